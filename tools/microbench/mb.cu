// Microbenchmarks that decide the layer-kernel design: FP32 pipe rates
// (FFMA, FFMA2 with scalar-broadcast operand, FMUL2+FADD2), smem LDS rates.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){ u64 r; asm volatile("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;}
__device__ __forceinline__ float lo(u64 v){ float a,b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a+b;}

template<int ITER>
__global__ void ffma1(float* out, float w0, float w1){
  float a[16]; float x = threadIdx.x*1e-3f; float w[4]={w0,w1,w0*0.5f,w1*0.5f};
  #pragma unroll
  for(int i=0;i<16;i++) a[i]=i;
  for(int it=0; it<ITER; it++){
    #pragma unroll
    for(int i=0;i<16;i++) a[i]=__fmaf_rn(x, w[i&3], a[i]);
    x = a[it&15]*1e-9f + x;
  }
  float s=0; for(int i=0;i<16;i++) s+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int ITER>
__global__ void ffma2(float* out, float w0, float w1){
  u64 a[16]; u64 x = pk(threadIdx.x*1e-3f, 1.f); float w[4]={w0,w1,w0*0.5f,w1*0.5f};
  #pragma unroll
  for(int i=0;i<16;i++) a[i]=pk(i,i);
  for(int it=0; it<ITER; it++){
    #pragma unroll
    for(int i=0;i<16;i++){ asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[i]) : "l"(x), "l"(pk(w[i&3],w[i&3]))); }
    asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(a[it&15]));
  }
  float s=0; for(int i=0;i<16;i++) s+=lo(a[i]); out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int ITER>
__global__ void mul2add2(float* out, float w0, float w1){
  u64 a[16]; u64 x = pk(threadIdx.x*1e-3f, 1.f); float w[4]={w0,w1,w0*0.5f,w1*0.5f};
  #pragma unroll
  for(int i=0;i<16;i++) a[i]=pk(i,i);
  for(int it=0; it<ITER; it++){
    #pragma unroll
    for(int i=0;i<16;i++){ u64 p; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(x), "l"(pk(w[i&3],w[i&3])));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(p)); }
    asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(a[it&15]));
  }
  float s=0; for(int i=0;i<16;i++) s+=lo(a[i]); out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int ITER>
__global__ void mul1add1(float* out, float w0, float w1){
  float a[16]; float x = threadIdx.x*1e-3f; float w[4]={w0,w1,w0*0.5f,w1*0.5f};
  #pragma unroll
  for(int i=0;i<16;i++) a[i]=i;
  for(int it=0; it<ITER; it++){
    #pragma unroll
    for(int i=0;i<16;i++) a[i]=__fadd_rn(a[i], __fmul_rn(x, w[i&3]));
    x = a[it&15]*1e-9f + x;
  }
  float s=0; for(int i=0;i<16;i++) s+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// FFMA2 where the packed operand is a pair-add of smem-broadcast weights
template<int ITER>
__global__ void lds64(float* out){
  __shared__ float2 s[64*32];
  for(int i=threadIdx.x;i<64*32;i+=blockDim.x) s[i]=make_float2(i,i+1);
  __syncthreads();
  float acc=0; int lane=threadIdx.x&31; int idx=(threadIdx.x>>5)&63;
  for(int it=0; it<ITER; it++){
    #pragma unroll
    for(int i=0;i<16;i++){ float2 v=s[((idx+i)&63)*32+lane]; acc+=v.x*v.y; }
    idx += (int)acc & 1;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
template<int ITER>
__global__ void ldsbc128(float* out){
  __shared__ float4 s[256];
  for(int i=threadIdx.x;i<256;i+=blockDim.x) s[i]=make_float4(i,i+1,i+2,i+3);
  __syncthreads();
  float acc=0; int idx=(threadIdx.x>>5)&63;
  for(int it=0; it<ITER; it++){
    #pragma unroll
    for(int i=0;i<16;i++){ float4 v=s[(idx+i)&255]; acc+=v.x*v.y+v.z*v.w; }
    idx += (int)acc & 1;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
__global__ void copyk(const float4* __restrict__ a, float4* __restrict__ b, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int smemoptin; cudaDeviceGetAttribute(&smemoptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("{\"sms\":%d,\"clock_khz\":%d,\"l2_bytes\":%d,\"smem_optin\":%d}\n", sms, clk, l2, smemoptin);
  float* out; CK(cudaMalloc(&out, 148*64*1024*sizeof(float)));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int IT=4096; int blocks=sms*4, threads=512; float ms;
  auto run=[&](const char* name, auto kern, double ops_per_thread_iter){
    for(int rep=0;rep<2;rep++){ cudaEventRecord(e0); kern(); cudaEventRecord(e1); cudaEventSynchronize(e1);}
    cudaEventElapsedTime(&ms,e0,e1);
    double ops = (double)blocks*threads*IT*ops_per_thread_iter;
    printf("{\"bench\":\"%s\",\"ms\":%.4f,\"Gops\":%.1f,\"ops_per_clk_per_sm_at_clk\":%.2f}\n", name, ms, ops/ms/1e6, ops/(ms*1e-3)/sms/(clk*1e3));
  };
  run("ffma_scalar(fma/s)", [&]{ffma1<IT><<<blocks,threads>>>(out,0.5f,0.25f);}, 16);
  run("ffma2(fma/s, 2 per instr)", [&]{ffma2<IT><<<blocks,threads>>>(out,0.5f,0.25f);}, 32);
  run("fmul2+fadd2(edge/s)", [&]{mul2add2<IT><<<blocks,threads>>>(out,0.5f,0.25f);}, 32);
  run("fmul+fadd scalar(edge/s)", [&]{mul1add1<IT><<<blocks,threads>>>(out,0.5f,0.25f);}, 16);
  run("lds64 conflict-free(loads/s)", [&]{lds64<IT><<<blocks,threads>>>(out);}, 16);
  run("lds128 broadcast(loads/s)", [&]{ldsbc128<IT><<<blocks,threads>>>(out);}, 16);
  size_t n = (size_t)1<<28; float4 *a,*b; CK(cudaMalloc(&a,n*16)); CK(cudaMalloc(&b,n*16)); cudaMemset(a,0,n*16);
  for(int rep=0;rep<3;rep++){ cudaEventRecord(e0); copyk<<<sms*8,512>>>(a,b,n); cudaEventRecord(e1); cudaEventSynchronize(e1);}
  cudaEventElapsedTime(&ms,e0,e1); printf("{\"bench\":\"copy\",\"GBps\":%.1f}\n", 2.0*n*16/ms/1e6);
  CK(cudaGetLastError());
  return 0;
}
