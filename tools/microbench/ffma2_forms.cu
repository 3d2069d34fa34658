// FFMA2 operand forms on sm_100a: issue rate of the packed fp32 FMA with the
// multiplier in a register, a uniform register, or an immediate (the
// Graph-Challenge weight 1/16), and the scalar FFMA immediate form.
// Reports FMA lanes per clock per SM (148 SMs, 8 warps per SMSP, 16
// independent accumulator pairs per thread).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_forms ffma2_forms.cu
#include <cuda_runtime.h>
#include <cstdio>

typedef unsigned long long u64;

__device__ __forceinline__ float2 f2(u64 v) { return *reinterpret_cast<float2 *>(&v); }

template <int MODE>
__global__ void bench(float *out, float wreg, const float *wvec, int iters, long long *cycles) {
  float2 acc[16];
  float s[16];
#pragma unroll
  for (int i = 0; i < 16; i++) { acc[i] = make_float2(i * 1e-3f, threadIdx.x * 1e-3f); s[i] = i; }
  float2 y = make_float2(threadIdx.x * 1e-6f, 1e-6f);
  // MODE 0/3: a per-thread register (opaque to the compiler); 4/5: the kernel
  // parameter, which ptxas keeps in a uniform register
  const float w = wvec[threadIdx.x];  // a per-thread register (every entry is wreg)
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
      if (MODE == 0) acc[i] = __ffma2_rn(y, make_float2(w, w), acc[i]);        // register
      if (MODE == 1) acc[i] = __ffma2_rn(y, make_float2(0.0625f, 0.0625f), acc[i]);  // immediate
      if (MODE == 2) s[i] = __fmaf_rn(y.x, 0.0625f, s[i]);                       // FFMA imm
      if (MODE == 3) s[i] = __fmaf_rn(y.x, w, s[i]);                             // FFMA reg
      if (MODE == 4) acc[i] = __ffma2_rn(y, make_float2(wreg, wreg), acc[i]);   // uniform reg
      if (MODE == 5) s[i] = __fmaf_rn(y.x, wreg, s[i]);                          // FFMA uniform
    }
    // keep y live and varying so nothing is hoisted
    y.x += 1e-9f;
  }
  long long t1 = clock64();
  float r = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) r += acc[i].x + acc[i].y + s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char *name, int lanes_per_op) {
  const int blocks = 148, threads = 1024, iters = 4096;
  float *out, *wv;
  long long *cyc;
  cudaMalloc(&wv, threads * 4);
  float h[1024];
  for (int i = 0; i < threads; i++) h[i] = 0.0625f;
  cudaMemcpy(wv, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  bench<MODE><<<blocks, threads>>>(out, 0.0625f, wv, 16, cyc);
  cudaDeviceSynchronize();
  bench<MODE><<<blocks, threads>>>(out, 0.0625f, wv, iters, cyc);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; i++) mx = c[i] > mx ? c[i] : mx;
  // per SM: 32 warps x 32 threads x iters x 16 ops x lanes_per_op FMAs
  double fmas = 32.0 * 32 * iters * 16 * lanes_per_op;
  printf("%-28s %7.1f FMA/clk/SM\n", name, fmas / mx);
  cudaFree(out);
  cudaFree(cyc);
  cudaFree(wv);
}

int main() {
  run<0>("FFMA2 register weight", 2);
  run<1>("FFMA2 immediate weight", 2);
  run<2>("FFMA immediate weight", 1);
  run<3>("FFMA register weight", 1);
  run<4>("FFMA2 uniform-register weight", 2);
  run<5>("FFMA uniform-register weight", 1);
  return 0;
}
