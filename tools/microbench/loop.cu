// Isolated record-loop benchmark: the consumer inner loop of layer.cu with
// records and feature rows resident in shared memory (no producer, no HBM).
// Measures the FFMA2 issue rate the loop itself can reach per warp count.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ void fma2_acc(u64 &acc, u64 y, float w) {
  float2 a = *reinterpret_cast<float2 *>(&acc);
  const float2 yy = *reinterpret_cast<const float2 *>(&y);
  a = __ffma2_rn(yy, make_float2(w, w), a);
  acc = *reinterpret_cast<u64 *>(&a);
}

template <int UNROLL, int MODE>
__global__ void loop_kernel(float *out, int reps, int cnt, float wparam = 0.0625f) {
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t *recs = reinterpret_cast<uint32_t *>(smem);
  char *ybase = smem + 64 * 1024;
  // records: 38 per group, 16 groups: offsets spread over 143 rows
  for (int i = tid; i < 16 * 64 * 8; i += blockDim.x) {
    int r = i / 8, w = i % 8;
    recs[i] = w == 0 ? (((r * 37) % 143) * 512) | ((r % 5 == 0) ? 0x3fu : 0x7fu)
                     : __float_as_uint(0.0625f);
  }
  for (int i = tid; i < 143 * 128; i += blockDim.x) reinterpret_cast<float *>(ybase)[i] = (i % 7) * 0.25f;
  __syncthreads();
  u64 acc[14];
  for (int r = 0; r < 14; r++) acc[r] = 0;
  const uint32_t *g = recs + (warp % 16) * 64 * 8;
  const char *yb = ybase + 16 * lane;
  for (int rep = 0; rep < reps; rep++) {
    const uint32_t *rp = g, *end = g + cnt * 8;
#pragma unroll UNROLL
    for (; rp < end; rp += 8) {
      uint4 a, b;
      if (MODE == 6 || MODE == 7) {  // one record word: offset | mask
        const uint32_t r0 = *rp;
        a = make_uint4(r0 & 0xffff00u, r0 & 0x7fu, 0, 0);
        b = make_uint4(0, 0, 0, 0);
      } else if (MODE == 2 || MODE == 4) {  // weights from registers (no record loads)
        a = make_uint4((uint32_t)(rp - g) * 64u % (143u * 512u), __float_as_uint(0.0625f),
                       __float_as_uint(0.0625f), __float_as_uint(0.0625f));
        b = make_uint4(__float_as_uint(0.0625f), __float_as_uint(0.0625f),
                       __float_as_uint(0.0625f), __float_as_uint(0.0625f));
      } else {
        a = *reinterpret_cast<const uint4 *>(rp);
        b = *reinterpret_cast<const uint4 *>(rp + 4);
      }
      float w[7] = {__uint_as_float(a.y), __uint_as_float(a.z), __uint_as_float(a.w),
                    __uint_as_float(b.x), __uint_as_float(b.y), __uint_as_float(b.z),
                    __uint_as_float(b.w)};
      ulonglong2 y;
      if (MODE == 0 || MODE == 2 || MODE == 5 || MODE == 6 || MODE == 7)
        y = *reinterpret_cast<const ulonglong2 *>(yb + (a.x & ~0xffu));
      else if (MODE == 1) y = *reinterpret_cast<const ulonglong2 *>(yb);  // fixed row
      else y = make_ulonglong2((u64)a.x * 3u + lane, (u64)a.x + rep);  // MODE 3/4: no y load
      if (MODE == 6 || MODE == 7) {  // mask bits + one weight from the constant bank
        const uint32_t mask = MODE == 6 ? (a.y & 0x7fu) : 0x7fu;
#pragma unroll
        for (int k = 0; k < 7; k++) {
          if (mask & (1u << k)) {
            fma2_acc(acc[2 * k], y.x, wparam);
            fma2_acc(acc[2 * k + 1], y.y, wparam);
          }
        }
      } else if (MODE == 5) {  // h-major order: 7 FFMA2 reusing y.x, then 7 reusing y.y
#pragma unroll
        for (int k = 0; k < 7; k++) fma2_acc(acc[2 * k], y.x, w[k]);
#pragma unroll
        for (int k = 0; k < 7; k++) fma2_acc(acc[2 * k + 1], y.y, w[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 7; k++) {
          fma2_acc(acc[2 * k], y.x, w[k]);
          fma2_acc(acc[2 * k + 1], y.y, w[k]);
        }
      }
    }
  }
  float s = 0;
  for (int r = 0; r < 14; r++) {
    float2 v = *reinterpret_cast<float2 *>(&acc[r]);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + tid] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  cudaMalloc(&out, 148 * 1024 * 4 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = 64 * 1024 + 143 * 512;
  auto run = [&](auto kern, const char *name, int warps, int ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 200, cnt = 38;
    kern<<<sms * ctas, warps * 32, smem>>>(out, 2, cnt, 0.0625f);
    cudaEventRecord(e0);
    kern<<<sms * ctas, warps * 32, smem>>>(out, reps, cnt, 0.0625f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ffma2 = (double)sms * ctas * warps * reps * cnt * 14;
    double per_smsp_clk = ffma2 / (ms * 1e-3) / (sms * 4) / 1.965e9;
    printf("{\"loop\":\"%s\",\"warps\":%d,\"ctas_per_sm\":%d,\"ffma2_per_smsp_clk\":%.3f,\"frac_of_0.5\":%.3f}\n",
           name, warps, ctas, per_smsp_clk, per_smsp_clk / 0.5);
  };
  run(loop_kernel<4, 0>, "unroll4", 16, 1);
  run(loop_kernel<4, 0>, "unroll4", 8, 1);
  run(loop_kernel<4, 0>, "unroll4", 16, 2);
  run(loop_kernel<2, 0>, "unroll2", 16, 1);
  run(loop_kernel<8, 0>, "unroll8", 16, 1);
  run(loop_kernel<4, 1>, "unroll4_fixedrow", 16, 1);
  run(loop_kernel<4, 5>, "hmajor", 16, 1);
  run(loop_kernel<4, 5>, "hmajor", 16, 2);
  run(loop_kernel<4, 6>, "mask_const_w", 16, 1);
  run(loop_kernel<4, 7>, "fullmask_const_w", 16, 1);
  run(loop_kernel<4, 6>, "mask_const_w", 16, 2);
  run(loop_kernel<4, 2>, "no_weight_lds", 16, 1);
  run(loop_kernel<4, 3>, "no_y_lds", 16, 1);
  run(loop_kernel<4, 4>, "no_lds", 16, 1);
  if (cudaGetLastError() != cudaSuccess) printf("error\n");
  return 0;
}
