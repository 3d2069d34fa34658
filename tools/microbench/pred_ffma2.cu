// Does a predicated-off FFMA2 cost FMA-pipe time? 14 FFMA2 per step guarded
// by a runtime row mask (R2P), mask = all rows vs no rows vs 5 of 7, 20 warps
// per SM (the layer kernel's consumer count). Prints ns per step per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ void fma2(u64 &acc, u64 y, float w) {
  float2 a = *reinterpret_cast<float2 *>(&acc);
  const float2 yy = *reinterpret_cast<const float2 *>(&y);
  a = __ffma2_rn(yy, make_float2(w, w), a);
  acc = *reinterpret_cast<u64 *>(&a);
}
__global__ void k(const uint32_t *masks, int iters, float w, float *out) {
  u64 acc[14];
  for (int i = 0; i < 14; i++) acc[i] = 0;
  const uint32_t m0 = masks[0], m1 = masks[1], m2 = masks[2], m3 = masks[3];
  u64 y = ((u64)__float_as_uint(1.0f + threadIdx.x) << 32) | __float_as_uint(2.0f);
  for (int it = 0; it < iters; it++) {
    const uint32_t wd[4] = {m0 ^ (uint32_t)(it & 0), m1, m2, m3};
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int r = 0; r < 7; r++)
        if (wd[j] & (1u << r)) {
          fma2(acc[2 * r], y, w);
          fma2(acc[2 * r + 1], y, w);
        }
    y += 1;
  }
  float s = 0;
  for (int i = 0; i < 14; i++) { float2 a = *reinterpret_cast<float2 *>(&acc[i]); s += a.x + a.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  uint32_t *m; float *o;
  cudaMalloc(&m, 16); cudaMalloc(&o, 148 * 640 * 4);
  const int iters = 20000;
  for (uint32_t mask : {0x7fu, 0x0u, 0x1fu, 0x3u}) {
    uint32_t h[4] = {mask, mask, mask, mask};
    cudaMemcpy(m, h, 16, cudaMemcpyHostToDevice);
    k<<<148, 640>>>(m, 100, 0.5f, o);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<148, 640>>>(m, iters, 0.5f, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int on = __builtin_popcount(mask) * 2 * 4;
    printf("mask 0x%02x: %d FFMA2 on / 56 per step: %.3f ns per step per SM-warp-slot; "
           "on-FFMA2 rate %.1f /clk/SM @1.965GHz\n", mask, on, ms * 1e6 / iters,
           (double)on * 20 * iters / (ms * 1e-3) / 1.965e9 / 1.0);
  }
  return 0;
}
