// The layer kernel's mask-record loop (accumulate_mask<7, FMA, 4> of
// csrc/layer.cu) in isolation: records and staged rows resident in shared
// memory, no producer, no epilogue. Reports the FFMA2 rate per SM
// sub-partition for 4..28 warps per SM, with realistic 38-record groups
// (26 full masks, 12 partial), all-full masks, and per-record variants, to
// tell how many warps must be in the loop to saturate the FP32 pipe
// (peak 0.5 FFMA2 / clk / SMSP).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o maskloop maskloop.cu
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
struct YV {
  u64 v[2];
  __device__ __forceinline__ void load_s(uint32_t a) {
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "r"(a));
  }
};
template <int R>
__device__ __forceinline__ void mask_record(u64 *acc, uint32_t wd, const YV &y, float w) {
#pragma unroll
  for (int k = 0; k < R; k++)
    if (wd & (2u << k)) {
      fma2_acc(acc[2 * k], y.v[0], w);
      fma2_acc(acc[2 * k + 1], y.v[1], w);
    }
}
template <int R, int UNROLL>
__device__ __forceinline__ void accumulate_mask(u64 *acc, const uint32_t *recs, int cnt,
                                                uint32_t ybase, float w) {
  const uint4 *rp = reinterpret_cast<const uint4 *>(recs);
  const uint4 *const end = rp + (cnt >> 2);
#pragma unroll UNROLL
  for (; rp < end; rp++) {
    const uint4 q = *rp;
    const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
    YV y[4];
#pragma unroll
    for (int j = 0; j < 4; j++) y[j].load_s(ybase + (wd[j] >> 15));
#pragma unroll
    for (int j = 0; j < 4; j++) mask_record<R>(acc, wd[j], y[j], w);
  }
}

// software-pipelined: the next quad's words one quad ahead, each record's
// staged row one record ahead of its FFMA2s
template <int R, int UNROLL>
__device__ __forceinline__ void accumulate_mask_pipe(u64 *acc, const uint32_t *recs, int cnt,
                                                     uint32_t ybase, float w) {
  const uint4 *rp = reinterpret_cast<const uint4 *>(recs);
  const int nq = cnt >> 2, rem = cnt & 3;
  if (cnt <= 0) return;
  uint4 q = rp[0];
  YV y0;
  y0.load_s(ybase + (q.x >> 15));
#pragma unroll UNROLL
  for (int i = 0; i < nq; i++) {
    const uint4 qn = (i + 1 < nq || rem) ? rp[i + 1] : make_uint4(0u, 0u, 0u, 0u);
    YV y1, y2, y3;
    y1.load_s(ybase + (q.y >> 15));
    mask_record<R>(acc, q.x, y0, w);
    y2.load_s(ybase + (q.z >> 15));
    mask_record<R>(acc, q.y, y1, w);
    y3.load_s(ybase + (q.w >> 15));
    mask_record<R>(acc, q.z, y2, w);
    y0.load_s(ybase + (qn.x >> 15));
    mask_record<R>(acc, q.w, y3, w);
    q = qn;
  }
  if (rem) {
    mask_record<R>(acc, q.x, y0, w);
    if (rem > 1) {
      y0.load_s(ybase + (q.y >> 15));
      mask_record<R>(acc, q.y, y0, w);
    }
    if (rem > 2) {
      y0.load_s(ybase + (q.z >> 15));
      mask_record<R>(acc, q.z, y0, w);
    }
  }
}

// MODE 1: every row unpredicated; 2: staged rows replaced by registers (no
// feature LDS); 3: neither record nor feature loads (pure FFMA2 stream)
template <int R, int MODE>
__device__ __forceinline__ void accumulate_mode(u64 *acc, const uint32_t *recs, int cnt,
                                                uint32_t ybase, float w) {
  const uint4 *rp = reinterpret_cast<const uint4 *>(recs);
  const uint4 *const end = rp + (cnt >> 2);
  u64 yr0 = ybase, yr1 = ybase + 1;
#pragma unroll 2
  for (; rp < end; rp++) {
    const uint4 q = MODE == 3 ? make_uint4(0xfeu, 0xfeu, 0xfeu, 0xfeu) : *rp;
    const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
    YV y[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (MODE >= 2) {
        y[j].v[0] = yr0 + j;
        y[j].v[1] = yr1 ^ wd[j];
      } else {
        y[j].load_s(ybase + (wd[j] >> 15));
      }
    }
#pragma unroll
    for (int j = 0; j < 4; j++) mask_record<R>(acc, MODE == 1 ? 0xfeu : wd[j], y[j], w);
    yr0 += 4;
  }
}

// MODE 4: full-mask records (bit 14 clear) run 14 unpredicated FFMA2;
// partial records (bit 14 set) carry a jump code in bits 8..11 (prefix
// rows 0..hi: code hi; suffix rows lo..6: code 5 + lo) and run exactly their
// rows through a fall-through switch
__device__ __forceinline__ void rowfma(u64 *acc, const YV &y, float w, int k) {
  fma2_acc(acc[2 * k], y.v[0], w);
  fma2_acc(acc[2 * k + 1], y.v[1], w);
}
__device__ __forceinline__ void run_record(u64 *acc, uint32_t wd, const YV &y, float w) {
  if (!(wd & 0x4000u)) {
#pragma unroll
    for (int k = 0; k < 7; k++) rowfma(acc, y, w, k);
    return;
  }
  switch ((wd >> 8) & 15u) {
    case 5: rowfma(acc, y, w, 5);  // fall through
    case 4: rowfma(acc, y, w, 4);
    case 3: rowfma(acc, y, w, 3);
    case 2: rowfma(acc, y, w, 2);
    case 1: rowfma(acc, y, w, 1);
    case 0: rowfma(acc, y, w, 0); break;
    case 6: rowfma(acc, y, w, 1);
    case 7: rowfma(acc, y, w, 2);
    case 8: rowfma(acc, y, w, 3);
    case 9: rowfma(acc, y, w, 4);
    case 10: rowfma(acc, y, w, 5);
    case 11: rowfma(acc, y, w, 6); break;
    default: break;
  }
}
template <int UNROLL>
__device__ __forceinline__ void accumulate_jump(u64 *acc, const uint32_t *recs, int cnt,
                                                uint32_t ybase, float w) {
  const uint4 *rp = reinterpret_cast<const uint4 *>(recs);
  const uint4 *const end = rp + (cnt >> 2);
#pragma unroll UNROLL
  for (; rp < end; rp++) {
    const uint4 q = *rp;
    const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
    YV y[4];
#pragma unroll
    for (int j = 0; j < 4; j++) y[j].load_s(ybase + (wd[j] >> 15));
#pragma unroll
    for (int j = 0; j < 4; j++) run_record(acc, wd[j], y[j], w);
  }
}

template <int UNROLL, bool PIPE = false, int MODE = 0>
__global__ void __launch_bounds__(1024, 1)
    loop_kernel(float *out, int reps, int cnt, const float *wp) {
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t *recs = reinterpret_cast<uint32_t *>(smem);
  const int nrec = 20 * 40;
  char *ybase = smem + nrec * 4;
  const uint32_t full = (uint32_t)__cvta_generic_to_shared(ybase);
  // 20 groups of 40 words (38 records + 2 padding), group g's records on
  // staged rows 7g .. 7g+37 (sliding windows), mask = rows covering the row
  // (prefix / suffix patterns), or all rows when cnt < 0 (full masks)
  const bool allfull = cnt < 0;
  if (cnt < 0) cnt = -cnt;
  for (int i = tid; i < nrec; i += blockDim.x) {
    const int g = i / 40, j = i % 40;
    uint32_t m = 0;
    for (int k = 0; k < 7; k++)
      if (allfull || (j >= k && j < k + 32)) m |= 2u << k;
    uint32_t code = 0;
    if (m != 0xfeu && m != 0u) {  // contiguous rows lo..hi: prefix (lo = 0) or suffix (hi = 6)
      int lo = 0, hi = 6;
      while (!(m & (2u << lo))) lo++;
      while (!(m & (2u << hi))) hi--;
      code = 0x4000u | ((lo == 0 ? (uint32_t)hi : 5u + (uint32_t)lo) << 8);
    }
    if (m == 0u) code = 0x4000u | (15u << 8);  // padding word: no rows
    recs[i] = j < 38 ? ((uint32_t)(7 * g + j) << 24 | m | code) : (0x4000u | (15u << 8));
  }
  for (int i = tid; i < 171 * 128; i += blockDim.x) reinterpret_cast<float *>(ybase)[i] = (i % 7) * 0.25f;
  __syncthreads();
  const float w = wp[0];
  u64 acc[14];
  for (int r = 0; r < 14; r++) acc[r] = 0;
  const uint32_t *g = recs + (warp % 20) * 40;
  const uint32_t yb = full + 16 * lane;
  for (int rep = 0; rep < reps; rep++) {
    if (MODE == 4) accumulate_jump<UNROLL>(acc, g, cnt, yb, w);
    else if (MODE) accumulate_mode<7, MODE>(acc, g, cnt, yb, w);
    else if (PIPE) accumulate_mask_pipe<7, UNROLL>(acc, g, cnt, yb, w);
    else accumulate_mask<7, UNROLL>(acc, g, cnt, yb, w);
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
  float *out, *wp;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&wp, 4);
  const float w = 0.0625f;
  cudaMemcpy(wp, &w, 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = 20 * 40 * 4 + 171 * 512;
  auto run = [&](auto kern, const char *name, int warps, int cnt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 400;
    kern<<<sms, warps * 32, smem>>>(out, 2, cnt, wp);
    cudaEventRecord(e0);
    kern<<<sms, warps * 32, smem>>>(out, reps, cnt, wp);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const int c = cnt < 0 ? -cnt : cnt;
    const int per_rec = cnt < 0 ? 14 : 14;  // executed (incl. predicated-off) FFMA2
    double ffma2 = (double)sms * warps * reps * (c / 4 * 4) * per_rec;
    double per_smsp_clk = ffma2 / (ms * 1e-3) / (sms * 4) / 1.965e9;
    printf("{\"loop\":\"%s\",\"warps\":%d,\"slots_ffma2_per_smsp_clk\":%.3f,\"frac_of_0.5\":%.3f}\n",
           name, warps, per_smsp_clk, per_smsp_clk / 0.5);
  };
  for (int warps : {4, 8, 12, 16, 20, 24, 28, 32}) run(loop_kernel<2>, "u2_sliding", warps, 40);
  for (int warps : {8, 12, 16, 20, 24}) run(loop_kernel<2, false, 4>, "mode4_jump(slots=14/record)", warps, 40);
  for (int warps : {8, 20}) run(loop_kernel<2, false, 1>, "mode1_unpredicated", warps, 40);
  for (int warps : {8, 20}) run(loop_kernel<2, false, 2>, "mode2_no_feature_lds", warps, 40);
  for (int warps : {8, 20}) run(loop_kernel<2, false, 3>, "mode3_no_lds", warps, 40);
  for (int warps : {4, 8, 12, 16, 20, 24}) run(loop_kernel<1, true>, "pipe_u1", warps, 40);
  for (int warps : {4, 8, 12, 16, 20, 24}) run(loop_kernel<2, true>, "pipe_u2", warps, 40);
  for (int warps : {4, 8, 12, 16, 20}) run(loop_kernel<2>, "u2_fullmask", warps, -40);
  for (int warps : {4, 8, 12, 16, 20}) run(loop_kernel<2, true>, "pipe_u2_fullmask", warps, -40);
  for (int warps : {4, 8, 12, 16, 20}) run(loop_kernel<1>, "u1_sliding", warps, 40);
  for (int warps : {4, 8, 12, 16, 20}) run(loop_kernel<4>, "u4_sliding", warps, 40);
  if (cudaGetLastError() != cudaSuccess) printf("error\n");
  return 0;
}
