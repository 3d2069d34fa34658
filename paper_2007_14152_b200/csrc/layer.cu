// layer.cu -- the fused sparse layer for sm_100a:
//     Y_out = min(ReLU(W . Y_in + b), 32)   over the active features,
// fused with the activity test and the compaction of dead features.
//
// Replaces (paths under /root/reference/pkg/src/spdnn/):
//   kernels.staged_fused_relu   kernels.py:40-88   (gather-accumulate, bias, clamp)
//   engine.optimized_layer      engine.py:109-127  ((out > 0).any(axis=0))
//   engine.compact_active       engine.py:130-142  (keep alive features)
//   engine.infer layer loop     engine.py:264-285
//
// Work item = (row block b of the layer plan, tile t of 64 active features).
// Persistent CTAs pull items from a per-layer atomic counter and run a
// two-deep pipeline: while item k is computed out of smem buffer k&1, the
// cp.async copies of item k+1 (its staged input neurons and its union
// records) land in buffer (k+1)&1.
//
// Per item:
//   1. staging (cp.async): for every input neuron c of the block footprint,
//      the 64 features' values y_in[c][a_in[64t + f]] -> one 256-byte smem
//      row (y_in is neuron-major and a_in mostly contiguous, so the global
//      reads are 128-byte coalesced segments); plus the block's records;
//   2. each warp takes one row group (R rows) at a time; lane l holds
//      features (64t + l, 64t + l + 32) as one f32x2 register pair. Per union
//      record (one input neuron, ascending neuron index) one LDS.64 fetches
//      the pair and each row k accumulates it with weight w_k (0 where row k
//      does not connect). Every row therefore adds its own products in
//      ascending column order, interleaved with exact +0 terms: bit-equal to
//      the reference's CSR sum (kernels.py:27-37, separate mul and add).
//        FMA form  (all weights +-2^e): acc = fma(y, w, acc). The product is
//                  exact, so fma == fl(acc + fl(y*w)). A value small enough
//                  for y*w to underflow trips a guard flag and the engine
//                  reruns with the exact form (never seen on real data).
//        exact form (any weights): p = fma(y, w, -0) == fl(y*w), acc += p;
//   3. epilogue: v = fl(acc + bias), comparison clamp (NaN kept,
//      kernels.py:33-36), store y_out[row][64t + f], alive |= v > 0;
//   4. the CTA finishing the last row block of tile t appends the tile's
//      alive features to a_out / cat_out (pruning without a pass over Y).
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "common.h"

namespace {

constexpr int kTile = 64;
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;

typedef unsigned long long u64;

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(u64 v, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
// d = a * w + c per half, one rounding (FFMA2 with a broadcast scalar).
__device__ __forceinline__ u64 fma2(u64 a, float w, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(pack2(w, w)), "l"(c));
  return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ float clamp32(float v) {
  // comparison clamp in the reference's order; NaN falls through unchanged
  v = (v < 0.0f) ? 0.0f : v;
  v = (v > 32.0f) ? 32.0f : v;
  return v;
}

__device__ __forceinline__ void cp_async4(uint32_t saddr, const void *gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async8(uint32_t saddr, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

struct LayerArgs {
  spdnn_layer_dev L;
  const float *bias;
  const float *y_in;
  float *y_out;
  int64_t ld;
  const int32_t *a_in;
  const int64_t *cat_in;
  const int32_t *m_in;
  int32_t *a_out;
  int64_t *cat_out;
  int32_t *m_out;
  int32_t *tile_done;
  uint32_t *tile_alive;
  int32_t *work;
  uint32_t *guard;     // bit 0: an output in (0, tiny) was produced
  float tiny;          // FMA form is exact for next-layer inputs >= tiny
  float negz;          // -0.0f, opaque to the compiler (exact form)
  uint32_t buf_bytes;  // bytes of one pipeline buffer (ysm + rsm)
  uint32_t ysm_bytes;
};

template <int R>
struct Rec;
template <>
struct Rec<1> {
  static constexpr int W = 2;
  __device__ __forceinline__ static void load(const uint32_t *p, uint32_t &off, float *w) {
    uint2 a = *reinterpret_cast<const uint2 *>(p);
    off = a.x;
    w[0] = __uint_as_float(a.y);
  }
};
template <>
struct Rec<3> {
  static constexpr int W = 4;
  __device__ __forceinline__ static void load(const uint32_t *p, uint32_t &off, float *w) {
    uint4 a = *reinterpret_cast<const uint4 *>(p);
    off = a.x;
    w[0] = __uint_as_float(a.y);
    w[1] = __uint_as_float(a.z);
    w[2] = __uint_as_float(a.w);
  }
};
template <>
struct Rec<7> {
  static constexpr int W = 8;
  __device__ __forceinline__ static void load(const uint32_t *p, uint32_t &off, float *w) {
    uint4 a = *reinterpret_cast<const uint4 *>(p);
    uint4 b = *reinterpret_cast<const uint4 *>(p + 4);
    off = a.x;
    w[0] = __uint_as_float(a.y);
    w[1] = __uint_as_float(a.z);
    w[2] = __uint_as_float(a.w);
    w[3] = __uint_as_float(b.x);
    w[4] = __uint_as_float(b.y);
    w[5] = __uint_as_float(b.z);
    w[6] = __uint_as_float(b.w);
  }
};

// Accumulate one segment of union records into acc[0..R).
template <int R, bool FMA>
__device__ __forceinline__ void accumulate(u64 *acc, const uint32_t *recs, int cnt,
                                           const char *ysm, int lane, u64 negz2) {
  const char *ybase = ysm + lane * 8;
#pragma unroll 2
  for (int i = 0; i < cnt; i++) {
    uint32_t off;
    float w[R];
    Rec<R>::load(recs + i * Rec<R>::W, off, w);
    const u64 y = *reinterpret_cast<const u64 *>(ybase + off);
#pragma unroll
    for (int k = 0; k < R; k++) {
      if (FMA) acc[k] = fma2(y, w[k], acc[k]);
      else acc[k] = add2(acc[k], fma2(y, w[k], negz2));
    }
  }
}

// Bias, clamp, store, activity (+ FMA-form guard) for one finished group.
template <int R, bool FMA>
__device__ __forceinline__ void epilogue(const LayerArgs &A, const u64 *acc, int g, int t,
                                         int lane, bool v0, bool v1, uint32_t *s_alive) {
  bool al0 = false, al1 = false, tiny = false;
  const int j0 = t * kTile + lane;
#pragma unroll
  for (int k = 0; k < R; k++) {
    const int row = __ldg(A.L.rows + (int64_t)g * R + k);
    if (row < 0) continue;
    const float b = __ldg(A.bias + row);
    float x0, x1;
    unpack2(acc[k], x0, x1);
    x0 = clamp32(__fadd_rn(x0, b));
    x1 = clamp32(__fadd_rn(x1, b));
    float *dst = A.y_out + (int64_t)row * A.ld + j0;
    if (v0) dst[0] = x0;
    if (v1) dst[32] = x1;
    al0 |= (x0 > 0.0f);
    al1 |= (x1 > 0.0f);
    if (FMA) tiny |= (v0 && x0 > 0.0f && x0 < A.tiny) || (v1 && x1 > 0.0f && x1 < A.tiny);
  }
  const unsigned m0 = __ballot_sync(0xffffffffu, al0 && v0);
  const unsigned m1 = __ballot_sync(0xffffffffu, al1 && v1);
  if (lane == 0) {
    if (m0) atomicOr(&s_alive[0], m0);
    if (m1) atomicOr(&s_alive[1], m1);
  }
  if (FMA && tiny) atomicOr(A.guard, 1u);
}

struct Item {
  int t, b, ng, g_first, s_first, nst;
  int64_t seg0;
};

__device__ __forceinline__ Item decode(const LayerArgs &A, int item, int nb) {
  Item it;
  it.t = item / nb;
  it.b = item - it.t * nb;
  const int4 q = __ldg(reinterpret_cast<const int4 *>(A.L.blocks + (int64_t)it.b * 8));
  const int2 s = __ldg(reinterpret_cast<const int2 *>(A.L.blocks + (int64_t)it.b * 8 + 4));
  it.g_first = q.x;
  it.ng = q.y;
  it.s_first = q.z;
  it.nst = q.w;
  it.seg0 = (int64_t)(uint32_t)s.x | ((int64_t)s.y << 32);
  return it;
}

// Issue the cp.async copies of one stage of an item into buffer `sbuf`
// (shared-window address). Threads own fixed lanes (tid % 32).
template <int RW>
__device__ __forceinline__ void issue_stage(const LayerArgs &A, const Item &it, int s,
                                            uint32_t sbuf, int tid, int M) {
  const int lane = tid & 31;
  const int j0 = it.t * kTile + lane, j1 = j0 + 32;
  const bool v0 = j0 < M, v1 = j1 < M;
  const int c0 = v0 ? __ldg(A.a_in + j0) : 0;
  const int c1 = v1 ? __ldg(A.a_in + j1) : 0;
  const int64_t *st = A.L.stages + (int64_t)(it.s_first + s) * 4;
  const int64_t fp_off = __ldg(st + 0), rec_off = __ldg(st + 2);
  const int fp_cnt = (int)__ldg(st + 1), rec_cnt = (int)__ldg(st + 3);
  const uint32_t ydst = sbuf + lane * 8;
  for (int slot = tid >> 5; slot < fp_cnt; slot += kWarps) {
    const int64_t c = __ldg(A.L.fp + fp_off + slot);
    const float *src = A.y_in + c * A.ld;
    cp_async4(ydst + slot * 256, src + c0, v0);
    cp_async4(ydst + slot * 256 + 4, src + c1, v1);
  }
  const uint32_t rdst = sbuf + A.ysm_bytes;
  const uint32_t *rg = A.L.records + rec_off * RW;
  if (RW >= 4) {
    const int chunks = rec_cnt * RW / 4;
    for (int i = tid; i < chunks; i += kThreads) cp_async16(rdst + 16 * i, rg + 4 * i);
  } else {
    const int chunks = rec_cnt * RW / 2;
    for (int i = tid; i < chunks; i += kThreads) cp_async8(rdst + 8 * i, rg + 2 * i);
  }
}

template <int R, bool FMA>
__global__ void __launch_bounds__(kThreads) layer_kernel(LayerArgs A) {
  extern __shared__ __align__(16) char smem[];
  __shared__ int s_next;
  __shared__ uint32_t s_alive[2][2];

  constexpr int RW = Rec<R>::W;
  const int M = *A.m_in;
  if (M <= 0) return;
  const int nb = (int)A.L.num_blocks;
  const int tiles = (M + kTile - 1) / kTile;
  const int items = tiles * nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const u64 negz2 = pack2(A.negz, A.negz);

  if (tid == 0) s_next = atomicAdd(A.work, 1);
  if (tid < 4) s_alive[tid >> 1][tid & 1] = 0u;
  __syncthreads();
  int item = s_next;
  if (item < items) issue_stage<RW>(A, decode(A, item, nb), 0, sbase, tid, M);
  cp_async_commit();

  for (int k = 0; item < items; k++) {
    const int buf = k & 1;
    if (tid == 0) s_next = atomicAdd(A.work, 1);
    __syncthreads();  // B1: previous compute on buffer buf^1 is done; s_next visible
    const int next = s_next;
    if (next < items)
      issue_stage<RW>(A, decode(A, next, nb), 0, sbase + (buf ^ 1) * A.buf_bytes, tid, M);
    cp_async_commit();
    cp_async_wait<1>();  // this item's copies (all but the newest group) landed
    __syncthreads();     // B2: ... for every thread

    const Item it = decode(A, item, nb);
    const int j0 = it.t * kTile + lane;
    const bool v0 = j0 < M, v1 = j0 + 32 < M;
    char *ysm = smem + buf * A.buf_bytes;
    const uint32_t *rsm = reinterpret_cast<const uint32_t *>(ysm + A.ysm_bytes);
    uint32_t *alive = s_alive[buf];
    if (it.nst == 1) {
      for (int gl = warp; gl < it.ng; gl += kWarps) {
        const int2 sg = __ldg(reinterpret_cast<const int2 *>(A.L.segs) + it.seg0 + gl);
        u64 acc[R];
#pragma unroll
        for (int r = 0; r < R; r++) acc[r] = 0ull;
        accumulate<R, FMA>(acc, rsm + (int64_t)sg.x * RW, sg.y, ysm, lane, negz2);
        epilogue<R, FMA>(A, acc, it.g_first + gl, it.t, lane, v0, v1, alive);
      }
    } else {
      // multi-stage block (plan.cpp: at most kWarps groups, in practice one):
      // accumulators stay in registers while later stages reload this buffer
      u64 acc[R];
#pragma unroll
      for (int r = 0; r < R; r++) acc[r] = 0ull;
      for (int s = 0; s < it.nst; s++) {
        if (s) {
          __syncthreads();
          issue_stage<RW>(A, it, s, sbase + buf * A.buf_bytes, tid, M);
          cp_async_commit();
          cp_async_wait<0>();
          __syncthreads();
        }
        if (warp < it.ng) {
          const int2 sg =
              __ldg(reinterpret_cast<const int2 *>(A.L.segs) + it.seg0 + (int64_t)s * it.ng + warp);
          accumulate<R, FMA>(acc, rsm + (int64_t)sg.x * RW, sg.y, ysm, lane, negz2);
        }
      }
      if (warp < it.ng) epilogue<R, FMA>(A, acc, it.g_first + warp, it.t, lane, v0, v1, alive);
    }
    __syncthreads();  // B3: every warp's activity bits are in s_alive[buf]

    // tile bookkeeping by warp 0 alone; the other warps move on
    if (warp == 0) {
      int last = 0, base = 0;
      u64 mask = 0;
      if (lane == 0) {
        const uint32_t lo = alive[0], hi = alive[1];
        alive[0] = 0u;
        alive[1] = 0u;
        if (lo) atomicOr(&A.tile_alive[2 * it.t], lo);
        if (hi) atomicOr(&A.tile_alive[2 * it.t + 1], hi);
        __threadfence();
        const int done = atomicAdd(&A.tile_done[it.t], 1);
        if (done == nb - 1) {
          __threadfence();
          const uint32_t alo = atomicOr(&A.tile_alive[2 * it.t], 0u);
          const uint32_t ahi = atomicOr(&A.tile_alive[2 * it.t + 1], 0u);
          mask = (u64)alo | ((u64)ahi << 32);
          const int cnt = __popcll(mask);
          base = cnt ? atomicAdd(A.m_out, cnt) : 0;
          A.tile_done[it.t] = 0;
          A.tile_alive[2 * it.t] = 0u;
          A.tile_alive[2 * it.t + 1] = 0u;
          last = 1;
        }
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        base = __shfl_sync(0xffffffffu, base, 0);
        mask = __shfl_sync(0xffffffffu, mask, 0);
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int f = lane + 32 * h;
          if ((mask >> f) & 1ull) {
            const int rank = __popcll(mask & ((1ull << f) - 1ull));
            const int j = it.t * kTile + f;
            A.a_out[base + rank] = j;
            A.cat_out[base + rank] = A.cat_in[j];
          }
        }
      }
    }
    item = next;
  }
  cp_async_wait<0>();
}

// ---- launch configuration ---------------------------------------------------

template <int R>
void *kernel_ptr(bool fma) {
  return fma ? reinterpret_cast<void *>(&layer_kernel<R, true>)
             : reinterpret_cast<void *>(&layer_kernel<R, false>);
}

struct DevInfo {
  std::mutex mu;
  int device = -1, sms = 0;
  size_t optin = 0;
};
DevInfo g_dev;

int device_info(int &sms, size_t &optin) {
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lk(g_dev.mu);
  if (g_dev.device != dev) {
    int s = 0, o = 0;
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    g_dev.device = dev;
    g_dev.sms = s;
    g_dev.optin = (size_t)o;
  }
  sms = g_dev.sms;
  optin = g_dev.optin;
  return 0;
}

int launch_layer(LayerArgs &A, bool fma, cudaStream_t stream) {
  const spdnn_layer_dev &L = A.L;
  const int R = L.rows_per_group;
  void *fn = R == 1 ? kernel_ptr<1>(fma)
                    : (R == 3 ? kernel_ptr<3>(fma) : (R == 7 ? kernel_ptr<7>(fma) : nullptr));
  if (!fn) return spdnn_fail(SPDNN_EINVAL, "layer: rows_per_group must be 1, 3 or 7");
  int sms;
  size_t optin;
  if (device_info(sms, optin)) return spdnn_fail(SPDNN_ECUDA, "layer: no CUDA device");
  const size_t ysm = (size_t)L.max_fp_per_stage * kTile * 4;
  const size_t rsm = ((size_t)L.max_records_per_stage * L.record_words * 4 + 15) / 16 * 16;
  const size_t buf = (ysm + rsm + 127) / 128 * 128;
  const size_t smem = 2 * buf;
  if (smem + 1024 > optin) return spdnn_fail(SPDNN_ERANGE, "layer: staged tile exceeds shared memory");
  A.ysm_bytes = (uint32_t)ysm;
  A.buf_bytes = (uint32_t)buf;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem);
  if (e != cudaSuccess || per_sm < 1) return spdnn_fail(SPDNN_ECUDA, "layer: kernel does not fit on an SM");
  void *args[] = {&A};
  e = cudaLaunchKernel(fn, dim3(sms * per_sm), dim3(kThreads), args, smem, stream);
  if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  return SPDNN_OK;
}

// ---- layout conversion kernels ---------------------------------------------

// x: [m][n] feature-major -> y: [n][ld]; 32x32 tiles through smem. Flags the
// inputs the FMA form cannot take: bit 0 = 0 < |x| < tiny or |x| > huge,
// bit 1 = non-finite (NaN/inf would leak into non-connected rows through
// the zero-weight union slots; the engine then reruns one row per group).
__global__ void transpose_in_kernel(const float *__restrict__ x, int64_t n, int64_t m,
                                    float *__restrict__ y, int64_t ld, uint32_t *guard,
                                    float tiny, float huge) {
  __shared__ float tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  uint32_t flag = 0;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t j = j0 + i, c = c0 + threadIdx.x;
    float v = (j < m && c < n) ? x[j * n + c] : 0.0f;
    const float a = fabsf(v);
    if (!(a <= 3.0e38f)) flag |= 2u;  // NaN or inf
    else if ((a > 0.0f && a < tiny) || a > huge) flag |= 1u;
    tile[i][threadIdx.x] = v;
  }
  if (guard && __any_sync(0xffffffffu, flag != 0)) {
    const unsigned f = __reduce_or_sync(0xffffffffu, flag);
    if ((threadIdx.x & 31) == 0) atomicOr(guard, f);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, j = j0 + threadIdx.x;
    if (c < n && j < m) y[c * ld + j] = tile[threadIdx.x][i];
  }
}

// out[k][c] = y[c][a[perm[k]]]
__global__ void gather_out_kernel(const float *__restrict__ y, int64_t n, int64_t ld,
                                  const int32_t *__restrict__ a,
                                  const int64_t *__restrict__ perm, int64_t m,
                                  float *__restrict__ out) {
  __shared__ float tile[32][33];
  __shared__ int32_t col[32];
  const int64_t c0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  if (threadIdx.y == 0) {
    int64_t k = k0 + threadIdx.x;
    col[threadIdx.x] = k < m ? a[perm ? perm[k] : k] : 0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, k = k0 + threadIdx.x;
    tile[i][threadIdx.x] = (c < n && k < m) ? y[c * ld + col[threadIdx.x]] : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t k = k0 + i, c = c0 + threadIdx.x;
    if (k < m && c < n) out[k * n + c] = tile[threadIdx.x][i];
  }
}

int forward(const spdnn_layer_dev *layer, const float *bias, const float *y_in, float *y_out,
            int64_t ld, const int32_t *a_in, const int64_t *cat_in, const int32_t *m_in,
            int32_t *a_out, int64_t *cat_out, int32_t *m_out, const spdnn_scratch *scratch,
            int32_t *work, const spdnn_run_opts *opts, void *stream) {
  if (!layer || !bias || !y_in || !y_out || !a_in || !cat_in || !m_in || !a_out ||
      !cat_out || !m_out || !scratch || !work || ld < 1 || ld % kTile)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_layer_forward: bad argument");
  const bool fma = opts && opts->fma_form;
  if (fma && !scratch->guard)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_layer_forward: the FMA form needs scratch->guard");
  LayerArgs A;
  A.L = *layer;
  A.bias = bias;
  A.y_in = y_in;
  A.y_out = y_out;
  A.ld = ld;
  A.a_in = a_in;
  A.cat_in = cat_in;
  A.m_in = m_in;
  A.a_out = a_out;
  A.cat_out = cat_out;
  A.m_out = m_out;
  A.tile_done = scratch->tile_done;
  A.tile_alive = scratch->tile_alive;
  A.work = work;
  A.guard = scratch->guard;
  A.tiny = opts ? opts->tiny : 0.0f;
  A.negz = -0.0f;
  A.buf_bytes = 0;
  A.ysm_bytes = 0;
  if (A.L.num_blocks == 0) return SPDNN_OK;  // N == 0
  return launch_layer(A, fma, (cudaStream_t)stream);
}

}  // namespace

extern "C" int spdnn_layer_forward(const spdnn_layer_dev *layer, const float *bias,
                                   const float *y_in, float *y_out, int64_t ld,
                                   const int32_t *a_in, const int64_t *cat_in,
                                   const int32_t *m_in, int32_t *a_out, int64_t *cat_out,
                                   int32_t *m_out, const spdnn_scratch *scratch,
                                   int32_t *work, const spdnn_run_opts *opts, void *stream) {
  return forward(layer, bias, y_in, y_out, ld, a_in, cat_in, m_in, a_out, cat_out, m_out,
                 scratch, work, opts, stream);
}

extern "C" int spdnn_infer_layers(int64_t num_layers, const spdnn_layer_dev *layers,
                                  const float *bias, float *y0, float *y1, int64_t ld,
                                  int32_t *a0, int32_t *a1, int64_t *cat0, int64_t *cat1,
                                  int32_t *counts, const spdnn_scratch *scratch,
                                  const spdnn_run_opts *opts, void *stream) {
  if (num_layers < 0 || (num_layers > 0 && (!layers || !scratch)))
    return spdnn_fail(SPDNN_EINVAL, "spdnn_infer_layers: bad argument");
  float *y[2] = {y0, y1};
  int32_t *a[2] = {a0, a1};
  int64_t *cat[2] = {cat0, cat1};
  for (int64_t l = 0; l < num_layers; l++) {
    int i = (int)(l & 1), o = i ^ 1;
    int rc = forward(&layers[l], bias, y[i], y[o], ld, a[i], cat[i], counts + l, a[o], cat[o],
                     counts + l + 1, scratch, scratch->work + l, opts, stream);
    if (rc) return rc;
  }
  return SPDNN_OK;
}

extern "C" int spdnn_transpose_in(const float *x, int64_t n, int64_t m, float *y, int64_t ld,
                                  uint32_t *guard, float tiny, float huge, void *stream) {
  if (n == 0 || m == 0) return SPDNN_OK;
  if (!x || !y || ld < m) return spdnn_fail(SPDNN_EINVAL, "spdnn_transpose_in: bad argument");
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  transpose_in_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(x, n, m, y, ld, guard, tiny,
                                                                huge);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPDNN_OK : spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
}

extern "C" int spdnn_gather_out(const float *y, int64_t n, int64_t ld, const int32_t *a,
                                const int64_t *perm, int64_t m, float *out, void *stream) {
  if (n == 0 || m == 0) return SPDNN_OK;
  if (!y || !a || !out) return spdnn_fail(SPDNN_EINVAL, "spdnn_gather_out: bad argument");
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  gather_out_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(y, n, ld, a, perm, m, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPDNN_OK : spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
}

extern "C" int spdnn_layer_occupancy(int32_t rows_per_group, int32_t *ctas_per_sm,
                                     int32_t *threads_per_cta) {
  (void)rows_per_group;
  if (threads_per_cta) *threads_per_cta = kThreads;
  if (ctas_per_sm) *ctas_per_sm = 0;
  return SPDNN_OK;
}
