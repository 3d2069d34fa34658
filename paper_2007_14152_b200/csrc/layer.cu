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
// One persistent CTA per resident slot pulls items from a per-layer atomic
// counter. Per item:
//   1. stage the block footprint: for each input neuron c of the stage, the 64
//      features' values y_in[c][a_in[64t + f]] -> smem (cp.async, coalesced
//      128-byte rows because y_in is neuron-major and a_in is mostly
//      contiguous); and the stage's union records (cp.async, 16 B chunks);
//   2. each warp owns one row group (R rows) at a time; lane l holds features
//      (64t + l, 64t + l + 32) as one f32x2 pair. For every record (one input
//      neuron of the group union, ascending neuron index): one LDS.64 of the
//      pair, then per row k: p = y * w_k (mul.rn.f32x2), acc_k += p
//      (add.rn.f32x2). w_k = +0 where row k does not connect: p = +0 and the
//      add is exact, so each row's sum equals the reference's ascending CSR
//      sum bit for bit (kernels.py:27-37: separate fp32 mul and add);
//   3. epilogue: v = acc + bias (one fp32 add), comparison clamp (NaN kept,
//      kernels.py:33-36), store y_out[row][64t + f], alive |= v > 0;
//   4. the CTA that finishes the last row block of tile t (atomic per-tile
//      counter) appends the tile's alive features to a_out / cat_out and
//      bumps the survivor count: pruning without a separate pass over Y.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "common.h"

namespace {

constexpr int kTile = 64;

typedef unsigned long long u64;

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(u64 v, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
// d = a * w + c per half (one rounding). Used two ways:
//  * scaled form:  acc = fma(p, m, acc) with p = fl(y*w) staged in smem and
//    m in {1, 0}: p*1 and p*0 are exact, so this is fl(acc + p) or acc;
//  * generic form: p = fma(y, w, -0) == fl(y*w) exactly (x + -0 == x for
//    every x, including -0), then acc = add(acc, p).
// The -0 addend arrives as a kernel argument: ptxas contracts a visible
// mul.rn.f32x2 + add.rn.f32x2 pair into FFMA2 (observed with CUDA 12.9,
// even with --fmad=false), which would skip the product's rounding.
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

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
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
  float negz;  // -0.0f, opaque to the compiler (see fma2)
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
template <int R, bool SCALED>
__device__ __forceinline__ void accumulate(u64 *acc, const uint32_t *recs, int cnt,
                                           const char *ysm, int lane, u64 negz2) {
  const char *ybase = ysm + lane * 8;
#pragma unroll 4
  for (int i = 0; i < cnt; i++) {
    uint32_t off;
    float w[R];
    Rec<R>::load(recs + i * Rec<R>::W, off, w);
    u64 y = *reinterpret_cast<const u64 *>(ybase + off);
    if (SCALED) {
#pragma unroll
      for (int k = 0; k < R; k++) acc[k] = fma2(y, w[k], acc[k]);
    } else {
#pragma unroll
      for (int k = 0; k < R; k++) acc[k] = add2(acc[k], fma2(y, w[k], negz2));
    }
  }
}

// Bias, clamp, store, activity for one finished group.
template <int R>
__device__ __forceinline__ void epilogue(const LayerArgs &A, const u64 *acc, int g, int t,
                                         int lane, bool v0, bool v1, uint32_t *s_alive) {
  bool al0 = false, al1 = false;
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
  }
  const unsigned m0 = __ballot_sync(0xffffffffu, al0 && v0);
  const unsigned m1 = __ballot_sync(0xffffffffu, al1 && v1);
  if (lane == 0) {
    if (m0) atomicOr(&s_alive[0], m0);
    if (m1) atomicOr(&s_alive[1], m1);
  }
}

template <int R, bool SCALED, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) layer_kernel(LayerArgs A) {
  extern __shared__ __align__(16) char smem[];
  __shared__ int s_item;
  __shared__ uint32_t s_alive[2];
  __shared__ int s_last;
  __shared__ int s_base;
  __shared__ u64 s_mask;

  constexpr int RW = Rec<R>::W;
  const int M = *A.m_in;
  if (M <= 0) return;
  const int nb = (int)A.L.num_blocks;
  const int tiles = (M + kTile - 1) / kTile;
  const int64_t items = (int64_t)tiles * nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  char *ysm = smem;
  uint32_t *rsm =
      reinterpret_cast<uint32_t *>(smem + (size_t)A.L.max_fp_per_stage * kTile * 4);
  const u64 negz2 = pack2(A.negz, A.negz);

  for (;;) {
    if (tid == 0) s_item = atomicAdd(A.work, 1);
    if (tid < 2) s_alive[tid] = 0u;
    __syncthreads();
    const int item = s_item;
    if (item >= items) break;
    const int t = item / nb;
    const int b = item - t * nb;
    const int j0 = t * kTile + lane, j1 = j0 + 32;
    const bool v0 = j0 < M, v1 = j1 < M;
    const int c0 = v0 ? __ldg(A.a_in + j0) : 0;
    const int c1 = v1 ? __ldg(A.a_in + j1) : 0;

    const int32_t *blk = A.L.blocks + (int64_t)b * 8;
    const int g_first = blk[0], ng = blk[1], s_first = blk[2], nst = blk[3];
    const int64_t seg0 = (int64_t)(uint32_t)blk[4] | ((int64_t)blk[5] << 32);

    auto stage_in = [&](int s) {
      const int64_t *st = A.L.stages + (int64_t)(s_first + s) * 4;
      const int64_t fp_off = st[0], rec_off = st[2];
      const int fp_cnt = (int)st[1], rec_cnt = (int)st[3];
      if (SCALED) {
        // stage p = fl(y * w_c): the product every connected row adds
        constexpr int U = 4;
        const int total = fp_cnt * 32;
        for (int i0 = tid; i0 < total; i0 += WARPS * 32 * U) {
          float x0[U], x1[U], wc[U];
#pragma unroll
          for (int u = 0; u < U; u++) {
            const int i = i0 + u * WARPS * 32;
            x0[u] = 0.0f;
            x1[u] = 0.0f;
            wc[u] = 0.0f;
            if (i < total) {
              const int slot = i >> 5;
              const int64_t c = __ldg(A.L.fp + fp_off + slot);
              wc[u] = __ldg(A.L.fpw + fp_off + slot);
              const float *src = A.y_in + c * A.ld;
              if (v0) x0[u] = __ldg(src + c0);
              if (v1) x1[u] = __ldg(src + c1);
            }
          }
#pragma unroll
          for (int u = 0; u < U; u++) {
            const int i = i0 + u * WARPS * 32;
            if (i < total) {
              float2 pr = make_float2(__fmul_rn(x0[u], wc[u]), __fmul_rn(x1[u], wc[u]));
              reinterpret_cast<float2 *>(ysm)[i] = pr;
            }
          }
        }
      } else {
        for (int i = tid; i < fp_cnt * 32; i += WARPS * 32) {
          const int slot = i >> 5;
          const int64_t c = __ldg(A.L.fp + fp_off + slot);
          const float *src = A.y_in + c * A.ld;
          float *dst = reinterpret_cast<float *>(ysm) + slot * kTile + 2 * lane;
          cp_async4(dst, src + c0, v0);
          cp_async4(dst + 1, src + c1, v1);
        }
      }
      const uint32_t *rg = A.L.records + rec_off * RW;
      if (RW >= 4) {
        const int chunks = rec_cnt * RW / 4;
        for (int i = tid; i < chunks; i += WARPS * 32) cp_async16(rsm + 4 * i, rg + 4 * i);
      } else {
        const int chunks = rec_cnt * RW / 2;
        for (int i = tid; i < chunks; i += WARPS * 32) cp_async8(rsm + 2 * i, rg + 2 * i);
      }
      cp_async_wait_all();
      __syncthreads();
    };

    if (nst == 1) {
      stage_in(0);
      for (int gl = warp; gl < ng; gl += WARPS) {
        const int32_t *sg = A.L.segs + (seg0 + gl) * 2;
        u64 acc[R];
#pragma unroll
        for (int k = 0; k < R; k++) acc[k] = 0ull;
        accumulate<R, SCALED>(acc, rsm + (int64_t)sg[0] * RW, sg[1], ysm, lane, negz2);
        epilogue<R>(A, acc, g_first + gl, t, lane, v0, v1, s_alive);
      }
    } else {
      // multi-stage blocks hold at most WARPS groups (plan.cpp): one per warp,
      // accumulators stay in registers across stages
      u64 acc[R];
#pragma unroll
      for (int k = 0; k < R; k++) acc[k] = 0ull;
      for (int s = 0; s < nst; s++) {
        if (s) __syncthreads();
        stage_in(s);
        if (warp < ng) {
          const int32_t *sg = A.L.segs + (seg0 + (int64_t)s * ng + warp) * 2;
          accumulate<R, SCALED>(acc, rsm + (int64_t)sg[0] * RW, sg[1], ysm, lane, negz2);
        }
      }
      if (warp < ng) epilogue<R>(A, acc, g_first + warp, t, lane, v0, v1, s_alive);
    }
    __syncthreads();

    // ---- tile bookkeeping: last finisher of tile t appends its survivors
    if (tid == 0) {
      const uint32_t lo = s_alive[0], hi = s_alive[1];
      if (lo) atomicOr(&A.tile_alive[2 * t], lo);
      if (hi) atomicOr(&A.tile_alive[2 * t + 1], hi);
      __threadfence();
      const int done = atomicAdd(&A.tile_done[t], 1);
      int last = 0;
      if (done == nb - 1) {
        __threadfence();
        const uint32_t alo = atomicOr(&A.tile_alive[2 * t], 0u);
        const uint32_t ahi = atomicOr(&A.tile_alive[2 * t + 1], 0u);
        const u64 mask = (u64)alo | ((u64)ahi << 32);
        const int k = __popcll(mask);
        s_base = k ? atomicAdd(A.m_out, k) : 0;
        s_mask = mask;
        A.tile_done[t] = 0;
        A.tile_alive[2 * t] = 0u;
        A.tile_alive[2 * t + 1] = 0u;
        last = 1;
      }
      s_last = last;
    }
    __syncthreads();
    if (s_last && tid < kTile) {
      const u64 mask = s_mask;
      if ((mask >> tid) & 1ull) {
        const int rank = __popcll(mask & ((1ull << tid) - 1ull));
        const int j = t * kTile + tid;
        A.a_out[s_base + rank] = j;
        A.cat_out[s_base + rank] = A.cat_in[j];
      }
    }
    // the __syncthreads at the top of the loop protects s_* and smem reuse
  }
}

// ---- launch configuration ---------------------------------------------------

constexpr int kWarps = 16;

template <int R>
void *kernel_ptr(bool scaled) {
  return scaled ? reinterpret_cast<void *>(&layer_kernel<R, true, kWarps>)
                : reinterpret_cast<void *>(&layer_kernel<R, false, kWarps>);
}

size_t smem_bytes(const spdnn_layer_dev &L) {
  return (size_t)L.max_fp_per_stage * kTile * 4 +
         (size_t)L.max_records_per_stage * L.record_words * 4;
}

struct OccCache {
  std::mutex mu;
  int device = -1, sms = 0;
  size_t optin = 0;
};
OccCache g_occ;

int device_info(int &sms, size_t &optin) {
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lk(g_occ.mu);
  if (g_occ.device != dev) {
    int s = 0, o = 0;
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    g_occ.device = dev;
    g_occ.sms = s;
    g_occ.optin = (size_t)o;
  }
  sms = g_occ.sms;
  optin = g_occ.optin;
  return 0;
}

int launch_layer(const LayerArgs &A, cudaStream_t stream) {
  const spdnn_layer_dev &L = A.L;
  int R = L.rows_per_group;
  const bool sc = L.scaled != 0;
  void *fn = R == 1 ? kernel_ptr<1>(sc) : (R == 3 ? kernel_ptr<3>(sc) : (R == 7 ? kernel_ptr<7>(sc) : nullptr));
  if (!fn) return spdnn_fail(SPDNN_EINVAL, "layer: rows_per_group must be 1, 3 or 7");
  int sms;
  size_t optin;
  if (device_info(sms, optin)) return spdnn_fail(SPDNN_ECUDA, "layer: no CUDA device");
  size_t smem = smem_bytes(L);
  if (smem + 1024 > optin) return spdnn_fail(SPDNN_ERANGE, "layer: staged tile exceeds shared memory");
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWarps * 32, smem);
  if (e != cudaSuccess || per_sm < 1) return spdnn_fail(SPDNN_ECUDA, "layer: kernel does not fit on an SM");
  void *args[] = {const_cast<LayerArgs *>(&A)};
  e = cudaLaunchKernel(fn, dim3(sms * per_sm), dim3(kWarps * 32), args, smem, stream);
  if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  return SPDNN_OK;
}

// ---- layout conversion kernels ---------------------------------------------

// x: [m][n] feature-major -> y: [n][ld]; 32x32 tiles through smem.
__global__ void transpose_in_kernel(const float *__restrict__ x, int64_t n, int64_t m,
                                    float *__restrict__ y, int64_t ld) {
  __shared__ float tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t j = j0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (j < m && c < n) ? x[j * n + c] : 0.0f;
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

}  // namespace

extern "C" int spdnn_layer_forward(const spdnn_layer_dev *layer, const float *bias,
                                   const float *y_in, float *y_out, int64_t ld,
                                   const int32_t *a_in, const int64_t *cat_in,
                                   const int32_t *m_in, int32_t *a_out, int64_t *cat_out,
                                   int32_t *m_out, const spdnn_scratch *scratch,
                                   int32_t *work, void *stream) {
  if (!layer || !bias || !y_in || !y_out || !a_in || !cat_in || !m_in || !a_out ||
      !cat_out || !m_out || !scratch || !work || ld < 1 || ld % kTile)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_layer_forward: bad argument");
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
  A.negz = -0.0f;
  if (A.L.num_blocks == 0) return SPDNN_OK;  // N == 0
  return launch_layer(A, (cudaStream_t)stream);
}

extern "C" int spdnn_infer_layers(int64_t num_layers, const spdnn_layer_dev *layers,
                                  const float *bias, float *y0, float *y1, int64_t ld,
                                  int32_t *a0, int32_t *a1, int64_t *cat0, int64_t *cat1,
                                  int32_t *counts, const spdnn_scratch *scratch,
                                  void *stream) {
  if (num_layers < 0 || (num_layers > 0 && !layers))
    return spdnn_fail(SPDNN_EINVAL, "spdnn_infer_layers: bad argument");
  float *y[2] = {y0, y1};
  int32_t *a[2] = {a0, a1};
  int64_t *cat[2] = {cat0, cat1};
  for (int64_t l = 0; l < num_layers; l++) {
    int i = (int)(l & 1), o = i ^ 1;
    int rc = spdnn_layer_forward(&layers[l], bias, y[i], y[o], ld, a[i], cat[i], counts + l,
                                 a[o], cat[o], counts + l + 1, scratch, scratch->work + l,
                                 stream);
    if (rc) return rc;
  }
  return SPDNN_OK;
}

extern "C" int spdnn_transpose_in(const float *x, int64_t n, int64_t m, float *y, int64_t ld,
                                  void *stream) {
  if (n == 0 || m == 0) return SPDNN_OK;
  if (!x || !y || ld < m) return spdnn_fail(SPDNN_EINVAL, "spdnn_transpose_in: bad argument");
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  transpose_in_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(x, n, m, y, ld);
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
  if (threads_per_cta) *threads_per_cta = kWarps * 32;
  if (ctas_per_sm) *ctas_per_sm = 0;
  return SPDNN_OK;
}
