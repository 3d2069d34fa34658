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
// Work item = (tile t of 128 active features, row block b of the layer plan);
// one item fills one entry of a ring of 2-4 shared-memory buffers. One
// persistent CTA per SM (launched with programmatic stream serialization, so
// a layer's static prologue runs under the previous layer's tail), warp
// roles:
//   * 3 producer warps: item metadata (block descriptor, the tile's feature
//     columns, the staged-row list) is prefetched with cp.async into a small
//     ring several items ahead; per entry one expect_tx, TMA bulk copies of
//     the block metadata and records, and TMA gather4 of the staged rows
//     (4 input neurons x 128 features per op) -- or 4-byte cp.async when the
//     tile's columns have gaps (the layer after deaths);
//   * 20 consumer warps (mask records; 16 for per-row weight records): one
//     unit = one row group of the entry. Lane l holds features 4l..4l+3 as
//     two f32x2 pairs; per record (one input neuron, ascending neuron index)
//     one LDS.128 of the four values and two FFMA2 per connected row. Every
//     row adds its own products in ascending column order: bit-equal to the
//     reference's CSR sum (kernels.py:27-37, separate mul and add):
//        FMA form  (all weights +-2^e): acc = fma(y, w, acc); y*w is exact,
//                  so fma == fl(acc + fl(y*w)). Outputs small enough that the
//                  next layer's products could underflow set a guard bit and
//                  the engine reruns in the exact form.
//        exact form (any weights): p = fma(y, w, -0) == fl(y*w); acc += p.
//     Epilogue: v = fl(acc + bias), comparison clamp (NaN kept,
//     kernels.py:33-36), 16-byte store per row, activity bits by ballot;
//   * 1 publisher warp: once every unit of an entry has arrived, folds the
//     entry's activity bits into its tile and releases the slot; the item
//     that completes tile t appends the tile's alive features to a_out /
//     cat_out (pruning without a pass over Y).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "common.h"

namespace {

constexpr int kMaxBufs = 4;
#ifndef SPDNN_PDL
#define SPDNN_PDL 1  // programmatic dependent launch between consecutive layers
#endif
constexpr int kUsePdl = SPDNN_PDL;
#ifndef SPDNN_META_AHEAD
#define SPDNN_META_AHEAD 3
#endif
#ifndef SPDNN_FP_AHEAD
#define SPDNN_FP_AHEAD 2
#endif
constexpr int kMetaAhead = SPDNN_META_AHEAD;  // producer: block descriptors prefetched this many items ahead
constexpr int kFpAhead = SPDNN_FP_AHEAD;      // producer: staged-row lists prefetched this many items ahead (>= 2)
constexpr int kMetaRing = kMetaAhead + 2;     // metadata ring entries (> kMetaAhead)
static_assert(kFpAhead >= 2 && kFpAhead < kMetaAhead && kMetaAhead + 2 <= 8, "prefetch depths");
#ifndef SPDNN_MASK_CONSUMERS
#define SPDNN_MASK_CONSUMERS 20
#endif
#ifndef SPDNN_MASK_PRODUCERS
#define SPDNN_MASK_PRODUCERS 3
#endif
#ifndef SPDNN_MASK_UNROLL
#define SPDNN_MASK_UNROLL 2
#endif
constexpr int kMaskUnroll = SPDNN_MASK_UNROLL;  // 4-record quads per loop iteration  // ring depth: as many buffers as shared memory holds (<= 4)
constexpr int kHeaderBytes = 128;  // keeps every region 128-byte aligned (TMA dst)

typedef unsigned long long u64;

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
// acc = y * w + acc in place. The CUDA intrinsic (not inline asm) lets the
// register allocator keep each accumulator in place (inline-asm "+l" operands
// cost 7 IMAD.MOV per record on the FMA pipe).
__device__ __forceinline__ void fma2_acc(u64 &acc, u64 y, float w) {
  float2 a = *reinterpret_cast<float2 *>(&acc);
  const float2 yy = *reinterpret_cast<const float2 *>(&y);
  a = __ffma2_rn(yy, make_float2(w, w), a);
  acc = *reinterpret_cast<u64 *>(&a);
}
// acc = acc + fl(y * w): the product rounded first. ptxas contracts even
// __fmul2_rn + __fadd2_rn into one FFMA2 (CUDA 12.9), so the product is an
// fma with a -0 addend the compiler cannot see (x + -0 == x for every x).
__device__ __forceinline__ void mul_add2_acc(u64 &acc, u64 y, float w, u64 negz2) {
  float2 a = *reinterpret_cast<float2 *>(&acc);
  const float2 yy = *reinterpret_cast<const float2 *>(&y);
  const float2 p = __ffma2_rn(yy, make_float2(w, w), *reinterpret_cast<const float2 *>(&negz2));
  a = __fadd2_rn(a, p);
  acc = *reinterpret_cast<u64 *>(&a);
}


// ---- async copy + mbarrier primitives -------------------------------------

__device__ __forceinline__ void cp_async4(uint32_t saddr, const void *gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t cnt) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar),
               "r"(cnt)
               : "memory");
}
// One arrival on `bar` once every cp.async this thread issued so far has landed
// (the barrier's expected count includes it: .noinc).
__device__ __forceinline__ void mbar_cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
// Blocks (suspended, up to the time hint) until the phase with `parity` is done.
#ifndef SPDNN_WAIT_TEST
#define SPDNN_WAIT_TEST 0  // 1: spin on test_wait instead of the suspending try_wait
#endif
#ifndef SPDNN_WAIT_HINT_NS
#define SPDNN_WAIT_HINT_NS 0  // 0: try_wait without a suspend-time hint
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#if SPDNN_WAIT_TEST
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
#elif SPDNN_WAIT_HINT_NS > 0
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(SPDNN_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
// Division by a runtime divisor d >= 1 for n < 2^31 (the producer splits every
// claimed item into tile and block, and ring counters into slot and phase):
// one multiply-high and two shifts instead of the ~20-instruction sequence.
struct FastDiv {
  uint32_t d, m;
  int s;  // -1: d == 1
  __device__ explicit FastDiv(uint32_t d_) : d(d_), m(0), s(-1) {
    if (d > 1) {
      const int l = 32 - __clz(d - 1);  // ceil(log2 d)
      m = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
      s = l - 1;
    }
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (s < 0) return n;
    const uint32_t t1 = __umulhi(m, n);
    return (t1 + ((n - t1) >> 1)) >> s;
  }
};

// TMA tile gather: rows r0..r3 of the 2-D tensor, columns [col, col + box),
// into 4 consecutive smem rows; completion as tx bytes on `bar`
__device__ __forceinline__ void tma_gather4(uint32_t sdst, const CUtensorMap *tmap, int col,
                                            int r0, int r1, int r2, int r3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(sdst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(bar)
      : "memory");
}
// TMA bulk copy global -> this CTA's shared memory, completion as tx bytes
__device__ __forceinline__ void bulk_g2s(uint32_t sdst, const void *gsrc, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(sdst), "l"(gsrc), "r"(bytes), "r"(bar)
      : "memory");
}

// ---- optional cycle accounting (build with -DSPDNN_PROFILE; diagnostics) ----
// Per warp, clock64() spans between marks are summed into 8 slots and added to
// g_prof at exit: consumers [0..7], producers [8..15]; read and reset with
// spdnn_profile_read().
__device__ unsigned long long g_prof[16];
// ring-chain timings (SPDNN_PROFILE): [0] issue (slot granted -> header posted),
// [1] fill (posted -> first consumer has data), [2] consume (first consumer ->
// last unit arrived), [3] release (last unit -> producer regains the slot),
// [4] entries, [5] releases; SM-local clock64 differences summed over entries
__device__ unsigned long long g_chain[8];
// per-entry timeline of CTA 0 (build with -DSPDNN_TRACE; diagnostics): for
// ring entries k < 96, clock64 at [0] rows free (grant), [1] producer warp 0
// issued its gathers, [2] units done (empty), [3] publisher done (free),
// [4] header posted, [5]/[6]/[7] consumer warp 0 start / loop done / unit
// done, [8]/[9]/[10] the same for the last consumer warp, [11] publisher
// saw empty; read with spdnn_trace_read()
__device__ long long g_trace[96][12];
// per-launch, per-CTA %globaltimer marks (build with -DSPDNN_LTRACE;
// diagnostics): [0] kernel entry, [1] consumer warp 0 past the grid
// dependency wait, [2] its first entry's data, [3] its exit, [4] the
// producer's first slot grant, [5] entries this CTA consumed
__device__ long long g_ltrace[64][160][6];
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef SPDNN_LTRACE
#define LTRACE(i, v)                                                     \
  do {                                                                  \
    if (lane == 0 && blockIdx.x < 160) g_ltrace[A.trace_slot & 63][blockIdx.x][(i)] = (v); \
  } while (0)
#else
#define LTRACE(i, v) \
  do {               \
  } while (0)
#endif
#ifdef SPDNN_TRACE
#define TRACE(k, i)                                                    \
  do {                                                                 \
    if (blockIdx.x == 0 && lane == 0 && (k) < 96) g_trace[(k)][(i)] = clock64(); \
  } while (0)
#else
#define TRACE(k, i) \
  do {              \
  } while (0)
#endif
#ifdef SPDNN_PROFILE
#define PROF_DECL                          \
  unsigned long long pf_[8] = {0};         \
  long long pt_ = clock64();
#define PROF_MARK(i)                       \
  {                                        \
    const long long n_ = clock64();        \
    pf_[i] += (unsigned long long)(n_ - pt_); \
    pt_ = n_;                              \
  }
#define PROF_FLUSH(base)                   \
  if (lane == 0)                           \
    for (int i_ = 0; i_ < 8; i_++) atomicAdd(&g_prof[(base) + i_], pf_[i_]);
#else
#define PROF_DECL
#define PROF_MARK(i)
#define PROF_FLUSH(base)
#endif

struct LayerArgs {
  CUtensorMap tmap_in;  // y_in as a 2-D tensor [N rows][ld cols], box 128 x 1
  spdnn_layer_dev L;
  const float *bias;
  const float *y_in;
  float *y_out;
  int64_t ld;
  uint32_t ld_bytes;   // 4 * ld (< 2^32): one output row of the feature buffer
  const int32_t *a_in;
  const int64_t *cat_in;
  const int32_t *m_in;
  // split survivor layout (scratch->split): al_in[0] = how many leading input
  // features form whole tiles of consecutive columns (the rest start at
  // a_in / cat_in + pk_off); al_out: the same counters for this layer's
  // survivors (aligned, packed), NULL = the packed layout
  const int32_t *al_in;
  int32_t *al_out;
  int64_t pk_off;
  int32_t *a_out;
  int64_t *cat_out;
  int32_t *m_out;
  int32_t *tile_done;
  uint32_t *tile_alive;
  int32_t *work;
  uint32_t *guard;     // bit 0: an output in (0, tiny) was produced (FMA form)
  float tiny;
  uint32_t tiny_bits_m1;  // bits(tiny) - 1: v in (0, tiny) <=> bits(v) - 1 < this
  float negz;          // -0.0f, opaque to the compiler (exact form)
  uint32_t buf_bytes;  // one ring buffer: header | meta | records | y rows
  uint32_t meta_bytes;
  uint32_t rec_bytes;
  int nbuf;            // ring depth
  uint32_t mring_off;  // producer metadata ring (after the nbuf buffers)
  uint32_t mentry_bytes;
  int gpi;             // consumer work units (row groups) per item = max groups per block
  uint32_t act_off;    // activity bytes: [nbuf][gpi][32 lanes], one byte per lane and unit
  int trace_slot;      // SPDNN_LTRACE: row of g_ltrace this launch writes (layer % 64)
};

// Ring-buffer header written by the producer (one per buffer fill).
struct Header {
  int item;     // -1: no more work
  int entry;    // ring entry number (stale-phase check)
  int t, b;
  int nst;
  int ng;
  int rec_cnt;  // records of this stage (multi-stage: all belong to group 0)
  int fp_cnt;
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
// R = 4 and 5 share the 8-word record of R = 6 (offset + up to 7 weights)
template <>
struct Rec<4> {
  static constexpr int W = 8;
  __device__ __forceinline__ static void load(const uint32_t *p, uint32_t &off, float *w) {
    uint4 a = *reinterpret_cast<const uint4 *>(p);
    uint4 b = *reinterpret_cast<const uint4 *>(p + 4);
    off = a.x;
    w[0] = __uint_as_float(a.y);
    w[1] = __uint_as_float(a.z);
    w[2] = __uint_as_float(a.w);
    w[3] = __uint_as_float(b.x);
  }
};
template <>
struct Rec<5> {
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
  }
};
template <>
struct Rec<6> {
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

// acc[2k], acc[2k+1]: row k, features (4l, 4l+1) and (4l+2, 4l+3).
// Records are walked with a bumped pointer; the feature row of a record is at
// ybase + record.offset.
// ---- per-configuration constants ---------------------------------------
// FPL = fp32 features per lane (2 or 4): a work item covers 32 * FPL features;
// a staged input neuron is a (128 * FPL)-byte smem row. FPL = 4 reuses every
// weight over more features, FPL = 2 halves the accumulator registers and
// buys twice the resident consumer warps.
// MASK = one-word mask records (uniform weights): no weight registers per
// record in flight, so the consumer loop fits 80 registers and 20 consumer
// warps (6 warps per scheduler instead of 5) hide the smem latency better.
template <int FPL, bool MASK>
struct Cfg;
template <>
struct Cfg<4, false> {
  static constexpr int kConsumers = 16, kProducers = 3;
};
template <>
struct Cfg<4, true> {
  static constexpr int kConsumers = SPDNN_MASK_CONSUMERS, kProducers = SPDNN_MASK_PRODUCERS;
};
template <bool MASK>
struct Cfg<2, MASK> {
  static constexpr int kConsumers = 28, kProducers = 3;
};
template <int FPL, bool MASK = false>
struct Geo {
  static constexpr int kTileF = 32 * FPL;      // features per item
  static constexpr int kRow = 4 * kTileF;      // staged row bytes
  static constexpr int kC = Cfg<FPL, MASK>::kConsumers;
  static constexpr int kP = Cfg<FPL, MASK>::kProducers;
  static constexpr int kThreads = (kC + kP + 1) * 32;  // + the publisher warp
  // record offsets are slot * SPDNN_STAGED_ROW_BYTES (512): shift to this row size
  static constexpr int kOffShift = FPL == 4 ? 0 : 1;
};

template <int FPL>
struct YVec;
template <>
struct YVec<4> {
  u64 v[2];
  __device__ __forceinline__ void load(const char *p) {
    const ulonglong2 t = *reinterpret_cast<const ulonglong2 *>(p);
    v[0] = t.x;
    v[1] = t.y;
  }
  // from a 32-bit shared-window address (one LEA.HI forms it from a record)
  __device__ __forceinline__ void load_s(uint32_t a) {
    asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "r"(a));
  }
};
template <>
struct YVec<2> {
  u64 v[1];
  __device__ __forceinline__ void load(const char *p) { v[0] = *reinterpret_cast<const u64 *>(p); }
  __device__ __forceinline__ void load_s(uint32_t a) {
    asm("ld.shared.u64 %0, [%1];" : "=l"(v[0]) : "r"(a));
  }
};

// acc[(FPL/2)*k + h]: row k, features (FPL*l + 2h, FPL*l + 2h + 1).
template <int R, bool FMA, int FPL, int UNROLL>
__device__ __forceinline__ void accumulate(u64 *acc, const uint32_t *recs, int cnt,
                                           const char *ybase, u64 negz2) {
  constexpr int RW = Rec<R>::W, H = FPL / 2;
  const uint32_t *rp = recs;
  const uint32_t *const end = recs + cnt * RW;
#pragma unroll UNROLL
  for (; rp < end; rp += RW) {
    uint32_t off;
    float w[R];
    Rec<R>::load(rp, off, w);
    YVec<FPL> y;
    y.load(ybase + (off >> Geo<FPL>::kOffShift));
#pragma unroll
    for (int k = 0; k < R; k++) {
#pragma unroll
      for (int h = 0; h < H; h++) {
        if (FMA) fma2_acc(acc[H * k + h], y.v[h], w[k]);
        else mul_add2_acc(acc[H * k + h], y.v[h], w[k], negz2);
      }
    }
  }
}

// Mask records (uniform weight w): 4 one-word records per 16-byte load; word
// = staged-row slot << 24 | row mask << 1, so the row's byte offset is
// word >> 15 (one LEA.HI with the base) and row k is bit k+1. Rows whose bit is clear add nothing --
// exactly the reference's sum, which never visits those columns. Each
// group's run is padded to a multiple of 4 with zero words (no-ops).
template <int R, bool FMA, int FPL>
__device__ __forceinline__ void mask_record(u64 *acc, uint32_t wd, const YVec<FPL> &y, float w,
                                            u64 negz2) {
  constexpr int H = FPL / 2;
#pragma unroll
  for (int k = 0; k < R; k++) {
    if (wd & (2u << k)) {  // row k = mask bit k+1
#pragma unroll
      for (int h = 0; h < H; h++) {
        if (FMA) fma2_acc(acc[H * k + h], y.v[h], w);
        else mul_add2_acc(acc[H * k + h], y.v[h], w, negz2);
      }
    }
  }
}

template <int R, bool FMA, int FPL>
__device__ __forceinline__ void accumulate_mask(u64 *acc, const uint32_t *recs, int cnt,
                                                uint32_t ybase, float w, u64 negz2) {
  const uint4 *rp = reinterpret_cast<const uint4 *>(recs);
  const uint4 *const end = rp + (cnt >> 2);
#pragma unroll kMaskUnroll
  for (; rp < end; rp++) {
    const uint4 q = *rp;
    const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
    YVec<FPL> y[4];
#pragma unroll
    for (int j = 0; j < 4; j++) y[j].load_s(ybase + (wd[j] >> (15 + Geo<FPL>::kOffShift)));
#pragma unroll
    for (int j = 0; j < 4; j++) mask_record<R, FMA, FPL>(acc, wd[j], y[j], w, negz2);
  }
  // the last 1-3 records of the run (cnt is exact; the run is stored padded
  // to a whole 16-byte quad with zero words, which are not executed): two
  // warp-uniform branches instead of 14 predicated-off FFMA2 per padding word
  const int rem = cnt & 3;
  if (rem) {
    const uint4 q = *rp;
    YVec<FPL> y;
    y.load_s(ybase + (q.x >> (15 + Geo<FPL>::kOffShift)));
    mask_record<R, FMA, FPL>(acc, q.x, y, w, negz2);
    if (rem > 1) {
      y.load_s(ybase + (q.y >> (15 + Geo<FPL>::kOffShift)));
      mask_record<R, FMA, FPL>(acc, q.y, y, w, negz2);
    }
    if (rem > 2) {
      y.load_s(ybase + (q.z >> (15 + Geo<FPL>::kOffShift)));
      mask_record<R, FMA, FPL>(acc, q.z, y, w, negz2);
    }
  }
}

// NaN-propagating max / min (max.NaN.f32): the reference's comparison clamp
// `v < 0 -> 0, v > 32 -> 32` keeps NaN; v is never -0 (the accumulator starts
// at +0 and round-to-nearest sums never produce -0), so max(v, +0) == v there.
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float min_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// The clamp of a value that is not NaN and not -0 (the FMA form's inputs are
// screened so sums stay finite, and round-to-nearest never yields -0 here):
// on the float bit pattern read as int32, order is preserved among
// non-negatives and every negative float is a negative int, so
// min(bits, bits(32)) followed by relu is min(max(v, 0), 32) -- one
// instruction (min.relu.s32) instead of two FMNMX.
__device__ __forceinline__ float clamp_finite(float v) {
  int r;
  asm("min.relu.s32 %0, %1, %2;" : "=r"(r) : "r"(__float_as_int(v)), "r"(0x42000000));
  return __int_as_float(r);
}

// Bias, clamp, store for one finished group; returns the lane's activity bits.
// All rows are finished into the accumulator registers first and stored
// after, so no store's source registers are overwritten while it is queued.
template <int R, bool FMA, int FPL, bool FULL>
__device__ __forceinline__ uint32_t finish_rows(const LayerArgs &A, u64 *acc, const int *rows,
                                                const float *bias, int j0, int valid,
                                                bool &tiny) {
  constexpr int H = FPL / 2;
  // row k's output address is one wide multiply-add off this base (the FMA
  // pipe is the kernel's bottleneck: no per-row re-derivation of ld * 4)
  const uint64_t obase = reinterpret_cast<uint64_t>(A.y_out) + 4ull * (uint32_t)j0;
  const uint32_t ldb = A.ld_bytes;
  // FMA form (finite values guaranteed, else the run is redone): per feature the
  // running unsigned min of bits(v) - 1 gives both tests: v > 0 exists <=> the
  // min is not 0xffffffff, and a v in (0, tiny) exists <=> min < bits(tiny) - 1.
  // Exact form: NaN may occur (non-finite inputs), alive uses a float max.
  float mx[FPL];
  uint32_t mn[FPL];
#pragma unroll
  for (int q = 0; q < FPL; q++) {
    mx[q] = 0.0f;
    mn[q] = 0xffffffffu;
  }
#pragma unroll
  for (int k = 0; k < R; k++) {
    const float2 b2 = make_float2(bias[k], bias[k]);
#pragma unroll
    for (int h = 0; h < H; h++) {
      float2 v = __fadd2_rn(*reinterpret_cast<float2 *>(&acc[H * k + h]), b2);
      if (FMA) {
        v.x = clamp_finite(v.x);
        v.y = clamp_finite(v.y);
      } else {
        v.x = min_nan(max_nan(v.x, 0.0f), 32.0f);
        v.y = min_nan(max_nan(v.y, 0.0f), 32.0f);
      }
      *reinterpret_cast<float2 *>(&acc[H * k + h]) = v;
    }
  }
#pragma unroll
  for (int k = 0; k < R; k++) {
    const float *x = reinterpret_cast<const float *>(&acc[H * k]);
#pragma unroll
    for (int q = 0; q < FPL; q++) {
      if (FMA) mn[q] = min(mn[q], __float_as_uint(x[q]) - 1u);  // padding rows give 0 -> no-op
      else if (rows[k] >= 0) mx[q] = fmaxf(mx[q], x[q]);
    }
    if (rows[k] < 0) continue;
#ifdef SPDNN_ABLATE_STORE
    if (rows[k] >= 0) continue;  // diagnostics: no output stores
#endif
    // one IMAD.WIDE.U32 per row: row * (ld * 4) + (y_out + 4 * j0)
    uint64_t da;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(da) : "r"((uint32_t)rows[k]), "r"(ldb), "l"(obase));
    float *dst = reinterpret_cast<float *>(da);
    if (FULL) {
      if (FPL == 4)
        asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(da), "f"(x[0]), "f"(x[1]),
                     "f"(x[2]), "f"(x[3])
                     : "memory");
      else
        asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(da), "f"(x[0]), "f"(x[1])
                     : "memory");
    } else {
#pragma unroll
      for (int q = 0; q < FPL; q++)
        if (q < valid) dst[q] = x[q];
    }
  }
  uint32_t am = 0, lo = 0xffffffffu;
#pragma unroll
  for (int q = 0; q < FPL; q++) {
    const bool in = FULL || q < valid;
    if (FMA) {
      am |= (in && mn[q] != 0xffffffffu) ? (1u << q) : 0u;
      if (in) lo = min(lo, mn[q]);
    } else {
      am |= (in && mx[q] > 0.0f) ? (1u << q) : 0u;
    }
  }
  if (FMA) tiny = lo < A.tiny_bits_m1;
  return am;
}


template <int R, bool FMA, int FPL>
__device__ __forceinline__ void epilogue(const LayerArgs &A, u64 *acc, const int *rows,
                                         const float *bias, int t, int lane, int M,
                                         uint8_t *act) {
  constexpr int T = Geo<FPL>::kTileF;
  const int j0 = t * T + FPL * lane;
  const int valid = M - j0;  // features of this lane that exist (may be <= 0)
  bool tiny = false;
  const uint32_t am = (t + 1) * T <= M
                          ? finish_rows<R, FMA, FPL, true>(A, acc, rows, bias, j0, valid, tiny)
                          : finish_rows<R, FMA, FPL, false>(A, acc, rows, bias, j0, valid, tiny);
  if (FMA && tiny) atomicOr(A.guard, 1u);
  // the lane's activity bits (bit q <=> feature FPL*lane + q is > 0), one
  // plain byte store: the publisher warp ORs the item's units together
  act[lane] = (uint8_t)am;
}

// Extra stages of a lone oversized group (rare: a row group whose inputs
// exceed the staging caps): its records are consumed straight from global
// memory, the feature values gathered through a_in. Slow, correct.
template <int R, bool FMA, int FPL, bool MASK>
__device__ void accumulate_global(const LayerArgs &A, u64 *acc, int b, int t, int lane, int M,
                                  u64 negz2) {
  const int nal = A.al_in ? *A.al_in : 0x7fffffff;
  constexpr int RW = MASK ? 1 : Rec<R>::W, H = FPL / 2, T = Geo<FPL>::kTileF;
  const float w0 = __uint_as_float(A.L.weight_bits);
  const int nst = __ldg(A.L.blocks + (int64_t)b * 8 + 2);
  const int first_extra = __ldg(A.L.blocks + (int64_t)b * 8 + 3);
  int pos[FPL];
  bool ok[FPL];
#pragma unroll
  for (int q = 0; q < FPL; q++) {
    const int j = t * T + FPL * lane + q;
    ok[q] = j < M;
    pos[q] = ok[q] ? __ldg(A.a_in + (A.al_in && j >= nal ? A.pk_off + (j - nal) : (int64_t)j)) : 0;
  }
  for (int s = 1; s < nst; s++) {
    const int4 sd = __ldg(reinterpret_cast<const int4 *>(A.L.stages) + first_extra + s - 1);
    const uint32_t *recs = A.L.records + (int64_t)sd.z * RW;
    for (int i = 0; i < sd.w; i++) {
      uint32_t off;
      float w[R];
      if (MASK) {
        const uint32_t wd = __ldg(recs + i);
        off = wd >> 15;
#pragma unroll
        for (int k = 0; k < R; k++) w[k] = (wd >> (k + 1)) & 1u ? w0 : 0.0f;
        if ((wd & (((1u << R) - 1u) << 1)) == 0u) continue;  // padding word
      } else {
        Rec<R>::load(recs + i * RW, off, w);  // (global loads)
      }
      const int64_t c = __ldg(A.L.meta + sd.x + off / SPDNN_STAGED_ROW_BYTES);
      const float *row = A.y_in + c * A.ld;
      float v[FPL];
#pragma unroll
      for (int q = 0; q < FPL; q++) v[q] = ok[q] ? __ldg(row + pos[q]) : 0.0f;
#pragma unroll
      for (int h = 0; h < H; h++) {
        const u64 y = pack2(v[2 * h], v[2 * h + 1]);
#pragma unroll
        for (int k = 0; k < R; k++) {
          if (MASK && w[k] == 0.0f) continue;  // row not connected: no term
          if (FMA) fma2_acc(acc[H * k + h], y, w[k]);
          else mul_add2_acc(acc[H * k + h], y, w[k], negz2);
        }
      }
    }
  }
}

template <int R, bool FMA, int FPL, bool MASK>
__global__ void __launch_bounds__(Geo<FPL, MASK>::kThreads, 1)
    layer_kernel(const __grid_constant__ LayerArgs A) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) u64 s_full[kMaxBufs], s_empty[kMaxBufs], s_free[kMaxBufs];
  __shared__ __align__(8) u64 s_rfree[kMaxBufs];
  __shared__ float s_wmask;
#ifdef SPDNN_PROFILE
  __shared__ long long s_tgr[kMaxBufs], s_tpost[kMaxBufs], s_tempty[kMaxBufs];
  __shared__ unsigned long long s_tfirst[kMaxBufs];
#endif
  __shared__ int s_items[8];  // producer: item index of ring entry j (j & 7)

  using G = Geo<FPL, MASK>;
  constexpr int RW = MASK ? 1 : Rec<R>::W, T = G::kTileF, C = G::kC, P = G::kP, H = FPL / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Programmatic dependent launch: the next layer's grid may be scheduled as
  // soon as every CTA here got this far (its CTAs start as SMs free up and run
  // their static prologue under this layer's tail). Everything the previous
  // layer wrote -- m_in, a_in, cat_in, y_in, the tile scratch -- is read only
  // after griddepcontrol.wait (dep_wait below).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid == 0) LTRACE(0, gtime());
  const int nb = (int)A.L.num_blocks;
  int M = 0, tiles = 0, items = 0x7fffffff;  // set by dep_wait
  int nal = 0x7fffffff;  // input features [0, nal) sit at their own index in a_in / cat_in
  // where input feature j's column and category are (split layout: the
  // aligned tiles, then the packed survivors at pk_off)
  auto pos = [&](int j) -> int64_t { return j < nal ? (int64_t)j : A.pk_off + (j - nal); };
  auto dep_wait = [&]() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    M = *A.m_in;
    if (A.al_in) nal = *A.al_in;
    tiles = (M + T - 1) / T;
    items = tiles * nb;
  };
  const int nbuf = A.nbuf, gpi = A.gpi;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(&s_full[0]);
  const uint32_t empty0 = (uint32_t)__cvta_generic_to_shared(&s_empty[0]);
  const uint32_t free0 = (uint32_t)__cvta_generic_to_shared(&s_free[0]);
  const uint32_t rfree0 = (uint32_t)__cvta_generic_to_shared(&s_rfree[0]);

  if (tid == 0) {
    s_wmask = __uint_as_float(A.L.weight_bits);
    for (int i = 0; i < nbuf; i++) {
      // the header arrival + one per producer thread (its row copies landed)
      // + the tx bytes of the TMA copies
      mbar_init(full0 + 8 * i, 1 + P * 32);
      mbar_init(empty0 + 8 * i, gpi * 32);  // every lane of every work unit (row group)
      mbar_init(free0 + 8 * i, 32);         // every publisher lane: activity bytes read
      mbar_init(rfree0 + 8 * i, gpi * 32);  // every unit's lanes: staged rows read
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp < C || warp >= C + P) {
    dep_wait();
    if (warp == 0) LTRACE(1, gtime());
    if (M <= 0) return;
  }

  if (warp >= C && warp < C + P) {
    // ======================= producer warps =======================
    // Per item (= ring fill): TMA bulk copies of the block's metadata and
    // union records and -- when the tile's feature columns are contiguous
    // (the steady state: every tile after a layer without deaths) -- TMA
    // gather4 of the staged rows, 4 input neurons x T features per op. Tiles
    // with gaps left by features that died in the previous layer are
    // gathered with 4-byte cp.async, the staged rows split over the
    // producer warps (named barrier 1 keeps them in step).
    //
    // Items are claimed from the layer's atomic counter kMetaAhead + 2
    // entries ahead (the claim's result is stored one iteration after it was
    // issued, so it never stalls), and each item's metadata is prefetched
    // into a shared-memory ring with cp.async, never through registers (a
    // register copy of a pending load would wait for it): the block
    // descriptor and the tile's feature columns kMetaAhead items ahead, the
    // staged-row list (whose address is in the descriptor) two items ahead.
    const int pw = warp - C;
    const int ptid = pw * 32 + lane;
    // This thread's first gather4 quad: quads are dealt round-robin over the
    // producer warps (lane-major), because a TMA instruction takes uniform
    // operands -- a warp issues its lanes' ops one after another, so 34 quads
    // in one warp would serialise ~34 issue rounds behind the others.
    const int qd0 = lane * P + pw;
    const FastDiv fnb((uint32_t)nb), fnbuf((uint32_t)nbuf);
    auto tile_of = [&](int item) { return (int)fnb.div((uint32_t)item); };
    auto pbar = [] { asm volatile("bar.sync 1, %0;\n" ::"n"(P * 32) : "memory"); };
    char *const mring = smem + A.mring_off;
    auto ment = [&](int j) { return mring + (j % kMetaRing) * A.mentry_bytes; };
    // entry layout: int desc[8] | int ain[T] | int fp[fpcap]
    auto item_of = [&](int j) { return s_items[j & 7]; };
    // descriptor (static: the layer's plan) and feature columns (written by
    // the previous layer) of item j
    auto prefetch_desc = [&](int j, bool blk, bool ain) {
      const int item = item_of(j);
      if (item >= items) return;
      const int t = tile_of(item), b = item - t * nb;
      const uint32_t e = (uint32_t)__cvta_generic_to_shared(ment(j));
      if (ptid < 2) {
        if (blk) cp_async16(e + 16 * ptid, A.L.blocks + (int64_t)b * 8 + 4 * ptid);
      } else if (ptid < 2 + T / 4) {
        const int q = ptid - 2;  // a_in has ld >= (t+1)*T entries; lanes past M are masked
        if (ain) cp_async16(e + 32 + 16 * q, A.a_in + pos(t * T) + 4 * q);
      }
    };
    auto prefetch_fp = [&](int j) {  // staged-row list of item j (descriptor landed)
      const int item = item_of(j);
      if (item >= items) return;
      const char *en = ment(j);
      const int meta_off = reinterpret_cast<const int *>(en)[4];
      const int fp_cnt = reinterpret_cast<const int *>(en)[5];
      const uint32_t e = (uint32_t)__cvta_generic_to_shared(en) + 32 + 4 * T;
      for (int q = ptid; 4 * q < fp_cnt; q += P * 32)
        cp_async16(e + 16 * q, A.L.meta + meta_off + 4 * q);
    };
    PROF_DECL
    int claim = 0;
    // entries 0..kMetaAhead are dealt statically, round j giving CTA c item
    // j*G + ((c + 17j) mod G): a small layer (few items) is spread over all
    // SMs instead of a few CTAs claiming the lookahead depth each, and the
    // per-round rotation keeps a CTA from meeting the same block every round
    // when the block count divides G. Later entries are claimed dynamically
    // (load balance at the tail) from item (kMetaAhead+1)*G on, so a CTA's
    // items stay increasing (the first one past the end stops the producer).
    const int G = (int)gridDim.x;
    const int dyn0 = (kMetaAhead + 1) * G;
    if (ptid == 0) {
      for (int j = 0; j <= kMetaAhead; j++)
        s_items[j] = j * G + (int)((blockIdx.x + 17u * j) % (unsigned)G);
      claim = dyn0 + atomicAdd(A.work, 1);  // entry kMetaAhead + 1
    }
    pbar();
    // static prologue (the plan only), overlapping the previous layer's tail
    for (int j = 0; j < kMetaAhead; j++) prefetch_desc(j, true, false);
    cp_async_commit();
    cp_async_wait<0>();
    pbar();
    for (int j = 0; j < kFpAhead; j++) prefetch_fp(j);
    cp_async_commit();
    // the feature columns of the first entries are fetched together with
    // the active count (one round trip): the tile of a statically dealt item
    // is known without M, and a tile inside the a_in allocation is safe to
    // read even if it turns out to lie past M (such items are never filled)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int j = 0; j < kMetaAhead; j++) {
      const int t0 = tile_of(item_of(j));
      if ((int64_t)(t0 + 1) * T <= A.ld) {
        const uint32_t e = (uint32_t)__cvta_generic_to_shared(ment(j));
        if (ptid >= 2 && ptid < 2 + T / 4)
          cp_async16(e + 32 + 16 * (ptid - 2), A.a_in + t0 * T + 4 * (ptid - 2));
      }
    }
    cp_async_commit();
    dep_wait();  // (griddepcontrol.wait again: returns at once) + M
    if (M <= 0) {
      cp_async_wait<0>();
      return;
    }
    if (A.al_in) {  // split input: a first tile among the packed survivors is refetched
      cp_async_wait<0>();  // (after the speculative copies: cp.async copies are unordered)
      for (int j = 0; j < kMetaAhead; j++) {
        const int t0 = tile_of(item_of(j));
        if (t0 * T >= nal && t0 < tiles) {
          const uint32_t e = (uint32_t)__cvta_generic_to_shared(ment(j));
          if (ptid >= 2 && ptid < 2 + T / 4)
            cp_async16(e + 32 + 16 * (ptid - 2), A.a_in + pos(t0 * T) + 4 * (ptid - 2));
        }
      }
      cp_async_commit();
    }
    cp_async_wait<0>();
    pbar();
    for (int k = 0;; k++) {
      // item k: descriptor (group k - kMetaAhead) and staged rows (group
      // k - kFpAhead) have landed once at most one group (the newest) is
      // pending; so have item k+1's (L2 prefetch) and item k+kFpAhead's
      // descriptor (group k - 2)
      if (ptid == 0) {
        s_items[(k + kMetaAhead + 1) & 7] = claim;  // claimed one iteration ago
        claim = dyn0 + atomicAdd(A.work, 1);         // entry k + kMetaAhead + 2
      }
      cp_async_wait<1>();
      pbar();
      const int item = item_of(k);
      if (item >= items) {
        cp_async_wait<0>();
        if (pw == 0) {
          // end markers in the next nbuf entries; a consumer warp waits at most
          // ceil(C / gpi) <= nbuf entries past the last one it served
          for (int e = 0; e < nbuf; e++, k++) {
            const int slot = k % nbuf;
            mbar_wait(free0 + 8 * slot, ((uint32_t)(k / nbuf) & 1u) ^ 1u);
            if (lane == 0) {
              Header *h = reinterpret_cast<Header *>(smem + slot * A.buf_bytes);
              h->item = -1;
              h->entry = k;
              mbar_arrive_cnt(full0 + 8 * slot, 1 + P * 32);  // (no copies)
            }
            __syncwarp();
          }
        }
        break;
      }
      const int *en = reinterpret_cast<const int *>(ment(k));
      const int t = tile_of(item), b = item - t * nb;
      const int ng = en[1], nst = en[2], meta_off = en[4], fp_cnt = en[5];
      const int rec_off = en[6], rec_cnt = en[7];
      const int *ain = en + 8;
      const int *sfp = en + 8 + T;
      // feature columns 32q + lane (q < FPL) of tile t
      const int valid = min(T, M - t * T);
      int src[FPL];
#pragma unroll
      for (int q = 0; q < FPL; q++) src[q] = 32 * q + lane < valid ? ain[32 * q + lane] : -1;
      const int p0 = ain[0];
      bool mine_contig = true;
#pragma unroll
      for (int q = 0; q < FPL; q++) mine_contig &= src[q] < 0 || src[q] == p0 + 32 * q + lane;
      const bool contig = __all_sync(0xffffffffu, mine_contig) && (p0 & 3) == 0;
      int4 c4 = make_int4(0, 0, 0, 0);
      if (4 * qd0 < fp_cnt) {
        c4 = *reinterpret_cast<const int4 *>(sfp + 4 * qd0);
        if (4 * qd0 + 1 >= fp_cnt) c4.y = c4.x;
        if (4 * qd0 + 2 >= fp_cnt) c4.z = c4.x;
        if (4 * qd0 + 3 >= fp_cnt) c4.w = c4.x;
      }
      PROF_MARK(3);  // [3] metadata from the prefetch ring

      const uint32_t kq = fnbuf.div((uint32_t)k);
      const int slot = k - (int)kq * nbuf;
      const uint32_t phase = kq & 1u;
      // Refill of ring slot `slot` (entry k; the slot last held entry k - nbuf),
      // in three steps that each wait only for what they overwrite:
      //   1. the staged rows, once every unit of k - nbuf is past its record
      //      loop (rows_free) -- the epilogues still run;
      //   2. block metadata and records, once every unit is done (empty);
      //   3. the header arrival, once the publisher has read the units'
      //      activity bytes (free), which entry k's units overwrite.
      if (pw == 0) mbar_wait(rfree0 + 8 * slot, phase ^ 1u);  // others park at the bar.sync below
#ifdef SPDNN_PROFILE
      if (ptid == 0) {
        const long long now = clock64();
        if (k >= nbuf) {
          atomicAdd(&g_chain[3], (unsigned long long)(now - s_tempty[slot]));
          atomicAdd(&g_chain[5], 1ull);
        }
        s_tgr[slot] = now;
        s_tfirst[slot] = ~0ull;
      }
#endif
      if (pw == 0) TRACE(k, 0);
      if (ptid == 0 && k == 0) LTRACE(4, gtime());
      PROF_MARK(0);  // [0] waiting for the slot's rows
      const uint32_t full = full0 + 8 * slot;
      const uint32_t buf = sbase + slot * A.buf_bytes;
      const uint32_t smeta = buf + kHeaderBytes;
      const uint32_t srec = smeta + A.meta_bytes;
      const uint32_t sy = srec + A.rec_bytes;
      const int meta_words = ((fp_cnt + 3) & ~3) + ((2 * ng + 2 * R * ng + 3) & ~3);
      const uint32_t rec_b = (uint32_t)((rec_cnt * RW * 4 + 15) & ~15);
      const int quads = (fp_cnt + 3) >> 2;
#ifdef SPDNN_ABLATE_STAGE
      const bool gather = false;  // diagnostics: staged rows are not copied
#else
      const bool gather = contig;
#endif
      if (ptid == 0)  // the phase cannot complete before the header's arrival
        mbar_expect_tx(full, (uint32_t)meta_words * 4u + rec_b +
                                 (gather ? (uint32_t)quads * 4u * G::kRow : 0u));
      pbar();  // the rows may be overwritten; expected bytes registered
      PROF_MARK(1);  // [1] barrier A
      if (gather) {
        if (qd0 < quads)
          tma_gather4(sy + (uint32_t)qd0 * 4u * G::kRow, &A.tmap_in, p0, c4.x, c4.y, c4.z, c4.w,
                      full);
        for (int qd = P * 32 + ptid; qd < quads; qd += P * 32) {  // footprints > 512 rows
          int4 c = *reinterpret_cast<const int4 *>(sfp + 4 * qd);
          if (4 * qd + 1 >= fp_cnt) c.y = c.x;
          if (4 * qd + 2 >= fp_cnt) c.z = c.x;
          if (4 * qd + 3 >= fp_cnt) c.w = c.x;
          tma_gather4(sy + (uint32_t)qd * 4u * G::kRow, &A.tmap_in, p0, c.x, c.y, c.z, c.w, full);
        }
        mbar_arrive(full);  // (the bytes complete the phase, not this arrival)
        if (pw == 0) TRACE(k, 1);
        PROF_MARK(6);  // [6] TMA gather4 issue (contiguous tiles)
      } else if (!contig) {
        // staged rows s = 32 pw .. : the warp's 32 lanes copy the row's T
        // features with 4-byte cp.async (tiles whose columns have gaps: the
        // layer right after one in which features died); each producer
        // thread's arrival on the full barrier fires once its copies landed
        for (int s0 = pw * 32; s0 < fp_cnt; s0 += P * 32) {
          const int my = s0 + lane < fp_cnt ? sfp[s0 + lane] : 0;
          const int cnt = min(32, fp_cnt - s0);
          for (int i = 0; i < cnt; i++) {
            const int64_t c = __shfl_sync(0xffffffffu, my, i);
            const float *row = A.y_in + c * A.ld;
            const uint32_t dst = sy + (uint32_t)(s0 + i) * G::kRow + 4 * lane;
#pragma unroll
            for (int q = 0; q < FPL; q++) cp_async4(dst + 128 * q, row + max(src[q], 0), src[q] >= 0);
          }
        }
        mbar_cp_async_arrive(full);
        PROF_MARK(7);  // [7] 4-byte cp.async gathers (tiles with gaps)
      } else {
        mbar_arrive(full);  // (diagnostics build without row staging)
      }
      if (pw == 0) {
        mbar_wait(empty0 + 8 * slot, phase ^ 1u);  // every unit of k - nbuf is done
        TRACE(k, 2);
        if (lane == 0) {
          if (meta_words) bulk_g2s(smeta, A.L.meta + meta_off, meta_words * 4, full);
          if (rec_b) bulk_g2s(srec, A.L.records + (int64_t)rec_off * RW, rec_b, full);
        }
        PROF_MARK(2);  // [2] bulk copies of meta + records
        mbar_wait(free0 + 8 * slot, phase ^ 1u);  // activity bytes of k - nbuf read
        TRACE(k, 3);
      }
      if (ptid == 0) {
        Header *h = reinterpret_cast<Header *>(smem + slot * A.buf_bytes);
        h->item = item;
        h->entry = k;
        h->t = t;
        h->b = b;
        h->nst = nst;
        h->ng = ng;
        h->rec_cnt = rec_cnt;
        h->fp_cnt = fp_cnt;
#ifdef SPDNN_PROFILE
        s_tpost[slot] = clock64();
#endif
        mbar_arrive(full);
        TRACE(k, 4);
      }
      // metadata for items k + kMetaAhead (descriptor) and k + kFpAhead
      // (staged rows; its descriptor landed with this iteration's wait):
      // ring entry k's slot is reused by k + kMetaRing > k + kMetaAhead only.
      // Issued after the header went out: off the slot turnaround path.
      prefetch_desc(k + kMetaAhead, true, true);
      prefetch_fp(k + kFpAhead);
      cp_async_commit();
      PROF_MARK(5);  // [5] header
    }
    PROF_FLUSH(8)
    return;
  }

  // the global part of a finished item (tile t, this lane's activity word
  // wv): OR it into the tile's words, count the tile's finished blocks, and
  // the item that completes tile t appends the tile's survivors to a_out /
  // cat_out (pruning without a pass over Y)
  auto account = [&](const int t, uint32_t wv) {
    if (lane < FPL && wv) atomicOr(&A.tile_alive[FPL * t + lane], wv);
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      // release our activity bits before the count; the last arrival
      // acquires everyone's (acq_rel instead of a full __threadfence)
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;\n"
                   : "=r"(old)
                   : "l"(A.tile_done + t)
                   : "memory");
      last = old == nb - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      if (lane < FPL) {
        wv = atomicOr(&A.tile_alive[FPL * t + lane], 0u);
        A.tile_alive[FPL * t + lane] = 0u;
      }
      if (lane == 0) A.tile_done[t] = 0;
      uint32_t mw[FPL];
      int tot = 0, below = 0;
#pragma unroll
      for (int q = 0; q < FPL; q++) {
        mw[q] = __shfl_sync(0xffffffffu, wv, q);
        tot += __popc(mw[q]);
        below += __popc(mw[q] & ((1u << lane) - 1u));  // alive features of lanes < this
      }
      // split layout: a whole tile of survivors is appended as an aligned
      // tile (its columns stay consecutive: the next layer stages it with
      // TMA gather4 even after deaths elsewhere); other survivors are packed
      const bool whole = A.al_out && tot == T && (t + 1) * T <= M;
      int64_t base = 0;
      if (lane == 0 && tot) {
        const int old = atomicAdd(A.m_out, tot);  // the layer's survivor count
        if (!A.al_out) base = old;
        else if (whole) base = atomicAdd(A.al_out, T);
        else base = A.pk_off + atomicAdd(A.al_out + 1, tot);
      }
      base = __shfl_sync(0xffffffffu, base, 0);
      // this lane's features FPL*lane + q, in feature order
      int64_t rank = base + below;
#pragma unroll
      for (int q = 0; q < FPL; q++) {
        if ((mw[q] >> lane) & 1u) {
          const int j = t * T + FPL * lane + q;
          A.a_out[rank] = j;
          A.cat_out[rank] = A.cat_in[pos(j)];
          rank++;
        }
      }
    }
  };

  if (warp == C + P) {
    // ======================= publisher warp =======================
    // Once every unit of ring entry k has arrived on empty[slot]: OR the
    // units' activity bytes into the tile's words, release the slot to the
    // producer (free[slot]), then account() for the item off the fill path.
    for (int k = 0;; k++) {
      const int slot = k % nbuf;
      const uint32_t phase = (uint32_t)(k / nbuf) & 1u;
      mbar_wait(full0 + 8 * slot, phase);
      const int item = reinterpret_cast<const volatile Header *>(smem + slot * A.buf_bytes)->item;
      const int t = reinterpret_cast<const volatile Header *>(smem + slot * A.buf_bytes)->t;
      if (item < 0) break;
      mbar_wait(empty0 + 8 * slot, phase);
      TRACE(k, 11);
#ifdef SPDNN_PROFILE
      if (lane == 0) {
        const long long now = clock64();
        const long long first = (long long)s_tfirst[slot];
        atomicAdd(&g_chain[0], (unsigned long long)(s_tpost[slot] - s_tgr[slot]));
        atomicAdd(&g_chain[1], (unsigned long long)(first - s_tpost[slot]));
        atomicAdd(&g_chain[2], (unsigned long long)(now - first));
        atomicAdd(&g_chain[4], 1ull);
        s_tempty[slot] = now;
      }
#endif
      // OR the units' activity bytes (this lane's FPL features), then turn
      // them into the tile's q-major words (word q bit l <=> feature FPL*l+q)
      const int ng = reinterpret_cast<const volatile Header *>(smem + slot * A.buf_bytes)->ng;
      const uint8_t *act = reinterpret_cast<const uint8_t *>(smem + A.act_off) + slot * gpi * 32;
      uint32_t am = 0u;
      for (int g = 0; g < ng; g++) am |= act[g * 32 + lane];
      uint32_t wv = 0u;
#pragma unroll
      for (int q = 0; q < FPL; q++) {
        const uint32_t word = __ballot_sync(0xffffffffu, (am >> q) & 1u);
        if (lane == q) wv = word;
      }
      mbar_arrive(free0 + 8 * slot);  // each lane's activity reads are done
      account(t, wv);
    }
    return;
  }

  // ======================= consumer warps =======================
  // Work unit u = (ring entry k = u / gpi, row group g = u % gpi); warp w
  // takes units w, w + C, ... launch_layer only admits mappings in which a
  // warp consumed the slot's previous entry itself before it waits on the
  // slot again, so the parity wait below always targets the current phase.
  const u64 negz2 = pack2(A.negz, A.negz);
  // the uniform weight, read from shared memory once: taken from the kernel
  // parameter, ptxas re-loads it from the constant bank before every
  // predicated FFMA2 instead of keeping it in a register
  const float w_mask = s_wmask;
  // unit u = warp + j*C  ->  (entry k, group g, ring slot, phase), advanced
  // incrementally (no per-unit integer division).
  int k = warp / gpi, g = warp - (warp / gpi) * gpi;
  int slot = k % nbuf;
  uint32_t phase = (uint32_t)(k / nbuf) & 1u;
  PROF_DECL
  for (;; ) {
    const char *buf = smem + slot * A.buf_bytes;
    mbar_wait(full0 + 8 * slot, phase);  // (launch_layer: never a stale phase)
    // the whole header in two 16-byte loads issued together (the fields are
    // otherwise loaded one by one behind the branches that test them)
    Header h;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(h.item), "=r"(h.entry), "=r"(h.t), "=r"(h.b)
                 : "r"((uint32_t)__cvta_generic_to_shared(buf)));
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(h.nst), "=r"(h.ng), "=r"(h.rec_cnt), "=r"(h.fp_cnt)
                 : "r"((uint32_t)__cvta_generic_to_shared(buf) + 16));
    if (warp == 0 && k == 0) LTRACE(2, gtime());
    if (warp == 0) TRACE(k, 5);
    if (warp == C - 1) TRACE(k, 8);
    PROF_MARK(0);  // [0] waiting for data
#ifdef SPDNN_PROFILE
    if (lane == 0 && h.item >= 0) atomicMin(&s_tfirst[slot], (unsigned long long)clock64());
#endif
    if (h.item < 0) break;
    if (g < h.ng) {
      const int32_t *meta = reinterpret_cast<const int32_t *>(buf + kHeaderBytes);
      const uint32_t *recs = reinterpret_cast<const uint32_t *>(buf + kHeaderBytes + A.meta_bytes);
      const char *ybase = buf + kHeaderBytes + A.meta_bytes + A.rec_bytes + 4 * FPL * lane;
      const int seg_base = (h.fp_cnt + 3) & ~3;
      u64 acc[H * R];
#pragma unroll
      for (int r = 0; r < H * R; r++) acc[r] = 0ull;
#ifdef SPDNN_ABLATE_COMPUTE
      if (false) {  // diagnostics: no record loop
#else
      if (MASK) {
#endif
        accumulate_mask<R, FMA, FPL>(acc, recs + meta[seg_base + 2 * g],
                                     meta[seg_base + 2 * g + 1],
                                     (uint32_t)__cvta_generic_to_shared(ybase), w_mask, negz2);
      } else if (!MASK) {
        accumulate<R, FMA, FPL, 4>(acc, recs + (int64_t)meta[seg_base + 2 * g] * RW,
                                   meta[seg_base + 2 * g + 1], ybase, negz2);
      }
      if (h.nst > 1) accumulate_global<R, FMA, FPL, MASK>(A, acc, h.b, h.t, lane, M, negz2);
      // this lane is done with the staged rows: the producer may refill them
      // while the epilogue runs
      mbar_arrive(rfree0 + 8 * slot);
      if (warp == 0) TRACE(k, 6);
      if (warp == C - 1) TRACE(k, 9);
      PROF_MARK(1);  // [1] record loop
      // output rows and their biases (staged with the block metadata) are read
      // only now, so they hold no registers across the record loop
      asm volatile("" ::: "memory");
      int rows[R];
      float bias[R];
      const int *mrows = meta + seg_base + 2 * h.ng + R * g;
      const float *mbias = reinterpret_cast<const float *>(meta + seg_base + 2 * h.ng + R * h.ng) + R * g;
#pragma unroll
      for (int r = 0; r < R; r++) {
        rows[r] = mrows[r];
        bias[r] = mbias[r];
      }
      epilogue<R, FMA, FPL>(A, acc, rows, bias, h.t, lane, M,
                            reinterpret_cast<uint8_t *>(smem + A.act_off) + (slot * gpi + g) * 32);
      PROF_MARK(2);  // [2] epilogue
    } else {
      mbar_arrive(rfree0 + 8 * slot);  // (a unit past the block's groups)
    }
    // every lane arrives (release) after its activity byte store; the
    // publisher warp folds the entry's bytes into the tile once all have
    mbar_arrive(empty0 + 8 * slot);
    if (warp == 0) TRACE(k, 7);
    if (warp == C - 1) TRACE(k, 10);
    g += C;
    while (g >= gpi) {
      g -= gpi;
      k++;
      if (++slot == nbuf) {
        slot = 0;
        phase ^= 1u;
      }
    }
    PROF_MARK(3);  // [3] unit bookkeeping, tile publishing
  }
  if (warp == 0) {
    LTRACE(3, gtime());
    LTRACE(5, (long long)k);
  }
  PROF_FLUSH(0)
}

// ---- launch configuration ---------------------------------------------------

template <int R, int FPL, bool MASK>
void *kernel_ptr(bool fma) {
  return fma ? reinterpret_cast<void *>(&layer_kernel<R, true, FPL, MASK>)
             : reinterpret_cast<void *>(&layer_kernel<R, false, FPL, MASK>);
}

template <int FPL, bool MASK>
void *kernel_for(int R, bool fma) {
  switch (R) {
    case 1: return kernel_ptr<1, FPL, MASK>(fma);
    case 3: return kernel_ptr<3, FPL, MASK>(fma);
    case 4: return kernel_ptr<4, FPL, MASK>(fma);
    case 5: return kernel_ptr<5, FPL, MASK>(fma);
    case 6: return kernel_ptr<6, FPL, MASK>(fma);
    case 7: return kernel_ptr<7, FPL, MASK>(fma);
    default: return nullptr;
  }
}

struct DevInfo {
  std::mutex mu;
  int device = -1, sms = 0;
  size_t optin = 0;
};
DevInfo g_dev;

struct LaunchCache {
  struct Entry {
    size_t smem_set = 0;                 // largest dynamic smem size set on the kernel
    std::map<size_t, int> occ;           // smem size -> CTAs per SM
  };
  std::mutex mu;
  std::map<std::pair<int, const void *>, Entry> map;
};
LaunchCache g_launch;

// (the caller's current device is returned in `dev`: g_dev may be switched to
// another device by a concurrent caller as soon as the lock is released)
int device_info(int &dev, int &sms, size_t &optin) {
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

template <int FPL, bool MASK>
int launch_layer(LayerArgs &A, bool fma, cudaStream_t stream, bool pdl) {
  using G = Geo<FPL, MASK>;
  const spdnn_layer_dev &L = A.L;
  void *fn = kernel_for<FPL, MASK>(L.rows_per_group, fma);
  if (!fn) return spdnn_fail(SPDNN_EINVAL, "layer: rows_per_group must be 1 or 3..7");
  if (MASK != (L.uniform != 0) || (MASK && L.record_words != 1))
    return spdnn_fail(SPDNN_EINVAL, "layer: record format does not match the layout");
  int dev, sms;
  size_t optin;
  if (device_info(dev, sms, optin)) return spdnn_fail(SPDNN_ECUDA, "layer: no CUDA device");
  auto up128 = [](size_t x) { return (x + 127) / 128 * 128; };
  const size_t meta = up128((size_t)L.max_meta_per_block * 4);
  const size_t rec = up128((size_t)L.max_records_per_stage * L.record_words * 4 + 16);
  const size_t ys = (size_t)((L.max_fp_per_stage + 3) & ~3) * G::kRow;  // gather4: rows in 4s
  const size_t buf = (kHeaderBytes + meta + rec + ys + 127) / 128 * 128;
  // producer metadata ring: descriptor | feature columns | staged-row list
  const size_t fpcap = (size_t)((L.max_fp_per_stage + 3) & ~3);
  const size_t mentry = ((8 + G::kTileF + fpcap) * 4 + 15) / 16 * 16;
  const size_t mring = (size_t)kMetaRing * mentry;
  const size_t budget = optin - 2048 - mring;  // static shared memory + reserve
  // + the per-unit activity bytes of each entry (gpi <= max(groups, C))
  const size_t act_unit = 32, act_max = (size_t)std::max(L.max_groups_per_block, G::kC) * act_unit;
  const int nbmax = (int)std::min<size_t>(kMaxBufs, budget / (buf + act_max));
  if (nbmax < 2) return spdnn_fail(SPDNN_ERANGE, "layer: staged tile exceeds shared memory");
  // Ring depth and units per entry (gpi). Every admitted mapping has each
  // consumer warp consume the slot's previous entry itself before it waits
  // on the slot again, so a parity wait can never see a stale phase:
  //   gpi >= C: each warp visits every entry;
  //   gpi | C with (C/gpi) | nbuf: each warp visits every (C/gpi)-th entry.
  // Among those, the most units with work per warp slot, then the deepest ring.
  const int C = G::kC, mg = std::max(1, L.max_groups_per_block);
  int nbuf = 0, gpi = 0;
  double best = -1.0;
  for (int nb = nbmax; nb >= 2; nb--) {
    auto consider = [&](int gp, double util) {
      if (util > best + 1e-9) {
        best = util;
        nbuf = nb;
        gpi = gp;
      }
    };
    if (mg >= C) consider(mg, 1.0);
    for (int d = mg; d < C; d++)
      if (C % d == 0 && nb % (C / d) == 0) consider(d, (double)mg / d);
    if (mg < C) consider(C, (double)mg / C);
  }
  const size_t smem = (size_t)nbuf * buf + mring + (size_t)nbuf * gpi * act_unit;
  A.mring_off = (uint32_t)(nbuf * buf);
  A.act_off = (uint32_t)(nbuf * buf + mring);
  A.mentry_bytes = (uint32_t)mentry;
  A.meta_bytes = (uint32_t)meta;
  A.rec_bytes = (uint32_t)rec;
  A.buf_bytes = (uint32_t)buf;
  A.nbuf = nbuf;
  A.gpi = gpi;
  // the smem attribute and the occupancy query cost several microseconds of
  // host time each; a layer loop launches every ~30 us at small batches, so
  // both are cached per (device, kernel): the attribute only ever grows
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(g_launch.mu);
    LaunchCache::Entry &en = g_launch.map[std::make_pair(dev, fn)];
    if (smem > en.smem_set) {
      cudaError_t e0 = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem);
      if (e0 != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e0));
      en.smem_set = smem;
      en.occ.clear();
    }
    auto it = en.occ.find(smem);
    if (it == en.occ.end()) {
      cudaError_t e0 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, G::kThreads, smem);
      if (e0 != cudaSuccess || per_sm < 1)
        return spdnn_fail(SPDNN_ECUDA, "layer: kernel does not fit on an SM");
      en.occ[smem] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  cudaError_t e;
  void *args[] = {&A};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms * per_sm);
  cfg.blockDim = dim3(G::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelExC(&cfg, fn, args);
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

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// y [n][ld] fp32 as a 2-D tensor whose box is one 128-feature row segment:
// the producer's gather4 fetches 4 such rows (4 input neurons) per TMA op.
int make_tensor_map(const float *y, int64_t n, int64_t ld, int box_cols, CUtensorMap *out) {
  auto enc = tensor_map_encoder();
  if (!enc) return spdnn_fail(SPDNN_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 1u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(y), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return spdnn_fail(SPDNN_ECUDA, "cuTensorMapEncodeTiled failed");
  return SPDNN_OK;
}

struct TmapCache {
  std::mutex mu;
  std::map<std::tuple<const float *, int64_t, int64_t, int>, CUtensorMap> maps;
};
TmapCache g_tmaps;

int tensor_map_for(const float *y, int64_t n, int64_t ld, int box_cols, CUtensorMap *out) {
  std::lock_guard<std::mutex> lk(g_tmaps.mu);
  auto key = std::make_tuple(y, n, ld, box_cols);
  auto it = g_tmaps.maps.find(key);
  if (it != g_tmaps.maps.end()) {
    *out = it->second;
    return SPDNN_OK;
  }
  if (g_tmaps.maps.size() > 64) g_tmaps.maps.clear();
  int rc = make_tensor_map(y, n, ld, box_cols, out);
  if (rc == SPDNN_OK) g_tmaps.maps[key] = *out;
  return rc;
}

int forward(const spdnn_layer_dev *layer, const float *bias, const float *y_in, float *y_out,
            int64_t ld, const int32_t *a_in, const int64_t *cat_in, const int32_t *m_in,
            int32_t *a_out, int64_t *cat_out, int32_t *m_out, const spdnn_scratch *scratch,
            int32_t *work, const spdnn_run_opts *opts, void *stream,
            const int32_t *al_in = nullptr, int32_t *al_out = nullptr) {
  // ld * 4 must fit 32 bits: the epilogue forms row addresses with one wide multiply
  if (!layer || !bias || !y_in || !y_out || !a_in || !cat_in || !m_in || !a_out ||
      !cat_out || !m_out || !scratch || !work || ld < 1 || ld % SPDNN_TILE_FEATURES ||
      ld >= (int64_t)1 << 30)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_layer_forward: bad argument");
  const bool fma = opts && opts->fma_form;
  if (fma && !scratch->guard)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_layer_forward: the FMA form needs scratch->guard");
  if (layer->num_blocks == 0) return SPDNN_OK;  // N == 0
  LayerArgs A;
  std::memset(&A, 0, sizeof(A));
  const int fpl = (opts && opts->features_per_lane == 2) ? 2 : 4;
  int rc = tensor_map_for(y_in, layer->neurons, ld, 32 * fpl, &A.tmap_in);
  if (rc) return rc;
  A.L = *layer;
  A.bias = bias;
  A.y_in = y_in;
  A.y_out = y_out;
  A.ld = ld;
  A.ld_bytes = (uint32_t)(ld * 4);
  A.a_in = a_in;
  A.cat_in = cat_in;
  A.m_in = m_in;
  A.a_out = a_out;
  A.cat_out = cat_out;
  A.m_out = m_out;
  A.al_in = al_in;
  A.al_out = al_out;
  A.pk_off = ld;  // split layout: a_* / cat_* hold 2 * ld entries
  A.tile_done = scratch->tile_done;
  A.tile_alive = scratch->tile_alive;
  A.work = work;
  A.guard = scratch->guard;
  A.tiny = opts ? opts->tiny : 0.0f;
  uint32_t tb;
  std::memcpy(&tb, &A.tiny, 4);
  A.tiny_bits_m1 = tb ? tb - 1u : 0u;
  A.negz = -0.0f;
  {
    static std::atomic<int> launches{0};
    A.trace_slot = launches.fetch_add(1) & 63;
  }
  const bool pdl = kUsePdl != 0;
  const bool mask = layer->uniform != 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (fpl == 2)
    return mask ? launch_layer<2, true>(A, fma, st, pdl) : launch_layer<2, false>(A, fma, st, pdl);
  return mask ? launch_layer<4, true>(A, fma, st, pdl) : launch_layer<4, false>(A, fma, st, pdl);
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

static int infer_layers(int64_t num_layers, const spdnn_layer_dev *layers, const float *bias,
                        float *y0, float *y1, int64_t ld, int32_t *a0, int32_t *a1,
                        int64_t *cat0, int64_t *cat1, int32_t *counts,
                        const spdnn_scratch *scratch, const spdnn_run_opts *opts, void *stream,
                        void *const *events) {
  if (num_layers < 0 || (num_layers > 0 && (!layers || !scratch)))
    return spdnn_fail(SPDNN_EINVAL, "spdnn_infer_layers: bad argument");
  for (int64_t l = 0; l < num_layers; l++) {
    const int i = (int)(l & 1), o = i ^ 1;
    float *y[2] = {y0, y1};
    int32_t *a[2] = {a0, a1};
    int64_t *cat[2] = {cat0, cat1};
    if (events && cudaEventRecord((cudaEvent_t)events[l], (cudaStream_t)stream) != cudaSuccess)
      return spdnn_fail(SPDNN_ECUDA, "spdnn_infer_layers_timed: event record failed");
    // split survivor layout between the layers of this call (scratch->split);
    // the last layer's survivors are packed, as spdnn_infer_layers returns them
    int32_t *sp = scratch->split;
    const int32_t *al_in = sp && l > 0 ? sp + 2 * l : nullptr;
    int32_t *al_out = sp && l + 1 < num_layers ? sp + 2 * (l + 1) : nullptr;
    int rc = forward(&layers[l], bias, y[i], y[o], ld, a[i], cat[i], counts + l, a[o], cat[o],
                     counts + l + 1, scratch, scratch->work + l, opts, stream, al_in, al_out);
    if (rc) return rc;
  }
  if (events && cudaEventRecord((cudaEvent_t)events[num_layers], (cudaStream_t)stream) !=
                    cudaSuccess)
    return spdnn_fail(SPDNN_ECUDA, "spdnn_infer_layers_timed: event record failed");
  return SPDNN_OK;
}

extern "C" int spdnn_infer_layers(int64_t num_layers, const spdnn_layer_dev *layers,
                                  const float *bias, float *y0, float *y1, int64_t ld,
                                  int32_t *a0, int32_t *a1, int64_t *cat0, int64_t *cat1,
                                  int32_t *counts, const spdnn_scratch *scratch,
                                  const spdnn_run_opts *opts, void *stream) {
  return infer_layers(num_layers, layers, bias, y0, y1, ld, a0, a1, cat0, cat1, counts, scratch,
                      opts, stream, nullptr);
}

extern "C" int spdnn_infer_layers_timed(int64_t num_layers, const spdnn_layer_dev *layers,
                                        const float *bias, float *y0, float *y1, int64_t ld,
                                        int32_t *a0, int32_t *a1, int64_t *cat0, int64_t *cat1,
                                        int32_t *counts, const spdnn_scratch *scratch,
                                        const spdnn_run_opts *opts, void *stream,
                                        void *const *events) {
  if (!events) return spdnn_fail(SPDNN_EINVAL, "spdnn_infer_layers_timed: null events");
  return infer_layers(num_layers, layers, bias, y0, y1, ld, a0, a1, cat0, cat1, counts, scratch,
                      opts, stream, events);
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

extern "C" int spdnn_profile_read(uint64_t *out, int32_t n, int32_t reset) {
  if (!out || n < 0 || n > 24) return spdnn_fail(SPDNN_EINVAL, "spdnn_profile_read: bad args");
  unsigned long long h[24];
  cudaError_t e = cudaMemcpyFromSymbol(h, g_prof, 16 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(h + 16, g_chain, 8 * sizeof(unsigned long long));
  if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  for (int i = 0; i < n; i++) out[i] = h[i];
  if (reset) {
    std::memset(h, 0, sizeof(h));
    e = cudaMemcpyToSymbol(g_prof, h, 16 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_chain, h, 8 * sizeof(unsigned long long));
    if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  }
  return SPDNN_OK;
}

extern "C" int spdnn_trace_read(int64_t *out, int32_t n) {
  if (!out || n < 0 || n > 96 * 12) return spdnn_fail(SPDNN_EINVAL, "spdnn_trace_read: bad args");
  long long h[96 * 12];
  cudaError_t e = cudaMemcpyFromSymbol(h, g_trace, sizeof(h));
  if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  for (int i = 0; i < n; i++) out[i] = h[i];
  return SPDNN_OK;
}

extern "C" int spdnn_ltrace_read(int64_t *out, int32_t n) {
  if (!out || n < 0 || n > 64 * 160 * 6)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_ltrace_read: bad args");
  static long long h[64 * 160 * 6];
  cudaError_t e = cudaMemcpyFromSymbol(h, g_ltrace, sizeof(h));
  if (e != cudaSuccess) return spdnn_fail(SPDNN_ECUDA, cudaGetErrorString(e));
  for (int i = 0; i < n; i++) out[i] = h[i];
  return SPDNN_OK;
}

extern "C" int spdnn_layer_occupancy(int32_t rows_per_group, int32_t *ctas_per_sm,
                                     int32_t *threads_per_cta) {
  (void)rows_per_group;
  if (threads_per_cta) *threads_per_cta = Geo<4, true>::kThreads;
  if (ctas_per_sm) *ctas_per_sm = 1;
  return SPDNN_OK;
}
