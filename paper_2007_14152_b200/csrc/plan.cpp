// plan.cpp -- one-time host conversion of a CSR layer into the B200 layout
// ("row-grouped union ELL"). Replaces the reference's staging plan + sliced
// ELL builders (spdnn/preprocess.py:148-190 build_staging_plan,
// :212-244 csr_to_sliced_ell) as called from engine.prepare_layer
// (spdnn/engine.py:77-85).
//
// Layout:
//   * rows are put in an order where consecutive rows share many input
//     columns (greedy nearest-overlap chain over the column->row index;
//     generic, no knowledge of how the network was generated);
//   * R consecutive rows form a group; the group's union U of input columns
//     (ascending neuron index) becomes one "record" per column: the staged
//     smem offset of that input neuron plus R weights (0 where a row does not
//     connect). Every row still visits its own columns in ascending order,
//     interleaved with exact +0 contributions, so its fp32 sum is bit-equal to
//     the reference's ascending CSR sum (spdnn/kernels.py:27-37);
//   * consecutive groups form a block whose input footprint (union of the
//     group unions) is staged once per 128-feature tile; a block whose single
//     group needs more than `footprint_cap` inputs is split into stages
//     (the reference's buffer_capacity stages, preprocess.py:148-190).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <new>
#include <stdexcept>
#include <utility>
#include <string>
#include <thread>
#include <vector>

#include "common.h"

struct spdnn_plan {
  int64_t n = 0;
  int R = 1, RW = 2;
  std::vector<int32_t> blocks;   // 8 ints per block (descriptor)
  std::vector<int32_t> stages;   // 4 ints per extra stage of a multi-stage block
  std::vector<int32_t> meta;     // per block: fp list, group segments, group rows
  std::vector<uint32_t> records;
  int64_t nnz = 0;
  int64_t num_groups = 0;
  int32_t max_fp = 0, max_rec = 0, max_meta = 0, max_groups = 0;
  int64_t num_fp = 0;
  int64_t union_records = 0;     // records excluding alignment padding
  int32_t pow2 = 0;              // every nonzero weight is +-2^e (FMA form allowed)
  int32_t wexp_min = 0, wexp_max = 0;
  int32_t uniform = 0;           // one-word mask records: every nonzero has these bits
  uint32_t weight_bits = 0;
};

namespace {


int record_words(int R, bool uniform) {
  return uniform ? 1 : (R == 1 ? 2 : (R == 3 ? 4 : 8));
}

// True when every stored weight has the same nonzero bit pattern: the layer
// is then described by its pattern alone and a record is one 32-bit word,
// staged-row slot << 24 | R-bit row mask (slots < 256: footprint_cap <= 256).
// Graph Challenge layers are all 1/16.
bool uniform_weights(int64_t nnz, const float *va, uint32_t &bits) {
  if (nnz == 0) return false;
  std::memcpy(&bits, &va[0], 4);
  if ((bits & 0x7fffffffu) == 0) return false;
  for (int64_t p = 1; p < nnz; p++) {
    uint32_t b;
    std::memcpy(&b, &va[p], 4);
    if (b != bits) return false;
  }
  return true;
}

bool valid_csr(int64_t n, const int64_t *rp, const int32_t *ci) {
  if (n < 0 || rp[0] != 0) return false;
  for (int64_t r = 0; r < n; r++) {
    if (rp[r + 1] < rp[r]) return false;
    for (int64_t p = rp[r]; p < rp[r + 1]; p++) {
      if (ci[p] < 0 || ci[p] >= n) return false;
      if (p > rp[r] && ci[p] <= ci[p - 1]) return false;
    }
  }
  return true;
}

// Greedy nearest-overlap chain: from the current row go to the unvisited row
// sharing the most input columns (ties -> lower index); when none shares a
// column, restart at the lowest unvisited row. Columns feeding more than
// `deg_cap` rows are skipped as candidate generators (bounded cost on dense
// columns; they still count toward nothing else).
// (n rows over ncol columns)
std::vector<int32_t> overlap_order_cols(int64_t n, int64_t ncol, const int64_t *rp,
                                        const int32_t *ci) {
  std::vector<int32_t> order;
  order.reserve(n);
  if (n == 0) return order;
  // column -> rows (CSC pattern)
  std::vector<int64_t> cp(ncol + 1, 0);
  for (int64_t p = 0; p < rp[n]; p++) cp[ci[p] + 1]++;
  for (int64_t c = 0; c < ncol; c++) cp[c + 1] += cp[c];
  std::vector<int32_t> cr(rp[n]);
  {
    std::vector<int64_t> fill(cp.begin(), cp.end() - 1);
    for (int64_t r = 0; r < n; r++)
      for (int64_t p = rp[r]; p < rp[r + 1]; p++) cr[fill[ci[p]]++] = (int32_t)r;
  }
  const int64_t deg_cap = 512;
  std::vector<uint8_t> visited(n, 0);
  std::vector<int32_t> cnt(n, 0);
  std::vector<int32_t> touched;
  touched.reserve(4096);
  int64_t next_free = 0;
  int64_t cur = 0;
  while ((int64_t)order.size() < n) {
    if (cur < 0) {
      while (visited[next_free]) next_free++;
      cur = next_free;
    }
    visited[cur] = 1;
    order.push_back((int32_t)cur);
    int64_t best = -1;
    int32_t bestc = 0;
    for (int64_t p = rp[cur]; p < rp[cur + 1]; p++) {
      int64_t c = ci[p];
      if (cp[c + 1] - cp[c] > deg_cap) continue;
      for (int64_t q = cp[c]; q < cp[c + 1]; q++) {
        int32_t r2 = cr[q];
        if (visited[r2]) continue;
        if (cnt[r2]++ == 0) touched.push_back(r2);
      }
    }
    for (int32_t r2 : touched) {
      int32_t k = cnt[r2];
      if (k > bestc || (k == bestc && r2 < best)) { bestc = k; best = r2; }
      cnt[r2] = 0;
    }
    touched.clear();
    cur = best;
  }
  return order;
}

std::vector<int32_t> overlap_order(int64_t n, const int64_t *rp, const int32_t *ci) {
  return overlap_order_cols(n, n, rp, ci);
}

// overlap_order over classes of identical rows: rows with the same column
// list (e.g. 2^v rows per window when the generator's offset/stride ratio has
// 2-adic valuation v) form one class; the greedy chain runs over one
// representative per class and each class is emitted in place, so a row
// group falls inside one class (its union is the rows' own columns: no
// padding). Without this, a column shared by more than deg_cap identical rows
// is skipped as a generator and the chain degrades to the identity order.
std::vector<int32_t> class_overlap_order(int64_t n, const int64_t *rp, const int32_t *ci) {
  std::vector<uint64_t> h((size_t)n);
  for (int64_t r = 0; r < n; r++) {
    uint64_t x = 1469598103934665603ull ^ (uint64_t)(rp[r + 1] - rp[r]);
    for (int64_t p = rp[r]; p < rp[r + 1]; p++) x = (x ^ (uint64_t)(uint32_t)ci[p]) * 1099511628211ull;
    h[(size_t)r] = x;
  }
  std::vector<int32_t> idx((size_t)n);
  for (int64_t r = 0; r < n; r++) idx[(size_t)r] = (int32_t)r;
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return h[a] < h[b]; });
  auto same = [&](int32_t a, int32_t b) {
    const int64_t la = rp[a + 1] - rp[a];
    return la == rp[b + 1] - rp[b] && std::equal(ci + rp[a], ci + rp[a] + la, ci + rp[b]);
  };
  // classes: members listed in ascending row index, representative = first
  std::vector<int32_t> cls_of((size_t)n, -1), reps;
  std::vector<std::vector<int32_t>> members;
  for (size_t i = 0; i < idx.size();) {
    size_t j = i;
    while (j < idx.size() && h[idx[j]] == h[idx[i]]) j++;
    // rows with equal hashes: split into classes of equal column lists
    for (size_t a = i; a < j; a++) {
      const int32_t r = idx[a];
      if (cls_of[r] >= 0) continue;
      const int32_t c = (int32_t)reps.size();
      reps.push_back(r);
      members.emplace_back();
      for (size_t b = a; b < j; b++)
        if (cls_of[idx[b]] < 0 && same(r, idx[b])) {
          cls_of[idx[b]] = c;
          members.back().push_back(idx[b]);
        }
    }
    i = j;
  }
  if ((int64_t)reps.size() == n) return overlap_order(n, rp, ci);
  // the representatives as a CSR, ordered by their smallest member row
  std::vector<int32_t> cord((size_t)reps.size());
  for (size_t c = 0; c < reps.size(); c++) {
    std::sort(members[c].begin(), members[c].end());
    cord[c] = (int32_t)c;
  }
  std::sort(cord.begin(), cord.end(),
            [&](int32_t a, int32_t b) { return members[a][0] < members[b][0]; });
  const int64_t nc = (int64_t)reps.size();
  std::vector<int64_t> rp2((size_t)nc + 1, 0);
  std::vector<int32_t> ci2;
  for (int64_t k = 0; k < nc; k++) {
    const int32_t r = reps[cord[k]];
    ci2.insert(ci2.end(), ci + rp[r], ci + rp[r + 1]);
    rp2[(size_t)k + 1] = (int64_t)ci2.size();
  }
  // column ids stay < n; the chain only compares column sets
  std::vector<int32_t> corder = overlap_order_cols(nc, n, rp2.data(), ci2.data());
  std::vector<int32_t> order;
  order.reserve((size_t)n);
  for (int32_t k : corder)
    for (int32_t r : members[cord[k]]) order.push_back(r);
  return order;
}

// Exponent range when every nonzero weight is +-2^e with e in the normal
// range: then y*w is exact for every normal product, which is what lets the
// kernel use a single FFMA2 per (row, column) (layer.cu, "FMA form").
bool pow2_weights(int64_t nnz, const float *va, int32_t &emin, int32_t &emax) {
  emin = 1000;
  emax = -1000;
  for (int64_t p = 0; p < nnz; p++) {
    uint32_t b;
    std::memcpy(&b, &va[p], 4);
    if ((b & 0x7fffffffu) == 0) continue;          // +-0: product is exactly 0
    const uint32_t ex = (b >> 23) & 0xffu, man = b & 0x7fffffu;
    if (man != 0 || ex == 0 || ex == 0xffu) return false;  // not a normal power of two
    const int32_t e = (int32_t)ex - 127;
    emin = std::min(emin, e);
    emax = std::max(emax, e);
  }
  if (emin > emax) { emin = 0; emax = 0; }  // no nonzero weights
  return true;
}

struct Group {
  int32_t rows[7];
  std::vector<int32_t> cols;  // ascending union
};

// Union of the group's rows, ascending (k-way merge via sort of the <= 7*K cols).
void group_union(const int64_t *rp, const int32_t *ci, const int32_t *rows, int R,
                 std::vector<int32_t> &out) {
  out.clear();
  for (int k = 0; k < R; k++) {
    if (rows[k] < 0) continue;
    out.insert(out.end(), ci + rp[rows[k]], ci + rp[rows[k] + 1]);
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
}

std::vector<Group> make_groups(int64_t n, const int64_t *rp, const int32_t *ci,
                               const std::vector<int32_t> &order, int R) {
  std::vector<Group> gs((n + R - 1) / R);
  for (size_t g = 0; g < gs.size(); g++) {
    for (int k = 0; k < 7; k++) gs[g].rows[k] = -1;
    for (int k = 0; k < R; k++) {
      int64_t i = (int64_t)g * R + k;
      if (i < n) gs[g].rows[k] = order[i];
    }
    group_union(rp, ci, gs[g].rows, R, gs[g].cols);
  }
  return gs;
}

int64_t total_records(const std::vector<Group> &gs) {
  int64_t s = 0;
  for (auto &g : gs) s += (int64_t)g.cols.size();
  return s;
}

// Issue-slot / smem-wavefront cost per union record, per warp:
// R=1: 4 issue, 3 wavefronts; R=3: 8 issue, 3 wavefronts; R=7: 17 issue,
// 4 wavefronts. Time ~ max(issue/4, wavefronts) smem-or-issue bound per SM.
double record_cost(int R) { return R == 1 ? 3.0 : (R == 3 ? 3.0 : 4.25); }
// Mask records (uniform weights), SM clocks per record: the staged-row load
// is 4 smem wavefronts plus a quarter of a broadcast record load; the FMA
// pipe retires 2 FFMA2 per clock per SM (R = 7: 14 FFMA2 = 7 clocks).
double mask_record_cost(int R) { return R == 7 ? 7.0 : (R == 6 ? 6.0 : 4.25); }
// Mask-record layers with at least this many rows group 6 rows instead of 7:
// measured on B200 16384 x 1920 +1.7 %, 65536 x 1920 +1.6 %,
// 4096 x 480 +-0, 1024 x 120 -1.8 % (with 32 connections per row a 6-row
// group's union holds 37 records and a 7-row group's 38: 13.5 % padded slots
// instead of 15.8 %, at 17 % more groups per layer)
constexpr int64_t kR6MinRows = 8192;

// The kernel keeps at least two ring entries in shared memory, so one
// block stage (staged rows + records + metadata + header) must fit half of
// the ~225 KB a CTA can use. The caps were tuned for one-word mask records;
// per-row weight records are 2-8 words, so the record cap, then the
// footprint cap, shrink until a stage fits.
spdnn_plan_params fit_caps(spdnn_plan_params p, int R, int RW) {
  // (227 KB - static smem - the producer's metadata ring) / 2, minus the
  // 128-byte rounding of every region
  const int64_t budget = 104 * 1024;
  auto stage_bytes = [&](int64_t s, int64_t rc) {
    const int64_t meta = s + 4 + 2 * (int64_t)p.max_groups + 2 * (int64_t)R * p.max_groups + 4;
    return s * SPDNN_STAGED_ROW_BYTES + rc * RW * 4 + 16 + meta * 4 + 128 + 3 * 128;
  };
  while (stage_bytes(p.footprint_cap, p.record_cap) > budget && p.record_cap > p.footprint_cap)
    p.record_cap = std::max(p.footprint_cap, p.record_cap - 8);
  while (stage_bytes(p.footprint_cap, p.record_cap) > budget && p.footprint_cap > 8) {
    p.footprint_cap -= 8;
    p.record_cap = std::max(p.footprint_cap, p.record_cap);
  }
  return p;
}

void pad4(std::vector<int32_t> &v) {
  while (v.size() % 4) v.push_back(0);
}

// Lay the groups out as blocks. Per block (include/spdnn_b200.h):
//   descriptor {g_first, ng, nst, first_extra_stage, meta_off, fp_cnt, rec_off, rec_cnt}
//   meta       [fp indices of stage 0][pad][ng x (rec_rel, cnt)][ng x R rows]
//              [ng x R bias slots][pad]
//   records    per group, its union columns in ascending order
// A block with more than one stage holds exactly one group; its stages 1..
// live in `stages` as {meta_off, fp_cnt, rec_off, rec_cnt} (meta = fp list).
void emit(spdnn_plan *pl, const int64_t *rp, const int32_t *ci, const float *va,
          const std::vector<Group> &gs, const spdnn_plan_params &p) {
  const int R = pl->R, RW = pl->RW;
  const int64_t n = pl->n;
  const int S = p.footprint_cap, RC = p.record_cap, GMAX = p.max_groups;
  std::vector<int32_t> stamp(n, -1);
  std::vector<int32_t> slot_of(n, 0);
  std::vector<int32_t> fp_block;
  int32_t blk_id = 0;
  auto weight = [&](int32_t row, int32_t col) -> float {
    const int32_t *b = ci + rp[row], *e = ci + rp[row + 1];
    const int32_t *it = std::lower_bound(b, e, col);
    return (it != e && *it == col) ? va[it - ci] : 0.0f;
  };
  // records of groups [g0, g0+ng) restricted to footprint columns [c_lo, c_hi)
  auto emit_records = [&](size_t g0, size_t ng, int64_t c_lo, int64_t c_hi,
                          std::vector<int32_t> *gseg) {
    const int32_t lo_col = c_hi > c_lo ? fp_block[c_lo] : 0;
    const int32_t hi_col = c_hi > c_lo ? fp_block[c_hi - 1] : -1;
    for (int64_t i = c_lo; i < c_hi; i++) slot_of[fp_block[i]] = (int32_t)(i - c_lo);
    const int64_t rec_off = (int64_t)pl->records.size() / RW;
    int64_t real = 0;  // records excluding padding words
    for (size_t gg = g0; gg < g0 + ng; gg++) {
      const int64_t start = (int64_t)pl->records.size() / RW - rec_off;
      int64_t cnt = 0;
      for (int32_t c : gs[gg].cols) {
        if (c < lo_col || c > hi_col) continue;
        const size_t base = pl->records.size();
        pl->records.resize(base + RW, 0u);
        // generic: word 0 = byte offset of the staged row; mask records:
        // slot << 24 | row mask (the kernel's address is base + word >> 15)
        pl->records[base] = pl->uniform ? (uint32_t)slot_of[c] << 24
                                        : (uint32_t)slot_of[c] * (uint32_t)SPDNN_STAGED_ROW_BYTES;
        for (int k = 0; k < R; k++) {
          const int32_t row = gs[gg].rows[k];
          const float w = row >= 0 ? weight(row, c) : 0.0f;
          uint32_t bits;
          std::memcpy(&bits, &w, 4);
          // row k is mask bit k+1: the kernel turns bits 1..6 into predicates
          // with one R2P and bit 7 with one LOP3 (bit 0 would cost two ops)
          if (pl->uniform) pl->records[base] |= (bits != 0u ? 2u : 0u) << k;
          else pl->records[base + 1 + k] = bits;
        }
        cnt++;
      }
      // mask records: each group's run is stored padded to a multiple of 4
      // words (the kernel reads 4 records per 16-byte load, so every run
      // starts 16-byte aligned); the padding words are mask 0 and the
      // segment keeps the exact count, so the kernel skips them
      real += cnt;
      const int64_t exact = cnt;
      if (pl->uniform)
        while (cnt % 4) {
          pl->records.push_back(0u);
          cnt++;
        }
      if (gseg) {
        gseg->push_back((int32_t)start);
        gseg->push_back((int32_t)exact);
      }
    }
    const int64_t rec_cnt = (int64_t)pl->records.size() / RW - rec_off;
    pl->union_records += real;
    // keep every stage's records 16-byte aligned for the bulk copy (R = 1
    // records are 8 bytes): pad with an unreferenced zero record
    while ((pl->records.size() * 4) % 16) pl->records.push_back(0u);
    pl->max_rec = std::max<int32_t>(pl->max_rec, (int32_t)rec_cnt);
    pl->max_fp = std::max<int32_t>(pl->max_fp, (int32_t)(c_hi - c_lo));
    return std::make_pair(rec_off, rec_cnt);
  };

  size_t g = 0;
  std::vector<int32_t> gseg;
  while (g < gs.size()) {
    // ---- choose the block's groups
    const size_t g0 = g;
    fp_block.clear();
    int64_t recs = 0;
    while (g < gs.size() && (int64_t)(g - g0) < GMAX) {
      int64_t newc = 0;
      for (int32_t c : gs[g].cols) newc += (stamp[c] != blk_id);
      if (g > g0 && ((int64_t)fp_block.size() + newc > S ||
                     recs + (int64_t)gs[g].cols.size() > RC))
        break;
      for (int32_t c : gs[g].cols)
        if (stamp[c] != blk_id) { stamp[c] = blk_id; fp_block.push_back(c); }
      recs += (int64_t)gs[g].cols.size();
      g++;
    }
    const size_t ng = g - g0;
    pl->max_groups = std::max<int32_t>(pl->max_groups, (int32_t)ng);
    std::sort(fp_block.begin(), fp_block.end());
    const int64_t nfp = (int64_t)fp_block.size();
    // a block overflows the caps only when it is a lone group (loop above)
    const int64_t nst = (nfp > S || recs > RC) ? (nfp + S - 1) / S : 1;
    // ---- stage 0: descriptor + meta + records
    const int64_t c_hi0 = nst == 1 ? nfp : std::min<int64_t>(nfp, S);
    const int64_t meta_off = (int64_t)pl->meta.size();
    pl->meta.insert(pl->meta.end(), fp_block.begin(), fp_block.begin() + c_hi0);
    pad4(pl->meta);
    gseg.clear();
    auto r0 = emit_records(g0, ng, 0, c_hi0, &gseg);
    pl->meta.insert(pl->meta.end(), gseg.begin(), gseg.end());
    for (size_t gg = g0; gg < g0 + ng; gg++)
      for (int k = 0; k < R; k++) pl->meta.push_back(gs[gg].rows[k]);
    // bias slots, one per group row: zero here, filled with bias[row] when the
    // model is uploaded (the layout does not depend on the bias values)
    pl->meta.insert(pl->meta.end(), (size_t)R * ng, 0);
    pad4(pl->meta);
    pl->max_meta = std::max<int32_t>(pl->max_meta, (int32_t)(pl->meta.size() - meta_off));
    const int64_t first_extra = (int64_t)pl->stages.size() / 4;
    const int32_t desc[8] = {(int32_t)g0, (int32_t)ng, (int32_t)nst, (int32_t)first_extra,
                             (int32_t)meta_off, (int32_t)c_hi0, (int32_t)r0.first,
                             (int32_t)r0.second};
    pl->blocks.insert(pl->blocks.end(), desc, desc + 8);
    // ---- further stages of a lone oversized group
    for (int64_t st = 1; st < nst; st++) {
      const int64_t c_lo = st * S, c_hi = std::min<int64_t>(nfp, (st + 1) * S);
      const int64_t moff = (int64_t)pl->meta.size();
      pl->meta.insert(pl->meta.end(), fp_block.begin() + c_lo, fp_block.begin() + c_hi);
      pad4(pl->meta);
      auto r = emit_records(g0, ng, c_lo, c_hi, nullptr);
      const int32_t sd[4] = {(int32_t)moff, (int32_t)(c_hi - c_lo), (int32_t)r.first,
                             (int32_t)r.second};
      pl->stages.insert(pl->stages.end(), sd, sd + 4);
    }
    blk_id++;
  }
  if (pl->meta.size() >= ((size_t)1 << 31) || pl->records.size() / RW >= ((size_t)1 << 31))
    throw std::length_error("layer layout exceeds 2^31 entries");
}

}  // namespace

extern "C" int spdnn_plan_build(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                const float *values, const spdnn_plan_params *params,
                                spdnn_plan **out) {
  if (!out || !params || n < 0 || (n > 0 && !row_ptr) ||
      (n > 0 && row_ptr[n] > 0 && (!col_idx || !values)))
    return spdnn_fail(SPDNN_EINVAL, "spdnn_plan_build: null argument");
  *out = nullptr;
  spdnn_plan_params p = *params;
  if (p.footprint_cap < 1 || p.max_groups < 1 || p.record_cap < p.footprint_cap)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_plan_build: bad params");
  if (p.rows_per_group < 0 || p.rows_per_group == 2 || p.rows_per_group > 7)
    return spdnn_fail(SPDNN_EINVAL, "spdnn_plan_build: rows_per_group must be 0, 1 or 3..7");
  if (n > 0 && !valid_csr(n, row_ptr, col_idx))
    return spdnn_fail(SPDNN_EINVAL, "spdnn_plan_build: CSR is not canonical");
  if ((int64_t)p.footprint_cap * SPDNN_STAGED_ROW_BYTES >= (int64_t)1 << 31)
    return spdnn_fail(SPDNN_ERANGE, "spdnn_plan_build: footprint cap too large");
  spdnn_plan *pl = new (std::nothrow) spdnn_plan();
  if (!pl) return spdnn_fail(SPDNN_ENOMEM, "spdnn_plan_build: out of memory");
  pl->n = n;
  pl->nnz = n > 0 ? row_ptr[n] : 0;
  try {
    uint32_t wb = 0;
    if (p.uniform_records && p.footprint_cap <= 256 && uniform_weights(pl->nnz, values, wb)) {
      pl->uniform = 1;
      pl->weight_bits = wb;
    }
    std::vector<int32_t> ident(n);
    for (int64_t i = 0; i < n; i++) ident[i] = (int32_t)i;
    int R = p.rows_per_group;
    std::vector<Group> best;
    if (R == 1 || n == 0) {
      R = 1;
      best = make_groups(n, row_ptr, col_idx, ident, 1);
    } else {
      std::vector<int32_t> order = p.reorder ? class_overlap_order(n, row_ptr, col_idx) : ident;
      if (R != 0) {
        best = make_groups(n, row_ptr, col_idx, order, R);
      } else {
        double best_cost = 0;
        const int top = pl->uniform && n >= kR6MinRows ? 6 : 7;
        for (int cand : {1, 3, top}) {
          auto gs = make_groups(n, row_ptr, col_idx, cand == 1 ? ident : order, cand);
          double cost = (double)total_records(gs) *
                        (pl->uniform ? mask_record_cost(cand) : record_cost(cand));
          if (best.empty() && cand == 1) { best = std::move(gs); R = 1; best_cost = cost; continue; }
          if (cost < best_cost) { best = std::move(gs); R = cand; best_cost = cost; }
        }
      }
    }
    pl->R = R;
    pl->RW = record_words(R, pl->uniform != 0);
    pl->num_groups = (int64_t)best.size();
    pl->pow2 = pow2_weights(pl->nnz, values, pl->wexp_min, pl->wexp_max) ? 1 : 0;
    emit(pl, row_ptr, col_idx, values, best, fit_caps(p, R, pl->RW));
  } catch (const std::bad_alloc &) {
    delete pl;
    return spdnn_fail(SPDNN_ENOMEM, "spdnn_plan_build: out of memory");
  } catch (const std::length_error &) {
    delete pl;
    return spdnn_fail(SPDNN_ERANGE, "spdnn_plan_build: layer layout exceeds 2^31 entries");
  }
  *out = pl;
  return SPDNN_OK;
}

extern "C" int spdnn_plan_build_many(int64_t num_layers, int64_t n,
                                     const int64_t *const *row_ptr,
                                     const int32_t *const *col_idx,
                                     const float *const *values,
                                     const spdnn_plan_params *params, int32_t threads,
                                     spdnn_plan **out) {
  if (num_layers < 0 || !out) return spdnn_fail(SPDNN_EINVAL, "spdnn_plan_build_many: bad args");
  for (int64_t l = 0; l < num_layers; l++) out[l] = nullptr;
  if (threads < 1) threads = 1;
  std::vector<int> rc(num_layers, 0);
  std::vector<std::string> msg(num_layers);
  std::vector<std::thread> pool;
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      int64_t l = next.fetch_add(1);
      if (l >= num_layers) break;
      rc[l] = spdnn_plan_build(n, row_ptr[l], col_idx[l], values[l], params, &out[l]);
      if (rc[l]) msg[l] = spdnn_last_error();  // thread-local: copy before leaving
    }
  };
  int nt = (int)std::min<int64_t>(threads, std::max<int64_t>(num_layers, 1));
  for (int t = 1; t < nt; t++) pool.emplace_back(worker);
  worker();
  for (auto &th : pool) th.join();
  for (int64_t l = 0; l < num_layers; l++)
    if (rc[l] != 0) {
      for (int64_t k = 0; k < num_layers; k++) { spdnn_plan_free(out[k]); out[k] = nullptr; }
      std::string m = "layer " + std::to_string(l) + ": " + msg[l];
      return spdnn_fail(rc[l], m.c_str());
    }
  return SPDNN_OK;
}

extern "C" int spdnn_plan_sizes(const spdnn_plan *pl, spdnn_plan_sizes_t *s) {
  if (!pl || !s) return spdnn_fail(SPDNN_EINVAL, "spdnn_plan_sizes: null argument");
  s->neurons = pl->n;
  s->rows_per_group = pl->R;
  s->record_words = pl->RW;
  s->num_blocks = (int64_t)pl->blocks.size() / 8;
  s->num_extra_stages = (int64_t)pl->stages.size() / 4;
  s->num_groups = pl->num_groups;
  s->num_meta = (int64_t)pl->meta.size();
  s->num_records = (int64_t)pl->records.size() / pl->RW;
  s->num_fp = 0;
  for (size_t b = 0; b < pl->blocks.size(); b += 8) s->num_fp += pl->blocks[b + 5];
  for (size_t st = 0; st < pl->stages.size(); st += 4) s->num_fp += pl->stages[st + 1];
  s->nnz = pl->nnz;
  s->padded_slots = pl->union_records * pl->R;
  s->max_fp_per_stage = pl->max_fp;
  s->max_records_per_stage = pl->max_rec;
  s->max_meta_per_block = pl->max_meta;
  s->max_groups_per_block = pl->max_groups;
  s->pow2 = pl->pow2;
  s->wexp_min = pl->wexp_min;
  s->wexp_max = pl->wexp_max;
  s->uniform = pl->uniform;
  s->weight_bits = pl->weight_bits;
  return SPDNN_OK;
}

extern "C" int spdnn_plan_export(const spdnn_plan *pl, int32_t *blocks, int32_t *stages,
                                 int32_t *meta, uint32_t *records) {
  if (!pl) return spdnn_fail(SPDNN_EINVAL, "spdnn_plan_export: null plan");
  auto cp = [](auto *dst, const auto &v) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(blocks, pl->blocks);
  cp(stages, pl->stages);
  cp(meta, pl->meta);
  cp(records, pl->records);
  return SPDNN_OK;
}

extern "C" void spdnn_plan_free(spdnn_plan *pl) { delete pl; }
