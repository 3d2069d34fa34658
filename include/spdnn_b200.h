/*
 * spdnn_b200.h -- C ABI of the B200 sparse-DNN inference path
 * (libspdnn_b200.so, built from paper_2007_14152_b200/csrc/).
 *
 * Plain pointers and sizes only. Device pointers are CUDA global-memory
 * addresses (the Python host layer allocates them with torch, but nothing
 * here depends on torch); `stream` is a cudaStream_t passed as void*.
 * Every entry point returns 0 on success and a nonzero SPDNN_E* code on
 * failure; spdnn_last_error() returns the message for the calling thread.
 * Entry points are reentrant: no global mutable state, one host thread per
 * device is the intended use (the reference calls its kernels concurrently
 * from worker threads, spdnn/parallel.py:302, tests/test_engine.py:264-287).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/spdnn/):
 *
 *   spdnn_plan_build / _sizes / _export / _free
 *       replace preprocess.build_staging_plan (preprocess.py:148-190) +
 *       csr_to_sliced_ell (preprocess.py:212-244) as called by
 *       engine.prepare_layer (engine.py:77-85): one-time host conversion of a
 *       CSR layer into the B200 layout ("row-grouped union ELL").
 *   spdnn_layer_forward
 *       replaces kernels.staged_fused_relu (kernels.py:40-88) as called by
 *       engine.optimized_layer (engine.py:109-127), fused with the activity
 *       test `(out > 0).any(axis=0)` (engine.py:127) and the stable
 *       compaction of engine.compact_active (engine.py:130-142).
 *   spdnn_transpose_in / spdnn_gather_out
 *       the FeatureBatch <-> device layout conversions around the loop
 *       (FeatureBatch data is (N, M) Fortran, model.py:82-114).
 *   spdnn_infer_layers
 *       replaces the layer loop of engine.infer (engine.py:235-290): all
 *       layers enqueued on one stream, device-side active counts, no host
 *       synchronisation inside the loop.
 */
#ifndef SPDNN_B200_H
#define SPDNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SPDNN_OK = 0,
  SPDNN_EINVAL = 1,   /* bad argument (the Python layer maps this to ModelError) */
  SPDNN_ECUDA = 2,    /* CUDA runtime error */
  SPDNN_ENOMEM = 3,
  SPDNN_ERANGE = 4    /* index exceeds the layout's range */
};

/* Feature-tile width: every work item covers 128 active features
 * (32 lanes x 4 fp32 features, two f32x2 register pairs per lane). One staged
 * input neuron is therefore a 512-byte shared-memory row. */
#define SPDNN_TILE_FEATURES 128
#define SPDNN_STAGED_ROW_BYTES 512

/* ---- one-time layout conversion (host, C++) ----------------------------- */

typedef struct spdnn_plan_params {
  int32_t rows_per_group;   /* R in {1, 3, 4, 5, 6, 7}; 0 = choose per layer */
  int32_t footprint_cap;    /* max input neurons staged per block stage */
  int32_t max_groups;       /* max row groups per block (<= warps per CTA) */
  int32_t record_cap;       /* max union records staged per block stage */
  int32_t reorder;          /* 1 = order rows by column overlap, 0 = identity */
  int32_t uniform_records;  /* 1 = when every stored weight has the same nonzero
                               bits, one-word mask records (see export) */
} spdnn_plan_params;

typedef struct spdnn_plan spdnn_plan; /* opaque host plan for one layer */

/* Sizes of the exported arrays plus padding statistics. */
typedef struct spdnn_plan_sizes_t {
  int64_t neurons;
  int32_t rows_per_group;   /* R actually used */
  int32_t record_words;     /* 32-bit words per union record (1, 2, 4 or 8) */
  int64_t num_blocks;
  int64_t num_extra_stages; /* stages beyond the first of multi-stage blocks */
  int64_t num_groups;
  int64_t num_meta;         /* int32 words of per-block metadata */
  int64_t num_records;      /* records array length (union records + 16-byte
                               alignment padding of R = 1 stages) */
  int64_t num_fp;           /* staged input neurons, summed over all stages */
  int64_t nnz;
  int64_t padded_slots;     /* union records * R: multiply-add slots per feature */
  int32_t max_fp_per_stage;
  int32_t max_records_per_stage;
  int32_t max_meta_per_block;
  int32_t max_groups_per_block;
  int32_t pow2;             /* 1: every nonzero weight is +-2^e (FMA form allowed) */
  int32_t wexp_min;         /* exponent range of the nonzero weights */
  int32_t wexp_max;
  int32_t uniform;          /* 1: mask records, every nonzero weight == weight_bits */
  uint32_t weight_bits;
} spdnn_plan_sizes_t;

/* Build the plan for one CSR layer (canonical CSR as in model.py:35-58).
 * Returns SPDNN_EINVAL on malformed CSR. */
int spdnn_plan_build(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                     const float *values, const spdnn_plan_params *params,
                     spdnn_plan **out);
/* Build plans for many layers on `threads` host threads. */
int spdnn_plan_build_many(int64_t num_layers, int64_t n,
                          const int64_t *const *row_ptr,
                          const int32_t *const *col_idx,
                          const float *const *values,
                          const spdnn_plan_params *params, int32_t threads,
                          spdnn_plan **out);
int spdnn_plan_sizes(const spdnn_plan *plan, spdnn_plan_sizes_t *sizes);
/* Copy the plan into caller-owned host buffers sized from spdnn_plan_sizes:
 *   blocks  int32[num_blocks * 8]  {g_first, ng, nst, first_extra_stage,
 *                                   meta_off, fp_cnt, rec_off, rec_cnt}
 *                                   (meta/records of the block's first stage)
 *   stages  int32[num_extra_stages * 4] {meta_off, fp_cnt, rec_off, rec_cnt}
 *           (a block with nst > 1 holds exactly one group)
 *   meta    int32[num_meta]: per block, 16-byte aligned:
 *           fp_cnt input neurons (smem slot order), pad to 4,
 *           ng x {record offset relative to rec_off, record count},
 *           ng x R output neurons (-1 = padding row),
 *           ng x R bias slots (fp32 bits; 0 from the builder, bias[row] once
 *           the model is on the device -- filled by the host layer), pad to 4
 *   records uint32[num_records * record_words]
 *           word 0 = smem byte offset of the input neuron's staged row
 *           (slot * SPDNN_STAGED_ROW_BYTES), words 1..R = fp32 weight bits
 *           per group row (0 = not connected); per group ascending neuron.
 *           Uniform layers (sizes.uniform): one word per record,
 *           slot << 24 | mask << 1 (bit k+1 = group row k connects; the
 *           weight is sizes.weight_bits), each group's run padded with zero
 *           words to a multiple of 4
 */
int spdnn_plan_export(const spdnn_plan *plan, int32_t *blocks, int32_t *stages,
                      int32_t *meta, uint32_t *records);
void spdnn_plan_free(spdnn_plan *plan);

/* ---- device execution ---------------------------------------------------- */

/* Device-resident plan of one layer (pointers into device memory). */
typedef struct spdnn_layer_dev {
  const int32_t *blocks;
  const int32_t *stages;
  const int32_t *meta;
  const uint32_t *records;
  int64_t num_blocks;
  int64_t neurons;          /* N: rows of the feature buffers */
  int32_t rows_per_group;
  int32_t record_words;
  int32_t max_fp_per_stage;
  int32_t max_records_per_stage;
  int32_t max_meta_per_block;
  int32_t max_groups_per_block;  /* work units (row groups) per item */
  int32_t uniform;               /* mask records (record_words == 1) */
  uint32_t weight_bits;          /* the weight of every connection when uniform */
} spdnn_layer_dev;

/* Per-inference scratch shared by every layer launch (device pointers). */
typedef struct spdnn_scratch {
  int32_t *tile_done;      /* [ceil(M_cap/64)] zero-initialised */
  uint32_t *tile_alive;    /* [ceil(M_cap/32)] zero-initialised (one bit per feature) */
  int32_t *work;           /* [num_layers] zero-initialised work counters */
  uint32_t *guard;         /* [1] zero-initialised; bit 0 = FMA-form guard
                              tripped (rerun in the exact form), bit 1 =
                              non-finite input (rerun with one row per group) */
  int32_t *split;          /* optional (NULL: off) [2 * (num_layers + 1)] zero-
                              initialised: between the layers of one
                              spdnn_infer_layers call, a tile whose 128 features
                              all survive is appended as a whole aligned tile and
                              the other survivors are packed from entry ld on,
                              so one death does not shift every later tile off
                              its consecutive columns (the TMA staging path);
                              the a0/a1/cat0/cat1 buffers must then hold 2 * ld
                              entries. The last layer's survivors are packed. */
} spdnn_scratch;

/* Arithmetic form of a launch (layer.cu):
 *   fma_form = 0 : exact form, any weights: p = fl(y*w) then acc = fl(acc+p)
 *   fma_form = 1 : acc = fma(y, w, acc); bit-identical when y*w is exact,
 *                  i.e. all weights +-2^e and no input in (0, tiny) --
 *                  tiny = 2^(-126 - min weight exponent); outputs below it
 *                  set guard bit 0 (the next layer would not be exact). */
typedef struct spdnn_run_opts {
  int32_t fma_form;
  float tiny;
  int32_t features_per_lane; /* 4 (default, 128-feature items) or 2 (64-feature
                                items, twice the resident consumer warps) */
} spdnn_run_opts;

/* One layer over the active features (engine.run_layer_step, engine.py:145-170):
 *   y_in   : float[N][ld]   neuron-major, the active feature j lives in column
 *            a_in[j], j < *m_in
 *   y_out  : float[N][ld]   output for active feature j in column j
 *   a_out / cat_out : surviving output columns and their categories, appended
 *            tile by tile (order across tiles is not fixed; categories are
 *            sorted once at the end, as the reference sorts, parallel.py:427)
 *   *m_out : incremented by the number of survivors (caller zeroes it)
 * `work` points at this launch's zeroed work counter. */
int spdnn_layer_forward(const spdnn_layer_dev *layer, const float *bias,
                        const float *y_in, float *y_out, int64_t ld,
                        const int32_t *a_in, const int64_t *cat_in,
                        const int32_t *m_in, int32_t *a_out, int64_t *cat_out,
                        int32_t *m_out, const spdnn_scratch *scratch,
                        int32_t *work, const spdnn_run_opts *opts, void *stream);

/* All layers back to back on `stream` (engine.infer's loop, engine.py:264-285).
 * Buffers ping-pong between index 0 and 1; counts[l] = active features
 * entering layer l (counts[0] must hold M_0; counts[1..L] zeroed by caller).
 * The final state is in buffer (num_layers % 2). */
int spdnn_infer_layers(int64_t num_layers, const spdnn_layer_dev *layers,
                       const float *bias, float *y0, float *y1, int64_t ld,
                       int32_t *a0, int32_t *a1, int64_t *cat0, int64_t *cat1,
                       int32_t *counts, const spdnn_scratch *scratch,
                       const spdnn_run_opts *opts, void *stream);

/* spdnn_infer_layers with a cudaEvent_t recorded on `stream` before every
 * layer (events[l]) and after the last (events[num_layers]): per-layer device
 * times without host round trips between launches (measurement). */
int spdnn_infer_layers_timed(int64_t num_layers, const spdnn_layer_dev *layers,
                             const float *bias, float *y0, float *y1, int64_t ld,
                             int32_t *a0, int32_t *a1, int64_t *cat0, int64_t *cat1,
                             int32_t *counts, const spdnn_scratch *scratch,
                             const spdnn_run_opts *opts, void *stream, void *const *events);

/* x: float[m][n] feature-major (FeatureBatch.data bytes) -> y: float[n][ld].
 * If guard != NULL: bit 0 |= some 0 < |x| < tiny or |x| > huge, bit 1 |= some
 * x is NaN or inf. */
int spdnn_transpose_in(const float *x, int64_t n, int64_t m, float *y,
                       int64_t ld, uint32_t *guard, float tiny, float huge,
                       void *stream);
/* out[k][:] = y[:, a[perm[k]]] for k < m (feature-major result, i.e. the
 * (N, m) Fortran FeatureBatch layout). perm may be NULL (identity). */
int spdnn_gather_out(const float *y, int64_t n, int64_t ld, const int32_t *a,
                     const int64_t *perm, int64_t m, float *out, void *stream);

/* Cycle accounting of the layer kernel when the library was built with
 * -DSPDNN_PROFILE (all zero otherwise): out[0..7] consumer-warp clock64 sums
 * (wait for data, record loop, epilogue, bookkeeping), out[8..15] producer
 * warps (empty-slot wait, barrier A, copy issue, metadata, barrier B, tail),
 * out[16..21] ring-entry chain sums (issue, fill, consume, release, entries,
 * releases). n <= 24. Diagnostics only. */
int spdnn_profile_read(uint64_t *out, int32_t n, int32_t reset);

/* Per-ring-entry clock64 timeline of CTA 0 of the last layer launches, when
 * the library was built with -DSPDNN_TRACE (zero otherwise): out[12*k + i]
 * for entry k < 96 (layer.cu, g_trace). n <= 1152. Diagnostics only. */
int spdnn_trace_read(int64_t *out, int32_t n);

/* Per-launch, per-CTA %globaltimer marks of the last 64 layer launches, when
 * built with -DSPDNN_LTRACE (layer.cu, g_ltrace): out[(slot*160 + cta)*6 + i],
 * slot = launch index % 64. n <= 61440. Diagnostics only. */
int spdnn_ltrace_read(int64_t *out, int32_t n);

/* Threadblocks per SM the layer kernel runs with (for diagnostics). */
int spdnn_layer_occupancy(int32_t rows_per_group, int32_t *ctas_per_sm,
                          int32_t *threads_per_cta);

const char *spdnn_last_error(void);
const char *spdnn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPDNN_B200_H */
