// Staging-path microbenchmark: how fast can one SM fill shared-memory slots
// with R random 512-byte feature-row segments (the layer kernel's per-item
// staging), by TMA gather4, by TMA bulk copies per row, or by 16-byte
// cp.async from all producer threads? A consumer warp releases each slot as
// soon as it lands, so the result is the staging rate alone.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tma_bench.cu -lcuda
//   ./tma_bench
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("err %s line %d\n", cudaGetErrorString(e), __LINE__);         \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

constexpr int kRowB = 512;

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra W_%=;\n}\n" ::"r"(bar), "r"(parity), "r"(1000000) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t sdst, const CUtensorMap *tmap, int col,
                                            int r0, int r1, int r2, int r3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(sdst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t sdst, const void *gsrc, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(sdst), "l"(gsrc), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void cp16(uint32_t s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}

// mode 0: gather4 (P producer warps, lane-dealt), 1: bulk per row, 2: cp.async 16 B
template <int P>
__global__ void __launch_bounds__((P + 1) * 32, 1)
    stage(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmb,
          int br, const float *y, int ld, int nrows_src,
          int rows, int nslot, int items, int mode, unsigned long long *cycles) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t f0 = (uint32_t)__cvta_generic_to_shared(&full[0]);
  const uint32_t e0 = (uint32_t)__cvta_generic_to_shared(&empty[0]);
  const int slot_b = rows * kRowB;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslot; i++) {
      mbar_init(f0 + 8 * i, mode == 2 ? P * 32 + 1 : 1);
      mbar_init(e0 + 8 * i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp < P) {
    const int ptid = warp * 32 + lane;
    unsigned h = blockIdx.x * 2654435761u + 12345u;
    for (int k = 0; k < items; k++) {
      const int s = k % nslot;
      const uint32_t ph = (k / nslot) & 1;
      mbar_wait(e0 + 8 * s, ph ^ 1);
      const uint32_t dst = sb + s * slot_b;
      const int col = ((h >> 8) % (ld / 128)) * 128;
      if (mode == 0) {
        if (ptid == 0) mbar_expect_tx(f0 + 8 * s, slot_b);
        asm volatile("bar.sync 1, %0;\n" ::"n"(P * 32));
        const int qd = lane * P + warp;
        if (qd < rows / 4) {
          unsigned r = h ^ (qd * 0x9E3779B9u);
          int rr[4];
          for (int j = 0; j < 4; j++) {
            r = r * 1664525u + 1013904223u;
            rr[j] = (r >> 4) % nrows_src;
          }
          tma_gather4(dst + qd * 4 * kRowB, &tm, col, rr[0], rr[1], rr[2], rr[3], f0 + 8 * s);
        }
      } else if (mode == 3) {
        // rows consecutive tensor rows from a random start: 2-D tile boxes of
        // br rows x 128 columns, dealt lane-major over the producer warps
        const int nbox = (rows + br - 1) / br;
        if (ptid == 0) mbar_expect_tx(f0 + 8 * s, nbox * br * kRowB);
        asm volatile("bar.sync 1, %0;\n" ::"n"(P * 32));
        const int r0 = (int)((h >> 4) % (unsigned)(nrows_src - rows - br));
        const int bx = lane * P + warp;
        if (bx < nbox) {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst + bx * br * kRowB),
              "l"(reinterpret_cast<uint64_t>(&tmb)), "r"(col), "r"(r0 + bx * br), "r"(f0 + 8 * s)
              : "memory");
        }
      } else if (mode == 1) {
        if (ptid == 0) mbar_expect_tx(f0 + 8 * s, slot_b);
        asm volatile("bar.sync 1, %0;\n" ::"n"(P * 32));
        for (int q = ptid; q < rows; q += P * 32) {
          unsigned r = (h ^ (q * 0x9E3779B9u)) * 1664525u + 1013904223u;
          const float *src = y + (size_t)((r >> 4) % nrows_src) * ld + col;
          bulk_g2s(dst + q * kRowB, src, kRowB, f0 + 8 * s);
        }
      } else {
        for (int q = warp; q < rows; q += P) {
          unsigned r = (h ^ (q * 0x9E3779B9u)) * 1664525u + 1013904223u;
          const float *src = y + (size_t)((r >> 4) % nrows_src) * ld + col;
          cp16(dst + q * kRowB + 16 * lane, src + 4 * lane);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(f0 + 8 * s)
                     : "memory");
        if (ptid == 0) mbar_arrive(f0 + 8 * s);
      }
      h = h * 747796405u + 2891336453u;
    }
  } else {
    for (int k = 0; k < items; k++) {
      const int s = k % nslot;
      mbar_wait(f0 + 8 * s, (k / nslot) & 1);
      if (lane == 0) mbar_arrive(e0 + 8 * s);
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int ld = 60032, nrows_big = 4096 * 4;  // 16384 x 60032 fp32 = 3.9 GB
  float *y;
  CK(cudaMalloc(&y, (size_t)nrows_big * ld * 4));
  CK(cudaMemset(y, 0, (size_t)nrows_big * ld * 4));
  unsigned long long *cyc;
  CK(cudaMalloc(&cyc, 8));
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap tm, tmb[3];
  const int brs[3] = {8, 32, 64};
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)nrows_big};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {128, 1}, es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("tensor map failed\n");
    return 1;
  }
  for (int i = 0; i < 3; i++) {
    cuuint32_t bb[2] = {128, (cuuint32_t)brs[i]};
    if (enc(&tmb[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, bb, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("box tensor map failed\n");
      return 1;
    }
  }
  printf("mode        br  rows slots srcrows   GB/s(all SMs)  B/clk/SM\n");
  struct Case { int mode, bri, rows, nslot, src; };
  std::vector<Case> cases;
  for (int rows : {136, 168})
    for (int nslot : {2, 3}) {
      cases.push_back({0, 0, rows, nslot, nrows_big});
      for (int bi = 0; bi < 3; bi++) cases.push_back({3, bi, rows, nslot, nrows_big});
      cases.push_back({2, 0, rows, nslot, nrows_big});
    }
  for (int rows : {168}) {
    cases.push_back({0, 0, rows, 2, 256 * 4});
    cases.push_back({3, 0, rows, 2, 256 * 4});
  }
  for (const Case &cs : cases) {
    const int br = brs[cs.bri];
    const int srows = cs.mode == 3 ? (cs.rows + br - 1) / br * br : (cs.rows + 3) / 4 * 4;
    const size_t sm_b = (size_t)srows * kRowB * cs.nslot;
    if (sm_b > 220 * 1024) continue;
    auto fn = stage<4>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_b));
    const int items = 400;
    // slot stride = srows rows (the kernel uses rows * kRowB as the slot size)
    fn<<<sms, 160, sm_b>>>(tm, tmb[cs.bri], br, y, ld, cs.src, srows, cs.nslot, 20, cs.mode, cyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(cyc, 0, 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    fn<<<sms, 160, sm_b>>>(tm, tmb[cs.bri], br, y, ld, cs.src, srows, cs.nslot, items, cs.mode, cyc);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    const double bytes = (double)sms * items * srows * kRowB;
    const char *nm = cs.mode == 0 ? "gather4" : (cs.mode == 3 ? "box" : "cp.async16");
    printf("%-10s %3d %5d %5d %7d   %10.1f   %8.2f\n", nm, cs.mode == 3 ? br : 4, srows,
           cs.nslot, cs.src, bytes / ms / 1e6, (double)items * srows * kRowB / ((double)c / sms));
  }
  return 0;
}
