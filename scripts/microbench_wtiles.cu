// Weight-streaming microbenchmark for the decode GEMMs (B200): the same grid and
// ring as dec_gemm_swap at 1.3B, B = 1 (67 weight-row tiles x 4 K ranges = 268
// CTAs, ~96 KB ring, two CTAs per SM), streaming W_in (8512 x 2048 bf16) with
//   (a) 2-D TMA boxes of 128 rows x 64 columns from the row-major matrix
//       (what the decode GEMM does: 128-byte row segments 4 KB apart), or
//   (b) 1-D bulk copies of 16 KB tiles from a tile-major copy (each 128 x 64
//       tile contiguous, a CTA's K range one contiguous 128 KB run).
// No math: the consumer just releases stages.  Prints GB/s per variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_09555_b200/csrc \
//      -o /tmp/mbw scripts/microbench_wtiles.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace ssd200;

constexpr int N = 8512, K = 2048, BM = 128, BK = 64, MAXSTAGES = 12;
constexpr uint32_t TILE = BM * BK * 2;  // 16 KB

template <bool TILED>
__global__ void __launch_bounds__(64) stream(const __grid_constant__ CUtensorMap tm,
                                             const uint8_t *tiled, float *sink, int STAGES,
                                             int KSPLIT) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[MAXSTAGES], empty[MAXSTAGES];
  const int ntn = N / BM + (N % BM ? 1 : 0);
  const int n_blk = blockIdx.x % ntn, ks = blockIdx.x / ntn;
  const int nkb = K / BK, kb0 = ks * nkb / KSPLIT, kb1 = (ks + 1) * nkb / KSPLIT;
  if (blockIdx.x >= ntn * KSPLIT) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      sm100::mbar_wait(&empty[s], ph ^ 1);
      sm100::mbar_arrive_expect_tx(&full[s], TILE);
      if (TILED) {
        const uint8_t *src = tiled + ((size_t)n_blk * nkb + kb) * TILE;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(sm100::smem_u32(sm + s * TILE)), "l"(src), "r"(TILE),
            "r"(sm100::smem_u32(&full[s])) : "memory");
      } else {
        sm100::tma_load_2d(sm + s * TILE, &tm, &full[s], kb * BK, n_blk * BM);
      }
      if (++s == STAGES) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    float acc = 0.f;
    for (int kb = kb0; kb < kb1; ++kb) {
      sm100::mbar_wait(&full[s], ph);
      acc += *reinterpret_cast<const float *>(sm + s * TILE + (kb & 63) * 4);
      sm100::mbar_arrive(&empty[s]);
      if (++s == STAGES) {
        s = 0;
        ph ^= 1;
      }
    }
    if (acc == 1.2345f) sink[0] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  const size_t bytes = (size_t)N * K * 2;
  const int ntn = N / BM + 1;
  uint8_t *w, *tiled;
  float *sink;
  cudaMalloc(&w, bytes);
  cudaMalloc(&tiled, (size_t)ntn * K / BK * TILE);
  cudaMalloc(&sink, 4);
  cudaMemset(w, 1, bytes);
  cudaMemset(tiled, 1, (size_t)ntn * K / BK * TILE);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {BK, BM}, es[2] = {1, 1};
  ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(stream<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(stream<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  // flush buffer larger than L2 between iterations
  uint8_t *flush;
  const size_t fb = 512ull << 20;
  cudaMalloc(&flush, fb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // (stages, k-split): smem per CTA = stages x 16 KB; CTAs per SM follow from it
  const int cfgs[][2] = {{5, 4}, {5, 8}, {3, 8}, {2, 16}, {3, 16}, {10, 2}, {12, 4}, {6, 4}, {4, 8}};
  for (auto &c : cfgs) {
    const int stages = c[0], ksplit = c[1];
    const size_t smem = stages * TILE + 1024;
    const int grid = ntn * ksplit;
    for (int tiledv = 0; tiledv < 2; ++tiledv) {
      float tot = 0.f;
      const int iters = 30;
      for (int it = 0; it < iters; ++it) {
        cudaMemsetAsync(flush, it, fb);
        cudaEventRecord(a);
        if (tiledv)
          stream<true><<<grid, 64, smem>>>(tm, tiled, sink, stages, ksplit);
        else
          stream<false><<<grid, 64, smem>>>(tm, tiled, sink, stages, ksplit);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        tot += ms;
      }
      const double us = tot / iters * 1e3;
      printf("stages %2d ksplit %2d grid %4d smem %3zu KB  %-22s %8.2f us  %7.0f GB/s\n", stages,
             ksplit, grid, smem >> 10, tiledv ? "tile-major 1-D bulk" : "row-major 2-D TMA", us,
             bytes / (us * 1e3));
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
