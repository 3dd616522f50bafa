// Weight-streaming tensor-core GEMM for decode batches (bf16 mode, 2 <= B <= 256):
//
//   part[s, b, n] = sum_{k in range s} W[n, k] X[b, k]        (f32 split-K partials)
//
// The operands are swapped against tc_gemm: the weight rows are the UMMA M side
// (128 per tile) and the batch rows the N side (BNB = B rounded up to 16 .. 256),
// so a k-block stages a 16 KB weight tile and only BNB x 128 B of activations —
// tc_gemm's 128-row activation tile (mostly zero padding at small B) would
// double the shared-memory fill per weight byte.  One work unit per CTA =
// (128 weight rows) x (one K range); the host picks the split so that the units
// cover the SMs.  The weight tiles of the first STAGES k-blocks are requested
// before griddepcontrol.wait (weights do not depend on the predecessor).
//
// Warps: 0 TMA producer, 1 TMEM allocator + single-thread tcgen05.mma issuer,
// 2..5 epilogue (one TMEM lane quarter each: lane = weight row, column = batch
// row; every store instruction writes 32 consecutive outputs of one batch row).
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace ssd200 {

// SMALL: a ~100 KB ring so that two CTAs (this GEMM's and the next kernel's)
// can share an SM and the next one's weight prefetch overlaps this one's tail
// (104 KB: 5 stages at BNB <= 32; B = 32 2.22 -> 2.19 ms vs 96 KB, 110 KB (6
// stages at BNB = 16) moved B = 1 / B = 8 by -1 % / +1 %)
#ifndef SSD200_DEC_SMALL_KB
#define SSD200_DEC_SMALL_KB 104u
#endif
template <int BNB, bool SMALL = false> struct DgCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr uint32_t A_BYTES = BM * BK * 2;   // 16 KB weight tile
  static constexpr uint32_t B_BYTES = BNB * BK * 2;  // activation tile
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t BUDGET = SMALL ? SSD200_DEC_SMALL_KB * 1024u : 192u * 1024u;
  static constexpr int STAGES = (int)(BUDGET / STAGE_BYTES) > 8 ? 8 : (int)(BUDGET / STAGE_BYTES);
  static constexpr int TMEM_COLS = BNB < 32 ? 32 : BNB;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
};

struct DgArgs {
  int N, K, B;        // weight rows, reduction length, batch rows
  int ksplit;
  float *out;         // (ksplit, B, ldo)
  long ldo, split_stride;
  unsigned *zero_ctr;  // in_proj: the state stream's chunk counter, zeroed after the wait
  int trace;          // launch-timeline slot (SSD200_TRACE builds), -1 = none
};

template <int BNB, bool SMALL = false>
__global__ void __launch_bounds__(192, 1)
    dec_gemm_swap(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                  DgArgs a) {
  using Cfg = DgCfg<BNB, SMALL>;
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  if (threadIdx.x == 0) SSD200_TRACE_MARK(a.trace, 0);
  uint8_t *smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = smem;
  uint8_t *sB = smem + STAGES * Cfg::A_BYTES;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tdone;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = (a.N + 127) / 128;
  const int n_blk = blockIdx.x % ntn, ks = blockIdx.x / ntn;
  const int num_kb = (a.K + BK - 1) / BK;
  const int kb0 = ks * num_kb / a.ksplit, kb1 = (ks + 1) * num_kb / a.ksplit;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmW);
    sm100::tma_prefetch(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(&tdone, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<Cfg::TMEM_COLS>(&tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  griddep_launch();  // the next kernel's CTAs may take SMs as ours retire

  if (warp == 0) {
    if (lane == 0) {
      // weight tiles of the first STAGES k-blocks before the dependency wait
      const int pre = min(STAGES, kb1 - kb0);
      for (int i = 0; i < pre; ++i) {
        sm100::mbar_arrive_expect_tx(&full[i], Cfg::STAGE_BYTES);
        sm100::tma_load_2d(sA + i * Cfg::A_BYTES, &tmW, &full[i], (kb0 + i) * BK, n_blk * 128);
      }
      griddep_wait();  // X comes from the predecessor (and out is free once it is done)
      SSD200_TRACE_MARK(a.trace, 1);
      if (a.zero_ctr && blockIdx.x == 0) *a.zero_ctr = 0u;
      for (int i = 0; i < pre; ++i)
        sm100::tma_load_2d(sB + i * Cfg::B_BYTES, &tmX, &full[i], (kb0 + i) * BK, 0);
      int s = pre % STAGES;
      uint32_t ph = pre == STAGES ? 1u : 0u;
      for (int kb = kb0 + pre; kb < kb1; ++kb) {
        sm100::mbar_wait(&empty[s], ph ^ 1);
        sm100::mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        sm100::tma_load_2d(sA + s * Cfg::A_BYTES, &tmW, &full[s], kb * BK, n_blk * 128);
        sm100::tma_load_2d(sB + s * Cfg::B_BYTES, &tmX, &full[s], kb * BK, 0);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_bf16(128, BNB, false, false);
      int s = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        sm100::mbar_wait(&full[s], ph);
        sm100::tc_fence_after();
        const uint32_t a0 = sm100::smem_u32(sA + s * Cfg::A_BYTES);
        const uint32_t b0 = sm100::smem_u32(sB + s * Cfg::B_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = sm100::sw128_desc(a0 + k * 32, 16, 1024);
          const uint64_t bd = sm100::sw128_desc(b0 + k * 32, 16, 1024);
          sm100::mma_bf16(tmem, ad, bd, idesc, (kb != kb0) || (k != 0));
        }
        sm100::mma_commit(&empty[s]);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      sm100::mma_commit(&tdone);
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 (weight rows)
    const int q = warp & 3;
    const int n = n_blk * 128 + q * 32 + lane;
    float *dst = a.out + (size_t)ks * a.split_stride + n;
    sm100::mbar_wait(&tdone, 0);
    sm100::tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    if constexpr (BNB == 16) {
      uint32_t r[16];
      sm100::tmem_ld16(trow, r);
      sm100::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < a.B && n < a.N) dst[(size_t)j * a.ldo] = __uint_as_float(r[j]);
    } else {
#pragma unroll 1
      for (int c0 = 0; c0 < BNB; c0 += 32) {
        if (c0 >= a.B) break;  // warp-uniform
        uint32_t r[32];
        sm100::tmem_ld32(trow + c0, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < a.B && n < a.N) dst[(size_t)(c0 + j) * a.ldo] = __uint_as_float(r[j]);
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    sm100::tc_fence_after();
    sm100::tmem_dealloc<Cfg::TMEM_COLS>(tmem);
  }
  if (threadIdx.x == 0) SSD200_TRACE_MARK(a.trace, 2);
}

}  // namespace ssd200
