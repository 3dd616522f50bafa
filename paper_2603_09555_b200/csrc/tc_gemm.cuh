// Persistent bf16 tensor-core GEMM for sm_100a:  D (M,N) = A (M,K) . B (N,K)^T
// with fp32 accumulation in TMEM and fused epilogues for the Mamba-2 block:
//
//   EPI_F32    store f32                      (tied head logits, decode u)
//   EPI_BF16   store bf16
//   EPI_INPROJ columns [0, n_split) -> bf16 [z | xBC]; columns >= n_split are
//              dt_raw: dt = clip(softplus(acc + dt_bias)) stored f32
//              (model.py:141-142 + ssd.py:115-136 fused)
//   EPI_RESID  hidden_f32 += acc, hidden_bf16 = bf16(hidden)  (model.py:168-173)
//
// Structure (one CTA per SM, 10 warps):
//   warp 0      TMA producer: A/B k-blocks (64 bf16 = 128 B rows, SWIZZLE_128B)
//               into a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (128 x BN x 16 per instruction), commits free smem stages
//   warps 2..9  epilogue (two per TMEM lane quarter, alternating 32-column
//               chunks; residual loads prefetched one chunk ahead):
//               tcgen05.ld 32x32b from TMEM -> registers -> global;
//               two TMEM accumulators so tile i's epilogue overlaps tile i+1's
//               mainloop.
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace ssd200 {

// TC_EPI_RESID_NORM: hidden += acc * rstd(row), rstd = 1/sqrt(sum_g ssq[g,row]/d + eps)
// (the partials are summed in slice order g = 0, 1, ..: a fixed function of the
// widths, so a row's scale does not depend on the batch it runs in):
// the gated RMSNorm's row scale applied after the GEMM (it commutes with it;
// norm_w is folded into W_out's columns at load time) — numerics.py:149-158.
enum {
  TC_EPI_F32 = 0,
  TC_EPI_BF16 = 1,
  TC_EPI_INPROJ = 2,
  TC_EPI_RESID = 3,
  TC_EPI_RESID_NORM = 4
};

struct TcEpilogue {
  void *C;        // F32: float*, BF16/INPROJ: bf16*, RESID: float* (hidden)
  long ldc;       // elements
  bf16 *C_lp;     // RESID: bf16 shadow (same ldc)
  int n_split;    // INPROJ: first dt column
  float *dt;      // INPROJ: (M, H) f32
  int H;
  const float *dt_bias;
  float dt_lo, dt_hi;
  const float *ssq;  // RESID_NORM: (ng, ssq_ld) partial sums of u^2, slice-major
  int ng;
  long ssq_ld;
  float inv_d, eps;
  // F32 only: split-K.  ksplit > 1 cuts the K blocks into ksplit ranges (extra
  // tiles for small-M GEMMs, decode batches); range s writes its partial
  // product to C + s * split_stride, the consumer sums them in a fixed order.
  int ksplit;
  long split_stride;
  int group_m;  // tile order: row blocks per group (<= 1: row-major), see tile_mn
  int stream;   // outputs / residual with evict-first (.cs) accesses: at prefill sizes they
                // have no L2 reuse, and plain ones evict the weight / activation tiles
                // the other CTAs are about to re-read (2.7B out_proj: 16.2 GB DRAM per
                // launch for 9.4 GB of operands and outputs)
};

__device__ __forceinline__ float4 ld_f4(const float *p, bool cs) {
  return cs ? __ldcs(reinterpret_cast<const float4 *>(p)) : *reinterpret_cast<const float4 *>(p);
}
__device__ __forceinline__ void st_f4(float *p, float4 v, bool cs) {
  if (cs) __stcs(reinterpret_cast<float4 *>(p), v);
  else *reinterpret_cast<float4 *>(p) = v;
}
__device__ __forceinline__ void st_u2(void *p, uint2 v, bool cs) {
  if (cs) __stcs(reinterpret_cast<uint2 *>(p), v);
  else *reinterpret_cast<uint2 *>(p) = v;
}
__device__ __forceinline__ void st_u4(void *p, uint4 v, bool cs) {
  if (cs) __stcs(reinterpret_cast<uint4 *>(p), v);
  else *reinterpret_cast<uint4 *>(p) = v;
}


// PAIR: a CTA pair (cluster of 2, cta_group::2) computes a 256 x BN tile; each
// CTA stages its 128 rows of A and half (BN / 2 rows) of B, the leader issues
// M = 256 MMAs that read both CTAs' shared memory, each CTA's TMEM holds its
// 128 x BN accumulator rows.  Halves the shared-memory traffic per MMA.
template <int BN, bool PAIR = false> struct TcCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;
  static constexpr int STAGES = (A_BYTES + B_BYTES) > 32768 ? 4 : 6;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // two accumulators
  // per epilogue warp: a 32-row x 16-word transpose buffer (padded) so that
  // global stores of the epilogue are row-contiguous (coalesced)
  static constexpr uint32_t XPOSE_BYTES = 8 * 32 * 17 * 4;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + XPOSE_BYTES + 1024 + 256;
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

template <int EPI>
__device__ __forceinline__ void tc_store_chunk(const TcEpilogue &ep, uint32_t (&r)[32], int m,
                                               int n0, int N, float rowscale, size_t coff = 0) {
  if (EPI == TC_EPI_RESID_NORM) {
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * rowscale);
  }
  const bool full = (n0 + 32 <= N);
  if (EPI == TC_EPI_F32) {
    float *dst = reinterpret_cast<float *>(ep.C) + coff + (size_t)m * ep.ldc + n0;
    if (full && ((ep.ldc & 3) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4 *>(dst + j) =
            make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                        __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) dst[j] = __uint_as_float(r[j]);
    }
  } else if (EPI == TC_EPI_BF16 || EPI == TC_EPI_INPROJ) {
    const int lim = (EPI == TC_EPI_INPROJ) ? ep.n_split : N;
    bf16 *dst = reinterpret_cast<bf16 *>(ep.C) + (size_t)m * ep.ldc + n0;
    if (n0 + 32 <= lim && ((ep.ldc & 7) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 v;
        v.x = pack_bf16x2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
        v.y = pack_bf16x2(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        v.z = pack_bf16x2(__uint_as_float(r[j + 4]), __uint_as_float(r[j + 5]));
        v.w = pack_bf16x2(__uint_as_float(r[j + 6]), __uint_as_float(r[j + 7]));
        *reinterpret_cast<uint4 *>(dst + j) = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int n = n0 + j;
        if (n >= N) continue;
        const float acc = __uint_as_float(r[j]);
        if (n < lim) {
          dst[j] = __float2bfloat16_rn(acc);
        } else if (EPI == TC_EPI_INPROJ) {
          const int h = n - ep.n_split;
          ep.dt[(size_t)m * ep.H + h] =
              clamp_(softplus(acc + ep.dt_bias[h]), ep.dt_lo, ep.dt_hi);
        }
      }
    }
  } else {  // TC_EPI_RESID / TC_EPI_RESID_NORM
    float *dst = reinterpret_cast<float *>(ep.C) + (size_t)m * ep.ldc + n0;
    bf16 *lp = ep.C_lp + (size_t)m * ep.ldc + n0;
    if (full && ((ep.ldc & 7) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float4 a = *reinterpret_cast<float4 *>(dst + j);
        float4 b = *reinterpret_cast<float4 *>(dst + j + 4);
        a.x += __uint_as_float(r[j + 0]);
        a.y += __uint_as_float(r[j + 1]);
        a.z += __uint_as_float(r[j + 2]);
        a.w += __uint_as_float(r[j + 3]);
        b.x += __uint_as_float(r[j + 4]);
        b.y += __uint_as_float(r[j + 5]);
        b.z += __uint_as_float(r[j + 6]);
        b.w += __uint_as_float(r[j + 7]);
        *reinterpret_cast<float4 *>(dst + j) = a;
        *reinterpret_cast<float4 *>(dst + j + 4) = b;
        uint4 v;
        v.x = pack_bf16x2(a.x, a.y);
        v.y = pack_bf16x2(a.z, a.w);
        v.z = pack_bf16x2(b.x, b.y);
        v.w = pack_bf16x2(b.z, b.w);
        *reinterpret_cast<uint4 *>(lp + j) = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (n0 + j >= N) continue;
        float v = dst[j] + __uint_as_float(r[j]);
        dst[j] = v;
        lp[j] = __float2bfloat16_rn(v);
      }
    }
  }
}

// Tile order: groups of group_m row blocks, row block fastest inside a
// group.  The CTAs in flight then share a few weight (B) tiles and a bounded set
// of activation (A) row blocks, so both stay in L2: the plain row-major order
// streamed every weight tile once per row block (2.7B in_proj: 24.8 GB of DRAM
// traffic per launch for ~7 GB of operands and outputs).
// (group_m = 1 is the row-major order, better when the weight has few column
// tiles: the out_proj's A row block is then read once for all of them.)
__device__ __forceinline__ void tile_mn(int mn, int num_m, int num_n, int group_m, int &m_blk,
                                        int &n_blk) {
  const int per_group = group_m * num_n;
  const int g = mn / per_group, r = mn - g * per_group;
  const int first = g * group_m;
  const int rows = min(num_m - first, group_m);
  m_blk = first + r % rows;
  n_blk = r / rows;
}

template <int BN, int EPI, bool PAIR = false>
__global__ void __launch_bounds__(320, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, TcEpilogue ep) {
  using Cfg = TcCfg<BN, PAIR>;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an offset so that the compiler
  // keeps the shared address space (LDS/STS rather than generic loads)
  uint8_t *smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = smem;
  uint8_t *sB = smem + STAGES * Cfg::A_BYTES;
  uint32_t *sX = reinterpret_cast<uint32_t *>(sB + STAGES * Cfg::B_BYTES);  // transpose buffers
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + STAGES * Cfg::B_BYTES + Cfg::XPOSE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RSTRIDE = 128;  // output rows per tile
  // pair mode: tiles are 256 rows per cluster; rank r owns rows [128 r, 128 r + 128)
  const uint32_t rank = PAIR ? sm100::cluster_rank() : 0u;
  const int cta0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nct = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  constexpr int TROWS = PAIR ? 256 : RSTRIDE;
  const int num_n = (N + BN - 1) / BN;
  const int num_m = (M + TROWS - 1) / TROWS;
  const int num_mn = num_m * num_n;
  const int gm = ep.group_m > 1 ? ep.group_m : 1;
  const int ksplit = (EPI == TC_EPI_F32 && ep.ksplit > 1) ? ep.ksplit : 1;
  const int num_tiles = num_mn * ksplit;
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&tfull[s], 1);
      sm100::mbar_init(&tempty[s], PAIR ? 16 : 8);  // pair: both CTAs' epilogue warps
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR)
      sm100::tmem_alloc_pair<Cfg::TMEM_COLS>(tmem_slot);
    else
      sm100::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) sm100::cluster_sync();  // both CTAs' barriers live before any remote arrive
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch();  // the next kernel's CTAs may take SMs as ours retire
  griddep_wait();    // the predecessor's outputs (A, residual, ssq) are visible

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = cta0; tile < num_tiles; tile += nct) {
        const int mn = tile % num_mn, ks = tile / num_mn;
        int m_blk, n_blk;
        tile_mn(mn, num_m, num_n, gm, m_blk, n_blk);
        const int kb0 = ks * num_kb / ksplit, kb1 = (ks + 1) * num_kb / ksplit;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[s], ph ^ 1);
          if constexpr (PAIR) {
            // both CTAs' bytes complete on the leader's full barrier
            const uint32_t fb = sm100::mapa_u32(sm100::smem_u32(&full[s]), 0);
            if (rank == 0) sm100::mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
            sm100::tma_load_2d_pair(sA + s * Cfg::A_BYTES, &tmA, fb, kb * BK,
                                    m_blk * 256 + (int)rank * 128);
            sm100::tma_load_2d_pair(sB + s * Cfg::B_BYTES, &tmB, fb, kb * BK,
                                    n_blk * BN + (int)rank * (BN / 2));
          } else {
          sm100::mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
          sm100::tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * BK,
                             m_blk * RSTRIDE);
          sm100::tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, &full[s], kb * BK, n_blk * BN);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // pair mode: the leader issues for both CTAs
      constexpr uint32_t idesc = sm100::idesc_bf16(PAIR ? 256 : BM, BN, false, false);
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int tile = cta0; tile < num_tiles; tile += nct, ++local) {
        const int as = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        sm100::mbar_wait(&tempty[as], aph ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        const int ks = tile / num_mn;
        const int kb0 = ks * num_kb / ksplit, kb1 = (ks + 1) * num_kb / ksplit;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[s], ph);
          sm100::tc_fence_after();
          const uint32_t a0 = sm100::smem_u32(sA + s * Cfg::A_BYTES);
          const uint32_t b0 = sm100::smem_u32(sB + s * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = sm100::sw128_desc(a0 + k * 32, 16, 1024);
            const uint64_t bd = sm100::sw128_desc(b0 + k * 32, 16, 1024);
            if constexpr (PAIR)
              sm100::mma_bf16_pair(d_tmem, ad, bd, idesc, (kb != kb0) || (k != 0));
            else
              sm100::mma_bf16(d_tmem, ad, bd, idesc, (kb != kb0) || (k != 0));
          }
          if constexpr (PAIR)
            sm100::mma_commit_pair(&empty[s], 3);
          else
            sm100::mma_commit(&empty[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (PAIR)
          sm100::mma_commit_pair(&tfull[as], 3);
        else
          sm100::mma_commit(&tfull[as]);
      }
    }
  } else {
    // 8 epilogue warps: two per TMEM lane quarter, alternating 32-column chunks
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;
    constexpr bool RESID = (EPI == TC_EPI_RESID || EPI == TC_EPI_RESID_NORM);
    const bool vec_ok = (ep.ldc & 7) == 0;
    int local = 0;
    for (int tile = cta0; tile < num_tiles; tile += nct, ++local) {
      const int mn = tile % num_mn;
      const size_t coff = (size_t)(tile / num_mn) * (size_t)ep.split_stride;
      int m_blk, n_blk;
      tile_mn(mn, num_m, num_n, gm, m_blk, n_blk);
      const int as = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      const int i_row = q * 32 + lane;                 // tile row == TMEM lane
      const int row0 = PAIR ? m_blk * 256 + (int)rank * 128 : m_blk * RSTRIDE;
      const int m = row0 + i_row;                      // global row
      // row-only inputs before the wait: the norm scale and the first residual chunk
      float rowscale = 1.f;
      if (EPI == TC_EPI_RESID_NORM && m < M) {
        float s = 0.f;
        for (int gg = 0; gg < ep.ng; ++gg) s += ep.ssq[(size_t)gg * ep.ssq_ld + m];
        rowscale = 1.f / sqrtf(s * ep.inv_d + ep.eps);
      }
      // transposed view of a 32 x 32 chunk: lanes 0-15 / 16-31 take rows 2i / 2i+1,
      // column (lane & 15) of each 16-column half -> row-contiguous global accesses
      uint32_t *xpb = sX + (warp - 2) * (32 * 17);
      const int m_w = row0 + q * 32;  // global row of this warp's lane 0
      const int tc = lane & 15, tr = lane >> 4;
      float hv[32];  // residual chunk, transposed layout (see fetch)
      // RESID with 16-byte aligned rows (rvec): in each 16-column half h, lane l takes rows
      // 8 i + (l >> 2) and columns 4 (l & 3) .. + 3 -> hv[16 h + 4 i + j] (float4 loads /
      // stores); otherwise the scalar layout [half h][pair i] -> hv[16 h + i]
      const bool rvec = RESID && (ep.ldc & 3) == 0 && (N & 3) == 0;
      const int vr = lane >> 2, vc = 4 * (lane & 3);
      auto fetch = [&](int cc, float(&dst)[32]) {
        const int n0 = n_blk * BN + cc;
        if (RESID && cc < BN && n0 < N) {
          if (rvec) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int mr = m_w + 8 * i + vr, n = n0 + 16 * h + vc;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (mr < M && n < N)
                  v = ld_f4(reinterpret_cast<const float *>(ep.C) + (size_t)mr * ep.ldc + n,
                            ep.stream);
                dst[16 * h + 4 * i + 0] = v.x;
                dst[16 * h + 4 * i + 1] = v.y;
                dst[16 * h + 4 * i + 2] = v.z;
                dst[16 * h + 4 * i + 3] = v.w;
              }
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int mr = m_w + 2 * i + tr, n = n0 + 16 * h + tc;
                dst[16 * h + i] = (mr < M && n < N)
                                      ? reinterpret_cast<const float *>(ep.C)[(size_t)mr * ep.ldc + n]
                                      : 0.f;
              }
          }
        }
      };
      fetch(half * 32, hv);
      sm100::mbar_wait(&tfull[as], aph);
      sm100::tc_fence_after();
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
#pragma unroll 1
      for (int cc = half * 32; cc < BN; cc += 64) {
        const int n0 = n_blk * BN + cc;
        if (n0 >= N) break;  // warp-uniform
        float hn[32];
        fetch(cc + 64, hn);  // next residual chunk in flight during this one
        uint32_t r[32];
        sm100::tmem_ld32(trow + cc, r);
        sm100::tmem_ld_wait();
        if constexpr (RESID) {
          // hidden += acc * rowscale: f32 + bf16 shadow, stored row-contiguously
          float *C = reinterpret_cast<float *>(ep.C);
          if (rvec) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                xpb[lane * 17 + j] = __float_as_uint(__uint_as_float(r[16 * h + j]) * rowscale);
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int rr = 8 * i + vr, mr = m_w + rr, n = n0 + 16 * h + vc;
                if (mr < M && n < N) {
                  float4 o;
                  o.x = hv[16 * h + 4 * i + 0] + __uint_as_float(xpb[rr * 17 + vc + 0]);
                  o.y = hv[16 * h + 4 * i + 1] + __uint_as_float(xpb[rr * 17 + vc + 1]);
                  o.z = hv[16 * h + 4 * i + 2] + __uint_as_float(xpb[rr * 17 + vc + 2]);
                  o.w = hv[16 * h + 4 * i + 3] + __uint_as_float(xpb[rr * 17 + vc + 3]);
                  st_f4(C + (size_t)mr * ep.ldc + n, o, ep.stream);
                  uint2 pk;
                  pk.x = pack_bf16x2(o.x, o.y);
                  pk.y = pack_bf16x2(o.z, o.w);
                  st_u2(ep.C_lp + (size_t)mr * ep.ldc + n, pk, ep.stream);
                }
              }
              __syncwarp();
            }
          } else
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              xpb[lane * 17 + j] = __float_as_uint(__uint_as_float(r[16 * h + j]) * rowscale);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int mr = m_w + 2 * i + tr, n = n0 + 16 * h + tc;
              if (mr < M && n < N) {
                const float o = hv[16 * h + i] + __uint_as_float(xpb[(2 * i + tr) * 17 + tc]);
                C[(size_t)mr * ep.ldc + n] = o;
                ep.C_lp[(size_t)mr * ep.ldc + n] = __float2bfloat16_rn(o);
              }
            }
            __syncwarp();
          }
        } else if (EPI == TC_EPI_INPROJ && n0 + 32 <= ep.n_split && vec_ok) {
          // bf16 z / xBC columns, stored row-contiguously: 16 bf16 pairs (64 B) per row,
          // lane l stores 16 B of row 8 i + (l >> 2)
          bf16 *C = reinterpret_cast<bf16 *>(ep.C);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            xpb[lane * 17 + j] = pack_bf16x2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = 8 * i + vr, mr = m_w + rr;
            if (mr < M) {
              uint4 v;
              v.x = xpb[rr * 17 + vc + 0];
              v.y = xpb[rr * 17 + vc + 1];
              v.z = xpb[rr * 17 + vc + 2];
              v.w = xpb[rr * 17 + vc + 3];
              st_u4(C + (size_t)mr * ep.ldc + n0 + 2 * vc, v, ep.stream);
            }
          }
          __syncwarp();
        } else if (m < M) {
          tc_store_chunk<EPI>(ep, r, m, n0, N, rowscale, coff);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) hv[j] = hn[j];
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)  // the leader's MMA waits for both CTAs' epilogues
          sm100::mbar_arrive_cluster(sm100::mapa_u32(sm100::smem_u32(&tempty[as]), 0));
        else
          sm100::mbar_arrive(&tempty[as]);
      }
    }
  }
  __syncthreads();
  if constexpr (PAIR) sm100::cluster_sync();  // the peer's MMAs / arrivals are done
  if (warp == 1) {
    __syncwarp();
    sm100::tc_fence_after();
    if constexpr (PAIR)
      sm100::tmem_dealloc_pair<Cfg::TMEM_COLS>(tmem_base);
    else
      sm100::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

}  // namespace ssd200
