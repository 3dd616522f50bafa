// ssd_tc_out — chunk outputs of the tensor-core SSD scan.
//
// One CTA per (batch b, chunk c, 128-row tile R of the chunk, head group g):
//   G = C_R . B^T   (128 x 128(R+1) x 128 UMMA, once; shared by every head, G = 1)
//   per head h:
//     M[l,s] = G[l,s] * e^{cs_l - cs_s} * dt_s  (s <= l)  -> bf16, written to TMEM
//       the decay is factorised per 32-column chunk J (r = last index of J):
//         e^{cs_l - cs_s} = e^{cs_l - cs_r} * e^{cs_r - cs_s},   both factors <= 1
//       so each (row, chunk) needs one ex2 and each column one ex2 per head;
//       only the diagonal chunk (s, l in the same 32-block) exponentiates
//       per element (ssd.py:147-148 / numerics.py:134-146 restated)
//     Ydiag = M . X_h        (K = 128(R+1)), A operand read from TMEM   ssd.py:149
//     Yoff  = C_R . prev_h^T (K = N = 128)                               ssd.py:196
//     y = Ydiag + e^{cs_l} Yoff + D_h x;  u = y * silu(z);  sum u^2       model.py:166-167
//   sum u^2 leaves as one partial per (SSQ_SLICE-head slice, column half) — independent of
//   the head grouping, so the norm's row scale is batch-invariant.
//
// M lives in TMEM (tcgen05.st by the math warps, consumed as the A operand of
// tcgen05.mma), double buffered: the math warps build M_{h+1} while the tensor
// core multiplies M_h, with no shared-memory round trip and no proxy fence.
// G itself is kept as bf16 in shared memory (the B-row staging area, free once
// G is computed) so TMEM holds only the two M buffers and two accumulator sets:
//   TMEM cols [0,128) M buffer 0, [128,256) M buffer 1 (bf16 pairs per column),
//             [256+128k, +64) Ydiag set k, [320+128k, +64) Yoff set k.
// X / prev tiles are double buffered as well, so head h's epilogue runs while
// the tensor core computes head h+1 and TMA fetches head h+2.
// Warp roles: warp 0 TMA, warp 1 MMA + TMEM owner, then OUT_KW math warps per
// TMEM lane quarter: warp k of a quarter builds columns [CW k, CW (k+1)) of
// every 32-column chunk of M, CW = 32 / OUT_KW (so the expensive diagonal chunk
// is shared evenly) and runs the epilogue on head columns [EW k, EW (k+1)),
// EW = 64 / OUT_KW.
// Block order: R = 1 / R = 0 tiles of one (b, c, g) side by side (L2 reuse).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace ssd200 {

// math warps per TMEM lane quarter: 8 math warps at 168 registers fill most of the
// register file (16 would leave 113 registers per thread)
constexpr int OUT_KW = 2;
// heads per sum-u^2 slice: head groups are whole slices, so the smallest group (and
// hence the output kernel's parallelism at small B) is one slice — 2 keeps B = 1,
// T = 2K at 256 CTAs for 32 heads; the out_proj then sums H / 2 * OUT_KW partials
constexpr int SSQ_SLICE = 2;
constexpr int OUT_CW = 32 / OUT_KW;    // columns of every 32-column M chunk per warp
constexpr int OUT_MW = 4 * OUT_KW;     // math warps
constexpr int OUT_EW = TC_P / OUT_KW;  // epilogue head columns per warp
constexpr int OUT_MATH = OUT_MW * 32;  // math threads
constexpr int OUT_THREADS = OUT_MATH + 64;

struct OutSmem {
  static constexpr uint32_t CR = 0;           // C rows of the tile: 2 x [128 l][64 n] (SW128)
  static constexpr uint32_t GB = 32768;       // B rows 2 x [NS s][64 n]; then G bf16 [128 l][NS s]
  static constexpr uint32_t X0 = GB + 65536;  // 2 x [256 s][64 p]
  static constexpr uint32_t P0 = X0 + 2 * 32768;  // 2 x [128 n][64 p]
  static constexpr uint32_t Z0 = P0 + 2 * 16384;  // gate z of the current head [128 l][64 p]
  static constexpr uint32_t WC = Z0 + 16384;       // per warp 4 x 8 OUT_CW f32 (cs2, cf, dt, cr)
  static constexpr uint32_t DH = WC + OUT_MW * 4 * 8 * OUT_CW * 4;  // D of the group's heads (<= 128)
  static constexpr uint32_t BAR = DH + 512;
  static constexpr uint32_t TOTAL = BAR + 256 + 1024;
  static constexpr int MAX_HG = 128;  // heads per CTA (DH table)
};

// 1024-byte aligned view of dynamic smem that keeps the shared address space
// visible to the compiler (STS/LDS instead of generic accesses)
__device__ __forceinline__ uint8_t *smem_align1k(uint8_t *raw) {
  const uint32_t a = sm100::smem_u32(raw);
  return raw + ((1024u - (a & 1023u)) & 1023u);
}

__global__ void __launch_bounds__(OUT_THREADS, 1)
    ssd_tc_out(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_prev,
               const __grid_constant__ CUtensorMap tm_z, const __grid_constant__ CUtensorMap tm_u,
               TcSsdArgs p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t *sm = smem_align1k(smem_raw);
  uint64_t *bar_cb = reinterpret_cast<uint64_t *>(sm + OutSmem::BAR);
  uint64_t *bar_g = bar_cb + 1;
  uint64_t *bar_x = bar_cb + 2;   // [2] X tile landed
  uint64_t *xfree = bar_cb + 4;   // [2] X tile consumed
  uint64_t *bar_p = bar_cb + 6;   // [2] prev tile landed
  uint64_t *pfree = bar_cb + 8;   // [2] prev tile consumed
  uint64_t *bar_y = bar_cb + 10;  // [2] accumulator set ready
  uint64_t *yfree = bar_cb + 12;  // [2] accumulator set read out
  uint64_t *mrdy = bar_cb + 14;   // [2] M buffer written (one arrival per math warp)
  uint64_t *bar_z = bar_cb + 16;  // z tile landed
  uint64_t *zfree = bar_cb + 17;  // z tile read (one arrival per math warp)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bar_cb + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // interleaved (default): the two row tiles of one (b, c, g) are neighbours in
  // launch order, so they run together and the X / prev tiles both read come
  // from L2 the second time; else the heavier R = 1 tiles first, then R = 0
  const int half_grid = gridDim.x >> 1;
  const int R = p.interleave ? ((blockIdx.x & 1) ^ 1) : (blockIdx.x < half_grid ? 1 : 0);
  int idx = p.interleave ? (blockIdx.x >> 1) : (R ? blockIdx.x : blockIdx.x - half_grid);
  const int g = idx % p.NG;
  idx /= p.NG;
  const int b = idx / p.Nc, c = idx % p.Nc;
  const int h0 = g * p.HG;
  const int NS = 128 * (R + 1);  // columns s of this row tile
  const uint32_t TM_M = 0, TM_Y = 256;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_act);
    sm100::tma_prefetch(&tm_prev);
    sm100::tma_prefetch(&tm_z);
    sm100::tma_prefetch(&tm_u);
    sm100::mbar_init(bar_cb, 1);
    sm100::mbar_init(bar_g, 1);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&bar_x[i], 1);
      sm100::mbar_init(&xfree[i], 1 + 4);  // MMA commit + each lane quarter's u store (it reuses the tile)
      sm100::mbar_init(&bar_p[i], 1);
      sm100::mbar_init(&pfree[i], 1);
      sm100::mbar_init(&bar_y[i], 1);
      sm100::mbar_init(&yfree[i], OUT_MATH);
      sm100::mbar_init(&mrdy[i], OUT_MW);
    }
    sm100::mbar_init(bar_z, 1);
    sm100::mbar_init(zfree, OUT_MW);  // one arrival per math warp once it has read its z
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<512>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch();
  griddep_wait();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      sm100::mbar_arrive_expect_tx(bar_cb, 32768 + 2 * NS * 128);
      for (int nb = 0; nb < 2; ++nb) {
        sm100::tma_load_3d(sm + OutSmem::CR + nb * 16384, &tm_act, bar_cb,
                           p.d_inner + TC_N + nb * 64, c * TC_L + R * 128, b);
        for (int q = 0; q <= R; ++q)
          sm100::tma_load_3d(sm + OutSmem::GB + nb * NS * 128 + q * 16384, &tm_act, bar_cb,
                             p.d_inner + nb * 64, c * TC_L + q * 128, b);
      }
      for (int i = 0; i < p.HG; ++i) {
        const int buf = i & 1, h = h0 + i;
        const uint32_t par = ((i >> 1) & 1) ^ 1;
        sm100::mbar_wait(&pfree[buf], par);
        sm100::mbar_arrive_expect_tx(&bar_p[buf], 16384);
        const int prow = (((b * p.Nc + c) * p.H + h) * TC_N);  // prev (b, c, h) as [n][p]
        sm100::tma_load_2d(sm + OutSmem::P0 + buf * 16384, &tm_prev, &bar_p[buf], 0, prow);
        sm100::mbar_wait(&xfree[buf], par);
        sm100::mbar_arrive_expect_tx(&bar_x[buf], NS * 128);
        for (int q = 0; q <= R; ++q)
          sm100::tma_load_3d(sm + OutSmem::X0 + buf * 32768 + q * 16384, &tm_act, &bar_x[buf],
                             h * TC_P, c * TC_L + q * 128, b);
        sm100::mbar_wait(zfree, (i & 1) ^ 1);  // single buffer: every warp has read head i-1's z
        sm100::mbar_arrive_expect_tx(bar_z, 16384);
        sm100::tma_load_3d(sm + OutSmem::Z0, &tm_z, bar_z, h * TC_P, c * TC_L + R * 128, b);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t cr = sm100::smem_u32(sm + OutSmem::CR);
      const uint32_t gb = sm100::smem_u32(sm + OutSmem::GB);
      sm100::mbar_wait(bar_cb, 0);
      sm100::tc_fence_after();
      const uint32_t idg = sm100::idesc_bf16(128, NS, false, false);
#pragma unroll
      for (int k = 0; k < TC_N / 16; ++k) {  // G into TMEM cols [0, NS) (before any M)
        const uint64_t ad = sm100::sw128_desc(cr + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        const uint64_t bd = sm100::sw128_desc(gb + (k >> 2) * NS * 128 + (k & 3) * 32, 16, 1024);
        sm100::mma_bf16(tmem + TM_M, ad, bd, idg, k > 0);
      }
      sm100::mma_commit(bar_g);
      constexpr uint32_t idy = sm100::idesc_bf16(128, TC_P, false, true);
      constexpr uint32_t ido = sm100::idesc_bf16(128, TC_P, false, true);
      for (int i = 0; i < p.HG; ++i) {
        const int buf = i & 1;
        const uint32_t par = (i >> 1) & 1;
        const uint32_t yd = tmem + TM_Y + buf * 128, yo = yd + 64;
        sm100::mbar_wait(&yfree[buf], par ^ 1);
        sm100::mbar_wait(&bar_p[buf], par);
        sm100::tc_fence_after();
        const uint32_t pb = sm100::smem_u32(sm + OutSmem::P0 + buf * 16384);
#pragma unroll
        for (int k = 0; k < TC_N / 16; ++k) {  // Yoff = C_R . prev^T (independent of M)
          const uint64_t ad = sm100::sw128_desc(cr + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sm100::sw128_desc(pb + k * 2048, 8192, 1024);  // [n][p]: MN-major
          sm100::mma_bf16(yo, ad, bd, ido, k > 0);
        }
        sm100::mma_commit(&pfree[buf]);
        sm100::mbar_wait(&bar_x[buf], par);
        sm100::mbar_wait(&mrdy[buf], par);
        sm100::tc_fence_after();
        const uint32_t xb = sm100::smem_u32(sm + OutSmem::X0 + buf * 32768);
        const uint32_t am = tmem + TM_M + buf * 128;
        for (int k = 0; k < NS / 16; ++k) {  // Ydiag = M . X, M from TMEM
          const uint64_t bd = sm100::sw128_desc(xb + k * 2048, 8192, 1024);
          sm100::mma_bf16_ts(yd, am + k * 8, bd, idy, k > 0);
        }
        sm100::mma_commit(&bar_y[buf]);  // accumulators ready, M buffer and X tile free
        sm100::mma_commit(&xfree[buf]);
      }
    }
  } else {
    // ------------------------------------------------------------ math warps
    constexpr int CW = OUT_CW, CL = CW / 4, CP = CW / 8;
    const int mw = warp - 2;        // 0 .. OUT_MW-1
    const int q = warp & 3;         // TMEM lane quarter
    const int kw = mw >> 2;         // column slice: CW columns of every 32-column chunk
    const int row = q * 32 + lane;  // tile row == TMEM lane
    const int l = R * 128 + row;    // row within the chunk
    const int t = c * TC_L + l;
    const bool valid = t < p.T;
    const int jd = 4 * R + q;  // this quarter's diagonal 32-column chunk
    const int nj = NS / 32;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const long csb = (long)p.Nc * TC_L;
    // warp table, entry CW j + e = column 32j + CW kw + e: cs*log2e, cf, dt;
    // cr[j] = cs_r*log2e (r = last column of chunk j)
    float *wcs = reinterpret_cast<float *>(sm + OutSmem::WC) + mw * (4 * 8 * CW);
    float *wcf = wcs + 8 * CW;
    float *wdt = wcs + 16 * CW;
    float *wcr = wcs + 24 * CW;
    float *d_s = reinterpret_cast<float *>(sm + OutSmem::DH);
    // G row of this thread: NS bf16 in 16-byte pieces XOR-swizzled by row
    // (conflict-free); pieces 4j + CP kw + [0, CP) are this warp's slice of chunk j
    uint8_t *grow = sm + OutSmem::GB + row * (NS * 2);
    const int gsw = row & 7;
    auto gpiece = [&](int pc) -> uint4 * {
      return reinterpret_cast<uint4 *>(grow + ((pc ^ gsw) << 4));
    };
    float ssq = 0.f;

    struct Pref {
      float cs[CL], dt[CL];
      float cr, csl;
    };
    // lane -> chunk j = lane/4, columns 32j + CW kw + CL (lane%4) + [0, CL)
    const int fj = lane >> 2, fcol = 32 * fj + CW * kw + CL * (lane & 3);
    auto fetch = [&](int i, Pref &f) {
      const int h = h0 + i;
      const float *csg = p.cs + ((long)b * p.H + h) * csb + (long)c * TC_L;
      const float *dtg = p.dtT + ((long)b * p.H + h) * csb + (long)c * TC_L;
      const float4 a = *reinterpret_cast<const float4 *>(csg + fcol);
      const float4 d = *reinterpret_cast<const float4 *>(dtg + fcol);
      f.cs[0] = a.x, f.cs[1] = a.y, f.cs[2] = a.z, f.cs[3] = a.w;
      f.dt[0] = d.x, f.dt[1] = d.y, f.dt[2] = d.z, f.dt[3] = d.w;
      f.cr = csg[32 * fj + 31];
      f.csl = csg[l];
    };
    // cf[s] = e^{cs_r - cs_s} dt_s
    auto commit = [&](const Pref &f) -> float {
      __syncwarp();  // every lane is done reading the previous head's table
      const float vr = f.cr * kLog2e;
      uint32_t *wcfb = reinterpret_cast<uint32_t *>(wcf);  // cf as bf16 pairs
#pragma unroll
      for (int k = 0; k < CL; k += 2) {
        const float v0 = f.cs[k] * kLog2e, v1 = f.cs[k + 1] * kLog2e;
        wcs[CL * lane + k] = v0;
        wcs[CL * lane + k + 1] = v1;
        wdt[CL * lane + k] = f.dt[k];
        wdt[CL * lane + k + 1] = f.dt[k + 1];
        __nv_bfloat162 cf2 = __floats2bfloat162_rn(ex2(vr - v0) * f.dt[k], ex2(vr - v1) * f.dt[k + 1]);
        wcfb[(CL * lane + k) / 2] = *reinterpret_cast<uint32_t *>(&cf2);
      }
      if ((lane & 3) == 0) wcr[fj] = vr;
      __syncwarp();
      return f.csl * kLog2e;
    };
    auto ld_table = [&](const float *tab, int j, float (&v)[CW]) {
#pragma unroll
      for (int k = 0; k < CW / 4; ++k) {
        const float4 a = *reinterpret_cast<const float4 *>(tab + CW * j + 4 * k);
        v[4 * k] = a.x, v[4 * k + 1] = a.y, v[4 * k + 2] = a.z, v[4 * k + 3] = a.w;
      }
    };
    auto ld_g = [&](int j, uint32_t (&gw)[CW / 2]) {
#pragma unroll
      for (int k = 0; k < CP; ++k) {
        const uint4 g = *gpiece(4 * j + CP * kw + k);
        gw[4 * k] = g.x, gw[4 * k + 1] = g.y, gw[4 * k + 2] = g.z, gw[4 * k + 3] = g.w;
      }
    };
    auto st_m = [&](uint32_t taddr, const uint32_t (&pk)[CW / 2], bool on) {
      sm100::tmem_st8_if(taddr, pk, on);
    };
    // M = G * decay * dt for this warp's slice of head hh -> TMEM M buffer hh & 1.
    // The off-diagonal chunks are computed branch-free (NJ is a compile-time
    // constant per row tile) so their loads and math interleave; chunks at or
    // past the diagonal are computed but not stored.
    auto build_m = [&](auto rt, int hh, float csl) {
      constexpr int NJ = 4 * (decltype(rt)::value + 1);
      const uint32_t mt = tmem + lane_off + TM_M + (hh & 1) * 128 + (CW / 2) * kw;
      {  // diagonal chunk: per-element decay, causal mask
        uint32_t gw[CW / 2], pd[CW / 2];
        float cs[CW], dt[CW];
        ld_g(jd, gw);
        ld_table(wcs, jd, cs);
        ld_table(wdt, jd, dt);
        const int s0 = 32 * jd + CW * kw;
#pragma unroll
        for (int e = 0; e < CW / 2; ++e) {
          const int s = s0 + 2 * e;
          const float g0 = __uint_as_float(gw[e] << 16);
          const float g1 = __uint_as_float(gw[e] & 0xffff0000u);
          const float m0 = s <= l ? g0 * ex2(csl - cs[2 * e]) * dt[2 * e] : 0.f;
          const float m1 = s + 1 <= l ? g1 * ex2(csl - cs[2 * e + 1]) * dt[2 * e + 1] : 0.f;
          __nv_bfloat162 v = __floats2bfloat162_rn(m0, m1);
          pd[e] = *reinterpret_cast<uint32_t *>(&v);
        }
        st_m(mt + 16 * jd, pd, true);
      }
      // off-diagonal chunks: M = (G * cf) * rf on packed bf16 pairs (M is bf16 anyway)
      const uint32_t *wcfb = reinterpret_cast<const uint32_t *>(wcf);
#pragma unroll
      for (int j = 0; j < NJ - 1; ++j) {
        uint32_t gw[CW / 2], cw[CW / 2], pk[CW / 2];
        ld_g(j, gw);
#pragma unroll
        for (int k = 0; k < CW / 8; ++k) {
          const uint4 a = *reinterpret_cast<const uint4 *>(wcfb + (CW / 2) * j + 4 * k);
          cw[4 * k] = a.x, cw[4 * k + 1] = a.y, cw[4 * k + 2] = a.z, cw[4 * k + 3] = a.w;
        }
        const __nv_bfloat162 rf2 = __float2bfloat162_rn(ex2(csl - wcr[j]));
#pragma unroll
        for (int e = 0; e < CW / 2; ++e) {
          const __nv_bfloat162 m = __hmul2(__hmul2(*reinterpret_cast<const __nv_bfloat162 *>(&gw[e]),
                                                   *reinterpret_cast<const __nv_bfloat162 *>(&cw[e])),
                                           rf2);
          pk[e] = *reinterpret_cast<const uint32_t *>(&m);
        }
        st_m(mt + 16 * j, pk, j < jd);
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&mrdy[hh & 1]);
    };
    auto build = [&](int hh, float csl) {
      if (R) build_m(std::integral_constant<int, 1>{}, hh, csl);
      else build_m(std::integral_constant<int, 0>{}, hh, csl);
    };

    Pref nxt;
    fetch(0, nxt);
    float csl = commit(nxt);
    if (p.HG > 1) fetch(1, nxt);
    // ---- G: TMEM f32 -> bf16 smem rows (this warp's column slices)
    sm100::mbar_wait(bar_g, 0);
    sm100::tc_fence_after();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < nj && j <= jd) {
        uint32_t r[CW];
        sm100::tmem_ld16(tmem + lane_off + TM_M + 32 * j + CW * kw, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < CP; ++k) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(r[8 * k + 2 * e]),
                                                     __uint_as_float(r[8 * k + 2 * e + 1]));
            w[e] = *reinterpret_cast<uint32_t *>(&v);
          }
          *gpiece(4 * j + CP * kw + k) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
    for (int k = threadIdx.x - 64; k < p.HG; k += OUT_MATH) d_s[k] = p.D[h0 + k];
    sm100::tc_fence_before();
    named_bar(1, OUT_MATH);  // every G column read out of TMEM before M overwrites it
    sm100::tc_fence_after();
    {  // chunks above the diagonal are zero in both M buffers for every head
      const uint32_t zero[CW / 2] = {};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool on = j < nj && j > jd;
        st_m(tmem + lane_off + TM_M + 16 * j + (CW / 2) * kw, zero, on);
        st_m(tmem + lane_off + TM_M + 128 + 16 * j + (CW / 2) * kw, zero, on);
      }
    }
    build(0, csl);
    constexpr int EW = OUT_EW;  // epilogue columns per warp
    const int pc = kw * EW;
    for (int i = 0; i < p.HG; ++i) {
      const int buf = i & 1, h = h0 + i;
      uint4 xv[EW / 8], zv[EW / 8];  // x (D skip) and z (gate) of head i, columns [pc, pc+EW)
      const float el = ex2(csl);
      const float Dh = d_s[i];
      if (i + 1 < p.HG) {  // M_{i+1} into the other buffer while the tensor core runs head i
        csl = commit(nxt);
        if (i + 2 < p.HG) fetch(i + 2, nxt);
        build(i + 1, csl);
      }
      sm100::mbar_wait(bar_z, i & 1);  // z tile of head i (TMA, SWIZZLE_128B)
#pragma unroll
      for (int cc = 0; cc < EW / 8; ++cc)
        zv[cc] = *reinterpret_cast<const uint4 *>(sm + OutSmem::Z0 + sw128_off(row, pc / 8 + cc));
      sm100::mbar_wait(&bar_y[buf], (i >> 1) & 1);  // MMA(i) done
      // D-skip x from the X tile the MMA just consumed (row l of the chunk); u later
      // overwrites the same positions and leaves from there, so the tile is released
      // only once that store has read it
      uint8_t *xt = sm + OutSmem::X0 + buf * 32768 + R * 16384;
#pragma unroll
      for (int cc = 0; cc < EW / 8; ++cc)
        xv[cc] = *reinterpret_cast<const uint4 *>(xt + sw128_off(row, pc / 8 + cc));
      sm100::tc_fence_after();
      // ---- epilogue(i) on columns [pc, pc+EW) in 16-column steps, overlapping MMA(i+1)
      const uint32_t ydt = tmem + lane_off + TM_Y + buf * 128 + pc;
      const __nv_bfloat162 *xe = reinterpret_cast<const __nv_bfloat162 *>(xv);
      const __nv_bfloat162 *ze = reinterpret_cast<const __nv_bfloat162 *>(zv);
#pragma unroll
      for (int hs = 0; hs < EW / 16; ++hs) {
        uint32_t yd[16], yo[16];
        sm100::tmem_ld16(ydt + 16 * hs, yd);
        sm100::tmem_ld16(ydt + 64 + 16 * hs, yo);
        sm100::tmem_ld_wait();
        if (hs == EW / 16 - 1) {
          sm100::tc_fence_before();
          sm100::mbar_arrive(&yfree[buf]);
        }
        uint32_t out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 xf = __bfloat1622float2(xe[8 * hs + j]);
          const float2 zf = __bfloat1622float2(ze[8 * hs + j]);
          const float y0 = __uint_as_float(yd[2 * j]) + el * __uint_as_float(yo[2 * j]) + Dh * xf.x;
          const float y1 =
              __uint_as_float(yd[2 * j + 1]) + el * __uint_as_float(yo[2 * j + 1]) + Dh * xf.y;
          const float u0 = y0 * silu_tanh(zf.x), u1 = y1 * silu_tanh(zf.y);
          ssq += u0 * u0 + u1 * u1;
          __nv_bfloat162 v = __floats2bfloat162_rn(u0, u1);
          out[j] = *reinterpret_cast<uint32_t *>(&v);
        }
        // u overwrites this thread's own x positions of the X tile (read above)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          *reinterpret_cast<uint4 *>(xt + sw128_off(row, pc / 8 + 2 * hs + k)) =
              make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
      }
      // z is consumed (every zv register fed the math above, so the loads are done):
      // the next head's z may land.  Releasing right after the loads let the TMA
      // overwrite the tile before a delayed LDS had read it (1 in ~15 runs differed).
      sm100::fence_proxy_async();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(zfree);
      // the quarter's 32 x 64 u tile leaves through TMA (rows past T are clipped);
      // the X buffer is released once the store has read it
      named_bar(4 + q, 32 * OUT_KW);
      if (kw == 0 && lane == 0) {
        sm100::tma_store_3d(&tm_u, xt + q * 4096, h * TC_P, c * TC_L + R * 128 + q * 32, b);
        sm100::bulk_commit();
        sm100::bulk_wait_read0();
        sm100::mbar_arrive(&xfree[buf]);
      }
      // sum u^2 of this warp's columns over the SSQ_SLICE-head slice that ends here:
      // one partial per (slice, column half), slice-major (n_slices * OUT_KW, rows),
      // so the out_proj's row scale sums the same partials in the same order
      // whatever head grouping (and hence batch) this launch used
      if (i % SSQ_SLICE == SSQ_SLICE - 1) {
        if (valid)
          p.ssq[(long)(((h0 + i) / SSQ_SLICE) * OUT_KW + kw) * ((long)p.B * p.T) + (long)b * p.T + t] = ssq;
        ssq = 0.f;
      }
    }
  }
  if (warp >= 2 && (warp - 2) < 4 && lane == 0)  // kw == 0: the u stores have completed
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem);
  }
}

}  // namespace ssd200
