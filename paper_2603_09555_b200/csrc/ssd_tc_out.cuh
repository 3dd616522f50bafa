// ssd_tc_out — chunk outputs of the tensor-core SSD scan.
//
// One CTA per (batch b, chunk c, 128-row tile R of the chunk, head group g):
//   G = C_R . B^T   (128 x 128(R+1) x 128 UMMA, once; shared by every head, G = 1)
//   per head h:
//     M[l,s] = G[l,s] * e^{cs_l - cs_s} * dt_s  (s <= l)  -> bf16, K-major SW128 smem
//       the decay is factorised per 32-column chunk J (r = last index of J):
//         e^{cs_l - cs_s} = e^{cs_l - cs_r} * e^{cs_r - cs_s},   both factors <= 1
//       so each (row, chunk) needs one ex2 and each column one ex2 per head;
//       only the diagonal chunk (s, l in the same 32-block) exponentiates
//       per element (ssd.py:147-148 / numerics.py:134-146 restated)
//     Ydiag = M . X_h        (K = 128(R+1))                        ssd.py:149
//     Yoff  = C_R . prev_h^T (K = N = 128)                          ssd.py:196
//     y = Ydiag + e^{cs_l} Yoff + D_h x;  u = y * silu(z);  sum u^2  model.py:166-167
// Pipeline: X / prev tiles and the two TMEM accumulator sets are double
// buffered, so head h's epilogue runs while the tensor core computes head
// h+1 and TMA fetches head h+2; per-head column constants are prefetched one
// head ahead into warp-private smem (no block barriers in the head loop).
// Warp roles (320 threads): warp 0 TMA, warp 1 MMA + TMEM owner, warps 2..9
// math — two warps per TMEM lane quarter, splitting the columns.
// Block order: the heavier R = 1 tiles first, then R = 0.
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace ssd200 {

struct OutSmem {
  static constexpr uint32_t CR = 0;                  // C rows of the tile: 2 x [128 l][64 n]
  static constexpr uint32_t BM = 32768;              // B rows (G operand), then M: 64 KB
  static constexpr uint32_t X0 = BM + 65536;         // 2 x [256 s][64 p]
  static constexpr uint32_t P0 = X0 + 2 * 32768;     // 2 x (2 x [64 p][64 n])
  static constexpr uint32_t WC = P0 + 2 * 16384;     // 8 warps x 3 x 256 f32 (cs2, cf, dt)
  static constexpr uint32_t SQ = WC + 8 * 3 * 1024;  // 128 f32: ssq of the second half
  static constexpr uint32_t BAR = SQ + 512;
  static constexpr uint32_t TOTAL = BAR + 256 + 1024;
};

constexpr int OUT_THREADS = 320;
constexpr int OUT_MATH = 256;

// 1024-byte aligned view of dynamic smem that keeps the shared address space
// visible to the compiler (STS/LDS instead of generic accesses)
__device__ __forceinline__ uint8_t *smem_align1k(uint8_t *raw) {
  const uint32_t a = sm100::smem_u32(raw);
  return raw + ((1024u - (a & 1023u)) & 1023u);
}

__global__ void __launch_bounds__(OUT_THREADS, 1)
    ssd_tc_out(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_prev,
               TcSsdArgs p, const bf16 *__restrict__ act, long act_ld) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t *sm = smem_align1k(smem_raw);
  uint64_t *bar_cb = reinterpret_cast<uint64_t *>(sm + OutSmem::BAR);
  uint64_t *bar_g = bar_cb + 1;
  uint64_t *bar_x = bar_cb + 2;   // [2]
  uint64_t *xfree = bar_cb + 4;   // [2]
  uint64_t *bar_p = bar_cb + 6;   // [2]
  uint64_t *pfree = bar_cb + 8;   // [2]
  uint64_t *bar_m = bar_cb + 10;
  uint64_t *bar_y = bar_cb + 11;  // [2]
  uint64_t *yfree = bar_cb + 13;  // [2]
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bar_cb + 15);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half_grid = gridDim.x >> 1;
  const int R = blockIdx.x < half_grid ? 1 : 0;
  int idx = R ? blockIdx.x : blockIdx.x - half_grid;
  const int g = idx % p.NG;
  idx /= p.NG;
  const int b = idx / p.Nc, c = idx % p.Nc;
  const int h0 = g * p.HG;
  const int NS = 128 * (R + 1);  // columns s of this row tile
  // TMEM: G [0,256), accumulator set k: Ydiag [256+128k, +64), Yoff [320+128k, +64)
  const uint32_t TM_G = 0, TM_Y = 256;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_act);
    sm100::tma_prefetch(&tm_prev);
    sm100::mbar_init(bar_cb, 1);
    sm100::mbar_init(bar_g, 1);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&bar_x[i], 1);
      sm100::mbar_init(&xfree[i], 1);
      sm100::mbar_init(&bar_p[i], 1);
      sm100::mbar_init(&pfree[i], 1);
      sm100::mbar_init(&bar_y[i], 1);
      sm100::mbar_init(&yfree[i], OUT_MATH);
    }
    sm100::mbar_init(bar_m, OUT_MATH);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<512>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      sm100::mbar_arrive_expect_tx(bar_cb, 32768 + 2 * NS * 128);
      for (int nb = 0; nb < 2; ++nb) {
        sm100::tma_load_3d(sm + OutSmem::CR + nb * 16384, &tm_act, bar_cb,
                           p.d_inner + TC_N + nb * 64, c * TC_L + R * 128, b);
        for (int q = 0; q <= R; ++q)
          sm100::tma_load_3d(sm + OutSmem::BM + nb * NS * 128 + q * 16384, &tm_act, bar_cb,
                             p.d_inner + nb * 64, c * TC_L + q * 128, b);
      }
      for (int i = 0; i < p.HG; ++i) {
        const int buf = i & 1, h = h0 + i;
        const uint32_t par = ((i >> 1) & 1) ^ 1;
        sm100::mbar_wait(&pfree[buf], par);
        sm100::mbar_arrive_expect_tx(&bar_p[buf], 16384);
        const int prow = (((b * p.Nc + c) * p.H + h) * TC_P);
        for (int nb = 0; nb < 2; ++nb)
          sm100::tma_load_2d(sm + OutSmem::P0 + buf * 16384 + nb * 8192, &tm_prev, &bar_p[buf],
                             nb * 64, prow);
        sm100::mbar_wait(&xfree[buf], par);
        sm100::mbar_arrive_expect_tx(&bar_x[buf], NS * 128);
        for (int q = 0; q <= R; ++q)
          sm100::tma_load_3d(sm + OutSmem::X0 + buf * 32768 + q * 16384, &tm_act, &bar_x[buf],
                             h * TC_P, c * TC_L + q * 128, b);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t cr = sm100::smem_u32(sm + OutSmem::CR);
      const uint32_t bm = sm100::smem_u32(sm + OutSmem::BM);
      sm100::mbar_wait(bar_cb, 0);
      sm100::tc_fence_after();
      const uint32_t idg = sm100::idesc_bf16(128, NS, false, false);
#pragma unroll
      for (int k = 0; k < TC_N / 16; ++k) {
        const uint64_t ad = sm100::sw128_desc(cr + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        const uint64_t bd = sm100::sw128_desc(bm + (k >> 2) * NS * 128 + (k & 3) * 32, 16, 1024);
        sm100::mma_bf16(tmem + TM_G, ad, bd, idg, k > 0);
      }
      sm100::mma_commit(bar_g);
      constexpr uint32_t idy = sm100::idesc_bf16(128, TC_P, false, true);
      constexpr uint32_t ido = sm100::idesc_bf16(128, TC_P, false, false);
      for (int i = 0; i < p.HG; ++i) {
        const int buf = i & 1;
        const uint32_t par = (i >> 1) & 1;
        const uint32_t yd = tmem + TM_Y + buf * 128, yo = yd + 64;
        sm100::mbar_wait(&yfree[buf], par ^ 1);
        sm100::mbar_wait(&bar_p[buf], par);
        sm100::mbar_wait(bar_m, i & 1);
        sm100::tc_fence_after();
        const uint32_t pb = sm100::smem_u32(sm + OutSmem::P0 + buf * 16384);
#pragma unroll
        for (int k = 0; k < TC_N / 16; ++k) {  // Yoff = C_R . prev^T
          const uint64_t ad = sm100::sw128_desc(cr + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sm100::sw128_desc(pb + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
          sm100::mma_bf16(yo, ad, bd, ido, k > 0);
        }
        sm100::mma_commit(&pfree[buf]);
        sm100::mbar_wait(&bar_x[buf], par);
        sm100::tc_fence_after();
        const uint32_t xb = sm100::smem_u32(sm + OutSmem::X0 + buf * 32768);
        for (int k = 0; k < NS / 16; ++k) {  // Ydiag = M . X
          const uint64_t ad = sm100::sw128_desc(bm + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sm100::sw128_desc(xb + k * 2048, 8192, 1024);
          sm100::mma_bf16(yd, ad, bd, idy, k > 0);
        }
        sm100::mma_commit(&bar_y[buf]);  // accumulators ready; M buffer free
        sm100::mma_commit(&xfree[buf]);  // X buffer free
      }
    }
  } else {
    // ------------------------------------------------------------ math warps
    const int mw = warp - 2;           // 0..7
    const int q = warp & 3;            // TMEM lane quarter
    const int hf = mw >> 2;            // column-chunk parity owned by this warp
    const int row = q * 32 + lane;     // tile row == TMEM lane
    const int l = R * 128 + row;       // row within the chunk
    const int t = c * TC_L + l;
    const bool valid = t < p.T;
    const int jd = 4 * R + q;          // this warp's diagonal 32-column chunk
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const long csb = (long)p.Nc * TC_L;
    float *wcs = reinterpret_cast<float *>(sm + OutSmem::WC) + mw * 768;
    float *wcf = wcs + 256;
    float *wdt = wcs + 512;
    float *sq_s = reinterpret_cast<float *>(sm + OutSmem::SQ);
    uint8_t *mbuf = sm + OutSmem::BM;
    const long trow = (long)b * p.T + (valid ? t : 0);
    const bf16 *xrow = act + trow * act_ld;
    const bf16 *zrow = p.z + trow * p.z_ld;
    float ssq = 0.f;

    // per-head column constants for this warp's chunks j = hf, hf+2, .. <= jd
    struct Pref {
      float cs[4], dt[4], csl;
    };
    auto fetch = [&](int i, Pref &f) {
      const int h = h0 + i;
      const float *csg = p.cs + ((long)b * p.H + h) * csb + (long)c * TC_L;
      const float *dtg = p.dtT + ((long)b * p.H + h) * csb + (long)c * TC_L;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = hf + 2 * u;
        if (j <= jd) {
          f.cs[u] = csg[j * 32 + lane];
          f.dt[u] = dtg[j * 32 + lane];
        }
      }
      f.csl = csg[l];
    };
    // write cs*log2e, dt and cf[s] = e^{cs_r - cs_s} dt_s (r = last index of
    // s's 32-chunk) into the warp's table; returns this row's cs_l * log2e
    auto commit = [&](const Pref &f) -> float {
      __syncwarp();  // every lane is done reading the previous head's table
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = hf + 2 * u;
        if (j <= jd) {
          const int s = j * 32 + lane;
          const float v = f.cs[u] * kLog2e;
          const float vr = __shfl_sync(0xffffffffu, v, 31);
          wcs[s] = v;
          wdt[s] = f.dt[u];
          wcf[s] = ex2(vr - v) * f.dt[u];
        }
      }
      __syncwarp();
      return f.csl * kLog2e;
    };
    // M = G * decay * dt into the smem M buffer (K-major, SWIZZLE_128B)
    auto build_m = [&](float csl) {
      auto emit = [&](int s0, const uint32_t(&pk)[16]) {
        uint8_t *blk = mbuf + (s0 >> 6) * 16384;
        const int ch0 = (s0 & 63) >> 3;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          *reinterpret_cast<uint4 *>(blk + sw128_off(row, ch0 + cc)) =
              make_uint4(pk[4 * cc], pk[4 * cc + 1], pk[4 * cc + 2], pk[4 * cc + 3]);
      };
      auto off_diag = [&](int s0, const uint32_t(&r)[32], uint32_t(&pk)[16]) {
        const float rf = ex2(csl - wcs[s0 + 31]);
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float m0 = __uint_as_float(r[e]) * rf * wcf[s0 + e];
          const float m1 = __uint_as_float(r[e + 1]) * rf * wcf[s0 + e + 1];
          __nv_bfloat162 v = __floats2bfloat162_rn(m0, m1);
          pk[e >> 1] = *reinterpret_cast<uint32_t *>(&v);
        }
      };
      int j = hf;
      for (; j + 2 < jd; j += 4) {  // two off-diagonal chunks, both TMEM loads in flight
        uint32_t r0[32], r1[32], pk[16];
        sm100::tmem_ld32(tmem + lane_off + TM_G + j * 32, r0);
        sm100::tmem_ld32(tmem + lane_off + TM_G + (j + 2) * 32, r1);
        sm100::tmem_ld_wait();
        off_diag(j * 32, r0, pk);
        emit(j * 32, pk);
        off_diag((j + 2) * 32, r1, pk);
        emit((j + 2) * 32, pk);
      }
      for (; j <= jd; j += 2) {
        uint32_t r[32], pk[16];
        sm100::tmem_ld32(tmem + lane_off + TM_G + j * 32, r);
        sm100::tmem_ld_wait();
        const int s0 = j * 32;
        if (j < jd) {
          off_diag(s0, r, pk);
        } else {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int s = s0 + e;
            const float m0 = s <= l ? __uint_as_float(r[e]) * ex2(csl - wcs[s]) * wdt[s] : 0.f;
            const float m1 =
                s + 1 <= l ? __uint_as_float(r[e + 1]) * ex2(csl - wcs[s + 1]) * wdt[s + 1] : 0.f;
            __nv_bfloat162 v = __floats2bfloat162_rn(m0, m1);
            pk[e >> 1] = *reinterpret_cast<uint32_t *>(&v);
          }
        }
        emit(s0, pk);
      }
      for (; j < NS / 32; j += 2) {  // chunks above the diagonal are zero
        const uint32_t zpk[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        emit(j * 32, zpk);
      }
      sm100::fence_proxy_async();
      sm100::tc_fence_before();
      sm100::mbar_arrive(bar_m);
    };

    Pref nxt;
    fetch(0, nxt);
    float csl = commit(nxt);
    sm100::mbar_wait(bar_g, 0);
    sm100::tc_fence_after();
    build_m(csl);
    const int pc = hf * 32;
    for (int i = 0; i < p.HG; ++i) {
      const int buf = i & 1, h = h0 + i;
      if (i + 1 < p.HG) fetch(i + 1, nxt);  // global loads in flight during the wait
      uint4 xv[4], zv[4];                    // x (D skip) and z (gate) rows of head i
      const uint4 *xg = reinterpret_cast<const uint4 *>(xrow + h * TC_P + pc);
      const uint4 *zg = reinterpret_cast<const uint4 *>(zrow + h * TC_P + pc);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        xv[cc] = xg[cc];
        zv[cc] = zg[cc];
      }
      const float el = ex2(csl);
      const float Dh = p.D[h];
      sm100::mbar_wait(&bar_y[buf], (i >> 1) & 1);  // MMA(i) done: M buffer free
      sm100::tc_fence_after();
      if (i + 1 < p.HG) {
        csl = commit(nxt);
        build_m(csl);                                 // tensor core starts head i+1
      }
      // ---- epilogue(i) on columns p in [32 hf, 32 hf + 32), overlapping MMA(i+1)
      const uint32_t ydt = tmem + lane_off + TM_Y + buf * 128 + pc;
      uint32_t yd[32], yo[32];
      sm100::tmem_ld32(ydt, yd);
      sm100::tmem_ld32(ydt + 64, yo);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&yfree[buf]);
      const __nv_bfloat162 *xe = reinterpret_cast<const __nv_bfloat162 *>(xv);
      const __nv_bfloat162 *ze = reinterpret_cast<const __nv_bfloat162 *>(zv);
      uint32_t out[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float2 xf = __bfloat1622float2(xe[j]);
        const float2 zf = __bfloat1622float2(ze[j]);
        const float y0 = __uint_as_float(yd[2 * j]) + el * __uint_as_float(yo[2 * j]) + Dh * xf.x;
        const float y1 =
            __uint_as_float(yd[2 * j + 1]) + el * __uint_as_float(yo[2 * j + 1]) + Dh * xf.y;
        const float u0 = y0 * silu_fast(zf.x), u1 = y1 * silu_fast(zf.y);
        ssq += u0 * u0 + u1 * u1;
        __nv_bfloat162 v = __floats2bfloat162_rn(u0, u1);
        out[j] = *reinterpret_cast<uint32_t *>(&v);
      }
      if (valid) {
        bf16 *urow = p.u_out + ((long)b * p.T + t) * p.d_inner + h * TC_P + pc;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          *reinterpret_cast<uint4 *>(urow + cc * 8) =
              make_uint4(out[4 * cc], out[4 * cc + 1], out[4 * cc + 2], out[4 * cc + 3]);
      }
    }
    if (hf == 1) sq_s[row] = ssq;
    named_bar(1, OUT_MATH);
    if (hf == 0 && valid) p.ssq[((long)b * p.T + t) * p.NG + g] = ssq + sq_s[row];
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem);
  }
}

}  // namespace ssd200
