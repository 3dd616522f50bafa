// Tensor-core chunked SSD scan for the bf16 mode at the production head
// dims (P = 64, N = 128, L = 256, G = 1) — ssd.py:139-257 restated for
// tcgen05 / TMEM / TMA, with the D skip and the gate of the gated RMSNorm
// (model.py:166-167) fused into the output epilogue.
//
//   ssd_tc_cumsum  cs = inclusive cumsum of a*dt per (b, h, chunk)        [ssd.py:244-245]
//   ssd_tc_state   S_c^T (N x P) = B_c^T . (X * dt * e^{cs_end - cs})     [ssd.py:152-160]
//                  one 128x64x256 UMMA per head, A = B (MN-major), B = X~ (MN-major)
//   ssd_tc_pass    s_c = e^{cs_end,c} s_{c-1} + S_c, O(Nc) per (b, h)     [ssd.py:163-184]
//   ssd_tc_out     per (b, chunk, 128-row tile R, head group):
//                  G = C_R . B^T  (once, shared by every head: G = 1)      [ssd.py:147]
//                  per head: M = G * e^{cs_l - cs_s} * dt_s (s <= l) -> bf16 smem,
//                  Ydiag = M . X   and   Yoff = C_R . prev^T  (two UMMAs) [ssd.py:148-149,196]
//                  y = Ydiag + e^{cs_l} Yoff + D x;  u = y * silu(z);  sum u^2
//                  -> u (bf16) and per-row partial sum u^2; the out_proj GEMM
//                  applies rsqrt(mean + eps) (norm_w folded into W_out).
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace ssd200 {

constexpr int TC_P = 64, TC_N = 128, TC_L = 256;

struct TcSsdArgs {
  int B, T, H, Nc, NG, HG;  // HG = heads per group = H / NG
  int interleave;           // ssd_tc_out block order (see there)
  int d_inner;
  const bf16 *z;      // gate, (rows, z_ld) — first d_inner columns of the in_proj output
  long z_ld;
  const float *dt;    // (rows, H)
  const float *a;     // (H)
  const float *D;     // (H)
  const float *init;  // (B, H, P, N) or null
  float *cs;          // (B, H, Nc*L)
  float *dtT;         // (B, H, Nc*L) dt transposed (0 past T)
  float *cs_end;      // (B, H, Nc)
  float *S;           // (B, Nc, H, P, N) f32: each chunk's own end state
  bf16 *prev;         // (B, Nc, H, N, P) bf16: state entering each chunk (transposed)
  float *final_state; // (B, H, P, N)
  bf16 *u_out;        // (rows, d_inner)
  float *ssq;         // (H/SSQ_SLICE * OUT_KW, rows) partial sums of u^2 per (head slice, column half)
};

__device__ __forceinline__ unsigned long long clk64() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// swizzled (SWIZZLE_128B) byte offset of 16-byte chunk `ch` (0..7) of row r
__device__ __forceinline__ uint32_t sw128_off(int r, int ch) {
  return (uint32_t)r * 128u + (uint32_t)((ch ^ (r & 7)) << 4);
}

// ------------------------------------------------------------------ conv1d
// Causal depthwise conv (k = 4) + SiLU over the xBC columns, numerics.py:169-189.
// One CTA = 256 channels x 64 tokens: one TMA load brings the [64+3, 256]
// bf16 tile (3-row history halo; rows before the buffer start are zero-filled)
// into smem; thread (quad q, quarter h) slides the window down channels
// 4q .. 4q+3 over rows [16h, 16h+16), restarting it at sequence starts.
constexpr int CONV_ROWS = 64, CONV_COLS = 256;

__global__ void __launch_bounds__(256) conv_silu_tma(const __grid_constant__ CUtensorMap tm_xbc,
                                                     const float *__restrict__ w_,
                                                     const float *__restrict__ bias,
                                                     bf16 *__restrict__ out, long ld_out, int T,
                                                     int C, long rows) {
  __shared__ __align__(128) bf16 tile[CONV_ROWS + 3][CONV_COLS];
  __shared__ __align__(8) uint64_t bar;
  const int c0 = blockIdx.x * CONV_COLS;
  const long r0 = (long)blockIdx.y * CONV_ROWS;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  griddep_launch();
  griddep_wait();
  if (threadIdx.x == 0) {
    sm100::mbar_arrive_expect_tx(&bar, (CONV_ROWS + 3) * CONV_COLS * 2);
    sm100::tma_load_2d(&tile[0][0], &tm_xbc, &bar, c0, (int)(r0 - 3));
  }
  // thread (quad qd, quarter qr): channels 4 qd .. 4 qd + 3 over rows [16 qr, 16 qr + 16)
  const int qd = threadIdx.x & 63, qr = threadIdx.x >> 6;
  const int c = c0 + 4 * qd;
  float w[4][4], bs[4] = {0.f, 0.f, 0.f, 0.f};
  const bool ok = c + 3 < C;
  if (ok) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 a = reinterpret_cast<const float4 *>(w_)[c + j];
      w[j][0] = a.x;
      w[j][1] = a.y;
      w[j][2] = a.z;
      w[j][3] = a.w;
      bs[j] = bias[c + j];
    }
  }
  sm100::mbar_wait(&bar, 0);
  if (!ok) return;
  auto ld4 = [&](int row, float (&v)[4]) {
    const uint2 u = *reinterpret_cast<const uint2 *>(&tile[row][4 * qd]);
    const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.x));
    const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.y));
    v[0] = lo.x;
    v[1] = lo.y;
    v[2] = hi.x;
    v[3] = hi.y;
  };
  const int i0 = qr * 16;  // first output row of this thread (tile row i0 + 3)
  long r = r0 + i0;
  int t = (int)(r % T);
  // window: x[t-3], x[t-2], x[t-1] from the tile rows i0, i0+1, i0+2 (masked at sequence start)
  float h3[4], h2[4], h1[4];
  ld4(i0, h3);
  ld4(i0 + 1, h2);
  ld4(i0 + 2, h1);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (t < 3) h3[j] = 0.f;
    if (t < 2) h2[j] = 0.f;
    if (t < 1) h1[j] = 0.f;
  }
#pragma unroll 4
  for (int i = 0; i < 16; ++i, ++r, ++t) {
    if (r >= rows) break;
    if (t == T) {  // next sequence: zero history
      t = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) h1[j] = h2[j] = h3[j] = 0.f;
    }
    float x[4], o[4];
    ld4(i0 + i + 3, x);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o[j] = silu_fast(w[j][0] * h3[j] + w[j][1] * h2[j] + w[j][2] * h1[j] + w[j][3] * x[j] + bs[j]);
      h3[j] = h2[j];
      h2[j] = h1[j];
      h1[j] = x[j];
    }
    const __nv_bfloat162 lo = __floats2bfloat162_rn(o[0], o[1]);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(o[2], o[3]);
    uint2 pk;
    pk.x = *reinterpret_cast<const uint32_t *>(&lo);
    pk.y = *reinterpret_cast<const uint32_t *>(&hi);
    *reinterpret_cast<uint2 *>(out + r * ld_out + c) = pk;
  }
}

// ------------------------------------------------------------------ cumsum
// grid (B*Nc, ceil(H/8)), 256 threads: one warp per (b, chunk, head).
__global__ __launch_bounds__(256) void ssd_tc_cumsum(TcSsdArgs p) {
  griddep_launch();
  griddep_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x / p.Nc, c = blockIdx.x % p.Nc;
  const int h = blockIdx.y * 8 + warp;
  if (h >= p.H) return;
  const float ah = p.a[h];
  float v[8], dv[8], run = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int t = c * TC_L + lane * 8 + j;
    const float d = t < p.T ? p.dt[((long)b * p.T + t) * p.H + h] : 0.f;
    dv[j] = d;
    run += ah * d;
    v[j] = run;
  }
  float *dtd = p.dtT + ((long)b * p.H + h) * ((long)p.Nc * TC_L) + (long)c * TC_L + lane * 8;
  *reinterpret_cast<float4 *>(dtd) = make_float4(dv[0], dv[1], dv[2], dv[3]);
  *reinterpret_cast<float4 *>(dtd + 4) = make_float4(dv[4], dv[5], dv[6], dv[7]);
  float tot = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float n = __shfl_up_sync(0xffffffffu, tot, o);
    if (lane >= o) tot += n;
  }
  const float excl = tot - run;
  float *dst = p.cs + ((long)b * p.H + h) * ((long)p.Nc * TC_L) + (long)c * TC_L + lane * 8;
#pragma unroll
  for (int j = 0; j < 8; ++j) dst[j] = v[j] + excl;
  if (lane == 31) p.cs_end[((long)b * p.H + h) * p.Nc + c] = tot;
}

// ------------------------------------------------------------------ chunk states
struct StateSmem {
  static constexpr uint32_t BT = 0;                 // B chunk as MN-major A: 2 x [256 l][64 n]
  static constexpr uint32_t X0 = 65536;             // 2 x [256 l][64 p]
  static constexpr uint32_t BAR = X0 + 2 * 32768;   // barriers
  static constexpr uint32_t TOTAL = BAR + 256 + 1024;
};

// grid (B*Nc*NG), 192 threads: warp0 TMA, warp1 MMA, warps 2-5 math.
__global__ void __launch_bounds__(192, 1)
    ssd_tc_state(const __grid_constant__ CUtensorMap tm_act, TcSsdArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bar_b = reinterpret_cast<uint64_t *>(sm + StateSmem::BAR);
  uint64_t *bar_x = bar_b + 1;     // [2] TMA X landed
  uint64_t *bar_xs = bar_b + 3;    // [2] X scaled by math
  uint64_t *bar_s = bar_b + 5;     // [2] accumulator ready
  uint64_t *xfree = bar_b + 7;     // [2] X buffer consumed by MMA
  uint64_t *tfree = bar_b + 9;     // [2] accumulator drained
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bar_b + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x % p.NG;
  const int bc = blockIdx.x / p.NG;
  const int b = bc / p.Nc, c = bc % p.Nc;
  const int h0 = g * p.HG;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_act);
    sm100::mbar_init(bar_b, 1);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&bar_x[i], 1);
      sm100::mbar_init(&bar_xs[i], 128);
      sm100::mbar_init(&bar_s[i], 1);
      sm100::mbar_init(&xfree[i], 1);
      sm100::mbar_init(&tfree[i], 4);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<128>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch();
  griddep_wait();

  if (warp == 0) {
    if (lane == 0) {
      sm100::mbar_arrive_expect_tx(bar_b, 65536);
      for (int j = 0; j < 2; ++j)
        for (int q = 0; q < 2; ++q)
          sm100::tma_load_3d(sm + StateSmem::BT + j * 32768 + q * 16384, &tm_act, bar_b,
                             p.d_inner + j * 64, c * TC_L + q * 128, b);
      for (int i = 0; i < p.HG; ++i) {
        const int buf = i & 1;
        sm100::mbar_wait(&xfree[buf], ((i >> 1) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&bar_x[buf], 32768);
        for (int q = 0; q < 2; ++q)
          sm100::tma_load_3d(sm + StateSmem::X0 + buf * 32768 + q * 16384, &tm_act, &bar_x[buf],
                             (h0 + i) * TC_P, c * TC_L + q * 128, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_bf16(128, TC_P, true, true);
      sm100::mbar_wait(bar_b, 0);
      const uint32_t a0 = sm100::smem_u32(sm + StateSmem::BT);
      for (int i = 0; i < p.HG; ++i) {
        const int buf = i & 1;
        sm100::mbar_wait(&bar_xs[buf], (i >> 1) & 1);
        sm100::mbar_wait(&tfree[buf], ((i >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
        const uint32_t x0 = sm100::smem_u32(sm + StateSmem::X0 + buf * 32768);
#pragma unroll
        for (int k = 0; k < TC_L / 16; ++k) {
          const uint64_t ad = sm100::sw128_desc(a0 + k * 2048, 32768, 1024);
          const uint64_t bd = sm100::sw128_desc(x0 + k * 2048, 32768, 1024);
          sm100::mma_bf16(tmem + buf * TC_P, ad, bd, idesc, k > 0);
        }
        sm100::mma_commit(&bar_s[buf]);
        sm100::mma_commit(&xfree[buf]);
      }
    }
  } else {
    const int tid = threadIdx.x - 64;  // 0..127
    const int q = warp & 3;
    const long csb = (long)p.Nc * TC_L;
    // scale X rows by dt_l * exp(cs_end - cs_l), in place (the row's 128 B
    // hold its 64 bf16 in swizzled order; a row-uniform scale ignores it)
    auto scale = [&](int i) {
      const int buf = i & 1, h = h0 + i;
      sm100::mbar_wait(&bar_x[buf], (i >> 1) & 1);
      const float *cs = p.cs + ((long)b * p.H + h) * csb + (long)c * TC_L;
      const float cend = p.cs_end[((long)b * p.H + h) * p.Nc + c];
      uint8_t *xb = sm + StateSmem::X0 + buf * 32768;
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int l = tid + rr * 128;
        const int t = c * TC_L + l;
        const float *dtr = p.dtT + ((long)b * p.H + h) * csb + (long)c * TC_L;
        // the same bf16 row weight and packed multiply as ssd_tc_chunkscan, so both
        // scan variants give bitwise-equal chunk states (batch invariance)
        const __nv_bfloat162 w2 = __float2bfloat162_rn(
            t < p.T ? dtr[l] * ex2((cend - cs[l]) * kLog2e) : 0.f);
        uint4 *row = reinterpret_cast<uint4 *>(xb + l * 128);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const int pc = (ch + l) & 7;  // lane-rotated chunk order: conflict-free phases
          uint4 v = row[pc];
          __nv_bfloat162 *e = reinterpret_cast<__nv_bfloat162 *>(&v);
#pragma unroll
          for (int j = 0; j < 4; ++j) e[j] = __hmul2(e[j], w2);
          row[pc] = v;
        }
      }
      sm100::fence_proxy_async();
      sm100::mbar_arrive(&bar_xs[buf]);
    };
    if (p.HG > 0) scale(0);
    for (int i = 0; i < p.HG; ++i) {
      if (i + 1 < p.HG) scale(i + 1);
      const int buf = i & 1, h = h0 + i;
      sm100::mbar_wait(&bar_s[buf], (i >> 1) & 1);
      sm100::tc_fence_after();
      const int n = q * 32 + lane;
      float *dst = p.S + ((((long)b * p.Nc + c) * p.H + h) * TC_P) * TC_N + n;
#pragma unroll
      for (int pc = 0; pc < TC_P; pc += 32) {
        uint32_t r[32];
        sm100::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * TC_P + pc, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[(long)(pc + j) * TC_N] = __uint_as_float(r[j]);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tfree[buf]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    sm100::tc_fence_after();
    sm100::tmem_dealloc<128>(tmem);
  }
}

// ------------------------------------------------------------------ state pass
// grid (B*H, P*N/256), 256 threads; sequential over chunks, loads batched.
__global__ __launch_bounds__(256) void ssd_tc_pass(TcSsdArgs p) {
  griddep_launch();
  griddep_wait();
  const int bh = blockIdx.x;
  const int b = bh / p.H, h = bh % p.H;
  const int e = blockIdx.y * 256 + threadIdx.x;
  constexpr int PN = TC_P * TC_N;
  float s = p.init ? p.init[(long)bh * PN + e] : 0.f;
  const float *ce = p.cs_end + (long)bh * p.Nc;
  for (int c0 = 0; c0 < p.Nc; c0 += 8) {
    float own[8], dec[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      if (c < p.Nc) {
        own[j] = p.S[(((long)b * p.Nc + c) * p.H + h) * PN + e];
        dec[j] = ce[c];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      if (c < p.Nc) {
        // prev is stored [n][p] per (b, c, h); e indexes S's [p][n] layout
        p.prev[(((long)b * p.Nc + c) * p.H + h) * PN + (e % TC_N) * TC_P + e / TC_N] =
            __float2bfloat16_rn(s);
        s = expf(dec[j]) * s + own[j];
      }
    }
  }
  p.final_state[(long)bh * PN + e] = s;
}

// ------------------------------------------------------------------ fused states + pass
// One CTA per (b, h) walks the chunks in order (ssd.py:152-184 fused):
//   S_c^T = B_c^T . (X_c * dt * e^{cs_end - cs})   (UMMA 128 x 64 x 256, TMEM)
//   prev_c = s ;  s = e^{cs_end,c} s + S_c          (running state in registers:
//                                                    thread n holds s[:, n])
// Two smem stages (B^T 64 KB + X 32 KB) and two TMEM accumulators pipeline
// chunk c+1's load/scale/MMA under chunk c's state update.  Eight math warps
// (two per TMEM lane quarter): each scales one X row per chunk and keeps half
// of one state row (32 of the 64 head columns) — the per-chunk critical path
// (scale, TMEM read-out, bf16 prev store, state update) is latency-bound, so
// more warps per scheduler shorten it.
constexpr int CHUNKSCAN_THREADS = 64 + 256;  // TMA warp, MMA warp, 8 math warps

struct ScanSmem {
  static constexpr uint32_t STG = 98304;  // Bt [2 n-blocks][256 l][64 n] + X [256 l][64 p]
  static constexpr uint32_t XO = 65536;
  static constexpr uint32_t BAR = 2 * STG;
  static constexpr uint32_t TOTAL = BAR + 256 + 1024;
};

// mc = CTAs per cluster (1 or 4): the heads h..h+3 of one batch row share every
// chunk's B tile, so with mc = 4 each CTA loads a quarter of it and multicasts it
// to the cluster (and a stage is refilled only once all four have consumed it).
__global__ void __launch_bounds__(CHUNKSCAN_THREADS, 1)
    ssd_tc_chunkscan(const __grid_constant__ CUtensorMap tm_act, TcSsdArgs p, int mc) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + ScanSmem::BAR);  // [2] TMA landed
  uint64_t *xsd = full + 2;    // [2] X scaled
  uint64_t *sfull = full + 4;  // [2] accumulator ready
  uint64_t *stfree = full + 6; // [2] stage consumed by the MMA
  uint64_t *tfree = full + 8;  // [2] accumulator drained
  uint32_t *tslot = reinterpret_cast<uint32_t *>(full + 10);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x / p.H, h = blockIdx.x % p.H;
  const int Nc = p.Nc;
  const long csb = (long)Nc * TC_L;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_act);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&xsd[i], 256);
      sm100::mbar_init(&sfull[i], 1);
      sm100::mbar_init(&stfree[i], mc);  // every CTA of the cluster frees the stage
      sm100::mbar_init(&tfree[i], 256);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<128>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  if (mc > 1) sm100::cluster_sync();  // barriers initialised cluster-wide before any multicast
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch();
  griddep_wait();
  const uint16_t mask = (uint16_t)((1u << mc) - 1u);
  const int crank = mc > 1 ? (int)sm100::cluster_rank() : 0;

  if (warp == 0) {
    if (lane == 0) {
      for (int c = 0; c < Nc; ++c) {
        const int st = c & 1;
        uint8_t *stg = sm + st * ScanSmem::STG;
        sm100::mbar_wait(&stfree[st], ((c >> 1) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&full[st], ScanSmem::STG);
        if (mc == 4) {  // this CTA's quarter of B, to all four CTAs
          const int j = crank >> 1, q = crank & 1;
          sm100::tma_load_3d_mc(stg + j * 32768 + q * 16384, &tm_act, &full[st],
                                p.d_inner + j * 64, c * TC_L + q * 128, b, mask);
        } else {
          for (int j = 0; j < 2; ++j)
            for (int q = 0; q < 2; ++q)
              sm100::tma_load_3d(stg + j * 32768 + q * 16384, &tm_act, &full[st],
                                 p.d_inner + j * 64, c * TC_L + q * 128, b);
        }
        for (int q = 0; q < 2; ++q)
          sm100::tma_load_3d(stg + ScanSmem::XO + q * 16384, &tm_act, &full[st], h * TC_P,
                             c * TC_L + q * 128, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_bf16(128, TC_P, true, true);
      for (int c = 0; c < Nc; ++c) {
        const int st = c & 1;
        const uint32_t par = (c >> 1) & 1;
        sm100::mbar_wait(&xsd[st], par);
        sm100::mbar_wait(&tfree[st], par ^ 1);
        sm100::tc_fence_after();
        const uint32_t a0 = sm100::smem_u32(sm + st * ScanSmem::STG);
        const uint32_t x0 = a0 + ScanSmem::XO;
#pragma unroll
        for (int k = 0; k < TC_L / 16; ++k) {
          const uint64_t ad = sm100::sw128_desc(a0 + k * 2048, 32768, 1024);
          const uint64_t bd = sm100::sw128_desc(x0 + k * 2048, 32768, 1024);
          sm100::mma_bf16(tmem + st * TC_P, ad, bd, idesc, k > 0);
        }
        sm100::mma_commit(&sfull[st]);
        if (mc > 1)
          sm100::mma_commit_mc(&stfree[st], mask);  // the stage may be refilled cluster-wide
        else
          sm100::mma_commit(&stfree[st]);
      }
    }
  } else {
    const int tid = threadIdx.x - 64;  // 0..255: X row in the scale step
    const int q = warp & 3;            // TMEM lane quarter
    const int half = (warp - 2) >> 2;  // state columns [32 half, 32 half + 32)
    const int n = q * 32 + lane;       // state row (TMEM lane)
    const float *csg = p.cs + ((long)b * p.H + h) * csb;
    const float *dtg = p.dtT + ((long)b * p.H + h) * csb;
    const float *ceg = p.cs_end + ((long)b * p.H + h) * Nc;
    // row weight w_l = dt_l e^{cs_end - cs_l} of a chunk: loaded one chunk ahead
    // so the global-load latency stays off the scale step
    struct RowW {
      float dt, cs, cend;
    };
    auto load_w = [&](int c, RowW &f) {
      if (c >= Nc) return;
      const long t = (long)c * TC_L + tid;
      f.dt = t < p.T ? dtg[t] : 0.f;
      f.cs = csg[t];
      f.cend = ceg[c];
    };
    auto scale = [&](int c, const RowW &f) {
      const int st = c & 1;
      sm100::mbar_wait(&full[st], (c >> 1) & 1);
      uint8_t *xb = sm + st * ScanSmem::STG + ScanSmem::XO;
      const int l = tid;
      const __nv_bfloat162 w2 = __float2bfloat162_rn(f.dt * ex2((f.cend - f.cs) * kLog2e));
      uint4 *row = reinterpret_cast<uint4 *>(xb + l * 128);
      // every 16-byte chunk of the row gets the same weight, so visit them in a
      // lane-rotated order (the 8 lanes of a shared-memory phase hit 8 bank
      // groups); all 8 loads are issued before the first multiply
      uint4 v[8];
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) v[ch] = row[(ch + l) & 7];
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {  // packed bf16 multiply (X is a bf16 MMA operand)
        __nv_bfloat162 *e = reinterpret_cast<__nv_bfloat162 *>(&v[ch]);
#pragma unroll
        for (int j = 0; j < 4; ++j) e[j] = __hmul2(e[j], w2);
      }
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) row[(ch + l) & 7] = v[ch];
      sm100::fence_proxy_async();
      sm100::mbar_arrive(&xsd[st]);
    };
    float s[32];
    const long sbase = ((long)b * p.H + h) * TC_P * TC_N + n;
#pragma unroll
    for (int pp = 0; pp < 32; ++pp)
      s[pp] = p.init ? p.init[sbase + (long)(32 * half + pp) * TC_N] : 0.f;
    // chunk k's weights live in wa (k even) / wb (k odd); chunk k+2's are fetched
    // right after scale(k), two chunks before they are needed
    RowW wa, wb;
    load_w(0, wa);
    load_w(1, wb);
    scale(0, wa);
    load_w(2, wa);
    float dnext = ceg[0];  // e^{cs_end} decay of the next chunk, loaded one chunk ahead
    for (int c = 0; c < Nc; ++c) {
      const float dlog = dnext;
      if (c + 1 < Nc) dnext = ceg[c + 1];
      if (c + 1 < Nc) {
        const int k = c + 1;
        if (k & 1) {
          scale(k, wb);
          load_w(k + 2, wb);
        } else {
          scale(k, wa);
          load_w(k + 2, wa);
        }
      }
      const int st = c & 1;
      const float decay = expf(dlog);
      sm100::mbar_wait(&sfull[st], (c >> 1) & 1);
      sm100::tc_fence_after();
      uint32_t r0[32];
      sm100::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + st * TC_P + 32 * half, r0);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&tfree[st]);
      // state entering chunk c, stored [n][p]: this thread's 32 values are contiguous
      uint4 *pv = reinterpret_cast<uint4 *>(
          p.prev + ((((long)b * Nc + c) * p.H + h) * TC_N + n) * TC_P + 32 * half);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 v = __floats2bfloat162_rn(s[8 * g + 2 * e], s[8 * g + 2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t *>(&v);
        }
        pv[g] = make_uint4(w[0], w[1], w[2], w[3]);
      }
#pragma unroll
      for (int pp = 0; pp < 32; ++pp) s[pp] = decay * s[pp] + __uint_as_float(r0[pp]);
    }
#pragma unroll
    for (int pp = 0; pp < 32; ++pp) p.final_state[sbase + (long)(32 * half + pp) * TC_N] = s[pp];
  }
  __syncthreads();
  if (mc > 1) sm100::cluster_sync();  // no CTA leaves while peers may still signal it
  if (warp == 1) {
    __syncwarp();
    sm100::tc_fence_after();
    sm100::tmem_dealloc<128>(tmem);
  }
}

}  // namespace ssd200

#include "ssd_tc_out.cuh"
