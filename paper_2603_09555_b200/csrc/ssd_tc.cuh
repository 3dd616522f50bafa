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
  bf16 *prev;         // (B, Nc, H, P, N) bf16: state entering each chunk
  float *final_state; // (B, H, P, N)
  bf16 *u_out;        // (rows, d_inner)
  float *ssq;         // (rows, NG) partial sum of u^2
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// swizzled (SWIZZLE_128B) byte offset of 16-byte chunk `ch` (0..7) of row r
__device__ __forceinline__ uint32_t sw128_off(int r, int ch) {
  return (uint32_t)r * 128u + (uint32_t)((ch ^ (r & 7)) << 4);
}

// ------------------------------------------------------------------ cumsum
// grid (B*Nc, ceil(H/8)), 256 threads: one warp per (b, chunk, head).
__global__ __launch_bounds__(256) void ssd_tc_cumsum(TcSsdArgs p) {
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
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                            ~(uintptr_t)1023);
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
        const float w = t < p.T ? dtr[l] * ex2((cend - cs[l]) * kLog2e) : 0.f;
        uint4 *row = reinterpret_cast<uint4 *>(xb + l * 128);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint4 v = row[ch];
          __nv_bfloat162 *e = reinterpret_cast<__nv_bfloat162 *>(&v);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 f = __bfloat1622float2(e[j]);
            e[j] = __floats2bfloat162_rn(f.x * w, f.y * w);
          }
          row[ch] = v;
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
        p.prev[(((long)b * p.Nc + c) * p.H + h) * PN + e] = __float2bfloat16_rn(s);
        s = expf(dec[j]) * s + own[j];
      }
    }
  }
  p.final_state[(long)bh * PN + e] = s;
}

}  // namespace ssd200

#include "ssd_tc_out.cuh"
