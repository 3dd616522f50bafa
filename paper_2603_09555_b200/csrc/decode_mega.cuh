// Persistent decode step (bf16 mode, batch <= DEC_MAX_B): one cooperative
// kernel runs the whole token step — every layer's in_proj / SSM update /
// out_proj and the tied head — decode.py:77-144.
//
// One CTA per SM.  Warp 8 is a producer that streams, in order, this CTA's
// row groups of every weight matrix the step touches (W_in[0], W_out[0],
// W_in[1], ..., E) with cp.async.bulk into a 3-deep 64 KB smem ring.  The
// weights never depend on activations, so the producer runs ahead across the
// grid barriers and HBM stays busy while the consumers synchronise.
// Warps 0..7 consume: phases separated by a sense-reversing grid barrier
//   P1  u = h_lp . W_in^T + conv window / SiLU / dt epilogue   (per row group)
//   P2  SSM state update + y + D skip + gate, sum u^2          (per (b, h, row split))
//   P3  hidden += rstd * (u . W_out'^T), bf16 shadow           (per row group)
//   H   logits = rmsnorm(hidden) . E^T, argmax partials; last barrier; pick.
#pragma once

#include "common.cuh"
#include "decode.cuh"

namespace ssd200 {

constexpr int MEGA_CW = 16;                    // consumer warps
constexpr int MEGA_CT = MEGA_CW * 32;          // consumer threads
constexpr int MEGA_THREADS = MEGA_CT + 32;     // + one producer warp
constexpr uint32_t MEGA_STAGE = 64 * 1024;
constexpr int MEGA_STAGES = 3;  // ring capacity; `stages` (2 or 3) is used

struct MegaArgs {
  int B, L, V, stages;
  int d_model, d_inner, conv_dim, d_in_proj, H, P, G, N, k, PS;
  float eps, dt_lo, dt_hi;
  const ssd200_layer_t *layers;  // device array [L]
  const bf16 *E;                 // (V, d_model)
  const float *final_w;
  float *hidden;     // (B, d_model)
  bf16 *hidden_lp;   // (B, d_model)
  float *ssm;        // (L, B, H, P, N) in place
  float *conv;       // (L, B, conv_dim, k-1) in place
  float *z, *act, *dt;  // scratch (B, d_inner) / (B, conv_dim) / (B, H)
  bf16 *u;           // (B, d_inner)
  float *usq;        // (B, d_inner) u^2 per element (summed by the out_proj prologue)
  float *logits;     // (B, V) or null
  float *amax_val;   // (grid, B)
  int *amax_idx;
  int64_t *argmax_out;  // (B) or null
  unsigned *bar_count, *bar_epoch;
  unsigned long long *trace;  // debug: per-phase %globaltimer stamps of CTA 0 (or null)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slot layout: [l*8 + k] consumer stamps, [4096 + m] producer stamps
#define MEGA_TRACE(slot)                                                   \
  do {                                                                     \
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[slot] = gtimer(); \
  } while (0)

// grid barrier: every CTA adds 1 (fire-and-forget release reduction) and
// waits until the counter reaches (index+1) * gridDim.  The counter is zeroed
// by mega_embed before every launch.  Only the 256 consumer threads call it.
__device__ __forceinline__ void mega_grid_sync(const MegaArgs &a, unsigned &index) {
  named_barrier_sync(1, MEGA_CT);
  if (threadIdx.x == 0) {
    const unsigned target = (++index) * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar_count) : "memory");
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(a.bar_count) : "memory");
    } while (cur < target);
  }
  named_barrier_sync(1, MEGA_CT);
}

// token embedding + barrier reset, launched right before decode_mega
__global__ void mega_embed(const int64_t *__restrict__ tok, const bf16 *__restrict__ E,
                           int d_model, float *__restrict__ hid, bf16 *__restrict__ hid_lp,
                           unsigned *bar_count) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *bar_count = 0u;
  const int r = blockIdx.x;
  const bf16 *src = E + (size_t)tok[r] * d_model;
  for (int c = threadIdx.x; c < d_model; c += blockDim.x) {
    const bf16 v = src[c];
    hid[(size_t)r * d_model + c] = __bfloat162float(v);
    hid_lp[(size_t)r * d_model + c] = v;
  }
}

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// L2 prefetch of a large contiguous range in <= 1 MB pieces (16-byte granular)
__device__ __forceinline__ void prefetch_range(const void *p, size_t bytes) {
  const char *c = static_cast<const char *>(p);
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(c) & ~(uintptr_t)15;
  size_t n = (bytes + (reinterpret_cast<uintptr_t>(c) - a0) + 15) & ~(size_t)15;
  const char *q = reinterpret_cast<const char *>(a0);
  while (n) {
    const uint32_t chunk = n > (1u << 20) ? (1u << 20) : (uint32_t)n;
    prefetch_l2(q, chunk);
    q += chunk;
    n -= chunk;
  }
}

// this CTA's share [g0, g1) of `groups` row groups
__device__ __forceinline__ void mega_share(int groups, int &g0, int &g1) {
  g0 = (int)((long)groups * blockIdx.x / gridDim.x);
  g1 = (int)((long)groups * (blockIdx.x + 1) / gridDim.x);
}

// rows per 64 KB stage for reduction length K (bf16)
__device__ __forceinline__ int mega_rows(int K) { return (int)(MEGA_STAGE / (K * 2)); }

// BT: batch rows computed (a.B rounded up to 1, 2, 4 or 8; extra rows are zero)
template <int BT>
__global__ void __launch_bounds__(MEGA_THREADS, 1) decode_mega(MegaArgs a) {
  extern __shared__ __align__(128) uint8_t msm[];
  __shared__ __align__(8) uint64_t full[MEGA_STAGES], empty[MEGA_STAGES];
  __shared__ float s_scale[DEC_MAX_B];
  __shared__ float s_best[MEGA_CW][DEC_MAX_B];
  __shared__ int s_bidx[MEGA_CW][DEC_MAX_B];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int B = a.B;
  uint8_t *ring = msm;
  const int S = a.stages;
  bf16 *xs = reinterpret_cast<bf16 *>(msm + (size_t)S * MEGA_STAGE);  // (B, K<=d_inner)
  if (threadIdx.x == 0) {
    for (int s = 0; s < MEGA_STAGES; ++s) {
      mbar_init_s(&full[s], 1);
      mbar_init_s(&empty[s], MEGA_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == MEGA_CW) {
    // ------------------------------------------------ producer: the weight stream
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      auto stream = [&](const bf16 *W, int N, int K) {
        const int rows = mega_rows(K);
        const int groups = (N + rows - 1) / rows;
        int g0, g1;
        mega_share(groups, g0, g1);
        for (int gi = g0; gi < g1; ++gi) {
          const int r0 = gi * rows, nr = min(rows, N - r0);
          mbar_wait_s(&empty[s], ph ^ 1);
          mbar_expect_s(&full[s], (uint32_t)nr * K * 2);
          for (int r = 0; r < nr; ++r)
            bulk_g2s(ring + (size_t)s * MEGA_STAGE + (size_t)r * K * 2, W + (size_t)(r0 + r) * K,
                     (uint32_t)K * 2, &full[s]);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      };
      // L2 prefetch of this CTA's share of one layer (weights + SSM state rows):
      // HBM keeps streaming one layer ahead of the smem ring, whatever the
      // consumers are waiting on.
      auto share_bytes = [&](int N, int K, size_t &off, size_t &len) {
        const int rows = mega_rows(K);
        const int groups = (N + rows - 1) / rows;
        int g0, g1;
        mega_share(groups, g0, g1);
        const int r0 = g0 * rows, r1 = min(N, g1 * rows);
        off = (size_t)r0 * K * 2;
        len = r1 > r0 ? (size_t)(r1 - r0) * K * 2 : 0;
      };
      auto prefetch_layer = [&](int l) {
        size_t off, len;
        share_bytes(a.d_in_proj, a.d_model, off, len);
        if (len) prefetch_range(static_cast<const char *>(a.layers[l].W_in) + off, len);
        share_bytes(a.d_model, a.d_inner, off, len);
        if (len) prefetch_range(static_cast<const char *>(a.layers[l].W_out) + off, len);
        const long rows_tot = (long)a.B * a.H * a.P;
        const long q0 = rows_tot * blockIdx.x / gridDim.x, q1 = rows_tot * (blockIdx.x + 1) / gridDim.x;
        if (q1 > q0)
          prefetch_range(a.ssm + ((size_t)l * rows_tot + q0) * a.N, (size_t)(q1 - q0) * a.N * 4);
      };
      prefetch_layer(0);
      for (int l = 0; l < a.L; ++l) {
        if (l + 1 < a.L) prefetch_layer(l + 1);
        stream(static_cast<const bf16 *>(a.layers[l].W_in), a.d_in_proj, a.d_model);
        if (a.trace && blockIdx.x == 0) a.trace[4096 + 2 * l] = gtimer();
        stream(static_cast<const bf16 *>(a.layers[l].W_out), a.d_model, a.d_inner);
        if (a.trace && blockIdx.x == 0) a.trace[4096 + 2 * l + 1] = gtimer();
      }
      {
        size_t off, len;
        share_bytes(a.V, a.d_model, off, len);  // the tied head's share of E
        if (len) prefetch_range(reinterpret_cast<const char *>(a.E) + off, len);
      }
      stream(a.E, a.V, a.d_model);
      if (a.trace && blockIdx.x == 0) a.trace[4096 + 2 * a.L] = gtimer();
    }
    return;
  }

  // ------------------------------------------------ consumers (warps 0..7)
  unsigned bar_idx = 0;
  int s = 0;
  uint32_t ph = 0;
  float best[DEC_MAX_B];
  int bidx[DEC_MAX_B];
#pragma unroll
  for (int b = 0; b < DEC_MAX_B; ++b) {
    best[b] = -INFINITY;
    bidx[b] = 0x7fffffff;
  }
  // one GEMV phase over this CTA's row groups; epi(n, b, v) per (row, batch)
  auto gemv = [&](int N, int K, auto &&pre, auto &&epi) {
    const int rows = mega_rows(K);
    const int groups = (N + rows - 1) / rows;
    const int kchunks = K / 256;
    int g0, g1;
    mega_share(groups, g0, g1);
    for (int gi = g0; gi < g1; ++gi) {
      const uint8_t *stage = ring + (size_t)s * MEGA_STAGE;
      const int nrows = min(rows, N - gi * rows);
      bool waited = false;
      for (int rr = warp; rr < rows; rr += MEGA_CW) {
        const int n = gi * rows + rr;
        const bool ok = rr < nrows;
        auto e = pre(n, ok);
        if (!waited) {
          mbar_wait_s(&full[s], ph);
          waited = true;
        }
        if (ok) {
          // 4 chunks of loads in flight, 4 independent accumulators per batch row
          float acc[BT][4];
#pragma unroll
          for (int b = 0; b < BT; ++b)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[b][u] = 0.f;
          const uint4 *wr = reinterpret_cast<const uint4 *>(stage + (size_t)rr * K * 2) + lane;
          const uint4 *xr = reinterpret_cast<const uint4 *>(xs) + lane;
          const int kq = K / 8;  // uint4 per row
          for (int c0 = 0; c0 < kchunks; c0 += 4) {
            uint4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c0 + u < kchunks) w[u] = wr[(c0 + u) * 32];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c0 + u < kchunks) {
#pragma unroll
                for (int b = 0; b < BT; ++b)
                  acc[b][u] += dot8(w[u], xr[(size_t)b * kq + (c0 + u) * 32]);
              }
          }
          float v = 0.f;
#pragma unroll
          for (int b = 0; b < BT; ++b) {
            const float t = warp_sum((acc[b][0] + acc[b][1]) + (acc[b][2] + acc[b][3]));
            if (lane == b) v = t;
          }
          if (lane < B) epi(n, lane, v, e);
        }
      }
      if (!waited) mbar_wait_s(&full[s], ph);
      __syncwarp();
      if (lane == 0) mbar_arrive_s(&empty[s]);
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    }
  };
  struct NoPre {
    float old, w0, w1, w2, w3, c0, c1, c2, bias;
  };

  for (int l = 0; l < a.L; ++l) {
    const ssd200_layer_t lw = a.layers[l];
    const float *conv_w = static_cast<const float *>(lw.conv_w);
    const float *conv_b = static_cast<const float *>(lw.conv_b);
    const float *dt_bias = static_cast<const float *>(lw.dt_bias);
    float *conv = a.conv + (size_t)l * B * a.conv_dim * (a.k - 1);
    // ---------------- P1: in_proj + conv / dt epilogue
    MEGA_TRACE(l * 8 + 0);
    {
      const uint4 *src = reinterpret_cast<const uint4 *>(a.hidden_lp);
      uint4 *dst = reinterpret_cast<uint4 *>(xs);
      for (int i = threadIdx.x; i < BT * a.d_model / 8; i += MEGA_CT)
        dst[i] = i < B * a.d_model / 8 ? src[i] : make_uint4(0, 0, 0, 0);
      named_barrier_sync(1, MEGA_CT);
      MEGA_TRACE(l * 8 + 1);
      gemv(
          a.d_in_proj, a.d_model,
          [&](int n, bool ok) {
            NoPre e{};
            if (ok && lane < B && a.k == 4 && n >= a.d_inner && n < a.d_inner + a.conv_dim) {
              const int ch = n - a.d_inner;
              const float *ci = conv + ((size_t)lane * a.conv_dim + ch) * 3;
              e.c0 = ci[0];
              e.c1 = ci[1];
              e.c2 = ci[2];
              e.w0 = conv_w[ch * 4];
              e.w1 = conv_w[ch * 4 + 1];
              e.w2 = conv_w[ch * 4 + 2];
              e.w3 = conv_w[ch * 4 + 3];
              e.bias = conv_b[ch];
            }
            return e;
          },
          [&](int n, int b, float v, const NoPre &e) {
            if (n < a.d_inner) {
              a.z[(size_t)b * a.d_inner + n] = v;
            } else if (n < a.d_inner + a.conv_dim) {
              const int ch = n - a.d_inner, km = a.k - 1;
              float *co = conv + ((size_t)b * a.conv_dim + ch) * km;
              if (a.k == 4) {  // taps oldest first (numerics.py:187-188)
                const float t = e.c0 * e.w0 + e.c1 * e.w1 + e.c2 * e.w2 + v * e.w3;
                a.act[(size_t)b * a.conv_dim + ch] = silu(t + e.bias);
                co[0] = e.c1;
                co[1] = e.c2;
                co[2] = v;
              } else {
                float win[16];
                for (int j = 0; j < km; ++j) win[j] = co[j];
                win[km] = v;
                float t = 0.f;
                for (int j = 0; j <= km; ++j) t += win[j] * conv_w[(size_t)ch * a.k + j];
                a.act[(size_t)b * a.conv_dim + ch] = silu(t + conv_b[ch]);
                for (int j = 0; j < km; ++j) co[j] = win[j + 1];
              }
            } else {
              const int h = n - a.d_inner - a.conv_dim;
              a.dt[(size_t)b * a.H + h] = clamp_(softplus(v + dt_bias[h]), a.dt_lo, a.dt_hi);
            }
          });
    }
    MEGA_TRACE(l * 8 + 2);
    if (a.trace && l == 1 && threadIdx.x == 0) a.trace[5000 + blockIdx.x] = gtimer();
    mega_grid_sync(a, bar_idx);
    if (a.trace && l == 1 && threadIdx.x == 0) a.trace[5200 + blockIdx.x] = gtimer();
    MEGA_TRACE(l * 8 + 3);
    // ---------------- P2: SSM step + D skip + gate, one warp per (b, h, p) row
    {
      const float *A = static_cast<const float *>(lw.a);
      const float *Dv = static_cast<const float *>(lw.D);
      float *ssm = a.ssm + (size_t)l * B * a.H * a.P * a.N;
      // stage B / C of every (batch row, group): G * N <= 256 floats each
      float *sbc = reinterpret_cast<float *>(xs);  // (B, 2, G*N)
      const int gn = a.G * a.N;
      for (int i = threadIdx.x; i < B * 2 * gn; i += MEGA_CT) {
        const int b = i / (2 * gn), j = i % (2 * gn);
        sbc[i] = a.act[(size_t)b * a.conv_dim + a.d_inner + j];
      }
      named_barrier_sync(1, MEGA_CT);
      const int total = B * a.H * a.P;
      const int hpg = a.H / a.G;
      // contiguous rows per CTA (their state was L2-prefetched by the producer)
      const int q0 = (int)((long)total * blockIdx.x / gridDim.x);
      const int q1 = (int)((long)total * (blockIdx.x + 1) / gridDim.x);
      for (int r = q0 + warp; r < q1; r += MEGA_CW) {
        const int b = r / (a.H * a.P);
        const int hp = r % (a.H * a.P);
        const int h = hp / a.P, pp = hp % a.P;
        const int g = h / hpg;
        const float *bs = sbc + (size_t)b * 2 * gn + g * a.N;
        const float *cs = sbc + (size_t)b * 2 * gn + gn + g * a.N;
        const float dt = a.dt[(size_t)b * a.H + h];
        const float xv = a.act[(size_t)b * a.conv_dim + h * a.P + pp];
        const float zv = a.z[(size_t)b * a.d_inner + h * a.P + pp];
        const float decay = expf(A[h] * dt);  // decode.py:126-129
        const float dx = dt * xv;
        float4 *st = reinterpret_cast<float4 *>(ssm + ((((size_t)b * a.H + h) * a.P) + pp) * a.N);
        float acc = 0.f;
        for (int n4 = lane; n4 < a.N / 4; n4 += 32) {
          float4 hv = st[n4];
          const int n = n4 * 4;
          hv.x = decay * hv.x + dx * bs[n];
          hv.y = decay * hv.y + dx * bs[n + 1];
          hv.z = decay * hv.z + dx * bs[n + 2];
          hv.w = decay * hv.w + dx * bs[n + 3];
          st[n4] = hv;
          acc = fmaf(cs[n], hv.x, acc);
          acc = fmaf(cs[n + 1], hv.y, acc);
          acc = fmaf(cs[n + 2], hv.z, acc);
          acc = fmaf(cs[n + 3], hv.w, acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) {
          const float y = acc + Dv[h] * xv;  // decode.py:132
          const float uu = y * silu(zv);
          a.u[(size_t)b * a.d_inner + h * a.P + pp] = __float2bfloat16_rn(uu);
          a.usq[(size_t)b * a.d_inner + h * a.P + pp] = uu * uu;
        }
      }
    }
    MEGA_TRACE(l * 8 + 4);
    mega_grid_sync(a, bar_idx);
    MEGA_TRACE(l * 8 + 5);
    // ---------------- P3: out_proj + norm row scale + residual
    {
      const uint4 *src = reinterpret_cast<const uint4 *>(a.u);
      uint4 *dst = reinterpret_cast<uint4 *>(xs);
      for (int i = threadIdx.x; i < BT * a.d_inner / 8; i += MEGA_CT)
        dst[i] = i < B * a.d_inner / 8 ? src[i] : make_uint4(0, 0, 0, 0);
      if (warp < B) {
        const float4 *q = reinterpret_cast<const float4 *>(a.usq + (size_t)warp * a.d_inner);
        float t = 0.f;
        for (int j = lane; j < a.d_inner / 4; j += 32) {
          const float4 v = q[j];
          t += (v.x + v.y) + (v.z + v.w);
        }
        t = warp_sum(t);
        if (lane == 0) s_scale[warp] = 1.f / sqrtf(t / (float)a.d_inner + a.eps);
      }
      named_barrier_sync(1, MEGA_CT);
      MEGA_TRACE(l * 8 + 6);
      gemv(
          a.d_model, a.d_inner,
          [&](int n, bool ok) {
            NoPre e{};
            if (ok && lane < B) e.old = a.hidden[(size_t)lane * a.d_model + n];
            return e;
          },
          [&](int n, int b, float v, const NoPre &e) {
            const float nv = e.old + s_scale[b] * v;
            a.hidden[(size_t)b * a.d_model + n] = nv;
            a.hidden_lp[(size_t)b * a.d_model + n] = __float2bfloat16_rn(nv);
          });
    }
    MEGA_TRACE(l * 8 + 7);
    mega_grid_sync(a, bar_idx);
  }
  MEGA_TRACE(4000);
  // ---------------- head: final RMSNorm + tied head + argmax partials
  {
    if (warp < B) {
      const float4 *hr = reinterpret_cast<const float4 *>(a.hidden + (size_t)warp * a.d_model);
      float ss = 0.f;
      for (int k = lane; k < a.d_model / 4; k += 32) {
        const float4 v = hr[k];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
      ss = warp_sum(ss);
      if (lane == 0) s_scale[warp] = 1.f / sqrtf(ss / (float)a.d_model + a.eps);
    }
    named_barrier_sync(1, MEGA_CT);
    for (int i = threadIdx.x; i < BT * a.d_model; i += MEGA_CT) {
      const int b = i / a.d_model, k = i % a.d_model;
      xs[i] = b < B ? __float2bfloat16_rn(a.hidden[(size_t)b * a.d_model + k] * s_scale[b] *
                                          a.final_w[k])
                    : __float2bfloat16_rn(0.f);
    }
    named_barrier_sync(1, MEGA_CT);
    gemv(
        a.V, a.d_model, [&](int, bool) { return NoPre{}; },
        [&](int n, int b, float v, const NoPre &) {
          if (a.logits) a.logits[(size_t)b * a.V + n] = v;
#pragma unroll
          for (int bb = 0; bb < DEC_MAX_B; ++bb)
            if (bb == b && v > best[bb]) {  // rows ascend per warp: strict > keeps the lowest id
              best[bb] = v;
              bidx[bb] = n;
            }
        });
#pragma unroll
    for (int bb = 0; bb < DEC_MAX_B; ++bb)
      if (lane == bb) {
        s_best[warp][bb] = best[bb];
        s_bidx[warp][bb] = bidx[bb];
      }
    named_barrier_sync(1, MEGA_CT);
    if (threadIdx.x < B) {
      const int bb = threadIdx.x;
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int w = 0; w < MEGA_CW; ++w) {
        const float ov = s_best[w][bb];
        const int oi = s_bidx[w][bb];
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      a.amax_val[blockIdx.x * B + bb] = bv;
      a.amax_idx[blockIdx.x * B + bb] = bi;
    }
  }
  MEGA_TRACE(4001);
  if (a.argmax_out) {
    mega_grid_sync(a, bar_idx);
    if (blockIdx.x == 0 && warp < B) {
      const int b = warp;
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int i = lane; i < (int)gridDim.x; i += 32) {
        const float v = a.amax_val[i * B + b];
        const int j = a.amax_idx[i * B + b];
        if (v > bv || (v == bv && j < bi)) {
          bv = v;
          bi = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) a.argmax_out[b] = bi == 0x7fffffff ? 0 : bi;
    }
  }
}

}  // namespace ssd200
