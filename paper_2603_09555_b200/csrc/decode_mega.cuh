// Persistent decode step (bf16 mode, batch <= DEC_MAX_B): one cooperative
// kernel runs the whole token step — every layer's in_proj / SSM update /
// out_proj and the tied head — decode.py:77-144.
//
// One CTA per SM.  The last warp is a producer that streams, in order, this
// CTA's weight rows of every matrix the step touches (W_in[0], W_out[0],
// W_in[1], ..., E) with cp.async.bulk into a 64 KB-stage smem ring.  The
// weights never depend on activations, so the producer runs ahead across the
// synchronisation points and HBM stays busy while the consumers wait.
//
// Work split per layer (16 consumer warps):
//   A  each CTA owns a contiguous range of d_inner channels [k0, k1): it
//      computes the in_proj rows of its own z and x channels and of the dt of
//      the heads they touch, plus a 1/grid share of the B / C rows (streamed
//      first).  B / C go through the conv and are published to global memory
//      with a release-counter (no grid barrier); z, x (post conv) and dt stay
//      in shared memory.  Once every B / C row is published, the CTA runs the
//      SSM update of its own channels (h <- e^{a dt} h + dt x B, y = C.h + D x,
//      u = y silu(z)) with purely local inputs and writes u + its sum u^2.
//   -- grid barrier --
//   B  hidden += rstd * (u . W_out'^T), bf16 shadow (rows of d_model split over
//      CTAs).
//   -- grid barrier --
//   H  logits = rmsnorm(hidden) . E^T, argmax partials; last barrier; pick.
#pragma once

#include "common.cuh"
#include "decode.cuh"

namespace ssd200 {

constexpr int MEGA_CW = 16;                    // consumer warps
constexpr int MEGA_CT = MEGA_CW * 32;          // consumer threads
constexpr int MEGA_THREADS = MEGA_CT + 32;     // + one producer warp
constexpr uint32_t MEGA_STAGE = 64 * 1024;
constexpr int MEGA_STAGES = 3;  // ring capacity; `stages` (2 or 3) is used
constexpr int MEGA_MAX_NK = 64;   // own d_inner channels per CTA
constexpr int MEGA_MAX_DT = 16;   // heads touched by one CTA's channels

struct MegaArgs {
  int B, L, V, stages, pf_ahead;
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
  float *upart;      // (grid, B) per-CTA partial sums of u^2 of the current layer
  float *logits;     // (B, V) or null
  float *amax_val;   // (grid, B)
  int *amax_idx;
  int64_t *argmax_out;  // (B) or null
  unsigned *bar_count;
  unsigned *bc_flag;  // B / C rows published so far this step (release counter)
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
    if (a.trace && index == 4) a.trace[5400 + blockIdx.x] = gtimer();
#ifdef MEGA_DIAG_NOFENCE
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar_count) : "memory");
#else
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar_count) : "memory");
#endif
    // relaxed polling (no per-iteration fence), one acquire fence once it flips
    unsigned cur;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.bar_count) : "memory");
    } while (cur < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (a.trace && index == 4) a.trace[5600 + blockIdx.x] = gtimer();
  }
  named_barrier_sync(1, MEGA_CT);
}

// token embedding + barrier reset, launched right before decode_mega
__global__ void mega_embed(const int64_t *__restrict__ tok, const bf16 *__restrict__ E,
                           int d_model, float *__restrict__ hid, bf16 *__restrict__ hid_lp,
                           unsigned *bar_count) {
  if (blockIdx.x == 0 && threadIdx.x < 2) bar_count[threadIdx.x] = 0u;  // barrier + B/C flag
  const int r = blockIdx.x;
  const bf16 *src = E + (size_t)tok[r] * d_model;
  for (int c = threadIdx.x; c < d_model; c += blockDim.x) {
    const bf16 v = src[c];
    hid[(size_t)r * d_model + c] = __bfloat162float(v);
    hid_lp[(size_t)r * d_model + c] = v;
  }
}

// rows per 64 KB stage for reduction length K (bf16)
__device__ __forceinline__ int mega_rows(int K) { return (int)(MEGA_STAGE / (K * 2)); }

// This CTA's in_proj rows for one layer, in stream order: its share of the
// B / C rows first (other CTAs wait for them), then the dt rows of the heads
// its channels touch, then its z rows and x rows.
struct MegaOwn {
  int nbc, bc0, ndt, h_lo, nk, k0;
  __device__ MegaOwn(const MegaArgs &a) {
    const int gn2 = 2 * a.G * a.N;
    bc0 = (int)((long)gn2 * blockIdx.x / gridDim.x);
    nbc = (int)((long)gn2 * (blockIdx.x + 1) / gridDim.x) - bc0;
    k0 = (int)((long)a.d_inner * blockIdx.x / gridDim.x);
    nk = (int)((long)a.d_inner * (blockIdx.x + 1) / gridDim.x) - k0;
    h_lo = k0 / a.P;
    ndt = nk ? (k0 + nk - 1) / a.P - h_lo + 1 : 0;
  }
  __device__ int count() const { return nbc + ndt + 2 * nk; }
  __device__ int row(int i, const MegaArgs &a) const {
    if (i < nbc) return 2 * a.d_inner + bc0 + i;
    i -= nbc;
    if (i < ndt) return 2 * a.d_inner + 2 * a.G * a.N + h_lo + i;
    i -= ndt;
    return i < nk ? k0 + i : a.d_inner + k0 + (i - nk);
  }
};

// BT: batch rows computed (a.B rounded up to 1, 2, 4 or 8; extra rows are zero)
template <int BT>
__global__ void __launch_bounds__(MEGA_THREADS, 1) decode_mega(MegaArgs a) {
  extern __shared__ __align__(128) uint8_t msm[];
  __shared__ __align__(8) uint64_t full[MEGA_STAGES], empty[MEGA_STAGES];
  __shared__ float s_scale[DEC_MAX_B];
  __shared__ float s_best[MEGA_CW][DEC_MAX_B];
  __shared__ int s_bidx[MEGA_CW][DEC_MAX_B];
  __shared__ float s_z[DEC_MAX_B][MEGA_MAX_NK];  // own channels: gate z
  __shared__ float s_x[DEC_MAX_B][MEGA_MAX_NK];  // own channels: x after conv + SiLU
  __shared__ float s_dt[DEC_MAX_B][MEGA_MAX_DT];
  __shared__ float s_uu[DEC_MAX_B][MEGA_MAX_NK];  // own channels: u^2
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int B = a.B;
  uint8_t *ring = msm;
  const int S = a.stages;
  bf16 *xs = reinterpret_cast<bf16 *>(msm + (size_t)S * MEGA_STAGE);  // (B, K<=d_inner)
  const MegaOwn own(a);
  const int gn = a.G * a.N;
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
    // Segment j of the step: 2l = this CTA's W_in rows of layer l, 2l+1 = its
    // W_out share, 2L = its share of E; rows are bulk-copied into the ring.
    // With pf_ahead > 0 a second cursor runs pf_ahead stages ahead of the copies
    // and prefetches those stages into L2, so HBM keeps streaming while the ring
    // is full during the grid-wide synchronisations (bounded: prefetching a
    // whole layer ahead was measured to slow the step down).
    if (lane == 0) {
      int s = 0, pstage = 0;
      uint32_t ph = 0;
      const int nseg = 2 * a.L + 1;
      auto share = [&](int N, int &r0, int &nr) {  // this CTA's contiguous share of N rows
        r0 = (int)((long)N * blockIdx.x / gridDim.x);
        nr = (int)((long)N * (blockIdx.x + 1) / gridDim.x) - r0;
      };
      int r0_out, nr_out, r0_e, nr_e;
      share(a.d_model, r0_out, nr_out);
      share(a.V, r0_e, nr_e);
      auto seg_w = [&](int j) -> const bf16 * {
        return j == 2 * a.L ? a.E
                            : static_cast<const bf16 *>((j & 1) ? a.layers[j >> 1].W_out
                                                                : a.layers[j >> 1].W_in);
      };
      auto seg_k = [&](int j) { return (j < 2 * a.L && (j & 1)) ? a.d_inner : a.d_model; };
      auto seg_n = [&](int j) { return j == 2 * a.L ? nr_e : (j & 1) ? nr_out : own.count(); };
      auto seg_row = [&](int j, int i) {
        return j == 2 * a.L ? r0_e + i : (j & 1) ? r0_out + i : own.row(i, a);
      };
      // L2 prefetch cursor (segment pj, first row pi0), pq = its stage index
      int pj = 0, pi0 = 0, pq = 0, q = 0;
      auto pf_next = [&]() {
        while (pj < nseg && pi0 >= seg_n(pj)) {
          ++pj;
          pi0 = 0;
        }
        if (pj >= nseg) return false;
        const int K = seg_k(pj), nr = min(mega_rows(K), seg_n(pj) - pi0);
        const bf16 *W = seg_w(pj);
        for (int r = 0; r < nr;) {
          const int row0 = seg_row(pj, pi0 + r);
          int run = 1;
          while (r + run < nr && seg_row(pj, pi0 + r + run) == row0 + run) ++run;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(W + (size_t)row0 * K),
                       "r"((uint32_t)run * K * 2)
                       : "memory");
          r += run;
        }
        pi0 += nr;
        ++pq;
        return true;
      };
      for (int j = 0; j < nseg; ++j) {
        const bf16 *W = seg_w(j);
        const int K = seg_k(j), nrows = seg_n(j), per = mega_rows(K);
        for (int i0 = 0; i0 < nrows; i0 += per) {
          const int nr = min(per, nrows - i0);
          if (a.pf_ahead > 0) {
            if (pq <= q) {  // keep the prefetch cursor past this stage
              while (pq <= q && pf_next()) {
              }
            }
            while (pq <= q + a.pf_ahead && pf_next()) {
            }
          }
          ++q;
          mbar_wait_s(&empty[s], ph ^ 1);
          if (a.trace && blockIdx.x == 0 && pstage < 512) a.trace[6000 + pstage] = gtimer();
          ++pstage;
          mbar_expect_s(&full[s], (uint32_t)nr * K * 2);
          // one bulk copy per run of memory-contiguous rows (the TMA queue holds a
          // bounded number of copies in flight, so bigger copies mean more bytes)
          for (int r = 0; r < nr;) {
            const int row0 = seg_row(j, i0 + r);
            int run = 1;
            while (r + run < nr && seg_row(j, i0 + r + run) == row0 + run) ++run;
            bulk_g2s(ring + (size_t)s * MEGA_STAGE + (size_t)r * K * 2, W + (size_t)row0 * K,
                     (uint32_t)run * K * 2, &full[s]);
            r += run;
          }
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        if (a.trace && blockIdx.x == 0) a.trace[4096 + j] = gtimer();
      }
    }
    return;
  }

  // ------------------------------------------------ consumers (warps 0..MEGA_CW-1)
  unsigned bar_idx = 0;
  int s = 0, cstage = 0;
  uint32_t ph = 0;
  float best[DEC_MAX_B];
  int bidx[DEC_MAX_B];
#pragma unroll
  for (int b = 0; b < DEC_MAX_B; ++b) {
    best[b] = -INFINITY;
    bidx[b] = 0x7fffffff;
  }
  // one GEMV over a row list of nrows rows (row i -> matrix row rowf(i));
  // pre(n, ok) prefetches epilogue inputs, epi(n, b, v, e) per (row, batch row)
  auto gemv = [&](int K, int nrows, auto &&rowf, auto &&pre, auto &&epi, auto &&post) {
    const int per = mega_rows(K);
    const int kchunks = K / 256;
    for (int i0 = 0; i0 < nrows; i0 += per) {
      const uint8_t *stage = ring + (size_t)s * MEGA_STAGE;
      const int nr = min(per, nrows - i0);
      bool waited = false;
      for (int rr = warp; rr < per; rr += MEGA_CW) {
        const bool ok = rr < nr;
        const int n = ok ? rowf(i0 + rr) : 0;
        auto e = pre(n, ok);
        if (!waited) {
          mbar_wait_s(&full[s], ph);
          waited = true;
          if (a.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && cstage < 512)
            a.trace[6600 + cstage] = gtimer();
        }
        if (ok) {
          // U chunks of loads in flight (fewer for wide batches: registers), W
          // unpacked once per chunk and reused by every batch row
          constexpr int U = BT <= 2 ? 4 : (BT == 4 ? 2 : 1);
          float acc[BT][U];
#pragma unroll
          for (int b = 0; b < BT; ++b)
#pragma unroll
            for (int u = 0; u < U; ++u) acc[b][u] = 0.f;
          const uint4 *wr = reinterpret_cast<const uint4 *>(stage + (size_t)rr * K * 2) + lane;
          const uint4 *xr = reinterpret_cast<const uint4 *>(xs) + lane;
          const int kq = K / 8;  // uint4 per row
          for (int c0 = 0; c0 < kchunks; c0 += U) {
            uint4 w[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (c0 + u < kchunks) w[u] = wr[(c0 + u) * 32];
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (c0 + u < kchunks) {
                float wf[8];
                const __nv_bfloat162 *wp = reinterpret_cast<const __nv_bfloat162 *>(&w[u]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 f = __bfloat1622float2(wp[j]);
                  wf[2 * j] = f.x;
                  wf[2 * j + 1] = f.y;
                }
#pragma unroll
                for (int b = 0; b < BT; ++b) {
                  const uint4 xv = xr[(size_t)b * kq + (c0 + u) * 32];
                  const __nv_bfloat162 *xp = reinterpret_cast<const __nv_bfloat162 *>(&xv);
                  float t = acc[b][u];
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const float2 f = __bfloat1622float2(xp[j]);
                    t = fmaf(wf[2 * j], f.x, t);
                    t = fmaf(wf[2 * j + 1], f.y, t);
                  }
                  acc[b][u] = t;
                }
              }
          }
#pragma unroll
          for (int b = 0; b < BT; ++b)
#pragma unroll
            for (int u = 1; u < U; ++u) acc[b][0] += acc[b][u];
          float v = 0.f;
#pragma unroll
          for (int b = 0; b < BT; ++b) {
            const float t = warp_sum(acc[b][0]);
            if (lane == b) v = t;
          }
          if (lane < B) epi(n, lane, v, e);
          post(n);
        }
      }
      if (!waited) mbar_wait_s(&full[s], ph);
      ++cstage;
      __syncwarp();
      if (lane == 0) mbar_arrive_s(&empty[s]);
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    }
  };
  struct Pre {
    float old, w0, w1, w2, w3, c0, c1, c2, bias;
  };
  auto no_post = [](int) {};
  const int gn2 = 2 * gn;

  for (int l = 0; l < a.L; ++l) {
    const ssd200_layer_t lw = a.layers[l];
    const float *conv_w = static_cast<const float *>(lw.conv_w);
    const float *conv_b = static_cast<const float *>(lw.conv_b);
    const float *dt_bias = static_cast<const float *>(lw.dt_bias);
    float *conv = a.conv + (size_t)l * B * a.conv_dim * (a.k - 1);
    // ---------------- A: this CTA's in_proj rows + conv / dt epilogue
    MEGA_TRACE(l * 8 + 0);
    {
      const uint4 *src = reinterpret_cast<const uint4 *>(a.hidden_lp);
      uint4 *dst = reinterpret_cast<uint4 *>(xs);
      for (int i = threadIdx.x; i < BT * a.d_model / 8; i += MEGA_CT)
        dst[i] = i < B * a.d_model / 8 ? src[i] : make_uint4(0, 0, 0, 0);
      named_barrier_sync(1, MEGA_CT);
      MEGA_TRACE(l * 8 + 1);
      gemv(
          a.d_model, own.count(), [&](int i) { return own.row(i, a); },
          [&](int n, bool ok) {
            Pre e{};
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
          [&](int n, int b, float v, const Pre &e) {
            if (n < a.d_inner) {
              s_z[b][n - own.k0] = v;
            } else if (n < a.d_inner + a.conv_dim) {
              const int ch = n - a.d_inner, km = a.k - 1;
              float *co = conv + ((size_t)b * a.conv_dim + ch) * km;
              float act;
              if (a.k == 4) {  // taps oldest first (numerics.py:187-188)
                const float t = e.c0 * e.w0 + e.c1 * e.w1 + e.c2 * e.w2 + v * e.w3;
                act = silu(t + e.bias);
                co[0] = e.c1;
                co[1] = e.c2;
                co[2] = v;
              } else {
                float win[16];
                for (int j = 0; j < km; ++j) win[j] = co[j];
                win[km] = v;
                float t = 0.f;
                for (int j = 0; j <= km; ++j) t += win[j] * conv_w[(size_t)ch * a.k + j];
                act = silu(t + conv_b[ch]);
                for (int j = 0; j < km; ++j) co[j] = win[j + 1];
              }
              if (ch < a.d_inner)
                s_x[b][ch - own.k0] = act;
              else
                a.act[(size_t)b * a.conv_dim + ch] = act;  // B / C: read by every CTA
            } else {
              const int h = n - a.d_inner - a.conv_dim;
              s_dt[b][h - own.h_lo] = clamp_(softplus(v + dt_bias[h]), a.dt_lo, a.dt_hi);
            }
          },
          [&](int n) {
            if (n >= 2 * a.d_inner && n < a.d_inner + a.conv_dim) {  // publish a B / C row
              __syncwarp();
              if (lane == 0)
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bc_flag) : "memory");
            }
          });
    }
    MEGA_TRACE(l * 8 + 2);
    // ---------------- SSM update of this CTA's channels (every B / C row published)
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)(l + 1) * gn2;
      unsigned cur;
      do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.bc_flag) : "memory");
      } while (cur < target);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    named_barrier_sync(1, MEGA_CT);
    MEGA_TRACE(l * 8 + 3);
    {
      const float *A = static_cast<const float *>(lw.a);
      const float *Dv = static_cast<const float *>(lw.D);
      float *sbc = reinterpret_cast<float *>(xs);  // (B, 2, G*N) from L2 (written by other CTAs)
      for (int i = threadIdx.x; i < B * gn2; i += MEGA_CT) {
        const int b = i / gn2, j = i % gn2;
        sbc[i] = __ldcg(&a.act[(size_t)b * a.conv_dim + a.d_inner + j]);
      }
      named_barrier_sync(1, MEGA_CT);
      const int hpg = a.H / a.G;
      const int hl = lane & 15, half = lane >> 4;
      const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
      const int rows = B * own.nk;
      float *ssm_l = a.ssm + (size_t)l * B * a.d_inner * a.N;
      for (int r0 = 2 * warp; r0 < rows; r0 += 2 * MEGA_CW) {
        const int r = r0 + half;
        if (r < rows) {
          const int b = r / own.nk, kk = r % own.nk, k = own.k0 + kk;
          const int h = k / a.P;
          const int g = h / hpg;
          const float *bs = sbc + (size_t)b * gn2 + g * a.N;
          const float *cs = sbc + (size_t)b * gn2 + gn + g * a.N;
          const float dt = s_dt[b][h - own.h_lo];
          const float xv = s_x[b][kk], zv = s_z[b][kk];
          const float Ah = A[h], Dh = Dv[h];
          float4 *st = reinterpret_cast<float4 *>(ssm_l + ((size_t)b * a.d_inner + k) * a.N);
          float4 hv[4];
          const int nq = a.N / 64;  // float4 per lane (N <= 256)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nq) hv[q] = st[hl + 16 * q];
          const float decay = expf(Ah * dt);  // decode.py:126-129
          const float dx = dt * xv;
          float acc = 0.f;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nq) {
              const int n = 4 * (hl + 16 * q);
              hv[q].x = decay * hv[q].x + dx * bs[n];
              hv[q].y = decay * hv[q].y + dx * bs[n + 1];
              hv[q].z = decay * hv[q].z + dx * bs[n + 2];
              hv[q].w = decay * hv[q].w + dx * bs[n + 3];
              st[hl + 16 * q] = hv[q];
              acc = fmaf(cs[n], hv[q].x, acc);
              acc = fmaf(cs[n + 1], hv[q].y, acc);
              acc = fmaf(cs[n + 2], hv[q].z, acc);
              acc = fmaf(cs[n + 3], hv[q].w, acc);
            }
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(hmask, acc, o);
          if (hl == 0) {
            const float y = acc + Dh * xv;  // decode.py:132
            const float uu = y * silu(zv);
            a.u[(size_t)b * a.d_inner + k] = __float2bfloat16_rn(uu);
            s_uu[b][kk] = uu * uu;
          }
        }
      }
      named_barrier_sync(1, MEGA_CT);
      if (warp < B) {  // fixed-order sum (deterministic)
        float t = 0.f;
        for (int kk = lane; kk < own.nk; kk += 32) t += s_uu[warp][kk];
        t = warp_sum(t);
        if (lane == 0) a.upart[(size_t)blockIdx.x * B + warp] = t;
      }
    }
    MEGA_TRACE(l * 8 + 4);
    mega_grid_sync(a, bar_idx);
    MEGA_TRACE(l * 8 + 5);
    // ---------------- B: out_proj + norm row scale + residual
    {
      const uint4 *src = reinterpret_cast<const uint4 *>(a.u);
      uint4 *dst = reinterpret_cast<uint4 *>(xs);
      for (int i = threadIdx.x; i < BT * a.d_inner / 8; i += MEGA_CT)
        dst[i] = i < B * a.d_inner / 8 ? __ldcg(src + i) : make_uint4(0, 0, 0, 0);
      if (warp < B) {  // fixed-order sum of the per-CTA partials (deterministic)
        float t = 0.f;
        for (int i = lane; i < (int)gridDim.x; i += 32) t += __ldcg(&a.upart[(size_t)i * B + warp]);
        t = warp_sum(t);
        if (lane == 0) s_scale[warp] = 1.f / sqrtf(t / (float)a.d_inner + a.eps);
      }
      named_barrier_sync(1, MEGA_CT);
      MEGA_TRACE(l * 8 + 6);
      const int r0 = (int)((long)a.d_model * blockIdx.x / gridDim.x);
      const int nr = (int)((long)a.d_model * (blockIdx.x + 1) / gridDim.x) - r0;
      gemv(
          a.d_inner, nr, [&](int i) { return r0 + i; },
          [&](int n, bool ok) {
            Pre e{};
            if (ok && lane < B) e.old = a.hidden[(size_t)lane * a.d_model + n];
            return e;
          },
          [&](int n, int b, float v, const Pre &e) {
            const float nv = e.old + s_scale[b] * v;
            a.hidden[(size_t)b * a.d_model + n] = nv;
            a.hidden_lp[(size_t)b * a.d_model + n] = __float2bfloat16_rn(nv);
          },
          no_post);
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
    const int hr0 = (int)((long)a.V * blockIdx.x / gridDim.x);
    const int hnr = (int)((long)a.V * (blockIdx.x + 1) / gridDim.x) - hr0;
    gemv(
        a.d_model, hnr, [&](int i) { return hr0 + i; }, [&](int, bool) { return Pre{}; },
        [&](int n, int b, float v, const Pre &) {
          if (a.logits) a.logits[(size_t)b * a.V + n] = v;
#pragma unroll
          for (int bb = 0; bb < DEC_MAX_B; ++bb)
            if (bb == b && v > best[bb]) {  // rows ascend per warp: strict > keeps the lowest id
              best[bb] = v;
              bidx[bb] = n;
            }
        },
        no_post);
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
