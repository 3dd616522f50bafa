// Cached decode step for the bf16 mode (decode.py:77-144): the per-layer
// state stream (dec_ssm_stream), the norm + residual finish (dec_out_finish)
// and the greedy argmax of the head (argmax_part / argmax_final).  The
// weight-streaming projections are dec_gemm_swap (decode_gemm.cuh).
#pragma once

#include "common.cuh"

namespace ssd200 {

__device__ __forceinline__ void named_barrier_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------------------
// bulk-copy (cp.async.bulk) + mbarrier helpers of the state stream
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void mbar_init_s(uint64_t *bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(n));
}
__device__ __forceinline__ void mbar_expect_s(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint64_t *bar, uint32_t parity) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// ---------------------------------------------------------------------------
// Decode (bf16 mode): at wide batches the SSM state dominates the
// step's bytes (1.3B, B = 64: 13.2 GB of f32 state read + written vs 2.7 GB of
// weights), so the layer's middle is one streaming kernel.
//
// dec_ssm_stream: a persistent TMA pipeline over the (row, head) state tiles
// (P x N f32 = 32 KB, contiguous in the cache).  A producer warp keeps S tiles
// in flight with cp.async.bulk — per tile: the state tile, the raw in_proj
// x / z / B / C slices of every split-K partial, the conv windows of the tile's
// x and B / C channels and its x conv taps; the tile index, whether B / C are
// new and the raw dt (summed over the partials by the producer's lanes) go in
// the stage's header — and refills a stage as soon as its tile is done.  Tiles
// come either as a contiguous static range per CTA or, at wide batches, as
// chunks of consecutive tiles handed out by an atomic counter (the first chunk
// of each CTA is static, so its state is requested before the dependency
// wait): a static split leaves the CTAs that started late or share their SM
// with a slower neighbour finishing up to ~18 % after the others (1.3B,
// B = 256).  Which CTA updates a tile does not change its arithmetic.  Eight
// consumer warps, per tile:
//   conv taps + SiLU for the tile's x channels and its row's B / C channels
//     (decode.py:103-108; the x windows are rolled here, each is owned by one
//     tile; the shared B / C windows are rolled by dec_out_finish, after every
//     tile has read them),
//   h <- e^{a dt} h + dt x B ; y = C.h + D x ; u = y silu(z)      decode.py:111-133
// all from shared memory; h leaves straight from registers (streaming stores).
// The layer's per-head scalars and B / C conv taps are copied once per CTA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src))), "r"(bytes)
               : "memory");
}
// expect tx bytes on the current phase without arriving
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}

struct DecStreamArgs {
  int B, H, P, G, N, d_inner, conv_dim;
  const float *proj;  // (nsplit, B, ldp) raw in_proj partials [z | x | B | C | dt_raw]
  long ldp, sstride;
  int nsplit;
  const float *conv_in;  // (B, conv_dim, 3)
  float *conv_out;       // x windows rolled here (may alias conv_in)
  const float *conv_w, *conv_b, *dt_bias, *a, *D;
  float dt_lo, dt_hi;
  const float *ssm_in;
  float *ssm_out;  // may alias ssm_in
  bf16 *u;         // (B, d_inner)
  float *ssq;      // (B, H)
  int stages;
  uint32_t stage_bytes;
  // dynamic tile hand-out: chunk > 0 tiles per chunk, ctr = chunk counter (zeroed
  // by this layer's in_proj after its own dependency wait); chunk = 0: static ranges
  int chunk;
  unsigned *ctr;
  // one tile per CTA (small batches): the consumer threads load their state rows
  // straight into registers at kernel entry, so the stage holds no state tile and
  // the CTA is small enough to share an SM with two in_proj CTAs — it launches (and
  // its state loads start) while the in_proj is still streaming weights
  int reg_state;
  int trace;  // launch-timeline slot (SSD200_TRACE builds), -1 = none
  int trace2; // consumer sub-phases: first tile landed, B / C conv done, last tile done
};
constexpr int DSS_MAX_STAGES = 8;

// byte offsets inside a stage (nsplit raw partials of x, z, B, C; conv windows;
// the x conv taps and biases of the tile's head)
struct DssLayout {
  uint32_t xr, zr, br, cr, xw, bw, cw, xcw, xcb, total;
  // with_state = false: the state tile is not staged (small batches keep it in registers)
  __host__ __device__ DssLayout(int P, int N, int ns, bool with_state = true) {
    xr = with_state ? (uint32_t)P * N * 4 : 0u;
    zr = xr + ns * P * 4;
    br = zr + ns * P * 4;
    cr = br + ns * N * 4;
    xw = cr + ns * N * 4;
    bw = xw + P * 12;
    cw = bw + N * 12;
    xcw = cw + N * 12;
    xcb = xcw + P * 16;
    total = (xcb + P * 4 + 127) & ~127u;
  }
};
// per-CTA parameter block behind the ring: dt_bias | a | D (H floats each,
// padded to 16 B), then the B / C conv taps (2 G N float4) and biases (2 G N)
__host__ __device__ inline uint32_t dss_par_scalars(int H) { return (3u * H * 4u + 15u) & ~15u; }
__host__ __device__ inline uint32_t dss_par_bytes(int H, int G, int N) {
  return dss_par_scalars(H) + 2u * G * N * 20u;
}

// sum_j p[j * stride] for j = 0 .. n-1, added in j order (the split-K partials'
// fixed reduction order), with the first 16 loads issued together: a dependent
// load -> add chain cost one memory latency per split
__device__ __forceinline__ float sum_splits(const float *__restrict__ p, long stride, int n) {
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = j < n ? __ldcg(p + j * stride) : 0.f;
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < n) acc += v[j];
  for (int j = 16; j < n; ++j) acc += __ldcg(p + j * stride);
  return acc;
}

// CW consumer warps (RPW = P / CW rows each) + 1 producer warp
template <int NQ, int RPW, int CW>
__global__ __launch_bounds__(CW * 32 + 32, CW == 8 ? 2 : 1) void dec_ssm_stream(DecStreamArgs a) {
  constexpr int CT = CW * 32;
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) uint64_t full[DSS_MAX_STAGES], done[DSS_MAX_STAGES], pbar;
  __shared__ float red[DSS_MAX_STAGES][CW];
  __shared__ int s_tile[DSS_MAX_STAGES];    // tile index (-1: no more tiles)
  __shared__ int s_nbc[DSS_MAX_STAGES];     // the stage carries a new (row, group)'s B / C
  __shared__ float2 s_dt[DSS_MAX_STAGES];   // (dt, e^{a dt}) of the stage's tile
  __shared__ __align__(16) float bcact[2][2 * 256];  // [B N | C N] per (row, group), double buffered
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) SSD200_TRACE_MARK(a.trace, 0);
  const int P = a.P, N = a.N, N4 = N >> 2, H = a.H, G = a.G, ns = a.nsplit;
  const int ntiles = a.B * H;
  const int S = a.stages;
  const bool regst = a.reg_state != 0;
  const DssLayout L(P, N, ns, !regst);
  const uint32_t tile_bytes = (uint32_t)P * N * 4;
  // per tile: state + x taps (requested early) and x / z partials + x windows; per new
  // (row, group): B / C partials + windows
  const uint32_t early_bytes = (regst ? 0u : tile_bytes) + P * 20;
  const uint32_t rest_bytes = (uint32_t)ns * 2 * P * 4 + P * 12;
  const uint32_t bc_bytes = (uint32_t)ns * 2 * N * 4 + 2 * N * 12;
  const int hpg = H / G;
  float *s_dtb = reinterpret_cast<float *>(dsm + (size_t)S * a.stage_bytes);
  float *s_a = s_dtb + H, *s_D = s_dtb + 2 * H;
  const float4 *s_bcw =
      reinterpret_cast<const float4 *>(dsm + (size_t)S * a.stage_bytes + dss_par_scalars(H));
  const float *s_bcb = reinterpret_cast<const float *>(s_bcw + 2 * G * N);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init_s(&full[s], 1);
      mbar_init_s(&done[s], CW);
    }
    mbar_init_s(&pbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {
    // ---------------- producer warp: loads, refills (lane 0 issues, all lanes load dt)
    // the tile sequence: static range [t0, t1), or chunk blockIdx.x, then grabbed chunks
    const bool dyn = a.chunk > 0;
    const int t0 = dyn ? blockIdx.x * a.chunk : (int)((long)ntiles * blockIdx.x / gridDim.x);
    const int t1 = dyn ? min(ntiles, t0 + a.chunk)
                       : (int)((long)ntiles * (blockIdx.x + 1) / gridDim.x);
    int cur = t0, end = t1, prev_key = -1;
    auto next_tile = [&](bool may_grab) -> int {
      if (cur >= end) {
        if (!dyn || !may_grab) return -1;
        int c = 0;
        if (lane == 0) c = (int)gridDim.x + (int)atomicAdd(a.ctr, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        cur = c * a.chunk;
        end = min(ntiles, cur + a.chunk);
        if (cur >= ntiles) {
          cur = end = ntiles;
          return -1;
        }
      }
      return cur++;
    };
    // early part of a stage (no dependency on this step's earlier kernels): the
    // state tile (last written by this layer's previous step) and the x taps
    auto fill_early = [&](int s, int t) {
      if (lane == 0) {
        const int h = t % H;
        uint8_t *st = dsm + (size_t)s * a.stage_bytes;
        mbar_expect_tx_only(&full[s], early_bytes);
        if (!regst) bulk_g2s(st, a.ssm_in + (size_t)t * P * N, tile_bytes, &full[s]);
        bulk_g2s(st + L.xcw, a.conv_w + (size_t)h * P * 4, P * 16, &full[s]);
        bulk_g2s(st + L.xcb, a.conv_b + (size_t)h * P, P * 4, &full[s]);
      }
    };
    // the rest (after the dependency wait): in_proj partials, conv windows, dt_raw;
    // the arrive publishes the stage header
    auto fill_rest = [&](int s, int t) {
      const int b = t / H, h = t % H, g = h / hpg, key = b * G + g;
      const bool nbc = key != prev_key;
      prev_key = key;
      if (lane == 0) {
        uint8_t *st = dsm + (size_t)s * a.stage_bytes;
        uint64_t *bar = &full[s];
        mbar_expect_tx_only(bar, rest_bytes + (nbc ? bc_bytes : 0u));
        for (int j = 0; j < ns; ++j) {
          const float *pr = a.proj + j * a.sstride + (size_t)b * a.ldp;
          bulk_g2s(st + L.xr + j * P * 4, pr + a.d_inner + h * P, P * 4, bar);
          bulk_g2s(st + L.zr + j * P * 4, pr + h * P, P * 4, bar);
          if (nbc) {
            bulk_g2s(st + L.br + j * N * 4, pr + 2 * a.d_inner + g * N, N * 4, bar);
            bulk_g2s(st + L.cr + j * N * 4, pr + 2 * a.d_inner + G * N + g * N, N * 4, bar);
          }
        }
        const float *cwin = a.conv_in + (size_t)b * a.conv_dim * 3;
        bulk_g2s(st + L.xw, cwin + (size_t)h * P * 3, P * 12, bar);
        if (nbc) {
          bulk_g2s(st + L.bw, cwin + (size_t)(a.d_inner + g * N) * 3, N * 12, bar);
          bulk_g2s(st + L.cw, cwin + (size_t)(a.d_inner + G * N + g * N) * 3, N * 12, bar);
        }
      }
      // dt_raw: lane j loads split j, lane 0 adds them in split order (sum_splits' order)
      float v = 0.f;
      for (int j0 = 0; j0 < ns; j0 += 32) {
        const int j = j0 + lane;
        const float x = j < ns ? __ldcg(a.proj + (size_t)j * a.sstride + (size_t)b * a.ldp +
                                        a.d_inner + a.conv_dim + h)
                               : 0.f;
        for (int q = 0; q < 32 && j0 + q < ns; ++q) v += __shfl_sync(0xffffffffu, x, q);
      }
      if (lane == 0) {
        // dt = clip(softplus(dt_raw + dt_bias)) and the decay e^{a dt}, once per tile
        // (decode.py:111-114); the layer's scalars have landed before any fill_rest
        const float dt = clamp_(softplus(v + s_dtb[h]), a.dt_lo, a.dt_hi);
        s_tile[s] = t;
        s_nbc[s] = nbc ? 1 : 0;
        s_dt[s] = make_float2(dt, expf(s_a[h] * dt));
        mbar_arrive_s(&full[s]);
      }
    };
    auto fill_end = [&](int s) {
      if (lane == 0) {
        s_tile[s] = -1;
        mbar_arrive_s(&full[s]);
      }
    };
    if (lane == 0) {
      mbar_expect_s(&pbar, dss_par_bytes(H, G, N));
      bulk_g2s(s_dtb, a.dt_bias, H * 4, &pbar);
      bulk_g2s(s_a, a.a, H * 4, &pbar);
      bulk_g2s(s_D, a.D, H * 4, &pbar);
      bulk_g2s(const_cast<float4 *>(s_bcw), a.conv_w + (size_t)a.d_inner * 4, 2 * G * N * 16, &pbar);
      bulk_g2s(const_cast<float *>(s_bcb), a.conv_b + a.d_inner, 2 * G * N * 4, &pbar);
    }
    int early[DSS_MAX_STAGES];
    int npre = 0;
    for (; npre < S; ++npre) {
      early[npre] = next_tile(false);
      if (early[npre] < 0) break;
      fill_early(npre, early[npre]);
    }
    griddep_wait();  // the in_proj partials (and the zeroed chunk counter)
    SSD200_TRACE_MARK(a.trace, 1);
    mbar_wait_s(&pbar, 0);  // dt_bias / a for the tile headers
    int nissued = 0;
    bool ended = false;
    for (int s = 0; s < S && !ended; ++s) {
      if (s < npre) {
        fill_rest(s, early[s]);
        ++nissued;
      } else {
        const int t = next_tile(true);
        if (t < 0) {
          fill_end(s);
          ended = true;
        } else {
          fill_early(s, t);
          fill_rest(s, t);
          ++nissued;
        }
      }
    }
    // let the out_proj launch once this CTA's first tile (the critical loads) has
    // landed: its CTAs then stream W_out into their rings while this grid computes
    // (they wait for this grid before reading u / ssq), instead of queueing their
    // weight tiles ahead of these small loads on the same SMs
    if (nissued > 0) mbar_wait_s(&full[0], 0);
    griddep_launch();
    for (int li = 0; li < nissued; ++li) {
      const int s = li % S;
      mbar_wait_s(&done[s], (uint32_t)(li / S) & 1u);  // the consumer warps finished tile li
      if (lane == 0) {
        float tsum = 0.f;
#pragma unroll
        for (int w = 0; w < CW; ++w) tsum += red[s][w];  // fixed order: deterministic
        a.ssq[s_tile[s]] = tsum;
      }
      __syncwarp();
      if (!ended) {  // stage s is free: the consumers stored the tile from registers
        const int t = next_tile(true);
        if (t < 0) {
          fill_end(s);
          ended = true;
        } else {
          fill_early(s, t);
          fill_rest(s, t);
          ++nissued;
        }
      }
    }
    if (lane == 0) SSD200_TRACE_MARK(a.trace, 2);
    return;
  }
  // ---------------- consumers
  float4 hreg[RPW][NQ];
  if (regst) {  // this CTA's single tile (static split, one tile per CTA)
    const int t = (int)((long)ntiles * blockIdx.x / gridDim.x);
    if (t < (int)((long)ntiles * (blockIdx.x + 1) / gridDim.x)) {
      const float4 *hg = reinterpret_cast<const float4 *>(a.ssm_in + (size_t)t * P * N);
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (lane + 32 * q < N4) hreg[r][q] = __ldcs(hg + (warp * RPW + r) * N4 + lane + 32 * q);
    }
  }
  mbar_wait_s(&pbar, 0);
  int bce = 1;
  long long cy[6] = {0, 0, 0, 0, 0, 0}, ct = SSD200_CYC_NOW();
  for (int li = 0;; ++li) {
    const int s = li % S;
    uint8_t *st = dsm + (size_t)s * a.stage_bytes;
    mbar_wait_s(&full[s], (uint32_t)(li / S) & 1u);
    { const long long c = SSD200_CYC_NOW(); cy[0] += c - ct; ct = c; }
    if (threadIdx.x == 0 && li == 0) SSD200_TRACE_MARK(a.trace2, 0);
    const int t = s_tile[s];
    if (t < 0) break;
    const int b = t / H, h = t % H, g = h / hpg;
    const bool nbc = s_nbc[s] != 0;
    bce ^= nbc ? 1 : 0;
    float *bca = bcact[bce];
    if (nbc) {
      // the row's B / C channels (shared by every head of the group): conv taps
      // (oldest first) + SiLU, once per (row, group) in this CTA's tile sequence
      for (int j = threadIdx.x; j < 2 * N; j += CT) {
        const bool isc = j >= N;
        const int jj = isc ? j - N : j;
        const int pj = (isc ? G * N : 0) + g * N + jj;
        const float *rawp = reinterpret_cast<const float *>(st + (isc ? L.cr : L.br));
        float v = 0.f;
        for (int q = 0; q < ns; ++q) v += rawp[q * N + jj];
        const float *win = reinterpret_cast<const float *>(st + (isc ? L.cw : L.bw)) + jj * 3;
        const float4 cwt = s_bcw[pj];
        bca[j] = silu_fast(win[0] * cwt.x + win[1] * cwt.y + win[2] * cwt.z + v * cwt.w +
                           s_bcb[pj]);
      }
    }
    if (threadIdx.x == 0 && li == 0) SSD200_TRACE_MARK(a.trace2, 1);
    { const long long c = SSD200_CYC_NOW(); cy[1] += c - ct; ct = c; }
    const float2 dtd = s_dt[s];
    const float dt = dtd.x, decay = dtd.y, Dh = s_D[h];
    // this warp's rows need only their own x and z: lanes 0..RPW-1 run the x conv
    // (and roll the x windows, which this tile owns: roll_and_insert, decode.py:65-69),
    // lanes 16..16+RPW-1 sum z over the split-K partials
    float mine = 0.f;
    if (lane < RPW) {
      const int p = warp * RPW + lane, ch = h * P + p;
      const float *rawp = reinterpret_cast<const float *>(st + L.xr);
      float v = 0.f;
      for (int q = 0; q < ns; ++q) v += rawp[q * P + p];
      const float *win = reinterpret_cast<const float *>(st + L.xw) + p * 3;
      const float4 cwt = reinterpret_cast<const float4 *>(st + L.xcw)[p];
      const float w0 = win[0], w1 = win[1], w2 = win[2];
      mine = silu_fast(w0 * cwt.x + w1 * cwt.y + w2 * cwt.z + v * cwt.w +
                       reinterpret_cast<const float *>(st + L.xcb)[p]);
      float *co = a.conv_out + ((size_t)b * a.conv_dim + ch) * 3;
      co[0] = w1;
      co[1] = w2;
      co[2] = v;
    } else if (lane >= 16 && lane < 16 + RPW) {
      const float *zr = reinterpret_cast<const float *>(st + L.zr);
      const int p = warp * RPW + lane - 16;
      for (int q = 0; q < ns; ++q) mine += zr[q * P + p];
    }
    // (the x conv above ran before this barrier, overlapping the other warps' B / C work)
    if (nbc) named_barrier_sync(1, CT);
    float xrow[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) xrow[r] = __shfl_sync(0xffffffffu, mine, r);
    { const long long c = SSD200_CYC_NOW(); cy[2] += c - ct; ct = c; }
    const float4 *hs = reinterpret_cast<const float4 *>(st);
    float4 *ho = reinterpret_cast<float4 *>(a.ssm_out + (size_t)t * P * N);
    const float4 *bs = reinterpret_cast<const float4 *>(bca);
    const float4 *cs = reinterpret_cast<const float4 *>(bca + N);
    float4 bq[NQ], cq[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (lane + 32 * q < N4) {
        bq[q] = bs[lane + 32 * q];
        cq[q] = cs[lane + 32 * q];
      }
    // RPW rows per warp, all loads / FMAs of the rows independent (ILP)
    float acc[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int p = warp * RPW + r;
      const float dx = dt * xrow[r];
      float tt = 0.f;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int n4 = lane + 32 * q;
        if (n4 < N4) {
          float4 v = regst ? hreg[r][q] : hs[p * N4 + n4];
          v.x = decay * v.x + dx * bq[q].x;
          v.y = decay * v.y + dx * bq[q].y;
          v.z = decay * v.z + dx * bq[q].z;
          v.w = decay * v.w + dx * bq[q].w;
          __stcs(ho + p * N4 + n4, v);  // streaming store straight from registers
          tt = fmaf(cq[q].x, v.x, tt);
          tt = fmaf(cq[q].y, v.y, tt);
          tt = fmaf(cq[q].z, v.z, tt);
          tt = fmaf(cq[q].w, v.w, tt);
        }
      }
      acc[r] = tt;
    }
    { const long long c = SSD200_CYC_NOW(); cy[3] += c - ct; ct = c; }
    // y_p = C . h_p: reduce the RPW row sums over the 32 lanes
    float yv;
    int prow;
    bool owner;
    if constexpr (RPW > 1) {
      // transposing butterfly: log2(RPW) levels halve the row set per lane (RPW - 1
      // shuffles in all), then plain xor levels; afterwards every lane of an aligned
      // group of 32 / RPW lanes holds the total of row warp * RPW + rsel
      int rsel = 0;
#pragma unroll
      for (int hf = RPW / 2, o = 16; hf >= 1; hf >>= 1, o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i2 = 0; i2 < hf; ++i2) {
          const float send = up ? acc[i2] : acc[i2 + hf];
          const float keep = up ? acc[i2 + hf] : acc[i2];
          acc[i2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
        if (up) rsel += hf;
      }
#pragma unroll
      for (int o = 16 / RPW; o > 0; o >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
      yv = acc[0];
      prow = warp * RPW + rsel;
      owner = (lane & (32 / RPW - 1)) == 0;
    } else {
      yv = warp_sum(acc[0]);
      prow = warp;
      owner = lane == 0;
    }
    float uu = 0.f;
    const float xv = __shfl_sync(0xffffffffu, mine, prow - warp * RPW);
    const float zv = __shfl_sync(0xffffffffu, mine, 16 + prow - warp * RPW);
    if (owner) {
      const float y = yv + Dh * xv;  // decode.py:132
      const float uv = y * silu_fast(zv);
      a.u[(size_t)b * a.d_inner + h * P + prow] = __float2bfloat16_rn(uv);
      uu = uv * uv;
    }
    uu = warp_sum(uu);
    if (lane == 0) red[s][warp] = uu;
    __syncwarp();
    if (lane == 0) mbar_arrive_s(&done[s]);
    { const long long c = SSD200_CYC_NOW(); cy[4] += c - ct; ct = c; cy[5] += 1; }
  }
  if (threadIdx.x == 0) {
    SSD200_TRACE_MARK(a.trace2, 2);
    for (int k = 0; k < 6; ++k) SSD200_CYC_ADD(k, cy[k]);
  }
}

// hidden += rsqrt(sum_h ssq[b, h] / d_inner + eps) * sum_s part[s, b, :]
// (gated RMSNorm row scale after the out_proj, norm_w folded into W_out;
// residual in f32 + bf16 shadow) — model.py:166-173.  grid (chunks, B); the
// blocks past d_model roll the row's shared B / C conv windows (read by every
// tile of dec_ssm_stream, so rolled only now): roll_and_insert, decode.py:65-69.
struct DecFinishArgs {
  const float *part;  // (nsplit_out, B, d_model)
  int nsplit;
  long sstride;
  const float *ssq;   // (B, H)
  int H;
  float inv_d, eps;
  const float *hidden_in;  // residual before this update (may alias hidden)
  float *hidden;
  bf16 *lp;
  int d_model;
  // B / C windows
  const float *proj;  // (nsplit_in, B, ldp)
  long ldp, psstride;
  int pnsplit, d_inner, conv_dim;
  const float *conv_in;
  float *conv_out;
  // head-group-sharded mode: pout[b, :d_model] = partial, pout[b, d_model] = sum u^2
  float *pout;
  long pld;
  int trace;  // launch-timeline slot (SSD200_TRACE builds), -1 = none
};
__global__ __launch_bounds__(256) void dec_out_finish(DecFinishArgs a) {
  __shared__ float sc;
  const int b = blockIdx.y;
  const int nb_h = (a.d_model + 255) / 256;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = (int)blockIdx.x < nb_h && n < a.d_model;
  const long i = (long)b * a.d_model + n;
  // the next layer's in_proj may launch at once and prefetch its weights while the
  // out_proj drains (it waits for this grid before reading hidden_lp)
  if (threadIdx.x == 0) SSD200_TRACE_MARK(a.trace, 0);
  griddep_launch();
  griddep_wait();  // the residual, the partials and sum u^2 are all predecessor outputs
  if (threadIdx.x == 0) SSD200_TRACE_MARK(a.trace, 1);
  const float hold = (live && !a.pout) ? a.hidden_in[i] : 0.f;
  if ((int)blockIdx.x >= nb_h) {
    const int c = a.d_inner + ((int)blockIdx.x - nb_h) * 256 + threadIdx.x;  // B / C channel
    if (c >= a.conv_dim) return;
    const float v = sum_splits(a.proj + (long)b * a.ldp + a.d_inner + c, a.psstride, a.pnsplit);
    const float *ci = a.conv_in + ((long)b * a.conv_dim + c) * 3;
    float *co = a.conv_out + ((long)b * a.conv_dim + c) * 3;
    const float w1 = ci[1], w2 = ci[2];
    co[0] = w1;
    co[1] = w2;
    co[2] = v;
    return;
  }
  // every load of the block in flight together: warp 0's sum u^2 terms (up to 8
  // heads per lane, more in a second pass), then the split-K partials
  constexpr int QH = 8;
  float sq[QH];
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < QH; ++k) {
      const int h = threadIdx.x + 32 * k;
      sq[k] = h < a.H ? a.ssq[(long)b * a.H + h] : 0.f;
    }
  }
  const float acc = live ? sum_splits(a.part + (long)b * a.d_model + n, a.sstride, a.nsplit) : 0.f;
  if (threadIdx.x < 32) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < QH; ++k)
      if (threadIdx.x + 32 * k < a.H) t += sq[k];
    for (int h = threadIdx.x + 32 * QH; h < a.H; h += 32) t += a.ssq[(long)b * a.H + h];
    t = warp_sum(t);  // fixed shuffle tree: deterministic
    if (threadIdx.x == 0) {
      sc = 1.f / sqrtf(t * a.inv_d + a.eps);
      if (a.pout && blockIdx.x == 0) a.pout[(long)b * a.pld + a.d_model] = t;
    }
  }
  __syncthreads();
  if (!live) return;
  if (a.pout) {
    a.pout[(long)b * a.pld + n] = acc;
    return;
  }
  const float v = hold + sc * acc;
  a.hidden[i] = v;
  a.lp[i] = __float2bfloat16_rn(v);
  if (threadIdx.x == 0) SSD200_TRACE_MARK(a.trace, 2);
}

// greedy pick over wide logits (decode.py:72-74, ties -> lowest id): grid
// (chunks, rows) partial maxima, then one warp per row over the partials
__global__ __launch_bounds__(256) void argmax_part(const float *__restrict__ lg, long ld, int V,
                                                   int chunk, float *__restrict__ pv,
                                                   int *__restrict__ pi) {
  __shared__ float sv[8];
  __shared__ int si[8];
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.y, c0 = blockIdx.x * chunk;
  const int c1 = min(V, c0 + chunk);
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const float v = lg[(long)r * ld + c];
    if (v > bv) {  // ascending per thread: strict > keeps the lowest id
      bv = v;
      bi = c;
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
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < (int)(blockDim.x >> 5); ++w2)
      if (sv[w2] > bv || (sv[w2] == bv && si[w2] < bi)) {
        bv = sv[w2];
        bi = si[w2];
      }
    pv[(long)r * gridDim.x + blockIdx.x] = bv;
    pi[(long)r * gridDim.x + blockIdx.x] = bi;
  }
}

__global__ void argmax_final(const float *__restrict__ pv, const int *__restrict__ pi, int nparts,
                             int64_t *__restrict__ out) {
  griddep_wait();
  const int r = blockIdx.x, lane = threadIdx.x;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = lane; i < nparts; i += 32) {
    const float v = pv[(long)r * nparts + i];
    const int j = pi[(long)r * nparts + i];
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
  if (lane == 0) out[r] = bi == 0x7fffffff ? 0 : bi;
}

}  // namespace ssd200
