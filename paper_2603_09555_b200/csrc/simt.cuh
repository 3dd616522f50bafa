// Generic CUDA-core kernels (any dims), templated on the compute type T
// (float or double).  They carry the f32 / f64 parity modes end to end and
// provide the elementwise / decode pieces the bf16 tensor-core mode reuses.
// Each kernel cites the reference arithmetic it reproduces
// (paths relative to /root/reference/pkg/src/ssd_engine).
#pragma once

#include "common.cuh"

namespace ssd200 {

// =========================================================================
// embedding gather — model.py:198, decode.py:96
// =========================================================================
template <typename T, typename TE>
__global__ void embed_kernel(const int64_t *__restrict__ tok, const TE *__restrict__ E, int d_model,
                             int vocab, T *__restrict__ hid, bf16 *__restrict__ hid_lp) {
  const int r = blockIdx.x;
  const int64_t id = tok[r];
  const bool ok = id >= 0 && id < vocab;  // device-resident ids: a bad id poisons its row
  const TE *src = E + (size_t)(ok ? id : 0) * d_model;
  for (int c = threadIdx.x; c < d_model; c += blockDim.x) {
    T v = ok ? cvt<T>(src[c]) : (T)NAN;
    hid[(size_t)r * d_model + c] = v;
    if (hid_lp) hid_lp[(size_t)r * d_model + c] = cvt<bf16>(v);
  }
}

// =========================================================================
// SIMT GEMM: C (M,N) [=|+=] A (M,K) . B, B either (K,N) "KN" (reference
// weight layout) or (N,K) "NK" (the tied head reads embedding rows).
// 64x64 tile, BK=16, 256 threads, 4x4 outputs per thread, no TF32.
// =========================================================================
enum { EPI_STORE = 0, EPI_ADD = 1 };

template <typename T, bool B_NK, int EPI>
__global__ __launch_bounds__(256) void gemm_simt(const T *__restrict__ A, long lda,
                                                 const T *__restrict__ B, long ldb, T *C, long ldc,
                                                 int M, int N, int K) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);

  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int idx = tid + 256 * i;
      int m = idx >> 4, k = idx & 15;
      int gm = m0 + m, gk = k0 + k;
      As[k][m] = (gm < M && gk < K) ? A[(size_t)gm * lda + gk] : T(0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int idx = tid + 256 * i;
      if (B_NK) {
        int n = idx >> 4, k = idx & 15;
        int gn = n0 + n, gk = k0 + k;
        Bs[k][n] = (gn < N && gk < K) ? B[(size_t)gn * ldb + gk] : T(0);
      } else {
        int k = idx >> 6, n = idx & 63;
        int gn = n0 + n, gk = k0 + k;
        Bs[k][n] = (gn < N && gk < K) ? B[(size_t)gk * ldb + gn] : T(0);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      T *dst = C + (size_t)gm * ldc + gn;
      if (EPI == EPI_ADD)
        *dst = *dst + acc[i][j];
      else
        *dst = acc[i][j];
    }
  }
}

// =========================================================================
// GEMV for few rows with the KN weight layout (f32/f64 decode projections):
// Y (M,N) [=|+=] X (M,K) . W (K,N).  block (32,8): x over columns, y over K.
// =========================================================================
template <typename T, int EPI>
__global__ __launch_bounds__(256) void gemv_kn(const T *__restrict__ X, long ldx,
                                               const T *__restrict__ W, long ldw, T *Y, long ldy,
                                               int M, int N, int K) {
  constexpr int MB = 8, KT = 128;
  __shared__ T xs[MB][KT];
  __shared__ T red[8][MB][33];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int n = blockIdx.x * 32 + tx;
  const int m0 = blockIdx.y * MB;
  T acc[MB];
#pragma unroll
  for (int r = 0; r < MB; ++r) acc[r] = T(0);
  for (int k0 = 0; k0 < K; k0 += KT) {
    for (int i = tid; i < MB * KT; i += 256) {
      int r = i / KT, k = i % KT;
      xs[r][k] = (m0 + r < M && k0 + k < K) ? X[(size_t)(m0 + r) * ldx + k0 + k] : T(0);
    }
    __syncthreads();
    if (n < N) {
      for (int k = ty; k < KT && k0 + k < K; k += 8) {
        T w = W[(size_t)(k0 + k) * ldw + n];
#pragma unroll
        for (int r = 0; r < MB; ++r) acc[r] = fma(xs[r][k], w, acc[r]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < MB; ++r) red[ty][r][tx] = acc[r];
  __syncthreads();
  {
    const int r = ty;  // 8 warps <-> 8 rows
    if (n < N && m0 + r < M) {
      T s = T(0);
      for (int j = 0; j < 8; ++j) s += red[j][r][tx];
      T *dst = Y + (size_t)(m0 + r) * ldy + n;
      if (EPI == EPI_ADD)
        *dst = *dst + s;
      else
        *dst = s;
    }
  }
}

// =========================================================================
// GEMV for few rows with the NK layout: Y (M,N) [=|+=] X (M,K) . W (N,K)^T.
// Used by the tied head (embedding rows) and the bf16 decode projections
// (K-major weights).  Block = 8 warps, each warp owns NPW output columns and
// walks their weight rows lane-strided; x tiles are staged in smem.
// Optional Ylp receives a bf16 copy of the result (residual shadow).
// =========================================================================
template <typename T, typename TX, typename TW, int EPI>
__global__ __launch_bounds__(256) void gemv_nk(const TX *__restrict__ X, long ldx,
                                               const TW *__restrict__ W, long ldw, T *Y, long ldy,
                                               bf16 *Ylp, int M, int N, int K) {
  constexpr int MB = 4, NPW = 4, KT = 512;
  __shared__ T xs[MB][KT];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (blockIdx.x * 8 + warp) * NPW;
  const int m0 = blockIdx.y * MB;
  T acc[NPW][MB];
#pragma unroll
  for (int j = 0; j < NPW; ++j)
#pragma unroll
    for (int r = 0; r < MB; ++r) acc[j][r] = T(0);
  for (int k0 = 0; k0 < K; k0 += KT) {
    for (int i = threadIdx.x; i < MB * KT; i += 256) {
      int r = i / KT, k = i % KT;
      xs[r][k] = (m0 + r < M && k0 + k < K) ? cvt<T>(X[(size_t)(m0 + r) * ldx + k0 + k]) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NPW; ++j) {
      int n = nb + j;
      if (n >= N) break;
      const TW *wr = W + (size_t)n * ldw + k0;
      for (int k = lane; k < KT && k0 + k < K; k += 32) {
        T w = cvt<T>(wr[k]);
#pragma unroll
        for (int r = 0; r < MB; ++r) acc[j][r] = fma(xs[r][k], w, acc[j][r]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NPW; ++j) {
    int n = nb + j;
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      T s = warp_sum(acc[j][r]);
      if (lane == 0 && n < N && m0 + r < M) {
        T *dst = Y + (size_t)(m0 + r) * ldy + n;
        T v = (EPI == EPI_ADD) ? *dst + s : s;
        *dst = v;
        if (Ylp) Ylp[(size_t)(m0 + r) * ldy + n] = cvt<bf16>(v);
      }
    }
  }
}

// =========================================================================
// causal depthwise conv + SiLU over the xBC columns — numerics.py:169-189
// (taps oldest first, bias after the taps, zero left padding).
// =========================================================================
// grid (ceil(C/256), rows/ROWS_PER_BLOCK): each thread walks ROWS consecutive
// tokens of one channel, keeping the k-1 previous inputs in registers.
// KC > 0: compile-time kernel width (the production k = 4, fully in
// registers); KC == 0: runtime k <= 16.
template <typename T, typename TI, typename TO, int KC = 0, int ROWS = 16>
__global__ __launch_bounds__(256) void conv_silu_prefill(const TI *__restrict__ xbc, long ld_in,
                                                         const T *__restrict__ w,
                                                         const T *__restrict__ bias,
                                                         TO *__restrict__ out, long ld_out,
                                                         int Tlen, int C, int k_rt, long rows) {
  const int k = KC > 0 ? KC : k_rt;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const long r0 = (long)blockIdx.y * ROWS;
  if (c >= C) return;
  T wk[KC > 0 ? KC : 16], win[KC > 0 ? KC : 16];
#pragma unroll
  for (int j = 0; j < k; ++j) wk[j] = w[(size_t)c * k + j];
  const T bc = bias[c];
  const int t0 = (int)(r0 % Tlen);
  // history before r0 within the same sequence (zero before t = 0)
#pragma unroll
  for (int j = 0; j < k - 1; ++j) {
    const int src = t0 - (k - 1) + j;
    win[j] = src >= 0 ? cvt<T>(xbc[(r0 - t0 + src) * ld_in + c]) : T(0);
  }
  T xin[ROWS];  // all loads in flight before the dependent taps
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const long r = r0 + i;
    xin[i] = r < rows ? cvt<T>(xbc[r * ld_in + c]) : T(0);
  }
  int t = t0;
#pragma unroll
  for (int i = 0; i < ROWS; ++i, ++t) {
    const long r = r0 + i;
    if (r >= rows) break;
    if (t == Tlen) {  // crossed into the next sequence: reset the history
      t = 0;
#pragma unroll
      for (int j = 0; j < k - 1; ++j) win[j] = T(0);
    }
    win[k - 1] = xin[i];
    T acc = T(0);
#pragma unroll
    for (int j = 0; j < k; ++j) acc += wk[j] * win[j];  // taps oldest first
    out[r * ld_out + c] = cvt<TO>(silu(acc + bc));
#pragma unroll
    for (int j = 0; j < k - 1; ++j) win[j] = win[j + 1];
  }
}

// bf16 path, k = KC: a thread owns 8 consecutive channels (one 16-byte load
// per token) for ROWS consecutive tokens; block (32, 8) covers 256 channels x
// 8*ROWS tokens.  Needs C % 8 == 0 and 16-byte aligned rows.
template <int KC, int ROWS>
__global__ __launch_bounds__(256, 2) void conv_silu_bf16x8(const bf16 *__restrict__ xbc, long ld_in,
                                                        const float *__restrict__ w,
                                                        const float *__restrict__ bias,
                                                        bf16 *__restrict__ out, long ld_out,
                                                        int Tlen, int C, long rows) {
  const int c0 = (blockIdx.x * 32 + threadIdx.x) * 8;
  const long r0 = ((long)blockIdx.y * 8 + threadIdx.y) * ROWS;
  if (c0 >= C || r0 >= rows) return;
  float wk[8][KC], bc[8], win[8][KC];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
#pragma unroll
    for (int j = 0; j < KC; ++j) wk[e][j] = w[(size_t)(c0 + e) * KC + j];
    bc[e] = bias[c0 + e];
  }
  const int t0 = (int)(r0 % Tlen);
#pragma unroll
  for (int j = 0; j < KC - 1; ++j) {
    const int src = t0 - (KC - 1) + j;
    uint4 v = src >= 0 ? *reinterpret_cast<const uint4 *>(xbc + (r0 - t0 + src) * ld_in + c0)
                       : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h[e]);
      win[2 * e][j] = f.x;
      win[2 * e + 1][j] = f.y;
    }
  }
  uint4 xin[ROWS];
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const long r = r0 + i;
    xin[i] = r < rows ? *reinterpret_cast<const uint4 *>(xbc + r * ld_in + c0) : make_uint4(0, 0, 0, 0);
  }
  int t = t0;
#pragma unroll
  for (int i = 0; i < ROWS; ++i, ++t) {
    const long r = r0 + i;
    if (r >= rows) break;
    if (t == Tlen) {
      t = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int j = 0; j < KC - 1; ++j) win[e][j] = 0.f;
    }
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&xin[i]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h[e]);
      win[2 * e][KC - 1] = f.x;
      win[2 * e + 1][KC - 1] = f.y;
    }
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int j = 0; j < KC; ++j) {  // taps oldest first (numerics.py:187-188)
        a0 += wk[e][j] * win[e][j];
        a1 += wk[e + 1][j] * win[e + 1][j];
      }
      __nv_bfloat162 v = __floats2bfloat162_rn(silu_fast(a0 + bc[e]), silu_fast(a1 + bc[e + 1]));
      o[e >> 1] = *reinterpret_cast<uint32_t *>(&v);
    }
    *reinterpret_cast<uint4 *>(out + r * ld_out + c0) = make_uint4(o[0], o[1], o[2], o[3]);
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int j = 0; j < KC - 1; ++j) win[e][j] = win[e][j + 1];
  }
}

// conv tail: last k-1 pre-activation xBC inputs, newest last, zero-padded
// when T < k-1 — model.py:144-147.
template <typename T, typename TI>
__global__ void conv_tail_kernel(const TI *__restrict__ xbc, long ld_in, T *__restrict__ tail,
                                 int Bsz, int Tlen, int C, int k) {
  griddep_launch();
  griddep_wait();
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int km = k - 1;
  if (i >= (long)Bsz * C * km) return;
  const int j = (int)(i % km);
  const int c = (int)((i / km) % C);
  const int b = (int)(i / ((long)km * C));
  const int src = Tlen - km + j;
  tail[i] = src >= 0 ? cvt<T>(xbc[((long)b * Tlen + src) * ld_in + c]) : T(0);
}

// dt = clip(softplus(dt_raw + dt_bias), lo, hi) — ssd.py:115-136.
template <typename T, typename TI>
__global__ void dt_kernel(const TI *__restrict__ raw, long ld_in, const T *__restrict__ dt_bias,
                          T *__restrict__ dt, long rows, int H, T lo, T hi) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * H) return;
  const int h = (int)(i % H);
  const long r = i / H;
  dt[i] = clamp_(softplus(cvt<T>(raw[r * ld_in + h]) + dt_bias[h]), lo, hi);
}

// =========================================================================
// chunked SSD scan, generic dims — ssd.py:139-257 as three passes:
//   (1) chunk states  S_c = sum_l (B_l e^{cs_end-cs_l}) (X_l dt_l)   [:152-160]
//   (2) O(Nc) state pass s_c = e^{cs_end_c} s_{c-1} + S_c           [:163-184]
//   (3) outputs Y = (C B^T * e^{cs_l-cs_s}) Xbar + (C prev^T) e^{cs_l}
//       (+ D x)                                                      [:139-149,187-198]
// Inputs may be strided views into the in_proj/conv buffers.
// =========================================================================
template <typename T, typename TI> struct SsdArgs {
  const TI *X;
  long x_ts;  // token stride of X (elements)
  const T *dt;
  long dt_ts;
  const T *a;
  const TI *Bm;
  const TI *Cm;
  long bc_ts;
  const T *D;
  const T *init;
  T *Y;
  long y_ts;
  T *final_state;
  T *S;       // workspace (B, Nc, H, P, N): own states, then entering states
  T *cs_end;  // workspace (B, H, Nc)
  int B, T_, H, P, G, N, L, Nc;
};

constexpr int SSD_MAX_PN_PER_THREAD = 32;  // P*N <= 8192 with 256 threads

template <typename T>
__device__ __forceinline__ void chunk_cumsum(const T *dts, T ah, T *cs, int L) {
  // inclusive cumsum of a*dt, left to right — numerics.py:96-101, ssd.py:244-245
  if (threadIdx.x == 0) {
    T run = T(0);
    for (int l = 0; l < L; ++l) {
      run += dts[l] * ah;
      cs[l] = run;
    }
  }
}

template <typename T, typename TI>
__global__ __launch_bounds__(256) void ssd_chunk_state(SsdArgs<T, TI> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int TL = 16;
  const int L = p.L, P = p.P, N = p.N;
  T *cs = reinterpret_cast<T *>(smem_raw);
  T *wl = cs + L;
  T *dts = wl + L;
  T *xs = dts + L;      // TL x P : X * dt
  T *bs = xs + TL * P;  // TL x N : B * e^{cs_end - cs_l}
  const int c = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int g = h / (p.H / p.G);
  const int tid = threadIdx.x;
  const long t0 = (long)c * L;
  for (int l = tid; l < L; l += blockDim.x) {
    long t = t0 + l;
    dts[l] = t < p.T_ ? p.dt[((long)b * p.T_ + t) * p.dt_ts + h] : T(0);
  }
  __syncthreads();
  chunk_cumsum(dts, p.a[h], cs, L);
  __syncthreads();
  const T cend = cs[L - 1];
  for (int l = tid; l < L; l += blockDim.x) wl[l] = exp_(cend - cs[l]);
  if (tid == 0) p.cs_end[((long)b * p.H + h) * p.Nc + c] = cend;
  const int PN = P * N;
  T acc[SSD_MAX_PN_PER_THREAD];
#pragma unroll
  for (int i = 0; i < SSD_MAX_PN_PER_THREAD; ++i) acc[i] = T(0);
  for (int l0 = 0; l0 < L; l0 += TL) {
    __syncthreads();
    for (int i = tid; i < TL * P; i += blockDim.x) {
      int li = i / P, pp = i % P;
      long t = t0 + l0 + li;
      T v = T(0);
      if (l0 + li < L && t < p.T_)
        v = cvt<T>(p.X[((long)b * p.T_ + t) * p.x_ts + (long)h * P + pp]) * dts[l0 + li];
      xs[i] = v;
    }
    for (int i = tid; i < TL * N; i += blockDim.x) {
      int li = i / N, nn = i % N;
      long t = t0 + l0 + li;
      T v = T(0);
      if (l0 + li < L && t < p.T_)
        v = cvt<T>(p.Bm[((long)b * p.T_ + t) * p.bc_ts + (long)g * N + nn]) * wl[l0 + li];
      bs[i] = v;
    }
    __syncthreads();
    const int lmax = min(TL, L - l0);
#pragma unroll
    for (int i = 0; i < SSD_MAX_PN_PER_THREAD; ++i) {
      int e = tid + i * 256;
      if (e < PN) {
        int pp = e / N, nn = e % N;
        T s = acc[i];
        for (int li = 0; li < lmax; ++li) s = fma(bs[li * N + nn], xs[li * P + pp], s);
        acc[i] = s;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < SSD_MAX_PN_PER_THREAD; ++i) {
    int e = tid + i * 256;
    if (e < PN) p.S[(((long)b * p.Nc + c) * p.H + h) * PN + e] = acc[i];
  }
}

template <typename T>
__global__ void ssd_state_pass(T *S, const T *__restrict__ cs_end, const T *__restrict__ init,
                               T *__restrict__ final_state, int H, int PN, int Nc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int h = blockIdx.y, b = blockIdx.z;
  if (e >= PN) return;
  T s = init ? init[((long)b * H + h) * PN + e] : T(0);
  for (int c = 0; c < Nc; ++c) {
    long idx = (((long)b * Nc + c) * H + h) * PN + e;
    T own = S[idx];
    S[idx] = s;  // state entering chunk c
    s = exp_(cs_end[((long)b * H + h) * Nc + c]) * s + own;
  }
  final_state[((long)b * H + h) * PN + e] = s;
}

template <typename T, typename TI>
__global__ __launch_bounds__(256) void ssd_chunk_out(SsdArgs<T, TI> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int RT = 16, ST = 32, MAXO = 16;  // rows per block, s tile, outputs/thread
  const int L = p.L, P = p.P, N = p.N;
  T *cs = reinterpret_cast<T *>(smem_raw);
  T *dts = cs + L;
  T *Cr = dts + L;      // RT x N
  T *Bs = Cr + RT * N;        // ST x (N+1): padded against bank conflicts
  T *Xs = Bs + ST * (N + 1);  // ST x P (Xbar)
  T *Mt = Xs + ST * P;  // RT x ST
  const int nRT = (L + RT - 1) / RT;
  const int c = blockIdx.x / nRT, rt = blockIdx.x % nRT;
  const int h = blockIdx.y, b = blockIdx.z;
  const int g = h / (p.H / p.G);
  const int tid = threadIdx.x;
  const long t0 = (long)c * L;
  const int l0 = rt * RT;
  for (int l = tid; l < L; l += blockDim.x) {
    long t = t0 + l;
    dts[l] = t < p.T_ ? p.dt[((long)b * p.T_ + t) * p.dt_ts + h] : T(0);
  }
  for (int i = tid; i < RT * N; i += blockDim.x) {
    int r = i / N, nn = i % N;
    long t = t0 + l0 + r;
    Cr[i] = (l0 + r < L && t < p.T_)
                ? cvt<T>(p.Cm[((long)b * p.T_ + t) * p.bc_ts + (long)g * N + nn])
                : T(0);
  }
  __syncthreads();
  chunk_cumsum(dts, p.a[h], cs, L);
  __syncthreads();

  T acc[MAXO];
#pragma unroll
  for (int i = 0; i < MAXO; ++i) acc[i] = T(0);
  const int smax = min(l0 + RT, L);
  for (int s0 = 0; s0 < smax; s0 += ST) {
    for (int i = tid; i < ST * N; i += blockDim.x) {
      int si = i / N, nn = i % N;
      long t = t0 + s0 + si;
      Bs[si * (N + 1) + nn] = (s0 + si < L && t < p.T_)
                  ? cvt<T>(p.Bm[((long)b * p.T_ + t) * p.bc_ts + (long)g * N + nn])
                  : T(0);
    }
    for (int i = tid; i < ST * P; i += blockDim.x) {
      int si = i / P, pp = i % P;
      long t = t0 + s0 + si;
      Xs[i] = (s0 + si < L && t < p.T_)
                  ? cvt<T>(p.X[((long)b * p.T_ + t) * p.x_ts + (long)h * P + pp]) * dts[s0 + si]
                  : T(0);
    }
    __syncthreads();
    for (int i = tid; i < RT * ST; i += blockDim.x) {
      int r = i / ST, si = i % ST;
      int l = l0 + r, s = s0 + si;
      T m = T(0);
      if (l < L && s <= l) {
        T gsum = T(0);
        for (int nn = 0; nn < N; ++nn) gsum = fma(Cr[r * N + nn], Bs[si * (N + 1) + nn], gsum);
        m = gsum * exp_(cs[l] - cs[s]);  // (C.B^T) * exp(segsum), ssd.py:147-148
      }
      Mt[i] = m;
    }
    __syncthreads();
    const int smx = min(ST, smax - s0);
#pragma unroll
    for (int i = 0; i < MAXO; ++i) {
      int e = tid + i * 256;
      if (e < RT * P) {
        int r = e / P, pp = e % P;
        T s = acc[i];
        for (int si = 0; si < smx; ++si) s = fma(Mt[r * ST + si], Xs[si * P + pp], s);
        acc[i] = s;
      }
    }
    __syncthreads();
  }
  // readout of the entering state: (C . prev^T) * exp(cs_l)  (ssd.py:196-198)
  const T *prev = p.S + (((long)b * p.Nc + c) * p.H + h) * (long)P * N;
#pragma unroll
  for (int i = 0; i < MAXO; ++i) {
    int e = tid + i * 256;
    if (e < RT * P) {
      int r = e / P, pp = e % P;
      int l = l0 + r;
      long t = t0 + l;
      if (l < L && t < p.T_) {
        T off = T(0);
        for (int nn = 0; nn < N; ++nn) off = fma(Cr[r * N + nn], prev[(long)pp * N + nn], off);
        T y = acc[i] + off * exp_(cs[l]);
        if (p.D) y += p.D[h] * cvt<T>(p.X[((long)b * p.T_ + t) * p.x_ts + (long)h * P + pp]);
        p.Y[((long)b * p.T_ + t) * p.y_ts + (long)h * P + pp] = y;
      }
    }
  }
}

// =========================================================================
// gated RMSNorm — numerics.py:149-158: u = y*silu(z); u / sqrt(mean(u^2)+eps) * w
// one block per row
// =========================================================================
template <typename T, typename TZ, typename TO>
__global__ __launch_bounds__(256) void gated_norm_kernel(const T *__restrict__ y, long ldy,
                                                         const TZ *__restrict__ z, long ldz,
                                                         const T *__restrict__ w,
                                                         TO *__restrict__ out, long ldo, int D,
                                                         T eps) {
  __shared__ T red[32];
  griddep_wait();  // no-op unless launched as a programmatic dependent (the bf16 head)
  griddep_launch();
  const long r = blockIdx.x;
  T ss = T(0);
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    T u = y[r * ldy + c] * silu(cvt<T>(z[r * ldz + c]));
    ss += u * u;
  }
  ss = block_sum(ss, red);
  const T denom = sqrt_(ss / T(D) + eps);
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    T u = y[r * ldy + c] * silu(cvt<T>(z[r * ldz + c]));
    out[r * ldo + c] = cvt<TO>(w ? (u / denom) * w[c] : u / denom);
  }
}

// ungated RMSNorm — numerics.py:161-166 (final norm before the tied head)
template <typename T, typename TO>
__global__ __launch_bounds__(256) void rmsnorm_rows(const T *__restrict__ x, long ldx,
                                                    const T *__restrict__ w,
                                                    TO *__restrict__ out, long ldo, int D, T eps) {
  __shared__ T red[32];
  griddep_wait();  // no-op unless launched as a programmatic dependent (the bf16 head)
  griddep_launch();
  const long r = blockIdx.x;
  T ss = T(0);
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    T v = x[r * ldx + c];
    ss += v * v;
  }
  ss = block_sum(ss, red);
  const T denom = sqrt_(ss / T(D) + eps);
  for (int c = threadIdx.x; c < D; c += blockDim.x)
    out[r * ldo + c] = cvt<TO>((x[r * ldx + c] / denom) * w[c]);
}

// =========================================================================
// greedy argmax, ties -> lowest id (decode.py:72-74); one block per row
// =========================================================================
template <typename T>
__global__ __launch_bounds__(256) void argmax_rows(const T *__restrict__ logits, long ld, int V,
                                                   int64_t *__restrict__ out) {
  __shared__ T bv[256];
  __shared__ int bi[256];
  const long r = blockIdx.x;
  T best = -INFINITY;
  int idx = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    T x = logits[r * ld + v];
    if (x > best || (x == best && v < idx)) {
      best = x;
      idx = v;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      T o = bv[threadIdx.x + s];
      int oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = bi[0] == 0x7fffffff ? 0 : bi[0];
}

// =========================================================================
// decode: conv window roll + readout — decode.py:103-108, roll_and_insert
// (:65-69).  One thread per (b, channel); conv_out may alias conv_in.
// =========================================================================
template <typename T, typename TU>
__global__ void decode_conv(const TU *__restrict__ u, long ldu, int col0, const T *conv_in,
                            T *conv_out, const T *__restrict__ w, const T *__restrict__ bias,
                            T *__restrict__ act, int Bsz, int C, int k) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)Bsz * C) return;
  const int c = (int)(i % C);
  const int b = (int)(i / C);
  const int km = k - 1;
  T win[16];
  for (int j = 0; j < km; ++j) win[j] = conv_in[((long)b * C + c) * km + j];
  win[km] = cvt<T>(u[(long)b * ldu + col0 + c]);
  T acc = T(0);
  for (int j = 0; j < k; ++j) acc += win[j] * w[(long)c * k + j];
  act[i] = silu(acc + bias[c]);
  for (int j = 0; j < km; ++j) conv_out[((long)b * C + c) * km + j] = win[j + 1];
}

// decode: state update + readout + D skip — decode.py:111-132.
// grid (H, B); warps over head rows p, lanes over state columns n.
// ssm_out may alias ssm_in (each element is read then written by one thread).
template <typename T, typename TU>
__global__ __launch_bounds__(128) void decode_ssm(const TU *__restrict__ u, long ldu, int dt_col0,
                                                  const T *__restrict__ act, int d_inner,
                                                  const T *__restrict__ dt_bias,
                                                  const T *__restrict__ a,
                                                  const T *__restrict__ D, const T *ssm_in,
                                                  T *ssm_out, T *__restrict__ y, long ldy, int H,
                                                  int P, int G, int N, T lo, T hi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *bs = reinterpret_cast<T *>(smem_raw);
  T *csh = bs + N;
  const int h = blockIdx.x, b = blockIdx.y;
  const int g = h / (H / G);
  const int conv_dim = d_inner + 2 * G * N;
  const T *arow = act + (long)b * conv_dim;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    bs[n] = arow[d_inner + g * N + n];
    csh[n] = arow[d_inner + G * N + g * N + n];
  }
  __syncthreads();
  const T dt = clamp_(softplus(cvt<T>(u[(long)b * ldu + dt_col0 + h]) + dt_bias[h]), lo, hi);
  const T decay = exp_(a[h] * dt);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const long base = (((long)b * H + h) * P) * N;
  for (int pp = warp; pp < P; pp += nw) {
    const T xv = arow[(long)h * P + pp];
    const T dx = dt * xv;
    T acc = T(0);
    for (int n = lane; n < N; n += 32) {
      long idx = base + (long)pp * N + n;
      T hv = decay * ssm_in[idx] + dx * bs[n];
      ssm_out[idx] = hv;
      acc = fma(csh[n], hv, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) y[(long)b * ldy + (long)h * P + pp] = acc + D[h] * xv;
  }
}

}  // namespace ssd200
