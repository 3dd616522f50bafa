// C-ABI entry points (include/ssd200.h): validation, workspace carving and
// the per-layer launch sequences.  No allocation, no host sync.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <set>
#include <tuple>
#include <string>
#include <type_traits>

#include "../../include/ssd200.h"
#include "common.cuh"
#include "simt.cuh"
#include "decode.cuh"
#include "ssd_tc.cuh"
#include "tc_gemm.cuh"
#include "decode_gemm.cuh"

using namespace ssd200;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;
thread_local void *const *g_phase_ev = nullptr;  // bench instrumentation only
thread_local int g_nphase = 0;

// launch-timeline slots (SSD200_TRACE diagnostic builds; -1 otherwise)
#ifdef SSD200_TRACE
std::mutex g_trace_mu;
int g_trace_next = 0;
char g_trace_name[TRACE_SLOTS][32];
int trace_slot(const char *name) {
  std::lock_guard<std::mutex> lk(g_trace_mu);
  if (g_trace_next >= TRACE_SLOTS) return -1;
  snprintf(g_trace_name[g_trace_next], 32, "%s", name);
  return g_trace_next++;
}
__global__ void trace_init_kernel() {
  for (int i = threadIdx.x; i < TRACE_SLOTS; i += blockDim.x)
    for (int k = 0; k < 6; ++k) g_trace[i][k] = (k & 1) ? 0ull : ~0ull;
  if (threadIdx.x < 16) g_cyc[threadIdx.x] = 0ull;
}
#else
inline int trace_slot(const char *) { return -1; }
#endif

// Implementation choices come with each call (ssd200_dims_t.tuning); TuneScope
// makes them visible to the launch helpers for the duration of that call only.
ssd200_tuning_t make_default_tuning() {
  ssd200_tuning_t t{};
  t.size = (int)sizeof(ssd200_tuning_t);
  t.prefill_pdl = 1;         // 370M B=1 T=2K +11%, neutral at B=4 T=8K
  t.gemm_pair = 1;           // 370M prefill +3.6%, 2.7B +11%
  t.pair_min_tiles = 64;     // pairs win from 64 tiles (370M B=1 T=4K 559K -> 616K tok/s)
  t.scan_variant = 0;
  t.chunkscan_multicast = 1;
  t.out_waves = 1;
  t.dec_pdl = 1;
  t.dec_swap = 1;
  t.dec_small_ring = -1;
  t.dec_small_max = 32;      // 1.3B: small ring B = 32 2.34 -> 2.25 ms, big ring B = 40 2.59 -> 2.49,
                             // B = 48 2.89 -> 2.75 ms
  t.dec_split_in = 0;
  t.dec_split_out = 0;
  t.stream_stages = 0;
  t.stream_cps = 0;
  t.stream_cw = 8;
  t.out_interleave = 1;
  t.gemm_group_m = 0;
  t.gemm_stream = 1;
  t.stream_chunk = 0;
  t.stream_reg_state = 1;
  return t;
}
const ssd200_tuning_t kDefaultTuning = make_default_tuning();
thread_local const ssd200_tuning_t *g_tune = nullptr;
inline const ssd200_tuning_t &tune() { return g_tune ? *g_tune : kDefaultTuning; }
struct TuneScope {
  const ssd200_tuning_t *prev;
  explicit TuneScope(const ssd200_dims_t *d) : prev(g_tune) {
    g_tune = (d && d->tuning && d->tuning->size == (int)sizeof(ssd200_tuning_t)) ? d->tuning
                                                                                  : nullptr;
  }
  ~TuneScope() { g_tune = prev; }
};

// bench phases of a prefill layer.  PH_SCAN: the chunk states (tensor-core path:
// cumsum + chunk walk) or the whole SIMT scan; PH_GATE: the gated output — the
// tensor-core output kernel (intra-chunk + cross-chunk outputs, D skip, gate) or
// the SIMT gated norm
enum { PH_IN_PROJ = 0, PH_CONV = 1, PH_SCAN = 2, PH_GATE = 3, PH_OUT_PROJ = 4 };

inline void phase_mark(int p, int end, cudaStream_t st) {
  if (g_phase_ev && p < g_nphase)
    cudaEventRecord(static_cast<cudaEvent_t>(g_phase_ev[2 * p + end]), st);
}

void set_err(const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

#define REQUIRE(cond, code, ...) \
  do {                           \
    if (!(cond)) {               \
      set_err(__VA_ARGS__);      \
      return code;               \
    }                            \
  } while (0)

int check_launch(const char *what) {
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err("%s: %s", what, cudaGetErrorString(e));
    return SSD200_ELAUNCH;
  }
  return SSD200_OK;
}

#define LAUNCH_CHECK(what)             \
  do {                                 \
    int _rc = check_launch(what);      \
    if (_rc) return _rc;               \
  } while (0)

inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// simple bump allocator over the caller's workspace
struct Carve {
  char *base;
  size_t used = 0, cap;
  Carve(void *p, size_t c) : base(static_cast<char *>(p)), cap(c) {}
  template <typename T> T *take(size_t n) {
    size_t off = used;
    used = align_up(used + n * sizeof(T));
    return reinterpret_cast<T *>(base ? base + off : nullptr);
  }
  bool ok() const { return used <= cap; }
};

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// SM count of the calling thread's current device (cached per device)
int num_sms() {
  static std::atomic<int> cache[64];
  const int dev = current_device();
  if (dev < 0 || dev >= 64) return 148;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// opt a kernel into `bytes` of dynamic shared memory on the current device
// (the attribute is per device; set once per (kernel, device, size), thread-safe)
template <typename... KArgs>
void smem_attr(void (*kern)(KArgs...), int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void *, int, int>> done;
  const auto key = std::make_tuple(reinterpret_cast<const void *>(kern), current_device(), bytes);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert(key).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// --------------------------------------------------------------- TMA maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 map over a row-major (rows, cols) matrix with leading dim ld,
// box = (64 cols = 128 B, box_rows), SWIZZLE_128B.
int make_map_2d(CUtensorMap *m, const void *ptr, long rows, long cols, long ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  REQUIRE(fn, SSD200_ELAUNCH, "cuTensorMapEncodeTiled unavailable");
  REQUIRE(((uintptr_t)ptr & 15) == 0, SSD200_EINVAL, "TMA base pointer not 16-byte aligned");
  REQUIRE((ld * 2) % 16 == 0, SSD200_EINVAL, "TMA row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  REQUIRE(r == CUDA_SUCCESS, SSD200_ELAUNCH, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SSD200_OK;
}

// 2-D bf16 map without swizzle, box (box_cols, box_rows)
int make_map_2d_plain(CUtensorMap *m, const void *ptr, long rows, long cols, long ld, int box_cols,
                      int box_rows) {
  EncodeTiledFn fn = encode_fn();
  REQUIRE(fn, SSD200_ELAUNCH, "cuTensorMapEncodeTiled unavailable");
  REQUIRE(((uintptr_t)ptr & 15) == 0, SSD200_EINVAL, "TMA base pointer not 16-byte aligned");
  REQUIRE((ld * 2) % 16 == 0, SSD200_EINVAL, "TMA row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  REQUIRE(r == CUDA_SUCCESS, SSD200_ELAUNCH, "cuTensorMapEncodeTiled(plain) failed (%d)", (int)r);
  return SSD200_OK;
}

// launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor drains; it waits (griddepcontrol.wait) before reading
// the predecessor's outputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// decode kernels: always PDL (their weight streams start before the wait)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  return launch_ex(tune().dec_pdl, kern, grid, block, smem, st, args...);
}
// prefill kernels: PDL per ssd200_tuning_t.prefill_pdl
template <typename... KArgs, typename... Args>
cudaError_t launch_pf(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t st, Args... args) {
  return launch_ex(tune().prefill_pdl, kern, grid, block, smem, st, args...);
}

template <int BN, int EPI>
int launch_tc_gemm_bn(const bf16 *A, long lda, const bf16 *B, long ldb, int M, int N, int K,
                      const TcEpilogue &ep, cudaStream_t st, bool pdl) {
  using Cfg = TcCfg<BN>;
  CUtensorMap ta, tb;
  int rc = make_map_2d(&ta, A, M, K, lda, Cfg::BM);
  if (rc) return rc;
  rc = make_map_2d(&tb, B, N, K, ldb, BN);
  if (rc) return rc;
  smem_attr(tc_gemm_kernel<BN, EPI>, (int)Cfg::SMEM);
  const int ks = (EPI == TC_EPI_F32 && ep.ksplit > 1) ? ep.ksplit : 1;
  const int tiles = ((M + Cfg::BM - 1) / Cfg::BM) * ((N + BN - 1) / BN) * ks;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  cudaError_t e = launch_ex(pdl || tune().prefill_pdl, tc_gemm_kernel<BN, EPI>, dim3(grid), dim3(320),
                            Cfg::SMEM, st, ta, tb, M, N, K, ep);
  REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "tc_gemm_kernel: %s", cudaGetErrorString(e));
  LAUNCH_CHECK("tc_gemm_kernel");
  return SSD200_OK;
}

// CTA-pair variant (cluster of 2, cta_group::2, 256-row tiles)
template <int BN, int EPI>
int launch_tc_gemm_pair(const bf16 *A, long lda, const bf16 *B, long ldb, int M, int N, int K,
                        const TcEpilogue &ep, cudaStream_t st, bool pdl) {
  using Cfg = TcCfg<BN, true>;
  CUtensorMap ta, tb;
  int rc = make_map_2d(&ta, A, M, K, lda, Cfg::BM);
  if (rc) return rc;
  rc = make_map_2d(&tb, B, N, K, ldb, BN / 2);
  if (rc) return rc;
  smem_attr(tc_gemm_kernel<BN, EPI, true>, (int)Cfg::SMEM);
  const int tiles = ((M + 255) / 256) * ((N + BN - 1) / BN);
  const int pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = (pdl || tune().prefill_pdl) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, EPI, true>, ta, tb, M, N, K, ep);
  REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "tc_gemm_kernel (pair): %s", cudaGetErrorString(e));
  LAUNCH_CHECK("tc_gemm_kernel (pair)");
  return SSD200_OK;
}

// D (M,N) = A (M,K) . B (N,K)^T, bf16 operands, fused epilogue.
template <int EPI>
int tc_gemm(const bf16 *A, long lda, const bf16 *B, long ldb, int M, int N, int K,
            const TcEpilogue &ep_in, cudaStream_t st, bool pdl = false) {
  TcEpilogue ep = ep_in;
  // grouped tile order for wide weights (many 256-column tiles): in_proj 2.7B B=32
  // 24.8 -> 13.6 GB of DRAM traffic; row-major for narrow ones (out_proj)
  const int gm = tune().gemm_group_m;
  ep.group_m = gm > 0 ? gm : ((N + 255) / 256 > 16 ? 16 : 1);
  // evict-first epilogue accesses once the output dwarfs L2 (>= 1 GB as f32): 2.7B at
  // C4 +0.8 %, in_proj / out_proj DRAM reads 10.7 -> 9.9 / 12.2 -> 11.5 GB per launch;
  // at 370M B = 4 (0.1-0.6 GB) the next kernel still finds part of the output in L2
  // and evict-first measured -1 % (profiles/r02_prefill_ab_gemm_stream.txt)
  ep.stream = tune().gemm_stream == 2 ||
              (tune().gemm_stream == 1 && (double)M * N * 4.0 >= 1024.0 * 1024 * 1024);
  pdl = pdl && tune().dec_pdl;
  REQUIRE(M > 0 && N > 0 && K > 0, SSD200_EINVAL, "tc_gemm: empty problem");
  REQUIRE(K % 8 == 0, SSD200_EINVAL, "tc_gemm: K must be a multiple of 8");
  REQUIRE(ep.ksplit <= 1 || (EPI == TC_EPI_F32 && ep.ksplit <= (K + 63) / 64), SSD200_EINVAL,
          "tc_gemm: split-K needs the F32 epilogue and at least one K block per split");
  if (EPI == TC_EPI_F32 && ep.ksplit > 1)  // split-K: always 128-wide tiles (most tiles)
    return launch_tc_gemm_bn<128, EPI>(A, lda, B, ldb, M, N, K, ep, st, pdl);
  {
    // CTA pairs when 256 x 256 tiles still cover the SMs several times
    const long tiles_pair = (long)((M + 255) / 256) * ((N + 255) / 256);
    // measured: pairs win from 64 tiles (370M B=1 T=4K 559K -> 616K tok/s, B=2 T=2K
    // 655K -> 685K); at 32 tiles (B=1 T=2K out_proj) the 128-wide single tiles win
    const long min_pair = tune().pair_min_tiles > 0 ? tune().pair_min_tiles : 64;
    if (tune().gemm_pair && N > 128 && tiles_pair >= min_pair)
      return launch_tc_gemm_pair<256, EPI>(A, lda, B, ldb, M, N, K, ep, st, pdl);
  }
  // 128-wide tiles when 256-wide ones would leave SMs idle (few row tiles: decode batches)
  // (prefill at B = 1 / short T: the out_proj's 256-wide tiles covered 64 of 148 SMs)
  const long tiles256 = (long)((M + 127) / 128) * ((N + 255) / 256);
  if (N <= 128 || tiles256 < num_sms())
    return launch_tc_gemm_bn<128, EPI>(A, lda, B, ldb, M, N, K, ep, st, pdl);
  return launch_tc_gemm_bn<256, EPI>(A, lda, B, ldb, M, N, K, ep, st, pdl);
}

// --------------------------------------------------------------- SSD scan
inline size_t scan_ws_bytes(size_t elt, long B, long T, long H, long P, long N, long L) {
  long Nc = (T + L - 1) / L;
  return align_up(B * Nc * H * P * N * elt) + align_up(B * H * Nc * elt);
}

template <typename T, typename TI>
int run_scan(SsdArgs<T, TI> a, void *ws, size_t ws_bytes, cudaStream_t st) {
  REQUIRE(a.L >= 1 && a.L <= 2048, SSD200_EUNSUPPORTED, "chunk_size %d outside [1, 2048]", a.L);
  REQUIRE((long)a.P * a.N <= 256L * SSD_MAX_PN_PER_THREAD, SSD200_EUNSUPPORTED,
          "head_dim*d_state = %d exceeds %d", a.P * a.N, 256 * SSD_MAX_PN_PER_THREAD);
  REQUIRE(a.P <= 256, SSD200_EUNSUPPORTED, "head_dim > 256");
  REQUIRE(a.H % a.G == 0, SSD200_EINVAL, "head count %d not divisible by group count %d", a.H,
          a.G);
  a.Nc = (a.T_ + a.L - 1) / a.L;
  Carve cv(ws, ws_bytes);
  a.S = cv.take<T>((size_t)a.B * a.Nc * a.H * a.P * a.N);
  a.cs_end = cv.take<T>((size_t)a.B * a.H * a.Nc);
  REQUIRE(cv.ok(), SSD200_EWORKSPACE, "scan workspace %zu < %zu", ws_bytes, cv.used);
  const size_t smem1 = (3 * (size_t)a.L + 16 * (size_t)a.P + 16 * (size_t)a.N) * sizeof(T);
  const size_t smem3 =
      (2 * (size_t)a.L + 16 * (size_t)a.N + 32 * ((size_t)a.N + 1) + 32 * (size_t)a.P + 16 * 32) *
      sizeof(T);
  REQUIRE(smem1 <= 220 * 1024 && smem3 <= 220 * 1024, SSD200_EUNSUPPORTED,
          "scan shared memory too large");
  smem_attr(ssd_chunk_state<T, TI>, 220 * 1024);
  smem_attr(ssd_chunk_out<T, TI>, 220 * 1024);
  ssd_chunk_state<T, TI><<<dim3(a.Nc, a.H, a.B), 256, smem1, st>>>(a);
  LAUNCH_CHECK("ssd_chunk_state");
  const int PN = a.P * a.N;
  ssd_state_pass<T><<<dim3((PN + 255) / 256, a.H, a.B), 256, 0, st>>>(a.S, a.cs_end, a.init,
                                                                       a.final_state, a.H, PN,
                                                                       a.Nc);
  LAUNCH_CHECK("ssd_state_pass");
  const int nRT = (a.L + 15) / 16;
  ssd_chunk_out<T, TI><<<dim3(a.Nc * nRT, a.H, a.B), 256, smem3, st>>>(a);
  LAUNCH_CHECK("ssd_chunk_out");
  return SSD200_OK;
}

int check_dims(const ssd200_dims_t *d) {
  REQUIRE(d, SSD200_EINVAL, "null dims");
  REQUIRE(d->dtype == SSD200_F32 || d->dtype == SSD200_F64 || d->dtype == SSD200_BF16,
          SSD200_EINVAL, "unknown dtype %d", d->dtype);
  REQUIRE(d->d_model > 0 && d->d_inner > 0 && d->n_heads > 0 && d->head_dim > 0 &&
              d->d_state > 0 && d->n_groups > 0 && d->conv_kernel >= 1 && d->chunk_size >= 1,
          SSD200_EINVAL, "non-positive model dims");
  REQUIRE(d->n_heads * d->head_dim == d->d_inner, SSD200_EINVAL, "n_heads*head_dim != d_inner");
  REQUIRE(d->n_heads % d->n_groups == 0, SSD200_EINVAL, "n_heads %% n_groups != 0");
  REQUIRE(d->conv_kernel <= 16, SSD200_EUNSUPPORTED, "conv_kernel > 16");
  REQUIRE(!d->tuning || d->tuning->size == (int)sizeof(ssd200_tuning_t), SSD200_EINVAL,
          "tuning.size %d != sizeof(ssd200_tuning_t) %d (header / library mismatch)",
          d->tuning->size, (int)sizeof(ssd200_tuning_t));
  return SSD200_OK;
}

struct Widths {
  long conv_dim, d_in_proj, gn;
};
inline Widths widths(const ssd200_dims_t *d) {
  Widths w;
  w.gn = (long)d->n_groups * d->d_state;
  w.conv_dim = d->d_inner + 2 * w.gn;
  w.d_in_proj = 2L * d->d_inner + 2 * w.gn + d->n_heads;
  return w;
}

inline unsigned blocks_for(long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

template <typename T, typename TI, typename TO>
void launch_conv(const TI *in, long ld_in, const T *w, const T *bias, TO *out, long ld_out, int Tn,
                 int C, int k, long rows, cudaStream_t st) {
  if constexpr (std::is_same<TI, bf16>::value && std::is_same<TO, bf16>::value &&
                std::is_same<T, float>::value) {
    if (k == 4 && C % 8 == 0 && ld_in % 8 == 0 && ld_out % 8 == 0 &&
        ((uintptr_t)in & 15) == 0 && ((uintptr_t)out & 15) == 0) {
      constexpr int ROWS = 8;
      const dim3 g8(blocks_for(C, 256), blocks_for(rows, 8 * ROWS));
      conv_silu_bf16x8<4, ROWS><<<g8, dim3(32, 8), 0, st>>>(in, ld_in, w, bias, out, ld_out, Tn,
                                                          C, rows);
      return;
    }
  }
  const dim3 grid(blocks_for(C), blocks_for(rows, 16));
  if (k == 4)
    conv_silu_prefill<T, TI, TO, 4><<<grid, 256, 0, st>>>(in, ld_in, w, bias, out, ld_out, Tn, C,
                                                          k, rows);
  else
    conv_silu_prefill<T, TI, TO, 0><<<grid, 256, 0, st>>>(in, ld_in, w, bias, out, ld_out, Tn, C,
                                                          k, rows);
}

// ----------------------------------------------------- tensor-core SSD path
// Production Mamba-2 head dims: the tcgen05 scan (ssd_tc.cuh) handles these;
// anything else runs the generic CUDA-core scan.
inline bool tc_ssd_eligible(const ssd200_dims_t *d) {
  // (H % 8: the in_proj row pitch 2 d_inner + 2 N + H stays 16-byte aligned for TMA)
  return d->head_dim == TC_P && d->d_state == TC_N && d->chunk_size == TC_L &&
         d->n_groups == 1 && d->conv_kernel >= 1 && d->n_heads % 8 == 0;
}

struct TcScanWs {
  float *cs, *cs_end, *S, *dtT;
  bf16 *prev;
};

inline size_t tc_scan_carve(int B, int Tn, int H, void *base, TcScanWs *o) {
  const long Nc = (Tn + TC_L - 1) / TC_L;
  Carve cv(base, SIZE_MAX);
  float *S = cv.take<float>((size_t)B * Nc * H * TC_P * TC_N);
  bf16 *prev = cv.take<bf16>((size_t)B * Nc * H * TC_P * TC_N);
  float *cs = cv.take<float>((size_t)B * H * Nc * TC_L);
  float *dtT = cv.take<float>((size_t)B * H * Nc * TC_L);
  float *ce = cv.take<float>((size_t)B * H * Nc);
  if (o) *o = TcScanWs{cs, ce, S, dtT, prev};
  return cv.used;
}

inline size_t tc_scan_ws_bytes(int B, int Tn, int H) { return tc_scan_carve(B, Tn, H, nullptr, nullptr); }

// 3-D bf16 map over (B, T, cols) with row pitch ld: box (64 cols, box_rows, 1)
int make_map_3d(CUtensorMap *m, const void *ptr, long B, long T, long cols, long ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  REQUIRE(fn, SSD200_ELAUNCH, "cuTensorMapEncodeTiled unavailable");
  REQUIRE(((uintptr_t)ptr & 15) == 0, SSD200_EINVAL, "TMA base pointer not 16-byte aligned");
  REQUIRE((ld * 2) % 16 == 0, SSD200_EINVAL, "TMA row stride must be a multiple of 16 bytes");
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)T, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)ld * 2 * T};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  REQUIRE(r == CUDA_SUCCESS, SSD200_ELAUNCH, "cuTensorMapEncodeTiled(3d) failed (%d)", (int)r);
  return SSD200_OK;
}

// smallest divisor of H giving at least `target` CTAs over `units` work units
// (at most max_hg heads per group, heads per group a multiple of `mult`)
inline int pick_groups(int H, long units, long target, int max_hg = 1 << 30, int mult = 1) {
  auto ok = [&](int ng) { return H % ng == 0 && H / ng <= max_hg && (H / ng) % mult == 0; };
  for (int ng = 1; ng <= H; ++ng)
    if (ok(ng) && units * ng >= target) return ng;
  for (int ng = 1; ng <= H; ++ng)
    if (ok(ng)) return ng;
  return H;
}

// act: post-conv xBC (B*T, conv_dim) bf16; z: gate (B*T, z_ld) bf16.
// Writes u (B*T, d_inner) bf16, ssq (B*T, NG) f32, final state (B,H,P,N) f32.
int run_tc_scan(const ssd200_dims_t *d, const ssd200_layer_t *w, const bf16 *act, long conv_dim,
                const bf16 *z, long z_ld, const float *dt, float *final_state, bf16 *u_out,
                float *ssq, int *ng_out, void *scan_ws, int B, int Tn, cudaStream_t st) {
  smem_attr(ssd_tc_state, (int)StateSmem::TOTAL);
  smem_attr(ssd_tc_out, (int)OutSmem::TOTAL);
  smem_attr(ssd_tc_chunkscan, (int)ScanSmem::TOTAL);
  const int H = d->n_heads;
  TcSsdArgs a{};
  a.B = B;
  a.T = Tn;
  a.H = H;
  a.Nc = (Tn + TC_L - 1) / TC_L;
  a.d_inner = d->d_inner;
  a.z = z;
  a.z_ld = z_ld;
  a.dt = dt;
  a.a = static_cast<const float *>(w->a);
  a.D = static_cast<const float *>(w->D);
  a.init = nullptr;
  TcScanWs ws;
  tc_scan_carve(B, Tn, H, scan_ws, &ws);
  a.cs = ws.cs;
  a.dtT = ws.dtT;
  a.cs_end = ws.cs_end;
  a.S = ws.S;
  a.prev = ws.prev;
  a.final_state = final_state;
  a.u_out = u_out;
  a.ssq = ssq;
  CUtensorMap tm_act, tm_prev, tm_z, tm_u;
  int rc = make_map_3d(&tm_act, act, B, Tn, conv_dim, conv_dim, 128);
  if (rc) return rc;
  rc = make_map_3d(&tm_z, z, B, Tn, d->d_inner, z_ld, 128);
  if (rc) return rc;
  rc = make_map_3d(&tm_u, u_out, B, Tn, d->d_inner, d->d_inner, 32);
  if (rc) return rc;
  rc = make_map_2d(&tm_prev, ws.prev, (long)B * a.Nc * H * TC_N, TC_P, TC_P, 128);
  if (rc) return rc;
  const long sms = num_sms();
  // chunk cumsums
  phase_mark(PH_SCAN, 0, st);
  REQUIRE(launch_pf(ssd_tc_cumsum, dim3(B * a.Nc, (H + 7) / 8), dim3(256), 0, st, a) ==
              cudaSuccess,
          SSD200_ELAUNCH, "ssd_tc_cumsum launch");
  LAUNCH_CHECK("ssd_tc_cumsum");
  // measured (370M, T = 2K..16K): the fused walk beats parallel states + pass from
  // B * H = 32 up (B = 1: 240 K -> 392 K tok/s at T = 2K, 640 K -> 755 K at T = 16K)
  const int variant = tune().scan_variant;
  if (variant == 1 || (variant == 0 && (long)B * H >= sms / 6)) {
    // chunk states + inter-chunk pass fused: one CTA per (b, h), chunks in order
    // clusters of 4 heads of one batch row share each chunk's B tile by multicast
    const int mc = (H % 4 == 0 && tune().chunkscan_multicast) ? 4 : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(B * H);
    cfg.blockDim = dim3(CHUNKSCAN_THREADS);
    cfg.dynamicSmemBytes = ScanSmem::TOTAL;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = mc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = tune().prefill_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, ssd_tc_chunkscan, tm_act, a, mc);
    REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "ssd_tc_chunkscan: %s", cudaGetErrorString(e));
    LAUNCH_CHECK("ssd_tc_chunkscan");
  } else {
    // few (b, h) pairs: parallel chunk states, then the O(Nc) pass
    a.NG = pick_groups(H, (long)B * a.Nc, 2 * sms);
    a.HG = H / a.NG;
    REQUIRE(launch_pf(ssd_tc_state, dim3(B * a.Nc * a.NG), dim3(192), StateSmem::TOTAL, st,
                       tm_act, a) == cudaSuccess,
            SSD200_ELAUNCH, "ssd_tc_state launch");
    LAUNCH_CHECK("ssd_tc_state");
    REQUIRE(launch_pf(ssd_tc_pass, dim3(B * H, TC_P * TC_N / 256), dim3(256), 0, st, a) ==
                cudaSuccess,
            SSD200_ELAUNCH, "ssd_tc_pass launch");
    LAUNCH_CHECK("ssd_tc_pass");
  }
  phase_mark(PH_SCAN, 1, st);
  // outputs (+ D skip + gate)
  // head groups of whole SSQ_SLICE-head slices: sum u^2 leaves per slice, so the grouping
  // (which depends on B) does not change any row's result
  a.interleave = tune().out_interleave;
  a.NG = pick_groups(H, (long)B * a.Nc * 2, (tune().out_waves > 0 ? tune().out_waves : 1) * sms, OutSmem::MAX_HG, SSQ_SLICE);
  a.HG = H / a.NG;
  phase_mark(PH_GATE, 0, st);
  REQUIRE(launch_pf(ssd_tc_out, dim3(B * a.Nc * 2 * a.NG), dim3(OUT_THREADS), OutSmem::TOTAL, st,
                     tm_act, tm_prev, tm_z, tm_u, a) == cudaSuccess,
          SSD200_ELAUNCH, "ssd_tc_out launch");
  LAUNCH_CHECK("ssd_tc_out");
  phase_mark(PH_GATE, 1, st);
  *ng_out = (H / SSQ_SLICE) * OUT_KW;  // sum u^2 partials per row, (slice, column half)
  return SSD200_OK;
}

// ------------------------------------------------------------ prefill layer
// workspace carve (identical in sizing and launch)
template <typename T> struct PrefillWs {
  void *xn;    // pre-norm only: rmsnorm(hidden) * pre_norm_w, (rows, d_model) T or bf16
  void *u;     // f32/f64: (rows, d_in_proj) T;  bf16: (rows, d_inner+conv_dim) bf16
  void *act;   // post-conv xBC: T or bf16 (rows, conv_dim); reused for the normed y
  T *dt;       // (rows, H)
  T *y;        // (rows, d_inner)
  void *scan;  // scan workspace
  size_t scan_bytes;
};

template <typename T>
bool carve_prefill(const ssd200_dims_t *d, int B, int Tn, void *ws, size_t cap, PrefillWs<T> &o,
                   size_t *need) {
  Widths w = widths(d);
  const long rows = (long)B * Tn;
  const bool lp = d->dtype == SSD200_BF16;
  Carve cv(ws, cap);
  o.xn = lp ? (void *)cv.take<bf16>(rows * d->d_model) : (void *)cv.take<T>(rows * d->d_model);
  if (lp) {
    o.u = cv.take<bf16>(rows * (d->d_inner + w.conv_dim));
    o.act = cv.take<bf16>(rows * w.conv_dim);
  } else {
    o.u = cv.take<T>(rows * w.d_in_proj);
    o.act = cv.take<T>(rows * w.conv_dim);
  }
  o.dt = cv.take<T>(rows * d->n_heads);
  o.y = cv.take<T>(rows * d->d_inner);
  o.scan_bytes = (lp && tc_ssd_eligible(d))
                     ? tc_scan_ws_bytes(B, Tn, d->n_heads)
                     : scan_ws_bytes(sizeof(T), B, Tn, d->n_heads, d->head_dim, d->d_state,
                                     d->chunk_size);
  o.scan = cv.take<char>(o.scan_bytes);
  if (need) *need = cv.used;
  return cv.ok();
}

template <typename T>
int prefill_layer_simt(const ssd200_dims_t *d, const ssd200_layer_t *w, T *hidden, T *ssm_out,
                       T *conv_out, int B, int Tn, void *ws, size_t ws_bytes, cudaStream_t st) {
  PrefillWs<T> o;
  size_t need = 0;
  REQUIRE(carve_prefill<T>(d, B, Tn, ws, ws_bytes, o, &need), SSD200_EWORKSPACE,
          "prefill workspace %zu < %zu", ws_bytes, need);
  Widths wd = widths(d);
  const long rows = (long)B * Tn;
  T *u = static_cast<T *>(o.u);
  T *act = static_cast<T *>(o.act);
  const int k = d->conv_kernel;
  // optional residual pre-norm (ssd200_layer_t.pre_norm_w): in_proj reads the normed copy
  const T *xin = hidden;
  if (w->pre_norm_w) {
    rmsnorm_rows<T, T><<<(unsigned)rows, 256, 0, st>>>(hidden, d->d_model,
                                                      static_cast<const T *>(w->pre_norm_w),
                                                      static_cast<T *>(o.xn), d->d_model,
                                                      d->d_model, (T)d->norm_eps);
    LAUNCH_CHECK("pre_norm");
    xin = static_cast<const T *>(o.xn);
  }
  // in_proj: u = hidden . W_in   (model.py:141)
  gemm_simt<T, false, EPI_STORE><<<dim3(blocks_for(wd.d_in_proj, 64), blocks_for(rows, 64)),
                                   256, 0, st>>>(xin, d->d_model,
                                                 static_cast<const T *>(w->W_in), wd.d_in_proj,
                                                 u, wd.d_in_proj, (int)rows, (int)wd.d_in_proj,
                                                 d->d_model);
  LAUNCH_CHECK("gemm_simt in_proj");
  // conv tail (pre-activation) + conv/SiLU + dt
  if (k > 1) {
    conv_tail_kernel<T, T><<<blocks_for((long)B * wd.conv_dim * (k - 1)), 256, 0, st>>>(
        u + d->d_inner, wd.d_in_proj, conv_out, B, Tn, (int)wd.conv_dim, k);
    LAUNCH_CHECK("conv_tail");
  }
  launch_conv<T, T, T>(u + d->d_inner, wd.d_in_proj, static_cast<const T *>(w->conv_w),
                       static_cast<const T *>(w->conv_b), act, wd.conv_dim, Tn, (int)wd.conv_dim,
                       k, rows, st);
  LAUNCH_CHECK("conv_silu_prefill");
  dt_kernel<T, T><<<blocks_for(rows * d->n_heads), 256, 0, st>>>(
      u + d->d_inner + wd.conv_dim, wd.d_in_proj, static_cast<const T *>(w->dt_bias), o.dt, rows,
      d->n_heads, (T)d->dt_min, (T)d->dt_max);
  LAUNCH_CHECK("dt_kernel");
  // SSD (+ D skip)
  SsdArgs<T, T> sa{};
  sa.X = act;
  sa.x_ts = wd.conv_dim;
  sa.dt = o.dt;
  sa.dt_ts = d->n_heads;
  sa.a = static_cast<const T *>(w->a);
  sa.Bm = act + d->d_inner;
  sa.Cm = act + d->d_inner + wd.gn;
  sa.bc_ts = wd.conv_dim;
  sa.D = static_cast<const T *>(w->D);
  sa.init = nullptr;
  sa.Y = o.y;
  sa.y_ts = d->d_inner;
  sa.final_state = ssm_out;
  sa.B = B;
  sa.T_ = Tn;
  sa.H = d->n_heads;
  sa.P = d->head_dim;
  sa.G = d->n_groups;
  sa.N = d->d_state;
  sa.L = d->chunk_size;
  int rc = run_scan<T, T>(sa, o.scan, o.scan_bytes, st);
  if (rc) return rc;
  // gated norm -> act (reused), then out_proj + residual
  gated_norm_kernel<T, T, T><<<(unsigned)rows, 256, 0, st>>>(
      o.y, d->d_inner, u, wd.d_in_proj, static_cast<const T *>(w->norm_w), act, d->d_inner,
      d->d_inner, (T)d->norm_eps);
  LAUNCH_CHECK("gated_norm");
  gemm_simt<T, false, EPI_ADD><<<dim3(blocks_for(d->d_model, 64), blocks_for(rows, 64)), 256, 0,
                                 st>>>(act, d->d_inner, static_cast<const T *>(w->W_out),
                                       d->d_model, hidden, d->d_model, (int)rows, d->d_model,
                                       d->d_inner);
  LAUNCH_CHECK("gemm_simt out_proj");
  return SSD200_OK;
}

// sum of the slice partial sums of u^2 ((ng, rows), slice-major) -> column `col`
// of a strided row
__global__ void ssq_groups_kernel(const float *__restrict__ ssq, int ng, long rows,
                                  float *__restrict__ dst, long ld, int col) {
  const long r = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float s = 0.f;
  for (int g = 0; g < ng; ++g) s += ssq[g * rows + r];
  dst[r * ld + col] = s;
}

// head-sharded residual update: hidden += partial * rsqrt(ssq / d_inner + eps)
// (partial rows of width ld, ssq in column d_model), bf16 shadow (model.py:166-173)
__global__ void resid_norm_finish_kernel(float *__restrict__ hidden, bf16 *__restrict__ lp,
                                         const float *__restrict__ part, long ld, long rows,
                                         int d_model, float inv_d, float eps) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * d_model) return;
  const long r = i / d_model, n = i % d_model;
  // same formula as dec_out_finish / the out_proj epilogue: only the all-reduce
  // order separates a head-sharded row from an unsharded one
  const float sc = 1.f / sqrtf(part[r * ld + d_model] * inv_d + eps);
  const float v = hidden[i] + sc * part[r * ld + n];
  hidden[i] = v;
  lp[i] = __float2bfloat16_rn(v);
}

// partial != nullptr: head-group-sharded mode (no residual update; writes
// partial[r, :d_model] = u_local . W_out'_local and partial[r, d_model] = sum u_local^2)
int prefill_layer_bf16(const ssd200_dims_t *d, const ssd200_layer_t *w, float *hidden,
                       bf16 *hidden_lp, float *ssm_out, float *conv_out, int B, int Tn, void *ws,
                       size_t ws_bytes, cudaStream_t st, float *partial = nullptr,
                       long partial_ld = 0) {
  REQUIRE(hidden_lp, SSD200_EINVAL, "bf16 mode needs the hidden_lp shadow");
  REQUIRE(!partial || tc_ssd_eligible(d), SSD200_EUNSUPPORTED,
          "head-sharded prefill needs the tensor-core scan (P=64, N=128, L=256, G=1, local heads "
          "a multiple of 8)");
  PrefillWs<float> o;
  size_t need = 0;
  REQUIRE(carve_prefill<float>(d, B, Tn, ws, ws_bytes, o, &need), SSD200_EWORKSPACE,
          "prefill workspace %zu < %zu", ws_bytes, need);
  Widths wd = widths(d);
  const long rows = (long)B * Tn;
  const long n_split = d->d_inner + wd.conv_dim;
  bf16 *u = static_cast<bf16 *>(o.u);
  bf16 *act = static_cast<bf16 *>(o.act);
  const int k = d->conv_kernel;
  // in_proj on tensor cores, dt epilogue fused
  TcEpilogue ep{};
  ep.C = u;
  ep.ldc = n_split;
  ep.n_split = (int)n_split;
  ep.dt = o.dt;
  ep.H = d->n_heads;
  ep.dt_bias = static_cast<const float *>(w->dt_bias);
  ep.dt_lo = (float)d->dt_min;
  ep.dt_hi = (float)d->dt_max;
  REQUIRE(!(partial && w->pre_norm_w), SSD200_EUNSUPPORTED,
          "head-sharded prefill has no residual pre-norm");
  phase_mark(PH_IN_PROJ, 0, st);
  const bf16 *xin = hidden_lp;
  if (w->pre_norm_w) {  // optional residual pre-norm: in_proj reads rmsnorm(hidden) * w (bf16)
    rmsnorm_rows<float, bf16><<<(unsigned)rows, 256, 0, st>>>(
        hidden, d->d_model, static_cast<const float *>(w->pre_norm_w), static_cast<bf16 *>(o.xn),
        d->d_model, d->d_model, (float)d->norm_eps);
    LAUNCH_CHECK("pre_norm");
    xin = static_cast<const bf16 *>(o.xn);
  }
  int rc = tc_gemm<TC_EPI_INPROJ>(xin, d->d_model, static_cast<const bf16 *>(w->W_in),
                                  d->d_model, (int)rows, (int)wd.d_in_proj, d->d_model, ep, st);
  if (rc) return rc;
  phase_mark(PH_IN_PROJ, 1, st);
  phase_mark(PH_CONV, 0, st);
  {
    if (k > 1) {
      REQUIRE(launch_pf(conv_tail_kernel<float, bf16>,
                         dim3(blocks_for((long)B * wd.conv_dim * (k - 1))), dim3(256), 0, st,
                         (const bf16 *)(u + d->d_inner), (long)n_split, conv_out, B, Tn,
                         (int)wd.conv_dim, k) == cudaSuccess,
              SSD200_ELAUNCH, "conv_tail launch");
      LAUNCH_CHECK("conv_tail");
    }
    if (k == 4 && n_split % 8 == 0 && d->d_inner % 8 == 0 && wd.conv_dim % 4 == 0) {
      // TMA-tiled streaming conv (ssd_tc.cuh)
      CUtensorMap tmx;
      rc = make_map_2d_plain(&tmx, u + d->d_inner, rows, wd.conv_dim, n_split, CONV_COLS,
                             CONV_ROWS + 3);
      if (rc) return rc;
      REQUIRE(launch_pf(conv_silu_tma,
                         dim3(blocks_for(wd.conv_dim, CONV_COLS), blocks_for(rows, CONV_ROWS)),
                         dim3(256), 0, st, tmx, static_cast<const float *>(w->conv_w),
                         static_cast<const float *>(w->conv_b), act, (long)wd.conv_dim, Tn,
                         (int)wd.conv_dim, rows) == cudaSuccess,
              SSD200_ELAUNCH, "conv_silu_tma launch");
      LAUNCH_CHECK("conv_silu_tma");
    } else {
      launch_conv<float, bf16, bf16>(u + d->d_inner, n_split,
                                     static_cast<const float *>(w->conv_w),
                                     static_cast<const float *>(w->conv_b), act, wd.conv_dim, Tn,
                                     (int)wd.conv_dim, k, rows, st);
      LAUNCH_CHECK("conv_silu_prefill");
    }
  }
  phase_mark(PH_CONV, 1, st);
  if (tc_ssd_eligible(d)) {
    // tensor-core scan with the D skip + gate fused; the norm's row scale is
    // applied by the out_proj epilogue (norm_w folded into W_out).
    bf16 *u_gated = reinterpret_cast<bf16 *>(o.y);
    float *ssq = reinterpret_cast<float *>(reinterpret_cast<char *>(o.y) +
                                           align_up((size_t)rows * d->d_inner * 2));
    int ng = 1;
    rc = run_tc_scan(d, w, act, wd.conv_dim, u, n_split, o.dt, ssm_out, u_gated, ssq, &ng, o.scan,
                     B, Tn, st);  // marks PH_SCAN and PH_GATE
    if (rc) return rc;
    TcEpilogue er{};
    phase_mark(PH_OUT_PROJ, 0, st);
    if (partial) {  // this rank's share: unscaled partial + local sum u^2
      ssq_groups_kernel<<<blocks_for(rows), 256, 0, st>>>(ssq, ng, rows, partial, partial_ld,
                                                          d->d_model);
      LAUNCH_CHECK("ssq_groups");
      er.C = partial;
      er.ldc = partial_ld;
      rc = tc_gemm<TC_EPI_F32>(u_gated, d->d_inner, static_cast<const bf16 *>(w->W_out),
                               d->d_inner, (int)rows, d->d_model, d->d_inner, er, st);
      phase_mark(PH_OUT_PROJ, 1, st);
      return rc;
    }
    er.C = hidden;
    er.ldc = d->d_model;
    er.C_lp = hidden_lp;
    er.ssq = ssq;
    er.ng = ng;
    er.ssq_ld = rows;
    er.inv_d = 1.f / (float)d->d_inner;
    er.eps = (float)d->norm_eps;
    rc = tc_gemm<TC_EPI_RESID_NORM>(u_gated, d->d_inner, static_cast<const bf16 *>(w->W_out),
                                    d->d_inner, (int)rows, d->d_model, d->d_inner, er, st);
    phase_mark(PH_OUT_PROJ, 1, st);
    return rc;
  }
  SsdArgs<float, bf16> sa{};
  sa.X = act;
  sa.x_ts = wd.conv_dim;
  sa.dt = o.dt;
  sa.dt_ts = d->n_heads;
  sa.a = static_cast<const float *>(w->a);
  sa.Bm = act + d->d_inner;
  sa.Cm = act + d->d_inner + wd.gn;
  sa.bc_ts = wd.conv_dim;
  sa.D = static_cast<const float *>(w->D);
  sa.init = nullptr;
  sa.Y = o.y;
  sa.y_ts = d->d_inner;
  sa.final_state = ssm_out;
  sa.B = B;
  sa.T_ = Tn;
  sa.H = d->n_heads;
  sa.P = d->head_dim;
  sa.G = d->n_groups;
  sa.N = d->d_state;
  sa.L = d->chunk_size;
  phase_mark(PH_SCAN, 0, st);
  rc = run_scan<float, bf16>(sa, o.scan, o.scan_bytes, st);
  if (rc) return rc;
  phase_mark(PH_SCAN, 1, st);
  phase_mark(PH_GATE, 0, st);
  bf16 *normed = act;  // act is dead after the scan
  gated_norm_kernel<float, bf16, bf16><<<(unsigned)rows, 256, 0, st>>>(
      o.y, d->d_inner, u, n_split, nullptr /* norm_w folded into W_out */, normed, d->d_inner,
      d->d_inner, (float)d->norm_eps);
  LAUNCH_CHECK("gated_norm");
  phase_mark(PH_GATE, 1, st);
  TcEpilogue er{};
  er.C = hidden;
  er.ldc = d->d_model;
  er.C_lp = hidden_lp;
  phase_mark(PH_OUT_PROJ, 0, st);
  rc = tc_gemm<TC_EPI_RESID>(normed, d->d_inner, static_cast<const bf16 *>(w->W_out), d->d_inner,
                             (int)rows, d->d_model, d->d_inner, er, st);
  phase_mark(PH_OUT_PROJ, 1, st);
  return rc;
}

// ------------------------------------------------------------- decode layer
template <typename T> struct DecodeWs {
  void *xn;          // pre-norm only: (B, d_model) T (bf16 in bf16 mode)
  T *u, *act, *y, *normed_T;
  bf16 *normed_lp;
  float *part;       // wide-batch bf16: out_proj split-K partials
  float *ssq;        // wide-batch bf16: (B, H) sum u^2
  unsigned *ctr;     // wide-batch bf16: the state stream's chunk counter
};

// split-K factors of the bf16 decode GEMMs: enough
// (row tile x column tile x K range) work units to cover the SMs, >= 4 K blocks
// of 64 per range.  The weights are read once either way; only the f32
// partials (a few MB) are extra traffic.
struct DecSplits {
  int in, out;
};
inline DecSplits dec_splits(const ssd200_dims_t *d, int B) {
  Widths w = widths(d);
  auto pick = [](long tiles, int K) {
    const long kb = (K + 63) / 64;
    long s = (long)num_sms() / (tiles > 0 ? tiles : 1);
    if (s > kb / 4) s = kb / 4;
    return (int)(s < 1 ? 1 : s);
  };
  const long mt = B <= 256 ? 1 : (B + 127) / 128;  // dec_gemm_swap: one tile covers the batch
  DecSplits r;
  r.in = pick(mt * ((w.d_in_proj + 127) / 128), d->d_model);
  const bool small = tune().dec_small_ring < 0 ? B <= tune().dec_small_max : tune().dec_small_ring != 0;
  if (small && B <= 256) {  // two CTAs per SM: twice the units
    const int s2 = 2 * ((int)num_sms() / (int)((w.d_in_proj + 127) / 128));
    int cap = (d->d_model + 63) / 64 / 4;
    if (cap < 1) cap = 1;
    r.in = s2 < 1 ? 1 : (s2 > cap ? cap : s2);
  }
  r.out = pick(mt * ((d->d_model + 127) / 128), d->d_inner);
  const int si = tune().dec_split_in, so = tune().dec_split_out;
  if (si > 0 && si <= (d->d_model + 63) / 64) r.in = si;
  if (so > 0 && so <= (d->d_inner + 63) / 64) r.out = so;
  return r;
}

inline bool dec_big_eligible(const ssd200_dims_t *d) {
  return (d->head_dim == 16 || d->head_dim == 32 || d->head_dim == 64) &&
         d->d_state % 4 == 0 &&
         d->d_state <= 256 && d->n_heads % d->n_groups == 0 && d->d_inner % 4 == 0 &&
         d->n_heads % 4 == 0 && d->conv_kernel == 4 &&
         DssLayout(d->head_dim, d->d_state, 16).total * 2 <= 200u * 1024u;
}

template <typename T>
bool carve_decode(const ssd200_dims_t *d, int B, void *ws, size_t cap, DecodeWs<T> &o,
                  size_t *need, bool force_big = false) {
  Widths w = widths(d);
  Carve cv(ws, cap);
  const bool big = std::is_same<T, float>::value && d->dtype == SSD200_BF16 &&
                   dec_big_eligible(d);
  const DecSplits sp = big ? dec_splits(d, B) : DecSplits{1, 1};
  o.xn = cv.take<T>((size_t)B * d->d_model);
  o.u = cv.take<T>((size_t)sp.in * B * w.d_in_proj);
  o.part = big ? cv.take<float>((size_t)sp.out * B * d->d_model) : nullptr;
  o.ssq = big ? cv.take<float>((size_t)B * d->n_heads) : nullptr;
  o.ctr = big ? cv.take<unsigned>(4) : nullptr;
  o.act = cv.take<T>((size_t)B * w.conv_dim);
  o.y = cv.take<T>((size_t)B * d->d_inner);
  o.normed_T = cv.take<T>((size_t)B * d->d_inner);
  o.normed_lp = cv.take<bf16>((size_t)B * d->d_inner);
  if (need) *need = cv.used;
  return cv.ok();
}

constexpr int GEMV_MAX_ROWS = 16;
// bf16: beyond the streaming-GEMV batch sizes the tensor-core GEMM wins (measured
// at B = 16: SIMT gemv_nk 315 us vs tc_gemm ~80 us for the 1.3B in_proj)
constexpr int GEMV_BF16_MAX_ROWS = 8;

// part[s, b, n] = sum_{k in range s} W[n, k] X[b, k] for decode batches: the
// weight-streaming swapped-operand GEMM (decode_gemm.cuh) for B <= 256, else tc_gemm
template <int BNB, bool SMALL>
int launch_dec_gemm_cfg(const bf16 *W, int N, int K, const bf16 *X, int B, float *out, long ldo,
                        int ksplit, long split_stride, cudaStream_t st, unsigned *zero_ctr) {
  using Cfg = DgCfg<BNB, SMALL>;
  CUtensorMap tw, tx;
  int rc = make_map_2d(&tw, W, N, K, K, 128);
  if (rc) return rc;
  rc = make_map_2d(&tx, X, B, K, K, BNB);
  if (rc) return rc;
  smem_attr(dec_gemm_swap<BNB, SMALL>, (int)Cfg::SMEM);
  DgArgs a{N, K, B, ksplit, out, ldo, split_stride, zero_ctr, trace_slot("dec_gemm")};
  const int grid = ((N + 127) / 128) * ksplit;
  cudaError_t e =
      launch_pdl(dec_gemm_swap<BNB, SMALL>, dim3(grid), dim3(192), Cfg::SMEM, st, tw, tx, a);
  REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "dec_gemm_swap: %s", cudaGetErrorString(e));
  LAUNCH_CHECK("dec_gemm_swap");
  return SSD200_OK;
}
template <int BNB>
int launch_dec_gemm_bnb(const bf16 *W, int N, int K, const bf16 *X, int B, float *out, long ldo,
                        int ksplit, long split_stride, cudaStream_t st, unsigned *zero_ctr) {
  // the small ring (two CTAs per SM) measured faster up to B = 32 (B = 1: 1.18 -> 1.06 ms
  // with the in_proj split 4), slower from B = 64 (3.37 vs 3.47 ms) and at B = 256
  const bool small = tune().dec_small_ring < 0 ? B <= tune().dec_small_max : tune().dec_small_ring != 0;
  return small
             ? launch_dec_gemm_cfg<BNB, true>(W, N, K, X, B, out, ldo, ksplit, split_stride, st,
                                              zero_ctr)
             : launch_dec_gemm_cfg<BNB, false>(W, N, K, X, B, out, ldo, ksplit, split_stride, st,
                                               zero_ctr);
}

int dec_gemm(const bf16 *W, int N, int K, const bf16 *X, int B, float *out, long ldo, int ksplit,
             long split_stride, cudaStream_t st, unsigned *zero_ctr = nullptr) {
  REQUIRE(ksplit >= 1 && ksplit <= (K + 63) / 64, SSD200_EINVAL, "dec_gemm: bad split");
  if (B <= 256 && tune().dec_swap) {
    if (B <= 16) return launch_dec_gemm_bnb<16>(W, N, K, X, B, out, ldo, ksplit, split_stride, st, zero_ctr);
    if (B <= 32) return launch_dec_gemm_bnb<32>(W, N, K, X, B, out, ldo, ksplit, split_stride, st, zero_ctr);
    if (B <= 64) return launch_dec_gemm_bnb<64>(W, N, K, X, B, out, ldo, ksplit, split_stride, st, zero_ctr);
    if (B <= 128)
      return launch_dec_gemm_bnb<128>(W, N, K, X, B, out, ldo, ksplit, split_stride, st, zero_ctr);
    return launch_dec_gemm_bnb<256>(W, N, K, X, B, out, ldo, ksplit, split_stride, st, zero_ctr);
  }
  TcEpilogue ep{};
  ep.C = out;
  ep.ldc = ldo;
  ep.ksplit = ksplit;
  ep.split_stride = split_stride;
  return tc_gemm<TC_EPI_F32>(X, K, W, K, B, N, K, ep, st, true);
}

// bf16 decode layer, 4 PDL-chained launches:
//   tc_gemm F32 split-K in_proj -> dec_ssm_stream (TMA-pipelined conv + state
//   update + gate + sum u^2) -> tc_gemm F32 split-K out_proj -> dec_out_finish
//   (norm row scale + residual, B / C conv windows rolled).
// Split-K keeps every SM streaming weights at B = 16..128, where the
// (row tile x column tile) grid alone covers a fraction of the SMs.
// pout != nullptr: head-group-sharded mode: hidden is not
// updated; pout[b, :d_model] = the local out_proj partial, pout[b, d_model] =
// the local sum of u^2, for the caller's all-reduce + ssd200_resid_norm_finish.
int decode_layer_big(const ssd200_dims_t *d, const ssd200_layer_t *w, float *hidden,
                     bf16 *hidden_lp, const float *ssm_in, float *ssm_out, const float *conv_in,
                     float *conv_out, int B, DecodeWs<float> &o, cudaStream_t st,
                     float *pout = nullptr, long pld = 0) {
  Widths wd = widths(d);
  const DecSplits sp = dec_splits(d, B);
  const long s_in = (long)B * wd.d_in_proj, s_out = (long)B * d->d_model;
  {
    const bf16 *xin = hidden_lp;
    if (w->pre_norm_w) {  // optional residual pre-norm
      REQUIRE(hidden, SSD200_EUNSUPPORTED, "head-sharded decode has no residual pre-norm");
      rmsnorm_rows<float, bf16><<<B, 256, 0, st>>>(hidden, d->d_model,
                                                   static_cast<const float *>(w->pre_norm_w),
                                                   static_cast<bf16 *>(o.xn), d->d_model,
                                                   d->d_model, (float)d->norm_eps);
      LAUNCH_CHECK("pre_norm");
      xin = static_cast<const bf16 *>(o.xn);
    }
    // the in_proj zeroes the state stream's chunk counter after its own dependency
    // wait (every earlier grab of it is then complete)
    int rc = dec_gemm(static_cast<const bf16 *>(w->W_in), (int)wd.d_in_proj, d->d_model, xin,
                      B, o.u, wd.d_in_proj, sp.in, s_in, st, o.ctr);
    if (rc) return rc;
  }
  DecStreamArgs sa{};
  sa.B = B;
  sa.H = d->n_heads;
  sa.P = d->head_dim;
  sa.G = d->n_groups;
  sa.N = d->d_state;
  sa.d_inner = d->d_inner;
  sa.conv_dim = (int)wd.conv_dim;
  sa.proj = o.u;
  sa.ldp = wd.d_in_proj;
  sa.sstride = s_in;
  sa.nsplit = sp.in;
  sa.conv_in = conv_in;
  sa.conv_out = conv_out;
  sa.conv_w = static_cast<const float *>(w->conv_w);
  sa.conv_b = static_cast<const float *>(w->conv_b);
  sa.dt_bias = static_cast<const float *>(w->dt_bias);
  sa.a = static_cast<const float *>(w->a);
  sa.D = static_cast<const float *>(w->D);
  sa.dt_lo = (float)d->dt_min;
  sa.dt_hi = (float)d->dt_max;
  sa.ssm_in = ssm_in;
  sa.ssm_out = ssm_out;
  sa.u = o.normed_lp;
  sa.ssq = o.ssq;
  // one tile per CTA (static split) -> state in registers (see DecStreamArgs::reg_state);
  // measured at 1.3B: B = 1 0.964 -> 0.945 ms, B = 2 (128 CTAs) 0.994 -> 1.001 ms, hence
  // only while the tiles fill at most half of the SMs
  const bool reg_state = tune().stream_reg_state && tune().stream_chunk <= 0 &&
                         2 * B * d->n_heads <= num_sms();
  sa.reg_state = reg_state ? 1 : 0;
  const DssLayout lay(d->head_dim, d->d_state, sp.in, !reg_state);
  sa.stage_bytes = lay.total;
  sa.trace = trace_slot("dec_ssm_stream");
  sa.trace2 = trace_slot("  stream phases");
  // CTAs per SM: two independent pipelines per SM (measured at 1.3B with the
  // small-ring decode GEMMs: B = 8 1.42 -> 1.29, B = 64 3.97 -> 3.51, B = 256
  // 12.1 -> 10.9 ms/step; neutral at B = 1, where there are fewer tiles than SMs)
  const int ntiles_all = B * d->n_heads;
  const int cps = tune().stream_cps == 1 ? 1
                  : tune().stream_cps == 2 ? 2
                  : (ntiles_all > num_sms() ? 2 : 1);  // B = 4 (256 tiles): 1.095 -> 1.018 ms
  const uint32_t par_bytes = dss_par_bytes(d->n_heads, d->n_groups, d->d_state);
  int stages = (int)((cps == 2 ? 105u * 1024u : 214u * 1024u) - par_bytes) / (int)lay.total;
  if (tune().stream_stages > 0 && tune().stream_stages < stages) stages = tune().stream_stages;
  REQUIRE(stages >= 2, SSD200_EUNSUPPORTED, "decode state tile too large for the smem ring");
  const int ntiles = B * d->n_heads;
  const int grid = ntiles < cps * num_sms() ? ntiles : cps * num_sms();
  // no more stages than a CTA has tiles: at small batches (one tile per CTA) the
  // ring then leaves the SM's shared memory to the out_proj CTAs that launch
  // early and stream W_out while this grid runs
  const int per_cta = (ntiles + grid - 1) / grid;
  if (stages > per_cta) stages = per_cta;
  sa.stages = stages > DSS_MAX_STAGES ? DSS_MAX_STAGES : stages;
  const size_t smem = (size_t)sa.stages * lay.total + par_bytes;
  cudaError_t e;
  // tile hand-out: static ranges, or (wide batches) chunks from a counter the
  // in_proj zeroes — only dec_gemm_swap does (B <= 256)
  const bool can_dyn = B <= 256 && tune().dec_swap;
  int chunk = 0;
  if (tune().stream_chunk > 0) chunk = tune().stream_chunk;
  else if (tune().stream_chunk == 0 && per_cta >= 4)  // 1.3B B = 256: 11.1 (static) -> 10.3 ms
    // chunks of 3 from 8 tiles per CTA (1.3B B = 64 3.29 -> 3.22 ms, 780M B = 128 4.27 -> 4.20
    // ms vs chunks of 1; B = 256 equal to 4)
    chunk = per_cta >= 8 ? 3 : 1;
  sa.chunk = can_dyn ? chunk : 0;
  sa.ctr = o.ctr;
  const int cw = tune().stream_cw == 16 ? 16 : 8;  // consumer warps
  const int nq = d->d_state <= 128 ? 1 : 2, rpw = d->head_dim / cw;
  e = cudaErrorInvalidValue;
#define DSS_CASE(NQ, RPW, CW)                                                                  \
  if (nq == NQ && rpw == RPW && cw == CW) {                                                    \
    smem_attr(dec_ssm_stream<NQ, RPW, CW>, 214 * 1024);                                        \
    e = launch_pdl(dec_ssm_stream<NQ, RPW, CW>, dim3(grid), dim3(CW * 32 + 32), smem, st, sa); \
  }
    DSS_CASE(1, 1, 8) DSS_CASE(1, 2, 8) DSS_CASE(1, 4, 8) DSS_CASE(1, 8, 8)
    DSS_CASE(2, 1, 8) DSS_CASE(2, 2, 8) DSS_CASE(2, 4, 8) DSS_CASE(2, 8, 8)
    DSS_CASE(1, 1, 16) DSS_CASE(1, 2, 16) DSS_CASE(1, 4, 16)
    DSS_CASE(2, 1, 16) DSS_CASE(2, 2, 16) DSS_CASE(2, 4, 16)
#undef DSS_CASE
  REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "dec_ssm_stream: %s", cudaGetErrorString(e));
  LAUNCH_CHECK("dec_ssm_stream");

  int rc = dec_gemm(static_cast<const bf16 *>(w->W_out), d->d_model, d->d_inner, o.normed_lp, B,
                    o.part, d->d_model, sp.out, s_out, st);
  if (rc) return rc;
  DecFinishArgs fa{};
  fa.part = o.part;
  fa.nsplit = sp.out;
  fa.sstride = s_out;
  fa.ssq = o.ssq;
  fa.H = d->n_heads;
  fa.inv_d = 1.f / (float)d->d_inner;
  fa.eps = (float)d->norm_eps;
  fa.hidden_in = hidden;
  fa.hidden = hidden;
  fa.lp = hidden_lp;
  fa.d_model = d->d_model;
  fa.proj = o.u;
  fa.ldp = wd.d_in_proj;
  fa.psstride = s_in;
  fa.pnsplit = sp.in;
  fa.d_inner = d->d_inner;
  fa.conv_dim = (int)wd.conv_dim;
  fa.conv_in = conv_in;
  fa.conv_out = conv_out;
  fa.pout = pout;
  fa.pld = pld;
  const int gbx = (d->d_model + 255) / 256 + (int)((wd.conv_dim - d->d_inner + 255) / 256);
  fa.trace = trace_slot("dec_out_finish");
  e = launch_pdl(dec_out_finish, dim3(gbx, B), dim3(256), 0, st, fa);
  REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "dec_out_finish: %s", cudaGetErrorString(e));
  LAUNCH_CHECK("dec_out_finish");
  return SSD200_OK;
}

template <typename T>
int decode_layer_impl(const ssd200_dims_t *d, const ssd200_layer_t *w, T *hidden,
                      bf16 *hidden_lp, const T *ssm_in, T *ssm_out, const T *conv_in,
                      T *conv_out, int B, void *ws, size_t ws_bytes, cudaStream_t st) {
  DecodeWs<T> o;
  size_t need = 0;
  REQUIRE(carve_decode<T>(d, B, ws, ws_bytes, o, &need), SSD200_EWORKSPACE,
          "decode workspace %zu < %zu", ws_bytes, need);
  Widths wd = widths(d);
  const bool lp = d->dtype == SSD200_BF16;
  const int k = d->conv_kernel;
  if constexpr (std::is_same<T, float>::value) {
    if (lp && dec_big_eligible(d)) {
      REQUIRE(hidden_lp, SSD200_EINVAL, "bf16 mode needs the hidden_lp shadow");
      return decode_layer_big(d, w, hidden, hidden_lp, ssm_in, ssm_out, conv_in, conv_out, B, o,
                              st);
    }
  }
  // optional residual pre-norm: in_proj reads rmsnorm(hidden) * pre_norm_w
  const T *xin = hidden;
  const bf16 *xin_lp = hidden_lp;
  if (w->pre_norm_w) {
    if (lp) {
      rmsnorm_rows<T, bf16><<<B, 256, 0, st>>>(hidden, d->d_model,
                                              static_cast<const T *>(w->pre_norm_w),
                                              static_cast<bf16 *>(o.xn), d->d_model, d->d_model,
                                              (T)d->norm_eps);
      xin_lp = static_cast<const bf16 *>(o.xn);
    } else {
      rmsnorm_rows<T, T><<<B, 256, 0, st>>>(hidden, d->d_model,
                                           static_cast<const T *>(w->pre_norm_w),
                                           static_cast<T *>(o.xn), d->d_model, d->d_model,
                                           (T)d->norm_eps);
      xin = static_cast<const T *>(o.xn);
    }
    LAUNCH_CHECK("pre_norm");
  }
  // in_proj
  if (lp) {
    REQUIRE(hidden_lp, SSD200_EINVAL, "bf16 mode needs the hidden_lp shadow");
    const bf16 *Win = static_cast<const bf16 *>(w->W_in);
    if (B <= GEMV_BF16_MAX_ROWS) {
      gemv_nk<float, bf16, bf16, EPI_STORE>
          <<<dim3(blocks_for(wd.d_in_proj, 32), blocks_for(B, 4)), 256, 0, st>>>(
              xin_lp, d->d_model, Win, d->d_model, (float *)o.u, wd.d_in_proj, nullptr, B,
              (int)wd.d_in_proj, d->d_model);
      LAUNCH_CHECK("gemv_nk in_proj");
    } else {
      TcEpilogue ep{};
      ep.C = o.u;
      ep.ldc = wd.d_in_proj;
      int rc = tc_gemm<TC_EPI_F32>(xin_lp, d->d_model, Win, d->d_model, B, (int)wd.d_in_proj,
                                   d->d_model, ep, st);
      if (rc) return rc;
    }
  } else {
    const T *Win = static_cast<const T *>(w->W_in);
    if (B <= GEMV_MAX_ROWS) {
      gemv_kn<T, EPI_STORE><<<dim3(blocks_for(wd.d_in_proj, 32), blocks_for(B, 8)), dim3(32, 8),
                              0, st>>>(xin, d->d_model, Win, wd.d_in_proj, o.u, wd.d_in_proj,
                                       B, (int)wd.d_in_proj, d->d_model);
    } else {
      gemm_simt<T, false, EPI_STORE><<<dim3(blocks_for(wd.d_in_proj, 64), blocks_for(B, 64)),
                                       256, 0, st>>>(xin, d->d_model, Win, wd.d_in_proj, o.u,
                                                     wd.d_in_proj, B, (int)wd.d_in_proj,
                                                     d->d_model);
    }
    LAUNCH_CHECK("in_proj (decode)");
  }
  // conv window roll + readout
  REQUIRE(k >= 1 && k <= 16, SSD200_EUNSUPPORTED, "conv_kernel");

  decode_conv<T, T><<<blocks_for((long)B * wd.conv_dim), 256, 0, st>>>(
      o.u, wd.d_in_proj, d->d_inner, conv_in, conv_out, static_cast<const T *>(w->conv_w),
      static_cast<const T *>(w->conv_b), o.act, B, (int)wd.conv_dim, k);
  LAUNCH_CHECK("decode_conv");
  // state update + readout + D skip
  decode_ssm<T, T><<<dim3(d->n_heads, B), 128, 2 * d->d_state * sizeof(T), st>>>(
      o.u, wd.d_in_proj, (int)(d->d_inner + wd.conv_dim), o.act, d->d_inner,
      static_cast<const T *>(w->dt_bias), static_cast<const T *>(w->a),
      static_cast<const T *>(w->D), ssm_in, ssm_out, o.y, d->d_inner, d->n_heads, d->head_dim,
      d->n_groups, d->d_state, (T)d->dt_min, (T)d->dt_max);
  LAUNCH_CHECK("decode_ssm");
  // gated norm + out_proj + residual
  if (lp) {
    gated_norm_kernel<float, float, bf16><<<B, 256, 0, st>>>(
        (const float *)o.y, d->d_inner, (const float *)o.u, wd.d_in_proj,
        nullptr /* norm_w folded into W_out */, o.normed_lp, d->d_inner, d->d_inner,
        (float)d->norm_eps);
    LAUNCH_CHECK("gated_norm (decode)");
    const bf16 *Wout = static_cast<const bf16 *>(w->W_out);
    if (B <= GEMV_BF16_MAX_ROWS) {
      gemv_nk<float, bf16, bf16, EPI_ADD>
          <<<dim3(blocks_for(d->d_model, 32), blocks_for(B, 4)), 256, 0, st>>>(
              o.normed_lp, d->d_inner, Wout, d->d_inner, (float *)hidden, d->d_model, hidden_lp,
              B, d->d_model, d->d_inner);
      LAUNCH_CHECK("gemv_nk out_proj");
    } else {
      TcEpilogue er{};
      er.C = hidden;
      er.ldc = d->d_model;
      er.C_lp = hidden_lp;
      int rc = tc_gemm<TC_EPI_RESID>(o.normed_lp, d->d_inner, Wout, d->d_inner, B, d->d_model,
                                     d->d_inner, er, st);
      if (rc) return rc;
    }
  } else {
    gated_norm_kernel<T, T, T><<<B, 256, 0, st>>>(o.y, d->d_inner, o.u, wd.d_in_proj,
                                                  static_cast<const T *>(w->norm_w), o.normed_T,
                                                  d->d_inner, d->d_inner, (T)d->norm_eps);
    LAUNCH_CHECK("gated_norm (decode)");
    const T *Wout = static_cast<const T *>(w->W_out);
    if (B <= GEMV_MAX_ROWS) {
      gemv_kn<T, EPI_ADD><<<dim3(blocks_for(d->d_model, 32), blocks_for(B, 8)), dim3(32, 8), 0,
                            st>>>(o.normed_T, d->d_inner, Wout, d->d_model, hidden, d->d_model,
                                  B, d->d_model, d->d_inner);
    } else {
      gemm_simt<T, false, EPI_ADD><<<dim3(blocks_for(d->d_model, 64), blocks_for(B, 64)), 256, 0,
                                     st>>>(o.normed_T, d->d_inner, Wout, d->d_model, hidden,
                                           d->d_model, B, d->d_model, d->d_inner);
    }
    LAUNCH_CHECK("out_proj (decode)");
  }
  return SSD200_OK;
}

// ------------------------------------------------------------------- head
template <typename T>
int head_simt(const ssd200_dims_t *d, int V, const T *hidden, long hrs, const T *fw, const T *E,
              T *logits, int64_t *amax, int rows, void *ws, size_t ws_bytes, cudaStream_t st) {
  Carve cv(ws, ws_bytes);
  T *normed = cv.take<T>((size_t)rows * d->d_model);
  T *lg = logits ? logits : cv.take<T>((size_t)rows * V);
  REQUIRE(cv.ok(), SSD200_EWORKSPACE, "head workspace %zu < %zu", ws_bytes, cv.used);
  rmsnorm_rows<T, T><<<rows, 256, 0, st>>>(hidden, hrs, fw, normed, d->d_model, d->d_model,
                                           (T)d->norm_eps);
  LAUNCH_CHECK("rmsnorm_rows");
  if (rows <= GEMV_MAX_ROWS) {
    gemv_nk<T, T, T, EPI_STORE><<<dim3(blocks_for(V, 32), blocks_for(rows, 4)), 256, 0, st>>>(
        normed, d->d_model, E, d->d_model, lg, V, nullptr, rows, V, d->d_model);
  } else {
    gemm_simt<T, true, EPI_STORE><<<dim3(blocks_for(V, 64), blocks_for(rows, 64)), 256, 0, st>>>(
        normed, d->d_model, E, d->d_model, lg, V, rows, V, d->d_model);
  }
  LAUNCH_CHECK("head gemm");
  if (amax) {
    argmax_rows<T><<<rows, 256, 0, st>>>(lg, V, V, amax);
    LAUNCH_CHECK("argmax_rows");
  }
  return SSD200_OK;
}

int head_bf16(const ssd200_dims_t *d, int V, const float *hidden, long hrs, const float *fw,
              const bf16 *E, float *logits, int64_t *amax, int rows, void *ws, size_t ws_bytes,
              cudaStream_t st) {
  Carve cv(ws, ws_bytes);
  bf16 *normed = cv.take<bf16>((size_t)rows * d->d_model);
  float *lg = logits ? logits : cv.take<float>((size_t)rows * V);
  constexpr int AM_CHUNK = 2048;
  const int nparts = (V + AM_CHUNK - 1) / AM_CHUNK;
  float *pv = cv.take<float>((size_t)rows * nparts);
  int *pi = cv.take<int>((size_t)rows * nparts);
  REQUIRE(cv.ok(), SSD200_EWORKSPACE, "head workspace %zu < %zu", ws_bytes, cv.used);
  {  // PDL: the norm's launch overlaps the last layer's finish (it waits for it)
    cudaError_t e = launch_pdl(rmsnorm_rows<float, bf16>, dim3(rows), dim3(256), 0, st, hidden,
                               (long)hrs, fw, normed, (long)d->d_model, d->d_model,
                               (float)d->norm_eps);
    REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "rmsnorm_rows: %s", cudaGetErrorString(e));
  }
  LAUNCH_CHECK("rmsnorm_rows");
  if (rows <= 256 && tune().dec_swap && d->d_model % 8 == 0) {
    // decode batches: the embedding streamed once as the UMMA M side (decode_gemm.cuh)
    int rc = dec_gemm(E, V, d->d_model, normed, rows, lg, V, 1, 0, st);
    if (rc) return rc;
  } else if (rows <= GEMV_MAX_ROWS) {
    gemv_nk<float, bf16, bf16, EPI_STORE>
        <<<dim3(blocks_for(V, 32), blocks_for(rows, 4)), 256, 0, st>>>(
            normed, d->d_model, E, d->d_model, lg, V, nullptr, rows, V, d->d_model);
    LAUNCH_CHECK("head gemv");
  } else {
    TcEpilogue ep{};
    ep.C = lg;
    ep.ldc = V;
    int rc = tc_gemm<TC_EPI_F32>(normed, d->d_model, E, d->d_model, rows, V, d->d_model, ep, st);
    if (rc) return rc;
  }
  if (amax) {  // (chunk, row) partial maxima, then one warp per row
    cudaError_t e = launch_pdl(argmax_part, dim3(nparts, rows), dim3(256), 0, st,
                               (const float *)lg, (long)V, V, AM_CHUNK, pv, pi);
    REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "argmax_part: %s", cudaGetErrorString(e));
    LAUNCH_CHECK("argmax_part");
    e = launch_pdl(argmax_final, dim3(rows), dim3(32), 0, st, (const float *)pv,
                   (const int *)pi, nparts, amax);
    REQUIRE(e == cudaSuccess, SSD200_ELAUNCH, "argmax_final: %s", cudaGetErrorString(e));
    LAUNCH_CHECK("argmax_final");
  }
  return SSD200_OK;
}

}  // namespace

// =============================================================== C ABI
extern "C" {

int ssd200_abi_version(void) { return 4; }

void ssd200_tuning_defaults(ssd200_tuning_t *t) {
  if (t) *t = kDefaultTuning;
}

const char *ssd200_last_error(void) { return g_err.c_str(); }

size_t ssd200_chunk_scan_workspace(int dtype, int batch, int seqlen, int heads, int head_dim,
                                   int d_state, int chunk) {
  size_t elt = dtype == SSD200_F64 ? 8 : 4;
  if (batch < 1 || seqlen < 1 || chunk < 1) return 0;
  return scan_ws_bytes(elt, batch, seqlen, heads, head_dim, d_state, chunk);
}

int ssd200_chunk_scan(int dtype, const void *X, const void *dt, const void *a, const void *Bmat,
                      const void *Cmat, const void *D, const void *init_state, void *Y,
                      void *final_state, int batch, int seqlen, int heads, int head_dim,
                      int groups, int d_state, int chunk, void *workspace,
                      size_t workspace_bytes, ssd200_stream_t stream) {
  REQUIRE(X && dt && a && Bmat && Cmat && Y && final_state, SSD200_EINVAL, "null pointer");
  REQUIRE(batch >= 1 && seqlen >= 1 && heads >= 1 && head_dim >= 1 && groups >= 1 &&
              d_state >= 1 && chunk >= 1,
          SSD200_EINVAL, "need T >= 1 and L >= 1, got T=%d, L=%d", seqlen, chunk);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == SSD200_F32 || dtype == SSD200_F64) {
    auto fill = [&](auto tag) {
      using T = decltype(tag);
      SsdArgs<T, T> s{};
      s.X = static_cast<const T *>(X);
      s.x_ts = (long)heads * head_dim;
      s.dt = static_cast<const T *>(dt);
      s.dt_ts = heads;
      s.a = static_cast<const T *>(a);
      s.Bm = static_cast<const T *>(Bmat);
      s.Cm = static_cast<const T *>(Cmat);
      s.bc_ts = (long)groups * d_state;
      s.D = static_cast<const T *>(D);
      s.init = static_cast<const T *>(init_state);
      s.Y = static_cast<T *>(Y);
      s.y_ts = (long)heads * head_dim;
      s.final_state = static_cast<T *>(final_state);
      s.B = batch;
      s.T_ = seqlen;
      s.H = heads;
      s.P = head_dim;
      s.G = groups;
      s.N = d_state;
      s.L = chunk;
      return run_scan<T, T>(s, workspace, workspace_bytes, st);
    };
    return dtype == SSD200_F32 ? fill(float{}) : fill(double{});
  }
  set_err("ssd200_chunk_scan: dtype %d not supported (F32/F64)", dtype);
  return SSD200_EINVAL;
}

int ssd200_embed(const ssd200_dims_t *d, const int64_t *tokens, int rows, int vocab,
                 const void *embedding, void *hidden, void *hidden_lp, ssd200_stream_t stream) {
  int rc = check_dims(d);
  if (rc) return rc;
  REQUIRE(tokens && embedding && hidden && rows >= 1 && vocab >= 1, SSD200_EINVAL,
          "embed: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d->dtype == SSD200_F32)
    embed_kernel<float, float><<<rows, 256, 0, st>>>(tokens, (const float *)embedding, d->d_model,
                                                     vocab, (float *)hidden, nullptr);
  else if (d->dtype == SSD200_F64)
    embed_kernel<double, double><<<rows, 256, 0, st>>>(tokens, (const double *)embedding,
                                                       d->d_model, vocab, (double *)hidden, nullptr);
  else {
    REQUIRE(hidden_lp, SSD200_EINVAL, "bf16 mode needs hidden_lp");
    embed_kernel<float, bf16><<<rows, 256, 0, st>>>(tokens, (const bf16 *)embedding, d->d_model,
                                                    vocab, (float *)hidden, (bf16 *)hidden_lp);
  }
  LAUNCH_CHECK("embed_kernel");
  return SSD200_OK;
}

size_t ssd200_prefill_layer_workspace(const ssd200_dims_t *d, int batch, int seqlen) {
  TuneScope scope(d);
  if (check_dims(d) || batch < 1 || seqlen < 1) return 0;
  size_t need = 0;
  if (d->dtype == SSD200_F64) {
    PrefillWs<double> o;
    carve_prefill<double>(d, batch, seqlen, nullptr, 0, o, &need);
  } else {
    PrefillWs<float> o;
    carve_prefill<float>(d, batch, seqlen, nullptr, 0, o, &need);
  }
  return need;
}

int ssd200_prefill_layer(const ssd200_dims_t *d, const ssd200_layer_t *w, void *hidden,
                         void *hidden_lp, void *ssm_out, void *conv_out, int batch, int seqlen,
                         void *workspace, size_t workspace_bytes, ssd200_stream_t stream) {
  TuneScope scope(d);
  int rc = check_dims(d);
  if (rc) return rc;
  REQUIRE(w && hidden && ssm_out && batch >= 1 && seqlen >= 1, SSD200_EINVAL,
          "prefill_layer: bad arguments");
  REQUIRE(d->conv_kernel == 1 || conv_out, SSD200_EINVAL, "prefill_layer: conv_out is null");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (d->dtype) {
    case SSD200_F32:
      return prefill_layer_simt<float>(d, w, (float *)hidden, (float *)ssm_out, (float *)conv_out,
                                       batch, seqlen, workspace, workspace_bytes, st);
    case SSD200_F64:
      return prefill_layer_simt<double>(d, w, (double *)hidden, (double *)ssm_out,
                                        (double *)conv_out, batch, seqlen, workspace,
                                        workspace_bytes, st);
    default:
      return prefill_layer_bf16(d, w, (float *)hidden, (bf16 *)hidden_lp, (float *)ssm_out,
                                (float *)conv_out, batch, seqlen, workspace, workspace_bytes, st);
  }
}

int ssd200_prefill_layer_partial(const ssd200_dims_t *d, const ssd200_layer_t *w,
                                 const void *hidden_lp, float *partial, long partial_ld,
                                 void *ssm_out, void *conv_out, int batch, int seqlen,
                                 void *workspace, size_t workspace_bytes, ssd200_stream_t stream) {
  TuneScope scope(d);
  int rc = check_dims(d);
  if (rc) return rc;
  REQUIRE(d->dtype == SSD200_BF16, SSD200_EUNSUPPORTED, "prefill_layer_partial: bf16 mode only");
  REQUIRE(w && hidden_lp && partial && ssm_out && batch >= 1 && seqlen >= 1 &&
              partial_ld >= d->d_model + 1 && partial_ld % 4 == 0,
          SSD200_EINVAL, "prefill_layer_partial: bad arguments");
  REQUIRE(d->conv_kernel == 1 || conv_out, SSD200_EINVAL, "prefill_layer_partial: conv_out is null");
  return prefill_layer_bf16(d, w, nullptr, (bf16 *)const_cast<void *>(hidden_lp), (float *)ssm_out,
                            (float *)conv_out, batch, seqlen, workspace, workspace_bytes,
                            static_cast<cudaStream_t>(stream), partial, partial_ld);
}

int ssd200_resid_norm_finish(int d_model, int d_inner_full, double eps, void *hidden,
                             void *hidden_lp, const float *partial, long partial_ld, long rows,
                             ssd200_stream_t stream) {
  REQUIRE(hidden && hidden_lp && partial && rows >= 1 && d_model >= 1 && d_inner_full >= 1 &&
              partial_ld >= d_model + 1,
          SSD200_EINVAL, "resid_norm_finish: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  resid_norm_finish_kernel<<<blocks_for(rows * d_model), 256, 0, st>>>(
      (float *)hidden, (bf16 *)hidden_lp, partial, partial_ld, rows, d_model,
      1.f / (float)d_inner_full, (float)eps);
  LAUNCH_CHECK("resid_norm_finish");
  return SSD200_OK;
}

size_t ssd200_decode_layer_workspace(const ssd200_dims_t *d, int batch) {
  TuneScope scope(d);
  if (check_dims(d) || batch < 1) return 0;
  size_t need = 0;
  if (d->dtype == SSD200_F64) {
    DecodeWs<double> o;
    carve_decode<double>(d, batch, nullptr, 0, o, &need);
  } else {
    DecodeWs<float> o;  // the wide-batch carve is a superset (also covers the partial entry)
    carve_decode<float>(d, batch, nullptr, 0, o, &need, true);
  }
  return need;
}

int ssd200_decode_layer_partial(const ssd200_dims_t *d, const ssd200_layer_t *w,
                                const void *hidden_lp, float *partial, long partial_ld,
                                const void *ssm_in, void *ssm_out, const void *conv_in,
                                void *conv_out, int batch, void *workspace,
                                size_t workspace_bytes, ssd200_stream_t stream) {
  TuneScope scope(d);
  int rc = check_dims(d);
  if (rc) return rc;
  REQUIRE(d->dtype == SSD200_BF16 && dec_big_eligible(d), SSD200_EUNSUPPORTED,
          "head-sharded decode needs bf16, conv_kernel 4, head_dim 16/32/64, local heads a "
          "multiple of 4");
  REQUIRE(batch >= 1 && batch <= 256, SSD200_EINVAL, "batch must be in [1, 256]");
  REQUIRE(hidden_lp && partial && ssm_in && ssm_out && conv_in && conv_out, SSD200_EINVAL,
          "null pointer");
  REQUIRE(partial_ld >= d->d_model + 1 && partial_ld % 4 == 0, SSD200_EINVAL,
          "partial_ld must be a multiple of 4 and >= d_model + 1");
  DecodeWs<float> o;
  size_t need = 0;
  REQUIRE(carve_decode<float>(d, batch, workspace, workspace_bytes, o, &need, true),
          SSD200_EWORKSPACE, "decode workspace %zu < %zu", workspace_bytes, need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return decode_layer_big(d, w, nullptr, (bf16 *)hidden_lp, (const float *)ssm_in,
                          (float *)ssm_out, (const float *)conv_in, (float *)conv_out, batch, o,
                          st, partial, partial_ld);
}

int ssd200_decode_layer(const ssd200_dims_t *d, const ssd200_layer_t *w, void *hidden,
                        void *hidden_lp, const void *ssm_in, void *ssm_out, const void *conv_in,
                        void *conv_out, int batch, void *workspace, size_t workspace_bytes,
                        ssd200_stream_t stream) {
  TuneScope scope(d);
  int rc = check_dims(d);
  if (rc) return rc;
  REQUIRE(w && hidden && ssm_in && ssm_out && batch >= 1, SSD200_EINVAL,
          "decode_layer: bad arguments");
  REQUIRE(d->conv_kernel == 1 || (conv_in && conv_out), SSD200_EINVAL,
          "decode_layer: conv state is null");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d->dtype == SSD200_F64)
    return decode_layer_impl<double>(d, w, (double *)hidden, nullptr, (const double *)ssm_in,
                                     (double *)ssm_out, (const double *)conv_in,
                                     (double *)conv_out, batch, workspace, workspace_bytes, st);
  return decode_layer_impl<float>(d, w, (float *)hidden, (bf16 *)hidden_lp,
                                  (const float *)ssm_in, (float *)ssm_out,
                                  (const float *)conv_in, (float *)conv_out, batch, workspace,
                                  workspace_bytes, st);
}

size_t ssd200_decode_layers_workspace(const ssd200_dims_t *d, int batch) {
  return ssd200_decode_layer_workspace(d, batch);
}

int ssd200_decode_layers(const ssd200_dims_t *d, const ssd200_layer_t *layers, int n_layers,
                         void *hidden, void *hidden_lp, const void *ssm_in, void *ssm_out,
                         const void *conv_in, void *conv_out, int batch, void *workspace,
                         size_t workspace_bytes, ssd200_stream_t stream) {
  TuneScope scope(d);
  int rc = check_dims(d);
  if (rc) return rc;
  REQUIRE(layers && n_layers >= 1 && hidden && ssm_in && ssm_out && batch >= 1, SSD200_EINVAL,
          "decode_layers: bad arguments");
  REQUIRE(d->conv_kernel == 1 || (conv_in && conv_out), SSD200_EINVAL,
          "decode_layers: conv state is null");
  const Widths wd = widths(d);
  const size_t esz = d->dtype == SSD200_F64 ? 8 : 4;
  const size_t ss = (size_t)batch * d->n_heads * d->head_dim * d->d_state * esz;
  const size_t cs = (size_t)batch * wd.conv_dim * (d->conv_kernel - 1) * esz;
  const char *si = static_cast<const char *>(ssm_in), *ci = static_cast<const char *>(conv_in);
  char *so = static_cast<char *>(ssm_out), *co = static_cast<char *>(conv_out);
  for (int i = 0; i < n_layers; ++i) {
    rc = ssd200_decode_layer(d, &layers[i], hidden, hidden_lp, si + i * ss, so + i * ss,
                             ci ? ci + i * cs : nullptr, co ? co + i * cs : nullptr, batch,
                             workspace, workspace_bytes, stream);
    if (rc) return rc;
  }
  return SSD200_OK;
}

size_t ssd200_head_workspace(const ssd200_dims_t *d, int vocab, int rows) {
  TuneScope scope(d);
  if (check_dims(d) || rows < 1 || vocab < 1) return 0;
  size_t elt = d->dtype == SSD200_F64 ? 8 : 4;
  size_t nel = d->dtype == SSD200_BF16 ? 2 : elt;
  // + argmax partials: (chunk or CTA, row) value / index pairs
  const size_t parts = (size_t)rows * ((vocab + 2047) / 2048 + 2 * 1024);
  return align_up((size_t)rows * d->d_model * nel) + align_up((size_t)rows * vocab * elt) +
         2 * align_up(parts * 4);
}

int ssd200_head(const ssd200_dims_t *d, int vocab, const void *hidden, int64_t hidden_row_stride,
                const void *final_norm_w, const void *embedding, void *logits,
                int64_t *argmax_out, int rows, void *workspace, size_t workspace_bytes,
                ssd200_stream_t stream) {
  TuneScope scope(d);
  int rc = check_dims(d);
  if (rc) return rc;
  REQUIRE(hidden && final_norm_w && embedding && rows >= 1 && vocab >= 1, SSD200_EINVAL,
          "head: bad arguments");
  REQUIRE(logits || argmax_out, SSD200_EINVAL, "head: nothing to compute");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d->dtype == SSD200_F32)
    return head_simt<float>(d, vocab, (const float *)hidden, hidden_row_stride,
                            (const float *)final_norm_w, (const float *)embedding,
                            (float *)logits, argmax_out, rows, workspace, workspace_bytes, st);
  if (d->dtype == SSD200_F64)
    return head_simt<double>(d, vocab, (const double *)hidden, hidden_row_stride,
                             (const double *)final_norm_w, (const double *)embedding,
                             (double *)logits, argmax_out, rows, workspace, workspace_bytes, st);
  return head_bf16(d, vocab, (const float *)hidden, hidden_row_stride,
                   (const float *)final_norm_w, (const bf16 *)embedding, (float *)logits,
                   argmax_out, rows, workspace, workspace_bytes, st);
}

int ssd200_gemm_bf16(const void *A, const void *B, void *C, int M, int N, int K,
                     ssd200_stream_t stream) {
  REQUIRE(A && B && C, SSD200_EINVAL, "gemm: null pointer");
  TcEpilogue ep{};
  ep.C = C;
  ep.ldc = N;
  return tc_gemm<TC_EPI_F32>((const bf16 *)A, K, (const bf16 *)B, K, M, N, K, ep,
                             static_cast<cudaStream_t>(stream));
}

uint64_t ssd200_launch_count(void) { return g_launches; }

int ssd200_set_phase_events(void *const *events, int n_phases) {
  REQUIRE(n_phases >= 0 && n_phases <= 5, SSD200_EINVAL, "n_phases must be in [0, 5]");
  g_phase_ev = n_phases ? events : nullptr;
  g_nphase = events ? n_phases : 0;
  return SSD200_OK;
}

#ifdef SSD200_TRACE
// diagnostic builds: reset the device timeline (and, with reset_slots, the
// slot counter: call before capturing / issuing the launches to trace)
int ssd200_trace_reset(int reset_slots, ssd200_stream_t stream) {
  if (reset_slots) {
    std::lock_guard<std::mutex> lk(g_trace_mu);
    g_trace_next = 0;
  }
  trace_init_kernel<<<1, 256, 0, (cudaStream_t)stream>>>();
  return cudaGetLastError() == cudaSuccess ? SSD200_OK : SSD200_ELAUNCH;
}
// copies n = min(max_slots, used slots) rows of 6 timestamps (ns) and names
// (32 chars each); returns n or < 0
int ssd200_trace_read(unsigned long long *out, char *names, int max_slots) {
  int n;
  {
    std::lock_guard<std::mutex> lk(g_trace_mu);
    n = g_trace_next < max_slots ? g_trace_next : max_slots;
    memcpy(names, g_trace_name, (size_t)n * 32);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return SSD200_ELAUNCH;
  if (cudaMemcpyFromSymbol(out, g_trace, (size_t)n * 6 * sizeof(unsigned long long)) !=
      cudaSuccess)
    return SSD200_ELAUNCH;
  return n;
}
int ssd200_trace_cycles(unsigned long long *out16) {
  if (cudaDeviceSynchronize() != cudaSuccess) return SSD200_ELAUNCH;
  return cudaMemcpyFromSymbol(out16, g_cyc, 16 * sizeof(unsigned long long)) == cudaSuccess
             ? SSD200_OK : SSD200_ELAUNCH;
}
#endif

}  // extern "C"
