/*
 * ssd200 — C ABI of the B200 (sm_100a) Mamba-2 SSD inference hot path.
 *
 * The reference engine (/root/reference/pkg/src/ssd_engine) has no FFI: its
 * boundary is the Python API re-exported in __init__.py:7-24.  Each entry
 * point below replaces the arithmetic behind one of those calls; the Python
 * package paper_2603_09555_b200 keeps the reference signatures and calls in
 * here (see INTEGRATION.md for the ctypes binding a maintainer would add).
 *
 * Rules: raw device pointers + explicit dims + a cudaStream_t; the caller owns
 * every buffer (workspace sizes via *_workspace()); no allocation, no host
 * synchronisation, no exceptions across the ABI.  Every call returns 0 on
 * success or a negative status; ssd200_last_error() gives a thread-local
 * message.  All launches are enqueued on `stream` and are CUDA-graph
 * capturable.
 *
 * Layouts (row-major, "row" = one token):
 *   hidden       (rows, d_model)          residual stream, f32 (f64 in f64 mode)
 *   hidden_lp    (rows, d_model)          bf16 shadow of hidden (bf16 mode only)
 *   ssm state    (batch, H, P, N)         compute dtype (f32 in bf16 mode)
 *   conv state   (batch, conv_dim, k-1)   newest column last (decode.py:49-69)
 *   W_in         f32/f64: (d_model, d_in_proj)  [reference layout, model.py:76]
 *                bf16:    (d_in_proj, d_model)  [K-major for tcgen05]
 *   W_out        f32/f64: (d_inner, d_model);  bf16: (d_model, d_inner)
 *   embedding    (vocab, d_model) weight dtype; the tied head reads it as-is.
 */
#ifndef SSD200_H
#define SSD200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *ssd200_stream_t; /* a cudaStream_t */

enum ssd200_dtype { SSD200_F32 = 0, SSD200_F64 = 1, SSD200_BF16 = 2 };

enum ssd200_status {
  SSD200_OK = 0,
  SSD200_EINVAL = -1,       /* bad argument (shape, null pointer, range) */
  SSD200_ELAUNCH = -2,      /* a CUDA launch failed */
  SSD200_EUNSUPPORTED = -3, /* dims outside what this build supports */
  SSD200_EWORKSPACE = -4    /* workspace too small */
};

/* Implementation choices of the bf16 tensor-core path, passed PER CALL through
 * ssd200_dims_t.tuning (NULL = the measured defaults from
 * ssd200_tuning_defaults).  There is no library-global option state: two
 * callers on one thread never see each other's choices.  Every setting
 * computes the same function; those marked [order] change the order of f32
 * partial sums (results agree to rounding, not bitwise). */
typedef struct ssd200_tuning {
  int size;                /* sizeof(ssd200_tuning_t), checked */
  int prefill_pdl;         /* programmatic dependent launch between prefill kernels (1) */
  int gemm_pair;           /* CTA-pair (cta_group::2) 256x256 prefill GEMM tiles (1) */
  int pair_min_tiles;      /* ... from this many 256x256 tiles (64) */
  int scan_variant;        /* 0 auto, 1 fused per-(b,h) chunk walk, 2 parallel chunk states + pass */
  int chunkscan_multicast; /* chunk walk: 4-CTA clusters share each chunk's B tile by TMA multicast (1) */
  int out_waves;           /* output kernel: head groups until >= out_waves x SMs CTAs (1) */
  int dec_pdl;             /* PDL between the decode kernels (1) */
  int dec_swap;            /* decode GEMMs: swapped-operand weight-streaming kernel (1) or tc_gemm (0) */
  int dec_small_ring;      /* [order] decode GEMMs: ~100 KB ring (1), 192 KB (0), -1 auto (B <= dec_small_max) */
  int dec_small_max;       /* largest batch on the ~100 KB ring when dec_small_ring is auto (32) */
  int dec_split_in;        /* [order] decode in_proj split-K factor (0 auto) */
  int dec_split_out;       /* [order] decode out_proj split-K factor (0 auto) */
  int stream_stages;       /* decode state stream: ring stages (0 = as many as fit) */
  int stream_cps;          /* decode state stream: CTAs per SM (0 auto, 1, 2) */
  int stream_cw;           /* decode state stream: consumer warps (8 or 16) */
  int out_interleave;      /* SSD output kernel: the two row tiles of a chunk run side by side (1) */
  int gemm_group_m;        /* prefill GEMM tile order: row blocks per group (0 auto, 1 row-major) */
  int gemm_stream;         /* prefill GEMM epilogues: outputs and residual with evict-first (.cs)
                              accesses, so they do not evict the operands' L2 reuse: 0 off,
                              1 when the output exceeds 1 GB as f32 (1), 2 always */
  int stream_chunk;        /* decode state stream tile hand-out: 0 auto (once a CTA's fair share
                              is >= 4 tiles, chunks from an atomic counter: 1 tile, 3 from a
                              share of 8), -1 static contiguous ranges, > 0 tiles per chunk */
  int stream_reg_state;    /* decode state stream with one tile per CTA (2 B x H <= SMs, static
                              tiles): the state rows go to registers at kernel entry, not through
                              the smem ring (1) */
} ssd200_tuning_t;

void ssd200_tuning_defaults(ssd200_tuning_t *t);

/* Model widths + numerics (model.py:20-70).  a = -exp(A_log) is host-computed
 * (ssd.py:99-112) so the bf16e ablation rounds exactly like the reference. */
typedef struct ssd200_dims {
  int dtype; /* enum ssd200_dtype: compute mode */
  int d_model, d_inner, n_heads, head_dim, d_state, n_groups, conv_kernel, chunk_size;
  double norm_eps, dt_min, dt_max;
  const ssd200_tuning_t *tuning; /* NULL = defaults (see ssd200_tuning_t) */
} ssd200_dims_t;

typedef struct ssd200_layer {
  const void *W_in, *conv_w, *conv_b, *dt_bias, *a, *D, *norm_w, *W_out;
  /* optional (d_model) weight of a residual pre-norm, compute dtype (f32 in
   * bf16 mode): the block then runs in_proj on rmsnorm(hidden) * pre_norm_w
   * (norm_eps) and adds its output to the un-normalised hidden — the layout
   * of real state-spaces/mamba2 checkpoints (backbone.layers.N.norm), which
   * the reference block drops (converter/mapping.json:75-78).  NULL = the
   * reference block (model.py:124-174). */
  const void *pre_norm_w;
} ssd200_layer_t;

int ssd200_abi_version(void);
const char *ssd200_last_error(void);

/* ---- ssd_forward (ssd.py:209-257): chunked SSD scan --------------------
 * X (B,T,H,P), dt (B,T,H) [post-softplus, >=0], a (H) [<=0], Bmat/Cmat
 * (B,T,G,N), D (H) or NULL (adds D*x, model.py:166), init_state (B,H,P,N) or
 * NULL -> Y (B,T,H,P), final_state (B,H,P,N).  dtype F32 or F64. */
size_t ssd200_chunk_scan_workspace(int dtype, int batch, int seqlen, int heads, int head_dim,
                                   int d_state, int chunk);
int ssd200_chunk_scan(int dtype, const void *X, const void *dt, const void *a, const void *Bmat,
                      const void *Cmat, const void *D, const void *init_state, void *Y,
                      void *final_state, int batch, int seqlen, int heads, int head_dim,
                      int groups, int d_state, int chunk, void *workspace,
                      size_t workspace_bytes, ssd200_stream_t stream);

/* ---- embedding gather (model.py:198, decode.py:96) ----------------------
 * tokens int64 (rows).  Host callers range-check ids like model.py:191-195;
 * for ids that live on the device (no host sync) the kernel checks them: an
 * id outside [0, vocab) yields a NaN row (never an out-of-bounds read). */
int ssd200_embed(const ssd200_dims_t *d, const int64_t *tokens, int rows, int vocab,
                 const void *embedding, void *hidden, void *hidden_lp, ssd200_stream_t stream);

/* ---- block_forward (model.py:124-174) over (batch, seqlen) ---------------
 * hidden/hidden_lp updated in place; writes the layer's final SSM state and
 * conv tail (pre-activation, newest last, zero-padded when T<k-1). */
size_t ssd200_prefill_layer_workspace(const ssd200_dims_t *d, int batch, int seqlen);
int ssd200_prefill_layer(const ssd200_dims_t *d, const ssd200_layer_t *w, void *hidden,
                         void *hidden_lp, void *ssm_out, void *conv_out, int batch, int seqlen,
                         void *workspace, size_t workspace_bytes, ssd200_stream_t stream);

/* ---- head-group-sharded block_forward (bf16) --------------
 * d describes THIS rank's shard (d_inner = local heads * head_dim, n_heads =
 * local heads, a multiple of 8); w holds the shard's weights (its z/x/dt
 * columns of W_in, its x conv channels + the replicated B/C ones, its D /
 * dt_bias / a, and its rows of W_out with norm_w folded in).  Instead of
 * updating hidden it writes, per row r, partial[r, 0:d_model] = u_local .
 * W_out'_local and partial[r, d_model] = sum of u_local^2 (row pitch
 * partial_ld, a multiple of 4, >= d_model + 1).  The caller sums partial
 * over the ranks (one all-reduce) and applies ssd200_resid_norm_finish.
 * Workspace: ssd200_prefill_layer_workspace(d, ...). */
int ssd200_prefill_layer_partial(const ssd200_dims_t *d, const ssd200_layer_t *w,
                                 const void *hidden_lp, float *partial, long partial_ld,
                                 void *ssm_out, void *conv_out, int batch, int seqlen,
                                 void *workspace, size_t workspace_bytes, ssd200_stream_t stream);
/* hidden += partial[:, :d_model] * rsqrt(partial[:, d_model] / d_inner_full + eps),
 * hidden_lp = bf16(hidden)  (model.py:166-173 after the all-reduce) */
int ssd200_resid_norm_finish(int d_model, int d_inner_full, double eps, void *hidden,
                             void *hidden_lp, const float *partial, long partial_ld, long rows,
                             ssd200_stream_t stream);

/* ---- head-group-sharded decode_step layer (bf16) ----------
 * As ssd200_prefill_layer_partial for one token per row: d / w describe THIS
 * rank's shard (local heads a multiple of 4); the rank's cache slices
 * (ssm (batch, H_local, P, N), conv (batch, conv_dim_local, k-1)) are updated
 * (in place when aliased); hidden is NOT updated: partial[b, 0:d_model] =
 * u_local . W_out'_local and partial[b, d_model] = sum u_local^2.  The caller
 * sums partial over the ranks (one all-reduce) and applies
 * ssd200_resid_norm_finish.  Workspace: ssd200_decode_layer_workspace(d, batch). */
int ssd200_decode_layer_partial(const ssd200_dims_t *d, const ssd200_layer_t *w,
                                const void *hidden_lp, float *partial, long partial_ld,
                                const void *ssm_in, void *ssm_out, const void *conv_in,
                                void *conv_out, int batch, void *workspace,
                                size_t workspace_bytes, ssd200_stream_t stream);

/* ---- one decode_step layer (decode.py:99-140) ----------------------------
 * ssm_out/conv_out may alias ssm_in/conv_in (in-place update for generate). */
size_t ssd200_decode_layer_workspace(const ssd200_dims_t *d, int batch);
int ssd200_decode_layer(const ssd200_dims_t *d, const ssd200_layer_t *w, void *hidden,
                        void *hidden_lp, const void *ssm_in, void *ssm_out, const void *conv_in,
                        void *conv_out, int batch, void *workspace, size_t workspace_bytes,
                        ssd200_stream_t stream);

/* ---- every layer of one decode_step (decode.py:99-140) ---------------------
 * layers: HOST array of n_layers ssd200_layer_t.  ssm (n_layers, batch, H, P, N)
 * and conv (n_layers, batch, conv_dim, k-1) contiguous; out may alias in.
 * hidden / hidden_lp hold the embedded tokens on entry and the residual stream
 * after the last layer on return (ssd200_decode_layer per layer, one ABI call
 * per token step).  Workspace: ssd200_decode_layers_workspace. */
size_t ssd200_decode_layers_workspace(const ssd200_dims_t *d, int batch);
int ssd200_decode_layers(const ssd200_dims_t *d, const ssd200_layer_t *layers, int n_layers,
                         void *hidden, void *hidden_lp, const void *ssm_in, void *ssm_out,
                         const void *conv_in, void *conv_out, int batch, void *workspace,
                         size_t workspace_bytes, ssd200_stream_t stream);

/* ---- final RMSNorm + tied head (+ greedy argmax) (model.py:204-205,
 * decode.py:72-74,142-143) -------------------------------------------------
 * Reads `rows` rows of hidden spaced hidden_row_stride elements apart.
 * logits (rows, vocab) f32 (f64 in f64 mode) or NULL; argmax_out (rows) int64
 * or NULL (ties -> lowest id). */
size_t ssd200_head_workspace(const ssd200_dims_t *d, int vocab, int rows);
int ssd200_head(const ssd200_dims_t *d, int vocab, const void *hidden, int64_t hidden_row_stride,
                const void *final_norm_w, const void *embedding, void *logits,
                int64_t *argmax_out, int rows, void *workspace, size_t workspace_bytes,
                ssd200_stream_t stream);

/* ---- raw bf16 tensor-core GEMM (tcgen05 + TMA + TMEM), for tests/bench --
 * C (M,N) f32 = A (M,K) bf16 row-major  x  B^T where B is (N,K) bf16 row-major.
 * K % 8 == 0 (16-byte TMA row pitch); ragged M/N/K tiles are zero-filled. */
int ssd200_gemm_bf16(const void *A, const void *B, void *C, int M, int N, int K,
                     ssd200_stream_t stream);

/* ---- instrumentation (bench.py) -----------------------------------------
 * Number of kernels this library has launched from the calling thread. */
uint64_t ssd200_launch_count(void);
/* Phase timing: when set (non-NULL), ssd200_prefill_layer records
 * events[2*p] before and events[2*p+1] after phase p on the call's stream
 * (p: 0 in_proj, 1 conv, 2 scan, 3 gated norm, 4 out_proj); events are
 * cudaEvent_t handles owned by the caller.  Pass NULL to disable. */
int ssd200_set_phase_events(void *const *events, int n_phases);

#ifdef __cplusplus
}
#endif

#endif /* SSD200_H */
