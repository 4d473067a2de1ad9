/*
 * fsa_b200.h — C ABI of the B200-native FuseSampleAgg operator (sm_100a).
 *
 * Drop-in boundary for the reference's compiled-kernel layer (numba, CPU):
 *   reference  pkg/src/fsa/kernels.py            this ABI
 *   ---------------------------------------      -----------------------------------------
 *   fused_1hop(...)          kernels.py:127-149  fsa_fused_1hop_fwd   (X != NULL)
 *   sample_1hop(...)         kernels.py:87-97    fsa_fused_1hop_fwd   (X == NULL, out == NULL)
 *   fused_2hop(...)          kernels.py:152-198  fsa_fused_2hop_fwd   (X != NULL)
 *   sample_2hop(...)         kernels.py:99-120   fsa_fused_2hop_fwd   (X == NULL, out == NULL)
 *   invert_targets +
 *   scatter_from_grad        kernels.py:296-338  fsa_fused_1hop_bwd / fsa_fused_2hop_bwd
 *     (with the denominators fused.py:216-217 / fused.py:248-250 computed on device)
 *   derive_state             kernels.py:71-73    fsa_derive_states    (test hook)
 *   xorshift_steps           kernels.py:76-80    fsa_xorshift_steps   (test hook)
 *
 * Conventions (kernels.py:1-5 and SURVEY.md §8b):
 *   - every pointer argument except `stream` is a DEVICE pointer; the caller allocates every
 *     output, the op writes in place, nothing is allocated inside;
 *   - calls are asynchronous and stream-ordered on `stream` (a cudaStream_t, NULL = legacy);
 *   - return value: FSA_OK or an fsa_status (argument errors detected on the host);
 *     data-dependent errors (seed / saved index out of range, negative take) are detected on
 *     device, the offending item is skipped, and a bit is OR-ed into the workspace error word,
 *     readable with fsa_read_error();
 *   - results are bitwise independent of launch geometry and of how a batch is sharded across
 *     GPUs: sampling streams are keyed on the GLOBAL batch position `root_offset + i`
 *     (root_offset = 0 reproduces the reference exactly, kernels.py:92,135,160,175);
 *   - workspace: size from fsa_ws_bytes(op, ...); it must be zero-filled when first
 *     allocated; every op leaves its persistent part zeroed again, so one buffer can be
 *     reused for any number of calls of the same op kind on the same stream.  A backward
 *     workspace carries per-node counters laid out for one graph size N: reuse it only with
 *     the same N (a different N needs a fresh zero-filled buffer).
 */
#ifndef FSA_B200_H_
#define FSA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum fsa_status {
  FSA_OK = 0,
  FSA_ERR_ARG = 1,        /* invalid shape / fanout / null pointer            */
  FSA_ERR_DTYPE = 2,      /* unsupported dtype code                            */
  FSA_ERR_WORKSPACE = 3,  /* workspace too small                               */
  FSA_ERR_CUDA = 4,       /* a CUDA runtime call failed (see fsa_last_cuda_error) */
  FSA_ERR_ALIGN = 5       /* misaligned feature / output pointer               */
};

enum fsa_dtype { FSA_F32 = 0, FSA_F64 = 1, FSA_BF16 = 2, FSA_F16 = 3 };

/* bits of the device error word */
enum fsa_device_error {
  FSA_DEVERR_SEED_RANGE = 1,  /* "seed out of range"        fused.py:84-85   */
  FSA_DEVERR_INDEX_RANGE = 2, /* "saved index out of range" fused.py:213,245 */
  FSA_DEVERR_NEG_TAKE = 4     /* "negative take count"      fused.py:211-212 */
};

enum fsa_op { FSA_OP_FWD1 = 1, FSA_OP_FWD2 = 2, FSA_OP_BWD1 = 3, FSA_OP_BWD2 = 4 };

/* phases of the replay backward (fsa_fused_*_bwd_phase): PLAN needs only the saved ids (per-node
 * counts, segment reservation, scatter of multi-hit slots); TERMS needs grad_out and the saved
 * ids, not PLAN (the per-group quotient table grad_out[row] / den in the workspace), so the two
 * may run concurrently on different streams; ROWS needs both (the gradient row writes; grad_out
 * is not read).  PLAN and TERMS (either order or concurrent), then ROWS, on the same workspace
 * == one fsa_fused_*_bwd call. */
enum fsa_bwd_phase {
  FSA_BWD_PLAN = 1,
  FSA_BWD_TERMS = 2,
  FSA_BWD_ROWS = 4,
  FSA_BWD_APPLY = 6, /* TERMS | ROWS */
  FSA_BWD_ALL = 7
};

/* phases of the 2-hop forward (fsa_fused_2hop_fwd_phase): SAMPLE writes s1/s2/take1/take2 (all
 * the replay backward's PLAN needs), GATHER the feature means.  SAMPLE then GATHER on the same
 * workspace == one fsa_fused_2hop_fwd call. */
enum fsa_fwd_phase { FSA_FWD_SAMPLE = 1, FSA_FWD_GATHER = 2, FSA_FWD_ALL = 3 };

const char* fsa_version(void);
const char* fsa_status_string(int status);
int fsa_last_cuda_error(void);
/* select the CUDA device for subsequent calls from this host thread */
int fsa_set_device(int device);

/* Number of kernels this library has launched in this process (all ops, all devices). */
unsigned long long fsa_launch_count(void);
/* Per-kernel CUDA-event timing: fsa_profile(1) clears and starts recording events around every
 * kernel launch on its launching stream, fsa_profile(0) stops.  fsa_profile_read synchronises
 * the recorded events and returns, per kernel name (48-byte slots in `names`), the summed
 * device time and the launch count. */
int fsa_profile(int enable);
int fsa_profile_read(int max_kernels, char* names, double* total_ms, int64_t* launches, int* n_kernels);

/* Per-block timeline of this library's kernels on the current device, for profiling: with a
 * device buffer of slots*blocks*2 uint64 (fsa_trace_geometry; starts set to UINT64_MAX, ends to
 * 0), every block of every kernel folds its first-warp start and last-warp end (%globaltimer,
 * ns) into buf[(slot*blocks + blockIdx)*2 + {0,1}]; slot = kernel kind (see TraceSlot in the
 * source).  fsa_trace(NULL) turns it off (the default). */
int fsa_trace(void* buf);
int fsa_trace_geometry(int* slots, int* blocks);

/* Workspace bytes for `op`.  FWD1: (B, k1=k); FWD2: (B, k1, k2); BWD1: (B, k1=k, D, dtype, N);
 * BWD2: (B, k1, k2, D, dtype, N) -- a backward workspace holds the term table, G x D values in
 * the accumulation type (fp64 for FSA_F64, else fp32).  Unused arguments are ignored; 0 means
 * an invalid request. */
size_t fsa_ws_bytes(int op, int64_t B, int32_t k1, int32_t k2, int64_t D, int dtype, int64_t N);

/* Synchronously read (and optionally clear) the device error word of a workspace. */
int fsa_read_error(void* ws, int clear, int* flags, void* stream);

/* ---- forward: fused sample + mean ------------------------------------------------------
 * rowptr int32[N+1], col int32[E]: CSR with ascending, de-duplicated rows (graph.py:108-151).
 * X [N, D] of `dtype` with row stride x_stride (elements); out [B, D] row stride out_stride.
 * seeds int64[B].  save != 0 writes the replay indices (−1 padded, fused.py:40-77):
 *   1-hop: samples int32[B,k], takes int32[B]
 *   2-hop: s1 int32[B,k1], s2 int32[B,k1,k2], take1 int32[B], take2 int32[B,k1]
 * X == NULL and out == NULL gives the sampling-only kernels (sample_1hop / sample_2hop). */
int fsa_fused_1hop_fwd(const int32_t* rowptr, const int32_t* col, int64_t N,
                       const void* X, int64_t D, int64_t x_stride, int dtype,
                       const int64_t* seeds, int64_t B, int64_t root_offset,
                       int32_t k, uint64_t base_seed, int save,
                       int32_t* samples, int32_t* takes,
                       void* out, int64_t out_stride,
                       void* ws, size_t ws_bytes, void* stream);

int fsa_fused_2hop_fwd(const int32_t* rowptr, const int32_t* col, int64_t N,
                       const void* X, int64_t D, int64_t x_stride, int dtype,
                       const int64_t* seeds, int64_t B, int64_t root_offset,
                       int32_t k1, int32_t k2, uint64_t base_seed, int save,
                       int32_t* s1, int32_t* s2, int32_t* take1, int32_t* take2,
                       void* out, int64_t out_stride,
                       void* ws, size_t ws_bytes, void* stream);

/* Same as above with the base seed read from device memory (one uint64) when the kernels run,
 * so a captured CUDA graph can be replayed with a new seed per step. */
int fsa_fused_1hop_fwd_dseed(const int32_t* rowptr, const int32_t* col, int64_t N,
                             const void* X, int64_t D, int64_t x_stride, int dtype,
                             const int64_t* seeds, int64_t B, int64_t root_offset,
                             int32_t k, const uint64_t* base_seed, int save,
                             int32_t* samples, int32_t* takes,
                             void* out, int64_t out_stride,
                             void* ws, size_t ws_bytes, void* stream);

int fsa_fused_2hop_fwd_dseed(const int32_t* rowptr, const int32_t* col, int64_t N,
                             const void* X, int64_t D, int64_t x_stride, int dtype,
                             const int64_t* seeds, int64_t B, int64_t root_offset,
                             int32_t k1, int32_t k2, const uint64_t* base_seed, int save,
                             int32_t* s1, int32_t* s2, int32_t* take1, int32_t* take2,
                             void* out, int64_t out_stride,
                             void* ws, size_t ws_bytes, void* stream);

/* fsa_fused_2hop_fwd in phases (enum fsa_fwd_phase); base_seed_dev, when not NULL, replaces
 * base_seed by a device-resident value (as the _dseed variant). */
int fsa_fused_2hop_fwd_phase(const int32_t* rowptr, const int32_t* col, int64_t N,
                             const void* X, int64_t D, int64_t x_stride, int dtype,
                             const int64_t* seeds, int64_t B, int64_t root_offset,
                             int32_t k1, int32_t k2, uint64_t base_seed, const uint64_t* base_seed_dev,
                             int save, int32_t* s1, int32_t* s2, int32_t* take1, int32_t* take2,
                             void* out, int64_t out_stride,
                             void* ws, size_t ws_bytes, void* stream, int phase);

/* ---- backward: deterministic saved-index replay (no float atomics) ----------------------
 * grad_out [B, D] (row stride g_stride) of `dtype`.  For every touched node v the op writes
 *   grad_x[v, :] = (((+0.0 + a_1) + a_2) + ...)   a_i = grad_out[t_i / K] / denom[t_i]
 * over the slots t_1 < t_2 < ... that sampled v (ascending flat slot order, kernels.py:296-338),
 * denom = max(take,1) (1-hop) or max(t1,1)*max(t2,1) (2-hop, one division by the product).
 * zero_mode: 0 = untouched rows of grad_x are left as they are (caller keeps them zero),
 *            1 = grad_x is zero-filled first (the reference's out.fill(0), fused.py:290-296).
 * grad_x may be NULL when grad_rows != NULL (sparse-COO output only).
 * Optional outputs: touched int32[B*K] receives the distinct touched node ids (any order)
 * and n_touched int32[1] their count; grad_rows [B*K, D] receives the row of touched[q] at
 * row q (requires touched). */
int fsa_fused_1hop_bwd(const void* grad_out, int64_t B, int64_t D, int64_t g_stride, int dtype,
                       const int32_t* samples, const int32_t* takes, int32_t k, int64_t N,
                       void* grad_x, int zero_mode,
                       int32_t* touched, int32_t* n_touched, void* grad_rows,
                       void* ws, size_t ws_bytes, void* stream);

int fsa_fused_2hop_bwd(const void* grad_out, int64_t B, int64_t D, int64_t g_stride, int dtype,
                       const int32_t* s1, const int32_t* s2, int32_t k1, int32_t k2, int64_t N,
                       void* grad_x, int zero_mode,
                       int32_t* touched, int32_t* n_touched, void* grad_rows,
                       void* ws, size_t ws_bytes, void* stream);

/* The same two ops split into phases (enum fsa_bwd_phase): a step scheduler can run PLAN, which
 * reads only the ids, concurrently with the forward's gather or the head that produces grad_out
 * (grad_out may be NULL unless the TERMS bit is set), and TERMS as soon as grad_out exists.
 * Phases must follow each other on the same workspace, stream-ordered. */
int fsa_fused_1hop_bwd_phase(const void* grad_out, int64_t B, int64_t D, int64_t g_stride, int dtype,
                             const int32_t* samples, const int32_t* takes, int32_t k, int64_t N,
                             void* grad_x, int zero_mode,
                             int32_t* touched, int32_t* n_touched, void* grad_rows,
                             void* ws, size_t ws_bytes, void* stream, int phase);

int fsa_fused_2hop_bwd_phase(const void* grad_out, int64_t B, int64_t D, int64_t g_stride, int dtype,
                             const int32_t* s1, const int32_t* s2, int32_t k1, int32_t k2, int64_t N,
                             void* grad_x, int zero_mode,
                             int32_t* touched, int32_t* n_touched, void* grad_rows,
                             void* ws, size_t ws_bytes, void* stream, int phase);

/* fsa_fused_2hop_bwd_phase into a dense gradient with row stride gx_stride (elements, >= D) of
 * which the op may write the first gx_cols columns (D <= gx_cols <= gx_stride).  When gx_cols
 * reaches D rounded up to 64 bytes, the row writers store whole 64-byte bursts (the padding
 * columns get zeros): a persistent, op-owned buffer of padded rows is then written without
 * partial bursts (400-byte fp32 rows, 1,204-byte bf16 rows).  No COO output. */
int fsa_fused_2hop_bwd_phase_rows(const void* grad_out, int64_t B, int64_t D, int64_t g_stride, int dtype,
                                  const int32_t* s1, const int32_t* s2, int32_t k1, int32_t k2, int64_t N,
                                  void* grad_x, int64_t gx_stride, int64_t gx_cols, int zero_mode,
                                  void* ws, size_t ws_bytes, void* stream, int phase);

/* grad[rows[i], :] = 0 for i < n_rows, rows[i] < 0 skipped (duplicates harmless): sparse
 * re-zero of a persistent gradient buffer between steps, e.g. with the previous step's flat
 * s2 / samples as `rows`. */
int fsa_zero_rows(void* grad, int64_t D, int dtype, const int32_t* rows, int64_t n_rows, void* stream);
/* The same for rows of stride gx_stride, writing the first gx_cols columns (whole 64-byte bursts
 * when gx_cols reaches D rounded up to 64 bytes, as fsa_fused_2hop_bwd_phase_rows). */
int fsa_zero_rows_strided(void* grad, int64_t D, int64_t gx_stride, int64_t gx_cols, int dtype,
                          const int32_t* rows, int64_t n_rows, void* stream);

/* ---- test hooks (device arrays of length n) ---------------------------------------------- */
int fsa_derive_states(const uint64_t* base_seed, const int64_t* root, const int64_t* hop,
                      const int64_t* index, int64_t n, uint64_t* out, void* stream);
int fsa_xorshift_steps(uint64_t state, int64_t n, uint64_t* out, void* stream);
/* out[i] = T^dist[i](states[i]) through the GF(2) jump tables */
int fsa_jump(const uint64_t* states, const int64_t* dist, int64_t n, uint64_t* out, void* stream);
/* Adds to *mismatches (device u64) the number of inputs where the backward's reciprocal-based
 * division differs bitwise from IEEE division: every divisor 1..dmax against every fp32
 * significand of two binades, plus sampled fp64 inputs. */
int fsa_div_check(int dmax, unsigned long long* mismatches, void* stream);
/* Micro-benchmark of the sampler's draw loop: n draws per lane from modulus m0 (mode 0 Barrett,
 * 1 fraction test, 2 / 3 the same as two interleaved streams per lane).  lanes <= 32: one warp,
 * out[0] = clock64 cycles of lane 0; lanes > 32 (a multiple of 256): lanes / 256 CTAs of 256
 * threads, for the caller to time with events (the GPU's draw throughput, the sampler roofline).
 * n must be a multiple of 256. */
int fsa_bench_draws(int mode, int n, uint32_t m0, int k, int lanes, unsigned long long* out, void* stream);
/* ---- unfused comparator (baseline.py:63-194): the same sums with every intermediate in HBM ----
 * fsa_gather_rows: out[t] = X[ids[t]] (zero row for -1)                 (kernels.gather_rows)
 * fsa_group_mean:  out[g] = (+0 + sum_{l < take[g]} row(g*k + l)) / max(1, take[g]) with
 *                  row(i) = src[remap ? remap[i] : i]; src_acc / out_acc select the accumulation
 *                  type (fp32, fp64 for FSA_F64) instead of `dtype` for src / out rows
 *                  (kernels.agg_1hop_block, partials_2hop_block/_dedup, agg_2hop_from_partials)
 * fsa_baseline_*_bwd: the replay backward with the per-slot gradient block materialised in
 *                  d_gathered [B*k(1*k2)][dg_stride] (accumulation type, dg_stride a multiple of 8
 *                  and >= D, 16-B aligned) between the division and the ordered scatter
 *                  (kernels.expand_grad + scatter_from_block); same workspace as fsa_fused_*_bwd. */
int fsa_gather_rows(const void* X, int64_t D, int64_t x_stride, int dtype, const int32_t* ids, int64_t n,
                    void* out, int64_t out_stride, void* stream);
int fsa_group_mean(const void* src, int64_t src_stride, int src_acc, const int32_t* remap, const int32_t* take,
                   int32_t k, int64_t G, int64_t D, int dtype, void* out, int64_t out_stride, int out_acc,
                   void* stream);
int fsa_baseline_1hop_bwd(const void* grad_out, int64_t B, int64_t D, int64_t g_stride, int dtype,
                          const int32_t* samples, const int32_t* takes, int32_t k, int64_t N, void* grad_x,
                          int zero_mode, void* d_gathered, int64_t dg_stride, void* ws, size_t ws_bytes,
                          void* stream);
int fsa_baseline_2hop_bwd(const void* grad_out, int64_t B, int64_t D, int64_t g_stride, int dtype,
                          const int32_t* s1, const int32_t* s2, int32_t k1, int32_t k2, int64_t N, void* grad_x,
                          int zero_mode, void* d_gathered, int64_t dg_stride, void* ws, size_t ws_bytes,
                          void* stream);

/* Performance knobs for experiments (results never change): what = 1, the sampler's bucket-length
 * divisor (value >= 1; 0, the default: 1 for a phase of >= 2^24 draws, else 2); what = 2, the gather's L2 prefetch of a root's rows (0/1,
 * default 0); what = 3, CTAs per SM of the sparse re-zero (1..8, default 1); what = 4, CTAs per SM of the
 * backward's slot count (1..64, default 8); what = 5, CTAs per SM of the multi-hit row
 * writer (1..8; 0, the default: 2, launched beside the singles, for rows wider than one
 * 32-lane chunk span, else 4 after them); what = 6, the 2-hop forward's first hop (1: one warp per root
 * samples, finalises and plans it in one kernel, the default; 2: the tile sampler with
 * separate planning passes, faster for dense graphs with long first-hop chains). */
int fsa_tune(int what, int value);
/* out[i] = x[i] % m[i] through the Barrett path used by the sampler (2 <= m <= 2^30) */
int fsa_umod(const uint64_t* x, const uint32_t* m, int64_t n, uint32_t* out, void* stream);

/* Row stage of the training step's SAGE-mean classifier head (fp32; with two library GEMMs it
 * replaces head_forward + cross_entropy + head_backward, pkg/src/fsa/train.py:111-160). For B
 * seeds: concat = [X[seeds] | agg], hidden = ReLU(concat W1 + b1), logits = hidden W2 + b2, the
 * softmax cross-entropy against labels, dlogits = (softmax - onehot) / B, dhidden, and
 * d agg -> grad_agg [B x D] (row stride grad_stride). The workspace receives, in order (each
 * region 256-byte aligned): [concat | 1] [B x (2D+1)], [hidden | 1] [B x (H+1)], dhidden [B x H],
 * dlogits [B x C] and the per-row losses [B], so that [concat | 1]^T dhidden = [dW1; db1],
 * [hidden | 1]^T dlogits = [dW2; db2] and loss = mean(row losses). Row-major, element strides;
 * H % 4 == 0, H <= 512, W1 / W2 16-byte aligned. Labels outside [0, C) give NaN rows. One
 * kernel on `stream`. */
/* AdamW of the training step (fp32; pkg/src/fsa/train.py:163-184) over n_tensors (<= 8)
 * parameter / gradient / first-moment / second-moment arrays of sizes[k] elements (host arrays of
 * device pointers). When every gradient element is finite: *step_count (device double) += 1, the
 * bias corrections are derived from it in double, and every parameter takes the reference's
 * update in its operation order (fp32, no contraction); *ok_out (device byte) = 1. Otherwise
 * nothing changes and *ok_out = 0 (the reference raises NonFiniteGradientError). Two kernels on
 * `stream`; ws: fsa_adamw_ws_bytes() bytes of device scratch, zero before the first call (the
 * kernels leave it zero, so a persistent buffer needs no memset per step). */
size_t fsa_adamw_ws_bytes(void);
int fsa_adamw_step(int n_tensors, float* const* params, const float* const* grads, float* const* exp_avg,
                   float* const* exp_avg_sq, const int64_t* sizes, double* step_count, double lr, double beta1,
                   double beta2, double weight_decay, double eps, unsigned char* ok_out, void* ws, size_t ws_bytes,
                   void* stream);
size_t fsa_sage_head_ws_bytes(int64_t B, int32_t D, int32_t H, int32_t C);
size_t fsa_sage_head_smem_bytes(int32_t D, int32_t H, int32_t C);
int fsa_sage_head_rows(const float* X, int64_t x_stride, const int64_t* seeds, const float* agg, int64_t agg_stride,
                       const int64_t* labels, int64_t B, int32_t D, int32_t H, int32_t C, const float* W1,
                       const float* b1, const float* W2, const float* b2, float* grad_agg, int64_t grad_stride,
                       void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FSA_B200_H_ */
