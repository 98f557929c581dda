/*
 * oscar.h — C ABI of liboscar.so, the B200 (sm_100a) hot path of OSCAR (arXiv 2605.17757).
 *
 * The three calls follow the paper's statement of the problem:
 *   calibrate(Q, S·V) -> R_K, R_V   Alg. 1 `Calibrate`, §3
 *   quantize_append(K, V)           Alg. 1 `Prefill`/`QuantizeAndWrite`,
 *                                   §4 "KV Cache Update"
 *   attend(q) -> o                  Alg. 1 `DecodeStep` attention, §4 "Decoding
 *                                   Attention Kernel"
 *
 * Conventions (all calls):
 *  - Pointers are DEVICE pointers owned by the caller unless stated otherwise; the library
 *    never allocates device memory after oscar_create and never frees caller memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All device
 *    work is enqueued asynchronously on it; no call synchronizes the host except
 *    oscar_calib_finalize when `info` is non-NULL (documented there).
 *  - bf16 tensors are passed as `const void*` holding IEEE bfloat16 bit patterns.
 *  - Row-vector convention: rotated row x̃ = x · R, R stored row-major R[k][j].
 *  - Errors: argument validation is synchronous and returns a status; oscar_last_error()
 *    returns a thread-local message for the last non-OK status of the calling thread.
 *    Launch failures return OSCAR_ERR_CUDA; asynchronous device faults surface at the
 *    caller's next synchronization.  There is no CPU fallback: every entry point that
 *    computes runs CUDA kernels for sm_100a or fails.
 *  - Out of contract (not checked on the hot path): non-finite inputs, |x̃| >= 2^15 (fp16
 *    metadata range), slots / pages out of range, two rows written to one slot in one call.
 *
 * Packed cache FORMAT: pool[num_pages][H_kv][page_bytes], slot = page·P + off.
 * One (page, kv-head) block: K codes [P][d·b/8] ‖ V codes [P/4][d·b/8][4] (rows byte-
 * interleaved in 4-token groups) ‖ meta [P][d/G][4] fp16 (s_K, m_K, s_V, m_V), padded to a
 * multiple of 256 B.  Code i of a row occupies bits [b·i, b·i+b) of the row's little-endian
 * bitstream ("four 2-bit values packed per byte").  Dequantized x̂ = s·c + m, i.e.
 * m = -s·z of App A.5.
 */
#ifndef OSCAR_H_
#define OSCAR_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define OSCAR_API __attribute__((visibility("default")))
#else
#define OSCAR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OSCAR_OK = 0,
  OSCAR_ERR_ARG = 1,          /* invalid argument value (NULL, negative size, G∤d, ...)  */
  OSCAR_ERR_DIM = 2,          /* non-power-of-two head_dim                               */
  OSCAR_ERR_UNSUPPORTED = 3,  /* valid but not implemented on this GPU path (e.g. d≠128) */
  OSCAR_ERR_CUDA = 4,         /* a CUDA runtime/launch error                             */
  OSCAR_ERR_CONVERGENCE = 5   /* Jacobi eigensolver hit its sweep cap                    */
} oscar_status;

typedef struct oscar_ctx oscar_ctx; /* opaque; immutable after create (except oscar_set_variant,
                                      which must not race with other calls) => thread-safe */

typedef struct {
  int32_t head_dim;        /* d; must be a power of two; this build implements d = 128       */
  int32_t num_q_heads;     /* H_q of this rank's shard                                       */
  int32_t num_kv_heads;    /* H_kv of this shard; H_q % H_kv == 0, g = H_q / H_kv (GQA).
                              Attend implements g <= 8 (OSCAR_ERR_UNSUPPORTED otherwise);
                              calibration takes any g: a context with H_kv = 1 accumulates one
                              covariance over all query heads (NEXT-4 shared-rotation mode,
                              P:L140-144; reading Z14's alternative)                         */
  int32_t bits;            /* b in {2, 3, 4}; b = 3 (codes straddle bytes, reading Z23) runs on
                              the simple CUDA-core kernels, b = 2, 4 also on the tensor-core ones */
  int32_t group_size;      /* G in {32, 64, 128}, G | d; same for K and V (reading Z7)        */
  int32_t page_size;       /* P tokens per page; multiple of 16; 0 => 64                       */
  float clip_ratio_k;      /* rho_K in (0, 1]; 1 = no clipping (App A.5)         */
  float clip_ratio_v;      /* rho_V in (0, 1]                                                  */
  float softmax_scale;     /* 0 => 1/sqrt(d)                                          */
  int32_t attend_pages_per_split; /* split-K granularity of attend; 0 => automatic           */
} oscar_config;

/* Create / destroy a context.  Validates the config (OSCAR_ERR_ARG / _DIM / _UNSUPPORTED). */
OSCAR_API oscar_status oscar_create(const oscar_config* cfg, oscar_ctx** out);
OSCAR_API void oscar_destroy(oscar_ctx* ctx);
OSCAR_API const char* oscar_last_error(void);
OSCAR_API const char* oscar_version(void);

/* Bytes of one (page, kv-head) block; the caller allocates pool[num_pages][H_kv][page_bytes]
 * (256-byte aligned base).  Returns 0 for a NULL ctx. */
OSCAR_API size_t oscar_page_bytes(const oscar_ctx* ctx);

/* ---------------------------------------------------------------- calibrate(Q, S, V)
 * Accumulate the unnormalized covariance targets of §3 for this call's N tokens:
 *   acc[h][0] += Σ_n Σ_{i in G_h} q_{n,i}ᵀ q_{n,i}        (C_Q)
 *   acc[h][1] += Σ_n Σ_{i in G_h} sv_{n,i}ᵀ sv_{n,i}      (C_S = VᵀSᵀSV = (SV)ᵀ(SV))
 * Q, SV: bf16 [N][H_q][d] row-major (16-B aligned bases take the tcgen05 kernel, others the
 * CUDA-core one); SV is the per-query-head attention output S·V before
 * W_O (C_S depends on S and V only through SV).  Query head i belongs to KV head i / g.
 * acc: fp64 [H_kv][2][d][d], caller-zeroed before the first call; each call ADDS.
 * Multi-GPU: shard tokens, then all-reduce acc (SUM) across ranks before finalize.
 * N = 0 is a no-op; N < 0 or NULL pointers -> OSCAR_ERR_ARG. */
OSCAR_API oscar_status oscar_calib_accumulate(const oscar_ctx* ctx, const void* Q, const void* SV,
                                    int64_t N, double* acc, void* stream);

/* S·V on the device for the C_S target: SV = softmax(Q Kᵀ·scale + M) V per query
 * head (Alg. 1), M causal including the diagonal and block-diagonal
 * across the calibration sequences (reading Z16); query head i attends KV head i/g.  Computed by a
 * flash-attention forward on the tensor cores: variant 0 on tcgen05 (TMA tiles, S and O in TMEM;
 * needs 16-B aligned Q, K, V, otherwise the variant-1 kernel runs), variant 1 on mma.sync; both
 * bf16 operands with P rounded to bf16, fp32 softmax statistics and accumulation.
 * Q: bf16 [N][H_q][d]; K, V: bf16 [N][H_kv][d]; seq_starts: device int32 [n_seq], the first
 * token of each calibration sequence (seq_starts[0] = 0, strictly increasing, < N); SV: bf16
 * [N][H_q][d] (output; pass it to oscar_calib_accumulate as SV).  N = 0 is a no-op. */
OSCAR_API oscar_status oscar_calib_sv(const oscar_ctx* ctx, const void* Q, const void* K, const void* V,
                            const int32_t* seq_starts, int32_t n_seq, int64_t N, void* SV, void* stream);

/* Finalize n_mats (layer, kv-head) pairs: C = acc / n_rows (n_rows = N_total·g), eigen-
 * decompose with a one-CTA parallel cyclic Jacobi in fp64 (λ descending, ties by index,
 * each eigenvector sign-fixed so its largest-|entry| is positive; Alg. 1), and
 * compose R = U · H_Had · P_br with (x R)_j = (x U H)_{beta(j)} (Eq. 3).
 * acc: fp64 [n_mats][2][d][d]; R_K, R_V: fp32 [n_mats][d][d]; evals: fp64 [n_mats][2][d]
 * or NULL.  info: device int32 [n_mats][2] receiving the sweeps used (or -1 if the 100-
 * sweep cap was hit), or NULL.  If info is non-NULL this call synchronizes `stream` and
 * returns OSCAR_ERR_CONVERGENCE if any matrix did not converge (offline path only). */
OSCAR_API oscar_status oscar_calib_finalize(const oscar_ctx* ctx, const double* acc, int32_t n_mats,
                                  int64_t n_rows, float* R_K, float* R_V, double* evals,
                                  int32_t* info, void* stream);

/* CalibrateClip (Alg. 1; the procedure is unspecified in the paper — reading Z34 follows
 * SPEC S:L152-160): for each KV head h and each candidate ratio rho_g of `grid`, the frozen-error
 * surrogates of Theorem 1 of clip + quantize at rho_g,
 *   obj[h][0][g] = tr(R_K[h]ᵀ C_Q[h] R_K[h] · E_K),  E_K = Σ_j e_jᵀ e_j,
 *   e_j = dequant(quant(clip(k_j R_K[h], rho_g))) − k_j R_K[h]            (App A.5, ctx bits / G)
 * and obj[h][1][g] likewise for V with R_V and C_S.  K, V: bf16 [N][H_kv][d] calibration rows;
 * R_K, R_V: fp32 [H_kv][d][d]; acc: fp64 [H_kv][2][d][d] (C_Q, C_S sums of calib_accumulate;
 * the normalization does not change the argmin); grid: host float[n_grid], values in (0, 1],
 * 1 <= n_grid <= 16; obj: device fp64 [H_kv][2][n_grid] (overwritten).  The per-layer choice is
 * argmin_g Σ_h obj[h][side][g] (the sum in head order, ties to the earlier grid entry),
 * written by the library to choice: device int32 [2] = (index for rho_K, index for rho_V), or
 * NULL to skip the selection.  N = 0 -> obj = 0 (and choice = (0, 0)). */
OSCAR_API oscar_status oscar_calib_clip(const oscar_ctx* ctx, const void* K, const void* V, int64_t N,
                              const float* R_K, const float* R_V, const double* acc,
                              const float* grid, int32_t n_grid, double* obj, int32_t* choice,
                              void* stream);

/* ---------------------------------------------------------------- quantize_append(K, V)
 * For each of the T rows and each KV head h: x̃ = x·R_h (K with R_K, V with R_V), per-token
 * percentile clip (rho from the config), per-(token, group) min-max quantization to b-bit
 * codes with fp16 (s, m) metadata (reading Z4 operation order), bit-pack, and store into
 * the slot's page block (FORMAT above).
 * K, V: bf16 [T][H_kv][d]; slots: int64 [T] (page·P + offset); R_K, R_V: fp32 [H_kv][d][d];
 * pool: see oscar_page_bytes.  T = 0 is a no-op.  K and V row bases 16-B aligned take the
 * tensor-core kernel (TMA); other alignments are accepted and run the simple kernel.
 * R_V = NULL selects the pre-rotated-V mode ("absorb R_V into W_V"):
 * V rows are taken as already rotated (identity rotation); pass NULL to oscar_attend too. */
OSCAR_API oscar_status oscar_quantize_append(const oscar_ctx* ctx, const void* K, const void* V,
                                   const int64_t* slots, int64_t T, const float* R_K,
                                   const float* R_V, void* pool, void* stream);

/* ---------------------------------------------------------------- attend(q) -> o
 * Decode attention over the packed cache, in the rotated frame (north star; equal in exact
 * arithmetic to Alg. 1): q̃ = q·R_K[h]; ℓ_t = scale·q̃·k̂_t over the first
 * seq_lens[b] tokens of sequence b (unmasked, reading Z20); p = softmax(ℓ); õ = Σ p_t v̂_t;
 * o = õ·R_V[h]ᵀ.  Split-K over pages with an online-softmax merge.
 * q: bf16 [B][H_q][d]; page_table: int32 [B][max_pages]; seq_lens: int32 [B] (<= max_pages·P,
 * 0 => o = 0, lse = -inf); pool as written by oscar_quantize_append; workspace: device bytes
 * >= oscar_attend_workspace_bytes(ctx, B, max_pages), 256-B aligned (its sub-buffers are laid
 * out on 256-B boundaries; a base not 16-B aligned -> OSCAR_ERR_ARG); out: [B][H_q][d] bf16 (out_fp32 = 0)
 * or fp32 (out_fp32 = 1); lse: fp32 [B][H_q] natural-log sum-exp of ℓ, or NULL.
 * R_V = NULL (pre-rotated-V mode, NEXT-2): o = õ, returned in V's own (rotated) frame. */
OSCAR_API size_t oscar_attend_workspace_bytes(const oscar_ctx* ctx, int32_t B, int32_t max_pages);
OSCAR_API oscar_status oscar_attend(const oscar_ctx* ctx, const void* q, const int32_t* page_table,
                          const int32_t* seq_lens, int32_t B, int32_t max_pages,
                          const void* pool, const float* R_K, const float* R_V,
                          void* workspace, size_t workspace_bytes, void* out, int32_t out_fp32,
                          float* lse, void* stream);

/* One decode step of Alg. 1 `DecodeStep` on the packed cache: QuantizeAndWrite
 * of the step's new K and V rows (rotate by R_K / R_V, clip, min-max quantize,
 * pack) at position seq_lens[b] - 1 of sequence b — slot page_table[b][(L-1)/P]·P + (L-1)%P —
 * then attend(q) over the seq_lens[b] tokens, the new one included (reading Z20).  Same result
 * as oscar_quantize_append of those rows followed by oscar_attend; one fused prologue kernel
 * does the appends and the q rotation, and the attention kernel starts streaming the other
 * pages while it runs.  k_new, v_new: bf16 [B][H_kv][d].  seq_lens[b] = 0 appends nothing and
 * returns o = 0.  pool is written.  Other arguments as oscar_attend. */
OSCAR_API oscar_status oscar_decode_step(const oscar_ctx* ctx, const void* q, const void* k_new,
                               const void* v_new, const int32_t* page_table,
                               const int32_t* seq_lens, int32_t B, int32_t max_pages, void* pool,
                               const float* R_K, const float* R_V, void* workspace,
                               size_t workspace_bytes, void* out, int32_t out_fp32, float* lse,
                               void* stream);

/* attend over the mixed-precision cache (§4 "KV Cache Layout" P:L537-548: bf16 sink ‖ INT2
 * history ‖ bf16 recent window; Alg. 1 DecodeStep P:L1627-1635): the INT2 history is the first
 * seq_lens[b] tokens of page_table[b] in the pool (as oscar_attend), and the bf16 tokens (sink +
 * recent, RAW rows as appended, Alg. 1) are seg_k / seg_v: bf16
 * [B][H_kv][seg_cap][d], the first seg_lens[b] rows valid (their order is irrelevant).  A third
 * kernel computes the bf16 partial (original frame) and the same LSE merge combines it with the
 * INT2 partials.  1 <= seg_cap <= 1024.  Demotion of the oldest recent row is the
 * caller's oscar_quantize_append of that row.  Other arguments as oscar_attend. */
OSCAR_API oscar_status oscar_attend_mixed(const oscar_ctx* ctx, const void* q, const int32_t* page_table,
                                const int32_t* seq_lens, int32_t B, int32_t max_pages, const void* pool,
                                const float* R_K, const float* R_V, const void* seg_k, const void* seg_v,
                                const int32_t* seg_lens, int32_t seg_cap, void* workspace,
                                size_t workspace_bytes, void* out, int32_t out_fp32, float* lse,
                                void* stream);

/* ---------------------------------------------------------------- test hooks
 * Stage-isolated entry points used by the parity tests.  Each takes the kernel route that
 * oscar_quantize_append takes for the same T and context (variant 0: T <= 64 -> the decode-size
 * kernel, else the tcgen05 kernel when no clipping is configured; variant 1, clipping, or row
 * bases that are not 16-B aligned -> the simple CUDA-core kernel), so the stages checked are
 * those of the kernel that writes the pool.
 * oscar_rotate: Xrot[t][h][:] = X[t][h][:] · R[h] in fp32 (App A.5), exactly the
 *   rotated values that kernel's epilogue would quantize (tcgen05: the fp32 TMEM accumulator of
 *   [x x]·[R_hi; R_lo]).  X: bf16 [T][H_kv][d]; R: fp32 [H_kv][d][d]; Xrot: fp32 [T][H_kv][d].
 * oscar_quantize_rotated: clip + quantize + pack + store of already-rotated fp32 rows through
 *   that kernel's own epilogue (skips the rotation: "identical rotated inputs"); Krot, Vrot:
 *   fp32 [T][H_kv][d]. */
OSCAR_API oscar_status oscar_rotate(const oscar_ctx* ctx, const void* X, const float* R, float* Xrot,
                          int64_t T, void* stream);
OSCAR_API oscar_status oscar_quantize_rotated(const oscar_ctx* ctx, const float* Krot, const float* Vrot,
                                    const int64_t* slots, int64_t T, void* pool, void* stream);
/* oscar_rotate_fwht: the north star's second rotation form, measured against oscar_rotate
 * (DESIGN.md §7.2): Xrot = ((X · U[h]) · H_Had) · P_br with U the d×d matrix of sorted, sign-
 * normalized eigenvectors (R = U·H·P_br, Eq. 3; H Sylvester-ordered and normalized,
 * App A.1; out[j] = in[β(j)]) — a tcgen05 GEMM with U followed by a
 * Walsh–Hadamard transform in registers.  X: bf16 [T][H_kv][d], 16-B aligned; U: fp32
 * [H_kv][d][d]; Xrot: fp32 [T][H_kv][d].  OSCAR_ERR_UNSUPPORTED when the tensor-core append
 * path does not apply (clipping configured, misaligned rows). */
OSCAR_API oscar_status oscar_rotate_fwht(const oscar_ctx* ctx, const void* X, const float* U, float* Xrot,
                               int64_t T, void* stream);

/* Kernel variant selection for measurements: 0 = default (fastest), 1 =
 * the simple CUDA-core reference kernels.  Applies to quantize_append and attend. */
OSCAR_API oscar_status oscar_set_variant(oscar_ctx* ctx, int32_t variant);

#ifdef __cplusplus
}
#endif
#endif /* OSCAR_H_ */
