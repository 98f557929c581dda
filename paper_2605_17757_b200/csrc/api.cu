// C ABI of liboscar.so (include/oscar.h): validation, context, launches on the caller's stream.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <new>
#include <string>

#include "common.cuh"

namespace oscar {
cudaError_t launch_append_simple(const oscar_ctx& c, int mode, const void* K, const void* V,
                                 const float* Krot, const float* Vrot, const int64_t* slots,
                                 int64_t T, const float* RK, const float* RV, void* pool,
                                 float* rot_out, cudaStream_t s);
cudaError_t launch_append_tc(const oscar_ctx& c, int mode, const void* K, const void* V, const float* xin_k,
                             const float* xin_v, const int64_t* slots, int64_t T, const float* RK,
                             const float* RV, void* pool, float* rot_out, cudaStream_t s);
bool append_tc_supported(const oscar_ctx& c);
bool append_tc_aligned(const void* K, const void* V);
bool cov_tc_supported(const oscar_ctx& c);
bool append_small_ok(const oscar_ctx& c, int64_t T);
cudaError_t launch_append_small(const oscar_ctx& c, int mode, const void* K, const void* V, const float* xin_k,
                                const float* xin_v, const int64_t* slots, int64_t T, const float* RK,
                                const float* RV, void* pool, float* rot_out, cudaStream_t s);
cudaError_t launch_cov_accum_tc(const oscar_ctx& c, const void* Q, const void* SV, int64_t N, double* acc,
                                cudaStream_t s);
}  // namespace oscar

namespace {
thread_local std::string g_last_error;

oscar_status fail(oscar_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
oscar_status fail(oscar_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

oscar_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return OSCAR_OK;
  return fail(OSCAR_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Which quantize_append kernel serves a call (the test hooks oscar_rotate / oscar_quantize_rotated
// take the same route, so they isolate the stages of the kernel that produces the pool):
//   variant 0: T <= 64 -> append_small_kernel (decode-size latency path); else the tensor-core
//              append_tc_kernel when it applies (no clipping, 16-B aligned row bases);
//   otherwise (variant 1, clipping, misaligned rows): append_simple_kernel.
enum class AppendPath { kSmall, kTc, kSimple };
AppendPath append_path(const oscar_ctx& c, int64_t T, const void* X0, const void* X1) {
  if (c.variant != 0) return AppendPath::kSimple;
  if (oscar::append_small_ok(c, T)) return AppendPath::kSmall;
  if (oscar::append_tc_supported(c) && oscar::append_tc_aligned(X0, X1)) return AppendPath::kTc;
  return AppendPath::kSimple;
}

cudaError_t launch_append(const oscar_ctx& c, int mode, const void* K, const void* V, const float* xin_k,
                          const float* xin_v, const int64_t* slots, int64_t T, const float* RK,
                          const float* RV, void* pool, float* rot_out, cudaStream_t s) {
  const void* a = mode == 2 ? (const void*)xin_k : K;
  const void* b = mode == 2 ? (const void*)xin_v : V;
  switch (append_path(c, T, a, b)) {
    case AppendPath::kSmall:
      return oscar::launch_append_small(c, mode, K, V, xin_k, xin_v, slots, T, RK, RV, pool, rot_out, s);
    case AppendPath::kTc:
      return oscar::launch_append_tc(c, mode, K, V, xin_k, xin_v, slots, T, RK, RV, pool, rot_out, s);
    default:
      return oscar::launch_append_simple(c, mode, K, V, xin_k, xin_v, slots, T, RK, RV, pool, rot_out, s);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}  // namespace

extern "C" {

const char* oscar_last_error(void) { return g_last_error.c_str(); }
const char* oscar_version(void) { return "oscar-b200 0.1.0 (sm_100a)"; }

oscar_status oscar_create(const oscar_config* cfg, oscar_ctx** out) {
  if (!cfg || !out) return fail(OSCAR_ERR_ARG, "oscar_create: NULL argument");
  const oscar_config& c = *cfg;
  if (c.head_dim <= 0 || (c.head_dim & (c.head_dim - 1)))
    return fail(OSCAR_ERR_DIM, "head_dim %d is not a power of two", c.head_dim);
  if (c.head_dim != oscar::kD)
    return fail(OSCAR_ERR_UNSUPPORTED, "this build implements head_dim 128 only (got %d)", c.head_dim);
  if (c.num_q_heads <= 0 || c.num_kv_heads <= 0 || c.num_q_heads % c.num_kv_heads)
    return fail(OSCAR_ERR_ARG, "need H_q %% H_kv == 0 and both > 0 (got %d, %d)", c.num_q_heads,
                c.num_kv_heads);
  // any GQA ratio calibrates (num_kv_heads = 1 is NEXT-4's shared-rotation mode); attend
  // implements g <= 8 and checks it per call
  if (c.bits != 2 && c.bits != 3 && c.bits != 4)
    return fail(OSCAR_ERR_ARG, "bits must be 2, 3 or 4 (got %d)", c.bits);
  if (c.group_size != 32 && c.group_size != 64 && c.group_size != 128)
    return fail(OSCAR_ERR_ARG, "group_size must be 32, 64 or 128 (got %d)", c.group_size);
  const int P = c.page_size == 0 ? 64 : c.page_size;
  if (P < 16 || P > 256 || P % 16) return fail(OSCAR_ERR_ARG, "page_size must be a multiple of 16 in [16, 256] (got %d)", P);
  if (!(c.clip_ratio_k > 0.f && c.clip_ratio_k <= 1.f) || !(c.clip_ratio_v > 0.f && c.clip_ratio_v <= 1.f))
    return fail(OSCAR_ERR_ARG, "clip ratios must be in (0, 1]");
  if (c.softmax_scale < 0.f || !std::isfinite(c.softmax_scale))
    return fail(OSCAR_ERR_ARG, "softmax_scale must be >= 0 and finite");
  if (c.attend_pages_per_split < 0) return fail(OSCAR_ERR_ARG, "attend_pages_per_split must be >= 0");

  oscar_ctx* x = new (std::nothrow) oscar_ctx();
  if (!x) return fail(OSCAR_ERR_ARG, "out of host memory");
  x->cfg = c;
  x->d = c.head_dim; x->hq = c.num_q_heads; x->hkv = c.num_kv_heads; x->g = c.num_q_heads / c.num_kv_heads;
  x->bits = c.bits; x->G = c.group_size; x->P = P; x->ng = x->d / x->G;
  x->row_bytes = x->d * x->bits / 8;
  x->vcodes_off = P * x->row_bytes;
  x->meta_off = 2 * P * x->row_bytes;
  const int raw = 2 * P * x->row_bytes + P * x->ng * 8;
  x->page_bytes = (raw + 255) / 256 * 256;
  auto clip_idx = [&](float rho) {
    if (rho >= 1.f) return -1;
    return (int)std::ceil((double)rho * x->d) - 1;
  };
  x->clip_k_idx = clip_idx(c.clip_ratio_k);
  x->clip_v_idx = clip_idx(c.clip_ratio_v);
  x->scale = c.softmax_scale > 0.f ? c.softmax_scale : 1.f / std::sqrt((float)x->d);
  x->pages_per_split = c.attend_pages_per_split;
  x->variant = 0;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms = 148;
  cudaGetLastError();
  x->num_sms = sms > 0 ? sms : 148;
  *out = x;
  return OSCAR_OK;
}

void oscar_destroy(oscar_ctx* ctx) { delete ctx; }

size_t oscar_page_bytes(const oscar_ctx* ctx) { return ctx ? (size_t)ctx->page_bytes : 0; }

oscar_status oscar_set_variant(oscar_ctx* ctx, int32_t variant) {
  if (!ctx || variant < 0 || variant > 1) return fail(OSCAR_ERR_ARG, "oscar_set_variant: bad argument");
  ctx->variant = variant;
  return OSCAR_OK;
}

oscar_status oscar_calib_accumulate(const oscar_ctx* ctx, const void* Q, const void* SV,
                                    int64_t N, double* acc, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (N < 0) return fail(OSCAR_ERR_ARG, "N must be >= 0 (got %lld)", (long long)N);
  if (N == 0) return OSCAR_OK;
  if (!Q || !SV || !acc) return fail(OSCAR_ERR_ARG, "oscar_calib_accumulate: NULL pointer");
  if (ctx->variant == 0 && oscar::cov_tc_supported(*ctx) && aligned16(Q) && aligned16(SV))
    return cuda_status(oscar::launch_cov_accum_tc(*ctx, Q, SV, N, acc, as_stream(stream)), "cov_accum_tc");
  return cuda_status(oscar::launch_cov_accum(*ctx, Q, SV, N, acc, as_stream(stream)), "cov_accum");
}

oscar_status oscar_calib_sv(const oscar_ctx* ctx, const void* Q, const void* K, const void* V,
                            const int32_t* seq_starts, int32_t n_seq, int64_t N, void* SV, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (N < 0 || N > 0x7fffffffLL) return fail(OSCAR_ERR_ARG, "N must be in [0, 2^31) (got %lld)", (long long)N);
  if (N == 0) return OSCAR_OK;
  if (n_seq < 1) return fail(OSCAR_ERR_ARG, "n_seq must be >= 1");
  if (!Q || !K || !V || !seq_starts || !SV) return fail(OSCAR_ERR_ARG, "oscar_calib_sv: NULL pointer");
  if (ctx->variant == 0 && oscar::calib_sv_tc_supported(*ctx) && aligned16(Q) && aligned16(K) && aligned16(V))
    return cuda_status(oscar::launch_calib_sv_tc(*ctx, Q, K, V, seq_starts, n_seq, N, SV, as_stream(stream)),
                       "calib_sv_tc");
  return cuda_status(oscar::launch_calib_sv(*ctx, Q, K, V, seq_starts, n_seq, N, SV, as_stream(stream)), "calib_sv");
}

oscar_status oscar_calib_clip(const oscar_ctx* ctx, const void* K, const void* V, int64_t N,
                              const float* R_K, const float* R_V, const double* acc,
                              const float* grid, int32_t n_grid, double* obj, int32_t* choice,
                              void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (N < 0) return fail(OSCAR_ERR_ARG, "N must be >= 0 (got %lld)", (long long)N);
  if (!grid || n_grid < 1 || n_grid > oscar::kMaxClipGrid)
    return fail(OSCAR_ERR_ARG, "grid must hold 1..%d ratios", oscar::kMaxClipGrid);
  if (!obj) return fail(OSCAR_ERR_ARG, "oscar_calib_clip: NULL obj");
  int32_t kidx[oscar::kMaxClipGrid];
  for (int g = 0; g < n_grid; ++g) {
    if (!(grid[g] > 0.f && grid[g] <= 1.f)) return fail(OSCAR_ERR_ARG, "clip ratios must be in (0, 1]");
    kidx[g] = (int32_t)std::ceil((double)grid[g] * ctx->d) - 1;     // reading Z6 nearest rank
  }
  cudaStream_t s = as_stream(stream);
  oscar_status st;
  if (N == 0) {
    st = cuda_status(cudaMemsetAsync(obj, 0, sizeof(double) * ctx->hkv * 2 * n_grid, s), "calib_clip");
  } else {
    if (!K || !V || !R_K || !R_V || !acc) return fail(OSCAR_ERR_ARG, "oscar_calib_clip: NULL pointer");
    st = cuda_status(oscar::launch_calib_clip(*ctx, K, V, N, R_K, R_V, acc, kidx, n_grid, obj, s), "calib_clip");
  }
  if (st != OSCAR_OK || !choice) return st;
  return cuda_status(oscar::launch_clip_select(*ctx, obj, n_grid, choice, s), "calib_clip select");
}

oscar_status oscar_calib_finalize(const oscar_ctx* ctx, const double* acc, int32_t n_mats,
                                  int64_t n_rows, float* R_K, float* R_V, double* evals,
                                  int32_t* info, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (n_mats <= 0 || n_rows <= 0) return fail(OSCAR_ERR_ARG, "n_mats and n_rows must be > 0 (empty dump)");
  if (!acc || !R_K || !R_V) return fail(OSCAR_ERR_ARG, "oscar_calib_finalize: NULL pointer");
  cudaStream_t s = as_stream(stream);
  oscar_status st = cuda_status(
      oscar::launch_jacobi_compose(*ctx, acc, n_mats, 1.0 / (double)n_rows, R_K, R_V, evals, info, s),
      "jacobi_compose");
  if (st != OSCAR_OK || !info) return st;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "calib_finalize sync");
  const int n = 2 * n_mats;
  int32_t* h = new int32_t[n];
  e = cudaMemcpy(h, info, sizeof(int32_t) * n, cudaMemcpyDeviceToHost);
  int bad = -1;
  for (int i = 0; e == cudaSuccess && i < n; ++i)
    if (h[i] < 0) { bad = i; break; }
  delete[] h;
  if (e != cudaSuccess) return cuda_status(e, "calib_finalize info copy");
  if (bad >= 0) return fail(OSCAR_ERR_CONVERGENCE, "Jacobi did not converge for matrix %d", bad);
  return OSCAR_OK;
}

oscar_status oscar_quantize_append(const oscar_ctx* ctx, const void* K, const void* V,
                                   const int64_t* slots, int64_t T, const float* R_K,
                                   const float* R_V, void* pool, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (T < 0) return fail(OSCAR_ERR_ARG, "T must be >= 0");
  if (T == 0) return OSCAR_OK;
  if (!K || !V || !slots || !R_K || !pool) return fail(OSCAR_ERR_ARG, "oscar_quantize_append: NULL pointer");
  return cuda_status(launch_append(*ctx, 0, K, V, nullptr, nullptr, slots, T, R_K, R_V, pool, nullptr,
                                   as_stream(stream)), "quantize_append");
}

oscar_status oscar_rotate(const oscar_ctx* ctx, const void* X, const float* R, float* Xrot,
                          int64_t T, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (T < 0) return fail(OSCAR_ERR_ARG, "T must be >= 0");
  if (T == 0) return OSCAR_OK;
  if (!X || !R || !Xrot) return fail(OSCAR_ERR_ARG, "oscar_rotate: NULL pointer");
  // the K half of the kernel quantize_append would use, writing its fp32 rotated rows
  return cuda_status(launch_append(*ctx, 1, X, X, nullptr, nullptr, nullptr, T, R, R, nullptr, Xrot,
                                   as_stream(stream)), "rotate");
}

oscar_status oscar_rotate_fwht(const oscar_ctx* ctx, const void* X, const float* U, float* Xrot,
                               int64_t T, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (T < 0) return fail(OSCAR_ERR_ARG, "T must be >= 0");
  if (T == 0) return OSCAR_OK;
  if (!X || !U || !Xrot) return fail(OSCAR_ERR_ARG, "oscar_rotate_fwht: NULL pointer");
  if (!oscar::append_tc_supported(*ctx) || !aligned16(X))
    return fail(OSCAR_ERR_UNSUPPORTED, "oscar_rotate_fwht: needs the tensor-core append path (no clipping, "
                                       "16-B aligned rows)");
  return cuda_status(oscar::launch_append_tc(*ctx, 3, X, X, nullptr, nullptr, nullptr, T, U, U, nullptr, Xrot,
                                             as_stream(stream)), "rotate_fwht");
}

oscar_status oscar_quantize_rotated(const oscar_ctx* ctx, const float* Krot, const float* Vrot,
                                    const int64_t* slots, int64_t T, void* pool, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (T < 0) return fail(OSCAR_ERR_ARG, "T must be >= 0");
  if (T == 0) return OSCAR_OK;
  if (!Krot || !Vrot || !slots || !pool) return fail(OSCAR_ERR_ARG, "oscar_quantize_rotated: NULL pointer");
  return cuda_status(launch_append(*ctx, 2, nullptr, nullptr, Krot, Vrot, slots, T, nullptr, nullptr, pool,
                                   nullptr, as_stream(stream)), "quantize_rotated");
}

size_t oscar_attend_workspace_bytes(const oscar_ctx* ctx, int32_t B, int32_t max_pages) {
  if (!ctx || B <= 0 || max_pages <= 0) return 0;
  return oscar::attend_workspace_bytes(*ctx, B, max_pages);
}

oscar_status oscar_attend(const oscar_ctx* ctx, const void* q, const int32_t* page_table,
                          const int32_t* seq_lens, int32_t B, int32_t max_pages,
                          const void* pool, const float* R_K, const float* R_V,
                          void* workspace, size_t workspace_bytes, void* out, int32_t out_fp32,
                          float* lse, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (ctx->g > 8 || (ctx->g & (ctx->g - 1)))
    return fail(OSCAR_ERR_UNSUPPORTED, "attend: GQA ratio %d not in {1, 2, 4, 8}", ctx->g);
  if (B < 0 || max_pages < 0) return fail(OSCAR_ERR_ARG, "B and max_pages must be >= 0");
  if (B == 0) return OSCAR_OK;
  if (max_pages == 0) return fail(OSCAR_ERR_ARG, "max_pages must be > 0");
  if (!q || !page_table || !seq_lens || !pool || !R_K || !workspace || !out)
    return fail(OSCAR_ERR_ARG, "oscar_attend: NULL pointer");
  const size_t need = oscar::attend_workspace_bytes(*ctx, B, max_pages);
  if (workspace_bytes < need)
    return fail(OSCAR_ERR_ARG, "workspace too small: %zu < %zu", workspace_bytes, need);
  if (!aligned16(workspace)) return fail(OSCAR_ERR_ARG, "workspace must be 16-B (preferably 256-B) aligned");
  return cuda_status(oscar::launch_attend(*ctx, q, page_table, seq_lens, B, max_pages, pool, R_K, R_V,
                                          workspace, out, out_fp32, lse, as_stream(stream), nullptr,
                                          nullptr, nullptr, 0),
                     "attend");
}

oscar_status oscar_decode_step(const oscar_ctx* ctx, const void* q, const void* k_new, const void* v_new,
                               const int32_t* page_table, const int32_t* seq_lens, int32_t B,
                               int32_t max_pages, void* pool, const float* R_K, const float* R_V,
                               void* workspace, size_t workspace_bytes, void* out, int32_t out_fp32,
                               float* lse, void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (ctx->g > 8 || (ctx->g & (ctx->g - 1)))
    return fail(OSCAR_ERR_UNSUPPORTED, "attend: GQA ratio %d not in {1, 2, 4, 8}", ctx->g);
  if (B < 0 || max_pages < 0) return fail(OSCAR_ERR_ARG, "B and max_pages must be >= 0");
  if (B == 0) return OSCAR_OK;
  if (max_pages == 0) return fail(OSCAR_ERR_ARG, "max_pages must be > 0");
  if (!q || !k_new || !v_new || !page_table || !seq_lens || !pool || !R_K || !workspace || !out)
    return fail(OSCAR_ERR_ARG, "oscar_decode_step: NULL pointer");
  const size_t need = oscar::attend_workspace_bytes(*ctx, B, max_pages);
  if (workspace_bytes < need)
    return fail(OSCAR_ERR_ARG, "workspace too small: %zu < %zu", workspace_bytes, need);
  if (!aligned16(workspace)) return fail(OSCAR_ERR_ARG, "workspace must be 16-B (preferably 256-B) aligned");
  return cuda_status(oscar::launch_attend(*ctx, q, page_table, seq_lens, B, max_pages, pool, R_K, R_V,
                                          workspace, out, out_fp32, lse, as_stream(stream), nullptr,
                                          nullptr, nullptr, 0, k_new, v_new),
                     "decode_step");
}

oscar_status oscar_attend_mixed(const oscar_ctx* ctx, const void* q, const int32_t* page_table,
                                const int32_t* seq_lens, int32_t B, int32_t max_pages, const void* pool,
                                const float* R_K, const float* R_V, const void* seg_k, const void* seg_v,
                                const int32_t* seg_lens, int32_t seg_cap, void* workspace,
                                size_t workspace_bytes, void* out, int32_t out_fp32, float* lse,
                                void* stream) {
  if (!ctx) return fail(OSCAR_ERR_ARG, "NULL ctx");
  if (ctx->g > 8 || (ctx->g & (ctx->g - 1)))
    return fail(OSCAR_ERR_UNSUPPORTED, "attend: GQA ratio %d not in {1, 2, 4, 8}", ctx->g);
  if (B < 0 || max_pages < 0 || seg_cap < 0) return fail(OSCAR_ERR_ARG, "negative size");
  if (B == 0) return OSCAR_OK;
  if (max_pages == 0) return fail(OSCAR_ERR_ARG, "max_pages must be > 0");
  if (seg_cap == 0 || seg_cap > 1024)
    return fail(OSCAR_ERR_ARG, "seg_cap must be in [1, 1024] (got %d)", seg_cap);
  if (!q || !page_table || !seq_lens || !pool || !R_K || !workspace || !out || !seg_k || !seg_v ||
      !seg_lens)
    return fail(OSCAR_ERR_ARG, "oscar_attend_mixed: NULL pointer");
  const size_t need = oscar::attend_workspace_bytes(*ctx, B, max_pages);
  if (workspace_bytes < need)
    return fail(OSCAR_ERR_ARG, "workspace too small: %zu < %zu", workspace_bytes, need);
  if (!aligned16(workspace)) return fail(OSCAR_ERR_ARG, "workspace must be 16-B (preferably 256-B) aligned");
  return cuda_status(oscar::launch_attend(*ctx, q, page_table, seq_lens, B, max_pages, pool, R_K, R_V,
                                          workspace, out, out_fp32, lse, as_stream(stream), seg_k, seg_v,
                                          seg_lens, seg_cap),
                     "attend_mixed");
}

}  // extern "C"
