// Shared internals of liboscar.so (CUDA, sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "oscar.h"

struct oscar_ctx {
  oscar_config cfg;
  int d, hq, hkv, g, bits, G, P, ng;     // ng = d / G groups per row
  int row_bytes;                          // d * bits / 8
  int vcodes_off, meta_off, page_bytes;   // FORMAT offsets inside one (page, head) block
  int clip_k_idx, clip_v_idx;             // nearest-rank index ceil(rho*d)-1, or -1 = off
  float scale;                            // softmax scale (1/sqrt(d) by default)
  int pages_per_split;                    // 0 = auto
  int variant;                            // 0 = fastest, 1 = simple reference kernels
  int num_sms;
};

namespace oscar {

constexpr int kD = 128;                   // head_dim implemented by this build
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- launch declarations
// calib.cu
cudaError_t launch_cov_accum(const oscar_ctx& c, const void* Q, const void* SV, int64_t N,
                             double* acc, cudaStream_t s);
// calib_sv.cu (S·V for C_S on device, NEXT-3)
cudaError_t launch_calib_sv(const oscar_ctx& c, const void* Q, const void* K, const void* V,
                            const int32_t* starts, int n_seq, int64_t N, void* SV, cudaStream_t s);
// calib_sv_tc.cu (the same on tcgen05, variant 0)
bool calib_sv_tc_supported(const oscar_ctx& c);
cudaError_t launch_calib_sv_tc(const oscar_ctx& c, const void* Q, const void* K, const void* V,
                               const int32_t* starts, int n_seq, int64_t N, void* SV, cudaStream_t s);
// clip.cu (CalibrateClip surrogate objectives, reading Z34)
constexpr int kMaxClipGrid = 16;
cudaError_t launch_calib_clip(const oscar_ctx& c, const void* K, const void* V, int64_t N,
                              const float* RK, const float* RV, const double* acc,
                              const int32_t* kidx, int n_grid, double* obj, cudaStream_t s);
// CalibrateClip selection (reading Z34): choice[side] = argmin_g Σ_h obj[h][side][g]
cudaError_t launch_clip_select(const oscar_ctx& c, const double* obj, int n_grid, int32_t* choice,
                               cudaStream_t s);
cudaError_t launch_jacobi_compose(const oscar_ctx& c, const double* acc, int n_mats,
                                  double inv_rows, float* RK, float* RV, double* evals,
                                  int32_t* info, cudaStream_t s);
// attend.cu
size_t attend_workspace_bytes(const oscar_ctx& c, int B, int max_pages);
cudaError_t launch_attend(const oscar_ctx& c, const void* q, const int32_t* page_table,
                          const int32_t* seq_lens, int B, int max_pages, const void* pool,
                          const float* RK, const float* RV, void* ws, void* out, int out_fp32,
                          float* lse, cudaStream_t s, const void* seg_k, const void* seg_v,
                          const int32_t* seg_lens, int seg_cap, const void* k_new = nullptr,
                          const void* v_new = nullptr);

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// ---------------------------------------------------------------- packed page FORMAT
// (include/oscar.h).  Placement of rows / bytes inside one (page, head) block:
//   K row u        -> row position fmt_krow(u) (even tokens of each 16-token tile first)
//   V byte j of u  -> vcodes_off + fmt_vbyte(u, j, rb): a 32-bit word holds byte j of the 4
//                     tokens of a 4-token group; words are grouped in 16-byte chunks
//                     (chunk 32·(k/4) + 4·(j%8) + group-in-tile, k = j/8) so that the
//                     decode kernel's per-lane 16-byte loads are bank-conflict free
//   meta (u, grp)  -> meta_off + fmt_meta(u, grp, ng): fp16 (s_K, m_K) at +0 and (s_V, m_V)
//                     at +16 of a 32-B chunk [tile of 16][grp][group-in-tile]; the token in
//                     its 4-token group selects the 4-byte slot
__host__ __device__ __forceinline__ int fmt_krow(int u) {
  return 16 * (u >> 4) + 8 * (u & 1) + ((u & 15) >> 1);
}
// b = 3 (rb = 48, reading Z36: a 2-bit low plane ‖ a 1-bit high plane per row): the 32 low-plane
// bytes of a 16-token tile take the 2-bit layout (512 B), the 16 high-plane bytes e = 4m + i
// follow at 512 + 16·(4i + token group) + 4m + token-in-group
__host__ __device__ __forceinline__ int fmt_vbyte(int u, int j, int rb) {
  if (rb == 48 && j >= 32) {
    const int e = j - 32;
    return 16 * rb * (u >> 4) + 512 + 16 * (4 * (e & 3) + ((u >> 2) & 3)) + 4 * (e >> 2) + (u & 3);
  }
  const int k = j >> 3, lane = 4 * (j & 7) + ((u >> 2) & 3);
  const int word = 128 * (k >> 2) + 4 * lane + (k & 3);
  return 16 * rb * (u >> 4) + 4 * word + (u & 3);
}
// offset of the (s_K, m_K) pair; the (s_V, m_V) pair is at +16
__host__ __device__ __forceinline__ int fmt_meta(int u, int grp, int ng) {
  return 128 * ng * (u >> 4) + 128 * grp + 32 * ((u >> 2) & 3) + 4 * (u & 3);
}

}  // namespace oscar
