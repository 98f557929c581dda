// Parameters shared by the attend kernels (attend.cu, attend_mma.cu).
#pragma once
#include "common.cuh"

namespace oscar {

struct AttnParams {
  int hq, hkv, g, P, bits, G, ng;
  int row_bytes, vcodes_off, meta_off, page_bytes;
  int max_pages, pps, n_splits, batch;
  const int32_t* page_table;   // [B][max_pages]
  const int32_t* seq_lens;     // [B]
  const uint8_t* pool;
  float* qt;                   // [B][H_q][128] q̃ = q R_K scale log2e
  float* ws_o;                 // [B][H_q][n_splits][128] unnormalized partial õ
  float* ws_m;                 // [B][H_q][n_splits] running max (log2 domain)
  float* ws_l;                 // [B][H_q][n_splits] running sum
  int16_t* qint;               // [B][H_q][128] round(q̃ / qscale), |.| <= 32639 (IMMA path)
  float* qscale;               // [B][H_q] max|q̃| / 32639
  int32_t* qsum;               // [B][H_q][8] Σ_{c in group} qint
  uint32_t* qfrag;             // [B][H_kv][NT*16][32] IMMA A fragments (hi/lo int8 of qint)
  int32_t* work;               // work-item counter of the persistent partial kernel
  int nt;                      // ceil(g * ng / 8)
  int balanced;                // 1: tensor-core partial kernel's balanced decomposition (n_splits =
                               //    split slots per unit; the merge recomputes each unit's count)
  int n_warps, pmin;           // balanced: warps of the persistent grid, minimum pages per warp
  // optional bf16 segment (sink + recent window, NEXT-1): partial in the ORIGINAL frame
  float* seg_o;                // [B][H_q][128] unnormalized Σ p v (null: no segment)
  float* seg_m;                // [B][H_q]
  float* seg_l;                // [B][H_q]
  int len_adj;                 // decode step: 1 (the partial kernels attend over seq_len - 1
                               // tokens; the merge kernel appends and folds the new token)
  // rank-weighted decomposition of the tensor-core partial kernel (attend_mma.cu, RangeMap):
  // per_sm CTAs resident on each of num_sms SMs, cta_warps warps each; zone q (the CTAs that
  // arrived q-th on their SM) gets ranges weighted rwts[q]
  int num_sms, per_sm, cta_warps, rwts[4];
  unsigned long long* tl;      // timing probe builds only (-DOSCAR_PROBE_TL): per-CTA/warp
                               // %globaltimer marks; null otherwise
};

// Layout of the `work` area of the workspace (ints): [0] unused, [1] arrivals, [2] overflow
// count, [4 .. 64) bitmap of claimed virtual CTA slots (up to 1920).  Zeroed by the prologue
// kernel before every partial kernel.
__host__ __device__ __forceinline__ int work_ints(int) { return 64; }

// Ranges of the rank-weighted balanced decomposition.  Warp issue priority on an SM falls with
// the warp slot (measured, tools/timeline_probe.py: with equal ranges the CTAs in warp slots
// 0-3 / 4-7 / 8-11 / 12-15 of an SM streamed for 58.4 / 63.0 / 68.3 / 74.1 µs, per-SM totals
// equal), so the CTA in slots 4q..4q+3 takes a range of zone q, weighted w[q].  W ranges over T pages, per_zone ranges per zone; boundary(r) = ⌊S(r)·T / S(W)⌋ with S(r)
// the summed weight of ranges 0..r-1; rof(x) = the range holding page x.  Shared by the partial
// and the merge kernel so both see identical boundaries.
struct RangeMap {
  int64_t T, W;
  int per_zone;
  int w[4];
  __host__ __device__ __forceinline__ int64_t S(int64_t r) const {
    int64_t s = 0, b0 = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t b1 = q == 3 ? r : min(r, b0 + per_zone);
      if (b1 > b0) s += (b1 - b0) * w[q];
      b0 = b1 > b0 ? b1 : b0;
    }
    return s;
  }
  __host__ __device__ __forceinline__ int64_t boundary(int64_t r) const {
    return r >= W ? T : S(r) * T / S(W);
  }
  __host__ __device__ __forceinline__ int64_t rof(int64_t x) const {   // largest r < W: boundary(r) <= x
    int64_t l = 0, h = W;
    while (h - l > 1) {
      const int64_t m = (l + h) >> 1;
      if (boundary(m) <= x) l = m; else h = m;
    }
    return l;
  }
};
__host__ __device__ __forceinline__ RangeMap make_range_map(const AttnParams& p, int64_t T) {
  RangeMap m;
  m.T = T;
  m.W = min((int64_t)(p.n_warps / p.hkv), max((int64_t)1, T / p.pmin));
  m.per_zone = (p.num_sms * p.cta_warps + p.hkv - 1) / p.hkv;
  for (int q = 0; q < 4; ++q) m.w[q] = q < p.per_sm ? p.rwts[q] : p.rwts[p.per_sm - 1];
  return m;
}

// timeline probe (tools/timeline_probe.py): slot base of each kernel kind in the probe buffer
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int kind, int idx, int slot) {
#ifdef OSCAR_PROBE_TL
  if (tl) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tl[(size_t)kind * 32768 + (size_t)idx * 4 + slot] = t;
  }
#endif
}

bool attend_mma_supported(const oscar_ctx& c);
int attend_mma_total_warps(const oscar_ctx& c, int B);
int attend_mma_cta_warps();                   // warps per CTA of the partial kernel
cudaError_t launch_attend_mma(const AttnParams& p, cudaStream_t s);
bool attend_mma_tq(const oscar_ctx& c);      // the partial kernel uses the token-row QK layout

// IMMA QK k-slot -> channel map (see attend_mma.cu): in K-step kk (0..3), lane t's B
// registers hold channels 32t .. 32t+31 of the token row; slot = 4t + m (+16 for b1).
__host__ __device__ __forceinline__ int qk_channel(int bits, int kk, int slot) {
  const int t = (slot & 15) >> 2, m = slot & 3, hi = slot >> 4;
  if (bits == 2) return 32 * t + 16 * hi + 4 * m + kk;
  return 32 * t + 16 * hi + 8 * (kk >> 1) + 2 * m + (kk & 1);
}

}  // namespace oscar
