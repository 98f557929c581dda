// Parameters shared by the attend kernels (attend.cu, attend_mma.cu).
#pragma once
#include "common.cuh"

namespace oscar {

constexpr int kNewTok = 2 * 128 + 8;   // floats per (b, h) of the decode step's new-token record

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
  float* newtok;               // decode step: [B][H_kv][kNewTok] k̂, v̂, logits q̃·k̂ (g) of the
                               // new token (prologue -> merge)
  int32_t* nsplit;             // [B] split partials per (sequence, head) (prologue -> merge)
  int len_adj;                 // decode step: 1 (the partial kernels attend over seq_len - 1
                               // tokens; the merge kernel appends and folds the new token)
  unsigned long long* tl;      // timing probe builds only (-DOSCAR_PROBE_TL): per-CTA/warp
                               // %globaltimer marks; null otherwise
};

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
