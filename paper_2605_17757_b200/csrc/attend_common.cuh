// Parameters shared by the attend kernels (attend.cu, attend_mma.cu).
#pragma once
#include "common.cuh"

namespace oscar {

struct AttnParams {
  int hq, hkv, g, P, bits, G, ng;
  int row_bytes, vcodes_off, meta_off, page_bytes;
  int max_pages, pps, n_splits;
  const int32_t* page_table;   // [B][max_pages]
  const int32_t* seq_lens;     // [B]
  const uint8_t* pool;
  float* qt;                   // [B][H_q][128] q̃ = q R_K scale log2e
  float* ws_o;                 // [B][H_q][n_splits][128] unnormalized partial õ
  float* ws_m;                 // [B][H_q][n_splits] running max (log2 domain)
  float* ws_l;                 // [B][H_q][n_splits] running sum
};

bool attend_mma_supported(const oscar_ctx& c);

}  // namespace oscar
