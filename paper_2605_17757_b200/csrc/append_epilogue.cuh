// Clip + per-group min-max quantize + pack + store of one rotated row (App A.5, P:L1235-1311;
// Alg. 1 QuantizeAndWrite P:L1639-1643).  Operation order = reading Z4:
//   s = (mx - mn) / q_max [fp32 RN]; s16 = fp16_rn(s); m16 = fp16_rn(mn);
//   inv = s16 > 0 ? 1 / float(s16) : 0; dx = x - float(m16) [RN];
//   c = clamp(rint(dx·inv, product exact), 0, q_max).
#pragma once
#include "common.cuh"

namespace oscar {

struct EpiParams {
  int hkv, P, page_bytes, row_bytes, vcodes_off, meta_off, ng, G, bits;
  int clip_k_idx, clip_v_idx;
};

inline EpiParams make_epi_params(const oscar_ctx& c) {
  EpiParams e;
  e.hkv = c.hkv; e.P = c.P; e.page_bytes = c.page_bytes; e.row_bytes = c.row_bytes;
  e.vcodes_off = c.vcodes_off; e.meta_off = c.meta_off; e.ng = c.ng; e.G = c.G; e.bits = c.bits;
  e.clip_k_idx = c.clip_k_idx; e.clip_v_idx = c.clip_v_idx;
  return e;
}

// Quantize one group given its min / max; returns the codes of x[0..n) and the metadata.
__device__ __forceinline__ void minmax_params(float mn, float mx, float qmax, __half& s16,
                                              __half& m16, float& m, float& inv) {
  const float s = __fdiv_rn(__fsub_rn(mx, mn), qmax);
  s16 = __float2half_rn(s);
  m16 = __float2half_rn(mn);
  const float sf = __half2float(s16);
  m = __half2float(m16);
  inv = sf > 0.f ? __fdiv_rn(1.f, sf) : 0.f;
}

// reading Z4: c = clamp(rint(RN(x - m)·inv), 0, qmax) with the product exact: one FFMA with the
// 1.5·2^23 magic constant rounds the exact product to an integer (half-even); the clamp acts on
// the float bits (any |product| >= 2^22 lands outside [magic, magic + qmax] on the right side)
__device__ __forceinline__ int quant_code(float x, float m, float inv, int qmax) {
  const float tq = __fmaf_rn(__fsub_rn(x, m), inv, 12582912.f);
  return min(max(__float_as_int(tq), 0x4B400000), 0x4B400000 + qmax) - 0x4B400000;
}

// Nearest-rank clip threshold over a 128-value row held 4 per lane (reading Z6):
// tau = the value v with #{|x| < v} <= k < #{|x| <= v}.
__device__ __forceinline__ float warp_row_rank_select(const float a[4], int k) {
  int less[4] = {0, 0, 0, 0}, le[4] = {0, 0, 0, 0};
  for (int src = 0; src < 32; ++src) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float o = __shfl_sync(0xffffffffu, a[q], src);
#pragma unroll
      for (int i = 0; i < 4; ++i) { less[i] += (o < a[i]); le[i] += (o <= a[i]); }
    }
  }
  float tau = -1.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (less[i] <= k && k < le[i]) tau = a[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tau = fmaxf(tau, __shfl_xor_sync(0xffffffffu, tau, o));
  return tau;
}

// One warp owns one row: lane holds channels 4*lane .. 4*lane+3 in y[] (bits in {2, 3, 4}).
// deq (optional): the lane's 4 dequantized values s16·c + m16 (App A.5), fp32
__device__ __forceinline__ void quantize_store_row_warp(const EpiParams& ep, float y[4], int lane,
                                                        int64_t slot, int h, int isV,
                                                        uint8_t* __restrict__ pool, float* deq = nullptr) {
  const int cidx = isV ? ep.clip_v_idx : ep.clip_k_idx;
  if (cidx >= 0) {
    const float a[4] = {fabsf(y[0]), fabsf(y[1]), fabsf(y[2]), fabsf(y[3])};
    const float tau = warp_row_rank_select(a, cidx);
#pragma unroll
    for (int i = 0; i < 4; ++i) y[i] = fminf(fmaxf(y[i], -tau), tau);
  }
  float mn = fminf(fminf(y[0], y[1]), fminf(y[2], y[3]));
  float mx = fmaxf(fmaxf(y[0], y[1]), fmaxf(y[2], y[3]));
  const int lanes_per_group = ep.G / 4;
  for (int o = 1; o < lanes_per_group; o <<= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int qmax = (1 << ep.bits) - 1;
  __half s16, m16;
  float m, inv;
  minmax_params(mn, mx, (float)qmax, s16, m16, m, inv);
  int c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = quant_code(y[i], m, inv, qmax);
  if (deq) {
    const float sf = __half2float(s16);
#pragma unroll
    for (int i = 0; i < 4; ++i) deq[i] = fmaf(sf, (float)c[i], m);
  }

  if (!pool) return;                          // (dequantized values only)
  const int64_t page = slot / ep.P;
  const int off = (int)(slot % ep.P);
  uint8_t* blk = pool + (page * ep.hkv + h) * (int64_t)ep.page_bytes;
  const int rb = ep.row_bytes;
  if (ep.bits == 3) {
    // reading Z36 planes: low-plane byte `lane` = the 2-bit fields of code & 3; the high bits of
    // this lane's channels 4·lane + f (= 16j + 4i + f with j = lane / 4, i = lane % 4) form the
    // nibble (lane / 4) % 2 of high byte 4·(lane / 8) + lane % 4, shared with lane ^ 4
    const uint32_t lo = (uint32_t)(c[0] & 3) | ((uint32_t)(c[1] & 3) << 2) | ((uint32_t)(c[2] & 3) << 4) |
                        ((uint32_t)(c[3] & 3) << 6);
    const uint32_t nib = (uint32_t)(c[0] >> 2) | ((uint32_t)(c[1] >> 2) << 1) | ((uint32_t)(c[2] >> 2) << 2) |
                         ((uint32_t)(c[3] >> 2) << 3);
    const uint32_t other = __shfl_xor_sync(0xffffffffu, nib, 4);
    const int jh = 32 + 4 * (lane >> 3) + (lane & 3);
    const uint8_t hb = (uint8_t)(((lane >> 2) & 1) ? (other | (nib << 4)) : (nib | (other << 4)));
    if (!isV) {
      blk[fmt_krow(off) * rb + lane] = (uint8_t)lo;
      if (!((lane >> 2) & 1)) blk[fmt_krow(off) * rb + jh] = hb;
    } else {
      blk[ep.vcodes_off + fmt_vbyte(off, lane, rb)] = (uint8_t)lo;
      if (!((lane >> 2) & 1)) blk[ep.vcodes_off + fmt_vbyte(off, jh, rb)] = hb;
    }
  } else {
  // reading Z22 bitstream: this lane's 4 codes are bits [4·b·lane, 4·b·lane + 4b); byte j of the
  // row (bits 8j .. 8j+7) lies in the fields of lanes a = 8j/(4b) and a + 1
  const int fb = 4 * ep.bits;                // bits per lane field
  const uint32_t field = (uint32_t)c[0] | ((uint32_t)c[1] << ep.bits) | ((uint32_t)c[2] << (2 * ep.bits)) |
                         ((uint32_t)c[3] << (3 * ep.bits));
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int j = lane + 32 * m;             // byte index inside the row
    const int a = min((8 * j) / fb, 31);
    const uint32_t lo = __shfl_sync(0xffffffffu, field, a);
    const uint32_t hi = __shfl_sync(0xffffffffu, field, min(a + 1, 31));
    const uint32_t both = lo | (hi << fb);
    const uint8_t v = (uint8_t)(both >> (8 * j - fb * a));
    if (j < rb) {
      if (!isV) blk[fmt_krow(off) * rb + j] = v;
      else blk[ep.vcodes_off + fmt_vbyte(off, j, rb)] = v;
    }
  }
  }
  if ((lane % lanes_per_group) == 0) {
    const int grp = lane / lanes_per_group;
    const __half2 sm = __halves2half2(s16, m16);
    *reinterpret_cast<__half2*>(blk + ep.meta_off + fmt_meta(off, grp, ep.ng) + (isV ? 16 : 0)) = sm;
  }
}

}  // namespace oscar
