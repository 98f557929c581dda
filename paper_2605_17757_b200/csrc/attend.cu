// attend(q) -> o : decode attention over the packed paged cache (Alg. 1 DecodeStep attention
// P:L1632-1635, in the rotated frame of the north star; §4 "Decoding Attention Kernel"
// split-K partial kernel + online-softmax merge kernel).
//   q_rotate_kernel        q̃ = q · R_K[h] · scale · log2(e)   (fp32, workspace)
//   attend_partial_simple  variant 1: CUDA-core reference partial kernel (one CTA per
//                          (split, kv head, sequence)); the tensor-core kernel is in
//                          attend_mma.cu (variant 0)
//   attend_merge_kernel    LSE merge over splits, o = õ · R_Vᵀ, bf16/fp32 store, lse
#include "common.cuh"
#include "attend_common.cuh"

namespace oscar {

// ------------------------------------------------------------------ q rotation
// grid (B, H_kv); 128 threads: thread c computes column c of q̃ for the g heads of the group.
// Also emits the 15-bit integer form used by the IMMA QK path: qscale = max|q̃| / 32639,
// qint = rint(q̃ / qscale) (|qint| <= 32639 = 127·256 + 127, so hi/lo int8 never overflow),
// qsum[grp] = Σ_{c in grp} qint.
__global__ void __launch_bounds__(128) q_rotate_kernel(const uint16_t* __restrict__ q,
                                                       const float* __restrict__ RK, int Hq,
                                                       int g, int G, float qscale,
                                                       float* __restrict__ qt,
                                                       int16_t* __restrict__ qint,
                                                       float* __restrict__ qsc,
                                                       int32_t* __restrict__ qsum,
                                                       uint32_t* __restrict__ qfrag, int bits,
                                                       int nt, int32_t* __restrict__ work) {
  extern __shared__ __align__(16) float Rs[];            // R_K[h] staged: [128][128] fp32
  __shared__ float qs[8][kD];
  __shared__ float red[8][4];
  __shared__ int gsum[8][8];
  __shared__ int16_t qis[8][kD];
  const int b = blockIdx.x, h = blockIdx.y, c = threadIdx.x;
  const int warp = c >> 5, lane = c & 31;
  if (work && b == 0 && h == 0 && c == 0) *work = 0;     // reset the work-item counter
  {
    const float4* R4 = reinterpret_cast<const float4*>(RK + (size_t)h * kD * kD);
#pragma unroll 8
    for (int e = c; e < kD * kD / 4; e += 128) reinterpret_cast<float4*>(Rs)[e] = R4[e];
  }
  for (int i = 0; i < g; ++i) qs[i][c] = bf16_to_f32(q[((size_t)b * Hq + h * g + i) * kD + c]);
  if (c < 64) gsum[c >> 3][c & 7] = 0;
  __syncthreads();
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
  for (int k = 0; k < kD; ++k) {
    const float r = Rs[k * kD + c];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < g) acc[i] = fmaf(qs[i][k], r, acc[i]);
  }
  for (int i = 0; i < g; ++i) {
    acc[i] *= qscale;
    qt[((size_t)b * Hq + h * g + i) * kD + c] = acc[i];
    float m = fabsf(acc[i]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[i][warp] = m;
  }
  __syncthreads();
  for (int i = 0; i < g; ++i) {
    const float mx = fmaxf(fmaxf(red[i][0], red[i][1]), fmaxf(red[i][2], red[i][3]));
    const float s = mx > 0.f ? mx / 32639.f : 1.f;
    const int v = max(-32639, min(32639, __float2int_rn(acc[i] / s)));
    const size_t row = (size_t)b * Hq + h * g + i;
    qint[row * kD + c] = (int16_t)v;
    qis[i][c] = (int16_t)v;
    if (c == 0) qsc[row] = s;
    int ws = v;
    for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
    if (lane == 0) atomicAdd(&gsum[i][(c / G)], ws);   // G >= 32: a warp lies in one group
  }
  __syncthreads();
  if (c < g * 8) {
    const int i = c >> 3, grp = c & 7;
    qsum[((size_t)b * Hq + h * g + i) * 8 + grp] = gsum[i][grp];
  }
  // IMMA A fragments for attend_partial_mma: word (j, kk, r) of lane (gid, t) holds the
  // hi (r even) / lo (r odd) int8 of qint[head][channel] for combo 8j + gid = grp·g + head,
  // zero outside the combo's group (see attend_mma.cu)
  if (qfrag) {
    const int ng = kD / G, nc = g * ng;
    uint32_t* dst = qfrag + ((size_t)b * gridDim.y + h) * nt * 16 * 32;
    for (int w = c; w < nt * 16 * 32; w += 128) {
      const int ln = w & 31, rest = w >> 5;
      const int r = rest & 3, kk = (rest >> 2) & 3, j = rest >> 4;
      const int gid = ln >> 2, t = ln & 3, cb = 8 * j + gid;
      uint32_t v = 0;
      if (cb < nc) {
        const int grp = cb / g, hd = cb % g;
        for (int m = 0; m < 4; ++m) {
          const int ch = qk_channel(bits, kk, 4 * t + m + ((r & 2) ? 16 : 0));
          if (ch / G != grp) continue;
          const int qv = qis[hd][ch];
          const int hi8 = (qv + 128) >> 8;
          const int val = (r & 1) ? (qv - 256 * hi8) : hi8;
          v |= (uint32_t)(val & 0xff) << (8 * m);
        }
      }
      dst[w] = v;
    }
  }
}

// ------------------------------------------------------------------ simple partial kernel
// grid (n_splits, H_kv, B); 128 threads (thread c <-> channel c in PV).  Page-by-page:
// stage the (page, head) block in smem, scores for all (token, head) pairs, online softmax
// per head (log2 domain), PV accumulation in registers.
__global__ void __launch_bounds__(128) attend_partial_simple(AttnParams p) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  float* qs = reinterpret_cast<float*>(sm_raw);              // [g][128]
  float* qsum = qs + 8 * kD;                                  // [g][ng]
  float* sc = qsum + 8 * 8;                                   // [g][P]
  float* mrun = sc + 8 * p.P;                                 // [g]
  float* lrun = mrun + 8;                                     // [g]
  float* alpha = lrun + 8;                                    // [g]
  uint8_t* pg = reinterpret_cast<uint8_t*>(alpha + 8);        // page block
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  const int g = p.g, P = p.P;
  const int seq_len = p.seq_lens[b];
  const int page0 = split * p.pps;
  const int page1 = min(page0 + p.pps, (seq_len + P - 1) / P);

  for (int e = tid; e < g * kD; e += 128)
    qs[e] = p.qt[((size_t)b * p.hq + h * g) * kD + e];
  if (tid < 8) { mrun[tid] = -INFINITY; lrun[tid] = 0.f; }
  __syncthreads();
  if (tid < g * p.ng) {
    const int i = tid / p.ng, grp = tid % p.ng;
    float s = 0.f;
    for (int c = grp * p.G; c < (grp + 1) * p.G; ++c) s += qs[i * kD + c];
    qsum[i * 8 + grp] = s;
  }
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int qmax = (1 << p.bits) - 1;
  const int rb = p.row_bytes;

  for (int pi = page0; pi < page1; ++pi) {
    __syncthreads();
    const int64_t page = p.page_table[(size_t)b * p.max_pages + pi];
    const uint4* src = reinterpret_cast<const uint4*>(p.pool + (page * p.hkv + h) * (int64_t)p.page_bytes);
    for (int e = tid; e < p.page_bytes / 16; e += 128) reinterpret_cast<uint4*>(pg)[e] = src[e];
    __syncthreads();
    const int valid = min(P, seq_len - pi * P);
    const uint8_t* meta = pg + p.meta_off;
    // scores
    for (int e = tid; e < g * P; e += 128) {
      const int i = e / P, t = e % P;
      float s = -INFINITY;
      if (t < valid) {
        s = 0.f;
        const uint8_t* krow = pg + fmt_krow(t) * rb;
        for (int grp = 0; grp < p.ng; ++grp) {
          float dot = 0.f;
          for (int c = grp * p.G; c < (grp + 1) * p.G; ++c) {
            const int bit = c * p.bits;
            const int code = (krow[bit >> 3] >> (bit & 7)) & qmax;
            dot = fmaf(qs[i * kD + c], (float)code, dot);
          }
          const __half* mt = reinterpret_cast<const __half*>(meta + fmt_meta(t, grp, p.ng));
          s += __half2float(mt[0]) * dot + __half2float(mt[1]) * qsum[i * 8 + grp];
        }
      }
      sc[i * P + t] = s;
    }
    __syncthreads();
    // online softmax per head: warp w handles heads w, w+4
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int i = warp; i < g; i += 4) {
        float mx = -INFINITY;
        for (int t = lane; t < P; t += 32) mx = fmaxf(mx, sc[i * P + t]);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float mnew = fmaxf(mrun[i], mx);
        float sum = 0.f;
        for (int t = lane; t < P; t += 32) {
          const float pv = exp2f(sc[i * P + t] - mnew);
          sc[i * P + t] = pv;
          sum += pv;
        }
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();
        if (lane == 0) {
          const float a = exp2f(mrun[i] - mnew);
          alpha[i] = a;
          lrun[i] = lrun[i] * a + sum;
          mrun[i] = mnew;
        }
      }
    }
    __syncthreads();
    // PV: thread c accumulates channel c for all heads
    {
      const int c = tid;
      const int grp = c / p.G;
      const int bit = c * p.bits;
      const int jb = bit >> 3, sh = bit & 7;
      for (int i = 0; i < g; ++i) acc[i] *= alpha[i];
      for (int t = 0; t < valid; ++t) {
        const int code = (pg[p.vcodes_off + fmt_vbyte(t, jb, rb)] >> sh) & qmax;
        const __half* mt = reinterpret_cast<const __half*>(meta + fmt_meta(t, grp, p.ng) + 16);
        const float v = fmaf(__half2float(mt[0]), (float)code, __half2float(mt[1]));
        for (int i = 0; i < g; ++i) acc[i] = fmaf(sc[i * P + t], v, acc[i]);
      }
    }
  }
  __syncthreads();
  // partial outputs
  for (int i = 0; i < g; ++i) {
    const size_t row = ((size_t)b * p.hq + h * g + i) * p.n_splits + split;
    p.ws_o[row * kD + tid] = acc[i];
    if (tid == 0) { p.ws_m[row] = mrun[i]; p.ws_l[row] = lrun[i]; }
  }
}

// ------------------------------------------------------------------ merge
// grid (B·H_q); 128 threads; dynamic smem n_splits floats.  Combines the splits of one
// (sequence, q-head) row in the log2 domain (weights w_s = 2^(m_s - M)), then
// o = õ · R_V[h]ᵀ (warp w computes output channels w, w+4, ...; coalesced rows of R_V).
__global__ void __launch_bounds__(128) attend_merge_kernel(AttnParams p, const float* __restrict__ RV,
                                                           void* __restrict__ out, int out_fp32,
                                                           float* __restrict__ lse) {
  extern __shared__ float wsplit[];
  __shared__ __align__(16) float ot[kD];
  __shared__ float red[4];
  const int row = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = (row % p.hq) / p.g;
  const int ns = p.n_splits;
  const size_t row0 = (size_t)row * ns;
  float M = -INFINITY;
  for (int s = tid; s < ns; s += 128) M = fmaxf(M, p.ws_m[row0 + s]);
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  if (lane == 0) red[warp] = M;
  __syncthreads();
  M = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float L = 0.f;
  for (int s = tid; s < ns; s += 128) {
    const float w = M == -INFINITY ? 0.f : exp2f(p.ws_m[row0 + s] - M);   // 0 for empty splits
    wsplit[s] = w;
    L += p.ws_l[row0 + s] * w;
  }
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  if (lane == 0) red[warp] = L;
  __syncthreads();
  L = red[0] + red[1] + red[2] + red[3];
  float o = 0.f;
  const float* po = p.ws_o + row0 * kD + tid;
#pragma unroll 8
  for (int s = 0; s < ns; ++s) o = fmaf(po[(size_t)s * kD], wsplit[s], o);
  ot[tid] = (L > 0.f) ? o / L : 0.f;
  if (tid == 0 && lse) lse[row] = (L > 0.f) ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
  __syncthreads();
  const float* R = RV + (size_t)h * kD * kD;
  const float4 o4 = reinterpret_cast<const float4*>(ot)[lane];
#pragma unroll 4
  for (int c = warp; c < kD; c += 4) {
    const float4 r4 = reinterpret_cast<const float4*>(R + (size_t)c * kD)[lane];
    float v = r4.x * o4.x + r4.y * o4.y + r4.z * o4.z + r4.w * o4.w;
    for (int of = 16; of > 0; of >>= 1) v += __shfl_xor_sync(0xffffffffu, v, of);
    if (lane == 0) {
      const size_t idx = (size_t)row * kD + c;
      if (out_fp32) static_cast<float*>(out)[idx] = v;
      else static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
    }
  }
}

// ------------------------------------------------------------------ host side
// Pages per split (per work item).  Simple kernel: ~8 CTAs per SM over the grid.  Tensor-core
// kernel: warp-granular items, ~3 per warp of a nominal 16-warps/SM residency, 8..32 pages.
static int choose_pps(const oscar_ctx& c, int B, int max_pages) {
  if (c.pages_per_split > 0) return c.pages_per_split;
  const long units = (long)B * c.hkv;
  if (c.variant == 0 && attend_mma_supported(c)) {
    long pps = units * max_pages / (3L * c.num_sms * 16);
    pps = pps < 8 ? 8 : (pps > 32 ? 32 : pps);
    return (int)pps;
  }
  const long target = (long)c.num_sms * 8;
  long splits = (target + units - 1) / units;
  if (splits < 1) splits = 1;
  if (splits > max_pages) splits = max_pages;
  return (int)((max_pages + splits - 1) / splits);
}

size_t attend_workspace_bytes(const oscar_ctx& c, int B, int max_pages) {
  const int pps = choose_pps(c, B, max_pages);
  const size_t ns = (size_t)((max_pages + pps - 1) / pps);
  const size_t rows = (size_t)B * c.hq;
  const size_t nt = (size_t)((c.g * c.ng + 7) / 8);
  return rows * kD * 4 + rows * ns * (kD + 2) * 4 + rows * (kD * 2 + 4 + 32) +
         (size_t)B * c.hkv * nt * 16 * 32 * 4 + 1024;
}

int attend_mma_total_warps(const oscar_ctx& c);                              // attend_mma.cu
cudaError_t launch_attend_mma(const AttnParams& p, int total_warps, cudaStream_t s);

cudaError_t launch_attend(const oscar_ctx& c, const void* q, const int32_t* page_table,
                          const int32_t* seq_lens, int B, int max_pages, const void* pool,
                          const float* RK, const float* RV, void* ws, void* out, int out_fp32,
                          float* lse, cudaStream_t s) {
  const bool mma = c.variant == 0 && attend_mma_supported(c);
  AttnParams p{};
  p.hq = c.hq; p.hkv = c.hkv; p.g = c.g; p.P = c.P; p.bits = c.bits; p.G = c.G; p.ng = c.ng;
  p.row_bytes = c.row_bytes; p.vcodes_off = c.vcodes_off; p.meta_off = c.meta_off;
  p.page_bytes = c.page_bytes; p.max_pages = max_pages;
  p.pps = choose_pps(c, B, max_pages);
  p.n_splits = (max_pages + p.pps - 1) / p.pps;
  p.page_table = page_table; p.seq_lens = seq_lens;
  p.pool = static_cast<const uint8_t*>(pool);
  p.nt = (c.g * c.ng + 7) / 8;
  p.n_items = B * c.hkv * p.n_splits;
  p.batch = B;
  // workspace carve-up (attend_workspace_bytes)
  const size_t rows = (size_t)B * c.hq;
  p.qt = static_cast<float*>(ws);
  p.ws_o = p.qt + rows * kD;
  p.ws_m = p.ws_o + rows * p.n_splits * kD;
  p.ws_l = p.ws_m + rows * p.n_splits;
  p.qsum = reinterpret_cast<int32_t*>(p.ws_l + rows * p.n_splits);
  p.qscale = reinterpret_cast<float*>(p.qsum + rows * 8);
  p.qint = reinterpret_cast<int16_t*>(p.qscale + rows);
  p.qfrag = reinterpret_cast<uint32_t*>(p.qint + rows * kD);
  p.work = reinterpret_cast<int32_t*>(p.qfrag + (size_t)B * c.hkv * p.nt * 16 * 32);

  const int qsmem = kD * kD * 4;
  cudaError_t e = cudaFuncSetAttribute(q_rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, qsmem);
  if (e != cudaSuccess) return e;
  q_rotate_kernel<<<dim3(B, c.hkv), 128, qsmem, s>>>(static_cast<const uint16_t*>(q), RK, c.hq, c.g, c.G,
                                                     c.scale * kLog2e, p.qt, p.qint, p.qscale, p.qsum,
                                                     mma ? p.qfrag : nullptr, c.bits, p.nt,
                                                     mma ? p.work : nullptr);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (!mma) {
    const int smem = (8 * kD + 64 + 8 * c.P + 24) * 4 + c.page_bytes;
    e = cudaFuncSetAttribute(attend_partial_simple, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attend_partial_simple<<<dim3(p.n_splits, c.hkv, B), 128, smem, s>>>(p);
  } else {
    e = launch_attend_mma(p, attend_mma_total_warps(c), s);
    if (e != cudaSuccess) return e;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  attend_merge_kernel<<<(unsigned)(B * c.hq), 128, p.n_splits * 4, s>>>(p, RV, out, out_fp32, lse);
  return cudaGetLastError();
}

}  // namespace oscar
