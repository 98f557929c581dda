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
__global__ void __launch_bounds__(128) q_rotate_kernel(const uint16_t* __restrict__ q,
                                                       const float* __restrict__ RK, int Hq,
                                                       int g, float qscale,
                                                       float* __restrict__ qt) {
  __shared__ float qs[8][kD];
  const int b = blockIdx.x, h = blockIdx.y, c = threadIdx.x;
  for (int i = 0; i < g; ++i) qs[i][c] = bf16_to_f32(q[((size_t)b * Hq + h * g + i) * kD + c]);
  __syncthreads();
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const float* R = RK + (size_t)h * kD * kD;
  for (int k = 0; k < kD; ++k) {
    const float r = R[k * kD + c];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < g) acc[i] = fmaf(qs[i][k], r, acc[i]);
  }
  for (int i = 0; i < g; ++i) qt[((size_t)b * Hq + h * g + i) * kD + c] = acc[i] * qscale;
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
        const __half* mt = reinterpret_cast<const __half*>(meta + fmt_meta(t, grp, p.ng));
        const float v = fmaf(__half2float(mt[2]), (float)code, __half2float(mt[3]));
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
// grid (B, H_kv); 128 threads.  Combines the splits of the g heads of one KV group in the
// log2 domain, then o = õ · R_V[h]ᵀ (warp w computes output channels w, w+4, ...).
__global__ void __launch_bounds__(128) attend_merge_kernel(AttnParams p, const float* __restrict__ RV,
                                                           void* __restrict__ out, int out_fp32,
                                                           float* __restrict__ lse) {
  __shared__ __align__(16) float ot[8][kD];
  const int b = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const int g = p.g;
  for (int i = 0; i < g; ++i) {
    const size_t row0 = ((size_t)b * p.hq + h * g + i) * p.n_splits;
    float M = -INFINITY;
    for (int s = 0; s < p.n_splits; ++s) M = fmaxf(M, p.ws_m[row0 + s]);
    float L = 0.f, o = 0.f;
    if (M != -INFINITY) {
      for (int s = 0; s < p.n_splits; ++s) {
        const float w = exp2f(p.ws_m[row0 + s] - M);   // 0 for empty splits
        L += p.ws_l[row0 + s] * w;
        o += p.ws_o[(row0 + s) * kD + tid] * w;
      }
    }
    ot[i][tid] = (L > 0.f) ? o / L : 0.f;
    if (tid == 0 && lse) lse[(size_t)b * p.hq + h * g + i] = (L > 0.f) ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const float* R = RV + (size_t)h * kD * kD;
  for (int c = warp; c < kD; c += 4) {
    const float4 r4 = reinterpret_cast<const float4*>(R + (size_t)c * kD)[lane];
    for (int i = 0; i < g; ++i) {
      const float4 o4 = reinterpret_cast<const float4*>(&ot[i][0])[lane];
      float v = r4.x * o4.x + r4.y * o4.y + r4.z * o4.z + r4.w * o4.w;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) {
        const size_t idx = ((size_t)b * p.hq + h * g + i) * kD + c;
        if (out_fp32) static_cast<float*>(out)[idx] = v;
        else static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
      }
    }
  }
}

// ------------------------------------------------------------------ host side
static int choose_pps(const oscar_ctx& c, int B, int max_pages) {
  if (c.pages_per_split > 0) return c.pages_per_split;
  // aim for ~8 CTAs (of 4 warps) per SM in flight over the whole grid
  const long units = (long)B * c.hkv;
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
  return rows * kD * 4 + rows * ns * (kD + 2) * 4 + 256;
}

cudaError_t launch_attend_mma(const AttnParams& p, cudaStream_t s);  // attend_mma.cu

cudaError_t launch_attend(const oscar_ctx& c, const void* q, const int32_t* page_table,
                          const int32_t* seq_lens, int B, int max_pages, const void* pool,
                          const float* RK, const float* RV, void* ws, void* out, int out_fp32,
                          float* lse, cudaStream_t s) {
  AttnParams p{};
  p.hq = c.hq; p.hkv = c.hkv; p.g = c.g; p.P = c.P; p.bits = c.bits; p.G = c.G; p.ng = c.ng;
  p.row_bytes = c.row_bytes; p.vcodes_off = c.vcodes_off; p.meta_off = c.meta_off;
  p.page_bytes = c.page_bytes; p.max_pages = max_pages;
  p.pps = choose_pps(c, B, max_pages);
  p.n_splits = (max_pages + p.pps - 1) / p.pps;
  p.page_table = page_table; p.seq_lens = seq_lens;
  p.pool = static_cast<const uint8_t*>(pool);
  const size_t rows = (size_t)B * c.hq;
  p.qt = static_cast<float*>(ws);
  p.ws_o = p.qt + rows * kD;
  p.ws_m = p.ws_o + rows * p.n_splits * kD;
  p.ws_l = p.ws_m + rows * p.n_splits;

  q_rotate_kernel<<<dim3(B, c.hkv), 128, 0, s>>>(static_cast<const uint16_t*>(q), RK, c.hq, c.g,
                                                 c.scale * kLog2e, p.qt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (c.variant == 1 || !attend_mma_supported(c)) {
    const int smem = (8 * kD + 64 + 8 * c.P + 24) * 4 + c.page_bytes;
    e = cudaFuncSetAttribute(attend_partial_simple, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attend_partial_simple<<<dim3(p.n_splits, c.hkv, B), 128, smem, s>>>(p);
  } else {
    e = launch_attend_mma(p, s);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  attend_merge_kernel<<<dim3(B, c.hkv), 128, 0, s>>>(p, RV, out, out_fp32, lse);
  return cudaGetLastError();
}

}  // namespace oscar
