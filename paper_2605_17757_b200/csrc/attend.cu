// attend(q) -> o : decode attention over the packed paged cache (Alg. 1 DecodeStep attention
// P:L1632-1635, in the rotated frame of the north star; §4 "Decoding Attention Kernel"
// split-K partial kernel + online-softmax merge kernel).
//   attend_prologue_kernel q̃ = q · R_K[h] · scale · log2(e) (+ the decode step's append)
//   attend_partial_simple  variant 1: CUDA-core reference partial kernel (one CTA per
//                          (split, kv head, sequence)); the tensor-core kernel is in
//                          attend_mma.cu (variant 0)
//   attend_merge_kernel    LSE merge over splits, o = õ · R_Vᵀ, bf16/fp32 store, lse
#include <algorithm>
#include <type_traits>
#include "common.cuh"
#include "attend_common.cuh"
#include "append_epilogue.cuh"
#include "ptx.cuh"

#ifndef OSCAR_PDL_MERGE
#define OSCAR_PDL_MERGE 1
#endif

#ifndef OSCAR_CARVEOUT
#define OSCAR_CARVEOUT 1
#endif

namespace oscar {

// ------------------------------------------------------------------ prologue
// q rotation (B1): grid (B, H_kv), NW = 8 warps (16 for g = 8).  Rows rotated per CTA: the GQ
// query heads of group h by R_K[h] (staged in smem, see below).  Warp w owns the contraction slice
// of 128 / NW rows of R_K (lane l: columns 4l..4l+3) and forms partial dots for every row; the NW
// partials per (row, channel) are summed through smem.
// Then:
//   * warps 0..GQ-1: q̃ = q·R_K·scale·log₂e (fp32, kept for the simple kernel and for the decode
//     step's new-token logit) and the 15-bit integer form of the IMMA QK path: qscale = max|q̃| /
//     32639, qint = rint(q̃/qscale) (|qint| <= 32639 = 127·256 + 127, so the hi/lo int8 split
//     never overflows), qsum[grp] = Σ_{c in grp} qint; then all threads write the per-lane IMMA
//     operand fragments of the group.
// Decode step (oscar_decode_step; Alg. 1 DecodeStep P:L1627-1635, reading Z35): the step's new
// K / V rows ride along as two more rows of the same contraction (x̃_K = k·R_K, x̃_V = v·R_V), then
// warps GQ / GQ + 1 run QuantizeAndWrite of the K / V row (shared clip/min-max/pack
// epilogue, store at slot page_table[b][(L-1)/P]·P + (L-1)%P) and leave the DEQUANTIZED rows
// k̂, v̂ (exactly what the pool now holds) in the workspace (newtok); the merge kernel folds the
// new token in as one more partial (logit q̃·k̂, weight 1, value v̂).  Same result as appending
// first and attending over seq_len tokens.  The partial kernels attend over the first
// seq_len - 1 tokens only: the slot written here lies past every token they use (masked), so
// their early page prefetch may overlap this store.
// PDL: launched behind whatever precedes it on the stream; R_K[h] / R_V[h] are bulk-copied to smem
// before griddepcontrol.wait (rotations are never produced by a kernel that triggers its dependents
// early — none of this library's kernels that do write them, and a kernel without the trigger
// completes before this one launches), q, the new rows and the page table after it.  It then
// lets the partial kernel launch at once; the partial kernel's early page prefetch only reads
// pool pages.
struct PrologueParams {
  const uint16_t* q;            // [B][H_q][128] bf16
  const float* RK;              // [H_kv][128][128]
  int Hq, lgG, bits, nt;
  float qscale;                 // softmax scale · log2(e)
  float* qt;
  int16_t* qint;
  float* qsc;
  int32_t* qsum;
  uint32_t* qfrag;              // null: simple kernel path
  int tq;                       // 1: fragments for the token-row QK layout of attend_partial_mma
  int32_t* work;                // null: simple kernel path
  const uint16_t* knew;         // decode step: [B][H_kv][128] bf16 new K / V rows (null: attend)
  const uint16_t* vnew;
  const float* RV;              // [H_kv][128][128]; null: pre-rotated V (identity)
  float* newtok;                // decode step: [B][H_kv][kNewTok] fp32 k̂, v̂, logits q̃·k̂ (g)
  int32_t* nsplit;              // [B] split partials per (sequence, head) of the balanced
                                // decomposition (attend_mma.cu Decomp), for the merge kernel
  int balanced, n_warps, pmin, len_adj, P, batch;
  const int32_t* page_table;    // decode step: slot of the new row
  const int32_t* seq_lens;
  int max_pages;
  uint8_t* pool;
  EpiParams ep;
  unsigned long long* tl;       // timing probe (OSCAR_PROBE_TL)
};

// warps of the prologue: 8 (16 for g = 8: g q-row warps + the K and V row warps), so that two
// partial-kernel CTAs fit beside it on an SM (64 registers per thread, 16 K per CTA)
template <int GQ>
constexpr int kProWarps = GQ + 2 <= 8 ? 8 : 16;
// 8 warps: <= 64 registers (two partial CTAs beside the prologue CTA); 16 warps (g = 8): one
// partial CTA fits either way, so the register cap is left at 128 (no spills)
#ifndef OSCAR_PRO16_MINB
#define OSCAR_PRO16_MINB 1
#endif
template <int GQ>
constexpr int kProMinBlocks = kProWarps<GQ> == 8 ? 4 : OSCAR_PRO16_MINB;

template <int GQ>
__global__ void __launch_bounds__(kProWarps<GQ> * 32, kProMinBlocks<GQ>)
attend_prologue_kernel(PrologueParams pp) {
  constexpr int NR = GQ + 2;                         // q heads, then the decode step's K and V rows
  constexpr int NW = kProWarps<GQ>, NT = NW * 32, KW = kD / NW;   // warps, threads, R rows per warp
  // dynamic smem: R_K[h] (64 KB) then R_V[h] (64 KB, decode step), bulk-copied before the wait;
  // the [16][NR][128] partial dots reuse it once every warp has finished its dots
  extern __shared__ __align__(128) float psm[];
  float* Rks = psm;
  float* Rvs = psm + kD * kD;
  float* ps = psm;
  __shared__ __align__(16) float xs[NR][kD];         // input rows (fp32)
  __shared__ __align__(16) float ys[NR][kD];         // rotated rows
  __shared__ int16_t qis[GQ][kD];
  __shared__ __align__(8) uint64_t rbar;
  const int b = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const int w = tid >> 5, lane = tid & 31;
  const bool step = pp.knew != nullptr;
  const bool rotv = step && pp.RV != nullptr;
  if (threadIdx.x == 0) tl_mark(pp.tl, 0, blockIdx.y * gridDim.x + blockIdx.x, 0);
  // R_K[h] (and R_V[h] for the decode step's V row) into smem: issued before the wait
  if (tid == 0) {
    constexpr uint32_t bytes = kD * kD * 4;
    ptx::mbar_init(&rbar, 1);
    ptx::mbar_init_fence();
#ifdef OSCAR_PROBE_NOR
    ptx::mbar_arrive(&rbar);                         // timing probe only: R not loaded (results invalid)
    if (false)
#else
    ptx::mbar_expect_tx(&rbar, rotv ? 2 * bytes : bytes);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(ptx::su32(Rks)), "l"(pp.RK + (size_t)h * kD * kD), "r"(bytes), "r"(ptx::su32(&rbar)) : "memory");
    if (rotv)
#endif
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(ptx::su32(Rvs)), "l"(pp.RV + (size_t)h * kD * kD), "r"(bytes), "r"(ptx::su32(&rbar)) : "memory");
  }
  // launched with PDL behind whatever precedes it on the stream: wait for it before reading q and
  // the new rows (they may be its outputs), then let the partial kernel launch
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (threadIdx.x == 0) tl_mark(pp.tl, 0, blockIdx.y * gridDim.x + blockIdx.x, 1);
  const int G = 1 << pp.lgG;
  if (pp.work && b == 0 && h == 0 && tid == 0) *pp.work = 0;   // reset the work-item counter
  // balanced decomposition: split count of sequence b (warp 15, CTA h = 0; loads overlapping the
  // rotation), the same formula as the partial kernel's Decomp::rof
  if (pp.balanced && h == 0 && w == NW - 1) {
    int lt = 0, tot = 0;
    for (int bb = lane; bb < pp.batch; bb += 32) {
      const int n = (max(pp.seq_lens[bb] - pp.len_adj, 0) + pp.P - 1) / pp.P;
      tot += n;
      lt += bb < b ? n : 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
      lt += __shfl_xor_sync(0xffffffffu, lt, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if (lane == 0) {
      const int npg = (max(pp.seq_lens[b] - pp.len_adj, 0) + pp.P - 1) / pp.P;
      const int64_t T = tot;
      const int64_t W = min((int64_t)(pp.n_warps / gridDim.y), max((int64_t)1, T / pp.pmin));
      auto rof = [&](int64_t x) { return ((x + 1) * W - 1) / T; };
      pp.nsplit[b] = npg > 0 ? (int)(rof(lt + npg - 1) - rof(lt) + 1) : 0;
    }
  }
  // decode step: the new row's slot (warps GQ, GQ + 1), its loads overlapping the rotation
  // (the length is loaded beside the rows; the dependent page-table load is issued after the
  // rows have arrived, so its latency overlaps the contraction instead of delaying the barrier)
  int Lstep = 0;
  int64_t slot = 0;
  if (step && (w == GQ || w == GQ + 1)) Lstep = pp.seq_lens[b];
#ifdef OSCAR_PROBE_NOPRO
  return;                                            // timing probe only (results invalid)
#endif
  const int nrow = step ? NR : GQ;
  for (int e = tid; e < nrow * (kD / 4); e += NT) {
    const int r = e >> 5, l4 = e & 31;
    const uint16_t* src = r < GQ ? pp.q + ((size_t)b * pp.Hq + (size_t)h * GQ + r) * kD
                                 : (r == GQ ? pp.knew : pp.vnew) + ((size_t)b * gridDim.y + h) * kD;
    const uint2 u = reinterpret_cast<const uint2*>(src)[l4];
    reinterpret_cast<float4*>(xs[r])[l4] =
        make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                    __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
  }
  __syncthreads();
  if (step && (w == GQ || w == GQ + 1) && Lstep > 0) {
    const int pos = Lstep - 1;
    slot = (int64_t)pp.page_table[(size_t)b * pp.max_pages + pos / pp.ep.P] * pp.ep.P + pos % pp.ep.P;
  }
  ptx::mbar_wait(&rbar, 0);                          // R_K (R_V) resident
  // warp w contracts rows KW·w .. KW·w + KW - 1 of R (lane: columns 4l..4l+3)
  float4 acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    const float4 mk = reinterpret_cast<const float4*>(Rks + (size_t)(KW * w + i) * kD)[lane];
#pragma unroll
    for (int r = 0; r < GQ + 1; ++r) {
      if (r == GQ && !step) break;
      const float x = xs[r][KW * w + i];
      acc[r].x = fmaf(x, mk.x, acc[r].x); acc[r].y = fmaf(x, mk.y, acc[r].y);
      acc[r].z = fmaf(x, mk.z, acc[r].z); acc[r].w = fmaf(x, mk.w, acc[r].w);
    }
    if (rotv) {
      const float4 mv = reinterpret_cast<const float4*>(Rvs + (size_t)(KW * w + i) * kD)[lane];
      const float x = xs[GQ + 1][KW * w + i];
      acc[GQ + 1].x = fmaf(x, mv.x, acc[GQ + 1].x); acc[GQ + 1].y = fmaf(x, mv.y, acc[GQ + 1].y);
      acc[GQ + 1].z = fmaf(x, mv.z, acc[GQ + 1].z); acc[GQ + 1].w = fmaf(x, mv.w, acc[GQ + 1].w);
    }
  }
  __syncthreads();                                   // every warp is done with R: ps reuses it
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (r >= GQ && !step) break;
    if (r == GQ + 1 && !rotv) break;
    reinterpret_cast<float4*>(ps + ((size_t)w * NR + r) * kD)[lane] = acc[r];
  }
  __syncthreads();
  for (int e = tid; e < nrow * kD; e += NT) {
    const int r = e >> 7, c = e & (kD - 1);
    float y = 0.f;
    if (r == GQ + 1 && !rotv) {
      y = xs[r][c];                                  // pre-rotated V (NEXT-2): identity
    } else {
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) y += ps[((size_t)ww * NR + r) * kD + c];
    }
    ys[r][c] = y;
  }
  __syncthreads();
  if (threadIdx.x == 0) tl_mark(pp.tl, 0, blockIdx.y * gridDim.x + blockIdx.x, 3);
  if (step && (w == GQ || w == GQ + 1)) {
    // QuantizeAndWrite of the new K (warp GQ) / V (warp GQ + 1) row; its dequantized row k̂ / v̂
    // goes to newtok for the merge kernel.  These two warps are done after this: the rest of
    // the CTA synchronises without them (named barrier 1), so this chain overlaps the q path.
    const int isV = w - GQ;
    if (Lstep > 0) {
      const float4 y4 = reinterpret_cast<const float4*>(ys[GQ + isV])[lane];
      float yy[4] = {y4.x, y4.y, y4.z, y4.w}, dq[4];
      quantize_store_row_warp(pp.ep, yy, lane, slot, h, isV, pp.pool, dq);
      float* nt = pp.newtok + ((size_t)b * gridDim.y + h) * kNewTok;
      reinterpret_cast<float4*>(nt + isV * kD)[lane] = make_float4(dq[0], dq[1], dq[2], dq[3]);
      if (!isV) {
        // the new token's logit (log2 units) per head: q̃·k̂ with q̃ = ys·scale·log₂e as stored
        // in qt below
#pragma unroll
        for (int r = 0; r < GQ; ++r) {
          const float4 qv = reinterpret_cast<const float4*>(ys[r])[lane];
          float d = (qv.x * pp.qscale) * dq[0] + (qv.y * pp.qscale) * dq[1] + (qv.z * pp.qscale) * dq[2] +
                    (qv.w * pp.qscale) * dq[3];
          for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (lane == 0) nt[2 * kD + r] = d;
        }
      }
    }
    return;
  }
  if (w < GQ) {
    const size_t row = (size_t)b * pp.Hq + (size_t)h * GQ + w;
    float4 a = reinterpret_cast<const float4*>(ys[w])[lane];
    a.x *= pp.qscale; a.y *= pp.qscale; a.z *= pp.qscale; a.w *= pp.qscale;
    reinterpret_cast<float4*>(pp.qt + row * kD)[lane] = a;
    float mx = fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w)));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float s = mx > 0.f ? mx / 32639.f : 1.f;
    const float is = mx > 0.f ? 32639.f / mx : 1.f;   // one division; the clamp absorbs rounding
    const int v0 = max(-32639, min(32639, __float2int_rn(a.x * is)));
    const int v1 = max(-32639, min(32639, __float2int_rn(a.y * is)));
    const int v2 = max(-32639, min(32639, __float2int_rn(a.z * is)));
    const int v3 = max(-32639, min(32639, __float2int_rn(a.w * is)));
    const uint2 pk = make_uint2((uint32_t)(v0 & 0xffff) | ((uint32_t)v1 << 16),
                                (uint32_t)(v2 & 0xffff) | ((uint32_t)v3 << 16));
    reinterpret_cast<uint2*>(pp.qint + row * kD)[lane] = pk;
    reinterpret_cast<uint2*>(qis[w])[lane] = pk;
    if (lane == 0) pp.qsc[row] = s;
    int gs = v0 + v1 + v2 + v3;                    // lanes of one group: G/4 consecutive lanes
    for (int o = 1; o < (G >> 2); o <<= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
    if ((lane & ((G >> 2) - 1)) == 0) pp.qsum[row * 8 + (lane * 4 >> pp.lgG)] = gs;
  }
  if (step) asm volatile("bar.sync 1, %0;\n" ::"r"(NT - 64) : "memory");   // all but warps GQ, GQ + 1
  else __syncthreads();
  // the fragment writers: every thread still running, renumbered 0 .. nft - 1
  const int ft = step && w > GQ + 1 ? tid - 64 : tid, nft = step ? NT - 64 : NT;
  // IMMA A fragments for attend_partial_mma: word (j, kk, r) of lane (gid, t) holds the
  // hi (r even) / lo (r odd) int8 of qint[head][channel] for combo 8j + gid = grp·g + head,
  // zero outside the combo's group (see attend_mma.cu)
  if (pp.qfrag && pp.tq) {
    // token-row QK layout (attend_mma.cu, TQ): B-fragment word (jt, kk, r) of lane (gid, t)
    // holds, for column gid = (head 4·jt + gid/2, hi|lo = gid&1), the int8 of qint at the
    // k-slots 4t + i + 16r (i = 0..3) <-> channel 16·j + 4·i + 2(kk&1) + r, j = t or 4 + t
    // for kk < 2 or >= 2
    constexpr int NTQ = (GQ + 3) / 4;
    uint32_t* dst = pp.qfrag + ((size_t)b * gridDim.y + h) * NTQ * 8 * 32;
    for (int wd = ft; wd < NTQ * 8 * 32; wd += nft) {
      const int ln = wd & 31, rest = wd >> 5;
      const int r = rest & 1, kk = (rest >> 1) & 3, jt = rest >> 3;
      const int gid = ln >> 2, t = ln & 3;
      const int hd = 4 * jt + (gid >> 1), lo = gid & 1;
      uint32_t v = 0;
      if (hd < GQ) {
        // G = 32: k-slot 4t + i + 16r of k-step kk <-> field t of byte i of word 2kk + r
        const bool g32 = pp.lgG == 5;
        const int j = g32 ? 2 * kk + r : ((kk >> 1) ? 4 + t : t);
        const int sft = g32 ? t : 2 * (kk & 1) + r;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int qv = qis[hd][16 * j + 4 * i + sft];
          const int hi8 = (qv + 128) >> 8;
          const int val = lo ? (qv - 256 * hi8) : hi8;
          v |= (uint32_t)(val & 0xff) << (8 * i);
        }
      }
      dst[wd] = v;
    }
  } else if (pp.qfrag) {
    const int nc = GQ << (7 - pp.lgG);
    uint32_t* dst = pp.qfrag + ((size_t)b * gridDim.y + h) * pp.nt * 16 * 32;
    for (int wd = ft; wd < pp.nt * 16 * 32; wd += nft) {
      const int ln = wd & 31, rest = wd >> 5;
      const int r = rest & 3, kk = (rest >> 2) & 3, j = rest >> 4;
      const int gid = ln >> 2, t = ln & 3, cb = 8 * j + gid;
      uint32_t v = 0;
      if (cb < nc) {
        const int grp = cb / GQ, hd = cb - grp * GQ;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int ch = qk_channel(pp.bits, kk, 4 * t + m + ((r & 2) ? 16 : 0));
          if ((ch >> pp.lgG) != grp) continue;
          const int qv = qis[hd][ch];
          const int hi8 = (qv + 128) >> 8;
          const int val = (r & 1) ? (qv - 256 * hi8) : hi8;
          v |= (uint32_t)(val & 0xff) << (8 * m);
        }
      }
      dst[wd] = v;
    }
  }
  if (ft == 0) tl_mark(pp.tl, 0, blockIdx.y * gridDim.x + blockIdx.x, 2);
}

// ------------------------------------------------------------------ simple partial kernel
// grid (n_splits, H_kv, B); 128 threads (thread c <-> channel c in PV).  Page-by-page:
// stage the (page, head) block in smem, scores for all (token, head) pairs, online softmax
// per head (log2 domain), PV accumulation in registers.
// The K row is read as 32-bit words: channels 32j..32j+31 are the BITS words BITS·j.. of the
// row (little-endian bit stream, codes straddling words taken with a funnel shift); one
// 32-channel chunk never crosses a quantization group (G ∈ {32, 64, 128}).  PV reads the V
// codes of a 4-token group with one 32-bit load per byte column (fmt_vbyte interleaving).
template <int BITS, int GQ>
__global__ void __launch_bounds__(128) attend_partial_simple(AttnParams p) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  float* qs = reinterpret_cast<float*>(sm_raw);              // [g][128]
  float* qsum = qs + 8 * kD;                                  // [g][ng]
  float* sc = qsum + 8 * 8;                                   // [P][g]
  float* mrun = sc + 8 * p.P;                                 // [g]
  float* lrun = mrun + 8;                                     // [g]
  float* alpha = lrun + 8;                                    // [g]
  uint8_t* pg = reinterpret_cast<uint8_t*>(alpha + 8);        // page block
  float2* vmf = reinterpret_cast<float2*>(pg + ((p.page_bytes + 15) & ~15));   // [P][ng]
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  constexpr int g = GQ;
  const int P = p.P;
  const int seq_len = max(p.seq_lens[b] - p.len_adj, 0);
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
  float acc[GQ];
#pragma unroll
  for (int i = 0; i < GQ; ++i) acc[i] = 0.f;
  const int qmax = (1 << p.bits) - 1;
  const int rb = p.row_bytes;
  const int ns = 128 % P == 0 ? min(128 / P, g) : 0;

  for (int pi = page0; pi < page1; ++pi) {
    __syncthreads();
    const int64_t page = p.page_table[(size_t)b * p.max_pages + pi];
    const uint4* src = reinterpret_cast<const uint4*>(p.pool + (page * p.hkv + h) * (int64_t)p.page_bytes);
    for (int e = tid; e < p.page_bytes / 16; e += 128) reinterpret_cast<uint4*>(pg)[e] = src[e];
    __syncthreads();
    const int valid = min(P, seq_len - pi * P);
    const uint8_t* meta = pg + p.meta_off;
    // (s_V, m_V) of every (token, group) as float2, read by the PV loop (one LDS.64 per token)
    for (int e = tid; e < valid * p.ng; e += 128) {
      const int t = e / p.ng, grp = e - t * p.ng;
      const __half2 h2 = *reinterpret_cast<const __half2*>(meta + fmt_meta(t, grp, p.ng) + 16);
      vmf[e] = __half22float2(h2);
    }
    // scores: thread -> token t and heads i0, i0 + ns, ... (the code unpack is shared by
    // the heads); ns = 128 / P thread slices when P divides 128, else one (t, head) pair each
    auto score_token = [&](auto NHc, int t, int i0, int istep) {
      constexpr int nh = decltype(NHc)::value;
      if (t >= valid) {
#pragma unroll
        for (int k = 0; k < nh; ++k) sc[t * GQ + i0 + k * istep] = -INFINITY;
        return;
      }
      const uint32_t* kw = reinterpret_cast<const uint32_t*>(pg + fmt_krow(t) * rb);
      float s[nh], dot[nh];
#pragma unroll
      for (int k = 0; k < nh; ++k) { s[k] = 0.f; dot[k] = 0.f; }
#pragma unroll
      for (int j = 0; j < kD / 32; ++j) {
        // channels 32j .. 32j+31: b in {2, 4}: the BITS words BITS·j.. of the bitstream; b = 3
        // (reading Z36): low-plane words 2j, 2j+1 and high-plane word 8 + j (channel
        // 32j + 4·k4 + r: high bit at bit 8·(k4 % 4) + 4·(k4 / 4) + r)
        constexpr int NW = BITS == 3 ? 3 : BITS;
        uint32_t w[NW + 1];
        if (BITS == 3) {
          w[0] = kw[2 * j]; w[1] = kw[2 * j + 1]; w[2] = kw[8 + j];
        } else {
#pragma unroll
          for (int u = 0; u < NW; ++u) w[u] = kw[BITS * j + u];
        }
        w[NW] = 0u;
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          float4 qv[nh];
#pragma unroll
          for (int k = 0; k < nh; ++k)
            qv[k] = reinterpret_cast<const float4*>(qs + (i0 + k * istep) * kD)[8 * j + k4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            uint32_t v;
            if (BITS == 3) {
              const uint32_t lo2 = (w[k4 >> 2] >> (2 * (4 * (k4 & 3) + r))) & 3u;
              const uint32_t hi1 = (w[2] >> (8 * (k4 & 3) + 4 * (k4 >> 2) + r)) & 1u;
              v = lo2 | (hi1 << 2);
            } else {
              const int bit = BITS * (4 * k4 + r), wi = bit >> 5, sh = bit & 31;
              v = sh + BITS <= 32 ? (w[wi] >> sh) : __funnelshift_r(w[wi], w[wi + 1], sh);
            }
            const float cf = (float)(v & ((1u << BITS) - 1u));
#pragma unroll
            for (int k = 0; k < nh; ++k)
              dot[k] = fmaf(r == 0 ? qv[k].x : r == 1 ? qv[k].y : r == 2 ? qv[k].z : qv[k].w, cf, dot[k]);
          }
        }
        if ((32 * (j + 1)) % p.G == 0) {
          const int grp = (32 * j) / p.G;
          const __half* mt = reinterpret_cast<const __half*>(meta + fmt_meta(t, grp, p.ng));
          const float sK = __half2float(mt[0]), mK = __half2float(mt[1]);
#pragma unroll
          for (int k = 0; k < nh; ++k) {
            s[k] += sK * dot[k] + mK * qsum[(i0 + k * istep) * 8 + grp]; dot[k] = 0.f; }
        }
      }
#pragma unroll
      for (int k = 0; k < nh; ++k) sc[t * GQ + i0 + k * istep] = s[k];
    };
    using I1 = std::integral_constant<int, 1>;
    if (ns > 0 && tid / P < ns) {
      const int nh = g / ns;
      if constexpr (g >= 8) { if (nh == 8) score_token(std::integral_constant<int, 8>{}, tid % P, tid / P, ns); }
      if constexpr (g >= 4) { if (nh == 4) score_token(std::integral_constant<int, 4>{}, tid % P, tid / P, ns); }
      if constexpr (g >= 2) { if (nh == 2) score_token(std::integral_constant<int, 2>{}, tid % P, tid / P, ns); }
      if (nh == 1) score_token(I1{}, tid % P, tid / P, ns);
    } else if (ns == 0) {
      for (int e = tid; e < g * P; e += 128) score_token(I1{}, e % P, e / P, 1);
    }
    __syncthreads();
    // online softmax per head: warp w handles heads w, w+4
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int i = warp; i < g; i += 4) {
        float mx = -INFINITY;
        for (int t = lane; t < P; t += 32) mx = fmaxf(mx, sc[t * GQ + i]);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float mnew = fmaxf(mrun[i], mx);
        float sum = 0.f;
        for (int t = lane; t < P; t += 32) {
          const float pv = exp2f(sc[t * GQ + i] - mnew);
          sc[t * GQ + i] = pv;
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
      // the code's byte(s): b in {2, 4} one byte at bit sh; b = 3 (reading Z36) the low-plane
      // byte c/4 at bit 2(c%4) and the high-plane byte 32 + 4(j/2) + i (c = 16j + 4i + f) at bit
      // 4(j%2) + f, gathered by one PRMT as bits 0-7 / 8-15
      const int bit = BITS == 3 ? 2 * c : c * p.bits;
      const int jb = bit >> 3, sh = bit & 7;
      const int jh = 32 + 4 * ((c >> 4) >> 1) + ((c >> 2) & 3), shh = 8 + 4 * ((c >> 4) & 1) + (c & 3);
#pragma unroll
      for (int i = 0; i < g; ++i) acc[i] *= alpha[i];
      for (int t4 = 0; t4 < valid; t4 += 4) {
        const uint32_t w0 = *reinterpret_cast<const uint32_t*>(pg + p.vcodes_off + fmt_vbyte(t4, jb, rb));
        const uint32_t w1 = BITS == 3 ? *reinterpret_cast<const uint32_t*>(pg + p.vcodes_off + fmt_vbyte(t4, jh, rb))
                          : (sh + BITS > 8
                             ? *reinterpret_cast<const uint32_t*>(pg + p.vcodes_off + fmt_vbyte(t4, jb + 1, rb)) : 0u);
        auto pv_tok = [&](int u) {
          const int t = t4 + u;
          const uint32_t word = __byte_perm(w0, w1, u | ((4 + u) << 4));   // byte u of w0, w1
          const int code = BITS == 3 ? (int)(((word >> sh) & 3u) | (((word >> shh) & 1u) << 2))
                                     : (int)((word >> sh) & (uint32_t)qmax);
          const float2 sm = vmf[t * p.ng + grp];
          const float v = fmaf(sm.x, (float)code, sm.y);
#pragma unroll
          for (int i = 0; i < g; ++i) acc[i] = fmaf(sc[t * GQ + i], v, acc[i]);
        };
        if (t4 + 4 <= valid) {
#pragma unroll
          for (int u = 0; u < 4; ++u) pv_tok(u);
        } else {
          for (int u = 0; u < valid - t4; ++u) pv_tok(u);
        }
      }
    }
  }
  __syncthreads();
  // partial outputs
#pragma unroll
  for (int i = 0; i < g; ++i) {
    const size_t row = ((size_t)b * p.hq + h * g + i) * p.n_splits + split;
    p.ws_o[row * kD + tid] = acc[i];
    if (tid == 0) { p.ws_m[row] = mrun[i]; p.ws_l[row] = lrun[i]; }
  }
}

// ------------------------------------------------------------------ merge
// LSE merge of the split-K partials + un-rotation o = õ·R_Vᵀ (reading Z21).
// grid (B, H_kv, g / HC), 256 threads (8 warps): one CTA per (sequence, KV head) and HC query
// heads of its group — HC = g normally (the heads share one copy of R_V[h]), HC = 1 for small
// batches (more CTAs, more warps per head's splits).  Launched with PDL: the tensor-core partial
// kernel triggers it right after its own wait (the prologue is complete), so its CTAs become
// resident as partial CTAs retire; before griddepcontrol.wait it touches only the caller's inputs
// and the prologue's outputs: R_V[h] (64 KB) bulk-copied into smem, the split count, the decode
// step's new-token logit and v̂.  Then warp w serves head w mod g, splits s ≡ w / g (mod 8/g):
// each lane loads batches of 4 splits, two batches in flight (partial row float4 = channels
// 4l..4l+3, split max and sum) and folds them with a running max;
// the 8/g warps of a head and the NEXT-1 segment are combined through smem.  Un-rotation:
// thread (c', half) forms output channel c' of every other head from smem, the contraction index
// rotated by lane % 8 (c = 4·((k + lane mod 8) mod 32)): conflict-free R_V rows, broadcast õ.
//
// Decode step (Alg. 1 DecodeStep; reading Z35): the prologue has stored the step's
// new K/V row (QuantizeAndWrite) and left its dequantized rows k̂, v̂ in the workspace (newtok);
// this kernel folds the new token in as one more partial: logit q̃·k̂, weight 1, value v̂.
namespace {
__device__ __forceinline__ uint32_t msmem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
}  // namespace

struct StepParams {
  int step;                     // 1: decode step (the prologue appended the new row)
  const int32_t* seq_lens;
};

template <int HC>
#ifndef OSCAR_MERGE_MINB
#define OSCAR_MERGE_MINB 1
#endif
__global__ void __launch_bounds__(256, OSCAR_MERGE_MINB) attend_merge_kernel(AttnParams p, const float* __restrict__ RV,
                                                           void* __restrict__ out, int out_fp32,
                                                           float* __restrict__ lse, StepParams sp) {
#ifdef OSCAR_PROBE_NOMERGE
  return;                                            // timing probe only (results invalid)
#endif
  constexpr int WPH = 8 / HC;                        // warps per query head
#ifndef OSCAR_MERGE_NB
#define OSCAR_MERGE_NB 4      // same-box A/B (C2 decode step): 2 79.9, 4 79.8, 6 81.5, 8 81.0, 16 81.5 us
#endif
  constexpr int NB = OSCAR_MERGE_NB;                 // splits per load batch (two in flight) per warp
  constexpr int HPT = (HC + 1) / 2;                  // heads per thread in the un-rotation
  extern __shared__ __align__(128) float Rs[];       // [128][128] R_V[h]
  __shared__ __align__(16) float po[8][kD];
  __shared__ __align__(16) float ot[HC][kD];
  __shared__ __align__(16) float vhat[kD];           // decode step: v̂ of the new token
  __shared__ float pm[8], pl[8], sws[HC], nlog[HC];
  __shared__ __align__(8) uint64_t bar;
  const int b = blockIdx.x, h = blockIdx.y, tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int hz = blockIdx.z * HC;                    // first query head (within the group) of this CTA
  const int tl_idx = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (tid == 0) tl_mark(p.tl, 2, tl_idx, 0);
  // the next call's prologue may become resident now: it waits for this grid's completion
  // before touching anything
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (RV && tid == 0) {
    const uint32_t bb = msmem_u32(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bb), "r"(kD * kD * 4) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     msmem_u32(Rs)),
                 "l"(RV + (size_t)h * kD * kD), "r"(kD * kD * 4), "r"(bb)
                 : "memory");
  }
  auto wait_rv = [&]() {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_R%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra WAIT_R%=;\n}\n" ::"r"(msmem_u32(&bar))
        : "memory");
  };
  // ---- decode step: the new token's partial — logit q̃·k̂ (log2 units) per head, value v̂; k̂, v̂
  // from the prologue (newtok)
  const int Lnew = sp.step ? sp.seq_lens[b] : 0;
  if (Lnew > 0) {
    const float* nt = p.newtok + ((size_t)b * p.hkv + h) * kNewTok;
    if (tid < kD / 4) reinterpret_cast<float4*>(vhat)[tid] = __ldcg(reinterpret_cast<const float4*>(nt + kD) + tid);
    if (tid >= 64 && tid < 64 + HC) nlog[tid - 64] = __ldcg(nt + 2 * kD + hz + tid - 64);
  }
  // split partials of this unit: all n_splits slots (simple kernel), or the count of warps whose
  // range covers the unit under the balanced decomposition (from the prologue)
  __shared__ int ns_s;
  if (tid == 96) ns_s = p.balanced ? __ldcg(p.nsplit + b) : p.n_splits;
  __syncthreads();
  const int ns = ns_s;
  if (tid == 0) tl_mark(p.tl, 2, tl_idx, 1);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (tid == 0) tl_mark(p.tl, 2, tl_idx, 2);
  {
    const int hd = w % HC, part = w / HC;
    const size_t rbh = (size_t)b * p.hq + (size_t)h * p.g + hz + hd;
    auto prow = [&](int s) -> size_t { return rbh * p.n_splits + s; };
    float mw = -INFINITY, Lw = 0.f;
    float4 ow = make_float4(0.f, 0.f, 0.f, 0.f);
    // software-pipelined fold: the loads of the next batch of NB splits are in flight while
    // the current batch is folded (running max; empty splits have m = -inf and weight 0)
    auto load = [&](int s0, float4 (&x)[NB], float (&ms)[NB], float (&ls)[NB]) {
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const int s = s0 + k * WPH;
        const bool ok = s < ns;
        const size_t r = ok ? prow(s) : 0;
        x[k] = ok ? __ldcg(reinterpret_cast<const float4*>(p.ws_o + r * kD) + lane)
                  : make_float4(0.f, 0.f, 0.f, 0.f);
        ms[k] = ok ? __ldcg(p.ws_m + r) : -INFINITY;
        ls[k] = ok ? __ldcg(p.ws_l + r) : 0.f;
      }
    };
    auto fold = [&](float4 (&x)[NB], float (&ms)[NB], float (&ls)[NB]) {
      float nm = mw;
#pragma unroll
      for (int k = 0; k < NB; ++k) nm = fmaxf(nm, ms[k]);
      const float alpha = mw == nm ? 1.f : exp2f(mw - nm);      // 0 from -inf
      ow.x *= alpha; ow.y *= alpha; ow.z *= alpha; ow.w *= alpha;
      Lw *= alpha;
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const float wt = ms[k] == -INFINITY ? 0.f : exp2f(ms[k] - nm);   // 0 for empty splits
        ow.x = fmaf(x[k].x, wt, ow.x); ow.y = fmaf(x[k].y, wt, ow.y);
        ow.z = fmaf(x[k].z, wt, ow.z); ow.w = fmaf(x[k].w, wt, ow.w);
        Lw = fmaf(ls[k], wt, Lw);
      }
      mw = nm;
    };
    float4 xa[NB], xb[NB];
    float ma[NB], mb[NB], la[NB], lb[NB];
    constexpr int STEP = WPH * NB;
    load(part, xa, ma, la);
    for (int s0 = part; s0 < ns; s0 += 2 * STEP) {
      if (s0 + STEP < ns) load(s0 + STEP, xb, mb, lb);
      fold(xa, ma, la);
      if (s0 + STEP >= ns) break;
      if (s0 + 2 * STEP < ns) load(s0 + 2 * STEP, xa, ma, la);
      fold(xb, mb, lb);
    }
    __syncthreads();                                 // (decode step) po was scratch above
    reinterpret_cast<float4*>(po[w])[lane] = ow;
    if (lane == 0) { pm[w] = mw; pl[w] = Lw; }
  }
  __syncthreads();
  const bool seg = p.seg_o != nullptr;
  for (int e = tid; e < HC * kD; e += 256) {
    const int hd = e >> 7, c = e & (kD - 1);
    const size_t row = (size_t)b * p.hq + (size_t)h * p.g + hz + hd;
    const float mnew = Lnew > 0 ? nlog[hd] : -INFINITY;
    float M = fmaxf(seg ? p.seg_m[row] : -INFINITY, mnew);
#pragma unroll
    for (int j = 0; j < WPH; ++j) M = fmaxf(M, pm[hd + HC * j]);
    float L = 0.f, o = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int j = 0; j < WPH; ++j) {
        const float wj = exp2f(pm[hd + HC * j] - M);
        L = fmaf(pl[hd + HC * j], wj, L);
        o = fmaf(po[hd + HC * j][c], wj, o);
      }
      if (Lnew > 0) {                                // the step's new token: weight 1, value v̂
        const float wn = exp2f(mnew - M);
        L += wn;
        o = fmaf(vhat[c], wn, o);
      }
    }
    const float wseg = (seg && M != -INFINITY) ? exp2f(p.seg_m[row] - M) : 0.f;
    if (seg) L = fmaf(p.seg_l[row], wseg, L);
    const float inv = L > 0.f ? 1.f / L : 0.f;
    ot[hd][c] = o * inv;
    if (c == 0) {
      sws[hd] = wseg * inv;
      if (lse) lse[row] = L > 0.f ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
    }
  }
  __syncthreads();
  const int cp = tid & (kD - 1), hh = tid >> 7;
  float acc[HPT];
  if (RV) {
    wait_rv();
#pragma unroll
    for (int j = 0; j < HPT; ++j) acc[j] = 0.f;
    const float4* Rrow = reinterpret_cast<const float4*>(Rs + (size_t)cp * kD);
#pragma unroll 8
    for (int k = 0; k < kD / 4; ++k) {
      // contraction chunk rotated by lane % 8: the 8 chunk positions cover the 32 banks, so the
      // R_V row reads are conflict-free (4 wavefronts per warp, the minimum for 512 B) and the
      // õ reads touch 8 distinct chunks (1 wavefront, broadcast)
      const int c4 = (k + (lane & 7)) & 31;
      const float4 r = Rrow[c4];
#pragma unroll
      for (int j = 0; j < HPT; ++j) {
        const int hd = hh + 2 * j;
        if (hd < HC) {
          const float4 x = reinterpret_cast<const float4*>(ot[hd])[c4];
          acc[j] = fmaf(r.x, x.x, fmaf(r.y, x.y, fmaf(r.z, x.z, fmaf(r.w, x.w, acc[j]))));
        }
      }
    }
  } else {                                           // pre-rotated V (NEXT-2): o = õ
#pragma unroll
    for (int j = 0; j < HPT; ++j) acc[j] = hh + 2 * j < HC ? ot[hh + 2 * j][cp] : 0.f;
  }
#pragma unroll
  for (int j = 0; j < HPT; ++j) {
    const int hd = hh + 2 * j;
    if (hd >= HC) continue;
    const size_t row = (size_t)b * p.hq + (size_t)h * p.g + hz + hd;
    float v = acc[j];
    if (seg) v = fmaf(p.seg_o[row * kD + cp], sws[hd], v);
    const size_t idx = row * kD + cp;
    if (out_fp32) static_cast<float*>(out)[idx] = v;
    else static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
  }
  if (tid == 0) tl_mark(p.tl, 2, tl_idx, 3);
}

// ------------------------------------------------------------------ bf16 segment (NEXT-1)
// grid (B, H_kv); one warp per query head.  Attention partial over the raw bf16 rows of the
// sink + recent segment (§4, "an additional kernel for BF16 KV cache
// attention"): scores q·k·scale·log2e in fp32 (lane = token), max / sum by warp shuffles,
// p staged in smem, then Σ p v with lane = 4 channels.  Output in the ORIGINAL frame.

__global__ void __launch_bounds__(256) attend_segment_kernel(AttnParams p, const uint16_t* __restrict__ q,
                                                             const uint16_t* __restrict__ sk,
                                                             const uint16_t* __restrict__ sv,
                                                             const int32_t* __restrict__ seg_lens,
                                                             int seg_cap, float qscale) {
  extern __shared__ __align__(16) float ssm[];
  const int b = blockIdx.x, h = blockIdx.y, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* qs = ssm + w * (kD + seg_cap);
  float* pr = qs + kD;
  const size_t row = (size_t)b * p.hq + (size_t)h * p.g + w;
  {
    const uint2 u = reinterpret_cast<const uint2*>(q + row * kD)[lane];
    qs[4 * lane + 0] = __uint_as_float(u.x << 16) * qscale;
    qs[4 * lane + 1] = __uint_as_float(u.x & 0xffff0000u) * qscale;
    qs[4 * lane + 2] = __uint_as_float(u.y << 16) * qscale;
    qs[4 * lane + 3] = __uint_as_float(u.y & 0xffff0000u) * qscale;
  }
  __syncwarp();
  const int n = seg_lens[b];
  const size_t base = ((size_t)b * p.hkv + h) * (size_t)seg_cap * kD;
  float M = -INFINITY;
  for (int t = lane; t < n; t += 32) {
    const uint4* kr = reinterpret_cast<const uint4*>(sk + base + (size_t)t * kD);
    float s = 0.f;
#pragma unroll 4
    for (int c8 = 0; c8 < kD / 8; ++c8) {
      const uint4 u = kr[c8];
      const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s = fmaf(qs[8 * c8 + 2 * e], __uint_as_float(wv[e] << 16), s);
        s = fmaf(qs[8 * c8 + 2 * e + 1], __uint_as_float(wv[e] & 0xffff0000u), s);
      }
    }
    pr[t] = s;
    M = fmaxf(M, s);
  }
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  __syncwarp();
  float L = 0.f;
  for (int t = lane; t < n; t += 32) {
    const float e = exp2f(pr[t] - M);
    pr[t] = e;
    L += e;
  }
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  __syncwarp();
  float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int t = 0; t < n; ++t) {
    const uint2 u = reinterpret_cast<const uint2*>(sv + base + (size_t)t * kD)[lane];
    const float e = pr[t];
    o4.x = fmaf(e, __uint_as_float(u.x << 16), o4.x);
    o4.y = fmaf(e, __uint_as_float(u.x & 0xffff0000u), o4.y);
    o4.z = fmaf(e, __uint_as_float(u.y << 16), o4.z);
    o4.w = fmaf(e, __uint_as_float(u.y & 0xffff0000u), o4.w);
  }
  reinterpret_cast<float4*>(p.seg_o + row * kD)[lane] = o4;
  if (lane == 0) { p.seg_m[row] = M; p.seg_l[row] = L; }
}

// ------------------------------------------------------------------ host side
// Split-K granularity.
// Tensor-core path (balanced decomposition, attend_mma.cu): every warp of the persistent grid gets
// an equal contiguous range of the call's page-heads, at least pmin pages long; pmin bounds the
// split slots a unit can need: <= ceil(max_pages / pmin) + 2 (pmin = attend_pages_per_split when
// set, else the smallest value >= 4 that keeps the slots <= 64).
static int mma_pmin(const oscar_ctx& c, int max_pages) {
  if (c.pages_per_split > 0) return c.pages_per_split;
  const int pm = (max_pages + 61) / 62;
  return pm < 4 ? 4 : pm;
}
// CUDA-core kernel (variant 1, b = 3): pages per split of a (split, kv head, sequence) grid with
// ~8 resident CTAs per SM; aim at ~8 waves of short splits (at least 4 pages) so the last wave is
// a small fraction of the kernel (3-bit C2 shape: 52 -> 7 pages per split, 1.00 -> 0.81 ms)
static int choose_pps(const oscar_ctx& c, int B, int max_pages) {
  if (c.pages_per_split > 0) return c.pages_per_split;
  const long units = (long)B * c.hkv;
  const long target = (long)c.num_sms * 64;
  long splits = (target + units - 1) / units;
  if (splits < 1) splits = 1;
  if (splits > max_pages) splits = max_pages;
  long pps = (max_pages + splits - 1) / splits;
  const long lo = max_pages < 4 ? (max_pages > 0 ? max_pages : 1) : 4;
  return (int)(pps < lo ? lo : pps);
}
// split slots per (sequence, query head) in the workspace
static int n_split_slots(const oscar_ctx& c, int B, int max_pages) {
  if (c.variant == 0 && attend_mma_supported(c)) {
    const int pm = mma_pmin(c, max_pages);
    return (max_pages + pm - 1) / pm + 2;
  }
  const int pps = choose_pps(c, B, max_pages);
  return (max_pages + pps - 1) / pps;
}

// Workspace carve-up: every sub-buffer starts on a 256-B boundary (the kernels use 8- and 16-B
// vector accesses on them, and B·H_q may be odd).
struct WsLayout {
  size_t qt, ws_o, ws_m, ws_l, qsum, qscale, qint, qfrag, work, seg_o, seg_m, seg_l, newtok, nsplit, total;
};
static WsLayout ws_layout(const oscar_ctx& c, int B, int max_pages) {
  const size_t ns = (size_t)n_split_slots(c, B, max_pages);
  const size_t rows = (size_t)B * c.hq;
  const size_t nt = (size_t)((c.g * c.ng + 7) / 8);
  WsLayout w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) / 256 * 256;
    return o;
  };
  w.qt = take(rows * kD * 4);
  w.ws_o = take(rows * ns * kD * 4);
  w.ws_m = take(rows * ns * 4);
  w.ws_l = take(rows * ns * 4);
  w.qsum = take(rows * 8 * 4);
  w.qscale = take(rows * 4);
  w.qint = take(rows * kD * 2);
  w.qfrag = take((size_t)B * c.hkv * nt * 16 * 32 * 4);
  w.work = take(64 * 4);
  w.seg_o = take(rows * kD * 4);
  w.seg_m = take(rows * 4);
  w.seg_l = take(rows * 4);
  w.newtok = take((size_t)B * c.hkv * kNewTok * 4);
  w.nsplit = take((size_t)B * 4);
  w.total = off;
  return w;
}

size_t attend_workspace_bytes(const oscar_ctx& c, int B, int max_pages) {
  return ws_layout(c, B, max_pages).total;
}


#ifdef OSCAR_PROBE_TL
static unsigned long long* g_tl = nullptr;
extern "C" __attribute__((visibility("default"))) void oscar_probe_timeline(unsigned long long* tl) { g_tl = tl; }
#else
static unsigned long long* const g_tl = nullptr;
#endif

cudaError_t launch_attend(const oscar_ctx& c, const void* q, const int32_t* page_table,
                          const int32_t* seq_lens, int B, int max_pages, const void* pool,
                          const float* RK, const float* RV, void* ws, void* out, int out_fp32,
                          float* lse, cudaStream_t s, const void* seg_k, const void* seg_v,
                          const int32_t* seg_lens, int seg_cap, const void* k_new, const void* v_new) {
  const bool mma = c.variant == 0 && attend_mma_supported(c);
  AttnParams p{};
  p.hq = c.hq; p.hkv = c.hkv; p.g = c.g; p.P = c.P; p.bits = c.bits; p.G = c.G; p.ng = c.ng;
  p.row_bytes = c.row_bytes; p.vcodes_off = c.vcodes_off; p.meta_off = c.meta_off;
  p.page_bytes = c.page_bytes; p.max_pages = max_pages;
  p.n_splits = n_split_slots(c, B, max_pages);
  if (mma) {
    p.balanced = 1;
    p.pmin = mma_pmin(c, max_pages);
    p.n_warps = attend_mma_total_warps(c, B);
  } else {
    p.pps = choose_pps(c, B, max_pages);
  }
  p.page_table = page_table; p.seq_lens = seq_lens;
  p.pool = static_cast<const uint8_t*>(pool);
  p.tl = g_tl;
  p.nt = (c.g * c.ng + 7) / 8;
  p.batch = B;
  // workspace carve-up (ws_layout: 256-B aligned sub-buffers)
  {
    const WsLayout w = ws_layout(c, B, max_pages);
    uint8_t* base = static_cast<uint8_t*>(ws);
    p.qt = reinterpret_cast<float*>(base + w.qt);
    p.ws_o = reinterpret_cast<float*>(base + w.ws_o);
    p.ws_m = reinterpret_cast<float*>(base + w.ws_m);
    p.ws_l = reinterpret_cast<float*>(base + w.ws_l);
    p.qsum = reinterpret_cast<int32_t*>(base + w.qsum);
    p.qscale = reinterpret_cast<float*>(base + w.qscale);
    p.qint = reinterpret_cast<int16_t*>(base + w.qint);
    p.qfrag = reinterpret_cast<uint32_t*>(base + w.qfrag);
    p.work = reinterpret_cast<int32_t*>(base + w.work);
    p.newtok = reinterpret_cast<float*>(base + w.newtok);
    p.nsplit = reinterpret_cast<int32_t*>(base + w.nsplit);
    if (seg_k) {
      p.seg_o = reinterpret_cast<float*>(base + w.seg_o);
      p.seg_m = reinterpret_cast<float*>(base + w.seg_m);
      p.seg_l = reinterpret_cast<float*>(base + w.seg_l);
    }
  }

  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  int lgG = 0;
  while ((1 << lgG) < c.G) ++lgG;
  cudaError_t e = cudaSuccess;
  {
    PrologueParams pp{};
    pp.q = static_cast<const uint16_t*>(q); pp.RK = RK;
    pp.Hq = c.hq; pp.lgG = lgG; pp.bits = c.bits; pp.nt = p.nt; pp.qscale = c.scale * kLog2e;
    pp.qt = p.qt; pp.qint = p.qint; pp.qsc = p.qscale; pp.qsum = p.qsum;
    pp.qfrag = mma ? p.qfrag : nullptr;
    pp.tq = mma && attend_mma_tq(c) ? 1 : 0; pp.work = mma ? p.work : nullptr;
    pp.knew = static_cast<const uint16_t*>(k_new); pp.vnew = static_cast<const uint16_t*>(v_new);
    pp.RV = RV; pp.newtok = p.newtok;
    pp.nsplit = p.nsplit; pp.balanced = p.balanced; pp.n_warps = p.n_warps; pp.pmin = p.pmin;
    pp.len_adj = k_new != nullptr ? 1 : 0; pp.P = c.P; pp.batch = B;
    pp.page_table = page_table; pp.seq_lens = seq_lens; pp.max_pages = max_pages;
    pp.pool = static_cast<uint8_t*>(const_cast<void*>(pool));
    pp.ep = make_epi_params(c);
    pp.tl = g_tl;
    void (*fn)(PrologueParams) = c.g == 1 ? attend_prologue_kernel<1> : c.g == 2 ? attend_prologue_kernel<2>
                               : c.g == 4 ? attend_prologue_kernel<4> : attend_prologue_kernel<8>;
    const int pnw = c.g + 2 <= 8 ? 8 : 16;
    const int psmem = std::max(pnw * (c.g + 2) * kD, (k_new && RV ? 2 : 1) * kD * kD) * (int)sizeof(float);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem);
    if (e != cudaSuccess) return e;
#if OSCAR_CARVEOUT
    // full shared-memory carveout on the prologue and the partial kernel, so that partial CTAs
    // can become resident beside the prologue's
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
#endif
    // PDL launch: its CTAs may become resident while the previous kernel of the stream drains;
    // the kernel's first instruction waits for that kernel's completion, so every later read
    // (and the partial kernel's early page prefetch) sees the caller's writes
    cudaLaunchConfig_t pcfg{};
    pcfg.gridDim = dim3((unsigned)B, (unsigned)c.hkv);
    pcfg.blockDim = dim3(32 * pnw);
    pcfg.dynamicSmemBytes = psmem;
    pcfg.stream = s;
    pcfg.attrs = pdl;
    pcfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&pcfg, fn, pp);
    if (e != cudaSuccess) return e;
  }
  // decode step: the partial kernels attend over the first seq_len - 1 tokens; the merge kernel
  // appends the new row and folds it in as one more partial (attend_merge_kernel)
  p.len_adj = k_new != nullptr ? 1 : 0;
  if (!mma) {
    const int smem = (8 * kD + 64 + 8 * c.P + 24) * 4 + ((c.page_bytes + 15) & ~15) + c.P * (kD / c.G) * 8;
#define OSCAR_SIMPLE(BB) (c.g == 1 ? attend_partial_simple<BB, 1> : c.g == 2 ? attend_partial_simple<BB, 2> \
                               : c.g == 4 ? attend_partial_simple<BB, 4> : attend_partial_simple<BB, 8>)
    void (*sfn)(AttnParams) = c.bits == 2 ? OSCAR_SIMPLE(2) : c.bits == 3 ? OSCAR_SIMPLE(3) : OSCAR_SIMPLE(4);
#undef OSCAR_SIMPLE
    e = cudaFuncSetAttribute(sfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    sfn<<<dim3(p.n_splits, c.hkv, B), 128, smem, s>>>(p);
  } else {
    e = launch_attend_mma(p, s);
    if (e != cudaSuccess) return e;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (seg_k) {
    const int ssmem = c.g * (kD + seg_cap) * 4;
    e = cudaFuncSetAttribute(attend_segment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem);
    if (e != cudaSuccess) return e;
    attend_segment_kernel<<<dim3(B, c.hkv), 32 * c.g, ssmem, s>>>(
        p, static_cast<const uint16_t*>(q), static_cast<const uint16_t*>(seg_k),
        static_cast<const uint16_t*>(seg_v), seg_lens, seg_cap, c.scale * kLog2e);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  {
    // small batches: one CTA per query head (the fold of many splits gets 8 warps per head)
#ifndef OSCAR_MERGE_PER_HEAD_MUL
#define OSCAR_MERGE_PER_HEAD_MUL 4
#endif
    const bool per_head = (long)B * c.hkv * OSCAR_MERGE_PER_HEAD_MUL <= (long)c.num_sms;
    void (*fn)(AttnParams, const float*, void*, int, float*, StepParams) =
        per_head ? attend_merge_kernel<1>
      : c.g == 1 ? attend_merge_kernel<1> : c.g == 2 ? attend_merge_kernel<2>
      : c.g == 4 ? attend_merge_kernel<4> : attend_merge_kernel<8>;
    const int hc = per_head ? 1 : c.g;
    const int msmem = RV ? kD * kD * 4 : 0;
    StepParams sp{};
    sp.step = k_new != nullptr ? 1 : 0;
    sp.seq_lens = seq_lens;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, msmem);
    if (e != cudaSuccess) return e;
#if OSCAR_CARVEOUT
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
#endif
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)B, (unsigned)c.hkv, (unsigned)(c.g / hc));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = msmem;
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = OSCAR_PDL_MERGE;
    e = cudaLaunchKernelEx(&cfg, fn, p, RV, out, out_fp32, lse, sp);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace oscar
