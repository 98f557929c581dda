// Tensor-core split-K decode attention over the packed cache (variant 0).
// Paper: Alg. 1 DecodeStep attention in the rotated frame; §4 "Decoding
// Attention Kernel" (unpack bytes, apply the stored scale/zero, accumulate in
// floating point; split-K partials merged with online softmax by attend_merge_kernel).
//
// Persistent, warp-granular: every warp of the (fully resident) grid takes one KV head of an
// equal contiguous range of the call's pages (balanced decomposition, struct Decomp: a range
// may span sequences, each (sequence, head) piece is one split partial) and
// streams its 5120-B page blocks through a private smem ring with cp.async.bulk + mbarrier
// (evict-first L2 policy; prefetch runs across unit boundaries).  Per page, in chunks of up to
// 64 tokens:
//   QK  : IMMA m16n8k32 s8 x u8 -> s32.  A = q̃ quantized to 15 bits and split hi/lo int8
//         (rows = (hi|lo) x (group, head) "combos", zero outside the combo's group; built once
//         per (b, h) by attend_prologue_kernel), B = the raw 2/4-bit codes moved to the top bits of
//         each byte (a left shift = IMAD on the FMA pipe, + one LOP3 per 4 codes; the 2^(8-b)
//         byte scale is folded into qscale / qsum).  Exact integer dots per (token, head, group); the fp32
//         epilogue applies s_K, m_K (x̂ = s·c + m).
//   soft: online softmax in the log2 domain, one max per 64-token chunk; the running max
//         follows every increase (OSCAR_LAZY = 0), so the dominant token's weight is exactly
//         1 and its PV operand p·s_V is exact in fp16 (a lazy +8 threshold let p reach 2^8 and
//         put the fp16 rounding of p·s_V on the dominant term: 2.3e-3 max-abs at full size).
//   PV  : HMMA m16n8k16 f16 -> f32.  A = V codes transposed (channels x tokens): the codes are
//         masked straight into the fp16 mantissa (subnormal c·2^(b·q)·2^-24, exact), one LOP3
//         per 2 codes, and each accumulator row is rescaled by 2^(24-b·q) at the end;
//         B = p·s_V per (token, combo) column; the m_V term is a rank-1 FFMA sum.
#include <mutex>
#include <type_traits>

#include "attend_common.cuh"
#include "ptx.cuh"

#ifndef OSCAR_CARVEOUT
#define OSCAR_CARVEOUT 1
#endif

namespace oscar {

namespace {

constexpr int kWarps = 4;
#ifndef OSCAR_CHUNK
#define OSCAR_CHUNK 4
#endif
#ifndef OSCAR_CHUNK_NT2
#define OSCAR_CHUNK_NT2 4
#endif
#ifndef OSCAR_MINB_NT2
#define OSCAR_MINB_NT2 3
#endif
#ifndef OSCAR_LAZY
#define OSCAR_LAZY 0
#endif
#ifndef OSCAR_MINB
#define OSCAR_MINB 3      // 3 CTAs x 4 warps per SM, <= 168 registers: C2 decode step 83.1 -> 79.4 us (same-box A/B)
#endif
#ifndef OSCAR_TQ
#define OSCAR_TQ 1      // token-row QK layout where it applies (A/B: -DOSCAR_TQ=0)
#endif


__device__ __forceinline__ void imma16832(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A unsigned (codes), B signed (q̃): the token-row QK layout
__device__ __forceinline__ void imma16832_us(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void hmma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, uint32_t b) {
  const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&a), *reinterpret_cast<const __half2*>(&b));
  return *reinterpret_cast<const uint32_t*>(&r);
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2: one issue slot for two lanes of math)
struct f2 { float x, y; };
__device__ __forceinline__ uint64_t f2_u64(f2 a) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ f2 u64_f2(uint64_t r) {
  f2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)), "l"(f2_u64(c)));
  return u64_f2(r);
}
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(r);
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(r);
}
// (low halves, high halves) of two half2 words as fp32 pairs
__device__ __forceinline__ void halves_f2(uint32_t w0, uint32_t w1, f2& lo, f2& hi) {
  const __half2 a = *reinterpret_cast<const __half2*>(&w0), b = *reinterpret_cast<const __half2*>(&w1);
  lo = f2{__low2float(a), __low2float(b)};
  hi = f2{__high2float(a), __high2float(b)};
}

using ptx::mbar_init;
using ptx::mbar_wait;
using ptx::bulk_load;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return ptx::su32(p); }

// PV M-tile row -> channel: row gid of M-tile i (+64 for rows gid+8); CPB codes per byte
template <int BITS>
__device__ __forceinline__ int pv_channel(int i, int gid, int upper) {
  constexpr int CPB = 8 / BITS;
  return CPB * gid + 8 * CPB * (i / CPB) + (i % CPB) + (upper ? 64 : 0);
}

struct Item {
  int b, h, split, page0, np, seq_len;
};

// Balanced work decomposition: the pages of all sequences, in sequence order
// (sequence b has npg(b) = ceil(len_b / P) pages), are cut into Wr equal contiguous ranges; warp
// gw takes range gw / H_kv for KV head gw % H_kv, so the H_kv warps of a range read the same
// physical pages (heads side by side in the pool) at the same time.  A range may span sequences;
// each (sequence, head) piece is one split partial.  pre[b] = Σ_{b' < b} npg(b') (CTA shared
// memory).  The range holding sequence page x is rof(x) = ⌊((x + 1)·Wr − 1) / T⌋; the piece of
// range r goes to split slot r − rof(pre[b]), which the merge kernel recomputes.
struct Decomp {
  const int* pre;
  int B;
  int64_t T, W;        // pages of all sequences, ranges
  __device__ __forceinline__ int64_t rof(int64_t x) const { return ((x + 1) * W - 1) / T; }
  // sequence b and page k of sequence page x
  __device__ __forceinline__ void locate(int64_t x, int& b, int& k) const {
    int l = 0, r = B;
    while (r - l > 1) {
      const int m = (l + r) >> 1;
      if (pre[m] <= x) l = m; else r = m;
    }
    b = l;
    k = (int)(x - pre[l]);
  }
};

}  // namespace

template <int BITS, int GQ, int NG, bool TQ>
__global__ void __launch_bounds__(kWarps * 32, (GQ * NG <= 8 ? OSCAR_MINB : OSCAR_MINB_NT2))
attend_partial_mma(AttnParams p, int S) {
  static_assert(!TQ || ((BITS == 2 || BITS == 3) && GQ >= 2 && (NG <= 2 || (NG == 4 && GQ == 4))),
                "token-row QK layout: 2- or 3-bit, g >= 2 (G = 32: g = 4)");
  constexpr int NTQ = (GQ + 3) / 4;           // TQ: QK N-tiles of 4 heads x (hi|lo)
  constexpr int NC = GQ * NG;                 // (group, head) combos
  constexpr int NT = (NC + 7) / 8;            // 8-combo tiles (QK M-tiles / PV N-tiles)
  // PVG (TQ, g = 8, two groups): PV M-tiles are group-pure (rows gid / gid + 8 take V words
  // 2p / 2p + 1 = channels 64p + 4·gid + q and + 32), so each multiplies only the 8 head
  // columns of its own group: one N-tile instead of two, half the PV HMMAs and accumulators
  // G = 32, g = 4 (PVG too): M-tile pair p takes V words 2p (rows gid: group 2p) / 2p + 1 (rows
  // gid + 8: group 2p + 1); its 8 columns are the 4 heads of group 2p, then of group 2p + 1
  constexpr bool PVG = TQ && ((GQ == 8 && NG == 2) || (GQ == 4 && NG == 4));
  // 3-bit codes (reading Z36): a 2-bit low plane in the 2-bit places plus a 1-bit high plane;
  // LB = bits of the low plane every in-place operand below is built from
  constexpr int LB = BITS == 3 ? 2 : BITS;
  constexpr int NTA = PVG ? 1 : NT;           // PV accumulator N-tiles
  constexpr int NBS = PVG ? 2 : NT;           // PV B-operand sets (per M-tile pair, or per N-tile)
  constexpr int kChunk = NT > 1 ? OSCAR_CHUNK_NT2 : OSCAR_CHUNK;   // 16-token sub-tiles per softmax chunk
  constexpr int RB = 16 * BITS;               // packed row bytes (d = 128)
  constexpr int G = 128 / NG;
  constexpr int CPB = 8 / LB;
  constexpr int VW = BITS == 3 ? 4 : RB / 8;  // low-plane V words per lane per 16-token tile
  constexpr uint32_t kCodeMask = LB == 2 ? 0x00030003u : 0x000F000Fu;
  constexpr uint32_t kByteMask = BITS == 2 ? 0x03030303u : 0x0F0F0F0Fu;
  extern __shared__ __align__(128) unsigned char smem[];

#ifdef OSCAR_PROBE_NOPARTIAL
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  return;                                            // timing probe only (results invalid)
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, t = lane & 3;
  const int page_bytes = p.page_bytes, P = p.P;
  unsigned char* ring = smem + (size_t)warp * S * page_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * S * page_bytes) + warp * S;

  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncwarp();
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(policy));

  // ---- balanced decomposition: prefix of pages per sequence (warp 0), then this warp's range
  int* pre = reinterpret_cast<int*>(smem + (size_t)kWarps * S * (page_bytes + 8));
  if (warp == 0) {
    int run = 0;
    for (int b0 = 0; b0 < p.batch; b0 += 32) {
      const int bb = b0 + lane;
      const int n = bb < p.batch ? (max(p.seq_lens[bb] - p.len_adj, 0) + P - 1) / P : 0;
      int inc = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (bb < p.batch) pre[bb] = run + inc - n;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) pre[p.batch] = run;
  }
  __syncthreads();
  Decomp dc;
  dc.pre = pre; dc.B = p.batch;
  dc.T = pre[p.batch];
  dc.W = min((int64_t)(p.n_warps / p.hkv), max((int64_t)1, dc.T / p.pmin));
  const int gw = blockIdx.x * kWarps + warp;
  const int rng = gw / p.hkv, my_h = gw - rng * p.hkv;
  const int64_t lo = rng < dc.W ? (int64_t)rng * dc.T / dc.W : dc.T;
  const int64_t hi = rng < dc.W ? (int64_t)(rng + 1) * dc.T / dc.W : dc.T;
  const int64_t nstream = hi - lo;
  // loader: page indices of stream positions [wb, wb + 32) in window c, [wb + 32, wb + 64) in
  // window n, one per lane; the next window is loaded 32 pages ahead of its use
  int pid_c = 0, pid_n = 0, wb = 0;
  auto load_window = [&](int base, int& pid) {
    pid = 0;
    const int64_t x = lo + base + lane;
    if (x < hi) {
      int bb, kx;
      dc.locate(x, bb, kx);
      pid = p.page_table[(size_t)bb * p.max_pages + kx];
    }
  };
  load_window(0, pid_c);
  load_window(32, pid_n);
  // stages are used in order, one mbarrier each.  (Pages are only read by this call until the
  // merge kernel, which appends the decode step's row, so every page may be prefetched before
  // griddepcontrol.wait.)
  int lq = 0, s_issue = 0, inflight = 0;
  auto issue_one = [&]() -> bool {
    if (lq >= nstream) return false;
    if (lq - wb >= 32) {                       // window c exhausted: shift, prefetch the next
      pid_c = pid_n; wb += 32;
      load_window(wb + 32, pid_n);
    }
    const int li = lq - wb;
    const int64_t page = __shfl_sync(0xffffffffu, pid_c, li);
    if (lane == 0)
      bulk_load(ring + (size_t)s_issue * page_bytes, p.pool + (page * p.hkv + my_h) * (int64_t)page_bytes,
                page_bytes, &bars[s_issue], policy);
    s_issue = s_issue + 1 == S ? 0 : s_issue + 1;
    ++lq;
    ++inflight;
    return true;
  };
  if (lane == 0) tl_mark(p.tl, 1, gw, 0);
  // the first pages depend only on the caller's inputs: start streaming before the prologue ends
  while (inflight < S && issue_one()) {}
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#ifndef OSCAR_PARTIAL_EARLY_TRIGGER
#define OSCAR_PARTIAL_EARLY_TRIGGER 1
#endif
#if OSCAR_PARTIAL_EARLY_TRIGGER
  // the merge grid may launch now (the prologue is complete): its CTAs take the SMs' resources as
  // partial CTAs retire and do their pre-wait work beside this grid's tail
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  if (lane == 0) tl_mark(p.tl, 1, gw, 1);
  while (inflight < S && issue_one()) {}

  const int hh = gid % GQ;                    // every tile of this lane serves head hh
  const bool real = NC >= 8 || gid < NC;
  int s_use = 0;
  uint32_t ph_use = 0;

  for (int64_t x = lo; x < hi;) {
    Item I;
    {
      int kx;
      dc.locate(x, I.b, kx);
      I.h = my_h;
      I.page0 = kx;
      I.np = (int)min((int64_t)(pre[I.b + 1] - pre[I.b] - kx), hi - x);
      I.seq_len = max(p.seq_lens[I.b] - p.len_adj, 0);
      I.split = (int)(rng - dc.rof(pre[I.b]));
      x += I.np;
    }
    const size_t qrow = (size_t)I.b * p.hq + (size_t)I.h * GQ + hh;
    constexpr float kBScale = (float)(1 << (8 - BITS));   // B bytes carry c·2^(8-BITS)
    const float qscale = real ? p.qscale[qrow] * (1.f / kBScale) : 0.f;
    int grp_of[NT];
    float qsumf[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int c = 8 * j + gid;
      grp_of[j] = c < NC ? c / GQ : 0;
      qsumf[j] = c < NC ? (float)p.qsum[qrow * 8 + grp_of[j]] * kBScale : 0.f;
    }
    // QK operand fragments of this (b, h), built by the prologue kernel: A (q rows, TQ = false)
    // or B (q columns, TQ = true)
    uint32_t aq[TQ ? 1 : NT][4][4];
    uint32_t bq[TQ ? NTQ : 1][4][2];
    if constexpr (!TQ) {
      const uint32_t* qf = p.qfrag + ((size_t)I.b * p.hkv + I.h) * NT * 16 * 32 + lane;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int r = 0; r < 4; ++r) aq[j][kk][r] = qf[(j * 16 + kk * 4 + r) * 32];
    } else {
      const uint32_t* qf = p.qfrag + ((size_t)I.b * p.hkv + I.h) * NTQ * 8 * 32 + lane;
#pragma unroll
      for (int jt = 0; jt < NTQ; ++jt)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int r = 0; r < 2; ++r) bq[jt][kk][r] = qf[(jt * 8 + kk * 2 + r) * 32];
    }
    // TQ: this lane's heads in the score layout are hq = 4·jt + t
    float qscale_h[NTQ], qs_h[NTQ][NG];
    if constexpr (TQ) {
#pragma unroll
      for (int jt = 0; jt < NTQ; ++jt) {
        const int hq = 4 * jt + t;
        const size_t row = (size_t)I.b * p.hq + (size_t)I.h * GQ + hq;
        qscale_h[jt] = hq < GQ ? p.qscale[row] * (1.f / kBScale) : 0.f;
#pragma unroll
        for (int g = 0; g < NG; ++g) qs_h[jt][g] = hq < GQ ? (float)p.qsum[row * 8 + g] * kBScale : 0.f;
      }
    }
    float acc[8][NTA][4];
    f2 mv2[NT];                               // Σ p·m_V of this lane's combo over its tokens (2 partial sums)
    float accm[TQ ? NBS : 1][4];              // TQ: Σ p·m_V through the tensor core (rows all equal)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      mv2[j] = f2{0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (TQ && j < NBS) accm[j][e] = 0.f;
        if (j < NTA) {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i][j][e] = 0.f;
        }
      }
    }
    // scores are kept relative to m_run (log2 domain); m_run starts at 0 and the first chunk
    // of the item moves it to that chunk's max, later chunks only when the max grows
    float m_run = 0.f;
    f2 l2{0.f, 0.f};                          // Σ p of this lane's tokens (2 partial sums)
    float m_h[NTQ];                           // TQ: per head of this lane
    f2 l_h[NTQ];
#pragma unroll
    for (int jt = 0; jt < NTQ; ++jt) { m_h[jt] = 0.f; l_h[jt] = f2{0.f, 0.f}; }
    bool fresh = true;

    // one page: chunks of up to 4 sub-tiles (64 tokens)
    // FULLSUB = 4: a completely valid 64-token page (compile-time shape, no masks);
    // FULLSUB = 0: generic page (any P, masked tail)
    auto page_body = [&](const unsigned char* pg, int valid, auto full_c) {
      constexpr int FULLSUB = decltype(full_c)::value;
      constexpr bool FULL = FULLSUB > 0;
      const unsigned char* vcodes = pg + (FULL ? 64 * RB : p.vcodes_off);
      const unsigned char* meta = pg + (FULL ? 128 * RB : p.meta_off);
      const int n_sub = FULL ? FULLSUB : ((valid + 15) >> 4);
      for (int c0 = 0; c0 < n_sub; c0 += kChunk) {
        float sc[kChunk][4];
        float tmax = -INFINITY;
#pragma unroll
        for (int sl = 0; sl < kChunk; ++sl) {
          const int st = c0 + sl;
          if (st >= n_sub) {
#pragma unroll
            for (int e = 0; e < 4; ++e) sc[sl][e] = -INFINITY;
            continue;
          }
          // ---- QK: B = K codes of tokens 2n + nt of the tile
          int cq[NT][2][4];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            uint32_t w[BITS];
            const unsigned char* row = pg + (size_t)(16 * st + 8 * nt + gid) * RB + t * (RB / 4);
            if (BITS == 2) {
              const uint2 u = *reinterpret_cast<const uint2*>(row);
              w[0] = u.x; w[1] = u.y;
            } else {
              const uint4 u = *reinterpret_cast<const uint4*>(row);
              w[0] = u.x; w[1] = u.y; w[2 % BITS] = u.z; w[3 % BITS] = u.w;
            }
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
              for (int e = 0; e < 4; ++e) cq[j][nt][e] = 0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint32_t b0, b1;
              // codes moved to the top bits of each byte with a left shift (a multiply: FMA
              // pipe) and one mask: every B byte is c·2^(8-BITS), folded into qscale
              constexpr uint32_t kTopMask = kByteMask << (8 - BITS);
              if (BITS == 2) {
                b0 = (w[0] * (1u << (6 - 2 * kk))) & kTopMask;
                b1 = (w[1] * (1u << (6 - 2 * kk))) & kTopMask;
              } else {
                b0 = (w[kk >> 1] * (1u << (4 - 4 * (kk & 1)))) & kTopMask;
                b1 = (w[2 + (kk >> 1)] * (1u << (4 - 4 * (kk & 1)))) & kTopMask;
              }
#pragma unroll
              for (int j = 0; j < NT; ++j) imma16832(cq[j][nt], aq[j][kk], b0, b1);
            }
          }
          // ---- scores of tokens 4t + e for head hh (log2 domain, relative to m_run), as the
          // pairs e = (0, 1) and (2, 3)
          f2 part[2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint4 mk4 = *reinterpret_cast<const uint4*>(meta + 128 * NG * st + 128 * grp_of[j] + 32 * t);
            const uint32_t mw[4] = {mk4.x, mk4.y, mk4.z, mk4.w};
            const f2 qs2{qsumf[j], qsumf[j]};
#pragma unroll
            for (int pe = 0; pe < 2; ++pe) {
              // token 4t+e <-> (N-tile e&1, column 2t + e/2): e = 2pe (nt 0), 2pe+1 (nt 1), col = pe
              const int d0 = cq[j][0][pe] * 256 + cq[j][0][2 + pe];
              const int d1 = cq[j][1][pe] * 256 + cq[j][1][2 + pe];
              f2 sk, mk;
              halves_f2(mw[2 * pe], mw[2 * pe + 1], sk, mk);
              part[pe] = ffma2(sk, f2{(float)d0, (float)d1}, ffma2(mk, qs2, part[pe]));
            }
          }
#pragma unroll
          for (int x = GQ; x < 8 && x < NC; x <<= 1)
#pragma unroll
            for (int pe = 0; pe < 2; ++pe)
              part[pe] = fadd2(part[pe], f2{__shfl_xor_sync(0xffffffffu, part[pe].x, x * 4),
                                            __shfl_xor_sync(0xffffffffu, part[pe].y, x * 4)});
          const f2 qsc{qscale, qscale}, nm{-m_run, -m_run};
#pragma unroll
          for (int pe = 0; pe < 2; ++pe) {
            const f2 v = ffma2(part[pe], qsc, nm);
            sc[sl][2 * pe] = v.x;
            sc[sl][2 * pe + 1] = v.y;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            bool ok = real;
            if (!FULL) ok = ok && (16 * st + 4 * t + e) < valid;
            if (!ok) sc[sl][e] = -INFINITY;
            tmax = fmaxf(tmax, sc[sl][e]);
          }
        }
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
        // ---- online-softmax rescale: first chunk of the item, or max grown by > 2^8
        const bool first = fresh;
        const bool need = first ? tmax > -INFINITY : tmax > (float)OSCAR_LAZY;
        fresh = false;
        if (__any_sync(0xffffffffu, need)) {
          const float shift = need ? tmax : 0.f;
          const float alpha = first ? 1.f : ex2_ftz(-shift);   // nothing accumulated yet if first
#pragma unroll
          for (int sl = 0; sl < kChunk; ++sl)
#pragma unroll
            for (int e = 0; e < 4; ++e) sc[sl][e] -= shift;
          m_run += shift;
          l2 = fmul2(l2, f2{alpha, alpha});
          const float a0 = __shfl_sync(0xffffffffu, alpha, 8 * t);
          const float a1 = __shfl_sync(0xffffffffu, alpha, 8 * t + 4);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            mv2[j] = fmul2(mv2[j], f2{alpha, alpha});
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              acc[i][j][0] *= a0; acc[i][j][2] *= a0;
              acc[i][j][1] *= a1; acc[i][j][3] *= a1;
            }
          }
        }
        // ---- PV per sub-tile
#pragma unroll
        for (int sl = 0; sl < kChunk; ++sl) {
          const int st = c0 + sl;
          if (st >= n_sub) break;
          float pr[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) pr[e] = ex2_ftz(sc[sl][e]);   // exp2(-inf) = 0
          const f2 p01{pr[0], pr[1]}, p23{pr[2], pr[3]};
          l2 = fadd2(l2, fadd2(p01, p23));
          uint32_t bpv[NT][2];
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint4 mv4 = *reinterpret_cast<const uint4*>(meta + 128 * NG * st + 128 * grp_of[j] + 32 * t + 16);
            uint32_t mw[4] = {mv4.x, mv4.y, mv4.z, mv4.w};
            if (!FULL) {   // masked tokens may carry garbage metadata: keep them out
#pragma unroll
              for (int e = 0; e < 4; ++e) mw[e] = pr[e] == 0.f ? 0u : mw[e];
            }
            // p·s_V and p·m_V in fp32 (one fp16 rounding of the MMA operand; the m_V sum exact)
            f2 s01, m01, s23, m23;
            halves_f2(mw[0], mw[1], s01, m01);
            halves_f2(mw[2], mw[3], s23, m23);
            const f2 w01 = fmul2(p01, s01), w23 = fmul2(p23, s23);
            mv2[j] = ffma2(p01, m01, ffma2(p23, m23, mv2[j]));
            bpv[j][0] = pack_half2(w01.x, w23.x);   // k-slots 2t, 2t+1 <-> tokens 4t, 4t+2
            bpv[j][1] = pack_half2(w01.y, w23.y);   // k-slots 2t+8, 2t+9 <-> tokens 4t+1, 4t+3
          }
          uint32_t vw[VW];
          {
            const uint4* vp = reinterpret_cast<const uint4*>(vcodes + (size_t)st * 16 * RB) + 4 * gid + t;
#pragma unroll
            for (int u = 0; u < VW / 4; ++u) {
              const uint4 x = vp[32 * u];
              vw[4 * u] = x.x; vw[4 * u + 1] = x.y; vw[4 * u + 2] = x.z; vw[4 * u + 3] = x.w;
            }
          }
          uint32_t vs[VW];
#pragma unroll
          for (int k = 0; k < VW; ++k) vs[k] = vw[k] >> 8;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int q = i % CPB;
            const uint32_t msk = kCodeMask << (BITS * q);
            uint32_t a[4];
            a[0] = vw[i / CPB] & msk;             // row gid,   tokens (4t, 4t+2)
            a[1] = vw[VW / 2 + i / CPB] & msk;    // row gid+8, tokens (4t, 4t+2)
            a[2] = vs[i / CPB] & msk;             // row gid,   tokens (4t+1, 4t+3)
            a[3] = vs[VW / 2 + i / CPB] & msk;    // row gid+8, tokens (4t+1, 4t+3)
#pragma unroll
            for (int j = 0; j < NT; ++j) hmma16816(acc[i][j], a, bpv[j][0], bpv[j][1]);
          }
        }
      }
    };

    // TQ page body: QK with the tokens as the MMA rows.  A = K codes of K-tile rows gid /
    // gid + 8 (tokens 2·gid, 2·gid + 1 of the 16-token sub-tile, FORMAT fmt_krow), lane t taking
    // words t and 4 + t of each row so every 32-channel k-step stays inside one quantization
    // group (G >= 64) and accumulates into that group's C; B = q̃ hi/lo int8 columns (4 heads x
    // (hi|lo) per N-tile).  Each lane then owns the scores of its two tokens for head 4·jt + t —
    // no cross-group shuffles, no duplicated softmax.  PV is the kernel's usual HMMA with the
    // B operand gathered by two shuffles (p pairs as half2) and formed by HMUL2 with s_V; the
    // Σ p·m_V term runs as an extra HMMA against an all-ones A tile.
    auto page_body_tq = [&](const unsigned char* pg, int valid, auto full_c) {
      constexpr int FULLSUB = decltype(full_c)::value;
      constexpr bool FULL = FULLSUB > 0;
      const unsigned char* vcodes = pg + (FULL ? 64 * RB : p.vcodes_off);
      const unsigned char* meta = pg + (FULL ? 128 * RB : p.meta_off);
      const int n_sub = FULL ? FULLSUB : ((valid + 15) >> 4);
      const int hc = gid % GQ;                  // PV: head of this lane's combo column(s)
      for (int c0 = 0; c0 < n_sub; c0 += kChunk) {
        float sc[kChunk][NTQ][2];
        float tmax[NTQ];
#pragma unroll
        for (int jt = 0; jt < NTQ; ++jt) tmax[jt] = -INFINITY;
#pragma unroll
        for (int sl = 0; sl < kChunk; ++sl) {
          const int st = c0 + sl;
          if (st >= n_sub) {
#pragma unroll
            for (int jt = 0; jt < NTQ; ++jt) sc[sl][jt][0] = sc[sl][jt][1] = -INFINITY;
            continue;
          }
          // one ldmatrix.x4: matrices (rows 0-7 | 8-15) x (bytes 0-15 | 16-31) of the K tile, so
          // lane (gid, t) receives words t and 4 + t of rows gid and gid + 8
          uint32_t wa[NG == 4 ? 8 : 2], wb[NG == 4 ? 8 : 2];
          [[maybe_unused]] uint32_t ha4[NG == 4 && BITS == 3 ? 4 : 1], hb4[NG == 4 && BITS == 3 ? 4 : 1];
          if constexpr (NG == 4) {
            // G = 32: lane t takes 2-bit field t of every word of rows gid / gid + 8 (k-step g =
            // words 2g, 2g + 1 = group g)
            const uint4* ra = reinterpret_cast<const uint4*>(pg + (size_t)(16 * st + gid) * RB);
            const uint4* rb = reinterpret_cast<const uint4*>(pg + (size_t)(16 * st + 8 + gid) * RB);
            const uint4 a0 = ra[0], a1 = ra[1], b0 = rb[0], b1 = rb[1];
            wa[0] = a0.x; wa[1] = a0.y; wa[2] = a0.z; wa[3] = a0.w;
            wa[4] = a1.x; wa[5] = a1.y; wa[6] = a1.z; wa[7] = a1.w;
            wb[0] = b0.x; wb[1] = b0.y; wb[2] = b0.z; wb[3] = b0.w;
            wb[4] = b1.x; wb[5] = b1.y; wb[6] = b1.z; wb[7] = b1.w;
            if constexpr (BITS == 3) {           // the 4 high-plane words of both rows
              const uint4 a2 = ra[2], b2 = rb[2];
              ha4[0] = a2.x; ha4[1] = a2.y; ha4[2] = a2.z; ha4[3] = a2.w;
              hb4[0] = b2.x; hb4[1] = b2.y; hb4[2] = b2.z; hb4[3] = b2.w;
            }
          } else {
            const int mi = lane >> 3;
            const uint32_t addr = smem_u32(pg + (size_t)(16 * st + 8 * (mi >> 1) + (lane & 7)) * RB + 16 * (mi & 1));
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
                         : "=r"(wa[0]), "=r"(wa[1]), "=r"(wb[0]), "=r"(wb[1])
                         : "r"(addr));
          }
          // 3-bit: the high-plane words of low words t and 4 + t (high word j / 2, nibble j % 2
          // = t % 2) of rows gid / gid + 8, normalized so the lane's nibble sits in bits 4-7
          [[maybe_unused]] uint32_t ha[2], hb[2];
          if constexpr (BITS == 3 && NG != 4) {
            const uint32_t* ra = reinterpret_cast<const uint32_t*>(pg + (size_t)(16 * st + gid) * RB + 32);
            const uint32_t* rb = reinterpret_cast<const uint32_t*>(pg + (size_t)(16 * st + 8 + gid) * RB + 32);
            const int sh = (t & 1) ? 0 : 4;
            ha[0] = ra[t >> 1] << sh; ha[1] = ra[2 + (t >> 1)] << sh;
            hb[0] = rb[t >> 1] << sh; hb[1] = rb[2 + (t >> 1)] << sh;
          }
          int cq[NTQ][NG][4];
#pragma unroll
          for (int jt = 0; jt < NTQ; ++jt)
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
              for (int e = 0; e < 4; ++e) cq[jt][g][e] = 0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            uint32_t a[4];
            if constexpr (NG == 4 && BITS == 3) {
              // 3-bit, G = 32: field t to bits 5-6 (lo·32)
              auto lo5 = [&](uint32_t w) { return (t < 3 ? (w << (5 - 2 * t)) : (w >> 1)) & 0x60606060u; };
              a[0] = lo5(wa[2 * kk]);
              a[1] = lo5(wb[2 * kk]);
              a[2] = lo5(wa[2 * kk + 1]);
              a[3] = lo5(wb[2 * kk + 1]);
            } else if constexpr (NG == 4) {
              // k-step kk = group kk: field t of words 2kk (a0, a1) and 2kk + 1 (a2, a3)
              const uint32_t mul = 1u << (6 - 2 * t);
              a[0] = (wa[2 * kk] * mul) & 0xC0C0C0C0u;
              a[1] = (wb[2 * kk] * mul) & 0xC0C0C0C0u;
              a[2] = (wa[2 * kk + 1] * mul) & 0xC0C0C0C0u;
              a[3] = (wb[2 * kk + 1] * mul) & 0xC0C0C0C0u;
            } else if (BITS == 2) {
              // k-step kk: word kk/2 (group kk/2 when G = 64), 2-bit fields 2(kk&1) (a0, a1) and
              // 2(kk&1)+1 (a2, a3) moved to the top of each byte (c·64, folded into qscale)
              const int wi = kk >> 1, s0 = 6 - 4 * (kk & 1);
              a[0] = (wa[wi] << s0) & 0xC0C0C0C0u;
              a[1] = (wb[wi] << s0) & 0xC0C0C0C0u;
              a[2] = (wa[wi] << (s0 - 2)) & 0xC0C0C0C0u;
              a[3] = (wb[wi] << (s0 - 2)) & 0xC0C0C0C0u;
            } else {
              // 3-bit: the low field to bits 5-6 (lo·32) — fields f0 = 2(kk&1) and f0 + 1
              const int wi = kk >> 1;
              if ((kk & 1) == 0) {
                a[0] = (wa[wi] << 5) & 0x60606060u;
                a[1] = (wb[wi] << 5) & 0x60606060u;
                a[2] = (wa[wi] << 3) & 0x60606060u;
                a[3] = (wb[wi] << 3) & 0x60606060u;
              } else {
                a[0] = (wa[wi] << 1) & 0x60606060u;
                a[1] = (wb[wi] << 1) & 0x60606060u;
                a[2] = (wa[wi] >> 1) & 0x60606060u;
                a[3] = (wb[wi] >> 1) & 0x60606060u;
              }
            }
            const int g = NG == 4 ? kk : (NG == 2 ? (kk >> 1) : 0);
#pragma unroll
            for (int jt = 0; jt < NTQ; ++jt) imma16832_us(cq[jt][g], a, bq[jt][kk][0], bq[jt][kk][1]);
            if constexpr (BITS == 3) {
              // the high bit to bit 7 (hi·128): code·32 = lo·32 + hi·128 into the same C
              uint32_t ah[4];
              if constexpr (NG == 4) {
                // low words 2kk (even: high bit t) and 2kk + 1 (odd: 4 + t) -> high word kk
                ah[0] = (ha4[kk] << (7 - t)) & 0x80808080u;
                ah[1] = (hb4[kk] << (7 - t)) & 0x80808080u;
                ah[2] = (ha4[kk] << (3 - t)) & 0x80808080u;
                ah[3] = (hb4[kk] << (3 - t)) & 0x80808080u;
              } else {
                const int wi = kk >> 1, f0 = 2 * (kk & 1);
                ah[0] = (ha[wi] << (3 - f0)) & 0x80808080u;
                ah[1] = (hb[wi] << (3 - f0)) & 0x80808080u;
                ah[2] = (ha[wi] << (2 - f0)) & 0x80808080u;
                ah[3] = (hb[wi] << (2 - f0)) & 0x80808080u;
              }
#pragma unroll
              for (int jt = 0; jt < NTQ; ++jt) imma16832_us(cq[jt][g], ah, bq[jt][kk][0], bq[jt][kk][1]);
            }
          }
          // scores of tokens 2·gid (e = 0) and 2·gid + 1 (e = 1) for head 4·jt + t
#pragma unroll
          for (int jt = 0; jt < NTQ; ++jt) {
            f2 part{0.f, 0.f};
#pragma unroll
            for (int g = 0; g < NG; ++g) {
              const uint2 mk = *reinterpret_cast<const uint2*>(meta + 128 * NG * st + 128 * g + 32 * (gid >> 1) + 8 * (gid & 1));
              f2 sk, mq;
              halves_f2(mk.x, mk.y, sk, mq);
              const int d0 = cq[jt][g][0] * 256 + cq[jt][g][1];
              const int d1 = cq[jt][g][2] * 256 + cq[jt][g][3];
              part = ffma2(sk, f2{(float)d0, (float)d1}, ffma2(mq, f2{qs_h[jt][g], qs_h[jt][g]}, part));
            }
            const f2 v = ffma2(part, f2{qscale_h[jt], qscale_h[jt]}, f2{-m_h[jt], -m_h[jt]});
            sc[sl][jt][0] = v.x;
            sc[sl][jt][1] = v.y;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              bool ok = 4 * jt + t < GQ;
              if (!FULL) ok = ok && (16 * st + 2 * gid + e) < valid;
              if (!ok) sc[sl][jt][e] = -INFINITY;
              tmax[jt] = fmaxf(tmax[jt], sc[sl][jt][e]);
            }
          }
        }
        bool need_any = false;
        float alpha[NTQ];
        const bool first = fresh;
        fresh = false;
#pragma unroll
        for (int jt = 0; jt < NTQ; ++jt) {
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) tmax[jt] = fmaxf(tmax[jt], __shfl_xor_sync(0xffffffffu, tmax[jt], o));
          const bool need = first ? tmax[jt] > -INFINITY : tmax[jt] > (float)OSCAR_LAZY;
          const float shift = need ? tmax[jt] : 0.f;
          alpha[jt] = first ? 1.f : ex2_ftz(-shift);
          if (need) {
#pragma unroll
            for (int sl = 0; sl < kChunk; ++sl) { sc[sl][jt][0] -= shift; sc[sl][jt][1] -= shift; }
            m_h[jt] += shift;
            l_h[jt] = fmul2(l_h[jt], f2{alpha[jt], alpha[jt]});
          }
          need_any = need_any || (need && !first);
        }
        if (__any_sync(0xffffffffu, need_any)) {
          // accumulator column (combo 8j + 2t + e) of head (8j + 2t + e) % GQ: its alpha lives
          // in lane t' = head % 4, slot head / 4
#pragma unroll
          for (int j = 0; j < NBS; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              // PVG: every set's column 2t + e is head 2t + e
              const int hq = PVG ? (2 * t + e) % GQ : (8 * j + 2 * t + e) % GQ;
              float a = __shfl_sync(0xffffffffu, alpha[0], hq & 3);
              if (NTQ > 1) {
                const float a1 = __shfl_sync(0xffffffffu, alpha[NTQ - 1], hq & 3);
                a = hq >= 4 ? a1 : a;
              }
              accm[j][e] *= a; accm[j][e + 2] *= a;
              if (j < NTA) {
#pragma unroll
                for (int i = 0; i < 8; ++i) { acc[i][j][e] *= a; acc[i][j][e + 2] *= a; }
              }
            }
        }
        // ---- PV per sub-tile
#pragma unroll
        for (int sl = 0; sl < kChunk; ++sl) {
          const int st = c0 + sl;
          if (st >= n_sub) break;
          uint32_t P[NTQ];
#pragma unroll
          for (int jt = 0; jt < NTQ; ++jt) {
            const float p0 = ex2_ftz(sc[sl][jt][0]), p1 = ex2_ftz(sc[sl][jt][1]);   // exp2(-inf) = 0
            l_h[jt] = fadd2(l_h[jt], f2{p0, p1});
            P[jt] = pack_half2(p0, p1);
          }
          // (p(4t), p(4t+1)) from lane (2t, hc%4), (p(4t+2), p(4t+3)) from lane (2t+1, hc%4)
          uint32_t X = __shfl_sync(0xffffffffu, P[0], 8 * t + (hc & 3));
          uint32_t Y = __shfl_sync(0xffffffffu, P[0], 8 * t + 4 + (hc & 3));
          if (NTQ > 1) {
            const uint32_t X1 = __shfl_sync(0xffffffffu, P[NTQ - 1], 8 * t + (hc & 3));
            const uint32_t Y1 = __shfl_sync(0xffffffffu, P[NTQ - 1], 8 * t + 4 + (hc & 3));
            if (hc >= 4) { X = X1; Y = Y1; }
          }
          const uint32_t p02 = __byte_perm(X, Y, 0x5410), p13 = __byte_perm(X, Y, 0x7632);
          uint32_t bpv[NBS][2];
#pragma unroll
          for (int j = 0; j < NBS; ++j) {
            // PVG: set j = M-tile pair j; column gid -> group j (g = 8) or 2j + gid / 4 (G = 32)
            const int gc = PVG ? (NG == 4 ? 2 * j + (gid >> 2) : j) : min((8 * j + gid) / GQ, NG - 1);
            const uint4 mv4 = *reinterpret_cast<const uint4*>(meta + 128 * NG * st + 128 * gc + 32 * t + 16);
            uint32_t mw[4] = {mv4.x, mv4.y, mv4.z, mv4.w};
            if (!FULL) {   // masked tokens may carry garbage metadata: keep them out
#pragma unroll
              for (int e = 0; e < 4; ++e) mw[e] = (16 * st + 4 * t + e) < valid ? mw[e] : 0u;
            }
            const uint32_t s02 = __byte_perm(mw[0], mw[2], 0x5410), s13 = __byte_perm(mw[1], mw[3], 0x5410);
            const uint32_t m02 = __byte_perm(mw[0], mw[2], 0x7632), m13 = __byte_perm(mw[1], mw[3], 0x7632);
            bpv[j][0] = hmul2_u32(p02, s02);   // k-slots 2t, 2t+1 <-> tokens 4t, 4t+2
            bpv[j][1] = hmul2_u32(p13, s13);   // k-slots 2t+8, 2t+9 <-> tokens 4t+1, 4t+3
            const uint32_t ones[4] = {0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u};
            hmma16816(accm[j], ones, hmul2_u32(p02, m02), hmul2_u32(p13, m13));
          }
          uint32_t vw[VW];
          {
            const uint4* vp = reinterpret_cast<const uint4*>(vcodes + (size_t)st * 16 * RB) + 4 * gid + t;
#pragma unroll
            for (int u = 0; u < VW / 4; ++u) {
              const uint4 x = vp[32 * u];
              vw[4 * u] = x.x; vw[4 * u + 1] = x.y; vw[4 * u + 2] = x.z; vw[4 * u + 3] = x.w;
            }
          }
          // 3-bit: high-plane word k = high byte 4k + gid % 4 of this lane's 4 tokens (FORMAT,
          // reading Z36); the lane's nibble gid / 4 moved to bits 0-3 of each byte
          [[maybe_unused]] uint32_t vh[BITS == 3 ? 4 : 1];
          if constexpr (BITS == 3) {
            const uint4 x = *reinterpret_cast<const uint4*>(vcodes + (size_t)st * 16 * RB + 512 + 16 * (4 * (gid & 3) + t));
            const int sh = 4 * (gid >> 2);
            vh[0] = x.x >> sh; vh[1] = x.y >> sh; vh[2] = x.z >> sh; vh[3] = x.w >> sh;
          }
          uint32_t vs[VW];
#pragma unroll
          for (int k = 0; k < VW; ++k) vs[k] = vw[k] >> 8;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int q = i % CPB;
            const uint32_t msk = kCodeMask << (LB * q);
            uint32_t a[4];
            if constexpr (PVG) {               // M-tile i: group p = i / CPB, words 2p / 2p + 1
              const int pg2 = 2 * (i / CPB);
              a[0] = vw[pg2] & msk;
              a[1] = vw[pg2 + 1] & msk;
              a[2] = vs[pg2] & msk;
              a[3] = vs[pg2 + 1] & msk;
              hmma16816(acc[i][0], a, bpv[i / CPB][0], bpv[i / CPB][1]);
              if constexpr (BITS == 3) {
                const uint32_t mh = 0x00040004u << (2 * q);
                uint32_t ah[4];
                ah[0] = (vh[pg2] << (q + 2)) & mh;
                ah[1] = (vh[pg2 + 1] << (q + 2)) & mh;
                ah[2] = (vh[pg2] >> (6 - q)) & mh;
                ah[3] = (vh[pg2 + 1] >> (6 - q)) & mh;
                hmma16816(acc[i][0], ah, bpv[i / CPB][0], bpv[i / CPB][1]);
              }
            } else {
              a[0] = vw[i / CPB] & msk;
              a[1] = vw[VW / 2 + i / CPB] & msk;
              a[2] = vs[i / CPB] & msk;
              a[3] = vs[VW / 2 + i / CPB] & msk;
#pragma unroll
              for (int j = 0; j < NTA; ++j) hmma16816(acc[i][j], a, bpv[j][0], bpv[j][1]);
              if constexpr (BITS == 3) {
                // the high bit at mantissa bit 2q + 2 of each half (4·hi·4^q·2^-24): tokens
                // (4t, 4t+2) from bytes 0 / 2, (4t+1, 4t+3) from bytes 1 / 3 of word i/4 (+2 upper)
                const uint32_t mh = 0x00040004u << (2 * q);
                uint32_t ah[4];
                ah[0] = (vh[i / CPB] << (q + 2)) & mh;
                ah[1] = (vh[2 + i / CPB] << (q + 2)) & mh;
                ah[2] = (vh[i / CPB] >> (6 - q)) & mh;
                ah[3] = (vh[2 + i / CPB] >> (6 - q)) & mh;
#pragma unroll
                for (int j = 0; j < NTA; ++j) hmma16816(acc[i][j], ah, bpv[j][0], bpv[j][1]);
              }
            }
          }
        }
      }
    };

    for (int k = 0; k < I.np; ++k) {
      mbar_wait(&bars[s_use], ph_use);
      const unsigned char* pg = ring + (size_t)s_use * page_bytes;
      const int valid = min(P, I.seq_len - (I.page0 + k) * P);
      if constexpr (TQ) {
        if (valid == 64 && P == 64) page_body_tq(pg, valid, std::integral_constant<int, 4>{});
        else page_body_tq(pg, valid, std::integral_constant<int, 0>{});
      } else {
        if (valid == 64 && P == 64) page_body(pg, valid, std::integral_constant<int, 4>{});
        else page_body(pg, valid, std::integral_constant<int, 0>{});
      }
      // release the stage (every lane's reads are done) and refill it
      __syncwarp();
      if (++s_use == S) { s_use = 0; ph_use ^= 1u; }
      --inflight;
      issue_one();
    }

    // ---- write this item's partial (unnormalized õ in the rotated frame, m, l)
    float l_run = l2.x + l2.y;
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    float l_hd[NTQ];                          // TQ: Σ p of head 4·jt + t over the 8 gid lanes
#pragma unroll
    for (int jt = 0; jt < NTQ; ++jt) {
      l_hd[jt] = l_h[jt].x + l_h[jt].y;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) l_hd[jt] += __shfl_xor_sync(0xffffffffu, l_hd[jt], o);
    }
    float mv_acc[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      mv_acc[j] = mv2[j].x + mv2[j].y;
      mv_acc[j] += __shfl_xor_sync(0xffffffffu, mv_acc[j], 1);
      mv_acc[j] += __shfl_xor_sync(0xffffffffu, mv_acc[j], 2);
    }
    const size_t row0 = ((size_t)I.b * p.hq + (size_t)I.h * GQ) * p.n_splits + I.split;
    if constexpr (PVG) {
      // M-tile pair p = i / CPB; rows gid / gid + 8 = channels 64p + CPB·gid + q (+ 32).  g = 8:
      // column = head, both row halves valid; G = 32: columns 0-3 (heads of group 2p) pair with
      // the rows gid, columns 4-7 (group 2p + 1) with the rows gid + 8
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = 2 * t + (e & 1);
        const bool upper = (e >> 1) != 0;
        if (NG == 4 && (col >= 4) != upper) continue;
        const int head = col % GQ;
        const size_t row = row0 + (size_t)head * p.n_splits;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float unscale = (float)(1 << (24 - LB * (i % CPB)));
          const int ch = 64 * (i / CPB) + CPB * gid + (i % CPB) + (upper ? 32 : 0);
          p.ws_o[row * 128 + ch] = fmaf(acc[i][0][e], unscale, accm[i / CPB][e & 1]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < (PVG ? 0 : NT); ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = 2 * t + (e & 1);
        const int cc = 8 * j + col;
        const float mvs = TQ ? accm[j % NBS][e & 1]                         // this lane's column
                             : __shfl_sync(0xffffffffu, mv_acc[j], 4 * col);   // combo col = gid of lane 4·col
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float unscale = (float)(1 << (24 - LB * (i % CPB)));
          const int ch = pv_channel<LB>(i, gid, e >> 1);
          if (cc < NC && ch / G == cc / GQ) {
            const size_t row = row0 + (size_t)(cc % GQ) * p.n_splits;
            p.ws_o[row * 128 + ch] = fmaf(acc[i][j % NTA][e], unscale, mvs);
          }
        }
      }
    if constexpr (TQ) {
#pragma unroll
      for (int jt = 0; jt < NTQ; ++jt)
        if (gid == 0 && 4 * jt + t < GQ) {
          const size_t row = row0 + (size_t)(4 * jt + t) * p.n_splits;
          p.ws_m[row] = I.np > 0 ? m_h[jt] : -INFINITY;
          p.ws_l[row] = l_hd[jt];
        }
    } else if (t == 0 && gid < GQ) {
      const size_t row = row0 + (size_t)gid * p.n_splits;
      p.ws_m[row] = I.np > 0 ? m_run : -INFINITY;
      p.ws_l[row] = l_run;
    }
  }
  if (lane == 0) tl_mark(p.tl, 1, gw, 2);
#ifdef OSCAR_PROBE_TL
  if (lane == 0 && p.tl) {
    unsigned smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    p.tl[(size_t)32768 + (size_t)gw * 4 + 3] = smid | (wid << 16) | ((unsigned long long)gw << 32);
  }
#endif
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");   // let the merge kernel launch
}

// ---------------------------------------------------------------- dispatch
namespace {
using KernelFn = void (*)(AttnParams, int);

template <int BITS>
KernelFn pick_g(int g, int ng) {
#define OSCAR_CASE(GQ_, NG_) \
  if (g == GQ_ && ng == NG_) return attend_partial_mma<BITS, GQ_, NG_, false>;
  OSCAR_CASE(1, 1) OSCAR_CASE(1, 2) OSCAR_CASE(1, 4)
  OSCAR_CASE(2, 1) OSCAR_CASE(2, 2) OSCAR_CASE(2, 4)
  OSCAR_CASE(4, 1) OSCAR_CASE(4, 2) OSCAR_CASE(4, 4)
  OSCAR_CASE(8, 1) OSCAR_CASE(8, 2)
#undef OSCAR_CASE
  return nullptr;
}

// token-row QK layout (TQ): 2-bit codes, G in {64, 128} with g in {2, 4, 8}, G = 32 with g = 4
KernelFn pick_tq(int g, int ng) {
#define OSCAR_CASE(GQ_, NG_) \
  if (g == GQ_ && ng == NG_) return attend_partial_mma<2, GQ_, NG_, true>;
  OSCAR_CASE(2, 1) OSCAR_CASE(2, 2) OSCAR_CASE(4, 1) OSCAR_CASE(4, 2) OSCAR_CASE(4, 4) OSCAR_CASE(8, 1)
  OSCAR_CASE(8, 2)
#undef OSCAR_CASE
  return nullptr;
}

// 3-bit (reading Z36 planes) on the token-row layout: the same shapes as 2-bit
KernelFn pick_tq3(int g, int ng) {
#define OSCAR_CASE(GQ_, NG_) \
  if (g == GQ_ && ng == NG_) return attend_partial_mma<3, GQ_, NG_, true>;
  OSCAR_CASE(2, 1) OSCAR_CASE(2, 2) OSCAR_CASE(4, 1) OSCAR_CASE(4, 2) OSCAR_CASE(4, 4) OSCAR_CASE(8, 1)
  OSCAR_CASE(8, 2)
#undef OSCAR_CASE
  return nullptr;
}

KernelFn pick(int bits, int g, int ng) {
  if (bits == 2 && OSCAR_TQ) {
    if (KernelFn f = pick_tq(g, ng)) return f;
  }
  if (bits == 3 && OSCAR_TQ) return pick_tq3(g, ng);
  if (bits == 2) return pick_g<2>(g, ng);
  if (bits == 4) return pick_g<4>(g, ng);
  return nullptr;
}

// ring stages per warp: 2-4 within ~48 KB per CTA; large pages (P = 256 at 4 bits: 36 KB) fall
// back to what fits in the 227-KB CTA limit (1 stage), 0 if not even that
#ifndef OSCAR_RING_KB
#define OSCAR_RING_KB 48
#endif
int stages_for(int page_bytes) {
  int S = (OSCAR_RING_KB * 1024) / (kWarps * page_bytes);
  S = S < 2 ? 2 : (S > 4 ? 4 : S);
  while (S > 0 && kWarps * S * (page_bytes + 8) > 227 * 1024) --S;
  return S;
}
}  // namespace

bool attend_mma_tq(const oscar_ctx& c) {
  return OSCAR_TQ && ((c.bits == 2 && pick_tq(c.g, c.ng) != nullptr) || (c.bits == 3 && pick_tq3(c.g, c.ng) != nullptr));
}

bool attend_mma_supported(const oscar_ctx& c) {
  return c.d == 128 && pick(c.bits, c.g, c.ng) != nullptr && c.P % 16 == 0 && stages_for(c.page_bytes) > 0;
}

// dynamic smem of the partial kernel: per-warp page rings + their mbarriers + the CTA's page
// prefix pre[B + 1] (balanced decomposition)
static int mma_smem(int page_bytes, int B) {
  return kWarps * stages_for(page_bytes) * (page_bytes + 8) + ((B + 1) * 4 + 15) / 16 * 16;
}

// Warps of the persistent grid: SMs x resident CTAs per SM x 4 (every CTA resident at once)
int attend_mma_total_warps(const oscar_ctx& c, int B) {
  KernelFn fn = pick(c.bits, c.g, c.ng);
  if (!fn) return 0;
  const int smem = mma_smem(c.page_bytes, B);
  // resident CTAs per SM, cached per (kernel, smem): the query is a few µs of host time
  // (contexts may be used from several host threads: the cache is guarded)
  static std::mutex mu;
  static struct { KernelFn fn; int smem, per_sm; } cache[64];
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache)
    if (e.fn == fn && e.smem == smem) return c.num_sms * e.per_sm * kWarps;
  int per_sm = 0;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWarps * 32, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 2;
  }
  if (per_sm < 1) per_sm = 1;
  for (auto& e : cache)
    if (e.fn == nullptr) { e.fn = fn; e.smem = smem; e.per_sm = per_sm; break; }
  return c.num_sms * per_sm * kWarps;
}

cudaError_t launch_attend_mma(const AttnParams& p, cudaStream_t s) {
  KernelFn fn = pick(p.bits, p.g, p.ng);
  if (!fn) return cudaErrorNotSupported;
  const int S = stages_for(p.page_bytes);
  const int smem = mma_smem(p.page_bytes, p.batch);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
#if OSCAR_CARVEOUT
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);   // see launch_attend
  if (e != cudaSuccess) return e;
#endif
  const int grid = p.n_warps / kWarps;
  // programmatic dependent launch: the first page loads overlap attend_prologue_kernel;
  // griddepcontrol.wait in the kernel orders every read of the prologue's outputs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, fn, p, S);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace oscar
