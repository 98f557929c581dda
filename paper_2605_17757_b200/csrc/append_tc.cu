// Tensor-core quantize_append (variant 0).  Alg. 1 `Prefill` rotate-before-
// write + `QuantizeAndWrite`; §4 "KV Cache Update".
//
// Persistent CTA per (kv head, K|V) "pair" slice, 18 warps:
//   warp 0      TMA producer: 128-token x 128-channel bf16 tiles of K (or V) for one head,
//               two 64-channel SWIZZLE_128B boxes per tile, 4-stage smem ring
//   warp 1      TMEM allocator (256 columns = 2 fp32 accumulators) + single-thread tcgen05.mma
//               issuer: x̃ = [x x]·[R_hi; R_lo] as 16 UMMA 128x128x16 (bf16 -> fp32 TMEM).  The
//               bf16 hi/lo split of the fp32 R keeps rotated values within 1e-5 of the fp64
//               product; R_hi, R_lo stay resident in smem (K-major SW128).
//   warps 2-17  epilogue, 4 per TMEM lane quarter = (channel half) x (tile parity): tcgen05.ld
//               32x32b (thread = token row, 64 channels), per-group min/max, fp16 (s, m), codes
//               (reading Z4: one FFMA + bit clamp per code), pack, store into the slot's page
//               block (FORMAT, common.cuh); V codes of whole 16-token tiles are staged in smem in
//               FORMAT order and written as 16-B chunks.
// Scope of this kernel: b in {2, 3, 4}, G in {32, 64, 128} (a G = 128 group spans the two channel
// halves: the two warps swap min/max through smem), no clipping; other configs use the simple
// kernel (append.cu).
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace oscar {

namespace {

#ifndef OSCAR_TREE_MINMAX
#define OSCAR_TREE_MINMAX 0      // 1: tree min/max (measured slower: 611 vs 586 us, C2 prefill)
#endif
constexpr int kTok = 128;          // tokens per tile (UMMA M)
constexpr int kStages = 4;
#ifndef OSCAR_APPEND_L2PF
#define OSCAR_APPEND_L2PF 0
#endif
#ifndef OSCAR_APPEND_ACC
#define OSCAR_APPEND_ACC 2
#endif
#ifndef OSCAR_APPEND_N256
#define OSCAR_APPEND_N256 1      // C2 prefill (2-bit, G = 64): 0.576 -> 0.549 ms (same-box A/B)
#endif
constexpr int kAcc = OSCAR_APPEND_ACC;          // TMEM fp32 accumulators (128 columns each; N256: 256)
constexpr int kEpiWarps = 16;                   // 4 per TMEM lane quarter: (channel half, tile parity)
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kTileBytes = kTok * kD * 2;       // 32 KB bf16 tile
constexpr int kBBytes = kD * kD * 2;            // 32 KB bf16 R part

#ifndef OSCAR_VSTAGE_PAD
#define OSCAR_VSTAGE_PAD 64      // 64 B: the two staged tiles of a half-warp pair land on disjoint banks (4-bit 0.629 -> 0.625 ms)
#endif
constexpr int kVStage = 2 * (16 * 64 + OSCAR_VSTAGE_PAD);   // V codes of one 32-token quarter (b <= 4), 2 padded tiles

struct TcSmem {
  alignas(1024) uint8_t Bhi[kBBytes];           // [2 k-chunks][128 rows n][128 B], SW128
  alignas(1024) uint8_t Blo[kBBytes];
  alignas(1024) uint8_t A[kStages][kTileBytes]; // [stage][2 k-chunks][128 rows tok][128 B]
  alignas(16) uint8_t vstage[2][4][kVStage];    // per (tile parity, lane quarter): FORMAT-ordered V codes
  float2 xch[2][2][4][2][32];                   // G = 128: (buffer, parity, quarter, half, lane) min/max
  uint64_t full[kStages], empty[kStages], tfull[kAcc], tempty[kAcc];
  uint32_t tmem_base;
};

using namespace ptx;
// instruction descriptor: kind::f16, A = B = BF16, D = F32, both K-major, M = 128, N = 128
constexpr uint32_t kIdesc = idesc_bf16(128, 128, false, false);
// N256 (MODE 0 / 1): one UMMA 128x256x16 per k-step against B = [R_hi | R_lo] side by side along N
// (D = [x·R_hi | x·R_lo], the epilogue adds the halves): half the MMA instructions and a quarter
// less shared-memory operand traffic than two 128x128x16 passes (A is read once per k-step)
constexpr uint32_t kIdesc256 = idesc_bf16(128, 256, false, false);

struct TcParams {
  const int64_t* slots;
  int64_t T;
  const float* RK;
  const float* RV;
  uint8_t* pool;
  int hkv, P, page_bytes, row_bytes, vcodes_off, meta_off, ng, G, bits;
  int cpp, tiles_per_pair;
  int lgP;                          // log2(P) if P is a power of two, else -1
  // test hooks (MODE != 0): fp32 rotated rows in (MODE 2) / out (MODE 1), [T][hkv][128]
  const float* xin_k;
  const float* xin_v;
  float* rot_out;
};

// Σ_i 0x4B400000 << (BITS·i) mod 2^32 over the codes of one 32-bit word: the constant part of
// the accumulated magic-add float bits
template <int BITS>
__device__ __forceinline__ constexpr uint32_t magic_words() {
  uint32_t k = 0;
  for (int i = 0; i < 32 / BITS; ++i) k += 0x4B400000u << (BITS * i);
  return k;
}

// packed fp32x2 arithmetic (one issue slot for two lanes of math; each lane rounds as the
// scalar instruction would: the results are bit-identical to FADD / FFMA)
__device__ __forceinline__ uint64_t pk2(uint32_t a, uint32_t b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ void unpk2(uint64_t r, uint32_t& a, uint32_t& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// packed f32x2 epilogue arithmetic, same-box A/B at the C2 prefill shape (scalar vs f32x2, ms):
// 2-bit G = 64 0.557 vs 0.573; G = 32 0.604 vs 0.592; G = 128 0.619 vs 0.594; 3-bit G = 64 0.658 vs
// 0.647; 4-bit G = 64 0.626 vs 0.623; G = 32 0.647 vs 0.625 -> on except for 2-bit G = 64
#ifndef OSCAR_APPEND_F2
#define OSCAR_APPEND_F2 (!(BITS == 2 && G == 64))
#endif
#ifndef OSCAR_APPEND_F2ADD
#define OSCAR_APPEND_F2ADD OSCAR_APPEND_F2     // the x·R_hi + x·R_lo sum alone as f32x2
#endif

}  // namespace

// MODE 0: production (TMA -> tcgen05 rotation -> quantize/pack/store epilogue).
// MODE 1 (oscar_rotate hook): TMA -> tcgen05 rotation; the epilogue warps write the TMEM rows
//        they would quantize as fp32 x̃ (K half only: one "pair" per head).
// MODE 2 (oscar_quantize_rotated hook): no TMA / MMA; the epilogue warps take the given fp32 x̃
//        rows in place of the TMEM load and run the identical quantize/pack/store code.
// MODE 3 (oscar_rotate_fwht): the north star's alternative rotation form, x̃ = ((x·U)·H)·P_br
//        (Eq. 3, App A.1): the same tcgen05 GEMM with U (the sorted
//        eigenvectors, hi/lo bf16) in place of R, then per row the Walsh–Hadamard transform in
//        registers — the stride-64 butterfly first (H_128 = H_2 ⊗ H_64: each thread reads its own
//        and its partner half's TMEM columns, no exchange), then strides 1..32 over the thread's
//        64 values — the 1/√128 scale and the bit-reversed column scatter out[j] = z[β(j)].
//        Written as fp32 rows like MODE 1, so the two rotation forms compare stage for stage.
template <int BITS, int G, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
append_tc_kernel(const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PDL: a following kernel may launch now (the attend prologue is launched without PDL and so
  // still starts after this kernel completes)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int pair = blockIdx.x / p.cpp, sub = blockIdx.x % p.cpp;
  const int h = (MODE == 1 || MODE == 3) ? pair : pair >> 1, isV = (MODE == 1 || MODE == 3) ? 0 : pair & 1;
  const int ntiles = sub < p.tiles_per_pair ? (p.tiles_per_pair - sub + p.cpp - 1) / p.cpp : 0;
  // (4-bit G = 32, the heaviest epilogue, stays on two N = 128 passes: 0.632 vs 0.640 ms)
  constexpr bool N256 = OSCAR_APPEND_N256 && MODE != 3 && !(BITS == 4 && G == 32);
  constexpr int kAccCols = N256 ? 256 : 128;    // TMEM columns per accumulator

  // ---- R -> bf16 hi/lo, transposed to K-major (row n = output channel, k contiguous), SW128
  {
    // R_V = NULL: pre-rotated V (NEXT-2) -> identity (exact in bf16: R_lo = 0)
    const float* Rb = isV ? p.RV : p.RK;
    const float* R = Rb ? Rb + (size_t)h * kD * kD : nullptr;
    for (int idx = threadIdx.x; idx < kD * 16; idx += kThreads) {
      const int n = idx & 127, kc16 = idx >> 7;            // 16 chunks of 8 k
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k0 = 8 * kc16 + 2 * e, k1 = k0 + 1;
        const float r0 = R ? R[(size_t)k0 * kD + n] : (k0 == n ? 1.f : 0.f);
        const float r1 = R ? R[(size_t)k1 * kD + n] : (k1 == n ? 1.f : 0.f);
        const __nv_bfloat16 h0 = __float2bfloat16_rn(r0), h1 = __float2bfloat16_rn(r1);
        const __nv_bfloat16 l0 = __float2bfloat16_rn(r0 - __bfloat162float(h0));
        const __nv_bfloat16 l1 = __float2bfloat16_rn(r1 - __bfloat162float(h1));
        hi[e] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
        lo[e] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
      }
      const int kchunk = kc16 >> 3, c16 = kc16 & 7;
      if (N256) {
        // [2 k-chunks][256 rows: R_hi columns, then R_lo columns][128 B] across Bhi ‖ Blo
        const int off = kchunk * (2 * kD * 128) + n * 128 + ((c16 ^ (n & 7)) << 4);
        *reinterpret_cast<uint4*>(S.Bhi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(S.Bhi + off + kD * 128) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      } else {
        const int off = kchunk * (kD * 128) + n * 128 + ((c16 ^ (n & 7)) << 4);
        *reinterpret_cast<uint4*>(S.Bhi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(S.Blo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], 1); }
    for (int a = 0; a < kAcc; ++a) { mbar_init(&S.tfull[a], 1); mbar_init(&S.tempty[a], kEpiWarps / 2); }
  }
  if (warp == 1) tmem_alloc(&S.tmem_base, kAccCols * kAcc);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // B writes -> async proxy
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ================= TMA producer
    if (MODE != 2 && lane == 0) {
      const CUtensorMap* map = isV ? &mapV : &mapK;
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        mbar_wait(&S.empty[s], ((i / kStages) & 1) ^ 1);
        mbar_expect_tx(&S.full[s], kTileBytes);
        const int tok0 = (sub + i * p.cpp) * kTok;
        tma_load_3d(S.A[s], map, 0, h, tok0, &S.full[s]);
        tma_load_3d(S.A[s] + kTileBytes / 2, map, 64, h, tok0, &S.full[s]);
        if (OSCAR_APPEND_L2PF > 0 && i + OSCAR_APPEND_L2PF < ntiles) {
          // the ring holds only kStages tiles: pull the tile OSCAR_APPEND_L2PF ahead into L2 so
          // its TMA load later sees L2 rather than DRAM latency
          const int tokp = (sub + (i + OSCAR_APPEND_L2PF) * p.cpp) * kTok;
          tma_prefetch_3d(map, 0, h, tokp);
          tma_prefetch_3d(map, 64, h, tokp);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    for (int i = 0; i < (MODE == 2 ? 0 : ntiles); ++i) {
      const int s = i % kStages, a = i % kAcc;
      mbar_wait(&S.tempty[a], ((i / kAcc) & 1) ^ 1);
      mbar_wait(&S.full[s], (i / kStages) & 1);
      fence_after();
      if (lane == 0) {
        const uint32_t dt = tmem + a * kAccCols;
        const uint32_t abase = su32(S.A[s]), bh = su32(S.Bhi), bl = su32(S.Blo);
#ifndef OSCAR_PROBE_PARTS
#define OSCAR_PROBE_PARTS 2      // timing probe only: 1 = the R_hi pass alone (results invalid)
#endif
        if (N256) {
#pragma unroll
          for (int kc = 0; kc < 2; ++kc)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_f16<kIdesc256>(dt, kmajor_sw128_desc(abase + kc * (kTileBytes / 2) + kk * 32),
                                  kmajor_sw128_desc(bh + kc * (2 * kD * 128) + kk * 32), (kc | kk) != 0);
        }
#pragma unroll
        for (int part = 0; part < (N256 ? 0 : OSCAR_PROBE_PARTS); ++part) {
          const uint32_t bbase = part ? bl : bh;
#pragma unroll
          for (int kc = 0; kc < 2; ++kc)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t ko = kc * (kTileBytes / 2) + kk * 32;
              umma_f16<kIdesc>(dt, kmajor_sw128_desc(abase + ko),
                               kmajor_sw128_desc(bbase + kc * (kBBytes / 2) + kk * 32), (part | kc | kk) != 0);
            }
        }
        umma_commit(&S.empty[s]);     // smem stage free once these MMAs complete
        umma_commit(&S.tfull[a]);     // accumulator ready for the epilogue
      }
      __syncwarp();
    }
  } else {
    // ================= epilogue: thread = token row, 64 channels (half of the row); the warps
    // of a lane quarter split by (channel half, tile parity), so the two TMEM accumulators are
    // drained concurrently
    const int ew = warp - 2;
    const int quarter = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (ew >> 2) & 1;               // channels [64·half, 64·half + 64)
    const int par = ew >> 3;                      // tiles i with i % 2 == par (accumulator par)
    const int r = quarter * 32 + lane;            // row (token) within the tile
    constexpr int QMAX = (1 << BITS) - 1;
    constexpr int GH = G < 64 ? G : 64;           // channels of a group inside this half
    constexpr int GPH = 64 / GH;                  // groups (or group halves, G = 128) in this half
    int xbuf = 0;
    // slot of this thread's token, loaded one tile ahead (its latency is off the critical path)
    auto load_slot = [&](int i) -> int64_t {
      const int64_t tk = (int64_t)(sub + i * p.cpp) * kTok + r;
      return (MODE != 1 && MODE != 3 && i < ntiles && tk < p.T) ? p.slots[tk] : -1;
    };
    int64_t slot_next = load_slot(par);
    for (int i = par; i < ntiles; i += 2) {
      const int a = i % kAcc;
      const int64_t slot = slot_next;
      slot_next = load_slot(i + 2);
      uint32_t v[64];
      if constexpr (MODE == 3) {
        // z = x·U·H_128 for this row: stride-64 butterfly from both halves' TMEM columns (32 at a
        // time), then the 64-point transform of this half in registers
        mbar_wait(&S.tfull[a], (i / kAcc) & 1);
        fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + a * kAccCols;
        float y[64];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t x0[16], x1[16];
          OSCAR_TMEM_LD16(tbase + 16 * ch, x0);
          OSCAR_TMEM_LD16(tbase + 64 + 16 * ch, x1);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k)
            y[16 * ch + k] = half ? __uint_as_float(x0[k]) - __uint_as_float(x1[k])
                                  : __uint_as_float(x0[k]) + __uint_as_float(x1[k]);
        }
        fence_before();
        // both halves read this accumulator: the arrival count of tempty is one per epilogue warp
        // of this parity (kEpiWarps / 2), as in the other modes
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.tempty[a]);
#pragma unroll
        for (int st = 1; st < 64; st <<= 1)
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (!(c & st)) {
              const float u0 = y[c], u1 = y[c + st];
              y[c] = u0 + u1;
              y[c + st] = u0 - u1;
            }
        const int64_t tk = (int64_t)(sub + i * p.cpp) * kTok + r;
        if (tk < p.T) {
          float* dst = p.rot_out + (tk * p.hkv + h) * kD;
          constexpr float kNorm = 0.08838834764831845f;   // 1/sqrt(128)
          // out[j] = z[β(j)]: z index 64·half + c lands on column j = β(64·half + c)
#pragma unroll
          for (int c = 0; c < 64; ++c) dst[__brev((unsigned)(64 * half + c)) >> 25] = y[c] * kNorm;
        }
        continue;
      }
      if constexpr (MODE != 2) {
        mbar_wait(&S.tfull[a], (i / kAcc) & 1);
        fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + a * kAccCols + half * 64;
        if (N256) {
          // x̃ = x·R_hi + x·R_lo: columns c and 128 + c of the accumulator
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t lo16[16];
            OSCAR_TMEM_LD16(taddr + 16 * q4, (v + 16 * q4));
            OSCAR_TMEM_LD16(taddr + 128 + 16 * q4, lo16);
            tmem_ld_wait();
            if (OSCAR_APPEND_F2ADD) {
#pragma unroll
              for (int k = 0; k < 16; k += 2)
                unpk2(fadd2(pk2(v[16 * q4 + k], v[16 * q4 + k + 1]), pk2(lo16[k], lo16[k + 1])), v[16 * q4 + k],
                      v[16 * q4 + k + 1]);
            } else {
#pragma unroll
              for (int k = 0; k < 16; ++k)
                v[16 * q4 + k] = __float_as_uint(__uint_as_float(v[16 * q4 + k]) + __uint_as_float(lo16[k]));
            }
          }
        } else {
          OSCAR_TMEM_LD32(taddr, v);
          OSCAR_TMEM_LD32(taddr + 32, (v + 32));
          tmem_ld_wait();
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.tempty[a]);
      } else {
        // hook: the given fp32 x̃ row (zeros past T) in place of the TMEM accumulator
        const int64_t tk = (int64_t)(sub + i * p.cpp) * kTok + r;
        const float* src = (isV ? p.xin_v : p.xin_k) + (tk * p.hkv + h) * kD + half * 64;
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 f = tk < p.T ? reinterpret_cast<const float4*>(src)[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * c4] = __float_as_uint(f.x); v[4 * c4 + 1] = __float_as_uint(f.y);
          v[4 * c4 + 2] = __float_as_uint(f.z); v[4 * c4 + 3] = __float_as_uint(f.w);
        }
      }
      if constexpr (MODE == 1) {
        // hook: the rotated row as the epilogue sees it (fp32 TMEM values)
        const int64_t tk = (int64_t)(sub + i * p.cpp) * kTok + r;
        if (tk < p.T) {
          float4* dst = reinterpret_cast<float4*>(p.rot_out + (tk * p.hkv + h) * kD + half * 64);
#pragma unroll
          for (int c4 = 0; c4 < 16; ++c4)
            dst[c4] = make_float4(__uint_as_float(v[4 * c4]), __uint_as_float(v[4 * c4 + 1]),
                                  __uint_as_float(v[4 * c4 + 2]), __uint_as_float(v[4 * c4 + 3]));
        }
        continue;
      }

#ifdef OSCAR_PROBE_NOEPI
      if (v[0] != 0x7fffffffu) continue;           // timing probe only: TMEM drained, nothing stored
#endif
      const bool valid = slot >= 0;
      // V fast path: the quarter's 32 tokens go to 32 consecutive slots starting on a 16-token
      // tile, i.e. two whole 16-token FORMAT tiles -> stage the FORMAT-ordered bytes in smem and
      // write 16-B chunks.  Both warps of the quarter (the two channel halves) see the same rows,
      // so they take the same branch and meet at the same named barrier.
      const int64_t slot0 = __shfl_sync(0xffffffffu, slot, 0);
      const bool fastV = isV && __all_sync(0xffffffffu, valid && slot == slot0 + lane && (slot0 & 15) == 0);
      // (G = 128: rows past T still take part in the partner exchange below; they store nothing)
      if (!valid && G != 128) continue;
      // (page, offset) of the slot: shift / mask when P is a power of two (the 64-bit division
      // costs ~40 instructions per row)
      const int64_t page = !valid ? 0 : (p.lgP >= 0 ? (slot >> p.lgP) : slot / p.P);
      const int u = !valid ? 0 : (p.lgP >= 0 ? (int)(slot & (p.P - 1)) : (int)(slot % p.P));
      uint8_t* blk = p.pool + (page * p.hkv + h) * (int64_t)p.page_bytes;
      // codes: the magic add leaves float bits 0x4B400000 + code; accumulate bits << shift with
      // one LEA per code and remove the constant part once per word.
      // b = 3 (reading Z36 planes): packed[0..3] = this half's 16 low-plane bytes (the 2-bit
      // stream of code & 3), packed[4..5] = its 8 high-plane bytes (channel 64·half + idx: high
      // bit at bit 8·((idx % 16) / 4) + 4·((idx / 16) % 2) + idx % 4 of word idx / 32)
      uint32_t packed[BITS * 2];
#pragma unroll
      for (int w = 0; w < BITS * 2; ++w) packed[w] = BITS == 3 ? 0u : 0u - magic_words<BITS>();
      auto put = [&](int idx, uint32_t fbits) {
        if (BITS == 3) {
          packed[idx >> 4] |= (fbits & 3u) << (2 * (idx & 15));
          packed[4 + (idx >> 5)] |= ((fbits >> 2) & 1u) << (8 * ((idx & 15) >> 2) + 4 * ((idx >> 4) & 1) + (idx & 3));
        } else {
          const int bit = idx * BITS, wd = bit >> 5, sh = bit & 31;
          packed[wd] += fbits << sh;
        }
      };
      // row byte of this half's packed byte jb (b = 3: low plane 16·half + jb, then high plane)
      auto row_byte = [&](int jb) -> int {
        if (BITS == 3) return jb < 16 ? 16 * half + jb : 32 + 8 * half + (jb - 16);
        return half * (8 * BITS) + jb;
      };
#pragma unroll
      for (int gi = 0; gi < GPH; ++gi) {
#if OSCAR_TREE_MINMAX
        // min / max as balanced trees (depth log2 GH instead of a GH-long dependency chain)
        float tmn[GH / 2], tmx[GH / 2];
#pragma unroll
        for (int c = 0; c < GH / 2; ++c) {
          const float x0 = __uint_as_float(v[gi * GH + 2 * c]), x1 = __uint_as_float(v[gi * GH + 2 * c + 1]);
          tmn[c] = fminf(x0, x1);
          tmx[c] = fmaxf(x0, x1);
        }
#pragma unroll
        for (int w = GH / 4; w >= 1; w >>= 1)
#pragma unroll
          for (int c = 0; c < w; ++c) {
            tmn[c] = fminf(tmn[c], tmn[c + w]);
            tmx[c] = fmaxf(tmx[c], tmx[c + w]);
          }
        float mn = tmn[0], mx = tmx[0];
#else
        float mn = __uint_as_float(v[gi * GH]), mx = mn;
#pragma unroll
        for (int c = 1; c < GH; ++c) {
          const float x = __uint_as_float(v[gi * GH + c]);
          mn = fminf(mn, x);
          mx = fmaxf(mx, x);
        }
#endif
        if (G == 128) {
          // the group spans both channel halves: swap min/max with the partner warp (same rows)
          S.xch[xbuf][par][quarter][half][lane] = make_float2(mn, mx);
          asm volatile("bar.sync %0, 64;\n" ::"r"(1 + quarter + 4 * par) : "memory");
          const float2 o = S.xch[xbuf][par][quarter][half ^ 1][lane];
          mn = fminf(mn, o.x);
          mx = fmaxf(mx, o.y);
          xbuf ^= 1;
        }
        const float s = __fdiv_rn(__fsub_rn(mx, mn), (float)QMAX);
        const __half s16 = __float2half_rn(s), m16 = __float2half_rn(mn);
        const float sf = __half2float(s16), m = __half2float(m16);
        const float inv = sf > 0.f ? __fdiv_rn(1.f, sf) : 0.f;
        // reading Z4: rint(RN(x - m)·inv) with the exact product: one FFMA with the 1.5·2^23
        // magic constant (round-half-even), clamp on the float bits (same exponent).  The code
        // is monotone in x, so when the group's min and max land inside [0, q_max] no value of
        // the group needs the clamp (the usual case: only ranges below the fp16 resolution of
        // their offset can push an end out)
        const int lo_b = __float_as_int(__fmaf_rn(__fsub_rn(mn, m), inv, 12582912.f));
        const int hi_b = __float_as_int(__fmaf_rn(__fsub_rn(mx, m), inv, 12582912.f));
        if (lo_b >= 0x4B400000 && hi_b <= 0x4B400000 + QMAX) {
          if (OSCAR_APPEND_F2) {
            // the same FADD (x - m) and FFMA (·inv + magic) two values at a time
            const uint64_t nm2 = pk2(__float_as_uint(-m), __float_as_uint(-m));
            const uint64_t inv2 = pk2(__float_as_uint(inv), __float_as_uint(inv));
            const uint64_t mg2 = pk2(__float_as_uint(12582912.f), __float_as_uint(12582912.f));
#pragma unroll
            for (int c = 0; c < GH; c += 2) {
              uint32_t t0, t1;
              unpk2(ffma2(fadd2(pk2(v[gi * GH + c], v[gi * GH + c + 1]), nm2), inv2, mg2), t0, t1);
              put(gi * GH + c, t0);
              put(gi * GH + c + 1, t1);
            }
          } else {
#pragma unroll
            for (int c = 0; c < GH; ++c) {
              const float tq = __fmaf_rn(__fsub_rn(__uint_as_float(v[gi * GH + c]), m), inv, 12582912.f);
              put(gi * GH + c, __float_as_uint(tq));   // code index within the half row
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < GH; ++c) {
            const float tq = __fmaf_rn(__fsub_rn(__uint_as_float(v[gi * GH + c]), m), inv, 12582912.f);
            const uint32_t bits = (uint32_t)min(max(__float_as_int(tq), 0x4B400000), 0x4B400000 + QMAX);
            put(gi * GH + c, bits);
          }
        }
        const int grp = (half * 64 + gi * GH) / G;
        if (valid && (G < 128 || half == 0))
          *reinterpret_cast<__half2*>(blk + p.meta_off + fmt_meta(u, grp, p.ng) + (isV ? 16 : 0)) =
              __halves2half2(s16, m16);
      }
      if (!valid) continue;
      constexpr int HB = 8 * BITS;                // bytes of this half row
      constexpr int RB = 16 * BITS;               // bytes of a row
      if (!isV) {
        uint8_t* rowp = blk + fmt_krow(u) * p.row_bytes;
        if (BITS == 3) {                          // low plane 16 B, high plane 8 B of this half
          *reinterpret_cast<uint4*>(rowp + 16 * half) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          *reinterpret_cast<uint2*>(rowp + 32 + 8 * half) = make_uint2(packed[4], packed[5]);
        } else {
          uint8_t* dst = rowp + half * HB;
#pragma unroll
          for (int w4 = 0; w4 < HB / 16; ++w4)
            *reinterpret_cast<uint4*>(dst + 16 * w4) =
                make_uint4(packed[4 * w4], packed[4 * w4 + 1], packed[4 * w4 + 2], packed[4 * w4 + 3]);
        }
      } else if (fastV) {
        constexpr int TILE = 16 * RB + OSCAR_VSTAGE_PAD;   // staged 16-token tile (+ pad: bank shift)
        const uint32_t stg = su32(S.vstage[par][quarter]);
        // this token's bytes at their FORMAT offsets inside its 16-token tile (fmt_vbyte is
        // additive: the token part fmt_vbyte(u, 0) + the compile-time byte part fmt_vbyte(0, j))
        const uint32_t base = stg + (lane >> 4) * TILE + fmt_vbyte(lane & 15, 0, RB);
        auto put = [&](auto half_c) {
          constexpr int H = decltype(half_c)::value;
#pragma unroll
          for (int jb = 0; jb < HB; ++jb) {
            const int rbyte = BITS == 3 ? (jb < 16 ? 16 * H + jb : 32 + 8 * H + (jb - 16)) : H * HB + jb;
            asm volatile("st.shared.u8 [%0], %1;\n" ::"r"(base + fmt_vbyte(0, rbyte, RB)),
                         "r"(packed[jb >> 2] >> (8 * (jb & 3))) : "memory");
          }
        };
        if (half) put(std::integral_constant<int, 1>{});
        else put(std::integral_constant<int, 0>{});
        const int bar_id = 1 + quarter + 4 * par;
        asm volatile("bar.sync %0, 64;\n" ::"r"(bar_id) : "memory");
        // copy out: 2 tiles x 16·RB bytes, 16 B per thread per pass (64 threads)
        const int tp = half * 32 + lane;
#pragma unroll
        for (int pass = 0; pass < (2 * RB + 63) / 64; ++pass) {
          const int cidx = pass * 64 + tp;        // 16-B chunk within the quarter
          if (cidx >= 2 * RB) break;              // (3-bit: 96 chunks)
          const int tile = cidx / RB;             // RB chunks of 16 B per 16-token tile
          const int64_t sl = slot0 + 16 * tile;
          const int64_t pg = p.lgP >= 0 ? (sl >> p.lgP) : sl / p.P;
          const int off = p.lgP >= 0 ? (int)(sl & (p.P - 1)) : (int)(sl % p.P);
          uint8_t* dst = p.pool + (pg * p.hkv + h) * (int64_t)p.page_bytes + p.vcodes_off +
                         16 * RB * (off >> 4) + 16 * (cidx % RB);
          uint4 q;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                       : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(stg + tile * TILE + 16 * (cidx % RB)));
          *reinterpret_cast<uint4*>(dst) = q;
        }
        asm volatile("bar.sync %0, 64;\n" ::"r"(bar_id) : "memory");   // staging reusable
      } else {
        uint8_t* vb = blk + p.vcodes_off;
#pragma unroll
        for (int jb = 0; jb < HB; ++jb)
          vb[fmt_vbyte(u, row_byte(jb), p.row_bytes)] = (uint8_t)(packed[jb >> 2] >> (8 * (jb & 3)));
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc(tmem, kAccCols * kAcc);
  }
}

// ---------------------------------------------------------------- host side
namespace {
// K or V [T][hkv][128] bf16: box {64 channels, 1 head, 128 tokens}
bool make_map(CUtensorMap* m, const void* base, int64_t T, int hkv) {
  return ptx::make_bf16_map_3d(m, base, T, hkv, 1, kTok);
}

using TcFn = void (*)(CUtensorMap, CUtensorMap, TcParams);
template <int MODE>
TcFn pick(int bits, int G) {
#define OSCAR_TC(B_, G_) if (bits == B_ && G == G_) return append_tc_kernel<B_, G_, MODE>;
  OSCAR_TC(2, 32) OSCAR_TC(2, 64) OSCAR_TC(2, 128)
  OSCAR_TC(3, 32) OSCAR_TC(3, 64) OSCAR_TC(3, 128)
  OSCAR_TC(4, 32) OSCAR_TC(4, 64) OSCAR_TC(4, 128)
#undef OSCAR_TC
  return nullptr;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}  // namespace

// The tensor-core kernel covers every (b, G) without clipping; TMA needs 16-B aligned row bases
// (callers fall back to the simple kernel otherwise, api.cu).
bool append_tc_supported(const oscar_ctx& c) {
  return c.d == 128 && c.clip_k_idx < 0 && c.clip_v_idx < 0 && pick<0>(c.bits, c.G) != nullptr &&
         ptx::encode_tiled_fn() != nullptr;
}
bool append_tc_aligned(const void* K, const void* V) { return aligned16(K) && aligned16(V); }

// mode 0: quantize_append(K, V); mode 1: rotate hook (K = X, R_K = R, fp32 rows to rot_out);
// mode 2: quantize_rotated hook (xin_k, xin_v fp32 rows, no rotation)
cudaError_t launch_append_tc(const oscar_ctx& c, int mode, const void* K, const void* V, const float* xin_k,
                             const float* xin_v, const int64_t* slots, int64_t T, const float* RK,
                             const float* RV, void* pool, float* rot_out, cudaStream_t s) {
  // (MODE 3 writes only rotated rows: one instance serves every (b, G))
  TcFn fn = mode == 0 ? pick<0>(c.bits, c.G) : mode == 1 ? pick<1>(c.bits, c.G)
          : mode == 2 ? pick<2>(c.bits, c.G) : append_tc_kernel<2, 64, 3>;
  if (!fn) return cudaErrorNotSupported;
  CUtensorMap mk{}, mv{};
  if (mode != 2) {
    if (!aligned16(K) || !aligned16(V)) return cudaErrorMisalignedAddress;
    if (!make_map(&mk, K, T, c.hkv) || !make_map(&mv, V, T, c.hkv)) return cudaErrorInvalidValue;
  }
  TcParams p{};
  p.slots = slots; p.T = T; p.RK = RK; p.RV = RV; p.pool = static_cast<uint8_t*>(pool);
  p.hkv = c.hkv; p.P = c.P; p.page_bytes = c.page_bytes; p.row_bytes = c.row_bytes;
  p.vcodes_off = c.vcodes_off; p.meta_off = c.meta_off; p.ng = c.ng; p.G = c.G; p.bits = c.bits;
  p.xin_k = xin_k; p.xin_v = xin_v; p.rot_out = rot_out;
  p.lgP = -1;
  for (int k = 0; k < 16; ++k)
    if ((1 << k) == c.P) p.lgP = k;
  const int pairs = (mode == 1 || mode == 3) ? c.hkv : 2 * c.hkv;
  p.tiles_per_pair = (int)((T + kTok - 1) / kTok);
  int cpp = c.num_sms / pairs;
  if (cpp < 1) cpp = 1;
  if (cpp > p.tiles_per_pair) cpp = p.tiles_per_pair;
  p.cpp = cpp;
  const int smem = (int)sizeof(TcSmem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  fn<<<pairs * cpp, kThreads, smem, s>>>(mk, mv, p);
  return cudaGetLastError();
}

}  // namespace oscar
