// On-device S·V for the C_S target on the 5th-generation tensor cores (variant 0; SURVEY §8(f)
// NEXT-3; Alg. 1 `Calibrate` P:L1604-1606: S = softmax(Q Kᵀ/√d + M), C_S from S·V).
// Reading Z16: M is causal including the diagonal and block-diagonal across the calibration
// sequences; query head i uses KV head i/g.  Same result as calib_sv.cu (the mma.sync kernel,
// variant 1) up to fp32 summation order: P is rounded to bf16 before the P·V product in both.
//
// Persistent: one CTA per SM walks the (128-query block, query head) items, longest key ranges
// first, its rings' phases running on across items (Q and O are handed over through qempty /
// oempty).  One item = 128 queries of one query head; 10 warps:
//   warp 8  TMA producer: the Q tile once, then 128-key K and V tiles (two 64-channel SWIZZLE_128B
//           boxes each) into a 3-stage K ring (a stage frees once its Q·Kᵀ completes) and a 2-stage
//           V ring (freed by its P·V)
//   warp 9  TMEM allocator + single-thread tcgen05.mma issuer:
//             S_j  = Q·K_jᵀ      (A = Q K-major, B = K_j K-major)   -> TMEM columns 128·(j % 2)
//             O   += P_j·V_j     (A = P_j from TMEM, B = V_j MN-major) -> TMEM columns 256..383
//   warps 0-7  softmax (thread = query row = TMEM lane; warps q and q + 4 take key columns 0-63 /
//           64-127 of the rows of lane quarter q, combining max and sum through smem): per key block, pass 1 reads S and forms
//           the masked row max; the running max m moves only when the block max exceeds it by more
//           than 2^8 (then O is rescaled in TMEM by exp2(m_old - m_new)), otherwise P ≤ 2^8 stays
//           exact in range for bf16; pass 2 writes P = exp2(S·scale·log2e - m) as bf16 into one
//           of two TMEM P buffers (columns 384 / 448) the P·V MMA reads as its A operand, and sums
//           l.  At the end O / l -> SV bf16.
#include "common.cuh"
#include "ptx.cuh"

namespace oscar {

namespace {
using namespace ptx;

constexpr int kSvQ = 128;                     // queries per CTA (UMMA M)
constexpr int kSvK = 128;                     // keys per block
constexpr int kSvHalf = 128 * 128;            // one 64-channel (or 64-key) half tile: 128 rows x 128 B
constexpr int kSvThreads = 10 * 32;
constexpr int kSvStages = 3;                  // K ring (a stage frees once its Q·Kᵀ completes)
constexpr int kSvVStages = 2;                 // V ring (a stage frees once its P·V completes)
#ifndef OSCAR_SV_RESCALE_THR
#define OSCAR_SV_RESCALE_THR 8.f
#endif
constexpr float kRescaleThr = OSCAR_SV_RESCALE_THR;   // log2 units

struct SvSmem {
  alignas(1024) uint8_t Q[2][kSvHalf];        // [channel half][query row][128 B]
  alignas(1024) uint8_t K[kSvStages][2][kSvHalf];   // [stage][channel half][key row][128 B]
  alignas(1024) uint8_t V[kSvVStages][2][kSvHalf];  // [stage][channel half][key row][128 B]
  uint64_t qfull, kfull[kSvStages], kempty[kSvStages], vfull[kSvVStages], vempty[kSvVStages];
  uint64_t sfull[2], sempty[2], pfull[2], pvdone[2], qempty, oempty;
  uint32_t tmem_base;
  float xmax[2][2][128];                      // [block parity][column half][row] softmax max exchange
  float xl[2][128];                           // [column half][row] final row sums
};

constexpr uint32_t kIdescS = idesc_bf16(128, 128, false, false);   // A, B K-major
constexpr uint32_t kIdescPV = idesc_bf16(128, 128, false, true);   // B (V) MN-major

constexpr uint32_t kPCol = 384;               // TMEM columns of the two P buffers (64 each)

// sequence containing token n: the last s with starts[s] <= n
__device__ __forceinline__ int sv_seq_start(const int32_t* starts, int n_seq, int n) {
  int lo = 0, hi = n_seq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (starts[mid] <= n) lo = mid; else hi = mid - 1;
  }
  return starts[lo];
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

struct SvParams {
  const int32_t* starts;
  int n_seq, N, hq, hkv, nqb;
  float scale_log2;
  uint16_t* SV;
};
}  // namespace

__global__ void __launch_bounds__(kSvThreads, 1)
calib_sv_tc_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                   const __grid_constant__ CUtensorMap mapV, SvParams p) {
  extern __shared__ uint8_t smem_raw[];
  SvSmem& S = *reinterpret_cast<SvSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent: this CTA takes items it = blockIdx.x, blockIdx.x + gridDim.x, ... of the
  // (query block, query head) list, longest key ranges first; the rings' phases run on across
  // items (J = blocks this CTA has processed)
  const int n_items = p.nqb * p.hq;
  auto item = [&](int it, int& q0, int& qh, int& kbeg, int& nblk) {
    const int qb = p.nqb - 1 - it / p.hq;
    qh = it % p.hq;
    q0 = qb * kSvQ;
    const int qlast = min(q0 + kSvQ, p.N) - 1;
    kbeg = sv_seq_start(p.starts, p.n_seq, q0);
    nblk = (qlast - kbeg) / kSvK + 1;
  };

  if (threadIdx.x == 0) {
    mbar_init(&S.qfull, 1);
    mbar_init(&S.qempty, 1);
    mbar_init(&S.oempty, 8);
    for (int s = 0; s < kSvStages; ++s) { mbar_init(&S.kfull[s], 1); mbar_init(&S.kempty[s], 1); }
    for (int s = 0; s < kSvVStages; ++s) { mbar_init(&S.vfull[s], 1); mbar_init(&S.vempty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&S.sfull[s], 1); mbar_init(&S.sempty[s], 8); }
    for (int s = 0; s < 2; ++s) { mbar_init(&S.pfull[s], 8); mbar_init(&S.pvdone[s], 1); }
    mbar_init_fence();
  }
  if (warp == 9) tmem_alloc(&S.tmem_base, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 8) {
    // ================= TMA producer
    if (lane == 0) {
      int J = 0, n = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
        int q0, qh, kbeg, nblk;
        item(it, q0, qh, kbeg, nblk);
        const int h = qh / (p.hq / p.hkv);
        if (n >= 1) mbar_wait(&S.qempty, (n - 1) & 1);   // the previous item's Q·Kᵀ are done
        mbar_expect_tx(&S.qfull, 2 * kSvHalf);
        tma_load_3d(S.Q[0], &mapQ, 0, qh, q0, &S.qfull);
        tma_load_3d(S.Q[1], &mapQ, 64, qh, q0, &S.qfull);
        for (int j = 0; j < nblk; ++j, ++J) {
          const int s = J % kSvStages, ph = ((J / kSvStages) & 1) ^ 1, key0 = kbeg + j * kSvK;
          mbar_wait(&S.kempty[s], ph);
          mbar_expect_tx(&S.kfull[s], 2 * kSvHalf);
          tma_load_3d(S.K[s][0], &mapK, 0, h, key0, &S.kfull[s]);
          tma_load_3d(S.K[s][1], &mapK, 64, h, key0, &S.kfull[s]);
          const int vs = J % kSvVStages;
          mbar_wait(&S.vempty[vs], ((J / kSvVStages) & 1) ^ 1);
          mbar_expect_tx(&S.vfull[vs], 2 * kSvHalf);
          tma_load_3d(S.V[vs][0], &mapV, 0, h, key0, &S.vfull[vs]);
          tma_load_3d(S.V[vs][1], &mapV, 64, h, key0, &S.vfull[vs]);
        }
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer: S_j, then P_{j-1}·V_{j-1}
    int J0 = 0, n = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
      int q0, qh, kbeg, nblk;
      item(it, q0, qh, kbeg, nblk);
      mbar_wait(&S.qfull, n & 1);
      for (int j = 0; j <= nblk; ++j) {
        if (j < nblk) {
          const int J = J0 + j, s = J & 1, ks = J % kSvStages;
          mbar_wait(&S.kfull[ks], (J / kSvStages) & 1);
          mbar_wait(&S.sempty[s], ((J >> 1) & 1) ^ 1);
          fence_after();
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_f16<kIdescS>(tmem + 128 * s, kmajor_sw128_desc(su32(S.Q[kk >> 2]) + (kk & 3) * 32),
                                kmajor_sw128_desc(su32(S.K[ks][kk >> 2]) + (kk & 3) * 32), kk != 0);
            umma_commit(&S.sfull[s]);
            umma_commit(&S.kempty[ks]);     // K_j consumed
            if (j == nblk - 1) umma_commit(&S.qempty);   // Q free for the next item
          }
          __syncwarp();
        }
        if (j >= 1) {
          const int jj = j - 1, JJ = J0 + jj, s = JJ % kSvVStages;
          mbar_wait(&S.vfull[s], (JJ / kSvVStages) & 1);
          mbar_wait(&S.pfull[JJ & 1], (JJ >> 1) & 1);
          // the first P·V of an item overwrites O: the previous item's O must have been read
          if (jj == 0 && n >= 1) mbar_wait(&S.oempty, (n - 1) & 1);
          fence_after();
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_f16_ts<kIdescPV>(tmem + 256, tmem + kPCol + 64 * (JJ & 1) + 8 * kk,
                                    mnmajor_sw128_desc(su32(S.V[s][0]) + kk * 2048, kSvHalf), (jj | kk) != 0);
            umma_commit(&S.vempty[s]);      // V_jj consumed
            umma_commit(&S.pvdone[JJ & 1]); // O holds blocks 0..jj; P buffer JJ % 2 free
          }
          __syncwarp();
        }
      }
      J0 += nblk;
    }
  } else {
    // ================= softmax: thread = query row r, key / channel columns [64·ch, 64·ch + 64)
    // (two warps per TMEM lane quarter: warps q and q + 4 split the row's columns; the row max and
    // the row sum are combined through shared memory, named barrier 1 + q)
    const int quarter = warp & 3, ch = warp >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const int cb = 64 * ch;                          // first column of this warp
    int J0 = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    int q0, qh, kbeg, nblk;
    item(it, q0, qh, kbeg, nblk);
    const int qi = q0 + r;
    const bool live = qi < p.N;
    const int lo = live ? sv_seq_start(p.starts, p.n_seq, qi) : 0x7fffffff;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int J = J0 + j, b = J & 1, key0 = kbeg + j * kSvK;
      mbar_wait(&S.sfull[b], (J >> 1) & 1);
      fence_after();
      // keys key0 + c valid for this row: lo <= key <= qi
      const int cmin = lo - key0, cmax = live ? qi - key0 : -1;
      // columns every row of the warp may see in full (the usual case below the diagonal) take the
      // unmasked loops
      const bool full = __all_sync(0xffffffffu, cmin <= cb && cmax >= cb + 63);
      // pass 1: masked max of this half (log2 units; scale > 0, so max(s)·scale = max(s·scale))
      float bm = -INFINITY;
#pragma unroll 1
      for (int c0 = cb; c0 < cb + 64; c0 += 32) {
        uint32_t v[32];
        OSCAR_TMEM_LD32(trow + 128 * b + c0, v);
        tmem_ld_wait();
        if (full) {
          float x = __uint_as_float(v[0]);
#pragma unroll
          for (int k = 1; k < 32; ++k) x = fmaxf(x, __uint_as_float(v[k]));
          bm = fmaxf(bm, x * p.scale_log2);
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int c = c0 + k;
            if (c >= cmin && c <= cmax) bm = fmaxf(bm, __uint_as_float(v[k]) * p.scale_log2);
          }
        }
      }
      S.xmax[b][ch][r] = bm;
      asm volatile("bar.sync %0, 64;\n" ::"r"(1 + quarter) : "memory");
      bm = fmaxf(bm, S.xmax[b][ch ^ 1][r]);
      // P buffer J % 2 free: P_{J-2}·V_{J-2} done (possibly the previous item's)
      if (J >= 2) {
        mbar_wait(&S.pvdone[J & 1], ((J >> 1) - 1) & 1);
        fence_after();
      }
      // (both warps of the row take the same decision; the TMEM load / store below are
      // warp-collective: the rescale runs for the whole warp, lanes that keep their max multiply
      // by 1)
      const bool upd = bm > m + kRescaleThr || (m == -INFINITY && bm > -INFINITY);
      const bool resc = upd && m != -INFINITY;
      float a = 1.f;
      if (resc) { a = ex2(m - bm); l *= a; }
      if (upd) m = bm;
      if (__any_sync(0xffffffffu, resc)) {
        // O holds blocks 0..j-1 once P_{j-1}·V_{j-1} is done (the MMAs complete in issue order)
        if (j >= 1) {
          mbar_wait(&S.pvdone[(J - 1) & 1], ((J - 1) >> 1) & 1);
          fence_after();
        }
#pragma unroll 1
        for (int c0 = cb; c0 < cb + 64; c0 += 32) {
          uint32_t o[32];
          OSCAR_TMEM_LD32(trow + 256 + c0, o);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * a);
          OSCAR_TMEM_ST32(trow + 256 + c0, o);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      }
      // pass 2: P = exp2(s·scale - m) (0 where masked) as bf16 into P[key half ch][row r]
#pragma unroll 1
      for (int c0 = cb; c0 < cb + 64; c0 += 32) {
        uint32_t v[32];
        OSCAR_TMEM_LD32(trow + 128 * b + c0, v);
        tmem_ld_wait();
        uint32_t pk[16];
        if (full) {
          float l0 = 0.f, l1 = 0.f;
#pragma unroll
          for (int k = 0; k < 32; k += 2) {
            const float p0 = ex2(fmaf(__uint_as_float(v[k]), p.scale_log2, -m));
            const float p1 = ex2(fmaf(__uint_as_float(v[k + 1]), p.scale_log2, -m));
            l0 += p0; l1 += p1;
            pk[k >> 1] = pack_bf16x2(p0, p1);
          }
          l += l0 + l1;
        } else {
#pragma unroll
          for (int k = 0; k < 32; k += 2) {
            const int c = c0 + k;
            const float p0 = (c >= cmin && c <= cmax) ? ex2(__uint_as_float(v[k]) * p.scale_log2 - m) : 0.f;
            const float p1 = (c + 1 >= cmin && c + 1 <= cmax) ? ex2(__uint_as_float(v[k + 1]) * p.scale_log2 - m) : 0.f;
            l += p0 + p1;
            pk[k >> 1] = pack_bf16x2(p0, p1);
          }
        }
        // keys c0 .. c0 + 31 -> TMEM columns kPCol + 64·(j % 2) + c0 / 2 .. + 15 of this lane
        OSCAR_TMEM_ST16(trow + kPCol + 64 * (J & 1) + c0 / 2, pk);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.sempty[b]);
        mbar_arrive(&S.pfull[J & 1]);
      }
    }
    // row sum of both halves, then O / l -> SV bf16 [N][H_q][128] (this warp's 64 channels)
    S.xl[ch][r] = l;
    asm volatile("bar.sync %0, 64;\n" ::"r"(1 + quarter) : "memory");
    l += S.xl[ch ^ 1][r];
    const int JL = J0 + nblk - 1;                     // this item's last block
    mbar_wait(&S.pvdone[JL & 1], (JL >> 1) & 1);
    fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    uint16_t* dst = p.SV + ((size_t)qi * p.hq + qh) * kD;
#pragma unroll 1
    for (int c0 = cb; c0 < cb + 64; c0 += 32) {
      uint32_t o[32];
      OSCAR_TMEM_LD32(trow + 256 + c0, o);
      tmem_ld_wait();
      if (live) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          reinterpret_cast<uint4*>(dst + c0)[q] = make_uint4(
              pack_bf16x2(__uint_as_float(o[8 * q]) * inv, __uint_as_float(o[8 * q + 1]) * inv),
              pack_bf16x2(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv),
              pack_bf16x2(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv),
              pack_bf16x2(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv));
      }
    }
    // O read: the next item's first P·V may overwrite it
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.oempty);
    J0 += nblk;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 9) {
    fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- host side
bool calib_sv_tc_supported(const oscar_ctx& c) {
  return c.d == 128 && ptx::encode_tiled_fn() != nullptr;
}

cudaError_t launch_calib_sv_tc(const oscar_ctx& c, const void* Q, const void* K, const void* V,
                               const int32_t* starts, int n_seq, int64_t N, void* SV, cudaStream_t s) {
  if ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(K) | reinterpret_cast<uintptr_t>(V)) & 15)
    return cudaErrorMisalignedAddress;
  CUtensorMap mq, mk, mv;
  if (!ptx::make_bf16_map_3d(&mq, Q, N, c.hq, 1, kSvQ) || !ptx::make_bf16_map_3d(&mk, K, N, c.hkv, 1, kSvK) ||
      !ptx::make_bf16_map_3d(&mv, V, N, c.hkv, 1, kSvK))
    return cudaErrorInvalidValue;
  SvParams p{};
  p.starts = starts; p.n_seq = n_seq; p.N = (int)N; p.hq = c.hq; p.hkv = c.hkv;
  p.nqb = (int)((N + kSvQ - 1) / kSvQ);
  p.scale_log2 = c.scale * kLog2e;
  p.SV = static_cast<uint16_t*>(SV);
  const int smem = (int)sizeof(SvSmem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(calib_sv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long items = (long)p.nqb * c.hq;
  const int grid = (int)(items < c.num_sms ? items : c.num_sms);   // persistent: one CTA per SM
  calib_sv_tc_kernel<<<grid, kSvThreads, smem, s>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

}  // namespace oscar
