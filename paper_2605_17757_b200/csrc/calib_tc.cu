// Tensor-core covariance accumulation (variant 0): the C_Q / C_S targets of
// §3 (C_S = (SV)ᵀ(SV)) as a tcgen05 contraction Σ_rows xᵀx.
//
// Persistent CTAs, 6 warps: warp 0 = TMA producer (128-row x 128-channel bf16 tiles of the
// rows of one KV head, i.e. (token, query head in its GQA group) pairs; two 64-channel
// SWIZZLE_128B boxes per tile), warp 1 = TMEM allocator + single-thread tcgen05.mma issuer,
// warps 2-5 = flush.  The SAME smem tile is both operands, MN-major:
//   D[i][j] += Σ_r X[r][i] X[r][j]   (A = Xᵀ: M = channel i; B = X: N = channel j; K = rows)
// Each work unit accumulates kRowsPerUnit rows in fp32 TMEM (reading H4: bounded fp32 chunk)
// and is then flushed with fp64 red.add into acc[h][which][128][128]; two TMEM accumulators
// let the next unit's MMAs overlap the flush.
#include "common.cuh"
#include "ptx.cuh"

namespace oscar {

namespace {

constexpr int kRows = 128;            // rows per tile (UMMA K extent of one tile = 8 x K16)
constexpr int kStagesC = 2;
constexpr int kTileB = kRows * kD * 2;
constexpr int kRowsPerUnit = 1024;    // fp32 TMEM accumulation span before the fp64 smem add
constexpr int kThreadsC = 6 * 32;

struct CovSmem {
  alignas(1024) uint8_t A[kStagesC][kTileB];   // [stage][2 channel chunks][128 rows][128 B]
  double accd[kD * kD];                         // per-CTA fp64 partial, [j][i]
  uint64_t full[kStagesC], empty[kStagesC], tfull[2], tempty[2];
  uint32_t tmem_base;
};

using namespace ptx;
// kind::f16, A = B = BF16, D = F32, A and B MN-major, M = 128, N = 128
constexpr uint32_t kIdescCov = idesc_bf16(128, 128, true, true);

struct CovParams {
  double* acc;             // [H_kv][2][128][128]
  int64_t rows;            // N * g rows per (kv head, which)
  int g, hkv, units_per_pair, cpp;
};

}  // namespace

__global__ void __launch_bounds__(kThreadsC, 1)
cov_accum_tc_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapS, CovParams p) {
  extern __shared__ uint8_t smem_raw[];
  CovSmem& S = *reinterpret_cast<CovSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA serves one (kv head, Q|S) pair: units sub, sub + cpp, ... of 1024 rows each
  const int pair = blockIdx.x / p.cpp, sub = blockIdx.x % p.cpp;
  const int n_my = sub < p.units_per_pair ? (p.units_per_pair - 1 - sub) / p.cpp + 1 : 0;
  auto unit_info = [&](int k, int64_t& row0, int& ntiles) {
    row0 = (int64_t)(sub + k * p.cpp) * kRowsPerUnit;
    const int64_t left = p.rows - row0;
    ntiles = (int)((left < kRowsPerUnit ? left : kRowsPerUnit) + kRows - 1) / kRows;
  };
  for (int e = threadIdx.x; e < kD * kD; e += kThreadsC) S.accd[e] = 0.0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesC; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&S.tfull[a], 1); mbar_init(&S.tempty[a], 4); }
    mbar_init_fence();
  }
  if (warp == 1) {
    tmem_alloc(&S.tmem_base, 256);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;   // global tile counter (stage ring)
      for (int k = 0; k < n_my; ++k) {
        int ntiles;
        int64_t row0;
        unit_info(k, row0, ntiles);
        const int h = pair >> 1, which = pair & 1;
        const CUtensorMap* map = which ? &mapS : &mapQ;
        for (int i = 0; i < ntiles; ++i, ++it) {
          const int s = it % kStagesC;
          mbar_wait(&S.empty[s], ((it / kStagesC) & 1) ^ 1);
          mbar_expect_tx(&S.full[s], kTileB);
          // rows r = token·g + i_g of KV head h: box {64 ch, g heads, 128/g tokens}
          const int tok0 = (int)((row0 + (int64_t)i * kRows) / p.g);
          tma_load_3d(S.A[s], map, 0, h * p.g, tok0, &S.full[s]);
          tma_load_3d(S.A[s] + kTileB / 2, map, 64, h * p.g, tok0, &S.full[s]);
        }
      }
    }
  } else if (warp == 1) {
    int it = 0;
    for (int k = 0; k < n_my; ++k) {
      int ntiles;
      int64_t row0;
      unit_info(k, row0, ntiles);
      const int a = k & 1;
      mbar_wait(&S.tempty[a], ((k >> 1) & 1) ^ 1);
      fence_after();
      for (int i = 0; i < ntiles; ++i, ++it) {
        const int s = it % kStagesC;
        mbar_wait(&S.full[s], (it / kStagesC) & 1);
        fence_after();
        if (lane == 0) {
          const uint32_t base = su32(S.A[s]);
#pragma unroll
          for (int kk = 0; kk < kRows / 16; ++kk) {
            const uint64_t d = mnmajor_sw128_desc(base + kk * 2048, kTileB / 2);
            umma_f16<kIdescCov>(tmem + a * 128, d, d, (i | kk) != 0);
          }
          umma_commit(&S.empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit(&S.tfull[a]);
      __syncwarp();
    }
  } else {
    // flush warps 2..5: TMEM lane quarter = warp % 4, row i = quarter·32 + lane (channel i);
    // each unit's fp32 TMEM sum is added into the CTA's fp64 smem partial, which is added to
    // the global accumulator once at the end
    const int quarter = warp & 3;
    const int i = quarter * 32 + lane;
    for (int k = 0; k < n_my; ++k) {
      const int a = k & 1;
      mbar_wait(&S.tfull[a], (k >> 1) & 1);
      fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < kD; c0 += 32) {
        uint32_t v[32];
        OSCAR_TMEM_LD32(tmem + ((uint32_t)(quarter * 32) << 16) + a * 128 + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) S.accd[(c0 + j) * kD + i] += (double)__uint_as_float(v[j]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.tempty[a]);
    }
    if (n_my > 0) {
      double* dst = p.acc + (size_t)pair * kD * kD + (size_t)i * kD;
#pragma unroll 4
      for (int j = 0; j < kD; ++j) atomicAdd(dst + j, S.accd[j * kD + i]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------- host side
namespace {
// rows r = token·g + i_g of KV head h: box {64 channels, g heads, 128/g tokens}
bool make_cov_map(CUtensorMap* m, const void* base, int64_t N, int hq, int g) {
  return ptx::make_bf16_map_3d(m, base, N, hq, g, kRows / g);
}
}  // namespace

bool cov_tc_supported(const oscar_ctx& c) {
  return c.d == 128 && (128 % c.g) == 0 && ptx::encode_tiled_fn() != nullptr;
}

cudaError_t launch_cov_accum_tc(const oscar_ctx& c, const void* Q, const void* SV, int64_t N, double* acc,
                                cudaStream_t s) {
  if ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(SV)) & 15) return cudaErrorMisalignedAddress;
  CUtensorMap mq, ms;
  if (!make_cov_map(&mq, Q, N, c.hq, c.g) || !make_cov_map(&ms, SV, N, c.hq, c.g)) return cudaErrorInvalidValue;
  CovParams p{};
  p.acc = acc;
  p.rows = N * c.g;
  p.g = c.g;
  p.hkv = c.hkv;
  p.units_per_pair = (int)((p.rows + kRowsPerUnit - 1) / kRowsPerUnit);
  const int pairs = 2 * c.hkv;
  int cpp = c.num_sms / pairs;
  if (cpp < 1) cpp = 1;
  if (cpp > p.units_per_pair) cpp = p.units_per_pair;
  p.cpp = cpp;
  const int grid = pairs * cpp;
  const int smem = (int)sizeof(CovSmem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(cov_accum_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cov_accum_tc_kernel<<<grid, kThreadsC, smem, s>>>(mq, ms, p);
  return cudaGetLastError();
}

}  // namespace oscar
