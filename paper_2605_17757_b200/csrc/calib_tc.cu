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
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

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

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// MN-major SWIZZLE_128B descriptor: 64 elements (128 B) contiguous along M/N per row, rows =
// K; LBO = byte stride between the two 64-channel blocks, SBO = 1024 B between 8-row groups.
__device__ __forceinline__ uint64_t mn_sw128_desc(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16, A = B = BF16, D = F32, A and B MN-major, M = 128, N = 128
constexpr uint32_t kIdescCov = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                               ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t dt, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(dt), "l"(a), "l"(b), "r"(kIdescCov), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}

#define OSCAR_CLD32(base, v)                                                                         \
  asm volatile(                                                                                       \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                    \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),           \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),       \
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),    \
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),    \
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                             \
      : "r"(base))

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
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su32(&S.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
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
            const uint64_t d = mn_sw128_desc(base + kk * 2048, kTileB / 2);
            umma(tmem + a * 128, d, d, (i | kk) != 0);
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
        OSCAR_CLD32(tmem + ((uint32_t)(quarter * 32) << 16) + a * 128 + c0, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_c() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

bool make_cov_map(CUtensorMap* m, const void* base, int64_t N, int hq, int g) {
  auto fn = encode_fn_c();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)hq, (cuuint64_t)N};
  cuuint64_t strides[2] = {(cuuint64_t)kD * 2, (cuuint64_t)hq * kD * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)g, (cuuint32_t)(kRows / g)};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

bool cov_tc_supported(const oscar_ctx& c) {
  return c.d == 128 && (128 % c.g) == 0 && encode_fn_c() != nullptr;
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
