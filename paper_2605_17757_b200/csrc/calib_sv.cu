// On-device S·V for the C_S target (Alg. 1 `Calibrate` P:L1604-1606:
// S = softmax(Q Kᵀ/√d + M), C_S from S·V).  Reading Z16: M is causal including the
// diagonal and block-diagonal across the calibration sequences; query head i uses KV head i/g.
//
// A flash-attention forward on the legacy tensor-core path (mma.sync m16n8k16 bf16 -> fp32):
// one CTA = 64 queries of one query head (4 warps x 16 rows); key blocks of 64 rows are staged
// in shared memory (K row-major, V transposed, both padded against bank conflicts); S = Q Kᵀ
// per warp in registers, online softmax in the log2 domain, P (bf16) re-used as the A operand
// of P·V.  Output SV bf16 [N][H_q][d] (the layout oscar_calib_accumulate takes).
#include "common.cuh"

namespace oscar {

namespace {
constexpr int kQB = 64;                  // queries per CTA
constexpr int kKB = 64;                  // keys per block
constexpr int kKS = kD + 8;              // K smem row stride (bf16): 272 B, conflict-free b loads
constexpr int kVS = kKB + 8;             // Vt smem row stride (bf16): 144 B

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// sequence containing token n: the last s with starts[s] <= n
__device__ __forceinline__ int seq_start_of(const int32_t* starts, int n_seq, int n) {
  int lo = 0, hi = n_seq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (starts[mid] <= n) lo = mid; else hi = mid - 1;
  }
  return starts[lo];
}
}  // namespace

__global__ void __launch_bounds__(128) calib_sv_kernel(const uint16_t* __restrict__ Q, const uint16_t* __restrict__ K,
                                                       const uint16_t* __restrict__ V,
                                                       const int32_t* __restrict__ starts, int n_seq, int N,
                                                       int hq, int hkv, float scale_log2,
                                                       uint16_t* __restrict__ SV) {
  __shared__ __align__(16) uint16_t Ks[kKB * kKS];
  __shared__ __align__(16) uint16_t Vt[kD * kVS];
  const int qb = blockIdx.x, qh = blockIdx.y, h = qh / (hq / hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t = lane & 3;
  const int q0 = qb * kQB;
  const int r0 = q0 + 16 * warp + gid, r1 = r0 + 8;           // this lane's two query rows
  const int rv0 = min(r0, N - 1), rv1 = min(r1, N - 1);
  const int lo0 = seq_start_of(starts, n_seq, rv0), lo1 = seq_start_of(starts, n_seq, rv1);
  // key range of the CTA: [first key any row needs, last row]
  const int qlast = min(q0 + kQB, N) - 1;
  const int kbeg = seq_start_of(starts, n_seq, q0);
  const int kend = qlast;                                        // inclusive

  // Q fragments (A operand), 8 k-steps over d
  uint32_t qa[8][4];
  {
    const uint32_t* q0p = reinterpret_cast<const uint32_t*>(Q + ((size_t)rv0 * hq + qh) * kD);
    const uint32_t* q1p = reinterpret_cast<const uint32_t*>(Q + ((size_t)rv1 * hq + qh) * kD);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = q0p[8 * ks + t];
      qa[ks][1] = q1p[8 * ks + t];
      qa[ks][2] = q0p[8 * ks + 4 + t];
      qa[ks][3] = q1p[8 * ks + 4 + t];
    }
  }
  float o[16][4];
#pragma unroll
  for (int nd = 0; nd < 16; ++nd)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[nd][e] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int kb = kbeg; kb <= kend; kb += kKB) {
    __syncthreads();
    // stage K rows (row-major) and V transposed for keys kb .. kb+63
    for (int e = threadIdx.x; e < kKB * (kD / 2); e += 128) {
      const int r = e / (kD / 2), c2 = e % (kD / 2);
      const int key = kb + r;
      uint32_t kv = 0u, vv = 0u;
      if (key < N) {
        kv = reinterpret_cast<const uint32_t*>(K + ((size_t)key * hkv + h) * kD)[c2];
        vv = reinterpret_cast<const uint32_t*>(V + ((size_t)key * hkv + h) * kD)[c2];
      }
      reinterpret_cast<uint32_t*>(Ks + r * kKS)[c2] = kv;
      Vt[(2 * c2) * kVS + r] = (uint16_t)(vv & 0xFFFFu);
      Vt[(2 * c2 + 1) * kVS + r] = (uint16_t)(vv >> 16);
    }
    __syncthreads();
    // S = Q Kᵀ for 8 n-tiles of 8 keys
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;
      const uint32_t* kr = reinterpret_cast<const uint32_t*>(Ks + (8 * nt + gid) * kKS);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) mma_bf16(s[nt], qa[ks], kr[8 * ks + t], kr[8 * ks + 4 + t]);
    }
    // mask (block-diagonal causal, reading Z16), scale, block row max
    float bm0 = -INFINITY, bm1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb + 8 * nt + 2 * t + (e & 1);
        const bool up = e >= 2;
        const int r = up ? r1 : r0, lo = up ? lo1 : lo0;
        const bool ok = key >= lo && key <= r && r < N;
        s[nt][e] = ok ? s[nt][e] * scale_log2 : -INFINITY;
        if (up) bm1 = fmaxf(bm1, s[nt][e]); else bm0 = fmaxf(bm0, s[nt][e]);
      }
#pragma unroll
    for (int x = 1; x <= 2; x <<= 1) {
      bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, x));
      bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, x));
    }
    const float mn0 = fmaxf(m0, bm0), mn1 = fmaxf(m1, bm1);
    const float a0 = mn0 == -INFINITY ? 1.f : exp2f(m0 - mn0);
    const float a1 = mn1 == -INFINITY ? 1.f : exp2f(m1 - mn1);
    m0 = mn0; m1 = mn1;
    l0 *= a0; l1 *= a1;
#pragma unroll
    for (int nd = 0; nd < 16; ++nd) {
      o[nd][0] *= a0; o[nd][1] *= a0;
      o[nd][2] *= a1; o[nd][3] *= a1;
    }
    // P = exp2(s - m), row sums, and P·V with P re-used as A fragments
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = m0 == -INFINITY ? 0.f : exp2f(s[nt][0] - m0);
      s[nt][1] = m0 == -INFINITY ? 0.f : exp2f(s[nt][1] - m0);
      s[nt][2] = m1 == -INFINITY ? 0.f : exp2f(s[nt][2] - m1);
      s[nt][3] = m1 == -INFINITY ? 0.f : exp2f(s[nt][3] - m1);
      l0 += s[nt][0] + s[nt][1];
      l1 += s[nt][2] + s[nt][3];
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int nd = 0; nd < 16; ++nd) {
        const uint32_t* vr = reinterpret_cast<const uint32_t*>(Vt + (8 * nd + gid) * kVS);
        mma_bf16(o[nd], pa, vr[8 * kk + t], vr[8 * kk + 4 + t]);
      }
    }
  }
  // normalize and store SV (bf16)
#pragma unroll
  for (int x = 1; x <= 2; x <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, x);
    l1 += __shfl_xor_sync(0xffffffffu, l1, x);
  }
  const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) {
    const int c = 8 * nd + 2 * t;
    if (r0 < N)
      *reinterpret_cast<uint32_t*>(SV + ((size_t)r0 * hq + qh) * kD + c) = pack_bf16(o[nd][0] * i0, o[nd][1] * i0);
    if (r1 < N)
      *reinterpret_cast<uint32_t*>(SV + ((size_t)r1 * hq + qh) * kD + c) = pack_bf16(o[nd][2] * i1, o[nd][3] * i1);
  }
}

cudaError_t launch_calib_sv(const oscar_ctx& c, const void* Q, const void* K, const void* V,
                            const int32_t* starts, int n_seq, int64_t N, void* SV, cudaStream_t s) {
  const dim3 grid((unsigned)((N + kQB - 1) / kQB), (unsigned)c.hq);
  calib_sv_kernel<<<grid, 128, 0, s>>>(static_cast<const uint16_t*>(Q), static_cast<const uint16_t*>(K),
                                       static_cast<const uint16_t*>(V), starts, n_seq, (int)N, c.hq, c.hkv,
                                       c.scale * kLog2e, static_cast<uint16_t*>(SV));
  return cudaGetLastError();
}

}  // namespace oscar
