// On-device calibration (Alg. 1 `Calibrate`):
//   cov_accum_kernel      — unnormalized C_Q / C_S partial sums (§3)
//   jacobi_compose_kernel — one CTA per matrix: parallel cyclic Jacobi (fp64 A in smem,
//                           fp32 V in smem), descending sort + sign convention, then
//                           R = U · H_Had · P_br by a warp-shuffle FWHT (App A.1 P:L1068-1077,
//                           Eq. 3, P_br convention pinned by P:L209-240).
#include "common.cuh"

namespace oscar {

// ------------------------------------------------------------------------------------
// cov_accum: grid (ceil(N / kTokPerCta), H_kv, 2); 256 threads.  Each CTA forms the fp32
// partial Σ xᵀx over its kTokPerCta tokens × g query heads (rows of one KV group) with an
// 8x8 register tile per thread, then adds it into the fp64 accumulator (reading H4).
// ------------------------------------------------------------------------------------
constexpr int kTokPerCta = 512;
constexpr int kRowTile = 32;

__global__ void __launch_bounds__(256) cov_accum_kernel(const uint16_t* __restrict__ Q,
                                                        const uint16_t* __restrict__ SV,
                                                        int64_t N, int Hq, int g,
                                                        double* __restrict__ acc) {
  __shared__ __align__(16) float xs[kRowTile][kD];
  const int h = blockIdx.y, which = blockIdx.z;
  const uint16_t* X = which == 0 ? Q : SV;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float c[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) c[i][j] = 0.f;

  const int64_t tok0 = (int64_t)blockIdx.x * kTokPerCta;
  const int64_t tok1 = (N < tok0 + kTokPerCta) ? N : tok0 + kTokPerCta;
  const int64_t rows = (tok1 - tok0) * g;   // row r -> token tok0 + r / g, head h*g + r % g
  for (int64_t r0 = 0; r0 < rows; r0 += kRowTile) {
    __syncthreads();
    // load kRowTile rows x 128 bf16 -> fp32 (8 bf16 = 16 B per thread-iteration)
    for (int e = threadIdx.x; e < kRowTile * (kD / 8); e += blockDim.x) {
      const int rr = e / (kD / 8), c8 = e % (kD / 8);
      const int64_t r = r0 + rr;
      float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (r < rows) {
        const int64_t tok = tok0 + r / g;
        const int head = h * g + (int)(r % g);
        const uint4 u = *reinterpret_cast<const uint4*>(X + ((tok * Hq + head) * kD + c8 * 8));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[2 * k] = __uint_as_float(w[k] << 16);
          v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) xs[rr][c8 * 8 + k] = v[k];
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < kRowTile; ++rr) {
      const float4 a0 = *reinterpret_cast<const float4*>(&xs[rr][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&xs[rr][ty * 8 + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&xs[rr][tx * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&xs[rr][tx * 8 + 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) c[i][j] = fmaf(a[i], b[j], c[i][j]);
    }
  }
  double* dst = acc + ((int64_t)h * 2 + which) * kD * kD;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) atomicAdd(dst + (ty * 8 + i) * kD + tx * 8 + j, (double)c[i][j]);
}

cudaError_t launch_cov_accum(const oscar_ctx& c, const void* Q, const void* SV, int64_t N,
                             double* acc, cudaStream_t s) {
  if (N == 0) return cudaSuccess;
  dim3 grid((unsigned)((N + kTokPerCta - 1) / kTokPerCta), c.hkv, 2);
  cov_accum_kernel<<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(Q),
                                        static_cast<const uint16_t*>(SV), N, c.hq, c.g, acc);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// jacobi_compose: grid (n_mats * 2), 512 threads, ~199 KB dynamic smem.
// Round-robin (circle) ordering: 127 rounds of 64 disjoint (p, q) pairs per sweep.
// Rotation per Golub & Van Loan sym.schur2: tau = (a_qq - a_pp) / (2 a_pq),
// t = sign(tau) / (|tau| + sqrt(1 + tau^2)), c = 1/sqrt(1 + t^2), s = t c;
// A <- Jᵀ A J (rows then columns), V <- V J.
// Layout: A (fp64) and V (fp32) rows padded to kLd = 129 elements, and one WARP per pair in both
// passes: the row pass reads A[p][j], A[q][j] with lane = j (consecutive), the column pass
// A[i][p], A[i][q] and V[i][p], V[i][q] with lane = i (stride 129: distinct banks) — the
// previous 8-threads-per-pair mapping strided 128 B / 16 rows across lanes (8-16-way bank
// conflicts, ~19 µs per round).  The column pass also zeroes the annihilated A[p][q], A[q][p].
// ------------------------------------------------------------------------------------
constexpr int kJacThreads = 512;
constexpr int kJacWarps = kJacThreads / 32;
constexpr int kMaxSweeps = 100;
constexpr double kJacTol = 1e-12;   // max |offdiag| <= kJacTol * ||A||_F
constexpr int kLd = kD + 1;

struct JacSmem {
  double A[kD][kLd];
  float V[kD][kLd];
  double cs[kD / 2], sn[kD / 2];
  int pp[kD / 2], qq[kD / 2];
  double red[kJacThreads / 32];
  int rank[kD];
  float sign[kD];
  double lam[kD];
};

__device__ __forceinline__ int circle_player(int r, int pos) {
  return pos == 0 ? 0 : ((pos - 1 + r) % (kD - 1)) + 1;
}

__device__ double block_reduce(double v, bool is_max, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : v + w;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < kJacThreads / 32; ++i) r = is_max ? fmax(r, red[i]) : r + red[i];
  return r;
}

__global__ void __launch_bounds__(kJacThreads, 1)
jacobi_compose_kernel(const double* __restrict__ acc, double inv_rows, float* __restrict__ RK,
                      float* __restrict__ RV, double* __restrict__ evals,
                      int32_t* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacSmem& S = *reinterpret_cast<JacSmem*>(smem_raw);
  const int mat = blockIdx.x >> 1, which = blockIdx.x & 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* src = acc + (size_t)blockIdx.x * kD * kD;   // [n_mats][2][d][d]

  double fro2 = 0.0;
  for (int e = tid; e < kD * kD; e += kJacThreads) {
    const int i = e / kD, j = e % kD;
    // symmetrize (the accumulator is symmetric up to fp64 atomic-order rounding)
    const double v = 0.5 * (src[i * kD + j] + src[j * kD + i]) * inv_rows;
    S.A[i][j] = v;
    S.V[i][j] = (i == j) ? 1.f : 0.f;
    fro2 += v * v;
  }
  const double fro = sqrt(block_reduce(fro2, false, S.red));

  int sweeps = 0;
  bool converged = false;
  for (; sweeps <= kMaxSweeps; ++sweeps) {
    double off = 0.0;
    for (int e = tid; e < kD * kD; e += kJacThreads) {
      const int i = e / kD, j = e % kD;
      if (i != j) off = fmax(off, fabs(S.A[i][j]));
    }
    off = block_reduce(off, true, S.red);
    if (off <= kJacTol * fro) { converged = true; break; }
    if (sweeps == kMaxSweeps) break;
    for (int r = 0; r < kD - 1; ++r) {
      if (tid < kD / 2) {
        const int p = circle_player(r, tid), q = circle_player(r, kD - 1 - tid);
        const double apq = S.A[p][q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double tau = (S.A[q][q] - S.A[p][p]) / (2.0 * apq);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
        }
        S.cs[tid] = c; S.sn[tid] = s; S.pp[tid] = p; S.qq[tid] = q;
      }
      __syncthreads();
      // rows: (JᵀA)_p = c A_p - s A_q ; (JᵀA)_q = s A_p + c A_q   (warp per pair, lane = column)
      for (int k = warp; k < kD / 2; k += kJacWarps) {
        const int p = S.pp[k], q = S.qq[k];
        const double c = S.cs[k], s = S.sn[k];
#pragma unroll
        for (int m = 0; m < kD / 32; ++m) {
          const int j = lane + 32 * m;
          const double ap = S.A[p][j], aq = S.A[q][j];
          S.A[p][j] = c * ap - s * aq;
          S.A[q][j] = s * ap + c * aq;
        }
      }
      __syncthreads();
      // columns of A and of V (warp per pair, lane = row); the annihilated pair set to 0
      for (int k = warp; k < kD / 2; k += kJacWarps) {
        const int p = S.pp[k], q = S.qq[k];
        const double c = S.cs[k], s = S.sn[k];
#pragma unroll
        for (int m = 0; m < kD / 32; ++m) {
          const int i = lane + 32 * m;
          const double ap = S.A[i][p], aq = S.A[i][q];
          S.A[i][p] = (i == q) ? 0.0 : c * ap - s * aq;
          S.A[i][q] = (i == p) ? 0.0 : s * ap + c * aq;
          const double vp = S.V[i][p], vq = S.V[i][q];
          S.V[i][p] = (float)(c * vp - s * vq);
          S.V[i][q] = (float)(s * vp + c * vq);
        }
      }
      __syncthreads();
    }
  }
  if (info && tid == 0) info[blockIdx.x] = converged ? sweeps : -1;

  // ---- descending order (ties by index), sign convention (largest-|entry| positive)
  if (tid < kD) S.lam[tid] = S.A[tid][tid];
  __syncthreads();
  if (tid < kD) {
    const double li = S.lam[tid];
    int rk = 0;
    for (int j = 0; j < kD; ++j) rk += (S.lam[j] > li) || (S.lam[j] == li && j < tid);
    S.rank[tid] = rk;
    float best = -1.f; int bi = 0;
    for (int k = 0; k < kD; ++k) {
      const float a = fabsf(S.V[k][tid]);
      if (a > best) { best = a; bi = k; }
    }
    S.sign[tid] = S.V[bi][tid] < 0.f ? -1.f : 1.f;
    if (evals) evals[(size_t)blockIdx.x * kD + rk] = li;
  }
  __syncthreads();
  // U_sorted[r][rank_i] = sign_i * V[r][i], staged in S.A (fp64)
  for (int e = tid; e < kD * kD; e += kJacThreads) {
    const int r = e / kD, i = e % kD;
    S.A[r][S.rank[i]] = (double)(S.sign[i] * S.V[r][i]);
  }
  __syncthreads();
  // ---- R = U · H_Had · P_br: per row, FWHT (Sylvester order) then out[beta(e)] = y[e]
  float* R = (which == 0 ? RK : RV) + (size_t)mat * kD * kD;
  const double norm = 0.08838834764831845;   // 1/sqrt(128)
  for (int r = warp; r < kD; r += kJacThreads / 32) {
    double y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = S.A[r][4 * lane + k];
    // strides 1, 2 inside the lane
    { double a = y[0], b = y[1]; y[0] = a + b; y[1] = a - b; a = y[2]; b = y[3]; y[2] = a + b; y[3] = a - b; }
    { double a = y[0], b = y[2]; y[0] = a + b; y[2] = a - b; a = y[1]; b = y[3]; y[1] = a + b; y[3] = a - b; }
    // strides 4..64 across lanes
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const bool upper = lane & m;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double o = __shfl_xor_sync(0xffffffffu, y[k], m);
        y[k] = upper ? (o - y[k]) : (y[k] + o);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = 4 * lane + k;
      const int be = __brev((unsigned)e) >> (32 - 7);
      R[r * kD + be] = (float)(y[k] * norm);
    }
  }
}

cudaError_t launch_jacobi_compose(const oscar_ctx& c, const double* acc, int n_mats,
                                  double inv_rows, float* RK, float* RV, double* evals,
                                  int32_t* info, cudaStream_t s) {
  const int smem = (int)sizeof(JacSmem);
  cudaError_t e = cudaFuncSetAttribute(jacobi_compose_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  jacobi_compose_kernel<<<n_mats * 2, kJacThreads, smem, s>>>(acc, inv_rows, RK, RV, evals, info);
  return cudaGetLastError();
}

}  // namespace oscar
