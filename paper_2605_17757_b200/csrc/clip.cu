// CalibrateClip surrogate objectives on the GPU (Alg. 1 `CalibrateClip` P:L1609; reading Z34,
// DESIGN.md §3): for every KV head h, side (K with C_Q, V with C_S) and candidate ratio rho,
//   L(rho) = tr(Rᵀ C R · E(rho)),  E(rho) = Σ_j e_jᵀ e_j,  e_j = Q(clip(x_j R, rho)) − x_j R
// (frozen-error surrogates of Theorem 1), accumulated in fp64.
//
// grid (chunks, H_kv, 2), 256 threads.  Each CTA first forms M = Rᵀ (C R) in shared memory
// (fp64 C from the calibration accumulators, fp32 R), then its 8 warps take rows j of its chunk:
// lane = channels 4l .. 4l+3; x̃ = x R from the smem R; for each rho: nearest-rank clip (Z6),
// the append path's quantizer (minmax_params / quant_code, Z4), e = dequant − x̃, and
// e·M·eᵀ with M rows from smem.  Per-lane fp64 partials, one atomicAdd per (warp, rho).
#include "append_epilogue.cuh"

namespace oscar {

namespace {
constexpr int kClipWarps = 8;

struct ClipParams {
  const uint16_t* X[2];      // K, V bf16 [N][H_kv][d]
  const float* R[2];         // R_K, R_V fp32 [H_kv][d][d]
  const double* acc;         // [H_kv][2][d][d] (C_Q, C_S sums)
  int64_t N;
  int hkv, bits, G, n_grid;
  int kidx[kMaxClipGrid];    // nearest-rank index ceil(rho·d) - 1 per candidate
  double* obj;               // [H_kv][2][n_grid]
};
}  // namespace

__global__ void __launch_bounds__(kClipWarps * 32) calib_clip_kernel(ClipParams p) {
  extern __shared__ __align__(16) float csm[];
  float* Rs = csm;                          // [d][d]
  float* Ms = csm + kD * kD;                // [d][d]
  float* Ts = csm + 2 * kD * kD;            // [d][d] C·R (then per-warp row buffers)
  const int h = blockIdx.y, side = blockIdx.z, tid = threadIdx.x;
  const float* R = p.R[side] + (size_t)h * kD * kD;
  const double* C = p.acc + ((size_t)h * 2 + side) * kD * kD;
  for (int e = tid; e < kD * kD; e += blockDim.x) Rs[e] = R[e];
  __syncthreads();
  // T = C·R (fp64 accumulate), then M = Rᵀ·T
  for (int e = tid; e < kD * kD; e += blockDim.x) {
    const int i = e / kD, c = e % kD;
    double acc = 0.0;
    for (int k = 0; k < kD; ++k) acc += C[(size_t)i * kD + k] * (double)Rs[k * kD + c];
    Ts[e] = (float)acc;
  }
  __syncthreads();
  for (int e = tid; e < kD * kD; e += blockDim.x) {
    const int a = e / kD, c = e % kD;
    double acc = 0.0;
    for (int i = 0; i < kD; ++i) acc += (double)Rs[i * kD + a] * (double)Ts[i * kD + c];
    Ms[e] = (float)acc;
  }
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  float* xb = Ts + warp * 2 * kD;           // per-warp: x row, e row
  float* eb = xb + kD;
  const uint16_t* X = p.X[side];
  const int qmax = (1 << p.bits) - 1;
  const int lanes_per_group = p.G / 4;
  double part[kMaxClipGrid];
#pragma unroll
  for (int g = 0; g < kMaxClipGrid; ++g) part[g] = 0.0;

  const int64_t per = (p.N + gridDim.x - 1) / gridDim.x;
  const int64_t j0 = blockIdx.x * per, j1 = min(p.N, j0 + per);
  for (int64_t j = j0 + warp; j < j1; j += kClipWarps) {
    const uint16_t* xr = X + ((size_t)j * p.hkv + h) * kD;
#pragma unroll
    for (int i = 0; i < 4; ++i) xb[4 * lane + i] = bf16_to_f32(xr[4 * lane + i]);
    __syncwarp();
    float y[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < kD; ++k) {
      const float xk = xb[k];
      const float4 r4 = reinterpret_cast<const float4*>(Rs + k * kD)[lane];
      y[0] = fmaf(xk, r4.x, y[0]); y[1] = fmaf(xk, r4.y, y[1]);
      y[2] = fmaf(xk, r4.z, y[2]); y[3] = fmaf(xk, r4.w, y[3]);
    }
    const float a[4] = {fabsf(y[0]), fabsf(y[1]), fabsf(y[2]), fabsf(y[3])};
    for (int g = 0; g < p.n_grid; ++g) {
      float yc[4] = {y[0], y[1], y[2], y[3]};
      if (p.kidx[g] < kD - 1) {             // rho < 1: nearest-rank clip (Z6)
        const float tau = warp_row_rank_select(a, p.kidx[g]);
#pragma unroll
        for (int i = 0; i < 4; ++i) yc[i] = fminf(fmaxf(yc[i], -tau), tau);
      }
      float mn = fminf(fminf(yc[0], yc[1]), fminf(yc[2], yc[3]));
      float mx = fmaxf(fmaxf(yc[0], yc[1]), fmaxf(yc[2], yc[3]));
      for (int o = 1; o < lanes_per_group; o <<= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      __half s16, m16;
      float m, inv;
      minmax_params(mn, mx, (float)qmax, s16, m16, m, inv);
      const float sf = __half2float(s16);
      float e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = fmaf(sf, (float)quant_code(yc[i], m, inv, qmax), m) - y[i];
      __syncwarp();
      reinterpret_cast<float4*>(eb)[lane] = make_float4(e[0], e[1], e[2], e[3]);
      __syncwarp();
      float z[4] = {0.f, 0.f, 0.f, 0.f};
      for (int r = 0; r < kD; ++r) {
        const float er = eb[r];
        const float4 m4 = reinterpret_cast<const float4*>(Ms + r * kD)[lane];
        z[0] = fmaf(er, m4.x, z[0]); z[1] = fmaf(er, m4.y, z[1]);
        z[2] = fmaf(er, m4.z, z[2]); z[3] = fmaf(er, m4.w, z[3]);
      }
      part[g] += (double)e[0] * z[0] + (double)e[1] * z[1] + (double)e[2] * z[2] + (double)e[3] * z[3];
    }
    __syncwarp();
  }
  for (int g = 0; g < p.n_grid; ++g) {
    double v = part[g];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) atomicAdd(&p.obj[((size_t)h * 2 + side) * p.n_grid + g], v);
  }
}

cudaError_t launch_calib_clip(const oscar_ctx& c, const void* K, const void* V, int64_t N,
                              const float* RK, const float* RV, const double* acc,
                              const int32_t* kidx, int n_grid, double* obj, cudaStream_t s) {
  ClipParams p{};
  p.X[0] = static_cast<const uint16_t*>(K);
  p.X[1] = static_cast<const uint16_t*>(V);
  p.R[0] = RK; p.R[1] = RV; p.acc = acc; p.N = N;
  p.hkv = c.hkv; p.bits = c.bits; p.G = c.G; p.n_grid = n_grid; p.obj = obj;
  for (int g = 0; g < n_grid; ++g) p.kidx[g] = kidx[g];
  cudaError_t e = cudaMemsetAsync(obj, 0, sizeof(double) * c.hkv * 2 * n_grid, s);
  if (e != cudaSuccess) return e;
  const int smem = 3 * kD * kD * (int)sizeof(float);
  e = cudaFuncSetAttribute(calib_clip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int chunks = (int)((N + 255) / 256);
  const int per_slice = (c.num_sms * 2 + 2 * c.hkv - 1) / (2 * c.hkv);   // ~2 CTAs per SM in total
  if (chunks > per_slice) chunks = per_slice;
  if (chunks < 1) chunks = 1;
  calib_clip_kernel<<<dim3(chunks, c.hkv, 2), kClipWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

// CalibrateClip selection (Alg. 1 P:L1609 "c_K, c_V <- CalibrateClip", reading Z34; S:L190 one
// pair per layer): thread `side` sums its objective over the KV heads in head order (fp64) for
// every grid entry and keeps the first minimum.
__global__ void clip_select_kernel(const double* __restrict__ obj, int hkv, int n_grid,
                                   int32_t* __restrict__ choice) {
  const int side = threadIdx.x;
  if (side >= 2) return;
  int best = 0;
  double bv = 0.0;
  for (int g = 0; g < n_grid; ++g) {
    double tot = 0.0;
    for (int h = 0; h < hkv; ++h) tot += obj[((size_t)h * 2 + side) * n_grid + g];
    if (g == 0 || tot < bv) { bv = tot; best = g; }
  }
  choice[side] = best;
}

cudaError_t launch_clip_select(const oscar_ctx& c, const double* obj, int n_grid, int32_t* choice,
                               cudaStream_t s) {
  clip_select_kernel<<<1, 32, 0, s>>>(obj, c.hkv, n_grid, choice);
  return cudaGetLastError();
}

}  // namespace oscar
