// quantize_append — Alg. 1 `Prefill` rotate-before-write + `QuantizeAndWrite`
// (P:L1639-1643); §4 "KV Cache Update".  This file holds the simple reference
// kernel (variant 1): rotation on CUDA cores in fp32, then clip / min-max / round / pack.
// The decode-size kernel (append_small_kernel, below) and the decode step's prologue
// (attend.cu) share its epilogue, quantize_store_row_warp (append_epilogue.cuh); the tensor-core
// kernel (variant 0, append_tc.cu) has its own thread-per-token epilogue with the same reading-Z4
// arithmetic, parity-tested through its own hooks.
#include "common.cuh"
#include "append_epilogue.cuh"

namespace oscar {

constexpr int kAppTok = 32;   // tokens per CTA in the simple kernel

// grid (ceil(T / kAppTok), H_kv, 2 [K, V]); 128 threads; dynamic smem = R (64 KB) + 2 tiles.
// mode 0: bf16 rows + R -> quantize into pool; 1: bf16 rows + R -> fp32 rotated out;
// mode 2: fp32 rotated rows -> quantize into pool.
__global__ void __launch_bounds__(128) append_simple_kernel(
    int mode, const uint16_t* __restrict__ K, const uint16_t* __restrict__ V,
    const float* __restrict__ Krot, const float* __restrict__ Vrot,
    const int64_t* __restrict__ slots, int64_t T, const float* __restrict__ RK,
    const float* __restrict__ RV, uint8_t* __restrict__ pool, float* __restrict__ rot_out,
    EpiParams ep) {
  extern __shared__ __align__(16) float sm[];
  float* Rs = sm;                       // [128][128]
  float* xs = sm + kD * kD;             // [kAppTok][128]
  float* ys = xs + kAppTok * kD;        // [kAppTok][128]
  const int h = blockIdx.y, isV = blockIdx.z;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");   // PDL (see append_tc.cu)
  const int64_t t0 = (int64_t)blockIdx.x * kAppTok;
  const int nt = (int)((T - t0) < (int64_t)kAppTok ? (T - t0) : (int64_t)kAppTok);
  const int tid = threadIdx.x;

  if (mode != 2) {
    const float* Rb = isV ? RV : RK;      // R_V = NULL: pre-rotated V (NEXT-2) -> identity
    if (Rb) {
      const float* R = Rb + (size_t)h * kD * kD;
      for (int e = tid; e < kD * kD / 4; e += 128)
        reinterpret_cast<float4*>(Rs)[e] = reinterpret_cast<const float4*>(R)[e];
    } else {
      for (int e = tid; e < kD * kD; e += 128) Rs[e] = (e / kD == e % kD) ? 1.f : 0.f;
    }
    const uint16_t* X = isV ? V : K;
    for (int e = tid; e < kAppTok * kD; e += 128) {
      const int r = e / kD, c = e % kD;
      xs[e] = (r < nt) ? bf16_to_f32(X[((t0 + r) * ep.hkv + h) * kD + c]) : 0.f;
    }
    __syncthreads();
    float acc[kAppTok];
#pragma unroll
    for (int r = 0; r < kAppTok; ++r) acc[r] = 0.f;
    for (int k = 0; k < kD; ++k) {
      const float rk = Rs[k * kD + tid];
#pragma unroll
      for (int r = 0; r < kAppTok; ++r) acc[r] = fmaf(xs[r * kD + k], rk, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < kAppTok; ++r) ys[r * kD + tid] = acc[r];
    if (mode == 1) {
      for (int r = 0; r < nt; ++r)
        rot_out[((t0 + r) * ep.hkv + h) * kD + tid] = acc[r];
      return;
    }
  } else {
    const float* X = isV ? Vrot : Krot;
    for (int e = tid; e < kAppTok * kD; e += 128) {
      const int r = e / kD, c = e % kD;
      ys[e] = (r < nt) ? X[((t0 + r) * ep.hkv + h) * kD + c] : 0.f;
    }
  }
  __syncthreads();
  // epilogue: warp w handles rows w, w+4, ...; lane owns channels 4*lane .. 4*lane+3
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < nt; r += 4) {
    const float4 y4 = *reinterpret_cast<const float4*>(&ys[r * kD + 4 * lane]);
    float y[4] = {y4.x, y4.y, y4.z, y4.w};
    quantize_store_row_warp(ep, y, lane, slots[t0 + r], h, isV, pool);
  }
}

cudaError_t launch_append_simple(const oscar_ctx& c, int mode, const void* K, const void* V,
                                 const float* Krot, const float* Vrot, const int64_t* slots,
                                 int64_t T, const float* RK, const float* RV, void* pool,
                                 float* rot_out, cudaStream_t s) {
  const int smem = (kD * kD + 2 * kAppTok * kD) * (int)sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(append_simple_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((T + kAppTok - 1) / kAppTok), c.hkv, 2);
  append_simple_kernel<<<grid, 128, smem, s>>>(
      mode, static_cast<const uint16_t*>(K), static_cast<const uint16_t*>(V), Krot, Vrot, slots,
      T, RK, RV, static_cast<uint8_t*>(pool), rot_out, make_epi_params(c));
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Decode-size appends (a few tokens): latency-bound, so one CTA per (token, head, K|V) row.
// Thread c forms x̃_c = Σ_k x_k R[k][c] in fp32 with R read straight from L2 (coalesced
// columns, 32 loads in flight), then warp 0 runs the shared quantize/pack/store epilogue.
// ------------------------------------------------------------------------------------
constexpr int kSmallAppendMaxT = 64;

__global__ void __launch_bounds__(128) append_small_kernel(const uint16_t* __restrict__ K,
                                                           const uint16_t* __restrict__ V,
                                                           const int64_t* __restrict__ slots,
                                                           const float* __restrict__ RK,
                                                           const float* __restrict__ RV,
                                                           uint8_t* __restrict__ pool, EpiParams ep,
                                                           const float* __restrict__ xin_k,
                                                           const float* __restrict__ xin_v,
                                                           float* __restrict__ rot_out) {
  __shared__ __align__(16) float xs[kD];
  __shared__ __align__(16) float ys[kD];
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");   // PDL (see append_tc.cu)
  const int t = blockIdx.x, h = blockIdx.y, isV = blockIdx.z, c = threadIdx.x;
  const int64_t row = (int64_t)t * ep.hkv + h;
  const float* xin = isV ? xin_v : xin_k;  // quantize_rotated hook: given fp32 x̃, no rotation
  if (!xin) {
    const uint16_t* X = isV ? V : K;
    xs[c] = bf16_to_f32(X[row * kD + c]);
  }
  __syncthreads();
  const float* Rb = isV ? RV : RK;        // R_V = NULL: pre-rotated V (NEXT-2) -> identity
  float acc = xin ? xin[row * kD + c] : xs[c];
  if (Rb && !xin) {
    const float* R = Rb + (size_t)h * kD * kD + c;
    acc = 0.f;
#pragma unroll 32
    for (int k = 0; k < kD; ++k) acc = fmaf(xs[k], R[(size_t)k * kD], acc);
  }
  if (rot_out) {                           // rotate hook: the fp32 x̃ the epilogue would quantize
    rot_out[row * kD + c] = acc;
    return;
  }
  ys[c] = acc;
  __syncthreads();
  if (c < 32) {
    const float4 y4 = reinterpret_cast<const float4*>(ys)[c];
    float y[4] = {y4.x, y4.y, y4.z, y4.w};
    quantize_store_row_warp(ep, y, c, slots[t], h, isV, pool);
  }
}

bool append_small_ok(const oscar_ctx& c, int64_t T) { return T <= kSmallAppendMaxT; }

// mode 0: quantize_append; mode 1: rotate hook (K = X, R_K = R -> rot_out, K half only);
// mode 2: quantize_rotated hook (xin_k / xin_v fp32 rows, no rotation)
cudaError_t launch_append_small(const oscar_ctx& c, int mode, const void* K, const void* V, const float* xin_k,
                                const float* xin_v, const int64_t* slots, int64_t T, const float* RK,
                                const float* RV, void* pool, float* rot_out, cudaStream_t s) {
  append_small_kernel<<<dim3((unsigned)T, c.hkv, mode == 1 ? 1 : 2), 128, 0, s>>>(
      static_cast<const uint16_t*>(K), static_cast<const uint16_t*>(V), slots, RK, RV,
      static_cast<uint8_t*>(pool), make_epi_params(c), mode == 2 ? xin_k : nullptr, mode == 2 ? xin_v : nullptr,
      mode == 1 ? rot_out : nullptr);
  return cudaGetLastError();
}

}  // namespace oscar
