// Microbenchmark: legacy mma.sync throughput on sm_100a (HMMA f16 m16n8k16, IMMA s8/u8 m16n8k32)
// and SHF/LOP3/HFMA2 issue rate context. Used once to choose the decode-attention MMA path.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void hmma_loop(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t b0 = a0 ^ 0x3c003c00u, b1 = a1 ^ 0x3c003c00u;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void imma_loop(int* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t b0 = a0 ^ 0x01010101u, b1 = a1 ^ 0x02020202u;
  int c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* dout; int* iout;
  cudaMalloc(&dout, 148 * 16 * 1024 * 4); cudaMalloc(&iout, 148 * 16 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int rep = 0; rep < 2; ++rep) {
      hmma_loop<<<148 * 2, warps * 32>>>(dout, iters);
      cudaEventRecord(e0);
      hmma_loop<<<148 * 2, warps * 32>>>(dout, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * warps * 148 * 2;
      if (rep) printf("HMMA f16 m16n8k16 warps/CTA=%d: %.1f TFLOP/s  (%.3f ms)\n", warps, flops / ms / 1e9, ms);
      imma_loop<<<148 * 2, warps * 32>>>(iout, iters);
      cudaEventRecord(e0);
      imma_loop<<<148 * 2, warps * 32>>>(iout, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * warps * 148 * 2;
      if (rep) printf("IMMA s8 m16n8k32 warps/CTA=%d: %.1f TOP/s  (%.3f ms)\n", warps, ops / ms / 1e9, ms);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
