// Throughput / latency of legacy mma.sync m16n8k16 (f16 -> f32) and of the
// LOP3+HFMA2 decode on sm_100a.  Independent-accumulator chains per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void mma_tput(float* out, int iters) {
  float acc[CHAINS][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c00, b1 = a0 ^ 0x3800;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1.2345f) out[0] = s;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096;
  for (int warps = 1; warps <= 16; warps *= 2) {
#define RUN(CH) { mma_tput<CH><<<148, 32 * warps>>>(out, iters); cudaDeviceSynchronize(); cudaEventRecord(a); mma_tput<CH><<<148, 32 * warps>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); \
      double n = 148.0 * warps * iters * CH; double cyc = ms * 1e-3 * 1.965e9; \
      printf("warps/SM=%2d chains=%d: %.2f cycles per HMMA per SM, %.1f cycles/HMMA/warp (%.0f FMA/clk/SM)\n", warps, CH, cyc / (n / 148), cyc / (iters * CH), n / 148 * 2048 / cyc); }
    RUN(1) RUN(4) RUN(8)
  }
  return 0;
}
