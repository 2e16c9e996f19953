// Issue rate of LOP3 (alu pipe), HFMA2 imm-form / 3-reg (fma pipe) and mixes on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
__device__ __forceinline__ uint32_t H(__half2 h){return *reinterpret_cast<uint32_t*>(&h);}
__device__ __forceinline__ __half2 U(uint32_t u){return *reinterpret_cast<__half2*>(&u);}
template <int MODE>
__global__ void k(uint32_t* out, int iters) {
  uint32_t a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * (i + 1);
  uint32_t m; asm volatile("mov.b32 %0, 0x64006400;" : "=r"(m));
  uint32_t c; asm volatile("mov.b32 %0, 0x3c003c00;" : "=r"(c));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("lop3.b32 %0, %0, 0x70007, %1, 0xEA;" : "+r"(a[i]) : "r"(m));
      if (MODE == 1) a[i] = H(__hfma2(U(a[i]), __float2half2_rn(0.125f), U(c)));
      if (MODE == 2) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(m), "r"(c));
      if (MODE == 3) { if (i & 1) a[i] = H(__hfma2(U(a[i]), __float2half2_rn(0.125f), U(c)));
                       else asm volatile("lop3.b32 %0, %0, 0x70007, %1, 0xEA;" : "+r"(a[i]) : "r"(m)); }
      if (MODE == 4) asm volatile("shr.b32 %0, %0, 9;" : "+r"(a[i]));
      if (MODE == 5) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
      if (MODE == 6) { if (i & 1) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
                       else asm volatile("lop3.b32 %0, %0, 0x70007, %1, 0xEA;" : "+r"(a[i]) : "r"(m)); }
      if (MODE == 7) asm volatile("fma.rn.f32 %0, %0, 0f3f000000, 0f3f800000;" : "+r"(a[i]));
    }
  }
  uint32_t s = 0; for (int i = 0; i < 16; ++i) s ^= a[i];
  if (s == 0x12345) out[0] = s;
}
int main() {
  uint32_t* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"LOP3 (reg magic)", "HFMA2 imm", "HFMA2 3-reg", "LOP3+HFMA2imm 1:1", "SHF", "HADD2", "LOP3+HADD2 1:1", "FFMA imm"};
  for (int mode = 0; mode < 8; ++mode)
    for (int nw : {8, 16, 32}) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : mode == 5 ? k<5> : mode == 6 ? k<6> : k<7>;
      int iters = 4096;
      f<<<148, 32 * nw>>>(out, iters); cudaDeviceSynchronize();
      cudaEventRecord(a); f<<<148, 32 * nw>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double instr_per_smsp = (double)nw / 4 * iters * 16;
      printf("%-20s warps/SM=%2d: %.2f SMSP-cycles per warp-instr\n", names[mode], nw, ms * 1e-3 * 1.965e9 / instr_per_smsp);
    }
}
