// Back-to-back tcgen05.mma kind::i8 (M=128, K=32) throughput on sm_100a: A from
// TMEM ("TS") or shared memory ("SS"), N = 8 / 16 / 64, NI issuing warps, each
// accumulating into its own D.  Cycles per MMA per issuer and per SM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <int N, bool TS, int NI>
__global__ void k(unsigned long long* out, int iters) {
  __shared__ __align__(1024) uint8_t a_s[128 * 64];   // A: 128 x 64 u8 (core matrices 8 rows x 16 B)
  __shared__ __align__(1024) uint8_t b_s[64 * 64];    // B: up to 64 x 64 s8
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (int)sizeof(a_s) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(a_s)[i] = 0x01020304u;
  for (int i = threadIdx.x; i < (int)sizeof(b_s) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(b_s)[i] = 0x01010101u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(NI)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  long long t0 = 0, t1 = 0;
  if ((threadIdx.x & 31) == 0 && warp < NI) {
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t d_t = tb + 64 + warp * 64;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int j = i & 1;
      const uint64_t bd = desc(sa(b_s) + j * 2 * (N / 8) * 128, (N / 8) * 128, 128);
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_t), "r"(tb + 8 * j), "l"(bd), "r"(idesc), "r"(i));
      } else {
        const uint64_t ad = desc(sa(a_s) + j * 2 * 16 * 128, 16 * 128, 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_t), "l"(ad), "l"(bd), "r"(idesc), "r"(i));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
    asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n}" ::"r"(sa(&bar)));
    t1 = clock64();
    if (blockIdx.x == 0 && warp == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
template <int N, bool TS, int NI>
void run(unsigned long long* d, int iters) {
  k<N, TS, NI><<<148, 128>>>(d, iters);
  cudaDeviceSynchronize();
  k<N, TS, NI><<<148, 128>>>(d, iters);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("i8 %s N=%2d NI=%d: %6.1f cycles per MMA per issuer, %6.1f per MMA per SM  [%s]\n", TS ? "TS" : "SS", N, NI, (double)h / iters,
         (double)h / iters / NI, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int it = 4096;
  run<8, true, 1>(d, it); run<8, true, 2>(d, it); run<8, true, 4>(d, it);
  run<8, false, 1>(d, it); run<8, false, 2>(d, it); run<8, false, 4>(d, it);
  run<16, true, 4>(d, it); run<16, false, 4>(d, it); run<64, true, 4>(d, it); run<64, false, 4>(d, it);
  return 0;
}
