// Round-trip cost of the decode -> MMA handshake used by owq_gemv_kernel:
// NWG producer warpgroups write one 128x64 fp16 item into a TMEM slot ring
// (tcgen05.st 32x32b.x32), publish it on an mbarrier (afull); one issuer warp per
// warpgroup waits, issues 4 tcgen05.mma (M=128 N=16 K=16, A from TMEM, B from
// smem) and tcgen05.commit's the slot back (aempty).  Reports cycles per item
// per CTA for several variants.  No decode arithmetic.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
template <bool HINT>
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  if (HINT)
    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 0x989680;\n\t@!P bra W_%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
  else
    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// MODE bit 0: STTM the item; bit 1: issue the 4 MMAs; bit 2: mbarrier wait with suspend hint
template <int NWG, int R, int MODE, int P = 1, int I = 1>
__global__ void k(unsigned long long* out, int items) {
  constexpr bool HINT = MODE & 4;
  __shared__ __align__(1024) uint8_t b_s[16 * 64 * 2];
  __shared__ __align__(8) uint64_t afull[NWG * R], aempty[NWG * R], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (int)sizeof(b_s) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(b_s)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NWG * R; ++i) { mbar_init(&afull[i], 4); mbar_init(&aempty[i], 1); }
    mbar_init(&done, NWG * I);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  const long long t0 = clock64();
  if (warp < 4 * NWG) {
    const int wg = warp >> 2, q = warp & 3;
    const uint32_t trow = tb + ((uint32_t)(q * 32) << 16) + wg * R * 32;
    uint32_t e[32];
    for (int j = 0; j < 32; ++j) e[j] = 0x3c003c00u ^ (j << 3);
    uint32_t slot = 0, rnd = 0;
    for (int it = 0; it < items; ++it) {
      if (rnd && (slot % P) == 0) mbar_wait<HINT>(&aempty[wg * R + slot + P - 1], (rnd - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE & 1) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(trow + slot * 32),
            "r"(e[0]), "r"(e[1]), "r"(e[2]), "r"(e[3]), "r"(e[4]), "r"(e[5]), "r"(e[6]), "r"(e[7]), "r"(e[8]),
            "r"(e[9]), "r"(e[10]), "r"(e[11]), "r"(e[12]), "r"(e[13]), "r"(e[14]), "r"(e[15]), "r"(e[16]),
            "r"(e[17]), "r"(e[18]), "r"(e[19]), "r"(e[20]), "r"(e[21]), "r"(e[22]), "r"(e[23]), "r"(e[24]),
            "r"(e[25]), "r"(e[26]), "r"(e[27]), "r"(e[28]), "r"(e[29]), "r"(e[30]), "r"(e[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if ((slot % P) == P - 1) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[wg * R + slot]);
      }
      if (++slot == R) { slot = 0; ++rnd; }
    }
  } else if (warp < 4 * NWG + NWG * I) {
    const int wg = (warp - 4 * NWG) / I, ii = (warp - 4 * NWG) % I;
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t d_t = tb + NWG * R * 32 + (wg * I + ii) * 16;
      for (int it = ii * P; it < items; it += I * P) {
       for (int it2 = it; it2 < it + P; ++it2) {
        const uint32_t slot = it2 % R, rnd = it2 / R;
        if ((slot % P) == 0) {
          mbar_wait<HINT>(&afull[wg * R + slot + P - 1], rnd & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (MODE & 2) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t bd = desc(sa(b_s) + j * 512, 256, 128);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_t),
                         "r"(tb + wg * R * 32 + slot * 32 + 8 * j), "l"(bd), "r"(idesc), "r"((it2 != ii * P || j) ? 1u : 0u));
          }
        }
        if ((slot % P) == P - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&aempty[wg * R + slot])) : "memory");
       }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&done)) : "memory");
      mbar_wait<HINT>(&done, 0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int NWG, int R, int MODE, int P = 1, int I = 1>
void run(unsigned long long* d, int items) {
  k<NWG, R, MODE, P, I><<<148, 32 * (4 * NWG + NWG * I)>>>(d, items);
  cudaDeviceSynchronize();
  k<NWG, R, MODE, P, I><<<148, 32 * (4 * NWG + NWG * I)>>>(d, items);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("I=%d P=%d NWG=%d R=%d sttm=%d mma=%d hint=%d: %7.1f cycles per item per WG, %6.1f per item per CTA [%s]\n", I, P, NWG, R, MODE & 1,
         (MODE >> 1) & 1, (MODE >> 2) & 1, (double)h / items, (double)h / items / NWG, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int items = 2048;
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  switch (v) {
    case 0: run<1, 4, 3, 1, 1>(d, items); break;
    case 1: run<3, 4, 3, 1, 1>(d, items); break;
    case 2: run<3, 4, 3, 1, 2>(d, items); break;
    case 3: run<3, 4, 3, 2, 2>(d, items); break;
    case 4: run<3, 2, 3, 1, 2>(d, items); break;
    case 5: run<4, 2, 3, 1, 2>(d, items); break;
    case 6: run<2, 6, 3, 1, 3>(d, items); break;
    case 7: run<2, 6, 3, 2, 3>(d, items); break;
    case 8: run<2, 4, 3, 1, 4>(d, items); break;
    case 9: run<1, 8, 3, 1, 8>(d, items); break;
    case 10: run<1, 8, 3, 1, 4>(d, items); break;
    case 11: run<2, 6, 2, 1, 3>(d, items); break;
  }
  fflush(stdout);
  return 0;
}
