// Decode ceiling without the rest of the GEMV: W warps per SM each decode 7
// items (128-row super-step records in shared memory, layout v3 3-bit) per
// "stage" into TMEM with tcgen05.st.32x32b.x16, as the GEMV's decode role does,
// with no MMA, no TMA, no barriers between stages.  MODE 0 = decode + STTM,
// 1 = decode only (results folded), 2 = STTM of the raw words only.
// Prints cycles per stage per warp (max over warps of CTA 0).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void st16(uint32_t t, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(t),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
               "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
struct Sh { uint32_t m3, m4, m5, m6; };
__device__ __forceinline__ void decode3(const uint32_t* w, uint32_t* o, const Sh& h) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    o[i] = w[i] & 0x07070707u;
    o[6 + i] = __umulhi(w[i], h.m3) & 0x07070707u;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    o[12 + r] = (__umulhi(w[r], h.m6) & 0x03030303u) | (__umulhi(w[4 + (r >> 1)], (r & 1) ? h.m5 : h.m4) & 0x04040404u);
}
constexpr int kIPW = 7, kSS = 128 * 24;
// BUSY extra warps spin on integer ALU work for the whole run (a stand-in for
// the GEMV's other roles); BUSYLO: the busy warps take the LOW warp ids.
template <int MODE, int BUSY = 0, bool BUSYLO = false>
__global__ void probe(unsigned long long* out, int stages) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < 2 * kIPW * kSS / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  const int awarp = BUSYLO ? nw - 1 : 0;   // a decode warp allocates and frees TMEM
  if (warp == awarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  const int dwarps = nw - BUSY;
  const bool busy = BUSYLO ? warp < BUSY : warp >= dwarps;
  if (busy) {
    uint32_t x = threadIdx.x, y = 1;
    while (!done) {
#pragma unroll
      for (int i = 0; i < 32; ++i) { x = (x ^ (y << 3)) + 0x9E3779B9u; y = (y & x) | 7u; }
    }
    if (x == 0x1234567u) out[1] = x + y;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    return;
  }
  const int dw = BUSYLO ? warp - BUSY : warp;
  const int q = warp & 3, wg = dw >> 2, row = q * 32 + lane;
  const uint32_t tcol = tb + ((uint32_t)(q * 32) << 16) + (uint32_t)((wg % 4) * kIPW * 16);
  Sh h;
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m3) : "n"(1u << 29));
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m4) : "n"(1u << 28));
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m5) : "n"(1u << 27));
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m6) : "n"(1u << 26));
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int st = 0; st < stages; ++st) {
    const uint32_t base = sa(sm) + (uint32_t)((st & 1) * kIPW * kSS);
    const uint32_t a_lo = base + row * 16, a_hi = base + 2048 + row * 8;
#pragma unroll
    for (int t = 0; t < kIPW; ++t) {
      uint32_t w[6], o[16];
      const uint4 a = lds128(a_lo + t * kSS);
      const uint2 b = lds64(a_hi + t * kSS);
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y;
      if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i] = w[i % 6];
        st16(tcol + t * 16, o);
      } else {
        decode3(w, o, h);
        if (MODE == 0) st16(tcol + t * 16, o);
        else {
#pragma unroll
          for (int i = 0; i < 16; ++i) acc += o[i];
        }
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  const long long t1 = clock64();
  if (acc == 0x1234567u) out[1] = acc;
  if (blockIdx.x == 0 && lane == 0) out[2 + dw] = (unsigned long long)(t1 - t0);
  // last decode warp out releases the busy warps
  asm volatile("bar.sync 1, %0;" ::"r"(dwarps * 32));
  if (dw == 0 && lane == 0) done = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == awarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
  (void)nw;
}
template <int MODE, int BUSY = 0, bool BUSYLO = false>
void run(unsigned long long* d, int warps, int stages) {
  const int smem = 2 * kIPW * kSS;
  cudaFuncSetAttribute(probe<MODE, BUSY, BUSYLO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<MODE, BUSY, BUSYLO><<<148, (warps + BUSY) * 32, smem>>>(d, stages);
  cudaDeviceSynchronize();
  unsigned long long h[64];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[2 + w] > mx ? h[2 + w] : mx;
  printf("mode %d busy %d%s warps %2d: %7.1f cycles per stage per warp (%d items of 128x64 per warp-group stage)\n", MODE, BUSY, BUSYLO ? "(low ids)" : "", warps,
         (double)mx / stages, kIPW);
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  for (int w : {4, 8, 12, 16}) {
    run<0>(d, w, 400);
    run<1>(d, w, 400);
    run<2>(d, w, 400);
  }
  run<0, 4, false>(d, 8, 400);
  run<0, 4, true>(d, 8, 400);
  run<0, 8, false>(d, 8, 400);
  run<0, 8, true>(d, 8, 400);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
