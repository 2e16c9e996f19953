// Box calibration probe: read-only HBM stream peak with
// 128-bit ld.global.nc loads, and with cp.async.bulk (TMA 1D) into shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void read_ldg(const int4* __restrict__ p, size_t n, int* out) {
  int acc = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  #pragma unroll 8
  for (; i < n; i += stride) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int STAGES, int CHUNK>
__global__ void read_tma(const char* __restrict__ p, size_t bytes, int* out) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  size_t nchunks = bytes / CHUNK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  int acc = 0;
  if (threadIdx.x == 0) {
    size_t c = blockIdx.x; int it = 0;
    // prologue
    for (int s = 0; s < STAGES && c + (size_t)s * gridDim.x < nchunks; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + s * CHUNK);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(d), "l"(p + (c + (size_t)s * gridDim.x) * CHUNK), "r"(CHUNK), "r"(b) : "memory");
    }
    for (; c < nchunks; c += gridDim.x, ++it) {
      int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" :: "r"(b), "r"(ph));
      acc ^= *(volatile int*)(smem + s * CHUNK);
      size_t nc = c + (size_t)STAGES * gridDim.x;
      if (nc < nchunks) {
        uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + s * CHUNK);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(d), "l"(p + nc * CHUNK), "r"(CHUNK), "r"(b) : "memory");
      }
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}


template <int STAGES, int CHUNK>
__global__ void read_tma_range(const char* __restrict__ p, size_t bytes, int* out) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const size_t per = (bytes / gridDim.x) / 1024 * 1024;
  const size_t beg = (size_t)blockIdx.x * per;
  const int nchunks = (int)(per / CHUNK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  int acc = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES && s < nchunks; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + s * CHUNK);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(d), "l"(p + beg + (size_t)s * CHUNK), "r"(CHUNK), "r"(b) : "memory");
    }
    for (int c = 0; c < nchunks; ++c) {
      int s = c % STAGES; uint32_t ph = (c / STAGES) & 1;
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" :: "r"(b), "r"(ph));
      acc ^= *(volatile int*)(smem + s * CHUNK);
      int nc = c + STAGES;
      if (nc < nchunks) {
        uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + s * CHUNK);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(d), "l"(p + beg + (size_t)nc * CHUNK), "r"(CHUNK), "r"(b) : "memory");
      }
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}
template <int ST, int CH, typename K>
void run_range(K k, const char* p, size_t bytes, int* out, int sms, const char* name) {
  cudaError_t e0 = cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH);
  if (e0 != cudaSuccess) printf("attr: %s\n", cudaGetErrorString(e0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<sms, 32, ST * CH>>>(p, bytes, out); cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(a); k<<<sms, 32, ST * CH>>>(p, bytes, out); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  printf("%s stages=%d chunk=%d bytes=%zu : %.2f us, %.1f GB/s [%s]\n", name, ST, CH, bytes, best * 1e3, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int dev = 0, sms = 0, l2 = 0, clk = 0, memclk = 0, busw = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  CK(cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, dev));
  CK(cudaDeviceGetAttribute(&busw, cudaDevAttrGlobalMemoryBusWidth, dev));
  printf("sms=%d l2=%d clk_khz=%d memclk_khz=%d busw=%d\n", sms, l2, clk, memclk, busw);
  size_t bytes = (size_t)4 << 30;
  char* p; int* out; CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(p, 1, bytes));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int occ = 1; occ <= 8; occ *= 2) for (int threads = 256; threads <= 1024; threads *= 2) {
    int grid = sms * occ * (1024 / threads) / 1; if (threads * occ > 2048) continue;
    read_ldg<<<grid, threads>>>((const int4*)p, bytes / 16, out);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(a); read_ldg<<<grid, threads>>>((const int4*)p, bytes / 16, out); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    printf("ldg grid=%d threads=%d : %.1f GB/s\n", grid, threads, bytes / best / 1e6);
  }
  {
    constexpr int ST = 6, CH = 32768;
    CK(cudaFuncSetAttribute(read_tma<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
    for (int occ = 1; occ <= 1; ++occ) {
      read_tma<ST, CH><<<sms * occ, 32, ST * CH>>>(p, bytes, out); CK(cudaDeviceSynchronize());
      float best = 1e9;
      for (int r = 0; r < 5; ++r) { cudaEventRecord(a); read_tma<ST, CH><<<sms * occ, 32, ST * CH>>>(p, bytes, out); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
      printf("tma stages=%d chunk=%d grid=%d : %.1f GB/s\n", ST, CH, sms * occ, bytes / best / 1e6);
    }
  }
  {
    constexpr int ST = 4, CH = 24576;
    CK(cudaFuncSetAttribute(read_tma<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
    read_tma<ST, CH><<<sms, 32, ST * CH>>>(p, bytes, out); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(a); read_tma<ST, CH><<<sms, 32, ST * CH>>>(p, bytes, out); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    printf("tma stages=%d chunk=%d grid=%d : %.1f GB/s\n", ST, CH, sms, bytes / best / 1e6);
  }
  // 57 MB working set (OPT-175B qkvo layer size) rotated over 12 buffers > L2
  {
    size_t lb = 57u << 20; int nb = 12; float tot = 0;
    read_ldg<<<sms * 8, 256>>>((const int4*)p, lb / 16, out); CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < 48; ++r) read_ldg<<<sms * 8, 256>>>((const int4*)(p + (r % nb) * lb), lb / 16, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&tot, a, b);
    printf("ldg 57MB rotated x48: %.2f us/launch, %.1f GB/s\n", tot * 1000 / 48, 48.0 * lb / tot / 1e6);
  }
  for (size_t mb : {57ul, 227ul, 1024ul}) {
    size_t by = (mb << 20);
    run_range<5, 36864>(read_tma_range<5, 36864>, p, by, out, sms, "tma-range");
    run_range<4, 24576>(read_tma_range<4, 24576>, p, by, out, sms, "tma-range");
    run_range<8, 24576>(read_tma_range<8, 24576>, p, by, out, sms, "tma-range");
    run_range<6, 32768>(read_tma_range<6, 32768>, p, by, out, sms, "tma-range");
  }
  return 0;
}
