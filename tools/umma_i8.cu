// tcgen05.mma kind::i8 on sm_100a: A (u8, 128 x K) from TMEM written with
// tcgen05.st (4 consecutive K per 32-bit column, byte 0 = lowest k), B (s8,
// N x K, K-major core matrices 8 rows x 16 B) from shared memory, D s32 in TMEM.
// Part 1 checks exactness against a host reference; part 2 measures the
// decode->MMA handshake (STTM x16 per item of 64 codes, 2 MMAs of K=32).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <int N>
__host__ __device__ constexpr uint32_t idesc_i8() {   // D s32, A u8, B s8, K-major, M = 128
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void st16(uint32_t t, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(t),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
               "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void ld16(uint32_t t, uint32_t* d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
                 "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]) : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- part 1: correctness, K = 64 (2 MMAs), N = 16
constexpr int K = 64, N = 16;
__global__ void check(const uint8_t* A, const int8_t* Bm, int* D) {
  __shared__ __align__(128) int8_t bs[N * K];   // [kc 0..3][nb 0..1][8 rows][16 B]
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K, kc = k / 16, nb = n / 8, r = n % 8;
    bs[(kc * (N / 8) + nb) * 128 + r * 16 + (k % 16)] = Bm[n * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  {
    const int row = warp * 32 + lane;
    uint32_t r[16];
    for (int c = 0; c < 16; ++c)
      r[c] = A[row * K + 4 * c] | (A[row * K + 4 * c + 1] << 8) | (A[row * K + 4 * c + 2] << 16) | ((uint32_t)A[row * K + 4 * c + 3] << 24);
    st16(tb + ((uint32_t)(warp * 32) << 16), r);
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    for (int j = 0; j < 2; ++j)
      mma_i8(tb + 32, tb + 8 * j, desc(sa(bs) + j * 2 * (N / 8) * 128, (N / 8) * 128, 128), idesc_i8<N>(), j);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
  }
  asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n}" ::"r"(sa(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t d[16];
    ld16(tb + 32 + ((uint32_t)(warp * 32) << 16), d);
    const int row = warp * 32 + lane;
    for (int n = 0; n < N; ++n) D[row * N + n] = (int)d[n];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tb));
}

// ---- part 2: pipeline throughput (NWG producer warpgroups, I issuers per WG)
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}
template <int NWG, int R, int I, int NN>
__global__ void pipe(unsigned long long* out, int items) {
  __shared__ __align__(1024) uint8_t b_s[64 * 64];
  __shared__ __align__(8) uint64_t afull[NWG * R], aempty[NWG * R], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (int)sizeof(b_s) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(b_s)[i] = 0x01010101u;
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
    const uint32_t trow = tb + ((uint32_t)(q * 32) << 16) + wg * R * 16;
    uint32_t e[16];
    for (int j = 0; j < 16; ++j) e[j] = 0x01020304u ^ (j << 3);
    uint32_t slot = 0, rnd = 0;
    for (int it = 0; it < items; ++it) {
      if (rnd) mbar_wait(&aempty[wg * R + slot], (rnd - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      st16(trow + slot * 16, e);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[wg * R + slot]);
      if (++slot == R) { slot = 0; ++rnd; }
    }
  } else if (warp < 4 * NWG + NWG * I) {
    const int wg = (warp - 4 * NWG) / I, ii = (warp - 4 * NWG) % I;
    if (lane == 0) {
      const uint32_t d_t = tb + NWG * R * 16 + (wg * I + ii) * NN;
      for (int it = ii; it < items; it += I) {
        const uint32_t slot = it % R, rnd = it / R;
        mbar_wait(&afull[wg * R + slot], rnd & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 2; ++j)
          mma_i8(d_t, tb + wg * R * 16 + slot * 16 + 8 * j, desc(sa(b_s) + j * 2 * (NN / 8) * 128, (NN / 8) * 128, 128), idesc_i8<NN>(),
                 (it != ii || j) ? 1u : 0u);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&aempty[wg * R + slot])) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&done)) : "memory");
      mbar_wait(&done, 0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
template <int NWG, int R, int I, int NN>
void run(unsigned long long* d, int items) {
  pipe<NWG, R, I, NN><<<148, 32 * (4 * NWG + NWG * I)>>>(d, items);
  cudaDeviceSynchronize();
  pipe<NWG, R, I, NN><<<148, 32 * (4 * NWG + NWG * I)>>>(d, items);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("i8 pipe NWG=%d R=%d I=%d N=%d: %7.1f cycles per item per WG, %6.1f per item per CTA [%s]\n", NWG, R, I, NN, (double)h / items,
         (double)h / items / NWG, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  if (v == 0) {
    static uint8_t hA[128 * K];
    static int8_t hB[N * K];
    static int hD[128 * N];
    srand(1);
    for (int i = 0; i < 128 * K; ++i) hA[i] = rand() % 16;
    for (int i = 0; i < N * K; ++i) hB[i] = (int8_t)(rand() % 256 - 128);
    uint8_t* dA; int8_t* dB; int* dD;
    CK(cudaMalloc(&dA, sizeof hA)); CK(cudaMalloc(&dB, sizeof hB)); CK(cudaMalloc(&dD, sizeof hD));
    CK(cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice));
    check<<<1, 128>>>(dA, dB, dD);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        long s = 0;
        for (int k = 0; k < K; ++k) s += (long)hA[m * K + k] * hB[n * K + k];
        if (s != hD[m * N + n]) { if (bad < 5) printf("m=%d n=%d got %d want %ld\n", m, n, hD[m * N + n], s); ++bad; }
      }
    printf("i8 check: %d mismatches of %d\n", bad, 128 * N);
  }
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int items = 2048;
  switch (v) {
    case 1: run<1, 8, 1, 16>(d, items); break;
    case 2: run<4, 4, 1, 16>(d, items); break;
    case 3: run<4, 4, 2, 16>(d, items); break;
    case 4: run<3, 6, 2, 16>(d, items); break;
    case 5: run<4, 4, 1, 64>(d, items); break;
    case 6: run<2, 8, 2, 16>(d, items); break;
    case 7: run<4, 2, 2, 32>(d, items); break;
  }
  return 0;
}
