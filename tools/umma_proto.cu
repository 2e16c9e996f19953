// Prototype: tcgen05.mma kind::f16, M=128 N=16 K=16, A from TMEM (written with
// tcgen05.st 32x32b), B from shared memory (K-major, no swizzle, core matrices
// 8 rows x 16 B), D fp32 in TMEM read back with tcgen05.ld.  Checked on the host.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int M = 128, N = 16, KSTEPS = 4;   // K = 64 (4 MMAs of K=16)

__global__ void proto(const __half* A, const __half* Bm, float* D, int nsteps) {
  // A: [128][64] row-major fp16, Bm: [N][64] (batch-major x), D: [128][N] fp32
  __shared__ __align__(128) uint8_t xs[N * 64 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B core-matrix layout: core (kc, nb) at (kc * (N/8) + nb) * 128; row r: 16 B = x[nb*8 + r][kc*8 .. +7]
  for (int i = tid; i < N * 64; i += blockDim.x) {
    const int n = i / 64, k = i % 64, kc = k / 8, nb = n / 8, r = n % 8;
    reinterpret_cast<__half*>(xs)[((kc * (N / 8) + nb) * 128 + r * 16) / 2 + (k % 8)] = Bm[n * 64 + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  // A columns [0, 32): lane = row, column c = fp16 pair (k = 2c, 2c+1); D columns [32, 48)
  if (warp < 4) {
    const int row = warp * 32 + lane;
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) {
      __half2 h = __halves2half2(A[row * 64 + 2 * c], A[row * 64 + 2 * c + 1]);
      r[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    const uint32_t ta = tb + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");   // smem B written by generic stores -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < nsteps; ++j) {
      const uint32_t baddr = sa(xs) + j * 2 * (N / 8) * 128;     // k-chunks 2j, 2j+1
      const uint64_t lbo = (N / 8) * 128, sbo = 128;
      const uint64_t desc = (uint64_t)((baddr >> 4) & 0x3FFF) | (((lbo >> 4) & 0x3FFF) << 16) |
                            (((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
      const uint32_t a_t = tb + j * 8;            // 8 columns = 16 fp16 per row
      const uint32_t d_t = tb + 32;
      const uint32_t acc = j > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_t),
          "r"(a_t), "l"(desc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
  }
  // wait for the MMAs
  asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n}" ::"r"(sa(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t d[16];
    const uint32_t ta = tb + 32 + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                   "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + lane;
    for (int n = 0; n < N; ++n) D[row * N + n] = __uint_as_float(d[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tb));
}

int main() {
  const int K = 64;
  __half hA[M * K], hB[N * K];
  float ref[M * N], out[M * N];
  for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) hA[m * K + k] = __float2half((float)(((m * 7 + k * 3) % 15) - 7));
  for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) hB[n * K + k] = __float2half((float)((n * 5 + k * 11) % 9 - 4) * 0.25f + (k == 5 ? n : 0));
  for (int steps = 1; steps <= KSTEPS; steps *= 2) {
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
      double s = 0; for (int k = 0; k < 16 * steps; ++k) s += (double)__half2float(hA[m * K + k]) * __half2float(hB[n * K + k]);
      ref[m * N + n] = (float)s;
    }
    __half *dA, *dB; float* dD;
    CK(cudaMalloc(&dA, sizeof hA)); CK(cudaMalloc(&dB, sizeof hB)); CK(cudaMalloc(&dD, sizeof out));
    CK(cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0, sizeof out));
    proto<<<1, 128>>>(dA, dB, dD, steps);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dD, sizeof out, cudaMemcpyDeviceToHost));
    int bad = 0; double maxe = 0;
    for (int i = 0; i < M * N; ++i) { double e = fabs(out[i] - ref[i]); maxe = fmax(maxe, e); bad += e > 1e-3; }
    printf("steps=%d (K=%d): mismatches %d / %d, max abs err %.3g; D[0][0..3] = %g %g %g %g ref %g %g %g %g\n", steps, 16 * steps, bad, M * N, maxe,
           out[0], out[1], out[2], out[3], ref[0], ref[1], ref[2], ref[3]);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
  }
  return 0;
}
