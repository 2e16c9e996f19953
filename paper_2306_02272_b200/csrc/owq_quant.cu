// owq_quant.cu -- OWQ quantization on the GPU: the step
// that produces the hot path's inputs, in fp64 so that its decisions (weak
// columns, grids, codes) are those of the paper's algorithm as the oracle
// states it:
//
//   H = 2 X X^T                               (Eq. 3; reading s1)
//   dead columns: H_jj := 1, W[:, j] := 0; H += percdamp mean(diag H) I   (s2)
//   Delta W = W - RTN_b(W), min-max grid per row / group on all columns  (s4)
//   sens_j = H_jj (undamped) ||Delta W_:,j||^2                  (Eq. 5)
//   weak = top-k sens (ties -> smaller index)                   (s5)
//   perm = non-weak ascending ++ weak ascending                 (s6)
//   U = upper Cholesky of (H_p)^-1                              (Eq. 1 row form)
//   OPTQ sweep over the non-weak positions, grids fitted when a group opens,
//   on its current (compensated) values, truncation-searched
//   codes un-permuted; weak codes := z; weak values = fp16 of the compensated
//   columns                                                     (s10)
//
// B200 mapping: everything is fp64 (DFMA on CUDA cores); the O(K^3) and
// O(M K^2) work is DGEMM-shaped (H, the Cholesky trailing updates, the
// triangular inverse, OPTQ's lazy-batch trailing updates) and runs in one tiled
// DGEMM kernel; the sequential parts (a 32-column Cholesky panel, the
// in-block OPTQ column sweep) run one thread per row with the block in shared
// memory.  U = R^-1 where R = P L' P and L' = chol(P H_p P) (P = index
// reversal): one Cholesky + one triangular inverse instead of the oracle's
// chol -> inv -> chol (same U up to rounding).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "owq.h"

namespace owq {
namespace qz {

// ---------------------------------------------------------------- fp64 GEMM
// C[m][n] = alpha * sum_k A(m, k) B(k, n) + beta * C[m][n]
// A(m, k) = TA ? A[k * lda + m] : A[m * lda + k];  B(k, n) = TB ? B[n * ldb + k] : B[k * ldb + n]
constexpr int GT = 64, GK = 16;
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) dgemm_kernel(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                    int64_t lda, const double* __restrict__ B, int64_t ldb,
                                                    double beta, double* __restrict__ C, int64_t ldc) {
  __shared__ double As[GK][GT + 1], Bs[GK][GT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * GT, n0 = blockIdx.x * GT;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += GK) {
    for (int e = threadIdx.x; e < GK * GT; e += 256) {
      const int kk = e / GT, mm = e % GT;
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? (TA ? A[(int64_t)k * lda + m] : A[(int64_t)m * lda + k]) : 0.0;
      const int n = n0 + mm;
      Bs[kk][mm] = (n < N && k < K) ? (TB ? B[(int64_t)n * ldb + k] : B[(int64_t)k * ldb + n]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) {
        double* c = C + (int64_t)m * ldc + n;
        *c = alpha * acc[i][j] + (beta == 0.0 ? 0.0 : beta * *c);
      }
    }
}

template <bool TA, bool TB>
static void dgemm(cudaStream_t s, int M, int N, int K, double alpha, const double* A, int64_t lda, const double* B,
                  int64_t ldb, double beta, double* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((N + GT - 1) / GT, (M + GT - 1) / GT);
  dgemm_kernel<TA, TB><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ double fp16_rne(double v) { return (double)__half2float(__double2half(v)); }

// grid (s, z) of a value range: reading s7 (0 on the grid), s12 (s rounded to fp16)
__device__ __forceinline__ void grid_from_range(double xmin, double xmax, int maxq, double& s, double& z) {
  xmin = fmin(xmin, 0.0);
  xmax = fmax(xmax, 0.0);
  if (xmin == 0.0 && xmax == 0.0) { xmin = -1.0; xmax = 1.0; }
  s = fp16_rne((xmax - xmin) / maxq);
  if (s == 0.0) s = 5.9604644775390625e-08;   // 2^-24
  z = fmin(fmax(rint(-xmin / s), 0.0), (double)maxq);
}
__device__ __forceinline__ double quant(double w, double s, double z, int maxq) {
  return fmin(fmax(rint(w / s) + z, 0.0), (double)maxq);
}

// block reductions (256 threads)
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (threadIdx.x == 0) sh[0] = r;
  }
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}
__device__ void block_minmax(double& lo, double& hi, double* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { sh[threadIdx.x >> 5] = lo; sh[32 + (threadIdx.x >> 5)] = hi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    double a = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : INFINITY;
    double b = threadIdx.x < (blockDim.x >> 5) ? sh[32 + threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (threadIdx.x == 0) { sh[0] = a; sh[32] = b; }
  }
  __syncthreads();
  lo = sh[0];
  hi = sh[32];
  __syncthreads();
}

// ---------------------------------------------------------------- Hessian conditioning
__global__ void diag_dead_kernel(double* H, int K, double* diag_orig, uint8_t* dead, double* W, int M) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  const double d = H[(int64_t)j * K + j];
  diag_orig[j] = d;
  dead[j] = d == 0.0;
  if (d == 0.0) {
    H[(int64_t)j * K + j] = 1.0;
    for (int i = 0; i < M; ++i) W[(int64_t)i * K + j] = 0.0;
  }
}
__global__ void damp_kernel(double* H, int K, double percdamp, int* bad) {
  __shared__ double sh[64];
  double v = 0.0;
  for (int j = threadIdx.x; j < K; j += blockDim.x) v += H[(int64_t)j * K + j];
  const double mean = block_sum(v, sh) / K;
  const double damp = percdamp * mean;
  for (int j = threadIdx.x; j < K; j += blockDim.x) H[(int64_t)j * K + j] += damp;
  if (threadIdx.x == 0 && !(mean > 0.0)) *bad = 1;
}

// ---------------------------------------------------------------- Eq. 5 sensitivity
// one CTA per row: RTN with the min-max grid per row / group on ALL columns (s4)
__global__ void rtn_delta_sq_kernel(const double* W, int M, int K, int group, int maxq, double* D) {
  __shared__ double sh[64];
  const int i = blockIdx.x;
  const double* w = W + (int64_t)i * K;
  const int gsz = group ? group : K;
  for (int c0 = 0; c0 < K; c0 += gsz) {
    const int c1 = min(K, c0 + gsz);
    double lo = INFINITY, hi = -INFINITY;
    for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) { lo = fmin(lo, w[j]); hi = fmax(hi, w[j]); }
    block_minmax(lo, hi, sh);
    double s, z;
    grid_from_range(lo, hi, maxq, s, z);
    for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
      const double d = w[j] - s * (quant(w[j], s, z, maxq) - z);
      D[(int64_t)i * K + j] = d * d;
    }
  }
}
__global__ void sensitivity_kernel(const double* D, int M, int K, const double* diag_orig, const uint8_t* dead,
                                   double* sens) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  double a = 0.0;
  for (int i = 0; i < M; ++i) a += D[(int64_t)i * K + j];
  sens[j] = dead[j] ? 0.0 : diag_orig[j] * a;
}

// top-k (ties -> smaller index), then weak list ascending and perm = non-weak ++ weak.
// One CTA of 1024 threads.
__global__ void select_kernel(const double* sens, int K, int k, uint8_t* flag, int* perm, uint16_t* weak_idx) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int cnt[1024];
  for (int j = threadIdx.x; j < K; j += blockDim.x) flag[j] = 0;
  __syncthreads();
  for (int t = 0; t < k; ++t) {
    double bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int j = threadIdx.x; j < K; j += blockDim.x)
      if (!flag[j] && (sens[j] > bv || (sens[j] == bv && j < bi))) { bv = sens[j]; bi = j; }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      bv = sv[0];
      bi = si[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) { bv = sv[w]; bi = si[w]; }
      flag[bi] = 1;
    }
    __syncthreads();
  }
  // ordered compaction: thread t owns the contiguous chunk [t*per, (t+1)*per)
  const int per = (K + blockDim.x - 1) / blockDim.x;
  const int a = threadIdx.x * per, b = min(K, a + per);
  int nw = 0;
  for (int j = a; j < b; ++j) nw += flag[j];
  cnt[threadIdx.x] = nw;
  __syncthreads();
  if (threadIdx.x == 0) {                // exclusive scan (1024 entries)
    int run = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) { const int c = cnt[t]; cnt[t] = run; run += c; }
  }
  __syncthreads();
  int wpos = cnt[threadIdx.x];
  int npos = a - wpos;                   // non-weak before this chunk
  for (int j = a; j < b; ++j) {
    if (flag[j]) { weak_idx[wpos] = (uint16_t)j; perm[K - k + wpos] = j; ++wpos; }
    else { perm[npos] = j; ++npos; }
  }
}

// A[a][b] = H[perm[K-1-a]][perm[K-1-b]]  (permuted, then index-reversed)
__global__ void gather_rev_kernel(const double* H, const int* perm, int K, double* A) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)K * K) return;
  const int a = (int)(e / K), b = (int)(e % K);
  A[e] = H[(int64_t)perm[K - 1 - a] * K + perm[K - 1 - b]];
}

// ---------------------------------------------------------------- Cholesky (lower, in place), 32-wide panels
constexpr int PB = 32;
__global__ void potrf_diag_kernel(double* A, int K, int k0, int nb, int* bad) {
  __shared__ double T[PB][PB + 1];
  const int t = threadIdx.x;   // PB x PB threads
  const int r = t / PB, c = t % PB;
  if (r < nb && c < nb) T[r][c] = A[(int64_t)(k0 + r) * K + k0 + c];
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (t == 0) {
      const double d = T[j][j];
      if (!(d > 0.0)) *bad = 1;
      T[j][j] = sqrt(fmax(d, 1e-300));
    }
    __syncthreads();
    if (c == j && r > j && r < nb) T[r][j] /= T[j][j];
    __syncthreads();
    if (r > j && c > j && c <= r && r < nb) T[r][c] -= T[r][j] * T[c][j];
    __syncthreads();
  }
  if (r < nb && c < nb) A[(int64_t)(k0 + r) * K + k0 + c] = c <= r ? T[r][c] : 0.0;
}
// rows i >= k0 + nb: L21[i, :] = A21[i, :] L11^-T (forward substitution per row)
__global__ void trsm_panel_kernel(double* A, int K, int k0, int nb) {
  __shared__ double L[PB][PB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) L[e / nb][e % nb] = A[(int64_t)(k0 + e / nb) * K + k0 + e % nb];
  __syncthreads();
  const int i = k0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  double* row = A + (int64_t)i * K + k0;
  double v[PB];
#pragma unroll
  for (int c = 0; c < PB; ++c) v[c] = c < nb ? row[c] : 0.0;
#pragma unroll
  for (int c = 0; c < PB; ++c) {
    if (c < nb) {
      double a = v[c];
#pragma unroll
      for (int m = 0; m < c; ++m) a -= v[m] * L[c][m];
      v[c] = a / L[c][c];
    }
  }
#pragma unroll
  for (int c = 0; c < PB; ++c) if (c < nb) row[c] = v[c];
}
__global__ void zero_upper_kernel(double* A, int K) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)K * K) return;
  const int a = (int)(e / K), b = (int)(e % K);
  if (b > a) A[e] = 0.0;
}

// R[a][b] = L'[K-1-a][K-1-b] (upper)
__global__ void reverse_kernel(const double* L, int K, double* R) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)K * K) return;
  const int a = (int)(e / K), b = (int)(e % K);
  R[e] = L[(int64_t)(K - 1 - a) * K + (K - 1 - b)];
}

// inverse of an upper-triangular diagonal block (n <= 32) of R into U (same place)
__global__ void trinv_small_kernel(const double* R, double* U, int ld, int o, int n) {
  __shared__ double T[PB][PB + 1], V[PB][PB + 1];
  const int t = threadIdx.x, r = t / PB, c = t % PB;
  if (r < n && c < n) T[r][c] = R[(int64_t)(o + r) * ld + o + c];
  __syncthreads();
  // column c of V = T^-1 by back substitution (thread c)
  if (t < n) {
    const int j = t;
    for (int i = PB - 1; i >= 0; --i) {
      if (i >= n) continue;
      if (i > j) { V[i][j] = 0.0; continue; }
      double a = i == j ? 1.0 : 0.0;
      for (int m = i + 1; m <= j; ++m) a -= T[i][m] * V[m][j];
      V[i][j] = a / T[i][i];
    }
  }
  __syncthreads();
  if (r < n && c < n) U[(int64_t)(o + r) * ld + o + c] = V[r][c];
}

// U = R^-1 for the upper-triangular block [o, o+n) (recursive halving with GEMMs):
// [[R11 R12] [0 R22]]^-1 = [[U11, -U11 R12 U22], [0, U22]]
static void trinv(cudaStream_t s, const double* R, double* U, int ld, int o, int n, double* T) {
  if (n <= PB) {
    trinv_small_kernel<<<1, PB * PB, 0, s>>>(R, U, ld, o, n);
    return;
  }
  const int h = ((n / 2) + PB - 1) / PB * PB;
  trinv(s, R, U, ld, o, h, T);
  trinv(s, R, U, ld, o + h, n - h, T);
  // T = U11 R12 (h x (n-h)), U12 = -T U22
  dgemm<false, false>(s, h, n - h, h, 1.0, U + (int64_t)o * ld + o, ld, R + (int64_t)o * ld + o + h, ld, 0.0, T, n - h);
  dgemm<false, false>(s, h, n - h, n - h, -1.0, T, n - h, U + (int64_t)(o + h) * ld + o + h, ld, 0.0,
                      U + (int64_t)o * ld + o + h, ld);
}

// ---------------------------------------------------------------- OPTQ sweep
// Wp[i][p] = W[i][perm[p]]
__global__ void gather_cols_kernel(const double* W, const int* perm, int M, int K, double* Wp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * K) return;
  const int i = (int)(e / K), p = (int)(e % K);
  Wp[e] = W[(int64_t)i * K + perm[p]];
}

// grid of each row on positions [c0, c1) of Wp (current values), truncation search
// (reading s8) or min-max; one CTA per row
__global__ void fit_kernel(const double* Wp, int M, int K, int c0, int c1, int maxq, int points, double* sg,
                           double* zg, int G, int gi) {
  __shared__ double sh[64];
  const int i = blockIdx.x;
  const double* w = Wp + (int64_t)i * K;
  double lo = INFINITY, hi = -INFINITY;
  for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) { lo = fmin(lo, w[j]); hi = fmax(hi, w[j]); }
  block_minmax(lo, hi, sh);
  const double xmin0 = fmin(lo, 0.0), xmax0 = fmax(hi, 0.0);
  double best_e = INFINITY, best_s = 0, best_z = 0;
  for (int pi = 0; pi < points; ++pi) {
    const double pp = 1.0 - pi / 100.0;
    double s, z;
    grid_from_range(pp * xmin0, pp * xmax0, maxq, s, z);
    double e = 0.0;
    for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
      const double d = w[j] - s * (quant(w[j], s, z, maxq) - z);
      e += d * d;
    }
    e = block_sum(e, sh);
    if (e < best_e) { best_e = e; best_s = s; best_z = z; }
  }
  if (threadIdx.x == 0) { sg[(int64_t)i * G + gi] = best_s; zg[(int64_t)i * G + gi] = best_z; }
}

// In-block OPTQ column sweep (Eq. 1, Cholesky-row form): one thread per row;
// positions [b0, b1) of Wp with U's diagonal block in shared memory.  Writes
// the codes (order positions) and the scaled errors E for the trailing update.
constexpr int SB = 128;       // max block width (a scale group, or 128 columns at g = 0)
constexpr int SR = 64;        // rows per CTA
__global__ void __launch_bounds__(SR) sweep_kernel(double* Wp, int M, int K, const double* U, int b0, int b1,
                                                   const double* sg, const double* zg, int G, int gi, int maxq,
                                                   uint8_t* codes_p, double* E) {
  extern __shared__ double sm[];
  const int n = b1 - b0;
  double* Ub = sm;                      // [n][n]
  double* Wr = sm + n * n;              // [SR][n + 1]
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) Ub[e] = U[(int64_t)(b0 + e / n) * K + b0 + e % n];
  const int r0 = blockIdx.x * SR;
  for (int e = threadIdx.x; e < SR * n; e += blockDim.x) {
    const int rr = e / n, c = e % n;
    Wr[rr * (n + 1) + c] = r0 + rr < M ? Wp[(int64_t)(r0 + rr) * K + b0 + c] : 0.0;
  }
  __syncthreads();
  const int i = r0 + threadIdx.x;
  if (i >= M) return;
  const double s = sg[(int64_t)i * G + gi], z = zg[(int64_t)i * G + gi];
  double* w = Wr + threadIdx.x * (n + 1);
  for (int c = 0; c < n; ++c) {
    const double q = quant(w[c], s, z, maxq);
    const double e = (w[c] - s * (q - z)) / Ub[c * n + c];
    codes_p[(int64_t)i * K + b0 + c] = (uint8_t)q;
    E[(int64_t)i * SB + c] = e;
    for (int l = c + 1; l < n; ++l) w[l] -= e * Ub[c * n + l];
  }
}

// codes (original order), weak codes := z, fp16 scale / zero / weak values
__global__ void assemble_kernel(const uint8_t* codes_p, const int* perm, const uint8_t* flag, const double* Wp,
                                const double* sg, const double* zg, int M, int K, int k, int group, int G,
                                uint8_t* codes, uint16_t* scale, uint16_t* zero, uint16_t* weak_val) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * K) return;
  const int i = (int)(e / K), p = (int)(e % K);
  const int j = perm[p];
  const int gi = group ? j / group : 0;
  if (p < K - k) {
    codes[(int64_t)i * K + j] = codes_p[(int64_t)i * K + p];
  } else {
    codes[(int64_t)i * K + j] = (uint8_t)zg[(int64_t)i * G + gi];
    weak_val[(int64_t)i * k + (p - (K - k))] = __half_as_ushort(__double2half(Wp[(int64_t)i * K + p]));
  }
  if (p < G) {
    scale[(int64_t)i * G + p] = __half_as_ushort(__double2half(sg[(int64_t)i * G + p]));
    zero[(int64_t)i * G + p] = __half_as_ushort(__double2half(zg[(int64_t)i * G + p]));
  }
}
__global__ void fill_kernel(double* a, int64_t n, double v) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) a[e] = v;
}

static inline unsigned blocks(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

struct Ws {     // workspace carve-up
  double *H, *A, *U, *T, *Wp, *D, *E, *sens, *diag, *sg, *zg;
  int* perm;
  uint8_t *flag, *dead, *codes_p;
  int* bad;
};
static size_t carve(Ws* w, uint8_t* base, int M, int K, int G) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* p = base ? base + off : nullptr;
    off += (bytes + 255) / 256 * 256;
    return p;
  };
  const size_t KK = (size_t)K * K * 8, MK = (size_t)M * K * 8;
  Ws t;
  t.H = (double*)take(KK); t.A = (double*)take(KK); t.U = (double*)take(KK); t.T = (double*)take(KK / 2 + 8);
  t.Wp = (double*)take(MK); t.D = (double*)take(MK); t.E = (double*)take((size_t)M * SB * 8);
  t.sens = (double*)take((size_t)K * 8); t.diag = (double*)take((size_t)K * 8);
  t.sg = (double*)take((size_t)M * G * 8); t.zg = (double*)take((size_t)M * G * 8);
  t.perm = (int*)take((size_t)K * 4); t.flag = take(K); t.dead = take(K); t.codes_p = take((size_t)M * K);
  t.bad = (int*)take(4);
  if (w) *w = t;
  return off;
}

}  // namespace qz
}  // namespace owq

using namespace owq::qz;

extern "C" {

size_t owq_quantize_workspace_bytes(int32_t c_out, int32_t c_in, int32_t n_samples, const owq_quant_params* prm) {
  if (!prm || c_out <= 0 || c_in <= 0 || c_in > 65536 || n_samples <= 0) return 0;
  const int G = prm->group_size ? (c_in + prm->group_size - 1) / prm->group_size : 1;
  return carve(nullptr, nullptr, c_out, c_in, G) + 256;
}

owq_status owq_quantize_gpu(int32_t M, int32_t K, int32_t N, const double* d_W, const double* d_X,
                            const owq_quant_params* prm, uint8_t* d_codes, uint16_t* d_scale, uint16_t* d_zero,
                            uint16_t* d_weak_idx, uint16_t* d_weak_val, void* d_ws, size_t ws_bytes, void* stream) {
  if (!prm || !d_W || !d_X || !d_codes || !d_scale || !d_zero || !d_ws) return OWQ_ERR_INVALID_ARG;
  if (M <= 0 || K <= 0 || N <= 0 || K > 65536) return OWQ_ERR_INVALID_ARG;
  const int bits = prm->bits, g = prm->group_size, k = prm->n_weak;
  if (bits < 2 || bits > 8) return OWQ_ERR_UNSUPPORTED;
  if (g < 0 || (g && g > SB) || k < 0 || k >= K) return OWQ_ERR_UNSUPPORTED;   // groups up to 128 columns
  if (k > 0 && (!d_weak_idx || !d_weak_val)) return OWQ_ERR_INVALID_ARG;
  if (!(prm->percdamp > 0.0)) return OWQ_ERR_INVALID_ARG;
  const int G = g ? (K + g - 1) / g : 1;
  if (ws_bytes < owq_quantize_workspace_bytes(M, K, N, prm)) return OWQ_ERR_BUFFER_TOO_SMALL;
  cudaStream_t s = (cudaStream_t)stream;
  Ws w;
  uint8_t* base = (uint8_t*)(((uintptr_t)d_ws + 255) & ~(uintptr_t)255);
  carve(&w, base, M, K, G);
  const int maxq = (1 << bits) - 1;
  cudaMemsetAsync(w.bad, 0, 4, s);
  // W working copy (dead columns are zeroed in it)
  cudaMemcpyAsync(w.D, d_W, (size_t)M * K * 8, cudaMemcpyDeviceToDevice, s);
  double* Wc = w.D;
  // H = 2 X X^T  (Eq. 3)
  dgemm<false, true>(s, K, K, N, 2.0, d_X, N, d_X, N, 0.0, w.H, K);
  diag_dead_kernel<<<blocks(K), 256, 0, s>>>(w.H, K, w.diag, w.dead, Wc, M);
  damp_kernel<<<1, 1024, 0, s>>>(w.H, K, prm->percdamp, w.bad);
  // Eq. 5 sensitivity on RTN Delta W (min-max grid on all columns), top-k, perm
  rtn_delta_sq_kernel<<<M, 256, 0, s>>>(Wc, M, K, g, maxq, w.Wp);
  sensitivity_kernel<<<blocks(K), 256, 0, s>>>(w.Wp, M, K, w.diag, w.dead, w.sens);
  select_kernel<<<1, 1024, 0, s>>>(w.sens, K, k, w.flag, w.perm, d_weak_idx ? d_weak_idx : (uint16_t*)w.T);
  // U: upper Cholesky factor of (H_p)^-1 = (P L' P)^-1, L' = chol(P H_p P)
  gather_rev_kernel<<<blocks((int64_t)K * K), 256, 0, s>>>(w.H, w.perm, K, w.A);
  for (int k0 = 0; k0 < K; k0 += PB) {
    const int nb = std::min(PB, K - k0);
    potrf_diag_kernel<<<1, PB * PB, 0, s>>>(w.A, K, k0, nb, w.bad);
    const int rest = K - k0 - nb;
    if (rest > 0) {
      trsm_panel_kernel<<<blocks(rest, 128), 128, 0, s>>>(w.A, K, k0, nb);
      dgemm<false, true>(s, rest, rest, nb, -1.0, w.A + (int64_t)(k0 + nb) * K + k0, K, w.A + (int64_t)(k0 + nb) * K + k0,
                         K, 1.0, w.A + (int64_t)(k0 + nb) * K + k0 + nb, K);
    }
  }
  zero_upper_kernel<<<blocks((int64_t)K * K), 256, 0, s>>>(w.A, K);
  reverse_kernel<<<blocks((int64_t)K * K), 256, 0, s>>>(w.A, K, w.H);   // R (upper) into H's buffer
  fill_kernel<<<blocks((int64_t)K * K), 256, 0, s>>>(w.U, (int64_t)K * K, 0.0);
  trinv(s, w.H, w.U, K, 0, K, w.T);
  // OPTQ sweep over the nq non-weak positions, lazy blocks aligned to the scale groups
  gather_cols_kernel<<<blocks((int64_t)M * K), 256, 0, s>>>(Wc, w.perm, M, K, w.Wp);
  fill_kernel<<<blocks((int64_t)M * G), 256, 0, s>>>(w.sg, (int64_t)M * G, 1.0);   // groups with only weak columns: s = 1,
  fill_kernel<<<blocks((int64_t)M * G), 256, 0, s>>>(w.zg, (int64_t)M * G, 0.0);   // z = 0 (the oracle's rule)
  const int nq = K - k;
  const int points = prm->clip ? 80 : 1;   // p = 1 - i/100, i < 80 (reading s8); 1 point = min-max
  // block boundaries: the positions where the (original-index) group changes, cut to <= SB
  if (g == 0) fit_kernel<<<M, 256, 0, s>>>(w.Wp, M, K, 0, nq, maxq, points, w.sg, w.zg, G, 0);
  // group runs in position order (the non-weak columns of one original group are
  // consecutive positions): the host walks the weak flags (one copy + sync; the
  // quantizer runs offline, off the hot path)
  std::vector<uint8_t> hflag(K);
  if (g) {
    cudaMemcpyAsync(hflag.data(), w.flag, K, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return OWQ_ERR_CUDA;
  }
  const size_t sweep_smem = (size_t)(SB * SB + SR * (SB + 1)) * 8;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sweep_smem) != cudaSuccess)
      return OWQ_ERR_CUDA;
    attr = true;
  }
  int pos = 0;
  int col = 0;   // original column cursor (g > 0)
  while (pos < nq) {
    int b1, gi = 0;
    if (g) {
      // next group with a non-weak column
      while (col < K && hflag[col]) ++col;
      gi = col / g;
      int cnt = 0;
      for (int j = gi * g; j < std::min(K, gi * g + g); ++j) cnt += !hflag[j];
      b1 = pos + cnt;
      col = std::min(K, gi * g + g);
      fit_kernel<<<M, 256, 0, s>>>(w.Wp, M, K, pos, b1, maxq, points, w.sg, w.zg, G, gi);
    } else {
      b1 = std::min(nq, pos + SB);
    }
    const int n = b1 - pos;
    sweep_kernel<<<blocks(M, SR), SR, (size_t)(n * n + SR * (n + 1)) * 8, s>>>(w.Wp, M, K, w.U, pos, b1, w.sg, w.zg, G,
                                                                               gi, maxq, w.codes_p, w.E);
    // trailing update of every later position (including the weak ones): Wp[:, b1:] -= E U[pos:b1, b1:]
    if (b1 < K)
      dgemm<false, false>(s, M, K - b1, n, -1.0, w.E, SB, w.U + (int64_t)pos * K + b1, K, 1.0, w.Wp + b1, K);
    pos = b1;
  }
  assemble_kernel<<<blocks((int64_t)M * K), 256, 0, s>>>(w.codes_p, w.perm, w.flag, w.Wp, w.sg, w.zg, M, K, k, g, G,
                                                         d_codes, d_scale, d_zero, d_weak_val);
  if (cudaGetLastError() != cudaSuccess) return OWQ_ERR_CUDA;
  int bad = 0;   // all-zero Hessian or a non-positive Cholesky pivot
  if (cudaMemcpyAsync(&bad, w.bad, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return OWQ_ERR_CUDA;
  return bad ? OWQ_ERR_INVALID_ARG : OWQ_OK;
}

}  // extern "C"
