// owq_prefill.cu -- the mixed OWQ matmul for many tokens (SURVEY §8(f) NEXT-2,
// "prefill"): Y = W_hat X with X = B tokens x C_in (X in R^{C_in x N};
// the same representation as the GEMV), B = 17 .. any, per-row scales,
// blob layout 3 (the tensor-core layout of the GEMV).
//
// At 64-2048 tokens the product is a dense contraction (2 B flops per code
// byte x 8/3), so it runs on the 5th-generation tensor cores:
//   A (weights)  = the EXACT integer (q - z) as fp16 (|q - z| <= 15), decoded
//                  from the packed codes by 4 warps (thread = row): the layout-3
//                  LOP3 decode to code bytes, one PRMT per 2 codes that places
//                  them under the 1024 fp16 exponent (1024 + q), one HSUB2 of
//                  1024 + z -- written to shared memory in the UMMA K-major
//                  core-matrix layout;
//   B (tokens)   = x fp16 as given, cp.async'ed into the same layout;
//   D            = fp32 in TMEM (128 rows x 256 tokens), tcgen05.mma.kind::f16,
//                  4 MMAs (K = 16) per 64-column super-step, one issuing thread.
// fp16 x fp16 products are exact in the fp32 accumulator; the scale s is
// applied once per row after the sum (reading s19: never an fp16-rounded
// s (q - z), SURVEY §8(c) scheme D).  The fp16 weak columns are folded in by
// the epilogue (fp16 x fp16 in fp32).
//
// Tile: one CTA = two 128-row blocks (sharing one x tile; two D accumulators
// fill the 512 TMEM columns) x 256 tokens; grid = (token tiles, row-block
// pairs), token tile fastest so the CTAs sharing weights run together and read
// the codes from L2.  3-stage ring: codes (TMA bulk), A tiles (8 decode warps,
// which are also the epilogue), B tile (4 loader warps, cp.async groups with
// one stage of lookahead); the MMA warp commits each stage's MMAs to the
// stage's `empty` barrier.  Measured 385-425 dense-equivalent TFLOP/s at 1-2k
// tokens (profiles/r2_prefill_time.txt): bound by moving the x tile through
// L2 with cp.async, not by the tensor cores.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "owq.h"
#include "owq_layout.h"
#include "owq_ptx.cuh"

namespace owq {
namespace pf {

using namespace owq::ptx;

constexpr int NT = 256;                  // tokens per CTA (MMA N)
constexpr uint32_t A_BYTES = 128 * 64 * 2;       // 16 KB per row-block: [8 K-chunks][16 row groups][8 rows][16 B]
constexpr uint32_t B_BYTES = NT * 64 * 2;        // 32 KB: 256 token rows x 128 B (128-byte swizzle)
constexpr uint32_t C_MAX = 128 * 8 * 4;          // codes of one row-block super-step (4-bit: 8 words per row)
// RB 128-row blocks per CTA share each x tile: 2 by default (one D of 256 TMEM
// columns each), 1 when two-row-block CTAs would leave SMs idle (few tokens)
template <int RB_>
struct PfCfg {
  static constexpr int RB = RB_;
  static constexpr int NST = RB == 2 ? 3 : 4;                                 // pipeline stages
  static constexpr uint32_t STAGE = RB * A_BYTES + B_BYTES + RB * C_MAX;
  static constexpr int kDecW = 4 * RB;            // decode (then epilogue) warps: thread = row
  static constexpr int kLoadW = 1;                // x loader warp (one lane issues the TMA tile loads)
  static constexpr int kProdW = kDecW + kLoadW, kMmaW = kProdW + 1;
  static constexpr int kThreads = (kMmaW + 1) * 32;
  static constexpr uint32_t kSmem = NST * STAGE + 1024 + 256;
  static constexpr uint32_t kTmemCols = RB * NT;
};

struct Params {
  CUtensorMap xmap;    // x [B][K] fp16, box 64 columns x NT tokens, 128-byte swizzle (zero fill out of range)
  const uint8_t* blob;
  const __half* x;     // [B][K]
  void* y;             // [B][M]
  Geo g;
  int32_t B, y_f32;
  int32_t KS, sps;     // K splits and super-steps per split (KS = 1: no split)
  float* part;         // KS > 1: [KS][B][Mp] fp32 partial rows (Mp = nrb x 128), summed by owq_prefill_reduce_kernel
};

// one row's 64 codes of a super-step -> 16 words of 4 code bytes (layout 3)
template <int BITS>
__device__ __forceinline__ void decode_row(const uint32_t* w, uint32_t* o) {
  if (BITS == 4) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i] = w[i] & 0x0F0F0F0Fu;
      o[8 + i] = (w[i] >> 4) & 0x0F0F0F0Fu;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      o[i] = w[i] & 0x07070707u;
      o[6 + i] = (w[i] >> 3) & 0x07070707u;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      o[12 + r] = ((w[r] >> 6) & 0x03030303u) | ((w[4 + (r >> 1)] >> ((r & 1) ? 5 : 4)) & 0x04040404u);
  }
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

#ifdef OWQ_EXPERIMENTS
// per-stage clock64 stamps of CTA (0, 0): events 0 producer after empty, 1 decode
// after full, 2 decode arrive, 3 MMA after afull, 4 MMA after bfull, 5 loader after
// empty, 6 loader arrive; per CTA: globaltimer start, loader pdl done, dfull seen, exit
__device__ long long g_pf_trace[8][256];
__device__ unsigned long long g_pf_cta[4][2048];
#define PF_TR(ev, l) do { if (blockIdx.x == 0 && blockIdx.y == 0 && (l) < 256) g_pf_trace[ev][l] = clock64(); } while (0)
#define PF_CTA(ev) do { const int c_ = blockIdx.y * gridDim.x + blockIdx.x; unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); if (c_ < 2048) g_pf_cta[ev][c_] = t_; } while (0)
#else
#define PF_TR(ev, l) do { } while (0)
#define PF_CTA(ev) do { } while (0)
#endif

template <int BITS, int RB_>
__global__ void __launch_bounds__(PfCfg<RB_>::kThreads, 1) owq_prefill_kernel(const __grid_constant__ Params p) {
  using C = PfCfg<RB_>;
  constexpr int RB = C::RB, NST = C::NST, kDecW = C::kDecW, kProdW = C::kProdW, kMmaW = C::kMmaW;
  constexpr uint32_t STAGE = C::STAGE;
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geo& g = p.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, rb0 = blockIdx.y * RB;
  const int nss = g.nss;
  const int split = blockIdx.z;                                      // K split (p.KS > 1, prefill with a workspace)
  const int ss0 = split * p.sps, nl = min(nss, ss0 + p.sps) - ss0;   // this CTA's super-steps
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + NST * STAGE);
  uint64_t* full = bars;               // codes landed (TMA tx)
  uint64_t* afull = full + NST;        // A tiles written (RB x 128 threads)
  uint64_t* bfull = afull + NST;       // B tile landed (TMA tx)
  uint64_t* empty = bfull + NST;       // the stage's MMAs completed (tcgen05.commit)
  uint64_t* dfull = empty + NST;       // all MMAs completed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dfull + 1);
  auto A = [&](int s, int h) { return base + (size_t)s * STAGE + (size_t)h * A_BYTES; };
  auto Bt = [&](int s) { return base + (size_t)s * STAGE + RB * A_BYTES; };
  auto Cd = [&](int s, int h) { return base + (size_t)s * STAGE + RB * A_BYTES + B_BYTES + (size_t)h * C_MAX; };
  const int nrb_here = min(RB, g.nrb - rb0);   // row-blocks of this CTA (the last CTA may have one)
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&afull[s], RB * 128);
      mbar_init(&bfull[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(dfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kProdW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t ssb = (uint32_t)g.ss_bytes;
  if (threadIdx.x == 0) PF_CTA(0);

  if (warp == kProdW) {
    // ------------------------------------------------ producer: codes of each super-step (TMA bulk)
    if (lane == 0) {
      pdl_launch_dependents();
      for (int l = 0; l < nl; ++l) {
        const int ss = ss0 + l;
        const int s = l % NST;
        if (l >= NST) mbar_wait(&empty[s], (uint32_t)((l / NST) - 1) & 1u);
        PF_TR(0, ss);
        mbar_expect_tx(&full[s], ssb * nrb_here);
        for (int h = 0; h < nrb_here; ++h)
          bulk_g2s(Cd(s, h), p.blob + g.units_off + item_offset(g, rb0 + h, ss), ssb, &full[s]);
      }
    }
  } else if (warp == kMmaW) {
    // ------------------------------------------------ MMA issue (one thread): per row-block h,
    // D_h (TMEM columns 256 h ..) += A_h x B
    constexpr uint32_t idesc = idesc_f16(128, NT);
    for (int l = 0; l < nl; ++l) {
        const int ss = ss0 + l;
      const int s = l % NST;
      const uint32_t ph = (uint32_t)(l / NST) & 1u;
      mbar_wait(&afull[s], ph);
      if (lane == 0) PF_TR(3, ss);
      mbar_wait(&bfull[s], ph);
      if (lane == 0) PF_TR(4, ss);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t b0 = smem_u32(Bt(s));
        for (int h = 0; h < nrb_here; ++h) {
          const uint32_t a0 = smem_u32(A(s, h));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)   // K = 16 per MMA: A two 8-element core-matrix columns, B 32 bytes into each swizzled row
            tc_mma_f16_ss(tmem + (uint32_t)(h * NT), umma_desc(a0 + kk * 2 * 2048, 2048, 128),
                          umma_desc_sw128(b0 + kk * 32), idesc, (l | kk) != 0 ? 1u : 0u);
        }
        tc_commit(&empty[s]);
        if (l == nl - 1) tc_commit(dfull);
      }
      __syncwarp();
    }
  } else if (warp < kDecW) {
    // ------------------------------------------------ decode: thread = weight row of row-block h
    const int h = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const int rb = rb0 + h;
    const bool live = h < nrb_here;
    const uint32_t szw = live ? __ldg(reinterpret_cast<const uint32_t*>(p.blob + g.sz_off + (int64_t)rb * kSZBlockBytes) + r) : 0u;
    const float z = __high2float(*reinterpret_cast<const __half2*>(&szw));
    const __half2 zz = __float2half2_rn(1024.f + z);   // exact: z <= 15
    const uint32_t zzw = *reinterpret_cast<const uint32_t*>(&zz);
    constexpr int WPR = BITS == 3 ? 6 : 8;
    for (int l = 0; l < nl; ++l) {
        const int ss = ss0 + l;
      const int s = l % NST;
      mbar_wait(&full[s], (uint32_t)(l / NST) & 1u);
      if (threadIdx.x == 0) PF_TR(1, ss);
      if (!live) {          // the CTA's second row-block does not exist: nothing to decode
        mbar_arrive(&afull[s]);
        continue;
      }
      const uint8_t* rec = Cd(s, h);
      uint32_t w[8], o[16];
#pragma unroll
      for (int i = 0; i < WPR; ++i) w[i] = *reinterpret_cast<const uint32_t*>(rec + row_word_byte(BITS, r, i));
      decode_row<BITS>(w, o);
      const uint32_t arow = smem_u32(A(s, h)) + (uint32_t)(r >> 3) * 128u + (uint32_t)(r & 7) * 16u;
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) {   // columns 8kc .. 8kc+7 = code words 2kc, 2kc+1
        const uint32_t w0 = o[2 * kc], w1 = o[2 * kc + 1];
        const uint32_t h0 = hsub2(prmt(w0, 0x64646464u, 0x4140u), zzw);   // (q - z) of columns 8kc, 8kc+1
        const uint32_t h1 = hsub2(prmt(w0, 0x64646464u, 0x4342u), zzw);
        const uint32_t h2 = hsub2(prmt(w1, 0x64646464u, 0x4140u), zzw);
        const uint32_t h3 = hsub2(prmt(w1, 0x64646464u, 0x4342u), zzw);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(arow + kc * 2048u), "r"(h0), "r"(h1), "r"(h2),
                     "r"(h3)
                     : "memory");
      }
      fence_proxy_async();
      mbar_arrive(&afull[s]);
      if (threadIdx.x == 0) PF_TR(2, ss);
    }
    // ---- epilogue (the decode warps): thread = row, TMEM lane quarter = warp % 4, D_h.
    // The weak fold reads x at the weak columns from shared memory: per 16 tokens
    // the 8 warps gather x[tokens][widx] once (k x 16 values), and the rows' fp16
    // weak values are staged once when they fit.  (Round 2's first version loaded
    // both from global memory inside the token loop: 200+ us of a 500 us CTA at
    // 12288^2 x 2048 tokens, tools/pf_trace.py.)  The ring is free once dfull
    // completed (all MMAs done), so the staging reuses it.
    {
    const int q = warp & 3;
    const int et = threadIdx.x;                      // 0 .. 8 x 32 - 1 (decode warps)
    constexpr int kEpiT = kDecW * 32;
    const int64_t tok0 = (int64_t)tile * NT;
    const int64_t grow = (int64_t)rb * kRowBlock + r;
    const uint32_t szw = live ? __ldg(reinterpret_cast<const uint32_t*>(p.blob + g.sz_off + (int64_t)rb * kSZBlockBytes) + r) : 0u;
    const float sc = __low2float(*reinterpret_cast<const __half2*>(&szw));
    pdl_wait();   // y (and x) belong to earlier kernels until they complete
    mbar_wait(dfull, 0);
    if (threadIdx.x == 0) PF_CTA(2);
    if (threadIdx.x == 0) PF_TR(7, 15);
    tc_fence_after();
    const uint16_t* widx = reinterpret_cast<const uint16_t*>(p.blob + g.widx_off);
    const uint8_t* wrec = p.blob + g.units_off + (int64_t)rb * g.rb_bytes + (int64_t)g.nss * g.ss_bytes;
    const int k = split == 0 ? g.k : 0;   // the weak fold goes into the first K split only
    auto wval = [&](int tt) {
      const int ch = tt / kWeakChunk, c = tt % kWeakChunk;
      return ch < g.nfull ? *reinterpret_cast<const __half*>(wrec + (int64_t)ch * kWeakChunkBytes + (r * kWeakChunk + c) * 2)
                          : *reinterpret_cast<const __half*>(wrec + (int64_t)g.nfull * kWeakChunkBytes + (r * g.ktail + c) * 2);
    };
    // x at the weak columns: all NT tokens at once when they fit next to the staged
    // weak values ([c16][k][16]), else two token groups at a time ([2][k][16]); the
    // weak indices are staged too.  Loads are issued four / eight at a time (the loops
    // were latency-bound on one dependent global load per element).
    const size_t ring = (size_t)NST * STAGE;
    const size_t wis_bytes = ((size_t)k * 2 + 127) & ~(size_t)127;
    const bool xall = (size_t)k * NT * 2 + 128 + (size_t)RB * k * 256 + wis_bytes <= ring;
    const size_t xw_bytes = ((size_t)k * (xall ? NT : 32) * 2 + 127) & ~(size_t)127;   // else two token groups per pass
    uint16_t* wis = reinterpret_cast<uint16_t*>(base);                      // [k] weak indices
    __half* xw = reinterpret_cast<__half*>(base + wis_bytes);
    __half* wsm = reinterpret_cast<__half*>(base + wis_bytes + xw_bytes);  // [RB][k][128]
    const bool wstaged = wis_bytes + xw_bytes + (size_t)RB * k * 256 <= ring;
    for (int tt = et; tt < k; tt += kEpiT) wis[tt] = __ldg(widx + tt);
    if (wstaged && live)
      for (int t0 = 0; t0 < k; t0 += 4) {
        __half wv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) wv[u] = t0 + u < k ? wval(t0 + u) : __float2half(0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t0 + u < k) wsm[((size_t)h * k + t0 + u) * 128 + r] = wv[u];
      }
    named_sync(1, kEpiT);   // wis (and wsm) written
    if (et == 0) PF_TR(7, 0);
    auto gather = [&](int c0, int nc) {   // token groups c0 .. c0 + nc - 1 -> xw[(c - c0)][tt][16]
      const int total = nc * k * 16;
      for (int i0 = et; i0 < total; i0 += 8 * kEpiT) {
        __half xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * kEpiT;
          xv[u] = __float2half(0.f);
          if (i < total) {
            const int c = i / (k * 16), rem = i - c * k * 16, tt = rem >> 4, jj = rem & 15;
            const int64_t n = tok0 + (c0 + c) * 16 + jj;
            if (n < p.B) xv[u] = p.x[n * g.K + wis[tt]];
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u * kEpiT < total) xw[i0 + u * kEpiT] = xv[u];
      }
    };
    if (xall) {
      gather(0, NT / 16);
      named_sync(1, kEpiT);
    }
    if (et == 0) PF_TR(7, 1);
    // two token groups per pass: two TMEM loads behind one wait, each weak value read
    // once, the fold as FFMA2 pairs; the pass's 32 tokens x 256 rows of y are staged
    // in shared memory and written as 16-byte vectors along the rows (each warp
    // writing 2-byte elements of 32 rows per token measured ~4000 cycles per pass).
    const int ysz = p.y_f32 ? 4 : 2;
    uint8_t* ystage = base + wis_bytes + xw_bytes + (wstaged ? (((size_t)RB * k * 256 + 127) & ~(size_t)127) : 0);
    const bool ystaged = p.KS == 1 && (size_t)(ystage - base) + (size_t)32 * RB * 128 * ysz <= ring;
    const int rows_here = nrb_here * 128;
    for (int c16 = 0; c16 < NT / 16; c16 += 2) {
      if (!xall) {
        named_sync(1, kEpiT);   // the previous token groups' readers are done with xw
        gather(c16, 2);
        named_sync(1, kEpiT);
      } else if (ystaged) {
        named_sync(1, kEpiT);   // the previous pass's ystage readers are done
      }
      if (live) {
        const __half* xg = xw + (xall ? (size_t)c16 * k * 16 : 0);
        uint32_t d[32];
        tc_ld16_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * NT + c16 * 16), d);
        tc_ld16_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * NT + c16 * 16 + 16), d + 16);
        tc_wait_ld32(d);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = sc * __uint_as_float(d[j]);
        // fp16 weak columns x the tokens' fp16 activations at their indices
        for (int tt = 0; tt < k; ++tt) {
          const float wf = __half2float(wstaged ? wsm[((size_t)h * k + tt) * 128 + r] : wval(tt));
          const unsigned long long wf2 = ((unsigned long long)__float_as_uint(wf) << 32) | __float_as_uint(wf);
#pragma unroll
          for (int gq = 0; gq < 2; ++gq) {
            const uint4* xv = reinterpret_cast<const uint4*>(xg + ((size_t)gq * k + tt) * 16);
            const uint4 x0 = xv[0], x1 = xv[1];
            const uint32_t xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&xs[c]));
              const unsigned long long fx = ((unsigned long long)__float_as_uint(f.y) << 32) | __float_as_uint(f.x);
              float& a0 = v[16 * gq + 2 * c];
              float& a1 = v[16 * gq + 2 * c + 1];
              unsigned long long acc = ((unsigned long long)__float_as_uint(a1) << 32) | __float_as_uint(a0);
              asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(wf2), "l"(fx));
              a0 = __uint_as_float((uint32_t)acc);
              a1 = __uint_as_float((uint32_t)(acc >> 32));
            }
          }
        }
        if (p.KS > 1) {
          // K split: this split's fp32 partial rows (owq_prefill_reduce_kernel sums them)
          const int64_t Mp = (int64_t)g.nrb * kRowBlock;
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int64_t n = tok0 + c16 * 16 + jj;
            if (n < p.B) __stcg(&p.part[((int64_t)split * p.B + n) * Mp + grow], v[jj]);
          }
        } else if (ystaged) {
          // ystage[token j][row h*128 + r]
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const size_t o = ((size_t)jj * RB * 128 + (size_t)h * 128 + r) * ysz;
            if (p.y_f32) *reinterpret_cast<float*>(ystage + o) = v[jj];
            else *reinterpret_cast<__half*>(ystage + o) = __float2half_rn(v[jj]);
          }
        } else if (grow < g.M) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int64_t n = tok0 + c16 * 16 + jj;
            if (n < p.B) {
              if (p.y_f32) reinterpret_cast<float*>(p.y)[n * g.M + grow] = v[jj];
              else reinterpret_cast<__half*>(p.y)[n * g.M + grow] = __float2half_rn(v[jj]);
            }
          }
        }
      }
      if (ystaged) {
        named_sync(1, kEpiT);   // the pass's 32 tokens are staged
        // each token's rows_here rows are contiguous in y: 16-byte vectors, rows past M
        // (the last row-block) element by element
        const int vec = 16 / ysz;                       // elements per vector
        const int per_tok = rows_here / vec;
        for (int i = et; i < 32 * per_tok; i += kEpiT) {
          const int jj = i / per_tok, e0 = (i - jj * per_tok) * vec;
          const int64_t n = tok0 + c16 * 16 + jj;
          if (n >= p.B) continue;
          const int64_t row0 = (int64_t)rb0 * 128 + e0;
          const uint8_t* src = ystage + ((size_t)jj * RB * 128 + e0) * ysz;
          uint8_t* dst = reinterpret_cast<uint8_t*>(p.y) + (n * g.M + row0) * ysz;
          if (row0 + vec <= g.M && !(reinterpret_cast<uintptr_t>(dst) & 15)) {
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
          } else {
            for (int e = 0; e < vec && row0 + e < g.M; ++e) {
              if (p.y_f32) reinterpret_cast<float*>(dst)[e] = reinterpret_cast<const float*>(src)[e];
              else reinterpret_cast<__half*>(dst)[e] = reinterpret_cast<const __half*>(src)[e];
            }
          }
        }
      }
    }
    }
  } else if (warp < kProdW) {
    // ------------------------------------------------ x loader: one lane, TMA tensor tiles of
    // 64 columns x NT tokens in the 128-byte-swizzled K-major layout the MMA reads
    // (round 2's first version used 4 warps of 16-byte cp.async, whose issue
    // stalled behind the decode warps' shared-memory stores)
    const int64_t tok0 = (int64_t)tile * NT;
    if (lane == 0) {
      pdl_wait();   // x belongs to earlier kernels until they complete
      PF_CTA(1);
      for (int l = 0; l < nl; ++l) {
        const int ss = ss0 + l;
        const int s = l % NST;
        if (l >= NST) mbar_wait(&empty[s], (uint32_t)((l / NST) - 1) & 1u);
        PF_TR(5, ss);
        mbar_expect_tx(&bfull[s], B_BYTES);
        tma_load_2d(Bt(s), &p.xmap, ss * 64, (int)tok0, &bfull[s]);
        PF_TR(6, ss);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProdW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
  }
  if (threadIdx.x == 0) PF_CTA(3);
}

template <int RB>
static owq_status launch_rb(Params& p, const Geo& g, int B, cudaStream_t stream);

// y[n][row] = sum over the K splits, in split order, of the fp32 partial rows
// (four rows per thread)
__global__ void owq_prefill_reduce_kernel(const float* __restrict__ part, int KS, int B, int64_t M, int64_t Mp,
                                          void* y, int y_f32) {
  pdl_wait();   // the partials come from the prefill kernel just before
  const int64_t q4 = (M + 3) / 4;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * q4) return;
  const int64_t n = i / q4, row = (i - n * q4) * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int sp = 0; sp < KS; ++sp) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(part + ((int64_t)sp * B + n) * Mp + row));
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  const float vv[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (row + e >= M) break;
    if (y_f32) reinterpret_cast<float*>(y)[n * M + row + e] = vv[e];
    else reinterpret_cast<__half*>(y)[n * M + row + e] = __float2half_rn(vv[e]);
  }
}

// Row-blocks per CTA (waves x per-CTA time, a one-row-block CTA taking ~0.6 of a
// two-row-block one: half the decode and MMAs, the same x tile) and K splits.
// Precision: the tensor core's fp32 accumulation over a long K loop is not
// round-to-nearest per add -- one TMEM accumulator over 192 super-steps (K =
// 12288) already exceeds the 2e-3 bound on near-zero outputs, K = 49152 reaches
// 1.3e-2 (tools/pf_precision.py) -- so every split is at most kPfChain
// super-steps and the splits are added in fp32 on CUDA cores in split order.
// Fill: when even one-row-block CTAs would fill at most half the SMs, more
// splits (up to 8, >= 4 super-steps each).
constexpr int kPfChain = 64;
struct PfPlan { int rb, ks, sps; };
static int pf_sms() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}
static PfPlan pf_plan(const Geo& g, int B, int sms) {
  const int64_t tiles = (B + NT - 1) / NT;
  const int64_t w2 = (tiles * ((g.nrb + 1) / 2) + sms - 1) / sms, w1 = (tiles * g.nrb + sms - 1) / sms;
  PfPlan pl{6 * w1 < 10 * w2 ? 1 : 2, 1, g.nss};
  int ks = (g.nss + kPfChain - 1) / kPfChain;                       // precision
  const int64_t ctas1 = tiles * g.nrb;
  if (2 * ctas1 <= sms) {                                            // fill
    int kf = (int)std::min<int64_t>(8, sms / ctas1);
    while (kf > 1 && (g.nss + kf - 1) / kf < 4) --kf;
    if (kf > ks) { ks = kf; pl.rb = 1; }
  }
  if (ks > 1) {
    pl.sps = (g.nss + ks - 1) / ks;
    pl.ks = (g.nss + pl.sps - 1) / pl.sps;
  }
  return pl;
}
size_t workspace_bytes(const Geo& g, int B) {
  const PfPlan pl = pf_plan(g, B, pf_sms());
  return pl.ks > 1 ? (size_t)pl.ks * B * g.nrb * kRowBlock * 4 : 0;
}

owq_status launch(const Geo& g, const void* blob, const uint16_t* x, int B, void* y, int y_f32, void* ws,
                  size_t ws_bytes, cudaStream_t stream) {
  Params p{};
  p.blob = (const uint8_t*)blob;
  p.x = (const __half*)x;
  p.y = y;
  p.g = g;
  p.B = B;
  p.y_f32 = y_f32 ? 1 : 0;
  {
    // x as a 2-D tensor map: dims {K, B}, row pitch 2K bytes (K % 8 == 0 checked by
    // the caller), box {64, NT}, 128-byte swizzle; rows past B and columns past K
    // read as zero.  The driver entry point is looked up once.
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !fn)
        return OWQ_ERR_CUDA;
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)g.K, (cuuint64_t)B};
    const cuuint64_t strides[1] = {(cuuint64_t)g.K * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)NT};
    const cuuint32_t estr[2] = {1, 1};
    if (encode(&p.xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(x), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return OWQ_ERR_CUDA;
  }
  PfPlan pl = pf_plan(g, B, pf_sms());
  if (pl.ks > 1 && (!ws || ws_bytes < (size_t)pl.ks * B * g.nrb * kRowBlock * 4))
    return OWQ_ERR_BUFFER_TOO_SMALL;   // the K split needs owq_prefill_workspace_bytes() of scratch
#ifdef OWQ_EXPERIMENTS
  if (const char* v = getenv("OWQ_PF_RB")) pl.rb = atoi(v) == 1 ? 1 : 2;
#endif
  p.KS = pl.ks;
  p.sps = pl.sps;
  p.part = pl.ks > 1 ? (float*)ws : nullptr;
  const owq_status st = pl.rb == 1 ? launch_rb<1>(p, g, B, stream) : launch_rb<2>(p, g, B, stream);
  if (st != OWQ_OK || pl.ks == 1) return st;
  // the deterministic sum of the splits (PDL: launches while the prefill drains)
  const int64_t q4 = (g.M + 3) / 4, n = (int64_t)B * q4;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((unsigned)((n + 255) / 256));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, owq_prefill_reduce_kernel, (const float*)p.part, pl.ks, B, (int64_t)g.M,
                     (int64_t)g.nrb * kRowBlock, y, y_f32 ? 1 : 0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "owq: launch of owq_prefill_reduce_kernel failed: %s\n", cudaGetErrorString(e));
    return OWQ_ERR_CUDA;
  }
  return OWQ_OK;
}

template <int RB>
static owq_status launch_rb(Params& p, const Geo& g, int B, cudaStream_t stream) {
  using C = PfCfg<RB>;
  auto kern = g.bits == 3 ? owq_prefill_kernel<3, RB> : owq_prefill_kernel<4, RB>;
  int dev = 0;
  cudaGetDevice(&dev);
  static bool configured[2][16] = {};
  if (!configured[g.bits == 3][dev & 15]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem) != cudaSuccess)
      return OWQ_ERR_CUDA;
    configured[g.bits == 3][dev & 15] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((unsigned)((B + NT - 1) / NT), (unsigned)((g.nrb + RB - 1) / RB), (unsigned)p.KS);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "owq: launch of owq_prefill_kernel failed: %s\n", cudaGetErrorString(e));
    return OWQ_ERR_CUDA;
  }
  return OWQ_OK;
}

// ============================================================================
// Small-batch tensor-core GEMM (B = 2 .. 32): the same A
// operand as the prefill -- the exact integer (q - z) as fp16 decoded into
// shared memory -- against x as the fp16 B operand with N = B padded to 16 /
// 32, so the MMA work per code does not grow with a digit expansion and TMEM
// holds only the small D accumulators.  Grouped scales: one D buffer per scale
// group (4 buffers in rotation); the epilogue warps drain a group's D into
// fp32 registers as tot += s_g D_g while the MMAs run on the next group.  The
// machine is filled by splitting K over the grid (split boundaries on group
// boundaries); partial rows go to the workspace and the last-arriving split of
// a row-block sums them in split order (deterministic), then resets its counter.
// ============================================================================
namespace sb {

// experiment builds only: OWQ_SB_SKIP switches roles' work off (timing); the
// product kernel has the skip mask folded to zero at compile time
#ifdef OWQ_EXPERIMENTS
#define SB_SKIP(m) (p.skip & (m))
#else
#define SB_SKIP(m) 0
#endif
#ifdef OWQ_EXPERIMENTS
// per-stage clock64 stamps of CTA (0, 0): [event][stage], events 0 producer after
// empty, 1 decode after full, 2 decode arrive afull, 3 MMA after afull, 4 MMA after
// bfull, 5 loader after empty, 6 loader arrive, 7 epilogue after dfull
__device__ long long g_sb_trace[8][64];
__device__ unsigned long long g_sb_cta[3][1024];   // per CTA: globaltimer at start, after the loader's pdl_wait, at exit
__device__ __forceinline__ unsigned long long sb_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SB_CTA(ev) do { const int c_ = blockIdx.y * gridDim.x + blockIdx.x; if (c_ < 1024) g_sb_cta[ev][c_] = sb_gtime(); } while (0)
#define SB_TR(ev, l) do { if (blockIdx.x == 0 && blockIdx.y == 0 && (l) < 64) g_sb_trace[ev][l] = clock64(); } while (0)
#else
#define SB_TR(ev, l) do { } while (0)
#define SB_CTA(ev) do { } while (0)
#endif

#ifndef OWQ_SB_NST
#define OWQ_SB_NST 4
#endif
constexpr int NST = OWQ_SB_NST;
#ifndef OWQ_SB_SPIN
#define OWQ_SB_SPIN 0
#endif
// ring waits: parked try_wait (0) or polling test_wait (1)
__device__ __forceinline__ void sb_wait(uint64_t* b, uint32_t parity) {
  if (OWQ_SB_SPIN) mbar_wait_spin(b, parity);
  else mbar_wait(b, parity);
}
#ifndef OWQ_SB_SUB
#define OWQ_SB_SUB 1
#endif
// super-steps per stage: 1 measured faster than 2 (8 decode warps; both are
// bound by shared-memory traffic: A is written and read as 2 B per code,
// DESIGN.md §6.5)
constexpr int SUB = OWQ_SB_SUB;
constexpr uint32_t A_BYTES = 128 * 64 * 2;
constexpr uint32_t C_MAX = 128 * 8 * 4;
constexpr int NDB = 4;                  // D buffers (one per drain in flight)
// Per-row scales: D is still drained into fp32 registers every kDrainSS
// super-steps.  One TMEM accumulator over all of K = 12288 (one split) lost
// precision (B = 32 parity error 4.8e-3 > the 2e-3 bound): one fp32 TMEM
// accumulator over a chain of 768 MMAs.
constexpr int kDrainSS = 8;
// warps: 0-7 decode (4 per sub-step, thread = row), 8-11 epilogue, 12 x loader, 13 producer, 14 MMA
constexpr int kDec = 4 * SUB, kEpi0 = kDec, kLoad = kEpi0 + 4, kProd = kLoad + 1, kMma = kProd + 1;
constexpr int kThreads = (kMma + 1) * 32;

struct Params {
  const uint8_t* blob;
  const __half* x;      // [B][K]
  void* y;              // [B][M]
  float* part;          // [KS][B][Mp] fp32 partial rows (KS > 1)
  uint32_t* counters;   // [nrb], zero between calls
  Geo g;
  int32_t B, y_f32, KS, sps;   // splits, super-steps per split (a multiple of SUB)
  int32_t gss;          // super-steps per D drain: the scale group, or kDrainSS with per-row scales
  int32_t skip;         // experiment builds only (OWQ_SB_SKIP): 1 decode, 2 MMA, 4 x copies, 8 code copies,
                        // 16 MMA-side proxy fence, 32 commits -> plain arrives (with 2)
};

template <int NT>
__host__ __device__ constexpr uint32_t stage_bytes() { return SUB * (A_BYTES + NT * 128 + C_MAX); }

// two resident CTAs per SM (register cap 93: N = 32 no longer takes 125 registers
// and one CTA per SM, 78.9 -> see DESIGN.md §6.5)
#ifndef OWQ_SB_MINB
#define OWQ_SB_MINB 2
#endif
constexpr int kMaxOcc = 3;   // resident CTAs per SM the planner and workspace_bytes() allow
template <int BITS, int NT>
__global__ void __launch_bounds__(kThreads, OWQ_SB_MINB) owq_gemm_sb_kernel(const Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t STG = stage_bytes<NT>();
  const Geo& g = p.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, rb = blockIdx.y;
  const int ss0 = split * p.sps, ss1 = min(g.nss, ss0 + p.sps);
  const int nsteps = ss1 - ss0;                  // super-steps of this split
  const int n = (nsteps + SUB - 1) / SUB;        // stages
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + NST * STG);
  uint64_t* afull = full + NST;
  uint64_t* bfull = afull + NST;
  uint64_t* empty = bfull + NST;
  uint64_t* dfull = empty + NST;      // [NDB]
  uint64_t* dempty = dfull + NDB;     // [NDB]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + NDB);
  int* flag = reinterpret_cast<int*>(tslot + 1);
  auto A = [&](int s, int u) { return base + (size_t)s * STG + (size_t)u * A_BYTES; };
  auto Bt = [&](int s, int u) { return base + (size_t)s * STG + SUB * A_BYTES + (size_t)u * (NT * 128); };
  auto Cd = [&](int s) { return base + (size_t)s * STG + SUB * (A_BYTES + NT * 128); };
  const bool grouped = g.group != 0;   // per-group scales (else per row: one (s, z) per row)
  if (threadIdx.x == 0) SB_CTA(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&afull[s], kDec * 32 + 32);   // decode threads + the loader lanes' cp.async arrivals
      mbar_init(&bfull[s], 1);                 // (unused)
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < NDB; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kProd) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t ssb = (uint32_t)g.ss_bytes;
  // scale group of stage l (stages never straddle a group: gss is a multiple of SUB)
  auto grp = [&](int l) { return (ss0 + SUB * l) / p.gss; };   // D drain (= scale group when grouped)
  auto sgrp = [&](int l) { return grouped ? grp(l) : 0; };      // (s, z) block
  auto nsub = [&](int l) { return min(SUB, nsteps - SUB * l); };

  if (warp == kProd) {
    if (lane == 0) {
      pdl_launch_dependents();
      for (int l = 0; l < n; ++l) {
        const int s = l % NST;
        if (l >= NST) sb_wait(&empty[s], (uint32_t)((l / NST) - 1) & 1u);
        SB_TR(0, l);
        const uint32_t bytes = ssb * (uint32_t)nsub(l);   // consecutive super-steps are contiguous in the blob
        if (SB_SKIP(8)) {
          mbar_arrive(&full[s]);
          continue;
        }
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(Cd(s), p.blob + g.units_off + item_offset(g, rb, ss0 + SUB * l), bytes, &full[s]);
      }
    }
  } else if (warp == kMma) {
    constexpr uint32_t idesc = idesc_f16(128, NT);
    int gcount = 0;
    int gpos = 0;   // super-steps into the current drain group (splits start on group boundaries)
    for (int l = 0; l < n; ++l) {
      const int s = l % NST;
      const uint32_t ph = (uint32_t)(l / NST) & 1u;
      const bool first = gpos == 0;
      gpos += SUB;
      const bool last = l == n - 1 || gpos == p.gss;
      if (gpos == p.gss) gpos = 0;
      const int buf = gcount % NDB;
      // one lane waits (parked waiters on a barrier cost every phase change)
      if (lane == 0 && first && gcount >= NDB) sb_wait(&dempty[buf], (uint32_t)((gcount / NDB) - 1) & 1u);
      if (lane == 0) sb_wait(&afull[s], ph);   // A decoded and the x tile landed
      if (lane == 0) SB_TR(3, l);
      if (lane == 0) SB_TR(4, l);
      if (!SB_SKIP(16)) fence_proxy_async();   // the landed cp.async (generic-proxy) writes, before the MMA's async-proxy reads
      tc_fence_after();
      if (lane == 0) {
        const int nu = SB_SKIP(2) ? 0 : nsub(l);
        for (int u = 0; u < nu; ++u)
          tc_mma_f16_ss_k64<2 * 2048, 2 * NT * 16>(tmem + (uint32_t)(buf * NT), umma_desc(smem_u32(A(s, u)), 2048, 128),
                                                   umma_desc(smem_u32(Bt(s, u)), NT * 16, 128), idesc,
                                                   (first && u == 0) ? 0u : 1u);
        if (SB_SKIP(32)) {
          mbar_arrive(&empty[s]);
          if (last) mbar_arrive(&dfull[buf]);
        } else {
          tc_commit(&empty[s]);
          if (last) tc_commit(&dfull[buf]);
        }
      }
      __syncwarp();
      if (last) ++gcount;
    }
  } else if (warp < kDec) {
    // decode: warps 4u .. 4u+3 decode sub-step u of each stage, thread = row; A = (q - z_group) fp16
    const int u = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    constexpr int WPR = BITS == 3 ? 6 : 8;
    // the row's (scale, zero) words of the split's groups, loaded two groups
    // ahead (one load per group in the stage loop left every group start waiting
    // on a global load, ~9 % of the stall samples at g128)
    auto ldsz = [&](int gi) {
      return gi < g.G ? __ldg(reinterpret_cast<const uint32_t*>(p.blob + g.sz_off + ((int64_t)rb * g.G + gi) * kSZBlockBytes) + r)
                      : 0u;
    };
    const int gfirst = sgrp(0);
    uint32_t sz0 = ldsz(gfirst), sz1 = grouped ? ldsz(gfirst + 1) : 0u, sz2 = grouped ? ldsz(gfirst + 2) : 0u;
    uint32_t zzw = 0;
    int zg = -1;
    for (int l = 0; l < n; ++l) {
      const int s = l % NST;
      const int gi = sgrp(l);
      if (gi != zg) {
        if (zg >= 0) {   // next group: shift the prefetch window
          sz0 = sz1;
          sz1 = sz2;
          sz2 = ldsz(gi + 2);
        }
        const __half2 zz = __float2half2_rn(1024.f + __high2float(*reinterpret_cast<const __half2*>(&sz0)));
        zzw = *reinterpret_cast<const uint32_t*>(&zz);
        zg = gi;
      }
      if (lane == 0) sb_wait(&full[s], (uint32_t)(l / NST) & 1u);
      __syncwarp();
      if (threadIdx.x == 0) SB_TR(1, l);
      if (u < nsub(l) && !SB_SKIP(1)) {
        const uint8_t* rec = Cd(s) + (size_t)u * ssb;
        uint32_t w[8], o[16];
#pragma unroll
        for (int i = 0; i < WPR; ++i) w[i] = *reinterpret_cast<const uint32_t*>(rec + row_word_byte(BITS, r, i));
        pf::decode_row<BITS>(w, o);
        const uint32_t arow = smem_u32(A(s, u)) + (uint32_t)(r >> 3) * 128u + (uint32_t)(r & 7) * 16u;
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) {
          const uint32_t w0 = o[2 * kc], w1 = o[2 * kc + 1];
          const uint32_t h0 = pf::hsub2(pf::prmt(w0, 0x64646464u, 0x4140u), zzw);
          const uint32_t h1 = pf::hsub2(pf::prmt(w0, 0x64646464u, 0x4342u), zzw);
          const uint32_t h2 = pf::hsub2(pf::prmt(w1, 0x64646464u, 0x4140u), zzw);
          const uint32_t h3 = pf::hsub2(pf::prmt(w1, 0x64646464u, 0x4342u), zzw);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(arow + kc * 2048u), "r"(h0), "r"(h1), "r"(h2),
                       "r"(h3)
                       : "memory");
        }
        fence_proxy_async();
      }
      mbar_arrive(&afull[s]);
      if (threadIdx.x == 0) SB_TR(2, l);
    }
  } else if (warp == kLoad) {
    // x loader: NT tokens x (SUB x 64) columns per stage (zero rows past B), up to
    // NST stages in flight; each lane's copies arrive on afull when they land
    pdl_wait();
    if (lane == 0) SB_CTA(1);
    for (int l = 0; l < n; ++l) {
      const int s = l % NST;
      if (lane == 0 && l >= NST) sb_wait(&empty[s], (uint32_t)((l / NST) - 1) & 1u);
      __syncwarp();
      if (lane == 0) SB_TR(5, l);
#pragma unroll
      for (int e = lane; e < (SB_SKIP(4) ? 0 : SUB * NT * 8); e += 32) {
        const int u = e / (NT * 8), e2 = e % (NT * 8);
        const int t = e2 >> 3, kc = e2 & 7;
        const int64_t col = (int64_t)(ss0 + SUB * l + u) * 64 + kc * 8;
        const bool ok = t < p.B && col < g.K && SUB * l + u < nsteps;
        cp_async16(smem_u32(Bt(s, u)) + (uint32_t)kc * (NT * 16) + (uint32_t)(t >> 3) * 128u + (uint32_t)(t & 7) * 16u,
                   ok ? p.x + (int64_t)t * g.K + col : p.x, ok ? 16u : 0u);
      }
      cp_async_arrive_noinc(&afull[s]);
      if (lane == 0) SB_TR(6, l);
    }
    cp_async_wait_all();
  } else {
    // epilogue (warps 8-11): thread = row; tot[b] = sum over the split's groups of s_g D_g
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int64_t grow = (int64_t)rb * kRowBlock + r;
    float tot[NT];
#pragma unroll
    for (int b = 0; b < NT; ++b) tot[b] = 0.f;
    int gcount = 0;
    auto ldsz = [&](int gi) {
      return gi < g.G ? __ldg(reinterpret_cast<const uint32_t*>(p.blob + g.sz_off + ((int64_t)rb * g.G + gi) * kSZBlockBytes) + r)
                      : 0u;
    };
    uint32_t sznext = ldsz(sgrp(0));   // the next group's (scale, zero), one group ahead
    for (int l = 0; l < n; ++l) {
      const bool last = l == n - 1 || grp(l) != grp(l + 1);
      if (!last) continue;
      const int gi = sgrp(l);
      const int buf = gcount % NDB;
      const uint32_t szw = sznext;
      if (grouped) sznext = ldsz(gi + 1);
      const float sc = __low2float(*reinterpret_cast<const __half2*>(&szw));
      if (lane == 0) sb_wait(&dfull[buf], (uint32_t)(gcount / NDB) & 1u);
      __syncwarp();
      if (r == 0) SB_TR(7, l);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < NT / 16; ++c) {
        uint32_t d[16];
        tc_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * NT + c * 16), d);
#pragma unroll
        for (int j = 0; j < 16; ++j) tot[c * 16 + j] = fmaf(sc, __uint_as_float(d[j]), tot[c * 16 + j]);
      }
      tc_fence_before();
      mbar_arrive(&dempty[buf]);
      ++gcount;
    }
    pdl_wait();   // y, the workspace and x (weak fold) belong to earlier kernels until they complete
    if (split == 0 && g.k > 0) {   // fp16 weak columns x gathered fp16 x, added once
      const uint16_t* widx = reinterpret_cast<const uint16_t*>(p.blob + g.widx_off);
      const uint8_t* wrec = p.blob + g.units_off + (int64_t)rb * g.rb_bytes + (int64_t)g.nss * g.ss_bytes;
      for (int tt = 0; tt < g.k; ++tt) {
        const int ch = tt / kWeakChunk, c = tt % kWeakChunk;
        const __half wv = ch < g.nfull
                              ? *reinterpret_cast<const __half*>(wrec + (int64_t)ch * kWeakChunkBytes + (r * kWeakChunk + c) * 2)
                              : *reinterpret_cast<const __half*>(wrec + (int64_t)g.nfull * kWeakChunkBytes + (r * g.ktail + c) * 2);
        const float wf = __half2float(wv);
        const int j = __ldg(widx + tt);
#pragma unroll
        for (int b = 0; b < NT; ++b)
          if (b < p.B) tot[b] = fmaf(wf, __half2float(p.x[(int64_t)b * g.K + j]), tot[b]);
      }
    }
    if (p.KS == 1) {
      if (grow < g.M)
#pragma unroll
        for (int b = 0; b < NT; ++b)
          if (b < p.B) {
            if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = tot[b];
            else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(tot[b]);
          }
    } else {
      const int64_t Mp = (int64_t)g.nrb * kRowBlock;
#pragma unroll
      for (int b = 0; b < NT; ++b)
        if (b < p.B) __stcg(&p.part[((int64_t)split * p.B + b) * Mp + grow], tot[b]);
      named_sync(1, 128);
      if (r == 0) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.counters + rb) : "memory");
        const int lastc = old == (unsigned)(p.KS - 1);
        if (lastc) p.counters[rb] = 0u;
        *flag = lastc;
      }
      named_sync(1, 128);
      if (*flag && grow < g.M) {
        for (int b = 0; b < p.B; ++b) {
          float v = 0.f;
          for (int sp = 0; sp < p.KS; ++sp) v += __ldcg(&p.part[((int64_t)sp * p.B + b) * Mp + grow]);
          if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = v;
          else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(v);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProd) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
  if (threadIdx.x == 0) SB_CTA(2);
}

// Splits of K (in super-steps, on drain-group boundaries): the split length that
// minimises the makespan  waves x (split / K + c)  over `slots` resident CTAs,
// c = 0.05 being a CTA's fixed cost (prologue, pipeline fill, fixup) relative to
// a full-K CTA.  (One CTA per row-block left 52 of 148 SMs idle at 12288^2;
// round 2's first planner rounded up to 2 x SMs and left a short second wave.)
static void plan(const Geo& g, int slots, int& KS, int& sps, int& gss) {
  gss = g.group ? g.group / 64 : kDrainSS;
  const int unit = gss;
  const int units = (g.nss + unit - 1) / unit;
  double best = 1e30;
  KS = 1;
  sps = units * unit;
  for (int upc = units; upc >= 1; --upc) {
    const int ks = (units + upc - 1) / upc;
    if (ks > 64) break;
    const int64_t waves = ((int64_t)ks * g.nrb + slots - 1) / slots;
    const double cost = (double)waves * ((double)upc / units + 0.05);
    if (cost < best - 1e-9) {
      best = cost;
      KS = ks;
      sps = upc * unit;
    }
  }
  KS = (g.nss + sps - 1) / sps;
}

size_t workspace_bytes(const Geo& g, int B, int sms) {
  int KS, KS2, sps, gss;
  plan(g, sms, KS, sps, gss);       // 1 .. kMaxOcc resident CTAs per SM (launch_t)
  plan(g, 2 * sms, KS2, sps, gss);
  KS = std::max(KS, KS2);
  plan(g, kMaxOcc * sms, KS2, sps, gss);
  KS = std::max(KS, KS2);
  return (size_t)g.nrb * 4 + 256 + (KS > 1 ? (size_t)KS * B * g.nrb * kRowBlock * 4 : 0);
}

template <int BITS, int NT>
static owq_status launch_t(Params& p, int sms, cudaStream_t stream) {
  auto kern = owq_gemm_sb_kernel<BITS, NT>;
  const uint32_t smem = NST * stage_bytes<NT>() + 1024 + 512;
  int dev = 0;
  cudaGetDevice(&dev);
  static int occupancy[16] = {};   // resident CTAs per SM (0 = not configured yet)
  if (!occupancy[dev & 15]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return OWQ_ERR_CUDA;
    // without a preference the driver picks the smallest carveout that fits ONE
    // CTA (measured: 1 resident CTA per SM at 92 KB)
    if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
      return OWQ_ERR_CUDA;
    // Resident CTAs per SM from shared memory and registers: the occupancy API
    // reports 1 for any kernel that allocates TMEM (tools/occ_probe.cu), but two
    // 128-column allocations fit and two CTAs were measured resident at once
    // (tools/sb_trace.py: 288 CTAs started within 0.8 us on 148 SMs).
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return OWQ_ERR_CUDA;
    int smem_sm = 0, regs_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    int occ = std::min<int>(kMaxOcc, smem_sm / (int)(smem + 1024));
    while (occ > 1 && occ * fa.numRegs * kThreads > regs_sm) --occ;
    occupancy[dev & 15] = std::max(occ, 1);
#ifdef OWQ_EXPERIMENTS
    fprintf(stderr, "owq sb<%d,%d>: %d resident CTAs per SM (smem %u, threads %d, regs %d)\n", BITS, NT, occupancy[dev & 15],
            smem, kThreads, fa.numRegs);
#endif
  }
  int slots = occupancy[dev & 15] * sms;
#ifdef OWQ_EXPERIMENTS
  if (const char* v = getenv("OWQ_SB_SLOTS")) slots = atoi(v);
#endif
  plan(p.g, slots, p.KS, p.sps, p.gss);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((unsigned)p.KS, (unsigned)p.g.nrb);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "owq: launch of owq_gemm_sb_kernel failed: %s\n", cudaGetErrorString(e));
    return OWQ_ERR_CUDA;
  }
  return OWQ_OK;
}

owq_status launch(const Geo& g, const void* blob, const uint16_t* x, int B, void* y, int y_f32, void* ws,
                  size_t ws_bytes, int sms, cudaStream_t stream) {
  if (B < 1 || B > 32) return OWQ_ERR_UNSUPPORTED;
  if (g.group && (g.group % (64 * SUB))) return OWQ_ERR_UNSUPPORTED;   // stages never straddle a scale group
  if (ws_bytes < workspace_bytes(g, B, sms)) return OWQ_ERR_BUFFER_TOO_SMALL;
  Params p{};
  p.blob = (const uint8_t*)blob;
  p.x = (const __half*)x;
  p.y = y;
  p.counters = (uint32_t*)ws;
  p.part = (float*)((uint8_t*)ws + ((size_t)g.nrb * 4 + 255) / 256 * 256);
  p.g = g;
  p.B = B;
  p.y_f32 = y_f32 ? 1 : 0;
#ifdef OWQ_EXPERIMENTS
  if (const char* v = getenv("OWQ_SB_SKIP")) p.skip = atoi(v);
#endif
  if (g.bits == 3) return B <= 16 ? launch_t<3, 16>(p, sms, stream) : launch_t<3, 32>(p, sms, stream);
  return B <= 16 ? launch_t<4, 16>(p, sms, stream) : launch_t<4, 32>(p, sms, stream);
}

}  // namespace sb
}  // namespace pf
}  // namespace owq

#ifdef OWQ_EXPERIMENTS
extern "C" int owq_exp_sb_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, owq::pf::sb::g_sb_trace, sizeof(owq::pf::sb::g_sb_trace));
}
extern "C" int owq_exp_pf_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, owq::pf::g_pf_trace, sizeof(owq::pf::g_pf_trace));
}
extern "C" int owq_exp_pf_cta(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, owq::pf::g_pf_cta, sizeof(owq::pf::g_pf_cta));
}
extern "C" int owq_exp_sb_cta(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, owq::pf::sb::g_sb_cta, sizeof(owq::pf::sb::g_sb_cta));
}
#endif
