// owq_gemv_cc.cu -- the CUDA-core OWQ GEMV (blob layout version 4, owq_layout_cc.h):
// y = diag(s) (Q - z) x + W_weak x[idx], batch 1..4 per launch.
//
// Why CUDA cores at batch 1 (tools/cc_probe.cu on this B200):
// the product has 2 flops per 3-bit code; the tensor-core path pays for it with
// an x-digit pre-pass, TMEM traffic and a decode -> MMA -> epilogue handshake per
// stage.  Here a code costs one LOP3 (it stays in place as an fp32 subnormal,
// q 2^(p-149)) and half an FFMA2 against x' = x 2^(111-p): the product
// q x 2^-38 is exact, the sum is fp32.  The zero point is factored out per
// (row, scale group): s (sum q x - z sum x) (reading s19).
//
// Persistent CTAs, byte-balanced stream-K over "units" (an item = 128 rows x 32
// columns of codes; one weak unit per row-block).  Warp roles:
//   producer (1 warp, one lane): TMA bulk copies of stages (runs of <= 16 items
//       of one row-block, contiguous in the blob) into a shared-memory ring.
//       It never waits on earlier kernels (weights are constant), so under
//       programmatic dependent launch the ring fills while the previous kernel
//       drains.
//   compute (8 warps): warp w takes items 2w, 2w+1 of each stage; lane l owns
//       rows 4l..4l+3 of the row-block.  Per item: x of the item's 32 columns
//       (lane l loads column l, zeroed at weak columns, scaled by 2^(111-p)),
//       shared through a per-warp smem slot; 3-4 LDS.128 of codes; 34-35 LOP3/
//       PRMT and 16 FFMA2 per row.  Per (row, scale-group part): one flush
//       tot += s (acc 2^38 - z sum x).  At a row-block end the warps' partial
//       rows are summed in a fixed order, the fp16 weak columns are folded in
//       (fp16 x fp16 in fp32), and y is written -- directly, or through the
//       stream-K fixup: the CTA holding a row-block's LAST unit sums the pieces
//       of the lower-index CTAs (which it only waits for at its own end, and
//       which never wait on it: forward progress needs only in-order dispatch).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>

#include "owq.h"
#include "owq_layout_cc.h"

namespace owq {
namespace cc {

#ifndef OWQ_CC_NW
#define OWQ_CC_NW 8          // compute warps per CTA
#endif
#ifndef OWQ_CC_S
#define OWQ_CC_S 4           // items per compute warp per stage
#endif
#ifndef OWQ_CC_MINB
#define OWQ_CC_MINB 1        // CTAs per SM the kernel is built for (registers / shared memory)
#endif
constexpr int kMaxGrid = 1024;

// Compile-time pipeline shape of one (bits, batch-rows) instantiation.
template <int BITS, int NB>
struct Cfg {
  static constexpr int NW = OWQ_CC_NW;
  static constexpr int W = BITS == 3 ? 3 : 4;               // code words per row and item
  static constexpr uint32_t ITEM = (uint32_t)W * 512u;
  static constexpr int MINB = OWQ_CC_MINB;
  static constexpr uint32_t BUDGET = MINB == 1 ? 227u * 1024u : 113u * 1024u;
  // items per warp and stage: OWQ_CC_S at batch 1 (fewer with more batch rows:
  // registers), halved until the ring holds >= 3 stages
  static constexpr int S0 = NB == 1 ? OWQ_CC_S : NB == 2 ? 2 : 1;
  static constexpr int S = (uint32_t)NW * S0 * ITEM * 3u <= BUDGET - 40u * 1024u ? S0
                           : (uint32_t)NW * (S0 / 2 > 0 ? S0 / 2 : 1) * ITEM * 3u <= BUDGET - 40u * 1024u ? (S0 / 2 > 0 ? S0 / 2 : 1)
                           : 1;
  static constexpr int CAP = NW * S;                        // items per stage
  static constexpr uint32_t STAGE = (uint32_t)CAP * ITEM;
  static constexpr int THREADS = (NW + 1) * 32;
  // shared memory besides the ring: x' slots, row partials (2 buffers), the summer's row
  static constexpr uint32_t FIXED = (uint32_t)(NW * 2 * S * NB * 32 + 2 * NW * NB * 128 + NB * 128) * 4u + 32u * 8u;
  static constexpr int NST0 = (int)((BUDGET - FIXED - 1024u) / STAGE);
  static constexpr int NST = NST0 > 8 ? 8 : NST0;
  static constexpr uint32_t SMEM = (uint32_t)NST * STAGE + FIXED;
  static_assert(NST >= 2, "ring");
};

struct Params {
  const uint8_t* blob;
  const __half* x;        // [NB][xK] (this launch's batch rows)
  void* y;                // [NB][M]
  uint32_t* slots;        // [grid][NB][128] partial rows as ~bits (0 = not written)
  Geo g;
  int64_t xK;
  int32_t y_f32;
  int32_t gl;             // log2(group / 32); 30 for per-row scales
  int32_t grid;
  int32_t span[kMaxGrid + 1];   // first unit of each CTA
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra W_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* a, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// two exact products (subnormal code patterns x scaled activations) into a pair of fp32 sums
__device__ __forceinline__ void ffma2(float2& acc, uint32_t c0, uint32_t c1, float x0, float x1) {
  unsigned long long a = ((unsigned long long)c1 << 32) | c0;
  unsigned long long b = ((unsigned long long)__float_as_uint(x1) << 32) | __float_as_uint(x0);
  unsigned long long d = ((unsigned long long)__float_as_uint(acc.y) << 32) | __float_as_uint(acc.x);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
  acc.x = __uint_as_float((uint32_t)d);
  acc.y = __uint_as_float((uint32_t)(d >> 32));
}

// The 32 codes of one row's step, each isolated in place (owq_layout_cc.h).
template <int BITS>
__device__ __forceinline__ void extract(const uint32_t* w, uint32_t* c) {
  if (BITS == 3) {
    const uint32_t t = prmt(prmt(w[0], w[1], 0x0073u), w[2], 0x0710u);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      c[i] = w[0] & (7u << (3 * i));
      c[8 + i] = w[1] & (7u << (3 * i));
      c[16 + i] = w[2] & (7u << (3 * i));
      c[24 + i] = t & (7u << (3 * i));
    }
  } else {
    const uint32_t t1 = prmt(prmt(w[0], w[1], 0x0073u), w[2], 0x0710u);
    const uint32_t t2 = prmt(w[3], w[3], 0x0003u);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      c[i] = w[0] & (15u << (4 * i));
      c[6 + i] = w[1] & (15u << (4 * i));
      c[12 + i] = w[2] & (15u << (4 * i));
      c[18 + i] = w[3] & (15u << (4 * i));
      c[24 + i] = t1 & (15u << (4 * i));
    }
    c[30] = t2 & 15u;
    c[31] = t2 & 0xF0u;
  }
}

// Stage walk shared by the producer and the compute warps: row-blocks of the
// CTA's unit range, each cut into runs of <= CAP code items.
template <int CAP>
struct Walk {
  int64_t rb, rb_last, u0, u1;    // current row-block; CTA unit range [u0, u1)
  int64_t n_rb;                   // units per row-block
  int32_t nsteps;
  int32_t s0, s1;                 // code items of rb in this CTA: [s0, s1)
  int32_t cur;                    // next stage start
  __device__ __forceinline__ void rb_init() {
    const int64_t base = rb * n_rb;
    const int64_t a = u0 > base ? u0 - base : 0, b = u1 < base + n_rb ? u1 - base : n_rb;
    s0 = (int32_t)(a < nsteps ? a : nsteps);
    s1 = (int32_t)(b < nsteps ? b : nsteps);
    cur = s0;
  }
  __device__ __forceinline__ void init(const Geo& g, int64_t ua, int64_t ub) {
    n_rb = units_per_rb(g);
    nsteps = g.nsteps;
    u0 = ua; u1 = ub;
    rb = ua / n_rb;
    rb_last = (ub - 1) / n_rb;
    rb_init();
  }
  // next stage of the current row-block: its item count (0 = row-block done)
  __device__ __forceinline__ int next(int32_t& start) {
    if (cur >= s1) return 0;
    start = cur;
    const int n = s1 - cur < CAP ? s1 - cur : CAP;
    cur += n;
    return n;
  }
  __device__ __forceinline__ bool next_rb() {
    if (rb >= rb_last) return false;
    ++rb;
    rb_init();
    return true;
  }
  // next stage of the whole walk, across row-blocks (0 = done)
  __device__ __forceinline__ int next_any(int32_t& start) {
    for (;;) {
      const int n = next(start);
      if (n > 0) return n;
      if (!next_rb()) return 0;
    }
  }
};

// x of one stage's items for one warp, prefetched into registers.
template <int S, int NB>
struct XPre {
  uint32_t m[S];          // weak-column bitmask words
  __half v[S][NB];        // x[b][column 32 (st + w S + t) + lane]
};

#ifdef OWQ_EXPERIMENTS
// per CTA (globaltimer ns): start, x available (after griddepcontrol.wait), main
// loop done, exit (tools/cc_trace.py)
__device__ unsigned long long g_cc_cta[4][1024];
#define CC_STAMP(ev) do { if (threadIdx.x == 0 && blockIdx.x < 1024) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_cc_cta[ev][blockIdx.x] = t_; } } while (0)
#else
#define CC_STAMP(ev) do { } while (0)
#endif
template <int BITS, int NB>
__global__ void __launch_bounds__(Cfg<BITS, NB>::THREADS, Cfg<BITS, NB>::MINB) owq_gemv_cc_kernel(const Params p) {
  using C = Cfg<BITS, NB>;
  constexpr int NW = C::NW, S = C::S, CAP = C::CAP, W = C::W, NST = C::NST;
  constexpr uint32_t ITEM = C::ITEM, STAGE = C::STAGE;
#ifndef OWQ_CC_XREG
#define OWQ_CC_XREG 2
#endif
  constexpr bool XREG = NB <= OWQ_CC_XREG;   // all of x' in registers (else reloaded per row)
  extern __shared__ __align__(128) uint8_t smem[];
  const Geo& g = p.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* xs = reinterpret_cast<float*>(smem + (size_t)NST * STAGE);   // [NW][2][S][NB][32]
  float* red = xs + NW * 2 * S * NB * 32;                              // [2][NW][NB][128]
  float* own = red + 2 * NW * NB * 128;                                // (unused spare) [NB][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(own + NB * 128);
  uint64_t* empty = full + NST;

  const int cta = blockIdx.x;
  const int64_t u0 = p.span[cta], u1 = p.span[cta + 1];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  CC_STAMP(0);
  if (u1 <= u0) return;
  const uint32_t ring0 = smem_u32(smem);

  if (warp == NW) {
    // ===================================================== producer (one lane)
    if (lane == 0) {
      pdl_launch_dependents();
      const uint64_t pol = evict_first();
      Walk<CAP> wk;
      wk.init(g, u0, u1);
      const uint8_t* units = p.blob + g.units_off;
      int s = 0, k = 0;
      uint32_t ph = 0;
      int32_t st;
      int n;
      while ((n = wk.next_any(st)) > 0) {
        if (k >= NST) mbar_wait(&empty[s], ph ^ 1u);
        const uint32_t bytes = (uint32_t)n * ITEM;
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(ring0 + (uint32_t)s * STAGE, units + item_offset(g, wk.rb, st), bytes, &full[s], pol);
        ++k;
        if (++s == NST) { s = 0; ph ^= 1u; }
      }
    }
    return;
  }

  // ======================================================= compute warps
  const int w = warp;
  const float xsc = __uint_as_float((uint32_t)(238 - cc_pos(BITS, lane)) << 23);   // 2^(111 - p(lane))
  const uint32_t xs_w = smem_u32(xs + w * 2 * S * NB * 32);
  const uint32_t* wmask = reinterpret_cast<const uint32_t*>(p.blob + g.wmask_off);
  const int64_t n_rb = units_per_rb(g);
  const int gl = p.gl;
  const uint8_t* szbase = p.blob + g.sz_off;

  auto cta_of = [&](int64_t unit) {   // span[c] <= unit < span[c + 1]
    int lo = 0, hi = p.grid;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (p.span[mid] <= unit) lo = mid; else hi = mid;
    }
    return lo;
  };
  const int64_t rb_first = u0 / n_rb;
  const bool first_partial = u0 > rb_first * n_rb && u1 >= (rb_first + 1) * n_rb;   // summer of rb_first
  const int c_first = first_partial ? cta_of(rb_first * n_rb) : cta;

  pdl_wait();   // x, y and the workspace belong to earlier kernels until they complete
  CC_STAMP(1);

  float tot[NB][4];
  float2 acc[NB][4][2];     // two FFMA2 chains per row (even / odd column pairs)
  float sx[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    sx[b] = 0.f;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      tot[b][r] = 0.f;
      acc[b][r][0] = acc[b][r][1] = make_float2(0.f, 0.f);
    }
  }
  int open_g = -1;          // scale group with unflushed sums (-1 = none)
  int64_t open_rb = -1;

  auto flush = [&]() {
    if (open_g < 0) return;
    const uint4 szv = __ldg(reinterpret_cast<const uint4*>(szbase + (open_rb * g.G + open_g) * kSZBlockBytes) + lane);
    const uint32_t szw[4] = {szv.x, szv.y, szv.z, szv.w};
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float Sx = sx[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Sx += __shfl_xor_sync(0xffffffffu, Sx, o);
      sx[b] = 0.f;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const __half2 h = *reinterpret_cast<const __half2*>(&szw[r]);
        const float sc = __low2float(h), z = __high2float(h);
        const float a = ((acc[b][r][0].x + acc[b][r][0].y) + (acc[b][r][1].x + acc[b][r][1].y)) * 274877906944.0f;   // 2^38
        tot[b][r] = fmaf(sc, fmaf(-z, Sx, a), tot[b][r]);
        acc[b][r][0] = acc[b][r][1] = make_float2(0.f, 0.f);
      }
    }
    open_g = -1;
  };

  // one item: codes of rows 4l..4l+3 at smem `it`, x' at smem `xa`
  auto do_item = [&](uint32_t it, uint32_t xa, int64_t rb, int32_t step, const float* xf) {
    const int gi = step >> gl;
    if (gi != open_g || rb != open_rb) {
      flush();
      open_g = gi;
      open_rb = rb;
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) sx[b] += xf[b];   // sum of x over the group's columns (zero-point term)
    uint4 cw[W];
#pragma unroll
    for (int c = 0; c < W; ++c) cw[c] = lds128(it + (uint32_t)(c * 512 + lane * 16));
    float xr[XREG ? NB : 1][32];
    if (XREG) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = lds128f(xa + (uint32_t)(b * 32 + 4 * q) * 4u);
          xr[XREG ? b : 0][4 * q] = v.x; xr[XREG ? b : 0][4 * q + 1] = v.y;
          xr[XREG ? b : 0][4 * q + 2] = v.z; xr[XREG ? b : 0][4 * q + 3] = v.w;
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      uint32_t wr[W];
#pragma unroll
      for (int c = 0; c < W; ++c) wr[c] = r == 0 ? cw[c].x : r == 1 ? cw[c].y : r == 2 ? cw[c].z : cw[c].w;
      uint32_t cd[32];
      extract<BITS>(wr, cd);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (XREG) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            ffma2(acc[b][r][i & 1], cd[2 * i], cd[2 * i + 1], xr[XREG ? b : 0][2 * i], xr[XREG ? b : 0][2 * i + 1]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 v = lds128f(xa + (uint32_t)(b * 32 + 4 * q) * 4u);
            ffma2(acc[b][r][0], cd[4 * q], cd[4 * q + 1], v.x, v.y);
            ffma2(acc[b][r][1], cd[4 * q + 2], cd[4 * q + 3], v.z, v.w);
          }
        }
      }
    }
  };

  // column map (NEXT-4 variants): stored position -> original column, loaded
  // one stage before the x it selects (the x load depends on it)
  const uint16_t* colmap = g.mapped ? reinterpret_cast<const uint16_t*>(p.blob + g.colmap_off) : nullptr;
  auto load_j = [&](uint32_t* jq, int32_t st, int n) {
#pragma unroll
    for (int t = 0; t < S; ++t) {
      const int i = w * S + t;
      const int64_t pos = (int64_t)(st + i) * kStep + lane;
      jq[t] = (i < n && pos < g.Ks) ? (uint32_t)__ldg(colmap + pos) : 0u;
    }
  };
  auto load_x = [&](XPre<S, NB>& xp, int32_t st, int n, const uint32_t* jq) {
#pragma unroll
    for (int t = 0; t < S; ++t) {
      const int i = w * S + t;
      const int64_t pos = (int64_t)(st + i) * kStep + lane;   // stored position
      xp.m[t] = 0u;
#pragma unroll
      for (int b = 0; b < NB; ++b) xp.v[t][b] = __ushort_as_half((unsigned short)0);
      if (i < n) {
        xp.m[t] = __ldg(wmask + st + i);
        if (pos < g.Ks) {
          const int64_t col = colmap ? (int64_t)jq[t] : pos;
#pragma unroll
          for (int b = 0; b < NB; ++b) xp.v[t][b] = p.x[(int64_t)b * p.xK + col];
        }
      }
    }
  };

  Walk<CAP> wk, nx, nj;
  wk.init(g, u0, u1);
  nx = wk;                       // x: two stages ahead; column map: three
  XPre<S, NB> xa_, xb_;
  uint32_t jq[S];
  {
    int32_t st;
    int n = nx.next_any(st);
    if (colmap) load_j(jq, st, n);
    load_x(xa_, st, n, jq);
    n = nx.next_any(st);
    if (colmap) load_j(jq, st, n);
    load_x(xb_, st, n, jq);
    nj = nx;
    if (colmap) {
      n = nj.next_any(st);
      load_j(jq, st, n);
    }
  }

  int s = 0, par = 0, xpar = 0;
  uint32_t ph = 0;
  float keep[NB];            // this thread's row of the summer piece (rb_first)
#pragma unroll
  for (int b = 0; b < NB; ++b) keep[b] = 0.f;
  bool have_keep = false;
  uint32_t* slots = p.slots;

  for (;;) {
    int32_t st;
    int n;
    while ((n = wk.next(st)) > 0) {
      // x' of this stage's items -> the warp's smem slot (one conversion per column)
      const XPre<S, NB> xc = xa_;
      xa_ = xb_;
      {
        int32_t st2;
        const int n2 = nx.next_any(st2);
        load_x(xb_, st2, n2, jq);
        if (colmap) {
          const int n3 = nj.next_any(st2);
          load_j(jq, st2, n3);
        }
      }
      const uint32_t xslot = xs_w + (uint32_t)(xpar * S * NB * 32) * 4u;
      xpar ^= 1;
      float xf[S][NB];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const bool weak = (xc.m[t] >> lane) & 1u;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          xf[t][b] = weak ? 0.f : __half2float(xc.v[t][b]);
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot + (uint32_t)((t * NB + b) * 32 + lane) * 4u), "f"(xf[t][b] * xsc)
                       : "memory");
        }
      }
      __syncwarp();
      mbar_wait(&full[s], ph);
      const uint32_t sb = ring0 + (uint32_t)s * STAGE + (uint32_t)(w * S) * ITEM;
      if (n == CAP) {
#pragma unroll
        for (int t = 0; t < S; ++t)
          do_item(sb + (uint32_t)t * ITEM, xslot + (uint32_t)(t * NB * 32) * 4u, wk.rb, st + w * S + t, xf[t]);
      } else {
#pragma unroll 1
        for (int t = 0; t < S; ++t)
          if (w * S + t < n) do_item(sb + (uint32_t)t * ITEM, xslot + (uint32_t)(t * NB * 32) * 4u, wk.rb, st + w * S + t, xf[t]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == NST) { s = 0; ph ^= 1u; }
    }
    // -------------------------------------------------- row-block wk.rb done in this CTA
    flush();
    const int64_t rb = wk.rb;
    const int64_t base = rb * n_rb;
    const bool has_weak = g.k > 0 && u0 <= base + g.nsteps && u1 > base + g.nsteps;
    const bool last_piece = u1 >= base + n_rb;    // holds the row-block's last unit
    const bool whole = u0 <= base && last_piece;
    if (has_weak) {
      // fp16 weak columns x gathered fp16 activations, fp32: warp w folds
      // chunks w, w + NW, ... (8 columns each) into its partial rows
      const uint8_t* wb = p.blob + g.weak_off + rb * g.weak_rb_bytes;
      const uint16_t* widx = reinterpret_cast<const uint16_t*>(p.blob + g.widx_off);
      for (int ch = w; ch < g.kpad / kWeakChunk; ch += NW) {
        uint4 a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = __ldg(reinterpret_cast<const uint4*>(wb + (int64_t)ch * kWeakChunkBytes) + 4 * lane + r);
        const uint4 iv = __ldg(reinterpret_cast<const uint4*>(widx + ch * kWeakChunk));
        const uint32_t iw[4] = {iv.x, iv.y, iv.z, iv.w};
        float xw[8][NB];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = (int)((iw[c >> 1] >> (16 * (c & 1))) & 0xFFFFu);
          const bool ok = ch * kWeakChunk + c < g.k;   // padding columns hold v = 0 and idx = 0
#pragma unroll
          for (int b = 0; b < NB; ++b) xw[c][b] = ok ? __half2float(p.x[(int64_t)b * p.xK + j]) : 0.f;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t av[4] = {a[r].x, a[r].y, a[r].z, a[r].w};
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const __half2 h2 = *reinterpret_cast<const __half2*>(&av[c >> 1]);
            const float wv = (c & 1) ? __high2float(h2) : __low2float(h2);
#pragma unroll
            for (int b = 0; b < NB; ++b) tot[b][r] = fmaf(wv, xw[c][b], tot[b][r]);
          }
        }
      }
    }
    float* rd = red + par * NW * NB * 128;
#pragma unroll
    for (int b = 0; b < NB; ++b)
      *reinterpret_cast<float4*>(rd + (w * NB + b) * 128 + 4 * lane) = make_float4(tot[b][0], tot[b][1], tot[b][2], tot[b][3]);
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int r = 0; r < 4; ++r) tot[b][r] = 0.f;
    named_sync(1, NW * 32);
    const int row = threadIdx.x;                  // threads 0..127: one row each
    if (row < kRowBlock) {
      float v[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float a = 0.f;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) a += rd[(ww * NB + b) * 128 + row];
        v[b] = a;
      }
      const int64_t grow = rb * kRowBlock + row;
      if (whole) {
        if (grow < g.M)
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = v[b];
            else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(v[b]);
          }
      } else if (last_piece) {
        // summer of rb (= rb_first): add the lower-index pieces at the CTA's end
#pragma unroll
        for (int b = 0; b < NB; ++b) keep[b] = v[b];
        have_keep = true;
      } else {
        // non-summer piece (this CTA's last row-block): publish as ~bits
#pragma unroll
        for (int b = 0; b < NB; ++b) st_relaxed(slots + ((int64_t)cta * NB + b) * kRowBlock + row, ~__float_as_uint(v[b]));
      }
    }
    par ^= 1;
    if (!wk.next_rb()) break;
  }

  CC_STAMP(2);
  // ---------------------------------------------------- summer: wait for the lower pieces
  if (have_keep && threadIdx.x < kRowBlock) {
    const int row = threadIdx.x;
    float v[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) v[b] = 0.f;
    for (int c = c_first; c < cta; ++c) {
      uint32_t wv[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) wv[b] = ld_relaxed(slots + ((int64_t)c * NB + b) * kRowBlock + row);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        uint32_t* a = slots + ((int64_t)c * NB + b) * kRowBlock + row;
        while (wv[b] == 0u) {
          __nanosleep(64);
          wv[b] = ld_relaxed(a);
        }
        st_relaxed(a, 0u);
        v[b] += __uint_as_float(~wv[b]);
      }
    }
    const int64_t grow = rb_first * kRowBlock + row;
    if (grow < g.M)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const float o = v[b] + keep[b];
        if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = o;
        else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(o);
      }
  }
  CC_STAMP(3);
}

// Device inverse of layout 4 (test hook): one thread per (row, column).
__global__ void owq_unpack_codes_cc_kernel(const uint8_t* blob, Geo g, uint8_t* codes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)g.M * g.Ks) return;
  const int64_t row = i / g.Ks, col = i - row * g.Ks;
  const int64_t rb = row / kRowBlock, rr = row % kRowBlock, step = col / kStep, j = col % kStep;
  const uint8_t* it = blob + g.units_off + item_offset(g, rb, step);
  const int lane = (int)(rr >> 2), r = (int)(rr & 3);
  uint32_t c = 0;
  for (int bit = 0; bit < g.bits; ++bit) {
    int word, pos;
    cc_bit_loc(g.bits, (int)j, bit, word, pos);
    const uint32_t v = *reinterpret_cast<const uint32_t*>(it + (word * 32 + lane) * 16 + r * 4);
    c |= ((v >> pos) & 1u) << bit;
  }
  codes[i] = (uint8_t)c;
}

// ---------------------------------------------------------------- host side
static int sms_of_current_device() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) return 148;
  return sms;
}

int grid_for(const Geo& g, int grid_req) {
  const int64_t T = (int64_t)g.nrb * rb_bytes(g);
  const int64_t maxu = std::max<int64_t>(g.item_bytes, g.weak_rb_bytes);
  const int64_t cap = std::max<int64_t>(1, T / maxu);
  int64_t G = grid_req > 0 ? grid_req : (int64_t)sms_of_current_device() * OWQ_CC_MINB;
  G = std::min<int64_t>(G, cap);
  return (int)std::min<int64_t>(G, kMaxGrid);
}

size_t workspace_bytes(int grid, int nb) { return (size_t)grid * nb * kRowBlock * 4; }

template <int BITS, int NB>
static owq_status launch_t(Params& p, cudaStream_t stream) {
  using C = Cfg<BITS, NB>;
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = owq_gemv_cc_kernel<BITS, NB>;
  static bool configured[16] = {};
  if (!configured[dev & 15]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
      return OWQ_ERR_CUDA;
    configured[dev & 15] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
#ifdef OWQ_EXPERIMENTS
  if (const char* v = getenv("OWQ_CC_PDL")) attr[0].val.programmaticStreamSerializationAllowed = atoi(v) ? 1 : 0;
#endif
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "owq: launch of owq_gemv_cc_kernel<%d,%d> (grid %d, smem %u) failed: %s\n", BITS, NB, p.grid,
            C::SMEM, cudaGetErrorString(e));
    return OWQ_ERR_CUDA;
  }
  return OWQ_OK;
}

// y = W_hat x for B rows (in launches of <= 4 rows), blob layout 4.
owq_status gemm(const Geo& g, const void* blob, const uint16_t* x, int B, void* y, int y_f32, void* ws, size_t ws_bytes,
                int grid_req, cudaStream_t stream) {
  const int grid = grid_for(g, grid_req);
  if (ws_bytes < workspace_bytes(grid, std::min(B, 4))) return OWQ_ERR_BUFFER_TOO_SMALL;
  // stream-K span table of this (geometry, grid), cached per host thread
  struct SpanCache { int64_t key[3]; int32_t span[kMaxGrid + 1]; };
  static thread_local SpanCache cache[8];
  static thread_local int cache_n = 0, cache_next = 0;
  const int64_t key[3] = {((int64_t)g.nrb << 32) | g.nsteps, ((int64_t)g.kpad << 32) | g.W, grid};   // nsteps covers Ks
  static thread_local Params p;   // large (span table); filled per call
  int hit = -1;
  for (int i = 0; i < cache_n && hit < 0; ++i)
    if (cache[i].key[0] == key[0] && cache[i].key[1] == key[1] && cache[i].key[2] == key[2]) hit = i;
  if (hit < 0) {
    hit = cache_next;
    cache_next = (cache_next + 1) % 8;
    if (cache_n < 8) ++cache_n;
    const int64_t T = (int64_t)g.nrb * rb_bytes(g);
    for (int c = 0; c <= grid; ++c)
      cache[hit].span[c] = (int32_t)first_unit_at(g, cdiv((int64_t)c * T, grid));
    double a = 0.0;   // span skew toward early CTAs (owq_gemv.cu); experiments only so far
#ifdef OWQ_EXPERIMENTS
    if (const char* v = getenv("OWQ_CC_SKEW")) a = atoi(v) / 100.0;
#endif
    if (a > 0.0 && cache[hit].span[grid] >= 8 * (int64_t)grid) {
      int32_t* sp = cache[hit].span;
      for (int c = 1; c < grid; ++c) {
        const double xx = (double)c / grid, F = xx + 0.5 * a * (xx - xx * xx);
        sp[c] = (int32_t)first_unit_at(g, (int64_t)std::ceil((double)T * F));
      }
      for (int c = 1; c < grid; ++c) sp[c] = std::max(sp[c], sp[c - 1] + 1);
      for (int c = grid - 1; c >= 1; --c) sp[c] = std::min(sp[c], sp[c + 1] - 1);
    }
    for (int i = 0; i < 3; ++i) cache[hit].key[i] = key[i];
  }
  std::copy(cache[hit].span, cache[hit].span + grid + 1, p.span);
  p.blob = (const uint8_t*)blob;
  p.slots = (uint32_t*)ws;
  p.g = g;
  p.xK = g.K;
  p.y_f32 = y_f32 ? 1 : 0;
  p.grid = grid;
  p.gl = 30;
  if (g.group) { int l = 0; while ((kStep << l) < g.group) ++l; p.gl = l; }
  for (int b0 = 0; b0 < B; b0 += 4) {
    const int nb = std::min(4, B - b0);
    p.x = reinterpret_cast<const __half*>(x) + (int64_t)b0 * g.K;
    p.y = (uint8_t*)y + (size_t)b0 * g.M * (y_f32 ? 4 : 2);
    owq_status st;
    if (g.bits == 3) {
      st = nb == 1 ? launch_t<3, 1>(p, stream) : nb == 2 ? launch_t<3, 2>(p, stream)
         : nb == 3 ? launch_t<3, 3>(p, stream) : launch_t<3, 4>(p, stream);
    } else {
      st = nb == 1 ? launch_t<4, 1>(p, stream) : nb == 2 ? launch_t<4, 2>(p, stream)
         : nb == 3 ? launch_t<4, 3>(p, stream) : launch_t<4, 4>(p, stream);
    }
    if (st != OWQ_OK) return st;
  }
  return OWQ_OK;
}

owq_status unpack(const Geo& g, const void* blob, uint8_t* codes, cudaStream_t stream) {
  const int64_t n = (int64_t)g.M * g.Ks;
  owq_unpack_codes_cc_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>((const uint8_t*)blob, g, codes);
  return cudaGetLastError() == cudaSuccess ? OWQ_OK : OWQ_ERR_CUDA;
}

}  // namespace cc
}  // namespace owq

#ifdef OWQ_EXPERIMENTS
extern "C" int owq_exp_cc_cta(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, owq::cc::g_cc_cta, sizeof(owq::cc::g_cc_cta));
}
#endif
