// owq_gemv.cu -- sm_100a kernels of the OWQ hot path (arXiv 2306.02272, P:114,
// P:276): y = diag(s) (Q - z) x + W_weak x[idx] with Q the zero-filled b-bit
// code matrix, one fused launch (+ one tiny x-digit pass), batch 1..16.
//
// Arithmetic (exact up to the final fp32 scaling): the codes q are the u8 A
// operand of tcgen05.mma kind::i8 as they are (no dequantisation);
// x is split into 6 balanced int8 digits, x * 2^24 = sum_i d_i 256^i, which is
// exact for every finite fp16 (its ulp is >= 2^-24 and |x| < 2^16), so
//   sum_k q_k x_k = 2^-24 sum_i 256^i D_i,   D_i = sum_k q_k d_ik  (int32, exact)
// and the zero point comes in through S = sum_k x_k 2^24 (int64, exact):
//   y = s * 2^-24 * (sum_i 256^i D_i - z * S)   per row and scale group.
//
// Persistent CTA per SM, byte-balanced stream-K over "items" (a super-step =
// 128 rows x 64 columns of codes, or a chunk of 8 weak columns).  Warp roles:
//   producer (1 warp)   : one lane streams stages (runs of items + the digit
//                         tiles and digit sums of their columns + scale/zero
//                         blocks) HBM/L2 -> a shared-memory ring with
//                         cp.async.bulk (TMA) and mbarriers.
//   decode (DWG x 4)    : one thread per output row: the row's 64 codes ->
//                         16 words of 4 code bytes (LOP3 / SHF only, see
//                         owq_layout.h), written to a TMEM slot with tcgen05.st.
//   MMA (1 warp per WG) : one lane issues 2 tcgen05.mma kind::i8 M=128 N=NN K=32
//                         per item (A = codes from TMEM, B = x digits from shared
//                         memory, D s32 in TMEM; one D per warpgroup and scale
//                         group, ping-pong) and tcgen05.commit -> mbarriers.
//   epilogue (4 warps)  : reads D (tcgen05.ld), combines the digits and the zero
//                         point exactly, applies the fp32 scale of the row/group,
//                         adds the fp16 weak columns x gathered x[idx] on CUDA
//                         cores (the paper's separate dense fp16 GEMV, P:276,
//                         folded in), and writes y -- directly, or through the
//                         stream-K fixup (last-arriving CTA sums the pieces in a
//                         fixed order: deterministic).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "owq.h"
#include "owq_layout.h"
#include "owq_layout_cc.h"

namespace owq {
namespace cc {   // owq_gemv_cc.cu
owq_status gemm(const Geo& g, const void* blob, const uint16_t* x, int B, void* y, int y_f32, void* ws, size_t ws_bytes,
                int grid_req, cudaStream_t stream);
owq_status unpack(const Geo& g, const void* blob, uint8_t* codes, cudaStream_t stream);
int grid_for(const Geo& g, int grid_req);
size_t workspace_bytes(int grid, int nb);
}  // namespace cc
namespace pf {   // owq_prefill.cu
owq_status launch(const Geo& g, const void* blob, const uint16_t* x, int B, void* y, int y_f32, void* ws,
                  size_t ws_bytes, cudaStream_t stream);
size_t workspace_bytes(const Geo& g, int B);
namespace sb {
owq_status launch(const Geo& g, const void* blob, const uint16_t* x, int B, void* y, int y_f32, void* ws,
                  size_t ws_bytes, int sms, cudaStream_t stream);
size_t workspace_bytes(const Geo& g, int B, int sms);
}  // namespace sb
}  // namespace pf
}  // namespace owq

namespace owq {

// Experiment hooks (environment knobs, per-CTA timestamp traces) exist only in
// builds with -DOWQ_EXPERIMENTS (tools/ab_build.sh); the product library ignores
// the environment and carries no trace code.
#ifdef OWQ_EXPERIMENTS
constexpr bool kTrace = true;
static int knob(const char* name, int def) {
  const char* v = getenv(name);
  return v ? atoi(v) : def;
}
#define OWQ_CLK() clock64()
#else
constexpr bool kTrace = false;
static inline int knob(const char*, int def) { return def; }
#define OWQ_CLK() 0ll
#endif

constexpr int kDigits = 6;          // int8 digits per x value (base 256, balanced)

// MMA N (digit rows of B) for a batch: 6 * B padded to a valid tcgen05 N
static inline int mma_n_for(int B) {
  static const int min_n = knob("OWQ_MINN", 8);
  const int r = std::max(kDigits * B, min_n);
  return r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : 96;
}
static inline int batch_pad(int B) { return (B + 1) & ~1; }   // digit-sum rows (16-byte aligned runs)

constexpr int kMaxGrid = 512;       // CTAs per launch (the span table rides in the kernel parameters)

struct Params {
  const uint8_t* blob;
  const __half* x;
  void* y;
  uint32_t* counters;
  uint32_t* slots;        // co-resident fixup: [cta][B][128] partial rows as ~bits (0 = not written)
  float* partial;
  const uint8_t* tiles;   // x digits, [nss][NN rows x 64 columns] in UMMA K-major core matrices
  const long long* sums;  // [nss][Bp] sum over the super-step of x * 2^24
  Geo g;
  int32_t B, Bp;
  int32_t y_f32;
  int32_t nst;            // pipeline stages
  int32_t cap;            // items per stage
  int32_t code_bytes;     // stage region for codes / weak chunks
  int32_t tile_off;       // digit tiles inside a stage
  int32_t sum_off;        // per-item digit sums inside a stage (in-kernel digit mode)
  int32_t x_off;          // end of the staged digit sums (grouped per-stage mode)
  int32_t sz_off;         // scale/zero blocks of the stage's groups (grouped per-stage mode)
  int32_t gstage;         // grouped per-stage mode: the epilogue consumes the ring (sums + s/z staged)
  int32_t stage_bytes;
  int64_t xK;             // row stride of x in elements
  int32_t group_log2;     // log2(group_size / 64)
  int32_t span[kMaxGrid + 1];  // first item of each CTA (stream-K split, host-computed)
  int32_t coresident;          // grid <= SM count: fixed summer per row-block (see the fixup)
  // per CTA: the CTAs holding the first / last item of the row-block of its first
  // item (bits 0-15 / 16-31) and of its last item (bits 32-47 / 48-63)
  uint64_t fix[kMaxGrid];
  unsigned long long* trace;   // experiments only (OWQ_TRACE)
  int32_t exp;                 // experiments only (OWQ_EXP): 3 = skip the TMEM stores
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* a, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// Off-critical-path wait: the thread may be suspended (time hint) instead of
// spinning, so long waits do not take issue slots from the decode/MMA warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 0x989680;\n\t"
      "@!P bra WAITS_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch (the kernels are launched with programmatic
// stream serialization): wait = all prerequisite grids completed and their
// memory visible; launch_dependents = the next kernel in the stream may start.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// tcgen05 (5th-gen tensor core + TMEM)
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
// Warp-uniform forms: the whole warp executes them, one elected lane issues.
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_elect(uint32_t d_t, uint32_t a_t, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_t),
      "r"(a_t), "l"(b_desc), "r"(idesc), "r"(acc));
}
// All 2*IPW MMAs of a full warpgroup share of a stage under ONE elect: item t,
// half j reads TMEM A columns a0 + 16t + 8j and the digit tile at
// b0 + t*TILE + j*2*LBO bytes (descriptor start field = address >> 4).
template <int IPW, uint32_t TILE, uint32_t LBO>
__device__ __forceinline__ void tc_mma_i8_stage(uint32_t d_t, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc) {
#define OWQ_MMA_T(t)                                                                              \
  "add.u32 a, %1, " #t "*16;\n\t"                                                                  \
  "add.u64 b, %2, " #t "*(%5/16);\n\t"                                                             \
  "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a], b, %3, p;\n\t"                                  \
  "setp.eq.u32 p, 0, 0;\n\t"                                                                      \
  "add.u32 a, a, 8;\n\t"                                                                           \
  "add.u64 b, b, %6/16;\n\t"                                                                       \
  "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a], b, %3, p;\n\t"
  static_assert(IPW >= 1 && IPW <= 7, "IPW");
  if (IPW == 1)
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t" OWQ_MMA_T(0) "}" ::"r"(d_t), "r"(a0), "l"(b0), "r"(idesc), "r"(acc),
                 "n"(TILE), "n"(2 * LBO));
  else if (IPW == 2)
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t" OWQ_MMA_T(0) OWQ_MMA_T(1) "}" ::"r"(d_t), "r"(a0), "l"(b0), "r"(idesc),
                 "r"(acc), "n"(TILE), "n"(2 * LBO));
  else if (IPW == 3)
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t" OWQ_MMA_T(0) OWQ_MMA_T(1) OWQ_MMA_T(2) "}" ::"r"(d_t), "r"(a0), "l"(b0),
                 "r"(idesc), "r"(acc), "n"(TILE), "n"(2 * LBO));
  else if (IPW == 4)
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t" OWQ_MMA_T(0) OWQ_MMA_T(1) OWQ_MMA_T(2) OWQ_MMA_T(3) "}" ::"r"(d_t),
                 "r"(a0), "l"(b0), "r"(idesc), "r"(acc), "n"(TILE), "n"(2 * LBO));
  else if (IPW == 5)
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t" OWQ_MMA_T(0) OWQ_MMA_T(1) OWQ_MMA_T(2) OWQ_MMA_T(3) OWQ_MMA_T(4) "}"
                 ::"r"(d_t), "r"(a0), "l"(b0), "r"(idesc), "r"(acc), "n"(TILE), "n"(2 * LBO));
  else if (IPW == 6)
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t" OWQ_MMA_T(0) OWQ_MMA_T(1) OWQ_MMA_T(2) OWQ_MMA_T(3) OWQ_MMA_T(4)
                 OWQ_MMA_T(5) "}" ::"r"(d_t), "r"(a0), "l"(b0), "r"(idesc), "r"(acc), "n"(TILE), "n"(2 * LBO));
  else
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t" OWQ_MMA_T(0) OWQ_MMA_T(1) OWQ_MMA_T(2) OWQ_MMA_T(3) OWQ_MMA_T(4)
                 OWQ_MMA_T(5) OWQ_MMA_T(6) "}" ::"r"(d_t), "r"(a0), "l"(b0), "r"(idesc), "r"(acc), "n"(TILE), "n"(2 * LBO));
#undef OWQ_MMA_T
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d_t, uint32_t a_t, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_t),
      "r"(a_t), "l"(b_desc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t* d) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
        "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_ld16_nowait(uint32_t taddr, uint32_t* d) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
        "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
      : "r"(taddr)
      : "memory");
}
// UMMA shared-memory descriptor, K-major, no swizzle (SM100 version = 1)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// instruction descriptor, kind::i8: D s32, A u8 (codes), B s8 (x digits), K-major, M = 128
template <int NN>
__host__ __device__ constexpr uint32_t idesc_i8() {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(kRowBlock >> 4) << 24);
}

// Codes of one row's super-step -> 16 words, word c = codes of columns 4c..4c+3
// as bytes (the bit map of owq_layout.h::code_bit_loc).  The ALU pipe (LOP3,
// SHF: half rate) is this kernel's binding resource, so the right shifts run on
// the otherwise idle FMA pipe as IMAD.HI: w >> k = umulhi(w, 2^(32-k)), with
// the multipliers held in registers (opaque to the compiler, which would turn a
// literal power of two back into SHF).
struct Shifts { uint32_t m3, m4, m5, m6; };
__device__ __forceinline__ Shifts make_shifts() {
  Shifts h;
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m3) : "n"(1u << 29));
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m4) : "n"(1u << 28));
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m5) : "n"(1u << 27));
  asm volatile("mov.b32 %0, %1;" : "=r"(h.m6) : "n"(1u << 26));
  return h;
}
template <int BITS>
__device__ __forceinline__ void decode_row(const uint32_t* w, uint32_t* o, const Shifts& h) {
  if (BITS == 4) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i] = w[i] & 0x0F0F0F0Fu;
      o[8 + i] = __umulhi(w[i], h.m4) & 0x0F0F0F0Fu;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      o[i] = w[i] & 0x07070707u;
      o[6 + i] = __umulhi(w[i], h.m3) & 0x07070707u;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      o[12 + r] = (__umulhi(w[r], h.m6) & 0x03030303u) |
                  (__umulhi(w[4 + (r >> 1)], (r & 1) ? h.m5 : h.m4) & 0x04040404u);
  }
}

// ---- x -> int8 digits (one CTA per super-step, one thread per (batch row, column))
// x * 2^24 = sum_{i<6} d_i 256^i with d_i in [-128, 127] (balanced base 256).
// tiles: [nss][NN*64] bytes; byte ((kc * NN/8 + nb) * 8 + r) * 16 + kk holds digit
// row n = 8 nb + r (= 6 b + i; rows >= 6 B are zero), column k = 16 kc + kk of the
// super-step.  sums: [nss][Bp] = sum over the super-step's columns of x * 2^24.
__device__ __forceinline__ long long x_fixed(__half h) { return (long long)(__half2float(h) * 16777216.0f); }
// The pass also zeroes the GEMV's stream-K counters when the GEMV grid is larger
// than the SM count (`nzero` 16-byte words at `zero`; a workspace shared by calls
// of other shapes may hold their data there).  CTAs past nss only zero.  (One
// CTA per super-step: a grid of two CTAs per SM looping over super-steps, to fit
// next to the running GEMV in one wave, measured slower.)
__global__ void owq_x_digits_kernel(const __half* __restrict__ x, int64_t xK, int B, int Bp, int K, int NN,
                                    uint8_t* __restrict__ tiles, long long* __restrict__ sums, int nss,
                                    uint4* __restrict__ zero, int64_t nzero) {
  __shared__ long long part[2 * OWQ_MAX_BATCH];
  // Let the GEMV start (prologue, weight prefetch, decode) as soon as SMs free up,
  // even before the previous GEMV has finished; everything it reads that depends on
  // earlier kernels (x, digit tiles / sums, workspace) is behind its own pdl_wait().
  pdl_launch_dependents();
  pdl_wait();                  // x and the workspace belong to earlier kernels until they complete
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nzero; i += (int64_t)gridDim.x * blockDim.x)
    zero[i] = make_uint4(0, 0, 0, 0);
  const int ss = blockIdx.x;
  if (ss >= nss) return;
  const int b = threadIdx.x >> 6, k = threadIdx.x & 63;   // blockDim = 64 * Bp
  const int nbk = NN / 8;
  const int64_t col = (int64_t)ss * kSuperStep + k;
  long long X = (b < B && col < K) ? x_fixed(x[(int64_t)b * xK + col]) : 0;
  uint8_t* tile = tiles + (int64_t)ss * NN * 64 + (k >> 4) * nbk * 128 + (k & 15);
  if (b < B) {
    long long t = X;
#pragma unroll
    for (int i = 0; i < kDigits; ++i) {
      const int d = (int)(signed char)(t & 0xFF);
      t = (t - d) >> 8;
      const int n = kDigits * b + i;
      tile[(n >> 3) * 128 + (n & 7) * 16] = (uint8_t)d;
    }
  }
  if (b == 0)   // zero the padding rows 6B .. NN-1 of this column
    for (int n = kDigits * B; n < NN; ++n) tile[(n >> 3) * 128 + (n & 7) * 16] = 0;
  long long v = X;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (k == 0) sums[(int64_t)ss * Bp + b] = part[2 * b] + part[2 * b + 1];
}

// group of code item li (row-block relative super-step index)
__device__ __forceinline__ int group_of(const Params& p, int li) { return p.g.group ? (li >> p.group_log2) : 0; }

// Per (MMA-N class, decode warpgroups): items per warpgroup per stage, largest
// batch.  Each warpgroup owns two TMEM A buffers (ping-pong) of kIPW items and
// two D accumulators of NN columns; kIPW is what fits in the 512 TMEM columns.
template <int BITS, int NN, int DWG_, bool GRP = false>
struct Cfg {
  static constexpr int DWG = DWG_;
  // MMA issuers per decode warpgroup: with 2, issuer i owns A buffer i (stages
  // alternate), so consecutive stages' MMAs issue concurrently (own D each).
  // Implemented, but measured slower at batch 1 (the decode becomes the limit and
  // the extra MMA concurrency adds TMEM contention): 1 everywhere.
  static constexpr int ISS = 1;
  // (In-kernel digit mode -- decode warps turning the stage's raw x into digit
  // tiles instead of the pre-pass -- was measured slower on B200, 12288^2 B=1:
  // 28.2 us vs 24.0 us, and removed.)
  static constexpr int kIPW0 = (512 - 2 * ISS * DWG * NN) / (2 * DWG * 16);
  // 7 items per warpgroup at batch 1 (measured -8 % vs 6); grouped-scale kernels
  // keep 6 so the per-stage D blocks (kGP) fit next to the A buffers
  static constexpr int kIPWMax = GRP ? 6 : 7;
  static constexpr int kIPW = kIPW0 > kIPWMax ? kIPWMax : kIPW0;
  static constexpr int kMaxB = NN == 8 ? 1 : NN == 16 ? 2 : NN == 32 ? 5 : NN == 64 ? 10 : 16;
  static constexpr int kDecodeWarps = 4 * DWG;            // DWG decode warpgroups
  static constexpr int kEpiWarp0 = kDecodeWarps;          // 4 epilogue warps (warp % 4 = TMEM lane quarter)
  static constexpr int kMmaWarp0 = kEpiWarp0 + 4;         // ISS MMA-issuer warps per warpgroup
  static constexpr int kProdWarp = kMmaWarp0 + DWG * ISS;
  // 17 warps would put 5 on one SMSP with the 120 registers __launch_bounds__ allows
  // -> launch failure; pad that case to 20 (96 registers)
  static constexpr int kWarps = ISS == 2 ? (kProdWarp + 1 + 3) / 4 * 4 : kProdWarp + 1;
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kTmemCols = 512;
  static constexpr int kACols = kSuperStep / 4;           // 16 TMEM columns (4 code bytes each) per item
  static constexpr int kABuf = kIPW * kACols;            // TMEM columns per A buffer
  static constexpr int kDCol0 = DWG * 2 * kABuf;          // A: [DWG][2] buffers, then D: [DWG*ISS][2][kGP] x NN columns
  // Grouped scales (g > 0) at batch 1: per-stage D with one block per scale-group
  // piece of a warpgroup's share (<= 4 pieces for g = 128 and 6 items), when TMEM fits.
  static constexpr int kGP = (GRP && NN == 8 && ISS == 1 && kDCol0 + DWG * 2 * 4 * NN <= kTmemCols) ? 4 : 1;
  static_assert(kDCol0 + DWG * ISS * 2 * kGP * NN <= kTmemCols, "TMEM budget");
  static_assert(kMaxB * kDigits <= NN, "digit rows");
  // per stage: decode warps arrive, each MMA warp commits (B is read from the stage)
  static constexpr int kEmptyCount = kDecodeWarps + DWG;
};

// Stage descriptor, written by the producer into shared memory before it
// arms the stage's full barrier (consumers read it after the wait: the
// mbarrier arrive/wait pair orders it).  n == 0 terminates the consumers.
struct StageDesc {
  int32_t rb;        // row-block
  int16_t li;        // first item (row-block relative)
  uint8_t n;         // items
  uint8_t flags;     // kRbEnd: last stage of this row-block in the CTA;
                     // kGroupCont: the stage's last scale group continues in the next stage
};
constexpr uint8_t kRbEnd = 1, kGroupCont = 2;

// Segments of a code stage: maximal runs of items of one scale group.  For
// per-row scales a stage is one segment.  `ends` = the segment's group has no
// further item in this CTA's sequence.
struct Seg {
  int pa, pb, gi;
  bool ends;
};
__device__ __forceinline__ Seg segment(const Params& p, int pa, const StageDesc& d) {
  Seg sg;
  sg.pa = pa;
  sg.gi = group_of(p, d.li + pa);
  if (p.g.group) {
    const int gend = ((sg.gi + 1) << p.group_log2) - d.li - 1;   // last stage position of this group
    sg.pb = gend < d.n - 1 ? gend : d.n - 1;
  } else {
    sg.pb = d.n - 1;
  }
  sg.ends = sg.pb + 1 < d.n || !(d.flags & kGroupCont);
  return sg;
}
// contiguous share of a stage's n items owned by warpgroup w: [lo, hi)
template <int DWG>
__device__ __forceinline__ void share(int n, int w, int& lo, int& hi) {
  const int per = (n + DWG - 1) / DWG;
  lo = w * per;
  hi = lo + per < n ? lo + per : n;
  if (lo > n) lo = n;
}
__device__ __forceinline__ StageDesc load_desc(const StageDesc* d) {
  const uint2 v = lds64(smem_addr(d));
  StageDesc r;
  r.rb = (int32_t)v.x;
  r.li = (int16_t)(v.y & 0xFFFF);
  r.n = (uint8_t)((v.y >> 16) & 0xFF);
  r.flags = (uint8_t)(v.y >> 24);
  return r;
}

template <int BITS, int NN, int DWG_, bool GRP>
__global__ void __launch_bounds__(Cfg<BITS, NN, DWG_, GRP>::kThreads, 1) owq_gemv_kernel(const Params p) {
  using C = Cfg<BITS, NN, DWG_, GRP>;
  constexpr int DWG = C::DWG, MAXB = C::kMaxB;
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geo& g = p.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NST = p.nst;
  uint8_t* ring = smem;
  __half* xw = reinterpret_cast<__half*>(smem + (size_t)NST * p.stage_bytes);   // [B][kpad] x at the weak columns
  long long* red = reinterpret_cast<long long*>(xw + (((size_t)p.B * g.kpad + 7) & ~(size_t)7));   // [2][4][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * 4 * OWQ_MAX_BATCH);
  uint64_t* full = bars;
  uint64_t* empty = full + NST;
  uint64_t* afull = empty + NST;       // [DWG][2]  A buffer written (4 warps)
  uint64_t* aempty = afull + DWG * 2;  // [DWG][2]  MMA done reading it
  constexpr int NDQ = DWG * C::ISS;    // D accumulator owners (warpgroup, issuer)
  uint64_t* dfull = aempty + DWG * 2;  // [NDQ][2]  group accumulator complete
  uint64_t* dempty = dfull + 2 * NDQ;  // [NDQ][2]  epilogue drained it
  uint64_t* tready = dempty + 2 * NDQ;  // [NST]  digit tiles of the stage landed (TMA tx); only the MMA waits on it
  StageDesc* desc = reinterpret_cast<StageDesc*>(tready + NST);       // [NST]
  uint4* mbox = reinterpret_cast<uint4*>((reinterpret_cast<uintptr_t>(desc + NST) + 15) & ~(uintptr_t)15);   // [DWG][2] decode -> MMA notes
  int64_t* span = reinterpret_cast<int64_t*>(mbox + 2 * DWG);         // [2] this CTA's item range
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(span + 2);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int64_t grid = gridDim.x, cta = blockIdx.x;
  if (threadIdx.x == 0) {
    if (kTrace && p.trace) p.trace[cta * 256 + 0] = gtime();
    span[0] = p.span[cta];
    span[1] = p.span[cta + 1];
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::kEmptyCount + (p.gstage ? 4 : 0));   // + the epilogue in grouped per-stage mode
      mbar_init(&tready[s], 1);
    }
    for (int i = 0; i < 2 * DWG; ++i) { mbar_init(&afull[i], 4); mbar_init(&aempty[i], 1); }
    for (int i = 0; i < 2 * NDQ; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == C::kProdWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t i0 = span[0], i1 = span[1];
  if (kTrace && p.trace && threadIdx.x == 0) {
    p.trace[cta * 256 + 58] = (unsigned long long)i0;
    p.trace[cta * 256 + 59] = (unsigned long long)i1;
    p.trace[cta * 256 + 61] = (unsigned long long)items_per_rb(g);
  }
  const int n_rb = items_per_rb(g);
  const uint32_t tile_bytes = (uint32_t)NN * kSuperStep;

  if (warp == C::kProdWarp) {
    // ==================================================================== producer
    if (lane == 0) {
      pdl_launch_dependents();
      const uint64_t pol = evict_first_policy(), pol_x = evict_last_policy();
      // Until the x-digit pass (the previous kernel) has completed, only the
      // weight codes are prefetched; the digit-tile copies of those stages are
      // issued after pdl_wait().
      bool dep = false;
      int npend = 0;
      int32_t pend_sli[8], pend_n[8], pend_s[8];
      auto resolve = [&]() {
        pdl_wait();
        dep = true;
        for (int i = 0; i < npend; ++i)
        {
          bulk_g2s(ring + (size_t)pend_s[i] * p.stage_bytes + p.tile_off, p.tiles + (int64_t)pend_sli[i] * tile_bytes,
                   (uint32_t)pend_n[i] * tile_bytes, &tready[pend_s[i]], pol_x);
          if (p.gstage)
            bulk_g2s(ring + (size_t)pend_s[i] * p.stage_bytes + p.sum_off, p.sums + (int64_t)pend_sli[i] * p.Bp,
                     (uint32_t)(pend_n[i] * p.Bp * 8), &tready[pend_s[i]], pol_x);
        }
        npend = 0;
      };
      // code stages only: weak chunks never enter the ring (the epilogue reads them)
      StageIter it;
      it.init(g, i0, i1, p.cap);
      auto next_code = [&](int64_t& rb_, int32_t& li_) {
        int32_t m;
        while ((m = it.next(rb_, li_)) > 0 && li_ >= g.nss) {}
        return m;
      };
      int64_t srb, nrb = 0;
      int32_t sli, nli = 0;
      int32_t n = next_code(srb, sli);
      int s = 0, k = 0;
      uint32_t ph = 0;
      while (n > 0) {
        const int32_t nn = next_code(nrb, nli);
        if (k >= NST) {
          if (!dep) resolve();
          mbar_wait(&empty[s], ph ^ 1u);
        }
        if (kTrace && p.trace && k < 32) p.trace[cta * 256 + 64 + k] = gtime();
        uint32_t fl = 0;
        if (nn == 0 || nrb != srb) fl |= kRbEnd;
        else if (group_of(p, nli) == group_of(p, sli + n - 1)) fl |= kGroupCont;
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_addr(&desc[s])), "r"((uint32_t)srb),
                     "r"((uint32_t)(sli & 0xFFFF) | ((uint32_t)n << 16) | (fl << 24)) : "memory");
        uint8_t* st = ring + (size_t)s * p.stage_bytes;
        const uint32_t cbytes = (uint32_t)stage_bytes(g, sli, n);
        {
          // codes -> full[s] (decode), digit tiles -> tready[s] (MMA only), so the
          // decode can run while the x-digit pass is still producing the tiles
          const uint32_t sumb = p.gstage ? (uint32_t)(n * p.Bp * 8) : 0u;
          uint32_t szb = 0;
          if (p.gstage) {
            const int gi0 = group_of(p, sli);
            szb = (uint32_t)((group_of(p, sli + n - 1) - gi0 + 1) * kSZBlockBytes);
            mbar_expect_tx(&full[s], cbytes + szb);
            bulk_g2s(st + p.sz_off, p.blob + g.sz_off + (srb * g.G + gi0) * kSZBlockBytes, szb, &full[s], pol);
          } else {
            mbar_expect_tx(&full[s], cbytes);
          }
          mbar_expect_tx(&tready[s], (uint32_t)n * tile_bytes + sumb);
          bulk_g2s(st, p.blob + g.units_off + item_offset(g, srb, sli), cbytes, &full[s], pol);
          if (dep) {
            bulk_g2s(st + p.tile_off, p.tiles + (int64_t)sli * tile_bytes, (uint32_t)n * tile_bytes, &tready[s], pol_x);
            if (sumb) bulk_g2s(st + p.sum_off, p.sums + (int64_t)sli * p.Bp, sumb, &tready[s], pol_x);
          } else {
            pend_sli[npend] = sli; pend_n[npend] = n; pend_s[npend] = s; ++npend;
          }
        }
        ++k;
        if (++s == NST) { s = 0; ph ^= 1u; }
        srb = nrb;
        sli = nli;
        n = nn;
      }
      if (!dep) resolve();
      // terminal descriptor: consumers leave their loops
      if (k >= NST) mbar_wait(&empty[s], ph ^ 1u);
      asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(smem_addr(&desc[s])), "r"(0u) : "memory");
      mbar_arrive(&full[s]);
    }
  } else if (warp < C::kDecodeWarps) {
    // ==================================================================== decode
    // Warpgroup wg decodes a contiguous share (<= kIPW items of 128 rows x 64
    // codes) of every code stage into one of its two TMEM A buffers and
    // publishes it to its MMA warp: afull + a mailbox note {stage, share, flags}.
    // Every code stage is published (possibly with no items) so the MMA warp
    // sees each group end; a note with n == 0 ends the MMA warp.  One warp per
    // warpgroup polls the mbarriers, the others wait on a named barrier.
    const int wg = warp >> 2, q = warp & 3;
    const int row = q * 32 + lane;                      // TMEM lane / row inside the row-block
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(wg * 2 * C::kABuf);
    constexpr uint32_t kSS = (uint32_t)kRowBlock * (BITS == 3 ? 6 : 8) * 4;   // bytes per super-step record
    constexpr uint32_t kHiStride = BITS == 3 ? 8u : 16u;   // words 4.. of a row
    const Shifts sh = make_shifts();
    const int nss = g.nss;
    const int bar_id = 3 + wg;
    uint32_t acnt = 0;                                  // A buffers published
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
      if (q == 0) mbar_wait(&full[s], ph);
      named_sync(bar_id, 128);
      const StageDesc d = load_desc(&desc[s]);
      if (d.n == 0) break;   // the MMA warps walk the stage sequence themselves: no terminal note
      const bool code = d.li < nss;
      if (code) {
        const uint32_t buf = acnt & 1u;
        if (acnt >= 2) {
          if (q == 0) mbar_wait(&aempty[wg * 2 + buf], ((acnt >> 1) & 1u) ^ 1u);
          named_sync(bar_id, 128);
        }
        ++acnt;
        int lo = 0, hi = 0;
        if (code) {
          share<DWG>(d.n, wg, lo, hi);
          tc_fence_after();
          const uint32_t sbase = smem_addr(ring + (size_t)s * p.stage_bytes);
          const uint32_t a_lo = sbase + (uint32_t)lo * kSS + (uint32_t)row * 16u;
          const uint32_t a_hi = sbase + (uint32_t)lo * kSS + 2048u + (uint32_t)row * kHiStride;
          const uint32_t tcol = trow + buf * (uint32_t)C::kABuf;
          auto load_item = [&](int t, uint32_t* w) {
            const uint4 a = lds128(a_lo + t * kSS);
            w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
            if (BITS == 3) {
              const uint2 b = lds64(a_hi + t * kSS);
              w[4] = b.x; w[5] = b.y;
            } else {
              const uint4 b = lds128(a_hi + t * kSS);
              w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
            }
          };
          auto store_item = [&](int t, const uint32_t* w) {
            uint32_t o[16];
            decode_row<BITS>(w, o, sh);
            tc_st16(tcol + t * C::kACols, o);
          };
          if (kTrace && p.exp == 3) {
          } else if (hi - lo == C::kIPW) {   // full share: unrolled, immediate offsets
#pragma unroll
            for (int t = 0; t < C::kIPW; ++t) {
              uint32_t w[8];
              load_item(t, w);
              store_item(t, w);
            }
          } else {
            for (int t = 0; t < hi - lo; ++t) {
              uint32_t w[8];
              load_item(t, w);
              store_item(t, w);
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
        }
        if (q == 0 && lane == 0)
          mbox[wg * 2 + buf] = make_uint4((uint32_t)s | (ph << 31), (uint32_t)(uint16_t)d.li,
                                          (uint32_t)d.n | ((uint32_t)lo << 8) | ((uint32_t)hi << 16) | ((uint32_t)d.flags << 24),
                                          (uint32_t)d.rb);
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[wg * 2 + buf]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == NST) { s = 0; ph ^= 1u; }
    }
  } else if (warp >= C::kMmaWarp0 && warp < C::kProdWarp) {
    // ==================================================================== MMA issue (ISS warps per warpgroup)
    // Each issuer walks the CTA's code-stage sequence itself (the producer's
    // partition).  Stage j goes to A buffer j & 1; issuer ii of warpgroup wg
    // issues the stages with (j & 1) == ii (every stage when ISS == 1) into its
    // own D accumulators, and commits its D (dfull) at every end of a scale group
    // it has open -- also when the group ends in the other issuer's stage.  The
    // whole warp runs this (warp-uniform); one elected lane issues each mma/commit.
    constexpr int ISS = C::ISS;
    const int wq = warp - C::kMmaWarp0, wg = wq / ISS, ii = wq % ISS;
    const int dq = wg * ISS + ii;                       // D owner index
    uint32_t dcnt = 0;
    bool open = false;          // D[dcnt & 1] holds a partial group sum
    int64_t orb = -1;
    int ogi = -1;               // the open group's row-block and group
    const int gl = g.group ? p.group_log2 : 30;
    const uint32_t a_wg = tmem + (uint32_t)(wg * 2 * C::kABuf);
    constexpr uint32_t kLbo = (NN / 8) * 128;          // K-adjacent core matrices
    const uint32_t ring0 = smem_addr(ring) + (uint32_t)p.tile_off;
    long long c_wait = 0, c_issue = 0, c_commit = 0, c_mma = 0, c_tready = 0, c_dempty = 0;   // trace only
    auto close_group = [&]() {
      tc_commit_elect(&dfull[dq * 2 + (dcnt & 1u)]);
      ++dcnt;
      open = false;
    };
    // The stage sequence comes from the producer's descriptors (desc[s], visible
    // once full[s] completed; a descriptor with n == 0 ends the sequence).
    int j = 0, kst = 0;
    for (;;) {
      const int s = j % NST;
      mbar_wait(&full[s], (uint32_t)(j / NST) & 1u);
      const StageDesc dsc = load_desc(&desc[s]);
      if (dsc.n == 0) break;
      const int64_t srb = dsc.rb;
      const int32_t sli = dsc.li, n = dsc.n;
      const uint32_t buf = (uint32_t)j & 1u;
      if (ISS == 1 || (int)buf == ii) {
        const long long t0 = OWQ_CLK();
        mbar_wait(&afull[wg * 2 + buf], ((uint32_t)j >> 1) & 1u);
        const long long t1 = OWQ_CLK();
        c_wait += t1 - t0;
        int lo, hi;
        share<DWG>(n, wg, lo, hi);
        mbar_wait(&tready[s], (uint32_t)(j / NST) & 1u);   // this stage's digit tiles
        c_tready += OWQ_CLK() - t1;
        if (kTrace && p.trace && dq == 0 && lane == 0 && kst < 32) p.trace[cta * 256 + 224 + kst] = gtime();
        tc_fence_after();
        const uint32_t stile = ring0 + (uint32_t)s * (uint32_t)p.stage_bytes;
        const bool cont = (dsc.flags & kGroupCont) != 0;   // the stage's last group continues in the next stage
        if (C::kGP > 1 && p.g.group) {
          // grouped scales: D of this stage = [buf][piece] blocks, drained by the
          // epilogue per stage (dempty of the stage that used this buffer before)
          if (j >= 2) mbar_wait(&dempty[wg * 2 + buf], (((uint32_t)j >> 1) - 1) & 1u);
          tc_fence_after();
          const int g0 = (sli + lo) >> gl;
          for (int pi = lo; pi < hi; ++pi) {
            const int gi = (sli + pi) >> gl;
            const bool first = pi == lo || gi != ((sli + pi - 1) >> gl);
            const uint32_t d_t = tmem + (uint32_t)(C::kDCol0 + ((wg * 2 + buf) * C::kGP + (gi - g0)) * NN);
            const uint32_t a_t = a_wg + buf * (uint32_t)C::kABuf + (uint32_t)(pi - lo) * C::kACols;
            const uint32_t tb = stile + (uint32_t)pi * tile_bytes;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
              tc_mma_i8_elect(d_t, a_t + 8 * jj, umma_desc(tb + jj * 2 * kLbo, kLbo, 128), idesc_i8<NN>(),
                              (!first || jj > 0) ? 1u : 0u);
            c_mma += 2;
          }
          tc_commit_elect(&dfull[wg * 2 + buf]);   // this stage's group pieces (possibly none)
        } else if (!p.g.group && hi - lo == C::kIPW) {
          // common case: one scale group, full share -> one asm block, one elect
          const uint32_t dbuf = dcnt & 1u;
          const long long td0 = OWQ_CLK();
          if (!open && dcnt >= 2) mbar_wait(&dempty[dq * 2 + dbuf], ((dcnt >> 1) - 1) & 1u);
          c_dempty += OWQ_CLK() - td0;
          tc_mma_i8_stage<C::kIPW, NN * kSuperStep, kLbo>(
              tmem + (uint32_t)(C::kDCol0 + (dq * 2 + dbuf) * C::kGP * NN), a_wg + buf * (uint32_t)C::kABuf,
              umma_desc(stile + (uint32_t)lo * tile_bytes, kLbo, 128), idesc_i8<NN>(), open ? 1u : 0u);
          open = true;
          orb = srb;
          ogi = 0;
          c_mma += 2 * C::kIPW;
          if (!cont) close_group();
        } else {
          StageDesc d;
          d.rb = (int32_t)srb; d.li = (int16_t)sli; d.n = (uint8_t)n; d.flags = cont ? kGroupCont : 0;
          for (int pa = 0; pa < n;) {
            const Seg sg = segment(p, pa, d);
            const int a0 = sg.pa > lo ? sg.pa : lo, a1 = sg.pb + 1 < hi ? sg.pb + 1 : hi;
            if (open && (orb != srb || ogi != sg.gi)) close_group();   // (cannot happen: closed at its end)
            for (int pi = a0; pi < a1; ++pi) {
              const uint32_t dbuf = dcnt & 1u;
              if (!open && dcnt >= 2) mbar_wait(&dempty[dq * 2 + dbuf], ((dcnt >> 1) - 1) & 1u);
              const uint32_t a_t = a_wg + buf * (uint32_t)C::kABuf + (uint32_t)(pi - lo) * C::kACols;
              const uint32_t d_t = tmem + (uint32_t)(C::kDCol0 + (dq * 2 + dbuf) * C::kGP * NN);
              const uint32_t tb = stile + (uint32_t)pi * tile_bytes;
#pragma unroll
              for (int jj = 0; jj < 2; ++jj)   // K = 32 columns each: TMEM columns 8jj.., core-matrix K-chunks 2jj, 2jj+1
                tc_mma_i8_elect(d_t, a_t + 8 * jj, umma_desc(tb + jj * 2 * kLbo, kLbo, 128), idesc_i8<NN>(),
                                (open || jj > 0) ? 1u : 0u);
              open = true;
              orb = srb;
              ogi = sg.gi;
              c_mma += 2;
            }
            if (sg.ends && open) close_group();
            pa = sg.pb + 1;
          }
        }
        const long long t2 = OWQ_CLK();
        tc_commit_elect(&aempty[wg * 2 + buf]);   // A buffer consumed once these MMAs complete
        tc_commit_elect(&empty[s]);                // ... and the stage's digit tiles
        const long long t3 = OWQ_CLK();
        c_issue += t2 - t1;
        c_commit += t3 - t2;
        if (kTrace && p.trace && dq == 0 && lane == 0 && kst < 32) p.trace[cta * 256 + 128 + kst] = gtime();
        ++kst;
      } else if (open) {
        // the other issuer's stage: does my open group end inside it?
        bool ends;
        if (orb != srb || (sli >> gl) != ogi) {
          ends = true;   // (defensive: the group ended before this stage)
        } else {
          const bool later = ((sli + n - 1) >> gl) != ogi;   // the stage reaches a later group
          ends = later || !(dsc.flags & kGroupCont);
        }
        if (ends) close_group();
      }
      ++j;
    }
    if (open && !(C::kGP > 1 && p.g.group)) close_group();
    if (kTrace && p.trace && lane == 0) {
      p.trace[cta * 256 + 1 + dq] = (unsigned long long)c_wait;
      p.trace[cta * 256 + 5 + dq] = (unsigned long long)c_issue;
      p.trace[cta * 256 + 9 + dq * 0] = (unsigned long long)c_commit;
      p.trace[cta * 256 + 52] = (unsigned long long)c_mma;
      p.trace[cta * 256 + 42 + dq] = (unsigned long long)c_tready;
      p.trace[cta * 256 + 46 + dq] = (unsigned long long)c_dempty;
    }
  } else if (warp >= C::kEpiWarp0 && warp < C::kMmaWarp0) {
    // ==================================================================== epilogue
    // Independent of the shared-memory ring: walks this CTA's item sequence
    // itself (the producer's stage partition, without waiting on stages),
    // prefetches each scale group's scale/zero, digit sums and the row's weak
    // values from global memory when the group opens, and only waits on the
    // D accumulators (dfull) at the group end.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int et = threadIdx.x - C::kEpiWarp0 * 32;     // 0..127
    pdl_wait();   // x may come from the previous kernels; digit sums (p.sums) from the x-digit pass
    {  // x gathered at the weak columns, x[b][idx[t]] (0 for padding)
      const uint16_t* widx = reinterpret_cast<const uint16_t*>(p.blob + g.widx_off);
      for (int i = et; i < p.B * g.kpad; i += 128) {
        const int b = i / g.kpad, t = i - b * g.kpad;
        xw[i] = t < g.k ? p.x[(int64_t)b * p.xK + widx[t]] : __float2half(0.f);
      }
    }
    named_sync(2, 128);
    constexpr double kPow256[6] = {1.0, 256.0, 65536.0, 16777216.0, 4294967296.0, 1099511627776.0};
    const int gl = g.group ? p.group_log2 : 30;
    float tot[MAXB];
    int64_t keep_rb = -1;                                // row-block this CTA sums at its end (fixup)
    long long sacc[MAXB];                                // this thread's share of the open group's digit sums
#pragma unroll
    for (int b = 0; b < MAXB; ++b) { tot[b] = 0.f; sacc[b] = 0; }
    constexpr int ISS = C::ISS;
    uint32_t dcnt[NDQ];
#pragma unroll
    for (int w = 0; w < NDQ; ++w) dcnt[w] = 0;
    uint32_t part = 0;                                   // D owners (warpgroup, issuer) with items in the open group
    int jc = 0;                                          // code-stage index (stage j -> issuer j & 1 when ISS == 2)
    bool gopen = false;
    bool sdirect = false;                                // the open group's digit sums are complete in sacc
    uint32_t szw = 0;                                    // the open group's (s, z) for this row
    uint4 wpre[2];                                       // this row's first two weak chunks of the row-block (prefetch)
    int64_t wpre_rb = -1;
    int ngend = 0, kst = 0, rr = 0;
    // pieces of this CTA's first and last row-block (host table; the row-blocks
    // in between are whole in this CTA)
    const int64_t rb_a = i0 / n_rb, rb_b = (i1 - 1) / n_rb;
    const uint64_t fx = p.fix[cta];
    auto pieces = [&](int64_t rb, int64_t& cf, int64_t& cl) {
      if (rb == rb_a) { cf = (int64_t)(fx & 0xFFFF); cl = (int64_t)((fx >> 16) & 0xFFFF); }
      else if (rb == rb_b) { cf = (int64_t)((fx >> 32) & 0xFFFF); cl = (int64_t)(fx >> 48); }
      else { cf = cta; cl = cta; }
    };
    StageIter it;
    it.init(g, i0, i1, p.cap);
    int64_t crb, nrb = -1;
    int32_t cli, nli = 0;
    int32_t cn = it.next(crb, cli);
    // grouped-scale per-stage mode (C::kGP > 1): the open group's running sums
    const bool gmode = C::kGP > 1 && g.group != 0;
    long long e_ring = 0, e_dfull = 0, e_ld = 0, e_comb = 0;   // trace only
    // exact int64 throughout: |X| < 2^40 makes |sum_i 256^i D_i| < 2^62 for any K
    int gm_g = -1;
    long long gm_v = 0, gm_s = 0;
    uint32_t gm_sz = 0;
    // (macro, not a lambda: a by-reference capture kept the group state in local memory)
#define OWQ_GM_FINISH()                                                                                 \
  do {                                                                                                  \
    if (gm_g >= 0) {                                                                                    \
      const __half2 szv_ = u2h(gm_sz);                                                                  \
      const long long vz_ = gm_v - (long long)__high2float(szv_) * gm_s; /* z is an integer code */     \
      tot[0] = fmaf(__low2float(szv_) * 5.9604644775390625e-08f, __ll2float_rn(vz_), tot[0]);           \
    }                                                                                                   \
    gm_g = -1;                                                                                          \
  } while (0)
    while (cn > 0) {
      int32_t nn = it.next(nrb, nli);
      if (cli < g.nss && gmode) {
        // one D buffer per stage and warpgroup: [piece] blocks of kGP x NN columns
        const int gA = cli >> gl;
        constexpr int kCapMax = DWG * C::kIPW;
        // the stage's digit sums and (s, z) blocks are staged in the ring (tready / full)
        const int rs = jc % NST;
        const uint32_t rph = (uint32_t)(jc / NST) & 1u;
        long long tq0 = OWQ_CLK();
        if (q == 0) {
          mbar_wait(&full[rs], rph);
          mbar_wait(&tready[rs], rph);
        }
        named_sync(2, 128);
        const uint32_t sb = smem_addr(ring + (size_t)rs * p.stage_bytes);
        (void)kCapMax;
        long long tq1 = OWQ_CLK();
        e_ring += tq1 - tq0;
        for (int w = 0; w < DWG; ++w) {
          long long tw0 = OWQ_CLK();
          if (q == 0) mbar_wait(&dfull[w * 2 + (jc & 1)], ((uint32_t)jc >> 1) & 1u);
          named_sync(2, 128);
          tc_fence_after();
          long long tw1 = OWQ_CLK();
          e_dfull += tw1 - tw0;
          int lo, hi;
          share<DWG>(cn, w, lo, hi);
          if (lo < hi) {
            const uint32_t tcol = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(C::kDCol0 + (w * 2 + (jc & 1)) * C::kGP * NN);
            const int g0 = (cli + lo) >> gl;
            long long tw2 = OWQ_CLK();
#pragma unroll
            for (int c16 = 0; c16 < C::kGP * NN / 16; ++c16) {   // two pieces (2 x NN columns) per load
              uint32_t dd[16];
              tc_ld16(tcol + 16 * c16, dd);
#pragma unroll
              for (int ph2 = 0; ph2 < 16 / NN; ++ph2) {
                const int pc = c16 * (16 / NN) + ph2;
                const int gp = g0 + pc;
                const int ia = ((gp << gl) - cli) > lo ? ((gp << gl) - cli) : lo;
                const int ib = (((gp + 1) << gl) - cli) < hi ? (((gp + 1) << gl) - cli) : hi;
                if (ia < ib) {
                  long long v = 0;
#pragma unroll
                  for (int i = 0; i < kDigits; ++i) v += (long long)(int)dd[ph2 * NN + i] << (8 * i);
                  long long sp = 0;
#pragma unroll 1
                  for (int t = ia; t < ib; ++t) {
                    const uint2 sv = lds64(sb + (uint32_t)p.sum_off + (uint32_t)(t * p.Bp) * 8u);
                    sp += (long long)(((unsigned long long)sv.y << 32) | sv.x);
                  }
                  if (gp != gm_g) {
                    OWQ_GM_FINISH();
                    gm_g = gp;
                    gm_v = 0;
                    gm_s = 0;
                    gm_sz = lds32(sb + (uint32_t)p.sz_off + (uint32_t)(gp - gA) * kSZBlockBytes + row * 4);
                  }
                  gm_v += v;
                  gm_s += sp;
                }
              }
            }
            e_comb += OWQ_CLK() - tw2;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[w * 2 + (jc & 1)]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rs]);   // done with the stage's staged sums and (s, z)
        ++jc;
      } else if (cli < g.nss) {
        for (int pa = 0; pa < cn;) {
          const int gi = (cli + pa) >> gl;
          const int gend = ((gi + 1) << gl) - cli - 1;   // last stage position of this group
          const int pb = gend < cn - 1 ? gend : cn - 1;
          const bool ends = pb + 1 < cn || !(nn > 0 && nrb == crb && nli < g.nss && (nli >> gl) == gi);
          if (wpre_rb != crb) {
            // row-block opens: prefetch this row's weak values of the CTA's first two
            // weak chunks of the row-block (full chunks only; the rest load on demand)
            wpre_rb = crb;
            const int64_t w0 = (i0 > crb * n_rb + g.nss ? i0 - crb * n_rb : g.nss) - g.nss;   // first weak chunk in this CTA
            const int64_t w1 = (i1 < (crb + 1) * n_rb ? i1 - crb * n_rb : n_rb) - g.nss;
            const uint8_t* wb = p.blob + g.units_off + item_offset(g, crb, g.nss);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              wpre[j] = make_uint4(0, 0, 0, 0);
              if (w0 + j < w1 && w0 + j < g.nfull)
                wpre[j] = __ldg(reinterpret_cast<const uint4*>(wb + (w0 + j) * kWeakChunkBytes + row * 16));
            }
          }
          if (!gopen) {
            // group opens: prefetch (s, z) of this row and this thread's share of the
            // group's digit sums (items gfirst .. glast of this CTA)
            gopen = true;
            szw = __ldg(reinterpret_cast<const unsigned int*>(p.blob + g.sz_off + ((int64_t)crb * g.G + gi) * kSZBlockBytes +
                                                              row * 4));
            const int gfirst = cli + pa;
            const int64_t cend = (i1 - crb * n_rb < (int64_t)g.nss ? i1 - crb * n_rb : (int64_t)g.nss) - 1;   // CTA's last code item in rb
            const int glast = (int)(((int64_t)((gi + 1) << gl) - 1 < cend) ? ((gi + 1) << gl) - 1 : cend);
            if (g.group && (glast - gfirst + 1) * MAXB <= 32) {
              // small group: every thread sums the whole group (no block reduction at its end)
              sdirect = true;
#pragma unroll 1
              for (int li = gfirst; li <= glast; ++li)
#pragma unroll
                for (int b = 0; b < MAXB; ++b)
                  if (b < p.B) sacc[b] += __ldg(&p.sums[(int64_t)li * p.Bp + b]);
            } else {
              for (int li = gfirst + et; li <= glast; li += 128)
#pragma unroll
                for (int b = 0; b < MAXB; ++b)
                  if (b < p.B) sacc[b] += __ldg(&p.sums[(int64_t)li * p.Bp + b]);
            }
          }
          {
            const int iss = ISS == 1 ? 0 : (jc & 1);
            if (cn == p.cap && !g.group) {   // full stage, one segment: every warpgroup has items
#pragma unroll
              for (int w = 0; w < DWG; ++w) part |= 1u << (w * ISS + iss);
            } else {
#pragma unroll
              for (int w = 0; w < DWG; ++w) {
                int lo, hi;
                share<DWG>(cn, w, lo, hi);
                if (lo <= pb && hi > pa) part |= 1u << (w * ISS + iss);
              }
            }
          }
          if (ends) {
            if (kTrace && p.trace && et == 0 && ngend < 4) p.trace[cta * 256 + 18 + 6 * ngend] = gtime();
            // block-reduce the digit-sum shares (the same for every row)
            long long S[MAXB];
            if (sdirect) {
#pragma unroll
              for (int b = 0; b < MAXB; ++b) { S[b] = sacc[b]; sacc[b] = 0; }
              sdirect = false;
            } else {
              long long* rd = red + (rr & 1) * 4 * OWQ_MAX_BATCH;
#pragma unroll
              for (int b = 0; b < MAXB; ++b) {
                long long v = sacc[b];
                sacc[b] = 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) rd[q * OWQ_MAX_BATCH + b] = v;
              }
              named_sync(2, 128);
#pragma unroll
              for (int b = 0; b < MAXB; ++b)
                S[b] = rd[b] + rd[OWQ_MAX_BATCH + b] + rd[2 * OWQ_MAX_BATCH + b] + rd[3 * OWQ_MAX_BATCH + b];
              ++rr;
            }
            if (kTrace && p.trace && et == 0 && ngend < 4) p.trace[cta * 256 + 19 + 6 * ngend] = gtime();
            const __half2 szv = u2h(szw);
            const float s_g = __low2float(szv);
            const double z_g = (double)__high2float(szv);
            double dacc[MAXB];
#pragma unroll
            for (int b = 0; b < MAXB; ++b) dacc[b] = 0.0;
#pragma unroll
            for (int w = 0; w < NDQ; ++w) {
              if (part & (1u << w)) {   // fixed order over D owners: deterministic
                const uint32_t dbuf = dcnt[w] & 1u;
                // one warp waits (suspending), the others block on the named barrier
                if (q == 0) mbar_wait(&dfull[w * 2 + dbuf], (dcnt[w] >> 1) & 1u);
                named_sync(2, 128);
                tc_fence_after();
                const uint32_t tcol = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(C::kDCol0 + (w * 2 + dbuf) * C::kGP * NN);
                constexpr int kL = (MAXB * kDigits + 15) / 16;
                if (kL <= 2) {
                  // small D: into registers, back to the MMA warp, then combine
                  uint32_t dall[kL][16];
#pragma unroll
                  for (int c16 = 0; c16 < kL; ++c16) tc_ld16_nowait(tcol + 16 * c16, dall[c16]);
                  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                  tc_fence_before();
                  __syncwarp();
                  if (lane == 0) mbar_arrive(&dempty[w * 2 + dbuf]);
#pragma unroll
                  for (int c16 = 0; c16 < kL; ++c16)
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                      const int col = 16 * c16 + j, b = col / kDigits, i = col % kDigits;
                      if (b < MAXB) dacc[b] += (double)(int)dall[c16][j] * kPow256[i];
                    }
                } else {
#pragma unroll
                  for (int c16 = 0; c16 < kL; ++c16) {
                    uint32_t dd[16];
                    tc_ld16(tcol + 16 * c16, dd);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                      const int col = 16 * c16 + j, b = col / kDigits, i = col % kDigits;
                      if (b < MAXB) dacc[b] += (double)(int)dd[j] * kPow256[i];
                    }
                  }
                  tc_fence_before();
                  __syncwarp();
                  if (lane == 0) mbar_arrive(&dempty[w * 2 + dbuf]);
                }
                ++dcnt[w];
              }
            }
            if (kTrace && p.trace && et == 0 && ngend < 4) p.trace[cta * 256 + 20 + 6 * ngend] = gtime();
#pragma unroll
            for (int b = 0; b < MAXB; ++b)
              tot[b] = fmaf(s_g, (float)((dacc[b] - z_g * (double)S[b]) * 5.9604644775390625e-08), tot[b]);
            if (kTrace && p.trace && et == 0 && ngend < 4) p.trace[cta * 256 + 21 + 6 * ngend] = gtime();
            ++ngend;
            part = 0;
            gopen = false;
          }
          pa = pb + 1;
        }
        ++jc;
        if (!g.group && C::ISS == 1 && gopen) {
          // Per-row scales: the stages between a group's first and last one need
          // nothing from the epilogue (they are full, so every warpgroup has
          // items) -- jump the walk to the group's last stage.
          const int64_t rb0 = crb * n_rb;
          const int64_t gs = i0 > rb0 ? i0 - rb0 : 0;                                  // group start (rb-relative)
          const int64_t ge = i1 - rb0 < (int64_t)g.nss ? i1 - rb0 : (int64_t)g.nss;   // group end
          const int64_t last = gs + (ge - gs - 1) / p.cap * p.cap;                     // its last stage
          if (last > (int64_t)cli + cn) {
#pragma unroll
            for (int w = 0; w < DWG; ++w) part |= 1u << w;
            it.rb = crb;
            it.li = (int32_t)last;
            it.left = i1 - (rb0 + last);
            nn = it.next(nrb, nli);
          }
        }
      } else {
        // weak chunks (straight from the blob, not through the ring): fp16 weak
        // columns x gathered activations, fp32 (unscaled)
        const uint8_t* wbase = p.blob + g.units_off + item_offset(g, crb, cli);
        const int64_t w0 = (i0 > crb * n_rb + g.nss ? i0 - crb * n_rb : g.nss) - g.nss;
        // four chunk loads in flight per batch (k = 153 has 20 chunks per row-block;
        // one load at a time left the epilogue latency-bound, DESIGN.md §6.2 k-sweep)
        for (int pi0 = 0; pi0 < cn; pi0 += 4) {
          uint4 av[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int pi = pi0 + u;
            const int gch = cli - g.nss + pi;
            av[u] = make_uint4(0, 0, 0, 0);
            if (pi < cn && gch < g.nfull) {
              const int jpre = (int)(gch - w0);
              av[u] = (wpre_rb == crb && jpre >= 0 && jpre < 2)
                          ? (jpre == 0 ? wpre[0] : wpre[1])
                          : __ldg(reinterpret_cast<const uint4*>(wbase + (size_t)pi * kWeakChunkBytes + row * 16));
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int pi = pi0 + u;
            if (pi >= cn) break;
            const int gch = cli - g.nss + pi;
            float v[8];
            if (gch < g.nfull) {
              const uint32_t aw[4] = {av[u].x, av[u].y, av[u].z, av[u].w};
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const float2 f = __half22float2(u2h(aw[c]));
                v[2 * c] = f.x;
                v[2 * c + 1] = f.y;
              }
            } else {
              const __half* tl = reinterpret_cast<const __half*>(wbase + (size_t)pi * kWeakChunkBytes);
#pragma unroll
              for (int c = 0; c < 8; ++c) v[c] = c < g.ktail ? __half2float(tl[row * g.ktail + c]) : 0.f;
            }
#pragma unroll
            for (int b = 0; b < MAXB; ++b) {
              if (b < p.B) {
                const uint4 xv = *reinterpret_cast<const uint4*>(xw + b * g.kpad + gch * kWeakChunk);
                const uint32_t xwv[4] = {xv.x, xv.y, xv.z, xv.w};
                float acc = tot[b];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const float2 f = __half22float2(u2h(xwv[c]));
                  acc = fmaf(v[2 * c], f.x, acc);
                  acc = fmaf(v[2 * c + 1], f.y, acc);
                }
                tot[b] = acc;
              }
            }
          }
        }
      }
      if (kTrace && p.trace && et == 0 && kst < 32) p.trace[cta * 256 + 160 + kst] = gtime();
      ++kst;

      if (gmode && (nn == 0 || nrb != crb || nli >= g.nss)) OWQ_GM_FINISH();   // the row-block's code part is done
      if (nn == 0 || nrb != crb) {
        // -------------------------------------------------- finish row-block crb
        if (kTrace && p.trace && et == 0) p.trace[cta * 256 + 50] = gtime();
        const int64_t ifirst = crb * n_rb, ilast = ifirst + n_rb - 1;
        const bool whole = ifirst >= i0 && ilast < i1;
        const int64_t grow = crb * kRowBlock + row;
        if (whole) {
          if (grow < g.M) {
#pragma unroll
            for (int b = 0; b < MAXB; ++b)
              if (b < p.B) {
                if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = tot[b];
                else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(tot[b]);
              }
          }
        } else {
          // pieces = CTAs holding the first .. last item of the row-block (none is empty)
          int64_t c_first, c_last;
          pieces(crb, c_first, c_last);
          const int npieces = (int)(c_last - c_first + 1);
          uint32_t* pw = p.slots;   // [cta][B][128]: each CTA has at most one non-summer piece (its first row-block)
#ifndef OWQ_SUMMER_LOW
#define OWQ_SUMMER_LOW 0   // A/B builds only: 1 = round 1's lowest-piece summer compiled in alone
#endif
          if ((OWQ_SUMMER_LOW || (kTrace && p.exp == 7)) && p.coresident) {
            // A/B only (OWQ_EXP=7 or -DOWQ_SUMMER_LOW=1): round 1's protocol, the lowest
            // piece sums.  Faster (12288^2: -0.3 us at B = 1, -4..7 us at B = 8..16,
            // profiles/r2_summer_ab.txt) but its summer waits on HIGHER-index CTAs: two
            // full grids on concurrent streams (the bench's q/k/v) can each hold SMs
            // the other's missing pieces need, so it is not the product protocol.
            if (cta != c_first) {
#pragma unroll
              for (int b = 0; b < MAXB; ++b)
                if (b < p.B) st_relaxed(pw + (cta * p.B + b) * kRowBlock + row, ~__float_as_uint(tot[b]));
            } else {
              for (int qq = 1; qq < npieces; ++qq) {
                uint32_t w[MAXB];
#pragma unroll
                for (int b = 0; b < MAXB; ++b)
                  w[b] = b < p.B ? ld_relaxed(pw + ((c_first + qq) * p.B + b) * kRowBlock + row) : 1u;
#pragma unroll
                for (int b = 0; b < MAXB; ++b)
                  if (b < p.B) {
                    uint32_t* a = pw + ((c_first + qq) * p.B + b) * kRowBlock + row;
                    while (w[b] == 0u) {
                      __nanosleep(32);
                      w[b] = ld_relaxed(a);
                    }
                    st_relaxed(a, 0u);
                    tot[b] += __uint_as_float(~w[b]);
                  }
              }
              if (grow < g.M) {
#pragma unroll
                for (int b = 0; b < MAXB; ++b)
                  if (b < p.B) {
                    if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = tot[b];
                    else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(tot[b]);
                  }
              }
            }
          } else if (p.coresident) {
            // Fixed summer = the CTA holding the row-block's LAST item (the
            // highest-index piece, CUTLASS's stream-K rule).  For that CTA the
            // row-block is its first one, so it parks its partial in its own
            // partial-row slot (same thread stores and reloads it; registers
            // live across the whole loop spilled the batch variants) and sums
            // after all its own work; every other piece is its CTA's last
            // row-block and is stored (as ~bits: a zero word = not written yet; the
            // workspace starts zeroed and the summer zeroes what it consumed)
            // before that CTA waits on anything.  A summer only ever waits on
            // lower-index CTAs, so progress needs in-order dispatch, not
            // co-residency of the whole grid.
            if (cta != c_last) {
#pragma unroll
              for (int b = 0; b < MAXB; ++b)
                if (b < p.B) st_relaxed(pw + (cta * p.B + b) * kRowBlock + row, ~__float_as_uint(tot[b]));
            } else {
#pragma unroll
              for (int b = 0; b < MAXB; ++b)
                if (b < p.B) p.partial[(cta * p.B + b) * kRowBlock + row] = tot[b];
              keep_rb = crb;
            }
          } else {
            // grids larger than the SM count: the last piece to arrive sums (acq_rel
            // counter; the x pass zeroes the counters)
#pragma unroll
            for (int b = 0; b < MAXB; ++b)
              if (b < p.B) __stcg(&p.partial[((crb + cta) * p.B + b) * kRowBlock + row], tot[b]);
            named_sync(2, 128);
            if (et == 0) {
              // releases this CTA's partial stores (ordered before by the barrier),
              // acquires the other pieces' stores when we are last
              unsigned old;
              asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.counters + crb) : "memory");
              const int last = old == (unsigned)(npieces - 1);
              if (last) p.counters[crb] = 0u;   // all pieces arrived: reset for the next call
              *flag = last;
            }
            named_sync(2, 128);
            if (*flag) {
              for (int b = 0; b < p.B; ++b) {
                float v = 0.f;
                for (int qq = 0; qq < npieces; ++qq) {
                  v += __ldcg(&p.partial[((crb + c_first + qq) * p.B + b) * kRowBlock + row]);
                }
                if (grow < g.M) {
                  if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = v;
                  else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(v);
                }
              }
            }
            named_sync(2, 128);
          }
        }
#pragma unroll
        for (int b = 0; b < MAXB; ++b) tot[b] = 0.f;
        if (kTrace && p.trace && et == 0) p.trace[cta * 256 + 56] = gtime();
      }
      crb = nrb;
      cli = nli;
      cn = nn;
    }
    if (!OWQ_SUMMER_LOW && keep_rb >= 0) {
      // summer of its first row-block: add the lower pieces in CTA order, then its own
      int64_t c_first, c_last;
      pieces(keep_rb, c_first, c_last);
      uint32_t* pw = p.slots;
      float v[MAXB];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) v[b] = 0.f;
      for (int64_t c = c_first; c < c_last; ++c) {
        // all batch rows of piece c in flight at once, then wait for the late ones
        // (one row at a time costs a round trip per row: +3 us at B = 8)
        uint32_t w[MAXB];
#pragma unroll
        for (int b = 0; b < MAXB; ++b) w[b] = b < p.B ? ld_relaxed(pw + (c * p.B + b) * kRowBlock + row) : 1u;
#pragma unroll
        for (int b = 0; b < MAXB; ++b)
          if (b < p.B) {
            uint32_t* a = pw + (c * p.B + b) * kRowBlock + row;
            while (w[b] == 0u) {
              __nanosleep(32);
              w[b] = ld_relaxed(a);
            }
            st_relaxed(a, 0u);
            v[b] += __uint_as_float(~w[b]);
          }
      }
      const int64_t grow = keep_rb * kRowBlock + row;
      if (grow < g.M) {
#pragma unroll
        for (int b = 0; b < MAXB; ++b)
          if (b < p.B) {
            const float r = v[b] + p.partial[(cta * p.B + b) * kRowBlock + row];
            if (p.y_f32) reinterpret_cast<float*>(p.y)[(int64_t)b * g.M + grow] = r;
            else reinterpret_cast<__half*>(p.y)[(int64_t)b * g.M + grow] = __float2half_rn(r);
          }
      }
    }
    if (kTrace && p.trace && et == 0) {
      p.trace[cta * 256 + 53] = (unsigned long long)e_ring;
      p.trace[cta * 256 + 54] = (unsigned long long)e_dfull;
      p.trace[cta * 256 + 55] = (unsigned long long)e_ld;
      p.trace[cta * 256 + 57] = (unsigned long long)e_comb;
    }
  }
  // teardown: every role is done with TMEM
  tc_fence_before();
  __syncthreads();
  if (warp == C::kProdWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
  }
  if (kTrace && p.trace && threadIdx.x == 0) p.trace[cta * 256 + 62] = gtime();
}

// Device inverse of the code layout (test hook): one CTA (128 threads = rows) per
// (row-block, super-step).
__global__ void owq_unpack_codes_kernel(const uint8_t* blob, Geo g, uint8_t* codes) {
  const int64_t item = blockIdx.x;
  const int rb = (int)(item / g.nss), ss = (int)(item % g.nss);
  const int rr = threadIdx.x;
  const int64_t row = (int64_t)rb * kRowBlock + rr;
  if (row >= g.M) return;
  const uint8_t* rec = blob + g.units_off + (int64_t)rb * g.rb_bytes + (int64_t)ss * g.ss_bytes;
  uint32_t w[8];
  for (int i = 0; i < words_per_row(g.bits); ++i) w[i] = *reinterpret_cast<const uint32_t*>(rec + row_word_byte(g.bits, rr, i));
  for (int cc = 0; cc < kSuperStep; ++cc) {
    const int64_t col = (int64_t)ss * kSuperStep + cc;
    if (col >= g.K) continue;
    uint32_t c = 0;
    for (int bit = 0; bit < g.bits; ++bit) {
      int word, pos;
      code_bit_loc(g.bits, cc, bit, word, pos);
      c |= ((w[word] >> pos) & 1u) << bit;
    }
    codes[row * g.K + col] = (uint8_t)c;
  }
}

// ---------------------------------------------------------------- host side
static int device_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) return 148;
  return sms;
}

// Grid: one CTA per SM by default, capped so that every CTA's byte window
// (T / grid) is at least the largest item -- then no CTA is empty and the
// pieces of a row-block are exactly the CTAs cta_of(first) .. cta_of(last).
static int64_t grid_for(const Geo& g, int grid) {
  int64_t G = grid > 0 ? grid : device_sms();
  const int64_t T = (int64_t)g.nrb * g.rb_bytes;
  const int64_t maxitem = std::max<int64_t>(g.ss_bytes, kWeakChunkBytes);
  const int64_t cap = std::max<int64_t>(1, T / maxitem);
  return G < cap ? G : cap;
}

// ---- blob registry: which layout a device blob holds, verified once ------------
// owq_pack registers the blobs it writes; any other blob pointer is verified
// once by reading its header (one device -> host copy on the call's stream),
// then remembered.  Keyed by (pointer, shape): a pointer reused for a blob of
// another shape misses and is re-read.  Unbounded (one entry per packed layer;
// OPT-175B has 576), process-wide, mutex-protected.
struct RegKey {
  const void* p;
  owq_shape s;
  bool operator==(const RegKey& o) const { return p == o.p && !std::memcmp(&s, &o.s, sizeof(owq_shape)); }
};
struct RegHash {
  size_t operator()(const RegKey& k) const {
    size_t h = std::hash<const void*>()(k.p);
    const int32_t* v = &k.s.c_out;
    for (int i = 0; i < 5; ++i) h = h * 1000003u ^ (size_t)(uint32_t)v[i];
    return h;
  }
};
static std::mutex g_reg_mu;
struct RegVal { int layout, Ks; };   // Ks: stored columns of a column-mapped layout-4 blob, else -1
static std::unordered_map<RegKey, RegVal, RegHash> g_reg;

void register_blob(const owq_shape* s, const void* d_packed, int layout, int Ks = -1) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_reg[RegKey{d_packed, *s}] = RegVal{layout, Ks};
}

// Layout of a device blob that must hold `s`: 3 or 4, or an error status (< 0 never: see out).
static owq_status blob_layout(const owq_shape* s, const void* d_packed, cudaStream_t stream, int& layout, int& Ks) {
  if (!s || !d_packed) return OWQ_ERR_INVALID_ARG;
  if (owq_packed_bytes(s) == 0) return OWQ_ERR_UNSUPPORTED;
  if (reinterpret_cast<uintptr_t>(d_packed) & 15) return OWQ_ERR_INVALID_ARG;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = g_reg.find(RegKey{d_packed, *s});
    if (it != g_reg.end()) { layout = it->second.layout; Ks = it->second.Ks; return OWQ_OK; }
  }
  uint8_t hb[128];   // >= sizeof either header struct
  if (cudaMemcpyAsync(hb, d_packed, sizeof(hb), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess)
    return OWQ_ERR_CUDA;
  uint32_t mv[2];
  std::memcpy(mv, hb, 8);
  if (mv[0] == kMagic && mv[1] == OWQ_LAYOUT_VERSION) {
    BlobHeader h;
    std::memcpy(&h, hb, sizeof(h));
    if (h.M != s->c_out || h.K != s->c_in || h.bits != s->bits || h.group != s->group_size || h.k != s->n_weak)
      return OWQ_ERR_BAD_BLOB;
    layout = OWQ_LAYOUT_VERSION;
  } else if (mv[0] == cc::kMagic && mv[1] == (uint32_t)OWQ_LAYOUT_CC) {
    cc::BlobHeader h;
    std::memcpy(&h, hb, sizeof(h));
    if (h.M != s->c_out || h.K != s->c_in || h.bits != s->bits || h.group != s->group_size || h.k != s->n_weak)
      return OWQ_ERR_BAD_BLOB;
    if (h.mapped && (h.Ks <= 0 || h.Ks > h.K)) return OWQ_ERR_BAD_BLOB;
    layout = OWQ_LAYOUT_CC;
    Ks = h.mapped ? h.Ks : -1;
  } else {
    return OWQ_ERR_BAD_BLOB;
  }
  if (layout != OWQ_LAYOUT_CC) Ks = -1;
  register_blob(s, d_packed, layout, Ks);
  return OWQ_OK;
}

// Workspace: [counters nrb u32][partials (nrb + grid) x B x 128 f32]
//            [x digit tiles nss x NN x 64 B][x digit sums nss x Bp x 8 B]
// Fixed-size prefix shared by every shape: one partial-row slot per (CTA, batch
// row) for the co-resident fixup's zero-word protocol (zero = not written yet;
// every call leaves it zero), so calls of other shapes never put data there.
static size_t ws_sync() { return (size_t)kMaxGrid * OWQ_MAX_BATCH * kRowBlock * 4; }
static size_t ws_counters(const Geo& g) { return ((size_t)g.nrb * 4 + 255) / 256 * 256; }
static size_t ws_partials(const Geo& g, int B, int64_t G) {
  return ((size_t)(g.nrb + G) * B * kRowBlock * 4 + 255) / 256 * 256;
}
static size_t ws_tiles(const Geo& g, int B) { return (size_t)g.nss * mma_n_for(B) * kSuperStep; }
static size_t ws_sums(const Geo& g, int B) { return (size_t)g.nss * batch_pad(B) * 8; }
static size_t ws_xpad(const Geo& g, int B) { return ((size_t)B * g.nss * kSuperStep * 2 + 255) / 256 * 256; }
static size_t ws_bytes_for(const Geo& g, int B, int64_t G) {
  return ws_sync() + ws_counters(g) + ws_partials(g, B, G) + ws_tiles(g, B) + ws_sums(g, B) + ws_xpad(g, B);
}

static unsigned long long* g_trace_buf = nullptr;   // experiments only (OWQ_TRACE)
static int64_t g_trace_grid = 0;

template <int BITS, int NN, int DWG, bool GRP = false>
static owq_status launch(const Params& p0, int64_t grid, cudaStream_t stream) {
  using C = Cfg<BITS, NN, DWG, GRP>;
  Params p = p0;
  const int64_t tile_bytes = (int64_t)NN * kSuperStep;
  int dev = 0, maxsmem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // x at the weak columns, the S reduction buffer, barriers + stage descriptors
  const size_t fixed = (((size_t)p.B * p.g.kpad + 7) & ~(size_t)7) * 2 + 2 * 4 * OWQ_MAX_BATCH * 8 + 512;
  const int64_t avail = (int64_t)maxsmem - (int64_t)fixed - 1024;
  // items per warpgroup per stage: fill the TMEM A buffers, but keep >= 4 stages
  const int64_t per_item = std::max<int64_t>(p.g.ss_bytes, kWeakChunkBytes) + tile_bytes +
                           0;
  static const int ipw_env = knob("OWQ_IPW", 0);
  int ipw = ipw_env > 0 && ipw_env < C::kIPW ? ipw_env : C::kIPW;
  while (ipw > 1 && 4 * (C::DWG * ipw * per_item + 2048) > avail) --ipw;
  p.cap = C::DWG * ipw;
  p.code_bytes = (int32_t)std::max<int64_t>((int64_t)p.cap * p.g.ss_bytes, (int64_t)p.cap * kWeakChunkBytes);
  p.tile_off = p.code_bytes;
  p.sum_off = p.tile_off + (int32_t)(p.cap * tile_bytes);
  p.gstage = (C::kGP > 1 && p.g.group) ? 1 : 0;
  p.x_off = p.sum_off + (int32_t)((p.gstage ? p.cap * p.Bp * 8 : 0) + 127) / 128 * 128;
  p.sz_off = p.x_off;
  const int sz_blocks = p.gstage ? (int)(p.cap * kSuperStep / p.g.group + 2) : 0;
  p.stage_bytes = (int32_t)((p.sz_off + sz_blocks * kSZBlockBytes + 127) / 128 * 128);
  int nst = (int)(avail / (p.stage_bytes + 32));
  static const int max_nst = knob("OWQ_NST", 8);
  nst = std::min(nst, max_nst);
  if (nst < 2) return OWQ_ERR_UNSUPPORTED;     // too many weak columns / batch rows for shared memory
  p.nst = nst;
  const size_t smem = (size_t)nst * p.stage_bytes + fixed + (size_t)nst * 32;
  auto kern = owq_gemv_kernel<BITS, NN, DWG, GRP>;
  // the attribute is per device: one record per device, atomically raised
  static std::atomic<size_t> configured[32];
  if (configured[dev & 31].load() < smem) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return OWQ_ERR_CUDA;
    size_t cur = configured[dev & 31].load();
    while (cur < smem && !configured[dev & 31].compare_exchange_weak(cur, smem)) {}
  }
  static const int pdl = knob("OWQ_PDL", 2);   // 0 off, 1 GEMV, 2 both
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl >= 1 ? 1 : 0;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "owq: launch of owq_gemv_kernel<%d,%d,%d> (grid %lld, smem %zu) failed: %s\n", BITS, NN, DWG,
            (long long)grid, smem, cudaGetErrorString(e));
    return OWQ_ERR_CUDA;
  }
  return OWQ_OK;
}

template <int BITS>
static owq_status launch_n(const Params& p, int64_t grid, cudaStream_t cs) {
  static const int dwg = knob("OWQ_DWG", 0);   // B = 1 only
  switch (mma_n_for(p.B)) {
    case 8:   // batch 1: 2 decode warpgroups x 6 items measured best (fewer TMEM stores racing the MMAs)
      if (dwg == 3) return launch<BITS, 8, 3>(p, grid, cs);
      if (dwg == 4) return launch<BITS, 8, 4>(p, grid, cs);
      if (p.g.group) return launch<BITS, 8, 2, true>(p, grid, cs);   // grouped scales: per-stage D blocks
      return launch<BITS, 8, 2>(p, grid, cs);
    case 16: return launch<BITS, 16, 3>(p, grid, cs);
    case 32: return launch<BITS, 32, 3>(p, grid, cs);
    case 64: return launch<BITS, 64, 2>(p, grid, cs);
    default: return launch<BITS, 96, 2>(p, grid, cs);
  }
}

static owq_status gemm_impl(const owq_shape* s, const void* d_packed, const uint16_t* d_x, int B, void* d_y,
                            int y_f32, void* d_ws, size_t ws_bytes, int grid_req, void* stream) {
  if (!d_x || !d_y || !d_ws) return OWQ_ERR_INVALID_ARG;
  if (B < 1 || B > OWQ_MAX_BATCH) return OWQ_ERR_UNSUPPORTED;
  int layout = 0, Ks = -1;
  owq_status st = blob_layout(s, d_packed, (cudaStream_t)stream, layout, Ks);
  if (st != OWQ_OK) return st;
  if (layout == OWQ_LAYOUT_CC)
    return cc::gemm(cc::make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak, Ks), d_packed, d_x, B, d_y,
                    y_f32, d_ws, ws_bytes, grid_req, (cudaStream_t)stream);
  const Geo g = make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak);
  // Grouped scales at B >= 4: the fp16-A batch kernel is faster (DESIGN.md §6.5:
  // LLaMA-7B up g128 B = 8 27.5 vs 57 us); an explicit grid request keeps this kernel.
  if (grid_req == 0 && g.group && B >= 4 && !(s->c_in & 7) && !(reinterpret_cast<uintptr_t>(d_x) & 15) &&
      ws_bytes >= ws_sync()) {
    const owq_status r = pf::sb::launch(g, d_packed, d_x, B, d_y, y_f32, (uint8_t*)d_ws + ws_sync(),
                                        ws_bytes - ws_sync(), device_sms(), (cudaStream_t)stream);
    if (r == OWQ_OK || r == OWQ_ERR_CUDA) return r;   // else (unsupported group / workspace): this kernel
  }
  const int64_t grid = grid_for(g, grid_req);
  if (grid > kMaxGrid || (int64_t)g.nrb * items_per_rb(g) >= (1ll << 31)) return OWQ_ERR_UNSUPPORTED;
  if (ws_bytes < ws_bytes_for(g, B, grid)) return OWQ_ERR_BUFFER_TOO_SMALL;
  Params p{};
  p.blob = (const uint8_t*)d_packed;
  p.x = (const __half*)d_x;
  p.y = d_y;
  p.slots = (uint32_t*)d_ws;
  p.counters = (uint32_t*)((uint8_t*)d_ws + ws_sync());
  p.partial = (float*)((uint8_t*)d_ws + ws_sync() + ws_counters(g));
  uint8_t* tiles = (uint8_t*)d_ws + ws_sync() + ws_counters(g) + ws_partials(g, B, grid);
  long long* sums = (long long*)(tiles + ws_tiles(g, B));
  p.tiles = tiles;
  p.sums = sums;
  p.g = g;
  {
    // Stream-K span table and row-block piece table of this (geometry, grid): a
    // few recent ones are kept per host thread (the tables are pure functions of
    // them and cost microseconds to rebuild on every call).
    struct SpanCache {
      int64_t key[4];
      int32_t span[kMaxGrid + 1];
      uint64_t fix[kMaxGrid];
    };
    static thread_local SpanCache cache[8];
    static thread_local int cache_n = 0, cache_next = 0;
    const int64_t key[4] = {g.nrb, g.rb_bytes, ((int64_t)g.nss << 32) | (int64_t)g.kpad, ((int64_t)g.ss_bytes << 32) | grid};
    int hit = -1;
    for (int i = 0; i < cache_n && hit < 0; ++i)
      if (!std::memcmp(cache[i].key, key, sizeof(key))) hit = i;
    if (hit < 0) {
      // CTA c's share of the bytes ~ 1 + a (1/2 - c/G).  In a chain of calls the
      // CTAs of a call start as the previous call's CTAs leave their SMs, in CTA
      // order, over several microseconds, and a late starter has had less time to
      // fill its ring before x is readable: giving the high
      // indices less work evens the finish.  a ~ 88 KB / (bytes per CTA), i.e.
      // ~2 us of one SM's HBM share, capped at 0.3 (measured: 12288^2 -7 %,
      // 49152 x 12288 -2 %; a reversed skew is slower).
      const double T = (double)g.nrb * g.rb_bytes;
      static const int skew_env = knob("OWQ_SKEW", -1);   // experiments: a = OWQ_SKEW / 100
      const int64_t n_items = (int64_t)g.nrb * items_per_rb(g);
      // only with >= 8 items per CTA; spans stay non-empty (the fixup's summer
      // waits on every CTA between a row-block's first and last piece)
      const double a = n_items < 8 * grid ? 0.0
                       : skew_env >= 0 ? skew_env / 100.0 : std::min(0.3, 88.0 * 1024.0 * grid / T);
      if (a <= 0.0) {
        for (int64_t c = 0; c <= grid; ++c) p.span[c] = (int32_t)cta_first_item(g, grid, c);
      } else {
        for (int64_t c = 0; c <= grid; ++c) {
          const double xx = (double)c / grid, F = xx + 0.5 * a * (xx - xx * xx);
          p.span[c] = c == grid ? (int32_t)cta_first_item(g, grid, c) : (int32_t)first_item_at(g, (int64_t)std::ceil(T * F));
        }
        for (int64_t c = 1; c < grid; ++c) p.span[c] = std::max(p.span[c], p.span[c - 1] + 1);
        for (int64_t c = grid - 1; c >= 1; --c) p.span[c] = std::min(p.span[c], p.span[c + 1] - 1);
      }
      {  // row-block pieces at each CTA's ends (the fixup's summer and piece count)
        const int64_t n_rb = items_per_rb(g);
        auto cta_of = [&](int64_t item) {   // span[c] <= item < span[c + 1]
          int64_t lo = 0, hi = grid;
          while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (p.span[mid] <= item) lo = mid; else hi = mid;
          }
          return (uint64_t)lo;
        };
        for (int64_t c = 0; c < grid; ++c) {
          const int64_t i0 = p.span[c], i1 = p.span[c + 1];
          if (i1 <= i0) { p.fix[c] = (uint64_t)c * 0x0001000100010001ull; continue; }
          const int64_t ra = i0 / n_rb, rbb = (i1 - 1) / n_rb;
          p.fix[c] = cta_of(ra * n_rb) | (cta_of(ra * n_rb + n_rb - 1) << 16) | (cta_of(rbb * n_rb) << 32) |
                     (cta_of(rbb * n_rb + n_rb - 1) << 48);
        }
      }
      hit = cache_next;
      cache_next = (cache_next + 1) % 8;
      if (cache_n < 8) ++cache_n;
      std::memcpy(cache[hit].key, key, sizeof(key));
      std::memcpy(cache[hit].span, p.span, sizeof(int32_t) * (grid + 1));
      std::memcpy(cache[hit].fix, p.fix, sizeof(uint64_t) * grid);
    } else {
      std::memcpy(p.span, cache[hit].span, sizeof(int32_t) * (grid + 1));
      std::memcpy(p.fix, cache[hit].fix, sizeof(uint64_t) * grid);
    }
  }
  p.coresident = grid <= device_sms() ? 1 : 0;   // one CTA per SM: every CTA is resident at once
  static const int force_counter = knob("OWQ_FORCE_COUNTER", 0);   // experiments: the counter fixup for every grid
  if (force_counter) p.coresident = 0;
  p.B = B;
  p.Bp = batch_pad(B);
  p.y_f32 = y_f32 ? 1 : 0;
  p.xK = g.K;
  cudaStream_t cs = (cudaStream_t)stream;
  // x -> exact int8 digits in UMMA tile order, plus per-super-step digit sums
  static const int skip = knob("OWQ_SKIP", 0);   // 1 no digit pass, 2 no GEMV (timing experiments)
  if (skip != 1) {
    static const int pdl = knob("OWQ_PDL", 2);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl >= 2 ? 1 : 0;
    // the stream-K counters (used by grids larger than the SM count) start at zero
    const int64_t nzero = grid > device_sms() ? (int64_t)ws_counters(g) / 16 : 0;
    const int64_t zctas = (nzero + 1023) / 1024;
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(g.nss, std::min<int64_t>(zctas, 1024)));
    cfg.blockDim = dim3((unsigned)(64 * p.Bp));
    cfg.stream = cs;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, owq_x_digits_kernel, (const __half*)p.x, (int64_t)p.xK, B, (int)p.Bp, (int)g.K,
                       mma_n_for(B), tiles, (long long*)sums, (int)g.nss, (uint4*)p.counters, nzero);
    if (cudaGetLastError() != cudaSuccess) return OWQ_ERR_CUDA;
  }
  // experiments only: OWQ_TRACE=<file> appends each call's per-CTA stamps to the
  // file; with OWQ_TRACE_DEFER set, calls only record (graph-capturable) and
  // owq_debug_trace_dump() writes the last launch's stamps.
#ifdef OWQ_EXPERIMENTS
  static const char* trace_path = getenv("OWQ_TRACE");
  static const bool trace_defer = getenv("OWQ_TRACE_DEFER") != nullptr;
#else
  static const char* trace_path = nullptr;
  static const bool trace_defer = false;
#endif
  if (trace_path && !g_trace_buf) {
    cudaMalloc(&g_trace_buf, 4096 * 256 * 8);
    cudaMemset(g_trace_buf, 0, 4096 * 256 * 8);
  }
  unsigned long long* trace_buf = trace_defer ? nullptr : g_trace_buf;
  if (trace_buf) cudaMemsetAsync(trace_buf, 0, 4096 * 256 * 8, cs);
  p.trace = g_trace_buf;
  g_trace_grid = grid;
  static const int exp_env = knob("OWQ_EXP", 0);
  p.exp = exp_env;

  p.group_log2 = 0;
  if (g.group) while ((kSuperStep << p.group_log2) < g.group) ++p.group_log2;
  const owq_status rs = skip == 2 ? OWQ_OK : (g.bits == 3 ? launch_n<3>(p, grid, cs) : launch_n<4>(p, grid, cs));
  if (trace_buf && rs == OWQ_OK) {   // experiments only: dump the per-CTA stamps
    std::vector<unsigned long long> h((size_t)grid * 256);
    cudaMemcpyAsync(h.data(), trace_buf, h.size() * 8, cudaMemcpyDeviceToHost, cs);
    cudaStreamSynchronize(cs);
    if (FILE* f = fopen(trace_path, "ab")) { fwrite(h.data(), 8, h.size(), f); fclose(f); }
  }
  return rs;
}

}  // namespace owq

// experiments only (not part of the C ABI in include/owq.h): write the stamps
// of the last traced launch (OWQ_TRACE + OWQ_TRACE_DEFER) to `path`.
extern "C" int owq_debug_trace_dump(const char* path) {
  if (!owq::g_trace_buf) return -1;
  std::vector<unsigned long long> h((size_t)owq::g_trace_grid * 256);
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  cudaMemcpy(h.data(), owq::g_trace_buf, h.size() * 8, cudaMemcpyDeviceToHost);
  FILE* f = fopen(path, "wb");
  if (!f) return -3;
  fwrite(h.data(), 8, h.size(), f);
  fclose(f);
  return 0;
}

using namespace owq;

extern "C" {

owq_status owq_pack(const owq_shape* s, const owq_host_layer* L, int flags, void* d_packed, size_t d_bytes,
                    void* stream) {
  if (!d_packed) return OWQ_ERR_INVALID_ARG;
  const int layout = (flags & OWQ_PACK_LAYOUT_CC) ? OWQ_LAYOUT_CC : OWQ_LAYOUT_VERSION;
  const size_t n = owq_packed_bytes_layout(s, layout);
  if (n == 0) return OWQ_ERR_UNSUPPORTED;
  if (d_bytes < n) return OWQ_ERR_BUFFER_TOO_SMALL;
  if (reinterpret_cast<uintptr_t>(d_packed) & 15) return OWQ_ERR_INVALID_ARG;
  std::vector<uint8_t> host(n);
  owq_status st = owq_pack_host(s, L, flags, host.data(), n);
  if (st != OWQ_OK) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  if (cudaMemcpyAsync(d_packed, host.data(), n, cudaMemcpyHostToDevice, cs) != cudaSuccess) return OWQ_ERR_CUDA;
  if (cudaStreamSynchronize(cs) != cudaSuccess) return OWQ_ERR_CUDA;
  register_blob(s, d_packed, layout);
  return OWQ_OK;
}

owq_status owq_pack_colmap(const owq_shape* s, const owq_host_layer* L, const owq_colmap* map, int flags,
                           void* d_packed, size_t d_bytes, void* stream) {
  if (!d_packed) return OWQ_ERR_INVALID_ARG;
  const size_t n = owq_packed_bytes_colmap(s, map);
  if (n == 0) return OWQ_ERR_INVALID_ARG;
  if (d_bytes < n) return OWQ_ERR_BUFFER_TOO_SMALL;
  if (reinterpret_cast<uintptr_t>(d_packed) & 15) return OWQ_ERR_INVALID_ARG;
  std::vector<uint8_t> host(n);
  owq_status st = owq_pack_host_colmap(s, L, map, flags, host.data(), n);
  if (st != OWQ_OK) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  if (cudaMemcpyAsync(d_packed, host.data(), n, cudaMemcpyHostToDevice, cs) != cudaSuccess) return OWQ_ERR_CUDA;
  if (cudaStreamSynchronize(cs) != cudaSuccess) return OWQ_ERR_CUDA;
  register_blob(s, d_packed, OWQ_LAYOUT_CC, map->k_stored);
  return OWQ_OK;
}

owq_status owq_unpack_codes(const owq_shape* s, const void* d_packed, uint8_t* d_codes, void* stream) {
  if (!d_codes) return OWQ_ERR_INVALID_ARG;
  int layout = 0, Ks = -1;
  owq_status st = blob_layout(s, d_packed, (cudaStream_t)stream, layout, Ks);
  if (st != OWQ_OK) return st;
  if (layout == OWQ_LAYOUT_CC)
    return cc::unpack(cc::make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak, Ks), d_packed, d_codes,
                      (cudaStream_t)stream);
  const Geo g = make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak);
  owq_unpack_codes_kernel<<<(unsigned)((int64_t)g.nrb * g.nss), kRowBlock, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)d_packed, g, d_codes);
  return cudaGetLastError() == cudaSuccess ? OWQ_OK : OWQ_ERR_CUDA;
}

size_t owq_workspace_bytes_grid(const owq_shape* s, int batch, int grid) {
  if (owq_packed_bytes(s) == 0 || batch < 1 || batch > OWQ_MAX_BATCH || grid < 0) return 0;
  const Geo g = make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak);
  // an upper bound for any n_weak: the requested grid before the per-shape cap
  const int64_t G = grid > 0 ? grid : device_sms();
  if (G > 1024) return 0;   // the CUDA-core kernel's limit (the tcgen05 kernel's is 512)
  // one workspace serves either layout of the layer and the small-batch f16 kernel
  const size_t sbw = ws_sync() + pf::sb::workspace_bytes(g, 32, device_sms());   // any batch <= 32
  const size_t v3 = G <= kMaxGrid ? ws_bytes_for(g, batch, G) : 0;
  return std::max(std::max(v3, cc::workspace_bytes((int)G, std::min(batch, 4))), sbw);
}

size_t owq_workspace_bytes(const owq_shape* s, int batch) { return owq_workspace_bytes_grid(s, batch, 0); }

owq_status owq_gemv(const owq_shape* s, const void* d_packed, const uint16_t* d_x, void* d_y, int y_f32, void* d_ws,
                    size_t ws_bytes, void* stream) {
  return gemm_impl(s, d_packed, d_x, 1, d_y, y_f32, d_ws, ws_bytes, 0, stream);
}

owq_status owq_gemm_small_batch(const owq_shape* s, const void* d_packed, const uint16_t* d_x, int batch, void* d_y,
                                int y_f32, void* d_ws, size_t ws_bytes, void* stream) {
  return gemm_impl(s, d_packed, d_x, batch, d_y, y_f32, d_ws, ws_bytes, 0, stream);
}

owq_status owq_gemm_batch_f16(const owq_shape* s, const void* d_packed, const uint16_t* d_x, int batch, void* d_y,
                              int y_f32, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_x || !d_y || !d_ws) return OWQ_ERR_INVALID_ARG;
  if (batch < 1 || batch > 32) return OWQ_ERR_UNSUPPORTED;
  int layout = 0, Ks = -1;
  owq_status st = blob_layout(s, d_packed, (cudaStream_t)stream, layout, Ks);
  if (st != OWQ_OK) return st;
  if (layout != OWQ_LAYOUT_VERSION || (s->c_in & 7)) return OWQ_ERR_UNSUPPORTED;
  if (reinterpret_cast<uintptr_t>(d_x) & 15) return OWQ_ERR_INVALID_ARG;
  if (ws_bytes < ws_sync()) return OWQ_ERR_BUFFER_TOO_SMALL;
  return pf::sb::launch(make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak), d_packed, d_x, batch, d_y, y_f32,
                        (uint8_t*)d_ws + ws_sync(), ws_bytes - ws_sync(), device_sms(), (cudaStream_t)stream);
}

static owq_status prefill_impl(const owq_shape* s, const void* d_packed, const uint16_t* d_x, int32_t n_tokens,
                               void* d_y, int y_f32, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_x || !d_y) return OWQ_ERR_INVALID_ARG;
  if (n_tokens < 1) return OWQ_ERR_INVALID_ARG;
  int layout = 0, Ks = -1;
  owq_status st = blob_layout(s, d_packed, (cudaStream_t)stream, layout, Ks);
  if (st != OWQ_OK) return st;
  if (layout != OWQ_LAYOUT_VERSION || s->group_size != 0 || (s->c_in & 7)) return OWQ_ERR_UNSUPPORTED;
  if (reinterpret_cast<uintptr_t>(d_x) & 15) return OWQ_ERR_INVALID_ARG;
  if (d_ws && (reinterpret_cast<uintptr_t>(d_ws) & 15)) return OWQ_ERR_INVALID_ARG;
  return pf::launch(make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak), d_packed, d_x, n_tokens, d_y, y_f32,
                    d_ws, d_ws ? ws_bytes : 0, (cudaStream_t)stream);
}

owq_status owq_gemm_prefill(const owq_shape* s, const void* d_packed, const uint16_t* d_x, int32_t n_tokens, void* d_y,
                            int y_f32, void* stream) {
  return prefill_impl(s, d_packed, d_x, n_tokens, d_y, y_f32, nullptr, 0, stream);
}

owq_status owq_gemm_prefill_ws(const owq_shape* s, const void* d_packed, const uint16_t* d_x, int32_t n_tokens,
                               void* d_y, int y_f32, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_ws && ws_bytes) return OWQ_ERR_INVALID_ARG;
  return prefill_impl(s, d_packed, d_x, n_tokens, d_y, y_f32, d_ws, ws_bytes, stream);
}

size_t owq_prefill_workspace_bytes(const owq_shape* s, int32_t n_tokens) {
  if (owq_packed_bytes(s) == 0 || n_tokens < 1) return 0;
  return pf::workspace_bytes(make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak), n_tokens);
}

owq_status owq_gemm_small_batch_grid(const owq_shape* s, const void* d_packed, const uint16_t* d_x, int batch,
                                     void* d_y, int y_f32, void* d_ws, size_t ws_bytes, int grid, void* stream) {
  if (grid < 0) return OWQ_ERR_INVALID_ARG;
  return gemm_impl(s, d_packed, d_x, batch, d_y, y_f32, d_ws, ws_bytes, grid, stream);
}

}  // extern "C"
