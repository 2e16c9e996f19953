// owq_layout_cc.h -- device layout version 4 ("cc"): the packed OWQ blob read by
// the CUDA-core GEMV (owq_gemv_cc.cu).  Shared by the host packer and the kernel.
//
// Arithmetic it is built for: a code q sitting at bits
// [p, p+b) of a 32-bit word w, with p + b <= 24, is isolated by ONE LOP3,
// m = w & (2^b - 1) << p, and m read as an fp32 bit pattern is the subnormal
// q * 2^(p-149) (patterns < 2^24 are linear in fp32: exponent field 0 or 1).
// Multiplying it by x' = x * 2^(111-p) gives q * x * 2^-38 EXACTLY (<= 4 + 11
// significant bits), two columns per FFMA2.  The zero point is factored out of
// the sum (s * (sum q x - z * sum x), reading s19), so the inner loop is one
// LOP3 per code plus half an FFMA2.
//
// Row-blocks of 128 output rows; steps of 32 columns.  One step of one row-block
// = one "item" = W words x 32 lanes x 4 rows (W = 3 at 3 bits, 4 at 4 bits):
//   u32 at item + (c * 32 + lane) * 16 + r * 4  = word c of row 4 * lane + r
// so lane `lane` of a warp reads its 4 rows' word c with one conflict-free
// LDS.128.  Inside a row's step (columns j = 0..31 of the step):
//   3-bit: j < 24 -> word j / 8, bits 3 (j % 8) ..;  j >= 24 -> the word t
//          assembled from the top bytes, t = {w0.b3, w1.b3, w2.b3, 0}, bits
//          3 (j - 24) ..  (t bit i = word i / 8, bit 24 + i % 8).
//   4-bit: j < 24 -> word j / 6, bits 4 (j % 6) ..;  24 <= j < 30 -> t1 =
//          {w0.b3, w1.b3, w2.b3, 0}, bits 4 (j - 24); j = 30, 31 -> t2 = {w3.b3},
//          bits 4 (j - 30).
// The code's bit offset inside its register is p(j) = 3 (j % 8) at 3 bits and
// 4 (j % 6 for j < 24, j - 24 for j < 30, j - 30) at 4 bits (cc_pos below).
//
// Regions after the 256-byte header:
//   units   [nrb][nsteps] items
//   sz      [nrb][G][128] (scale, zero) fp16 pairs (row-block-major)
//   weak    [nrb][kpad/8][128 rows][8] fp16 weak values (zero-padded to 8)
//   widx    [kpad] u16 weak-column indices (zero-padded)
//   wmask   [nsteps] u32, bit j of word s = stored column 32 s + j is weak
//   colmap  [nsteps * 32] u16 (only when Ks-mapped): original column
//           of each stored position (act-order / storage-favored variants,
//           P:411-412); without it stored position = original column.
// Ks = stored columns (K without a map); steps, groups and the weak mask run
// over stored positions; x and the weak indices keep the original K columns.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define OWQ_CC_HD __host__ __device__ __forceinline__
#else
#define OWQ_CC_HD inline
#endif

namespace owq {
namespace cc {

constexpr int kVersion = 4;
constexpr int kRowBlock = 128;
constexpr int kStep = 32;                     // columns per item
constexpr int kWeakChunk = 8;
constexpr int kWeakChunkBytes = kRowBlock * kWeakChunk * 2;
constexpr int kHeaderBytes = 256;
constexpr int kSZBlockBytes = kRowBlock * 4;

OWQ_CC_HD int words_per_row(int bits) { return bits == 3 ? 3 : 4; }
OWQ_CC_HD int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Geo {
  int32_t M, K, bits, group, k;
  int32_t nrb, nsteps, kpad, G, W;
  int32_t Ks, mapped;         // stored columns; 1 = a column map is stored
  int64_t item_bytes, rb_code_bytes, weak_rb_bytes;
  int64_t units_off, sz_off, weak_off, widx_off, wmask_off, colmap_off, total;
};

// Ks < 0: no column map (Ks = K).
OWQ_CC_HD Geo make_geo(int32_t M, int32_t K, int32_t bits, int32_t group, int32_t k, int32_t Ks = -1) {
  Geo g{};
  g.M = M; g.K = K; g.bits = bits; g.group = group; g.k = k;
  g.mapped = Ks >= 0 ? 1 : 0;
  g.Ks = Ks >= 0 ? Ks : K;
  g.nrb = (int32_t)cdiv(M, kRowBlock);
  g.nsteps = (int32_t)cdiv(g.Ks, kStep);
  g.kpad = (int32_t)cdiv(k, kWeakChunk) * kWeakChunk;
  g.G = group ? (int32_t)cdiv(g.Ks, group) : 1;
  g.W = words_per_row(bits);
  g.item_bytes = (int64_t)g.W * 32 * 16;
  g.rb_code_bytes = (int64_t)g.nsteps * g.item_bytes;
  g.weak_rb_bytes = (int64_t)(g.kpad / kWeakChunk) * kWeakChunkBytes;
  g.units_off = kHeaderBytes;
  g.sz_off = g.units_off + (int64_t)g.nrb * g.rb_code_bytes;
  g.weak_off = g.sz_off + (int64_t)g.nrb * g.G * kSZBlockBytes;
  g.widx_off = g.weak_off + (int64_t)g.nrb * g.weak_rb_bytes;
  g.wmask_off = g.widx_off + cdiv((int64_t)g.kpad * 2 + 2, 16) * 16;
  g.colmap_off = g.wmask_off + cdiv((int64_t)g.nsteps * 4, 16) * 16;
  g.total = g.colmap_off + (g.mapped ? cdiv((int64_t)g.nsteps * kStep * 2, 16) * 16 : 0);
  return g;
}

// Bit offset of column j (0..31 of a step) inside the register it is read from,
// and which register: 0..W-1 = the stored words, W = t (t1), W + 1 = t2.
OWQ_CC_HD int cc_pos(int bits, int j) {
  if (bits == 3) return 3 * (j & 7);
  if (j < 24) return 4 * (j % 6);
  if (j < 30) return 4 * (j - 24);
  return 4 * (j - 30);
}

// Location of bit `bit` of column j's code: stored word and bit position.
OWQ_CC_HD void cc_bit_loc(int bits, int j, int bit, int& word, int& pos) {
  if (bits == 3) {
    if (j < 24) { word = j >> 3; pos = 3 * (j & 7) + bit; return; }
    const int i = 3 * (j - 24) + bit;        // bit of t
    word = i >> 3; pos = 24 + (i & 7);
    return;
  }
  if (j < 24) { word = j / 6; pos = 4 * (j % 6) + bit; return; }
  if (j < 30) {
    const int i = 4 * (j - 24) + bit;        // bit of t1
    word = i >> 3; pos = 24 + (i & 7);
    return;
  }
  word = 3; pos = 24 + 4 * (j - 30) + bit;   // t2 = w3.b3
}

// Item (rb, step) byte offset relative to units_off.
OWQ_CC_HD int64_t item_offset(const Geo& g, int64_t rb, int64_t step) {
  return rb * g.rb_code_bytes + step * g.item_bytes;
}

// Stream-K work units: per row-block its nsteps code items, then (k > 0) one
// weak unit of weak_rb_bytes.  Units are balanced by bytes: CTA c of `grid`
// owns the units whose start offset lies in [c T / grid, (c + 1) T / grid).
OWQ_CC_HD int64_t units_per_rb(const Geo& g) { return (int64_t)g.nsteps + (g.k > 0 ? 1 : 0); }
OWQ_CC_HD int64_t rb_bytes(const Geo& g) { return g.rb_code_bytes + g.weak_rb_bytes; }

// First unit whose byte offset is >= b.
inline int64_t first_unit_at(const Geo& g, int64_t b) {
  const int64_t R = rb_bytes(g), n = units_per_rb(g);
  int64_t rb = b / R, r = b - rb * R;
  if (rb >= g.nrb) return (int64_t)g.nrb * n;
  int64_t u;
  if (r <= g.rb_code_bytes) u = cdiv(r, g.item_bytes);
  else u = n;                                 // past the weak unit's start -> next row-block
  if (u >= n) { rb += 1; u = 0; }
  return rb * n + u;
}

struct BlobHeader {          // first bytes of the blob (version 4)
  uint32_t magic, version;
  int32_t M, K, bits, group, k;
  int32_t nrb, nsteps, kpad, G, W;
  int64_t total;
  int32_t Ks, mapped;
};
constexpr uint32_t kMagic = 0x4257514Fu;     // same magic as version 3: the version field tells them apart

}  // namespace cc
}  // namespace owq
