// owq_layout.h -- device layout of the packed OWQ blob (layout version 3).
// Shared by the host packer (owq_pack.cpp) and the device kernels (*.cu).
// (Layout version 3: codes positioned for the tcgen05 kind::i8 A operand.)
// DESIGN.md §5 documents the bit map; include/owq.h summarises it.
//
// Row-blocks of 128 output rows (one tcgen05 M=128 tile, one thread per row).
// Per row-block: its super-steps (64 columns each) then its weak chunks.
//   super-step record: every row's 64 codes in WPR 32-bit words (WPR = 6 for
//     3-bit, 8 for 4-bit); words 0..3 of row r at r*16, words 4.. at
//     2048 + r*(WPR-4)*4 -- one LDS.128 (+ one LDS.64/128) per thread, no bank
//     conflicts.  Columns 4c..4c+3 of the super-step become TMEM column c of
//     the thread's row (4 unsigned bytes, byte 0 = column 4c).
//   weak chunk (8 weak columns): [128 rows][8] fp16; the ragged last chunk
//     (k % 8 columns) is [128][k % 8] fp16, unpadded.
// Then: scale/zero blocks [nrb][G][128 rows] of (s, z) fp16 pairs, and the
// u16 weak-column index list.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define OWQ_HD __host__ __device__ __forceinline__
#else
#define OWQ_HD inline
#endif

namespace owq {

constexpr int kRowBlock = 128;       // rows per row-block (tcgen05 M = 128)
constexpr int kSuperStep = 64;       // columns per super-step (4 MMAs of K = 16)
constexpr int kWeakChunk = 8;        // weak columns per chunk
constexpr int kWeakChunkBytes = kRowBlock * kWeakChunk * 2;   // 2 KiB
constexpr int kHeaderBytes = 256;
constexpr int kSZBlockBytes = kRowBlock * 4;                  // 128 x (s, z) fp16 pairs
constexpr uint32_t kMagic = 0x4257514Fu;                      // "OQWB"

// floor(a / b) for 0 <= a < 2^53, b > 0.  On the device a double-precision
// estimate plus an exact integer correction (a 64-bit integer division is a
// ~100-instruction subroutine; this runs in the kernel prologue).
OWQ_HD int64_t fdiv(int64_t a, int64_t b) {
#if defined(__CUDA_ARCH__)
  int64_t q = (int64_t)((double)a / (double)b);
  while (q * b > a) --q;
  while ((q + 1) * b <= a) ++q;
  return q;
#else
  return a / b;
#endif
}
OWQ_HD int64_t cdiv(int64_t a, int64_t b) { return fdiv(a + b - 1, b); }
OWQ_HD int words_per_row(int bits) { return bits == 3 ? 6 : 8; }

struct Geo {
  int32_t M, K, bits, group, k;
  int32_t nrb;       // row-blocks
  int32_t nss;       // super-steps per row
  int32_t kpad;      // k rounded up to a multiple of 8 (gathered-x buffer only)
  int32_t nfull;     // full weak chunks
  int32_t ktail;     // columns of the ragged last chunk (k % 8), stored unpadded
  int32_t tail_bytes;// 128 * ktail * 2
  int32_t G;         // scale/zero groups per row
  int64_t ss_bytes;  // bytes per super-step (all 128 rows)
  int64_t rb_bytes;  // bytes per row-block record (super-steps + weak chunks)
  int64_t units_off, sz_off, widx_off, total;
};

OWQ_HD Geo make_geo(int32_t M, int32_t K, int32_t bits, int32_t group, int32_t k) {
  Geo g{};
  g.M = M; g.K = K; g.bits = bits; g.group = group; g.k = k;
  g.nrb = (int32_t)cdiv(M, kRowBlock);
  g.nss = (int32_t)cdiv(K, kSuperStep);
  g.kpad = (int32_t)cdiv(k, kWeakChunk) * kWeakChunk;
  g.nfull = k / kWeakChunk;
  g.ktail = k % kWeakChunk;
  g.tail_bytes = kRowBlock * g.ktail * 2;
  g.G = group ? (int32_t)cdiv(K, group) : 1;
  g.ss_bytes = (int64_t)kRowBlock * words_per_row(bits) * 4;
  g.rb_bytes = (int64_t)g.nss * g.ss_bytes + (int64_t)g.nfull * kWeakChunkBytes + g.tail_bytes;
  g.units_off = kHeaderBytes;
  g.sz_off = g.units_off + (int64_t)g.nrb * g.rb_bytes;
  g.widx_off = g.sz_off + (int64_t)g.nrb * g.G * kSZBlockBytes;
  g.total = g.widx_off + cdiv((int64_t)g.kpad * 2, 16) * 16;
  if (g.total == g.widx_off) g.total += 16;
  return g;
}

// ---- work items and the byte-balanced stream-K split ---------------------------
// Items, in blob order: per row-block its nss super-steps, then its
// ceil(k/8) weak chunks.  CTA c of `grid` owns the items whose byte offset in
// the units region lies in [c*T/grid, (c+1)*T/grid), T = nrb * rb_bytes, so
// every CTA streams the same number of bytes (+- one item).
OWQ_HD int32_t items_per_rb(const Geo& g) { return g.nss + g.kpad / kWeakChunk; }

OWQ_HD int64_t item_offset(const Geo& g, int64_t rb, int32_t li) {   // relative to units_off
  return rb * g.rb_bytes + (li < g.nss ? (int64_t)li * g.ss_bytes
                                       : (int64_t)g.nss * g.ss_bytes + (int64_t)(li - g.nss) * kWeakChunkBytes);
}

// First item whose offset is >= b (b in [0, T]).
OWQ_HD int64_t first_item_at(const Geo& g, int64_t b) {
  const int32_t n = items_per_rb(g);
  int64_t rb = fdiv(b, g.rb_bytes);
  int64_t r = b - rb * g.rb_bytes;
  if (rb >= g.nrb) return (int64_t)g.nrb * n;
  const int64_t C = (int64_t)g.nss * g.ss_bytes;
  int64_t li;
  if (r <= C) li = cdiv(r, g.ss_bytes);
  else li = g.nss + cdiv(r - C, kWeakChunkBytes);
  if (li >= n) { rb += 1; li = 0; }
  return rb * n + li;
}

OWQ_HD int64_t cta_first_item(const Geo& g, int64_t grid, int64_t c) {
  const int64_t T = (int64_t)g.nrb * g.rb_bytes;
  return first_item_at(g, cdiv(c * T, grid));
}

OWQ_HD int64_t cta_of_item(const Geo& g, int64_t grid, int64_t item) {
  const int32_t n = items_per_rb(g);
  const int64_t rb = fdiv(item, n);
  const int64_t T = (int64_t)g.nrb * g.rb_bytes;
  return fdiv(item_offset(g, rb, (int32_t)(item - rb * n)) * grid, T);
}

// Stage sequence of one CTA: runs of at most `cap` items of one kind (code or
// weak) inside one row-block.  Every role of the CTA walks the same sequence.
struct StageIter {
  int64_t rb;
  int32_t li, n_rb, nss, cap;
  int64_t left;
  OWQ_HD void init(const Geo& g, int64_t first, int64_t last, int32_t cap_) {
    n_rb = items_per_rb(g); nss = g.nss; cap = cap_;
    rb = (int64_t)((uint32_t)first / (uint32_t)n_rb); li = (int32_t)(first - rb * n_rb); left = last - first;
  }
  // returns the number of items (0 = done); (srb, sli) = the stage's first item
  OWQ_HD int32_t next(int64_t& srb, int32_t& sli) {
    if (left <= 0) return 0;
    const int32_t lim = (li < nss ? nss : n_rb) - li;
    int32_t n = lim < cap ? lim : cap;
    if ((int64_t)n > left) n = (int32_t)left;
    srb = rb; sli = li;
    li += n; left -= n;
    if (li == n_rb) { li = 0; ++rb; }
    return n;
  }
};

// Bytes of a stage starting at item li with n items (the weak tail chunk is short).
OWQ_HD int32_t stage_bytes(const Geo& g, int32_t li, int32_t n) {
  if (li < g.nss) return (int32_t)(n * g.ss_bytes);
  const int32_t c0 = li - g.nss;
  const bool has_tail = g.ktail && (c0 + n - 1 == g.nfull);
  return (has_tail ? (n - 1) * kWeakChunkBytes + g.tail_bytes : n * kWeakChunkBytes);
}

// ---- bit map of one row's super-step -------------------------------------------
// Word w of row r inside the super-step record.
OWQ_HD int64_t row_word_byte(int bits, int r, int w) {
  return w < 4 ? (int64_t)r * 16 + w * 4 : 2048 + (int64_t)r * (words_per_row(bits) - 4) * 4 + (w - 4) * 4;
}

// Location of bit `bit` of the code of super-step column `col` (0..63).  The
// decoder emits 16 32-bit values per row, value c = the codes of columns
// 4c .. 4c+3 as bytes 0..3 (tcgen05 kind::i8 A operand, one TMEM column); byte
// b = col % 4 of value c = col / 4 sits in bits [8b, 8b+8) of a word:
//  4-bit: c < 8 -> word c, bits 8b+0..3;  c >= 8 -> word c-8, bits 8b+4..7.
//  3-bit: c < 6 -> word c, bits 8b+0..2;  6 <= c < 12 -> word c-6, bits 8b+3..5;
//         c = 12+r -> bits 0,1 in word r at 8b+6, 8b+7 and bit 2 in word
//         4 + r/2 at 8b + 6 + r%2.
// So value c costs one LOP3 (c < 6 / c < 8), one SHF + LOP3 (c < 12 / c >= 8),
// or two SHF + three LOP3 (3-bit c >= 12).
OWQ_HD void code_bit_loc(int bits, int col, int bit, int& word, int& pos) {
  const int c = col >> 2, b = col & 3;
  if (bits == 4) {
    word = c & 7;
    pos = 8 * b + (c >= 8 ? 4 : 0) + bit;
  } else if (c < 6) {
    word = c;
    pos = 8 * b + bit;
  } else if (c < 12) {
    word = c - 6;
    pos = 8 * b + 3 + bit;
  } else {
    const int r = c - 12;
    if (bit < 2) {
      word = r;
      pos = 8 * b + 6 + bit;
    } else {
      word = 4 + (r >> 1);
      pos = 8 * b + 6 + (r & 1);
    }
  }
}

struct BlobHeader {            // first 256 bytes of the blob
  uint32_t magic, version;
  int32_t M, K, bits, group, k;
  int32_t nrb, nss, kpad, nitems, G;
  int64_t total, sz_off, widx_off;
};

}  // namespace owq
