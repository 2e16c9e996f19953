// owq_layout.h -- device layout of the packed OWQ blob (layout version 1).
// Shared by the host packer (owq_pack.cpp) and the device kernels (*.cu).
// The bit map is documented in DESIGN.md §5; include/owq.h summarises it.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define OWQ_HD __host__ __device__ __forceinline__
#else
#define OWQ_HD inline
#endif

namespace owq {

constexpr int kRowBlock = 64;        // rows per row-block (4 mma row-tiles of 16)
constexpr int kSuperStep = 64;       // columns per super-step (4 mma k16 steps)
constexpr int kWeakChunk = 8;        // weak columns per mma m16n8k8 chunk
constexpr int kWeakChunkBytes = kRowBlock * kWeakChunk * 2;   // 1 KiB
constexpr int kHeaderBytes = 256;
constexpr int kSZBlockBytes = kRowBlock * 4;                  // 64 x (s, z) fp16 pairs
constexpr uint32_t kMagic = 0x4257514Fu;                      // "OQWB"

OWQ_HD int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Geo {
  int32_t M, K, bits, group, k;
  int32_t nrb;       // row-blocks
  int32_t nss;       // super-steps per row
  int32_t kpad;      // k rounded up to a multiple of 8 (gathered-x buffer only)
  int32_t nfull;     // full weak chunks (8 columns, mma-fragment order)
  int32_t ktail;     // columns of the ragged last chunk (k % 8), stored row-major
  int32_t tail_bytes;// 64 * ktail * 2 rounded up to 16
  int32_t G;         // scale/zero groups per row
  int64_t ss_bytes;  // bytes per super-step (all 32 lanes)
  int64_t rb_bytes;  // bytes per row-block record (code units + weak units)
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
  g.tail_bytes = (int32_t)cdiv((int64_t)kRowBlock * g.ktail * 2, 16) * 16;
  g.G = group ? (int32_t)cdiv(K, group) : 1;
  g.ss_bytes = 32 * (bits == 3 ? 48 : 64);
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
  int64_t rb = b / g.rb_bytes;
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
  const int64_t rb = item / n;
  const int64_t T = (int64_t)g.nrb * g.rb_bytes;
  return item_offset(g, rb, (int32_t)(item - rb * n)) * grid / T;
}

// Stage sequence of one CTA: runs of at most `cap` items of one kind (code or
// weak) inside one row-block.  Producer and consumers walk the same sequence.
struct StageIter {
  int64_t rb;
  int32_t li, n_rb, nss, cap;
  int64_t left;
  OWQ_HD void init(const Geo& g, int64_t first, int64_t last, int32_t cap_) {
    n_rb = items_per_rb(g); nss = g.nss; cap = cap_;
    rb = first / n_rb; li = (int32_t)(first - rb * n_rb); left = last - first;
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

// ---- bit map of one super-step -------------------------------------------------
// Lane l = 4*gq + t (gq = l/4 "groupID", t = l%4) owns, for each of the 4 packets
// s (mma k16 steps) of the super-step, 16 pairs P = 4*r + a (r = row-tile 0..3,
// a = mma A register 0..3).  Pair (P, half) holds the code of
//   row = 16*r + gq + 8*(a & 1),  col = 16*t + 4*s + 2*(a >> 1) + half
// inside the row-block / super-step.  A packet is 3 (3-bit) or 4 (4-bit) 32-bit
// words; word w of packet s is lane word n = s*WPP + w, stored at byte
// (n/4)*512 + l*16 + (n%4)*4 of the super-step record (one LDS.128 per 4 words).
OWQ_HD int words_per_packet(int bits) { return bits == 3 ? 3 : 4; }

OWQ_HD int pair_row(int P, int gq) { return 16 * (P >> 2) + gq + 8 * (P & 1); }
OWQ_HD int pair_col(int P, int t, int s, int half) { return 16 * t + 4 * s + 2 * ((P & 3) >> 1) + half; }

// Location (word within packet, bit within word) of bit `bit` of the code in (P, half).
//  3-bit: P 0..8  : word P/3, field at bit 3*(P%3)          (+16 for the high half)
//         P 9..14 : word (P-9)/2, field at bit 9+3*((P-9)%2) (+16)
//         P 15    : code bit j in word j at bit 15           (+16)
//  4-bit: word P/4, field at bit 4*(P%4)                     (+16)
OWQ_HD void code_bit_loc(int bits, int P, int half, int bit, int& word, int& pos) {
  if (bits == 4) {
    word = P >> 2;
    pos = 4 * (P & 3) + bit + 16 * half;
  } else if (P < 9) {
    word = P / 3;
    pos = 3 * (P % 3) + bit + 16 * half;
  } else if (P < 15) {
    word = (P - 9) / 2;
    pos = 9 + 3 * ((P - 9) % 2) + bit + 16 * half;
  } else {
    word = bit;
    pos = 15 + 16 * half;
  }
}

OWQ_HD int64_t lane_word_byte(int n, int lane) { return (int64_t)(n >> 2) * 512 + lane * 16 + (n & 3) * 4; }

// ---- weak block ----------------------------------------------------------------
// Chunk j (8 weak columns) of a row-block: lane l = 4*gq + t holds, for row-tile r,
// two fp16x2 registers of the mma m16n8k8 A fragment:
//   reg0 = (v[16r+gq][8j+2t], v[16r+gq][8j+2t+1]),  reg1 = rows + 8.
// Byte offset inside the chunk: l*32 + r*8 + reg*4 (+ 2 for the odd column).
// The ragged last chunk (k % 8 columns) is stored unpadded, row-major
// [64][k % 8] fp16 (padded to 16 bytes), right after the full chunks.
OWQ_HD int64_t weak_byte(int row_in_rb, int col_in_chunk) {
  int r = row_in_rb >> 4, rem = row_in_rb & 15, gq = rem & 7, reg = rem >> 3;
  int t = col_in_chunk >> 1, odd = col_in_chunk & 1;
  int lane = gq * 4 + t;
  return (int64_t)lane * 32 + r * 8 + reg * 4 + odd * 2;
}

// ---- scale / zero block --------------------------------------------------------
// For (row-block, group): 64 rows x (s, z) fp16 pairs; row 16r + gq + 8h at
// byte gq*32 + (2r + h)*4 (s in the low half, z in the high half).
OWQ_HD int sz_byte(int row_in_rb) {
  int r = row_in_rb >> 4, rem = row_in_rb & 15, gq = rem & 7, h = rem >> 3;
  return gq * 32 + (2 * r + h) * 4;
}

struct BlobHeader {            // first 256 bytes of the blob
  uint32_t magic, version;
  int32_t M, K, bits, group, k;
  int32_t nrb, nss, kpad, nitems, G;
  int64_t total, sz_off, widx_off;
};

}  // namespace owq
