// owq_pack.cpp -- host side of libowq: validation, the packer (paper
// representation -> device layout), its inverse, and tensor-parallel sharding.
// Runs once per layer, off the hot path.  No CUDA dependency (CPU tests use it).
//
// Paper representation: a complete b-bit matrix with zero-filled weak
// columns, fp16 weak columns, one u16 index per weak column; fp16 scale/zero
// per output row or per (row, group).
#include <cmath>
#include <cstring>
#include <vector>

#include "owq.h"
#include "owq_layout.h"
#include "owq_layout_cc.h"

using owq::Geo;

namespace {

float half_to_float(uint16_t h) {
  uint32_t sign = (uint32_t)(h >> 15) << 31, exp = (h >> 10) & 0x1f, man = h & 0x3ff;
  uint32_t bits;
  if (exp == 0) {
    if (man == 0) { bits = sign; }
    else {                                   // subnormal
      float f = std::ldexp((float)man, -24);
      return sign ? -f : f;
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | (man << 13);
  } else {
    bits = sign | ((exp + 112) << 23) | (man << 13);
  }
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

bool shape_ok(const owq_shape* s) {
  return s && s->c_out > 0 && s->c_in > 0 && s->c_in <= 65536 && s->n_weak >= 0 &&
         s->n_weak <= s->c_in && (s->bits == 3 || s->bits == 4) &&
         (s->group_size == 0 || (s->group_size >= 128 && (s->group_size & (s->group_size - 1)) == 0));
}

owq_status check_shape(const owq_shape* s) {
  if (!s) return OWQ_ERR_INVALID_ARG;
  if (s->c_out <= 0 || s->c_in <= 0 || s->n_weak < 0) return OWQ_ERR_INVALID_ARG;
  if (s->bits != 3 && s->bits != 4) return OWQ_ERR_UNSUPPORTED;
  if (s->group_size < 0 || (s->group_size && (s->group_size < 128 || (s->group_size & (s->group_size - 1)))))
    return OWQ_ERR_UNSUPPORTED;
  if (s->c_in > 65536 || s->n_weak > s->c_in) return OWQ_ERR_WEAK_INDEX;
  return OWQ_OK;
}

int n_groups(const owq_shape* s) { return s->group_size ? (s->c_in + s->group_size - 1) / s->group_size : 1; }

// Validated, decoded view of an owq_host_layer.
struct Layer {
  int M, K, bits, group, k, G;     // K = stored columns (= c_in without a column map)
  int Korig = 0;                   // c_in (x width) when a column map is present
  std::vector<uint16_t> colmap;    // stored position -> original column (empty: identity)
  std::vector<uint8_t> codes;      // [M][K], weak columns already zero-filled
  const uint16_t* scale;
  const uint16_t* zero;
  const uint16_t* widx;
  const uint16_t* wval;
};

owq_status load_layer(const owq_shape* s, const owq_host_layer* L, int flags, Layer& out) {
  owq_status st = check_shape(s);
  if (st != OWQ_OK) return st;
  if (!L || !L->codes || !L->scale || !L->zero) return OWQ_ERR_INVALID_ARG;
  if (s->n_weak > 0 && (!L->weak_idx || !L->weak_val)) return OWQ_ERR_INVALID_ARG;
  const int M = s->c_out, K = s->c_in, b = s->bits, k = s->n_weak, G = n_groups(s);
  const int maxq = (1 << b) - 1;
  for (int t = 0; t < k; ++t) {
    if (L->weak_idx[t] >= K) return OWQ_ERR_WEAK_INDEX;
    if (t && L->weak_idx[t] <= L->weak_idx[t - 1]) return OWQ_ERR_WEAK_INDEX;
  }
  for (int64_t i = 0; i < (int64_t)M * G; ++i) {
    float z = half_to_float(L->zero[i]);
    if (!(z >= 0.f && z <= (float)maxq && z == std::floor(z))) return OWQ_ERR_ZERO_POINT;
  }
  out.M = M; out.K = K; out.bits = b; out.group = s->group_size; out.k = k; out.G = G;
  out.scale = L->scale; out.zero = L->zero; out.widx = L->weak_idx; out.wval = L->weak_val;
  out.codes.assign((size_t)M * K, 0);
  const bool u8 = flags & OWQ_PACK_U8_CODES;
  const int64_t rs = ((int64_t)K * b + 7) / 8;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int i = 0; i < M; ++i) {
    uint8_t* dst = &out.codes[(size_t)i * K];
    if (u8) {
      const uint8_t* src = L->codes + (size_t)i * K;
      for (int j = 0; j < K; ++j) { dst[j] = src[j]; bad |= src[j] > maxq; }
    } else {
      const uint8_t* row = L->codes + i * rs;
      for (int j = 0; j < K; ++j) {
        int64_t pos = (int64_t)j * b;
        uint32_t w = row[pos >> 3] | ((pos >> 3) + 1 < rs ? (uint32_t)row[(pos >> 3) + 1] << 8 : 0u);
        dst[j] = (uint8_t)((w >> (pos & 7)) & maxq);
      }
    }
  }
  if (bad) return OWQ_ERR_CODE_RANGE;
  // zero fill of weak columns ("zero-filled weak columns"; reading s10: code := z)
  const bool strict = flags & OWQ_PACK_STRICT;
  int fill_err = 0;
#pragma omp parallel for schedule(static) reduction(| : fill_err)
  for (int i = 0; i < M; ++i) {
    for (int t = 0; t < k; ++t) {
      int j = L->weak_idx[t];
      int gi = out.group ? j / out.group : 0;
      uint8_t z = (uint8_t)half_to_float(out.zero[(size_t)i * G + gi]);
      uint8_t& c = out.codes[(size_t)i * K + j];
      if (c != z) {
        if (strict) fill_err = 1;
        c = z;
      }
    }
  }
  if (fill_err) return OWQ_ERR_ZERO_FILL;
  return OWQ_OK;
}

void write_blob(const Layer& L, uint8_t* blob) {
  const Geo g = owq::make_geo(L.M, L.K, L.bits, L.group, L.k);
  std::memset(blob, 0, (size_t)g.total);
  owq::BlobHeader h{};
  h.magic = owq::kMagic; h.version = OWQ_LAYOUT_VERSION;
  h.M = L.M; h.K = L.K; h.bits = L.bits; h.group = L.group; h.k = L.k;
  h.nrb = g.nrb; h.nss = g.nss; h.kpad = g.kpad; h.nitems = owq::items_per_rb(g); h.G = g.G;
  h.total = g.total; h.sz_off = g.sz_off; h.widx_off = g.widx_off;
  std::memcpy(blob, &h, sizeof(h));
  const int wpr = owq::words_per_row(L.bits);
#pragma omp parallel for schedule(dynamic, 1)
  for (int rb = 0; rb < g.nrb; ++rb) {
    uint8_t* rec = blob + g.units_off + (int64_t)rb * g.rb_bytes;
    for (int ss = 0; ss < g.nss; ++ss) {
      uint8_t* ssrec = rec + (int64_t)ss * g.ss_bytes;
      for (int rr = 0; rr < owq::kRowBlock; ++rr) {
        const int row = rb * owq::kRowBlock + rr;
        uint32_t words[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (row < L.M) {
          for (int cc = 0; cc < owq::kSuperStep; ++cc) {
            const int col = ss * owq::kSuperStep + cc;
            const uint32_t code = col < L.K ? L.codes[(size_t)row * L.K + col] : 0u;
            for (int bit = 0; bit < L.bits; ++bit) {
              if (!((code >> bit) & 1u)) continue;
              int word, pos;
              owq::code_bit_loc(L.bits, cc, bit, word, pos);
              words[word] |= 1u << pos;
            }
          }
        }
        for (int w = 0; w < wpr; ++w) std::memcpy(ssrec + owq::row_word_byte(L.bits, rr, w), &words[w], 4);
      }
    }
    uint8_t* weak = rec + (int64_t)g.nss * g.ss_bytes;
    for (int j = 0; j < g.nfull; ++j)
      for (int rr = 0; rr < owq::kRowBlock; ++rr)
        for (int c = 0; c < owq::kWeakChunk; ++c) {
          const int row = rb * owq::kRowBlock + rr, col = j * owq::kWeakChunk + c;
          const uint16_t v = row < L.M ? L.wval[(size_t)row * L.k + col] : 0;
          std::memcpy(weak + (int64_t)j * owq::kWeakChunkBytes + (rr * owq::kWeakChunk + c) * 2, &v, 2);
        }
    uint8_t* tail = weak + (int64_t)g.nfull * owq::kWeakChunkBytes;
    for (int rr = 0; rr < owq::kRowBlock; ++rr)
      for (int c = 0; c < g.ktail; ++c) {
        const int row = rb * owq::kRowBlock + rr, col = g.nfull * owq::kWeakChunk + c;
        const uint16_t v = row < L.M ? L.wval[(size_t)row * L.k + col] : 0;
        std::memcpy(tail + 2 * (rr * g.ktail + c), &v, 2);
      }
    for (int gi = 0; gi < g.G; ++gi) {
      uint8_t* sz = blob + g.sz_off + ((int64_t)rb * g.G + gi) * owq::kSZBlockBytes;
      for (int rr = 0; rr < owq::kRowBlock; ++rr) {
        const int row = rb * owq::kRowBlock + rr;
        uint16_t pair[2] = {0, 0};
        if (row < L.M) { pair[0] = L.scale[(size_t)row * g.G + gi]; pair[1] = L.zero[(size_t)row * g.G + gi]; }
        std::memcpy(sz + 4 * rr, pair, 4);
      }
    }
  }
  for (int t = 0; t < L.k; ++t) std::memcpy(blob + g.widx_off + 2 * t, &L.widx[t], 2);
}

// Layout version 4 (owq_layout_cc.h): items of 128 rows x 32 columns for the
// CUDA-core GEMV; codes placed so that each is one LOP3 away from an fp32
// subnormal (bit offset p(j) + bits <= 24 inside the register it is read from).
void write_blob_cc(const Layer& L, uint8_t* blob) {
  namespace C = owq::cc;
  const bool mapped = !L.colmap.empty() || L.Korig > 0;
  const C::Geo g = mapped ? C::make_geo(L.M, L.Korig, L.bits, L.group, L.k, L.K) : C::make_geo(L.M, L.K, L.bits, L.group, L.k);
  std::memset(blob, 0, (size_t)g.total);
  C::BlobHeader h{};
  h.magic = C::kMagic; h.version = C::kVersion;
  h.M = L.M; h.K = g.K; h.bits = L.bits; h.group = L.group; h.k = L.k;
  h.nrb = g.nrb; h.nsteps = g.nsteps; h.kpad = g.kpad; h.G = g.G; h.W = g.W; h.total = g.total;
  h.Ks = g.Ks; h.mapped = g.mapped;
  std::memcpy(blob, &h, sizeof(h));
#pragma omp parallel for schedule(dynamic, 1)
  for (int rb = 0; rb < g.nrb; ++rb) {
    for (int st = 0; st < g.nsteps; ++st) {
      uint8_t* it = blob + g.units_off + C::item_offset(g, rb, st);
      for (int rr = 0; rr < C::kRowBlock; ++rr) {
        const int row = rb * C::kRowBlock + rr;
        if (row >= L.M) continue;
        uint32_t words[4] = {0, 0, 0, 0};
        for (int j = 0; j < C::kStep; ++j) {
          const int col = st * C::kStep + j;
          const uint32_t code = col < L.K ? L.codes[(size_t)row * L.K + col] : 0u;
          for (int bit = 0; bit < L.bits; ++bit) {
            if (!((code >> bit) & 1u)) continue;
            int word, pos;
            C::cc_bit_loc(L.bits, j, bit, word, pos);
            words[word] |= 1u << pos;
          }
        }
        const int lane = rr >> 2, r = rr & 3;
        for (int c = 0; c < g.W; ++c) std::memcpy(it + (c * 32 + lane) * 16 + r * 4, &words[c], 4);
      }
    }
    for (int gi = 0; gi < g.G; ++gi) {
      uint8_t* sz = blob + g.sz_off + ((int64_t)rb * g.G + gi) * C::kSZBlockBytes;
      for (int rr = 0; rr < C::kRowBlock; ++rr) {
        const int row = rb * C::kRowBlock + rr;
        uint16_t pair[2] = {0, 0};
        if (row < L.M) { pair[0] = L.scale[(size_t)row * g.G + gi]; pair[1] = L.zero[(size_t)row * g.G + gi]; }
        std::memcpy(sz + 4 * rr, pair, 4);
      }
    }
    uint8_t* weak = blob + g.weak_off + (int64_t)rb * g.weak_rb_bytes;
    for (int t = 0; t < L.k; ++t)
      for (int rr = 0; rr < C::kRowBlock; ++rr) {
        const int row = rb * C::kRowBlock + rr;
        const uint16_t v = row < L.M ? L.wval[(size_t)row * L.k + t] : 0;
        std::memcpy(weak + (int64_t)(t / C::kWeakChunk) * C::kWeakChunkBytes + (rr * C::kWeakChunk + t % C::kWeakChunk) * 2, &v, 2);
      }
  }
  uint32_t* mask = reinterpret_cast<uint32_t*>(blob + g.wmask_off);
  for (int t = 0; t < L.k; ++t) std::memcpy(blob + g.widx_off + 2 * t, &L.widx[t], 2);
  if (mapped) {
    // weak mask over stored positions; the column map itself
    std::vector<char> is_weak((size_t)g.K, 0);
    for (int t = 0; t < L.k; ++t) is_weak[L.widx[t]] = 1;
    uint16_t* cm = reinterpret_cast<uint16_t*>(blob + g.colmap_off);
    for (int p = 0; p < g.Ks; ++p) {
      cm[p] = L.colmap[p];
      if (is_weak[L.colmap[p]]) mask[p >> 5] |= 1u << (p & 31);
    }
  } else {
    for (int t = 0; t < L.k; ++t) mask[L.widx[t] >> 5] |= 1u << (L.widx[t] & 31);
  }
}

// Layer with a column map (NEXT-4: act-order / storage-favored, layout 4 only):
// codes [M][Ks] and scale/zero [M][ceil(Ks/g)] in stored order; weak indices
// and values in original columns; stored positions of weak columns zero-filled.
owq_status load_layer_map(const owq_shape* s, const owq_host_layer* L, const owq_colmap* map, int flags, Layer& out) {
  owq_status st = check_shape(s);
  if (st != OWQ_OK) return st;
  if (!map || !map->colmap || map->k_stored <= 0 || map->k_stored > s->c_in) return OWQ_ERR_INVALID_ARG;
  if (!L || !L->codes || !L->scale || !L->zero) return OWQ_ERR_INVALID_ARG;
  if (s->n_weak > 0 && (!L->weak_idx || !L->weak_val)) return OWQ_ERR_INVALID_ARG;
  const int K = s->c_in, Ks = map->k_stored, k = s->n_weak;
  std::vector<char> seen((size_t)K, 0);
  for (int p = 0; p < Ks; ++p) {
    const int c = map->colmap[p];
    if (c >= K || seen[c]) return OWQ_ERR_INVALID_ARG;   // in range and injective
    seen[c] = 1;
  }
  for (int t = 0; t < k; ++t) {
    if (L->weak_idx[t] >= K) return OWQ_ERR_WEAK_INDEX;
    if (t && L->weak_idx[t] <= L->weak_idx[t - 1]) return OWQ_ERR_WEAK_INDEX;
  }
  // codes / grids over the stored positions, validated without the weak handling
  owq_shape ss = *s;
  ss.c_in = Ks;
  ss.n_weak = 0;
  owq_host_layer ls = *L;
  ls.weak_idx = nullptr;
  ls.weak_val = nullptr;
  st = load_layer(&ss, &ls, flags & ~OWQ_PACK_STRICT, out);
  if (st != OWQ_OK) return st;
  out.k = k; out.widx = L->weak_idx; out.wval = L->weak_val;
  out.Korig = K;
  out.colmap.assign(map->colmap, map->colmap + Ks);
  std::vector<char> is_weak((size_t)K, 0);
  for (int t = 0; t < k; ++t) is_weak[L->weak_idx[t]] = 1;
  int fill_err = 0;
  for (int i = 0; i < out.M; ++i)
    for (int p = 0; p < Ks; ++p)
      if (is_weak[out.colmap[p]]) {
        const int gi = out.group ? p / out.group : 0;
        const uint8_t z = (uint8_t)half_to_float(out.zero[(size_t)i * out.G + gi]);
        uint8_t& c = out.codes[(size_t)i * Ks + p];
        if (c != z) {
          if (flags & OWQ_PACK_STRICT) fill_err = 1;
          c = z;
        }
      }
  return fill_err ? OWQ_ERR_ZERO_FILL : OWQ_OK;
}

owq_status decode_cc(const void* h_blob, size_t bytes, owq_shape* shape_out, uint8_t* codes, uint16_t* scale,
                     uint16_t* zero, uint16_t* weak_idx, uint16_t* weak_val) {
  namespace C = owq::cc;
  C::BlobHeader h;
  std::memcpy(&h, h_blob, sizeof(h));
  owq_shape s{h.M, h.K, h.bits, h.group, h.k};
  if (!shape_ok(&s)) return OWQ_ERR_BAD_BLOB;
  const C::Geo g = h.mapped ? C::make_geo(h.M, h.K, h.bits, h.group, h.k, h.Ks) : C::make_geo(h.M, h.K, h.bits, h.group, h.k);
  if ((size_t)g.total > bytes || g.total != h.total) return OWQ_ERR_BAD_BLOB;
  const uint8_t* blob = (const uint8_t*)h_blob;
  if (shape_out) *shape_out = s;
  for (int row = 0; row < h.M; ++row) {
    const int rb = row / C::kRowBlock, rr = row % C::kRowBlock, lane = rr >> 2, r = rr & 3;
    if (codes)
      for (int col = 0; col < g.Ks; ++col) {
        const uint8_t* it = blob + g.units_off + C::item_offset(g, rb, col / C::kStep);
        uint32_t c = 0;
        for (int bit = 0; bit < h.bits; ++bit) {
          int word, pos;
          C::cc_bit_loc(h.bits, col % C::kStep, bit, word, pos);
          uint32_t v;
          std::memcpy(&v, it + (word * 32 + lane) * 16 + r * 4, 4);
          c |= ((v >> pos) & 1u) << bit;
        }
        codes[(size_t)row * g.Ks + col] = (uint8_t)c;
      }
    for (int gi = 0; gi < g.G; ++gi) {
      uint16_t pair[2];
      std::memcpy(pair, blob + g.sz_off + ((int64_t)rb * g.G + gi) * C::kSZBlockBytes + 4 * rr, 4);
      if (scale) scale[(size_t)row * g.G + gi] = pair[0];
      if (zero) zero[(size_t)row * g.G + gi] = pair[1];
    }
    if (weak_val)
      for (int t = 0; t < h.k; ++t)
        std::memcpy(&weak_val[(size_t)row * h.k + t],
                    blob + g.weak_off + (int64_t)rb * g.weak_rb_bytes + (int64_t)(t / C::kWeakChunk) * C::kWeakChunkBytes +
                        (rr * C::kWeakChunk + t % C::kWeakChunk) * 2, 2);
  }
  if (weak_idx)
    for (int t = 0; t < h.k; ++t) std::memcpy(&weak_idx[t], blob + g.widx_off + 2 * t, 2);
  return OWQ_OK;
}

owq_status read_header(const void* h_blob, size_t bytes, owq::BlobHeader& h, Geo& g) {
  if (!h_blob || bytes < (size_t)owq::kHeaderBytes) return OWQ_ERR_INVALID_ARG;
  std::memcpy(&h, h_blob, sizeof(h));
  if (h.magic != owq::kMagic || h.version != OWQ_LAYOUT_VERSION) return OWQ_ERR_BAD_BLOB;
  owq_shape s{h.M, h.K, h.bits, h.group, h.k};
  if (!shape_ok(&s)) return OWQ_ERR_BAD_BLOB;
  g = owq::make_geo(h.M, h.K, h.bits, h.group, h.k);
  if ((size_t)g.total > bytes || g.total != h.total) return OWQ_ERR_BAD_BLOB;
  return OWQ_OK;
}

// ---- tensor-parallel slicing ----------------------------------------------------
int64_t round_to(int64_t v, int64_t u) { return ((v + u / 2) / u) * u; }

void shard_bounds(const owq_shape* f, int mode, int world, int rank, int64_t& a, int64_t& b) {
  if (mode == OWQ_TP_ROWS) {
    auto bnd = [&](int r) -> int64_t {
      if (r >= world) return f->c_out;
      int64_t v = round_to((int64_t)r * f->c_out / world, 16);
      return v > f->c_out ? f->c_out : v;
    };
    a = bnd(rank); b = bnd(rank + 1);
  } else {
    int64_t u = f->group_size > 64 ? f->group_size : 64;
    auto bnd = [&](int r) -> int64_t {
      if (r >= world) return f->c_in;
      int64_t v = round_to((int64_t)r * f->c_in / world, u);
      return v > f->c_in ? f->c_in : v;
    };
    a = bnd(rank); b = bnd(rank + 1);
  }
}

// Build rank's slice as a Layer (codes u8 already zero-filled from the full layer).
owq_status slice_layer(const owq_shape* full, const owq_host_layer* FL, int mode, int world,
                       int rank, int flags, Layer& out, std::vector<uint16_t>& sc,
                       std::vector<uint16_t>& zr, std::vector<uint16_t>& wi,
                       std::vector<uint16_t>& wv, owq_shape& ss, int32_t& offset) {
  if ((mode != OWQ_TP_ROWS && mode != OWQ_TP_COLS) || world < 1 || rank < 0 || rank >= world)
    return OWQ_ERR_INVALID_ARG;
  Layer F;
  owq_status st = load_layer(full, FL, flags, F);
  if (st != OWQ_OK) return st;
  int64_t a, b;
  shard_bounds(full, mode, world, rank, a, b);
  if (b <= a) return OWQ_ERR_INVALID_ARG;        // empty slice: too many ranks for this shape
  offset = (int32_t)a;
  const int G = F.G;
  if (mode == OWQ_TP_ROWS) {
    const int m = (int)(b - a);
    ss = {m, F.K, F.bits, F.group, F.k};
    out = F;
    out.M = m;
    out.codes.assign(F.codes.begin() + a * F.K, F.codes.begin() + b * F.K);
    sc.assign(F.scale + a * G, F.scale + b * G);
    zr.assign(F.zero + a * G, F.zero + b * G);
    wi.assign(F.widx, F.widx + F.k);
    wv.assign(F.wval ? F.wval + a * F.k : nullptr, F.wval ? F.wval + b * F.k : nullptr);
  } else {
    const int kc = (int)(b - a);
    std::vector<int> cols;
    for (int t = 0; t < F.k; ++t)
      if (F.widx[t] >= a && F.widx[t] < b) cols.push_back(t);
    const int kl = (int)cols.size();
    const int g0 = F.group ? (int)(a / F.group) : 0;
    const int Gl = F.group ? (int)((kc + F.group - 1) / F.group) : 1;
    ss = {F.M, kc, F.bits, F.group, kl};
    out = F;
    out.K = kc; out.k = kl; out.G = Gl;
    out.codes.resize((size_t)F.M * kc);
    sc.resize((size_t)F.M * Gl); zr.resize((size_t)F.M * Gl);
    wi.resize(kl); wv.resize((size_t)F.M * kl);
    for (int i = 0; i < F.M; ++i) {
      std::memcpy(&out.codes[(size_t)i * kc], &F.codes[(size_t)i * F.K + a], kc);
      for (int q = 0; q < Gl; ++q) { sc[(size_t)i * Gl + q] = F.scale[(size_t)i * G + g0 + q]; zr[(size_t)i * Gl + q] = F.zero[(size_t)i * G + g0 + q]; }
      for (int t = 0; t < kl; ++t) wv[(size_t)i * kl + t] = F.wval[(size_t)i * F.k + cols[t]];
    }
    for (int t = 0; t < kl; ++t) wi[t] = (uint16_t)(F.widx[cols[t]] - a);
  }
  out.scale = sc.data(); out.zero = zr.data(); out.widx = wi.data(); out.wval = wv.data();
  return OWQ_OK;
}

}  // namespace

extern "C" {

size_t owq_packed_bytes(const owq_shape* s) {
  if (!shape_ok(s)) return 0;
  return (size_t)owq::make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak).total;
}

size_t owq_packed_bytes_layout(const owq_shape* s, int layout) {
  if (!shape_ok(s)) return 0;
  if (layout == OWQ_LAYOUT_VERSION) return owq_packed_bytes(s);
  if (layout == OWQ_LAYOUT_CC) return (size_t)owq::cc::make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak).total;
  return 0;
}

owq_status owq_pack_host(const owq_shape* s, const owq_host_layer* L, int flags, void* h_blob,
                         size_t blob_bytes) {
  if (!h_blob) return OWQ_ERR_INVALID_ARG;
  Layer lay;
  owq_status st = load_layer(s, L, flags, lay);
  if (st != OWQ_OK) return st;
  const bool cc = flags & OWQ_PACK_LAYOUT_CC;
  if (blob_bytes < owq_packed_bytes_layout(s, cc ? OWQ_LAYOUT_CC : OWQ_LAYOUT_VERSION)) return OWQ_ERR_BUFFER_TOO_SMALL;
  if (cc) write_blob_cc(lay, (uint8_t*)h_blob);
  else write_blob(lay, (uint8_t*)h_blob);
  return OWQ_OK;
}

size_t owq_packed_bytes_colmap(const owq_shape* s, const owq_colmap* map) {
  if (!shape_ok(s) || !map || map->k_stored <= 0 || map->k_stored > s->c_in) return 0;
  return (size_t)owq::cc::make_geo(s->c_out, s->c_in, s->bits, s->group_size, s->n_weak, map->k_stored).total;
}

owq_status owq_pack_host_colmap(const owq_shape* s, const owq_host_layer* L, const owq_colmap* map, int flags,
                                void* h_blob, size_t blob_bytes) {
  if (!h_blob) return OWQ_ERR_INVALID_ARG;
  Layer lay;
  owq_status st = load_layer_map(s, L, map, flags, lay);
  if (st != OWQ_OK) return st;
  if (blob_bytes < owq_packed_bytes_colmap(s, map)) return OWQ_ERR_BUFFER_TOO_SMALL;
  write_blob_cc(lay, (uint8_t*)h_blob);
  return OWQ_OK;
}

owq_status owq_blob_colmap_host(const void* h_blob, size_t bytes, int32_t* k_stored, uint16_t* colmap) {
  namespace C = owq::cc;
  if (!h_blob || bytes < (size_t)C::kHeaderBytes) return OWQ_ERR_INVALID_ARG;
  C::BlobHeader h;
  std::memcpy(&h, h_blob, sizeof(h));
  if (h.magic != C::kMagic || h.version != (uint32_t)OWQ_LAYOUT_CC) return OWQ_ERR_BAD_BLOB;
  const C::Geo g = h.mapped ? C::make_geo(h.M, h.K, h.bits, h.group, h.k, h.Ks) : C::make_geo(h.M, h.K, h.bits, h.group, h.k);
  if ((size_t)g.total > bytes) return OWQ_ERR_BAD_BLOB;
  if (k_stored) *k_stored = g.Ks;
  if (colmap)
    for (int p = 0; p < g.Ks; ++p) {
      uint16_t v = (uint16_t)p;
      if (h.mapped) std::memcpy(&v, (const uint8_t*)h_blob + g.colmap_off + 2 * p, 2);
      colmap[p] = v;
    }
  return OWQ_OK;
}

owq_status owq_blob_decode_host(const void* h_blob, size_t bytes, owq_shape* shape_out,
                                uint8_t* codes, uint16_t* scale, uint16_t* zero,
                                uint16_t* weak_idx, uint16_t* weak_val) {
  if (h_blob && bytes >= (size_t)owq::kHeaderBytes) {
    uint32_t mv[2];
    std::memcpy(mv, h_blob, 8);
    if (mv[0] == owq::cc::kMagic && mv[1] == (uint32_t)OWQ_LAYOUT_CC)
      return decode_cc(h_blob, bytes, shape_out, codes, scale, zero, weak_idx, weak_val);
  }
  owq::BlobHeader h;
  Geo g;
  owq_status st = read_header(h_blob, bytes, h, g);
  if (st != OWQ_OK) return st;
  const uint8_t* blob = (const uint8_t*)h_blob;
  if (shape_out) *shape_out = {h.M, h.K, h.bits, h.group, h.k};
  const int wpr = owq::words_per_row(h.bits);
  for (int rb = 0; rb < g.nrb; ++rb) {
    const uint8_t* rec = blob + g.units_off + (int64_t)rb * g.rb_bytes;
    for (int rr = 0; rr < owq::kRowBlock; ++rr) {
      const int row = rb * owq::kRowBlock + rr;
      if (row >= h.M) continue;
      if (codes) {
        for (int ss = 0; ss < g.nss; ++ss) {
          uint32_t words[8];
          for (int w = 0; w < wpr; ++w)
            std::memcpy(&words[w], rec + (int64_t)ss * g.ss_bytes + owq::row_word_byte(h.bits, rr, w), 4);
          for (int cc = 0; cc < owq::kSuperStep; ++cc) {
            const int col = ss * owq::kSuperStep + cc;
            if (col >= h.K) continue;
            uint32_t c = 0;
            for (int bit = 0; bit < h.bits; ++bit) {
              int word, pos;
              owq::code_bit_loc(h.bits, cc, bit, word, pos);
              c |= ((words[word] >> pos) & 1u) << bit;
            }
            codes[(size_t)row * h.K + col] = (uint8_t)c;
          }
        }
      }
      if (weak_val) {
        const uint8_t* weak = rec + (int64_t)g.nss * g.ss_bytes;
        for (int col = 0; col < h.k; ++col) {
          const int j = col / owq::kWeakChunk, c = col % owq::kWeakChunk;
          const uint8_t* src = j < g.nfull
              ? weak + (int64_t)j * owq::kWeakChunkBytes + (rr * owq::kWeakChunk + c) * 2
              : weak + (int64_t)g.nfull * owq::kWeakChunkBytes + 2 * (rr * g.ktail + c);
          std::memcpy(&weak_val[(size_t)row * h.k + col], src, 2);
        }
      }
      for (int gi = 0; gi < g.G; ++gi) {
        uint16_t pair[2];
        std::memcpy(pair, blob + g.sz_off + ((int64_t)rb * g.G + gi) * owq::kSZBlockBytes + 4 * rr, 4);
        if (scale) scale[(size_t)row * g.G + gi] = pair[0];
        if (zero) zero[(size_t)row * g.G + gi] = pair[1];
      }
    }
  }
  if (weak_idx)
    for (int t = 0; t < h.k; ++t) std::memcpy(&weak_idx[t], blob + g.widx_off + 2 * t, 2);
  return OWQ_OK;
}

owq_status owq_tp_shard_shape(const owq_shape* full, const owq_host_layer* FL, int mode,
                              int world, int rank, owq_shape* shard_out, int32_t* offset_out) {
  Layer L;
  std::vector<uint16_t> sc, zr, wi, wv;
  owq_shape ss;
  int32_t off;
  owq_status st = slice_layer(full, FL, mode, world, rank, 0, L, sc, zr, wi, wv, ss, off);
  if (st != OWQ_OK) return st;
  if (shard_out) *shard_out = ss;
  if (offset_out) *offset_out = off;
  return OWQ_OK;
}

owq_status owq_tp_shard_host(const owq_shape* full, const owq_host_layer* FL, int mode, int world,
                             int rank, int flags, void* h_blob, size_t blob_bytes) {
  if (!h_blob) return OWQ_ERR_INVALID_ARG;
  Layer L;
  std::vector<uint16_t> sc, zr, wi, wv;
  owq_shape ss;
  int32_t off;
  owq_status st = slice_layer(full, FL, mode, world, rank, flags, L, sc, zr, wi, wv, ss, off);
  if (st != OWQ_OK) return st;
  const bool cc = flags & OWQ_PACK_LAYOUT_CC;
  if (blob_bytes < owq_packed_bytes_layout(&ss, cc ? OWQ_LAYOUT_CC : OWQ_LAYOUT_VERSION)) return OWQ_ERR_BUFFER_TOO_SMALL;
  if (cc) write_blob_cc(L, (uint8_t*)h_blob);
  else write_blob(L, (uint8_t*)h_blob);
  return OWQ_OK;
}

owq_status owq_tp_bounds(const owq_shape* full, int mode, int world, int rank, int32_t* begin,
                         int32_t* end) {
  owq_status st = check_shape(full);
  if (st != OWQ_OK) return st;
  if ((mode != OWQ_TP_ROWS && mode != OWQ_TP_COLS) || world < 1 || rank < 0 || rank >= world)
    return OWQ_ERR_INVALID_ARG;
  int64_t a, b;
  shard_bounds(full, mode, world, rank, a, b);
  if (begin) *begin = (int32_t)a;
  if (end) *end = (int32_t)b;
  return OWQ_OK;
}

const char* owq_status_string(owq_status s) {
  switch (s) {
    case OWQ_OK: return "OWQ_OK";
    case OWQ_ERR_INVALID_ARG: return "OWQ_ERR_INVALID_ARG";
    case OWQ_ERR_UNSUPPORTED: return "OWQ_ERR_UNSUPPORTED";
    case OWQ_ERR_WEAK_INDEX: return "OWQ_ERR_WEAK_INDEX";
    case OWQ_ERR_ZERO_POINT: return "OWQ_ERR_ZERO_POINT";
    case OWQ_ERR_ZERO_FILL: return "OWQ_ERR_ZERO_FILL";
    case OWQ_ERR_BUFFER_TOO_SMALL: return "OWQ_ERR_BUFFER_TOO_SMALL";
    case OWQ_ERR_BAD_BLOB: return "OWQ_ERR_BAD_BLOB";
    case OWQ_ERR_CUDA: return "OWQ_ERR_CUDA";
    case OWQ_ERR_NCCL: return "OWQ_ERR_NCCL";
    case OWQ_ERR_CODE_RANGE: return "OWQ_ERR_CODE_RANGE";
  }
  return "OWQ_ERR_UNKNOWN";
}

}  // extern "C"
