/*
 * owq.h -- C ABI of libowq.so, the B200 (sm_100a) hot path of OWQ
 * (Outlier-aware Weight Quantization, arXiv 2306.02272).
 *
 * The operation (Sec. 4; Sec. 5.4):
 *
 *   y = W_hat x,   W_hat = (zero-filled b-bit matrix) + (fp16 weak columns)
 *
 *   "we store a complete low-precision matrix with zero-filled weak columns.
 *    Additionally, we store the weak columns as fp16 and use an extra single
 *    16-bit integer per column [...] the output of the matrix multiplication can
 *    be calculated as the sum of (zero-filled quantized weight matrix x fp16
 *    activation matrix) and (fp16 weak columns x corresponding fp16 activation
 *    channels)."
 *
 *   y[b][i] = sum_{j not weak} s[i][g(j)] * (q[i][j] - z[i][g(j)]) * x[b][j]
 *           + sum_{t < k} v[i][t] * x[b][idx[t]]
 *
 * W in R^{C_out x C_in}.  x is row-major [B][C_in] and y is [B][C_out]
 * (the transpose of the paper's C_in x N layout, reading s18).
 * g(j) = j / group_size (group_size 0 = one scale/zero per output row; P:362-388
 * for grouped grids).  Scale s and zero z are fp16; z is an integer code
 * (readings s7, s10).  Weak-column indices are u16, so
 * C_in <= 65536.
 *
 * Conventions
 *  - Every entry point validates on the host and returns an owq_status; no C++
 *    exception crosses the ABI.  Device calls are asynchronous on the given
 *    stream (cudaStream_t passed as void*; NULL = legacy default stream); a
 *    launch failure is returned as OWQ_ERR_CUDA, a fault inside a kernel
 *    surfaces at the caller's next synchronisation.
 *  - All buffers are caller-owned.  "d_" = device pointer, "h_" = host pointer.
 *    Nothing on the hot path (owq_gemv, owq_gemm_small_batch, owq_tp_gemv)
 *    allocates device memory or synchronises with the host.
 *  - fp16 values cross the ABI as uint16_t bit patterns (IEEE binary16) so this
 *    header is plain C99 with no CUDA headers.
 *
 * Device layout (the "packed blob", produced only by owq_pack / owq_pack_host;
 * version OWQ_LAYOUT_VERSION, self-describing: a 256-byte header repeats the
 * shape, so every call re-checks shape agreement).  Rows are grouped in
 * row-blocks of 128 (one tcgen05 M=128 tile; the last one padded); columns in
 * super-steps of 64 (the last one padded).  Per row-block the record holds
 * its super-steps followed by its weak-column chunks (8 columns each; the
 * ragged last chunk unpadded), so any run of items is one contiguous TMA bulk
 * copy.  Inside a super-step each row's 64 codes are 6 (3-bit) or 8 (4-bit)
 * 32-bit words, pre-positioned so that one LOP3 (or SHF + LOP3) yields four
 * consecutive codes as the bytes of one tcgen05 kind::i8 A-operand column.
 * DESIGN.md §5 gives the exact bit map;
 * owq_unpack_codes / owq_blob_decode_host invert it.
 */
#ifndef OWQ_H_
#define OWQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OWQ_LAYOUT_VERSION 3   /* tensor-core layout (tcgen05 kind::i8 GEMV)          */
#define OWQ_LAYOUT_CC 4        /* CUDA-core layout (FFMA2 GEMV), see owq_pack flags   */
#define OWQ_MAX_BATCH 16

typedef enum {
  OWQ_OK = 0,
  OWQ_ERR_INVALID_ARG = 1,     /* NULL pointer, non-positive size, bad mode      */
  OWQ_ERR_UNSUPPORTED = 2,     /* bits not in {3,4}; group_size not 0 or a power
                                  of two >= 128; batch outside [1,16]            */
  OWQ_ERR_WEAK_INDEX = 3,      /* weak_idx not strictly ascending, >= c_in,
                                  n_weak > c_in, or c_in > 65536                 */
  OWQ_ERR_ZERO_POINT = 4,      /* zero not an integer in [0, 2^bits - 1]        */
  OWQ_ERR_ZERO_FILL = 5,       /* OWQ_PACK_STRICT and a weak-column code != z  */
  OWQ_ERR_BUFFER_TOO_SMALL = 6,/* destination / workspace smaller than needed   */
  OWQ_ERR_BAD_BLOB = 7,        /* header magic/version/shape mismatch           */
  OWQ_ERR_CUDA = 8,            /* a CUDA runtime call or launch failed          */
  OWQ_ERR_NCCL = 9,            /* an NCCL call failed                           */
  OWQ_ERR_CODE_RANGE = 10      /* OWQ_PACK_U8_CODES and a code > 2^bits - 1     */
} owq_status;

/* Shape of one quantized linear layer (W in R^{C_out x C_in}). */
typedef struct {
  int32_t c_out;       /* M: output features (rows)                        */
  int32_t c_in;        /* K: input features (columns), 1..65536            */
  int32_t bits;        /* b: 3 or 4                         */
  int32_t group_size;  /* g: 0 = per output row, else a power of two >= 128 */
  int32_t n_weak;      /* k: number of fp16 weak columns, 0..c_in          */
} owq_shape;

/* The paper's representation in host memory ("interchange form"). */
typedef struct {
  const uint8_t  *codes;     /* canonical bit stream: row-major, LSB-first,
                                each row padded to a whole byte; row stride
                                ceil(c_in*bits/8) bytes  */
  const uint16_t *scale;     /* fp16 [c_out][G], G = g ? ceil(c_in/g) : 1     */
  const uint16_t *zero;      /* fp16 [c_out][G], integer-valued codes          */
  const uint16_t *weak_idx;  /* u16 [n_weak], strictly ascending, < c_in       */
  const uint16_t *weak_val;  /* fp16 [c_out][n_weak], row-major                */
} owq_host_layer;

/* owq_pack flags */
#define OWQ_PACK_STRICT 1    /* reject weak-column codes != z instead of zero-filling */
#define OWQ_PACK_U8_CODES 2  /* layer->codes is one code per byte, [c_out][c_in]       */
#define OWQ_PACK_LAYOUT_CC 4 /* write device layout 4 (CUDA-core GEMV) instead of 3      */

/* Bytes of the device blob for `shape` (header + padded code units + weak
 * units + scale/zero blocks + weak index list) in layout 3.  0 on an invalid
 * shape. */
size_t owq_packed_bytes(const owq_shape *shape);

/* Bytes of the device blob for `shape` in `layout` (OWQ_LAYOUT_VERSION = 3,
 * the tensor-core layout, or OWQ_LAYOUT_CC = 4, the CUDA-core layout: items of
 * 128 rows x 32 columns in which every code is one LOP3 away from an fp32
 * subnormal).  0 on an invalid shape or layout.  Both layouts
 * hold the same representation in the same number of code bytes
 * (b*M*K/8 up to row/column padding); the GEMV entry points read the layout
 * from the blob header and run the matching kernel. */
size_t owq_packed_bytes_layout(const owq_shape *shape, int layout);

/* Host packer (C++, runs once per layer, off the hot path): validates the
 * paper representation and writes the device layout into h_blob.  Weak-column
 * codes are rewritten to that row/group's zero point ("zero-filled", P:114,
 * reading s10) unless OWQ_PACK_STRICT.  Bit-exact, deterministic. */
owq_status owq_pack_host(const owq_shape *shape, const owq_host_layer *layer,
                         int flags, void *h_blob, size_t blob_bytes);

/* owq_pack_host into a temporary host buffer, then a copy to d_packed on
 * `stream`; returns after the copy completed (packing is offline).  With
 * OWQ_PACK_LAYOUT_CC in flags the blob is layout 4 and d_bytes must be at
 * least owq_packed_bytes_layout(shape, OWQ_LAYOUT_CC). */
owq_status owq_pack(const owq_shape *shape, const owq_host_layer *layer,
                    int flags, void *d_packed, size_t d_bytes, void *stream);

/* ---- representation variants (device layout 4 only) ----
 * act-order: OPTQ quantizes the columns in descending order of
 * diag(H) and forms its scale groups over that order; storage-favored
 * (P:486-490): the zero-filled weak columns are not stored at all.  Both are
 * a code matrix in STORED column order plus a column map: stored position p
 * holds original column colmap[p].  Scale/zero groups run over stored
 * positions (G = ceil(k_stored / group_size)); x keeps its c_in columns and
 * the weak indices stay original column indices.  Stored positions whose
 * column is weak are zero-filled (reading s10) unless OWQ_PACK_STRICT. */
typedef struct {
  int32_t k_stored;          /* stored columns: c_in (latency-favored, a
                                permutation) or c_in - n_weak (storage-favored) */
  const uint16_t *colmap;    /* [k_stored] original column of each stored
                                position; distinct, < c_in                      */
} owq_colmap;

/* Bytes of the layout-4 blob of `shape` with column map `map`; 0 if invalid. */
size_t owq_packed_bytes_colmap(const owq_shape *shape, const owq_colmap *map);

/* Pack a column-mapped layer: layer->codes is [c_out][k_stored] in stored
 * order (canonical stream, or one byte per code with OWQ_PACK_U8_CODES),
 * scale/zero [c_out][ceil(k_stored / g)], weak_idx/weak_val as in
 * owq_host_layer.  INVALID_ARG: a colmap entry out of range or repeated. */
owq_status owq_pack_host_colmap(const owq_shape *shape, const owq_host_layer *layer,
                                const owq_colmap *map, int flags,
                                void *h_blob, size_t blob_bytes);
owq_status owq_pack_colmap(const owq_shape *shape, const owq_host_layer *layer,
                           const owq_colmap *map, int flags,
                           void *d_packed, size_t d_bytes, void *stream);

/* Column map of a layout-4 blob (host test hook): *k_stored, and colmap
 * [k_stored] (identity for blobs packed without a map).  Any output may be NULL. */
owq_status owq_blob_colmap_host(const void *h_blob, size_t blob_bytes,
                                int32_t *k_stored, uint16_t *colmap);

/* Host inverse of the packer (test hook): recovers shape, one code per byte
 * [c_out][c_in] (weak columns hold the zero point), fp16 scale/zero [c_out][G],
 * weak_idx [n_weak], weak_val [c_out][n_weak].  Any output pointer may be NULL. */
/* (for a column-mapped blob, codes come back in stored order, [c_out][k_stored],
 * and scale/zero [c_out][ceil(k_stored / g)]) */
owq_status owq_blob_decode_host(const void *h_blob, size_t blob_bytes,
                                owq_shape *shape_out, uint8_t *codes,
                                uint16_t *scale, uint16_t *zero,
                                uint16_t *weak_idx, uint16_t *weak_val);

/* Device inverse of the code layout (test hook): one code per byte,
 * d_codes [c_out][c_in] row-major. */
owq_status owq_unpack_codes(const owq_shape *shape, const void *d_packed,
                            uint8_t *d_codes, void *stream);

/* Workspace of owq_gemv / owq_gemm_small_batch on the current device: a fixed
 * 4 MiB prefix of stream-K partial-row slots (one per CTA and batch row; a zero
 * word means "not written yet"), per-row-block arrival counters and fp32
 * partials for grids larger than the SM count, and the exact int8 digit tiles +
 * int64 digit sums of x written by each call's x pass.  The caller zero-fills
 * it ONCE; every call leaves the slots at zero again, so one workspace (sized
 * for the largest shape) serves sequential calls of any shapes.  One workspace
 * must not be used by two calls that may run concurrently. */
size_t owq_workspace_bytes(const owq_shape *shape, int batch);

/* Workspace for an explicit grid (owq_gemm_small_batch_grid; 0 = the default
 * grid of the current device), for either layout.  0 on an invalid shape,
 * batch or grid. */
size_t owq_workspace_bytes_grid(const owq_shape *shape, int batch, int grid);

/* y = W_hat x for one activation vector (batch 1).
 * d_x: fp16 [c_in] (finite values); d_y: [c_out], fp32 if y_f32 else fp16 (RNE).
 * Arithmetic: x * 2^24 is split into 6 exact int8 digits, the
 * codes are the u8 A operand of tcgen05.mma kind::i8 (s32 accumulate), and
 * s * 2^-24 * (sum_i 256^i D_i - z * sum x 2^24) is formed exactly in fp64 then
 * scaled in fp32; weak columns fp16 x fp16 in fp32.  Two launches on the
 * stream (x digit pass + fused GEMV).  Errors: INVALID_ARG (NULL pointers),
 * BAD_BLOB (header/shape mismatch), BUFFER_TOO_SMALL (workspace), CUDA. */
owq_status owq_gemv(const owq_shape *shape, const void *d_packed,
                    const uint16_t *d_x, void *d_y, int y_f32,
                    void *d_workspace, size_t ws_bytes, void *stream);

/* Y = W_hat X for B in [1, 16] activation rows: d_x fp16 [B][c_in] row-major,
 * d_y [B][c_out] (fp32 if y_f32).  Same arithmetic as owq_gemv; the MMA's N
 * dimension carries the 6 digit rows of every activation row (N = 8 / 16 / 32
 * / 64 / 96 for B = 1 / 2 / <= 5 / <= 10 / <= 16).  UNSUPPORTED if B is outside
 * [1, 16].  Layout-3 blobs with grouped scales at B >= 4 (c_in % 8 == 0, d_x
 * 16-byte aligned) run owq_gemm_batch_f16's kernel instead (faster there,
 * DESIGN.md §6.5); the result stays within the same error bound. */
owq_status owq_gemm_small_batch(const owq_shape *shape, const void *d_packed,
                                const uint16_t *d_x, int batch, void *d_y,
                                int y_f32, void *d_workspace, size_t ws_bytes,
                                void *stream);

/* Batched GEMV on tensor cores with an exact fp16 A operand:
 * Y = W_hat X for batch in [1, 32], layout-3 blobs, per-row or grouped scales
 * (any group_size owq_shape allows), c_in % 8 == 0, d_x 16-byte aligned.  A = the
 * exact integer (q - z) as fp16 in shared memory, B = x (N = batch padded to
 * 16 / 32), fp32 D in TMEM, one D per scale group drained by s_g; K split over
 * the grid with a deterministic last-arriver sum.  Workspace: the GEMV
 * workspace (owq_workspace_bytes with batch >= 2). */
owq_status owq_gemm_batch_f16(const owq_shape *shape, const void *d_packed,
                              const uint16_t *d_x, int batch, void *d_y, int y_f32,
                              void *d_workspace, size_t ws_bytes, void *stream);

/* Prefill: Y = W_hat X for any number of tokens (P:58 X in
 * R^{C_in x N}), d_x fp16 [n_tokens][c_in] (16-byte aligned, c_in % 8 == 0),
 * d_y [n_tokens][c_out] (fp32 if y_f32).  Tensor cores: A = the exact integer
 * (q - z) as fp16 decoded into shared memory, B = x, fp32 accumulation in TMEM
 * (tcgen05.mma kind::f16, 128 rows x 256 tokens per CTA); s applied per row after
 * the sum; fp16 weak columns folded in by the epilogue.  Layout 3 blobs with
 * per-row scales only: UNSUPPORTED for layout 4, group_size > 0 or c_in % 8 != 0.
 * No workspace. */
owq_status owq_gemm_prefill(const owq_shape *shape, const void *d_packed,
                            const uint16_t *d_x, int32_t n_tokens, void *d_y,
                            int y_f32, void *stream);

/* Prefill with a scratch workspace (16-byte aligned, any contents, at least
 * owq_prefill_workspace_bytes()): the K loop is split into pieces of at most 64
 * super-steps (4096 columns; the tensor core's fp32 accumulation over longer
 * loops exceeds the 2e-3 bound) and, when even one-row-block
 * CTAs would fill at most half the SMs, into up to 8 pieces; each piece stores
 * fp32 partial rows in the workspace and a second kernel adds them in piece
 * order (deterministic).  owq_gemm_prefill (no workspace) returns
 * OWQ_ERR_BUFFER_TOO_SMALL whenever a split is needed, i.e. c_in > 4096. */
owq_status owq_gemm_prefill_ws(const owq_shape *shape, const void *d_packed,
                               const uint16_t *d_x, int32_t n_tokens, void *d_y,
                               int y_f32, void *d_workspace, size_t ws_bytes,
                               void *stream);
/* Workspace bytes owq_gemm_prefill_ws needs at n_tokens on the current device
 * (0 = no split, owq_gemm_prefill suffices; 0 also for an invalid shape). */
size_t owq_prefill_workspace_bytes(const owq_shape *shape, int32_t n_tokens);

/* Test/tuning hook: same as owq_gemm_small_batch with an explicit grid size
 * (number of CTAs; 0 = one per SM; capped at one CTA per item; > 512 after the
 * cap -> UNSUPPORTED).  Small grids exercise the stream-K partial-sum path with
 * many pieces per row-block. */
owq_status owq_gemm_small_batch_grid(const owq_shape *shape, const void *d_packed,
                                     const uint16_t *d_x, int batch, void *d_y,
                                     int y_f32, void *d_workspace, size_t ws_bytes,
                                     int grid, void *stream);

/* ---------------- tensor parallelism over NCCL (one process per GPU) ------- */
#define OWQ_TP_ROWS 0   /* split c_out: each rank owns a row slice; all-gather y  */
#define OWQ_TP_COLS 1   /* split c_in: each rank owns a column slice; all-reduce  */

typedef struct owq_tp owq_tp;   /* owns one ncclComm_t */

/* 128-byte NCCL unique id, created on rank 0 and broadcast by the caller
 * (torch.distributed) before owq_tp_init on every rank. */
owq_status owq_tp_get_unique_id(void *id128);
owq_status owq_tp_init(const void *id128, int world, int rank, owq_tp **out);
owq_status owq_tp_destroy(owq_tp *tp);
/* Host poll of the communicator's asynchronous error state
 * (ncclCommGetAsyncError): OWQ_OK, or OWQ_ERR_NCCL once a collective enqueued by
 * owq_tp_gemv has failed (a peer died, a network error).  Non-blocking. */
owq_status owq_tp_check(owq_tp *tp);

/* Slice of `full` owned by `rank` (host only, no GPU needed).  ROWS: rows
 * [r0, r1) with r0 = round(rank*M/world) to a multiple of 16; every column,
 * every weak column.  COLS: columns [c0, c1), boundaries at multiples of
 * max(group_size, 64); weak columns inside the slice, re-based to the slice.
 * offset_out receives r0 (ROWS) or c0 (COLS). */
owq_status owq_tp_shard_shape(const owq_shape *full, const owq_host_layer *full_layer,
                              int mode, int world, int rank,
                              owq_shape *shard_out, int32_t *offset_out);

/* Pack rank's slice of `full_layer` into h_blob (host, no GPU). */
owq_status owq_tp_shard_host(const owq_shape *full, const owq_host_layer *full_layer,
                             int mode, int world, int rank, int flags,
                             void *h_blob, size_t blob_bytes);

/* owq_tp_shard_host + copy to d_packed_shard on `stream` (blocking). */
owq_status owq_tp_shard(const owq_shape *full, const owq_host_layer *full_layer,
                        int mode, int world, int rank, int flags,
                        void *d_packed_shard, size_t d_bytes, void *stream);

/* Workspace of owq_tp_gemv for this rank (zero-filled once by the caller). */
size_t owq_tp_workspace_bytes(const owq_shape *full, int mode, int world, int batch);

/* Tensor-parallel Y = W_hat X.  `shard` is this rank's slice shape (from
 * owq_tp_shard_shape).  ROWS: d_x is the full fp16 [B][c_in] on every rank;
 * local fused GEMV, then ncclAllGather of the y slices.  COLS: d_x is the
 * rank's column slice fp16 [B][c1-c0]; local fp32 partial Y (including the
 * rank's weak columns), then ncclAllReduce(sum, fp32).  d_y: the full
 * [B][c_out] on every rank (fp32 if y_f32).  Everything is enqueued on `stream`. */
owq_status owq_tp_gemv(owq_tp *tp, int mode, const owq_shape *full, const owq_shape *shard,
                       const void *d_packed_shard, const uint16_t *d_x, int batch,
                       void *d_y, int y_f32, void *d_workspace, size_t ws_bytes,
                       void *stream);

/* Host-only: [r0, r1) (ROWS) or [c0, c1) (COLS) owned by `rank`. */
owq_status owq_tp_bounds(const owq_shape *full, int mode, int world, int rank,
                         int32_t *begin, int32_t *end);

/* ---- OWQ quantization on the GPU (off the hot path) ----
 * The paper's algorithm (DESIGN.md §3 readings s1-s12) in fp64:
 * H = 2 X X^T (Eq. 3); dead columns H_jj := 1, W[:, j] := 0 and
 * H += percdamp * mean(diag H) * I; Eq. 5 sensitivity lambda_j ||dW_:,j||^2
 * with lambda_j the undamped H_jj and dW the min-max RTN error;
 * the n_weak most sensitive columns (ties -> smaller index) are kept in
 * fp16 and go last in the OPTQ order; OPTQ (Eq. 1) quantizes the
 * rest with a truncation-searched grid per row / original group fitted on
 * the group's current values; weak codes are zero-filled.
 * Output = the paper representation on the device: codes one per byte
 * [c_out][c_in] (pack with owq_pack + OWQ_PACK_U8_CODES after a copy),
 * fp16 scale / zero [c_out][G], u16 weak_idx [n_weak] ascending, fp16
 * weak_val [c_out][n_weak].  Synchronises the stream once (group runs) and at
 * the end (status).  UNSUPPORTED: bits outside [2, 8], group_size > 128,
 * n_weak >= c_in.  INVALID_ARG: NULL buffers, percdamp <= 0, or H not positive
 * definite after dampening. */
typedef struct {
  int32_t bits;         /* b */
  int32_t group_size;   /* g: 0 = per row, else <= 128 columns (original index groups) */
  int32_t n_weak;       /* k */
  int32_t clip;         /* 1 = truncation search over p = 1 - i/100, i < 80; 0 = min-max */
  double percdamp;      /* 0.01 (reading s2) */
} owq_quant_params;

size_t owq_quantize_workspace_bytes(int32_t c_out, int32_t c_in, int32_t n_samples,
                                    const owq_quant_params *params);
/* d_W: fp64 [c_out][c_in]; d_X: fp64 calibration features [c_in][n_samples]. */
owq_status owq_quantize_gpu(int32_t c_out, int32_t c_in, int32_t n_samples,
                            const double *d_W, const double *d_X, const owq_quant_params *params,
                            uint8_t *d_codes, uint16_t *d_scale, uint16_t *d_zero,
                            uint16_t *d_weak_idx, uint16_t *d_weak_val,
                            void *d_workspace, size_t ws_bytes, void *stream);

const char *owq_status_string(owq_status s);

#ifdef __cplusplus
}
#endif
#endif /* OWQ_H_ */
