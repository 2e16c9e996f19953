// owq_tp.cu -- tensor-parallel OWQ GEMV over NCCL (one process per GPU).
// Row split (c_out): each rank runs the fused GEMV on its rows, then
// ncclAllGather assembles y.  Column split (c_in): each rank produces an fp32
// partial y (its columns and its weak columns), then ncclAllReduce(sum).
// The paper runs on one A100; sharding is this build's addition
// (SURVEY §8(e)).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>

#include "owq.h"
#include "owq_layout.h"

struct owq_tp {
  ncclComm_t comm;
  int world, rank;
};

namespace {

// gathered [world][B*mmax]: rank r's slot holds its rows densely as [B][m_r];
// scatter them to y [B][M] at the rank's row offset.
__device__ __forceinline__ int row_bound(int r, int world, int M) {   // == shard_bounds (owq_pack.cpp)
  if (r >= world) return M;
  const int64_t v = (((int64_t)r * M / world) + 8) / 16 * 16;
  return v > M ? M : (int)v;
}

template <typename T>
__global__ void tp_scatter_rows(const T* __restrict__ g, T* __restrict__ y, int world, int B, int M, int mmax) {
  const int64_t slot = (int64_t)B * mmax, n = (int64_t)world * slot;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / slot);
    const int64_t rem = i - (int64_t)r * slot;
    const int o0 = row_bound(r, world, M), mr = row_bound(r + 1, world, M) - o0;
    if (rem >= (int64_t)B * mr) continue;
    const int b = (int)(rem / mr), j = (int)(rem - (int64_t)b * mr);
    y[(int64_t)b * M + o0 + j] = g[i];
  }
}

__global__ void tp_f32_to_f16(const float* __restrict__ a, __half* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __float2half_rn(a[i]);
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

int max_rows(const owq_shape* full, int world, int32_t* offs) {
  int mmax = 0;
  for (int r = 0; r < world; ++r) {
    int32_t a, b;
    owq_tp_bounds(full, OWQ_TP_ROWS, world, r, &a, &b);
    if (offs) { offs[r] = a; offs[r + 1] = b; }
    mmax = std::max(mmax, (int)(b - a));
  }
  return mmax;
}

}  // namespace

extern "C" {

owq_status owq_tp_get_unique_id(void* id128) {
  if (!id128) return OWQ_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return OWQ_ERR_NCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id128, &id, sizeof(id));
  return OWQ_OK;
}

owq_status owq_tp_init(const void* id128, int world, int rank, owq_tp** out) {
  if (!id128 || !out || world < 1 || rank < 0 || rank >= world) return OWQ_ERR_INVALID_ARG;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  owq_tp* tp = new owq_tp{nullptr, world, rank};
  if (ncclCommInitRank(&tp->comm, world, id, rank) != ncclSuccess) {
    delete tp;
    return OWQ_ERR_NCCL;
  }
  *out = tp;
  return OWQ_OK;
}

owq_status owq_tp_check(owq_tp* tp) {
  if (!tp) return OWQ_ERR_INVALID_ARG;
  ncclResult_t async = ncclSuccess;
  if (ncclCommGetAsyncError(tp->comm, &async) != ncclSuccess) return OWQ_ERR_NCCL;
  return async == ncclSuccess || async == ncclInProgress ? OWQ_OK : OWQ_ERR_NCCL;
}

owq_status owq_tp_destroy(owq_tp* tp) {
  if (!tp) return OWQ_ERR_INVALID_ARG;
  ncclResult_t r = ncclCommDestroy(tp->comm);
  delete tp;
  return r == ncclSuccess ? OWQ_OK : OWQ_ERR_NCCL;
}

owq_status owq_tp_shard(const owq_shape* full, const owq_host_layer* FL, int mode, int world, int rank,
                        int flags, void* d_packed, size_t d_bytes, void* stream) {
  if (!d_packed) return OWQ_ERR_INVALID_ARG;
  owq_shape ss;
  owq_status st = owq_tp_shard_shape(full, FL, mode, world, rank, &ss, nullptr);
  if (st != OWQ_OK) return st;
  const size_t n = owq_packed_bytes_layout(&ss, (flags & OWQ_PACK_LAYOUT_CC) ? OWQ_LAYOUT_CC : OWQ_LAYOUT_VERSION);
  if (d_bytes < n) return OWQ_ERR_BUFFER_TOO_SMALL;
  uint8_t* host = new uint8_t[n];
  st = owq_tp_shard_host(full, FL, mode, world, rank, flags, host, n);
  if (st == OWQ_OK) {
    cudaStream_t cs = (cudaStream_t)stream;
    if (cudaMemcpyAsync(d_packed, host, n, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaStreamSynchronize(cs) != cudaSuccess)
      st = OWQ_ERR_CUDA;
  }
  delete[] host;
  return st;
}

// Workspace layout: [local GEMV workspace][row offsets (world+1) int32][buffer]
size_t owq_tp_workspace_bytes(const owq_shape* full, int mode, int world, int batch) {
  if (owq_packed_bytes(full) == 0 || world < 1 || batch < 1 || batch > OWQ_MAX_BATCH) return 0;
  owq_shape local = *full;
  size_t buf;
  if (mode == OWQ_TP_ROWS) {
    local.c_out = max_rows(full, world, nullptr);
    buf = (size_t)world * batch * local.c_out * 4;
  } else if (mode == OWQ_TP_COLS) {
    buf = (size_t)batch * full->c_out * 4;
  } else {
    return 0;
  }
  local.n_weak = 0;
  return align256(owq_workspace_bytes(&local, batch)) + align256((size_t)(world + 1) * 4) + align256(buf);
}

owq_status owq_tp_gemv(owq_tp* tp, int mode, const owq_shape* full, const owq_shape* shard,
                       const void* d_packed, const uint16_t* d_x, int B, void* d_y, int y_f32, void* d_ws,
                       size_t ws_bytes, void* stream) {
  if (!tp || !full || !shard || !d_y || !d_ws) return OWQ_ERR_INVALID_ARG;
  const size_t need = owq_tp_workspace_bytes(full, mode, tp->world, B);
  if (need == 0) return OWQ_ERR_INVALID_ARG;
  if (ws_bytes < need) return OWQ_ERR_BUFFER_TOO_SMALL;
  cudaStream_t cs = (cudaStream_t)stream;
  owq_shape local = *full;
  if (mode == OWQ_TP_ROWS) local.c_out = max_rows(full, tp->world, nullptr);
  local.n_weak = 0;
  const size_t lws = align256(owq_workspace_bytes(&local, B));
  void* buf = (uint8_t*)d_ws + lws + align256((size_t)(tp->world + 1) * 4);
  const int M = full->c_out;
  if (mode == OWQ_TP_ROWS) {
    int32_t offs[1025];
    if (tp->world > 1024) return OWQ_ERR_UNSUPPORTED;
    const int mmax = max_rows(full, tp->world, offs);
    if (shard->c_out != offs[tp->rank + 1] - offs[tp->rank] || shard->c_in != full->c_in) return OWQ_ERR_INVALID_ARG;
    const size_t esz = y_f32 ? 4 : 2;
    const size_t count = (size_t)B * mmax;
    const bool direct = B == 1 && (size_t)mmax * tp->world == (size_t)M;
    uint8_t* gbuf = direct ? (uint8_t*)d_y : (uint8_t*)buf;
    uint8_t* mine = gbuf + (size_t)tp->rank * count * esz;
    // local rows -> this rank's slot of the gather buffer (dense [B][m_r])
    owq_status st = owq_gemm_small_batch(shard, d_packed, d_x, B, mine, y_f32, d_ws, lws, stream);
    if (st != OWQ_OK) return st;
    if (ncclAllGather(mine, gbuf, count, y_f32 ? ncclFloat32 : ncclFloat16, tp->comm, cs) != ncclSuccess)
      return OWQ_ERR_NCCL;
    if (!direct) {
      const int64_t n = (int64_t)tp->world * B * mmax;
      const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
      if (y_f32)
        tp_scatter_rows<float><<<blocks, 256, 0, cs>>>((const float*)gbuf, (float*)d_y, tp->world, B, M, mmax);
      else
        tp_scatter_rows<__half><<<blocks, 256, 0, cs>>>((const __half*)gbuf, (__half*)d_y, tp->world, B, M, mmax);
      if (cudaGetLastError() != cudaSuccess) return OWQ_ERR_CUDA;
    }
    return OWQ_OK;
  }
  if (mode == OWQ_TP_COLS) {
    if (shard->c_out != M) return OWQ_ERR_INVALID_ARG;
    float* part = y_f32 ? (float*)d_y : (float*)buf;
    owq_status st = owq_gemm_small_batch(shard, d_packed, d_x, B, part, 1, d_ws, lws, stream);
    if (st != OWQ_OK) return st;
    if (ncclAllReduce(part, part, (size_t)B * M, ncclFloat32, ncclSum, tp->comm, cs) != ncclSuccess)
      return OWQ_ERR_NCCL;
    if (!y_f32) {
      const int64_t n = (int64_t)B * M;
      tp_f32_to_f16<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, cs>>>(part, (__half*)d_y, n);
      if (cudaGetLastError() != cudaSuccess) return OWQ_ERR_CUDA;
    }
    return OWQ_OK;
  }
  return OWQ_ERR_INVALID_ARG;
}

}  // extern "C"
