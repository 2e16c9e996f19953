"""paper_2306_02272_b200 -- B200-native OWQ (arXiv 2306.02272) hot path.

Thin ctypes binding over ``libowq.so`` (include/owq.h).  Every function here
only marshals arguments: packing runs in the C++ packer, every step of the
GEMV runs in the sm_100a kernels.  There is no CPU fallback: importing works
without a GPU (the library loads), but any device call raises if CUDA or the
library is unavailable.

Names mirror the C ABI (owq_pack, owq_gemv, owq_gemm_small_batch, owq_tp_gemv,
...).  Device buffers are torch tensors; the stream is torch's current stream
unless one is passed.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "OwqError", "Shape", "lib", "canonical_pack", "owq_packed_bytes", "owq_pack_host",
    "owq_pack", "owq_blob_decode_host", "owq_unpack_codes", "owq_workspace_bytes",
    "workspace", "owq_gemv", "owq_gemm_small_batch", "owq_gemm_small_batch_grid",
    "owq_tp_get_unique_id", "owq_tp_init", "owq_tp_destroy", "owq_tp_bounds",
    "owq_tp_shard_shape", "owq_tp_shard_host", "owq_tp_shard", "owq_tp_workspace_bytes",
    "owq_tp_gemv", "OwqLinear", "OWQ_TP_ROWS", "OWQ_TP_COLS", "OWQ_PACK_STRICT",
    "OWQ_PACK_U8_CODES", "OWQ_PACK_LAYOUT_CC", "OWQ_LAYOUT_TC", "OWQ_LAYOUT_CC",
    "owq_packed_bytes_layout", "owq_workspace_bytes_grid", "owq_packed_bytes_colmap", "owq_pack_host_colmap",
    "owq_pack_colmap", "owq_blob_colmap_host", "choose_layout", "owq_quantize_gpu",
    "owq_quantize_workspace_bytes", "owq_gemm_prefill", "owq_gemm_batch_f16", "owq_tp_check",
    "owq_prefill_workspace_bytes", "prefill_workspace", "EXPORTED_SYMBOLS",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OWQ_LIB") or os.path.join(HERE, "libowq.so")   # OWQ_LIB: A/B experiments only

OWQ_TP_ROWS, OWQ_TP_COLS = 0, 1
OWQ_PACK_STRICT, OWQ_PACK_U8_CODES, OWQ_PACK_LAYOUT_CC = 1, 2, 4
OWQ_LAYOUT_TC, OWQ_LAYOUT_CC = 3, 4     # device layouts: tensor-core (tcgen05) / CUDA-core

# every symbol include/owq.h declares
EXPORTED_SYMBOLS = [
    "owq_packed_bytes", "owq_packed_bytes_layout", "owq_pack_host", "owq_pack", "owq_blob_decode_host",
    "owq_unpack_codes", "owq_workspace_bytes", "owq_workspace_bytes_grid", "owq_gemv", "owq_gemm_small_batch",
    "owq_gemm_small_batch_grid", "owq_tp_get_unique_id", "owq_tp_init", "owq_tp_destroy",
    "owq_tp_shard_shape", "owq_tp_shard_host", "owq_tp_shard", "owq_tp_workspace_bytes",
    "owq_tp_gemv", "owq_tp_bounds", "owq_status_string", "owq_packed_bytes_colmap",
    "owq_pack_host_colmap", "owq_pack_colmap", "owq_blob_colmap_host",
    "owq_quantize_workspace_bytes", "owq_quantize_gpu", "owq_gemm_prefill", "owq_gemm_batch_f16",
    "owq_tp_check", "owq_gemm_prefill_ws", "owq_prefill_workspace_bytes",
]


class OwqError(RuntimeError):
    pass


class Shape(ctypes.Structure):
    _fields_ = [("c_out", ctypes.c_int32), ("c_in", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("group_size", ctypes.c_int32), ("n_weak", ctypes.c_int32)]

    def __repr__(self):
        return (f"Shape(c_out={self.c_out}, c_in={self.c_in}, bits={self.bits}, "
                f"group_size={self.group_size}, n_weak={self.n_weak})")

    def tup(self):
        return (self.c_out, self.c_in, self.bits, self.group_size, self.n_weak)


class _QuantParams(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int32), ("group_size", ctypes.c_int32), ("n_weak", ctypes.c_int32),
                ("clip", ctypes.c_int32), ("percdamp", ctypes.c_double)]


class _ColMap(ctypes.Structure):
    _fields_ = [("k_stored", ctypes.c_int32), ("colmap", ctypes.c_void_p)]


class _HostLayer(ctypes.Structure):
    _fields_ = [("codes", ctypes.c_void_p), ("scale", ctypes.c_void_p), ("zero", ctypes.c_void_p),
                ("weak_idx", ctypes.c_void_p), ("weak_val", ctypes.c_void_p)]


_lib = None
_P = ctypes.c_void_p
_S = ctypes.POINTER(Shape)


def lib():
    """Load libowq.so (built in-tree by __graft_entry__.build()); fail loudly."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OwqError(f"{LIB_PATH} is missing: run `python -m paper_2306_02272_b200.build` "
                       "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    st = ctypes.c_int
    sz = ctypes.c_size_t
    sig = {
        "owq_packed_bytes": (sz, [_S]),
        "owq_packed_bytes_layout": (sz, [_S, ctypes.c_int]),
        "owq_workspace_bytes_grid": (sz, [_S, ctypes.c_int, ctypes.c_int]),
        "owq_pack_host": (st, [_S, ctypes.POINTER(_HostLayer), ctypes.c_int, _P, sz]),
        "owq_pack": (st, [_S, ctypes.POINTER(_HostLayer), ctypes.c_int, _P, sz, _P]),
        "owq_blob_decode_host": (st, [_P, sz, _S, _P, _P, _P, _P, _P]),
        "owq_unpack_codes": (st, [_S, _P, _P, _P]),
        "owq_workspace_bytes": (sz, [_S, ctypes.c_int]),
        "owq_gemv": (st, [_S, _P, _P, _P, ctypes.c_int, _P, sz, _P]),
        "owq_gemm_small_batch": (st, [_S, _P, _P, ctypes.c_int, _P, ctypes.c_int, _P, sz, _P]),
        "owq_gemm_small_batch_grid": (st, [_S, _P, _P, ctypes.c_int, _P, ctypes.c_int, _P, sz,
                                           ctypes.c_int, _P]),
        "owq_tp_get_unique_id": (st, [_P]),
        "owq_tp_init": (st, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
        "owq_tp_destroy": (st, [_P]),
        "owq_tp_check": (st, [_P]),
        "owq_tp_bounds": (st, [_S, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
        "owq_tp_shard_shape": (st, [_S, ctypes.POINTER(_HostLayer), ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _S, ctypes.POINTER(ctypes.c_int32)]),
        "owq_tp_shard_host": (st, [_S, ctypes.POINTER(_HostLayer), ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, _P, sz]),
        "owq_tp_shard": (st, [_S, ctypes.POINTER(_HostLayer), ctypes.c_int, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, _P, sz, _P]),
        "owq_tp_workspace_bytes": (sz, [_S, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "owq_tp_gemv": (st, [_P, ctypes.c_int, _S, _S, _P, _P, ctypes.c_int, _P, ctypes.c_int,
                             _P, sz, _P]),
        "owq_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "owq_packed_bytes_colmap": (sz, [_S, ctypes.POINTER(_ColMap)]),
        "owq_pack_host_colmap": (st, [_S, ctypes.POINTER(_HostLayer), ctypes.POINTER(_ColMap), ctypes.c_int, _P, sz]),
        "owq_pack_colmap": (st, [_S, ctypes.POINTER(_HostLayer), ctypes.POINTER(_ColMap), ctypes.c_int, _P, sz, _P]),
        "owq_blob_colmap_host": (st, [_P, sz, ctypes.POINTER(ctypes.c_int32), _P]),
        "owq_gemm_prefill": (st, [_S, _P, _P, ctypes.c_int32, _P, ctypes.c_int, _P]),
        "owq_gemm_prefill_ws": (st, [_S, _P, _P, ctypes.c_int32, _P, ctypes.c_int, _P, sz, _P]),
        "owq_prefill_workspace_bytes": (sz, [_S, ctypes.c_int32]),
        "owq_gemm_batch_f16": (st, [_S, _P, _P, ctypes.c_int, _P, ctypes.c_int, _P, sz, _P]),
        "owq_quantize_workspace_bytes": (sz, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.POINTER(_QuantParams)]),
        "owq_quantize_gpu": (st, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P,
                                  ctypes.POINTER(_QuantParams), _P, _P, _P, _P, _P, _P, sz, _P]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("OWQ_LIB") and not hasattr(L, name):
            continue   # A/B experiments against an older library: its missing entry points stay unusable
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status):
    if status != 0:
        raise OwqError(lib().owq_status_string(status).decode())


def _shape(s) -> Shape:
    if isinstance(s, Shape):
        return s
    if isinstance(s, dict):
        return Shape(s["M"], s["K"], s["bits"], s["group"], len(s["weak_idx"]))
    return Shape(*s)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream(stream):
    import torch
    if stream is None:
        # the current stream's raw handle without the Python Stream object
        # (torch.cuda.current_stream() costs several microseconds per call)
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            return raw(torch._C._cuda_getDevice())
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def canonical_pack(codes: np.ndarray, bits: int) -> np.ndarray:
    """One code per byte [M][K] -> the paper-side canonical stream (row-major,
    LSB-first, rows byte-padded)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    M, K = codes.shape
    planes = ((codes[:, :, None] >> np.arange(bits, dtype=np.uint8)) & 1).reshape(M, K * bits)
    return np.packbits(planes, axis=1, bitorder="little")


@dataclass
class _HostArrays:
    layer: _HostLayer
    keep: tuple


def _host_layer(codes, scale, zero, weak_idx, weak_val) -> _HostArrays:
    arrs = [np.ascontiguousarray(codes, dtype=np.uint8),
            np.ascontiguousarray(scale, dtype=np.uint16),
            np.ascontiguousarray(zero, dtype=np.uint16),
            np.ascontiguousarray(weak_idx, dtype=np.uint16),
            np.ascontiguousarray(weak_val, dtype=np.uint16)]
    L = _HostLayer(*[a.ctypes.data if a.size else None for a in arrs])
    return _HostArrays(L, tuple(arrs))


def _layer_from(rep: dict, flags: int):
    """rep: dict with codes (u8 [M][K] one per byte, or canonical if `canonical`),
    scale_f16/zero_f16/weak_val_f16 (u16 bit patterns), weak_idx (u16)."""
    canonical = rep.get("canonical", False)
    if not canonical:
        flags |= OWQ_PACK_U8_CODES
    return _host_layer(rep["codes"], rep["scale_f16"], rep["zero_f16"], rep["weak_idx"],
                       rep["weak_val_f16"]), flags


def owq_packed_bytes(shape) -> int:
    return int(lib().owq_packed_bytes(ctypes.byref(_shape(shape))))


def owq_packed_bytes_layout(shape, layout: int) -> int:
    return int(lib().owq_packed_bytes_layout(ctypes.byref(_shape(shape)), int(layout)))


def _layout_of(flags: int) -> int:
    return OWQ_LAYOUT_CC if flags & OWQ_PACK_LAYOUT_CC else OWQ_LAYOUT_TC


def owq_pack_host(shape, rep: dict, flags: int = 0) -> np.ndarray:
    s = _shape(shape)
    n = owq_packed_bytes_layout(s, _layout_of(flags))
    if n == 0:
        raise OwqError("OWQ_ERR_UNSUPPORTED")
    blob = np.empty(n, dtype=np.uint8)
    hl, flags = _layer_from(rep, flags)
    _check(lib().owq_pack_host(ctypes.byref(s), ctypes.byref(hl.layer), flags, blob.ctypes.data, n))
    return blob


def owq_pack(shape, rep: dict, flags: int = 0, device=None, stream=None):
    import torch
    s = _shape(shape)
    n = owq_packed_bytes_layout(s, _layout_of(flags))
    if n == 0:
        raise OwqError("OWQ_ERR_UNSUPPORTED")
    d = torch.empty(n, dtype=torch.uint8, device=device or "cuda")
    hl, flags = _layer_from(rep, flags)
    with torch.cuda.device(d.device):
        _check(lib().owq_pack(ctypes.byref(s), ctypes.byref(hl.layer), flags, d.data_ptr(), n,
                              _stream(stream)))
    return d


def _colmap(colmap):
    cm = np.ascontiguousarray(colmap, dtype=np.uint16)
    return _ColMap(int(cm.size), cm.ctypes.data), cm


def owq_packed_bytes_colmap(shape, colmap) -> int:
    m, keep = _colmap(colmap)
    return int(lib().owq_packed_bytes_colmap(ctypes.byref(_shape(shape)), ctypes.byref(m)))


def owq_pack_host_colmap(shape, rep: dict, colmap, flags: int = 0) -> np.ndarray:
    """NEXT-4 variants (act-order / storage-favored): rep["codes"] is [c_out][k_stored]
    in stored order, colmap[p] = original column of stored position p."""
    s = _shape(shape)
    m, keep = _colmap(colmap)
    n = int(lib().owq_packed_bytes_colmap(ctypes.byref(s), ctypes.byref(m)))
    if n == 0:
        raise OwqError("OWQ_ERR_INVALID_ARG (shape / column map)")
    blob = np.empty(n, dtype=np.uint8)
    hl, flags = _layer_from(rep, flags)
    _check(lib().owq_pack_host_colmap(ctypes.byref(s), ctypes.byref(hl.layer), ctypes.byref(m), flags,
                                      blob.ctypes.data, n))
    return blob


def owq_pack_colmap(shape, rep: dict, colmap, flags: int = 0, device=None, stream=None):
    import torch
    s = _shape(shape)
    m, keep = _colmap(colmap)
    n = int(lib().owq_packed_bytes_colmap(ctypes.byref(s), ctypes.byref(m)))
    if n == 0:
        raise OwqError("OWQ_ERR_INVALID_ARG (shape / column map)")
    d = torch.empty(n, dtype=torch.uint8, device=device or "cuda")
    hl, flags = _layer_from(rep, flags)
    with torch.cuda.device(d.device):
        _check(lib().owq_pack_colmap(ctypes.byref(s), ctypes.byref(hl.layer), ctypes.byref(m), flags,
                                     d.data_ptr(), n, _stream(stream)))
    return d


def owq_blob_colmap_host(blob: np.ndarray):
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    ks = ctypes.c_int32()
    _check(lib().owq_blob_colmap_host(blob.ctypes.data, blob.size, ctypes.byref(ks), None))
    cm = np.zeros(ks.value, np.uint16)
    _check(lib().owq_blob_colmap_host(blob.ctypes.data, blob.size, ctypes.byref(ks), cm.ctypes.data))
    return cm


def owq_blob_decode_host(blob: np.ndarray) -> dict:
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    s = Shape()
    _check(lib().owq_blob_decode_host(blob.ctypes.data, blob.size, ctypes.byref(s),
                                      None, None, None, None, None))
    M, K = s.c_out, s.c_in
    if int(blob[:8].view(np.uint32)[1]) == OWQ_LAYOUT_CC:
        K = owq_blob_colmap_host(blob).size          # stored columns
    G = 1 if s.group_size == 0 else -(-K // s.group_size)
    out = {"shape": s, "codes": np.zeros((M, K), np.uint8), "scale_f16": np.zeros((M, G), np.uint16),
           "zero_f16": np.zeros((M, G), np.uint16), "weak_idx": np.zeros(s.n_weak, np.uint16),
           "weak_val_f16": np.zeros((M, s.n_weak), np.uint16)}
    _check(lib().owq_blob_decode_host(blob.ctypes.data, blob.size, ctypes.byref(s),
                                      *[_ptr(out[k]) if out[k].size else None for k in
                                        ("codes", "scale_f16", "zero_f16", "weak_idx", "weak_val_f16")]))
    return out


def owq_unpack_codes(shape, d_packed, stream=None):
    import torch
    s = _shape(shape)
    out = torch.empty((s.c_out, s.c_in), dtype=torch.uint8, device=d_packed.device)
    _check(lib().owq_unpack_codes(ctypes.byref(s), d_packed.data_ptr(), out.data_ptr(), _stream(stream)))
    return out


def owq_workspace_bytes(shape, batch: int = 1) -> int:
    return int(lib().owq_workspace_bytes(ctypes.byref(_shape(shape)), batch))


def owq_workspace_bytes_grid(shape, batch: int = 1, grid: int = 0) -> int:
    return int(lib().owq_workspace_bytes_grid(ctypes.byref(_shape(shape)), batch, grid))


def workspace(shape, batch: int = 1, device=None, grid: int = 0):
    """Zero-filled workspace (every call leaves its stream-K slots and counters
    at zero again, so one workspace serves sequential calls of any shapes).
    The size comes from the C ABI (owq_workspace_bytes_grid) on `device`."""
    import torch
    dev = torch.device(device or "cuda")
    with torch.cuda.device(dev):
        n = owq_workspace_bytes_grid(shape, batch, grid)
    if n == 0:
        raise OwqError("OWQ_ERR_UNSUPPORTED (workspace for this shape / batch / grid)")
    return torch.zeros(max(n, 256), dtype=torch.uint8, device=dev)


def _out(s: Shape, B: int, y, y_f32: bool, device):
    import torch
    if y is None:
        y = torch.empty((B, s.c_out), dtype=torch.float32 if y_f32 else torch.float16, device=device)
    return y


def _check_io(s: Shape, d_packed, x, y, y_f32: bool, B: int, ws):
    """Every tensor the C ABI will dereference: dtype, contiguity, shape and
    device (the ABI takes raw pointers, so a wrong tensor would otherwise be
    read or written out of bounds)."""
    import torch
    dev = d_packed.device
    if d_packed.dtype != torch.uint8 or not d_packed.is_contiguous():
        raise OwqError("packed blob must be a contiguous uint8 tensor")
    if x.dtype != torch.float16:
        raise OwqError(f"x must be float16, got {x.dtype}")
    if x.device != dev:
        raise OwqError(f"x is on {x.device}, the layer on {dev}")
    if not x.is_contiguous():
        raise OwqError("x must be contiguous (row-major [B][c_in])")
    if tuple(x.shape) not in ((B, s.c_in),) and not (x.dim() == 1 and B == 1 and x.shape[0] == s.c_in):
        raise OwqError(f"x must be [{B}][{s.c_in}], got {tuple(x.shape)}")
    want = torch.float32 if y_f32 else torch.float16
    if y.dtype != want:
        raise OwqError(f"y must be {want} (y_f32={bool(y_f32)}), got {y.dtype}")
    if y.device != dev or not y.is_contiguous():
        raise OwqError("y must be contiguous and on the layer's device")
    if y.numel() != B * s.c_out:
        raise OwqError(f"y must hold [{B}][{s.c_out}] elements, got {tuple(y.shape)}")
    if ws is not None and (ws.device != dev or ws.dtype != torch.uint8 or not ws.is_contiguous()):
        raise OwqError("workspace must be a contiguous uint8 tensor on the layer's device")


def _on_device(dev):
    """torch.cuda.device(dev) unless dev is already current (saves ~2 us per call)."""
    import contextlib
    import torch
    if dev.index is None or dev.index == torch._C._cuda_getDevice():
        return contextlib.nullcontext()
    return torch.cuda.device(dev)


def owq_gemv(shape, d_packed, x, y=None, y_f32=False, ws=None, stream=None):
    """y = W_hat x for one fp16 vector x [c_in] (or [1][c_in]); returns y [1][c_out]."""
    s = _shape(shape)
    y = _out(s, 1, y, y_f32, x.device)
    _check_io(s, d_packed, x, y, y_f32, 1, ws)
    with _on_device(d_packed.device):
        ws = ws if ws is not None else workspace(s, 1, x.device)
        _check(lib().owq_gemv(ctypes.byref(s), d_packed.data_ptr(), x.data_ptr(), y.data_ptr(),
                              int(bool(y_f32)), ws.data_ptr(), ws.numel(), _stream(stream)))
    return y


def owq_gemm_small_batch(shape, d_packed, x, y=None, y_f32=False, ws=None, stream=None):
    """Y = W_hat X for fp16 X [B][c_in], B in [1, 16]; returns Y [B][c_out]."""
    s = _shape(shape)
    B = x.shape[0] if x.dim() == 2 else 1
    y = _out(s, B, y, y_f32, x.device)
    _check_io(s, d_packed, x, y, y_f32, B, ws)
    with _on_device(d_packed.device):
        ws = ws if ws is not None else workspace(s, B, x.device)
        _check(lib().owq_gemm_small_batch(ctypes.byref(s), d_packed.data_ptr(), x.data_ptr(), B,
                                          y.data_ptr(), int(bool(y_f32)), ws.data_ptr(), ws.numel(),
                                          _stream(stream)))
    return y


def owq_gemm_batch_f16(shape, d_packed, x, y=None, y_f32=False, ws=None, stream=None):
    """Y = W_hat X for fp16 X [B][c_in], B in [1, 32], on tensor cores with the exact
    (q - z) fp16 A operand (layout-3 blobs)."""
    s = _shape(shape)
    B = x.shape[0] if x.dim() == 2 else 1
    y = _out(s, B, y, y_f32, x.device)
    _check_io(s, d_packed, x, y, y_f32, B, ws)
    with _on_device(d_packed.device):
        ws = ws if ws is not None else workspace(s, min(max(B, 2), 16), x.device)
        _check(lib().owq_gemm_batch_f16(ctypes.byref(s), d_packed.data_ptr(), x.data_ptr(), B, y.data_ptr(),
                                        int(bool(y_f32)), ws.data_ptr(), ws.numel(), _stream(stream)))
    return y


def owq_prefill_workspace_bytes(shape, n_tokens: int) -> int:
    return int(lib().owq_prefill_workspace_bytes(ctypes.byref(_shape(shape)), int(n_tokens)))


def prefill_workspace(shape, n_tokens: int, device=None):
    """Scratch workspace for owq_gemm_prefill(..., ws=...) (K-split partial rows),
    or None when no split would be used at this token count."""
    import torch
    dev = torch.device(device or "cuda")
    with torch.cuda.device(dev):
        n = owq_prefill_workspace_bytes(shape, n_tokens)
    return torch.empty(n, dtype=torch.uint8, device=dev) if n else None


def owq_gemm_prefill(shape, d_packed, x, y=None, y_f32=False, ws=None, stream=None):
    """Y = W_hat X for fp16 X [n_tokens][c_in], any n_tokens (NEXT-2, tensor cores,
    layout-3 blobs with per-row scales); returns Y [n_tokens][c_out].  K is split
    into pieces of <= 4096 columns (precision) and, for few tokens on few rows,
    over more CTAs; the scratch comes from `ws` (prefill_workspace) or is
    allocated per call."""
    s = _shape(shape)
    B = x.shape[0] if x.dim() == 2 else 1
    y = _out(s, B, y, y_f32, x.device)
    _check_io(s, d_packed, x, y, y_f32, B, None)
    with _on_device(d_packed.device):
        if ws is None:
            ws = prefill_workspace(s, B, x.device)   # None when K needs no split
        if ws is None:
            _check(lib().owq_gemm_prefill(ctypes.byref(s), d_packed.data_ptr(), x.data_ptr(), B, y.data_ptr(),
                                          int(bool(y_f32)), _stream(stream)))
        else:
            if ws.device != x.device or ws.dtype.itemsize != 1 or not ws.is_contiguous():
                raise OwqError("OWQ_ERR_INVALID_ARG: prefill workspace must be a contiguous byte tensor on x's device")
            _check(lib().owq_gemm_prefill_ws(ctypes.byref(s), d_packed.data_ptr(), x.data_ptr(), B, y.data_ptr(),
                                             int(bool(y_f32)), ws.data_ptr(), ws.numel(), _stream(stream)))
    return y


def owq_gemm_small_batch_grid(shape, d_packed, x, grid: int, y=None, y_f32=False, ws=None, stream=None):
    s = _shape(shape)
    B = x.shape[0] if x.dim() == 2 else 1
    y = _out(s, B, y, y_f32, x.device)
    _check_io(s, d_packed, x, y, y_f32, B, ws)
    with _on_device(d_packed.device):
        ws = ws if ws is not None else workspace(s, B, x.device, grid=grid)
        _check(lib().owq_gemm_small_batch_grid(ctypes.byref(s), d_packed.data_ptr(), x.data_ptr(), B,
                                               y.data_ptr(), int(bool(y_f32)), ws.data_ptr(), ws.numel(),
                                               grid, _stream(stream)))
    return y


# ---------------------------------------------------------------- tensor parallel
def owq_tp_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().owq_tp_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def owq_tp_init(uid: bytes, world: int, rank: int):
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    h = ctypes.c_void_p()
    _check(lib().owq_tp_init(ctypes.cast(buf, ctypes.c_void_p), world, rank, ctypes.byref(h)))
    return h


def owq_tp_check(h):
    """Raise OwqError if an NCCL collective of this communicator failed (non-blocking poll)."""
    _check(lib().owq_tp_check(h))


def owq_tp_destroy(h):
    _check(lib().owq_tp_destroy(h))


def owq_tp_bounds(shape, mode: int, world: int, rank: int):
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().owq_tp_bounds(ctypes.byref(_shape(shape)), mode, world, rank, ctypes.byref(a),
                               ctypes.byref(b)))
    return a.value, b.value


def owq_tp_shard_shape(shape, rep: dict, mode: int, world: int, rank: int):
    s = _shape(shape)
    hl, flags = _layer_from(rep, 0)
    out, off = Shape(), ctypes.c_int32()
    _check(lib().owq_tp_shard_shape(ctypes.byref(s), ctypes.byref(hl.layer), mode, world, rank,
                                    ctypes.byref(out), ctypes.byref(off)))
    return out, off.value


def owq_tp_shard_host(shape, rep: dict, mode: int, world: int, rank: int, flags: int = 0):
    s = _shape(shape)
    ss, _ = owq_tp_shard_shape(s, rep, mode, world, rank)
    n = owq_packed_bytes(ss)
    blob = np.empty(n, np.uint8)
    hl, flags = _layer_from(rep, flags)
    _check(lib().owq_tp_shard_host(ctypes.byref(s), ctypes.byref(hl.layer), mode, world, rank, flags,
                                   blob.ctypes.data, n))
    return ss, blob


def owq_tp_shard(shape, rep: dict, mode: int, world: int, rank: int, flags: int = 0, device=None,
                 stream=None):
    import torch
    s = _shape(shape)
    ss, _ = owq_tp_shard_shape(s, rep, mode, world, rank)
    n = owq_packed_bytes(ss)
    d = torch.empty(n, dtype=torch.uint8, device=device or "cuda")
    hl, flags = _layer_from(rep, flags)
    _check(lib().owq_tp_shard(ctypes.byref(s), ctypes.byref(hl.layer), mode, world, rank, flags,
                              d.data_ptr(), n, _stream(stream)))
    return ss, d


def owq_tp_workspace_bytes(shape, mode: int, world: int, batch: int = 1) -> int:
    return int(lib().owq_tp_workspace_bytes(ctypes.byref(_shape(shape)), mode, world, batch))


def owq_tp_gemv(tp, mode, full, shard, d_packed, x, y, y_f32=False, ws=None, stream=None):
    f, s = _shape(full), _shape(shard)
    B = x.shape[0] if x.dim() == 2 else 1
    _check(lib().owq_tp_gemv(tp, mode, ctypes.byref(f), ctypes.byref(s), d_packed.data_ptr(),
                             x.data_ptr(), B, y.data_ptr(), int(bool(y_f32)), ws.data_ptr(),
                             ws.numel(), _stream(stream)))
    return y


def owq_quantize_workspace_bytes(c_out: int, c_in: int, n_samples: int, bits: int, n_weak: int,
                                 group: int = 0, clip: bool = True, percdamp: float = 0.01) -> int:
    prm = _QuantParams(bits, group, n_weak, int(bool(clip)), percdamp)
    return int(lib().owq_quantize_workspace_bytes(c_out, c_in, n_samples, ctypes.byref(prm)))


def owq_quantize_gpu(W, X, bits: int, n_weak: int, group: int = 0, clip: bool = True, percdamp: float = 0.01,
                     stream=None) -> dict:
    """OWQ quantization on the GPU (NEXT-1, owq.h owq_quantize_gpu): W fp64 [c_out][c_in],
    calibration X fp64 [c_in][n_samples], both contiguous CUDA tensors.  Returns the
    paper representation as CUDA tensors: codes u8 [M][K], scale_f16 / zero_f16 u16
    bit patterns [M][G], weak_idx u16 [k], weak_val_f16 u16 [M][k]."""
    import torch
    if W.dtype != torch.float64 or X.dtype != torch.float64 or not W.is_cuda or W.device != X.device:
        raise OwqError("W and X must be float64 CUDA tensors on one device")
    W, X = W.contiguous(), X.contiguous()
    M, K = W.shape
    if X.shape[0] != K:
        raise OwqError(f"X must be [{K}][n_samples], got {tuple(X.shape)}")
    N = X.shape[1]
    G = 1 if group == 0 else -(-K // group)
    dev = W.device
    out = {"codes": torch.empty((M, K), dtype=torch.uint8, device=dev),
           "scale_f16": torch.empty((M, G), dtype=torch.int16, device=dev),
           "zero_f16": torch.empty((M, G), dtype=torch.int16, device=dev),
           "weak_idx": torch.empty(max(n_weak, 1), dtype=torch.int16, device=dev),
           "weak_val_f16": torch.empty((M, max(n_weak, 1)), dtype=torch.int16, device=dev)}
    prm = _QuantParams(bits, group, n_weak, int(bool(clip)), percdamp)
    with _on_device(dev):
        nws = int(lib().owq_quantize_workspace_bytes(M, K, N, ctypes.byref(prm)))
        if nws == 0:
            raise OwqError("OWQ_ERR_INVALID_ARG (quantizer shape)")
        ws = torch.empty(nws, dtype=torch.uint8, device=dev)
        _check(lib().owq_quantize_gpu(M, K, N, W.data_ptr(), X.data_ptr(), ctypes.byref(prm),
                                      out["codes"].data_ptr(), out["scale_f16"].data_ptr(),
                                      out["zero_f16"].data_ptr(), out["weak_idx"].data_ptr(),
                                      out["weak_val_f16"].data_ptr(), ws.data_ptr(), nws, _stream(stream)))
    out["weak_idx"] = out["weak_idx"][:n_weak]
    out["weak_val_f16"] = out["weak_val_f16"][:, :n_weak]
    out.update(M=M, K=K, bits=bits, group=group)
    return out


def choose_layout(shape, max_batch: int = 1) -> int:
    """Device layout to pack a layer for, from the measured crossover on B200
    (profiles/r2_layout_table.txt): the CUDA-core kernel
    (layout 4) for batch-1 decode of grouped-scale layers and of layers up to
    ~48 M weights (lower fixed cost per call); the tcgen05 kernel (layout 3)
    for larger per-row layers and for batches > 1 (tensor cores)."""
    s = _shape(shape)
    if max_batch > 1:
        return OWQ_LAYOUT_TC
    if s.group_size > 0 or s.c_out * s.c_in <= 48 * 1024 * 1024:
        return OWQ_LAYOUT_CC
    return OWQ_LAYOUT_TC


class OwqLinear:
    """A packed OWQ layer resident in HBM: ``y = layer(x)`` (x fp16 [B][c_in])."""

    def __init__(self, rep: dict, device=None, max_batch: int = 16, flags: int = 0, layout: int = None):
        """layout: OWQ_LAYOUT_TC (tcgen05 kernel) or OWQ_LAYOUT_CC (CUDA-core kernel);
        None = choose_layout(shape, max_batch)."""
        import torch
        self.shape = _shape((rep["M"], rep["K"], rep["bits"], rep["group"], len(rep["weak_idx"])))
        self.device = torch.device(device or "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        if layout is None:
            layout = choose_layout(self.shape, max_batch)
        if layout == OWQ_LAYOUT_CC:
            flags |= OWQ_PACK_LAYOUT_CC
        self.layout = layout
        if rep.get("colmap") is not None:      # NEXT-4 variants: layout 4 with a column map
            self.layout = OWQ_LAYOUT_CC
            self.packed = owq_pack_colmap(self.shape, rep, rep["colmap"], flags, device=self.device)
        else:
            self.packed = owq_pack(self.shape, rep, flags, device=self.device)
        self.ws = workspace(self.shape, max_batch, self.device)

    @property
    def nbytes(self) -> int:
        return self.packed.numel()

    def __call__(self, x, y=None, y_f32=False, stream=None):
        if x.dim() == 1:
            x = x.unsqueeze(0)
        return owq_gemm_small_batch(self.shape, self.packed, x, y=y, y_f32=y_f32, ws=self.ws,
                                    stream=stream)
