#!/usr/bin/env python
"""OWQ hot-path benchmark (BASELINE.json metric: OWQ 3.01-bit GEMV us and
achieved HBM GB/s, batch 1, OPT shapes).

Step = one pass of the whole hot path over one batch: the six linear layers of
an OPT-175B decoder layer (q, k, v, out: 12288x12288; fc1: 49152x12288;
fc2: 12288x49152) at 3.01 bits (3-bit codes, per-row fp16 scale/zero, k fp16
weak columns per layer from the paper's budget rule), batch 1.  The
weights are synthetic (seeded, synth/), packed once and resident in HBM.  The
682 MB of packed weights per step exceed the 126 MB L2, so every timed launch
streams from HBM (no flush needed).

N = 1  : the stack on one GPU, K steps unrolled into one CUDA graph with
         external timing events between launches (per-launch durations).
N > 1  : tensor parallel (torchrun, one process per GPU, NCCL): q, k, v, fc1
         row-sharded (outputs stay sharded, as in Megatron), out and fc2
         column-sharded with an NCCL all-reduce -- 2 collectives per step.
--impl reference : the CPU oracle (oracle/) on a bounded sample of the same
         workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "OWQ 3.01-bit GEMV µs and achieved HBM GB/s (vs ~8 TB/s), batch 1, OPT shapes"
UNIT = "GB/s"
NOMINAL_HBM_GBS = 8000.0
D = 12288
# (name, c_out, c_in, k): k = floor(0.01 * sum(MK) / 6 / (16 M + 16)) (reading s13);
# tests/test_bench_config.py pins these against oracle.budget_to_k.
LAYERS = [("q", D, D, 15), ("k", D, D, 15), ("v", D, D, 15), ("out", D, D, 15),
          ("fc1", 4 * D, D, 3), ("fc2", D, 4 * D, 15)]
BITS = 3
WORKLOAD = "opt175b_decoder_linear_stack_3.01bit"
# Megatron-style TP: which layers are row-split (no collective) vs column-split (+all-reduce)
TP_MODE = {"q": 0, "k": 0, "v": 0, "fc1": 0, "out": 1, "fc2": 1}


def algorithmic_bytes(M, K, k, B, bits=BITS, G=1):
    """codes (zero-filled weak columns included) + fp16 scale/zero +
    fp16 weak values + u16 indices + fp16 x + fp16 y."""
    return bits * M * K / 8 + 4 * M * G + 2 * M * k + 2 * k + 2 * K * B + 2 * M * B


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.index = index
        self.ok = False
        self.period = float(os.environ.get("BENCH_CLOCK_PERIOD_S", "0.002"))
        if os.environ.get("BENCH_NO_CLOCKS"):   # experiments only
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle sample
def oracle_sample(layers_host, rows_per_layer):
    """Oracle fp64 matvec (oracle.matvec_rows) on the first `rows_per_layer`
    rows of every layer; returns (seconds, algorithmic bytes of the sample)."""
    import oracle as O
    t_total, nbytes = 0.0, 0.0
    for (name, M, K, k), h in zip(LAYERS, layers_host):
        rep = O.Rep(M=rows_per_layer, K=K, bits=BITS, group=0, codes=h["codes"],
                    scale=O.from_fp16_bits(h["scale_f16"]), zero=O.from_fp16_bits(h["zero_f16"]),
                    weak_idx=h["weak_idx"].astype(np.int64), weak_val=O.from_fp16_bits(h["weak_val_f16"]))
        x = h["x"].astype(np.float64)
        t0 = time.perf_counter()
        O.matvec_rows(rep, x, range(rows_per_layer))
        t_total += time.perf_counter() - t0
        nbytes += algorithmic_bytes(rows_per_layer, K, k, x.shape[0])
    return t_total, nbytes


def host_sample(rows, batch):
    """Seeded sample rows of the workload for the CPU oracle (same generators)."""
    import synth
    out = []
    for i, (name, M, K, k) in enumerate(LAYERS):
        d = synth.representation(rows, K, BITS, 0, k, seed=synth.SEED_BASE + 100 * i)
        d["x"] = synth.activations(batch, K, seed=synth.SEED_BASE + 100 * i + 1, outliers=d["weak_idx"][:8])
        out.append(d)
    return out


def cpu_threads():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits
    except Exception:
        return None


def run_reference(args):
    """--impl reference: the oracle, as it stands, on a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    rows = args.ref_rows
    sample = host_sample(rows, args.batch)
    lim = cpu_threads()
    ctx = lim(limits=1) if lim else None
    if ctx:
        ctx.__enter__()
    for _ in range(args.warmup):
        oracle_sample(sample, rows)
    times, nb = [], 0.0
    for _ in range(args.steps):
        t, nb = oracle_sample(sample, rows)
        times.append(t)
    if ctx:
        ctx.__exit__(None, None, None)
    tot = sum(times)
    value = nb * args.steps / tot / 1e9
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "batch": args.batch,
                   "sample": f"first {rows} rows of each of the 6 layers per step"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"oracle.matvec_rows (fp64) on the first {rows} rows of each layer, 1 thread"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def build_layers(dev, batch, world, rank, keep_rows):
    import torch

    import paper_2306_02272_b200 as owq
    import synth
    layers, host_keep = [], []
    for i, (name, M, K, k) in enumerate(LAYERS):
        d = synth.representation(M, K, BITS, 0, k, seed=synth.SEED_BASE + 100 * i)
        x = synth.activations(batch, K, seed=synth.SEED_BASE + 100 * i + 1, outliers=d["weak_idx"][:8])
        if keep_rows:
            host_keep.append({"codes": d["codes"][:keep_rows].copy(), "scale_f16": d["scale_f16"][:keep_rows].copy(),
                              "zero_f16": d["zero_f16"][:keep_rows].copy(), "weak_idx": d["weak_idx"].copy(),
                              "weak_val_f16": d["weak_val_f16"][:keep_rows].copy(), "x": x.copy()})
        full = owq.Shape(M, K, BITS, 0, k)
        L = {"name": name, "M": M, "K": K, "k": k, "full": full}
        if world == 1:
            L["shape"] = full
            L["packed"] = owq.owq_pack(full, d, device=dev)
            L["x"] = torch.from_numpy(x).to(dev)
            L["y"] = torch.empty((batch, M), dtype=torch.float16, device=dev)
            L["ws"] = owq.workspace(full, batch, dev)
            L["bytes"] = algorithmic_bytes(M, K, k, batch)
        else:
            mode = TP_MODE[name]
            ss, packed = owq.owq_tp_shard(full, d, mode, world, rank, device=dev)
            a, b = owq.owq_tp_bounds(full, mode, world, rank)
            L.update(mode=mode, shape=ss, packed=packed, a=a, b=b)
            if mode == 0:
                L["x"] = torch.from_numpy(x).to(dev)
                L["y"] = torch.empty((batch, ss.c_out), dtype=torch.float16, device=dev)
                L["ws"] = owq.workspace(ss, batch, dev)
            else:
                L["x"] = torch.from_numpy(np.ascontiguousarray(x[:, a:b])).to(dev)
                L["y"] = torch.empty((batch, M), dtype=torch.float16, device=dev)
                L["ws"] = torch.zeros(owq.owq_tp_workspace_bytes(full, mode, world, batch), dtype=torch.uint8, device=dev)
            L["bytes"] = algorithmic_bytes(M, K, k, batch)   # whole-layer bytes; summed once over ranks below
        del d
        layers.append(L)
    return layers, host_keep


def graph_upload(g, stream) -> bool:
    """cudaGraphUpload: move the instantiated graph to the device before the timed
    region (otherwise the first replay pays the upload of every node)."""
    import ctypes
    import glob
    try:
        import torch
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
        rt = ctypes.CDLL(cands[0] if cands else "libcudart.so")
        rt.cudaGraphUpload.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        return rt.cudaGraphUpload(ctypes.c_void_p(g.raw_cuda_graph_exec()), ctypes.c_void_p(stream.cuda_stream)) == 0
    except Exception as e:  # pragma: no cover
        print(f"[bench] cudaGraphUpload unavailable ({e})", file=sys.stderr)
        return False


def launch(L, tp=None, stream=None):
    import paper_2306_02272_b200 as owq
    if L.get("grid"):
        owq.owq_gemm_small_batch_grid(L["shape"], L["packed"], L["x"], L["grid"], y=L["y"], ws=L["ws"], stream=stream)
    elif tp is None or L.get("mode", 0) == 0:
        owq.owq_gemm_small_batch(L["shape"], L["packed"], L["x"], y=L["y"], ws=L["ws"])
    else:
        owq.owq_tp_gemv(tp, L["mode"], L["full"], L["shape"], L["packed"], L["x"], L["y"], ws=L["ws"])


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2306_02272_b200 as owq
    from paper_2306_02272_b200.build import build
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    if rank == 0:
        build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    owq.lib()
    keep = args.ref_rows if (rank == 0 and not args.no_cpu) else 0
    layers, host_keep = build_layers(dev, args.batch, world, rank, keep)
    tp = None
    if world > 1:
        uid = owq.owq_tp_get_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        tp = owq.owq_tp_init(obj[0], world, rank)
    step_bytes = sum(L["bytes"] for L in layers)
    stream = torch.cuda.Stream(device=dev)
    # q, k, v are independent (one input, three weights): on one GPU they run
    # concurrently on three streams with a third of the SMs each, so their fixed
    # per-call costs (prologue, pipeline fill/drain, digit pass) overlap; out,
    # fc1, fc2 depend on their predecessors and run in order on all SMs.
    concurrent = world == 1 and not args.sequential
    side = [torch.cuda.Stream(device=dev) for _ in range(3)] if concurrent else []
    if concurrent:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        qkv = [L for L in layers if L["name"] in ("q", "k", "v")]
        for j, L in enumerate(qkv):
            L["grid"] = sms // 3 + (1 if j < sms % 3 else 0)
            L["ws_seq"] = L["ws"]
            L["ws"] = owq.workspace(L["shape"], args.batch, dev, grid=L["grid"])

    def step(ls=None):
        ls = layers if ls is None else ls
        if not concurrent:
            for L in ls:
                launch(L, tp)
            return
        cur = torch.cuda.current_stream()
        for sd in side:
            sd.wait_stream(cur)
        for sd, L in zip(side, [L for L in ls if L.get("grid")]):
            with torch.cuda.stream(sd):
                launch(L, tp, stream=sd)
        for sd in side:
            cur.wait_stream(sd)
        for L in ls:
            if not L.get("grid"):
                launch(L, tp)
    # eager warm-up (verifies blobs, sets kernel attributes) before capture
    with torch.cuda.stream(stream):
        for _ in range(2):
            step()
    torch.cuda.synchronize()

    K, W = args.steps, args.warmup
    n_l = len(layers)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    graph_ok = world == 1 and not args.no_graph
    g = None
    if graph_ok:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for s in range(K):
                    step()
            wg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(wg, stream=stream):
                for _ in range(max(W, 3)):
                    step()
        except Exception as e:  # pragma: no cover - fall back to eager timing
            print(f"[bench] graph capture failed ({e}); timing eager launches", file=sys.stderr)
            g = None
    uploaded = g is not None and graph_upload(g, stream) and graph_upload(wg, stream)
    torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        # warm-up (untimed)
        with torch.cuda.stream(stream):
            if g is not None:
                wg.replay()
            else:
                for _ in range(W):
                    step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # timed region: exactly K steps (device events on the launching stream)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            if g is not None:
                g.replay()
            else:
                for s in range(K):
                    step()
            ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    # per-launch durations (roofline): per layer shape, R back-to-back calls in one
    # graph over the same-shape layers in rotation (working set > L2), CUDA events
    # around the replay on the launching stream
    per_layer_ms = [None] * n_l
    shapes = {}
    for i, L in enumerate(layers):
        shapes.setdefault((L["M"], L["K"]), []).append(i)
    R = max(8, min(2 * K, 60))
    seq_view = []
    for L in layers:   # per-launch (roofline) timing: every layer on all SMs
        Lv = dict(L)
        Lv.pop("grid", None)
        if "ws_seq" in L:
            Lv["ws"] = L["ws_seq"]
        seq_view.append(Lv)
    for idx in shapes.values():
        pool = [seq_view[i] for i in idx]
        nbytes = sum(L["bytes"] for L in pool)
        # rotate over >= 3x L2 of distinct weights so every call streams from HBM:
        # extra packed copies for shapes that occur once per step (fc1, fc2)
        while nbytes < 3 * 126e6 and world == 1:
            L0 = pool[len(pool) % len(idx)]
            Lc = dict(L0)
            Lc["packed"] = L0["packed"].clone()
            pool.append(Lc)
            nbytes += L0["bytes"]
        seq = [pool[j % len(pool)] for j in range(R)]
        if graph_ok:
            pg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(pg, stream=stream):
                for L in seq:
                    launch(L, tp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for rep_ in range(2):   # first replay warms up
                e0.record(stream)
                if graph_ok:
                    pg.replay()
                else:
                    for L in seq:
                        launch(L, tp)
                e1.record(stream)
        torch.cuda.synchronize()
        for i in idx:
            per_layer_ms[i] = e0.elapsed_time(e1) / R
    ms_step = ms_total / K
    value = step_bytes / (ms_step * 1e-3) / 1e9

    # ---------------------------------------------------------------- e2e (host buffers)
    e2e = None
    if not args.no_e2e:
        # The step's inputs (every layer's x) sit in one pinned host buffer and go
        # to the device in one copy; the step's results (every layer's y) come back
        # in one copy; in between, the layers are eager public-API calls, one
        # after another on all SMs (the three-stream q/k/v schedule costs more
        # host time than it saves when not captured in a graph).
        eager = [dict(L) for L in (seq_view if world == 1 else layers)]
        nx = [L["x"].numel() for L in eager]
        ny = [L["y"].numel() for L in eager]
        xh_all = torch.empty(sum(nx), dtype=torch.float16).pin_memory()
        yh_all = torch.empty(sum(ny), dtype=torch.float16).pin_memory()
        xd_all = torch.empty(sum(nx), dtype=torch.float16, device=dev)
        yd_all = torch.empty(sum(ny), dtype=torch.float16, device=dev)
        ox = oy = 0
        for L, a, b in zip(eager, nx, ny):
            xh_all[ox:ox + a].copy_(L["x"].reshape(-1).cpu())
            L["x"] = xd_all[ox:ox + a].view(L["x"].shape)
            L["y"] = yd_all[oy:oy + b].view(L["y"].shape)
            ox += a
            oy += b
        h2d = xh_all.numel() * 2
        d2h = yh_all.numel() * 2
        E = max(3, min(K, 50))

        def e2e_step():
            xd_all.copy_(xh_all, non_blocking=True)
            for L in eager:
                launch(L, tp)
            yh_all.copy_(yd_all, non_blocking=True)
            stream.synchronize()   # the host reads the step's result

        with torch.cuda.stream(stream):
            for _ in range(3):
                e2e_step()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(E):
                e2e_step()
            dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": round(step_bytes * E / dt / 1e9, 2), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(1e3 * dt / E, 4), "path": "one pinned H2D copy of every layer's x, eager public-API calls (all SMs, in order), one D2H copy of every y"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---------------------------------------------------------------- roofline / cpu baseline
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs")
    per_layer = {L["name"]: {"us": round(1e3 * t, 3), "GBps": round(L["bytes"] / (t * 1e-3) / 1e9, 1),
                             "bytes": int(L["bytes"])} for L, t in zip(layers, per_layer_ms)}
    kern_ms = sum(per_layer_ms)
    achieved = step_bytes / (kern_ms * 1e-3) / 1e9 if world == 1 else value
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get("bytes_per_step") and tr["bytes_per_step"] / len(layers)
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4) if peak else None, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, measured)" if peak else "missing",
                "frac_of_nominal_8TBps": round(achieved / NOMINAL_HBM_GBS, 4),
                "per_launch": "per layer shape: R back-to-back calls in one CUDA graph timed with CUDA events; "
                              "a call = the x-digit pass + the fused GEMV (both counted, so achieved is conservative)"}
    cpu = None
    if not args.no_cpu and host_keep:
        lim = cpu_threads()
        ctx = lim(limits=1) if lim else None
        if ctx:
            ctx.__enter__()
        # repeat the sample until about args.cpu_seconds of CPU work (bounded: at most 64 passes)
        t, nb, passes = 0.0, 0.0, 0
        while passes < 64 and (passes == 0 or t < args.cpu_seconds):
            dt, dnb = oracle_sample(host_keep, args.ref_rows)
            t, nb, passes = t + dt, nb + dnb, passes + 1
        if ctx:
            ctx.__exit__(None, None, None)
        cpu = {"value": round(nb / t / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"oracle.matvec_rows (fp64) on the first {args.ref_rows} rows of each of the 6 layers, "
                         f"{passes} passes, 1 thread",
               "seconds": round(t, 3)}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8*s8->s32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "layers": [[n, M, K_, k] for n, M, K_, k in LAYERS],
                   "bits": BITS, "group_size": 0, "batch": args.batch,
                   "parallelism": f"tp{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (682 MB of packed weights per step vs 126 MB L2); no flush",
                   "graph": g is not None, "graph_uploaded_before_timing": bool(uploaded) if g is not None else None,
                   "schedule": ("q, k, v concurrently on 3 streams (a third of the SMs each); out, fc1, fc2 in order"
                                if concurrent else "all six layers in order on all SMs"),
                   "arith": "codes (u8) x exact int8 digits of x*2^24 on tcgen05.mma kind::i8, s32 accumulate; "
                            "zero point and digits combined exactly (fp64), fp32 scale; weak columns fp16 x fp16, fp32"},
        "us_per_layer": per_layer,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        # our kernels per step: per layer the x-digit pass + the fused GEMV (+ 1 fp32->fp16 convert
        # per column-split, all-reduced layer under TP; row-split layers keep sharded outputs)
        "gpu_launches": K * (2 * len(layers) + (sum(1 for L in layers if L.get("mode", 0) == 1) if world > 1 else 0)),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if tp is not None:
        owq.owq_tp_destroy(tp)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="owq", choices=["owq", "reference"])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ref-rows", type=int, default=1024)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU work for the cpu_baseline sample (repeated passes over --ref-rows rows per layer)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--sequential", action="store_true", help="q, k, v one after another on all SMs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
