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
    """Seeded sample rows of the workload for the CPU oracle (same generators;
    q, k and v share one input, as in the GPU arm)."""
    import synth
    out = []
    for i, (name, M, K, k) in enumerate(LAYERS):
        d = synth.representation(rows, K, BITS, 0, k, seed=synth.SEED_BASE + 100 * i)
        if name in ("k", "v"):
            d["x"] = out[0]["x"]
        else:
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
# BASELINE configs measured beside the headline (per-layer device time, the
# layout choose_layout() picks; parity-test shapes, reported, not the headline)
SECONDARY = {
    "opt6.7b_3.01bit_b1": [("qkvo", 4096, 4096, 3, 0, 5, 1), ("fc1", 16384, 4096, 3, 0, 1, 1),
                           ("fc2", 4096, 16384, 3, 0, 5, 1)],
    "llama7b_4bit_g128": [(f"{n}_b{B}", M, K, 4, 128, k, B) for B in (1, 4, 8, 16)
                          for n, M, K, k in (("qkvo", 4096, 4096, 4), ("up", 11008, 4096, 1), ("down", 4096, 11008, 4))],
    "opt66b_3.01bit_b1": [("qkvo", 9216, 9216, 3, 0, 11, 1), ("fc1", 36864, 9216, 3, 0, 2, 1),
                          ("fc2", 9216, 36864, 3, 0, 11, 1)],
}


def build_layers(dev, batch, world, rank, keep_rows, layout_override=None):
    import torch

    import paper_2306_02272_b200 as owq
    import synth
    layers, host_keep = [], []
    x_shared = None
    for i, (name, M, K, k) in enumerate(LAYERS):
        d = synth.representation(M, K, BITS, 0, k, seed=synth.SEED_BASE + 100 * i)
        # q, k and v read the SAME activation (the model's structure); out, fc1, fc2 their own
        if name in ("q", "k", "v") and x_shared is not None:
            x = x_shared
        else:
            x = synth.activations(batch, K, seed=synth.SEED_BASE + 100 * i + 1, outliers=d["weak_idx"][:8])
        if name == "q":
            x_shared = x
        if keep_rows:
            host_keep.append({"codes": d["codes"][:keep_rows].copy(), "scale_f16": d["scale_f16"][:keep_rows].copy(),
                              "zero_f16": d["zero_f16"][:keep_rows].copy(), "weak_idx": d["weak_idx"].copy(),
                              "weak_val_f16": d["weak_val_f16"][:keep_rows].copy(), "x": x.copy()})
        full = owq.Shape(M, K, BITS, 0, k)
        L = {"name": name, "M": M, "K": K, "k": k, "full": full}
        if world == 1:
            L["shape"] = full
            L["layout"] = layout_override or owq.choose_layout(full, batch)
            flags = owq.OWQ_PACK_LAYOUT_CC if L["layout"] == owq.OWQ_LAYOUT_CC else 0
            L["packed"] = owq.owq_pack(full, d, flags=flags, device=dev)
            if name in ("k", "v"):
                L["x"] = layers[0]["x"]          # the same device tensor as q's input
            else:
                L["x"] = torch.from_numpy(x).to(dev)
            L["y"] = torch.empty((batch, M), dtype=torch.float16, device=dev)
            L["ws"] = owq.workspace(full, batch, dev)
            L["bytes"] = algorithmic_bytes(M, K, k, batch)
        else:
            mode = TP_MODE[name]
            ss, packed = owq.owq_tp_shard(full, d, mode, world, rank, device=dev)
            a, b = owq.owq_tp_bounds(full, mode, world, rank)
            L.update(mode=mode, shape=ss, packed=packed, a=a, b=b, layout=owq.OWQ_LAYOUT_TC)
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


def launches_per_call(L, world):
    """Our kernels per public call: tcgen05 layout = x-digit pass + GEMV; CUDA-core
    layout = one GEMV per 4 batch rows; + the fp32 -> fp16 convert of a
    column-split layer's all-reduced y under TP."""
    import paper_2306_02272_b200 as owq
    B = L["x"].shape[0]
    n = 2 if L.get("layout", owq.OWQ_LAYOUT_TC) == owq.OWQ_LAYOUT_TC else -(-B // 4)
    return n + (1 if world > 1 and L.get("mode", 0) == 1 else 0)


def time_graph_calls(seq, stream, tp=None, reps=2):
    """Device time of the calls in `seq`, captured back to back in one CUDA graph
    (events on the launching stream; the first replay warms up)."""
    import torch
    pg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(pg, stream=stream):
        for L in seq:
            launch(L, tp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for _ in range(reps):
            e0.record(stream)
            pg.replay()
            e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def measure_secondary(dev, stream, budget_s):
    """Per-layer device time of the SECONDARY configs (rotating packed copies >
    3x L2, back-to-back calls in one graph)."""
    import torch

    import paper_2306_02272_b200 as owq
    import synth
    out, t0 = {}, time.perf_counter()
    for cfg, rows in SECONDARY.items():
        res = {}
        for name, M, K, bits, group, k, B in rows:
            if time.perf_counter() - t0 > budget_s:
                res[name] = "skipped (time budget)"
                continue
            d = synth.representation(M, K, bits, group, k, seed=M + K + k)
            shape = owq.Shape(M, K, bits, group, k)
            lay = owq.choose_layout(shape, B)
            flags = owq.OWQ_PACK_LAYOUT_CC if lay == owq.OWQ_LAYOUT_CC else 0
            nb = owq.owq_packed_bytes_layout(shape, lay)
            ncop = max(1, min(8, -(-400_000_000 // nb)))
            packs = [owq.owq_pack(shape, d, flags=flags, device=dev) for _ in range(ncop)]
            x = torch.from_numpy(synth.activations(B, K, seed=1, outliers=d["weak_idx"])).to(dev)
            y = torch.empty((B, M), dtype=torch.float16, device=dev)
            ws = owq.workspace(shape, B, dev)
            R = 24
            seq = [{"shape": shape, "packed": packs[i % ncop], "x": x, "y": y, "ws": ws} for i in range(R)]
            with torch.cuda.stream(stream):
                for L in seq[:ncop]:
                    launch(L)
            ms = time_graph_calls(seq, stream) / R
            alg = algorithmic_bytes(M, K, k, B, bits=bits, G=(1 if group == 0 else -(-K // group)))
            res[name] = {"us": round(ms * 1e3, 2), "GBps": round(alg / (ms * 1e-3) / 1e9, 1),
                         "layout": "cc" if lay == owq.OWQ_LAYOUT_CC else "tc"}
            del packs
        out[cfg] = res
    return out


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["model"] = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return info


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
    layout_override = {"tc": owq.OWQ_LAYOUT_TC, "cc": owq.OWQ_LAYOUT_CC}.get(args.layout)
    layers, host_keep = build_layers(dev, args.batch, world, rank, keep, layout_override)
    tp = None
    if world > 1:
        uid = owq.owq_tp_get_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        tp = owq.owq_tp_init(obj[0], world, rank)
    step_bytes = sum(L["bytes"] for L in layers)
    stream = torch.cuda.Stream(device=dev)
    # q, k, v read one input and are independent of each other: on one GPU they run
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
    if world > 1:
        dist.barrier()

    K, W = args.steps, args.warmup
    n_l = len(layers)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    g = wg = sg = None
    if not args.no_graph:
        # K steps (and the warm-up) captured in CUDA graphs -- also under TP: the
        # NCCL collectives of owq_tp_gemv are graph-capturable
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for s in range(K):
                    step()
            wg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(wg, stream=stream):
                for _ in range(max(W, 3)):
                    step()
            sg = torch.cuda.CUDAGraph()     # one step (per-step distribution, outside the timed region)
            with torch.cuda.graph(sg, stream=stream):
                step()
        except Exception as e:  # pragma: no cover - fall back to eager timing
            print(f"[bench] graph capture failed ({e}); timing eager launches", file=sys.stderr)
            g = wg = sg = None
    uploaded = g is not None and graph_upload(g, stream) and graph_upload(wg, stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

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
    ms_step = ms_total / K
    value = step_bytes / (ms_step * 1e-3) / 1e9

    # per-step distribution (outside the timed region): K single-step replays
    step_ms = []
    if sg is not None:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(min(K, 100))]
        with torch.cuda.stream(stream):
            for a_, b_ in evs:
                a_.record(stream)
                sg.replay()
                b_.record(stream)
        torch.cuda.synchronize()
        step_ms = sorted(a_.elapsed_time(b_) for a_, b_ in evs)
    pct = (lambda q: round(step_ms[min(len(step_ms) - 1, int(q * len(step_ms)))], 5)) if step_ms else (lambda q: None)

    # per-launch durations (roofline): per layer shape, R back-to-back calls in one
    # graph over the same-shape layers in rotation (working set > L2), CUDA events
    # around the replay on the launching stream; + one call after an L2 flush
    per_layer_ms = [None] * n_l
    single_ms = {}
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
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for idx in shapes.values():
        pool = [seq_view[i] for i in idx]
        nbytes = sum(L["bytes"] for L in pool)
        while nbytes < 3 * 126e6 and world == 1:
            L0 = pool[len(pool) % len(idx)]
            Lc = dict(L0)
            Lc["packed"] = L0["packed"].clone()
            pool.append(Lc)
            nbytes += L0["bytes"]
        with torch.cuda.stream(stream):
            for L in pool:
                launch(L, tp)
        seq = [pool[j % len(pool)] for j in range(R)]
        if g is not None:
            ms = time_graph_calls(seq, stream, tp) / R
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for L in seq:
                    launch(L, tp)
                e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / R
        for i in idx:
            per_layer_ms[i] = ms
        # single-launch latency: one call with a cold L2 (256 MB written first)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.fill_(1)
            e0.record(stream)
            launch(pool[0], tp)
            e1.record(stream)
        torch.cuda.synchronize()
        single_ms[layers[idx[0]]["name"]] = e0.elapsed_time(e1)
    del flush

    # ---------------------------------------------------------------- e2e (host buffers)
    e2e = None
    if not args.no_e2e:
        # The step's inputs (q's x -- shared by k and v -- and the x of out, fc1,
        # fc2) sit in one pinned host buffer and go to the device in one copy;
        # the step's results (every layer's y) come back in one copy; in between,
        # the layers are eager public-API calls, one after another on all SMs.
        eager = [dict(L) for L in (seq_view if world == 1 else layers)]
        xs_unique = []
        for L in eager:
            if not any(L["x"] is u for u in xs_unique):
                xs_unique.append(L["x"])
        nx = [u.numel() for u in xs_unique]
        ny = [L["y"].numel() for L in eager]
        xh_all = torch.empty(sum(nx), dtype=torch.float16).pin_memory()
        yh_all = torch.empty(sum(ny), dtype=torch.float16).pin_memory()
        xd_all = torch.empty(sum(nx), dtype=torch.float16, device=dev)
        yd_all = torch.empty(sum(ny), dtype=torch.float16, device=dev)
        ox = 0
        views = {}
        for u, a in zip(xs_unique, nx):
            xh_all[ox:ox + a].copy_(u.reshape(-1).cpu())
            views[id(u)] = xd_all[ox:ox + a].view(u.shape)
            ox += a
        oy = 0
        for L, b in zip(eager, ny):
            L["x"] = views[id(L["x"])]
            L["y"] = yd_all[oy:oy + b].view(L["y"].shape)
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
               "ms_per_step": round(1e3 * dt / E, 4),
               "path": "one pinned H2D copy of the step's inputs (q/k/v share one x), eager public-API calls "
                       "(all SMs, in order), one D2H copy of every y"}
        # the same step captured once in a CUDA graph (H2D copy, the public-API calls,
        # D2H copy) and replayed: what a serving loop that graphs its decode step sees
        try:
            ge = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                with torch.cuda.graph(ge, stream=stream):
                    xd_all.copy_(xh_all, non_blocking=True)
                    for L in eager:
                        launch(L, tp)
                    yh_all.copy_(yd_all, non_blocking=True)
                for _ in range(3):
                    ge.replay()
                    stream.synchronize()
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                for _ in range(E):
                    ge.replay()
                    stream.synchronize()   # the host reads the step's result
                dtg = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([dtg], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dtg = float(t.item())
            e2e["graphed"] = {"value": round(step_bytes * E / dtg / 1e9, 2), "ms_per_step": round(1e3 * dtg / E, 4),
                              "path": "the same copies and calls captured in one CUDA graph, replayed and "
                                      "synchronised every step (wall clock)"}
        except Exception as ex:   # graph capture of the host-copy step unavailable: eager number only
            e2e["graphed"] = {"unavailable": str(ex)[:200]}

    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary:
        secondary = measure_secondary(dev, stream, args.secondary_seconds)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---------------------------------------------------------------- roofline / cpu baseline
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs")
    read_peak = None
    try:
        with open(os.path.join(ROOT, "profiles", "read_peak.json")) as f:
            read_peak = json.load(f).get("read_only_gbs_tma_1GiB")
    except Exception:
        pass
    per_layer = {L["name"]: {"us": round(1e3 * t, 3), "GBps": round(L["bytes"] / (t * 1e-3) / 1e9, 1),
                             "bytes": int(L["bytes"]), "single_launch_us_cold_l2": (round(1e3 * single_ms[L["name"]], 2) if L["name"] in single_ms else None),
                             "layout": "cc" if L.get("layout") == owq.OWQ_LAYOUT_CC else "tc"}
                 for L, t in zip(layers, per_layer_ms)}
    kern_ms = sum(per_layer_ms)
    achieved = step_bytes / (kern_ms * 1e-3) / 1e9 if world == 1 else value
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)["per_shape"]
        tag = {(D, D): "q", (4 * D, D): "fc1", (D, 4 * D): "fc2"}
        per = [tr[tag[(L["M"], L["K"])]] for L in layers]
        traffic = round(sum(t["dram_read_bytes"] + t["dram_write_bytes"] for t in per) / len(per), 1)
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4) if peak else None, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, measured)" if peak else "missing",
                "read_only_peak": read_peak,
                "frac_of_read_only_peak": round(achieved / read_peak, 4) if read_peak else None,
                "frac_of_nominal_8TBps": round(achieved / NOMINAL_HBM_GBS, 4),
                "per_launch": "per layer shape: R back-to-back calls in one CUDA graph timed with CUDA events; "
                              "achieved = sum of the layers' algorithmic bytes / sum of their per-call times "
                              "(a tcgen05-layout call = x-digit pass + GEMV, both counted)",
                "traffic_note": "mean per launch of dram__bytes_read.sum + dram__bytes_write.sum from "
                                "profiles/ncu_traffic.json (one --set full capture per layer shape)"}
    cpu = None
    if not args.no_cpu and host_keep:
        lim = cpu_threads()
        runs = []
        for threads in (1, None):
            ctx = lim(limits=threads) if lim else None
            if ctx:
                ctx.__enter__()
            # repeat the sample until about args.cpu_seconds of CPU work (bounded: at most 64 passes)
            t, nb, passes = 0.0, 0.0, 0
            while passes < 64 and (passes == 0 or t < args.cpu_seconds / 2):
                dt, dnb = oracle_sample(host_keep, args.ref_rows)
                t, nb, passes = t + dt, nb + dnb, passes + 1
            if ctx:
                ctx.__exit__(None, None, None)
            runs.append((threads or os.cpu_count(), nb / t / 1e9, passes, t))
        best = max(runs, key=lambda r: r[1])
        hi = host_info()
        cpu = {"value": round(best[1], 4), "unit": UNIT, "cores": best[0], "kind": "oracle",
               "sample": f"oracle.matvec_rows (fp64) on the first {args.ref_rows} rows of each of the 6 layers, "
                         f"{best[2]} passes, {best[0]} thread(s) (BLAS threads via threadpoolctl)",
               "seconds": round(best[3], 3),
               "runs": [{"threads": r[0], "GBps": round(r[1], 4), "passes": r[2], "seconds": round(r[3], 3)} for r in runs],
               "host": hi}
        if args.quantizer_time:
            import oracle as O
            import synth
            Wq, Xq, _ = synth.weights_and_calib(768, 768, N=2048, n_outliers=8, seed=2306)
            t0 = time.perf_counter()
            O.owq_quantize(Wq, Xq, 3, 8)
            cpu["oracle_quantizer_config1_s"] = round(time.perf_counter() - t0, 2)
    lays = {L.get("layout") for L in layers}
    arith = []
    if owq.OWQ_LAYOUT_TC in lays:
        arith.append("tcgen05 layout: codes (u8) x exact int8 digits of x*2^24 on tcgen05.mma kind::i8, s32 accumulate; "
                     "zero point and digits combined exactly (fp64), fp32 scale")
    if owq.OWQ_LAYOUT_CC in lays:
        arith.append("CUDA-core layout: exact products q*x (fp32 subnormal codes x 2^(111-p)-scaled x, FFMA2), fp32 sums, "
                     "factored zero point s*(sum q x - z sum x)")
    arith.append("weak columns fp16 x fp16 in fp32")
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8*s8->s32" if lays == {owq.OWQ_LAYOUT_TC} else "mixed (see config.arith)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "layers": [[n, M, K_, k] for n, M, K_, k in LAYERS],
                   "bits": BITS, "group_size": 0, "batch": args.batch,
                   "parallelism": f"tp{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (682 MB of packed weights per step vs 126 MB L2); no flush",
                   "graph": g is not None, "graph_uploaded_before_timing": bool(uploaded) if g is not None else None,
                   "schedule": ("q, k, v (one shared input) concurrently on 3 streams (a third of the SMs each); "
                                "out, fc1, fc2 in order" if concurrent else "all six layers in order on all SMs"),
                   "arith": "; ".join(arith)},
        "step_ms_p10_p50_p90": [pct(0.1), pct(0.5), pct(0.9)],
        "us_per_layer": per_layer,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": K * sum(launches_per_call(L, world) for L in layers),
        "clocks": clk.summary(),
        "secondary_configs": secondary,
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
    ap.add_argument("--layout", default="auto", choices=["auto", "tc", "cc"],
                    help="device layout of the headline layers (auto = choose_layout)")
    ap.add_argument("--no-secondary", action="store_true", help="skip the BASELINE config 2/3/4 per-layer lines")
    ap.add_argument("--secondary-seconds", type=float, default=60.0)
    ap.add_argument("--no-quantizer-time", dest="quantizer_time", action="store_false",
                    help="skip timing the oracle quantizer at config 1 (768x768, k = 8) for cpu_baseline")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
