"""World-size-2 tensor-parallel host logic on CPU (gloo): every rank builds its
shard through the C-ABI host sharder (owq_tp_shard_host), evaluates it with the
fp64 oracle, and the ranks combine exactly as owq_tp_gemv does on the GPU --
ROWS: all-gather of the row shards (padded to the largest shard) placed by
owq_tp_bounds; COLS: all-reduce(sum) of the partial products.  The result must
equal the full layer's oracle matvec."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2306_02272_b200 as owq
import synth
from owq_testutil import rep_from_synth

CASES = [  # M, K, bits, group, k
    (600, 512, 3, 0, 7),
    (272, 1024, 4, 128, 9),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for M, K, bits, g, k in CASES:
            d = synth.representation(M, K, bits, g, k, seed=11)
            shape = owq.Shape(M, K, bits, g, k)
            x = synth.activations(2, K, seed=12).astype(np.float64)
            for mode in (owq.OWQ_TP_ROWS, owq.OWQ_TP_COLS):
                a, b = owq.owq_tp_bounds(shape, mode, world, rank)
                ss, blob = owq.owq_tp_shard_host(shape, d, mode, world, rank)
                dec = owq.owq_blob_decode_host(blob)
                sr = O.Rep(M=ss.c_out, K=ss.c_in, bits=bits, group=g, codes=dec["codes"],
                           scale=O.from_fp16_bits(dec["scale_f16"]), zero=O.from_fp16_bits(dec["zero_f16"]),
                           weak_idx=dec["weak_idx"].astype(np.int64),
                           weak_val=O.from_fp16_bits(dec["weak_val_f16"]))
                if mode == owq.OWQ_TP_ROWS:
                    part = O.matvec(sr, x)                                   # [B, b - a]
                    mmax = max(owq.owq_tp_bounds(shape, mode, world, r)[1] - owq.owq_tp_bounds(shape, mode, world, r)[0]
                               for r in range(world))
                    buf = torch.zeros((2, mmax), dtype=torch.float64)
                    buf[:, : b - a] = torch.from_numpy(part)
                    gathered = [torch.zeros_like(buf) for _ in range(world)]
                    dist.all_gather(gathered, buf)
                    y = np.zeros((2, M))
                    for r in range(world):
                        ra, rb = owq.owq_tp_bounds(shape, mode, world, r)
                        y[:, ra:rb] = gathered[r][:, : rb - ra].numpy()
                else:
                    t = torch.from_numpy(O.matvec(sr, x[:, a:b]))
                    dist.all_reduce(t, op=dist.ReduceOp.SUM)
                    y = t.numpy()
                ref = O.matvec(rep_from_synth(d), x)
                out.append(float(np.max(np.abs(y - ref)) / max(1e-300, float(np.max(np.abs(ref))))))
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_tp_world2_gloo_matches_full_layer():
    world = 2
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert sorted(results.keys()) == list(range(world))
    for r in range(world):
        errs = results[r]
        assert len(errs) == 2 * len(CASES)
        assert max(errs) < 1e-12, errs
    assert list(results[0]) == list(results[1])
