"""Two-rank NCCL tensor parallelism on two GPUs: each rank
packs its shard through the C-ABI, runs owq_tp_gemv (row split: all-gather;
column split: fp32 all-reduce) and checks the full y against the fp64 oracle
and owq_tp_check for asynchronous NCCL errors.  Skips on a box with one GPU
(every gpurun box this round); tests/test_tp_gloo.py covers the same host
logic with world 2 on CPU."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle as O
    import paper_2306_02272_b200 as owq
    import synth
    from owq_testutil import TOL, rel_err, rep_from_synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    uid = [owq.owq_tp_get_unique_id() if rank == 0 else bytes(128)]
    dist.broadcast_object_list(uid, src=0)
    tp = owq.owq_tp_init(uid[0], world, rank)
    errs = []
    for (M, K, bits, group, k, B) in [(1024, 2048, 3, 0, 9, 1), (768, 4096, 4, 128, 5, 3)]:
        d = synth.representation(M, K, bits, group, k, seed=M + K)
        shape = owq.Shape(M, K, bits, group, k)
        x = synth.activations(B, K, seed=B, outliers=d["weak_idx"])
        ref = O.matvec(rep_from_synth(d), x.astype(np.float64))
        for mode in (owq.OWQ_TP_ROWS, owq.OWQ_TP_COLS):
            ss, packed = owq.owq_tp_shard(shape, d, mode, world, rank, device=dev)
            a, b = owq.owq_tp_bounds(shape, mode, world, rank)
            xs = x if mode == owq.OWQ_TP_ROWS else np.ascontiguousarray(x[:, a:b])
            ws = torch.zeros(owq.owq_tp_workspace_bytes(shape, mode, world, B), dtype=torch.uint8, device=dev)
            y = torch.empty((B, M), dtype=torch.float32, device=dev)
            owq.owq_tp_gemv(tp, mode, shape, ss, packed, torch.from_numpy(xs).to(dev), y, y_f32=True, ws=ws)
            torch.cuda.synchronize()
            owq.owq_tp_check(tp)
            errs.append(rel_err(y.cpu().numpy(), ref)[0])
    owq.owq_tp_destroy(tp)
    dist.destroy_process_group()
    q.put((rank, max(errs), TOL))


def test_tp_two_ranks_nccl():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one per rank); gpurun boxes have one")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = [q.get(timeout=10) for _ in procs]
    for rank, err, tol in res:
        assert err <= tol, (rank, err)
