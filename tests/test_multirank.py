"""Multi-rank host logic on CPU (gloo, world size 2): the cell partition and
the a6 global reductions.

Each rank takes its rc_partition block of C1, runs the oracle on it (the stand-in
for rc_step on a CPU box: the reductions see the same red/diag buffers the GPU
path writes), and reduces through paper_2312_13513_b200.dist.GlobalReductions.
Rank 0 checks the result against one unsharded oracle run: T_max and the
counters exactly, the heat-release sum to summation-order rounding.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    from _harness import inputs
    from workload import CONFIGS
    return inputs("C1", np.arange(CONFIGS["C1"].n_cells))


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    from _harness import run_oracle
    from paper_2312_13513_b200.dist import GlobalReductions, shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        case = _case()
        n = case["T_true"].shape[0]
        b, e = shard(n)
        sl = {k: (v[..., b:e] if isinstance(v, np.ndarray) and v.shape[-1] == n else v) for k, v in case.items()}
        out = run_oracle("C1", sl, chem=True)
        red = torch.tensor(out["red"], dtype=torch.float64)
        diag = torch.tensor(out["diag"], dtype=torch.int64)
        GlobalReductions("cpu")(red, diag)
        q.put((rank, b, e, red.numpy().tolist(), diag.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_partition_and_global_reductions_gloo():
    import torch.multiprocessing as mp
    from paper_2312_13513_b200 import build
    build.build()
    from _harness import run_oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the blocks tile [0, n) in order, 128-aligned boundaries
    case = _case()
    n = case["T_true"].shape[0]
    assert res[0][1] == 0 and res[-1][2] == n and res[0][2] == res[1][1] and res[0][2] % 128 == 0
    # every rank holds the global values, equal to one unsharded run
    full = run_oracle("C1", case, chem=True)
    for _, _, _, red, diag in res:
        assert red[0] == full["red"][0]                              # max is order-free: exact
        assert red[1] == pytest.approx(full["red"][1], rel=1e-12)    # Neumaier sums per rank, then a 2-term sum
        assert diag == list(full["diag"])
    assert res[0][3] == res[1][3] and res[0][4] == res[1][4]
