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


# ---------------------------------------------------------------- NEXT-1: z-slab halo exchange
MESH = (6, 5, 8, 1e-3, 1.2e-3, 0.9e-3)
NS = 3


def _gamma_inputs():
    """a seeded global field of the Laplacian inputs (rho, lambda, cp, D_k) on MESH, cells in index order"""
    nx, ny, nz = MESH[:3]
    rng = np.random.default_rng(11)
    n = nx * ny * nz
    return {"rho": rng.uniform(0.1, 1.2, n), "lam": rng.uniform(0.02, 0.2, n), "cp": rng.uniform(1e3, 2e3, n),
            "D": rng.uniform(1e-5, 1e-4, (NS, n))}


def _pack(f, sl):
    """[(ns + 3)][plane] pack of the planes `sl` of the fields (the layout rc_pack_planes writes)"""
    return np.concatenate([f["rho"][sl][None], f["lam"][sl][None], f["cp"][sl][None], f["D"][:, sl]])


def _halo_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2312_13513_b200.dist import exchange_halos, slab
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        nx, ny, nz, dx, dy, dz = MESH
        plane = nx * ny
        f = _gamma_inputs()
        z0, z1 = slab(nz)
        loc = slice(z0 * plane, z1 * plane)
        bottom = torch.from_numpy(_pack(f, slice(z0 * plane, (z0 + 1) * plane)))
        top = torch.from_numpy(_pack(f, slice((z1 - 1) * plane, z1 * plane)))
        lo, hi = exchange_halos(bottom, top)
        g = oracle.laplacian_gamma(NS, f["rho"][loc], f["D"][:, loc], f["lam"][loc], f["cp"][loc])
        hg = [oracle.laplacian_gamma(NS, h[0], h[3:], h[1], h[2]) for h in (lo.numpy(), hi.numpy())]
        up, dg = oracle.laplacian((nx, ny, z1 - z0, dx, dy, dz), g, hg[0], hg[1])
        q.put((rank, z0, z1, lo.numpy(), hi.numpy(), up, dg))
    finally:
        dist.destroy_process_group()


def test_slab_halo_exchange_gloo():
    """Two ranks own z-slabs of a periodic box; exchange_halos (batch_isend_irecv on the periodic ring,
    NCCL P2P on the GPU box) delivers the neighbours' boundary planes, and each rank's slab assembly
    with those halos equals the corresponding rows of the global periodic assembly."""
    import torch.multiprocessing as mp

    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nx, ny, nz = MESH[:3]
    plane, N = nx * ny, nx * ny * nz
    f = _gamma_inputs()
    gG = oracle.laplacian_gamma(NS, f["rho"], f["D"], f["lam"], f["cp"])
    upG, dgG = oracle.laplacian(MESH, gG)
    assert res[0][1] == 0 and res[-1][2] == nz and res[0][2] == res[1][1]
    for rank, z0, z1, lo, hi, up, dg in res:
        # halos: the planes z0 - 1 and z1 of the periodic box
        assert np.array_equal(lo, _pack(f, slice(((z0 - 1) % nz) * plane, ((z0 - 1) % nz + 1) * plane)))
        assert np.array_equal(hi, _pack(f, slice((z1 % nz) * plane, (z1 % nz + 1) * plane)))
        n = (z1 - z0) * plane
        sl = slice(z0 * plane, z1 * plane)
        for d in range(3):
            assert np.array_equal(up[:, d * n:(d + 1) * n], upG[:, d * N:(d + 1) * N][:, sl])
        np.testing.assert_allclose(dg, dgG[:, sl], rtol=1e-15)


# ---------------------------------------------------------------- bench.py's rank logic (--dry-run)
def _bench_ranks(args, world=2):
    import json
    import subprocess
    import sys
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", *args], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=600)
        assert p.returncode == 0, e[-2000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    return sorted(outs, key=lambda d: d["rank"])


def test_bench_rank_logic_strong_c5_gloo():
    """bench.py at N = 2 (strong scaling of C5, the 1e8-cell 8xB200 target): the ranks' rc_partition
    blocks tile [0, 1e8) with a 128-aligned boundary, each rank generates its cells, and the a6
    reductions leave the same global values on both ranks."""
    from workload import CONFIGS
    r = _bench_ranks(["--config", "C5", "--strong", "--dry-cells", "4096"])
    n = CONFIGS["C5"].n_cells
    assert r[0]["first"] == 0 and r[1]["last"] == n - 1 and r[0]["last"] + 1 == r[1]["first"]
    assert r[1]["first"] % 128 == 0 and r[0]["cells_total"] == n
    assert r[0]["red"] == r[1]["red"] and r[0]["diag"] == r[1]["diag"]
    assert 1500.0 < r[0]["red"][0] < 3000.0                         # max T of the generated flame states


def test_bench_rank_logic_weak_laplacian_halos_gloo():
    """bench.py --laplacian at N = 2 (weak scaling: each rank's C3 block is a z-slab of a box stacked in z):
    the halo exchange delivers the neighbours' boundary planes on the periodic ring."""
    r = _bench_ranks(["--config", "C3", "--laplacian", "--dry-cells", "1024"])
    (a0, a1), (b0, b1) = r[0]["slab"], r[1]["slab"]
    assert a1 == b0 and (b1 - a0) == 512
    assert r[0]["halo"] == [float(b1 - 1), float(b0)]                # below rank 0: rank 1's top (periodic)
    assert r[1]["halo"] == [float(a1 - 1), float(a0)]
