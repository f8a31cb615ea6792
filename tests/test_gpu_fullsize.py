"""BASELINE.json's 3D configs at their full per-GPU size, in the launch configuration bench.py times
(one rc_step over every cell, the default bf16 MLP), checked against the oracle on a hashed sample
of cells computed one by one, plus whole-field properties that hold at any size.

  C3  16,777,216 H2 cells (256^3), 8 nets      -- also covers C5's per-GPU block (1e8 / 8 = 12.5M cells
                                                   of the same recipe)
  C4  16,777,216 CH4 cells (256^3), 19 nets, KZ = 32 z rows

Gates as in test_gpu_parity.py (fp64 1e-10; o 2e-2; derived wdot / qdot 3e-2 and within 1.5x the
rounding floor of the operand-rounding emulation on the same cells)."""
import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import oracle
from _harness import Gpu, mech, run_oracle
from test_gpu_parity import _sample, check_chem, check_fp64
from workload import CONFIGS
from workload.cells import make_cells

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_13513_b200 import build
    build.build()


def _generate(cfg):
    """all cells of cfg, generated in parallel over 1M-cell blocks (spawned workers: this process
    already holds a CUDA context, so no fork)"""
    n = CONFIGS[cfg].n_cells
    step = 1 << 20
    bounds = [(b, min(n, b + step)) for b in range(0, n, step)]
    workers = max(1, min(len(os.sched_getaffinity(0)), 32, len(bounds)))
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        parts = list(ex.map(make_cells, [cfg] * len(bounds), [b for b, _ in bounds], [e for _, e in bounds]))
    c = {k: np.concatenate([p[k] for p in parts], axis=-1) for k in parts[0]}
    # h of every cell from the ORACLE's T-mode thermo (the input of both sides)
    om = oracle.Mech(mech(CONFIGS[cfg].mech))
    c["h"] = oracle.step(om, None, c["T_true"], c["p"], c["Y"], mode="T", transport=False, chem=False)["h"]
    return c


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_full_size_3d_configs_sampled(cfg):
    c = _generate(cfg)
    n = CONFIGS[cfg].n_cells
    assert c["p"].shape[0] == n
    g = Gpu(cfg).run(c)
    cols = _sample(cfg, 160)
    sub = {k: (v[..., cols] if isinstance(v, np.ndarray) else v) for k, v in c.items()}
    o = run_oracle(cfg, sub)
    check_fp64(g, o, cols)
    m = mech(CONFIGS[cfg].mech)
    eo, ew, eq = check_chem(g, o, m, cols, emu=(cfg, sub, "bf16_ideal"))
    print(f"{cfg} full size ({n} cells), sampled bf16 errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")
    # whole field: finite, no fallbacks beyond the oracle's, T_max is the field's max, mass conserved
    assert np.all(np.isfinite(g["T"])) and np.all(np.isfinite(g["wdot"])) and g["diag"][2] == 0
    assert g["red"][0] == g["T"].max()
    tot = np.abs(g["wdot"]).sum(axis=0) + 1e-300
    assert np.all(np.abs(g["wdot"].sum(axis=0)) <= 1e-12 * tot)
