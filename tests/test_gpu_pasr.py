"""LES PaSR option (reading R19) on the GPU vs the oracle's step 11,
through the C ABI (rc_cells.tau_mix), fused into the chemistry epilogue."""
import numpy as np
import pytest

from _harness import (BF16_DERIVED_TOL, BF16_TOL, TF32_DERIVED_TOL, TF32_TOL, Gpu, inputs, max_rel, mech,
                      rel_fro, run_oracle)
from workload import CONFIGS, make_bundle, tau_mix_at
from workload.cells import uniform

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_13513_b200 import build
    build.build()


def _conserves(m, w):
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    E = m["atoms"] * m["W_elem"][:, None] / W[None, :]
    tot = np.abs(w).sum(axis=0) + 1e-300
    assert np.all(np.abs(w.sum(axis=0)) <= 1e-12 * tot)
    assert np.all(np.abs(E @ w) <= 1e-12 * tot[None, :])


def test_exact_outputs_match_to_fp64():
    """All weights zero and b4 = 0.5: o = 0.5 exactly on both sides, so the PaSR-scaled wdot / qdot
    differ from the oracle only by fp64 rounding (kappa, the inverse transform and the projection)."""
    b = make_bundle("h2_9sp", hidden=(64, 32, 16))
    b["params"][:] = 0.0
    b["params"][:, -1] = 0.5
    c = inputs("C1")
    tau = tau_mix_at("C1", np.arange(1000))
    o = run_oracle("C1", c, b=b, tau_mix=tau)
    lam = run_oracle("C1", c, b=b)
    assert rel_fro(o["wdot"], lam["wdot"]) > 0.05           # the mixing times change the sources
    g = Gpu("C1", b=b).run(c, tau_mix=tau)
    assert rel_fro(g["wdot"], o["wdot"]) <= 1e-12, rel_fro(g["wdot"], o["wdot"])
    assert max_rel(g["qdot"], o["qdot"]) <= 1e-9
    _conserves(mech("h2_9sp"), g["wdot"])


@pytest.mark.parametrize("prec,tol,dtol", [(0, BF16_TOL, BF16_DERIVED_TOL), (1, TF32_TOL, TF32_DERIVED_TOL)])
def test_c1_full(prec, tol, dtol):
    c = inputs("C1")
    tau = tau_mix_at("C1", np.arange(1000))
    o = run_oracle("C1", c, tau_mix=tau)
    g = Gpu("C1", precision=prec).run(c, tau_mix=tau)
    eo, ew, eq = rel_fro(g["o"], o["o"]), rel_fro(g["wdot"], o["wdot"]), rel_fro(g["qdot"], o["qdot"])
    print(f"\n  PaSR C1 precision {prec}: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")
    assert eo <= tol and ew <= dtol and eq <= dtol
    _conserves(mech("h2_9sp"), g["wdot"])


def test_c2_paper_shape_sample():
    """Paper MLP (1600/800/400, 8 nets) on 128 hashed C2 cells with LES mixing times."""
    cols = np.unique((uniform(4545, np.arange(128)) * CONFIGS["C2"].n_cells).astype(np.int64))
    c = inputs("C2", idx=cols)
    tau = tau_mix_at("C2", cols)
    o = run_oracle("C2", c, tau_mix=tau)
    g = Gpu("C2").run(c, tau_mix=tau)
    eo, ew, eq = rel_fro(g["o"], o["o"]), rel_fro(g["wdot"], o["wdot"]), rel_fro(g["qdot"], o["qdot"])
    print(f"\n  PaSR C2 bf16: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")
    assert eo <= BF16_TOL and ew <= BF16_DERIVED_TOL and eq <= BF16_DERIVED_TOL
    _conserves(mech("h2_9sp"), g["wdot"])
