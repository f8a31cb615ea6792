"""Shared-net MLP variant (reading R20: ONE net d_in -> 1600 -> 800
-> 400 -> n_nets) on the GPU vs the oracle, through the C ABI (rc_mlp_desc.flags RC_MLP_SHARED)."""
import numpy as np
import pytest

from _harness import (BF16_DERIVED_TOL, BF16_TOL, TF32_DERIVED_TOL, TF32_TOL, Gpu, inputs, mech, rel_fro,
                      run_oracle)
from workload import CONFIGS, make_bundle
from workload.cells import uniform

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_13513_b200 import build
    build.build()


def _check(g, o, tol, dtol, tag):
    eo, ew, eq = rel_fro(g["o"], o["o"]), rel_fro(g["wdot"], o["wdot"]), rel_fro(g["qdot"], o["qdot"])
    per = " ".join(f"{rel_fro(g['o'][i], o['o'][i]):.1e}" for i in range(g["o"].shape[0]))
    print(f"\n  shared net {tag}: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}; per output {per}")
    assert eo <= tol and ew <= dtol and eq <= dtol, (eo, ew, eq)
    m = mech("h2_9sp")
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    E = m["atoms"] * m["W_elem"][:, None] / W[None, :]
    tot = np.abs(g["wdot"]).sum(axis=0) + 1e-300
    assert np.all(np.abs(g["wdot"].sum(axis=0)) <= 1e-12 * tot)
    assert np.all(np.abs(E @ g["wdot"]) <= 1e-12 * tot[None, :])


@pytest.mark.parametrize("prec,tol,dtol", [(0, BF16_TOL, BF16_DERIVED_TOL), (1, TF32_TOL, TF32_DERIVED_TOL)])
def test_c1_full(prec, tol, dtol):
    """C1 (1,000 cells, ragged last tile), small shared net (64/32/16 -> 8 outputs)."""
    b = make_bundle("h2_9sp", hidden=(64, 32, 16), shared=True)
    c = inputs("C1")
    o = run_oracle("C1", c, b=b)
    g = Gpu("C1", precision=prec, b=b).run(c)
    _check(g, o, tol, dtol, f"C1 precision {prec}")


@pytest.mark.parametrize("prec,tol,dtol", [(0, BF16_TOL, BF16_DERIVED_TOL), (1, TF32_TOL, TF32_DERIVED_TOL)])
def test_paper_shape_full_chunk_sampled(prec, tol, dtol):
    """Paper widths (fused layer-1/2 kernel in bf16, one net): 65,536 C2 cells through the GPU, 96
    hashed cells checked against the oracle."""
    b = make_bundle("h2_9sp", shared=True)
    n = 65536
    c = inputs("C2", begin=0, end=n)
    g = Gpu("C2", precision=prec, b=b).run(c)
    cols = np.unique((uniform(4646, np.arange(96)) * n).astype(np.int64))
    cs = {k: (v[:, cols] if v.ndim == 2 else v[cols]) for k, v in c.items()}
    o = run_oracle("C2", cs, b=b)
    gs = {k: g[k][:, cols] if g[k].ndim == 2 else g[k][cols] for k in ("o", "wdot", "qdot")}
    _check(gs, o, tol, dtol, f"C2 precision {prec}")


def test_ch4_shared_net_19_outputs():
    """CH4 (Ns = 20, 19 outputs: three 8-output MMA tiles in layer 4, the last one padded), bf16,
    small widths so every tile of 2,000 cells is checked."""
    b = make_bundle("ch4_20sp", hidden=(64, 32, 16), shared=True)
    assert b["n_nets"] == 19
    c = inputs("C4", begin=3_000_000, end=3_002_000)
    o = run_oracle("C4", c, b=b)
    g = Gpu("C4", precision=0, b=b).run(c)
    eo, ew = rel_fro(g["o"], o["o"]), rel_fro(g["wdot"], o["wdot"])
    print(f"\n  shared net CH4: o {eo:.2e} wdot {ew:.2e}")
    assert eo <= BF16_TOL and ew <= BF16_DERIVED_TOL


def test_shared_flag_rejects_tf32x3():
    import paper_2312_13513_b200 as rc
    M = rc.Mechanism(mech("h2_9sp"))
    b = make_bundle("h2_9sp", hidden=(64, 32, 16), shared=True)
    with pytest.raises(rc.RcError) as e:
        rc.MLPBundle(M, b, rc.RC_TF32X3)
    assert e.value.code == rc._rc.RC_EUNSUPPORTED


@pytest.mark.parametrize("prec", [0, 1])
def test_shared_net_layer3_overlap_bitwise_equals_serial(prec):
    """The shared net with the layer-3 overlap (layer 4 of a chunk after both of its
    layer-3 launches): three chunks with a ragged last one give bitwise the RC_MLP_SERIAL result."""
    import paper_2312_13513_b200 as rc
    b = make_bundle("h2_9sp", shared=True)
    n = 2 * 262144 + 30_000
    c = inputs("C2", begin=0, end=n)
    G = Gpu("C2", precision=prec, b=b)
    rc.rc_overlap_read(reset=True)
    ov = G.run(c)
    cnt = rc.rc_overlap_read(reset=True)
    print(f"\n  shared-net overlap counters (precision {prec}): {cnt}")
    assert cnt["pairs_ran"] + cnt["pairs_gave_up"] > 0
    G.mlp = rc.MLPBundle(G.mech, b, prec, flags=rc.RC_MLP_SERIAL)
    se = G.run(c)
    for k in ("T", "cp", "rho", "mu", "lambda", "qdot", "D", "wdot", "o", "red", "diag"):
        assert np.array_equal(ov[k], se[k]), k
