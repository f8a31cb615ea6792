"""Detailed-kinetics source term (reading R21) on the GPU vs the
oracle (orc_kinetics), through the C ABI (rc_kin_create / rc_kinetics).

Gate: fp64 throughout, so per cell and species |g - o| <= 1e-10 x the gross rate
W_k sum_r |nu_rk| (|q_f| + |q_r|) of that cell (the net rate is a difference of forward and reverse
rates that cancel near equilibrium, so the gross rate is its natural scale); qdot likewise against
sum_k |h_k| x gross rate; sum qdot 1e-10 relative."""
import numpy as np
import pytest

import oracle
from _harness import inputs, mech
from workload import CONFIGS, load_kinetics, tau_mix_at
from workload.cells import uniform

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_13513_b200 import build
    build.build()


def _run(c, T, tau=None, ld=None):
    import torch

    import paper_2312_13513_b200 as rc
    m = mech("h2_9sp")
    M = rc.Mechanism(m)
    K = rc.Kinetics(M, load_kinetics("h2_9sp"))
    n = T.shape[0]
    st = rc.CellState(n, 9, 0, ld=ld, sources=True)
    st.load(T, c["p"], c["Y"])
    st.set_tau_mix(tau)
    rc.rc_kinetics(M, K, st.cells(rc.RC_MODE_T, chem=True, transport=False))
    torch.cuda.synchronize()
    return st.host(), rc.rc_last_launch_count()


def _check(g, o, m):
    om = oracle.Mech(m)
    err = np.abs(g["wdot"] - o["wdot"]) / (o["wscale"] + 1e-300)
    assert err.max() <= TOL, err.max()
    n = g["qdot"].shape[0]
    hs = np.array([[abs(om.h_k(k, T)) for T in o["T"]] for k in range(m["ns"])]) if "T" in o else None
    qscale = (hs * o["wscale"]).sum(axis=0)
    assert np.max(np.abs(g["qdot"] - o["qdot"]) / (qscale + 1e-300)) <= TOL
    tot = np.abs(g["wdot"]).sum(axis=0) + 1e-300
    assert np.all(np.abs(g["wdot"].sum(axis=0)) <= 1e-12 * tot)
    return err.max(), n


def test_c1_full():
    m = mech("h2_9sp")
    c = inputs("C1")
    o = oracle.kinetics(oracle.Mech(m), oracle.Kin(load_kinetics("h2_9sp")), c["T_true"], c["p"], c["Y"])
    o["T"] = c["T_true"]
    g, launches = _run(c, c["T_true"])
    e, _ = _check(g, o, m)
    assert g["red"][1] == pytest.approx(o["red"][1], rel=TOL)
    assert launches >= 1
    print(f"\n  kinetics C1: max error / gross rate {e:.2e}")


def test_c2_sample_ragged_and_pasr():
    """1,031 hashed C2 jet-flame cells (ragged last tile, ld > n) with and without LES PaSR."""
    m = mech("h2_9sp")
    cols = np.unique((uniform(777, np.arange(1100)) * CONFIGS["C2"].n_cells).astype(np.int64))[:1031]
    c = inputs("C2", idx=cols)
    kin = oracle.Kin(load_kinetics("h2_9sp"))
    for tau in (None, tau_mix_at("C2", cols)):
        o = oracle.kinetics(oracle.Mech(m), kin, c["T_true"], c["p"], c["Y"], tau_mix=tau)
        o["T"] = c["T_true"]
        g, _ = _run(c, c["T_true"], tau=tau, ld=1040)
        e, _ = _check(g, o, m)
        print(f"\n  kinetics C2 sample (PaSR {tau is not None}): max error / gross rate {e:.2e}")


def test_kinetics_argument_errors():
    import paper_2312_13513_b200 as rc
    from workload import load_mech
    M = rc.Mechanism(mech("h2_9sp"))
    K = rc.Kinetics(M, load_kinetics("h2_9sp"))
    st = rc.CellState(64, 9, 0)                          # no wdot allocated
    with pytest.raises(rc.RcError) as e:
        rc.rc_kinetics(M, K, st.cells(rc.RC_MODE_T, chem=False))
    assert e.value.code == rc._rc.RC_EINVAL
    # a mechanism of another size
    M20 = rc.Mechanism(load_mech("ch4_20sp"))
    st20 = rc.CellState(64, 20, 0, sources=True)
    with pytest.raises(rc.RcError):
        rc.rc_kinetics(M20, K, st20.cells(rc.RC_MODE_T))
    # a reaction with four reactant molecules is refused at create
    k = load_kinetics("h2_9sp")
    k["nu_f"] = k["nu_f"].copy()
    k["nu_f"][0, 3] = 4
    with pytest.raises(rc.RcError) as e:
        rc.Kinetics(M, k)
    assert e.value.code == rc._rc.RC_EUNSUPPORTED
