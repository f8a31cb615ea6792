"""Pins of the oracle's LES PaSR step (step 11, reading R19; PAPER.md:112 names the
partially-stirred reactor model for the SGS turbulence-chemistry interaction without giving its
equations): kappa = tau_c / (tau_c + tau_mix), 1/tau_c = (1/2 sum_k |wdot_k|/W_k) / sum_k C+_k."""
import numpy as np
import pytest

import oracle
from _harness import bundle, mech
from workload import make_cells, tau_mix_at


@pytest.fixture(scope="module")
def om():
    return oracle.Mech(mech("h2_9sp"))


def test_hand_example(om):
    """rho = 1 kg/m^3 with 0.01 kmol/m^3 each of H2 (Y = 0.02016) and O2 (Y = 0.31998): sum C = 0.02.
    wdot_H2 = -0.02016 and wdot_O2 = +0.31998 kg/m^3/s are 0.01 kmol/m^3/s each, so half the molar
    turnover is 0.01 and tau_c = 0.02 / 0.01 = 2 s.  tau_mix = 2 s gives kappa = 1/2, tau_mix = 6 s
    gives 1/4, tau_mix = 0 gives 1."""
    Y = np.zeros(9); Y[0], Y[1] = 0.02016, 0.31998
    w = np.zeros(9); w[0], w[1] = -0.02016, 0.31998
    assert om.pasr_kappa(1.0, Y, w, 2.0) == pytest.approx(0.5, rel=1e-14)
    assert om.pasr_kappa(1.0, Y, w, 6.0) == pytest.approx(0.25, rel=1e-14)
    assert om.pasr_kappa(1.0, Y, w, 0.0) == 1.0
    # rho scales C, not |wdot|: rho = 2 doubles tau_c
    assert om.pasr_kappa(2.0, Y, w, 4.0) == pytest.approx(0.5, rel=1e-14)
    # negative Y carries no concentration (C+ = rho max(Y, 0) / W)
    Yn = Y.copy(); Yn[5] = -1e-3
    assert om.pasr_kappa(1.0, Yn, w, 2.0) == pytest.approx(0.5, rel=1e-14)


def test_limits(om):
    Y = np.full(9, 1.0 / 9)
    w = np.linspace(-1.0, 1.0, 9)
    assert om.pasr_kappa(1.2, Y, np.zeros(9), 1.0) == 1.0          # nothing reacts: kappa = 1
    assert om.pasr_kappa(1.2, Y, w, 0.0) == 1.0                    # no subgrid mixing time: laminar
    k = [om.pasr_kappa(1.2, Y, w, t) for t in (1e-9, 1e-6, 1e-3, 1.0, 1e3)]
    assert all(a > b for a, b in zip(k, k[1:]))                      # monotone in tau_mix
    assert k[-1] < 1e-3                                              # tau_mix >> tau_c: kappa -> tau_c / tau_mix
    # kappa depends on |wdot| only (sign-blind turnover)
    assert om.pasr_kappa(1.2, Y, -w, 1e-3) == k[2]


def test_field_step_scales_the_laminar_sources():
    """orc_step with tau_mix: per cell wdot = kappa * laminar wdot (kappa of that cell's laminar wdot),
    qdot = kappa * laminar qdot, and the scaled sources still conserve mass and elements."""
    m = mech("h2_9sp")
    om, ob = oracle.Mech(m), oracle.Mlp(bundle("h2_9sp", (64, 32, 16)))
    c = make_cells("C1", 0, 200)
    h = oracle.step(om, None, c["T_true"], c["p"], c["Y"], mode="T", transport=False, chem=False)["h"]
    tau = tau_mix_at("C1", np.arange(200))
    lam = oracle.step(om, ob, c["T_guess"], c["p"], c["Y"], h=h, transport=False)
    les = oracle.step(om, ob, c["T_guess"], c["p"], c["Y"], h=h, transport=False, tau_mix=tau)
    kap = np.array([om.pasr_kappa(lam["rho"][i], c["Y"][:, i], lam["wdot"][:, i], tau[i]) for i in range(200)])
    assert np.all((kap > 0.0) & (kap <= 1.0)) and kap.min() < 0.9   # the recipe exercises kappa < 1
    np.testing.assert_allclose(les["wdot"], lam["wdot"] * kap[None, :], rtol=1e-15, atol=0)
    np.testing.assert_allclose(les["qdot"], lam["qdot"] * kap, rtol=1e-12)
    tot = np.abs(les["wdot"]).sum(axis=0)
    assert np.all(np.abs(les["wdot"].sum(axis=0)) <= 1e-12 * tot)
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    E = m["atoms"] * m["W_elem"][:, None] / W[None, :]
    assert np.all(np.abs(E @ les["wdot"]) <= 1e-12 * tot[None, :])
