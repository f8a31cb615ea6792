"""Pins for the oracle's thermo (§3.1
"Newton's method and high-order temperature polynomials").  Each check is fixed
by mathematics or published data, not by re-running the oracle's formula."""
import json
import os

import numpy as np
import pytest

from conftest import synth_mech

RU = 8314.46261815324
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def W_of(m):
    return (m["atoms"].astype(float) * m["W_elem"][:, None]).sum(0)


def test_a1_only_species_closed_form(orc):
    # cp = a1 R/W at any T; h = a1 R T/W + a6 R/W
    nasa = np.zeros((2, 7)); nasa[:, 0] = 3.5; nasa[1, 5] = -1234.5
    m = orc.Mech(synth_mech(2, [7.0, 11.0], nasa=nasa))
    for T in (250.0, 999.0, 1000.0, 1001.0, 3100.0):
        assert m.cp_k(0, T) == pytest.approx(3.5 * RU / 7.0, rel=1e-15)
        assert m.h_k(0, T) == pytest.approx(3.5 * RU * T / 7.0, rel=1e-15)
        assert m.h_k(1, T) == pytest.approx((3.5 * T - 1234.5) * RU / 11.0, rel=1e-15)


def test_cp_is_dh_dT(orc, h2mech, ch4mech):
    # central difference of h equals cp; stay clear of T_mid
    for mech in (h2mech, ch4mech):
        m = orc.Mech(mech)
        for k in range(mech["ns"]):
            for T in (320.0, 600.0, 950.0, 1100.0, 1800.0, 2700.0):
                d = 1e-4 * T
                fd = (m.h_k(k, T + d) - m.h_k(k, T - d)) / (2 * d)
                assert fd == pytest.approx(m.cp_k(k, T), rel=1e-8), (mech["species"][k], T)


def test_nasa_continuity_at_Tmid(orc, h2mech, ch4mech):
    # transcription check of the GRI-Mech tables: both ranges agree at T_mid (App. A)
    for mech in (h2mech, ch4mech):
        m = orc.Mech(mech)
        for k, s in enumerate(mech["species"]):
            Tm = mech["T_mid"][k]
            tol = 3e-6 if s in ("N2", "CH3O") else 1e-7
            assert m.cp_k(k, Tm) == pytest.approx(m.cp_k(k, np.nextafter(Tm, 1e9)), rel=tol), s
            assert m.h_k(k, Tm) == pytest.approx(m.h_k(k, np.nextafter(Tm, 1e9)), rel=tol, abs=1.0), s


def test_formation_enthalpy_and_cp_298(orc, h2mech, ch4mech):
    g = json.load(open(os.path.join(GOLD, "thermo_298K.json")))
    seen = set()
    for mech in (h2mech, ch4mech):
        m = orc.Mech(mech)
        W = W_of(mech)
        for k, s in enumerate(mech["species"]):
            if s in g["dHf_kJ_per_mol"]:
                hf = m.h_k(k, 298.15) * W[k] / 1e6       # J/kg * kg/kmol -> kJ/mol
                assert hf == pytest.approx(g["dHf_kJ_per_mol"][s], abs=g["dHf_tol_kJ_per_mol"]), s
                seen.add(s)
            if s in g["cpR_298"]:
                assert m.cp_k(k, 298.15) * W[k] / RU == pytest.approx(g["cpR_298"][s], abs=g["cpR_tol"]), s
    assert seen == set(g["dHf_kJ_per_mol"])


def test_single_species_and_affine(orc, h2mech):
    m = orc.Mech(h2mech)
    ns = h2mech["ns"]
    rng = np.random.default_rng(0)
    for k in range(ns):
        Y = np.zeros(ns); Y[k] = 1.0
        for T in (400.0, 1500.0):
            assert m.cp(Y, T) == pytest.approx(m.cp_k(k, T), rel=1e-15)
            assert m.h(Y, T) == pytest.approx(m.h_k(k, T), rel=1e-15)
        assert m.W(Y) == pytest.approx(W_of(h2mech)[k], rel=1e-15)
    for _ in range(20):
        Y1, Y2 = rng.dirichlet(np.ones(ns)), rng.dirichlet(np.ones(ns))
        a, T = rng.uniform(), rng.uniform(300, 3000)
        lhs = m.h(a * Y1 + (1 - a) * Y2, T)
        rhs = a * m.h(Y1, T) + (1 - a) * m.h(Y2, T)
        assert lhs == pytest.approx(rhs, rel=1e-12, abs=1e-6 * abs(m.cp(Y1, T)))


def test_mean_molar_mass_dual_formula(orc, h2mech):
    # harmonic mass-fraction rule == mole-fraction route sum_k X_k W_k
    m = orc.Mech(h2mech)
    W = W_of(h2mech)
    Y = np.array([0.5, 0.5] + [0.0] * 7)  # equal mass H2/O2
    n = Y / W
    X = n / n.sum()
    assert m.W(Y) == pytest.approx(np.dot(X, W), rel=1e-15)
    rng = np.random.default_rng(1)
    for _ in range(10):
        Y = rng.dirichlet(np.ones(9))
        n = Y / W
        assert m.W(Y) == pytest.approx(np.dot(n / n.sum(), W), rel=1e-14)


def test_newton_round_trip(orc, h2mech, ch4mech):
    # T -> h -> T over 300-3000 K x random Y
    rng = np.random.default_rng(2)
    for mech in (h2mech, ch4mech):
        m = orc.Mech(mech)
        for T in np.linspace(300.0, 3000.0, 50):
            Y = rng.dirichlet(np.ones(mech["ns"]))
            h = m.h(Y, T)
            Tn, flags, it = m.T_from_h(Y, h, T * (1 + rng.uniform(-0.02, 0.02)))
            assert flags == 0
            assert Tn == pytest.approx(T, rel=1e-12)
            assert it <= 8


def test_newton_far_guess(orc, h2mech):
    # 300 K guess for a 2400 K state converges without bisection
    m = orc.Mech(h2mech)
    Y = np.array([0.0, 0.0, 0.2549, 0.0, 0.0, 0.0, 0.0, 0.0, 0.7451])
    h = m.h(Y, 2400.0)
    T, flags, it = m.T_from_h(Y, h, 300.0)
    assert flags == 0 and T == pytest.approx(2400.0, rel=1e-12)


def test_newton_constant_cp_one_step(orc):
    # h linear in T: the first update lands on the root; the
    # second iteration only confirms it
    m = orc.Mech(synth_mech(3, [2.0, 17.0, 40.0]))
    Y = np.array([0.2, 0.3, 0.5])
    cp = m.cp(Y, 1000.0)
    for T in (350.0, 1700.0, 2900.0):
        T_new, flags, it = m.T_from_h(Y, cp * T, 1000.0)
        assert flags == 0 and it == 2
        assert T_new == pytest.approx(T, rel=1e-15)


def test_newton_out_of_range_bisects(orc, h2mech):
    m = orc.Mech(h2mech)
    Y = np.array([0.0, 0.233, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.767])
    h_hi = m.h(Y, 5000.0) * 1.5   # above h(T_max): Newton clamps twice -> bisection
    T, flags, _ = m.T_from_h(Y, h_hi, 1000.0)
    assert flags & 1
    assert T == pytest.approx(5000.0, rel=1e-9)


def test_step_rho_identity_and_modes(orc, h2mech):
    from workload import make_cells
    m = orc.Mech(h2mech)
    c = make_cells("C1")
    n = c["p"].size
    tm = orc.step(m, None, c["T_true"], c["p"], c["Y"], mode="T", transport=False, chem=False)
    hm = orc.step(m, None, c["T_guess"], c["p"], c["Y"], h=tm["h"], mode="h", transport=False, chem=False)
    np.testing.assert_allclose(hm["T"], c["T_true"], rtol=1e-12)
    assert hm["diag"][0] == 0 and hm["diag"][1] == 0
    assert hm["diag"][3] == int(((c["Y"] < 0).any(axis=0)).sum())
    for i in range(0, n, 97):
        Wb = m.W(c["Y"][:, i])
        assert hm["rho"][i] * RU * hm["T"][i] / (c["p"][i] * Wb) == pytest.approx(1.0, rel=1e-15)
        assert hm["cp"][i] == pytest.approx(m.cp(c["Y"][:, i], hm["T"][i]), rel=1e-15)
    assert hm["red"][0] == hm["T"].max()
