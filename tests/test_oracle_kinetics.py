"""Pins of the oracle's detailed-kinetics source term (reading R21;
PAPER.md:114 names CVODE integration of detailed chemistry on the CPU, PAPER.md:231 the 9-species /
12-reaction H2 mechanism).  Checks against what mathematics and handbooks fix, not against a retyped
copy of oracle.c: thermodynamic identities, handbook entropies, the element-potential chemical
equilibrium (detailed balance), conservation, and special cases of the rate laws."""
import numpy as np
import pytest
from scipy.optimize import root

import oracle
from workload import load_kinetics, load_mech, make_cells

RU = 8314.46261815324
P0 = 101325.0


@pytest.fixture(scope="module")
def h2():
    m = load_mech("h2_9sp")
    return m, oracle.Mech(m), load_kinetics("h2_9sp")


def test_gibbs_function_identities(h2):
    """g = h/RT - s/R: with the (pinned) h_k, s/R = h/RT - g must satisfy ds/dT = cp/T (central
    difference), and S(298.15 K) must match JANAF standard entropies to 0.5 J/mol/K."""
    m, om, _ = h2
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    sR = lambda k, T: om.h_k(k, T) * W[k] / (RU * T) - om.g_k(k, T)
    for k in range(9):
        for T in (350.0, 800.0, 1500.0, 2500.0):
            d = 1e-4 * T
            dsdT = (sR(k, T + d) - sR(k, T - d)) / (2 * d)
            assert dsdT == pytest.approx(om.cp_k(k, T) * W[k] / RU / T, rel=1e-6)
    janaf = {"H2": 130.680, "O2": 205.147, "H2O": 188.834, "H": 114.716, "O": 161.058, "OH": 183.737, "N2": 191.609}
    for name, S in janaf.items():
        k = m["species"].index(name)
        assert sR(k, 298.15) * RU / 1000.0 == pytest.approx(S, abs=0.5), name


def _equilibrium(m, om, T, p, b):
    """Element-potential equilibrium at (T, p) for element amounts b: X_k = exp(-g_k + sum_e a_ek lam_e)
    (p0/p), sum_k X_k = 1, element ratios of X equal those of b.  Solved to 1e-14."""
    a = m["atoms"].astype(float)                           # [ne][ns]
    g = np.array([om.g_k(k, T) for k in range(m["ns"])])

    def X(lam):
        return np.exp(-g + a.T @ lam) * (P0 / p)

    def f(lam):  # log residuals: near-linear in the element potentials
        x = X(lam)
        e = a @ x
        return [np.log(x.sum()), np.log(e[0] / e[1]) - np.log(b[0] / b[1]), np.log(e[2] / e[1]) - np.log(b[2] / b[1])]

    # start: element potentials of a guessed major-species split (N2 0.65, H2O 0.3, H2 0.01)
    sp = m["species"]
    guess = {"N2": 0.65, "H2O": 0.3, "H2": 0.01}
    Ag = np.array([a[:, sp.index(k)] for k in guess])
    rhs = np.array([np.log(v * p / P0) + g[sp.index(k)] for k, v in guess.items()])
    sol = root(f, x0=np.linalg.solve(Ag, rhs), method="lm", tol=1e-15)
    assert np.max(np.abs(f(sol.x))) < 1e-12, f(sol.x)
    return X(sol.x)


@pytest.mark.parametrize("T,p", [(2500.0, 101325.0), (3000.0, 5 * 101325.0), (1800.0, 101325.0)])
def test_detailed_balance_at_equilibrium(h2, T, p):
    """At the chemical equilibrium found independently (element potentials, no rate law involved),
    every reversible reaction's net rate vanishes: pins K_c = exp(-sum nu g) (p0/RT)^(sum nu), the
    stoichiometry and the mass-action exponents of every reaction."""
    m, om, kd = h2
    kin = oracle.Kin(kd)
    b = m["atoms"].astype(float) @ np.array([2.0, 1.0, 0, 0, 0, 0, 0, 0, 3.76])  # moles H2:O2:N2 = 2:1:3.76
    X = _equilibrium(m, om, T, p, b)
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    Y = X * W / (X @ W)
    w, q, sc = kin.cell(om, T, p, Y)
    C = p / (RU * T) * X
    for r in range(kd["nr"]):
        fwd = kin.rate_constant(r, T, 0.0 if kd["type"][r] != 2 else (kd["eff"][r] @ C)) * np.prod(C ** kd["nu_f"][r])
        assert abs(q[r]) <= 1e-9 * fwd * (kd["eff"][r] @ C if kd["type"][r] == 1 else 1.0), (r, q[r], fwd)
    assert np.all(np.abs(w) <= 1e-9 * sc + 1e-300)


def test_conservation_on_flame_states(h2):
    m, om, kd = h2
    kin = oracle.Kin(kd)
    for cfg, n in (("C1", 1000), ("C2", 2000)):
        c = make_cells(cfg, 0, n) if cfg == "C1" else make_cells(cfg, 400_000, 400_000 + n)
        r = oracle.kinetics(om, kin, c["T_true"], c["p"], c["Y"])
        w = r["wdot"]
        tot = np.abs(w).sum(axis=0) + 1e-300
        assert np.all(np.abs(w.sum(axis=0)) <= 1e-12 * tot)
        W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
        E = m["atoms"] * m["W_elem"][:, None] / W[None, :]
        assert np.all(np.abs(E @ w) <= 1e-12 * tot[None, :])
        assert np.all(w[8] == 0.0)                           # N2 takes part in no reaction
        assert np.abs(w).max() > 1e2                          # real chemistry in the flame states
        # heat release positive where it is largest (exothermic H2 oxidation)
        assert r["qdot"].max() > -r["qdot"].min()


def test_rate_constant_special_cases(h2):
    m, om, kd = h2
    k = {key: np.array(v, copy=True) for key, v in kd.items() if isinstance(v, np.ndarray)}
    k["nr"] = kd["nr"]
    # elementary with b = 0, Ea = 0: k = A at any T
    k["b"][0], k["Ea"][0] = 0.0, 0.0
    # reaction 3 (falloff): Lindemann (a < 0) and Troe with Fcent = 1 must coincide
    kin_l = dict(k); kin_l["troe"] = k["troe"].copy(); kin_l["troe"][3] = [-1.0, 0, 0, 0]
    kin_t = dict(k); kin_t["troe"] = k["troe"].copy(); kin_t["troe"][3] = [1.0, 1.0, 1e300, 1e300]
    L, Tr, O = oracle.Kin(kin_l), oracle.Kin(kin_t), oracle.Kin(k)
    assert O.rate_constant(0, 1234.5, 0.0) == k["A"][0]
    for T in (800.0, 1500.0, 2500.0):
        kinf = k["A"][3] * T ** k["b"][3] * np.exp(-k["Ea"][3] / (RU * T))
        k0 = k["A0"][3] * T ** k["b0"][3] * np.exp(-k["Ea0"][3] / (RU * T))
        for M in (1e-6, 1e-2, 1.0, 1e3):
            assert Tr.rate_constant(3, T, M) == pytest.approx(L.rate_constant(3, T, M), rel=1e-13)
        # Lindemann limits: k -> k0 [M] at low, k -> k_inf at high pressure
        assert L.rate_constant(3, T, 1e-12 * kinf / k0) == pytest.approx(k0 * 1e-12 * kinf / k0, rel=1e-10)
        assert L.rate_constant(3, T, 1e12 * kinf / k0) == pytest.approx(kinf, rel=1e-10)
        # Troe blending stays within (0, 1] of the Lindemann value
        for M in (1e-4, 1e-1, 1e2):
            assert 0.0 < O.rate_constant(3, T, M) <= L.rate_constant(3, T, M)


def test_three_body_law(h2):
    """Only H, OH and N2 present: reaction 8 (H + OH + M <=> H2O + M, efficiencies 1 for these)
    proceeds forward only, q = k [M] C_H C_OH with [M] = C_H + C_OH + C_N2 (the textbook three-body
    law), and wdot_H2O = W_H2O (q_8 + nothing else producing water from these species)."""
    m, om, kd = h2
    kin = oracle.Kin(kd)
    T, p = 2000.0, 101325.0
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    X = np.zeros(9); X[3], X[5], X[8] = 0.01, 0.02, 0.97
    Y = X * W / (X @ W)
    w, q, _ = kin.cell(om, T, p, Y)
    C = p / (RU * T) * X
    k8 = kd["A"][7] * T ** kd["b"][7]
    assert q[7] == pytest.approx(k8 * C.sum() * C[3] * C[5], rel=1e-13)
    assert w[2] == pytest.approx(W[2] * q[7], rel=1e-13)   # H2O is made only by reaction 8 here
