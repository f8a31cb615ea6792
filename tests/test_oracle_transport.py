"""Pins for the oracle's transport (Wilke viscosity,
Mathur conductivity, mixture-averaged diffusivity, BASELINE.json north_star;
PAPER.md:112 "molecular transport models ... via the Cantera interface")."""
import json
import os

import numpy as np
import pytest

from conftest import synth_mech

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def const_visc_mech(W, mu_at_T, T):
    # sqrt(mu_k)/T^(1/4) = c0  ->  mu_k(T) = c0^2 sqrt(T): pick c0 so mu_k(T) = mu_at_T
    ns = len(W)
    visc = np.zeros((ns, 5))
    visc[:, 0] = np.sqrt(np.asarray(mu_at_T)) / T ** 0.25
    cond = np.zeros((ns, 5)); cond[:, 0] = 1.0
    diff = np.zeros((ns * (ns + 1) // 2, 5)); diff[:, 0] = 1.0
    return synth_mech(ns, W, visc=visc, cond=cond, diff=diff)


def test_wilke_textbook_example(orc):
    g = json.load(open(os.path.join(GOLD, "wilke_bsl_example.json")))
    mu_si = np.array(g["mu_poise"]) * 0.1            # poise -> Pa s
    m = orc.Mech(const_visc_mech(g["M"], mu_si, g["T"]))
    x = np.array(g["x"])
    W = np.array(g["M"])
    Y = x * W / np.dot(x, W)
    mu, _, _ = m.transport(g["T"], 101325.0, Y)
    assert mu == pytest.approx(g["mu_mix_poise"] * 0.1, rel=g["rel_tol"])


def test_wilke_identical_species(orc):
    # two copies of one species: Phi = 1 everywhere -> mu = mu_k for any split
    m = orc.Mech(const_visc_mech([28.0, 28.0, 28.0], [1.8e-5, 1.8e-5, 1.8e-5], 500.0))
    for a in (0.1, 0.5, 0.93):
        mu, _, _ = m.transport(500.0, 1e5, np.array([a, 1 - a, 0.0]))
        assert mu == pytest.approx(1.8e-5, rel=1e-14)


def test_pure_species_limits(orc, h2mech, ch4mech):
    for mech in (h2mech, ch4mech):
        m = orc.Mech(mech)
        ns = mech["ns"]
        for k in range(ns):
            Y = np.zeros(ns); Y[k] = 1.0
            for T, p in ((400.0, 101325.0), (2100.0, 2e5)):
                mu, lam, D = m.transport(T, p, Y)
                assert mu == pytest.approx(m.mu_k(k, T), rel=1e-14)
                assert lam == pytest.approx(m.lambda_k(k, T), rel=1e-14)
                assert D[k] == pytest.approx(m.D_jk(k, k, T, p), rel=1e-14)     # fallback D_kk
                for j in range(ns):
                    if j != k:   # trace species in pure k: D_j = D_jk (Blanc, one term)
                        assert D[j] == pytest.approx(m.D_jk(j, k, T, p), rel=1e-13)


def test_mathur_means(orc):
    # lambda = (arithmetic mean + harmonic mean)/2 of the species lambda_k weighted by X
    cond = np.zeros((2, 5)); cond[0, 0] = 0.02; cond[1, 0] = 0.18
    m = orc.Mech(synth_mech(2, [10.0, 10.0], visc=np.ones((2, 5)) * [1e-3, 0, 0, 0, 0], cond=cond,
                            diff=np.ones((3, 5)) * [1, 0, 0, 0, 0]))
    T = 900.0
    l1, l2 = 0.02 * np.sqrt(T), 0.18 * np.sqrt(T)
    for x in (0.25, 0.5, 0.8):
        _, lam, _ = m.transport(T, 1e5, np.array([x, 1 - x]))
        am = x * l1 + (1 - x) * l2
        hm = 1.0 / (x / l1 + (1 - x) / l2)
        assert lam == pytest.approx(0.5 * (am + hm), rel=1e-14)
    _, lam, _ = m.transport(T, 1e5, np.array([1.0, 0.0]))   # equal-lambda / pure limit
    assert lam == pytest.approx(l1, rel=1e-15)


def test_binary_mixture_averaged_D(orc, h2mech):
    # binary mixture: D_1m = (1 - Y_1) / (X_2 / D_12) = D_12 W_2 / Wbar
    m = orc.Mech(h2mech)
    W = (h2mech["atoms"] * h2mech["W_elem"][:, None]).sum(0)
    i, j = 0, 8  # H2 in N2
    for y in (0.01, 0.3, 0.9):
        Y = np.zeros(9); Y[i] = y; Y[j] = 1 - y
        T, p = 1300.0, 101325.0
        _, _, D = m.transport(T, p, Y)
        Wb = 1.0 / (y / W[i] + (1 - y) / W[j])
        D12 = m.D_jk(i, j, T, p)
        assert D[i] == pytest.approx(D12 * W[j] / Wb, rel=1e-13)
        assert D[j] == pytest.approx(D12 * W[i] / Wb, rel=1e-13)


def test_blanc_trace_limit(orc, ch4mech):
    # X_k = 0: D_k = 1 / sum_{j != k} X_j / D_jk (Blanc's law)
    m = orc.Mech(ch4mech)
    rng = np.random.default_rng(3)
    ns = ch4mech["ns"]
    W = (ch4mech["atoms"] * ch4mech["W_elem"][:, None]).sum(0)
    for _ in range(5):
        Y = rng.dirichlet(np.ones(ns)); k = rng.integers(ns); Y[k] = 0.0; Y /= Y.sum()
        T, p = rng.uniform(400, 2500), 101325.0
        _, _, D = m.transport(T, p, Y)
        X = Y / W / np.sum(Y / W)
        S = sum(X[j] / m.D_jk(j, k, T, p) for j in range(ns) if j != k)
        assert D[k] == pytest.approx(1.0 / S, rel=1e-13)


def test_negative_Y_clipped(orc, h2mech):
    # X+ = max(X, 0): a -1e-12 mass fraction behaves as 0 in the mixing rules
    m = orc.Mech(h2mech)
    Y = np.array([0.02, 0.2, 0.1, 0.0, 0.0, 0.0, 0.0, 0.0, 0.68])
    Yn = Y.copy(); Yn[5] = -1e-12
    a, b = m.transport(1500.0, 1e5, Y), m.transport(1500.0, 1e5, Yn)
    assert a[0] == pytest.approx(b[0], rel=1e-10) and a[1] == pytest.approx(b[1], rel=1e-10)


def neufeld_mu(W, eps, sig, T):
    ts = T / eps
    om = 1.16145 * ts ** -0.14874 + 0.52487 * np.exp(-0.77320 * ts) + 2.16178 * np.exp(-2.43787 * ts)
    return 2.6693e-6 * np.sqrt(W * T) / (sig ** 2 * om)


def test_fits_reproduce_chapman_enskog(orc, h2mech):
    # the fitted polynomials, evaluated by the oracle, track the Chapman-Enskog
    # values they were fitted to (parity against real Cantera data: unpinned)
    import json as _j
    raw = _j.load(open(os.path.join(os.path.dirname(__file__), "..", "data", "mech", "h2_9sp.json")))
    m = orc.Mech(h2mech)
    W = (h2mech["atoms"] * h2mech["W_elem"][:, None]).sum(0)
    for k, s in enumerate(h2mech["species"]):
        _, eps, sig, *_ = raw["lennard_jones"][s]
        for T in (300.0, 800.0, 1700.0, 3000.0):
            assert m.mu_k(k, T) == pytest.approx(neufeld_mu(W[k], eps, sig, T), rel=5e-3), s


def test_handbook_sanity(orc, h2mech):
    # physical plausibility (handbook values, loose): N2 and air at 300 K, H2-N2 diffusion
    m = orc.Mech(h2mech)
    N2, O2, H2 = 8, 1, 0
    assert m.mu_k(N2, 300.0) == pytest.approx(1.79e-5, rel=0.03)
    assert m.lambda_k(N2, 300.0) == pytest.approx(0.026, rel=0.10)
    assert m.D_jk(H2, N2, 300.0, 101325.0) == pytest.approx(7.8e-5, rel=0.05)
    Y = np.zeros(9); Y[O2] = 0.233; Y[N2] = 0.767
    mu, lam, _ = m.transport(300.0, 101325.0, Y)
    assert mu == pytest.approx(1.85e-5, rel=0.03)
    assert lam == pytest.approx(0.0263, rel=0.10)
