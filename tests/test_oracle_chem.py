"""Pins for the oracle's DNN chemistry (
PAPER.md:114 §2: per-species nets, hidden 1600/800/400, GELU, inputs T, p, Y)."""
import math

import numpy as np
import pytest
import torch

from workload import make_bundle, make_cells
from workload.bundle import split_params


def test_gelu_values(orc):
    # GELU(x) = x Phi(x) (exact erf form)
    assert orc.gelu(0.0) == 0.0
    assert orc.gelu(1.0) == pytest.approx(0.8413447460685429, rel=1e-15)
    assert abs(orc.gelu(-10.0)) < 1e-21
    assert orc.gelu(30.0) == 30.0
    assert orc.gelu(-1.0) == pytest.approx(-0.15865525393145707, rel=1e-14)


@pytest.mark.parametrize("hidden", [(64, 32, 16), (1600, 800, 400)])
def test_forward_matches_torch_float64(orc, hidden):
    b = make_bundle("h2_9sp", hidden=hidden)
    mlp = orc.Mlp(b)
    rng = np.random.default_rng(4)
    for net in (0, b["n_nets"] - 1):
        W1, b1, W2, b2, W3, b3, W4, b4 = [torch.from_numpy(np.array(a)) for a in split_params(b, net)]
        seq = torch.nn.Sequential(torch.nn.Linear(11, hidden[0]), torch.nn.GELU(), torch.nn.Linear(hidden[0], hidden[1]),
                                  torch.nn.GELU(), torch.nn.Linear(hidden[1], hidden[2]), torch.nn.GELU(),
                                  torch.nn.Linear(hidden[2], 1)).double()
        with torch.no_grad():
            for lin, (W, bb) in zip([seq[0], seq[2], seq[4], seq[6]], [(W1, b1), (W2, b2), (W3, b3), (W4, b4)]):
                lin.weight.copy_(W); lin.bias.copy_(bb)
            for _ in range(3):
                z = rng.normal(size=11)
                ref = seq(torch.from_numpy(z)[None]).item()
                assert mlp.forward(net, z) == pytest.approx(ref, rel=1e-12, abs=1e-14)


def test_forward_hand_computable(orc):
    # W2 = W3 = 0: o = w4 . GELU(b3) + b4 regardless of the input
    b = make_bundle("h2_9sp", hidden=(64, 32, 16))
    W1, b1, W2, b2, W3, b3, W4, b4 = split_params(b, 0)
    W2[:] = 0.0; W3[:] = 0.0
    mlp = orc.Mlp(b)
    g = [0.5 * x * (1 + math.erf(x / math.sqrt(2))) for x in b3]
    ref = sum(w * v for w, v in zip(W4[0], g)) + b4[0]
    for z in (np.zeros(11), np.ones(11) * 3.0):
        assert mlp.forward(0, z) == pytest.approx(ref, rel=1e-14)


def _mech_E(mech):
    W = (mech["atoms"] * mech["W_elem"][:, None]).sum(0)
    return mech["atoms"] * mech["W_elem"][:, None] / W[None, :]


@pytest.mark.parametrize("name", ["h2_9sp", "ch4_20sp"])
def test_projection_properties(orc, name):
    from workload import load_mech
    mech = load_mech(name)
    P = orc.Mech(mech).projection()
    E = _mech_E(mech)
    ns, ne = mech["ns"], mech["ne"]
    np.testing.assert_allclose(P @ P, P, atol=1e-14)
    np.testing.assert_allclose(P, P.T, atol=1e-15)
    np.testing.assert_allclose(E @ P, 0.0, atol=1e-14)
    np.testing.assert_allclose(np.ones(ns) @ P, 0.0, atol=1e-14)
    assert np.trace(P) == pytest.approx(ns - ne, abs=1e-12)          # rank ns - ne
    n2 = mech["species"].index("N2")                                   # sole N carrier
    np.testing.assert_allclose(P[n2], 0.0, atol=1e-15)
    np.testing.assert_allclose(P[:, n2], 0.0, atol=1e-15)
    # P is THE orthogonal projector onto null(E): P v = v for v in null(E)
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(E.T, mode="complete")
    v = Q[:, ne:] @ rng.normal(size=ns - ne)
    np.testing.assert_allclose(P @ v, v, atol=1e-14)


def _thermo_h(orc, om, c):
    t = orc.step(om, None, c["T_true"], c["p"], c["Y"], mode="T", transport=False, chem=False)
    return t["h"]


def test_zero_output_bundle_is_identity(orc, h2mech):
    # o = 0 and mu_y = 0 -> Delta = 0 -> Y* = (Y^lambda)^(1/lambda) = Y -> wdot ~ 0
    b = make_bundle("h2_9sp", hidden=(64, 32, 16))
    b["params"][:] = 0.0
    om, mlp = orc.Mech(h2mech), orc.Mlp(b)
    c = make_cells("C1")
    h = _thermo_h(orc, om, c)
    r = orc.step(om, mlp, c["T_guess"], c["p"], c["Y"], h=h)
    assert np.all(r["o"] == 0.0)
    scale = r["rho"] * np.abs(c["Y"]).max(axis=0) / b["dt"]
    assert np.all(np.abs(r["wdot"]) <= 1e-14 * scale[None, :])


def test_chem_conservation_and_batch_invariance(orc, h2mech):
    b = make_bundle("h2_9sp", hidden=(64, 32, 16))
    om, mlp = orc.Mech(h2mech), orc.Mlp(b)
    c = make_cells("C1")
    h = _thermo_h(orc, om, c)
    r = orc.step(om, mlp, c["T_guess"], c["p"], c["Y"], h=h)
    w = r["wdot"]
    E = _mech_E(h2mech)
    tot = np.abs(w).sum(axis=0)
    assert np.all(np.abs(w.sum(axis=0)) <= 1e-12 * tot)                    # sum_k wdot_k = 0
    assert np.all(np.abs(E @ w) <= 1e-12 * tot[None, :])                   # element conservation
    n2 = h2mech["species"].index("N2")
    assert np.all(w[n2] == 0.0)
    assert np.linalg.norm(w) > 0
    # qdot = -sum_k h_k(T) wdot_k = -(rho/dt) (h(T, Y + dY) - h(T, Y)) since h is affine in Y
    for i in range(0, 1000, 111):
        Yh = np.maximum(c["Y"][:, i], 0.0)
        dY = w[:, i] * b["dt"] / r["rho"][i]
        ref = -(r["rho"][i] / b["dt"]) * (om.h(Yh + dY, r["T"][i]) - om.h(Yh, r["T"][i]))
        assert r["qdot"][i] == pytest.approx(ref, rel=1e-6, abs=1e-9 * np.abs(r["qdot"]).max())
    # batch of 1000 == 10 batches of 100, bitwise
    for s in range(0, 1000, 100):
        sl = slice(s, s + 100)
        q = orc.step(om, mlp, c["T_guess"][sl], c["p"][sl], c["Y"][:, sl], h=h[sl], nthreads=3)
        for k in ("T", "cp", "rho", "mu", "lambda", "qdot"):
            assert np.array_equal(q[k], r[k][sl]), k
        for k in ("D", "o", "wdot"):
            assert np.array_equal(q[k], r[k][:, sl]), k
    # Neumaier sum of qdot equals the exactly-rounded sum (math.fsum)
    assert r["red"][1] == pytest.approx(math.fsum(r["qdot"]), rel=1e-15, abs=0.0)


def test_inverse_box_cox_single_net(orc, h2mech):
    # only b4 nonzero: o = b4 for every cell -> Y*_s = (Y_s^l + l (b4 sigma_y))^(1/l)
    b = make_bundle("h2_9sp", hidden=(64, 32, 16))
    b["params"][:] = 0.0
    b["params"][:, -1] = 0.5           # b4 of every net
    om, mlp = orc.Mech(h2mech), orc.Mlp(b)
    c = make_cells("C1", 400, 420)
    h = _thermo_h(orc, om, c)
    r = orc.step(om, mlp, c["T_guess"], c["p"], c["Y"], h=h)
    assert np.all(r["o"] == 0.5)
    P = om.projection()
    lam, d = b["lambda_bc"], 0.5 * b["y_std"][0]
    for i in range(20):
        Yh = np.maximum(c["Y"][:, i], 0.0)
        dY = np.zeros(9)
        for net, s in enumerate(b["species_of_net"]):
            a = Yh[s] ** lam + lam * d
            dY[s] = (a ** (1 / lam) if a > 0 else 0.0) - Yh[s]
        np.testing.assert_allclose(r["wdot"][:, i], r["rho"][i] * (P @ dY) / b["dt"], rtol=1e-11,
                                   atol=1e-13 * np.abs(r["wdot"][:, i]).max())


def _torch_net(b, net):
    """torch.nn float64 Sequential with net `net`'s weights (GELU MLP); for a shared
    bundle the one net with all n_nets outputs."""
    d, hid = b["d_in"], b["hidden"]
    dims = [d, *hid, b["n_nets"] if b.get("shared") else 1]
    layers = []
    for l in range(4):
        layers.append(torch.nn.Linear(dims[l], dims[l + 1]))
        if l < 3:
            layers.append(torch.nn.GELU(approximate="none"))
    seq = torch.nn.Sequential(*layers).double()
    W = split_params(b, net)
    with torch.no_grad():
        for l in range(4):
            seq[2 * l].weight.copy_(torch.from_numpy(np.array(W[2 * l])))
            seq[2 * l].bias.copy_(torch.from_numpy(np.array(W[2 * l + 1])))
    return seq


@pytest.mark.parametrize("hidden,cfg,n", [((64, 32, 16), "C1", 200), ((1600, 800, 400), "C2", 64)])
def test_step_field_path_matches_torch(orc, h2mech, hidden, cfg, n):
    """Pins orc_step's own MLP path (dense_t over transposed W1..W3, oracle.c) and the
    z-score of step 6: the o the GPU is compared
    against equals torch float64 Linear/GELU(erf) applied to z computed here from the
    definition x = [T, p, (max(Y,0)^lambda - 1)/lambda], z = (x - mu_x)/sigma_x.
    A transposed weight index, a dropped /sigma_x or a wrong Box-Cox fails it."""
    b = make_bundle("h2_9sp", hidden=hidden)
    om, mlp = orc.Mech(h2mech), orc.Mlp(b)
    c = make_cells(cfg, 0, n) if cfg == "C1" else make_cells(cfg, 300_000, 300_000 + n)
    r = orc.step(om, mlp, c["T_true"], c["p"], c["Y"], mode="T", transport=False)
    lam = b["lambda_bc"]
    x = np.vstack([c["T_true"][None], c["p"][None], (np.maximum(c["Y"], 0.0) ** lam - 1.0) / lam])   # [d_in][n]
    z = (x - b["x_mean"][:, None]) / b["x_std"][:, None]
    assert np.abs(z).max() < 50 and np.abs(z).std() > 0.1          # a real spread of inputs, not a saturated net
    for net in range(b["n_nets"]):
        with torch.no_grad():
            ref = _torch_net(b, net)(torch.from_numpy(np.ascontiguousarray(z.T))).numpy()[:, 0]
        np.testing.assert_allclose(r["o"][net], ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max())


def test_step_zscore_hand_computable(orc, h2mech):
    """x_mean = cell 0's own x and x_std = 1 make z(cell 0) = 0 exactly, so o(cell 0) =
    torch(0); x_mean = 0, x_std = 2 make z = x/2 (second point).  Pins the z-score
    (reading R4) independently of the bundle statistics."""
    b = make_bundle("h2_9sp", hidden=(64, 32, 16))
    c = make_cells("C1", 500, 532)
    lam = b["lambda_bc"]
    x = np.vstack([c["T_true"][None], c["p"][None], (np.maximum(c["Y"], 0.0) ** lam - 1.0) / lam])
    om = orc.Mech(h2mech)
    for xm, xs in ((x[:, 0].copy(), np.ones(b["d_in"])), (np.zeros(b["d_in"]), np.full(b["d_in"], 2.0))):
        bb = dict(b, x_mean=xm, x_std=xs)
        r = orc.step(om, orc.Mlp(bb), c["T_true"], c["p"], c["Y"], mode="T", transport=False)
        z0 = (x[:, 0] - xm) / xs
        if xs[0] == 1.0:
            assert np.all(np.abs(z0) <= 1e-12 * np.abs(x[:, 0]))
            z0 = np.zeros(b["d_in"])
        for net in (0, 3, 7):
            with torch.no_grad():
                ref = _torch_net(bb, net)(torch.from_numpy(z0)[None]).item()
            assert r["o"][net, 0] == pytest.approx(ref, rel=1e-12, abs=1e-14)


@pytest.mark.parametrize("hidden,cfg,n", [((64, 32, 16), "C1", 200), ((1600, 800, 400), "C2", 32)])
def test_shared_net_field_path_matches_torch(orc, h2mech, hidden, cfg, n):
    """NEXT-2 (reading R20): ONE net d_in -> h1 -> h2 -> h3 -> n_nets outputs.  orc_step's o[net]
    equals output `net` of a torch float64 Sequential ending in Linear(h3, n_nets), on z from the
    step-6 definition; orc_mlp_forward agrees; and wdot still conserves mass and elements."""
    b = make_bundle("h2_9sp", hidden=hidden, shared=True)
    assert b["params"].shape[0] == 1
    om, mlp = orc.Mech(h2mech), orc.Mlp(b)
    c = make_cells(cfg, 0, n) if cfg == "C1" else make_cells(cfg, 300_000, 300_000 + n)
    r = orc.step(om, mlp, c["T_true"], c["p"], c["Y"], mode="T", transport=False)
    lam = b["lambda_bc"]
    x = np.vstack([c["T_true"][None], c["p"][None], (np.maximum(c["Y"], 0.0) ** lam - 1.0) / lam])
    z = (x - b["x_mean"][:, None]) / b["x_std"][:, None]
    with torch.no_grad():
        ref = _torch_net(b, 0)(torch.from_numpy(np.ascontiguousarray(z.T))).numpy()   # [n][n_nets]
    np.testing.assert_allclose(r["o"], ref.T, rtol=1e-12, atol=1e-13 * np.abs(ref).max())
    for net in (0, b["n_nets"] - 1):
        assert mlp.forward(net, z[:, 0]) == pytest.approx(ref[0, net], rel=1e-12, abs=1e-14)
    tot = np.abs(r["wdot"]).sum(axis=0)
    assert np.all(np.abs(r["wdot"].sum(axis=0)) <= 1e-12 * tot)
    E = _mech_E(h2mech)
    assert np.all(np.abs(E @ r["wdot"]) <= 1e-12 * tot[None, :])


def test_shared_net_with_equal_output_rows_is_the_per_species_net(orc, h2mech):
    """A shared net whose output rows all equal net 0's W4 (and b4) is n_nets copies of the
    individual net 0: every o[net] equals the per-species bundle's o[0] bitwise (same summation
    order).  Pins the shared output-layer indexing against the per-species path."""
    bi = make_bundle("h2_9sp", hidden=(64, 32, 16))
    bs = make_bundle("h2_9sp", hidden=(64, 32, 16), shared=True)
    W = split_params(bi, 0)
    P = np.concatenate([np.ravel(W[k]) for k in range(6)] + [np.tile(W[6][0], bs["n_nets"]),
                                                             np.full(bs["n_nets"], W[7][0])])
    bs["params"] = P[None, :]
    c = make_cells("C1", 0, 64)
    om = orc.Mech(h2mech)
    ri = orc.step(om, orc.Mlp(bi), c["T_true"], c["p"], c["Y"], mode="T", transport=False)
    rs = orc.step(om, orc.Mlp(bs), c["T_true"], c["p"], c["Y"], mode="T", transport=False)
    for net in range(bs["n_nets"]):
        assert np.array_equal(rs["o"][net], ri["o"][0])
