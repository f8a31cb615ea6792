"""CUDA path vs oracle, element by element on the same seeded inputs, through
the C ABI (include/rc.h).  Gates (BASELINE.json north_star):
  fp64 thermo/transport (T, cp, rho, mu, lambda, D_k)  |g - o| <= 1e-10 |o|
  bf16 MLP output o ("relative 2e-2 of the output norm")   ||g - o|| / ||o|| <= 2e-2
  bf16 wdot, qdot, sum qdot (derived, R17)    ||g - o|| / ||o|| <= 3e-2
  TF32 MLP o ("relative 1e-3 of the output norm")      <= 1e-3
  TF32 wdot, qdot (derived, R18)              <= 2e-3
  and, on every sample with an emulation (tests/_emulate.py), o and wdot errors within
  EMU_FACTOR x those of an MLP that only rounds its operands (the rounding floor)
  T_max                                                 1e-10
  GPU wdot conserves mass and elements                  1e-12 of sum |wdot|
  sharded == unsharded                                  bitwise
"""
import numpy as np
import pytest

from _harness import (BF16_DERIVED_TOL, BF16_TOL, EMU_FACTOR, FP64_TOL, TF32_DERIVED_TOL, TF32_TOL, Gpu, bundle,
                      inputs, max_rel, mech, rel_fro, run_oracle)
from workload import CONFIGS
from workload.cells import uniform

pytestmark = pytest.mark.gpu



@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_13513_b200 import build
    build.build()


def _E(m):
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    return m["atoms"] * m["W_elem"][:, None] / W[None, :]


def check_fp64(g, o, cols=None):
    for k in ("T", "cp", "rho", "mu", "lambda"):
        gv = g[k] if cols is None else g[k][cols]
        assert max_rel(gv, o[k]) <= FP64_TOL, (k, max_rel(gv, o[k]))
    gD = g["D"] if cols is None else g["D"][:, cols]
    assert max_rel(gD, o["D"]) <= FP64_TOL, ("D", max_rel(gD, o["D"]))


def check_chem(g, o, m, cols=None, tol=BF16_TOL, dtol=BF16_DERIVED_TOL, emu=None):
    """emu = (cfg, cells, variant): also hold o and wdot to EMU_FACTOR x the errors of the
    rounding-only emulation of `variant` on the same cells (tests/_emulate.py)."""
    go = g["o"] if cols is None else g["o"][:, cols]
    gw = g["wdot"] if cols is None else g["wdot"][:, cols]
    gq = g["qdot"] if cols is None else g["qdot"][cols]
    eo, ew, eq = rel_fro(go, o["o"]), rel_fro(gw, o["wdot"]), rel_fro(gq, o["qdot"])
    per_net = " ".join(f"{rel_fro(go[i], o['o'][i]):.1e}" for i in range(go.shape[0]))
    print(f"\n  errors o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}; per-net relative o error {per_net}")
    if emu is not None:
        from _emulate import emulated_errors
        cfg, cells, variant = emu
        C = CONFIGS[cfg]
        mo, mw, mq, _ = emulated_errors(mech(C.mech), bundle(C.mech, C.hidden), cells, o, variant)
        print(f"  rounding floor ({variant} emulation) o {mo:.2e} wdot {mw:.2e} qdot {mq:.2e}; "
              f"GPU/floor o {eo / mo:.2f} wdot {ew / mw:.2f}")
        assert eo <= EMU_FACTOR * mo, ("o vs rounding floor", eo, mo)
        assert ew <= EMU_FACTOR * mw, ("wdot vs rounding floor", ew, mw)
    assert eo <= tol, ("o", eo)
    assert ew <= dtol, ("wdot", ew)
    assert eq <= dtol, ("qdot", eq)
    # conservation of the GPU's own wdot (its projection runs in fp64)
    tot = np.abs(gw).sum(axis=0) + 1e-300
    assert np.all(np.abs(gw.sum(axis=0)) <= 1e-12 * tot)
    assert np.all(np.abs(_E(m) @ gw) <= 1e-12 * tot[None, :])
    return eo, ew, eq


def test_c1_full_parity():
    """C1: 1,000 premixed cells (ragged: 7 full 128-row tiles + 104), small MLP."""
    c = inputs("C1")
    o = run_oracle("C1", c)
    g = Gpu("C1").run(c)
    check_fp64(g, o)
    eo, ew, eq = check_chem(g, o, mech("h2_9sp"), emu=("C1", c, "bf16_ideal"))
    assert g["red"][0] == pytest.approx(o["red"][0], rel=FP64_TOL)
    assert g["red"][1] == pytest.approx(o["red"][1], rel=BF16_DERIVED_TOL)
    assert np.array_equal(g["diag"][[0, 1, 3]], o["diag"][[0, 1, 3]])
    assert g["diag"][2] == 0
    # negY_out is decided on the bf16 MLP's dY: equal up to cells at the sign boundary
    assert abs(int(g["diag"][4]) - int(o["diag"][4])) <= max(2, o["diag"][4] // 20), (g["diag"][4], o["diag"][4])
    print(f"C1 bf16 errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")


def test_c1_transport_and_thermo_only_paths():
    c = inputs("C1", begin=100, end=357)
    o = run_oracle("C1", c, chem=False)
    g = Gpu("C1").run(c, chem=False)
    check_fp64(g, o)
    assert "wdot" not in g or g.get("wdot") is None


def _sample(cfg, n):
    N = CONFIGS[cfg].n_cells
    return np.unique((uniform(4242, np.arange(n)) * N).astype(np.int64))


@pytest.mark.parametrize("cfg", ["C2"])
def test_full_size_sampled(cfg):
    """BASELINE configs[1] at full size (1,048,576 cells, paper MLP 1600/800/400),
    the bench's launch configuration; the oracle checks a hashed sample."""
    n = CONFIGS[cfg].n_cells
    c = inputs(cfg, begin=0, end=n)
    g = Gpu(cfg).run(c)
    cols = _sample(cfg, 192)
    sub = {k: (v[..., cols] if isinstance(v, np.ndarray) else v) for k, v in c.items()}
    o = run_oracle(cfg, sub)
    check_fp64(g, o, cols)
    eo, ew, eq = check_chem(g, o, mech(CONFIGS[cfg].mech), cols, emu=(cfg, sub, "bf16_ideal"))
    print(f"{cfg} sampled bf16 errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")
    # whole-field properties that hold at any size
    assert np.all(np.isfinite(g["wdot"])) and g["diag"][2] == 0
    assert g["red"][0] == pytest.approx(g["T"].max(), rel=0, abs=0)
    tot = np.abs(g["wdot"]).sum(axis=0) + 1e-300
    assert np.all(np.abs(g["wdot"].sum(axis=0)) <= 1e-12 * tot)


def test_small_mlp_many_tiles_per_cta():
    """C1's narrow MLP (64/32/16: pass widths below one 64-column block) on 65,536 C2
    cells, so every persistent CTA pair runs several tiles (accumulator reuse, warps
    with no columns still releasing the accumulator); every cell checked."""
    c = inputs("C2", begin=0, end=65536)
    o = run_oracle("C1", c)
    g = Gpu("C1").run(c)
    check_fp64(g, o)
    eo, ew, eq = check_chem(g, o, mech("h2_9sp"))
    print(f"small MLP x 65536 cells bf16 errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")


def test_tf32_c1_full():
    """TF32 MLP (RC_TF32: tf32 operands, fp32 accumulate, exact-erf GELU) on all C1 cells."""
    c = inputs("C1")
    o = run_oracle("C1", c)
    g = Gpu("C1", precision=1).run(c)
    check_fp64(g, o)
    eo, ew, eq = check_chem(g, o, mech("h2_9sp"), tol=TF32_TOL, dtol=TF32_DERIVED_TOL, emu=("C1", c, "tf32"))
    print(f"C1 tf32 errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")


def test_tf32_paper_shape_sample():
    """TF32 MLP at the paper's widths (1600/800/400): C2 on 65,536 cells, hashed sample checked."""
    c = inputs("C2", begin=0, end=65536)
    g = Gpu("C2", precision=1).run(c)
    cols = np.unique((uniform(4242, np.arange(128)) * 65536).astype(np.int64))
    sub = {k: (v[..., cols] if isinstance(v, np.ndarray) else v) for k, v in c.items()}
    o = run_oracle("C2", sub)
    eo, ew, eq = check_chem(g, o, mech("h2_9sp"), cols, tol=TF32_TOL, dtol=TF32_DERIVED_TOL,
                            emu=("C2", sub, "tf32"))
    print(f"C2 tf32 sampled errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")


@pytest.mark.parametrize("cfg,n", [("C1", 1000), ("C2", 65536)])
def test_tf32x3_meets_1e3_on_outputs_and_wdot(cfg, n):
    """RC_TF32X3 (three tf32 MMAs per product on hi/lo operand pairs: fp32-accurate
    GEMMs): the 1e-3 gate holds for o and for the derived wdot/qdot too (R18)."""
    c = inputs(cfg, begin=0, end=n)
    g = Gpu(cfg, precision=2).run(c)
    cols = np.unique((uniform(4343, np.arange(128)) * n).astype(np.int64)) if n > 1000 else None
    sub = c if cols is None else {k: (v[..., cols] if isinstance(v, np.ndarray) else v) for k, v in c.items()}
    o = run_oracle(cfg, sub)
    if cols is None:
        check_fp64(g, o)
    eo, ew, eq = check_chem(g, o, mech("h2_9sp"), cols, tol=TF32_TOL, dtol=TF32_TOL)
    print(f"{cfg} tf32x3 errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")


def test_layerwise_path_paper_shape():
    """The layer-wise bf16 path (layer-1 kernel + layer-2 pair GEMM, h1 through the workspace;
    rc_mlp_desc.flags = RC_MLP_LAYERWISE) at the paper widths, the path the fused layer-1/2
    kernel replaces by default."""
    import paper_2312_13513_b200 as rc
    c = inputs("C2", begin=0, end=65536)
    G = Gpu("C2")
    G.mlp = rc.MLPBundle(G.mech, bundle("h2_9sp", CONFIGS["C2"].hidden), rc.RC_BF16, flags=rc._rc.RC_MLP_LAYERWISE)
    g = G.run(c)
    cols = np.unique((uniform(4444, np.arange(128)) * 65536).astype(np.int64))
    sub = {k: (v[..., cols] if isinstance(v, np.ndarray) else v) for k, v in c.items()}
    o = run_oracle("C2", sub)
    eo, ew, eq = check_chem(g, o, mech("h2_9sp"), cols, emu=("C2", sub, "bf16_ideal"))
    print(f"C2 layer-wise bf16 errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")
    # the fused kernel on the same cells: same arithmetic per output up to summation order
    f = Gpu("C2").run(c)
    assert rel_fro(f["o"], g["o"]) < 2e-3


@pytest.mark.parametrize("hidden", [(64, 48, 16), (128, 96, 48), (192, 240, 80), (1600, 768, 384), (2560, 800, 400)])
def test_odd_widths_create_and_run(hidden):
    """Every width rc_mlp_create accepts runs (pass widths without a kernel instance;
    KZ = 16 fused kernel whose whole-net W1 rows outgrow shared memory at h1 >= 2496 must take
    the layer-wise path up front).  Parity against the oracle on 256 C2 cells."""
    from workload import make_bundle
    b = make_bundle("h2_9sp", hidden=hidden)
    c = inputs("C2", begin=500_000, end=500_256)
    o = run_oracle("C2", c, b=b)
    g = Gpu("C2", b=b).run(c)
    check_fp64(g, o)
    eo, ew, eq = check_chem(g, o, mech("h2_9sp"))
    print(f"hidden {hidden} bf16 errors: o {eo:.2e} wdot {ew:.2e}")


def test_ch4_paper_shape_sample():
    """C4 (CH4/air, 20 species, 19 nets, d_in 22): parity on a hashed sample."""
    cols = _sample("C4", 256)
    c = inputs("C4", idx=cols)
    o = run_oracle("C4", c)
    g = Gpu("C4").run(c)
    check_fp64(g, o)
    check_chem(g, o, mech("ch4_20sp"), emu=("C4", c, "bf16_ideal"))


@pytest.mark.parametrize("prec", [0, 1])
def test_ch4_many_tiles_per_cluster(prec):
    """C4 on 65,536 contiguous cells (256 row blocks: every persistent cluster of the fused
    KZ = 32 kernel runs several tiles, so its per-chunk W1 ring continues across tiles and
    across the 19 nets), hashed sample checked; bf16 and TF32."""
    n = 65536
    c = inputs("C4", begin=2_000_000, end=2_000_000 + n)
    g = Gpu("C4", precision=prec).run(c)
    cols = np.unique((uniform(4646 + prec, np.arange(160)) * n).astype(np.int64))
    sub = {k: (v[..., cols] if isinstance(v, np.ndarray) else v) for k, v in c.items()}
    o = run_oracle("C4", sub)
    check_fp64(g, o, cols)
    tol, dtol = (BF16_TOL, BF16_DERIVED_TOL) if prec == 0 else (TF32_TOL, TF32_DERIVED_TOL)
    eo, ew, eq = check_chem(g, o, mech("ch4_20sp"), cols, tol=tol, dtol=dtol,
                            emu=("C4", sub, "bf16_ideal" if prec == 0 else "tf32"))
    print(f"C4 65536-cell precision {prec} errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")
    assert np.all(np.isfinite(g["wdot"])) and g["diag"][2] == 0


def test_inverse_box_cox_nonpositive_base():
    """SURVEY §8(c) step 8 / reading R3: with all weights zero and b4 = -1000 on the H2 net,
    o = -1000 exactly on both sides, a = Yh^lambda + lambda sigma_y o < 0, so Y*_H2 = 0
    (the a <= 0 branch); other nets have b4 = +0.5.  wdot / qdot follow in fp64 from an
    exact o, so they match the oracle to fp64 rounding, and negY_out (diag[4]) equals the
    oracle's count exactly."""
    from workload import make_bundle
    b = make_bundle("h2_9sp", hidden=(64, 32, 16))
    b["params"][:] = 0.0
    b["params"][:, -1] = 0.5
    b["params"][0, -1] = -1000.0     # net 0 predicts species 0 (H2)
    assert b["species_of_net"][0] == 0
    c = inputs("C1")
    o = run_oracle("C1", c, b=b)
    assert np.all(o["o"][0] == -1000.0)
    lam = b["lambda_bc"]
    assert np.all(np.maximum(c["Y"][0], 0) ** lam + lam * b["y_std"][0] * -1000.0 < 0)
    for prec in (0, 1):
        g = Gpu("C1", precision=prec, b=b).run(c)
        assert np.array_equal(g["o"], o["o"].astype(np.float32))
        assert rel_fro(g["wdot"], o["wdot"]) <= 1e-12, rel_fro(g["wdot"], o["wdot"])
        assert max_rel(g["qdot"], o["qdot"]) <= 1e-9
        assert o["diag"][4] > 0
        assert np.array_equal(g["diag"], o["diag"]), (g["diag"], o["diag"])


@pytest.mark.parametrize("mname,cfg,perm", [("h2_9sp", "C1", "identity"), ("h2_9sp", "C1", "reversed"),
                                            ("h2_9sp", "C1", "subset"), ("ch4_20sp", "C4", "identity"),
                                            ("ch4_20sp", "C4", "reversed")])
def test_projection_both_forms_exact_outputs(mname, cfg, perm):
    """The epilogue applies P = I - E^T (E E^T)^-1 E in factored form when net i predicts species i
    (the mechanisms' layout) and as columns of P otherwise; both against the oracle's P (step 9) on
    exact outputs: zero hidden weights and a distinct fp32-exact b4 per net, so o is exact on both sides and
    wdot / qdot differ only by fp64 rounding.  'reversed' maps net i to species n_nets - 1 - i,
    'subset' drops every other net (species without a net get dY = 0)."""
    from workload import make_bundle
    b = make_bundle(mname, hidden=(64, 32, 16))
    nn = b["n_nets"]
    if perm == "reversed":
        b["species_of_net"] = b["species_of_net"][::-1].copy()
    elif perm == "subset":
        keep = np.arange(0, nn, 2)
        b["n_nets"], b["species_of_net"] = keep.size, b["species_of_net"][keep].copy()
        for k in ("params", "y_mean", "y_std"):
            b[k] = b[k][keep].copy()
    b["params"][:] = 0.0
    b["params"][:, -1] = 0.25 + np.arange(b["n_nets"]) / 64.0   # exact in fp32 (the kernel's o)
    cols = None if cfg == "C1" else _sample(cfg, 96)
    c = inputs(cfg) if cols is None else inputs(cfg, idx=cols)
    o = run_oracle(cfg, c, b=b)
    g = Gpu(cfg, b=b).run(c)
    assert np.array_equal(g["o"], o["o"].astype(np.float32))
    assert rel_fro(g["wdot"], o["wdot"]) <= 1e-12, rel_fro(g["wdot"], o["wdot"])
    assert max_rel(g["qdot"], o["qdot"]) <= 1e-9
    assert np.array_equal(g["diag"], o["diag"]), (g["diag"], o["diag"])
    m = mech(mname)
    W = (m["atoms"] * m["W_elem"][:, None]).sum(0)
    E = m["atoms"] * m["W_elem"][:, None] / W[None, :]
    tot = np.abs(g["wdot"]).sum(axis=0) + 1e-300
    assert np.all(np.abs(E @ g["wdot"]) <= 1e-12 * tot[None, :])


@pytest.mark.parametrize("prec,tol,dtol", [(1, 1e-3, 2e-3), (2, 1e-3, 1e-3)])
def test_ch4_tf32_modes_sample(prec, tol, dtol):
    """C4 (d_in 22 -> 32-wide z rows, 19 nets) in the TF32 and TF32X3 modes."""
    cols = _sample("C4", 128)
    c = inputs("C4", idx=cols)
    o = run_oracle("C4", c)
    g = Gpu("C4", precision=prec).run(c)
    check_fp64(g, o)
    eo, ew, eq = check_chem(g, o, mech("ch4_20sp"), tol=tol, dtol=dtol, emu=("C4", c, "tf32") if prec == 1 else None)
    print(f"C4 precision {prec} errors: o {eo:.2e} wdot {ew:.2e} qdot {eq:.2e}")


def test_padding_untouched_and_single_cell():
    c = inputs("C1", begin=0, end=1)
    o = run_oracle("C1", c)
    g = Gpu("C1").run(c, ld=64)
    check_fp64(g, o)
    check_chem(g, o, mech("h2_9sp"))


def test_empty_is_noop():
    import torch
    import paper_2312_13513_b200 as rc
    G = Gpu("C1")
    st = rc.CellState(0, G.ns, G.n_nets, ld=2)
    ws = rc.aligned_workspace(G.mlp, 128)
    rc.rc_step(G.mech, G.mlp, st.cells(rc.RC_MODE_H, dt=G.dt), ws)
    torch.cuda.synchronize()
    assert st.diag.sum().item() == 0


def test_errors():
    import paper_2312_13513_b200 as rc
    G = Gpu("C1")
    st = rc.CellState(10, G.ns, G.n_nets)
    ws = rc.aligned_workspace(G.mlp, 10)
    with pytest.raises(rc.RcError) as e:
        rc.rc_step(G.mech, G.mlp, st.cells(rc.RC_MODE_H, dt=2e-6), ws)
    assert e.value.code == rc._rc.RC_EDTMISMATCH
    bad = st.cells(rc.RC_MODE_H, dt=G.dt)
    bad.ld = 5
    with pytest.raises(rc.RcError) as e:
        rc.rc_step(G.mech, G.mlp, bad, ws)
    assert e.value.code == rc._rc.RC_EINVAL
    bad = st.cells(rc.RC_MODE_H, dt=G.dt)
    bad.p = bad.p + 8
    with pytest.raises(rc.RcError) as e:
        rc.rc_step(G.mech, G.mlp, bad, ws)
    assert e.value.code == rc._rc.RC_EALIGN


def test_out_of_range_h_bisects_like_oracle():
    c = inputs("C1", begin=500, end=520)
    c["h"][3] = c["h"][3] + 5e7          # far above h(T_max): Newton clamps twice -> bisection
    c["h"][7] = -5e7 + c["h"][7]         # far below h(T_min)
    o = run_oracle("C1", c, chem=False)
    g = Gpu("C1").run(c, chem=False)
    assert o["diag"][0] == 2
    assert np.array_equal(g["diag"][:2], o["diag"][:2])
    assert max_rel(g["T"], o["T"]) <= FP64_TOL


@pytest.mark.parametrize("prec", [0, 1])
def test_sharded_equals_unsharded_bitwise(prec):
    """Cells are independent: running G shards (rc_partition) one after another
    reproduces the unsharded per-cell outputs bit for bit, for the fused
    bf16 and TF32 kernels alike; a repeated run is bitwise identical (deterministic)."""
    import paper_2312_13513_b200 as rc
    c = inputs("C2", begin=300000, end=300000 + 5000)
    G = Gpu("C2", precision=prec)
    whole = G.run(c)
    again = G.run(c)
    for k in ("T", "cp", "rho", "mu", "lambda", "qdot", "D", "wdot", "o", "red", "diag"):
        assert np.array_equal(again[k], whole[k]), k
    for world in (2, 3):
        for r in range(world):
            b, e = rc.rc_partition(5000, r, world)
            part = {k: (v[..., b:e] if isinstance(v, np.ndarray) else v) for k, v in c.items()}
            g = G.run(part)
            for k in ("T", "cp", "rho", "mu", "lambda", "qdot"):
                assert np.array_equal(g[k], whole[k][b:e]), (k, world, r)
            for k in ("D", "wdot", "o"):
                assert np.array_equal(g[k], whole[k][:, b:e]), (k, world, r)


def test_sub_batches_in_place_and_combined_reductions():
    """One step run as three sub-batches on views of the same component-major arrays
    (pointer offsets, shared ld), each with its own red/diag, then rc_combine_reductions:
    per-cell outputs bitwise equal to the single call, T_max exact, sum qdot to rounding."""
    import torch
    import paper_2312_13513_b200 as rc
    c = inputs("C1")
    G = Gpu("C1")
    whole = G.run(c)
    n = c["p"].shape[0]
    st = rc.CellState(n, G.ns, G.n_nets).load(c["T_guess"], c["p"], c["Y"], h=c["h"])
    ws = rc.aligned_workspace(G.mlp, n)
    parts = [(0, 384), (384, 768), (768, n)]
    red_parts = torch.zeros(len(parts), 2, dtype=torch.float64, device="cuda")
    diag_parts = torch.zeros(len(parts), 5, dtype=torch.int64, device="cuda")
    for i, (b, e) in enumerate(parts):
        cells = rc.make_cells(e - b, st.ld, rc.RC_MODE_H, st.T[b:], st.p[b:], st.Y[:, b:], h=st.h[b:], cp=st.cp[b:],
                              rho=st.rho[b:], mu=st.mu[b:], lam=st.lam[b:], D=st.D[:, b:], wdot=st.wdot[:, b:],
                              qdot=st.qdot[b:], o=st.o[:, b:], dt=G.dt, red=red_parts[i], diag=diag_parts[i])
        rc.rc_step(G.mech, G.mlp, cells, ws)
    red = torch.zeros(2, dtype=torch.float64, device="cuda")
    diag = torch.zeros(5, dtype=torch.int64, device="cuda")
    rc.rc_combine_reductions(red_parts, diag_parts, red, diag)
    torch.cuda.synchronize()
    g = st.host()
    for k, gk in (("T", "T"), ("cp", "cp"), ("rho", "rho"), ("mu", "mu"), ("lambda", "lam"), ("qdot", "qdot")):
        assert np.array_equal(g[gk], whole[k]), k
    for k in ("D", "wdot", "o"):
        assert np.array_equal(g[k], whole[k]), k
    r = red.cpu().numpy()
    assert r[0] == whole["red"][0]
    assert r[1] == pytest.approx(whole["red"][1], rel=1e-13)
    assert np.array_equal(diag.cpu().numpy(), whole["diag"])


def test_chunking_is_invisible_per_cell():
    """The MLP runs in chunks sized to the workspace (z for every cell + one chunk of
    activations): a third of rc_workspace_bytes gives several chunks with a ragged last one.
    Per-cell outputs are bitwise those of the one-chunk call; below the minimum (z of every
    cell + a 256-cell chunk) the call fails with RC_EINVAL before any launch."""
    import paper_2312_13513_b200 as rc
    n = 65536 + 300
    c = inputs("C2", begin=0, end=n)
    G = Gpu("C2")
    one = G.run(c)
    full = rc.aligned_workspace(G.mlp, n)
    part = full[: (full.numel() // 3) // 256 * 256]
    several = G.run(c, ws=part)
    for k in ("T", "cp", "rho", "mu", "lambda", "qdot"):
        assert np.array_equal(several[k], one[k]), k
    for k in ("D", "wdot", "o"):
        assert np.array_equal(several[k], one[k]), k
    assert several["red"][1] == pytest.approx(one["red"][1], rel=1e-12)
    with pytest.raises(rc.RcError) as e:
        G.run(c, ws=full[: 1 << 20])
    assert e.value.code == rc._rc.RC_EINVAL


def test_cuda_graph_capture_replays_rc_step_bitwise():
    """SURVEY A16/K10 (the per-step kernel suite launched as a CUDA graph): rc_step
    captured once with torch.cuda.graph and replayed gives bitwise the eager results (every kernel is
    deterministic; the tensor maps travel by value in the kernel parameters)."""
    import torch

    import paper_2312_13513_b200 as rc
    c = inputs("C2", begin=0, end=4096)
    G = Gpu("C2")
    n = 4096
    st = rc.CellState(n, G.ns, G.n_nets)
    st.load(c["T_guess"], c["p"], c["Y"], h=c["h"])
    ws = rc.aligned_workspace(G.mlp, n)
    cells = st.cells(rc.RC_MODE_H, dt=G.dt)
    T0 = st.T.clone()
    rc.rc_step(G.mech, G.mlp, cells, ws)            # eager (also warms the host-side caches)
    torch.cuda.synchronize()
    ref = st.host()
    st.T.copy_(T0)
    for t in (st.cp, st.rho, st.mu, st.lam, st.D, st.wdot, st.qdot, st.o):
        t.zero_()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        rc.rc_step(G.mech, G.mlp, cells, ws, side)
    for _ in range(2):                               # replay twice from the restored guess
        st.T.copy_(T0)
        graph.replay()
    torch.cuda.synchronize()
    out = st.host()
    for k in ("T", "cp", "rho", "mu", "lam", "D", "wdot", "qdot", "o", "red", "diag"):
        assert np.array_equal(out[k], ref[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [0, 1])
def test_layer3_overlap_bitwise_equals_serial(prec):
    """Layer 3 of chunk j - 1 overlapped with the fused layer-1/2 kernel of chunk j (DESIGN.md 6.4:
    side launches on the SMs the fused kernel's 4-CTA clusters leave idle, tiles from a shared
    counter, h2 in two alternating buffers) gives bitwise the one-stream result (RC_MLP_SERIAL) on a
    three-chunk call with a ragged last chunk; the side launches ran (rc_overlap_read)."""
    import paper_2312_13513_b200 as rc
    n = 2 * 262144 + 75_008
    c = inputs("C2", begin=0, end=n)
    G = Gpu("C2", precision=prec)
    rc.rc_overlap_read(reset=True)
    ov = G.run(c)
    cnt = rc.rc_overlap_read(reset=True)
    print(f"\n  overlap counters (precision {prec}): {cnt}")
    assert cnt["pairs_ran"] + cnt["pairs_gave_up"] > 0  # two side launches were made
    G.mlp = rc.MLPBundle(G.mech, bundle("h2_9sp", CONFIGS["C2"].hidden), prec, flags=rc.RC_MLP_SERIAL)
    se = G.run(c)
    assert rc.rc_overlap_read(reset=True)["pairs_ran"] == 0
    for k in ("T", "cp", "rho", "mu", "lambda", "qdot", "D", "wdot", "o", "red", "diag"):
        assert np.array_equal(ov[k], se[k]), k
    # and against the oracle on a hashed sample of the three chunks
    idx = np.unique(np.random.default_rng(7).integers(0, n, 96))
    cs = inputs("C2", idx=idx)
    ref = run_oracle("C2", cs, nthreads=0)
    assert rel_fro(ov["o"][:, idx], ref["o"]) <= (BF16_TOL if prec == 0 else TF32_TOL)


@pytest.mark.gpu
def test_cuda_graph_capture_with_layer3_overlap():
    """rc_step with the layer-3 overlap (auxiliary stream forked and joined by events inside the call)
    captured into a CUDA graph replays bitwise the eager result."""
    import torch

    import paper_2312_13513_b200 as rc
    n = 262144 + 40_000
    c = inputs("C2", begin=0, end=n)
    G = Gpu("C2")
    st = rc.CellState(n, G.ns, G.n_nets)
    st.load(c["T_guess"], c["p"], c["Y"], h=c["h"])
    ws = rc.aligned_workspace(G.mlp, n)
    cells = st.cells(rc.RC_MODE_H, dt=G.dt)
    T0 = st.T.clone()
    rc.rc_step(G.mech, G.mlp, cells, ws)
    torch.cuda.synchronize()
    ref = st.host()
    st.T.copy_(T0)
    for t in (st.cp, st.rho, st.mu, st.lam, st.D, st.wdot, st.qdot, st.o):
        t.zero_()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        rc.rc_step(G.mech, G.mlp, cells, ws, side)
    for _ in range(2):
        st.T.copy_(T0)
        graph.replay()
    torch.cuda.synchronize()
    out = st.host()
    for k in ("T", "cp", "rho", "mu", "lam", "D", "wdot", "qdot", "o", "red", "diag"):
        assert np.array_equal(out[k], ref[k]), k


@pytest.mark.gpu
def test_layer3_overlap_bitwise_equals_serial_ch4():
    """The same for CH4 (19 nets, KZ = 32 fused kernel): a 100,000-cell call runs as two chunks with
    the layer-3 side launch; bitwise equal to RC_MLP_SERIAL."""
    import paper_2312_13513_b200 as rc
    n = 100_000
    c = inputs("C4", begin=3_000_000, end=3_000_000 + n)
    G = Gpu("C4")
    rc.rc_overlap_read(reset=True)
    ov = G.run(c)
    cnt = rc.rc_overlap_read(reset=True)
    print(f"\n  CH4 overlap counters: {cnt}")
    assert cnt["pairs_ran"] + cnt["pairs_gave_up"] > 0
    G.mlp = rc.MLPBundle(G.mech, bundle("ch4_20sp", CONFIGS["C4"].hidden), 0, flags=rc.RC_MLP_SERIAL)
    se = G.run(c)
    for k in ("T", "cp", "rho", "mu", "lambda", "qdot", "D", "wdot", "o", "red", "diag"):
        assert np.array_equal(ov[k], se[k]), k


@pytest.mark.gpu
def test_layer3_side_launches_run_concurrently_with_fused_kernel():
    """The event timeline (rc_profile_timeline, one time axis for both streams) shows the layer-3 side
    launches running while fused-kernel launches run: their intervals intersect."""
    import paper_2312_13513_b200 as rc
    n = 3 * 262144
    c = inputs("C2", begin=0, end=n)
    G = Gpu("C2")
    G.run(c)  # warm the host-side caches
    rc.rc_overlap_read(reset=True)
    rc.rc_profile_enable(True)
    rc.rc_profile_read(reset=True)
    try:
        G.run(c)
        tl = rc.rc_profile_timeline()
        rc.rc_profile_read(reset=True)
    finally:
        rc.rc_profile_enable(False)
    cnt = rc.rc_overlap_read(reset=True)
    l12 = [(a, b) for s, a, b in tl if s == "L12"]
    fill = [(a, b) for s, a, b in tl if s == "L3_fill"]
    assert len(l12) == 3 and len(fill) == 2, (len(l12), len(fill))
    conc = sum(max(0.0, min(b1, b2) - max(a1, a2)) for a1, b1 in fill for a2, b2 in l12)
    print(f"\n  side launches {sum(b - a for a, b in fill):.3f} ms, {conc:.3f} ms of it during the fused kernel; {cnt}")
    if cnt["pairs_ran"] > 0:
        assert conc > 0.5 * min(b - a for a, b in l12)
