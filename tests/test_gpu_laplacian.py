"""Laplacian assembly consumer (Algorithm 1; ldu -> CSR,
PAPER.md:173) on the GPU vs the oracle, through the C ABI (rc_laplacian, rc_ldu_to_csr,
rc_pack_planes).  The property inputs (rho, D_k, lambda, cp) of both sides are the oracle's own
thermo/transport outputs on generator cells laid out on the mesh, so the comparison isolates the
assembly.  Gates: face coefficients bitwise (same arithmetic: (gamma_P + gamma_N)/2 |S|/|d|), diagonals
1e-14 relative (summation order); slab == periodic bitwise (gather mode); CSR == scipy's conversion."""
import numpy as np
import pytest

import oracle
from _harness import mech
from workload import make_cells

pytestmark = pytest.mark.gpu
MESH = (12, 10, 9, 4e-5, 4e-5, 4e-5)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_13513_b200 import build
    build.build()


@pytest.fixture(scope="module")
def props():
    """oracle thermo + transport of C3 generator cells (3D jet states) on MESH"""
    m = mech("h2_9sp")
    om = oracle.Mech(m)
    n = int(np.prod(MESH[:3]))
    c = make_cells("C3", 5_000_000, 5_000_000 + n)
    r = oracle.step(om, None, c["T_true"], c["p"], c["Y"], mode="T", chem=False)
    return {"rho": r["rho"], "lam": r["lambda"], "cp": r["cp"], "D": r["D"], "T": c["T_true"], "p": c["p"],
            "Y": c["Y"]}


def _device(props, sl=None, ld=None):
    import torch

    import paper_2312_13513_b200 as rc
    n = props["rho"].shape[0] if sl is None else sl.stop - sl.start
    sl = sl or slice(0, n)
    st = rc.CellState(n, 9, 0, ld=ld)
    st.load(props["T"][sl], props["p"][sl], props["Y"][:, sl])
    for k, v in (("rho", props["rho"]), ("lam", props["lam"]), ("cp", props["cp"])):
        getattr(st, k)[:n].copy_(torch.from_numpy(np.ascontiguousarray(v[sl])))
    st.D[:, :n].copy_(torch.from_numpy(np.ascontiguousarray(props["D"][:, sl])))
    return st


def _assemble(M, mesh, st, mode, halo=(None, None)):
    import torch

    import paper_2312_13513_b200 as rc
    n = int(np.prod(mesh[:3]))
    up = torch.empty(10, 3 * n, dtype=torch.float64, device="cuda")
    dg = torch.empty(10, n, dtype=torch.float64, device="cuda")
    rc.rc_laplacian(M, mesh, st.cells(rc.RC_MODE_T), up, dg, halo[0], halo[1], mode)
    torch.cuda.synchronize()
    return up, dg


def test_periodic_gather_and_atomic_match_oracle(props):
    import paper_2312_13513_b200 as rc
    M = rc.Mechanism(mech("h2_9sp"))
    g = oracle.laplacian_gamma(9, props["rho"], props["D"], props["lam"], props["cp"])
    upO, dgO = oracle.laplacian(MESH, g)
    st = _device(props, ld=1090)     # ld > n: the stride is honoured
    for mode in (rc.RC_LAP_GATHER, rc.RC_LAP_ATOMIC):
        up, dg = _assemble(M, MESH, st, mode)
        up, dg = up.cpu().numpy(), dg.cpu().numpy()
        assert np.array_equal(up, upO), (mode, np.max(np.abs(up - upO) / upO))
        np.testing.assert_allclose(dg, dgO, rtol=1e-14)


def test_slabs_with_packed_halos_equal_the_periodic_block_bitwise(props):
    """Two z-slabs assembled separately, each with the other slab's boundary planes packed by
    rc_pack_planes as halos (what exchange_halos moves between GPUs): identical to the whole block."""
    import torch

    import paper_2312_13513_b200 as rc
    M = rc.Mechanism(mech("h2_9sp"))
    nx, ny, nz, dx, dy, dz = MESH
    plane = nx * ny
    whole = _device(props)
    upW, dgW = _assemble(M, MESH, whole, rc.RC_LAP_GATHER)
    cuts = [(0, 4), (4, 9)]
    sts = [_device(props, slice(z0 * plane, z1 * plane)) for z0, z1 in cuts]
    packs = []
    for (z0, z1), st in zip(cuts, sts):
        b = torch.empty(12, plane, dtype=torch.float64, device="cuda")
        t = torch.empty(12, plane, dtype=torch.float64, device="cuda")
        rc.rc_pack_planes(M, (nx, ny, z1 - z0, dx, dy, dz), st.cells(rc.RC_MODE_T), b, t)
        packs.append((b, t))
    N = nx * ny * nz
    for s, ((z0, z1), st) in enumerate(zip(cuts, sts)):
        other = packs[1 - s]
        up, dg = _assemble(M, (nx, ny, z1 - z0, dx, dy, dz), st, rc.RC_LAP_GATHER, halo=(other[1], other[0]))
        n = (z1 - z0) * plane
        sl = slice(z0 * plane, z1 * plane)
        for d in range(3):
            assert torch.equal(up[:, d * n:(d + 1) * n], upW[:, d * N:(d + 1) * N][:, sl])
        assert torch.equal(dg, dgW[:, sl])


def test_ldu_to_csr_matches_scipy(props):
    import scipy.sparse as sp
    import torch

    import paper_2312_13513_b200 as rc
    M = rc.Mechanism(mech("h2_9sp"))
    nx, ny, nz = MESH[:3]
    N = nx * ny * nz
    up, dg = _assemble(M, MESH, _device(props), rc.RC_LAP_GATHER)
    rp = torch.empty(N + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(7 * N, dtype=torch.int32, device="cuda")
    val = torch.empty(10, 7 * N, dtype=torch.float64, device="cuda")
    rc.rc_ldu_to_csr(MESH, 10, up, dg, rp, col, val)
    torch.cuda.synchronize()
    upn, dgn = up.cpu().numpy(), dg.cpu().numpy()
    # the ldu triplets of the face list (owner c, +d neighbour) -> scipy CSR (sorted, canonical)
    c = np.arange(N)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    nb = [((i + 1) % nx) + nx * (j + ny * k), i + nx * (((j + 1) % ny) + ny * k), i + nx * (j + ny * ((k + 1) % nz))]
    for s in (0, 4, 9):
        rows = np.concatenate([c] + [c] * 3 + nb)
        cols = np.concatenate([c] + nb + [c] * 3)
        vals = np.concatenate([dgn[s]] + [upn[s, d * N:(d + 1) * N] for d in range(3)] * 2)
        A = sp.csr_matrix((vals, (rows, cols)), shape=(N, N))
        A.sort_indices()
        assert np.array_equal(rp.cpu().numpy(), A.indptr) and np.array_equal(col.cpu().numpy(), A.indices)
        assert np.array_equal(val[s].cpu().numpy(), A.data)
        # and the CSR operator equals the oracle's ldu product
        x = np.random.default_rng(s).normal(size=N)
        np.testing.assert_allclose(A @ x, oracle.ldu_matvec(MESH, upn[s], dgn[s], x), rtol=1e-12, atol=1e-12 * np.abs(dgn[s]).max())


def test_ch4_21_systems():
    """CH4 set: 20 species + energy = 21 systems through the runtime-ns path of the assembly; faces
    bitwise, diagonals 1e-14, CSR values equal to the ldu entries."""
    import torch

    import paper_2312_13513_b200 as rc
    m = mech("ch4_20sp")
    om = oracle.Mech(m)
    mesh = (10, 9, 8, 5e-5, 5e-5, 5e-5)
    n = 720
    c = make_cells("C4", 7_000_000, 7_000_000 + n)
    r = oracle.step(om, None, c["T_true"], c["p"], c["Y"], mode="T", chem=False)
    g = oracle.laplacian_gamma(20, r["rho"], r["D"], r["lambda"], r["cp"])
    upO, dgO = oracle.laplacian(mesh, g)
    M = rc.Mechanism(m)
    st = rc.CellState(n, 20, 0)
    st.load(c["T_true"], c["p"], c["Y"])
    for k, v in (("rho", r["rho"]), ("lam", r["lambda"]), ("cp", r["cp"])):
        getattr(st, k)[:n].copy_(torch.from_numpy(np.ascontiguousarray(v)))
    st.D[:, :n].copy_(torch.from_numpy(np.ascontiguousarray(r["D"])))
    up = torch.empty(21, 3 * n, dtype=torch.float64, device="cuda")
    dg = torch.empty(21, n, dtype=torch.float64, device="cuda")
    rc.rc_laplacian(M, mesh, st.cells(rc.RC_MODE_T), up, dg)
    torch.cuda.synchronize()
    assert np.array_equal(up.cpu().numpy(), upO)
    np.testing.assert_allclose(dg.cpu().numpy(), dgO, rtol=1e-14)
