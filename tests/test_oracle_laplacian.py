"""Pins of the oracle's Laplacian assembly (Algorithm 1):
closed forms on a constant coefficient, the discrete-Fourier eigenvalues of the 7-point Laplacian,
row sums, symmetry, exact linear interpolation, and slab decomposition with halo planes."""
import numpy as np
import pytest

import oracle

MESH = (8, 6, 5, 1e-3, 2e-3, 1.5e-3)     # nx, ny, nz, dx, dy, dz


def _faces(mesh):
    nx, ny, nz, dx, dy, dz = mesh
    return nx * ny * nz, (dy * dz / dx, dx * dz / dy, dx * dy / dz)


def test_constant_coefficient_closed_form():
    N, S = _faces(MESH)
    g0 = 2.5e-5
    up, dg = oracle.laplacian(MESH, np.full((1, N), g0))
    for d in range(3):
        assert np.all(up[0, d * N:(d + 1) * N] == g0 * S[d])
    np.testing.assert_allclose(dg[0], -2.0 * g0 * sum(S), rtol=1e-15)


def test_fourier_eigenvalues():
    """For constant gamma, phi = cos(2 pi (m_x i / nx + m_y j / ny + m_z k / nz)) is an eigenvector of the
    periodic 7-point Laplacian with eigenvalue sum_d gamma S_d/|d_d| (2 cos(2 pi m_d / n_d) - 2)."""
    nx, ny, nz = MESH[:3]
    N, S = _faces(MESH)
    g0 = 0.7
    up, dg = oracle.laplacian(MESH, np.full((1, N), g0))
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    for m in ((1, 0, 0), (2, 1, 0), (3, 2, 4), (0, 0, 2)):
        phi = np.cos(2 * np.pi * (m[0] * i / nx + m[1] * j / ny + m[2] * k / nz)).ravel()
        lam = sum(g0 * S[d] * (2 * np.cos(2 * np.pi * m[d] / (nx, ny, nz)[d]) - 2) for d in range(3))
        y = oracle.ldu_matvec(MESH, up[0], dg[0], phi)
        np.testing.assert_allclose(y, lam * phi, atol=1e-13 * abs(lam) + 1e-15)


def test_row_sums_and_symmetry():
    N, _ = _faces(MESH)
    rng = np.random.default_rng(3)
    g = rng.uniform(1e-6, 1e-4, size=(1, N))
    up, dg = oracle.laplacian(MESH, g)
    y = oracle.ldu_matvec(MESH, up[0], dg[0], np.ones(N))            # Laplacian of a constant
    assert np.max(np.abs(y)) <= 1e-15 * np.max(np.abs(dg[0]))
    x1, x2 = rng.normal(size=N), rng.normal(size=N)
    a = x2 @ oracle.ldu_matvec(MESH, up[0], dg[0], x1)
    b = x1 @ oracle.ldu_matvec(MESH, up[0], dg[0], x2)
    assert a == pytest.approx(b, rel=1e-13)
    assert np.all(up > 0) and np.all(dg < 0)


def test_linear_interpolation_is_exact_at_faces():
    """gamma = a + b x: away from the periodic wrap, gamma_f is the value at the face centre."""
    nx, ny, nz, dx = MESH[:4]
    N, S = _faces(MESH)
    i = np.arange(N) % nx
    g = 3.0 + 0.25 * (i + 0.5) * dx
    up, _ = oracle.laplacian(MESH, g[None])
    inner = i < nx - 1
    np.testing.assert_allclose(up[0, :N][inner], (3.0 + 0.25 * (i[inner] + 1.0) * dx) * S[0], rtol=1e-15)


def test_slab_decomposition_with_halo_planes_equals_periodic():
    """The z-slab [z0, z1) assembled with the gamma planes z0-1 and z1 as halos (what the multi-GPU path
    exchanges) reproduces the global periodic assembly of those cells exactly (same arithmetic)."""
    nx, ny, nz, dx, dy, dz = MESH
    N = nx * ny * nz
    plane = nx * ny
    rng = np.random.default_rng(5)
    g = rng.uniform(1e-6, 1e-4, size=(3, N))
    upG, dgG = oracle.laplacian(MESH, g)
    for z0, z1 in ((0, 2), (2, 5), (1, 4)):
        sl = slice(z0 * plane, z1 * plane)
        lo = g[:, ((z0 - 1) % nz) * plane:((z0 - 1) % nz + 1) * plane]
        hi = g[:, (z1 % nz) * plane:(z1 % nz + 1) * plane]
        up, dg = oracle.laplacian((nx, ny, z1 - z0, dx, dy, dz), g[:, sl], lo, hi)
        n = (z1 - z0) * plane
        for d in range(3):
            assert np.array_equal(up[:, d * n:(d + 1) * n], upG[:, d * N:(d + 1) * N][:, sl])
        np.testing.assert_allclose(dg, dgG[:, sl], rtol=1e-15)


def test_gamma_definition():
    rng = np.random.default_rng(1)
    n, ns = 10, 3
    rho, lam, cp = rng.uniform(0.1, 1, n), rng.uniform(0.01, 0.1, n), rng.uniform(1e3, 2e3, n)
    D = rng.uniform(1e-5, 1e-4, (ns, n))
    g = oracle.laplacian_gamma(ns, rho, D, lam, cp)
    assert np.array_equal(g[:ns], rho[None] * D) and np.array_equal(g[ns], lam / cp)
