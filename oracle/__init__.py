"""ctypes binding of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, nothing else.  It shares no
code with paper_2312_13513_b200/ (the CUDA path), and the CUDA path never
imports it.
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")
CFLAGS = ["-O3", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree with gcc (plain C11, no fused multiply-add)."""
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", SO, "-lm"])
    return SO


class _Mech(C.Structure):
    _fields_ = [("ns", C.c_int32), ("ne", C.c_int32), ("W_elem", C.c_void_p), ("atoms", C.c_void_p),
                ("nasa_lo", C.c_void_p), ("nasa_hi", C.c_void_p), ("T_lo", C.c_void_p), ("T_mid", C.c_void_p),
                ("T_hi", C.c_void_p), ("visc", C.c_void_p), ("cond", C.c_void_p), ("diff", C.c_void_p),
                ("inert", C.c_void_p)]


class _Mlp(C.Structure):
    _fields_ = [("n_nets", C.c_int32), ("d_in", C.c_int32), ("hidden", C.c_int32 * 3),
                ("species_of_net", C.c_void_p), ("params", C.c_void_p), ("x_mean", C.c_void_p),
                ("x_std", C.c_void_p), ("y_mean", C.c_void_p), ("y_std", C.c_void_p),
                ("lambda_bc", C.c_double), ("dt", C.c_double), ("shared", C.c_int32)]


class _Cells(C.Structure):
    _fields_ = [("n", C.c_int64), ("ld", C.c_int64), ("mode", C.c_int32), ("h", C.c_void_p), ("T", C.c_void_p),
                ("p", C.c_void_p), ("Y", C.c_void_p), ("cp", C.c_void_p), ("rho", C.c_void_p), ("mu", C.c_void_p),
                ("lam", C.c_void_p), ("D", C.c_void_p), ("o", C.c_void_p), ("wdot", C.c_void_p),
                ("qdot", C.c_void_p), ("red", C.c_double * 2), ("diag", C.c_int64 * 5), ("tau_mix", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i, vp = C.c_double, C.c_int, C.c_void_p
        for name, res, args in [
            ("orc_species_cp", d, [vp, i, d]), ("orc_species_h", d, [vp, i, d]), ("orc_mix_W", d, [vp, vp]),
            ("orc_mix_h", d, [vp, vp, d]), ("orc_mix_cp", d, [vp, vp, d]),
            ("orc_T_from_h", d, [vp, vp, d, d, vp, vp]),
            ("orc_transport_cell", None, [vp, d, d, vp, vp, vp, vp]),
            ("orc_species_mu", d, [vp, i, d]), ("orc_species_lambda", d, [vp, i, d]),
            ("orc_binary_D", d, [vp, i, i, d, d]), ("orc_gelu", d, [d]),
            ("orc_mlp_forward", d, [vp, i, vp]), ("orc_projection", i, [vp, vp]),
            ("orc_prologue_cell", None, [vp, vp, d, d, vp, vp, vp]), ("orc_step", i, [vp, vp, vp, i]),
            ("orc_pasr_kappa", d, [vp, d, vp, vp, d]),
            ("orc_laplacian_gamma", None, [i, C.c_int64, vp, vp, vp, vp, vp]),
            ("orc_laplacian", None, [vp, i, vp, vp, vp, vp, vp]), ("orc_ldu_matvec", None, [vp, vp, vp, vp, vp]),
            ("orc_species_g", d, [vp, i, d]), ("orc_rate_constant", d, [vp, i, d, d]),
            ("orc_kinetics_cell", None, [vp, vp, d, d, vp, vp, vp, vp]), ("orc_kinetics", i, [vp, vp, vp, vp, i]),
        ]:
            f = getattr(_lib, name)
            f.restype, f.argtypes = res, args
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class Mech:
    """Oracle view of a workload.load_mech() dict (keeps the numpy arrays alive)."""

    def __init__(self, m: dict):
        self.keep = {k: np.ascontiguousarray(m[k], dtype=dt) for k, dt in [
            ("W_elem", np.float64), ("atoms", np.int32), ("nasa_lo", np.float64), ("nasa_hi", np.float64),
            ("T_lo", np.float64), ("T_mid", np.float64), ("T_hi", np.float64), ("visc", np.float64),
            ("cond", np.float64), ("diff", np.float64), ("inert", np.uint8)]}
        self.ns, self.ne = int(m["ns"]), int(m["ne"])
        self.s = _Mech(self.ns, self.ne, *[_p(self.keep[k]) for k in [
            "W_elem", "atoms", "nasa_lo", "nasa_hi", "T_lo", "T_mid", "T_hi", "visc", "cond", "diff", "inert"]])
        self.ref = C.byref(self.s)

    # per-species / per-cell primitives (pins)
    def cp_k(self, k, T): return lib().orc_species_cp(self.ref, k, T)
    def h_k(self, k, T): return lib().orc_species_h(self.ref, k, T)
    def mu_k(self, k, T): return lib().orc_species_mu(self.ref, k, T)
    def lambda_k(self, k, T): return lib().orc_species_lambda(self.ref, k, T)
    def D_jk(self, j, k, T, p): return lib().orc_binary_D(self.ref, j, k, T, p)

    def W(self, Y):
        Y = np.ascontiguousarray(Y, dtype=np.float64); return lib().orc_mix_W(self.ref, _p(Y))

    def h(self, Y, T):
        Y = np.ascontiguousarray(Y, dtype=np.float64); return lib().orc_mix_h(self.ref, _p(Y), T)

    def cp(self, Y, T):
        Y = np.ascontiguousarray(Y, dtype=np.float64); return lib().orc_mix_cp(self.ref, _p(Y), T)

    def T_from_h(self, Y, h, T_guess):
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        fl, it = C.c_int(0), C.c_int(0)
        T = lib().orc_T_from_h(self.ref, _p(Y), h, T_guess, C.addressof(fl), C.addressof(it))
        return T, fl.value, it.value

    def transport(self, T, p, Y):
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        mu, lam, D = C.c_double(), C.c_double(), np.empty(self.ns)
        lib().orc_transport_cell(self.ref, T, p, _p(Y), C.addressof(mu), C.addressof(lam), _p(D))
        return mu.value, lam.value, D

    def pasr_kappa(self, rho, Y, wdot, tau_mix):
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        w = np.ascontiguousarray(wdot, dtype=np.float64)
        return lib().orc_pasr_kappa(self.ref, rho, _p(Y), _p(w), tau_mix)

    def g_k(self, k, T): return lib().orc_species_g(self.ref, k, T)

    def projection(self):
        P = np.empty((self.ns, self.ns))
        if lib().orc_projection(self.ref, _p(P)) != 0:
            raise RuntimeError("singular E E^T")
        return P


def gelu(x: float) -> float:
    return lib().orc_gelu(x)


class Mlp:
    """Oracle view of a workload.make_bundle() dict."""

    def __init__(self, b: dict):
        self.keep = {k: np.ascontiguousarray(b[k], dtype=np.float64) for k in
                     ["params", "x_mean", "x_std", "y_mean", "y_std"]}
        self.keep["species_of_net"] = np.ascontiguousarray(b["species_of_net"], dtype=np.int32)
        self.n_nets, self.d_in = int(b["n_nets"]), int(b["d_in"])
        self.s = _Mlp(self.n_nets, self.d_in, (C.c_int32 * 3)(*b["hidden"]),
                      _p(self.keep["species_of_net"]), _p(self.keep["params"]), _p(self.keep["x_mean"]),
                      _p(self.keep["x_std"]), _p(self.keep["y_mean"]), _p(self.keep["y_std"]),
                      float(b["lambda_bc"]), float(b["dt"]), int(bool(b.get("shared", False))))
        self.ref = C.byref(self.s)

    def forward(self, net: int, z):
        z = np.ascontiguousarray(z, dtype=np.float64)
        return lib().orc_mlp_forward(self.ref, net, _p(z))

    def prologue(self, mech: Mech, T, p, Y):
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        z, b = np.empty(self.d_in), np.empty(mech.ns)
        lib().orc_prologue_cell(mech.ref, self.ref, T, p, _p(Y), _p(z), _p(b))
        return z, b


def step(mech: Mech, mlp: "Mlp | None", T, p, Y, h=None, mode: str = "h", transport: bool = True,
         chem: bool = True, nthreads: int = 0, tau_mix=None) -> dict:
    """Run oracle steps 1-10 + a6 on host arrays. T is the guess (h-mode) or value (T-mode).

    Returns dict with T, h, cp, rho, mu, lambda, D[ns][n], o[n_nets][n], wdot[ns][n], qdot, red, diag.
    """
    n = int(np.asarray(T).shape[0])
    ns = mech.ns
    out = {"T": np.array(T, dtype=np.float64, copy=True),
           "h": np.array(h, dtype=np.float64, copy=True) if h is not None else np.empty(n),
           "cp": np.empty(n), "rho": np.empty(n)}
    p = np.ascontiguousarray(p, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    assert Y.shape == (ns, n)
    if mode == "h" and h is None:
        raise ValueError("h-mode needs h")
    if transport:
        out.update(mu=np.empty(n), **{"lambda": np.empty(n)}, D=np.empty((ns, n)))
    do_chem = chem and mlp is not None
    if do_chem:
        out.update(o=np.empty((mlp.n_nets, n)), wdot=np.empty((ns, n)), qdot=np.empty(n))
    c = _Cells(n, n, 0 if mode == "h" else 1, _p(out["h"]), _p(out["T"]), _p(p), _p(Y), _p(out["cp"]),
               _p(out["rho"]), _p(out.get("mu")), _p(out.get("lambda")), _p(out.get("D")), _p(out.get("o")),
               _p(out.get("wdot")), _p(out.get("qdot")))
    tau = None if tau_mix is None else np.ascontiguousarray(tau_mix, dtype=np.float64)
    c.tau_mix = _p(tau)
    rc = lib().orc_step(mech.ref, mlp.ref if do_chem else None, C.byref(c), nthreads)
    if rc != 0:
        raise RuntimeError(f"orc_step failed: {rc}")
    out["red"] = np.array(c.red[:])
    out["diag"] = np.array(c.diag[:], dtype=np.int64)
    return out


class _Kin(C.Structure):
    _fields_ = [("nr", C.c_int32), ("nu_f", C.c_void_p), ("nu_r", C.c_void_p), ("type", C.c_void_p),
                ("reversible", C.c_void_p), ("A", C.c_void_p), ("b", C.c_void_p), ("Ea", C.c_void_p),
                ("eff", C.c_void_p), ("A0", C.c_void_p), ("b0", C.c_void_p), ("Ea0", C.c_void_p), ("troe", C.c_void_p)]


KIN_KEYS = [("nu_f", np.int32), ("nu_r", np.int32), ("type", np.int32), ("reversible", np.int32), ("A", np.float64),
            ("b", np.float64), ("Ea", np.float64), ("eff", np.float64), ("A0", np.float64), ("b0", np.float64),
            ("Ea0", np.float64), ("troe", np.float64)]


class Kin:
    """Oracle view of a workload.load_kinetics() dict (detailed kinetics, NEXT-3)."""

    def __init__(self, k: dict):
        self.keep = {key: np.ascontiguousarray(k[key], dtype=dt) for key, dt in KIN_KEYS}
        self.nr = int(k["nr"])
        self.s = _Kin(self.nr, *[_p(self.keep[key]) for key, _ in KIN_KEYS])
        self.ref = C.byref(self.s)

    def rate_constant(self, r, T, M):
        return lib().orc_rate_constant(self.ref, r, T, M)

    def cell(self, mech: Mech, T, p, Y):
        """(wdot[ns], q_net[nr], gross-rate scale[ns]) of one cell."""
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        w, q, sc = np.empty(mech.ns), np.empty(self.nr), np.empty(mech.ns)
        lib().orc_kinetics_cell(mech.ref, self.ref, T, p, _p(Y), _p(w), _p(q), _p(sc))
        return w, q, sc


def kinetics(mech: Mech, kin: Kin, T, p, Y, tau_mix=None, nthreads: int = 0) -> dict:
    """Detailed-kinetics sources of a field (T given): wdot[ns][n], qdot, wscale[ns][n], red, diag."""
    n = int(np.asarray(T).shape[0])
    ns = mech.ns
    T = np.ascontiguousarray(T, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    out = {"wdot": np.empty((ns, n)), "qdot": np.empty(n), "wscale": np.empty((ns, n))}
    c = _Cells(n, n, 1, None, _p(T), _p(p), _p(Y), None, None, None, None, None, None, _p(out["wdot"]),
               _p(out["qdot"]))
    tau = None if tau_mix is None else np.ascontiguousarray(tau_mix, dtype=np.float64)
    c.tau_mix = _p(tau)
    if lib().orc_kinetics(mech.ref, kin.ref, C.byref(c), _p(out["wscale"]), nthreads) != 0:
        raise RuntimeError("orc_kinetics failed")
    out["red"] = np.array(c.red[:])
    out["diag"] = np.array(c.diag[:], dtype=np.int64)
    return out


class _MeshS(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
                ("dz", C.c_double)]


def laplacian_gamma(ns, rho, D, lam, cp):
    """gamma [ns+1][n]: rho D_k for species, lambda/cp for energy (NEXT-1 coefficients)."""
    n = int(np.asarray(rho).shape[0])
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (rho, D, lam, cp)]
    g = np.empty((ns + 1, n))
    lib().orc_laplacian_gamma(ns, n, *[_p(a) for a in arrs], _p(g))
    return g


def laplacian(mesh, gamma, halo_lo=None, halo_hi=None):
    """Algorithm 1 on the periodic mesh / slab: returns (upper [nsys][3N], diag [nsys][N]).
    mesh = (nx, ny, nz, dx, dy, dz)."""
    ms = _MeshS(*mesh)
    g = np.ascontiguousarray(gamma, dtype=np.float64)
    nsys, N = g.shape
    up, dg = np.empty((nsys, 3 * N)), np.empty((nsys, N))
    lo = None if halo_lo is None else np.ascontiguousarray(halo_lo, dtype=np.float64)
    hi = None if halo_hi is None else np.ascontiguousarray(halo_hi, dtype=np.float64)
    lib().orc_laplacian(C.byref(ms), nsys, _p(g), _p(lo), _p(hi), _p(up), _p(dg))
    return up, dg


def ldu_matvec(mesh, upper, diag, x):
    ms = _MeshS(*mesh)
    y = np.empty_like(np.asarray(x, dtype=np.float64))
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (upper, diag, x)]
    lib().orc_ldu_matvec(C.byref(ms), *[_p(a) for a in arrs], _p(y))
    return y
