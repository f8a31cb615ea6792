"""Shared test plumbing: seeded inputs -> oracle (CPU, fp64) and -> the CUDA
path (through the C ABI), on the SAME inputs.  The h fed to both sides is the
oracle's h(T_true) (T-mode), never a CUDA-path value."""
import numpy as np

import oracle
from workload import CONFIGS, load_mech, make_bundle, make_cells, make_cells_at

# Parity gates (BASELINE.json north_star; R17/R18 for the derived ones)
FP64_TOL = 1e-10          # thermo / transport / epilogue fp64 outputs, elementwise relative
BF16_TOL = 2e-2           # bf16 MLP output o, relative Frobenius (north_star)
TF32_TOL = 1e-3           # TF32 MLP output o (north_star: "relative 1e-3 of the output norm")
# wdot / qdot: an MLP that does nothing but round its operands (bf16 or tf32 RNE, fp32 accumulate,
# exact GELU; tests/_emulate.py) already reaches wdot 1.9-2.0e-2 (bf16) and 1.1-1.3e-3 (tf32) on
# the C2 parity samples: the O2 net's |o| is ~5x below the norm of o with random init weights and
# dominates wdot.  The derived gates are 1.5x that rounding floor (tests/test_emulation_gates.py
# re-derives it on CPU); the kernels are also held to EMU_FACTOR x the floor on every sample.
BF16_DERIVED_TOL = 3e-2
TF32_DERIVED_TOL = 2e-3
EMU_FACTOR = 1.5

_cache = {}


def mech(name):
    if name not in _cache:
        _cache[name] = load_mech(name)
    return _cache[name]


def bundle(mech_name, hidden):
    key = ("b", mech_name, tuple(hidden))
    if key not in _cache:
        _cache[key] = make_bundle(mech_name, hidden=hidden)
    return _cache[key]


def inputs(cfg, idx=None, begin=0, end=None):
    """cells (T_true, T_guess, p, Y) + the oracle's h(T_true, Y)."""
    c = make_cells_at(cfg, idx) if idx is not None else make_cells(cfg, begin, end)
    om = oracle.Mech(mech(CONFIGS[cfg].mech))
    t = oracle.step(om, None, c["T_true"], c["p"], c["Y"], mode="T", transport=False, chem=False)
    c["h"] = t["h"]
    return c


def run_oracle(cfg, c, chem=True, transport=True, nthreads=0, b=None, tau_mix=None):
    m = mech(CONFIGS[cfg].mech)
    om = oracle.Mech(m)
    ob = oracle.Mlp(b if b is not None else bundle(CONFIGS[cfg].mech, CONFIGS[cfg].hidden)) if chem else None
    return oracle.step(om, ob, c["T_guess"], c["p"], c["Y"], h=c["h"], transport=transport, chem=chem,
                       nthreads=nthreads, tau_mix=tau_mix)


class Gpu:
    """Handles for one config on the current CUDA device."""

    def __init__(self, cfg, precision=0, b=None):
        import paper_2312_13513_b200 as rc
        self.rc = rc
        self.cfg = cfg
        m = mech(CONFIGS[cfg].mech)
        self.mech = rc.Mechanism(m)
        b = b if b is not None else bundle(CONFIGS[cfg].mech, CONFIGS[cfg].hidden)
        self.mlp = rc.MLPBundle(self.mech, b, precision)
        self.ns = m["ns"]
        self.n_nets = b["n_nets"]
        self.dt = b["dt"]

    def run(self, c, ld=None, chem=True, transport=True, ws=None, tau_mix=None):
        import torch
        rc = self.rc
        n = c["p"].shape[0]
        st = rc.CellState(n, self.ns, self.n_nets if chem else 0, ld=ld)
        st.load(c["T_guess"], c["p"], c["Y"], h=c["h"])
        st.set_tau_mix(tau_mix)
        if ws is None:
            ws = rc.aligned_workspace(self.mlp, max(n, 1))
        rc.rc_step(self.mech, self.mlp if chem else None, st.cells(rc.RC_MODE_H, dt=self.dt, chem=chem,
                                                                    transport=transport), ws)
        torch.cuda.synchronize()
        out = st.host()
        out["lambda"] = out.pop("lam", None)
        out["launches"] = rc.rc_last_launch_count()
        return out


def rel_fro(g, o):
    g, o = np.asarray(g, dtype=np.float64), np.asarray(o, dtype=np.float64)
    return float(np.linalg.norm(g - o) / max(np.linalg.norm(o), 1e-300))


def max_rel(g, o):
    g, o = np.asarray(g, dtype=np.float64), np.asarray(o, dtype=np.float64)
    return float(np.max(np.abs(g - o) / np.maximum(np.abs(o), 1e-300)))
