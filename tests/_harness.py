"""Shared test plumbing: seeded inputs -> oracle (CPU, fp64) and -> the CUDA
path (through the C ABI), on the SAME inputs.  The h fed to both sides is the
oracle's h(T_true) (T-mode), never a CUDA-path value."""
import numpy as np

import oracle
from workload import CONFIGS, load_mech, make_bundle, make_cells, make_cells_at

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


def run_oracle(cfg, c, chem=True, transport=True, nthreads=0):
    m = mech(CONFIGS[cfg].mech)
    om = oracle.Mech(m)
    ob = oracle.Mlp(bundle(CONFIGS[cfg].mech, CONFIGS[cfg].hidden)) if chem else None
    return oracle.step(om, ob, c["T_guess"], c["p"], c["Y"], h=c["h"], transport=transport, chem=chem,
                       nthreads=nthreads)


class Gpu:
    """Handles for one config on the current CUDA device."""

    def __init__(self, cfg, precision=0):
        import paper_2312_13513_b200 as rc
        self.rc = rc
        self.cfg = cfg
        m = mech(CONFIGS[cfg].mech)
        self.mech = rc.Mechanism(m)
        b = bundle(CONFIGS[cfg].mech, CONFIGS[cfg].hidden)
        self.mlp = rc.MLPBundle(self.mech, b, precision)
        self.ns = m["ns"]
        self.n_nets = b["n_nets"]
        self.dt = b["dt"]

    def run(self, c, ld=None, chem=True, transport=True, ws=None):
        import torch
        rc = self.rc
        n = c["p"].shape[0]
        st = rc.CellState(n, self.ns, self.n_nets if chem else 0, ld=ld)
        st.load(c["T_guess"], c["p"], c["Y"], h=c["h"])
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
