"""Synthetic cell states (T_true, T_guess, p, Y) for the five BASELINE.json configs.

Recipe (DESIGN.md §"Input recipe"):
  C1  H2/air 1D premixed flame profile, 1,000 cells (SPEC.md-scale oracle case)
  C2  H2/air planar jet diffusion flame on a 1024^2 grid (quasi-DNS jet)
  C3  H2/air 3D smooth-field diffusion-flame states on 256^3 (the TGV mesh size)
  C4  CH4/air stratified premixed (Cambridge SWB5-like) on 256^3
  C5  H2/air, 500x500x400 = 1e8 cells, C3 recipe
All configs: p = 101325 (1 + 0.005 F_p); T_guess = T (1 + 0.02 (2u - 1)) emulating
the previous step's T; 0.1 % of cells get Y_k = -1e-12 on one minor species.
Every value is a function of (SEED, field id, global cell index) only.
The inert species (N2) is the residual 1 - sum(others), as "inert gases" are
excluded from prediction.
"""
from dataclasses import dataclass, field
import numpy as np

SEED = 231213513
U64 = np.uint64


def _splitmix64(x):
    x = (x + U64(0x9E3779B97F4A7C15)) & U64(0xFFFFFFFFFFFFFFFF)
    z = x
    z = (z ^ (z >> U64(30))) * U64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> U64(27))) * U64(0x94D049BB133111EB)
    return z ^ (z >> U64(31))


def uniform(field_id: int, idx: np.ndarray) -> np.ndarray:
    """u in [0,1) from (SEED, field_id, idx) by a SplitMix64 hash."""
    with np.errstate(over="ignore"):
        key = _splitmix64(np.asarray(idx, dtype=U64) ^ _splitmix64(
            np.full(1, SEED * 1000003 + field_id, dtype=U64)))
    return (key >> U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


class SmoothField:
    """F(x) = sum_{m<32} A_m cos(2 pi k_m . x + phi_m), A_m ~ |k|^(-5/6), unit variance."""

    def __init__(self, field_id: int, dim: int, kmax: float = 6.0, modes: int = 32):
        rng = np.random.default_rng(SEED + 7919 * field_id)
        kmag = rng.uniform(1.0, kmax, modes)
        d = rng.normal(size=(modes, dim))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        self.k = 2.0 * np.pi * d * kmag[:, None]
        self.phi = rng.uniform(0.0, 2.0 * np.pi, modes)
        a = kmag ** (-5.0 / 6.0)
        self.A = a / np.sqrt(0.5 * np.sum(a * a))

    def __call__(self, X: np.ndarray) -> np.ndarray:  # X [n, dim]
        out = np.zeros(X.shape[0])
        for m in range(len(self.A)):
            out += self.A[m] * np.cos(X @ self.k[m] + self.phi[m])
        return out


def _bell(c, c0, w):
    return np.exp(-((c - c0) / w) ** 2)


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


@dataclass
class Config:
    name: str
    mech: str
    grid: tuple
    hidden: tuple
    recipe: str
    note: str = ""
    n_cells: int = field(init=False)

    def __post_init__(self):
        self.n_cells = int(np.prod(self.grid))


CONFIGS = {
    "C1": Config("C1", "h2_9sp", (1000,), (64, 32, 16), "premixed1d", "H2/air 1D premixed profile, small MLP"),
    "C2": Config("C2", "h2_9sp", (1024, 1024), (1600, 800, 400), "jet2d", "H2/air 2D jet flame, paper MLP"),
    "C3": Config("C3", "h2_9sp", (256, 256, 256), (1600, 800, 400), "jet3d", "H2/air 3D LES-shaped states"),
    "C4": Config("C4", "ch4_20sp", (256, 256, 256), (1600, 800, 400), "swb", "CH4/air stratified premixed"),
    "C5": Config("C5", "h2_9sp", (500, 500, 400), (1600, 800, 400), "jet3d", "H2/air 1e8 cells"),
}

H2_SP = ["H2", "O2", "H2O", "H", "O", "OH", "HO2", "H2O2", "N2"]
CH4_SP = ["H2", "H", "O", "O2", "OH", "H2O", "HO2", "CH2", "CH2(S)", "CH3", "CH4", "CO", "CO2",
          "HCO", "CH2O", "CH3O", "C2H4", "C2H5", "C2H6", "N2"]
# molar masses used only to shape the synthetic composition (stoichiometry of the recipe)
_W = {"H2": 2.016, "O2": 31.998, "H2O": 18.015, "CH4": 16.043, "CO2": 44.009, "CO": 28.010}


def coords(cfg: Config, idx: np.ndarray) -> np.ndarray:
    """Cell centres in [0,1)^d; linear index i = ix + nx*iy + nx*ny*iz."""
    g = cfg.grid
    out = np.empty((idx.shape[0], len(g)))
    rem = idx.astype(np.int64)
    for d, n in enumerate(g):
        out[:, d] = ((rem % n) + 0.5) / n
        rem = rem // n
    return out


def _h2_premixed(cfg, idx, X):
    n = idx.shape[0]
    x = X[:, 0] - 0.5
    c = 0.5 * (1.0 + np.tanh(x / 0.08))
    Y = np.zeros((9, n))
    Y[0] = 0.02852 * (1.0 - c)
    Y[1] = 0.2264 * (1.0 - c)
    Y[3] = 4e-4 * _bell(c, 0.75, 0.15)
    Y[4] = 1.5e-3 * _bell(c, 0.70, 0.15)
    Y[5] = 6e-3 * _bell(c, 0.80, 0.20)
    Y[6] = 2e-4 * _bell(c, 0.30, 0.12)
    Y[7] = 5e-5 * _bell(c, 0.35, 0.12)
    rad = Y[3] + Y[4] + Y[5] + Y[6] + Y[7]
    Y[2] = np.maximum(0.2549 * c - rad, 0.0)
    T = 300.0 + 2100.0 * c
    return T, Y


def _h2_jet(cfg, idx, X, two_d: bool):
    n = idx.shape[0]
    dim = X.shape[1]
    F1, F2 = SmoothField(1, dim)(X), SmoothField(2, dim)(X)
    if two_d:
        xs, y = X[:, 0], X[:, 1]
        b = 0.05 + 0.15 * xs
        yw = y + 0.03 * F1
        dl = 0.02 + 0.03 * xs
        Zc = np.minimum(1.0, 0.15 / b)
        arg = (b - np.abs(yw - 0.5)) / dl
        e = _erf(arg)
        Z = Zc * 0.5 * (1.0 + e)
        chi = _sigmoid(3.0 * F2 + 1.0)
    else:
        Z = np.clip(0.3 + 0.25 * F1, 0.0, 1.0)
        chi = _sigmoid(2.0 * F2 + 0.5)
    YF_H2, YO_O2 = 0.0671, 0.233
    s = 0.5 * _W["O2"] / _W["H2"]
    Zst = YO_O2 / (s * YF_H2 + YO_O2)
    H2m, O2m = YF_H2 * Z, YO_O2 * (1.0 - Z)
    lean = Z <= Zst
    H2b = np.where(lean, 0.0, H2m - O2m / s)
    O2b = np.where(lean, O2m - s * H2m, 0.0)
    H2Ob = np.where(lean, H2m * _W["H2O"] / _W["H2"], O2m * 2.0 * _W["H2O"] / _W["O2"])
    TBS = 300.0 + 1900.0 * np.where(lean, Z / Zst, (1.0 - Z) / (1.0 - Zst))
    T = 300.0 + chi * (TBS - 300.0)
    Y = np.zeros((9, n))
    Y[0] = H2m + chi * (H2b - H2m)
    Y[1] = O2m + chi * (O2b - O2m)
    Y[2] = chi * H2Ob
    g = _bell(Z, Zst, 0.1)
    Y[3] = 4e-4 * chi * g
    Y[4] = 1.5e-3 * chi * g
    Y[5] = 6e-3 * chi * g
    Y[6] = 2e-4 * 4.0 * chi * (1.0 - chi) * g
    Y[7] = 5e-5 * 4.0 * chi * (1.0 - chi) * g
    return T, np.maximum(Y, 0.0)


def _erf(x):
    # profile shaping only (jet edge), not the method's arithmetic
    from scipy.special import erf
    return erf(x)


def _ch4_swb(cfg, idx, X):
    n = idx.shape[0]
    F1, F2 = SmoothField(11, 3)(X), SmoothField(12, 3)(X)
    r = np.sqrt((X[:, 0] - 0.5) ** 2 + (X[:, 1] - 0.5) ** 2) + 0.03 * F1
    z = X[:, 2]
    inner = 0.5 * (1.0 - np.tanh((r - 0.15) / 0.03))
    outer = 0.5 * (1.0 - np.tanh((r - 0.30) / 0.03))
    phi = 0.5 * outer + 0.5 * inner                    # 1.0 inner / 0.5 outer / 0 coflow
    zf = 0.2 + 0.6 * r + 0.05 * F2
    c = _sigmoid((z - zf) / 0.04) * np.minimum(1.0, phi / 0.05)
    YF = phi / (phi + 17.12)
    O2u, N2u = 0.233 * (1.0 - YF), 0.767 * (1.0 - YF)
    CO2b = 0.9 * YF * _W["CO2"] / _W["CH4"]
    COb = 0.1 * YF * _W["CO"] / _W["CH4"]
    H2Ob = 0.98 * YF * 2.0 * _W["H2O"] / _W["CH4"]
    H2b = 0.02 * YF * 2.0 * _W["H2"] / _W["CH4"]
    O2b = np.maximum(O2u - (CO2b + COb + H2Ob + H2b - YF), 0.0)
    Tb = np.where(phi >= 0.5, 1480.0 + 750.0 * (phi - 0.5) / 0.5, 300.0 + 1180.0 * phi / 0.5)
    T = 300.0 + c * (Tb - 300.0)
    sp = {s: i for i, s in enumerate(CH4_SP)}
    Y = np.full((20, n), 1e-10)
    Y[sp["CH4"]] = YF * (1.0 - c) + 1e-10
    Y[sp["O2"]] = O2u + c * (O2b - O2u)
    Y[sp["CO2"]] = c * CO2b + 1e-10
    Y[sp["H2O"]] = c * H2Ob + 1e-10
    pw = phi / (phi + 1e-3) * np.minimum(phi, 1.0)
    bells = {"CO": (2e-2, 0.6, 0.2), "H2": (1e-3, 0.6, 0.2), "OH": (3e-3, 0.8, 0.2), "H": (3e-4, 0.7, 0.15),
             "O": (5e-4, 0.7, 0.15), "HO2": (1e-4, 0.2, 0.1), "CH2O": (1e-3, 0.3, 0.12),
             "CH3": (5e-4, 0.4, 0.12), "CH3O": (1e-5, 0.35, 0.1), "HCO": (2e-5, 0.5, 0.1),
             "CH2": (1e-6, 0.5, 0.1), "CH2(S)": (1e-7, 0.5, 0.1), "C2H4": (1e-4, 0.4, 0.12),
             "C2H5": (1e-6, 0.4, 0.1), "C2H6": (5e-5, 0.3, 0.12)}
    for s, (pk, c0, w) in bells.items():
        Y[sp[s]] += pk * pw * _bell(c, c0, w)
    Y[sp["CO"]] += c * COb
    Y[sp["H2"]] += c * H2b
    return T, Y


MINOR = {"h2_9sp": [3, 4, 5, 6, 7], "ch4_20sp": [1, 2, 4, 6, 7, 8, 9, 13, 14, 15, 16, 17, 18]}


def tau_mix_at(cfg, idx: np.ndarray) -> np.ndarray:
    """LES subgrid mixing time per cell [s] for the PaSR option (rc_cells.tau_mix, R19):
    log-uniform in [1e-6, 1e-3] s along a smooth field (tau_mix = C_mix sqrt(nu_sgs / eps) of an LES
    with eps ~ 1e1..1e6 m^2/s^3), so kappa spans ~0.2..1 against the random-init nets' tau_c."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    idx = np.asarray(idx, dtype=np.int64)
    X = coords(cfg, idx)
    F = SmoothField(11, X.shape[1])(X)                   # ~N(0,1)-like smooth field
    u = 0.5 * (1.0 + np.tanh(F))                        # (0, 1)
    return 10.0 ** (-6.0 + 3.0 * u)


def make_cells(cfg, begin: int = 0, end: int | None = None, chunk: int = 1 << 20) -> dict:
    """States of global cells [begin, end) of config `cfg` (name or Config).

    Returns dict(T_true[n], T_guess[n], p[n], Y[ns][n]) as fp64 numpy, component-major.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    end = cfg.n_cells if end is None else end
    return make_cells_at(cfg, np.arange(begin, end, dtype=np.int64), chunk)


def make_cells_at(cfg, idx: np.ndarray, chunk: int = 1 << 20) -> dict:
    """States of the global cells listed in idx (any order, any subset)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    idx_all = np.asarray(idx, dtype=np.int64)
    n = idx_all.shape[0]
    ns = 9 if cfg.mech == "h2_9sp" else 20
    out = {"T_true": np.empty(n), "T_guess": np.empty(n), "p": np.empty(n), "Y": np.empty((ns, n))}
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        idx = idx_all[c0:c1]
        X = coords(cfg, idx)
        if cfg.recipe == "premixed1d":
            T, Y = _h2_premixed(cfg, idx, X)
        elif cfg.recipe == "jet2d":
            T, Y = _h2_jet(cfg, idx, X, True)
        elif cfg.recipe == "jet3d":
            T, Y = _h2_jet(cfg, idx, X, False)
        elif cfg.recipe == "swb":
            T, Y = _ch4_swb(cfg, idx, X)
        else:
            raise ValueError(cfg.recipe)
        # 0.1 % of cells: one minor species set to -1e-12 (exercises the clipping)
        u = uniform(101, idx)
        pick = u < 1e-3
        if pick.any():
            minors = MINOR[cfg.mech]
            which = (uniform(102, idx[pick]) * len(minors)).astype(np.int64)
            Y[np.array(minors)[which], np.nonzero(pick)[0]] = -1e-12
        inert = ns - 1                                   # N2 last in both species sets
        Y[inert] = 0.0
        Y[inert] = 1.0 - Y.sum(axis=0)
        Fp = SmoothField(3, X.shape[1])(X)
        out["p"][c0:c1] = 101325.0 * (1.0 + 0.005 * Fp)
        out["T_true"][c0:c1] = T
        out["T_guess"][c0:c1] = T * (1.0 + 0.02 * (2.0 * uniform(103, idx) - 1.0))
        out["Y"][:, c0:c1] = Y
    return out
