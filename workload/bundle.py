"""Random-init MLP bundle of the paper's shape (one net per
non-inert species, hidden 1600/800/400, GELU).  No trained weights exist
(SURVEY.md §0), so weights are PyTorch-default-style uniform draws
U(-1/sqrt(fan_in), 1/sqrt(fan_in)) for W and b, in fp64, seeded per net with
SEED + net (DESIGN.md input recipe).

Normalisation statistics (x_mean, x_std over the d_in = ns + 2 inputs
[T, p, BCT_1..ns]) are read from data/bundle_stats/<mech>.json, which
tools/make_bundle_stats.py wrote once from 65,536 generator cells using only
oracle/ (the Box-Cox transform belongs to the method, so it is not computed
here).  y_mean = 0, y_std = 0.02 (|Delta| ~ 1e-2 Box-Cox units); lambda_BC =
0.1; dt = 1e-6 s (readings R3, R4, R7).
"""
import json
import os

import numpy as np
import torch

from .mech import load_mech

SEED = 231213513
STATS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "bundle_stats")


def param_count(d_in: int, hidden, n_out: int = 1) -> int:
    h1, h2, h3 = hidden
    return h1 * d_in + h1 + h2 * h1 + h2 + h3 * h2 + h3 + n_out * h3 + n_out


def make_bundle(mech_name: str, hidden=(1600, 800, 400), lambda_bc: float = 0.1, dt: float = 1e-6,
                y_std: float = 0.02, stats: dict | None = None, shared: bool = False) -> dict:
    """shared=False: one net per non-inert species (reading R1), params [n_nets][P];
    shared=True: ONE net d_in -> hidden -> n_nets outputs (reading R20),
    params [1][P] with the output layer W4 [n_nets][h3], b4 [n_nets]."""
    m = load_mech(mech_name)
    ns = m["ns"]
    d_in = ns + 2
    nets = [k for k in range(ns) if not m["inert"][k]]
    n_out = len(nets) if shared else 1
    dims = [d_in, *hidden, n_out]
    params = np.empty((1 if shared else len(nets), param_count(d_in, hidden, n_out)), dtype=np.float64)
    for i in range(params.shape[0]):
        g = torch.Generator().manual_seed(SEED + i)
        parts = []
        for l in range(4):
            fan_in, fan_out = dims[l], dims[l + 1]
            bound = 1.0 / np.sqrt(fan_in)
            W = torch.empty(fan_out, fan_in, dtype=torch.float64).uniform_(-bound, bound, generator=g)
            b = torch.empty(fan_out, dtype=torch.float64).uniform_(-bound, bound, generator=g)
            parts += [W.reshape(-1), b]
        params[i] = torch.cat(parts).numpy()
    if stats is None:
        with open(os.path.join(STATS, mech_name + ".json")) as f:
            stats = json.load(f)
    return {
        "mech": mech_name,
        "n_nets": len(nets),
        "d_in": d_in,
        "hidden": tuple(hidden),
        "species_of_net": np.array(nets, dtype=np.int32),
        "params": params,                                   # [n_nets][param_count]
        "x_mean": np.array(stats["x_mean"], dtype=np.float64),
        "x_std": np.array(stats["x_std"], dtype=np.float64),
        "y_mean": np.zeros(len(nets)),
        "y_std": np.full(len(nets), y_std),
        "lambda_bc": lambda_bc,
        "dt": dt,
        "shared": bool(shared),
    }


def split_params(bundle: dict, net: int):
    """Views (W1, b1, W2, b2, W3, b3, W4, b4) of one net's flat fp64 parameters (of the shared
    net for shared bundles: W4 [n_nets][h3], b4 [n_nets]; pass net = 0)."""
    d, (h1, h2, h3) = bundle["d_in"], bundle["hidden"]
    n_out = bundle["n_nets"] if bundle.get("shared") else 1
    p = bundle["params"][net]
    out, o = [], 0
    for fi, fo in ((d, h1), (h1, h2), (h2, h3), (h3, n_out)):
        out.append(p[o:o + fi * fo].reshape(fo, fi)); o += fi * fo
        out.append(p[o:o + fo]); o += fo
    return out
