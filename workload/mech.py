"""Mechanism table reader: data/mech/<name>.json -> dict of numpy arrays.
No arithmetic beyond type conversion (species molar masses are derived by
each consumer itself)."""
import json
import os

import numpy as np

DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "mech")


def load_mech(name: str) -> dict:
    with open(os.path.join(DATA, name + ".json")) as f:
        j = json.load(f)
    m = {
        "name": j["name"],
        "species": list(j["species"]),
        "elements": list(j["elements"]),
        "ns": len(j["species"]),
        "ne": len(j["elements"]),
        "W_elem": np.array(j["atomic_weights"], dtype=np.float64),
        "atoms": np.array(j["atoms"], dtype=np.int32),            # [ne][ns]
        "nasa_lo": np.array(j["nasa_lo"], dtype=np.float64),       # [ns][7]
        "nasa_hi": np.array(j["nasa_hi"], dtype=np.float64),
        "T_lo": np.array(j["T_lo"], dtype=np.float64),
        "T_mid": np.array(j["T_mid"], dtype=np.float64),
        "T_hi": np.array(j["T_hi"], dtype=np.float64),
        "visc": np.array(j["visc"], dtype=np.float64),             # [ns][5]
        "cond": np.array(j["cond"], dtype=np.float64),             # [ns][5]
        "diff": np.array(j["diff"], dtype=np.float64),             # [ns(ns+1)/2][5]
        "inert": np.array(j["inert"], dtype=np.uint8),
    }
    for k in ("atoms", "nasa_lo", "nasa_hi", "visc", "cond", "diff"):
        m[k] = np.ascontiguousarray(m[k])
    return m


def load_kinetics(name: str) -> dict:
    """Detailed-kinetics table data/mech/<name>_kin.json (SI) -> numpy arrays:
    nu_f, nu_r [nr][ns] int32; type [nr] (0 elementary, 1 three-body, 2 falloff); reversible [nr];
    A, b, Ea [nr] (k = A T^b exp(-Ea / (R_u T))); eff [nr][ns] third-body efficiencies; A0, b0, Ea0
    [nr] low-pressure limit (falloff); troe [nr][4] = (a, T***, T*, T**), a < 0: Lindemann."""
    with open(os.path.join(DATA, name + "_kin.json")) as f:
        j = json.load(f)
    R = j["reactions"]
    k = {"name": j["name"], "species": list(j["species"]), "nr": len(R)}
    for key, dt in (("nu_f", np.int32), ("nu_r", np.int32), ("type", np.int32), ("reversible", np.int32),
                    ("A", np.float64), ("b", np.float64), ("Ea", np.float64), ("eff", np.float64),
                    ("A0", np.float64), ("b0", np.float64), ("Ea0", np.float64), ("troe", np.float64)):
        k[key] = np.ascontiguousarray(np.array([r[key] for r in R], dtype=dt))
    return k
