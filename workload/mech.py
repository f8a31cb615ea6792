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
