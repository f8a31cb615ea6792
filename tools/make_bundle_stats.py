"""Write data/bundle_stats/<mech>.json: z-score statistics of the MLP inputs
x = [T, p, BCT(Y_1)..BCT(Y_ns)] (reading R4).

The paper's nets were trained on DNS data whose statistics are not published
(PAPER.md:114); a random-init bundle still needs defined input statistics.
They are the mean / std over 65,536 generator cells (C3 recipe for H2, C4 for
CH4), with std floored at 1e-12 + 1e-3 |mean|.  The Box-Cox transform is the
method's arithmetic, so this committed script computes x only through oracle/
(prologue with mean 0, std 1), as the task's rule for stored values requires.

usage: python tools/make_bundle_stats.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle  # noqa: E402
from workload import load_mech, make_cells  # noqa: E402
from workload.bundle import STATS  # noqa: E402

for mech_name, cfg in (("h2_9sp", "C3"), ("ch4_20sp", "C4")):
    m = load_mech(mech_name)
    ns = m["ns"]
    d_in = ns + 2
    ident = {"x_mean": [0.0] * d_in, "x_std": [1.0] * d_in}
    om = oracle.Mech(m)
    b = {"n_nets": 1, "d_in": d_in, "hidden": (1, 1, 1), "species_of_net": np.zeros(1, np.int32),
         "params": np.zeros((1, 64)), "x_mean": np.zeros(d_in), "x_std": np.ones(d_in),
         "y_mean": np.zeros(1), "y_std": np.ones(1), "lambda_bc": 0.1, "dt": 1e-6}
    ob = oracle.Mlp(b)
    # 65,536 cells drawn uniformly (hashed) over the whole grid
    from workload import CONFIGS
    n_all = CONFIGS[cfg].n_cells
    from workload.cells import uniform
    sample = np.unique((uniform(991, np.arange(65536)) * n_all).astype(np.int64))
    from workload import make_cells_at
    c = make_cells_at(cfg, sample)
    X = np.empty((sample.size, d_in))
    for i in range(sample.size):
        z, _ = ob.prologue(om, c["T_true"][i], c["p"][i], c["Y"][:, i])
        X[i] = z
    mean = X.mean(axis=0)
    std = X.std(axis=0)
    std = np.maximum(std, 1e-12 + 1e-3 * np.abs(mean))
    with open(os.path.join(STATS, mech_name + ".json"), "w") as f:
        json.dump({"mech": mech_name, "source": f"{sample.size} hashed-random cells of {cfg} (field 991), via oracle prologue",
                   "x_mean": mean.tolist(), "x_std": std.tolist()}, f, indent=1)
    print(mech_name, mean, std)
