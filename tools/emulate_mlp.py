"""CPU emulation of the MLP precision modes against the fp64 oracle.

Question it answers: what o / wdot / qdot error does an MLP that only rounds its
operands (bf16-RNE or tf32-RNE weights and activations, fp32 accumulation, one
rounding per activation) make on the parity samples the GPU tests use?  If the
plain rounding already meets SURVEY §8(c)'s gates (2e-2 bf16, 1e-3 TF32 on o AND
wdot), any extra GPU error is the kernels' own and the gates stay where the
contract puts them.

Variants (all: weights pre-rounded RNE, fp32 accumulation, biases fp32):
  bf16_ideal   z, h1, h2 rounded to bf16 once each; exact-erf GELU in fp32 from the
               fp32 accumulator; h3 fp32 into the fp32 layer-4 dot
  bf16_tanh32  as bf16_ideal but the tanh-form GELU in fp32 (the fp32 MUFU GELU)
  bf16_r01     round-1 kernels: accumulator (+bias) rounded to bf16 BEFORE GELU, GELU
               evaluated with every op rounded to bf16 (tanh-form, bf16x2 arithmetic)
  tf32         z, h1, h2, h3 rounded to tf32 (RNE), exact-erf GELU in fp32

Reference: oracle.step (fp64, exact erf).  The sample is the GPU tests' hashed
sample (workload.cells.uniform(seed, ...)) for several seeds.  The o -> wdot map
below restates SURVEY §8(c) steps 8-10 (inverse Box-Cox, projection, rho dY/dt)
and is checked against the oracle's own wdot on the oracle's o before use.

usage: python tools/emulate_mlp.py [--cells 256] [--seeds 4242 4243 4244] [--cfg C2 C4]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from _emulate import emulate_o, oracle_z, rel, wdot_from_o  # noqa: E402
from workload import CONFIGS, load_mech, make_bundle, make_cells_at  # noqa: E402
from workload.cells import uniform  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=256)
    ap.add_argument("--seeds", type=int, nargs="+", default=[4242, 4243, 4244])
    ap.add_argument("--cfg", nargs="+", default=["C2", "C4"])
    ap.add_argument("--variants", nargs="+", default=["bf16_ideal", "bf16_tanh32", "bf16_r01", "tf32"])
    a = ap.parse_args()
    torch.set_num_threads(os.cpu_count() or 1)
    for cfg in a.cfg:
        C = CONFIGS[cfg]
        mech, b = load_mech(C.mech), make_bundle(C.mech, hidden=C.hidden)
        om, ob = oracle.Mech(mech), oracle.Mlp(b)
        P = om.projection()
        for seed in a.seeds:
            idx = np.unique((uniform(seed, np.arange(a.cells)) * C.n_cells).astype(np.int64))
            c = make_cells_at(cfg, idx)
            r = oracle.step(om, ob, c["T_true"], c["p"], c["Y"], mode="T", transport=False)
            w_chk, q_chk = wdot_from_o(mech, b, P, r["T"], r["rho"], c["Y"], r["o"])
            assert rel(w_chk, r["wdot"]) < 1e-10 and rel(q_chk, r["qdot"]) < 1e-10, "restated o->wdot map disagrees"
            z = oracle_z(om, ob, r["T"], c["p"], c["Y"])
            for v in a.variants:
                o = emulate_o(b, z, v)
                w, q = wdot_from_o(mech, b, P, r["T"], r["rho"], c["Y"], o)
                per = " ".join(f"{rel(o[i], r['o'][i]):.1e}" for i in range(o.shape[0]))
                print(f"{cfg} seed {seed} n={len(idx)} {v:12s} o {rel(o, r['o']):.2e} wdot {rel(w, r['wdot']):.2e} "
                      f"qdot {rel(q, r['qdot']):.2e} | per-net o {per}", flush=True)


if __name__ == "__main__":
    main()
