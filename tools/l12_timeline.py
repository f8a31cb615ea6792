"""Developer tool: event timeline of CTA 0 of the fused layer-1/2 kernel (one
C2 chunk).  usage (GPU): python tools/l12_timeline.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_13513_b200 as rc  # noqa: E402
from paper_2312_13513_b200 import _rc  # noqa: E402
from workload import load_mech, make_bundle, make_cells  # noqa: E402

m = load_mech("h2_9sp")
b = make_bundle("h2_9sp")
mech = rc.Mechanism(m)
mlp = rc.MLPBundle(mech, b)
n = 32768
c = make_cells("C2", 0, n)
st = rc.CellState(n, 9, b["n_nets"]).load(c["T_true"], c["p"], c["Y"])
rc.rc_thermo(mech, st.cells(rc.RC_MODE_T, chem=False, transport=False))
ws = rc.aligned_workspace(mlp, n)
dbg = torch.zeros(5 * 8 * 64, dtype=torch.int64, device="cuda")
for _ in range(2):
    rc.rc_step(mech, mlp, st.cells(rc.RC_MODE_H, dt=b["dt"]), ws)
_rc.lib().rc_debug_timeline(dbg.data_ptr())
rc.rc_step(mech, mlp, st.cells(rc.RC_MODE_H, dt=b["dt"]), ws)
torch.cuda.synchronize()
_rc.lib().rc_debug_timeline(None)
d = dbg.cpu().numpy().reshape(5, 8, 64).astype(np.float64)
t0 = d[d > 0].min()
d = np.where(d > 0, d - t0, np.nan)
names = ["mma_wait_a2full", "mma_a2full_ok", "A_acc1_ready", "A_a2_written", "drain(start,end)"]
for it in range(4):
    print(f"--- tile {it}")
    for c in range(25):
        print(f"  c={c:2d} " + " ".join(f"{names[r][:14]:>14s}={d[r, it, c]:9.0f}" for r in range(4)))
    print(f"  drain start {d[4, it, 0]:.0f} end {d[4, it, 1]:.0f}")
