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
dbg = torch.zeros(10 * 8 * 64, dtype=torch.int64, device="cuda")
for _ in range(2):
    rc.rc_step(mech, mlp, st.cells(rc.RC_MODE_H, dt=b["dt"]), ws)
_rc.lib().rc_debug_flags(int(os.environ.get("L12_FLAGS", "0")))
_rc.lib().rc_debug_timeline(dbg.data_ptr())
rc.rc_step(mech, mlp, st.cells(rc.RC_MODE_H, dt=b["dt"]), ws)
torch.cuda.synchronize()
_rc.lib().rc_debug_timeline(None)
_rc.lib().rc_debug_flags(0)
d = dbg.cpu().numpy().reshape(10, 8, 64).astype(np.float64)
t0 = d[d > 0].min()
d = np.where(d > 0, d - t0, np.nan)
names = ["mma_wait_a2full", "mma_a2full_ok", "A_acc1_ready", "A_a2_written", "drain(start,end)", "-",
         "M_a1empty_ok", "M_l2_issued", "-", "-"]
for it in range(2, 3):
    print(f"--- tile {it}")
    for c in range(25):
        print(f"  c={c:2d} " + " ".join(f"{names[r][:9]:>9s}={d[r, it, c]:7.0f}" for r in [0, 1, 2, 3]))
    print(f"  drain start {d[4, it, 0]:.0f} end {d[4, it, 1]:.0f}")
print("drain summary (clk): tile start -> first a2full, chunk period, drain start->end, drain end -> next tile's first L2")
for it in range(6):
    st, en = d[4, it, 0], d[4, it, 1]
    first = d[1, it, 0]
    last = d[1, it, 24]
    nxt = d[1, it + 1, 0] if it + 1 < 8 else np.nan
    print(f"tile {it}: chunks {first:8.0f}..{last:8.0f} ({(last-first)/24:6.0f}/chunk)  drain {st:8.0f}..{en:8.0f} ({en-st:6.0f})  next L2 at {nxt:8.0f} (+{nxt-en:6.0f})")

