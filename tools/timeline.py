"""One profiled C2 step's launches on one time axis (rc_profile_timeline): the gaps between
consecutive launches on the caller's stream, and the layer-3 side launches against the fused kernel.
usage (GPU): python tools/timeline.py [bench config args...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_13513_b200 as rc  # noqa: E402
from workload import load_mech, make_bundle, make_cells  # noqa: E402
import oracle  # noqa: E402  (h(T) of the inputs only)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
mech_d = load_mech("h2_9sp")
b = make_bundle("h2_9sp", hidden=(1600, 800, 400))
c = make_cells("C2", 0, n)
h = oracle.step(oracle.Mech(mech_d), None, c["T_true"], c["p"], c["Y"], mode="T", transport=False, chem=False)["h"]
mech = rc.Mechanism(mech_d)
mlp = rc.MLPBundle(mech, b, rc.RC_BF16)
st = rc.CellState(n, 9, b["n_nets"]).load(c["T_guess"], c["p"], c["Y"], h=h)
ws = rc.aligned_workspace(mlp, n)
cells = st.cells(rc.RC_MODE_H, dt=b["dt"])
T0 = st.T.clone()
for _ in range(3):
    st.T.copy_(T0)
    rc.rc_step(mech, mlp, cells, ws)
torch.cuda.synchronize()
rc.rc_profile_enable(True)
rc.rc_profile_read(reset=True)
st.T.copy_(T0)
rc.rc_step(mech, mlp, cells, ws)
torch.cuda.synchronize()
tl = rc.rc_profile_timeline()
rc.rc_profile_read(reset=True)
main = [(s, a, e) for s, a, e in tl if s != "L3_fill"]
fill = [(s, a, e) for s, a, e in tl if s == "L3_fill"]
print(f"step {max(e for _, _, e in tl) - min(a for _, a, _ in tl):.3f} ms, {len(main)} launches on the caller's stream")
gap = 0.0
for (s0, a0, e0), (s1, a1, e1) in zip(main, main[1:]):
    g = a1 - e0
    gap += max(g, 0.0)
    print(f"  {s0:10s} {a0:9.3f} -> {e0:9.3f} ({e0 - a0:7.3f})  gap to {s1:10s} {g * 1e3:8.1f} us")
s, a, e = main[-1]
print(f"  {s:10s} {a:9.3f} -> {e:9.3f} ({e - a:7.3f})")
print(f"total gap between launches on the caller's stream: {gap * 1e3:.1f} us")
for s, a, e in fill:
    print(f"  side {a:9.3f} -> {e:9.3f} ({e - a:7.3f})")
