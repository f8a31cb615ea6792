"""Timing experiment for the fused layer-1/2 kernel: build with -DL12TRACE, run one
bench step, print cluster 0's per-chunk clock64 stamps (MMA leader of each pair,
producer warp 0 and forwarder of every CTA, layer-1 issuer) and per-tile drain stamps."""
import ctypes as C
import os
import runpy
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
env = dict(os.environ, RC_EXTRA_NVCC_FLAGS="-DL12TRACE")
subprocess.check_call([sys.executable, os.path.join(ROOT, "paper_2312_13513_b200", "build.py"), "--force"], env=env)
sys.argv = ["bench.py", "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline"]
try:
    runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="__main__")
except SystemExit:
    pass
from paper_2312_13513_b200 import _rc  # noqa: E402

buf = np.zeros((4, 6, 64, 4), dtype=np.int64)
f = _rc.lib().rc_debug_l12trace
f.restype, f.argtypes = C.c_int, [C.c_void_p]
print("copy rc", f(buf.ctypes.data))
t0 = buf[buf > 0].min()
b = np.where(buf > 0, buf - t0, -1)
for g in list(range(0, 6)) + list(range(20, 32)) + list(range(44, 56)):
    m0, m2 = b[0, 0, g], b[2, 0, g]
    p = [b[r, 1, g] for r in range(4)]
    l1 = [b[r, 4, g] for r in (0, 2)]
    print(f"chunk {g:2d} MMA A: wait {m0[0]:8d} +{m0[1]-m0[0]:6d} iss {m0[2]-m0[1]:5d} | B: wait {m2[0]:8d} +{m2[1]-m2[0]:6d} | "
          + " ".join(f"P{r}: a1 {p[r][1]-p[r][0]:6d} ae {p[r][2]-p[r][1]:6d} st {p[r][3]-p[r][2]:5d} @{p[r][3]:8d}" for r in (0, 2))
          + " | " + " ".join(f"L1{2*i}: z {l[1]-l[0]:6d} ae@{l[2]:8d} +{l[3]-l[2]:6d}" for i, l in enumerate(l1)))
for it in range(4):
    print(f"tile {it}: " + " | ".join(
        f"CTA{r}: TMA zb {b[r,5,it,0]:8d}->{b[r,5,it,1]:8d} drain w0 {b[r,3,it,0]:8d} +{b[r,3,it,1]-b[r,3,it,0]:6d} "
        f"w8 {b[r,3,it,2]:8d} +{b[r,3,it,3]-b[r,3,it,2]:6d}" for r in range(4)))
