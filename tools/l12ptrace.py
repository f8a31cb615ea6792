"""Timing experiment for the pair-local fused layer-1/2 kernel: build with -DL12TRACE, run one
bench step, print pair 0's per-chunk clock64 stamps (MMA issuer, producer warp 0) and the
per-tile drain copy-out of warp 8."""
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

buf = np.zeros((2, 4, 64, 4), dtype=np.int64)
f = _rc.lib().rc_debug_l12ptrace
f.restype, f.argtypes = C.c_int, [C.c_void_p]
print("copy rc", f(buf.ctypes.data))
t0 = buf[buf > 0].min()
b = np.where(buf > 0, buf - t0, -1)
for g in list(range(0, 8)) + list(range(20, 32)) + list(range(44, 56)):
    m = b[0, 0, g]
    p = [b[r, 1, g] for r in range(2)]
    l1 = b[0, 3, g]
    print(f"chunk {g:2d} L1 @{l1[0]:8d} w1 {l1[1]-l1[0]:5d} a1e {l1[2]-l1[1]:5d} iss {l1[3]-l1[2]:4d} | MMA wait@{m[0]:8d} +{m[1]-m[0]:6d} l1 {m[2]-m[1]:5d} l2 {m[3]-m[2]:5d} | "
          + " ".join(f"P{r}: a1wait@{p[r][0]:8d} +{p[r][1]-p[r][0]:6d} gelu+freed {p[r][2]-p[r][1]:5d} st {p[r][3]-p[r][2]:5d} done@{p[r][3]:8d}" for r in range(2)))
for it in range(4):
    print(f"tile {it}: " + " | ".join(f"CTA{r}: drain @{b[r,2,it,0]:8d} copy-out {b[r,2,it,1]-b[r,2,it,0]:6d}" for r in range(2)))
