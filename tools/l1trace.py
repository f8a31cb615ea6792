"""Timing experiment for the layer-1 kernel: build with -DL1TRACE, run one bench
step, dump CTA 0's per-tile clock64 stamps (warps 0..15 epilogue: wait-start,
tfull acquired, released, stored; warp 17 MMA: wait-start, tempty acquired,
full acquired)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
env = dict(os.environ, RC_EXTRA_NVCC_FLAGS="-DL1TRACE")
subprocess.check_call([sys.executable, os.path.join(ROOT, "paper_2312_13513_b200", "build.py"), "--force"], env=env)
sys.argv = ["bench.py", "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline"]
import runpy  # noqa: E402

try:
    runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="__main__")
except SystemExit:
    pass
from paper_2312_13513_b200 import _rc  # noqa: E402

L = _rc.lib()
buf = np.zeros((24, 96, 8), dtype=np.int64)
f = L.rc_debug_l1trace
f.restype = C.c_int
f.argtypes = [C.c_void_p]
print("copy rc", f(buf.ctypes.data))
t0 = buf[buf > 0].min()
b = np.where(buf > 0, buf - t0, -1)
np.save(os.path.join(ROOT, "gpurun_out", "l1trace.npy"), b)
NE, WM = 16, 17
for it in range(0, 40):
    e = b[:NE, it, :]
    m = b[WM, it, :]
    print(f"tile {it:3d} MMA wait {m[0]:8d} tempty+{m[1]-m[0]:6d} full+{m[2]-m[1]:5d} | "
          f"epi start {e[:,0].min():8d}..{e[:,0].max():8d} tfull wait {np.mean(e[:,1]-e[:,0]):6.0f} "
          f"ld+rel {np.mean(e[:,2]-e[:,1]):5.0f} gelu+store {np.mean(e[:,3]-e[:,2]):6.0f}")
