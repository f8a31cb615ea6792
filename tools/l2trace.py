"""Timing experiment for the CTA-pair GEMM (layers 2 and 3): build with -DL2TRACE,
run one bench step, print cluster 0 / CTA 0's per-tile clock64 stamps:
MMA warp (17): wait-start, accumulator free, last commit issued;
epilogue warps 0..15: wait-start, accumulator full, released, tile done."""
import ctypes as C
import os
import runpy
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
env = dict(os.environ, RC_EXTRA_NVCC_FLAGS="-DL2TRACE")
subprocess.check_call([sys.executable, os.path.join(ROOT, "paper_2312_13513_b200", "build.py"), "--force"], env=env)
sys.argv = ["bench.py", "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline"]
try:
    runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="__main__")
except SystemExit:
    pass
from paper_2312_13513_b200 import _rc  # noqa: E402

buf = np.zeros((2, 20, 40, 4), dtype=np.int64)
f = _rc.lib().rc_debug_l2trace
f.restype, f.argtypes = C.c_int, [C.c_void_p]
print("copy rc", f(buf.ctypes.data))
for dot, name in ((0, "layer 2"), (1, "layer 3 (dot)")):
    b = buf[dot]
    if not (b > 0).any():  # layer 2 runs in the fused kernel unless bench.py --layerwise
        continue
    t0 = b[b > 0].min()
    b = np.where(b > 0, b - t0, -1)
    print(name)
    for it in range(0, 12):
        m, e = b[17, it], b[:16, it]
        print(f"  tile {it:2d} MMA: wait {m[0]:8d} free+{m[1]-m[0]:6d} mainloop {m[2]-m[1]:6d} | epi: full at {e[:,1].max():8d} "
              f"(wait {np.mean(e[:,1]-e[:,0]):6.0f}) release after {np.mean(e[:,2]-e[:,1]):6.0f} (max {np.max(e[:,2]-e[:,1]):6.0f}) "
              f"done after {np.mean(e[:,3]-e[:,1]):6.0f}")
