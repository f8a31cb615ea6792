"""Build the in-tree CUDA library librc_b200.so for sm_100a with nvcc.

Every kernel is compiled with -gencode arch=compute_100a,code=sm_100a
-lineinfo; the C ABI (include/rc.h) is the only exported surface.
usage: python -m paper_2312_13513_b200.build [--force]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "librc_b200.so")
SOURCES = ["capi.cpp", "thermo.cu", "transport.cu", "mlp_sm100.cu", "mlp_l1_sm100.cu", "mlp_l2_sm100.cu", "mlp_l12_sm100.cu", "kinetics.cu", "laplacian.cu"]
HEADERS = ["rc_internal.h", "ptx.cuh", "stream.cuh", "mlp_internal.h", "mlp_common.cuh", os.path.join("..", "..", "include", "rc.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
FLAGS += os.environ.get("RC_EXTRA_NVCC_FLAGS", "").split()  # experiments only (e.g. -D switches)


def _stale(objs):
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale(SOURCES):
        return SO
    objdir = os.path.join(CSRC, "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out)
        if p.returncode:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", *objs, "-o", SO]
    subprocess.check_call(link)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
