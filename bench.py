#!/usr/bin/env python
"""bench.py -- throughput of the full per-cell thermo + transport + DNN-chemistry
step (BASELINE.json metric: Mcells/s, % roofline) on 1..8 B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--precision bf16]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)
  python bench.py --impl reference ...                   (the CPU oracle, timed as it stands)

One step = rc_step over every local cell (a1 thermo Newton, a2 transport, a3-a5
MLP chemistry) + the a6 global reductions (NCCL all-reduce of max T and
sum qdot / counters when N > 1).  Inputs are synthetic states from workload/
(shapes of the paper's workloads, DESIGN.md input recipe) with random-init
weights of the paper's MLP shape.  Default workload: C2 =
BASELINE configs[1], 1,048,576 H2/air cells, MLP 11->1600->800->400->1 x 8 nets.
Multi-GPU is weak scaling: every rank owns C2-sized blocks of a periodic tiling
of the C2 grid (no halo, no data-path collective).
Prints ONE JSON line on rank 0.
"""
import argparse
import glob
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SUSTAINED = "bf16_tflops_sustained"
# executed FP64-pipe instructions per cell of kinetics_kernel (ncu, profiles/ncu_kinetics_r02.json)
KIN_FP64_INSTR_PER_CELL = {"h2_9sp": 1180}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "tf32", "tf32x3"])
    ap.add_argument("--strong", action="store_true", help="partition the config's cells (strong scaling)")
    ap.add_argument("--layerwise", action="store_true", help="rc_mlp_desc.flags = RC_MLP_LAYERWISE (comparison path)")
    ap.add_argument("--e2e-batches", type=int, default=1,
                    help="sub-batches of the e2e pipeline (copies of one overlap the compute of another)")
    ap.add_argument("--serial", action="store_true",
                    help="rc_mlp_desc.flags = RC_MLP_SERIAL: layer 3 not overlapped with the fused kernel (comparison)")
    ap.add_argument("--pasr", action="store_true", help="LES: PaSR scaling of wdot with per-cell tau_mix (NEXT-4)")
    ap.add_argument("--shared", action="store_true", help="one shared net with n_nets outputs (NEXT-2)")
    ap.add_argument("--laplacian", action="store_true",
                    help="add the NEXT-1 consumer: Algorithm 1 Laplacian assembly of the ns+1 species/energy "
                         "systems (+ ldu->CSR at N=1; z-slab halo exchange over NCCL P2P at N>1); 3D configs")
    ap.add_argument("--graph", action="store_true",
                    help="replay the step as one CUDA graph (PAPER.md:187); per-kernel timing is then unavailable")
    ap.add_argument("--chem", default="dnn", choices=["dnn", "kinetics"],
                    help="source term: the DNN (the paper's GPU path) or detailed kinetics (NEXT-3, the CVODE RHS)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU rank logic only (gloo): partition, generation, a6 reductions, NEXT-1 halo exchange")
    ap.add_argument("--dry-cells", type=int, default=65536, help="--dry-run: local cells generated per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the TF32 line beside the bf16 headline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle baseline")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, SUSTAINED: 1400.0}, "fallback"


# FP64 FMA rate measured on this pool's B200 by tools/microbench/peaks.cu (profiles/peaks_r01.json)
def fp64_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_r01.json")) as f:
            return json.load(f)["fp64_fma_tflops"], "measured (tools/microbench/peaks.cu)"
    except (OSError, KeyError):
        return 37.0, "fallback (148 SM x 64 DFMA/clk x 1.965 GHz)"


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region (B200_PROFILING.md
    clocks line).  NVML polled from a thread every 5 ms (nvidia-smi's start-up latency would
    miss most of a ~1 s timed region); falls back to nvidia-smi -lms if NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = None

    def _handle(self, nv):
        """NVML handle of this process's CUDA device, matched by PCI bus id (CUDA and NVML
        enumerate devices differently when CUDA_VISIBLE_DEVICES is set)."""
        nv.nvmlInit()
        want = None
        try:
            import torch
            want = str(torch.cuda.get_device_properties(self.index).pci_bus_id).lower()
        except Exception:
            pass
        n = nv.nvmlDeviceGetCount()
        for i in range(n):
            h = nv.nvmlDeviceGetHandleByIndex(i)
            bid = nv.nvmlDeviceGetPciInfo(h).busId
            bid = (bid.decode() if isinstance(bid, bytes) else str(bid)).lower()
            if want and (bid.endswith(want) or want.endswith(bid[-12:])):
                return h
        return nv.nvmlDeviceGetHandleByIndex(self.index if self.index < n else 0)

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            h = self._handle(nv)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((float(sm), float(mx), int(r)))
                except Exception:
                    pass
                time.sleep(0.005)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 5 ms polling during the timed steps"}


def generate(cfg, idx, world=1):
    """Host generation of this rank's cells (workload.make_cells_at), in parallel over 1M-cell chunks
    with this rank's share of the host cores: C5 gives every one of 8 ranks 12.5M cells (~45 s of
    single-core numpy); the cell values are a pure function of the global index, so the split
    changes nothing."""
    from workload import make_cells_at
    n = idx.size
    chunk = 1 << 20
    workers = max(1, min(len(os.sched_getaffinity(0)) // max(1, world), (n + chunk - 1) // chunk))
    if workers == 1 or n <= 2 * chunk:
        return make_cells_at(cfg, idx)
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    parts = [idx[i:i + chunk] for i in range(0, n, chunk)]
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
        res = list(ex.map(make_cells_at, [cfg] * len(parts), parts))
    return {k: np.concatenate([r[k] for r in res], axis=-1) for k in res[0]}


def run_dry(a):
    """--dry-run: the multi-rank host logic of run_ours on CPU (gloo) -- cell partition, generation of
    (the first --dry-cells of) the local block, the a6 global reductions, and with --laplacian the
    z-slab halo exchange -- so a world-size-2 CPU test can drive it (tests/test_multirank.py)."""
    import torch
    import torch.distributed as dist

    from paper_2312_13513_b200.dist import GlobalReductions, exchange_halos, slab
    from workload import CONFIGS
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    cfg = CONFIGS[a.config]
    idx, n_global = local_cells(cfg, rank, world, a.strong)
    sub = idx[:a.dry_cells]
    host = generate(cfg, sub, world)
    red = torch.tensor([float(host["T_true"].max()), float(host["p"].sum())], dtype=torch.float64)
    diag = torch.tensor([0, 0, 0, int((host["Y"] < 0).any(axis=0).sum()), 0], dtype=torch.int64)
    GlobalReductions("cpu")(red, diag)
    out = {"dry_run": True, "rank": rank, "world": world, "cells_local": int(idx.size), "first": int(idx[0]),
           "last": int(idx[-1]), "cells_total": int(idx.size) * world if not a.strong else int(n_global),
           "red": red.tolist(), "diag": diag.tolist()}
    if a.laplacian and len(cfg.grid) == 3:
        nx, ny, nz = cfg.grid
        z0, z1 = slab(nz * world, rank, world)            # weak scaling: rank blocks stacked in z
        plane = nx * ny
        bottom = torch.full((3, plane), float(z0), dtype=torch.float64)
        top = torch.full((3, plane), float(z1 - 1), dtype=torch.float64)
        lo, hi = exchange_halos(bottom, top)
        out["halo"] = [float(lo[0, 0]), float(hi[0, 0])]  # plane indices of the neighbours' boundary planes
        out["slab"] = [z0, z1]
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def local_cells(cfg, rank, world, strong):
    """Global cell indices owned by this rank.  Weak: a C-sized block per rank of a
    periodic tiling of the config grid; strong: rc_partition of the config."""
    import paper_2312_13513_b200 as rc
    n = cfg.n_cells
    if strong:
        b, e = rc.rc_partition(n, rank, world)
        return np.arange(b, e, dtype=np.int64), n
    return (np.arange(rank * n, (rank + 1) * n, dtype=np.int64) % n), n * world


def algorithmic(cfg, bundle, ns, n, precision="bf16"):
    """Per-step algorithmic work: bytes for the HBM-bound stages (the
    minimum each must move), FLOPs for the MLP, FP64 flops for transport."""
    d, (h1, h2, h3) = bundle["d_in"], bundle["hidden"]
    nout = bundle["n_nets"]
    nets = 1 if bundle.get("shared") else nout              # hidden-layer nets (NEXT-2 shared net: one)
    eb = {"bf16": 2, "tf32": 4, "tf32x3": 8}[precision]  # MLP activation bytes (tf32x3: hi + lo)
    kz = 16 if d + 2 <= 16 else 32                          # layer-1 input row (d inputs, 2 bias columns)
    flops_net = 2 * (d * h1 + h1 * h2 + h2 * h3 + h3 * nout // nets)
    npair = ns * (ns + 1) // 2
    return {
        "thermo_bytes": n * ((3 + ns) * 8 + 3 * 8),
        "transport_bytes": n * ((2 + ns) * 8 + (2 + ns) * 8),
        # FP64-pipe instructions of the factorised algorithm, x 2 flop per DFMA slot:
        # Wilke 3 ns nse (A, B, C sums), binary pairs 8 per pair j < k (4 Horner + 2 reciprocal
        # + 2 FMA), 32 per species (fits, reciprocals, sums, D_k), 120 per cell (ln T, sqrt, p/T^1.5)
        "transport_fp64_flops": n * 2 * (3 * ns * ((ns + 1) // 2 * 2) + 8 * (npair - ns) + 32 * ns + 120),
        "L1_flops": n * nets * 2 * d * h1,
        "L2_flops": n * nets * 2 * h1 * h2,
        "L3_flops": n * nets * 2 * (h2 * h3 + (0 if bundle.get("shared") else h3)),
        "L4_flops": n * 2 * h3 * nout if bundle.get("shared") else 0,
        "L4_bytes": n * (h3 * eb + nout * 4) if bundle.get("shared") else 0,  # h3 read, o written
        # detailed kinetics: FP64-pipe instructions per cell executed by the kernel (ncu
        # sm__inst_executed_pipe_fp64 per cell, profiles/ncu_kinetics_r02.json), x 2 flop per DFMA slot
        "kinetics_fp64_flops": n * 2 * KIN_FP64_INSTR_PER_CELL.get(cfg.mech, 0),
        # NEXT-1: in rho, lambda, cp, D_k; out upper (3 faces per cell) and diag of ns+1 systems
        "laplacian_bytes": n * ((3 + ns) * 8 + 4 * (ns + 1) * 8),
        # ldu -> CSR: in upper + diag; out 7 columns (int32) + 7 values per system + row pointer
        "csr_bytes": n * (4 * (ns + 1) * 8 + 7 * 4 + 7 * (ns + 1) * 8 + 8),
        "mlp_flops": n * nets * flops_net,
        "L1_bytes": n * nets * h1 * eb,               # h1 activations written
        # in: raw outputs o (fp32 per net), T, rho, Y; out: wdot, qdot
        "epilogue_bytes": n * (nout * 4 + 2 * 8 + ns * 8 + ns * 8 + 8),
        # in: T, p, Y; out: the layer-1 input row
        "prologue_bytes": n * ((2 + ns) * 8 + kz * eb),
    }


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_2312_13513_b200 as rc
    from paper_2312_13513_b200.dist import GlobalReductions
    from workload import CONFIGS, load_mech, make_bundle, make_cells_at

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[a.config]
    # this rank's cells, generated on the host BEFORE any CUDA context or NCCL communicator exists
    # (generate() forks worker processes for large blocks)
    idx, n_global = local_cells(cfg, rank, world, a.strong)
    n = idx.size
    host = generate(cfg, idx, world)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mech_d = load_mech(cfg.mech)
    bundle = make_bundle(cfg.mech, hidden=cfg.hidden, shared=a.shared)
    mech = rc.Mechanism(mech_d)
    prec = {"bf16": rc.RC_BF16, "tf32": rc.RC_TF32, "tf32x3": rc.RC_TF32X3}[a.precision]
    mlp = rc.MLPBundle(mech, bundle, prec, flags=(rc.RC_MLP_LAYERWISE if a.layerwise else 0) |
                       (rc.RC_MLP_SERIAL if a.serial else 0))
    ns, nets = mech_d["ns"], bundle["n_nets"]
    st = rc.CellState(n, ns, nets, outputs=("cp", "rho", "mu", "lam", "D", "wdot", "qdot"))
    st.load(host["T_true"], host["p"], host["Y"])
    if a.pasr:
        from workload import tau_mix_at
        st.set_tau_mix(tau_mix_at(cfg, idx))
    stream = torch.cuda.current_stream()
    # h of each cell from the previous step's state: h(T_true, Y) by the library's own T-mode thermo
    rc.rc_thermo(mech, st.cells(rc.RC_MODE_T, chem=False, transport=False), stream)
    T_guess = torch.from_numpy(host["T_guess"]).to("cuda")
    ws = rc.aligned_workspace(mlp, n)
    reduce_a6 = GlobalReductions("cuda")
    cells = st.cells(rc.RC_MODE_H, dt=bundle["dt"])
    if a.chem == "kinetics":
        from workload import load_kinetics
        kin = rc.Kinetics(mech, load_kinetics(cfg.mech))

    lap = None
    if a.laplacian:  # NEXT-1: the block is a z-slab (weak scaling: rank blocks stacked in z) of a periodic box
        if len(cfg.grid) != 3 or a.strong:
            raise SystemExit("--laplacian needs a 3D config (C3, C4, C5) and weak scaling")
        from paper_2312_13513_b200.dist import exchange_halos
        h_sp = 0.01 / cfg.grid[0]                      # uniform spacing: a ~1 cm box
        mesh = (*cfg.grid, h_sp, h_sp, h_sp)
        nsys, plane = ns + 1, cfg.grid[0] * cfg.grid[1]
        f64 = dict(dtype=torch.float64, device="cuda")
        lap = {"up": torch.empty(nsys, 3 * n, **f64), "dg": torch.empty(nsys, n, **f64)}
        if world > 1:
            lap.update(bot=torch.empty(ns + 3, plane, **f64), top=torch.empty(ns + 3, plane, **f64))
        else:
            lap.update(rp=torch.empty(n + 1, dtype=torch.int64, device="cuda"),
                       col=torch.empty(7 * n, dtype=torch.int32, device="cuda"), val=torch.empty(nsys, 7 * n, **f64))

    def consumer():
        if world > 1:  # halo planes of the neighbouring slabs (NCCL P2P), then the slab assembly
            rc.rc_pack_planes(mech, mesh, cells, lap["bot"], lap["top"], stream)
            lo, hi = exchange_halos(lap["bot"], lap["top"])
            rc.rc_laplacian(mech, mesh, cells, lap["up"], lap["dg"], lo, hi, rc.RC_LAP_GATHER, stream)
        else:
            rc.rc_laplacian(mech, mesh, cells, lap["up"], lap["dg"], None, None, rc.RC_LAP_GATHER, stream)
            rc.rc_ldu_to_csr(mesh, nsys, lap["up"], lap["dg"], lap["rp"], lap["col"], lap["val"], stream)

    def step():
        st.T[:n].copy_(T_guess)                       # each step restarts Newton from the same guess
        if a.chem == "kinetics":                       # a1 + a2 + detailed kinetics instead of a3-a5
            st.red.zero_()
            st.diag.zero_()
            rc.rc_thermo(mech, cells, stream)
            rc.rc_transport(mech, cells, stream)
            rc.rc_kinetics(mech, kin, cells, stream)
        else:
            rc.rc_step(mech, mlp, cells, ws, stream)
        if lap is not None:
            consumer()
        reduce_a6(st.red, st.diag)                     # a6: global max T and sums (NCCL over NVLink; no-op at N=1)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = rc.rc_last_launch_count()     # our kernels per rc_step (the T restore copy is torch's)
    if a.graph:  # the whole step (T restore + rc_step) captured once, replayed every step
        if world > 1 or a.laplacian or a.chem != "dnn":
            raise SystemExit("--graph: single-GPU DNN step only")
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            st.T[:n].copy_(T_guess)
            rc.rc_step(mech, mlp, cells, ws, cap)
        stream.wait_stream(cap)
        step = graph.replay
        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
    else:
        rc.rc_profile_enable(True)
    rc.rc_profile_read(reset=True)
    if hasattr(rc.lib(), "rc_overlap_read"):
        rc.rc_overlap_read(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / a.steps
    # the launches on one time axis (CUDA events on both streams): how long the layer-3 side launches
    # ran while a fused L1+L2 launch was running
    tl = rc.rc_profile_timeline() if hasattr(rc.lib(), "rc_profile_timeline") else []
    l12_iv = [(t0, t1) for s_, t0, t1 in tl if s_ == "L12"]
    fill_iv = [(t0, t1) for s_, t0, t1 in tl if s_ == "L3_fill"]
    fill_conc = sum(max(0.0, min(b1, b2) - max(a1, a2)) for a1, b1 in fill_iv for a2, b2 in l12_iv)
    prof = rc.rc_profile_read(reset=True)
    ovl = rc.rc_overlap_read(reset=True) if hasattr(rc.lib(), "rc_overlap_read") else {}
    rc.rc_profile_enable(False)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_cells = n * world if not a.strong else n_global
    value = total_cells / (ms_max * 1e-3) / 1e6

    # ---- end to end through the C ABI from pinned HOST buffers (H2D in, D2H out, every step)
    e2e = None
    if not a.no_e2e and a.chem == "dnn" and not a.laplacian:
        e2e = run_e2e(a, rc, mech, mlp, bundle, host, st, ws, n, ns, world, stream)

    out = None
    if rank == 0:
        pk, pk_src = peaks()
        f64, f64_src = fp64_peak()
        alg = algorithmic(cfg, bundle, ns, n, a.precision)
        K = a.steps

        def per(stage):
            ms_s, cnt = prof[stage]
            return ms_s / K, cnt / K

        # tensor peak of the MLP's own arithmetic: the measured bf16 figure x the guide's nominal ratio
        # (tf32 dense = 1/2 of bf16; tf32x3 spends three tf32 MMAs per useful product)
        tratio = {"bf16": 1.0, "tf32": 0.5, "tf32x3": 0.5 / 3}[a.precision]
        # the sustained peak was measured under the power cap (MEASURED_PEAKS clocks_under_load): it is the
        # peak of a kernel inside a long, power-capped step; a run whose SM clock never left the maximum
        # (a short step: the cap did not engage) is a kernel timed alone and is held to the burst peak
        cs0 = clk.summary()
        pmhz_s = (pk.get("clocks_under_load") or {}).get("sm_mhz_median")
        burst = bool(cs0.get("sm_mhz") and cs0["sm_mhz"] >= 0.95 * pk.get("sm_max_mhz", 1965.0) and "bf16_tflops" in pk)
        pkey = "bf16_tflops" if burst else SUSTAINED
        tpeak = round(pk[pkey] * tratio, 1)
        kernels = {}
        for st_name, work, unit, bound, peak in [
            ("thermo", alg["thermo_bytes"], "GB/s", "hbm", pk["hbm_gbs"]),
            ("transport", alg["transport_fp64_flops"], "TFLOP/s", "fp64", f64),
            ("prologue", alg["prologue_bytes"], "GB/s", "hbm", pk["hbm_gbs"]),
            ("L1", alg["L1_bytes"], "GB/s", "hbm", pk["hbm_gbs"]),  # K=16: bound by the h1 write, not the MMA
            ("L2", alg["L2_flops"], "TFLOP/s", "tensor", tpeak),
            ("L12", alg["L1_flops"] + alg["L2_flops"], "TFLOP/s", "tensor", tpeak),  # fused layers 1+2
            ("L3", alg["L3_flops"], "TFLOP/s", "tensor", tpeak),
            ("L3_fill", alg["L3_flops"], "TFLOP/s", "tensor", tpeak),
            ("L4", alg["L4_bytes"], "GB/s", "hbm", pk["hbm_gbs"]),  # shared net's output layer (CUDA cores)
            ("kinetics", alg["kinetics_fp64_flops"], "TFLOP/s", "fp64", f64),  # detailed kinetics (NEXT-3)
            ("laplacian", alg["laplacian_bytes"], "GB/s", "hbm", pk["hbm_gbs"]),     # NEXT-1 assembly
            ("csr", alg["csr_bytes"], "GB/s", "hbm", pk["hbm_gbs"]),                 # NEXT-1 ldu -> CSR
            ("epilogue", alg["epilogue_bytes"], "GB/s", "hbm", pk["hbm_gbs"]),
        ]:
            t_ms, cnt = per(st_name)
            if t_ms <= 0:
                continue
            if st_name in ("L3", "L3_fill") and prof["L3_fill"][0] > 0:
                # layer 3 overlapped with the fused kernel: the tiles the launches beside
                # it ran (rc_overlap_read) are their work, the rest the main launches'; the side launches
                # run on the SMs the fused kernel's clusters leave idle, their peak is that share of the GPU
                l3_tiles = K * (1 if bundle.get("shared") else bundle["n_nets"]) * (-(-n // 256))
                ffrac = min(1.0, ovl["tiles_fill"] / l3_tiles) if l3_tiles else 0.0
                work = work * (ffrac if st_name == "L3_fill" else 1.0 - ffrac)
                if st_name == "L3_fill":
                    fill_sms = 2 * ovl["pairs_ran"] / max(1, prof["L3_fill"][1])  # SMs per side launch that ran
                    peak = round(tpeak * fill_sms / torch.cuda.get_device_properties(0).multi_processor_count, 1)
            scale = 1e9 if unit == "GB/s" else 1e12
            ach = work / (t_ms * 1e-3) / scale
            kernels[st_name] = {"bound": bound, "achieved": round(ach, 2), "peak": peak, "unit": unit,
                                "frac": round(ach / peak, 4), "ms_per_step": round(t_ms, 4),
                                "launches_per_step": cnt, "share": None}
        tot_k = sum(v["ms_per_step"] for k, v in kernels.items() if k != "L3_fill")
        for k, v in kernels.items():
            v["share"] = round(v["ms_per_step"] / tot_k, 4) if tot_k and k != "L3_fill" else None
        if "L3_fill" in kernels:  # concurrent with L12 on the otherwise idle SMs: not on the step's critical path
            kernels["L3_fill"].update({"concurrent_with": "L12", "tiles_share": round(ffrac, 4),
                                       "ms_per_step_during_L12": round(fill_conc / K, 4),
                                       "pairs_ran": ovl["pairs_ran"], "pairs_gave_up": ovl["pairs_gave_up"]})
        fused = "L12" in kernels
        l2 = kernels.get("L12" if fused else "L2", {})
        traffic = None
        tfs = sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")))  # latest round's summary
        tf = tfs[-1] if tfs and a.precision == "bf16" else ""
        if os.path.exists(tf):
            try:
                tj = json.load(open(tf))
                traffic = tj.get("dominant_kernel_dram_bytes_per_launch", tj.get("L2_gemm_dram_bytes_per_launch"))
            except (OSError, ValueError):
                traffic = None
        mlp_ms = sum(per(s)[0] for s in ("L1", "L2", "L3", "L12", "L4"))
        # the roofline object describes the dominant kernel of the step that ran: the MLP's layer-1/2
        # GEMM for the DNN chemistry; the kinetics kernel when --chem kinetics replaces it (NEXT-3)
        if a.chem == "kinetics" and "kinetics" in kernels:
            kk = kernels["kinetics"]
            roofline = {"kernel": "kinetics_kernel (12 reactions, falloff, reverse rates; fp64)", "bound": "fp64",
                        "achieved": kk["achieved"], "peak": kk["peak"], "unit": kk["unit"], "frac": kk["frac"],
                        "traffic": None, "peak_source": f64_src,
                        "work_per_launch": "2 * KIN_FP64_INSTR_PER_CELL * cells FLOP (ncu-calibrated FP64 instruction count)"}
        else:
            roofline = {"kernel": (f"fused L1+L2 (z -> h1 1600 on chip -> h2 800, tcgen05 {a.precision}, 4-CTA clusters)"
                                   if fused else f"L2 GEMM (h1 1600 -> h2 800, tcgen05 {a.precision})"), "bound": "tensor",
                        "achieved": l2.get("achieved"), "peak": tpeak, "unit": "TFLOP/s",
                        "frac": l2.get("frac"), "traffic": traffic,
                        "peak_source": f"{pk_src} {pkey} (MEASURED_PEAKS.json)"
                                       + ("" if a.precision == "bf16" else f" x {tratio:.3f} ({a.precision}, nominal ratio)"),
                        "work_per_launch": ("2*cells_chunk*(d_in*1600 + 1600*800)*nets FLOP" if fused
                                            else "2*cells_chunk*1600*800*nets FLOP")}
            # the step is power-capped: the SM clock it ran at against the one the sustained peak was
            # measured at (MEASURED_PEAKS clocks_under_load); frac x peak_mhz / sm_mhz is the fraction
            # per clock cycle
            pmhz = pk.get("sm_max_mhz") if burst else pmhz_s
            cs = cs0
            if pmhz and cs.get("sm_mhz") and roofline.get("frac"):
                roofline.update({"sm_mhz": cs["sm_mhz"], "peak_sm_mhz": pmhz,
                                 "frac_per_clock": round(roofline["frac"] * pmhz / cs["sm_mhz"], 4)})
        out = {
            "metric": ("Mcells/s per thermo+transport+DNN-chem step" if a.chem == "dnn"
                       else "Mcells/s per thermo+transport+detailed-kinetics step (NEXT-3)"),
            "value": round(value, 4),
            "unit": "Mcells/s",
            "n_gpus": world,
            "steps": a.steps,
            "warmup": a.warmup,
            "ms_per_step": round(ms_max, 4),
            "higher_is_better": True,
            "scaling": "strong" if a.strong else "weak",
            "vs_baseline": None,
            "dtype": (f"{a.precision} MLP (fp32 accumulate) + f64 thermo/transport/epilogue" if a.chem == "dnn"
                      else "f64 (thermo, transport, detailed kinetics)"),
            "data": "synthetic (seeded manifold states, random-init paper-shape MLP weights)",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "cells_per_gpu": int(n), "cells_total": int(total_cells),
                       "mech": cfg.mech, "hidden": list(cfg.hidden), "nets": nets, "parallelism": f"cells dp{world}",
                       "l2": "working set > L2 (h2 of 262144-cell chunks x 8 nets 3.4 GB, z 32 MB; "
                             "cell state 0.2 GB) - no flush needed",
                       "precision": a.precision, **({"les_pasr": True} if a.pasr else {}),
                       **({"mlp": "one shared net, n_nets outputs (NEXT-2)"} if a.shared else {}),
                       **({"chem": "detailed kinetics, 12 reactions (NEXT-3)"} if a.chem == "kinetics" else {}),
                       **({"consumer": "Laplacian assembly of ns+1 systems (NEXT-1)"} if a.laplacian else {}),
                       **({"launch": "one CUDA graph per step"} if a.graph else {}),
                       **({"mlp_schedule": "serial (RC_MLP_SERIAL)"} if a.serial else
                          {"mlp_schedule": "layer 3 of chunk j-1 beside the fused L1+L2 kernel of chunk j on its idle SMs"}
                          if prof["L3_fill"][0] > 0 else {})},
            "roofline": roofline,
            # the whole MLP on the step's critical path (the layer-3 side launches run beside L12 and
            # are not counted in mlp_ms): its FLOPs over that time, against the same tensor peak
            "mlp_tflops": round(alg["mlp_flops"] / (mlp_ms * 1e-3) / 1e12, 2) if mlp_ms else None,
            "mlp_frac": round(alg["mlp_flops"] / (mlp_ms * 1e-3) / 1e12 / tpeak, 4) if mlp_ms and a.chem == "dnn" else None,
            "kernels": kernels,
            "clocks": clk.summary(),
            "gpu_launches": int(launches_per_step * a.steps),
            "e2e": e2e,
            "fp64_peak_source": f64_src,
        }
    if world > 1:
        dist.barrier()
    # ---- the TF32 MLP on the same cells (north_star's 1e-3 gate on o is met by TF32; bf16 is the
    # headline), a short device-timed run beside the default bf16 line
    if (rank == 0 and world == 1 and a.precision == "bf16" and a.chem == "dnn" and not a.shared and not a.laplacian
            and not a.graph and not a.no_variants):
        out["precision_variants"] = {"tf32": tf32_variant(a, rc, mech, bundle, cells, st, T_guess, n, stream)}
    # ---- CPU oracle baseline, rank 0 at N = 1 only
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, bundle, mech_d, a.cpu_seconds, a.chem)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def tf32_variant(a, rc, mech, bundle, cells, st, T_guess, n, stream):
    """The same step with the TF32 MLP (RC_TF32: layer-wise tcgen05 kind::tf32 GEMMs, exact-erf GELU)."""
    import torch
    mlp = rc.MLPBundle(mech, bundle, rc.RC_TF32)
    ws = rc.aligned_workspace(mlp, n)
    steps = max(3, min(10, a.steps))

    def step():
        st.T[:n].copy_(T_guess)
        rc.rc_step(mech, mlp, cells, ws, stream)

    for _ in range(max(1, a.warmup)):
        step()
    torch.cuda.synchronize()
    rc.rc_profile_enable(True)
    rc.rc_profile_read(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    prof = rc.rc_profile_read(reset=True)
    rc.rc_profile_enable(False)
    ms = e0.elapsed_time(e1) / steps
    pk, _ = peaks()
    tpeak = round(pk[SUSTAINED] * 0.5, 1)
    d, (h1, h2, h3) = bundle["d_in"], bundle["hidden"]
    fused = prof["L12"][0] > 0                         # the fused layer-1/2 kernel (tf32 instance)
    key = "L12" if fused else "L2"
    k_ms = prof[key][0] / steps
    k_flops = n * bundle["n_nets"] * 2 * ((d * h1 if fused else 0) + h1 * h2)
    del ws, mlp
    return {"value": round(n / (ms * 1e-3) / 1e6, 4), "unit": "Mcells/s", "ms_per_step": round(ms, 4), "steps": steps,
            key: {"bound": "tensor", "achieved": round(k_flops / (k_ms * 1e-3) / 1e12, 2) if k_ms else None,
                  "peak": tpeak, "unit": "TFLOP/s",
                  "frac": round(k_flops / (k_ms * 1e-3) / 1e12 / tpeak, 4) if k_ms else None,
                  "peak_source": "measured bf16 sustained x 1/2 (nominal dense tf32 ratio)"},
            "stage_ms": {k: round(v[0] / steps, 4) for k, v in prof.items() if v[0] > 0}}


def run_e2e(a, rc, mech, mlp, bundle, host, st, ws, n, ns, world, stream):
    """Same metric, timed from pinned host inputs to host outputs through the C ABI.

    Two device cell states alternate between steps (each split into B sub-batches, default one):
    the host->device copy of step k+1's inputs and the device->host copy of step k-1's outputs run
    on two copy streams while step k computes (rc_step on the caller's stream), and
    rc_combine_reductions forms each step's a6 values from the per-batch reductions (then the NCCL
    allreduce across ranks).  Every step copies its own inputs in and its outputs out.
    """
    import torch
    from paper_2312_13513_b200.dist import GlobalReductions
    B = a.e2e_batches if n % (a.e2e_batches * 128) == 0 else 1
    nb = n // B
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
    h_all = st.h[:n].cpu().numpy()
    hin_all, hout_all = [], []
    for b in range(B):  # host buffers, shared by the two device sets (copies of one stream are ordered)
        sl = slice(b * nb, (b + 1) * nb)
        hin_all.append({"h": pin(h_all[sl]), "T": pin(host["T_guess"][sl]), "p": pin(host["p"][sl]),
                        "Y": pin(host["Y"][:, sl])})
        hout_all.append({k: torch.empty((nb,) if k not in ("D", "wdot") else (ns, nb), dtype=torch.float64).pin_memory()
                         for k in ("T", "cp", "rho", "mu", "lam", "D", "wdot", "qdot")})
    sets = []  # [parity] -> (batches, cells, red_parts, diag_parts)
    for _ in range(2):
        batches = [(rc.CellState(nb, ns, mlp.n_nets, outputs=("cp", "rho", "mu", "lam", "D", "wdot", "qdot")),
                    hin_all[b], hout_all[b]) for b in range(B)]
        red_parts = torch.zeros(B, 2, dtype=torch.float64, device="cuda")
        diag_parts = torch.zeros(B, 5, dtype=torch.int64, device="cuda")
        cells = []
        for b, (sb, _, _) in enumerate(batches):
            c = sb.cells(rc.RC_MODE_H, dt=bundle["dt"])
            c.red, c.diag = red_parts[b].data_ptr(), diag_parts[b].data_ptr()
            cells.append(c)
        sets.append((batches, cells, red_parts, diag_parts))
    red = torch.zeros(2, dtype=torch.float64, device="cuda")
    diag = torch.zeros(5, dtype=torch.int64, device="cuda")
    reduce_a6 = GlobalReductions("cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    in_done = [[torch.cuda.Event() for _ in range(B)] for _ in range(2)]
    cmp_done = [[torch.cuda.Event() for _ in range(B)] for _ in range(2)]
    out_done = [[torch.cuda.Event() for _ in range(B)] for _ in range(2)]
    for e in [e for ev in cmp_done + out_done for e in ev]:
        e.record(stream)
    h2d = sum(t.numel() for hin in hin_all for t in hin.values()) * 8
    d2h = sum(t.numel() for hout in hout_all for t in hout.values()) * 8
    k_step = [0]

    def step():
        par = k_step[0] & 1
        k_step[0] += 1
        batches, cells, red_parts, diag_parts = sets[par]
        for b, (sb, hin, hout) in enumerate(batches):
            # this set's buffers were last used two steps ago: its compute has read the inputs and its
            # D2H has read the outputs (T included) before the H2D / compute rewrite them; compute
            # waits on in_done, which is recorded after this wait, so it is ordered too
            s_in.wait_event(out_done[par][b])
            with torch.cuda.stream(s_in):
                sb.h[:nb].copy_(hin["h"], non_blocking=True)
                sb.T[:nb].copy_(hin["T"], non_blocking=True)
                sb.p[:nb].copy_(hin["p"], non_blocking=True)
                sb.Y[:, :nb].copy_(hin["Y"], non_blocking=True)
                in_done[par][b].record(s_in)
            stream.wait_event(in_done[par][b])
            rc.rc_step(mech, mlp, cells[b], ws, stream)
            cmp_done[par][b].record(stream)
            s_out.wait_event(cmp_done[par][b])
            with torch.cuda.stream(s_out):
                for k, v in hout.items():
                    src = getattr(sb, k)
                    v.copy_(src[:nb] if src.dim() == 1 else src[:, :nb], non_blocking=True)
                out_done[par][b].record(s_out)
        rc.rc_combine_reductions(red_parts, diag_parts, red, diag, stream)
        reduce_a6(red, diag)

    for _ in range(max(1, a.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    for _ in range(a.steps):
        step()
    s_out.wait_stream(stream)
    e1.record(s_out)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    val = n * world / (t.item() * 1e-3) / 1e6
    return {"value": round(val, 4), "unit": "Mcells/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(t.item(), 4),
            "api": f"rc_step (C ABI) on two alternating device states ({B} sub-batch(es) each), pinned host buffers, "
                   f"H2D of step k+1 / D2H of step k-1 on copy streams overlapping step k, rc_combine_reductions + NCCL for a6"}


def oracle_time(cfg, bundle, mech_d, idx, chem="dnn"):
    import oracle
    from workload import load_kinetics, make_cells_at
    c = make_cells_at(cfg, idx)
    om, ob = oracle.Mech(mech_d), oracle.Mlp(bundle)
    h = oracle.step(om, None, c["T_true"], c["p"], c["Y"], mode="T", transport=False, chem=False)["h"]
    kin = oracle.Kin(load_kinetics(cfg.mech)) if chem == "kinetics" else None
    t0 = time.perf_counter()
    if kin is None:
        oracle.step(om, ob, c["T_guess"], c["p"], c["Y"], h=h)
    else:  # a1 + a2, then the detailed-kinetics sources at the converged T
        r = oracle.step(om, None, c["T_guess"], c["p"], c["Y"], h=h, chem=False)
        oracle.kinetics(om, kin, r["T"], c["p"], c["Y"])
    return time.perf_counter() - t0


def cpu_baseline(cfg, bundle, mech_d, seconds, chem="dnn"):
    """The fp64 oracle as it stands, on the box's host cores, on a bounded hashed sample."""
    import oracle
    from workload.cells import uniform
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    n_all = cfg.n_cells
    # probe with several cells per core (a 1-cell-per-thread probe overstates the per-cell cost)
    probe = np.unique((uniform(777, np.arange(max(64, 8 * cores))) * n_all).astype(np.int64))
    t_probe = oracle_time(cfg, bundle, mech_d, probe, chem)
    per_cell = t_probe / probe.size
    m = int(min(n_all, max(probe.size, seconds / max(per_cell, 1e-9))))
    idx = np.unique((uniform(778, np.arange(m)) * n_all).astype(np.int64))
    t = oracle_time(cfg, bundle, mech_d, idx, chem)
    what = "full step a1-a5" if chem == "dnn" else "a1 + a2 + detailed kinetics"
    return {"value": round(idx.size / t / 1e6, 8), "unit": "Mcells/s", "cores": cores, "kind": "oracle",
            "sample": f"{idx.size} hashed-random cells of {cfg.name} ({what}, fp64, {t:.1f} s)"}


def run_reference(a):
    """--impl reference: the CPU oracle (this tier's reference arm), timed as it stands."""
    import oracle
    from workload import CONFIGS, load_mech, make_bundle
    from workload.cells import uniform
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    oracle.build()
    cfg = CONFIGS[a.config]
    mech_d = load_mech(cfg.mech)
    bundle = make_bundle(cfg.mech, hidden=cfg.hidden)
    cores = len(os.sched_getaffinity(0))
    n_all = cfg.n_cells
    probe = np.unique((uniform(779, np.arange(max(64, 8 * cores))) * n_all).astype(np.int64))
    per_cell = oracle_time(cfg, bundle, mech_d, probe) / probe.size
    budget = min(10.0, 150.0 / max(1, a.steps + a.warmup))   # whole run within a few minutes
    m = int(min(n_all, max(cores, budget / max(per_cell, 1e-9))))
    times = []
    for s in range(a.warmup + a.steps):
        idx = np.unique((uniform(800 + s, np.arange(m)) * n_all).astype(np.int64))
        t = oracle_time(cfg, bundle, mech_d, idx)
        if s >= a.warmup:
            times.append((idx.size, t))
    cells = sum(c for c, _ in times)
    secs = sum(t for _, t in times)
    v = cells / secs / 1e6
    out = {"impl": "reference", "metric": "Mcells/s per thermo+transport+DNN-chem step", "value": round(v, 8),
           "unit": "Mcells/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
           "ms_per_step": round(1e3 * secs / len(times), 2), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": {"workload": f"{cfg.name}: {cfg.note}"},
           "cpu_baseline": {"value": round(v, 8), "unit": "Mcells/s", "cores": cores, "kind": "oracle",
                            "sample": f"{m} hashed-random cells of {cfg.name} per step"},
           "e2e": {"value": round(v, 8), "unit": "Mcells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.dry_run:
        run_dry(args)
    else:
        run_ours(args)
