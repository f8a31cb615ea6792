"""Summarise ncu output into profiles/ (tracked): the per-kernel launch list of a
bench step and the key counters of the full captures.

usage: python tools/ncu_summary.py TAG launches.csv [capture.ncu-rep ...]
writes profiles/ncu_TAG.json and profiles/traffic_TAG.json (DRAM bytes per launch
of each captured kernel; bench.py reports the layer-2 GEMM's as roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")
SCALE = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    name = re.sub(r"\(.*$", "", name)  # drop the argument list
    return name.replace("void ", "").replace("<unnamed>::", "").strip()


def launch_list(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    iK, iM, iU, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    agg = {}
    for r in rows[start + 1:]:
        if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
            continue
        t = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1e-9)
        k = short(r[iK])
        a = agg.setdefault(k, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += t * 1e6
    tot = sum(a["total_us"] for a in agg.values())
    for a in agg.values():
        a["total_us"] = round(a["total_us"], 2)
        a["avg_us"] = round(a["total_us"] / a["launches"], 2)
        a["share"] = round(a["total_us"] / tot, 4) if tot else None
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]))


KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", None),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", None),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", None),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
}


def capture(path):
    out = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        k = short(d.get("Kernel Name", "?"))
        e = {}
        for key, (m, mul) in KEYS.items():
            if m not in d:  # some metrics carry a section prefix ("TPC.TriageCompute.<name>")
                m = next((c for c in h if c.endswith("." + m) or c.endswith(m)), m)
            if m not in d or d[m] in ("", "n/a", "no data"):
                continue
            v = float(d[m].replace(",", ""))
            if mul is not None:
                v = v * SCALE.get(u.get(m, ""), 1) * mul if key == "duration_us" else v * SCALE.get(u.get(m, ""), 1)
            e[key] = round(v, 4) if isinstance(v, float) else v
        stalls = {m.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[m].replace(",", "") or 0) for m in h
                  if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued")
                  and d[m] not in ("n/a", "no data")}
        tot = sum(stalls.values())
        if tot:
            e["stall_top"] = {k2: round(v / tot, 3) for k2, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        if "dram_read_bytes" in e and "dram_write_bytes" in e:
            e["dram_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
        res.setdefault(k, e)  # first launch of each kernel in the capture
    return res


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    out = {"tag": tag, "launch_list": launch_list(lcsv),
           "note": "launch list: ncu --metrics gpu__time_duration.sum --clock-control none (serialised, "
                   "cold-cache per launch: use the shares, not the absolute times); captures: ncu --set full "
                   "--clock-control none, first captured launch of each kernel"}
    caps = {}
    for r in reps:
        caps.update(capture(r))
    out["captures"] = caps
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", f"ncu_{tag}.json"), "w"), indent=1)
    traffic = {k: v.get("dram_bytes") for k, v in caps.items()}
    l12 = next((v for k, v in traffic.items() if "l12_kernel" in k), None)  # fused layers 1+2 (default bf16 path)
    l2 = next((v for k, v in traffic.items() if "l2_pair_kernel" in k and ", 0, " in k), None)  # layer 2 (not DOT)
    json.dump({"per_launch_dram_bytes": traffic, "dominant_kernel_dram_bytes_per_launch": l12 if l12 else l2,
               "L2_gemm_dram_bytes_per_launch": l2,
               "source": f"ncu --set full, profiles/ncu_{tag}.json"},
              open(os.path.join(ROOT, "profiles", f"traffic_{tag}.json"), "w"), indent=1)
    print(json.dumps(out["launch_list"], indent=1)[:3000])
    for k, v in caps.items():
        print(k, v)


if __name__ == "__main__":
    main()
