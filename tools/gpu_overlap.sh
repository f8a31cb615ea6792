#!/bin/bash
# layer-3 overlap: its tests, the GPU suite, then an interleaved A/B of the bench
# (default = overlap, --serial = one stream) on one box
TAG=${1:-ov}
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "overlap" 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do
  for v in "" "--serial"; do
    name=ab${v:+_serial}_$r
    timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-variants $v ${ARGS} > $O/bench_${TAG}_$name.json 2> $O/bench_${TAG}_$name.err
    python - "$O/bench_${TAG}_$name.json" "$v" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).readline())
k = d["kernels"]
print(sys.argv[2] or "overlap", d["value"], d["clocks"]["sm_mhz"], {n: (v["ms_per_step"], v["frac"]) for n, v in k.items() if n.startswith("L")},
      {n: k[n].get(x) for n in k if n == "L3_fill" for x in ("pairs_ran", "pairs_gave_up", "tiles_share")})
PY
  done
done
