#!/bin/bash
# Laplacian (NEXT-1) parity tests + the C3 --laplacian bench (per-kernel times and fractions)
O=gpurun_out; mkdir -p $O
TAG=${1:-lap}
timeout 600 python -m pytest tests -m gpu -x -q -k "laplacian or halo" 2>&1 | tail -3
timeout 600 python bench.py --config C3 --laplacian --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $O/bench_lap_$TAG.json 2> $O/bench_lap_$TAG.err
python -c "
import json; d=json.loads(open('$O/bench_lap_$TAG.json').readline()); print(d['value'], {k:(round(v['ms_per_step'],3), round(v['frac'],3)) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 $O/bench_lap_$TAG.err
