#!/bin/bash
# parity tests, then short C2 / C3 / C4 benches printing the per-kernel times and roofline fractions
O=gpurun_out; mkdir -p $O
TAG=${1:-f}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for CFG in C2 C3 C4; do
  timeout 600 python bench.py --config $CFG --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${CFG}_$TAG.json 2> $O/bench_${CFG}_$TAG.err
  python -c "
import json,sys; d=json.loads(open('$O/bench_${CFG}_$TAG.json').readline()); print('$CFG', d['value'], {k:(round(v['ms_per_step'],3), round(v['frac'],3)) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 $O/bench_${CFG}_$TAG.err
done
