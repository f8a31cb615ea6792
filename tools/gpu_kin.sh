#!/bin/bash
# kinetics parity tests, kinetics benches (C2 default line, C3 steady state) and an ncu capture
O=gpurun_out; mkdir -p $O
TAG=${1:-k}
timeout 600 python -m pytest tests -m gpu -x -q -s -k "kinetics" 2>&1 | tail -8
timeout 300 python bench.py --chem kinetics --steps 10 --cpu-seconds 5 > $O/bench_kin_$TAG.json 2> $O/bench_kin_$TAG.err
timeout 300 python bench.py --chem kinetics --config C3 --steps 5 --no-cpu-baseline > $O/bench_kin_C3_$TAG.json 2> $O/bench_kin_C3_$TAG.err
for f in bench_kin_$TAG bench_kin_C3_$TAG; do python -c "
import json; d=json.load(open('$O/$f.json')); print('$f', d['value'], {k:(v['ms_per_step'], v['frac']) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 $O/$f.err; done
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kinetics_kernel -c 1 -o $O/prof_kin_$TAG -f \
  python bench.py --chem kinetics --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_kin_$TAG.log 2>&1; echo "ncu rc=$?"
fi
