#!/bin/bash
# kinetics parity tests, a kinetics bench (C2) and an ncu capture of the kinetics kernel
O=gpurun_out; mkdir -p $O
TAG=${1:-k}
timeout 600 python -m pytest tests -m gpu -x -q -s -k "kinetics" 2>&1 | tail -8
timeout 300 python bench.py --chem kinetics --steps 10 --cpu-seconds 5 > $O/bench_kin_$TAG.json 2> $O/bench_kin_$TAG.err
python -c "
import json; d=json.load(open('$O/bench_kin_$TAG.json')); print(d['value'], {k:(v['ms_per_step'], v['frac']) for k,v in d['kernels'].items()}, d.get('cpu_baseline'))" || tail -5 $O/bench_kin_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kinetics_kernel -c 1 -o $O/prof_kin_$TAG -f \
  python bench.py --chem kinetics --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_kin_$TAG.log 2>&1; echo "ncu rc=$?"
