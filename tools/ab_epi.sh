#!/bin/bash
# interleaved A/B of the cell-local kernels: the previous build (tools/ab/librc_prev.so) vs this build
N=${1:-2}
for cfg in C3 C4; do
for i in $(seq $N); do
  for v in prev new; do
    case $v in prev) E="RC_LIB=tools/ab/librc_prev.so";; new) E="";; esac
    env $E timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-variants ${ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; print('$cfg $v', d['value'], d['clocks']['sm_mhz'], {n:(v['ms_per_step'], v['frac']) for n,v in k.items() if not n.startswith('L')})"
  done
done
done
