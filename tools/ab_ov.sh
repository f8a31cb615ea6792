#!/bin/bash
# interleaved A/B on one box: the previous build (tools/ab/librc_head.so), this build serial, this build
# with the layer-3 overlap
N=${1:-2}
for i in $(seq $N); do
  for v in head serial overlap; do
    case $v in head) E="RC_LIB=tools/ab/librc_head.so"; X="";; serial) E=""; X="--serial";; overlap) E=""; X="";; esac
    env $E timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-variants $X ${ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; print('$v', d['value'], d['clocks']['sm_mhz'], {n:(v['ms_per_step'], v['frac']) for n,v in k.items() if n.startswith('L')})"
  done
done
