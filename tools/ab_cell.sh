#!/bin/bash
# interleaved A/B of library builds on the cell-local kernels: bash tools/ab_cell.sh "A.so B.so ..." "C3 C4" [rounds]
LIBS=$1; CFGS=$2; N=${3:-2}
for cfg in $CFGS; do
for i in $(seq $N); do
  for v in $LIBS; do
    RC_LIB=$v timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-variants 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; print('$cfg $(basename $v)', d['value'], d['clocks']['sm_mhz'], {n:(v['ms_per_step'], v['frac']) for n,v in k.items() if not n.startswith('L')})"
  done
done
done
