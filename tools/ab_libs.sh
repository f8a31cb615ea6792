#!/bin/bash
# interleaved A/B of library builds on one box: bash tools/ab_libs.sh "A.so B.so" [rounds] [bench args]
LIBS=$1; N=${2:-2}; shift 2; ARGS="$@"
for i in $(seq $N); do
  for v in $LIBS; do
    RC_LIB=$v timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-variants $ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; e=d.get('e2e') or {}
print('$(basename $v)', d['value'], 'e2e', e.get('value'), d['clocks']['sm_mhz'], {n:(v['ms_per_step'], v['frac']) for n,v in k.items() if n.startswith('L')})"
  done
done
