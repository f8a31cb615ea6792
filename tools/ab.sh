#!/bin/bash
# A/B timing of two library builds on the same box, interleaved (power-cap clock drift hits both):
# usage: bash tools/ab.sh A.so B.so [rounds]
A=$1; B=$2; N=${3:-3}
for i in $(seq $N); do
  for v in $A $B; do
    RC_LIB=$v timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$(basename $v)', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
  done
done
