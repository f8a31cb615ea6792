#!/bin/bash
# A/B timing of two library builds on a given config: bash tools/ab_cfg.sh A.so B.so CONFIG [rounds]
A=$1; B=$2; CFG=$3; N=${4:-2}
for i in $(seq $N); do
  for v in $A $B; do
    RC_LIB=$v timeout 600 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$(basename $v)', d['value'], {k:(round(v['ms_per_step'],3), v['frac']) for k,v in d['kernels'].items() if k in ('thermo','transport','prologue','epilogue')}, d['clocks']['sm_mhz'])"
  done
done
