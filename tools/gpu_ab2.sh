#!/bin/bash
# parity tests, then interleaved bench: quad (default) vs pair-local (RC_L12_PAIR=1) fused kernel
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
for q in 1 0; do
RC_L12_PAIR=$((1-q)) timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('quad=$q', d['value'], {k:(round(v['ms_per_step'],3)) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done; done
