#!/bin/bash
# parity tests + a 10-step bench (no trace, no profiler)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps ${STEPS:-10} --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], {k:(round(v['ms_per_step'],3), round(v['frac'],3)) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
