#!/bin/bash
# fused layer-1/2 kernel experiment: timeline trace, then parity + two benches of the normal build
O=gpurun_out; mkdir -p $O; TAG=${1:-x}
timeout 300 python tools/l12trace.py > $O/l12trace_$TAG.txt 2>&1; echo "trace rc=$?"
python paper_2312_13513_b200/build.py --force > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for L in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('run $L', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
