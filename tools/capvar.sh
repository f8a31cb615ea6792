# chunk-size (cells per MLP chunk) sweep, one bench each
for CAP in 32768 65536 131072; do
RC_MAX_CAP=$CAP timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('cap=$CAP', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
