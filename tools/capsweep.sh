for i in 1 2; do for C in 131072 262144 524288; do
RC_MAX_CAP=$C timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('cap=$C', d['value'], {k:(round(v['ms_per_step'],3)) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done; done
