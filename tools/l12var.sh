# fused layer-1/2 kernel: chunks of the next tile produced before the drain (RC_L12_LEADIN) sweep
for L in 0 1 2 3 4; do
RC_L12_LEADIN=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('lead_in=$L', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
