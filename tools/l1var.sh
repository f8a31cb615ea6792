# L1 kernel variants (compile-time switches), one bench each; rebuilds the default at the end
for V in "-DL1_SLEEP_MASK=3" "-DL1_SLEEP_MASK=0" "-DL1_SLEEP_MASK=11"; do
RC_EXTRA_NVCC_FLAGS="$V" python paper_2312_13513_b200/build.py --force > /dev/null 2>&1 || echo buildfail
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$V', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
python paper_2312_13513_b200/build.py --force > /dev/null 2>&1
