# pair GEMM: epilogue warps parked (default) vs spinning on the accumulator-full barrier
for V in "" "-DL2_EPI_SPIN"; do
RC_EXTRA_NVCC_FLAGS="$V" python paper_2312_13513_b200/build.py --force > /dev/null 2>&1 || echo buildfail
for r in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('[$V]', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
done
python paper_2312_13513_b200/build.py --force > /dev/null 2>&1
