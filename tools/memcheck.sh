#!/bin/bash
# compute-sanitizer memcheck of the smoke step and a 1-step C2 bench (fused quad and pair-local kernels)
O=gpurun_out; mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 $O/memcheck_smoke.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/memcheck_bench.txt 2>&1; echo "bench rc=$?"; tail -3 $O/memcheck_bench.txt
