#!/bin/bash
# quick GPU check: smoke + parity tests + bench (no profiler)
TAG=${1:-q}
O=gpurun_out; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | tail -15
timeout 600 python bench.py --no-cpu-baseline > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"; cat $O/bench_$TAG.json; tail -5 $O/bench_$TAG.err
