#!/bin/bash
# compute-sanitizer memcheck: the smoke step, a 1-step C2 bench (fused path, TMA-ring fp64 kernels,
# one-launch epilogue), and the NEXT-row GPU tests (kinetics, Laplacian/CSR/halo packing, shared net,
# PaSR) -- ragged tiles and ld > n included
O=gpurun_out; mkdir -p $O
TAG=${1:-r02}
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke_$TAG.txt 2>&1; echo "smoke rc=$?"; tail -2 $O/memcheck_smoke_$TAG.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/memcheck_bench_$TAG.txt 2>&1; echo "bench rc=$?"; tail -2 $O/memcheck_bench_$TAG.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q -k "kinetics or laplacian or slab or csr or shared or pasr or c1_full" > $O/memcheck_next_$TAG.txt 2>&1; echo "next rc=$?"; tail -3 $O/memcheck_next_$TAG.txt
