#!/bin/bash
# One GPU pass: smoke, parity tests, bench, ncu launch list, ncu full captures.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
tail -2 $O/smoke_$TAG.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu_$TAG.log
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
cat $O/bench_$TAG.json; tail -3 $O/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-variants > /dev/null 2>&1; echo "ncu list rc=$?"
# ncu serialises kernels: the layer-3 side launch then runs alone on its 16 SMs and takes
# every tile of its chunk, so the kernel shares of the overlapped step come from the serial schedule's list
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_serial_$TAG.csv \
  python bench.py --serial --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-variants > /dev/null 2>&1; echo "ncu list (serial) rc=$?"
# l12_kernel: fused layers 1+2; l2_pair_kernel: layer 3 (DOT; the serial schedule's full-grid launch);
# l1_kernel / layer-2 pair: bench.py --layerwise run
for K in l12_kernel l2_pair_kernel; do
  C=1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c $C \
    -o $O/prof_${K}_$TAG -f python bench.py --serial --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-variants > $O/ncu_${K}_$TAG.log 2>&1
  echo "ncu $K rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"l1_kernel|l2_pair_kernel" -s 4 -c 2 \
  -o $O/prof_layerwise_$TAG -f python bench.py --layerwise --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_layerwise_$TAG.log 2>&1
echo "ncu layer-wise rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"thermo_kernel" -s 1 -c 1 \
  -o $O/prof_thermo_$TAG -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_thermo_$TAG.log 2>&1; echo "ncu thermo rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"thermo_kernel|transport_kernel|chem_epilogue|prologue" -s 2 -c 4 \
  -o $O/prof_fp64_$TAG -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_fp64_$TAG.log 2>&1; echo "ncu fp64 rc=$?"
ls -la $O | tail -20
