#!/bin/bash
# round-end evidence: the standard round (smoke, GPU tests, bench, ncu launch list + full captures),
# then the NEXT-row and precision benches and ncu captures of their kernels
TAG=${1:-r02d}
O=gpurun_out; mkdir -p $O
bash tools/gpu_round.sh $TAG
for args in "--config C3" "--config C4" "--precision tf32" "--config C4 --precision tf32" "--shared" "--chem kinetics" "--config C3 --laplacian" "--pasr --config C4" "--graph"; do
  name=$(echo $args | tr -d '-' | tr ' ' '_')
  timeout 900 python bench.py $args --steps 5 --no-e2e --no-cpu-baseline --no-variants > $O/bench_${name}_$TAG.json 2> $O/bench_${name}_$TAG.err
  echo "$args rc=$?"; head -c 200 $O/bench_${name}_$TAG.json; echo
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kinetics_kernel|lap_gather|ldu_to_csr" -c 3 \
  -o $O/prof_next_$TAG -f python bench.py --config C3 --laplacian --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_next_$TAG.log 2>&1; echo "ncu next rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kinetics_kernel" -c 1 \
  -o $O/prof_kin_$TAG -f python bench.py --chem kinetics --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_kin_$TAG.log 2>&1; echo "ncu kin rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"l12_kernel|l4_kernel" -s 2 -c 2 \
  -o $O/prof_tf32_$TAG -f python bench.py --precision tf32 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-variants > $O/ncu_tf32_$TAG.log 2>&1; echo "ncu tf32 rc=$?"
