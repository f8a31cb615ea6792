#!/bin/bash
# ncu --set full of two chem-epilogue launches (C3 and C4)
O=gpurun_out; mkdir -p $O
TAG=${1:-f}
for CFG in C3 C4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chem_epilogue" -s 1 -c 1 \
  -o $O/prof_epi_${CFG}_$TAG -f python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_epi_${CFG}_$TAG.log 2>&1
echo "ncu $CFG rc=$?"
done
