#!/bin/bash
# ncu --set full of the cell-local kernels (thermo, transport, prologue, chem epilogue) in one bench step
O=gpurun_out; mkdir -p $O
TAG=${1:-f}; CFG=${2:-C3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-thermo_kernel|transport_kernel|chem_epilogue|prologue}" -s ${SKIP:-0} -c ${COUNT:-4} \
  -o $O/prof_fp64_${CFG}_$TAG -f python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_fp64_${CFG}_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 $O/ncu_fp64_${CFG}_$TAG.log
