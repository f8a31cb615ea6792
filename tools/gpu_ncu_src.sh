#!/bin/bash
# ncu --set full + source-level instruction mix of the cell-local kernels (C3 epilogue, C4 epilogue and
# transport, C3 thermo)
O=gpurun_out; mkdir -p $O
TAG=${1:-s}
run() {  # cfg kernel-regex name
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 0 -c 1 \
    -o $O/prof_$3_$TAG -f python bench.py --config $1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-variants > $O/ncu_$3_$TAG.log 2>&1
  echo "ncu $3 rc=$?"
  python tools/ncu_src.py $O/prof_$3_$TAG.ncu-rep "$2" 50 > $O/src_$3_$TAG.txt 2>&1
}
run C3 chem_epilogue epiC3
run C4 chem_epilogue epiC4
run C4 transport_kernel trC4
run C3 thermo_kernel thC3
