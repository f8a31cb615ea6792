#!/bin/bash
# GPU pass: parity tests (-s: per-net errors), then an interleaved A/B of the current library
# against a reference build (tools/ab.sh).  usage: bash tools/gpu_check_ab.sh TAG REF.so [rounds]
TAG=$1; REF=$2; N=${3:-2}
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -s > $O/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_$TAG.log
bash tools/ab.sh $REF paper_2312_13513_b200/librc_b200.so $N 2>&1 | tee $O/ab_$TAG.txt
