#!/bin/bash
# round-end evidence that fits gpurun's 64 MiB return: tools/gpu_final.sh, then the ncu summaries are
# made on the box (profiles/ncu_TAG.json, traffic_TAG.json, per-report raw counters) and copied into
# gpurun_out/; only the fused kernel's full capture is kept as a report
TAG=${1:-r02f}
O=gpurun_out
bash tools/gpu_final.sh $TAG
python tools/ncu_summary.py $TAG $O/launches_serial_$TAG.csv $O/prof_l12_kernel_$TAG.ncu-rep $O/prof_l2_pair_kernel_$TAG.ncu-rep \
  $O/prof_fp64_$TAG.ncu-rep > $O/ncu_summary_$TAG.log 2>&1; echo "summary rc=$?"
cp profiles/ncu_$TAG.json profiles/traffic_$TAG.json $O/ 2>/dev/null
for r in $O/prof_*_$TAG.ncu-rep; do python tools/ncu_raw.py $r > ${r%.ncu-rep}.txt 2>&1; done
for k in l12_kernel l2_pair_kernel fp64 thermo; do python tools/ncu_src.py $O/prof_${k}_$TAG.ncu-rep "." 30 > $O/src_${k}_$TAG.txt 2>&1; done
find $O -name "prof_*_$TAG.ncu-rep" ! -name "prof_l12_kernel_$TAG.ncu-rep" -delete
du -sh $O
