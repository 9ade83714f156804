#!/bin/bash
# Full ncu captures of the hot kernels at the north-star shape, summarised on the
# box (gpurun_out/ncu_summary.json + per-kernel stall pages).
rm -rf /tmp/reps; mkdir -p /tmp/reps  # a reused box keeps /tmp: never summarise a stale report
args=""
for k in "ul fp32 4480" "dl fp32 4480" "ul fp16 2240" "dl fp16 2240" "opt fp32 4480" "pev fp32 4096"; do
  set -- $k
  timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"reg_f|tmh_f|gram_f16|gram_chol|pev16|pev_tc" -s 2 -c 1 \
    -o /tmp/reps/full_$1_$2 python scripts/prof_kernel.py $1 $2 4 > /dev/null 2>&1
  args="$args ${1}_${2}_32_16=/tmp/reps/full_$1_$2.ncu-rep:134400:$3"
done
python scripts/ncu_summary.py gpurun_out/ncu_summary.json $args > /dev/null 2>&1
for f in /tmp/reps/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv --print-source sass > /tmp/reps/$b.src.csv 2>/dev/null
  python scripts/stall_summary.py /tmp/reps/$b.src.csv > gpurun_out/stalls_$b.txt 2>&1
done
