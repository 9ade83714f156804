rm -rf /tmp/reps; mkdir -p /tmp/reps  # a reused box keeps /tmp: never summarise a stale report
for d in ul dl; do
  timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"gram_f16" -s 2 -c 1 \
    -o /tmp/reps/full_${d}_gram python scripts/prof_kernel.py $d fp16 4 > /dev/null 2>&1
  ncu -i /tmp/reps/full_${d}_gram.ncu-rep --page source --csv --print-source sass > /tmp/reps/${d}.csv 2>/dev/null
  python scripts/stall_summary.py /tmp/reps/${d}.csv > gpurun_out/stalls_${d}_gram.txt 2>&1
  ncu -i /tmp/reps/full_${d}_gram.ncu-rep --page raw --csv > gpurun_out/raw_${d}_gram.csv 2>/dev/null
done
python scripts/ncu_summary.py gpurun_out/ncu_gram.json ul_fp16_32_16=/tmp/reps/full_ul_gram.ncu-rep:134400:2240 dl_fp16_32_16=/tmp/reps/full_dl_gram.ncu-rep:134400:2240 > /dev/null 2>&1
