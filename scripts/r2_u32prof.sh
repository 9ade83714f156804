rm -rf /tmp/reps; mkdir -p /tmp/reps
args=""
for k in "ul 11520 4 32 32 8704" "dl 11520 4 32 32 8704" "ul 2880 1 128 32 34048" "ul 720 1 512 32 135424"; do
  set -- $k
  timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"split_f|reg_f|mw_f" -s 2 -c 1 \
    -o /tmp/reps/u32_$1_$4 python scripts/prof_kernel.py $1 fp32 4 $2 $3 $4 $5 > /dev/null 2>&1
  P=$(( $2 * $3 ))
  args="$args ${1}_$4_$5=/tmp/reps/u32_$1_$4.ncu-rep:$P:$6"
done
python scripts/ncu_summary.py gpurun_out/ncu_u32.json $args > /dev/null 2>&1
for f in /tmp/reps/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv --print-source sass > /tmp/reps/$b.src.csv 2>/dev/null
  python scripts/stall_summary.py /tmp/reps/$b.src.csv > gpurun_out/stalls_$b.txt 2>&1
done
