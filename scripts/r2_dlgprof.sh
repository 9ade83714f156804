# source-level stall samples of the downlink kernel with and without the gain share (lab)
rm -rf /tmp/reps; mkdir -p /tmp/reps
for d in dl dlg; do
  timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"dl_reg_f32" -s 2 -c 1 -o /tmp/reps/$d python scripts/prof_kernel.py $d fp32 4 > /dev/null 2>&1
  ncu -i /tmp/reps/$d.ncu-rep --page source --csv --print-source cuda > /tmp/reps/${d}_cuda.csv 2>/dev/null
  python scripts/cuda_lines.py /tmp/reps/${d}_cuda.csv 60 > gpurun_out/${d}_lines.txt 2>&1
  ncu -i /tmp/reps/$d.ncu-rep --page raw --csv > gpurun_out/${d}_raw.csv 2>/dev/null
done
