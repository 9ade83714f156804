rm -rf /tmp/reps; mkdir -p /tmp/reps
timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"ul_reg_f32" -s 2 -c 1 -o /tmp/reps/sig python scripts/prof_kernel.py opt fp32 4 > /dev/null 2>&1
ncu -i /tmp/reps/sig.ncu-rep --page source --csv --print-source cuda > /tmp/reps/sig_cuda.csv 2>/dev/null
head -c 3000 /tmp/reps/sig_cuda.csv > gpurun_out/sig_cuda_head.txt
python scripts/cuda_lines.py /tmp/reps/sig_cuda.csv 40 > gpurun_out/sig_lines.txt 2>&1
