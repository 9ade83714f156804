# fused fp32 variance kernel (forward elimination): full ncu capture, SASS + CUDA-line stall pages
rm -rf /tmp/reps; mkdir -p /tmp/reps
timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"ul_reg_f32" -s 2 -c 1 -o /tmp/reps/sig python scripts/prof_kernel.py opt fp32 4 > gpurun_out/sigprof.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_sig.json sig=/tmp/reps/sig.ncu-rep:134400:4480 >> gpurun_out/sigprof.log 2>&1
ncu -i /tmp/reps/sig.ncu-rep --page source --csv --print-source sass > /tmp/reps/sig.csv 2>/dev/null
python scripts/stall_summary.py /tmp/reps/sig.csv > gpurun_out/stalls_sig.txt 2>&1
ncu -i /tmp/reps/sig.ncu-rep --page source --csv --print-source cuda > gpurun_out/sig_cuda_src.csv 2>/dev/null
cp /tmp/reps/sig.ncu-rep gpurun_out/
