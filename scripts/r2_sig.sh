# fused-variance uplink: parity, timing, one full ncu capture
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xchg.py tests/test_gpu_ref_parity.py tests/test_gpu_aux.py tests/test_cpp_api.py -m gpu -q -x > gpurun_out/sig_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sig_tests.log
python scripts/opt_bench.py > gpurun_out/opt_bench.log 2>&1
rm -rf /tmp/reps; mkdir -p /tmp/reps
timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"ul_reg_f32" -s 2 -c 1 -o /tmp/reps/sig python scripts/prof_kernel.py opt fp32 4 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_sig.json sig=/tmp/reps/sig.ncu-rep:134400:4480 > /dev/null 2>&1
ncu -i /tmp/reps/sig.ncu-rep --page source --csv --print-source sass > /tmp/reps/sig.csv 2>/dev/null
python scripts/stall_summary.py /tmp/reps/sig.csv > gpurun_out/stalls_sig.txt 2>&1
