rm -rf /tmp/reps; mkdir -p /tmp/reps
timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"pev_tc" -s 2 -c 1 -o /tmp/reps/full_pev_fp32 python scripts/prof_kernel.py pev fp32 4 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_pev.json pev_fp32_32_16=/tmp/reps/full_pev_fp32.ncu-rep:134400:4096 > /dev/null 2>&1
ncu -i /tmp/reps/full_pev_fp32.ncu-rep --page source --csv --print-source sass > /tmp/reps/p.csv 2>/dev/null
python scripts/stall_summary.py /tmp/reps/p.csv > gpurun_out/stalls_full_pev_fp32.txt 2>&1
