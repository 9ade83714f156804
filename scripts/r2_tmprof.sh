rm -rf /tmp/reps; mkdir -p /tmp/reps
DCDG_LIB_PATH=vlib/tm2/libdcdg.so timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"ul_tm" -s 2 -c 1 -o /tmp/reps/tm python scripts/prof_kernel.py ul fp32 4 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_tm.json tm=/tmp/reps/tm.ncu-rep:134400:4480 > /dev/null 2>&1
ncu -i /tmp/reps/tm.ncu-rep --page source --csv --print-source sass > /tmp/reps/tm.csv 2>/dev/null
python scripts/stall_summary.py /tmp/reps/tm.csv > gpurun_out/stalls_tm.txt 2>&1
