# ncu of the TMEM half-tile lab kernel (vlib/tmh) and ul_reg_f32
rm -rf /tmp/reps; mkdir -p /tmp/reps
DCDG_LIB_PATH=vlib/tmh/libdcdg.so timeout 300 ncu -f --set full --clock-control none -k regex:"ul_tmh" -s 2 -c 1 -o /tmp/reps/tmh python scripts/prof_kernel.py ul fp32 4 > gpurun_out/tmhprof.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_tmh.json tmh=/tmp/reps/tmh.ncu-rep:134400:4480 >> gpurun_out/tmhprof.log 2>&1
ncu -i /tmp/reps/tmh.ncu-rep --page raw --csv > gpurun_out/tmh_raw.csv 2>/dev/null
ncu -i /tmp/reps/tmh.ncu-rep --page source --csv --print-source sass > /tmp/reps/tmh.csv 2>/dev/null
python scripts/stall_summary.py /tmp/reps/tmh.csv > gpurun_out/stalls_tmh.txt 2>&1
