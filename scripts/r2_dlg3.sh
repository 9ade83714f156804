# launch list of the downlink + effective-gain stage (lab)
for v in base g0m; do
  DCDG_LIB_PATH=vlib/$v/libdcdg.so ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"dl_reg_f32|gain_reduce" -c 24 --csv --log-file gpurun_out/dlg_$v.csv python scripts/kbench.py 16800 3 > /dev/null 2>&1
done
