for v in pf2 pf3; do DCDG_LIB_PATH=vlib/$v/libdcdg.so timeout 600 python scripts/sweep_configs4.py - 32 > gpurun_out/u32_$v.log 2>&1; done
timeout 600 python scripts/sweep_configs4.py - 32 > gpurun_out/u32_pf1.log 2>&1
