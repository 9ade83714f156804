for r in 1 2; do python scripts/lab/u8_bench.py > gpurun_out/u8_base_$r.log 2>&1; DCDG_LIB_PATH=vlib/g8u8/libdcdg.so python scripts/lab/u8_bench.py > gpurun_out/u8_g8_$r.log 2>&1; done
