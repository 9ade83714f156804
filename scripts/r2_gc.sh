DCDG_LIB_PATH=vlib/sc0/libdcdg.so python scripts/opt_bench.py > gpurun_out/opt_sc0.log 2>&1
python scripts/opt_bench.py > gpurun_out/opt_sc1.log 2>&1
DCDG_LIB_PATH=vlib/sc0/libdcdg.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uplink_fp32" > gpurun_out/sc0_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sc0_tests.log
