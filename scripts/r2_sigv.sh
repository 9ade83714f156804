for v in sig8 sig9; do DCDG_LIB_PATH=vlib/$v/libdcdg.so python scripts/opt_bench.py >> gpurun_out/opt_bench_v.log 2>&1; done
DCDG_LIB_PATH=vlib/sig9/libdcdg.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xchg.py -m gpu -q -x > gpurun_out/sigv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sigv_tests.log
