# forward-elimination variance (DCDG_SIG_COLS=1) vs the sweep operator (vlib/sweepop): parity + timing
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_aux.py tests/test_gpu_gram.py tests/test_gpu_acceptance.py -m gpu -q -x > gpurun_out/cols_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cols_tests.log
for i in 1 2; do
python scripts/opt_bench.py >> gpurun_out/cols_bench.log 2>&1
DCDG_LIB_PATH=vlib/sweepop/libdcdg.so python scripts/opt_bench.py >> gpurun_out/cols_bench.log 2>&1
python scripts/pev_bench.py >> gpurun_out/cols_bench.log 2>&1
DCDG_LIB_PATH=vlib/sweepop/libdcdg.so python scripts/pev_bench.py >> gpurun_out/cols_bench.log 2>&1
done
