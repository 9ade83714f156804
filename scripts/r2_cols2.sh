# forward-elimination variance in all three variance sites (+ approximate reciprocal) vs the sweep operators (vlib/sweepop)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_aux.py tests/test_gpu_gram.py tests/test_gpu_acceptance.py tests/test_gpu_xchg.py -m gpu -q -x > gpurun_out/cols_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cols_tests.log
rm -f gpurun_out/cols_bench.log
for i in 1 2; do
python scripts/opt_bench.py >> gpurun_out/cols_bench.log 2>&1
DCDG_LIB_PATH=vlib/sweepop/libdcdg.so python scripts/opt_bench.py >> gpurun_out/cols_bench.log 2>&1
python scripts/pev_bench.py >> gpurun_out/cols_bench.log 2>&1
DCDG_LIB_PATH=vlib/sweepop/libdcdg.so python scripts/pev_bench.py >> gpurun_out/cols_bench.log 2>&1
done
