# forward elimination with the owner's pivot column left scaled (working tree) vs per-row selects (vlib/noscaled)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_acceptance.py tests/test_gpu_gram.py tests/test_gpu_aux.py -m gpu -q -x > gpurun_out/scaled_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/scaled_tests.log
rm -f gpurun_out/scaled_bench.log
for i in 1 2 3; do
python scripts/opt_bench.py >> gpurun_out/scaled_bench.log 2>&1
DCDG_LIB_PATH=vlib/noscaled/libdcdg.so python scripts/opt_bench.py >> gpurun_out/scaled_bench.log 2>&1
done
python scripts/pev_bench.py >> gpurun_out/scaled_bench.log 2>&1
DCDG_LIB_PATH=vlib/noscaled/libdcdg.so python scripts/pev_bench.py >> gpurun_out/scaled_bench.log 2>&1
