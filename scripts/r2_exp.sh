# fused-variance scale from exponent bits (working tree) vs HEAD (vlib/head)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_acceptance.py -m gpu -q -x > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
rm -f gpurun_out/exp_bench.log
for i in 1 2 3; do
python scripts/opt_bench.py >> gpurun_out/exp_bench.log 2>&1
DCDG_LIB_PATH=vlib/head/libdcdg.so python scripts/opt_bench.py >> gpurun_out/exp_bench.log 2>&1
done
