# uplink: last block of the last sweep without the (dead) residual update vs vlib/noskip
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_xchg.py -m gpu -q -x > gpurun_out/skip_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/skip_tests.log
rm -f gpurun_out/skip_bench.log
for i in 1 2 3; do
timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/skip_bench.log 2>&1
DCDG_LIB_PATH=vlib/noskip/libdcdg.so timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/skip_bench.log 2>&1
done
python scripts/opt_bench.py >> gpurun_out/skip_bench.log 2>&1
DCDG_LIB_PATH=vlib/noskip/libdcdg.so python scripts/opt_bench.py >> gpurun_out/skip_bench.log 2>&1
