# downlink register kernel at 12 warps/SM in 4-warp CTAs (vlib/dl12) vs 1-warp CTAs at 10 (default)
DCDG_LIB_PATH=vlib/dl12/libdcdg.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "downlink" > gpurun_out/dl12_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/dl12_tests.log
rm -f gpurun_out/dl12_bench.log
for i in 1 2; do
timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/dl12_bench.log 2>&1
DCDG_LIB_PATH=vlib/dl12/libdcdg.so timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/dl12_bench.log 2>&1
done
