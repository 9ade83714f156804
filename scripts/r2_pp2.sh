# two problems per 16-lane group (ul_pp2_f32) vs ul_reg_f32 (vlib/base): parity + kernel timing
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_decisions.py -m gpu -q -x > gpurun_out/pp2_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pp2_tests.log
rm -f gpurun_out/pp2_bench.log
for i in 1 2; do
timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/pp2_bench.log 2>&1
DCDG_LIB_PATH=vlib/base/libdcdg.so timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/pp2_bench.log 2>&1
DCDG_LIB_PATH=vlib/pp2split/libdcdg.so timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/pp2_bench.log 2>&1
done
