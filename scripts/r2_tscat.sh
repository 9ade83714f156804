# ul_tmh_f32 block reduction: reduce-scatter + smem broadcast (vlib/tscat) vs butterfly (default)
DCDG_LIB_PATH=vlib/tscat/libdcdg.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uplink" > gpurun_out/tscat_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tscat_tests.log
rm -f gpurun_out/tscat_bench.log
for i in 1 2 3; do
timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/tscat_bench.log 2>&1
DCDG_LIB_PATH=vlib/tscat/libdcdg.so timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/tscat_bench.log 2>&1
done
