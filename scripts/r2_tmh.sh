# odd coordinate blocks in TMEM at 8 lanes per problem, 3 warps per scheduler (vlib/tmh) vs ul_reg_f32 (default)
DCDG_LIB_PATH=vlib/tmh/libdcdg.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uplink" > gpurun_out/tmh_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tmh_tests.log
rm -f gpurun_out/tmh_bench.log
for i in 1 2; do
timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/tmh_bench.log 2>&1
DCDG_LIB_PATH=vlib/tmh/libdcdg.so timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/tmh_bench.log 2>&1
done
