# ul_tmh_f32 with 3 of the 4 odd blocks in TMEM (vlib/ntm3) vs 4 (default)
DCDG_LIB_PATH=vlib/ntm3/libdcdg.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uplink" > gpurun_out/ntm_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ntm_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uplink" >> gpurun_out/ntm_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ntm_tests.log
rm -f gpurun_out/ntm_bench.log
for i in 1 2 3; do
timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/ntm_bench.log 2>&1
DCDG_LIB_PATH=vlib/ntm3/libdcdg.so timeout 300 python scripts/kbench.py 16800 40 >> gpurun_out/ntm_bench.log 2>&1
done
