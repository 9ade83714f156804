# ul_tmh_f32 also at 64x16 (G=16) and 16x16 (G=4) vs the register kernels there (vlib/nomore)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_abi.py tests/test_gpu_decisions.py -q -x > gpurun_out/more_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/more_tests.log
timeout 600 python scripts/sweep_configs4.py gpurun_out/c4_more.json 16 > /dev/null 2>&1
DCDG_LIB_PATH=vlib/nomore/libdcdg.so timeout 600 python scripts/sweep_configs4.py gpurun_out/c4_nomore.json 16 > /dev/null 2>&1
timeout 600 python scripts/sweep_configs4.py gpurun_out/c4_more2.json 16 > /dev/null 2>&1
