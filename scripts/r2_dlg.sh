DCDG_LIB_PATH=vlib/base/libdcdg.so python scripts/kbench.py > gpurun_out/kbench_base.log 2>&1
python scripts/kbench.py > gpurun_out/kbench_new.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_aux.py tests/test_gpu_xchg.py tests/test_cpp_api.py -m gpu -q -x > gpurun_out/dlg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dlg_tests.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_dlg.log 2>&1
