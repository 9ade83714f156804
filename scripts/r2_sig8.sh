timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xchg.py tests/test_gpu_ref_parity.py tests/test_cpp_api.py tests/test_gpu_acceptance.py -m gpu -q -x > gpurun_out/sig8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sig8_tests.log
python scripts/lab/opt_shapes.py > gpurun_out/opt_shapes.json 2>&1
