timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_aux.py tests/test_gpu_gram.py tests/test_cpp_api.py -m gpu -q -x > gpurun_out/pev_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pev_tests.log
python scripts/pev_bench.py > gpurun_out/pev_bench.log 2>&1
python scripts/lab/opt_shapes.py > gpurun_out/opt_shapes.json 2>&1
