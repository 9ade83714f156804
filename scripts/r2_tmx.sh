# exchange (p2p window) instantiation on the TMEM uplink kernel: exchange suite, parity, multi-rank bench self-test
timeout 900 python -m pytest tests/test_gpu_xchg.py tests/test_gpu_parity.py tests/test_gpu_aux.py tests/test_abi.py -q -x > gpurun_out/tmx_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tmx_tests.log
BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --fast > gpurun_out/tmx_multi2.log 2>&1; echo "rc=$?" >> gpurun_out/tmx_multi2.log
