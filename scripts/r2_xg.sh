timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
BENCH_ONE_GPU=1 timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_g2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_g2.log
BENCH_ONE_GPU=1 timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --eager > gpurun_out/bench_g2e.log 2>&1; echo "rc=$?" >> gpurun_out/bench_g2e.log
