# multi-rank bench self-test on the one leased GPU (ranks share cuda:0; p2p windows over CUDA IPC)
BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/multi2.log 2>&1; echo "rc=$?" >> gpurun_out/multi2.log
BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu --fast > gpurun_out/multi4.log 2>&1; echo "rc=$?" >> gpurun_out/multi4.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/ref_small.log 2>&1; echo "rc=$?" >> gpurun_out/ref_small.log
