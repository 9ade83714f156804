timeout 120 python -X faulthandler scripts/lab/clock_sampler_check.py > gpurun_out/cs.log 2>&1
timeout 600 python -X faulthandler bench.py --no-cpu --fast > gpurun_out/bench_graph.log 2>&1
