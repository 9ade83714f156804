timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pev_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pev_tests.log
python scripts/lab/opt_shapes.py > gpurun_out/opt_shapes.json 2>&1
python scripts/pev_bench.py > gpurun_out/pev_bench.log 2>&1
