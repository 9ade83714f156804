#!/bin/bash
# One GPU session of the round-end evidence (run under gpurun from the repo root):
# tests, smoke, bench, the bench's ncu launch list, and full ncu captures of the
# hot kernels summarised on the box (the .ncu-rep files are too large to return).
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --fast > gpurun_out/b_ncu.log 2>&1
bash scripts/ncu_captures.sh
for f in /tmp/reps/*.ncu-rep; do
  ncu -i $f --page source --csv --print-source sass > /tmp/reps/$(basename $f .ncu-rep).src.csv 2>/dev/null
  python scripts/stall_summary.py /tmp/reps/$(basename $f .ncu-rep).src.csv > gpurun_out/stalls_$(basename $f .ncu-rep).txt 2>&1
done
