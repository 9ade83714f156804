DCDG_LIB_PATH=vlib/tm1/libdcdg.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uplink_fp32 and uniform" > gpurun_out/tm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tm_tests.log
for r in 1 2; do
DCDG_LIB_PATH=vlib/tm1/libdcdg.so python scripts/kbench.py > gpurun_out/kb_tm1_$r.log 2>&1
python scripts/kbench.py > gpurun_out/kb_tm0_$r.log 2>&1
done
