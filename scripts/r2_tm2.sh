DCDG_LIB_PATH=vlib/tm2/libdcdg.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uplink_fp32 and uniform or persistent" > gpurun_out/tm2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tm2_tests.log
for r in 1 2; do
DCDG_LIB_PATH=vlib/tm2/libdcdg.so timeout 300 python scripts/kbench.py > gpurun_out/kb_tm2_$r.log 2>&1
done
