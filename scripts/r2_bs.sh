for r in 1 2; do
python scripts/kbench.py > gpurun_out/kb_bs0_$r.log 2>&1
DCDG_LIB_PATH=vlib/bs2/libdcdg.so python scripts/kbench.py > gpurun_out/kb_bs2_$r.log 2>&1
done
DCDG_LIB_PATH=vlib/bs2/libdcdg.so timeout 600 python scripts/sweep_configs4.py - 16 > gpurun_out/u16_bs2.log 2>&1
timeout 600 python scripts/sweep_configs4.py - 16 > gpurun_out/u16_bs0.log 2>&1
DCDG_LIB_PATH=vlib/bs2/libdcdg.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xchg.py -m gpu -q -x > gpurun_out/bs2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bs2_tests.log
