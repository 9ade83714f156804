DCDG_LIB_PATH=vlib/gl1/libdcdg.so timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py -m gpu -q -x -k "gram or fp16" > gpurun_out/gl1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gl1_tests.log
for r in 1 2; do
python scripts/kbench.py > gpurun_out/kb_gl0_$r.log 2>&1
DCDG_LIB_PATH=vlib/gl1/libdcdg.so python scripts/kbench.py > gpurun_out/kb_gl1_$r.log 2>&1
done
DCDG_LIB_PATH=vlib/gl1/libdcdg.so python scripts/opt_bench.py > gpurun_out/opt_gl1.log 2>&1
