timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_aux.py tests/test_gpu_xchg.py tests/test_gpu_ref_parity.py tests/test_cpp_api.py -m gpu -q -x > gpurun_out/sb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sb_tests.log
for r in 1 2; do
python scripts/opt_bench.py > gpurun_out/opt_sb2_$r.log 2>&1
DCDG_LIB_PATH=vlib/sb1/libdcdg.so python scripts/opt_bench.py > gpurun_out/opt_sb1_$r.log 2>&1
done
python scripts/lab/opt_shapes.py > gpurun_out/opt_shapes_sb2.json 2>&1
DCDG_LIB_PATH=vlib/sb1/libdcdg.so python scripts/lab/opt_shapes.py > gpurun_out/opt_shapes_sb1.json 2>&1
python scripts/pev_bench.py > gpurun_out/pev_sb2.log 2>&1
