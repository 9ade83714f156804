# fused variance on the TMEM half-tile kernel (working tree) vs ul_reg_f32<...,SIG> (vlib/nosig_tm)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_acceptance.py tests/test_gpu_aux.py tests/test_cpp_api.py -m gpu -q -x > gpurun_out/tmsig_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tmsig_tests.log
rm -f gpurun_out/tmsig_bench.log
for i in 1 2 3; do
python scripts/opt_bench.py >> gpurun_out/tmsig_bench.log 2>&1
DCDG_LIB_PATH=vlib/nosig_tm/libdcdg.so python scripts/opt_bench.py >> gpurun_out/tmsig_bench.log 2>&1
done
