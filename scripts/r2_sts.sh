# fused-variance pivot-column stores: st.shared.v2 (default) vs two st.shared.f32 (vlib/sts32)
rm -f gpurun_out/sts_bench.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "optimal or uplink" > gpurun_out/sts_tests.log 2>&1
for i in 1 2 3; do
python scripts/opt_bench.py >> gpurun_out/sts_bench.log 2>&1
DCDG_LIB_PATH=vlib/sts32/libdcdg.so python scripts/opt_bench.py >> gpurun_out/sts_bench.log 2>&1
done
