for r in 1 2; do
for v in lb4s lb2s lb4; do DCDG_LIB_PATH=vlib/$v/libdcdg.so python scripts/kbench.py > gpurun_out/kb_${v}_$r.log 2>&1; done
python scripts/kbench.py > gpurun_out/kb_base_$r.log 2>&1
done
