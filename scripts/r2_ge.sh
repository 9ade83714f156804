DCDG_LIB_PATH=vlib/ge1/libdcdg.so python scripts/kbench.py > gpurun_out/kb_ge1.log 2>&1
python scripts/kbench.py > gpurun_out/kb_ge0.log 2>&1
DCDG_LIB_PATH=vlib/ge1/libdcdg.so python scripts/kbench.py > gpurun_out/kb_ge1b.log 2>&1
python scripts/kbench.py > gpurun_out/kb_ge0b.log 2>&1
