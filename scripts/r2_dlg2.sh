# downlink effective-gain placement variants (lab, scripts/kbench.py)
for v in base g2 g2m g0m; do
  for r in 1 2; do DCDG_LIB_PATH=vlib/$v/libdcdg.so python scripts/kbench.py > gpurun_out/kb_${v}_$r.log 2>&1; done
done
