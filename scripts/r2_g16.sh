# 16x16 tile: lanes per problem 4 (base) vs 8 (lab)
for v in base g8; do for r in 1 2; do
  DCDG_LIB_PATH=vlib/$v/libdcdg.so python scripts/sweep_configs4.py gpurun_out/c4_${v}_$r.json 16 > /dev/null 2>&1
done; done
