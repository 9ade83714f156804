timeout 600 python -m pytest tests/test_cpp_api.py -m gpu -q > gpurun_out/zc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zc_tests.log
for v in main; do
  if [ $v = main ]; then LIBD=$PWD/paper_1902_08653_b200; else LIBD=$PWD/vlib/$v; fi
  g++ -std=c++20 -O2 -pthread -I include -I /usr/local/cuda/include tests/cpp/bench_cpp_api.cpp -o /tmp/bench_cpp_$v \
    -L $LIBD -ldcdg -Wl,-rpath,$LIBD oracle/libdcdoracle.so -Wl,-rpath,$PWD/oracle -L /usr/local/cuda/lib64 -lcudart -ldl
  timeout 600 /tmp/bench_cpp_$v > gpurun_out/cpp_bench_$v.json 2> gpurun_out/cpp_bench_$v.err
done
