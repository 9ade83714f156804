timeout 600 python -m pytest tests/test_cpp_api.py -m gpu -q > gpurun_out/cpp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cpp_tests.log
g++ -std=c++20 -O2 -pthread -I include -I /usr/local/cuda/include tests/cpp/bench_cpp_api.cpp -o /tmp/bench_cpp_api \
  -L paper_1902_08653_b200 -ldcdg -Wl,-rpath,$PWD/paper_1902_08653_b200 oracle/libdcdoracle.so -Wl,-rpath,$PWD/oracle \
  -L /usr/local/cuda/lib64 -lcudart -ldl && timeout 600 /tmp/bench_cpp_api > gpurun_out/cpp_bench.json 2> gpurun_out/cpp_bench.err
