g++ -std=c++20 -O2 -pthread -I include -I /usr/local/cuda/include tests/cpp/bench_cpp_api.cpp -o /tmp/bench_cpp_api \
  -L paper_1902_08653_b200 -ldcdg -Wl,-rpath,$PWD/paper_1902_08653_b200 oracle/libdcdoracle.so -Wl,-rpath,$PWD/oracle \
  -L /usr/local/cuda/lib64 -lcudart -ldl && timeout 600 /tmp/bench_cpp_api > gpurun_out/cpp_bench.json 2> gpurun_out/cpp_bench.err
timeout 900 python scripts/acceptance_gpu.py gpurun_out/acceptance_gpu.json > gpurun_out/acceptance.log 2>&1
timeout 900 python scripts/sweep_configs4.py gpurun_out/configs4_sweep.json > gpurun_out/configs4.log 2>&1
