g++ -std=c++20 -O2 -I include -I /usr/local/cuda/include scripts/lab/call_latency.cpp -o /tmp/call_latency -L paper_1902_08653_b200 -ldcdg -Wl,-rpath,$PWD/paper_1902_08653_b200 -L /usr/local/cuda/lib64 -lcudart && /tmp/call_latency > gpurun_out/call_latency.json 2>&1
nproc >> gpurun_out/call_latency.json; lscpu | grep -i "model name\|mhz" >> gpurun_out/call_latency.json
