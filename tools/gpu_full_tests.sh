mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 3000 python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/gpu_tests.txt 2>&1
tail -45 gpurun_out/gpu_tests.txt
