mkdir -p gpurun_out
nproc > gpurun_out/host.txt
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/gpu_tests.txt 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -20 gpurun_out/gpu_tests.txt; tail -c 2500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
