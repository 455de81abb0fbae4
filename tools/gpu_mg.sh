mkdir -p gpurun_out
python -m pytest tests/test_sharded_capi.py tests/test_gpu_properties.py -x -q 2>&1 | tail -15 > gpurun_out/mg_tests.txt
cat gpurun_out/mg_tests.txt
