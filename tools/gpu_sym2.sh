mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_asm_sym.py -x -q > gpurun_out/sym2_tests.txt 2>&1
tail -25 gpurun_out/sym2_tests.txt
timeout 600 python tools/time_c2.py > gpurun_out/time_c2.txt 2>&1; tail -30 gpurun_out/time_c2.txt
