mkdir -p gpurun_out

python -m pytest tests/test_asm_sym.py -x -q 2>&1 | tail -15 > gpurun_out/sym_tests.txt
python tools/time_asm.py > gpurun_out/time_asm.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:asm3_sym -c 1 -o gpurun_out/sym_c3i python tools/prof_asm.py C3 > gpurun_out/ncu_sym.log 2>&1
head -40 gpurun_out/san_p3.txt; cat gpurun_out/sym_tests.txt gpurun_out/time_asm.txt
