mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_asm_sym.py -x -q > gpurun_out/sym2_tests.txt 2>&1
tail -3 gpurun_out/sym2_tests.txt
timeout 600 python tools/time_c2.py > gpurun_out/time_c2.txt 2>&1; tail -30 gpurun_out/time_c2.txt | cut -c1-200
if [ "$1" = ncu ]; then
python tools/prof_asm.py C2 > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:asm2_sym -s 1 -c 1 -o gpurun_out/sym2_c2 python tools/prof_asm.py C2 > gpurun_out/ncu_sym2.log 2>&1; tail -2 gpurun_out/ncu_sym2.log
fi
