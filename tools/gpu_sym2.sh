mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_asm_sym.py -x -q 2>&1 | tail -2
python tools/time_c2.py orders 2>&1 | grep -v Warn
if [ "$1" = ncu ]; then
python tools/prof_asm.py C2 > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:asm2_sym -c 1 -o gpurun_out/sym2_c2 python tools/prof_asm.py C2 > gpurun_out/ncu_sym2.log 2>&1; tail -1 gpurun_out/ncu_sym2.log
fi
