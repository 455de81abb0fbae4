#!/bin/bash
# GPU box: tests, F_exec counters, bench lines (ours + reference arm), the
# bench's ncu launch list and full captures of the assembly kernels.
O=gpurun_out/r
mkdir -p $O
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
timeout 2400 python -m pytest tests -q -m gpu -x > $O/gpu_tests.txt 2>&1; tail -2 $O/gpu_tests.txt
python tools/fexec.py C3 > $O/fexec_c3.log 2>&1; python tools/fexec.py C2 > $O/fexec_c2.log 2>&1
cp gpurun_out/C3_fexec.json gpurun_out/C2_fexec.json profiles/ 2>/dev/null
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
python tools/prof_asm.py C2 > $O/plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:asm2_sym -c 1 \
    -o $O/sym2_c2 python tools/prof_asm.py C2 > $O/ncu_sym2.log 2>&1
python tools/prof_asm.py C3 > $O/plain3.log 2>&1 && \
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:asm3_sym -c 1 \
    -o $O/sym3_c3 python tools/prof_asm.py C3 > $O/ncu_sym3.log 2>&1
ls $O
