#!/bin/bash
# Runs on the GPU box: bench lines, ncu launch list and full captures of the
# hot kernels into gpurun_out/prof/ (summarised into profiles/ afterwards).
set -x
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --workload C5 --no-cpu-baseline --no-assembly > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_c4.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:apply3d_kernel -s 2 -c 1 \
    -o $O/prof_c4 python tools/time_apply.py C4 > $O/ncu_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:apply3d_kernel -s 2 -c 1 \
    -o $O/prof_c5 python tools/time_apply.py C5 > $O/ncu_c5.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:asm3_stage12|asm_sweep" -s 2 -c 2 \
    -o $O/prof_asm_c3 python tools/prof_asm.py C3 > $O/ncu_asm.log 2>&1
python tools/f1_time.py 128 > $O/f1_c4_grid.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:geom_line_kernel -s 1 -c 1 \
    -o $O/prof_f1 python tools/f1_time.py 64 > $O/ncu_f1.log 2>&1
ls -la $O
