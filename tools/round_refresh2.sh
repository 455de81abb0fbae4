#!/bin/bash
# GPU box, end of round 2: F_exec counters, bench lines (ours + reference arm),
# the bench's ncu launch list, order sweep, launch lists + full captures of the
# three-pass kernels (p = 5, 6 at 64^3).
O=gpurun_out/r
mkdir -p $O
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
python tools/fexec.py C3 > $O/fexec_c3.log 2>&1; python tools/fexec.py C2 > $O/fexec_c2.log 2>&1
cp gpurun_out/C3_fexec.json gpurun_out/C2_fexec.json profiles/ 2>/dev/null
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
python tools/order_sweep.py > $O/order_sweep.txt 2>&1
for p in 5 6; do
  python tools/prof_asm.py 3,$p,64,3 > $O/plain_p$p.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file $O/launches_p$p.csv python tools/prof_asm.py 3,$p,64,3 > $O/ncu_p$p.log 2>&1
  python tools/launch_summary.py $O/launches_p$p.csv "python tools/prof_asm.py 3,$p,64,3" > $O/launches_p${p}_summary.txt
done
for k in asm3_xpass asm_ysweep "asm_sweep"; do
  ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$k -s 1 -c 1 \
      -f -o $O/full_${k}_p6 python tools/prof_asm.py 3,6,64,3 > $O/ncu_full_$k.log 2>&1
done
ls $O
