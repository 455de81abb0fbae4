#!/bin/bash
# GPU box: ncu launch lists of one warm 64^3 M+K assembly for the orders given
O=gpurun_out/tp
mkdir -p $O
for p in "$@"; do
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file $O/launches_p$p.csv python tools/prof_asm.py 3,$p,64,3 > $O/ncu_p$p.log 2>&1
  python tools/launch_summary.py $O/launches_p$p.csv "python tools/prof_asm.py 3,$p,64,3" > $O/launches_p${p}_summary.txt
  head -6 $O/launches_p${p}_summary.txt
done
