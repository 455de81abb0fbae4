#!/bin/bash
# GPU box: three-pass checks + timing, then the p = 6 launch list.
O=gpurun_out/tp
mkdir -p $O
python tools/three_pass_check.py 2>&1 | tail -14
for p in ${1:-6}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file $O/launches_p$p.csv python tools/prof_asm.py 3,$p,64,3 > $O/ncu_p$p.log 2>&1
  python tools/launch_summary.py $O/launches_p$p.csv "python tools/prof_asm.py 3,$p,64,3" | head -5 | tee $O/launches_p${p}_summary.txt
done
