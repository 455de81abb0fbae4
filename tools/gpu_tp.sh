#!/bin/bash
# GPU box: three-pass tests, then the ncu launch lists of one warm p = 5 / p = 6 assembly at 64^3.
O=gpurun_out/tp
mkdir -p $O
python -m pytest tests/test_three_pass.py -q -m gpu -x 2>&1 | tail -5
for p in 5 6; do
  python tools/prof_asm.py 3,$p,64,3 > $O/plain_p$p.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file $O/launches_p$p.csv python tools/prof_asm.py 3,$p,64,3 > $O/ncu_p$p.log 2>&1
  python tools/launch_summary.py $O/launches_p$p.csv "python tools/prof_asm.py 3,$p,64,3" | tee $O/launches_p${p}_summary.txt
done
