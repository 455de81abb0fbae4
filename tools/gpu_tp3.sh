#!/bin/bash
# GPU box: timing + launch list + one full capture of a kernel ($1 = regex, $2 = p)
O=gpurun_out/tp
mkdir -p $O
p=${2:-6}
python tools/three_pass_check.py time 2>&1 | tail -5
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/launches_p$p.csv python tools/prof_asm.py 3,$p,64,3 > $O/ncu_p$p.log 2>&1
python tools/launch_summary.py $O/launches_p$p.csv "python tools/prof_asm.py 3,$p,64,3" | head -5 | tee $O/launches_p${p}_summary.txt
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$1 -s 1 -c 1 \
    -f -o $O/full_$1_p$p python tools/prof_asm.py 3,$p,64,3 > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
