#!/bin/bash
# GPU box: one full capture of a kernel ($1 = regex, $2 = p) of the 64^3 M+K assembly
O=gpurun_out/tp
mkdir -p $O
p=${2:-6}
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$1 -s 1 -c 1 \
    -f -o $O/full_$1_p$p python tools/prof_asm.py 3,$p,64,3 > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
