#!/bin/bash
# GPU box: ncu launch lists of the fused apply at low orders
O=gpurun_out/ap; mkdir -p $O
for p in 2 3 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 8 --csv --log-file $O/ap_p$p.csv python tools/time_apply_p.py $p 2 > $O/ap_p$p.log 2>&1
  python tools/launch_summary.py $O/ap_p$p.csv "time_apply_p $p" | head -5
done
