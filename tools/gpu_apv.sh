#!/bin/bash
# GPU box: low-order apply tile-shape variants (measurement build variants/apv)
L=variants/apv/libigs_b200.so
for p in 2 3 4 5; do
  for kind in 2 3; do
    echo "base: $(python tools/time_apply_p.py $p $kind)"
    for v in 10 11 12 13; do
      out=$(IGS_LIB_PATH=$L IGS_APPLY_VARIANT=$v python tools/time_apply_p.py $p $kind 2>&1 | tail -1)
      echo "v$v: $out"
    done
  done
done
