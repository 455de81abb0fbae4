#!/bin/bash
# GPU box: tile-shape variants of the headline applies (measurement build variants/apv)
L=variants/apv/libigs_b200.so
for pk in "6 2" "8 3"; do
  set -- $pk
  echo "base: $(python tools/time_apply_p.py $1 $2)"
  for v in 20 21 22 23 24 25; do
    out=$(IGS_LIB_PATH=$L IGS_APPLY_VARIANT=$v python tools/time_apply_p.py $1 $2 2>&1 | tail -1)
    echo "v$v: $out"
  done
done
