#!/bin/bash
# GPU box: L2 promotion variants of the assembly kernels' tensor maps
cat > /tmp/t.py <<'PY'
import sys, json
sys.path.insert(0, ".")
from tools.time_asm import run
for c in [(3, 4, 64, 3, 0), (2, 5, 256, 2, 0), (3, 6, 64, 3, 0), (3, 5, 64, 3, 0), (3, 3, 64, 3, 0), (3, 2, 64, 3, 0)]:
    r = run(*c, reps=10); print(r["d"], r["p"], r["K"], round(r["ms"], 4))
PY
for v in base apromo128 apromo0; do
  echo "== $v"
  if [ $v = base ]; then python /tmp/t.py; else IGS_LIB_PATH=variants/$v/libigs_b200.so python /tmp/t.py; fi
done
