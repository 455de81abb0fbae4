#!/bin/bash
# GPU box: sustained C5 (50 applies) with the 8-row single-stage variant vs the production tile
L=variants/apv/libigs_b200.so
for r in 1 2; do
python bench.py --workload C5 --no-cpu-baseline --no-assembly 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['clocks'])"
IGS_LIB_PATH=$L IGS_APPLY_VARIANT=21 python bench.py --workload C5 --no-cpu-baseline --no-assembly 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('v21 ', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['clocks'])"
done
