#!/bin/bash
# GPU box: sustained C4 (100 applies) A/B: production (128-byte promotion at C4) vs 256 bytes
for r in 1 2 3; do
python bench.py --workload C4 --no-cpu-baseline --no-assembly 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prod128', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
IGS_LIB_PATH=variants/promo256/libigs_b200.so python bench.py --workload C4 --no-cpu-baseline --no-assembly 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('var256 ', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done
