timeout 900 python -m pytest tests/test_asm_sym.py -x -q 2>&1 | tail -2
for r in 1 2 3; do python tools/time_c3.py new; done
