timeout 900 python -m pytest tests/test_asm_sym.py -x -q 2>&1 | tail -1
for r in 1 2 3; do python tools/time_c3.py new; IGS_LIB_PATH=variants/prev/libigs_b200.so python tools/time_c3.py prev; done 2>&1 | grep -v Warn
