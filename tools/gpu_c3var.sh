for r in 1 2 3; do
python tools/time_c3.py base
for v in variants/*/; do IGS_LIB_PATH=$v/libigs_b200.so python tools/time_c3.py $v; done
done 2>&1 | grep -v Warn
for v in variants/*/; do IGS_LIB_PATH=$v/libigs_b200.so python -m pytest tests/test_asm_sym.py -x -q -k "not row_ranges" 2>&1 | tail -1; done
