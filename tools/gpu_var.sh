mkdir -p gpurun_out
python -m pytest tests/test_asm_sym.py -x -q 2>&1 | tail -2
for r in 1 2; do
python tools/time_c3.py base
for v in variants/*/; do [ -f $v/libigs_b200.so ] && IGS_LIB_PATH=$v/libigs_b200.so python tools/time_c3.py $v; done
done 2>&1 | tee gpurun_out/variants.txt
