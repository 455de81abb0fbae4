for r in 1 2; do
python tools/time_c2.py c2 base
for v in variants/t*/; do IGS_LIB_PATH=$v/libigs_b200.so python tools/time_c2.py c2 $v; done
done 2>&1 | grep -v Warn
