for r in 1 2; do
for v in 0 21 22 23; do
for c in C4 C5; do IGS_APPLY_VARIANT=$v IGS_LIB_PATH=variants/hip/libigs_b200.so python tools/time_apply.py $c 2>&1 | grep -v Warn | sed "s/^/v$v /" | cut -c1-60; done
done; done
