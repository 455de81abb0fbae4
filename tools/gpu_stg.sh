for r in 1 2; do
for p in 3 5 7; do
for v in 0 31 32; do
 for k in 2 3; do IGS_APPLY_VARIANT=$v IGS_LIB_PATH=variants/stg/libigs_b200.so python tools/time_apply_p.py $p $k 2>&1 | grep -v Warn | sed "s/^/v$v /"; done
done; done; done
