for r in 1 2 3; do
for c in C4 C5; do
for v in variants/*/ new; do
 if [ $v = new ]; then python tools/time_apply.py $c | sed "s/^/new /"; else IGS_LIB_PATH=$v/libigs_b200.so python tools/time_apply.py $c | sed "s|^|$v |"; fi
done; done; done 2>&1 | grep -v Warn | cut -c1-52
timeout 1500 python -m pytest tests -q -m gpu -x -k "apply or operator or full_size or smoke or sharded or parity or localized or geometry" 2>&1 | tail -1
