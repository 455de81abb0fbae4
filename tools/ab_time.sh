#!/bin/bash
# A/B timing on one box: builds HEAD (A) and the working tree (B) into
# gpurun_out-independent paths, then alternates their timings.
#   tools/ab_time.sh prepare      (here)   -> ab/libA.so, ab/libB.so
#   tools/ab_time.sh run C4 C5    (on the box)
set -e
cd "$(dirname "$0")/.."
if [ "$1" = prepare ]; then
  mkdir -p ab
  python paper_1809_05471_b200/build.py > /dev/null 2>&1
  cp paper_1809_05471_b200/libigs_b200.so ab/libB.so
  git stash -q
  python paper_1809_05471_b200/build.py > /dev/null 2>&1
  cp paper_1809_05471_b200/libigs_b200.so ab/libA.so
  git stash pop -q
  python paper_1809_05471_b200/build.py > /dev/null 2>&1
  ls -la ab
  exit 0
fi
shift
for r in 1 2 3; do
  for v in A B; do
    echo "== $v"
    IGS_LIB_PATH=ab/lib$v.so python tools/time_apply.py "$@" 2>/dev/null | grep -E "ms/apply|assemble"
  done
done
