#!/bin/bash
# GPU box: compute-sanitizer memcheck / synccheck / racecheck / initcheck over
# tools/sanitize.py; logs into gpurun_out/san/ (summaries go to profiles/).
O=gpurun_out/san
mkdir -p $O
python tools/sanitize.py all > $O/plain.log 2>&1 || { tail -20 $O/plain.log; exit 1; }
for tool in memcheck synccheck racecheck initcheck; do
  for w in apply asm; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --log-file $O/${tool}_$w.log \
        python tools/sanitize.py $w > $O/${tool}_$w.out 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${tool}_$w.log | tail -1)"
  done
done
