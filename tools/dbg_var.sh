for v in base variants/s2e1 variants/s2e2 variants/s2e3; do
  if [ $v = base ]; then L=""; else L="IGS_LIB_PATH=$v/libigs_b200.so"; fi
  echo "== $v"; env $L python tools/dbg_sym2.py 2>&1 | grep -E "^\(" | cut -c1-160
done
