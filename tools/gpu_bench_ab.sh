for r in 1 2 3; do
for v in variants/*/ new; do
 if [ $v = new ]; then L=""; else L="IGS_LIB_PATH=$v/libigs_b200.so"; fi
 env $L python bench.py --no-assembly --no-c5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,1), d['ms_per_step'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
