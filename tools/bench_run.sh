mkdir -p gpurun_out
python tools/fexec.py C3 > gpurun_out/fexec_c3.log 2>&1
python tools/fexec.py C2 > gpurun_out/fexec_c2.log 2>&1
cp gpurun_out/C3_fexec.json gpurun_out/C2_fexec.json profiles/ 2>/dev/null
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
