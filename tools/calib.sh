mkdir -p gpurun_out
python tools/fp64_peak.py > gpurun_out/fp64_peak.log 2>&1
python tools/fexec.py C3 > gpurun_out/fexec_c3.log 2>&1
python tools/fexec.py C2 > gpurun_out/fexec_c2.log 2>&1
tail -2 gpurun_out/fp64_peak.log gpurun_out/fexec_c3.log gpurun_out/fexec_c2.log
