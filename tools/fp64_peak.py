"""Measure the fp64 roofline denominators on this B200 and record them with
the SM clocks seen while they ran: profiles/fp64_peak.json (read by bench.py).

DMMA (mma.sync m8n8k4 f64) burst and sustained (back to back for ~4 s),
DFMA burst, and the plain copy bandwidth (tools/fp64_peak.cu)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from bench import ClockSampler  # noqa: E402

exe = "/tmp/igs_fp64_peak"
subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                os.path.join(REPO, "tools", "fp64_peak.cu")], check=True)
with ClockSampler(0) as clk_b:
    burst = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
with ClockSampler(0) as clk_s:
    sust = subprocess.run([exe, "sustained"], capture_output=True, text=True, check=True).stdout
lines = [json.loads(x) for x in (burst + sust).splitlines() if x.startswith("{")]
dmma = [x["dmma_tflops"] for x in lines if "dmma_tflops" in x]
dfma = [x["dfma_tflops"] for x in lines if "dfma_tflops" in x]
copy = [x["copy_gbs"] for x in lines if "copy_gbs" in x]
sus = [x["dmma_tflops_sustained"] for x in lines if "dmma_tflops_sustained" in x]
out = {"dmma_tflops_burst": max(dmma), "dmma_tflops_sustained": sus[0], "dfma_tflops_burst": max(dfma),
       "copy_gbs": max(copy), "device": lines[0], "clocks_burst": clk_b.summary(), "clocks_sustained": clk_s.summary(),
       "how": "tools/fp64_peak.cu: 592 CTAs x 8 warps, 4 independent m8n8k4 f64 chains per warp (DMMA), 8 DFMA "
              "chains per thread; best of 3 (burst) and 480 launches back to back (sustained); CUDA events"}
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
with open(os.path.join(REPO, "gpurun_out", "fp64_peak.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
