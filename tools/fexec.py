"""Executed fp64 work of the assembly kernels from ncu counters (SURVEY
§8(d): F_exec from DFMA / DADD / DMUL / DMMA counts), per assembly, written
to gpurun_out/<cfg>_fexec.json (copied to profiles/ and read by bench.py).

    python tools/fexec.py C3     (runs ncu on tools/prof_asm.py C3)"""

import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1]
metrics = ["sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
           "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "sm__ops_path_tensor_src_fp64.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__time_duration.sum"]
# the second assemble() call in prof_asm.py is the warm one: profile every
# launch of the package's kernels in it
cmd = ["ncu", "--profile-from-start", "off", "--metrics", ",".join(metrics), "--clock-control", "none", "--csv",
       "--print-units", "base", "python", os.path.join(REPO, "tools", "prof_asm.py"), cfg]
out = subprocess.run(cmd, capture_output=True, text=True, cwd=REPO).stdout
rows = list(csv.reader(io.StringIO(out[out.index('"ID"'):])))
hdr = rows[0]
iK, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iID = hdr.index("ID")
per = {}
for r in rows[1:]:
    if len(r) <= iV:
        continue
    per.setdefault(int(r[iID]), {"kernel": r[iK]})[r[iM]] = float(r[iV].replace(",", ""))
launches = [per[k] for k in sorted(per)]
# only the warm call is profiled (prof_asm.py brackets it with the profiler API);
# torch's own allocation kernels are not assembly work
warm = [x for x in launches if "cub" not in x["kernel"] and "elementwise" not in x["kernel"]]
dmma = sum(x.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0) for x in warm)
dfma = sum(x.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) for x in warm)
dadd = sum(x.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0) for x in warm)
dmul = sum(x.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) for x in warm)
res = {"config": cfg, "kernels": [x["kernel"][:80] for x in warm],
       "dmma_warp_inst": dmma, "dfma_thread_inst": dfma, "dadd_thread_inst": dadd, "dmul_thread_inst": dmul,
       "tensor_fp64_ops": sum(x.get("sm__ops_path_tensor_src_fp64.sum", 0) for x in warm),
       "exec_flops": 512.0 * dmma + 2.0 * dfma + dadd + dmul,
       "dram_bytes": sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in warm),
       "ncu_ms": sum(x.get("gpu__time_duration.sum", 0) for x in warm) / 1e6,
       "how": "ncu --metrics (DMMA warp instructions x 512 flop + 2 x DFMA + DADD + DMUL thread instructions) "
              "over the warm assemble() launches of tools/prof_asm.py"}
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
with open(os.path.join(REPO, "gpurun_out", f"{cfg}_fexec.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
