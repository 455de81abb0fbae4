"""One cold and one warm assembly of a BASELINE config (profiling target);
the warm call is bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off` sees only its launches."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads  # noqa: E402

name = sys.argv[1]
if "," in name:  # "d,p,K,kind"
    d_, p_, K_, kind_ = (int(v) for v in name.split(","))
    c = {"d": d_, "p": p_, "K": K_, "kind": kind_}
else:
    c = workloads.CONFIGS[name]
prob = workloads.make_problem(c["d"], c["p"], c["K"], c["kind"])
A = sumfac.assemble(prob)
torch.cuda.synchronize()
torch.cuda.profiler.start()
A = sumfac.assemble(prob)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", A.nnz)
