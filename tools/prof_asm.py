import sys, torch
sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads
name = sys.argv[1]
c = workloads.CONFIGS[name]
prob = workloads.make_problem(c["d"], c["p"], c["K"], c["kind"])
A = sumfac.assemble(prob)
torch.cuda.synchronize()
A = sumfac.assemble(prob)
torch.cuda.synchronize()
print("ok", A.nnz)
