import os, subprocess, sys
cases = [(5, 20, 5, 2), (5, 2, 3, 2), (5, 38, 1, 2)]
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads
p, K0, K1, kind = map(int, sys.argv[1:5])
prob = workloads.make_problem(2, p, [K0, K1], kind, seed=1) if False else None
from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots
from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule
bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in (K0, K1)]
quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
planes = workloads.synthetic_planes(2, list(quad.shape), kind, seed=3)
prob = sumfac.AssemblyProblem(bases, bases, quad, workloads.field_from_planes(2, kind, planes, quad.shape))
B = sumfac.assemble(prob, flags=8).values_np()
A = sumfac.assemble(prob).values_np()
torch.cuda.synchronize()
print("fused", sumfac.fused_path(prob), "rel", np.linalg.norm(A-B)/np.linalg.norm(B), "maxabs", np.abs(A-B).max())
'''
for c in cases:
    r = subprocess.run([sys.executable, "-c", code, *map(str, c)], capture_output=True, text=True,
                       env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"), timeout=300)
    print(c, r.returncode, r.stdout.strip()[-300:], r.stderr.strip()[-600:], flush=True)
