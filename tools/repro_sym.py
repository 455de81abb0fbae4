"""One symmetric fused assembly on a small mesh (sanitizer / debugging aid):
python tools/repro_sym.py p K0 K1 K2 kind"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads  # noqa: E402
from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots  # noqa: E402
from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule  # noqa: E402

p, K, kind = int(sys.argv[1]), [int(v) for v in sys.argv[2:5]], int(sys.argv[5])
bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=51)
prob = sumfac.AssemblyProblem(bases, bases, quad, workloads.field_from_planes(3, kind, planes, quad.shape))
A = sumfac.assemble(prob)
B = sumfac.assemble(prob, flags=8)
torch.cuda.synchronize()
va, vb = A.values_np(), B.values_np()
print("fused", sumfac.fused_path(prob), "rel", np.linalg.norm(va - vb) / np.linalg.norm(vb))
