"""Device timing of the fused apply at order p, 128^3, stiffness (kind 2) or
M+K (kind 3): python tools/time_apply_p.py p [kind] (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import matfree, workloads  # noqa: E402

p = int(sys.argv[1])
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = workloads.make_problem(3, p, 128, kind)
op = matfree.MatrixFreeOperator(prob)
n = prob.shape[1]
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    op.apply_device(x, y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    op.apply_device(x, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
balg = 8 * prob.coeff.n_planes * prob.quad.num_points + 16 * n
print(f"p={p} kind={kind}: {ms:.3f} ms, frac {balg / (ms / 1e3) / 6532.5e9:.3f}, fused={op.fused}")
