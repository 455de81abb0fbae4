"""C3 assembly device time (CUDA events, warm) of the library at IGS_LIB_PATH (A/B aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads  # noqa: E402

prob = workloads.make_problem(3, 4, 64, 3)
for _ in range(2):
    sumfac.assemble(prob)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    sumfac.assemble(prob)
e1.record()
torch.cuda.synchronize()
print(sys.argv[1] if len(sys.argv) > 1 else "", f"{e0.elapsed_time(e1) / 10:.3f} ms")
