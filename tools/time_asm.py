"""Device timing of the fused assembly: one-pass symmetric vs two-pass
(development aid; CUDA events, warm, pattern cached)."""

import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads  # noqa: E402


def run(d, p, K, kind, flags=0, reps=10):
    prob = workloads.make_problem(d, p, K, kind)
    sumfac.assemble(prob, flags=flags)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        A = sumfac.assemble(prob, flags=flags)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"d": d, "p": p, "K": K, "kind": kind, "flags": flags, "ms": ms, "nnz": A.nnz,
            "gnnz_s": A.nnz / ms / 1e6}


if __name__ == "__main__":
    cases = [(3, 4, 64, 3, 0), (3, 4, 64, 3, 8), (2, 5, 256, 2, 0), (3, 2, 64, 3, 0), (3, 3, 64, 3, 0),
             (3, 2, 64, 3, 8), (3, 3, 64, 3, 8)]
    for c in cases:
        print(json.dumps(run(*c)), flush=True)
