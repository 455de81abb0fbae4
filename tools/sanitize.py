"""Small invocations of every fused kernel (apply3d_kernel, asm3_sym, asm2_sym,
asm3_stage12 + asm_sweep, asm2_stage1 + asm_sweep, the generic stage kernels)
for compute-sanitizer (memcheck / racecheck / synccheck / initcheck); the
results are still checked against each other so a sanitizer-clean but wrong
run cannot pass.  Run as
    compute-sanitizer --tool <tool> python tools/sanitize.py [apply|asm|all]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import matfree, sumfac, workloads  # noqa: E402
from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots  # noqa: E402
from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule  # noqa: E402

TWO_PASS, GENERIC = 8, 1


def problem(p, K, kind, seed):
    d = len(K)
    bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=seed)
    return sumfac.AssemblyProblem(bases, bases, quad, workloads.field_from_planes(d, kind, planes, quad.shape))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("apply", "all"):
        for p, K, kind in [(2, (9, 5, 4), 3), (3, (6, 4, 5), 2), (4, (5, 9, 3), 3), (5, (4, 3, 5), 2),
                           (6, (6, 5, 4), 2), (7, (3, 4, 3), 3), (8, (3, 4, 3), 3), (8, (2, 3, 4), 2)]:
            prob = problem(p, K, kind, seed=p)
            op = matfree.MatrixFreeOperator(prob)
            x = np.random.default_rng(p).standard_normal(prob.shape[1])
            y = matfree.apply(op, x)
            yg = matfree.apply(matfree.MatrixFreeOperator(prob, force_generic=True), x)
            torch.cuda.synchronize()
            e = rel(y, yg)
            print(f"apply p={p} K={K} kind={kind} fused={op.fused} fused-vs-generic {e:.2e}", flush=True)
            assert e < 1e-12

    if what in ("asm", "all"):
        for p, K, kind in [(4, (5, 4, 6), 3), (2, (9, 6, 3), 2), (3, (4, 5, 3), 3), (5, (3, 4, 2), 2), (6, (2, 2, 3), 3),
                           (5, (20, 7), 3), (4, (24, 13), 2), (3, (34, 9), 3), (2, (48, 10), 1)]:
            prob = problem(p, K, kind, seed=10 + p)
            A = sumfac.assemble(prob).values_np()
            A2 = sumfac.assemble(prob, flags=TWO_PASS).values_np()
            Ag = sumfac.assemble(prob, flags=GENERIC).values_np()
            torch.cuda.synchronize()
            e2, eg = rel(A, A2), rel(A, Ag)
            print(f"asm p={p} K={K} kind={kind} path={sumfac.fused_path(prob)} vs two-pass {e2:.2e} vs generic {eg:.2e}", flush=True)
            assert e2 < 1e-12 and eg < 1e-12
    print("sanitize cases ok")
