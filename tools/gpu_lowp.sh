cat > /tmp/lp.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_1809_05471_b200 import matfree, workloads
for p in (2, 3, 4):
    prob = workloads.make_problem(3, p, 128, 2)
    op = matfree.MatrixFreeOperator(prob)
    n = prob.shape[1]
    x = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    for _ in range(3): op.apply_device(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): op.apply_device(x, y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    balg = 8 * prob.coeff.n_planes * prob.quad.num_points + 16 * n
    print(sys.argv[1], p, f"{ms:.3f} ms frac {balg / (ms / 1e3) / 6532.5e9:.3f}", flush=True)
PY
for r in 1 2; do
for v in 0 11 12 13; do IGS_APPLY_VARIANT=$v IGS_LIB_PATH=variants/lowp/libigs_b200.so python /tmp/lp.py v$v; done
done 2>&1 | grep -v Warn
