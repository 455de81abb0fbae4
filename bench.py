"""Benchmark of the matrix-free fp64 apply (BASELINE.json headline metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4]
                    [--impl ours|reference]

Default workload: C4 — d=3 stiffness apply y = K·x, p=6, 128^3 elements
(N = 133^3 = 2,352,637 DoFs, 453M quadrature points carrying 6 SPD
coefficient planes = 21.7 GB).  A step is one apply.  For N > 1 GPUs
(torchrun) the element layers of the last direction are split over the
ranks (sharded.py) with an NCCL (p-1)-layer halo: strong scaling.

Printed JSON (rank 0): value = DoFs/s of the whole job (N·K/t, device
time, max over ranks); e2e = the same through the public API with host
(pinned) x/y and the H2D/D2H copies inside the timed region; roofline of
the dominant kernel (apply3d) against the measured HBM copy bandwidth;
cpu_baseline = the CPU oracle (oracle/igs_oracle.py, a numpy restatement
of the reference algorithm) on a bounded z-slab sample.  The same line
carries `c5` (the largest single-GPU config, 50 applies, with its own
roofline / e2e / cpu_baseline) and `assembly` (C3 and C2, each checked
against the oracle's values in the run).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    "C4": dict(d=3, p=6, K=128, kind=2, applies=100, desc="d3 p6 128^3 stiffness apply"),
    "C5": dict(d=3, p=8, K=128, kind=3, applies=50, desc="d3 p8 128^3 mass+stiffness apply"),
}


def measured_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_peak():
    """P64 (TFLOP/s): the DMMA rate tools/fp64_peak.py measured on this pool's
    B200 with its clock record (profiles/fp64_peak.json), sustained figure."""
    try:
        with open(os.path.join(REPO, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["dmma_tflops_sustained"]), "profiles/fp64_peak.json (sustained DMMA, SM clock " \
            f"{d['clocks_sustained']['sm_mhz']:.0f} MHz, reasons {d['clocks_sustained']['reasons']})"
    except Exception:
        return 37.15, "fallback (round-1 burst microbenchmark)"


def ncu_profile(name):
    """ncu-measured per-launch facts committed under profiles/ (F_exec, DRAM traffic)."""
    try:
        with open(os.path.join(REPO, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def config_for(name, world):
    """The workload's config dict — identical in both arms (no torch needed)."""
    w = WORKLOADS[name]
    d, p, K = w["d"], w["p"], w["K"]
    nplanes = {1: 1, 2: d * (d + 1) // 2, 3: 1 + d * (d + 1) // 2}[w["kind"]]
    pts = (p * K) ** d
    return {"workload": name, "desc": w["desc"], "dofs": (K + p - 1) ** d, "points": pts, "planes": nplanes,
            "applies_per_step": 1, "baseline_applies": w["applies"],
            "partition": f"slowest-axis slabs x{world}",
            "l2": f"inputs > L2 ({8 * nplanes * pts / 1e9:.1f} GB of coefficient planes per step)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, streamed every 50 ms while the
    timed region runs (the recipe's clocks line, B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._proc = None
        self._t = None

    def _reader(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.strip().split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *exc):
        if self._proc is not None:
            time.sleep(0.1)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_baseline(w, min_seconds=10.0, seed=0):
    """Time the CPU oracle's slab-wise apply (oracle/igs_oracle.py apply_slab,
    the numpy restatement of the reference algorithm) on a bounded sample:
    one element layer of the last direction per task, all host cores, passes
    repeated until `min_seconds` of work.  Coefficient values do not change
    the work, so one layer of seeded planes (1 + 0.05·U) is reused for every
    layer; the rate is extrapolated from the layers done to whole applies."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import igs_oracle as O

    d, p, K = w["d"], w["p"], w["K"]
    cores = os.cpu_count() or 1
    sp = [O.uniform_space(p, K) for _ in range(d)]
    ths = O.first_order_set(d)
    pm = O.plane_map(d, w["kind"])
    n = int(np.prod([s.num_basis for s in sp]))
    x = O.recipe_x(n, seed)
    layer_pts = (p * K) ** (d - 1) * p
    nplanes = len({v for row in pm for v in row if v >= 0})
    rng = np.random.default_rng(seed)
    planes = 1.0 + 0.05 * rng.random((nplanes, layer_pts))
    layers = min(K, cores)

    def one(z):
        return O.apply_slab(sp, p, ths, ths, pm, planes, x, z, z + 1)

    done = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        while True:
            list(ex.map(one, range(layers)))
            done += layers
            if time.perf_counter() - t0 >= min_seconds:
                break
    t = time.perf_counter() - t0
    frac = done / K
    return {"value": n * frac / t, "unit": "DoF/s", "cores": cores, "kind": "port", "host": host_info(),
            "sample": f"{done} element layers ({frac:.2f} applies' worth, extrapolated to whole applies) of "
                      f"{w['desc']}, numpy oracle apply_slab on {cores} threads, one seeded layer of planes "
                      f"(1 + 0.05 U) reused for every layer, {t:.1f} s"}


def _sym_exec_model(p, K, e_cnt):
    """Executed DMMA / fp64 flops of asm3_sym<4,4,4> from its schedule (used
    only when the ncu-counted profiles/C3_fexec.json is absent): per (4x4-row
    tile, z point) stage 1 = 4 y-tiles x 2 n-tiles x 5 k-steps x 10 blocks,
    stage 2 = 4 m-tiles x 2 n-tiles x 4 k-steps x 9 groups DMMA (512 flop);
    stage 3 = 448 pairs x (4P + 2P^2 FMA)."""
    tiles = (-(-(K + p - 1) // 4)) ** 2
    dmma = (400 + 288) * tiles * e_cnt * p
    return 512.0 * dmma + 2.0 * 448 * (4 * p + 2 * p * p) * tiles * e_cnt * p


def assembly_section(reps=5, cpu=True, seed=0, rank=0, world=1):
    """C3 assembly (d=3, p=4, 64^3, mass+stiffness) measured in the same run:
    warm assembly (pattern cached, as the reference caches it), CUDA events,
    nnz/s; roofline against the measured fp64 DMMA peak with F_exec counted
    by ncu (profiles/C3_fexec.json); CPU baseline = the oracle's Alg. 1
    restatement on the same full-size problem (one core).  With N ranks the
    rows are split by DoF layers of z (sharded.SlabAssembly): each rank
    generates the coefficients of its slab plus the kernel's halo and writes
    its CSR slice, no collective; time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1809_05471_b200 import sumfac, workloads
    from paper_1809_05471_b200.sharded import SlabAssembly, SlabPartition
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    p, K, kind = 4, 64, workloads.MASS_STIFF
    bases, quad = workloads.spaces(3, p, K)
    part = SlabPartition(K, p, world)
    sa = SlabAssembly(part, rank)
    e_lo, e_hi = (0, K) if world == 1 else sa.halo_elements()
    planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=seed, z_range=(e_lo * p, e_hi * p))
    field = workloads.field_from_planes(3, kind, planes, quad.shape, slab=None if world == 1 else (e_lo, e_hi))
    prob = AssemblyProblem(bases, bases, quad, field, max_nnz=1 << 40)
    run = (lambda: sumfac.assemble(prob)) if world == 1 else (lambda: sa.assemble(prob))
    for _ in range(3):  # W >= 3 warm-up assemblies (the first also builds the tables and the pattern)
        run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    nnz = prob.pattern().nnz
    npts = quad.num_points
    b_alg = 8 * field.n_planes * npts + 8 * nnz             # planes read + values written (whole job)
    p64, p64_src = fp64_peak()
    p64 *= 1e12
    prof = ncu_profile("C3_fexec.json")
    if prof is not None and world == 1:
        f_exec, f_src = float(prof["exec_flops"]), "ncu counters (profiles/C3_fexec.json)"
        traffic = float(prof["dram_bytes"])
    else:
        f_exec, f_src = _sym_exec_model(p, K, e_hi - e_lo) * (world if world > 1 else 1), "kernel schedule"
        traffic = None
    f_merged = 2 * 10_390_000_000        # merged-block MACs (the algorithm's own count)
    f_ref = 2 * 16_030_801_920           # the reference FlopCounter's block updates
    peak_bw, _ = measured_peak()
    t = ms / 1e3
    fused = sumfac.fused_path(prob)
    out = {"workload": "C3", "desc": "d3 p4 64^3 mass+stiffness assembly (warm, pattern cached)",
           "value": nnz / t, "unit": "nnz/s", "ms": ms, "nnz": nnz, "fused": fused,
           "kernel": "asm3_sym<4,4,4> (one pass: stages 1-3 on chip, symmetric half + mirrored writes)",
           "gpu_launches_per_assembly": 2,
           "partition": f"z DoF-layer row blocks x{world} (slab + halo, no collective)",
           "clocks": clk.summary(),
           "roofline": {"bound": "fp64", "achieved": f_exec / t / 1e12, "peak": p64 / 1e12, "unit": "TFLOP/s",
                        "peak_source": p64_src,
                        "frac": max(f_exec / t / (p64 * world), b_alg / t / (peak_bw * 1e9 * world)),
                        "frac_rule": "SURVEY 8d: max(B_alg/(t BW), F_exec/(t P64)); the one-pass kernel is "
                                     "the whole assembly (plus a 1-thread row-offset launch)",
                        "exec_flops": f_exec, "exec_flops_source": f_src, "alg_flops_merged": f_merged,
                        "ref_flops": f_ref, "frac_merged_alg": f_merged / t / (p64 * world),
                        "frac_ref_equivalent": f_ref / t / (p64 * world),
                        "hbm_gbs": b_alg / t / 1e9, "alg_bytes": b_alg, "traffic": traffic}}
    # the two-kernel fused path (H through HBM) on the same problem, for comparison
    if world == 1:
        for _ in range(3):
            sumfac.assemble(prob, flags=8)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            sumfac.assemble(prob, flags=8)
        e1.record()
        torch.cuda.synchronize()
        out["two_pass_ms"] = e0.elapsed_time(e1) / reps
    # cold assembly (fresh problem: tabulation + pattern + values) and the CSR
    # hand-off to the host (f2), reported separately as SURVEY §8(d) asks
    if world == 1:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cold = AssemblyProblem(bases, bases, quad, field, max_nnz=1 << 40)
        A = sumfac.assemble(cold)
        torch.cuda.synchronize()
        out["cold_ms"] = (time.perf_counter() - t0) * 1e3
        pat = cold.pattern()
        hv = torch.empty(A.values.shape, dtype=A.values.dtype, pin_memory=True)
        hi_ = torch.empty(pat.indices_dev.shape, dtype=pat.indices_dev.dtype, pin_memory=True)
        hp = torch.empty(pat.indptr_dev.shape, dtype=pat.indptr_dev.dtype, pin_memory=True)
        e0.record()
        hv.copy_(A.values, non_blocking=True)
        hi_.copy_(pat.indices_dev, non_blocking=True)
        hp.copy_(pat.indptr_dev, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        d2h_ms = e0.elapsed_time(e1)
        nbytes = hv.numel() * 8 + hi_.numel() * hi_.element_size() + hp.numel() * 8
        out["csr_d2h"] = {"ms": d2h_ms, "bytes": nbytes, "gbs": nbytes / d2h_ms / 1e6,
                          "index_bytes": hi_.element_size()}
        del A, cold, hv, hi_, hp
        # the coefficient planes' upload (a caller with host-side F), timed alone
        hpl = torch.empty(planes.shape, dtype=planes.dtype, pin_memory=True)
        hpl.copy_(planes)
        dpl = torch.empty_like(planes)
        torch.cuda.synchronize()
        e0.record()
        dpl.copy_(hpl, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_ms = e0.elapsed_time(e1)
        out["planes_h2d"] = {"ms": h2d_ms, "bytes": hpl.numel() * 8, "gbs": hpl.numel() * 8 / h2d_ms / 1e6}
        out["e2e"] = {"value": nnz / ((ms + h2d_ms + d2h_ms) / 1e3), "unit": "nnz/s",
                      "h2d_bytes_per_step": hpl.numel() * 8, "d2h_bytes_per_step": nbytes,
                      "note": "warm assembly + planes upload + CSR download, each timed alone and summed"}
        del hpl, dpl
    if cpu and rank == 0 and world == 1:
        from oracle import igs_oracle as O

        sp = [O.uniform_space(4, K) for _ in range(3)]
        hplanes = planes.cpu().numpy()
        ths = O.first_order_set(3)
        t0 = time.perf_counter()
        vals = O.assemble_sumfac(sp, sp, ths, ths, hplanes, O.plane_map(3, 3))
        tc = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": vals.size / tc, "unit": "nnz/s", "cores": 1, "kind": "port",
                               "host": host_info(),
                               "sample": f"oracle Alg. 1 restatement (scipy CSR x dense per direction, as the "
                                         f"reference), the full C3 problem on the same planes: {vals.size} nnz, "
                                         f"{tc:.2f} s (values only, pattern excluded as in the warm GPU number)"}
        err = float(np.linalg.norm(A_vals_check(prob) - vals) / np.linalg.norm(vals))
        out["parity_vs_cpu"] = {"rel_frobenius": err, "tol": 1e-12}
        assert err <= 1e-12, f"C3 GPU vs oracle {err:.3e}"
    return out


def A_vals_check(prob):
    from paper_1809_05471_b200 import sumfac

    return sumfac.assemble(prob).values_np()


def assembly_c2_section(reps=10, cpu=True, seed=0):
    """C2 (BASELINE configs[1]: d=2, p=5, 256², stiffness) assembly, warm,
    CUDA events; the CPU baseline is the oracle's Alg. 1 restatement on the
    same full-size problem (one core), whose values are also checked."""
    import torch

    from paper_1809_05471_b200 import sumfac, workloads

    p, K = 5, 256
    prob = workloads.make_problem(2, p, K, workloads.STIFF, seed=seed)
    for _ in range(3):  # W >= 3 warm-up assemblies
        A = sumfac.assemble(prob)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        A = sumfac.assemble(prob)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    t = ms / 1e3
    nnz = A.nnz
    b_alg = 8 * prob.coeff.n_planes * prob.quad.num_points + 8 * nnz
    f_ref = 2 * 460_800_000                   # the reference FlopCounter
    p64, p64_src = fp64_peak()
    peak_bw, _ = measured_peak()
    prof = ncu_profile("C2_fexec.json")
    out = {"workload": "C2", "desc": "d2 p5 256^2 stiffness assembly (warm, pattern cached)",
           "value": nnz / t, "unit": "nnz/s", "ms": ms, "nnz": nnz, "fused": sumfac.fused_path(prob),
           "roofline": {"bound": "fp64", "frac_ref_equivalent": f_ref / t / (p64 * 1e12),
                        "hbm_frac": b_alg / t / (peak_bw * 1e9), "alg_bytes": b_alg, "ref_flops": f_ref,
                        "peak": p64, "unit": "TFLOP/s", "peak_source": p64_src}}
    if prof is not None:
        out["roofline"]["exec_flops"] = float(prof["exec_flops"])
        out["roofline"]["achieved"] = float(prof["exec_flops"]) / t / 1e12
        out["roofline"]["frac"] = max(float(prof["exec_flops"]) / t / (p64 * 1e12), b_alg / t / (peak_bw * 1e9))
        out["roofline"]["traffic"] = float(prof["dram_bytes"])
    if cpu:
        from oracle import igs_oracle as O

        sp = [O.uniform_space(p, K) for _ in range(2)]
        planes = prob.coeff.planes.cpu().numpy()
        ths = O.first_order_set(2)
        t0 = time.perf_counter()
        vals = O.assemble_sumfac(sp, sp, ths, ths, planes, O.plane_map(2, workloads.STIFF))
        tc = time.perf_counter() - t0
        err = float(np.linalg.norm(A.values_np() - vals) / np.linalg.norm(vals))
        assert err <= 1e-12, f"C2 GPU vs oracle {err:.3e}"
        out["parity_vs_cpu"] = {"rel_frobenius": err, "tol": 1e-12}
        out["cpu_baseline"] = {"value": vals.size / tc, "unit": "nnz/s", "cores": 1, "kind": "port",
                               "host": host_info(),
                               "sample": f"oracle Alg. 1 restatement, full C2 ({vals.size} nnz) on the same planes, "
                                         f"{tc:.2f} s"}
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    steps = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(w, min_seconds=1.0 if i < args.warmup else min(5.0, 150.0 / max(1, args.steps)))
        if i >= args.warmup:
            steps.append(cb["value"])
    value = float(np.median(steps))
    line = {"metric": "matrix-free fp64 apply throughput", "value": value, "unit": "DoF/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based coefficients, see DESIGN.md)",
            "config": config_for(args.workload, world),
            "cpu_baseline": {**cb, "value": value},
            "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measure_apply(name, args, rank, world, local, steps, with_cpu):
    """One apply workload (C4 / C5): device-timed steps, the dominant kernel
    alone (roofline), e2e through the public API with host buffers, clocks,
    and (rank 0, N=1) the CPU baseline.  Returns the result dict (rank 0)."""
    import torch
    import torch.distributed as dist

    from paper_1809_05471_b200 import matfree, workloads
    from paper_1809_05471_b200.sharded import NcclComm, NcclSlabApply, SlabPartition
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    w = WORKLOADS[name]
    d, p, K, kind = w["d"], w["p"], w["K"], w["kind"]
    part = SlabPartition(K, p, world)
    lo, hi = part.elements(rank)
    bases, quad = workloads.spaces(d, p, K)
    layer_pts = int(np.prod(quad.shape[:-1]))
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=0, z_range=(lo * p, hi * p))
    slab = None if world == 1 else (lo, hi)
    field = workloads.field_from_planes(d, kind, planes, quad.shape, slab=slab)
    prob = AssemblyProblem(bases, bases, quad, field)
    op = matfree.MatrixFreeOperator(prob)
    N = int(np.prod([b.num_basis for b in bases]))
    layer_n = N // (K + p - 1)
    olo, ohi = part.own_layers(rank)
    n_own = (ohi - olo) * layer_n
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x_own = torch.randn(n_own, dtype=torch.float64, device="cuda", generator=gen)
    y_own = torch.empty(n_own, dtype=torch.float64, device="cuda")
    if world == 1:
        def step(x, y):
            op.apply_device(x, y)
        launches = 2
    else:
        # the C-ABI data plane: igs_apply_sharded over an NCCL communicator of
        # the library (ghost gather on a communication stream overlapped with
        # the interior elements, boundary elements after it, ghost reduce)
        comm = NcclComm(rank, world)
        sharded = NcclSlabApply(op, part, rank, comm=comm, overlap=True)
        launches = 8  # x copy, interior apply3d + reduce, memset, boundary apply3d + reduce, halo add, y copy

        def step(x, y):
            sharded.apply(x, y)

    for _ in range(max(3, args.warmup)):
        step(x_own, y_own)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # --- device-timed region: `steps` applies, inputs (21.7+ GB) far larger than L2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(steps):
            step(x_own, y_own)
        e1.record()
        barrier()
    t_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = N * steps / (t_ms / 1e3)

    # --- dominant kernel alone (apply3d, no reduce): roofline
    f = prob.coeff
    npts_local = (hi - lo) * p * layer_pts
    n_local = (hi - lo + p - 1) * layer_n
    b_alg = 8 * f.n_planes * npts_local + 16 * n_local
    x_local = torch.randn(n_local, dtype=torch.float64, device="cuda", generator=gen)
    y_local = torch.empty(n_local, dtype=torch.float64, device="cuda")
    kreps = max(5, steps // 4)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(kreps):
        op.apply_device(x_local, y_local, kernel_only=True)
    k1.record()
    torch.cuda.synchronize()
    k_ms = k0.elapsed_time(k1) / kreps
    peak, peak_kind = measured_peak()
    achieved = b_alg / (k_ms / 1e3) / 1e9
    traffic = None
    prof = ncu_profile(f"{name}_traffic.json")
    if prof is not None:
        traffic = prof.get("dram_bytes_per_launch")

    # --- end to end through the public API: pinned host x -> device -> apply
    # -> host y every step, transfers overlapped with the neighbouring steps'
    # applies (matfree.HostPipeline: copy streams + events)
    x_host = torch.empty(n_own, dtype=torch.float64, pin_memory=True)
    x_host.copy_(x_own.cpu())
    y_hosts = [torch.empty(n_own, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    pipe = matfree.HostPipeline(step, n_own, n_own)
    pipe.run([x_host] * 2, y_hosts)
    barrier()
    e0.record()
    pipe.run([x_host] * steps, [y_hosts[i & 1] for i in range(steps)])
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = N * steps / (e2e_ms / 1e3)
    fused_flag = op.fused
    if world > 1:
        comm.check()
        dist.barrier()
        comm.close()
    del planes, field, prob, op
    step = None
    torch.cuda.empty_cache()
    cb = cpu_baseline(w) if (with_cpu and rank == 0 and world == 1) else None
    return {"value": value, "unit": "DoF/s", "steps": steps, "ms_per_step": t_ms / steps,
            "config": config_for(name, world), "fused": fused_flag,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": "apply3d_kernel", "kernel_ms": k_ms, "alg_bytes_per_launch": b_alg},
            "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": 8 * n_own,
                    "d2h_bytes_per_step": 8 * n_own},
            "gpu_launches": steps * launches, "clocks": clk.summary(), "cpu_baseline": cb}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100, help="applies per timed region (BASELINE C4: 100)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-assembly", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 section (the C4 run measures C5 too)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = measure_apply(args.workload, args, rank, world, local, args.steps, not args.no_cpu_baseline)
    c5 = None
    if args.workload == "C4" and not args.no_c5:
        # the largest single-GPU configuration (60 GB of planes), BASELINE's 50 applies
        try:
            c5 = measure_apply("C5", args, rank, world, local, WORKLOADS["C5"]["applies"],
                               not args.no_cpu_baseline)
        except Exception as exc:  # the headline line must still print
            c5 = {"error": repr(exc)}
    asm = None
    if not args.no_assembly:
        try:
            asm = assembly_section(cpu=not args.no_cpu_baseline, rank=rank, world=world)
            if world == 1:
                asm["c2"] = assembly_c2_section(cpu=not args.no_cpu_baseline)
        except Exception as exc:  # the apply line must still print
            asm = {"error": repr(exc)}
    if rank == 0:
        line = {
            "metric": "matrix-free fp64 apply throughput", "value": res["value"], "unit": "DoF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based coefficients, see DESIGN.md)",
            "config": res["config"], "roofline": res["roofline"], "e2e": res["e2e"],
            # per step: apply3d + reduce; rank 0 of a slab run: x copy, interior
            # and boundary applies (2 + 2), y copy (K5 kernels) — NCCL's own excluded
            "gpu_launches": res["gpu_launches"], "clocks": res["clocks"], "cpu_baseline": res["cpu_baseline"],
            "fused": res["fused"], "c5": c5, "assembly": asm,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
