"""2D assembly timing (development aid): the sumfac.assemble loop (host
overhead included) vs a CUDA-graph replay of the same call (device time),
one-pass vs two-pass; checked against each other."""

import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads  # noqa: E402


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return ev_time(g.replay, reps)


def case(d, p, K, kind, reps=50):
    prob = workloads.make_problem(d, p, K, kind)
    out = {"d": d, "p": p, "K": K, "kind": kind}
    for name, fl in (("one", 0), ("two", 8)):
        A = sumfac.assemble(prob, flags=fl)
        out[name + "_loop_ms"] = ev_time(lambda: sumfac.assemble(prob, flags=fl), reps)
        out[name + "_graph_ms"] = graph_time(lambda: sumfac.assemble(prob, flags=fl), reps)
        t0 = time.perf_counter()
        for _ in range(reps):
            sumfac.assemble(prob, flags=fl)
        torch.cuda.synchronize()
        out[name + "_host_us"] = (time.perf_counter() - t0) / reps * 1e6
        out[name + "_vals"] = A.values_np()
    a, b = out.pop("one_vals"), out.pop("two_vals")
    out["rel_one_vs_two"] = float(np.linalg.norm(a - b) / np.linalg.norm(b))
    out["nnz"] = int(a.size)
    out["gnnz_s_graph"] = a.size / out["one_graph_ms"] / 1e6
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "orders":
        for p in range(2, 7):
            o = case(2, p, 256, 2, reps=10)
            print(p, json.dumps({k: o[k] for k in ("one_graph_ms", "one_loop_ms", "two_graph_ms", "rel_one_vs_two")}))
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "c2":
        o = case(2, 5, 256, 2)
        print(sys.argv[2:] or "", json.dumps({k: o[k] for k in ("one_graph_ms", "two_graph_ms", "rel_one_vs_two")}))
        sys.exit(0)
    for c in [(2, 5, 256, 2), (2, 3, 64, 1), (2, 5, 128, 3), (2, 4, 256, 3), (2, 2, 512, 2), (2, 3, 256, 2)]:
        print(json.dumps(case(*c)), flush=True)
