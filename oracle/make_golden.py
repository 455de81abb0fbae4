"""Generate tests/golden/*.npz from the REFERENCE package itself.

Run here (the reference is importable from /root/reference/pkg/src); the
fixtures are committed so the GPU box — which has no /root/reference —
can check both the oracle restatement and the CUDA path against them.

    python oracle/make_golden.py

Coefficient fields follow SURVEY §8(d)'s recipe (oracle.igs_oracle.recipe_planes);
the fixtures store a checksum of each field plus the seed, so the tests
regenerate the field and detect generator drift.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from igasum import bspline, quadrature, sumfac, tensorspace, geometry  # noqa: E402

from oracle import igs_oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def ref_problem(d, p, K, kind, k=None, seed=0, max_nnz=1 << 28):
    k = p if k is None else k
    bases = [bspline.UnivariateBasis(bspline.uniform_open_knots(p, K)) for _ in range(d)]
    rules = [quadrature.per_element_rule(b.breakpoints, k) for b in bases]
    quad = quadrature.TensorQuadrature(rules)
    planes = O.recipe_planes(d, list(quad.shape), k, kind, seed)
    pm = O.plane_map(d, kind)
    F = O.dense_field(planes, pm)
    ths = geometry.first_order_derivative_set(d)
    field = geometry.CoefficientField(ths, ths, F, quad.shape)
    prob = sumfac.AssemblyProblem(bases, bases, quad, field, max_nnz=max_nnz)
    return prob, planes


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{path}: {os.path.getsize(path) / 1e6:.2f} MB")


def golden_gauss():
    arrs = {}
    for k in range(1, 17):
        r = quadrature.gauss_legendre(k)
        arrs[f"nodes_{k}"] = r.nodes
        arrs[f"weights_{k}"] = r.weights
    r = quadrature.per_element_rule([0.0, 0.25, 0.5, 0.75, 1.0], 3)
    arrs["pe_points"] = r.points
    arrs["pe_weights"] = r.weights
    save("gauss", **arrs)


def golden_tabulate():
    arrs = {}
    cases = []
    for p in range(1, 9):
        for K in (1, 3, 8):
            cases.append((p, K, "gauss"))
    cases += [(4, 5, "random"), (3, 4, "knots"), (5, 6, "reduced")]
    for idx, (p, K, kind) in enumerate(cases):
        if kind == "reduced":
            kv = bspline.uniform_open_knots(p, K, interior_multiplicity=2)
        else:
            kv = bspline.uniform_open_knots(p, K)
        b = bspline.UnivariateBasis(kv)
        if kind in ("gauss", "reduced"):
            pts = quadrature.per_element_rule(b.breakpoints, p).points
        elif kind == "random":
            pts = np.sort(np.random.default_rng(idx).uniform(0, 1, 40))
            pts = np.concatenate([[0.0], pts, [1.0]])
        else:
            pts = np.unique(kv.knots)
        md = p - 1
        t = bspline.tabulate(b, pts, md)
        arrs[f"c{idx}_meta"] = np.array([p, K, md])
        arrs[f"c{idx}_knots"] = kv.knots
        arrs[f"c{idx}_points"] = pts
        arrs[f"c{idx}_values"] = t.values
        arrs[f"c{idx}_first"] = t.first_active
    arrs["ncases"] = np.array([len(cases)])
    save("tabulate", **arrs)


def golden_pattern():
    arrs = {}
    cases = [
        (2, 2, 2, 2, 1, 1, 2),   # order-2, 2 elements -> 7 pairs
        (1, 5, 1, 5, 1, 1, 1),   # order 1 -> K diagonal pairs
        (3, 4, 3, 4, 1, 1, 3),
        (4, 6, 4, 6, 2, 2, 4),   # reduced smoothness
        (3, 4, 2, 4, 2, 1, 3),   # Taylor-Hood-like
        (5, 7, 5, 7, 1, 1, 2),
    ]
    for idx, (pt, Kt, ps, Ks, mt, ms, k) in enumerate(cases):
        bt = bspline.UnivariateBasis(bspline.uniform_open_knots(pt, Kt, interior_multiplicity=mt))
        bs = bspline.UnivariateBasis(bspline.uniform_open_knots(ps, Ks, interior_multiplicity=ms))
        rule = quadrature.per_element_rule(np.union1d(bt.breakpoints, bs.breakpoints), k)
        pairs = tensorspace.nnz_pattern_1d(bt, bs, rule)
        arrs[f"c{idx}_meta"] = np.array([pt, Kt, ps, Ks, mt, ms, k])
        arrs[f"c{idx}_pairs"] = pairs
        arrs[f"c{idx}_count"] = np.array([tensorspace.nnz_count_exact(bt, bs)])
    arrs["ncases"] = np.array([len(cases)])
    save("pattern", **arrs)


def golden_assembly():
    # (name, d, p, K, kind): C1 at full size; reduced C2/C3 with the same p.
    cases = [
        ("c1_full", 2, 3, 64, 1),
        ("c2_reduced", 2, 5, 16, 2),
        ("c3_reduced", 3, 4, 6, 3),
        ("d1_mk", 1, 4, 7, 3),
        ("d3_p2", 3, 2, 4, 2),
    ]
    for name, d, p, K, kind in cases:
        prob, planes = ref_problem(d, p, K, kind)
        counter = sumfac.FlopCounter()
        A = sumfac.assemble(prob, counter)
        pat = prob.pattern()
        save(f"asm_{name}", meta=np.array([d, p, K, kind]), indptr=pat.indptr, indices=pat.indices,
             values=A.values, planes_sum=np.array([planes.sum(), (planes ** 2).sum()]),
             counter=np.array(counter.as_tuple()))


def golden_apply():
    # Reduced C4 / C5 (same p, fewer elements) -> assembled matvec oracle.
    cases = [("c4_reduced", 3, 6, 6, 2), ("c5_reduced", 3, 8, 4, 3), ("c3_small", 3, 4, 5, 3),
             ("d2_stiff", 2, 5, 9, 2)]
    for name, d, p, K, kind in cases:
        prob, planes = ref_problem(d, p, K, kind)
        A = sumfac.assemble(prob)
        N = prob.shape[1]
        x = O.recipe_x(N)
        y = A.matvec(x)
        save(f"apply_{name}", meta=np.array([d, p, K, kind]), x=x, y=y,
             planes_sum=np.array([planes.sum(), (planes ** 2).sum()]))


def golden_blocks():
    # assemble_block and a non-identity dir_order at a small size.
    prob, planes = ref_problem(3, 3, 3, 3)
    ths = geometry.first_order_derivative_set(3)
    blk = sumfac.assemble_block(prob, ths[1], ths[2])
    perm = sumfac.assemble(prob, dir_order=(2, 0, 1))
    save("blocks_d3_p3", meta=np.array([3, 3, 3, 3]), block_12=blk.values, perm_201=perm.values,
         indptr=prob.pattern().indptr, indices=prob.pattern().indices)


AFFINE_M = np.array([[1.0, 0.2, 0.0], [0.0, 1.5, 0.1], [0.3, 0.0, 0.8]])
AFFINE_B = np.array([0.5, -0.25, 1.0])
DIFF_M = np.array([[2.0, 0.3, 0.1], [0.3, 1.0, 0.2], [0.1, 0.2, 1.5]])


def geometry_cases():
    """(name, map, elements per direction, points per element, pde) — the
    tests rebuild the same cases through the repo's API."""
    return [
        ("qa", geometry.quarter_annulus(), 3, 3, geometry.pde_convection_diffusion(convection="default")),
        ("tb", geometry.twisted_box(), 2, 3, geometry.pde_laplace()),
        ("af", geometry.affine_geometry(AFFINE_M, AFFINE_B), 2, 2,
         geometry.PDEData(diffusion=DIFF_M, convection=[1.0, -2.0, 0.5], reaction=0.7)),
        ("qf", geometry.quarter_annulus(0.5, 1.5), 2, 4,
         geometry.PDEData(diffusion="identity", reaction=lambda x: 1.0 + x[:, 0] ** 2)),
    ]


def golden_geometry():
    for name, geo, ne, k, pde in geometry_cases():
        rules = [quadrature.per_element_rule(np.linspace(0.0, 1.0, ne + 1), k) for _ in range(geo.d)]
        quad = quadrature.TensorQuadrature(rules)
        ev = geometry.eval_geometry(geo, quad)
        F = geometry.build_coefficient_field(ev, pde).values
        save(f"geo_{name}", meta=np.array([geo.d, ne, k]), phys=ev.phys, jac=ev.jac, det=ev.det, inv=ev.inv, F=F)
    # full pipeline: quarter annulus, p=3 on 4x4 elements, cdr pulled back
    p, K = 3, 4
    bases = [bspline.UnivariateBasis(bspline.uniform_open_knots(p, K)) for _ in range(2)]
    quad = quadrature.TensorQuadrature([quadrature.per_element_rule(b.breakpoints, p) for b in bases])
    field = geometry.PulledBackCoefficient(geometry.quarter_annulus(), geometry.pde_convection_diffusion(
        convection="default")).evaluate(quad)
    A = sumfac.assemble(sumfac.AssemblyProblem(bases, bases, quad, field))
    save("geo_qa_assembly", meta=np.array([2, p, K]), values=A.values, indptr=A.pattern.indptr,
         indices=A.pattern.indices)


def golden_naive():
    """The reference's own comparison oracles (sumfac.py:388-509): values and
    block_update counter of assemble_naive, and assemble_kronecker_dense, on a
    3D mass+stiffness case and a 2D Petrov-Galerkin case with reduced
    smoothness, a non-symmetric F and a custom rule in one direction."""
    prob, planes = ref_problem(3, 3, 3, 3)
    counter = sumfac.FlopCounter()
    A = sumfac.assemble_naive(prob, counter)
    save("naive_d3_p3", meta=np.array([3, 3, 3, 3]), values=A.values, counter=np.array(counter.as_tuple()),
         indptr=prob.pattern().indptr, indices=prob.pattern().indices)
    tk = [bspline.uniform_open_knots(3, 4, interior_multiplicity=2), bspline.uniform_open_knots(3, 3)]
    sk = [bspline.uniform_open_knots(2, 4), bspline.uniform_open_knots(2, 3)]
    rules = [quadrature.per_element_rule(np.unique(tk[0].knots), 3),
             quadrature.custom_rule(np.linspace(0.01, 0.99, 11), np.full(11, 1.0 / 11))]
    quad = quadrature.TensorQuadrature(rules)
    theta = [(0, 0), (1, 0), (0, 1)]
    F = np.random.default_rng(3).uniform(-1, 1, (quad.num_points, 3, 3))
    field = geometry.CoefficientField(theta, theta, F, quad.shape)
    prob = sumfac.AssemblyProblem([bspline.UnivariateBasis(k) for k in tk], [bspline.UnivariateBasis(k) for k in sk],
                                  quad, field)
    counter = sumfac.FlopCounter()
    A = sumfac.assemble_naive(prob, counter)
    D = sumfac.assemble_kronecker_dense(prob)
    save("naive_d2_pg", F=F, values=A.values, counter=np.array(counter.as_tuple()), dense=D,
         indptr=prob.pattern().indptr, indices=prob.pattern().indices)


if __name__ == "__main__" and len(sys.argv) > 1:
    for name in sys.argv[1:]:
        globals()["golden_" + name]()
elif __name__ == "__main__":
    golden_gauss()
    golden_tabulate()
    golden_pattern()
    golden_assembly()
    golden_apply()
    golden_blocks()
    golden_geometry()
    golden_naive()
