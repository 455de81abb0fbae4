"""Builders of the C `igs_problem` struct from the Python mirror objects.

Each builder returns (struct, keepalive) — `keepalive` holds the device
tensors the struct points at and must live as long as the struct is used.
"""

import ctypes

import numpy as np

from . import _lib


def _fill_dir(dst, basis, rule, table, keep):
    torch = _lib.require_cuda()
    dst.order = basis.order
    dst.num_basis = basis.num_basis
    dst.num_points = rule.num_points
    lo, hi = basis.device_csupp()
    pts, wts = rule.device()
    keep += [lo, hi, pts, wts]
    dst.csupp_lo = lo.data_ptr()
    dst.csupp_hi = hi.data_ptr()
    dst.points = pts.data_ptr()
    dst.weights = wts.data_ptr()
    if table is not None:
        dst.max_deriv = table.max_deriv
        dst.values = table.values.data_ptr()
        dst.first_active = table.first_active.data_ptr()
        keep += [table.values, table.first_active]
    else:
        dst.max_deriv = 0
    # Element structure for the fused kernels: a per-element rule built on
    # exactly this basis' breakpoints.
    if (rule.points_per_element > 0 and rule.elements == basis.num_elements
            and getattr(rule, "breakpoints", None) is not None
            and len(rule.breakpoints) == len(basis.breakpoints)
            and (rule.breakpoints == basis.breakpoints).all()):
        dst.num_elements = rule.elements
        dst.points_per_element = rule.points_per_element
        bp = basis.breakpoints
        h = np.diff(bp)
        dst.uniform = int(basis.max_smoothness and len(h) > 0
                          and float(np.max(np.abs(h - h[0]))) <= 1e-14 * float(abs(bp[-1] - bp[0])))
    else:
        dst.num_elements = 0
        dst.points_per_element = 0
        dst.uniform = 0
    del torch


def problem_struct_for_pattern(trial_bases, test_bases, rules):
    prob = _lib.IgsProblem()
    keep = []
    prob.d = len(rules)
    for k, (tr, te, rule) in enumerate(zip(trial_bases, test_bases, rules)):
        _fill_dir(prob.trial[k], tr, rule, None, keep)
        _fill_dir(prob.test[k], te, rule, None, keep)
    prob.n_theta = prob.n_eta = 1
    for i in range(_lib.MAX_DERIV_SET):
        for j in range(_lib.MAX_DERIV_SET):
            prob.plane_of[i][j] = -1
    for k in range(prob.d):
        prob.dir_order[k] = k
    return prob, keep


class _TableRule:
    """Rule stand-in built from a table's own points (weights unused)."""

    def __init__(self, table):
        self.points = table.points
        self.num_points = table.num_points
        self.points_per_element = 0
        self.elements = 0
        self.breakpoints = None
        self._t = table

    def device(self):
        pts = self._t.points_dev
        return pts, pts


def problem_struct_for_tables(tables):
    prob = _lib.IgsProblem()
    keep = []
    prob.d = len(tables)
    for k, t in enumerate(tables):
        rule = _TableRule(t)
        _fill_dir(prob.trial[k], t.basis, rule, t, keep)
        _fill_dir(prob.test[k], t.basis, rule, t, keep)
    prob.n_theta = prob.n_eta = 1
    for i in range(_lib.MAX_DERIV_SET):
        for j in range(_lib.MAX_DERIV_SET):
            prob.plane_of[i][j] = -1
    for k in range(prob.d):
        prob.dir_order[k] = k
    return prob, keep


def problem_struct(trial_bases, test_bases, rules, trial_tables, test_tables, theta_set, eta_set,
                   plane_of, n_planes, plane_stride, dir_order=None, num_pairs=None, slab=None):
    prob = _lib.IgsProblem()
    keep = []
    d = len(rules)
    prob.d = d
    for k in range(d):
        _fill_dir(prob.trial[k], trial_bases[k], rules[k], trial_tables[k], keep)
        _fill_dir(prob.test[k], test_bases[k], rules[k], test_tables[k], keep)
    if len(theta_set) > _lib.MAX_DERIV_SET or len(eta_set) > _lib.MAX_DERIV_SET:
        raise ValueError("at most 8 derivative multi-indices per set")
    prob.n_theta = len(theta_set)
    prob.n_eta = len(eta_set)
    for j, th in enumerate(theta_set):
        for k in range(d):
            prob.theta[j][k] = int(th[k])
    for i, et in enumerate(eta_set):
        for k in range(d):
            prob.eta[i][k] = int(et[k])
    for i in range(_lib.MAX_DERIV_SET):
        for j in range(_lib.MAX_DERIV_SET):
            prob.plane_of[i][j] = -1
    for i in range(len(eta_set)):
        for j in range(len(theta_set)):
            prob.plane_of[i][j] = int(plane_of[i][j])
    prob.n_planes = int(n_planes)
    prob.plane_stride = int(plane_stride)
    order = tuple(range(d)) if dir_order is None else tuple(dir_order)
    for k in range(d):
        prob.dir_order[k] = int(order[k])
    if num_pairs is not None:
        for k in range(d):
            prob.num_pairs[k] = int(num_pairs[k])
    if slab is not None:
        prob.slab_lo, prob.slab_hi = int(slab[0]), int(slab[1])
    return prob, keep


def byref(prob):
    return ctypes.byref(prob)
