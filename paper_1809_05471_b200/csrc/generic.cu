// Generic stage-by-stage kernels: the direction-by-direction recursion of
// the reference, one banded 1D contraction per launch, intermediates in HBM.
//
// This path covers everything the reference accepts (d = 1..3, Petrov-
// Galerkin trial != test, non-uniform / reduced-smoothness knots, custom
// point sets, arbitrary derivative index sets, any dir_order).  The fused
// kernels (apply3d.cu, assemble3d.cu) cover the BASELINE configurations at
// speed; `igs_fused_path` reports which one runs.
//
//   contraction MODE_EVAL  : Alg. 3 stage, coefficient -> points,
//                            tensorspace.py:134-153 (Q = _table_point_csr :115-131)
//   contraction MODE_TEST  : transpose of the above against test tables
//                            (Alg. 2)
//   contraction MODE_PAIR  : Alg. 1 stage against W = w·B_n·B_m
//                            (_Core.w_matrix sumfac.py:163-198, block_values :200-213)
//
// Layout: every intermediate is a 3-axis tensor [dir2][dir1][dir0] with
// direction 0 fastest — the reference's F-order point grid.  Contracting
// direction k replaces that axis' length in place, so after all directions
// the assembly values sit in [pair2][pair1][pair0] = the reference's
// assembly-value layout for the identity dir_order (tensorspace.py:306-322).
#include "igs_internal.cuh"

namespace igs {
namespace {

enum { MODE_EVAL = 0, MODE_TEST = 1, MODE_PAIR = 2 };

struct Op1D {
  // trial table (MODE_EVAL, MODE_PAIR)
  const double* vt; const int64_t* fat; int pt; int kt;
  // test table (MODE_TEST, MODE_PAIR)
  const double* vs; const int64_t* fas; int ps; int ks;
  const double* w;       // quadrature weights (MODE_PAIR)
  int64_t xtab;          // points in the full table (stride of values)
  int64_t x_off;         // first point of the slab
  int64_t n_off;         // first function of the slab (trial for EVAL, test for TEST)
  int64_t x_loc;         // points in the slab
  const int64_t* pair_n; // MODE_PAIR: trial function of each pair
  const int64_t* pair_m; // MODE_PAIR: test function of each pair
};

template <int MODE>
__global__ void contract_kernel(Op1D op, const double* __restrict__ in, double* __restrict__ out,
                                int64_t outer, int64_t Lin, int64_t Lout, int64_t inner,
                                int accumulate) {
  const int64_t total = outer * Lout * inner;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = g % inner;
    int64_t r = (g / inner) % Lout;
    int64_t o = g / (inner * Lout);
    const double* src = in + o * Lin * inner + i;
    double acc = 0.0;
    if (MODE == MODE_EVAL) {
      int64_t x = r + op.x_off;
      int64_t c0 = op.fat[x] - op.n_off;
      const double* v = op.vt + (int64_t)op.kt * op.pt * op.xtab + x;
      for (int j = 0; j < op.pt; ++j) acc = fma(v[j * op.xtab], src[(c0 + j) * inner], acc);
    } else if (MODE == MODE_TEST) {
      int64_t m = r + op.n_off;
      int64_t xa = lower_bound_i64(op.fas, op.xtab, m - op.ps + 1);
      int64_t xb = upper_bound_i64(op.fas, op.xtab, m);
      if (xa < op.x_off) xa = op.x_off;
      if (xb > op.x_off + op.x_loc) xb = op.x_off + op.x_loc;
      const double* v = op.vs + (int64_t)op.ks * op.ps * op.xtab;
      for (int64_t x = xa; x < xb; ++x)
        acc = fma(v[(m - op.fas[x]) * op.xtab + x], src[(x - op.x_off) * inner], acc);
    } else {
      int64_t n = op.pair_n[r], m = op.pair_m[r];
      int64_t xa = lower_bound_i64(op.fat, op.xtab, n - op.pt + 1);
      int64_t xa2 = lower_bound_i64(op.fas, op.xtab, m - op.ps + 1);
      int64_t xb = upper_bound_i64(op.fat, op.xtab, n);
      int64_t xb2 = upper_bound_i64(op.fas, op.xtab, m);
      if (xa2 > xa) xa = xa2;
      if (xb2 < xb) xb = xb2;
      const double* vt = op.vt + (int64_t)op.kt * op.pt * op.xtab;
      const double* vs = op.vs + (int64_t)op.ks * op.ps * op.xtab;
      for (int64_t x = xa; x < xb; ++x) {
        double coef = (op.w[x] * vt[(n - op.fat[x]) * op.xtab + x]) * vs[(m - op.fas[x]) * op.xtab + x];
        acc = fma(coef, src[x * inner], acc);
      }
    }
    double* dst = out + (o * Lout + r) * inner + i;
    *dst = accumulate ? *dst + acc : acc;
  }
}

struct PointwiseArgs {
  int n_theta, n_eta;
  int8_t plane_of[IGS_MAX_DERIV_SET][IGS_MAX_DERIV_SET];
  const double* planes;
  int64_t plane_stride;
  const double* u[IGS_MAX_DERIV_SET];  // per theta (nullptr if unused)
  double* g[IGS_MAX_DERIV_SET];        // per eta (nullptr if unused)
  const double* w[3];                  // per-direction weights (global tables)
  int64_t x[3];                        // local points per direction
  int64_t x_off_last;                  // slab offset in the last direction
  int d;
};

// g_eta = w(x) · Σ_theta F[eta, theta](x) · ∂^theta u(x)
__global__ void pointwise_kernel(PointwiseArgs a) {
  const int64_t npts = a.x[0] * a.x[1] * a.x[2];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npts;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i0 = q % a.x[0];
    int64_t i1 = (q / a.x[0]) % a.x[1];
    int64_t i2 = q / (a.x[0] * a.x[1]);
    // flat_weights order (quadrature.py:146-151): w_{d-1}·(...·(w_0·1))
    double w = a.w[0][i0 + (a.d == 1 ? a.x_off_last : 0)];
    if (a.d >= 2) w = a.w[1][i1 + (a.d == 2 ? a.x_off_last : 0)] * w;
    if (a.d >= 3) w = a.w[2][i2 + a.x_off_last] * w;
    double uv[IGS_MAX_DERIV_SET];
    for (int j = 0; j < a.n_theta; ++j) uv[j] = a.u[j] ? a.u[j][q] : 0.0;
    for (int i = 0; i < a.n_eta; ++i) {
      if (!a.g[i]) continue;
      double s = 0.0;
      for (int j = 0; j < a.n_theta; ++j) {
        int pl = a.plane_of[i][j];
        if (pl >= 0) s = fma(a.planes[pl * a.plane_stride + q], uv[j], s);
      }
      a.g[i][q] = w * s;
    }
  }
}

__global__ void pair_rows_kernel(const int64_t* rowptr, int64_t nrows, int64_t* pair_m) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= nrows) return;
  for (int64_t p = rowptr[m]; p < rowptr[m + 1]; ++p) pair_m[p] = m;
}

// Assembly-value layout [pair2][pair1][pair0] -> CSR order for rows
// [row_lo, row_hi) (the reference's value_perm, tensorspace.py:324-332,
// in closed form).
__global__ void scatter_csr_kernel(TensorPat t, const int64_t* pm0, const int64_t* pm1,
                                   const int64_t* pm2, const double* __restrict__ acc,
                                   int64_t P0, int64_t P1, int64_t P2, int64_t row_lo,
                                   int64_t row_hi, double* __restrict__ values) {
  int64_t total = P0 * P1 * P2;
  int64_t w[3], mi[3];
  int64_t base = tensor_row_start(t, row_lo, w, mi);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t p0 = g % P0, p1 = (g / P0) % P1, p2 = g / (P0 * P1);
    int64_t m0 = pm0[p0];
    int64_t m1 = t.d > 1 ? pm1[p1] : 0;
    int64_t m2 = t.d > 2 ? pm2[p2] : 0;
    int64_t m = m0 + t.ns[0] * (m1 + t.ns[1] * m2);
    if (m < row_lo || m >= row_hi) continue;
    int64_t start = tensor_row_start(t, m, w, mi);
    int64_t r0 = p0 - t.rp[0][m0];
    int64_t r1 = t.d > 1 ? p1 - t.rp[1][m1] : 0;
    int64_t r2 = t.d > 2 ? p2 - t.rp[2][m2] : 0;
    values[start - base + r2 * w[0] * w[1] + r1 * w[0] + r0] = acc[g];
  }
}

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = ceil_div(n, block);
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (unsigned)g;
}

igs_status launch_contract(int mode, const Op1D& op, const double* in, double* out,
                           const int64_t shape_in[3], int k, int64_t Lout, int accumulate,
                           cudaStream_t s) {
  int64_t outer = 1, inner = 1;
  for (int j = 0; j < k; ++j) inner *= shape_in[j];
  for (int j = k + 1; j < 3; ++j) outer *= shape_in[j];
  int64_t total = outer * Lout * inner;
  if (total == 0) return IGS_OK;
  const int block = 256;
  unsigned grid = grid_for(total, block);
  switch (mode) {
    case MODE_EVAL:
      contract_kernel<MODE_EVAL><<<grid, block, 0, s>>>(op, in, out, outer, shape_in[k], Lout, inner, accumulate);
      break;
    case MODE_TEST:
      contract_kernel<MODE_TEST><<<grid, block, 0, s>>>(op, in, out, outer, shape_in[k], Lout, inner, accumulate);
      break;
    default:
      contract_kernel<MODE_PAIR><<<grid, block, 0, s>>>(op, in, out, outer, shape_in[k], Lout, inner, accumulate);
  }
  IGS_LAUNCH_CHECK("contract_kernel");
  return IGS_OK;
}

Op1D eval_op(const igs_problem* p, const Dims& D, int k, int level) {
  const igs_dir& t = p->trial[k];
  Op1D op{};
  op.vt = t.values; op.fat = t.first_active; op.pt = t.order; op.kt = level;
  op.xtab = t.num_points;
  bool last = (k == p->d - 1);
  op.x_off = last ? D.x_off : 0;
  op.n_off = last ? D.nt_off : 0;
  op.x_loc = D.x[k];
  return op;
}

Op1D test_op(const igs_problem* p, const Dims& D, int k, int level) {
  const igs_dir& t = p->test[k];
  Op1D op{};
  op.vs = t.values; op.fas = t.first_active; op.ps = t.order; op.ks = level;
  op.xtab = t.num_points;
  bool last = (k == p->d - 1);
  op.x_off = last ? D.x_off : 0;
  op.n_off = last ? D.ns_off : 0;
  op.x_loc = D.x[k];
  return op;
}

int64_t prod3(const int64_t* s) { return s[0] * s[1] * s[2]; }

// Largest intermediate of an eval chain (N -> X per direction, 0..d-1).
int64_t eval_chain_max(const Dims& D, bool trial) {
  int64_t s[3] = {trial ? D.nt[0] : D.ns[0], trial ? D.nt[1] : D.ns[1], trial ? D.nt[2] : D.ns[2]};
  int64_t mx = prod3(s);
  for (int k = 0; k < D.d; ++k) {
    s[k] = D.x[k];
    mx = mx > prod3(s) ? mx : prod3(s);
  }
  return mx;
}

bool theta_used(const igs_problem* p, int j) {
  for (int i = 0; i < p->n_eta; ++i)
    if (p->plane_of[i][j] >= 0) return true;
  return false;
}
bool eta_used(const igs_problem* p, int i) {
  for (int j = 0; j < p->n_theta; ++j)
    if (p->plane_of[i][j] >= 0) return true;
  return false;
}

// Runs the eval chain of one trial derivative multi-index into `out`.
igs_status eval_chain(const igs_problem* p, const Dims& D, const int8_t* deriv, const double* x,
                      double* out, double* tA, double* tB, cudaStream_t s) {
  int64_t shape[3] = {D.nt[0], D.nt[1], D.nt[2]};
  const double* src = x;
  for (int k = 0; k < p->d; ++k) {
    double* dst = (k == p->d - 1) ? out : ((k % 2 == 0) ? tA : tB);
    Op1D op = eval_op(p, D, k, deriv[k]);
    IGS_TRY(launch_contract(MODE_EVAL, op, src, dst, shape, k, D.x[k], 0, s));
    shape[k] = D.x[k];
    src = dst;
  }
  return IGS_OK;
}

}  // namespace

size_t generic_apply_workspace(const igs_problem* p, const Dims& D) {
  Workspace ws(nullptr, 0, true);
  int64_t npts = D.x[0] * D.x[1] * D.x[2];
  int64_t tmax = eval_chain_max(D, true);
  int64_t tmax2 = eval_chain_max(D, false);
  if (tmax2 > tmax) tmax = tmax2;
  for (int j = 0; j < p->n_theta; ++j) ws.take<double>(npts);
  for (int i = 0; i < p->n_eta; ++i) ws.take<double>(npts);
  ws.take<double>(tmax);
  ws.take<double>(tmax);
  return ws.used + 256;
}

size_t generic_eval_workspace(const igs_problem* p, const Dims& D) {
  (void)p;
  Workspace ws(nullptr, 0, true);
  int64_t tmax = eval_chain_max(D, true);
  ws.take<double>(tmax);
  ws.take<double>(tmax);
  return ws.used + 256;
}

igs_status generic_apply(const igs_problem* p, const Dims& D, const double* planes,
                         const double* x, double* y, void* wsp, size_t ws_bytes, int flags,
                         cudaStream_t s) {
  Workspace ws(wsp, ws_bytes);
  int64_t npts = D.x[0] * D.x[1] * D.x[2];
  int64_t tmax = eval_chain_max(D, true);
  int64_t tmax2 = eval_chain_max(D, false);
  if (tmax2 > tmax) tmax = tmax2;
  double* u[IGS_MAX_DERIV_SET] = {};
  double* g[IGS_MAX_DERIV_SET] = {};
  for (int j = 0; j < p->n_theta; ++j) u[j] = ws.take<double>(npts);
  for (int i = 0; i < p->n_eta; ++i) g[i] = ws.take<double>(npts);
  double* tA = ws.take<double>(tmax);
  double* tB = ws.take<double>(tmax);
  if (!ws.ok()) return fail(IGS_EWORKSPACE, "workspace too small for the generic apply");
  const int64_t ny = D.ns[0] * D.ns[1] * D.ns[2];
  bool accumulate = (flags & IGS_FLAG_ACCUMULATE) != 0;
  bool any_block = false;
  for (int i = 0; i < p->n_eta; ++i) any_block |= eta_used(p, i);
  if (!any_block || npts == 0) {
    if (!accumulate) IGS_TRY(cuda_check(cudaMemsetAsync(y, 0, ny * sizeof(double), s), "memset y"));
    return IGS_OK;
  }
  // 1) interpolate every needed trial derivative to the points (Alg. 3)
  for (int j = 0; j < p->n_theta; ++j) {
    if (!theta_used(p, j)) { u[j] = nullptr; continue; }
    IGS_TRY(eval_chain(p, D, p->theta[j], x, u[j], tA, tB, s));
  }
  // 2) pointwise coefficient application
  PointwiseArgs a{};
  a.n_theta = p->n_theta; a.n_eta = p->n_eta;
  for (int i = 0; i < IGS_MAX_DERIV_SET; ++i)
    for (int j = 0; j < IGS_MAX_DERIV_SET; ++j) a.plane_of[i][j] = p->plane_of[i][j];
  a.planes = planes; a.plane_stride = p->plane_stride;
  for (int j = 0; j < p->n_theta; ++j) a.u[j] = u[j];
  for (int i = 0; i < p->n_eta; ++i) a.g[i] = eta_used(p, i) ? g[i] : nullptr;
  for (int k = 0; k < 3; ++k) {
    a.w[k] = k < p->d ? p->trial[k].weights : nullptr;
    a.x[k] = D.x[k];
  }
  a.x_off_last = D.x_off;
  a.d = p->d;
  pointwise_kernel<<<grid_for(npts, 256), 256, 0, s>>>(a);
  IGS_LAUNCH_CHECK("pointwise_kernel");
  // 3) test back, direction by direction, summing over eta into y
  bool written = false;
  for (int i = 0; i < p->n_eta; ++i) {
    if (!a.g[i]) continue;
    int64_t shape[3] = {D.x[0], D.x[1], D.x[2]};
    const double* src = g[i];
    for (int k = 0; k < p->d; ++k) {
      bool last = (k == p->d - 1);
      double* dst = last ? y : ((k % 2 == 0) ? tA : tB);
      int acc = last ? ((written || accumulate) ? 1 : 0) : 0;
      Op1D op = test_op(p, D, k, p->eta[i][k]);
      IGS_TRY(launch_contract(MODE_TEST, op, src, dst, shape, k, D.ns[k], acc, s));
      shape[k] = D.ns[k];
      src = dst;
    }
    written = true;
  }
  return IGS_OK;
}

igs_status generic_eval_field(const igs_problem* p, const Dims& D, const int8_t* deriv,
                              const double* coeffs, double* out, void* wsp, size_t ws_bytes,
                              cudaStream_t s) {
  Workspace ws(wsp, ws_bytes);
  int64_t tmax = eval_chain_max(D, true);
  double* tA = ws.take<double>(tmax);
  double* tB = ws.take<double>(tmax);
  if (!ws.ok()) return fail(IGS_EWORKSPACE, "workspace too small for eval_field");
  return eval_chain(p, D, deriv, coeffs, out, tA, tB, s);
}

// ---- assembly ----------------------------------------------------------

namespace {
int64_t assemble_chain_max(const igs_problem* p, const Dims& D) {
  int64_t s[3] = {D.x[0], D.x[1], D.x[2]};
  int64_t mx = prod3(s);
  for (int k = 0; k < p->d; ++k) {
    int dd = p->dir_order[k];
    s[dd] = p->num_pairs[dd];
    mx = mx > prod3(s) ? mx : prod3(s);
  }
  return mx;
}
}  // namespace

size_t generic_assemble_workspace(const igs_problem* p, const Dims& D) {
  Workspace ws(nullptr, 0, true);
  int64_t P = 1;
  for (int k = 0; k < p->d; ++k) P *= p->num_pairs[k];
  int64_t tmax = assemble_chain_max(p, D);
  ws.take<double>(P);
  ws.take<double>(tmax);
  ws.take<double>(tmax);
  for (int k = 0; k < p->d; ++k) ws.take<int64_t>(p->num_pairs[k]);
  return ws.used + 256;
}

igs_status generic_assemble(const igs_problem* p, const Dims& D, const int64_t* const* rowptr1d,
                            const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                            int block_eta, int block_theta, const double* planes, double* values,
                            void* wsp, size_t ws_bytes, cudaStream_t s) {
  Workspace ws(wsp, ws_bytes);
  int64_t P = 1;
  for (int k = 0; k < p->d; ++k) P *= p->num_pairs[k];
  int64_t tmax = assemble_chain_max(p, D);
  double* acc = ws.take<double>(P);
  double* tA = ws.take<double>(tmax);
  double* tB = ws.take<double>(tmax);
  int64_t* pair_m[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < p->d; ++k) pair_m[k] = ws.take<int64_t>(p->num_pairs[k]);
  if (!ws.ok()) return fail(IGS_EWORKSPACE, "workspace too small for the generic assembly");
  if (P == 0) return IGS_OK;
  for (int k = 0; k < p->d; ++k) {
    int64_t nr = D.ns[k];
    pair_rows_kernel<<<(unsigned)ceil_div(nr, 128), 128, 0, s>>>(rowptr1d[k], nr, pair_m[k]);
    IGS_LAUNCH_CHECK("pair_rows_kernel");
  }
  IGS_TRY(cuda_check(cudaMemsetAsync(acc, 0, P * sizeof(double), s), "memset acc"));
  // Blocks in the reference's loop order: theta outer, eta inner
  // (sumfac.py:220-224); exactly-zero blocks skipped.
  for (int j = 0; j < p->n_theta; ++j) {
    for (int i = 0; i < p->n_eta; ++i) {
      if (block_eta >= 0 && (i != block_eta || j != block_theta)) continue;
      int pl = p->plane_of[i][j];
      if (pl < 0) continue;
      int64_t shape[3] = {D.x[0], D.x[1], D.x[2]};
      const double* src = planes + pl * p->plane_stride;
      for (int kk = 0; kk < p->d; ++kk) {
        int k = p->dir_order[kk];
        bool last = (kk == p->d - 1);
        double* dst = last ? acc : ((kk % 2 == 0) ? tA : tB);
        Op1D op{};
        const igs_dir& tr = p->trial[k];
        const igs_dir& te = p->test[k];
        op.vt = tr.values; op.fat = tr.first_active; op.pt = tr.order; op.kt = p->theta[j][k];
        op.vs = te.values; op.fas = te.first_active; op.ps = te.order; op.ks = p->eta[i][k];
        op.w = tr.weights;
        op.xtab = tr.num_points;
        op.x_loc = D.x[k];
        op.pair_n = cols1d[k];
        op.pair_m = pair_m[k];
        IGS_TRY(launch_contract(MODE_PAIR, op, src, dst, shape, k, p->num_pairs[k], last ? 1 : 0, s));
        shape[k] = p->num_pairs[k];
        src = dst;
      }
    }
  }
  TensorPat t;
  t.d = p->d;
  for (int k = 0; k < 3; ++k) {
    t.rp[k] = k < p->d ? rowptr1d[k] : nullptr;
    t.cl[k] = k < p->d ? cols1d[k] : nullptr;
    t.ns[k] = D.ns[k];
    t.nt[k] = D.nt[k];
  }
  int64_t P0 = p->num_pairs[0], P1 = p->d > 1 ? p->num_pairs[1] : 1, P2 = p->d > 2 ? p->num_pairs[2] : 1;
  scatter_csr_kernel<<<grid_for(P, 256), 256, 0, s>>>(t, pair_m[0], pair_m[1], pair_m[2], acc, P0,
                                                       P1, P2, row_lo, row_hi, values);
  IGS_LAUNCH_CHECK("scatter_csr_kernel");
  return IGS_OK;
}

}  // namespace igs
