/*
 * Stand-alone C use of libigs_b200.so (no Python): the C-ABI alone builds a
 * 3D mass+stiffness problem (Gauss rules, tables, synthetic coefficients),
 * applies it matrix-free and assembles it, then checks two identities:
 *   1ᵀ A 1 = Σ_x w(x)·c(x)   (the stiffness part annihilates constants)
 *   the CSR matvec of the assembled values equals the apply, ≤ 1e-12.
 * Build (tests/test_capi_c_example.py does this on the GPU box):
 *   gcc -O2 tools/capi_example.c -Iinclude -I$CUDA/include -Lpaper_1809_05471_b200 -ligs_b200
 *       -L$CUDA/lib64 -lcudart -Wl,-rpath,... -o capi_example
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "igs_capi.h"

#define CHECK(x)                                                          \
  do {                                                                    \
    igs_status s_ = (x);                                                  \
    if (s_ != IGS_OK) {                                                   \
      fprintf(stderr, "%s failed: %s\n", #x, igs_last_error());           \
      return 1;                                                           \
    }                                                                     \
  } while (0)

static void* dmalloc(size_t bytes) {
  void* p = NULL;
  if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    exit(1);
  }
  return p;
}

static void* upload(const void* host, size_t bytes) {
  void* d = dmalloc(bytes);
  cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice);
  return d;
}

int main(void) {
  const int d = 3, p = 4, K = 6, k = 4;
  const int nknots = K + 2 * p - 1, N = K + p - 1, X = K * k, nbp = K + 1;
  double knots[64], bp[64], lo[64], hi[64];
  for (int i = 0; i < nknots; ++i) {
    int j = i - (p - 1);
    knots[i] = j <= 0 ? 0.0 : (j >= K ? 1.0 : (double)j / K);
  }
  for (int i = 0; i < nbp; ++i) bp[i] = (double)i / K;
  for (int n = 0; n < N; ++n) {
    lo[n] = knots[n];
    hi[n] = knots[n + p];
  }
  double* dknots = upload(knots, nknots * sizeof(double));
  double* dbp = upload(bp, nbp * sizeof(double));
  double* dlo = upload(lo, N * sizeof(double));
  double* dhi = upload(hi, N * sizeof(double));
  double* pts = dmalloc(X * sizeof(double));
  double* wts = dmalloc(X * sizeof(double));
  double* vals = dmalloc(2 * p * X * sizeof(double));
  int64_t* first = dmalloc(X * sizeof(int64_t));
  CHECK(igs_gauss_rule(k, dbp, nbp, pts, wts, NULL));
  CHECK(igs_tabulate(p, dknots, nknots, pts, X, 1, vals, first, NULL));

  igs_problem prob;
  memset(&prob, 0, sizeof(prob));
  prob.d = d;
  for (int a = 0; a < d; ++a) {
    igs_dir t;
    memset(&t, 0, sizeof(t));
    t.order = p;
    t.num_basis = N;
    t.num_points = X;
    t.max_deriv = 1;
    t.values = vals;
    t.first_active = first;
    t.weights = wts;
    t.csupp_lo = dlo;
    t.csupp_hi = dhi;
    t.points = pts;
    t.num_elements = K;
    t.points_per_element = k;
    t.uniform = 1;
    prob.trial[a] = t;
    prob.test[a] = t;
    prob.dir_order[a] = a;
  }
  /* first-order set (value, d/dx0, d/dx1, d/dx2); planes [c, a00, a11, a22, a01, a02, a12] */
  prob.n_theta = prob.n_eta = d + 1;
  for (int i = 0; i <= d; ++i)
    for (int a = 0; a < d; ++a) prob.theta[i][a] = prob.eta[i][a] = (int8_t)(i == a + 1);
  memset(prob.plane_of, -1, sizeof(prob.plane_of));
  int pl = 0;
  prob.plane_of[0][0] = (int8_t)pl++;
  for (int a = 0; a < d; ++a) prob.plane_of[1 + a][1 + a] = (int8_t)pl++;
  for (int a = 0; a < d; ++a)
    for (int b = a + 1; b < d; ++b) {
      prob.plane_of[1 + a][1 + b] = prob.plane_of[1 + b][1 + a] = (int8_t)pl;
      ++pl;
    }
  prob.n_planes = pl;
  const int64_t npts = (int64_t)X * X * X, ndof = (int64_t)N * N * N;
  prob.plane_stride = npts;

  double* planes = dmalloc((size_t)pl * npts * sizeof(double));
  const int64_t dims[3] = {X, X, X};
  CHECK(igs_fill_synthetic(d, dims, 0, X, 3, 7ull, planes, npts, NULL));

  /* 1D patterns (two-phase) -> tensor CSR */
  int64_t* rp[3];
  int64_t* cl[3];
  for (int a = 0; a < d; ++a) {
    int64_t cnt = 0;
    rp[a] = dmalloc((N + 1) * sizeof(int64_t));
    CHECK(igs_pattern_1d(&prob, a, rp[a], NULL, &cnt, NULL));
    cl[a] = dmalloc(cnt * sizeof(int64_t));
    CHECK(igs_pattern_1d(&prob, a, rp[a], cl[a], &cnt, NULL));
    prob.num_pairs[a] = cnt;
  }
  int64_t nnz = prob.num_pairs[0] * prob.num_pairs[1] * prob.num_pairs[2];
  int64_t* indptr = dmalloc((ndof + 1) * sizeof(int64_t));
  int64_t* indices = dmalloc(nnz * sizeof(int64_t));
  CHECK(igs_pattern(&prob, (const int64_t* const*)rp, (const int64_t* const*)cl, 0, ndof, 0, indptr, indices, 8,
                    NULL));

  /* apply to 1 and to a pseudo-random vector */
  size_t wsa = igs_workspace_bytes(&prob, IGS_OP_APPLY, 0);
  size_t wsb = igs_workspace_bytes(&prob, IGS_OP_ASSEMBLE, 0);
  void* ws = dmalloc(wsa > wsb ? wsa : wsb);
  double* hx = malloc(ndof * sizeof(double));
  double* hy = malloc(ndof * sizeof(double));
  for (int64_t i = 0; i < ndof; ++i) hx[i] = 1.0;
  double* x = upload(hx, ndof * sizeof(double));
  double* y = dmalloc(ndof * sizeof(double));
  CHECK(igs_apply(&prob, planes, x, y, ws, wsa, 0, NULL));
  cudaMemcpy(hy, y, ndof * sizeof(double), cudaMemcpyDeviceToHost);
  double total = 0.0;
  for (int64_t i = 0; i < ndof; ++i) total += hy[i];
  /* Σ_x w(x) c(x) from the device planes and weights */
  double* hc = malloc(npts * sizeof(double));
  double hw[64];
  cudaMemcpy(hc, planes, npts * sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(hw, wts, X * sizeof(double), cudaMemcpyDeviceToHost);
  double mass = 0.0;
  for (int64_t q = 0; q < npts; ++q) mass += hw[q % X] * hw[(q / X) % X] * hw[q / ((int64_t)X * X)] * hc[q];
  printf("1^T A 1 = %.15f, sum w c = %.15f\n", total, mass);
  if (fabs(total - mass) > 1e-12 * fabs(mass)) {
    fprintf(stderr, "measure identity violated\n");
    return 1;
  }

  /* assembled values: CSR matvec on the host equals the apply */
  unsigned long long r = 88172645463325252ull;
  for (int64_t i = 0; i < ndof; ++i) {
    r ^= r << 13;
    r ^= r >> 7;
    r ^= r << 17;
    hx[i] = (double)(r >> 11) / 9007199254740992.0 - 0.5;
  }
  cudaMemcpy(x, hx, ndof * sizeof(double), cudaMemcpyHostToDevice);
  CHECK(igs_apply(&prob, planes, x, y, ws, wsa, 0, NULL));
  cudaMemcpy(hy, y, ndof * sizeof(double), cudaMemcpyDeviceToHost);
  double* values = dmalloc(nnz * sizeof(double));
  CHECK(igs_assemble_values(&prob, (const int64_t* const*)rp, (const int64_t* const*)cl, 0, ndof, -1, -1, planes,
                            values, ws, wsb, 0, NULL));
  double* hv = malloc(nnz * sizeof(double));
  int64_t* hp = malloc((ndof + 1) * sizeof(int64_t));
  int64_t* hi_ = malloc(nnz * sizeof(int64_t));
  cudaMemcpy(hv, values, nnz * sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(hp, indptr, (ndof + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost);
  cudaMemcpy(hi_, indices, nnz * sizeof(int64_t), cudaMemcpyDeviceToHost);
  double num = 0.0, den = 0.0;
  for (int64_t m = 0; m < ndof; ++m) {
    double s = 0.0;
    for (int64_t e = hp[m]; e < hp[m + 1]; ++e) s += hv[e] * hx[hi_[e]];
    num += (s - hy[m]) * (s - hy[m]);
    den += hy[m] * hy[m];
  }
  printf("nnz %lld, |CSR x - apply x| / |apply x| = %.3e\n", (long long)nnz, sqrt(num / den));
  if (!(sqrt(num / den) <= 1e-12)) {
    fprintf(stderr, "assembly and apply disagree\n");
    return 1;
  }
  printf("capi example ok\n");
  return 0;
}
