// K1 — Gauss-Legendre rules per element and banded B-spline tabulation.
//
// Compiled with -fmad=false so that every +,-,*,/ is an individually
// rounded IEEE operation, like the reference's Python float arithmetic:
// the tables then agree with bspline.tabulate to the last bit or two.
//
//   igs_gauss_rule : quadrature.py:34-65 (Newton on the Legendre recurrence,
//                    tolerance 1e-15, <= 100 steps, mirrored halves) and
//                    quadrature.py:87-106 (affine map into every element).
//   igs_tabulate   : bspline.py:314-333 over eval_all_derivs
//                    (bspline.py:169-239, the de Boor triangle + derivative
//                    recurrence, NURBS book A2.3) and find_span
//                    (bspline.py:153-166).
// One thread per point; setup-time kernels (tables are tiny: <= 131 KB at
// every BASELINE config), so they favour exactness over throughput.
#include "igs_internal.cuh"

namespace igs {
namespace {

constexpr int kMaxOrder = IGS_MAX_ORDER;

__global__ void gauss_rule_kernel(int k, const double* __restrict__ bp, int nel,
                                  double* __restrict__ pts, double* __restrict__ wts) {
  // Thread t handles reference node i (one half, mirrored) for element e.
  int half = (k + 1) / 2;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)half * nel) return;
  int i = (int)(t % half);
  int e = (int)(t / half);
  bool middle = (2 * i + 1 == k);
  const double pi = 3.141592653589793;
  double x = middle ? 0.0 : cos(pi * (i + 0.75) / (k + 0.5));
  double dp = 1.0;
  for (int it = 0; it < 100; ++it) {
    double p0 = 1.0, p1 = 0.0;
    for (int j = 1; j <= k; ++j) {
      double pn = ((2 * j - 1) * x * p0 - (j - 1) * p1) / j;
      p1 = p0;
      p0 = pn;
    }
    dp = k * (x * p0 - p1) / (x * x - 1.0);
    double dx = p0 / dp;
    x -= dx;
    if (fabs(dx) <= 1e-15) break;
  }
  if (middle) x = 0.0;
  double w = 2.0 / ((1.0 - x * x) * dp * dp);
  double node_lo = -fabs(x), node_hi = fabs(x);
  double lo = bp[e], hi = bp[e + 1];
  double mid = 0.5 * (lo + hi), hw = 0.5 * (hi - lo);
  int64_t base = (int64_t)e * k;
  pts[base + i] = mid + hw * node_lo;
  wts[base + i] = hw * w;
  pts[base + (k - 1 - i)] = mid + hw * node_hi;
  wts[base + (k - 1 - i)] = hw * w;
}

// Error flags written by the tabulation kernel (bitwise OR).
enum { kErrDomain = 1, kErrUnsorted = 2 };

__global__ void tabulate_kernel(int p, const double* __restrict__ U, int nknots,
                                const double* __restrict__ pts, int npts, int md,
                                double* __restrict__ values, int64_t* __restrict__ first,
                                int* __restrict__ err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  const int deg = p - 1;
  const int nbasis = nknots - p;
  const double a = U[0], b = U[nknots - 1];
  double x = pts[i];
  if (i + 1 < npts && pts[i + 1] < x) atomicOr(err, kErrUnsorted);
  if (!(a <= x && x <= b)) {
    atomicOr(err, kErrDomain);
    return;
  }
  // find_span: searchsorted(U, x, 'right') - 1, or N-1 at x == b.
  int span;
  if (x >= b) {
    span = nbasis - 1;
  } else {
    int lo = 0, hi = nknots;  // first index with U[idx] > x
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (U[mid] <= x) lo = mid + 1; else hi = mid;
    }
    span = lo - 1;
  }
  // de Boor triangle: ndu[j][r] holds basis values (upper) and knot
  // differences (lower).
  double ndu[kMaxOrder][kMaxOrder];
  double left[kMaxOrder], right[kMaxOrder];
  ndu[0][0] = 1.0;
  for (int j = 1; j < p; ++j) {
    left[j] = x - U[span + 1 - j];
    right[j] = U[span + j] - x;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      ndu[j][r] = right[r + 1] + left[j - r];
      double temp = ndu[r][j - 1] / ndu[j][r];
      ndu[r][j] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    ndu[j][j] = saved;
  }
  const int64_t stride_k = (int64_t)p * npts;
  for (int r = 0; r < p; ++r) values[(int64_t)r * npts + i] = ndu[r][deg];
  if (md > 0) {
    double ders[kMaxOrder][kMaxOrder];
    double acoef[2][kMaxOrder];
    for (int r = 0; r < p; ++r) {
      int s1 = 0, s2 = 1;
      acoef[0][0] = 1.0;
      for (int k = 1; k <= md; ++k) {
        double dd = 0.0;
        int rk = r - k, pk = deg - k;
        if (r >= k) {
          acoef[s2][0] = acoef[s1][0] / ndu[pk + 1][rk];
          dd = acoef[s2][0] * ndu[rk][pk];
        }
        int j1 = (rk >= -1) ? 1 : -rk;
        int j2 = (r - 1 <= pk) ? k - 1 : deg - r;
        for (int j = j1; j <= j2; ++j) {
          acoef[s2][j] = (acoef[s1][j] - acoef[s1][j - 1]) / ndu[pk + 1][rk + j];
          dd += acoef[s2][j] * ndu[rk + j][pk];
        }
        if (r <= pk) {
          acoef[s2][k] = -acoef[s1][k - 1] / ndu[pk + 1][r];
          dd += acoef[s2][k] * ndu[r][pk];
        }
        ders[k][r] = dd;
        int t = s1; s1 = s2; s2 = t;
      }
    }
    double fact = (double)deg;
    for (int k = 1; k <= md; ++k) {
      for (int r = 0; r < p; ++r) values[k * stride_k + (int64_t)r * npts + i] = ders[k][r] * fact;
      fact *= (double)(deg - k);
    }
  }
  first[i] = span - deg;
}

}  // namespace
}  // namespace igs

using namespace igs;

extern "C" igs_status igs_gauss_rule(int32_t k, const double* breakpoints, int32_t nbp,
                                     double* points, double* weights, void* stream) {
  if (k < 1 || k > 64) return fail(IGS_EARG, "node count outside [1, 64]");
  if (nbp < 2) return fail(IGS_EARG, "need at least 2 distinct breakpoints");
  if (!breakpoints || !points || !weights) return fail(IGS_EARG, "null pointer");
  int nel = nbp - 1;
  int64_t threads = (int64_t)((k + 1) / 2) * nel;
  int block = 128;
  gauss_rule_kernel<<<(unsigned)ceil_div(threads, block), block, 0, as_stream(stream)>>>(
      k, breakpoints, nel, points, weights);
  IGS_LAUNCH_CHECK("gauss_rule_kernel");
  return IGS_OK;
}

extern "C" igs_status igs_tabulate(int32_t order, const double* knots, int32_t nknots,
                                   const double* points, int32_t npts, int32_t max_deriv,
                                   double* values, int64_t* first_active, void* stream) {
  if (order < 1 || order > IGS_MAX_ORDER) return fail(IGS_ECAPACITY, "spline order outside [1, 16]");
  if (max_deriv < 0 || max_deriv >= order)
    return fail(IGS_EDERIV, "derivative order " + std::to_string(max_deriv) +
                                " not supported for spline order " + std::to_string(order));
  if (nknots < 2 * order) return fail(IGS_EARG, "need at least 2*order knots");
  if (npts == 0) return IGS_OK;
  if (!knots || !points || !values || !first_active) return fail(IGS_EARG, "null pointer");
  cudaStream_t s = as_stream(stream);
  int* err = nullptr;
  IGS_TRY(cuda_check(cudaMallocAsync(&err, sizeof(int), s), "cudaMallocAsync"));
  cudaMemsetAsync(err, 0, sizeof(int), s);
  int block = 128;
  tabulate_kernel<<<(unsigned)ceil_div(npts, block), block, 0, s>>>(
      order, knots, nknots, points, npts, max_deriv, values, first_active, err);
  igs_status st = cuda_check(cudaGetLastError(), "tabulate_kernel");
  int host_err = 0;
  cudaMemcpyAsync(&host_err, err, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(err, s);
  if (st != IGS_OK) return st;
  IGS_TRY(cuda_check(cudaStreamSynchronize(s), "tabulate sync"));
  if (host_err & kErrUnsorted) return fail(IGS_EARG, "points must be sorted ascending");
  if (host_err & kErrDomain) return fail(IGS_EDOMAIN, "point outside the basis domain");
  return IGS_OK;
}
