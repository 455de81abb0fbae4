// the reference's independent comparison oracles,
// assemble_naive (sumfac.py:388-477) and assemble_kronecker_dense
// (:480-509), as one direct-quadrature kernel: every CSR entry (m, n) sums
//
//   Σ_{(θ,η) blocks, F ≠ 0} Σ_x  Π_δ w_δ(x_δ) B^{θ_δ}_{n_δ}(x_δ) B^{η_δ}_{m_δ}(x_δ) · F_{η,θ}(x)
//
// over the box of points where both supports overlap — the reference's
// _support_column_ranges (sumfac.py:382-385: searchsorted of the knot
// supports in the points), so the update counter it records matches too.
// Independent of Alg. 1 (no W operators, no intermediates): it is the GPU
// cross-check of K3 at small sizes, not a fast path.
#include "igs_internal.cuh"

namespace igs {
namespace {

struct NaiveArgs {
  igs_problem p;
  const int64_t* indptr;
  const void* indices;
  int ibytes;
  int64_t row_lo, row_hi;       // rows; entries [e_lo, e_hi) = indptr[row_lo], indptr[row_hi]
  int64_t e_lo, e_hi;
  const double* planes;
  double* values;
  unsigned long long* updates;  // Σ over (entry, block) of the box sizes (nullable)
};

__device__ __forceinline__ int64_t lower_bound(const double* a, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t upper_bound(const double* a, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// B^{k}_n(x) from the banded table (0 outside the band)
__device__ __forceinline__ double band(const igs_dir& t, int k, int64_t n, int64_t x) {
  const int64_t j = n - t.first_active[x];
  if (j < 0 || j >= t.order || k > t.max_deriv) return 0.0;
  return t.values[((int64_t)k * t.order + j) * t.num_points + x];
}

__global__ void naive_kernel(const NaiveArgs a) {
  const igs_problem& p = a.p;
  const int d = p.d;
  for (int64_t e = a.e_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.e_hi;
       e += (int64_t)gridDim.x * blockDim.x) {
    // row of entry e: largest m in [row_lo, row_hi) with indptr[m] <= e
    int64_t l = a.row_lo, r = a.row_hi;
    while (r - l > 1) {
      const int64_t mid = (l + r) >> 1;
      if (a.indptr[mid] <= e) l = mid; else r = mid;
    }
    const int64_t m = l;
    const int64_t n = a.ibytes == 4 ? (int64_t)static_cast<const int32_t*>(a.indices)[e]
                                    : static_cast<const int64_t*>(a.indices)[e];
    int64_t mi[3] = {0, 0, 0}, ni[3] = {0, 0, 0}, x0[3] = {0, 0, 0}, x1[3] = {1, 1, 1};
    int64_t mr = m, nr = n;
    bool empty = false;
    for (int k = 0; k < d; ++k) {
      mi[k] = mr % p.test[k].num_basis;
      mr /= p.test[k].num_basis;
      ni[k] = nr % p.trial[k].num_basis;
      nr /= p.trial[k].num_basis;
      const igs_dir& tt = p.trial[k];
      const igs_dir& ts = p.test[k];
      const int64_t X = tt.num_points;
      const int64_t lt = lower_bound(tt.points, X, tt.csupp_lo[ni[k]]);
      const int64_t ht = upper_bound(tt.points, X, tt.csupp_hi[ni[k]]);
      const int64_t ls = lower_bound(ts.points, X, ts.csupp_lo[mi[k]]);
      const int64_t hs = upper_bound(ts.points, X, ts.csupp_hi[mi[k]]);
      x0[k] = lt > ls ? lt : ls;
      x1[k] = ht < hs ? ht : hs;
      if (x1[k] <= x0[k]) empty = true;
    }
    double val = 0.0;
    unsigned long long upd = 0;
    if (!empty) {
      const int64_t box = (x1[0] - x0[0]) * (x1[1] - x0[1]) * (x1[2] - x0[2]);
      const int64_t X0 = p.trial[0].num_points;
      const int64_t X1 = d > 1 ? p.trial[1].num_points : 1;
      for (int j = 0; j < p.n_theta; ++j)
        for (int i = 0; i < p.n_eta; ++i) {
          const int pl = p.plane_of[i][j];
          if (pl < 0) continue;
          const double* F = a.planes + (int64_t)pl * p.plane_stride;
          double s2 = 0.0;
          for (int64_t z = x0[2]; z < x1[2]; ++z) {
            double f2 = 1.0;
            if (d > 2)
              f2 = p.test[2].weights[z] * band(p.trial[2], p.theta[j][2], ni[2], z) *
                   band(p.test[2], p.eta[i][2], mi[2], z);
            double s1 = 0.0;
            for (int64_t y = x0[1]; y < x1[1]; ++y) {
              double f1 = 1.0;
              if (d > 1)
                f1 = p.test[1].weights[y] * band(p.trial[1], p.theta[j][1], ni[1], y) *
                     band(p.test[1], p.eta[i][1], mi[1], y);
              double s0 = 0.0;
              const double* Fr = F + (z * X1 + y) * X0;
              for (int64_t x = x0[0]; x < x1[0]; ++x) {
                const double f0 = p.test[0].weights[x] * band(p.trial[0], p.theta[j][0], ni[0], x) *
                                  band(p.test[0], p.eta[i][0], mi[0], x);
                s0 = fma(f0, Fr[x], s0);
              }
              s1 = fma(f1, s0, s1);
            }
            s2 = fma(f2, s1, s2);
          }
          val += s2;
          upd += (unsigned long long)box;
        }
    }
    a.values[e - a.e_lo] = val;
    if (a.updates && upd) atomicAdd(a.updates, upd);
  }
}

}  // namespace
}  // namespace igs

using namespace igs;

extern "C" igs_status igs_assemble_naive(const igs_problem* prob, const int64_t* indptr, const void* indices,
                                         int32_t index_bytes, int64_t row_lo, int64_t row_hi, int64_t entry_lo,
                                         int64_t entry_hi, const double* planes, double* values,
                                         uint64_t* updates, void* stream) {
  if (!prob || !indptr) return fail(IGS_EARG, "null argument");
  if (row_lo < 0 || row_hi < row_lo) return fail(IGS_EARG, "bad row range");
  if (prob->d < 1 || prob->d > 3) return fail(IGS_EARG, "dimension must be 1..3");
  if (index_bytes != 4 && index_bytes != 8) return fail(IGS_EARG, "index_bytes must be 4 or 8");
  if (prob->slab_lo != prob->slab_hi) return fail(IGS_EARG, "the naive oracle takes whole fields (no slab)");
  for (int k = 0; k < prob->d; ++k) {
    const igs_dir& t = prob->trial[k];
    const igs_dir& s = prob->test[k];
    if (t.num_points != s.num_points) return fail(IGS_EARG, "trial/test point counts differ");
    if (!t.points || !s.points || !t.csupp_lo || !s.csupp_lo || !t.csupp_hi || !s.csupp_hi || !s.weights)
      return fail(IGS_EARG, "naive oracle needs points, weights and knot supports");
  }
  const int64_t e_lo = entry_lo, e_hi = entry_hi;
  if (e_hi < e_lo || e_lo < 0) return fail(IGS_EARG, "bad entry range");
  const int64_t n = e_hi - e_lo;
  if (n == 0) return IGS_OK;
  if (!indices || !values || (!planes && prob->n_planes > 0)) return fail(IGS_EARG, "null argument");
  NaiveArgs a{};
  a.p = *prob;
  a.indptr = indptr;
  a.indices = indices;
  a.ibytes = index_bytes;
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  a.e_lo = e_lo;
  a.e_hi = e_hi;
  a.planes = planes;
  a.values = values;
  a.updates = reinterpret_cast<unsigned long long*>(updates);
  cudaStream_t st = as_stream(stream);
  const int64_t blocks = min64(ceil_div(n, 128), 148 * 32);
  naive_kernel<<<(unsigned)blocks, 128, 0, st>>>(a);
  IGS_LAUNCH_CHECK("naive_kernel");
  return IGS_OK;
}
