// K2 — sparsity patterns.
//
//   igs_pattern_1d : the 1D interaction set {(n,m) : X ∩ csupp φ_n ∩ csupp ψ_m ≠ ∅}
//                    (tensorspace.py:168-208, Lemma 3.1).  Because csupp
//                    endpoints are non-decreasing in the function index, the
//                    trial functions meeting row m form a window found by two
//                    binary searches; each candidate is then checked exactly.
//   igs_pattern    : the tensor CSR (tensorspace.py:262-338).  Instead of the
//                    reference's lexsort, row offsets are closed-form products
//                    of the 1D row pointers:
//                      indptr[m] = rp0[m0]·w1·w2 + P0·rp1[m1]·w2 + P0·P1·rp2[m2]
//                    and column lists are Cartesian products of the 1D lists
//                    with direction 0 fastest, so every row comes out sorted.
#include "igs_internal.cuh"

#include <cub/device/device_scan.cuh>

namespace igs {
namespace {

__device__ __forceinline__ int64_t lower_bound_d(const double* a, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound_d(const double* a, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct Pat1DArgs {
  const double* pts; int64_t npts;
  const double* lo_t; const double* hi_t; int64_t nt;
  const double* lo_s; const double* hi_s; int64_t ns;
};

// Enumerates the trial functions of test row m; writes them if `cols`.
__device__ int64_t row_pairs(const Pat1DArgs& a, int64_t m, int64_t* cols) {
  int64_t ia = lower_bound_d(a.pts, a.npts, a.lo_s[m]);
  int64_t ib = upper_bound_d(a.pts, a.npts, a.hi_s[m]);
  if (ia >= ib) return 0;
  double x_first = a.pts[ia], x_last = a.pts[ib - 1];
  int64_t n_min = lower_bound_d(a.hi_t, a.nt, x_first);        // first n with hi >= x_first
  int64_t n_max = upper_bound_d(a.lo_t, a.nt, x_last) - 1;     // last n with lo <= x_last
  int64_t c = 0;
  for (int64_t n = n_min; n <= n_max; ++n) {
    int64_t ja = lower_bound_d(a.pts, a.npts, a.lo_t[n]);
    int64_t jb = upper_bound_d(a.pts, a.npts, a.hi_t[n]);
    if (ja < jb && (ja > ia ? ja : ia) < (jb < ib ? jb : ib)) {
      if (cols) cols[c] = n;
      ++c;
    }
  }
  return c;
}

__global__ void pat1d_count(Pat1DArgs a, int64_t* counts) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m < a.ns) counts[m] = row_pairs(a, m, nullptr);
  if (m == a.ns) counts[m] = 0;
}

__global__ void pat1d_fill(Pat1DArgs a, const int64_t* rowptr, int64_t* cols) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m < a.ns) row_pairs(a, m, cols + rowptr[m]);
}

__global__ void tensor_indptr(TensorPat t, int64_t row_lo, int64_t row_hi, int relative,
                              int64_t* indptr) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t nrows = row_hi - row_lo;
  if (r > nrows) return;
  int64_t w[3], mi[3];
  int64_t base = 0;
  if (relative) base = tensor_row_start(t, row_lo, w, mi);
  int64_t total_rows = t.ns[0] * t.ns[1] * t.ns[2];
  int64_t m = row_lo + r;
  int64_t v;
  if (m >= total_rows) {
    int64_t P = 1;
    for (int k = 0; k < t.d; ++k) P *= t.rp[k][t.ns[k]];
    v = P;
  } else {
    v = tensor_row_start(t, m, w, mi);
  }
  indptr[r] = v - base;
}

// One warp per row: lanes stride over the row's w0*w1*w2 entries, so the
// stores of a row are contiguous and coalesced.
template <class IndexT>
__global__ void tensor_indices(TensorPat t, int64_t row_lo, int64_t nrows,
                               IndexT* __restrict__ out) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= nrows) return;
  int64_t w[3], mi[3];
  int64_t base = tensor_row_start(t, row_lo, w, mi);
  int64_t m = row_lo + warp;
  int64_t start = tensor_row_start(t, m, w, mi);
  int64_t width = w[0] * w[1] * w[2];
  const int64_t* c0 = t.cl[0] + t.rp[0][mi[0]];
  const int64_t* c1 = t.d > 1 ? t.cl[1] + t.rp[1][mi[1]] : nullptr;
  const int64_t* c2 = t.d > 2 ? t.cl[2] + t.rp[2][mi[2]] : nullptr;
  for (int64_t e = lane; e < width; e += 32) {
    int64_t e0 = e % w[0], e1 = (e / w[0]) % w[1], e2 = e / (w[0] * w[1]);
    int64_t n0 = c0[e0];
    int64_t n1 = c1 ? c1[e1] : 0;
    int64_t n2 = c2 ? c2[e2] : 0;
    out[start - base + e] = (IndexT)(n0 + t.nt[0] * (n1 + t.nt[1] * n2));
  }
}

}  // namespace
}  // namespace igs

using namespace igs;

extern "C" igs_status igs_pattern_1d(const igs_problem* prob, int32_t dir, int64_t* rowptr,
                                     int64_t* cols, int64_t* count, void* stream) {
  IGS_TRY(validate_problem(prob, nullptr, 0));
  if (dir < 0 || dir >= prob->d) return fail(IGS_EARG, "direction out of range");
  const igs_dir& tr = prob->trial[dir];
  const igs_dir& te = prob->test[dir];
  if (!tr.csupp_lo || !tr.csupp_hi || !te.csupp_lo || !te.csupp_hi || (!tr.points && tr.num_points))
    return fail(IGS_EARG, "pattern needs csupp and point arrays");
  if (!rowptr) return fail(IGS_EARG, "null rowptr");
  cudaStream_t s = as_stream(stream);
  Pat1DArgs a{tr.points, tr.num_points, tr.csupp_lo, tr.csupp_hi, tr.num_basis,
              te.csupp_lo, te.csupp_hi, te.num_basis};
  int block = 128;
  if (cols == nullptr) {
    // Phase 1: counts -> exclusive scan in place (rowptr has ns+1 slots).
    pat1d_count<<<(unsigned)ceil_div(a.ns + 1, block), block, 0, s>>>(a, rowptr);
    IGS_LAUNCH_CHECK("pat1d_count");
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rowptr, rowptr, (int)(a.ns + 1), s);
    void* tmp = nullptr;
    IGS_TRY(cuda_check(cudaMallocAsync(&tmp, tmp_bytes, s), "cudaMallocAsync"));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, rowptr, rowptr, (int)(a.ns + 1), s);
    cudaFreeAsync(tmp, s);
    IGS_LAUNCH_CHECK("pattern scan");
    if (count) {
      IGS_TRY(cuda_check(cudaMemcpyAsync(count, rowptr + a.ns, sizeof(int64_t),
                                         cudaMemcpyDeviceToHost, s), "count copy"));
      IGS_TRY(cuda_check(cudaStreamSynchronize(s), "pattern sync"));
    }
    return IGS_OK;
  }
  pat1d_fill<<<(unsigned)ceil_div(a.ns, block), block, 0, s>>>(a, rowptr, cols);
  IGS_LAUNCH_CHECK("pat1d_fill");
  return IGS_OK;
}

extern "C" igs_status igs_pattern(const igs_problem* prob, const int64_t* const* rowptr1d,
                                  const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                                  int32_t relative, int64_t* indptr, void* indices,
                                  int32_t index_bytes, void* stream) {
  Dims D;
  IGS_TRY(validate_problem(prob, &D, 0));
  if (prob->slab_lo != 0 || prob->slab_hi != 0)
    return fail(IGS_EARG, "igs_pattern works on the full problem; use row ranges to partition");
  if (index_bytes != 4 && index_bytes != 8) return fail(IGS_EARG, "index_bytes must be 4 or 8");
  int64_t nrows_total = D.ns[0] * D.ns[1] * D.ns[2];
  if (row_lo < 0 || row_hi < row_lo || row_hi > nrows_total) return fail(IGS_EARG, "row range");
  int64_t ncols_total = D.nt[0] * D.nt[1] * D.nt[2];
  if (index_bytes == 4 && ncols_total > INT32_MAX)
    return fail(IGS_ECAPACITY, "int32 column indices overflow");
  TensorPat t;
  t.d = prob->d;
  for (int k = 0; k < 3; ++k) {
    t.rp[k] = k < t.d ? rowptr1d[k] : nullptr;
    t.cl[k] = k < t.d ? cols1d[k] : nullptr;
    t.ns[k] = D.ns[k];
    t.nt[k] = D.nt[k];
  }
  cudaStream_t s = as_stream(stream);
  int block = 256;
  int64_t nrows = row_hi - row_lo;
  if (indptr) {
    tensor_indptr<<<(unsigned)ceil_div(nrows + 1, block), block, 0, s>>>(t, row_lo, row_hi,
                                                                         relative, indptr);
    IGS_LAUNCH_CHECK("tensor_indptr");
  }
  if (indices && nrows > 0) {
    int64_t threads = nrows * 32;
    if (index_bytes == 4) {
      tensor_indices<int32_t><<<(unsigned)ceil_div(threads, block), block, 0, s>>>(
          t, row_lo, nrows, (int32_t*)indices);
    } else {
      tensor_indices<int64_t><<<(unsigned)ceil_div(threads, block), block, 0, s>>>(
          t, row_lo, nrows, (int64_t*)indices);
    }
    IGS_LAUNCH_CHECK("tensor_indices");
  }
  return IGS_OK;
}
