// Internal helpers shared by the libigs_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/igs_capi.h"

namespace igs {

// Thread-local last-error message (igs_last_error).
void set_error(const std::string& msg);
const std::string& get_error();

// Records `msg` and returns `s`; used as `return fail(IGS_EARG, "...")`.
inline igs_status fail(igs_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

inline igs_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return IGS_OK;
  return fail(IGS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define IGS_TRY(expr)                       \
  do {                                      \
    igs_status _s = (expr);                 \
    if (_s != IGS_OK) return _s;            \
  } while (0)

#define IGS_LAUNCH_CHECK(what) IGS_TRY(::igs::cuda_check(cudaGetLastError(), what))

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Bump allocator over the caller-provided workspace; 256-byte aligned.
struct Workspace {
  char* base;
  size_t cap;
  size_t used = 0;
  bool dry;  // dry run: only measure
  Workspace(void* b, size_t c, bool dry_run = false) : base((char*)b), cap(c), dry(dry_run) {}
  template <class T>
  T* take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + count * sizeof(T);
    if (dry) return nullptr;
    if (used > cap) return nullptr;
    return reinterpret_cast<T*>(base + off);
  }
  bool ok() const { return dry || used <= cap; }
};

// Number of DoFs / points of a problem, honouring the last-direction slab.
struct Dims {
  int d;
  int64_t nt[3];   // trial functions per direction (slab-restricted in the last dir)
  int64_t ns[3];   // test functions per direction
  int64_t x[3];    // points per direction (slab-restricted)
  int64_t x_off;   // first point layer of the slab (last direction)
  int64_t nt_off, ns_off;  // first DoF layer of the slab
};

enum { NEED_TABLES = 1, NEED_WEIGHTS = 2, NEED_ALL = 3 };
igs_status validate_problem(const igs_problem* p, Dims* dims, unsigned need = NEED_ALL);

// 1D banded matrix: row r multiplies in[col0[r] + t] by vals[r*width + t],
// t < cnt[r].  Used for Q (points x functions), Q^T and W (pairs x points).
struct Band {
  int64_t rows = 0;
  int32_t width = 0;
  int64_t* col0 = nullptr;
  int32_t* cnt = nullptr;
  double* vals = nullptr;
};

}  // namespace igs

namespace igs {

// Tensor CSR geometry from 1D m-major patterns (see pattern.cu).
struct TensorPat {
  int d;
  const int64_t* rp[3];
  const int64_t* cl[3];
  int64_t ns[3];  // test functions per direction
  int64_t nt[3];  // trial functions per direction
};

// Start offset of row m in the tensor CSR, plus its per-direction widths
// w[] and multi-index mi[]:
//   start = rp0[m0]·w1·w2 + P0·rp1[m1]·w2 + P0·P1·rp2[m2].
__device__ __forceinline__ int64_t tensor_row_start(const TensorPat& t, int64_t m, int64_t* w,
                                                    int64_t* mi) {
  int64_t P[3], rpm[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k < t.d) {
      mi[k] = m % t.ns[k];
      m /= t.ns[k];
      rpm[k] = t.rp[k][mi[k]];
      w[k] = t.rp[k][mi[k] + 1] - rpm[k];
      P[k] = t.rp[k][t.ns[k]];
    } else {
      mi[k] = 0; rpm[k] = 0; w[k] = 1; P[k] = 1;
    }
  }
  return rpm[0] * w[1] * w[2] + P[0] * rpm[1] * w[2] + P[0] * P[1] * rpm[2];
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound_i64(const int64_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace igs
