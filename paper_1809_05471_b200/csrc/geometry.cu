// f1 — coefficient field from a geometry map, on the device.
//
// Pointwise half of eval_geometry + build_coefficient_field (reference
// geometry.py:158-216, :121-155, :315-336): the spline fields of the map
// (component values and first derivatives, optionally weighted numerators
// and the weight for rational maps) come from Alg. 3 (igs_eval_field); this
// kernel forms the Jacobian J[c][k] = dG_c/dx_k (quotient rule for rational
// maps), its determinant and cofactor inverse, checks degeneracy against
// rtol·max|J|^d, and writes the pulled-back coefficient
//
//     F = |det J| · E · [[c, 0], [b, A]] · E^T,   E = diag(1, J^{-1})
//
// straight into the SoA coefficient planes of the hot path (plane_of map,
// blocks sharing a plane written once), with per-plane "any non-zero" flags
// so the host can drop exactly-zero blocks as the reference does
// (geometry.py:296).

#include <cstring>

#include "igs_internal.cuh"

namespace igs {
namespace {

// Where the Jacobian (and the mapped point) of point x come from:
//   FieldSrc — the spline fields precomputed by Alg. 3 (igs_eval_field);
//   MapSrc   — evaluated in place from the map's 1D tables and control
//              points (the f1 fused path: nothing but the planes is written).
struct FieldSrc {
  igs_pullback_args g;
  __device__ __forceinline__ void eval(int64_t x, double J[3][3], double X[3]) const {
    const int d = g.d;
    if (g.wval) {
      const double w = g.wval[x];
      const double w2 = w * w;
      for (int c = 0; c < d; ++c) {
        const double n = g.val[c][x];
        X[c] = n / w;
        for (int k = 0; k < d; ++k) J[c][k] = (g.grad[c][k][x] * w - n * g.wgrad[k][x]) / w2;
      }
    } else {
      for (int c = 0; c < d; ++c) {
        X[c] = g.val[c][x];
        for (int k = 0; k < d; ++k) J[c][k] = g.grad[c][k][x];
      }
    }
  }
};

constexpr int kMapMaxOrder = 8;

template <int PM>  // PM >= every direction's map order
struct MapSrc {
  igs_geometry_map m;
  // Σ over the map's active control points of the tensor basis (values and
  // first derivatives), the weighted numerators for rational maps; then the
  // quotient rule as FieldSrc (geometry.py:158-216).  Loops are unrolled to
  // PM with run-time guards, so the basis values stay in registers.
  __device__ __forceinline__ void eval(int64_t x, double J[3][3], double X[3]) const {
    const int d = m.d;
    int64_t fa[3] = {0, 0, 0};
    int64_t r = x;
    double b[3][2][PM];
    int P[3] = {1, 1, 1};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k < d) {
        const int64_t i = r % m.num_points[k];
        r /= m.num_points[k];
        P[k] = m.order[k];
        fa[k] = m.first_active[k][i];
#pragma unroll
        for (int j = 0; j < PM; ++j) {
          b[k][0][j] = j < P[k] ? m.values[k][(int64_t)j * m.num_points[k] + i] : 0.0;
          b[k][1][j] = j < P[k] ? m.values[k][((int64_t)P[k] + j) * m.num_points[k] + i] : 0.0;
        }
      } else {
#pragma unroll
        for (int j = 0; j < PM; ++j) b[k][0][j] = b[k][1][j] = 0.0;
        b[k][0][0] = 1.0;
      }
    }
    // acc[c][0] = value, acc[c][1 + k] = d/dx_k; c = 3: the weight spline
    double acc[4][4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[c][k] = 0.0;
    const bool rat = m.weights != nullptr;
    const int64_t N0 = m.num_basis[0], N01 = N0 * (d > 1 ? m.num_basis[1] : 1);
#pragma unroll
    for (int j2 = 0; j2 < PM; ++j2) {
      if (j2 >= P[2]) break;
#pragma unroll
      for (int j1 = 0; j1 < PM; ++j1) {
        if (j1 >= P[1]) break;
        const double yz0 = b[1][0][j1] * b[2][0][j2];
        const double yz1 = b[1][1][j1] * b[2][0][j2];
        const double yz2 = b[1][0][j1] * b[2][1][j2];
        const int64_t row = (fa[1] + j1) * N0 + (fa[2] + j2) * N01 + fa[0];
#pragma unroll
        for (int j0 = 0; j0 < PM; ++j0) {
          if (j0 >= P[0]) break;
          const int64_t n = row + j0;
          const double v = b[0][0][j0] * yz0;
          const double g0 = b[0][1][j0] * yz0;
          const double g1 = b[0][0][j0] * yz1;
          const double g2 = b[0][0][j0] * yz2;
          const double wn = rat ? m.weights[n] : 1.0;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (c >= d) break;
            const double cp = wn * m.control[n * d + c];
            acc[c][0] = fma(cp, v, acc[c][0]);
            acc[c][1] = fma(cp, g0, acc[c][1]);
            acc[c][2] = fma(cp, g1, acc[c][2]);
            acc[c][3] = fma(cp, g2, acc[c][3]);
          }
          if (rat) {
            acc[3][0] = fma(wn, v, acc[3][0]);
            acc[3][1] = fma(wn, g0, acc[3][1]);
            acc[3][2] = fma(wn, g1, acc[3][2]);
            acc[3][3] = fma(wn, g2, acc[3][3]);
          }
        }
      }
    }
    if (rat) {
      const double w = acc[3][0];
      const double w2 = w * w;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (c >= d) break;
        X[c] = acc[c][0] / w;
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (k < d) J[c][k] = (acc[c][1 + k] * w - acc[c][0] * acc[3][1 + k]) / w2;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (c >= d) break;
        X[c] = acc[c][0];
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (k < d) J[c][k] = acc[c][1 + k];
      }
    }
  }
};

struct PullArgs {
  igs_pullback_args g;               // PDE data, d, npts, rtol (FieldSrc: also the fields)
  int8_t plane_of[4][4];
  int n_planes;
  double* planes;
  int64_t pstride;
  double* phys;                      // [d][npts] or null
  unsigned long long* maxbits;       // max |J| as IEEE bits (non-negative doubles order as integers)
  unsigned long long* bad;           // first degenerate point
  unsigned long long* mindet;        // min |det J| as IEEE bits
  unsigned int* nonzero;             // [n_planes]
};

// Determinant and inverse by the reference's cofactor formulas
// (geometry.py:121-155); the cofactors are scaled by one reciprocal of the
// determinant (the reference divides each: <= 1 ulp apart).
__device__ __forceinline__ double invert(int d, const double J[3][3], double inv[3][3]) {
  if (d == 1) {
    inv[0][0] = 1.0 / J[0][0];
    return J[0][0];
  }
  if (d == 2) {
    const double a = J[0][0], b = J[0][1], c = J[1][0], dd = J[1][1];
    const double det = a * dd - b * c;
    const double r = 1.0 / det;
    inv[0][0] = dd * r;
    inv[0][1] = -b * r;
    inv[1][0] = -c * r;
    inv[1][1] = a * r;
    return det;
  }
  double cof[3][3];
  cof[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  cof[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  cof[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  cof[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  cof[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  cof[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  cof[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  cof[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  cof[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double det = J[0][0] * cof[0][0] + J[0][1] * cof[1][0] + J[0][2] * cof[2][0];
  const double r = 1.0 / det;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) inv[i][j] = cof[i][j] * r;
  return det;
}

struct PullAcc {
  unsigned nz = 0;  // plane flags (bit p)
  double jmax = 0.0;
  double dmin = 1.7976931348623157e308;
};

// Everything after the Jacobian for point x: determinant, inverse, the mapped
// point, F = |det J|·E·[[c,0],[b,A]]·E^T into the planes, the reductions.
template <int D>
__device__ __forceinline__ void pull_point(const PullArgs& a, int64_t x, const double J[3][3], const double X[3],
                                           PullAcc& r) {
  const igs_pullback_args& g = a.g;
  constexpr int d = D, n = D + 1;
  double inv[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int c = 0; c < d; ++c)
#pragma unroll
    for (int k = 0; k < d; ++k) r.jmax = fmax(r.jmax, fabs(J[c][k]));
  const double det = invert(d, J, inv);
  if (det != det) atomicMin(a.bad, (unsigned long long)x);
  else r.dmin = fmin(r.dmin, fabs(det));
  if (a.phys) {
#pragma unroll
    for (int c = 0; c < d; ++c) a.phys[c * g.npts + x] = X[c];
  }
  if (a.n_planes == 0) return;
  // mhat = [[c, 0], [b, A]]; ext = diag(1, inv)
  double mh[4][4];
#pragma unroll
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < n; ++j) mh[i][j] = 0.0;
  if (g.reaction) mh[0][0] = g.reaction[x * g.reaction_stride];
#pragma unroll
  for (int i = 0; i < d; ++i) {
    if (g.convection[i]) mh[1 + i][0] = g.convection[i][x * g.convection_stride];
#pragma unroll
    for (int j = 0; j < d; ++j)
      if (g.diffusion[i][j]) mh[1 + i][1 + j] = g.diffusion[i][j][x * g.diffusion_stride];
  }
  double ext[4][4];
#pragma unroll
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < n; ++j) ext[i][j] = (i == 0 || j == 0) ? (i == j ? 1.0 : 0.0) : inv[i - 1][j - 1];
  // t = ext · mhat, F = |det| · t · ext^T
  double t[4][4];
#pragma unroll
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < n; ++k) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n; ++j) s += ext[i][j] * mh[j][k];
      t[i][k] = s;
    }
  const double ad = fabs(det);
#pragma unroll
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int l = 0; l < n; ++l) {
      const int pl = a.plane_of[i][l];
      if (pl < 0) continue;
      // a plane shared by (i, l) and (l, i) is written from the upper triangle
      if (l < i && a.plane_of[l][i] == pl) continue;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < n; ++k) s += t[i][k] * ext[l][k];
      const double v = ad * s;
      a.planes[pl * a.pstride + x] = v;
      if (v != 0.0) r.nz |= 1u << pl;
    }
}

__device__ __forceinline__ void pull_reduce(const PullArgs& a, PullAcc& r) {
  for (int o = 16; o; o >>= 1) {
    r.nz |= __shfl_xor_sync(0xffffffffu, r.nz, o);
    r.jmax = fmax(r.jmax, __shfl_xor_sync(0xffffffffu, r.jmax, o));
    r.dmin = fmin(r.dmin, __shfl_xor_sync(0xffffffffu, r.dmin, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (r.jmax > 0.0) atomicMax(a.maxbits, (unsigned long long)__double_as_longlong(r.jmax));
    atomicMin(a.mindet, (unsigned long long)__double_as_longlong(r.dmin));
    for (int p = 0; p < a.n_planes; ++p)
      if (r.nz & (1u << p)) atomicOr(a.nonzero + p, 1u);
  }
}

// One pass over the points: Jacobian from `src`, then pull_point; max |J|
// and min |det J| reduced on the side so the degeneracy test |det J| <
// rtol·max|J|^d (geometry.py:158-216) needs a second pass only when it fails
// (NaN determinants are flagged directly).
template <class Src, int D>
__global__ void pullback_kernel(const PullArgs a, const Src src) {
  PullAcc r;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < a.g.npts;
       x += (int64_t)gridDim.x * blockDim.x) {
    double J[3][3], X[3];
    src.eval(x, J, X);
    pull_point<D>(a, x, J, X, r);
  }
  pull_reduce(a, r);
}

// f1 fused, sum-factorised per line of direction-0 points: for the line
// (i1, i2) the slower directions are contracted once into shared memory,
//   Y[n0][c][t] = Σ_{j1,j2} P_c[n0, f1+j1, f2+j2] · (B1 B2, B1' B2, B1 B2')[t],
// (c = d: the weight spline of a rational map, P_c weighted), then every
// point of the line needs only its P direction-0 terms (Alg. 3 restricted to
// one point row) before pull_point.
template <int PM, int D>
__global__ void geom_line_kernel(const PullArgs a, const igs_geometry_map m) {
  extern __shared__ double Ysm[];  // [N0][4][3]
  PullAcc r;
  constexpr int d = D;
  const bool rat = m.weights != nullptr;
  const int nc = rat ? d + 1 : d;
  const int64_t X0 = m.num_points[0], X1 = d > 1 ? m.num_points[1] : 1, X2 = d > 2 ? m.num_points[2] : 1;
  const int N0 = m.num_basis[0];
  const int64_t N1 = d > 1 ? m.num_basis[1] : 1;
  const int P0 = m.order[0], P1 = d > 1 ? m.order[1] : 1, P2 = d > 2 ? m.order[2] : 1;
  for (int64_t line = blockIdx.x; line < X1 * X2; line += gridDim.x) {
    const int64_t i1 = line % X1, i2 = line / X1;
    const int64_t f1 = d > 1 ? m.first_active[1][i1] : 0, f2 = d > 2 ? m.first_active[2][i2] : 0;
    __syncthreads();  // the previous line's Y is consumed
    for (int e = threadIdx.x; e < N0 * nc; e += blockDim.x) {
      const int n0 = e / nc, c = e % nc;
      double y0 = 0.0, y1 = 0.0, y2 = 0.0;
      for (int j2 = 0; j2 < P2; ++j2) {
        const double z0 = d > 2 ? m.values[2][(int64_t)j2 * X2 + i2] : 1.0;
        const double z1 = d > 2 ? m.values[2][((int64_t)P2 + j2) * X2 + i2] : 0.0;
        for (int j1 = 0; j1 < P1; ++j1) {
          const double q0 = d > 1 ? m.values[1][(int64_t)j1 * X1 + i1] : 1.0;
          const double q1 = d > 1 ? m.values[1][((int64_t)P1 + j1) * X1 + i1] : 0.0;
          const int64_t n = n0 + N0 * ((f1 + j1) + N1 * (f2 + j2));
          const double wn = rat ? m.weights[n] : 1.0;
          const double cp = c < d ? wn * m.control[n * d + c] : wn;
          y0 = fma(cp, q0 * z0, y0);
          y1 = fma(cp, q1 * z0, y1);
          y2 = fma(cp, q0 * z1, y2);
        }
      }
      double* Y = Ysm + (n0 * 4 + c) * 3;
      Y[0] = y0;
      Y[1] = y1;
      Y[2] = y2;
    }
    __syncthreads();
    for (int64_t i0 = threadIdx.x; i0 < X0; i0 += blockDim.x) {
      const int64_t f0 = m.first_active[0][i0];
      double acc[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[c][k] = 0.0;
#pragma unroll
      for (int j0 = 0; j0 < PM; ++j0) {
        if (j0 >= P0) break;
        const double v0 = m.values[0][(int64_t)j0 * X0 + i0];
        const double v1 = m.values[0][((int64_t)P0 + j0) * X0 + i0];
        const double* Y = Ysm + (f0 + j0) * 12;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nc) break;
          const double y0 = Y[c * 3], y1 = Y[c * 3 + 1], y2 = Y[c * 3 + 2];
          acc[c][0] = fma(y0, v0, acc[c][0]);
          acc[c][1] = fma(y0, v1, acc[c][1]);
          acc[c][2] = fma(y1, v0, acc[c][2]);
          acc[c][3] = fma(y2, v0, acc[c][3]);
        }
      }
      double J[3][3], X[3];
      if (rat) {
        const double w = acc[d][0];
        const double w2 = w * w;
#pragma unroll
        for (int c = 0; c < d; ++c) {
          X[c] = acc[c][0] / w;
#pragma unroll
          for (int k = 0; k < d; ++k) J[c][k] = (acc[c][1 + k] * w - acc[c][0] * acc[d][1 + k]) / w2;
        }
      } else {
#pragma unroll
        for (int c = 0; c < d; ++c) {
          X[c] = acc[c][0];
#pragma unroll
          for (int k = 0; k < d; ++k) J[c][k] = acc[c][1 + k];
        }
      }
      pull_point<D>(a, i0 + X0 * line, J, X, r);
    }
  }
  pull_reduce(a, r);
}

// Second pass, only when min |det J| fails the test: the first such point.
template <class Src>
__global__ void find_degenerate_kernel(const PullArgs a, const Src src, double lim) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < a.g.npts;
       x += (int64_t)gridDim.x * blockDim.x) {
    double J[3][3], X[3], inv[3][3];
    src.eval(x, J, X);
    const double det = invert(a.g.d, J, inv);
    if (!(fabs(det) >= lim)) atomicMin(a.bad, (unsigned long long)x);
  }
}

// Shared front end of both entry points: validation, workspace, launches,
// the degeneracy verdict.
// PM > 0: `src` is MapSrc<PM> and the main pass is the line-factorised
// geom_line_kernel (when its per-line table fits shared memory).
template <int PM, class Src>
igs_status run_pullback(const igs_pullback_args* args, const Src& src, const int8_t* plane_of, int32_t n_planes,
                        double* planes, int64_t plane_stride, double* phys, uint32_t* nonzero, int64_t* bad,
                        void* ws, size_t ws_bytes, void* stream, const igs_geometry_map* map = nullptr) {
  const int d = args->d;
  if (args->npts < 0) return fail(IGS_EARG, "negative point count");
  if (n_planes < 0 || n_planes > 16) return fail(IGS_EARG, "at most 16 planes");
  if (n_planes > 0 && !planes) return fail(IGS_EARG, "null planes");
  if (ws_bytes < 64 || !ws) return fail(IGS_EWORKSPACE, "pullback workspace needs 64 bytes");
  PullArgs a{};
  a.g = *args;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int8_t pl = (i <= d && j <= d) ? plane_of[i * 4 + j] : (int8_t)-1;
      if (pl >= n_planes) return fail(IGS_EARG, "plane_of entry beyond n_planes");
      a.plane_of[i][j] = pl;
    }
  a.n_planes = n_planes;
  a.planes = planes;
  a.pstride = plane_stride;
  a.phys = phys;
  a.maxbits = reinterpret_cast<unsigned long long*>(ws);
  a.bad = a.maxbits + 1;
  a.mindet = a.maxbits + 2;
  a.nonzero = nonzero;
  cudaStream_t st = as_stream(stream);
  unsigned long long h[3] = {0ull, ~0ull, ~0ull};
  IGS_TRY(cuda_check(cudaMemcpyAsync(ws, h, sizeof(h), cudaMemcpyHostToDevice, st), "pullback init"));
  if (n_planes > 0)
    IGS_TRY(cuda_check(cudaMemsetAsync(nonzero, 0, n_planes * sizeof(uint32_t), st), "pullback flags"));
  const int64_t blocks = min64(ceil_div(args->npts, 256), 148 * 16);
  if (args->npts > 0) {
    const size_t ysm = map ? (size_t)map->num_basis[0] * 12 * sizeof(double) : 0;
    bool done = false;
    if constexpr (PM > 0) {
      if (map && ysm <= 200 * 1024) {
        int64_t lines = args->npts / map->num_points[0];
        const unsigned lb = (unsigned)min64(lines, 148 * 16);
        if (d == 1) {
          IGS_TRY(cuda_check(cudaFuncSetAttribute(geom_line_kernel<PM, 1>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ysm), "smem"));
          geom_line_kernel<PM, 1><<<lb, 128, ysm, st>>>(a, *map);
        } else if (d == 2) {
          IGS_TRY(cuda_check(cudaFuncSetAttribute(geom_line_kernel<PM, 2>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ysm), "smem"));
          geom_line_kernel<PM, 2><<<lb, 128, ysm, st>>>(a, *map);
        } else {
          IGS_TRY(cuda_check(cudaFuncSetAttribute(geom_line_kernel<PM, 3>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ysm), "smem"));
          geom_line_kernel<PM, 3><<<lb, 128, ysm, st>>>(a, *map);
        }
        IGS_LAUNCH_CHECK("geom_line_kernel");
        done = true;
      }
    }
    if (!done) {
      if (d == 1) pullback_kernel<Src, 1><<<(unsigned)blocks, 256, 0, st>>>(a, src);
      else if (d == 2) pullback_kernel<Src, 2><<<(unsigned)blocks, 256, 0, st>>>(a, src);
      else pullback_kernel<Src, 3><<<(unsigned)blocks, 256, 0, st>>>(a, src);
      IGS_LAUNCH_CHECK("pullback_kernel");
    }
  }
  IGS_TRY(cuda_check(cudaMemcpyAsync(h, ws, sizeof(h), cudaMemcpyDeviceToHost, st), "pullback result"));
  IGS_TRY(cuda_check(cudaStreamSynchronize(st), "pullback sync"));
  unsigned long long b = h[1];
  if (args->npts > 0) {
    double lim = args->rtol;
    double scale, dmin;
    memcpy(&scale, &h[0], sizeof(double));
    memcpy(&dmin, &h[2], sizeof(double));
    for (int k = 0; k < d; ++k) lim *= scale;
    if (!(dmin >= lim)) {
      find_degenerate_kernel<Src><<<(unsigned)blocks, 256, 0, st>>>(a, src, lim);
      IGS_LAUNCH_CHECK("find_degenerate_kernel");
      IGS_TRY(cuda_check(cudaMemcpyAsync(&b, a.bad, sizeof(b), cudaMemcpyDeviceToHost, st), "pullback result"));
      IGS_TRY(cuda_check(cudaStreamSynchronize(st), "pullback sync"));
    }
  }
  *bad = b == ~0ull ? -1 : (int64_t)b;
  return IGS_OK;
}

}  // namespace
}  // namespace igs

using namespace igs;

extern "C" igs_status igs_geometry_pullback(const igs_pullback_args* args, const int8_t* plane_of,
                                            int32_t n_planes, double* planes, int64_t plane_stride,
                                            double* phys, uint32_t* nonzero, int64_t* bad, void* ws,
                                            size_t ws_bytes, void* stream) {
  if (!args || !plane_of || !bad || !nonzero) return fail(IGS_EARG, "null argument");
  const int d = args->d;
  if (d < 1 || d > 3) return fail(IGS_EARG, "geometry dimension must be 1..3");
  for (int c = 0; c < d; ++c) {
    if (!args->val[c]) return fail(IGS_EARG, "null component values");
    for (int k = 0; k < d; ++k)
      if (!args->grad[c][k]) return fail(IGS_EARG, "null component derivative");
    if (args->wval && !args->wgrad[c]) return fail(IGS_EARG, "null weight derivative");
  }
  FieldSrc src{*args};
  return run_pullback<0>(args, src, plane_of, n_planes, planes, plane_stride, phys, nonzero, bad, ws, ws_bytes,
                      stream);
}

extern "C" igs_status igs_geometry_planes(const igs_geometry_map* map, const igs_pullback_args* pde,
                                          const int8_t* plane_of, int32_t n_planes, double* planes,
                                          int64_t plane_stride, double* phys, uint32_t* nonzero, int64_t* bad,
                                          void* ws, size_t ws_bytes, void* stream) {
  if (!map || !pde || !plane_of || !bad || !nonzero) return fail(IGS_EARG, "null argument");
  const int d = map->d;
  if (d < 1 || d > 3 || pde->d != d) return fail(IGS_EARG, "geometry dimension must be 1..3 and match the PDE");
  int64_t npts = 1;
  for (int k = 0; k < d; ++k) {
    if (map->order[k] < 2 || map->order[k] > kMapMaxOrder)
      return fail(IGS_EARG, "map orders must be 2..8 (first derivatives tabulated)");
    if (!map->values[k] || !map->first_active[k] || map->num_points[k] < 0 || map->num_basis[k] < map->order[k])
      return fail(IGS_EARG, "bad map tables");
    npts *= map->num_points[k];
  }
  if (npts != pde->npts) return fail(IGS_EARG, "point grid does not match npts");
  if (!map->control) return fail(IGS_EARG, "null control points");
  int pm = 2;
  for (int k = 0; k < d; ++k) pm = map->order[k] > pm ? map->order[k] : pm;
#define IGS_MAP_CASE(PM)                                                                                  \
  case PM: {                                                                                              \
    MapSrc<PM> src{*map};                                                                                 \
    return run_pullback<PM>(pde, src, plane_of, n_planes, planes, plane_stride, phys, nonzero, bad, ws,   \
                            ws_bytes, stream, map);                                                       \
  }
  switch (pm) {
    IGS_MAP_CASE(2)
    IGS_MAP_CASE(3)
    IGS_MAP_CASE(4)
    IGS_MAP_CASE(5)
    IGS_MAP_CASE(6)
    IGS_MAP_CASE(7)
    IGS_MAP_CASE(8)
    default: return fail(IGS_EARG, "map orders must be 2..8");
  }
#undef IGS_MAP_CASE
}
