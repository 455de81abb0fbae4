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

#include "igs_internal.cuh"

namespace igs {
namespace {

struct PullArgs {
  igs_pullback_args g;
  int8_t plane_of[4][4];
  int n_planes;
  double* planes;
  int64_t pstride;
  double* phys;                      // [d][npts] or null
  unsigned long long* maxbits;       // max |J| as IEEE bits (non-negative)
  unsigned long long* bad;           // first degenerate point
  unsigned int* nonzero;             // [n_planes]
};

__device__ __forceinline__ void jacobian(const igs_pullback_args& g, int64_t x, double J[3][3]) {
  const int d = g.d;
  if (g.wval) {
    const double w = g.wval[x];
    const double w2 = w * w;
    for (int c = 0; c < d; ++c) {
      const double n = g.val[c][x];
      for (int k = 0; k < d; ++k) J[c][k] = (g.grad[c][k][x] * w - n * g.wgrad[k][x]) / w2;
    }
  } else {
    for (int c = 0; c < d; ++c)
      for (int k = 0; k < d; ++k) J[c][k] = g.grad[c][k][x];
  }
}

__global__ void jac_max_kernel(const PullArgs a) {
  double m = 0.0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < a.g.npts;
       x += (int64_t)gridDim.x * blockDim.x) {
    double J[3][3];
    jacobian(a.g, x, J);
    for (int c = 0; c < a.g.d; ++c)
      for (int k = 0; k < a.g.d; ++k) m = fmax(m, fabs(J[c][k]));
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(a.maxbits, (unsigned long long)__double_as_longlong(m));
}

// Determinant and inverse by the reference's cofactor formulas
// (geometry.py:121-155), same operation order.
__device__ __forceinline__ double invert(int d, const double J[3][3], double inv[3][3]) {
  if (d == 1) {
    inv[0][0] = 1.0 / J[0][0];
    return J[0][0];
  }
  if (d == 2) {
    const double a = J[0][0], b = J[0][1], c = J[1][0], dd = J[1][1];
    const double det = a * dd - b * c;
    inv[0][0] = dd / det;
    inv[0][1] = -b / det;
    inv[1][0] = -c / det;
    inv[1][1] = a / det;
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
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) inv[i][j] = cof[i][j] / det;
  return det;
}

__global__ void pullback_kernel(const PullArgs a) {
  const igs_pullback_args& g = a.g;
  const int d = g.d, n = d + 1;
  const double scale = __longlong_as_double((long long)*a.maxbits);
  double lim = g.rtol;
  for (int k = 0; k < d; ++k) lim *= scale;
  unsigned nz = 0;  // per-thread plane flags (bit p)
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < g.npts;
       x += (int64_t)gridDim.x * blockDim.x) {
    double J[3][3], inv[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    jacobian(g, x, J);
    const double det = invert(d, J, inv);
    if (!(fabs(det) >= lim)) atomicMin(a.bad, (unsigned long long)x);
    if (a.phys) {
      for (int c = 0; c < d; ++c) a.phys[c * g.npts + x] = g.wval ? g.val[c][x] / g.wval[x] : g.val[c][x];
    }
    // mhat = [[c, 0], [b, A]]; ext = diag(1, inv)
    double mh[4][4];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) mh[i][j] = 0.0;
    if (g.reaction) mh[0][0] = g.reaction[x * g.reaction_stride];
    for (int i = 0; i < d; ++i) {
      if (g.convection[i]) mh[1 + i][0] = g.convection[i][x * g.convection_stride];
      for (int j = 0; j < d; ++j)
        if (g.diffusion[i][j]) mh[1 + i][1 + j] = g.diffusion[i][j][x * g.diffusion_stride];
    }
    double ext[4][4];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) ext[i][j] = (i == 0 || j == 0) ? (i == j ? 1.0 : 0.0) : inv[i - 1][j - 1];
    // t = ext · mhat, F = |det| · t · ext^T
    double t[4][4];
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += ext[i][j] * mh[j][k];
        t[i][k] = s;
      }
    const double ad = fabs(det);
    for (int i = 0; i < n; ++i)
      for (int l = 0; l < n; ++l) {
        const int pl = a.plane_of[i][l];
        if (pl < 0) continue;
        // a plane shared by (i, l) and (l, i) is written from the upper triangle
        if (l < i && a.plane_of[l][i] == pl) continue;
        double s = 0.0;
        for (int k = 0; k < n; ++k) s += t[i][k] * ext[l][k];
        const double v = ad * s;
        a.planes[pl * a.pstride + x] = v;
        if (v != 0.0) nz |= 1u << pl;
      }
  }
  for (int o = 16; o; o >>= 1) nz |= __shfl_xor_sync(0xffffffffu, nz, o);
  if ((threadIdx.x & 31) == 0)
    for (int p = 0; p < a.n_planes; ++p)
      if (nz & (1u << p)) atomicOr(a.nonzero + p, 1u);
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
  if (args->npts < 0) return fail(IGS_EARG, "negative point count");
  if (n_planes < 0 || n_planes > 16) return fail(IGS_EARG, "at most 16 planes");
  if (n_planes > 0 && !planes) return fail(IGS_EARG, "null planes");
  if (ws_bytes < 64 || !ws) return fail(IGS_EWORKSPACE, "pullback workspace needs 64 bytes");
  for (int c = 0; c < d; ++c) {
    if (!args->val[c]) return fail(IGS_EARG, "null component values");
    for (int k = 0; k < d; ++k)
      if (!args->grad[c][k]) return fail(IGS_EARG, "null component derivative");
    if (args->wval && !args->wgrad[c]) return fail(IGS_EARG, "null weight derivative");
  }
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
  a.nonzero = nonzero;
  cudaStream_t st = as_stream(stream);
  const unsigned long long init[2] = {0ull, ~0ull};
  IGS_TRY(cuda_check(cudaMemcpyAsync(ws, init, sizeof(init), cudaMemcpyHostToDevice, st), "pullback init"));
  if (n_planes > 0)
    IGS_TRY(cuda_check(cudaMemsetAsync(nonzero, 0, n_planes * sizeof(uint32_t), st), "pullback flags"));
  if (args->npts > 0) {
    const int64_t blocks = min64(ceil_div(args->npts, 256), 148 * 16);
    jac_max_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
    IGS_LAUNCH_CHECK("jac_max_kernel");
    pullback_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
    IGS_LAUNCH_CHECK("pullback_kernel");
  }
  unsigned long long b = ~0ull;
  IGS_TRY(cuda_check(cudaMemcpyAsync(&b, a.bad, sizeof(b), cudaMemcpyDeviceToHost, st), "pullback result"));
  IGS_TRY(cuda_check(cudaStreamSynchronize(st), "pullback sync"));
  *bad = b == ~0ull ? -1 : (int64_t)b;
  return IGS_OK;
}
