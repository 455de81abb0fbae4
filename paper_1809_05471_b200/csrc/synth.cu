// Seeded synthetic coefficient planes for the BASELINE workloads.
//
// Counter-based: every value is a pure function of (seed, slot, global flat
// point index), so any slab is reproducible on any rank and by the numpy
// mirror in oracle/ (oracle/igs_oracle.py:synthetic_planes) with no RNG
// state to ship.  Distribution as in BASELINE.json: c ~ U[0.5, 1.5];
// A = I + 0.05·G·Gᵀ/d with G_ab ~ N(0,1) (Box-Muller).
#include "igs_internal.cuh"

namespace igs {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Uniform in [0, 1) with 53 random bits.
__device__ __forceinline__ double uni(uint64_t key, uint64_t q) {
  return (double)(mix64(key ^ q) >> 11) * 0x1.0p-53;
}

__global__ void fill_kernel(int d, int64_t layer, int64_t z_lo, int64_t z_hi, int kind,
                            uint64_t seed, double* planes, int64_t stride) {
  const int64_t local_total = (z_hi - z_lo) * layer;
  const double two_pi = 6.283185307179586;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < local_total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = z_lo * layer + t;  // global flat point index
    int pl = 0;
    if (kind & 1) {
      uint64_t key = mix64(seed + 0x632BE59BD9B4E019ull * 1ull);
      planes[(pl++) * stride + t] = 0.5 + uni(key, (uint64_t)q);
    }
    if (kind & 2) {
      double G[3][3];
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          int e = a * d + b;
          uint64_t k1 = mix64(seed + 0x632BE59BD9B4E019ull * (uint64_t)(2 * e + 2));
          uint64_t k2 = mix64(seed + 0x632BE59BD9B4E019ull * (uint64_t)(2 * e + 3));
          double u1 = uni(k1, (uint64_t)q), u2 = uni(k2, (uint64_t)q);
          G[a][b] = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
        }
      // diagonal entries first, then the upper triangle row-major
      for (int a = 0; a < d; ++a) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) s += G[a][c] * G[a][c];
        planes[(pl++) * stride + t] = 1.0 + (0.05 * s) / d;
      }
      for (int a = 0; a < d; ++a)
        for (int b = a + 1; b < d; ++b) {
          double s = 0.0;
          for (int c = 0; c < d; ++c) s += G[a][c] * G[b][c];
          planes[(pl++) * stride + t] = (0.05 * s) / d;
        }
    }
  }
}

}  // namespace
}  // namespace igs

using namespace igs;

extern "C" igs_status igs_fill_synthetic(int32_t d, const int64_t* point_dims, int64_t z_lo,
                                         int64_t z_hi, int32_t kind, uint64_t seed, double* planes,
                                         int64_t plane_stride, void* stream) {
  if (d < 1 || d > 3) return fail(IGS_EARG, "dimension must be 1..3");
  if (kind < 1 || kind > 3) return fail(IGS_EARG, "kind must be 1 (mass), 2 (stiffness) or 3");
  if (!point_dims || !planes) return fail(IGS_EARG, "null argument");
  // A "layer" is one index of the last direction: the product of the others.
  int64_t layer = 1;
  for (int k = 0; k + 1 < d; ++k) layer *= point_dims[k];
  int64_t XL = point_dims[d - 1];
  if (z_lo < 0 || z_hi < z_lo || z_hi > XL) return fail(IGS_EARG, "layer range");
  int64_t total = (z_hi - z_lo) * layer;
  if (total == 0) return IGS_OK;
  int block = 256;
  int64_t grid = ceil_div(total, block);
  if (grid > 148 * 32) grid = 148 * 32;
  fill_kernel<<<(unsigned)grid, block, 0, as_stream(stream)>>>(d, layer, z_lo, z_hi, kind, seed,
                                                               planes, plane_stride);
  IGS_LAUNCH_CHECK("fill_kernel");
  return IGS_OK;
}
