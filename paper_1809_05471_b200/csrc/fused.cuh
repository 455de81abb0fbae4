// Fused sm_100a kernels (apply3d.cu, assemble3d.cu): applicability checks,
// workspace sizing and launchers.
#pragma once
#include "igs_internal.cuh"

namespace igs {

bool fused_apply_supported(const igs_problem* p, const Dims& D);
size_t fused_apply_workspace(const igs_problem* p, const Dims& D);
igs_status fused_apply(const igs_problem* p, const Dims& D, const double* planes, const double* x,
                       double* y, void* ws, size_t ws_bytes, int flags, cudaStream_t s);

bool fused_assemble_supported(const igs_problem* p, const Dims& D);
size_t fused_assemble_workspace(const igs_problem* p, const Dims& D, int flags = 0);
igs_status fused_assemble(const igs_problem* p, const Dims& D, const int64_t* const* rowptr1d,
                          const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                          const double* planes, double* values, void* ws, size_t ws_bytes,
                          cudaStream_t s, int flags = 0);

// Shape class shared by the fused kernels: same spline order p in every
// direction, trial == test, first-order derivative sets (0, e_1..e_d),
// per-element rules with k points and maximum smoothness (function e+j is
// the j-th active one on element e).
struct FusedShape {
  int d, p, k;
  int64_t nel[3];   // elements per direction (slab-restricted in the last)
  int64_t nfn[3];   // functions per direction (slab-restricted)
  int64_t npt[3];   // points per direction (slab-restricted)
  int mass;         // mass term present (plane for F[0][0])
  int stiff;        // stiffness terms present
  int general;      // any other coupling (convection) present
};
bool fused_shape(const igs_problem* p, const Dims& D, FusedShape* fs);

}  // namespace igs
