// Temporary: fused kernels not yet built; every problem takes the generic path.
#include "fused.cuh"
namespace igs {
bool fused_apply_supported(const igs_problem*, const Dims&) { return false; }
size_t fused_apply_workspace(const igs_problem*, const Dims&) { return 0; }
igs_status fused_apply(const igs_problem*, const Dims&, const double*, const double*, double*,
                       void*, size_t, int, cudaStream_t) {
  return fail(IGS_ECAPACITY, "no fused apply");
}
bool fused_assemble_supported(const igs_problem*, const Dims&) { return false; }
size_t fused_assemble_workspace(const igs_problem*, const Dims&) { return 0; }
igs_status fused_assemble(const igs_problem*, const Dims&, const int64_t* const*,
                          const int64_t* const*, int64_t, int64_t, const double*, double*, void*,
                          size_t, cudaStream_t) {
  return fail(IGS_ECAPACITY, "no fused assembly");
}
}  // namespace igs
