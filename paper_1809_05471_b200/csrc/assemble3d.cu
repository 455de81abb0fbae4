// K3 fused assembly: not yet specialised; every assembly takes the generic path.
#include "fused.cuh"
namespace igs {
bool fused_assemble_supported(const igs_problem*, const Dims&) { return false; }
size_t fused_assemble_workspace(const igs_problem*, const Dims&) { return 0; }
igs_status fused_assemble(const igs_problem*, const Dims&, const int64_t* const*,
                          const int64_t* const*, int64_t, int64_t, const double*, double*, void*,
                          size_t, cudaStream_t) {
  return fail(IGS_ECAPACITY, "no fused assembly");
}
}  // namespace igs
