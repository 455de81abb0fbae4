// C-ABI entry points: validation, fused-vs-generic dispatch, workspace sizing.
#include "igs_internal.cuh"
#include "fused.cuh"

namespace igs {
size_t generic_apply_workspace(const igs_problem* p, const Dims& D);
size_t generic_eval_workspace(const igs_problem* p, const Dims& D);
size_t generic_assemble_workspace(const igs_problem* p, const Dims& D);
igs_status generic_apply(const igs_problem* p, const Dims& D, const double* planes,
                         const double* x, double* y, void* ws, size_t ws_bytes, int flags,
                         cudaStream_t s);
igs_status generic_eval_field(const igs_problem* p, const Dims& D, const int8_t* deriv,
                              const double* coeffs, double* out, void* ws, size_t ws_bytes,
                              cudaStream_t s);
igs_status generic_assemble(const igs_problem* p, const Dims& D, const int64_t* const* rowptr1d,
                            const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                            int block_eta, int block_theta, const double* planes, double* values,
                            void* ws, size_t ws_bytes, cudaStream_t s);
}  // namespace igs

using namespace igs;

extern "C" int32_t igs_fused_path(const igs_problem* prob, int32_t op) {
  Dims D;
  if (validate_problem(prob, &D) != IGS_OK) return 0;
  if (op == IGS_OP_APPLY) return fused_apply_supported(prob, D) ? 1 : 0;
  if (op == IGS_OP_ASSEMBLE) return fused_assemble_supported(prob, D) ? 1 : 0;
  return 0;
}

extern "C" size_t igs_workspace_bytes(const igs_problem* prob, int32_t op, int32_t flags) {
  Dims D;
  if (validate_problem(prob, &D, op == IGS_OP_EVAL_FIELD ? NEED_TABLES : NEED_ALL) != IGS_OK) return 0;
  bool generic = (flags & IGS_FLAG_FORCE_GENERIC) != 0;
  switch (op) {
    case IGS_OP_APPLY:
      if (!generic && fused_apply_supported(prob, D)) return fused_apply_workspace(prob, D);
      return generic_apply_workspace(prob, D);
    case IGS_OP_EVAL_FIELD:
      return generic_eval_workspace(prob, D);
    case IGS_OP_ASSEMBLE:
      if (!generic && fused_assemble_supported(prob, D)) return fused_assemble_workspace(prob, D, flags);
      return generic_assemble_workspace(prob, D);
    default:
      return 0;
  }
}

extern "C" igs_status igs_apply(const igs_problem* prob, const double* planes, const double* x,
                                double* y, void* ws, size_t ws_bytes, int32_t flags, void* stream) {
  Dims D;
  IGS_TRY(validate_problem(prob, &D));
  if (!x || !y) return fail(IGS_EARG, "null vector");
  if (!planes && prob->n_planes > 0) return fail(IGS_EARG, "null coefficient planes");
  cudaStream_t s = as_stream(stream);
  // TMA needs 16-byte aligned planes: a misaligned view takes the generic kernels
  const bool aligned = ((uintptr_t)planes & 15) == 0;
  if (!(flags & IGS_FLAG_FORCE_GENERIC) && aligned && fused_apply_supported(prob, D))
    return fused_apply(prob, D, planes, x, y, ws, ws_bytes, flags, s);
  return generic_apply(prob, D, planes, x, y, ws, ws_bytes, flags, s);
}

extern "C" igs_status igs_eval_field(const igs_problem* prob, const int8_t* deriv,
                                     const double* coeffs, double* out, void* ws, size_t ws_bytes,
                                     void* stream) {
  Dims D;
  IGS_TRY(validate_problem(prob, &D, NEED_TABLES));
  if (!deriv || !coeffs || !out) return fail(IGS_EARG, "null argument");
  for (int k = 0; k < prob->d; ++k) {
    if (deriv[k] < 0) return fail(IGS_EARG, "negative derivative level");
    if (deriv[k] >= prob->trial[k].order) return fail(IGS_EDERIV, "derivative level >= order");
    if (deriv[k] > prob->trial[k].max_deriv) return fail(IGS_EARG, "table does not hold derivative level");
  }
  return generic_eval_field(prob, D, deriv, coeffs, out, ws, ws_bytes, as_stream(stream));
}

extern "C" igs_status igs_assemble_values(const igs_problem* prob, const int64_t* const* rowptr1d,
                                          const int64_t* const* cols1d, int64_t row_lo,
                                          int64_t row_hi, int32_t block_eta, int32_t block_theta,
                                          const double* planes, double* values, void* ws,
                                          size_t ws_bytes, int32_t flags, void* stream) {
  // A slab (last-direction elements [slab_lo, slab_hi) held by `planes`)
  // restricts the coefficient data, not the matrix: rows, columns and the 1D
  // patterns stay global, and the row range must only need slab elements.
  const bool slab = prob->slab_lo != 0 || prob->slab_hi != 0;
  if (slab) {
    Dims Ds;
    IGS_TRY(validate_problem(prob, &Ds));
  }
  igs_problem g = *prob;
  g.slab_lo = g.slab_hi = 0;
  Dims D;
  IGS_TRY(validate_problem(&g, &D));
  int64_t nrows = D.ns[0] * D.ns[1] * D.ns[2];
  if (row_lo < 0 || row_hi < row_lo || row_hi > nrows) return fail(IGS_EARG, "row range");
  if ((block_eta < 0) != (block_theta < 0)) return fail(IGS_EARG, "block indices must both be set");
  if (block_eta >= prob->n_eta || block_theta >= prob->n_theta) return fail(IGS_EARG, "block index");
  if (!rowptr1d || !cols1d || !values) return fail(IGS_EARG, "null argument");
  for (int k = 0; k < prob->d; ++k)
    if (!rowptr1d[k] || !cols1d[k]) return fail(IGS_EARG, "null 1D pattern");
  cudaStream_t s = as_stream(stream);
  const bool aligned = ((uintptr_t)planes & 15) == 0;
  if (!(flags & IGS_FLAG_FORCE_GENERIC) && block_eta < 0 && aligned && fused_assemble_supported(prob, D))
    return fused_assemble(prob, D, rowptr1d, cols1d, row_lo, row_hi, planes, values, ws, ws_bytes, s, flags);
  if (slab) return fail(IGS_ECAPACITY, "slab assembly needs the fused 3D kernels (uniform p = k, full sum)");
  return generic_assemble(prob, D, rowptr1d, cols1d, row_lo, row_hi, block_eta, block_theta, planes,
                          values, ws, ws_bytes, s);
}
