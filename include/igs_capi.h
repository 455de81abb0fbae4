/*
 * igs_capi.h — C-ABI of the B200 sum-factorization library (libigs_b200.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `igasum` (arXiv:1809.05471, Bressan & Takacs): B-spline tabulation at Gauss
 * points, global sum-factorized assembly into CSR (Alg. 1), and the
 * matrix-free apply (Alg. 2 with Alg. 3 as its interpolation stage).
 *
 * Conventions (identical to the reference):
 *   - spline `order` = degree + 1; indices are 0-based;
 *   - flat DoF / point indices put direction 0 fastest
 *     (tensorspace.py:3-5, LexOrdering tensorspace.py:33-72);
 *   - CSR rows are test functions, columns ascending, band zeros stored
 *     (tensorspace.py:262-338);
 *   - the coefficient field F[x, eta_i, theta_j] excludes quadrature
 *     weights (geometry.py:279-312); weights enter through the 1D tables.
 *
 * Every pointer that is not explicitly marked "host" is a DEVICE pointer.
 * The library allocates nothing persistent, never frees caller memory and
 * keeps no global state except a thread-local last-error string.  All
 * kernels are enqueued on the caller's stream (`cudaStream_t` passed as
 * void*); calls are reentrant.  No C++ exception crosses this boundary.
 * Accumulation order is fixed, so results are bit-reproducible run to run
 * (SPEC.md:419); no floating-point atomics are used on outputs.
 */
#ifndef IGS_CAPI_H
#define IGS_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGS_ABI_VERSION 1
#define IGS_MAX_DIM 3
#define IGS_MAX_DERIV_SET 8   /* max |Theta|, |Eta| (first-order set in 3D has 4) */
#define IGS_MAX_ORDER 16      /* generic path; fused kernels cover orders 2..8 */

/* Status codes; the Python shim maps them 1:1 onto the reference's
 * exception classes (errors.py:4-17). */
typedef enum {
  IGS_OK = 0,
  IGS_EARG = 1,       /* ValueError / TypeError                       */
  IGS_EDOMAIN = 2,    /* DomainError (errors.py:4)                     */
  IGS_EDERIV = 3,     /* UnsupportedDerivativeError (errors.py:8)      */
  IGS_ECAPACITY = 4,  /* CapacityError (errors.py:12)                  */
  IGS_ECUDA = 5,      /* RuntimeError (CUDA launch / runtime failure)  */
  IGS_ENCCL = 6,      /* RuntimeError (collective failure)             */
  IGS_EWORKSPACE = 7  /* ValueError: workspace too small               */
} igs_status;

/* One direction's 1D data: the banded BasisEvalTable (bspline.py:258-311)
 * plus the 1D quadrature rule (quadrature.py:68-106). */
typedef struct {
  int32_t order;              /* spline order p                                   */
  int32_t num_basis;          /* N = len(knots) - order                           */
  int32_t num_points;         /* X = #quadrature points in this direction          */
  int32_t max_deriv;          /* table holds derivative levels 0..max_deriv        */
  const double* values;       /* [max_deriv+1][order][num_points]  (values[k,j,i]) */
  const int64_t* first_active;/* [num_points], non-decreasing                      */
  const double* weights;      /* [num_points] quadrature weights                   */
  const double* csupp_lo;     /* [num_basis] knots[n]            (bspline.py:128)  */
  const double* csupp_hi;     /* [num_basis] knots[n + order]    (bspline.py:129)  */
  const double* points;       /* [num_points] ascending                            */
  int32_t num_elements;       /* K: elements of a per-element rule, else 0         */
  int32_t points_per_element; /* k: points per element of a per-element rule, else 0 */
  int32_t uniform;            /* 1: equally spaced breakpoints (interior elements share
                                 one table up to rounding), lets fused kernels hoist it */
} igs_dir;

/* A trial/test pair on a tensor quadrature plus the coefficient layout:
 * the C view of AssemblyProblem (sumfac.py:232-337) and of the SPEC's
 * MatrixFreeOperator. */
typedef struct {
  int32_t d;                                  /* 1..3                                   */
  igs_dir trial[IGS_MAX_DIM];
  igs_dir test[IGS_MAX_DIM];
  int32_t n_theta, n_eta;                     /* derivative index sets (geometry.py:48) */
  int8_t theta[IGS_MAX_DERIV_SET][IGS_MAX_DIM];
  int8_t eta[IGS_MAX_DERIV_SET][IGS_MAX_DIM];
  /* plane_of[i][j]: which coefficient plane holds F[:, eta_i, theta_j];
   * -1 marks an exactly-zero block that is skipped (geometry.py:296,305). */
  int8_t plane_of[IGS_MAX_DERIV_SET][IGS_MAX_DERIV_SET];
  int32_t n_planes;
  int64_t plane_stride;                       /* doubles between consecutive planes     */
  int32_t dir_order[IGS_MAX_DIM];             /* assembly direction order (sumfac.py:157) */
  int64_t num_pairs[IGS_MAX_DIM];             /* 1D pattern sizes (igs_pattern_1d counts)  */
  /* Slab along the LAST direction (multi-GPU partition).
   * Elements [slab_lo, slab_hi) of direction d-1; coefficient planes hold
   * exactly the points of those elements; apply vectors hold DoF layers
   * [slab_lo, slab_hi + order - 1).  slab_lo = slab_hi = 0 means "all". */
  int32_t slab_lo, slab_hi;
} igs_problem;

/* Operation codes for igs_workspace_bytes. */
enum { IGS_OP_ASSEMBLE = 1, IGS_OP_APPLY = 2, IGS_OP_EVAL_FIELD = 3, IGS_OP_PATTERN = 4 };

/* Flags for igs_assemble_values / igs_apply. */
enum {
  IGS_FLAG_DEFAULT = 0,
  IGS_FLAG_FORCE_GENERIC = 1,   /* use the stage-by-stage kernels even when a fused one applies */
  IGS_FLAG_ACCUMULATE = 2,      /* y += A x instead of y = A x (apply only)              */
  IGS_FLAG_KERNEL_ONLY = 4,     /* measurement: run only the fused main kernel (apply:
                                   apply3d, y untouched; two-pass assembly: stage 1(+2),
                                   values untouched; the one-pass symmetric assembly is a
                                   single kernel and runs whole) — the roofline's
                                   dominant kernel                                       */
  IGS_FLAG_TWO_PASS = 8,        /* assembly: the two-kernel fused path (stage-1/2 kernel,
                                   intermediate H in HBM) even where the one-pass
                                   symmetric kernel (3D p = 2, 4; 2D) or the three-pass
                                   path (3D p = 5, 6) applies                            */
  IGS_FLAG_SPLIT_BOUNDARY = 16, /* igs_apply_sharded: interior / boundary launches even
                                   without a next rank (exercises the overlap path)     */
  IGS_FLAG_THREE_PASS = 32      /* assembly, 3D p = 3..6: one direction per pass (x on
                                   DMMA, y and z sweeps; G and H in the workspace) even
                                   where another fused kernel is the default (p = 4)    */
};

/* ---- diagnostics ---------------------------------------------------- */
const char* igs_last_error(void);            /* thread-local, never NULL */
const char* igs_status_string(igs_status s);
int32_t igs_abi_version(void);
/* Which kernel family igs_apply / igs_assemble_values would run for this
 * problem: 0 = generic stage-by-stage, 1 = fused sm_100a kernel. */
int32_t igs_fused_path(const igs_problem* prob, int32_t op);

/* ---- K1: quadrature + tabulation ------------------------------------ */
/* Gauss-Legendre rule mapped into every element (quadrature.py:34-65 and
 * :87-106): `breakpoints` [nbp] ascending distinct (device), outputs
 * points/weights [(nbp-1)*k] element-major.  1 <= k <= 64. */
igs_status igs_gauss_rule(int32_t k, const double* breakpoints, int32_t nbp,
                          double* points, double* weights, void* stream);

/* Banded basis/derivative table at sorted points (bspline.py:314-333,
 * eval_all_derivs bspline.py:169-239, find_span bspline.py:153-166).
 * values [max_deriv+1][order][npts], first_active [npts].
 * Out-of-domain points -> IGS_EDOMAIN; max_deriv >= order -> IGS_EDERIV;
 * unsorted points -> IGS_EARG (all detected on device, reported here). */
igs_status igs_tabulate(int32_t order, const double* knots, int32_t nknots,
                        const double* points, int32_t npts, int32_t max_deriv,
                        double* values, int64_t* first_active, void* stream);

/* ---- K2: sparsity pattern ------------------------------------------- */
/* 1D interaction pattern (tensorspace.py:168-208, Lemma 3.1) of direction
 * `dir` as m-major CSR: rowptr [num_test+1] (int64), cols [count] (int64).
 * Two-phase: pass cols = NULL to get rowptr and *count only. */
igs_status igs_pattern_1d(const igs_problem* prob, int32_t dir, int64_t* rowptr,
                          int64_t* cols, int64_t* count /* host */, void* stream);

/* Tensor CSR pattern rows [row_lo, row_hi) (tensorspace.py:262-338):
 * indptr [row_hi-row_lo+1] (relative to row_lo's first entry when
 * `relative` != 0, else global offsets); indices int32 or int64
 * (index_bytes = 4 or 8).  The 1D patterns are passed explicitly. */
igs_status igs_pattern(const igs_problem* prob, const int64_t* const* rowptr1d,
                       const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                       int32_t relative, int64_t* indptr, void* indices,
                       int32_t index_bytes, void* stream);

/* ---- workspace ------------------------------------------------------ */
size_t igs_workspace_bytes(const igs_problem* prob, int32_t op, int32_t flags);

/* ---- K3: assembly (Alg. 1; sumfac.py:200-229, :358-379) -------------- */
/* values [nnz of rows row_lo..row_hi) in CSR order.  `block` selects one
 * derivative block (eta index i, theta index j) as in assemble_block
 * (sumfac.py:358-370); pass i = j = -1 for the full sum (assemble,
 * sumfac.py:373-379).  rowptr1d/cols1d are the 1D patterns. */
igs_status igs_assemble_values(const igs_problem* prob, const int64_t* const* rowptr1d,
                               const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                               int32_t block_eta, int32_t block_theta,
                               const double* planes, double* values, void* ws,
                               size_t ws_bytes, int32_t flags, void* stream);

/* ---- a22: direct-quadrature comparison oracle ------------------------- */
/* assemble_naive (sumfac.py:388-477) on the device: every entry of rows
 * [row_lo, row_hi) — entries [entry_lo, entry_hi) = indptr[row_lo],
 * indptr[row_hi] (host copies) — sums the weighted integrand of every
 * non-zero (theta, eta) block over the box where the knot supports of its
 * trial and test functions overlap (_support_column_ranges :382-385), with
 * no W operators or intermediates: an independent check of K3.  values
 * [entry_hi - entry_lo].  `updates` (device uint64 or NULL) is incremented
 * by the box size of every (entry, block), the reference's block_update
 * count (:475).  Whole fields only (no slab).  Small sizes: the caller
 * applies the reference's nominal-work budget. */
igs_status igs_assemble_naive(const igs_problem* prob, const int64_t* indptr, const void* indices,
                              int32_t index_bytes, int64_t row_lo, int64_t row_hi, int64_t entry_lo,
                              int64_t entry_hi, const double* planes, double* values,
                              uint64_t* updates, void* stream);

/* ---- K4: matrix-free apply (Alg. 2 + Alg. 3) --------- */
/* y = A x (or y += A x with IGS_FLAG_ACCUMULATE).  x has the trial DoF
 * count, y the test DoF count (of the slab, see igs_problem). */
igs_status igs_apply(const igs_problem* prob, const double* planes, const double* x,
                     double* y, void* ws, size_t ws_bytes, int32_t flags, void* stream);

/* Alg. 3 / contract_to_points (tensorspace.py:134-153) for one derivative
 * multi-index `deriv` [d] (host array) of the TRIAL space: out [#points]. */
igs_status igs_eval_field(const igs_problem* prob, const int8_t* deriv, const double* coeffs,
                          double* out, void* ws, size_t ws_bytes, void* stream);

/* ---- synthetic coefficients (SURVEY §8d workloads) ------------------- */
/* Fills SoA coefficient planes of a (X0, X1, X2) point grid, point layers
 * [z_lo, z_hi) of the last direction, with the seeded counter-based
 * generator: c ~ U[0.5,1.5], A = I + 0.05 G G^T / d with G ~ N(0,1).
 * kind: 1 = mass [c]; 2 = stiffness [a00,a11,(a22),a01,(a02,a12)];
 * 3 = mass+stiffness [c, then the stiffness planes]. */
igs_status igs_fill_synthetic(int32_t d, const int64_t* point_dims /* host [d] */,
                              int64_t z_lo, int64_t z_hi, int32_t kind, uint64_t seed,
                              double* planes, int64_t plane_stride, void* stream);

/* ---- CSR export --------------------------------- */
/* Writes a HOST CSR matrix as MatrixMarket coordinate `real general`,
 * 1-based, 17 significant digits. */
igs_status igs_write_matrix_market(const char* path /* host */, int64_t nrows, int64_t ncols,
                                   const int64_t* indptr /* host */, const int64_t* indices /* host */,
                                   const double* values /* host */);

/* ---- f1: coefficient field from a geometry map ---------- */
/* Pointwise half of eval_geometry + build_coefficient_field
 * (geometry.py:158-216 Jacobians, :121-155 cofactor inverse, :315-336
 * pullback).  The spline fields of the map come from igs_eval_field (Alg. 3)
 * on the map's own bases tabulated at the quadrature points.  All arrays are
 * device arrays of npts doubles in the flat point order. */
typedef struct {
  int32_t d;                          /* 1..3, physical dimension = d            */
  int64_t npts;
  const double* val[IGS_MAX_DIM];     /* G_c (weighted numerator w·G_c if rational) */
  const double* grad[IGS_MAX_DIM][IGS_MAX_DIM]; /* d/dx_k of val[c]            */
  const double* wval;                 /* weight spline w (NULL: polynomial map)  */
  const double* wgrad[IGS_MAX_DIM];   /* d/dx_k of w                             */
  /* PDE data (geometry.py:219-276): NULL = absent; stride 0 = one constant,
   * stride 1 = one value per point. */
  const double* reaction;
  int64_t reaction_stride;
  const double* convection[IGS_MAX_DIM];
  int64_t convection_stride;
  const double* diffusion[IGS_MAX_DIM][IGS_MAX_DIM];
  int64_t diffusion_stride;
  double rtol;                        /* degenerate if |det J| < rtol·max|J|^d (1e-12) */
} igs_pullback_args;

/* F = |det J|·E·[[c,0],[b,A]]·E^T, E = diag(1, J^{-1}), written as planes:
 * plane_of (host, [4][4] row-major, eta i x theta j over the first-order
 * set) maps F[i][j] to a plane (-1: not stored; a plane shared by (i,j) and
 * (j,i) is written once).  nonzero (device [n_planes]) gets 1 for every plane
 * holding a non-zero value; phys (device [d][npts] or NULL) the mapped
 * points.  *bad (host) = first point with a degenerate Jacobian, else -1.
 * Synchronises the stream (the degeneracy verdict is returned).  ws >= 64 B. */
igs_status igs_geometry_pullback(const igs_pullback_args* args, const int8_t* plane_of /* host */,
                                 int32_t n_planes, double* planes, int64_t plane_stride, double* phys,
                                 uint32_t* nonzero, int64_t* bad /* host */, void* ws, size_t ws_bytes,
                                 void* stream);

/* f1 fused: the map's spline fields evaluated in place at every point (sum
 * over its active control points of the tensor basis from its 1D value /
 * first-derivative tables at the quadrature points; rational maps by the
 * quotient rule) and pulled back in the same pass — only the planes (and
 * optionally phys) are written, no field arrays.  PDE data, npts and rtol
 * come from `pde` (its val/grad/wval/wgrad are ignored); outputs and the
 * degeneracy verdict as igs_geometry_pullback.  Map orders 2..8. */
typedef struct {
  int32_t d;
  int32_t order[IGS_MAX_DIM];          /* map basis orders                           */
  int32_t num_basis[IGS_MAX_DIM];      /* map basis counts (control grid, dir 0 fastest) */
  int64_t num_points[IGS_MAX_DIM];     /* quadrature points per direction            */
  const double* values[IGS_MAX_DIM];   /* [2][order][num_points]: B and dB/dx tables  */
  const int64_t* first_active[IGS_MAX_DIM];
  const double* control;               /* [num control points][d]                    */
  const double* weights;               /* [num control points] or NULL (polynomial)  */
} igs_geometry_map;

igs_status igs_geometry_planes(const igs_geometry_map* map, const igs_pullback_args* pde,
                               const int8_t* plane_of /* host */, int32_t n_planes, double* planes,
                               int64_t plane_stride, double* phys, uint32_t* nonzero, int64_t* bad /* host */,
                               void* ws, size_t ws_bytes, void* stream);

/* ---- K5: halo pack / unpack-add for the slab-partitioned apply ------- */
/* Copies `nlayers` contiguous DoF layers (layer = N0*N1 doubles) — kept
 * as kernels so they can be captured in CUDA graphs. dst[i] (+)= src[i]. */
igs_status igs_layers_copy(const double* src, double* dst, int64_t count, int32_t add,
                           void* stream);

/* ---- multi-GPU data plane ----------------------- */
/* NCCL communicators for the slab partition.  NCCL is resolved at run time
 * (libnccl.so.2 already loaded by the host process, else the system one);
 * `comm` is an ncclComm_t passed as void*.  Failures return IGS_ENCCL with
 * NCCL's message in igs_last_error(). */
igs_status igs_nccl_unique_id(uint8_t* id /* host [128] */);
igs_status igs_nccl_comm_init(const uint8_t* id /* host [128] */, int32_t nranks, int32_t rank,
                              void** comm /* host out */);
igs_status igs_nccl_comm_destroy(void* comm);
/* Asynchronous communicator error (peer failure, transport error, timeout
 * detected by NCCL) -> IGS_ENCCL; with abort_on_error the communicator is
 * aborted so pending operations return. */
igs_status igs_nccl_check(void* comm, int32_t abort_on_error);

/* One rank's part of y = A x for the slab partition along the last
 * direction (replaces the reference's single-process matvec, sumfac.py:112,
 * for the SPEC apply): `prob` carries this rank's slab
 * [slab_lo, slab_hi) (rank 0 owns element 0, the last rank the last one),
 * `planes` that slab's coefficient points; x_own / y_own hold the rank's own
 * DoF layers [slab_lo, slab_hi) (the last rank also the trailing order-1
 * layers).  The (order-1)-layer halo moves by NCCL send/recv: ghost gather
 * of x from rank+1, ghost reduce of y into rank+1.  With `comm_stream` (may
 * be NULL) the gather overlaps the interior elements.  `comm` may be NULL
 * for nranks = 1. */
size_t igs_apply_sharded_workspace(const igs_problem* prob, int32_t rank, int32_t nranks, int32_t flags);
igs_status igs_apply_sharded(const igs_problem* prob, const double* planes, const double* x_own, double* y_own,
                             void* ws, size_t ws_bytes, void* comm, int32_t rank, int32_t nranks,
                             int32_t flags, void* stream, void* comm_stream);

#ifdef __cplusplus
}
#endif
#endif /* IGS_CAPI_H */
