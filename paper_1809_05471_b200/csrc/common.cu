// Error plumbing, problem validation and small utility kernels.
#include "igs_internal.cuh"

#include <cstring>

namespace igs {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
const std::string& get_error() { return g_last_error; }

// Structural checks of an igs_problem (the C mirror of the argument checks
// in AssemblyProblem.__init__, sumfac.py:241-268, and of
// _check_block_indices, sumfac.py:340-355).
igs_status validate_problem(const igs_problem* p, Dims* dims, unsigned need) {
  if (!p) return fail(IGS_EARG, "null problem");
  if (p->d < 1 || p->d > IGS_MAX_DIM) return fail(IGS_EARG, "dimension must be 1..3");
  if (p->n_theta < 1 || p->n_theta > IGS_MAX_DERIV_SET || p->n_eta < 1 ||
      p->n_eta > IGS_MAX_DERIV_SET)
    return fail(IGS_EARG, "derivative index sets must hold 1..8 multi-indices");
  const int d = p->d;
  for (int k = 0; k < d; ++k) {
    const igs_dir* dirs[2] = {&p->trial[k], &p->test[k]};
    for (const igs_dir* t : dirs) {
      if (t->order < 1 || t->order > IGS_MAX_ORDER)
        return fail(IGS_ECAPACITY, "spline order outside [1, 16]");
      if (t->num_basis < 1) return fail(IGS_EARG, "empty basis");
      if (t->num_points < 0) return fail(IGS_EARG, "negative point count");
      if (t->max_deriv < 0 || t->max_deriv >= t->order)
        return fail(IGS_EDERIV, "table derivative level outside [0, order)");
      if ((need & NEED_TABLES) && t->num_points > 0 && (!t->values || !t->first_active))
        return fail(IGS_EARG, "null table pointer");
      if ((need & NEED_WEIGHTS) && t->num_points > 0 && !t->weights)
        return fail(IGS_EARG, "null weight pointer");
    }
    if (p->trial[k].num_points != p->test[k].num_points)
      return fail(IGS_EARG, "trial and test tables are on different point sets");
  }
  for (int i = 0; i < p->n_theta; ++i)
    for (int k = 0; k < d; ++k) {
      int lv = p->theta[i][k];
      if (lv < 0) return fail(IGS_EARG, "negative derivative level");
      if (lv >= p->trial[k].order)
        return fail(IGS_EDERIV, "trial derivative exceeds order in direction " + std::to_string(k));
      if ((need & NEED_TABLES) && lv > p->trial[k].max_deriv)
        return fail(IGS_EARG, "trial table too shallow");
    }
  for (int i = 0; i < p->n_eta; ++i)
    for (int k = 0; k < d; ++k) {
      int lv = p->eta[i][k];
      if (lv < 0) return fail(IGS_EARG, "negative derivative level");
      if (lv >= p->test[k].order)
        return fail(IGS_EDERIV, "test derivative exceeds order in direction " + std::to_string(k));
      if ((need & NEED_TABLES) && lv > p->test[k].max_deriv)
        return fail(IGS_EARG, "test table too shallow");
    }
  for (int i = 0; i < p->n_eta; ++i)
    for (int j = 0; j < p->n_theta; ++j) {
      int pl = p->plane_of[i][j];
      if (pl < -1 || pl >= p->n_planes) return fail(IGS_EARG, "plane_of out of range");
    }
  bool seen[IGS_MAX_DIM] = {false, false, false};
  for (int k = 0; k < d; ++k) {
    int o = p->dir_order[k];
    if (o < 0 || o >= d || seen[o]) return fail(IGS_EARG, "dir_order must be a permutation of the directions");
    seen[o] = true;
  }
  Dims D;
  D.d = d;
  for (int k = 0; k < IGS_MAX_DIM; ++k) {
    D.nt[k] = k < d ? p->trial[k].num_basis : 1;
    D.ns[k] = k < d ? p->test[k].num_basis : 1;
    D.x[k] = k < d ? p->trial[k].num_points : 1;
  }
  D.x_off = D.nt_off = D.ns_off = 0;
  const int L = d - 1;
  if (p->slab_lo != 0 || p->slab_hi != 0) {
    const igs_dir& tl = p->trial[L];
    const igs_dir& sl = p->test[L];
    int kq = tl.points_per_element;
    if (kq <= 0 || tl.num_elements <= 0 || sl.points_per_element != kq)
      return fail(IGS_EARG, "slabs need a per-element rule in the last direction");
    if (tl.num_basis != tl.num_elements + tl.order - 1 || sl.num_basis != sl.num_elements + sl.order - 1)
      return fail(IGS_ECAPACITY, "slabs need maximum-smoothness knots in the last direction");
    if (p->slab_lo < 0 || p->slab_hi <= p->slab_lo || p->slab_hi > tl.num_elements)
      return fail(IGS_EARG, "slab range outside [0, num_elements]");
    D.x_off = (int64_t)p->slab_lo * kq;
    D.x[L] = (int64_t)(p->slab_hi - p->slab_lo) * kq;
    D.nt_off = p->slab_lo;
    D.nt[L] = p->slab_hi - p->slab_lo + tl.order - 1;
    D.ns_off = p->slab_lo;
    D.ns[L] = p->slab_hi - p->slab_lo + sl.order - 1;
  }
  if (dims) *dims = D;
  return IGS_OK;
}

namespace {
__global__ void layers_copy_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                   int64_t n, int add) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = add ? dst[i] + src[i] : src[i];
}
}  // namespace

}  // namespace igs

using namespace igs;

extern "C" const char* igs_last_error(void) { return get_error().c_str(); }

extern "C" const char* igs_status_string(igs_status s) {
  switch (s) {
    case IGS_OK: return "ok";
    case IGS_EARG: return "invalid argument";
    case IGS_EDOMAIN: return "point outside the domain";
    case IGS_EDERIV: return "unsupported derivative order";
    case IGS_ECAPACITY: return "capacity exceeded / unsupported configuration";
    case IGS_ECUDA: return "CUDA error";
    case IGS_ENCCL: return "collective error";
    case IGS_EWORKSPACE: return "workspace too small";
  }
  return "unknown status";
}

extern "C" int32_t igs_abi_version(void) { return IGS_ABI_VERSION; }

extern "C" igs_status igs_layers_copy(const double* src, double* dst, int64_t count, int32_t add,
                                      void* stream) {
  if (count == 0) return IGS_OK;
  if (!src || !dst || count < 0) return fail(IGS_EARG, "bad layer copy arguments");
  int block = 256;
  int64_t grid = ceil_div(count, block);
  if (grid > 148 * 16) grid = 148 * 16;
  layers_copy_kernel<<<(unsigned)grid, block, 0, as_stream(stream)>>>(src, dst, count, add);
  IGS_LAUNCH_CHECK("layers_copy_kernel");
  return IGS_OK;
}

// ---- TMA tensor maps over coefficient planes ---------------------------------
#include "tma.cuh"

namespace igs {

// L2 promotion of the assembly kernels' coefficient boxes (measurement
// builds override it; 256 bytes measured best or equal everywhere)
#ifndef IGS_ASM_L2_PROMO
#define IGS_ASM_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
igs_status planes_tensor_map(CUtensorMap* map, const double* planes, const int64_t dims[4],
                             int64_t pstride, const unsigned box[4]) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(IGS_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t gd[4] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2], (cuuint64_t)dims[3]};
  cuuint64_t gs[3] = {(cuuint64_t)dims[0] * 8, (cuuint64_t)(dims[0] * dims[1]) * 8, (cuuint64_t)pstride * 8};
  cuuint32_t bd[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(planes), gd, gs, bd, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      IGS_ASM_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(IGS_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return IGS_OK;
}

}  // namespace igs
