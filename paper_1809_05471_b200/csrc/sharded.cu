// Multi-GPU data plane of the slab-partitioned apply:
// igs_apply_sharded runs one rank's part of y = A x on its slab of elements
// [slab_lo, slab_hi) of the last direction, with the (p-1)-layer halo over
// NCCL point-to-point (NVLink / NVSwitch on one box):
//   1. ghost gather : x layers [hi, hi+p-1) from rank r+1      ncclSend/Recv
//   2. fused apply  : y over DoF layers [lo, hi+p-1)           apply3d + reduce
//   3. ghost reduce : trailing p-1 y layers added into rank r+1
// With a communication stream the gather overlaps the interior elements
// [lo, hi-p+1) (own x only); the boundary elements [hi-p+1, hi) run after
// it lands, accumulating (IGS_FLAG_ACCUMULATE).  NCCL is resolved at run
// time from the process (torch's libnccl.so.2 when loaded, else the system
// one), so the library has no link-time NCCL dependency; every NCCL failure
// maps to IGS_ENCCL with NCCL's message.
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "igs_internal.cuh"

namespace igs {
namespace {

// Minimal NCCL ABI (nccl.h): opaque communicator, 128-byte unique id.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclSuccess = 0, kNcclInProgress = 7, kNcclFloat64 = 8;

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
#define IGS_NCCL_SYM(field, name)                                          \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));          \
  if (!n.field) {                                                          \
    n.why = std::string("libnccl.so.2 lacks ") + name;                     \
    return;                                                                \
  }
    IGS_NCCL_SYM(GetUniqueId, "ncclGetUniqueId")
    IGS_NCCL_SYM(CommInitRank, "ncclCommInitRank")
    IGS_NCCL_SYM(CommDestroy, "ncclCommDestroy")
    IGS_NCCL_SYM(CommGetAsyncError, "ncclCommGetAsyncError")
    IGS_NCCL_SYM(CommAbort, "ncclCommAbort")
    IGS_NCCL_SYM(Send, "ncclSend")
    IGS_NCCL_SYM(Recv, "ncclRecv")
    IGS_NCCL_SYM(GroupStart, "ncclGroupStart")
    IGS_NCCL_SYM(GroupEnd, "ncclGroupEnd")
    IGS_NCCL_SYM(GetErrorString, "ncclGetErrorString")
#undef IGS_NCCL_SYM
    n.ok = true;
  });
  return n;
}

igs_status nccl_ready() {
  const Nccl& n = nccl();
  if (!n.ok) return fail(IGS_ENCCL, n.why);
  return IGS_OK;
}

igs_status nccl_check(ncclResult_t r, const char* what) {
  if (r == kNcclSuccess || r == kNcclInProgress) return IGS_OK;
  const Nccl& n = nccl();
  return fail(IGS_ENCCL, std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "nccl error"));
}

// The slab's geometry: layer = N0·N1 doubles, own / local layer counts.
struct SlabGeom {
  int p, lo, hi, K2;
  int64_t layer, n_own, n_local, g;  // g: halo doubles = (p-1)·layer
};

igs_status slab_geom(const igs_problem* prob, int rank, int nranks, SlabGeom* s) {
  if (prob->d != 3 && prob->d != 2) return fail(IGS_EARG, "sharded apply needs d = 2 or 3");
  const int L = prob->d - 1;
  const igs_dir& t = prob->trial[L];
  if (t.num_elements <= 0 || t.points_per_element <= 0)
    return fail(IGS_EARG, "sharded apply needs a per-element rule in the last direction");
  s->p = t.order;
  s->K2 = t.num_elements;
  const bool slab = prob->slab_lo || prob->slab_hi;
  s->lo = slab ? prob->slab_lo : 0;
  s->hi = slab ? prob->slab_hi : s->K2;
  if (s->lo < 0 || s->hi > s->K2 || s->hi <= s->lo) return fail(IGS_EARG, "bad slab");
  s->layer = 1;
  for (int k = 0; k < L; ++k) s->layer *= prob->trial[k].num_basis;
  const int last = rank == nranks - 1;
  if (last != (s->hi == s->K2)) return fail(IGS_EARG, "the last rank must own the last elements");
  if (rank == 0 && s->lo != 0) return fail(IGS_EARG, "rank 0 must own the first elements");
  s->n_local = (int64_t)(s->hi - s->lo + s->p - 1) * s->layer;
  s->n_own = last ? s->n_local : (int64_t)(s->hi - s->lo) * s->layer;
  s->g = (int64_t)(s->p - 1) * s->layer;
  return IGS_OK;
}

// A view of `prob` restricted to slab elements [a, b) (planes offset by the
// caller: the planes of the sub-slab start (a - lo)·k·layer_pts points in).
igs_problem sub_slab(const igs_problem* prob, int a, int b) {
  igs_problem q = *prob;
  q.slab_lo = a;
  q.slab_hi = b;
  return q;
}

int64_t layer_points(const igs_problem* prob) {
  int64_t n = 1;
  for (int k = 0; k + 1 < prob->d; ++k) n *= prob->trial[k].num_points;
  return n;
}

}  // namespace
}  // namespace igs

using namespace igs;

extern "C" igs_status igs_nccl_unique_id(uint8_t* id) {
  if (!id) return fail(IGS_EARG, "null id");
  IGS_TRY(nccl_ready());
  ncclUniqueId u;
  IGS_TRY(nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId"));
  std::memcpy(id, u.internal, sizeof(u.internal));
  return IGS_OK;
}

extern "C" igs_status igs_nccl_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, void** comm) {
  if (!id || !comm) return fail(IGS_EARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(IGS_EARG, "rank / nranks out of range");
  IGS_TRY(nccl_ready());
  ncclUniqueId u;
  std::memcpy(u.internal, id, sizeof(u.internal));
  ncclComm_t c = nullptr;
  IGS_TRY(nccl_check(nccl().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank"));
  *comm = c;
  return IGS_OK;
}

extern "C" igs_status igs_nccl_comm_destroy(void* comm) {
  if (!comm) return IGS_OK;
  IGS_TRY(nccl_ready());
  return nccl_check(nccl().CommDestroy(reinterpret_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

// Asynchronous communicator errors (a peer died, a transport failed): the
// caller polls this while it waits on the stream; a failed communicator is
// aborted so pending operations return.
extern "C" igs_status igs_nccl_check(void* comm, int32_t abort_on_error) {
  if (!comm) return fail(IGS_EARG, "null communicator");
  IGS_TRY(nccl_ready());
  ncclResult_t r = kNcclSuccess;
  IGS_TRY(nccl_check(nccl().CommGetAsyncError(reinterpret_cast<ncclComm_t>(comm), &r), "ncclCommGetAsyncError"));
  if (r != kNcclSuccess && r != kNcclInProgress) {
    if (abort_on_error) nccl().CommAbort(reinterpret_cast<ncclComm_t>(comm));
    return nccl_check(r, "communicator");
  }
  return IGS_OK;
}

extern "C" size_t igs_apply_sharded_workspace(const igs_problem* prob, int32_t rank, int32_t nranks,
                                              int32_t flags) {
  SlabGeom s;
  if (!prob || slab_geom(prob, rank, nranks, &s) != IGS_OK) return 0;
  const size_t apply_ws = igs_workspace_bytes(prob, IGS_OP_APPLY, flags & IGS_FLAG_FORCE_GENERIC);
  size_t split_ws = 0;
  if (s.hi - s.lo > s.p - 1) {
    igs_problem a = sub_slab(prob, s.lo, s.hi - s.p + 1), b = sub_slab(prob, s.hi - s.p + 1, s.hi);
    const size_t wa = igs_workspace_bytes(&a, IGS_OP_APPLY, flags & IGS_FLAG_FORCE_GENERIC);
    const size_t wb = igs_workspace_bytes(&b, IGS_OP_APPLY, flags & IGS_FLAG_FORCE_GENERIC);
    split_ws = wa > wb ? wa : wb;
  }
  const size_t aws = apply_ws > split_ws ? apply_ws : split_ws;
  auto up = [](size_t n) { return (n + 255) & ~size_t(255); };
  return up(s.n_local * 8) * 2 + up(s.g * 8) + up(aws) + 256;
}

extern "C" igs_status igs_apply_sharded(const igs_problem* prob, const double* planes, const double* x_own,
                                        double* y_own, void* ws, size_t ws_bytes, void* comm, int32_t rank,
                                        int32_t nranks, int32_t flags, void* stream, void* comm_stream) {
  if (!prob || !x_own || !y_own) return fail(IGS_EARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(IGS_EARG, "rank / nranks out of range");
  if (nranks > 1 && !comm) return fail(IGS_EARG, "a communicator is needed for more than one rank");
  SlabGeom s;
  IGS_TRY(slab_geom(prob, rank, nranks, &s));
  if (nranks > 1) IGS_TRY(nccl_ready());
  const size_t need = igs_apply_sharded_workspace(prob, rank, nranks, flags);
  if (!ws || ws_bytes < need) return fail(IGS_EWORKSPACE, "workspace too small for the sharded apply");
  Workspace w(ws, ws_bytes);
  double* xl = w.take<double>(s.n_local);
  double* yl = w.take<double>(s.n_local);
  double* halo = w.take<double>(s.g > 0 ? s.g : 1);
  const size_t aws_bytes = ws_bytes - ((w.used + 255) & ~size_t(255));
  void* aws = w.take<char>(aws_bytes);
  if (!w.ok()) return fail(IGS_EWORKSPACE, "workspace too small for the sharded apply");
  cudaStream_t st = as_stream(stream);
  cudaStream_t cs = comm_stream ? as_stream(comm_stream) : st;
  const Nccl& n = nccl();
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  const bool has_next = rank < nranks - 1, has_prev = rank > 0;
  const int fl = flags & IGS_FLAG_FORCE_GENERIC;
  // own x into the local vector (the ghost layers follow it)
  IGS_TRY(igs_layers_copy(x_own, xl, s.n_own, 0, st));
  const bool split = (has_next || (flags & IGS_FLAG_SPLIT_BOUNDARY)) && s.hi - s.lo > s.p - 1 && s.g > 0;
  cudaEvent_t ev_x = nullptr, ev_g = nullptr;
  auto cleanup = [&] {
    if (ev_x) cudaEventDestroy(ev_x);
    if (ev_g) cudaEventDestroy(ev_g);
  };
  if (cs != st) {
    if (cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_g, cudaEventDisableTiming) != cudaSuccess) {
      cleanup();
      return fail(IGS_ECUDA, "event creation failed");
    }
    cudaEventRecord(ev_x, st);          // x_local's own part is in place
    cudaStreamWaitEvent(cs, ev_x, 0);
  }
  // 1. ghost gather (on the communication stream)
  if (s.g > 0 && (has_prev || has_next)) {
    igs_status r = nccl_check(n.GroupStart(), "ncclGroupStart");
    if (r == IGS_OK && has_prev) r = nccl_check(n.Send(xl, (size_t)s.g, kNcclFloat64, rank - 1, c, cs), "ncclSend");
    if (r == IGS_OK && has_next)
      r = nccl_check(n.Recv(xl + s.n_own, (size_t)s.g, kNcclFloat64, rank + 1, c, cs), "ncclRecv");
    igs_status r2 = nccl_check(n.GroupEnd(), "ncclGroupEnd");
    if (r != IGS_OK || r2 != IGS_OK) {
      cleanup();
      return r != IGS_OK ? r : r2;
    }
  }
  if (cs != st) cudaEventRecord(ev_g, cs);
  igs_status r = IGS_OK;
  if (split) {
    // 2a. interior elements (own x only) while the ghosts are in flight
    const int cut = s.hi - s.p + 1;
    const int64_t kq = prob->trial[prob->d - 1].points_per_element;
    igs_problem a = sub_slab(prob, s.lo, cut), b = sub_slab(prob, cut, s.hi);
    const double* pb = planes + (int64_t)(cut - s.lo) * kq * layer_points(prob);
    r = igs_apply(&a, planes, xl, yl, aws, aws_bytes, fl, st);
    if (r == IGS_OK) {
      // the interior wrote layers [lo, cut + p - 1); the boundary adds into
      // [cut, hi + p - 1): its layers beyond the interior's start at zero
      const int64_t off = (int64_t)(cut - s.lo) * s.layer;
      r = cuda_check(cudaMemsetAsync(yl + (int64_t)(cut - s.lo + s.p - 1) * s.layer, 0,
                                     (size_t)(s.n_local - (int64_t)(cut - s.lo + s.p - 1) * s.layer) * 8, st),
                     "memset");
      if (r == IGS_OK && cs != st) cudaStreamWaitEvent(st, ev_g, 0);
      // 2b. the boundary elements need the ghost layers
      if (r == IGS_OK) r = igs_apply(&b, pb, xl + off, yl + off, aws, aws_bytes, fl | IGS_FLAG_ACCUMULATE, st);
    }
  } else {
    if (cs != st) cudaStreamWaitEvent(st, ev_g, 0);
    r = igs_apply(prob, planes, xl, yl, aws, aws_bytes, fl, st);
  }
  if (r != IGS_OK) {
    cleanup();
    return r;
  }
  // 3. ghost reduce: my trailing p-1 partial layers go to r+1; r-1's come in
  if (s.g > 0 && (has_prev || has_next)) {
    igs_status q = nccl_check(n.GroupStart(), "ncclGroupStart");
    if (q == IGS_OK && has_next)
      q = nccl_check(n.Send(yl + s.n_own, (size_t)s.g, kNcclFloat64, rank + 1, c, st), "ncclSend");
    if (q == IGS_OK && has_prev) q = nccl_check(n.Recv(halo, (size_t)s.g, kNcclFloat64, rank - 1, c, st), "ncclRecv");
    igs_status q2 = nccl_check(n.GroupEnd(), "ncclGroupEnd");
    if (q != IGS_OK || q2 != IGS_OK) {
      cleanup();
      return q != IGS_OK ? q : q2;
    }
    if (has_prev) r = igs_layers_copy(halo, yl, s.g, 1, st);
  }
  if (r == IGS_OK) r = igs_layers_copy(yl, y_own, s.n_own, 0, st);
  cleanup();  // events may be destroyed while pending work still references them
  return r;
}
