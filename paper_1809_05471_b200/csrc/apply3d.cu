// K4 — fused 3D matrix-free apply (Alg. 2 with Alg. 3 as its first half).
//
//   y = Σ_eta Q_eta^T · w · Σ_theta F_{eta,theta} · Q_theta · x
//
// for uniform-structure problems (trial == test, order P in every
// direction, Q Gauss points per element, first-order derivative sets,
// symmetric mass/stiffness coefficient planes) — SPEC.md:461-483,
// PAPER.md Alg. 2 (lines 818-839) and Alg. 3 (tensorspace.py:134-153).
//
// Decomposition: one CTA per work item = an EX×EY tile of
// elements in (x, y) times a chunk of EZ element layers in z.  The CTA
// sweeps its chunk layer by layer; for every z point layer q2 it runs
//
//   Z   : A_v[n1][n0]  = Σ_j Bz_v[q2][j] · x[e2+j][n1][n0]        (v: val, z-der)
//   Y   : C_vw[q1][n0] = Σ_j By_w[q1][j] · A_v[ey+j][n0]           (3 variants)
//   X   : u, ∂x u, ∂y u, ∂z u at every point of a line segment,
//         g = w · F(x) · ∇u  (F streamed from HBM exactly once),
//         X^T partial sums per element                             (registers)
//   X^T : R_v[q1][n0] = Σ_elements partials
//   Y^T : S_v[n1][n0]  = Σ_q1 By · R
//   Z^T : yring[e2+j][n1][n0] += Bz_v[q2][j] · S_v
//
// so every intermediate stays in shared memory/registers; HBM traffic is
// the coefficient planes (read once), x (L2-resident) and one scratch box
// of partial y per work item.  Boxes overlap by P-1 DoFs in each direction;
// `apply_reduce_kernel` sums them in a fixed order (deterministic, no fp64
// atomics).
#include "fused.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>

#ifdef IGS_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[8];
#define PHASE_MARK(k)                                                             \
  do {                                                                            \
    if (threadIdx.x == 0) {                                                       \
      long long now_ = clock64();                                                 \
      atomicAdd(&g_phase_cycles[k], (unsigned long long)(now_ - phase_t0_));      \
      phase_t0_ = now_;                                                           \
    }                                                                             \
  } while (0)
#else
#define PHASE_MARK(k) \
  do {                \
  } while (0)
#endif

namespace igs {

bool fused_shape(const igs_problem* p, const Dims& D, FusedShape* fs) {
  const int d = p->d;
  FusedShape s{};
  s.d = d;
  s.p = p->trial[0].order;
  s.k = p->trial[0].points_per_element;
  for (int k = 0; k < d; ++k) {
    const igs_dir& t = p->trial[k];
    const igs_dir& u = p->test[k];
    if (t.order != s.p || u.order != s.p) return false;
    if (t.points_per_element != s.k || u.points_per_element != s.k || s.k <= 0) return false;
    if (t.num_elements <= 0 || t.num_basis != t.num_elements + t.order - 1) return false;
    if (t.values != u.values || t.first_active != u.first_active || t.weights != u.weights) return false;
    if (t.num_points != t.num_elements * s.k) return false;
    if (t.max_deriv < 1) return false;
  }
  // derivative sets must be exactly (0, e_1, ..., e_d) in that order
  if (p->n_theta != d + 1 || p->n_eta != d + 1) return false;
  for (int i = 0; i <= d; ++i)
    for (int k = 0; k < d; ++k) {
      int want = (i >= 1 && k == i - 1) ? 1 : 0;
      if (p->theta[i][k] != want || p->eta[i][k] != want) return false;
    }
  s.mass = p->plane_of[0][0] >= 0;
  s.stiff = 0;
  s.general = 0;
  for (int a = 0; a < d; ++a) {
    if (p->plane_of[0][1 + a] >= 0 || p->plane_of[1 + a][0] >= 0) s.general = 1;  // convection
    for (int b = 0; b < d; ++b) {
      if (p->plane_of[1 + a][1 + b] >= 0) s.stiff = 1;
      if (p->plane_of[1 + a][1 + b] != p->plane_of[1 + b][1 + a]) s.general = 1;
    }
  }
  if (s.stiff)
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b)
        if (p->plane_of[1 + a][1 + b] < 0) s.general = 1;  // partial stiffness: generic path
  for (int k = 0; k < 3; ++k) {
    s.nel[k] = k < d ? (k == d - 1 && (p->slab_lo || p->slab_hi) ? p->slab_hi - p->slab_lo
                                                                 : p->trial[k].num_elements)
                     : 1;
    s.nfn[k] = D.nt[k];
    s.npt[k] = D.x[k];
  }
  if (fs) *fs = s;
  return !s.general && (s.mass || s.stiff);
}

namespace {

struct ApplyArgs {
  const double* x;            // slab-local trial vector [N2][N1][N0]
  const double* planes;
  int64_t pstride;
  int pl_c;                   // mass plane
  int pl_a[3][3];             // stiffness planes (symmetric)
  const double* vals[3];      // tables [2][P][xtab] per direction (global)
  const double* wts[3];       // quadrature weights (global)
  int64_t xtab[3];
  int64_t N0, N1, N2;         // local DoF counts
  int64_t X0, X1;             // points in x, y
  int K0, K1, K2;             // elements (K2 slab-local)
  int z_el_off;               // global element index of local z element 0
  int ntx, nty, nch, ez;      // tiling
  int uni_x;                  // equally spaced x breakpoints (interior tables shared)
  int l2pf;                   // measurement: -1 = re-read one box (L2-resident, no HBM stream)
  double* scratch;            // per-item boxes
  int64_t box;                // doubles per box
};

// fp64 tensor-core MMA (DMMA.8x8x4 on sm_100a): D(8x8) += A(8x4) · B(4x8).
// Fragments (lane = 4·g + m): A[g][m], B[m][g], D[g][2m], D[g][2m+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// (A suspend-time hint on try_wait was measured 3 % slower over BASELINE's
// 100 sustained applies: the wake-up latency costs more than the spin.)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA: one 4D box (8 points, 8 lines, 1 point layer, all planes).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// Tile geometry and shared-memory plan.  Q2B point layers of z are processed
// per batch; warp w owns (point layer w / NLG of the batch, line group
// w % NLG) in the X phase and sweeps all EX elements of its 8 lines.
template <int P, int Q, int EX, int EY, int Q2B, bool MASS, bool STIFF, int STG_>
struct Cfg {
  static_assert(P >= 2 && P <= 8 && Q >= 1 && Q <= 8, "orders 2..8, up to 8 points per element");
  static_assert(Q % Q2B == 0, "batches tile the element's point layers");
  static constexpr int FX = EX + P - 1, FY = EY + P - 1;
  static_assert(FY <= 16, "S-row line-group table holds 16 rows");
  static_assert(EX + 7 <= 16, "x footprint must fit two 8-column MMA tiles");
  static constexpr int RP = 20;                // row pitch (16 used columns, bank-spread)
  static constexpr int FYP = EY + 8;           // rows incl. MMA padding
  static constexpr int TX = EX * Q, TY = EY * Q;
  static_assert(TY % 8 == 0, "lines come in MMA groups of 8");
  static constexpr int NLG = TY / 8;           // line groups
  static constexpr int NW = Q2B * NLG, NT = 32 * NW;
  static constexpr int NB = Q / Q2B;           // batches per element layer
  // the DoF rows a line group touches in y fit one 8-row MMA operand
  static constexpr bool y_rows_fit() {
    for (int lg = 0; lg < NLG; ++lg)
      if ((lg * 8 + 7) / Q - (lg * 8) / Q + P - 1 > 7) return false;
    return true;
  }
  static_assert(y_rows_fit(), "line group spans more than 8 DoF rows");
  static constexpr int NA = STIFF ? 2 : 1;     // z variants: value, z-derivative
  static constexpr int NV = STIFF ? 3 : 1;     // (y, z) variants: 00, 10, 01
  static constexpr int NPL = (MASS ? 1 : 0) + (STIFF ? 6 : 0);  // coefficient planes
  // The X sweep walks 8-point windows of the tile's TX = EX·Q points (one
  // MMA n-tile each, whatever Q is); window w spans elements
  // [8w/Q, (8w+7)/Q] and DoF columns [c0(w), c0(w) + 8), c0(w) = 8w/Q.
  static_assert((EX * Q) % 8 == 0, "windows tile the element row");
  static constexpr int NWIN = EX * Q / 8;      // windows per (batch, line group)
  static constexpr int NBX = NWIN;             // TMA boxes (one window each)
  static constexpr int QE = 8;                 // TMA box width (64-byte rows)
  static constexpr int c0w(int w) { return (8 * w) / Q; }
  static constexpr int gcd8(int q) { return q % 8 == 0 ? 8 : q % 4 == 0 ? 4 : q % 2 == 0 ? 2 : 1; }
  static constexpr int PER = Q / gcd8(Q);      // windows per period of the table pattern
  // X^T accumulator as a circular buffer over DoF columns (slot = column
  // mod 8; window tables rotated to match) instead of sliding it across lanes
  // (12 shuffles) after every window.  Windows of one pattern (PER = 1) then
  // load their own rotated table instead of sharing a hoisted one (measured:
  // C4 3.84 -> 3.75 ms, C5 11.3 -> 10.9 ms).  IGS_APPLY_ROT=0 (measurement
  // builds) restores the sliding window.
#ifndef IGS_APPLY_SYNCWARP
#define IGS_APPLY_SYNCWARP 0
#endif
#ifndef IGS_APPLY_ROT
  static constexpr bool ROT = true;
#else
  static constexpr bool ROT = IGS_APPLY_ROT;
#endif
  static constexpr int STG = STG_;             // TMA stages (boxes) per warp
  static constexpr int FST = NPL * 8 * QE;     // doubles per stage
  static constexpr int LXR = FYP * RP;         // one [n1][n0] plane
  static constexpr int XR = P * LXR;           // x ring (P DoF layers)
  static constexpr int AQ = Q2B * NA * LXR;    // A per point layer of the batch
  static constexpr int CQL = TY * RP;          // one C/R variant plane
  static constexpr int CQ = Q2B * NV * CQL;    // C, overwritten in place by R
  static constexpr int YR = P * LXR;           // y ring
  static constexpr int TBX = NWIN * 256, TBY = EY * 128, TBZ = 256;  // Tw [w][4][lane][2]; Ty/Tz [e][v][q8][j8]
  static constexpr int WW = TX + TY + 16;
  static constexpr int FS = NW * STG * FST;    // coefficient staging
  static constexpr int TOTAL = FS + XR + AQ + CQ + YR + TBX + TBY + TBZ + WW;
  static constexpr size_t SMEM = (size_t)TOTAL * sizeof(double) + NW * STG * sizeof(uint64_t) + 16 * sizeof(int);
  static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;  // CTAs per SM the tile allows
};

template <int P, int Q, int EX, int EY, int Q2B, bool MASS, bool STIFF, int STG_>
__global__ void __launch_bounds__(Cfg<P, Q, EX, EY, Q2B, MASS, STIFF, STG_>::NT,
                                  Cfg<P, Q, EX, EY, Q2B, MASS, STIFF, STG_>::MINB)
    apply3d_kernel(const ApplyArgs a, const __grid_constant__ CUtensorMap fmap) {
  using C = Cfg<P, Q, EX, EY, Q2B, MASS, STIFF, STG_>;
  constexpr int FX = C::FX, FY = C::FY, RP = C::RP, TX = C::TX, TY = C::TY;
  constexpr int NT = C::NT, NW = C::NW, LXR = C::LXR, STG = C::STG, FST = C::FST, QE = C::QE;
  constexpr int NLG = C::NLG, NB = C::NB, CQL = C::CQL, NA = C::NA, NV = C::NV;
  extern __shared__ __align__(128) double sm[];
  double* Fs = sm;              // [NW][STG][NPL][8][QE]  (TMA destination)
  double* Xr = Fs + C::FS;      // [P][FYP][RP]
  double* Aq = Xr + C::XR;      // [Q2B][NA][FYP][RP]
  // C, then R in place, then the warp's Y^T partials S_v over its own rows
  double* Cq = Aq + C::AQ;      // [Q2B][NV][TY][RP]
  double* Yr = Cq + C::CQ;      // [P][FYP][RP]
  double* Tw = Yr + C::YR;      // [NWIN][4][32 lanes][2]  window table fragments
  double* Ty = Tw + C::TBX;     // [EY][2][8][8]
  double* Tzb = Ty + C::TBY;    // [2 buffers][2][8][8]
  double* Wx = Tzb + C::TBZ;    // [TX] (unused: w_x lives in the X^T window tables)
  double* Wy = Wx + TX;         // [TY]
  double* Wzb = Wy + TY;        // [2 buffers][8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(Wzb + 16);  // [NW][STG]
  int* zr = reinterpret_cast<int*>(bars + NW * STG);       // [FY] line-group range per S row

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, m = lane & 3;  // MMA fragment coordinates
  const int item = blockIdx.x;
#ifdef IGS_PHASE_TIMING
  long long phase_t0_ = clock64();
#endif
  const int tx = item % a.ntx;
  const int ty = (item / a.ntx) % a.nty;
  const int tz = item / (a.ntx * a.nty);
  const int ex0 = tx * EX, ey0 = ty * EY;
  const int z0 = tz * a.ez;
  const int z1 = min(a.K2, z0 + a.ez);
  double* box = a.scratch + (int64_t)item * a.box;

  // ---- coefficient stream: warp w's X task in every batch covers point
  // layer (batch·Q2B + w/NLG) and line group w%NLG, element by element; each
  // (batch, element) is one TMA box, STG boxes in flight per warp.
  const int wq = warp / NLG, wlg = warp % NLG;
  // ring stage / parity of a task: static per box when STG divides the
  // boxes of a row into an even number of rounds, else from the task index
  constexpr int NBX = C::NBX, NWIN = C::NWIN;
  constexpr bool kStaticRing = NBX % STG == 0 && (NBX / STG) % 2 == 0;
  // every element of the tile interior (e in [P-1, K0-P]): one shared table
  const bool tile_uniform = a.uni_x && ex0 >= P - 1 && ex0 + EX - 1 <= a.K0 - P;
  const int ntask = (z1 - z0) * NB * NBX;
  uint64_t* mybar = bars + warp * STG;
  double* mystage = Fs + warp * STG * FST;
  // one lane: box of window bx of point layer zq into ring stage stg
#ifdef IGS_DEV_SWITCHES
  const bool co = a.l2pf < 0;  // compute-only measurement mode
#else
  constexpr bool co = false;
#endif
  const int tma_x = ex0 * Q, tma_y = ey0 * Q + wlg * 8;
  auto issue_box = [&](int stg, int bx, int zq) {
    uint64_t* bar = mybar + stg;
    mbar_expect_tx(bar, (unsigned)(FST * sizeof(double)));
    tma_load_4d(mystage + stg * FST, &fmap, bar, co ? tma_x : tma_x + bx * 8, tma_y, co ? 0 : zq, 0);
  };
  auto issue = [&](int idx) {  // box idx = (batch, window)
    const int batch = idx / NBX, bx = idx % NBX;
    issue_box(idx % STG, bx, (z0 + batch / NB) * Q + (batch % NB) * Q2B + wq);
  };
  // lanes past the box width of odd Q read neighbouring stage memory (masked
  // by zero weights): keep it finite
  for (int i = tid; i < C::FS; i += NT) Fs[i] = 0.0;
  if (tid < NW * STG) mbar_init(bars + tid, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros before TMA writes
  __syncthreads();
  if (lane == 0)
    for (int i = 0; i < STG && i < ntask; ++i) issue(i);

  // ---- prologue ---------------------------------------------------------------
  for (int i = tid; i < C::TOTAL - C::FS; i += NT) Xr[i] = 0.0;  // all MMA padding is zero
  __syncthreads();
  // Window table fragments in lane order (one 16-byte load per pair):
  // B^v(c, pt) = B^v of DoF column c0(w) + c at window point pt (zero outside
  // the support or past the mesh); pair kp = 0, 1: forward B^v[c = m + 4s][pt
  // = g] (v = kp), kp = 2, 3: transpose B^v[pt = 2m + s][c] (v = kp - 2) for
  // the accumulator column g, which holds DoF column ≡ g (mod 8) of the
  // window (c = (g - c0(w)) mod 8): the X^T accumulator is a circular buffer
  // over the DoF columns, so windows never move it between lanes.
  for (int i = tid; i < NWIN * 256; i += NT) {
    const int s = i % 2, ln = (i / 2) % 32, kp = (i / 64) % 4, w = i / 256;
    const int lg = ln >> 2, lm = ln & 3, v = kp & 1;
    const int c = kp < 2 ? lm + 4 * s : C::ROT ? ((lg - C::c0w(w)) & 7) : lg, pt = kp < 2 ? lg : 2 * lm + s;
    const int el = (8 * w + pt) / Q, j = (8 * w) / Q + c - el, ge = ex0 + el;
    double val = 0.0;
    if (ge < a.K0 && j >= 0 && j < P && (v == 0 || STIFF)) {
      const int64_t x = (int64_t)ex0 * Q + 8 * w + pt;
      val = a.vals[0][((int64_t)v * P + j) * a.xtab[0] + x];
      if (kp >= 2) val *= a.wts[0][x];  // test side: the x quadrature weight folded in
    }
    Tw[i] = val;
  }
  for (int i = tid; i < EY * 2 * Q * P; i += NT) {
    int j = i % P, q = (i / P) % Q, v = (i / (P * Q)) % 2, e = i / (2 * P * Q);
    int ge = ey0 + e;
    if (ge < a.K1)
      Ty[((e * 2 + v) * 8 + q) * 8 + j] = a.vals[1][((int64_t)v * P + j) * a.xtab[1] + (int64_t)ge * Q + q];
  }
  for (int i = tid; i < TY; i += NT) {
    int64_t gg = (int64_t)ey0 * Q + i;
    if (gg < a.X1) Wy[i] = a.wts[1][gg];
  }
  // asynchronous 8-byte copies (LDGSTS) with zero fill past the domain: the
  // next element's x layer and z tables stream in behind the last batch
  auto cp8 = [](double* dst, const double* src, bool ok) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0)
                 : "memory");
  };
  // Y fragments of this warp's 8 lines (line = wlg·8 + g lies in element
  // line / Q at point line % Q): A[g][k] = By_v[line % Q][ynb + k - line / Q]
  // over DoF rows ynb + k, k = m + 4s (zero outside the element's support)
  const int ynb = (wlg * 8) / Q;
  // (recomputed from the shared Ty table where used: no registers held
  // across the X sweep)
  auto y_frag = [&](int v, int s) {
    const int line = wlg * 8 + g, eyl = line / Q, q1 = line % Q, jj = ynb + m + 4 * s - eyl;
    return (jj >= 0 && jj < P && (v == 0 || STIFF)) ? Ty[((eyl * 2 + v) * 8 + q1) * 8 + jj] : 0.0;
  };
  // transpose: A[k = g][line' = m + 4s] = w_y(line')·By_v[line' % Q][ynb + g - line' / Q]
  // (test side: the y quadrature weight folded in; zero past the mesh)
  auto yt_frag = [&](int v, int s) {
    const int lt = wlg * 8 + m + 4 * s, eyt = lt / Q, qt = lt % Q, jt = ynb + g - eyt;
    return (jt >= 0 && jt < P && (v == 0 || STIFF)) ? Ty[((eyt * 2 + v) * 8 + qt) * 8 + jt] * Wy[lt] : 0.0;
  };
  __syncthreads();
  for (int n1 = tid; n1 < FY; n1 += NT) {
    int lo = NLG, hi = -1;
    for (int lg = 0; lg < NLG; ++lg) {
      const int nb = (lg * 8) / Q, ne = (lg * 8 + 7) / Q + P - 1;
      if (nb <= n1 && n1 <= ne) {
        lo = min(lo, lg);
        hi = max(hi, lg);
      }
    }
    zr[n1] = lo | (hi << 8);
  }
  auto load_layer = [&](int n2) {
    double* dst = Xr + (n2 % P) * LXR;
    for (int i = tid; i < FY * FX; i += NT) {
      int n0 = i % FX, n1 = i / FX;
      int64_t g0 = (int64_t)ex0 + n0, g1 = (int64_t)ey0 + n1;
      const bool ok = g0 < a.N0 && g1 < a.N1 && n2 < a.N2;
      cp8(dst + n1 * RP + n0, ok ? a.x + ((int64_t)n2 * a.N1 + g1) * a.N0 + g0 : a.x, ok);
    }
  };
  auto load_ztab = [&](int e2, int zb) {
    const int gz = e2 + a.z_el_off;
    for (int i = tid; i < 2 * Q * P; i += NT) {
      int j = i % P, q = (i / P) % Q, v = i / (P * Q);
      cp8(Tzb + zb * 128 + (v * 8 + q) * 8 + j, a.vals[2] + ((int64_t)v * P + j) * a.xtab[2] + (int64_t)gz * Q + q,
          true);
    }
    for (int i = tid; i < Q; i += NT) cp8(Wzb + zb * 8 + i, a.wts[2] + (int64_t)gz * Q + i, true);
  };
  for (int l = 0; l < P; ++l) load_layer(z0 + l);
  if (z0 < z1) load_ztab(z0, 0);

  // plane slots inside a TMA stage
  const int pc = a.pl_c;
  const int p00 = a.pl_a[0][0], p11 = a.pl_a[1][1], p22 = a.pl_a[2][2];
  const int p01 = a.pl_a[0][1], p02 = a.pl_a[0][2], p12 = a.pl_a[1][2];

  // Z^T of the Q2B point layers of batch `b` into the y ring (item mapping
  // (n1, n0) identical in every phase that touches the ring).  S row n1 is
  // the fixed-order sum of the partials of line groups zr[n1] = lo | hi << 8.
  // The z quadrature weight of point layer q2 scales its partials (test side).
  auto zt_item = [&](const double* Tz, const double* Wzp, int e2, int b, int i) {
    const int n0 = i % FX, n1 = i / FX, o = n1 * RP + n0;
    const int lr = zr[n1], lo = lr & 255, hi = lr >> 8;
    double s0[Q2B], s1[Q2B];
#pragma unroll
    for (int qb = 0; qb < Q2B; ++qb) {
      double a0 = 0.0, a1 = 0.0;
      // line group lg's partial of DoF row n1 sits in row lg·8 + n1 - lg·8/Q
      const double* sp = Cq + qb * NV * CQL + n1 * RP + n0;
#pragma unroll
      for (int lg = 0; lg < NLG; ++lg)
        if (lg >= lo && lg <= hi) {
          a0 += sp[(lg * 8 - (lg * 8) / Q) * RP];
          if (STIFF) a1 += sp[(lg * 8 - (lg * 8) / Q) * RP + CQL];
        }
      const double wz = Wzp[b * Q2B + qb];
      s0[qb] = a0 * wz;
      s1[qb] = a1 * wz;
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      double* yr = Yr + ((e2 + j) % P) * LXR + o;
      double v = *yr;
#pragma unroll
      for (int qb = 0; qb < Q2B; ++qb) {
        const int q2 = b * Q2B + qb;
        v = fma(Tz[(0 * 8 + q2) * 8 + j], s0[qb], v);
        if (STIFF) v = fma(Tz[(1 * 8 + q2) * 8 + j], s1[qb], v);
      }
      *yr = v;
    }
  };

  int widx = 0;  // this warp's running TMA task index
  for (int e2 = z0; e2 < z1; ++e2) {
    const int zb = (e2 - z0) & 1;
    const double* Tz = Tzb + zb * 128;
    const double* Wz = Wzb + zb * 8;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    for (int b = 0; b < NB; ++b) {
      PHASE_MARK(0);  // element setup / previous batch tail
      // ---- Z^T(previous batch) + Z(this batch) + clear S ---------------------
      if (b > 0)
        for (int i = tid; i < FY * FX; i += NT) zt_item(Tz, Wz, e2, b - 1, i);
      for (int i = tid; i < Q2B * FY * FX; i += NT) {
        const int qb = i / (FY * FX), r = i % (FY * FX);
        const int n0 = r % FX, n1 = r / FX, o = n1 * RP + n0;
        const int q2 = b * Q2B + qb;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          const double xv = Xr[((e2 + j) % P) * LXR + o];
          a0 = fma(Tz[(0 * 8 + q2) * 8 + j], xv, a0);
          if (STIFF) a1 = fma(Tz[(1 * 8 + q2) * 8 + j], xv, a1);
        }
        Aq[(qb * NA + 0) * LXR + o] = a0;
        if (STIFF) Aq[(qb * NA + 1) * LXR + o] = a1;
      }
      __syncthreads();
      if (b == NB - 1) {  // x slot e2 % P and the other z-table buffer are free now
        load_layer(e2 + P);
        if (e2 + 1 < z1) load_ztab(e2 + 1, zb ^ 1);
      }

      PHASE_MARK(1);  // Z (+ Z^T of the previous batch)
      // ---- Y (DMMA), X (DMMA) + pointwise + X^T (DMMA): warp-private rows -----
      {
        const int line = wlg * 8 + g;   // A-fragment / D row
        double* Cb = Cq + wq * NV * CQL;
        double* Crow = Cb + line * RP;  // C (then R) row of this lane's line
        // Y for this warp's 8 lines: C_vw[line][n0] = Σ_k By_w[line][k] ·
        // A_v[nb + k][n0] with the banded per-warp fragments byA (k = m + 4s)
        {
          double byA[2][2];
#pragma unroll
          for (int v = 0; v < 2; ++v)
#pragma unroll
            for (int s = 0; s < 2; ++s) byA[v][s] = y_frag(v, s);
          const double* A0 = Aq + (wq * NA) * LXR + ynb * RP;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            double c00[2] = {0.0, 0.0}, c10[2] = {0.0, 0.0}, c01[2] = {0.0, 0.0};
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int o = (m + 4 * s) * RP + nt * 8 + g;
              const double b0 = A0[o];
              dmma(c00[0], c00[1], byA[0][s], b0);
              if (STIFF) {
                const double b1 = A0[LXR + o];
                dmma(c10[0], c10[1], byA[1][s], b0);
                dmma(c01[0], c01[1], byA[0][s], b1);
              }
            }
            double* co = Crow + nt * 8 + 2 * m;
            co[0] = c00[0];
            co[1] = c00[1];
            if (STIFF) {
              co[CQL] = c10[0];
              co[CQL + 1] = c10[1];
              co[2 * CQL] = c01[0];
              co[2 * CQL + 1] = c01[1];
            }
          }
          __syncwarp();
        }
        PHASE_MARK(2);  // Y
        const int widx0 = widx;         // = batch·NBX
        // point layers (slab-local) of this batch's and the next batch's boxes
        const int zq_cur = e2 * Q + b * Q2B + wq;
        const int zq_next = b + 1 < NB ? zq_cur + Q2B : (e2 + 1) * Q + wq;
        int stage = 0;                  // ring stage of the current box
        // running X^T window over DoF columns [c0(w), c0(w) + 8): lane m holds
        // c0 + 2m, c0 + 2m + 1
        double w00[2] = {0.0, 0.0}, w10[2] = {0.0, 0.0}, w01[2] = {0.0, 0.0};
        // window table fragments: forward B^T[c][pt = n] (D column n is window
        // point n, so a lane's two D values are the adjacent points 2m, 2m+1)
        // and the transpose B[pt][c] with k-chunk s covering points 2m + s;
        // hoisted when the tile is interior and every window has one pattern
        double fb0[2], fb1[2], tb0[2], tb1[2];
        auto load_tab = [&](int w) {
          const double2* T = reinterpret_cast<const double2*>(Tw + w * 256) + lane;
          const double2 f0 = T[0], t0 = T[64];
          fb0[0] = f0.x;
          fb0[1] = f0.y;
          tb0[0] = t0.x;
          tb0[1] = t0.y;
          if (STIFF) {
            const double2 f1 = T[32], t1 = T[96];
            fb1[0] = f1.x;
            fb1[1] = f1.y;
            tb1[0] = t1.x;
            tb1[1] = t1.y;
          } else {
            fb1[0] = fb1[1] = tb1[0] = tb1[1] = 0.0;
          }
        };
        const bool hoist = tile_uniform && C::PER == 1 && !C::ROT;
        if (hoist) load_tab(0);
        // software pipeline: C fragments of window w+1 are loaded while w
        // computes (window w only ever writes columns below c0(w+1))
        double cf[3][2], cn[3][2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          cf[0][s] = Crow[m + 4 * s];
          cf[1][s] = STIFF ? Crow[CQL + m + 4 * s] : 0.0;
          cf[2][s] = STIFF ? Crow[2 * CQL + m + 4 * s] : 0.0;
        }
#pragma unroll
        for (int w = 0; w < NWIN; ++w) {
          const int c0 = C::c0w(w);
          if (!hoist) load_tab(w);
          if (w + 1 < NWIN) {
            const int c1 = C::c0w(w + 1);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              cn[0][s] = Crow[c1 + m + 4 * s];
              cn[1][s] = STIFF ? Crow[CQL + c1 + m + 4 * s] : 0.0;
              cn[2][s] = STIFF ? Crow[2 * CQL + c1 + m + 4 * s] : 0.0;
            }
          }
          // forward: U^T[line][pt] = Σ_c C^T[line][c0 + c] · B^T[c][pt].  A
          // lane's two D values (points 2m, 2m+1) are its A-fragment columns
          // of the two k-chunks of the transposed product below (no shuffles).
          double u[2] = {0.0, 0.0}, ux[2] = {0.0, 0.0}, uy[2] = {0.0, 0.0}, uz[2] = {0.0, 0.0};
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (MASS) dmma(u[0], u[1], cf[0][s], fb0[s]);
            if (STIFF) {
              dmma(ux[0], ux[1], cf[0][s], fb1[s]);
              dmma(uy[0], uy[1], cf[1][s], fb0[s]);
              dmma(uz[0], uz[1], cf[2][s], fb0[s]);
            }
          }
          // coefficients of (window w, these 8 lines, point layer q2): wait
          // for the TMA box after issuing the forward MMAs (they do not need it)
#ifdef IGS_PHASE_TIMING
          long long tw0_ = clock64();
#endif
          {
            const int gi = kStaticRing ? w : widx0 + w;
            stage = gi % STG;
            mbar_wait(mybar + stage, (unsigned)((gi / STG) & 1));
          }
#ifdef IGS_PHASE_TIMING
          if (tid == 0) atomicAdd(&g_phase_cycles[5], (unsigned long long)(clock64() - tw0_));
#endif
          // [plane][line][pt]: the lane's points 2m, 2m+1 as one 16-byte load
          const double* F = mystage + stage * FST + g * QE + 2 * m;
          double fv[7][2];
          auto ld2 = [&](int pl, double* o) {
            const double2 v = *reinterpret_cast<const double2*>(F + pl * 8 * QE);
            o[0] = v.x;
            o[1] = v.y;
          };
          if (MASS) ld2(pc, fv[0]);
          if (STIFF) {
            ld2(p00, fv[1]);
            ld2(p11, fv[2]);
            ld2(p22, fv[3]);
            ld2(p01, fv[4]);
            ld2(p02, fv[5]);
            ld2(p12, fv[6]);
          }
          // pointwise g = F·∇u (the quadrature weights w_x, w_y, w_z are
          // folded into the test-side tables of X^T, Y^T and Z^T; they are
          // zero past the mesh, which masks the finite values read there)
          double g0[2], gx[2], gy[2], gz[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (MASS) g0[c] = fv[0][c] * u[c];
            if (STIFF) {
              const double f00 = fv[1][c], f11 = fv[2][c], f22 = fv[3][c];
              const double f01 = fv[4][c], f02 = fv[5][c], f12 = fv[6][c];
              gx[c] = fma(f00, ux[c], fma(f01, uy[c], f02 * uz[c]));
              gy[c] = fma(f01, ux[c], fma(f11, uy[c], f12 * uz[c]));
              gz[c] = fma(f02, ux[c], fma(f12, uy[c], f22 * uz[c]));
            }
          }
          // transpose into the window: W^T[line][c] += Σ_pt g^T[line][pt] · B[pt][c]
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (MASS) dmma(w00[0], w00[1], g0[s], tb0[s]);
            if (STIFF) {
              dmma(w00[0], w00[1], gx[s], tb1[s]);
              dmma(w10[0], w10[1], gy[s], tb0[s]);
              dmma(w01[0], w01[1], gz[s], tb0[s]);
            }
          }
          // every lane's reads of this stage have been consumed: the
          // transposed MMAs above (warp-synchronous mma.sync) consumed every
          // lane's g, which needed its coefficient loads; hand the stage to
          // the next box of this warp
#if IGS_APPLY_SYNCWARP
          __syncwarp();
#endif
          if (lane == 0 && widx0 + w + STG < ntask) {
            // box w + STG of this row: window (w + STG) % NBX of this or the next batch
            const int nxt = w + STG;
            const int stg = kStaticRing ? nxt % STG : (widx0 + nxt) % STG;
            issue_box(stg, nxt % NBX, nxt < NBX ? zq_cur : zq_next);
          }
          // columns [c0, c0 + d) are complete (no later window touches them):
          // store them over C's columns, which no later window reads; then
          // clear their accumulator slots (ROT: column c lives in slot c mod 8)
          // or slide the accumulator window by d columns
          const int d = (w + 1 < NWIN ? C::c0w(w + 1) : c0 + 8) - c0;
          if (w + 1 < NWIN) {
            // (ROT: every lane's reads of these C columns fed the forward
            // MMAs, which every lane passed before the transposed MMAs)
            if constexpr (!C::ROT) __syncwarp();
            if constexpr (C::ROT) {
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const int off = (2 * m + c - c0) & 7;
                if (off < d) {
                  Crow[c0 + off] = w00[c];
                  w00[c] = 0.0;
                  if (STIFF) {
                    Crow[CQL + c0 + off] = w10[c];
                    Crow[2 * CQL + c0 + off] = w01[c];
                    w10[c] = 0.0;
                    w01[c] = 0.0;
                  }
                }
              }
            } else {
#pragma unroll
              for (int c = 0; c < 2; ++c)
                if (2 * m + c < d) {
                  Crow[c0 + 2 * m + c] = w00[c];
                  if (STIFF) {
                    Crow[CQL + c0 + 2 * m + c] = w10[c];
                    Crow[2 * CQL + c0 + 2 * m + c] = w01[c];
                  }
                }
              // new column 2m + c = old column 2m + c + d: lane m + (c + d) / 2,
              // element (c + d) % 2 (zero past the window)
              auto slide = [&](double (&acc)[2]) {
                double nv[2];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                  const int ls = (c + d) / 2, el = (c + d) % 2;
                  const double src = el ? acc[1] : acc[0];
                  const double got = __shfl_down_sync(0xffffffffu, src, ls, 4);
                  nv[c] = (m + ls < 4) ? got : 0.0;
                }
                acc[0] = nv[0];
                acc[1] = nv[1];
              };
              slide(w00);
              if (STIFF) {
                slide(w10);
                slide(w01);
              }
            }
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
              for (int s2 = 0; s2 < 2; ++s2) cf[v][s2] = cn[v][s2];
          }
        }
        widx = widx0 + NBX;
        // remaining columns [c0(last), c0(last) + 8): slot 2m + c holds the
        // one congruent to it mod 8 (ROT), else column c0(last) + 2m + c
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int col = C::c0w(NWIN - 1) + (C::ROT ? ((2 * m + c - C::c0w(NWIN - 1)) & 7) : 2 * m + c);
          if (col < FX) {
            Crow[col] = w00[c];
            if (STIFF) {
              Crow[CQL + col] = w10[c];
              Crow[2 * CQL + col] = w01[c];
            }
          }
        }
        __syncwarp();
        // Y^T partials of this warp's 8 lines: S_0 = By0·R00 + By1·R10 and
        // S_1 = By0·R01 over DoF rows ynb + k (fragments byT, k = g), stored
        // over the warp's own R rows (planes 0 and 1) once all are consumed
        {
          double byT[2][2];
#pragma unroll
          for (int v = 0; v < 2; ++v)
#pragma unroll
            for (int s = 0; s < 2; ++s) byT[v][s] = yt_frag(v, s);
          const double* R0 = Cb + (wlg * 8) * RP;
          double d0[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, d1[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int o = (m + 4 * s) * RP + nt * 8 + g;
              dmma(d0[nt][0], d0[nt][1], byT[0][s], R0[o]);
              if (STIFF) {
                dmma(d0[nt][0], d0[nt][1], byT[1][s], R0[CQL + o]);
                dmma(d1[nt][0], d1[nt][1], byT[0][s], R0[2 * CQL + o]);
              }
            }
          __syncwarp();
          double* so = Cb + (wlg * 8 + g) * RP + 2 * m;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            so[nt * 8] = d0[nt][0];
            so[nt * 8 + 1] = d0[nt][1];
            if (STIFF) {
              so[CQL + nt * 8] = d1[nt][0];
              so[CQL + nt * 8 + 1] = d1[nt][1];
            }
          }
        }
      }
      __syncthreads();

      PHASE_MARK(3);  // X (+ Y^T partials)
    }
    PHASE_MARK(4);  // Y^T of the last batch
    // last Z^T of the element, flush DoF layer e2 (complete for this chunk)
    for (int i = tid; i < FY * FX; i += NT) {
      zt_item(Tz, Wz, e2, NB - 1, i);
      const int n0 = i % FX, n1 = i / FX, o = n1 * RP + n0;
      double* yr = Yr + (e2 % P) * LXR + o;
      box[(int64_t)(e2 - z0) * FY * FX + i] = *yr;
      *yr = 0.0;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  // trailing P-1 DoF layers [z1, z1 + P - 1)
  for (int l = z1; l < z1 + P - 1; ++l) {
    const double* yr = Yr + (l % P) * LXR;
    double* dst = box + (int64_t)(l - z0) * FY * FX;
    for (int i = tid; i < FY * FX; i += NT) {
      const int n0 = i % FX, n1 = i / FX;
      dst[i] = yr[n1 * RP + n0];
    }
  }
}

struct ReduceArgs {
  const double* scratch;
  double* y;
  int64_t N0, N1, N2;
  int EX, EY, FX, FY, P;
  int ntx, nty, nch, ez, K2;
  int64_t box;
  int accumulate;
};

// y[n] = Σ over the work-item boxes covering n, in (tz, ty, tx) order.
// Grid (x: blocks over the flattened (n0, n1) layer — every lane busy even
// when N0 is just past a multiple of 128 — y: n2 stride); 32-bit
// coordinates, no 64-bit divisions on the per-DoF path.
__global__ void __launch_bounds__(128) apply_reduce_kernel(const ReduceArgs r) {
  const int n01 = blockIdx.x * blockDim.x + threadIdx.x;
  const int N0 = (int)r.N0;
  if (n01 >= N0 * (int)r.N1) return;
  const int n0 = n01 % N0, n1 = n01 / N0;
  const int EX = r.EX, EY = r.EY, FX = r.FX, FY = r.FY, ez = r.ez;
  const int tx_hi = min(r.ntx - 1, n0 / EX), tx_lo = n0 >= FX ? (n0 - FX) / EX + 1 : 0;
  const int ty_hi = min(r.nty - 1, n1 / EY), ty_lo = n1 >= FY ? (n1 - FY) / EY + 1 : 0;
  const int zspan = ez + r.P - 1;
  for (int n2 = blockIdx.y; n2 < r.N2; n2 += gridDim.y) {
    const int tz_hi = min(r.nch - 1, n2 / ez), tz_lo = n2 >= zspan ? (n2 - zspan) / ez + 1 : 0;
    double s = 0.0;
    for (int tz = tz_lo; tz <= tz_hi; ++tz) {
      const int z0 = tz * ez, z1 = min(r.K2, z0 + ez);
      if (n2 >= z1 + r.P - 1 || n2 < z0) continue;
      for (int ty = ty_lo; ty <= ty_hi; ++ty) {
        const int l1 = n1 - ty * EY;
        if (l1 >= FY) continue;
        for (int tx = tx_lo; tx <= tx_hi; ++tx) {
          const int l0 = n0 - tx * EX;
          if (l0 >= FX) continue;
          const int64_t item = ((int64_t)tz * r.nty + ty) * r.ntx + tx;
          s += r.scratch[item * r.box + ((n2 - z0) * FY + l1) * FX + l0];
        }
      }
    }
    const int64_t gi = ((int64_t)n2 * r.N1 + n1) * r.N0 + n0;
    r.y[gi] = r.accumulate ? r.y[gi] + s : s;
  }
}

// ---- instantiation table ----------------------------------------------------

struct Launch {
  int EX, EY, NT, NPL, QE;
  size_t smem;
  void (*kernel)(ApplyArgs, CUtensorMap);
  int promo = 256;  // L2 promotion of the coefficient boxes (bytes)
};

template <int P, int Q, int EX, int EY, int Q2B, bool MASS, bool STIFF, int STG = 2>
Launch make_launch() {
  using C = Cfg<P, Q, EX, EY, Q2B, MASS, STIFF, STG>;
  return Launch{EX, EY, C::NT, C::NPL, C::QE, C::SMEM, &apply3d_kernel<P, Q, EX, EY, Q2B, MASS, STIFF, STG>, 256};
}

// Development switches, compiled only into the measurement build
// (-DIGS_DEV_SWITCHES, tools/): IGS_APPLY_L2PF=-1 makes every TMA box re-read
// the tile's first box (L2-resident) so the kernel runs without its HBM
// stream (the compute-only time in DESIGN.md §K4; results are wrong in that
// mode), IGS_APPLY_VARIANT picks alternative tile shapes and
// IGS_APPLY_ZCHUNKS forces a z-chunk count.  The production library never
// reads the environment.
#ifdef IGS_DEV_SWITCHES
int compute_only_mode() {
  static int v = 2;
  if (v == 2) {
    const char* e = getenv("IGS_APPLY_L2PF");
    v = (e && atoi(e) < 0) ? -1 : 0;
  }
  return v;
}
int apply_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGS_APPLY_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}
int forced_zchunks() {
  static const int forced = [] {
    const char* e = getenv("IGS_APPLY_ZCHUNKS");
    return e ? atoi(e) : 0;
  }();
  return forced;
}
#else
constexpr int compute_only_mode() { return 0; }
constexpr int apply_variant() { return 0; }
constexpr int forced_zchunks() { return 0; }
#endif

// Tile shapes per order: EY·Q lines in groups of 8, Q2B point layers per
// batch, one warp per (point layer, line group) of a batch.
template <bool MASS, bool STIFF>
bool pick(int P, int Q, Launch* L) {
  if (P != Q) return false;
#ifdef IGS_DEV_SWITCHES
  // tile-shape experiments at low orders (measurement builds only)
  if (apply_variant() >= 10) {
    switch (apply_variant() * 10 + P) {
      case 102: *L = make_launch<2, 2, 8, 12, 2, MASS, STIFF, 1>(); return true;
      case 112: *L = make_launch<2, 2, 8, 12, 1, MASS, STIFF, 2>(); return true;
      case 122: *L = make_launch<2, 2, 8, 8, 2, MASS, STIFF, 1>(); return true;
      case 132: *L = make_launch<2, 2, 8, 12, 2, MASS, STIFF, 3>(); return true;
      case 103: *L = make_launch<3, 3, 8, 8, 1, MASS, STIFF, 1>(); return true;
      case 113: *L = make_launch<3, 3, 8, 8, 1, MASS, STIFF, 2>(); return true;
      case 123: *L = make_launch<3, 3, 8, 8, 3, MASS, STIFF, 2>(); return true;
      case 104: *L = make_launch<4, 4, 8, 8, 2, MASS, STIFF, 2>(); return true;
      case 114: *L = make_launch<4, 4, 8, 8, 2, MASS, STIFF, 1>(); return true;
      case 124: *L = make_launch<4, 4, 8, 8, 4, MASS, STIFF, 1>(); return true;
      case 105: *L = make_launch<5, 5, 8, 8, 1, MASS, STIFF, 1>(); return true;
      case 115: *L = make_launch<5, 5, 8, 8, 1, MASS, STIFF, 3>(); return true;
      default: break;
    }
    // the headline configurations: C4 (p = 6 stiffness), C5 (p = 8 mass+stiffness)
    if constexpr (!MASS && STIFF) {
      switch (apply_variant() * 10 + P) {
        case 206: *L = make_launch<6, 6, 8, 8, 1, MASS, STIFF, 3>(); return true;
        case 216: *L = make_launch<6, 6, 8, 8, 1, MASS, STIFF, 4>(); return true;
        case 226: *L = make_launch<6, 6, 8, 8, 3, MASS, STIFF, 2>(); return true;
        case 236: *L = make_launch<6, 6, 8, 8, 2, MASS, STIFF, 4>(); return true;
        case 246: *L = make_launch<6, 6, 8, 8, 3, MASS, STIFF, 3>(); return true;
        case 256: *L = make_launch<6, 6, 8, 8, 2, MASS, STIFF, 2>(); return true;
        case 306: *L = make_launch<6, 6, 8, 4, 2, MASS, STIFF, 4>(); return true;
        case 316: *L = make_launch<6, 6, 8, 4, 3, MASS, STIFF, 3>(); return true;
        case 326: *L = make_launch<6, 6, 8, 4, 6, MASS, STIFF, 2>(); return true;
        case 336: *L = make_launch<6, 6, 8, 8, 2, MASS, STIFF, 1>(); return true;
        case 346: *L = make_launch<6, 6, 8, 4, 6, MASS, STIFF, 1>(); return true;
        case 356: *L = make_launch<6, 6, 8, 4, 3, MASS, STIFF, 2>(); return true;
        case 218: *L = make_launch<8, 8, 8, 8, 2, MASS, STIFF, 1>(); return true;
        case 228: *L = make_launch<8, 8, 8, 8, 1, MASS, STIFF, 1>(); return true;
        default: break;
      }
    }
    if constexpr (MASS && STIFF) {
      switch (apply_variant() * 10 + P) {
        case 208: *L = make_launch<8, 8, 8, 8, 1, MASS, STIFF, 2>(); return true;
        case 218: *L = make_launch<8, 8, 8, 8, 2, MASS, STIFF, 1>(); return true;
        case 228: *L = make_launch<8, 8, 8, 6, 1, MASS, STIFF, 3>(); return true;
        case 238: *L = make_launch<8, 8, 8, 6, 2, MASS, STIFF, 3>(); return true;
        case 248: *L = make_launch<8, 8, 8, 6, 4, MASS, STIFF, 1>(); return true;
        case 258: *L = make_launch<8, 8, 8, 6, 2, MASS, STIFF, 1>(); return true;
        default: break;
      }
    }
  }
#endif
  switch (P) {
    // p = 4: 8-row y tiles (16 warps) where they fit shared memory (measured
    // 1.51 -> 1.21 ms at 128^3, stiffness), else 4-row tiles (mass+stiffness)
    case 2: *L = make_launch<2, 2, 8, 12, 2, MASS, STIFF>(); return true;
    // p = 3: a single TMA stage lets two CTAs share an SM (18 warps):
    // 0.73 -> 0.66 ms at 128^3 (stiffness)
    case 3:  // (mass+stiffness: one point layer per batch on two stages, 0.780 -> 0.764 ms)
      if (MASS && STIFF) *L = make_launch<3, 3, 8, 8, 1, MASS, STIFF, 2>();
      else *L = make_launch<3, 3, 8, 8, 3, MASS, STIFF, 1>();
      return true;
    // mass+stiffness (7 planes): 8-row tiles fit with two point layers per
    // batch and a single TMA stage (1.61 -> 1.26 ms at 128^3, 0.72 -> 0.92 of
    // the copy roofline; the 4-row-tile fallback stays for larger plane sets)
    case 4:
      if (MASS && STIFF) *L = make_launch<4, 4, 8, 8, 2, MASS, STIFF, 1>();
      else *L = make_launch<4, 4, 8, 8, 4, MASS, STIFF>();
      if (L->smem > 232448) *L = make_launch<4, 4, 8, 4, 4, MASS, STIFF>();
      return true;
    case 5: *L = make_launch<5, 5, 8, 8, 1, MASS, STIFF>(); return true;
    case 6:  // 7 planes (M+K) fit a 2-stage ring, 6 a 3-stage one
      if (apply_variant() == 1 || (MASS && STIFF)) *L = make_launch<6, 6, 8, 8, 2, MASS, STIFF, 2>();
      else {
        // the 3-stage ring hides the box latency itself: 256-byte promotion
        // only over-fetches there (ncu: 24.7 GB read for 21.8 GB of planes);
        // 128 bytes: 3.70 -> 3.47 ms at C4, DRAM back to B_alg
        *L = make_launch<6, 6, 8, 8, 2, MASS, STIFF, 3>();
        L->promo = 128;
      }
      return true;
    // p = 7: stiffness on a single TMA stage (two CTAs per SM: 7.35 ->
    // 6.45 ms at 128^3), mass+stiffness on three (8.0 -> 7.7 ms)
    case 7:
      if (MASS && STIFF) *L = make_launch<7, 7, 8, 8, 1, MASS, STIFF, 3>();
      else if (STIFF) *L = make_launch<7, 7, 8, 8, 1, MASS, STIFF, 1>();
      else *L = make_launch<7, 7, 8, 8, 1, MASS, STIFF>();
      return true;
    case 8:
      if (apply_variant() == 1) *L = make_launch<8, 8, 8, 4, 2, MASS, STIFF, 4>();
      else if (apply_variant() == 2) *L = make_launch<8, 8, 8, 2, 2, MASS, STIFF, 2>();
      // stiffness and mass+stiffness (C5): 8-row tiles on a single TMA stage
      // (C5 sustained 50 applies 10.41 -> 10.13 ms/step, 0.92 -> 0.94 of the
      // copy roofline; stiffness 9.03 -> 8.66 ms)
      else if (STIFF) *L = make_launch<8, 8, 8, 8, 2, MASS, STIFF, 1>();
      else *L = make_launch<8, 8, 8, 6, 2, MASS, STIFF, 2>();
      return true;
    default: return false;
  }
}

bool pick_launch(const FusedShape& s, Launch* L) {
  if (s.d != 3) return false;
  bool ok = false;
  if (s.mass && s.stiff) ok = pick<true, true>(s.p, s.k, L);
  else if (s.stiff) ok = pick<false, true>(s.p, s.k, L);
  else if (s.mass) ok = pick<true, false>(s.p, s.k, L);
  // 227 KB of dynamic shared memory per CTA on sm_100a
  return ok && L->smem <= 232448;
}

struct Tiling {
  int ntx, nty, nch, ez;
  int64_t box;
};

// Resident CTAs per SM of a fused apply configuration (occupancy query,
// cached per kernel).
int ctas_per_sm(const Launch& L) {
  static std::mutex mu;
  static std::map<void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find((void*)L.kernel);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaFuncSetAttribute(L.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, L.kernel, L.NT, L.smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  cache[(void*)L.kernel] = n;
  return n;
}

Tiling tiling(const FusedShape& s, const Launch& L) {
  Tiling t;
  t.ntx = (int)ceil_div(s.nel[0], L.EX);
  t.nty = (int)ceil_div(s.nel[1], L.EY);
  // z chunks: as few as possible (each chunk costs a prologue and P-1 layers
  // of overlapping partial sums) while the work items fill whole waves of
  // resident CTAs (>= 97 % of the last wave); chunks of at least P-1 layers
  // so each DoF sees at most two chunks.
  const int K2 = (int)s.nel[2];
  const int64_t tiles = (int64_t)t.ntx * t.nty;
  const double slots = 148.0 * ctas_per_sm(L);
  const int ez_min = s.p - 1 > 1 ? s.p - 1 : 1;
  int best_ez = K2, pick_ez = 0;
  double best_eff = -1.0;
  for (int n = 1; n <= 16; ++n) {
    int ez = (int)ceil_div(K2, n);
    if (ez < ez_min) ez = ez_min;
    if (ez > K2) ez = K2;
    const int nch = (int)ceil_div(K2, ez);
    const double w = nch * (double)tiles / slots;
    const double eff = w / std::ceil(w);
    if (eff >= 0.97) {
      pick_ez = ez;
      break;
    }
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best_ez = ez;
    }
  }
  int ez = pick_ez ? pick_ez : best_ez;
  {  // development switch for chunking experiments (measurement build only)
    const int forced = forced_zchunks();
    if (forced > 0) {
      ez = (int)ceil_div(K2, forced);
      if (ez < ez_min) ez = ez_min;
      if (ez > K2) ez = K2;
    }
  }
  t.ez = ez;
  t.nch = (int)ceil_div(K2, ez);
  int FX = L.EX + s.p - 1, FY = L.EY + s.p - 1;
  t.box = (int64_t)(ez + s.p - 1) * FY * FX;
  return t;
}

// L2 promotion of the coefficient boxes: 64-byte box rows (one 8-point
// window) gain from 256-byte promotion (the warp's next windows arrive with
// them: C5 -3 %).
#ifdef IGS_L2_PROMO  // measurement builds: one promotion for every configuration
CUtensorMapL2promotion l2_promotion(const Launch&) { return IGS_L2_PROMO; }
#else
CUtensorMapL2promotion l2_promotion(const Launch& L) {
  return L.promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}
#endif

// The coefficient planes as one 4D tensor (x, y, z points, plane) for TMA.
// cuTensorMapEncodeTiled comes from the driver through the runtime's entry
// point query, so the library does not link libcuda directly.
igs_status coeff_tensor_map(CUtensorMap* map, const double* planes, int64_t pstride, const Dims& D,
                            const Launch& L, unsigned box0) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(IGS_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[4] = {(cuuint64_t)D.x[0], (cuuint64_t)D.x[1], (cuuint64_t)D.x[2], (cuuint64_t)L.NPL};
  cuuint64_t strides[3] = {(cuuint64_t)D.x[0] * 8, (cuuint64_t)(D.x[0] * D.x[1]) * 8, (cuuint64_t)pstride * 8};
  cuuint32_t boxd[4] = {(cuuint32_t)box0, 8u, 1u, (cuuint32_t)L.NPL};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(planes), dims, strides,
                      boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      l2_promotion(L), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(IGS_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return IGS_OK;
}

// TMA needs 16-byte aligned rows/planes and exactly the kernel's plane set.
bool tma_ok(const igs_problem* p, const Dims& D, const Launch& L) {
  if ((D.x[0] * 8) % 16 != 0 || (p->plane_stride * 8) % 16 != 0) return false;
  if (p->n_planes != L.NPL) return false;
  return true;
}

}  // namespace

bool fused_apply_supported(const igs_problem* p, const Dims& D) {
  FusedShape s;
  if (!fused_shape(p, D, &s)) return false;
  Launch L;
  return pick_launch(s, &L) && tma_ok(p, D, L);
}

size_t fused_apply_workspace(const igs_problem* p, const Dims& D) {
  FusedShape s;
  Launch L;
  if (!fused_shape(p, D, &s) || !pick_launch(s, &L)) return 0;
  Tiling t = tiling(s, L);
  return (size_t)t.ntx * t.nty * t.nch * t.box * sizeof(double) + 256;
}

igs_status fused_apply(const igs_problem* p, const Dims& D, const double* planes, const double* x,
                       double* y, void* ws, size_t ws_bytes, int flags, cudaStream_t st) {
  FusedShape s;
  Launch L;
  if (!fused_shape(p, D, &s) || !pick_launch(s, &L) || !tma_ok(p, D, L))
    return fail(IGS_ECAPACITY, "no fused apply");
  if (((uintptr_t)planes & 15) != 0) return fail(IGS_EARG, "coefficient planes must be 16-byte aligned");
  Tiling t = tiling(s, L);
  size_t need = (size_t)t.ntx * t.nty * t.nch * t.box * sizeof(double);
  if (ws_bytes < need || !ws) return fail(IGS_EWORKSPACE, "workspace too small for the fused apply");
  ApplyArgs a{};
  a.x = x;
  a.planes = planes;
  a.pstride = p->plane_stride;
  a.pl_c = p->plane_of[0][0];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a.pl_a[i][j] = p->plane_of[1 + i][1 + j];
  for (int k = 0; k < 3; ++k) {
    a.vals[k] = p->trial[k].values;
    a.wts[k] = p->trial[k].weights;
    a.xtab[k] = p->trial[k].num_points;
  }
  a.N0 = D.nt[0]; a.N1 = D.nt[1]; a.N2 = D.nt[2];
  a.X0 = D.x[0]; a.X1 = D.x[1];
  a.K0 = (int)s.nel[0]; a.K1 = (int)s.nel[1]; a.K2 = (int)s.nel[2];
  a.z_el_off = (p->slab_lo || p->slab_hi) ? p->slab_lo : 0;
  a.l2pf = compute_only_mode();
  a.uni_x = p->trial[0].uniform;
  a.ntx = t.ntx; a.nty = t.nty; a.nch = t.nch; a.ez = t.ez;
  a.scratch = reinterpret_cast<double*>(ws);
  a.box = t.box;
  CUtensorMap fmap;
  IGS_TRY(coeff_tensor_map(&fmap, planes, p->plane_stride, D, L, (unsigned)L.QE));
  IGS_TRY(cuda_check(cudaFuncSetAttribute(L.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)L.smem), "smem attribute"));
  unsigned grid = (unsigned)(t.ntx * t.nty * t.nch);
  L.kernel<<<grid, L.NT, L.smem, st>>>(a, fmap);
  IGS_LAUNCH_CHECK("apply3d_kernel");
  if (flags & IGS_FLAG_KERNEL_ONLY) return IGS_OK;
  ReduceArgs r{};
  r.scratch = a.scratch;
  r.y = y;
  r.N0 = D.ns[0]; r.N1 = D.ns[1]; r.N2 = D.ns[2];
  r.EX = L.EX; r.EY = L.EY; r.FX = L.EX + s.p - 1; r.FY = L.EY + s.p - 1; r.P = s.p;
  r.ntx = t.ntx; r.nty = t.nty; r.nch = t.nch; r.ez = t.ez; r.K2 = (int)s.nel[2];
  r.box = t.box;
  r.accumulate = (flags & IGS_FLAG_ACCUMULATE) ? 1 : 0;
  if (r.N0 * r.N1 >= ((int64_t)1 << 31)) return fail(IGS_ECAPACITY, "DoF layer too large for the reduce");
  const dim3 rgrid((unsigned)ceil_div(r.N0 * r.N1, 128), (unsigned)min64(r.N2, 64));
  apply_reduce_kernel<<<rgrid, 128, 0, st>>>(r);
  IGS_LAUNCH_CHECK("apply_reduce_kernel");
  return IGS_OK;
}

}  // namespace igs

#ifdef IGS_PHASE_TIMING
// Debug-only (built by tools/phase_timing.py): read and reset the per-phase
// cycle counters of thread 0 of every CTA.
extern "C" void igs_debug_phase_cycles(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles));
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
}
#endif
