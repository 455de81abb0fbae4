// K3 — fused global sum-factorized assembly (Alg. 1) for uniform-structure
// problems in 2D and 3D, written straight into CSR order.
//
// Same recursion as the reference (_Core.block_values, sumfac.py:200-213,
// with W_δ = w·B^θ_n·B^η_m as in _Core.w_matrix, sumfac.py:163-198), reorganised
// for the GPU:
//   * derivative blocks that share the per-direction variants of the later
//     directions are summed right after the earlier contraction (3D M+K:
//     10 blocks -> 9 stage-1 groups -> 4 stage-2 groups), so the work drops
//     from 32 to 21 GFLOP at C3 without changing what is summed;
//   * 1D pairs are addressed by slots s = m·(2p-1) + (n - m + p - 1) (the
//     band of row m), so every stage is a dense loop;
//   * the last direction is swept per (pair0[, pair1]) thread with a ring of
//     p rows x (2p-1) columns in registers: row m is final once the sweep has
//     passed its last element, and is written straight to its CSR slots
//     (closed-form offsets, no lexsort / value permutation).
//
//   3D: asm3_stage12 (per point layer z, tile of 4x4 rows in (x, y)):
//         G_g[pair0][y] = Σ_{blocks b in g} Σ_x W_x^{v0(b)} F_b      (smem)
//         H_h[pair1][pair0] = Σ_{g in h} Σ_y W_y^{v1(g)} G_g       -> HBM
//       asm3_stage3 (one thread per (pair0, pair1)):
//         ring[m2][n2] += Σ_h W_z^{v2(h)} H_h  ->  CSR
//   2D: asm2_stage1 (x) -> HBM, asm2_stage2 (y ring, chunked) -> CSR.
#include "fused.cuh"

namespace igs {
namespace {

constexpr int kMaxBlocks = 16;

// Block / group plan derived from (theta, eta, plane_of) on the host.
struct AsmPlan {
  int nb;                       // non-zero blocks
  int b_plane[kMaxBlocks];
  int b_v0[kMaxBlocks];         // variant code θ + 2η in direction 0
  int b_g[kMaxBlocks];          // stage-1 group of the block
  int ng;                       // stage-1 groups (keyed by the later directions' variants)
  int g_v1[kMaxBlocks];         // variant of direction 1 (3D) / last direction (2D)
  int g_h[kMaxBlocks];          // stage-2 group (3D)
  int nh;                       // stage-2 groups (3D: keyed by v2)
  int h_v2[kMaxBlocks];
};

bool build_plan(const igs_problem* p, AsmPlan* plan) {
  AsmPlan P{};
  const int d = p->d;
  int gkey[kMaxBlocks], hkey[kMaxBlocks];
  for (int j = 0; j < p->n_theta; ++j)
    for (int i = 0; i < p->n_eta; ++i) {
      int pl = p->plane_of[i][j];
      if (pl < 0) continue;
      if (P.nb >= kMaxBlocks) return false;
      int v[3] = {0, 0, 0};
      for (int k = 0; k < d; ++k) {
        int th = p->theta[j][k], et = p->eta[i][k];
        if (th > 1 || et > 1) return false;
        v[k] = th + 2 * et;
      }
      int key = d == 3 ? v[1] * 4 + v[2] : v[1];
      int g = -1;
      for (int q = 0; q < P.ng; ++q)
        if (gkey[q] == key) g = q;
      if (g < 0) {
        g = P.ng++;
        gkey[g] = key;
        P.g_v1[g] = v[1];
        if (d == 3) {
          int h = -1;
          for (int q = 0; q < P.nh; ++q)
            if (hkey[q] == v[2]) h = q;
          if (h < 0) {
            h = P.nh++;
            hkey[h] = v[2];
            P.h_v2[h] = v[2];
          }
          P.g_h[g] = h;
        }
      }
      P.b_plane[P.nb] = pl;
      P.b_v0[P.nb] = v[0];
      P.b_g[P.nb] = g;
      ++P.nb;
    }
  if (P.nb == 0) return false;
  *plan = P;
  return true;
}

struct TabArgs {
  const double* vals[3];  // [2][P][X] per direction
  const double* wts[3];
  int64_t X[3];           // points per direction
  int64_t N[3];           // functions per direction
  int K[3];               // elements per direction
  int md[3];              // deepest tabulated derivative level
};

// B^{lvl}_n(x) for point x of element e = x / Q (0 outside the band).
template <int P, int Q>
__device__ __forceinline__ double bval(const TabArgs& t, int dir, int lvl, int64_t n, int64_t x) {
  int64_t e = x / Q;
  int64_t j = n - e;
  if (j < 0 || j >= P || lvl > t.md[dir]) return 0.0;
  return t.vals[dir][((int64_t)lvl * P + j) * t.X[dir] + x];
}

// ---------------------------------------------------------------- 3D -------

struct Asm3Args {
  AsmPlan plan;
  TabArgs tab;
  const double* planes;
  int64_t pstride;
  double* H;          // [X2][nh][NS1][NS0]
  int64_t NS0, NS1;   // slot counts N·(2P-1)
  int nt0, nt1;       // row tiles
};

template <int P, int Q, int T>
struct A3Cfg {
  static constexpr int W = 2 * P - 1;        // band width
  static constexpr int PT = T * W;           // slots per tile per direction
  static constexpr int ER = T + P - 1;       // elements in the support region
  static constexpr int XR = ER * Q;          // points in the region
  static constexpr int NT = 256;
};

template <int P, int Q, int T>
__global__ void __launch_bounds__(256) asm3_stage12(const Asm3Args a) {
  using C = A3Cfg<P, Q, T>;
  constexpr int W = C::W, PT = C::PT, XR = C::XR, NT = C::NT;
  extern __shared__ double sm[];
  const AsmPlan& pl = a.plan;
  const int nb = pl.nb, ng = pl.ng, nh = pl.nh;
  double* Fs = sm;                         // [nb-planes][XR(y)][XR(x)] (by block)
  double* Gs = Fs + (size_t)nb * XR * XR;  // [ng][PT][XR(y)]
  const int tid = threadIdx.x;
  const int t0 = blockIdx.x % a.nt0, t1 = blockIdx.x / a.nt0;
  const int64_t x2 = blockIdx.y;
  const int a0 = t0 * T, a1 = t1 * T;           // first rows of the tile
  const int64_t xb0 = (int64_t)(a0 - (P - 1)) * Q, xb1 = (int64_t)(a1 - (P - 1)) * Q;  // first region points
  const int64_t X0 = a.tab.X[0], X1 = a.tab.X[1];
  // coefficient tile (distinct planes only once is not needed: F per block)
  for (int i = tid; i < nb * XR * XR; i += NT) {
    int b = i / (XR * XR), r = i % (XR * XR);
    int yl = r / XR, xl = r % XR;
    int64_t gx = xb0 + xl, gy = xb1 + yl;
    double v = 0.0;
    if (gx >= 0 && gx < X0 && gy >= 0 && gy < X1)
      v = __ldg(a.planes + (int64_t)pl.b_plane[b] * a.pstride + (x2 * X1 + gy) * X0 + gx);
    Fs[i] = v;
  }
  __syncthreads();
  // stage 1: G_g[s0][y] = Σ_b∈g Σ_x W0^{v0(b)}[pair0(s0)][x] F_b[y][x]
  for (int i = tid; i < PT * XR; i += NT) {
    const int s0 = i / XR, yl = i % XR;
    const int64_t m0 = a0 + s0 / W, n0 = m0 + (s0 % W) - (P - 1);
    double acc[kMaxBlocks];
    for (int g = 0; g < ng; ++g) acc[g] = 0.0;
    if (m0 < a.tab.N[0] && n0 >= 0 && n0 < a.tab.N[0]) {
      int64_t elo = (m0 > n0 ? m0 : n0) - (P - 1), ehi = m0 < n0 ? m0 : n0;
      if (elo < 0) elo = 0;
      if (ehi > a.tab.K[0] - 1) ehi = a.tab.K[0] - 1;
      for (int64_t e = elo; e <= ehi; ++e)
        for (int q = 0; q < Q; ++q) {
          const int64_t x = e * Q + q;
          const double w = a.tab.wts[0][x];
          const double bn0 = bval<P, Q>(a.tab, 0, 0, n0, x), bn1 = bval<P, Q>(a.tab, 0, 1, n0, x);
          const double bm0 = bval<P, Q>(a.tab, 0, 0, m0, x), bm1 = bval<P, Q>(a.tab, 0, 1, m0, x);
          const double wv[4] = {(w * bn0) * bm0, (w * bn1) * bm0, (w * bn0) * bm1, (w * bn1) * bm1};
          const double* fcol = Fs + (int64_t)yl * XR + (x - xb0);
          for (int b = 0; b < nb; ++b) acc[pl.b_g[b]] = fma(wv[pl.b_v0[b]], fcol[(int64_t)b * XR * XR], acc[pl.b_g[b]]);
        }
    }
    for (int g = 0; g < ng; ++g) Gs[((int64_t)g * PT + s0) * XR + yl] = acc[g];
  }
  __syncthreads();
  // stage 2: H_h[s1][s0] = Σ_{g∈h} Σ_y W1^{v1(g)}[pair1(s1)][y] G_g[s0][y]
  for (int i = tid; i < PT * PT; i += NT) {
    const int s1 = i / PT, s0 = i % PT;
    const int64_t m1 = a1 + s1 / W, n1 = m1 + (s1 % W) - (P - 1);
    const int64_t gs0 = (int64_t)a0 * W + s0, gs1 = (int64_t)a1 * W + s1;
    if (gs0 >= a.NS0 || gs1 >= a.NS1) continue;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (m1 < a.tab.N[1] && n1 >= 0 && n1 < a.tab.N[1]) {
      int64_t elo = (m1 > n1 ? m1 : n1) - (P - 1), ehi = m1 < n1 ? m1 : n1;
      if (elo < 0) elo = 0;
      if (ehi > a.tab.K[1] - 1) ehi = a.tab.K[1] - 1;
      for (int64_t e = elo; e <= ehi; ++e)
        for (int q = 0; q < Q; ++q) {
          const int64_t y = e * Q + q;
          const double w = a.tab.wts[1][y];
          const double bn0 = bval<P, Q>(a.tab, 1, 0, n1, y), bn1 = bval<P, Q>(a.tab, 1, 1, n1, y);
          const double bm0 = bval<P, Q>(a.tab, 1, 0, m1, y), bm1 = bval<P, Q>(a.tab, 1, 1, m1, y);
          const double wv[4] = {(w * bn0) * bm0, (w * bn1) * bm0, (w * bn0) * bm1, (w * bn1) * bm1};
          const int yl = (int)(y - xb1);
          for (int g = 0; g < ng; ++g)
            acc[pl.g_h[g]] = fma(wv[pl.g_v1[g]], Gs[((int64_t)g * PT + s0) * XR + yl], acc[pl.g_h[g]]);
        }
    }
    for (int h = 0; h < nh; ++h) a.H[((x2 * nh + h) * a.NS1 + gs1) * a.NS0 + gs0] = acc[h];
  }
}

struct Asm3bArgs {
  AsmPlan plan;
  TabArgs tab;
  const double* H;
  int64_t NS0, NS1;
  TensorPat pat;
  int64_t row_lo, row_hi;         // rows to write
  const int64_t* base;            // CSR offset of row_lo (device scalar)
  double* values;
};

// One thread per (slot0, slot1): sweep z with a ring of P rows x (2P-1) cols.
template <int P, int Q>
__global__ void __launch_bounds__(128) asm3_stage3(const Asm3bArgs a) {
  constexpr int W = 2 * P - 1;
  __shared__ double w2s[Q][4][P][P];  // W2^{v}[jn][jm] at the element's Q points
  const AsmPlan& pl = a.plan;
  const int nh = pl.nh;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s0 = gid % a.NS0, s1 = gid / a.NS0;
  const bool live = s1 < a.NS1;
  const int64_t N0 = a.tab.N[0], N1 = a.tab.N[1], N2 = a.tab.N[2];
  const int64_t m0 = s0 / W, n0 = m0 + (s0 % W) - (P - 1);
  const int64_t m1 = live ? s1 / W : 0, n1 = m1 + (live ? (s1 % W) : 0) - (P - 1);
  const bool valid = live && n0 >= 0 && n0 < N0 && n1 >= 0 && n1 < N1 && m0 < N0 && m1 < N1;
  // CSR geometry of this thread's (row, column) pairs in directions 0, 1
  int64_t w0 = 1, w1 = 1, rp0 = 0, rp1 = 0, r0 = 0, r1 = 0, P0 = 1, P1 = 1;
  if (valid) {
    rp0 = a.pat.rp[0][m0];
    w0 = a.pat.rp[0][m0 + 1] - rp0;
    rp1 = a.pat.rp[1][m1];
    w1 = a.pat.rp[1][m1 + 1] - rp1;
    P0 = a.pat.rp[0][N0];
    P1 = a.pat.rp[1][N1];
    r0 = n0 - a.pat.cl[0][rp0];
    r1 = n1 - a.pat.cl[1][rp1];
  }
  double ring[P][W];
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k < W; ++k) ring[r][k] = 0.0;
  const int K2 = a.tab.K[2];
  const int nthr = blockDim.x;
  auto flush = [&](int64_t m2, const double* row) {
    const int64_t rp2 = a.pat.rp[2][m2];
    const int64_t w2 = a.pat.rp[2][m2 + 1] - rp2;
    const int64_t lo2 = a.pat.cl[2][rp2];
    const int64_t m = m0 + N0 * (m1 + N1 * m2);
    if (m < a.row_lo || m >= a.row_hi) return;
    const int64_t start = rp0 * w1 * w2 + P0 * rp1 * w2 + P0 * P1 * rp2 - *a.base;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int64_t n2 = m2 + k - (P - 1);
      if (n2 >= 0 && n2 < N2) a.values[start + (n2 - lo2) * w0 * w1 + r1 * w0 + r0] = row[k];
    }
  };
  for (int eb = 0; eb < K2; eb += P) {
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int e2 = eb + r;
      if (e2 >= K2) break;
      __syncthreads();
      for (int i = threadIdx.x; i < Q * 4 * P * P; i += nthr) {
        int jm = i % P, jn = (i / P) % P, v = (i / (P * P)) % 4, q = i / (4 * P * P);
        int64_t x = (int64_t)e2 * Q + q;
        double w = a.tab.wts[2][x];
        double bn = (v & 1) > a.tab.md[2] ? 0.0 : a.tab.vals[2][((int64_t)(v & 1) * P + jn) * a.tab.X[2] + x];
        double bm = (v >> 1) > a.tab.md[2] ? 0.0 : a.tab.vals[2][((int64_t)(v >> 1) * P + jm) * a.tab.X[2] + x];
        w2s[q][v][jn][jm] = (w * bn) * bm;
      }
      __syncthreads();
      if (valid) {
        for (int q = 0; q < Q; ++q) {
          const int64_t x2 = (int64_t)e2 * Q + q;
          double h[4];
          for (int hh = 0; hh < nh; ++hh) h[hh] = __ldg(a.H + ((x2 * nh + hh) * a.NS1 + s1) * a.NS0 + s0);
#pragma unroll
          for (int jm = 0; jm < P; ++jm)
#pragma unroll
            for (int jn = 0; jn < P; ++jn) {
              double s = ring[(r + jm) % P][jn - jm + P - 1];
              for (int hh = 0; hh < nh; ++hh) s = fma(w2s[q][pl.h_v2[hh]][jn][jm], h[hh], s);
              ring[(r + jm) % P][jn - jm + P - 1] = s;
            }
        }
        // row m2 = e2 is final: write its 2P-1 columns, recycle the ring row
        flush(e2, ring[r % P]);
#pragma unroll
        for (int k = 0; k < W; ++k) ring[r % P][k] = 0.0;
      }
    }
  }
  // trailing rows m2 in [K2, K2 + P - 1) (their last element is K2 - 1)
  if (valid) {
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const int64_t m2 = K2 - 1 + t;
      const int slot = (int)(m2 % P);
#pragma unroll
      for (int s = 0; s < P; ++s)
        if (s == slot) flush(m2, ring[s]);
    }
  }
}

// ---------------------------------------------------------------- 2D -------

struct Asm2Args {
  AsmPlan plan;
  TabArgs tab;
  const double* planes;
  int64_t pstride;
  double* G;     // [X1][ng][NS0]
  int64_t NS0;
};

// G_g[y][s0] = Σ_b∈g Σ_x W0^{v0(b)}[pair0(s0)][x] F_b[y][x]
template <int P, int Q>
__global__ void __launch_bounds__(256) asm2_stage1(const Asm2Args a) {
  constexpr int W = 2 * P - 1;
  const AsmPlan& pl = a.plan;
  const int64_t X0 = a.tab.X[0], X1 = a.tab.X[1];
  const int64_t total = a.NS0 * X1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = i % a.NS0, y = i / a.NS0;
    const int64_t m0 = s0 / W, n0 = m0 + (s0 % W) - (P - 1);
    double acc[kMaxBlocks];
    for (int g = 0; g < pl.ng; ++g) acc[g] = 0.0;
    if (n0 >= 0 && n0 < a.tab.N[0]) {
      int64_t elo = (m0 > n0 ? m0 : n0) - (P - 1), ehi = m0 < n0 ? m0 : n0;
      if (elo < 0) elo = 0;
      if (ehi > a.tab.K[0] - 1) ehi = a.tab.K[0] - 1;
      for (int64_t e = elo; e <= ehi; ++e)
        for (int q = 0; q < Q; ++q) {
          const int64_t x = e * Q + q;
          const double w = a.tab.wts[0][x];
          const double bn0 = bval<P, Q>(a.tab, 0, 0, n0, x), bn1 = bval<P, Q>(a.tab, 0, 1, n0, x);
          const double bm0 = bval<P, Q>(a.tab, 0, 0, m0, x), bm1 = bval<P, Q>(a.tab, 0, 1, m0, x);
          const double wv[4] = {(w * bn0) * bm0, (w * bn1) * bm0, (w * bn0) * bm1, (w * bn1) * bm1};
          for (int b = 0; b < pl.nb; ++b)
            acc[pl.b_g[b]] = fma(wv[pl.b_v0[b]], __ldg(a.planes + (int64_t)pl.b_plane[b] * a.pstride + y * X0 + x),
                                 acc[pl.b_g[b]]);
        }
    }
    for (int g = 0; g < pl.ng; ++g) a.G[(y * pl.ng + g) * a.NS0 + s0] = acc[g];
  }
}

struct Asm2bArgs {
  AsmPlan plan;
  TabArgs tab;
  const double* G;
  int64_t NS0;
  int chunk;         // elements of direction 1 per thread chunk
  TensorPat pat;
  int64_t row_lo, row_hi;
  const int64_t* base;
  double* values;
};

// One thread per (slot0, chunk of y elements): ring over rows m1.  A chunk
// starts P-1 elements early so its first rows are complete (redundant work
// (P-1)/chunk); it writes rows m1 in [c·chunk, (c+1)·chunk) (+ the trailing
// P-1 rows for the last chunk).
template <int P, int Q>
__global__ void __launch_bounds__(128) asm2_stage2(const Asm2bArgs a) {
  constexpr int W = 2 * P - 1;
  const AsmPlan& pl = a.plan;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s0 = gid % a.NS0, c = gid / a.NS0;
  const int K1 = a.tab.K[1];
  const int nch = (K1 + a.chunk - 1) / a.chunk;
  if (c >= nch) return;
  const int64_t N0 = a.tab.N[0], N1 = a.tab.N[1];
  const int64_t m0 = s0 / W, n0 = m0 + (s0 % W) - (P - 1);
  if (m0 >= N0 || n0 < 0 || n0 >= N0) return;
  const int64_t rp0 = a.pat.rp[0][m0], w0 = a.pat.rp[0][m0 + 1] - rp0;
  const int64_t P0 = a.pat.rp[0][N0];
  const int64_t r0 = n0 - a.pat.cl[0][rp0];
  const int e_first = (int)c * a.chunk, e_last = min(K1, (int)(c + 1) * a.chunk);
  const int e_start = max(0, e_first - (P - 1));
  double ring[P][W];
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k < W; ++k) ring[r][k] = 0.0;
  auto flush = [&](int64_t m1, double* row) {
    if (m1 < e_first || m1 >= N1) return;
    if (m1 >= e_last && e_last != K1) return;
    const int64_t m = m0 + N0 * m1;
    if (m < a.row_lo || m >= a.row_hi) return;
    const int64_t rp1 = a.pat.rp[1][m1], lo1 = a.pat.cl[1][rp1];
    const int64_t start = rp0 * (a.pat.rp[1][m1 + 1] - rp1) + P0 * rp1 - *a.base;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int64_t n1 = m1 + k - (P - 1);
      if (n1 >= 0 && n1 < N1) a.values[start + (n1 - lo1) * w0 + r0] = row[k];
    }
  };
  for (int eb = e_start; eb < e_last; eb += P) {
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int e1 = eb + r;
      if (e1 >= e_last) break;
      const int rr = (e1 - e_start) % P;  // == r (eb steps by P from e_start)
      for (int q = 0; q < Q; ++q) {
        const int64_t y = (int64_t)e1 * Q + q;
        const double w = a.tab.wts[1][y];
        double bv[2][P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
          bv[0][j] = a.tab.vals[1][((int64_t)0 * P + j) * a.tab.X[1] + y];
          bv[1][j] = a.tab.md[1] >= 1 ? a.tab.vals[1][((int64_t)1 * P + j) * a.tab.X[1] + y] : 0.0;
        }
        for (int g = 0; g < pl.ng; ++g) {
          const double hv = __ldg(a.G + (y * pl.ng + g) * a.NS0 + s0);
          const int v = pl.g_v1[g];
#pragma unroll
          for (int jm = 0; jm < P; ++jm)
#pragma unroll
            for (int jn = 0; jn < P; ++jn) {
              double wt = (w * bv[v & 1][jn]) * bv[v >> 1][jm];
              ring[(r + jm) % P][jn - jm + P - 1] = fma(wt, hv, ring[(r + jm) % P][jn - jm + P - 1]);
            }
        }
      }
      (void)rr;
      flush(e1, ring[r % P]);
#pragma unroll
      for (int k = 0; k < W; ++k) ring[r % P][k] = 0.0;
    }
  }
  // trailing rows of the last chunk: m1 in [K1, K1 + P - 1)
  if (e_last == K1) {
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const int64_t m1 = K1 - 1 + t;
      const int slot = (int)((m1 - e_start) % P);
#pragma unroll
      for (int s = 0; s < P; ++s)
        if (s == slot) flush(m1, ring[s]);
    }
  }
}

// ---- host side ----------------------------------------------------------------

struct AsmShape {
  FusedShape fs;
  AsmPlan plan;
};

bool asm_shape(const igs_problem* p, const Dims& D, AsmShape* out) {
  AsmShape s;
  if (p->d != 2 && p->d != 3) return false;
  if (p->slab_lo || p->slab_hi) return false;
  const int d = p->d;
  s.fs.d = d;
  s.fs.p = p->trial[0].order;
  s.fs.k = p->trial[0].points_per_element;
  for (int k = 0; k < d; ++k) {
    const igs_dir& t = p->trial[k];
    const igs_dir& u = p->test[k];
    if (t.order != s.fs.p || u.order != s.fs.p) return false;
    if (t.points_per_element != s.fs.k || u.points_per_element != s.fs.k || s.fs.k <= 0) return false;
    if (t.num_elements <= 0 || t.num_basis != t.num_elements + t.order - 1) return false;
    if (t.values != u.values || t.first_active != u.first_active || t.weights != u.weights) return false;
    if (t.num_points != t.num_elements * s.fs.k) return false;
    if (p->dir_order[k] != k) return false;
    s.fs.nel[k] = t.num_elements;
    s.fs.nfn[k] = t.num_basis;
    s.fs.npt[k] = t.num_points;
  }
  if (!build_plan(p, &s.plan)) return false;
  // tables must hold the derivative levels the blocks use
  for (int k = 0; k < d; ++k)
    if (p->trial[k].max_deriv < 1) {
      for (int b = 0; b < s.plan.nb; ++b)
        if (s.plan.b_v0[b] != 0) return false;
    }
  if (s.fs.p < 2 || s.fs.p > 6 || s.fs.k != s.fs.p) return false;
  if (d == 3) {  // stage-1/2 tile must fit shared memory
    const int W = 2 * s.fs.p - 1, XR = (4 + s.fs.p - 1) * s.fs.k, PT = 4 * W;
    size_t smem = ((size_t)s.plan.nb * XR * XR + (size_t)s.plan.ng * PT * XR) * sizeof(double);
    if (smem > 232448) return false;
  }
  (void)D;
  if (out) *out = s;
  return true;
}

TabArgs tab_args(const igs_problem* p) {
  TabArgs t{};
  for (int k = 0; k < p->d; ++k) {
    t.vals[k] = p->trial[k].values;
    t.wts[k] = p->trial[k].weights;
    t.X[k] = p->trial[k].num_points;
    t.N[k] = p->trial[k].num_basis;
    t.K[k] = p->trial[k].num_elements;
    t.md[k] = p->trial[k].max_deriv;
  }
  return t;
}

constexpr int kTile = 4;

size_t asm_workspace(const AsmShape& s) {
  const int W = 2 * s.fs.p - 1;
  if (s.fs.d == 3) {
    return (size_t)s.fs.npt[2] * s.plan.nh * (s.fs.nfn[1] * W) * (s.fs.nfn[0] * W) * sizeof(double) + 512;
  }
  return (size_t)s.fs.npt[1] * s.plan.ng * (s.fs.nfn[0] * W) * sizeof(double) + 512;
}

template <int P, int Q>
igs_status launch3(const igs_problem* p, const AsmShape& s, TensorPat pat, int64_t row_lo, int64_t row_hi,
                   const int64_t* base, const double* planes, double* values, double* H, cudaStream_t st) {
  using C = A3Cfg<P, Q, kTile>;
  Asm3Args a{};
  a.plan = s.plan;
  a.tab = tab_args(p);
  a.planes = planes;
  a.pstride = p->plane_stride;
  a.H = H;
  a.NS0 = s.fs.nfn[0] * C::W;
  a.NS1 = s.fs.nfn[1] * C::W;
  a.nt0 = (int)ceil_div(s.fs.nfn[0], kTile);
  a.nt1 = (int)ceil_div(s.fs.nfn[1], kTile);
  size_t smem = ((size_t)s.plan.nb * C::XR * C::XR + (size_t)s.plan.ng * C::PT * C::XR) * sizeof(double);
  if (smem > 232448) return fail(IGS_ECAPACITY, "fused assembly tile does not fit shared memory");
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm3_stage12<P, Q, kTile>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                     "smem attribute"));
  dim3 grid((unsigned)(a.nt0 * a.nt1), (unsigned)s.fs.npt[2]);
  asm3_stage12<P, Q, kTile><<<grid, C::NT, smem, st>>>(a);
  IGS_LAUNCH_CHECK("asm3_stage12");
  Asm3bArgs b{};
  b.plan = s.plan;
  b.tab = a.tab;
  b.H = H;
  b.NS0 = a.NS0;
  b.NS1 = a.NS1;
  b.pat = pat;
  b.row_lo = row_lo;
  b.row_hi = row_hi;
  b.values = values;
  b.base = base;
  int64_t threads = a.NS0 * a.NS1;
  asm3_stage3<P, Q><<<(unsigned)ceil_div(threads, 128), 128, 0, st>>>(b);
  IGS_LAUNCH_CHECK("asm3_stage3");
  return IGS_OK;
}

template <int P, int Q>
igs_status launch2(const igs_problem* p, const AsmShape& s, TensorPat pat, int64_t row_lo, int64_t row_hi,
                   const int64_t* base, const double* planes, double* values, double* G, cudaStream_t st) {
  constexpr int W = 2 * P - 1;
  Asm2Args a{};
  a.plan = s.plan;
  a.tab = tab_args(p);
  a.planes = planes;
  a.pstride = p->plane_stride;
  a.G = G;
  a.NS0 = s.fs.nfn[0] * W;
  int64_t total = a.NS0 * s.fs.npt[1];
  int64_t grid = ceil_div(total, 256);
  if (grid > 148 * 32) grid = 148 * 32;
  asm2_stage1<P, Q><<<(unsigned)grid, 256, 0, st>>>(a);
  IGS_LAUNCH_CHECK("asm2_stage1");
  Asm2bArgs b{};
  b.plan = s.plan;
  b.tab = a.tab;
  b.G = G;
  b.NS0 = a.NS0;
  // enough (slot, chunk) threads to fill the GPU, chunks >= 4(P-1) elements
  int K1 = (int)s.fs.nel[1];
  int want = (int)ceil_div(148 * 1024, a.NS0);
  int chunk = (int)ceil_div(K1, want > 0 ? want : 1);
  if (chunk < 4 * (P - 1)) chunk = 4 * (P - 1);
  if (chunk > K1) chunk = K1;
  b.chunk = chunk;
  b.pat = pat;
  b.row_lo = row_lo;
  b.row_hi = row_hi;
  b.base = base;
  b.values = values;
  int64_t threads = a.NS0 * ceil_div(K1, chunk);
  asm2_stage2<P, Q><<<(unsigned)ceil_div(threads, 128), 128, 0, st>>>(b);
  IGS_LAUNCH_CHECK("asm2_stage2");
  return IGS_OK;
}

// CSR offset of the first row of the range (written into a device scalar
// so the stage kernels can subtract it; ranges start at row boundaries).
__global__ void row_start_kernel(TensorPat t, int64_t row, int64_t* out) {
  int64_t w[3], mi[3];
  *out = tensor_row_start(t, row, w, mi);
}

}  // namespace

bool fused_assemble_supported(const igs_problem* p, const Dims& D) {
  AsmShape s;
  return asm_shape(p, D, &s);
}

size_t fused_assemble_workspace(const igs_problem* p, const Dims& D) {
  AsmShape s;
  if (!asm_shape(p, D, &s)) return 0;
  return asm_workspace(s);
}

igs_status fused_assemble(const igs_problem* p, const Dims& D, const int64_t* const* rowptr1d,
                          const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                          const double* planes, double* values, void* ws, size_t ws_bytes,
                          cudaStream_t st) {
  AsmShape s;
  if (!asm_shape(p, D, &s)) return fail(IGS_ECAPACITY, "no fused assembly");
  if (ws_bytes < asm_workspace(s) || !ws) return fail(IGS_EWORKSPACE, "workspace too small for the fused assembly");
  TensorPat pat;
  pat.d = p->d;
  for (int k = 0; k < 3; ++k) {
    pat.rp[k] = k < p->d ? rowptr1d[k] : nullptr;
    pat.cl[k] = k < p->d ? cols1d[k] : nullptr;
    pat.ns[k] = D.ns[k];
    pat.nt[k] = D.nt[k];
  }
  int64_t* base = reinterpret_cast<int64_t*>(ws);
  double* buf = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + 256);
  row_start_kernel<<<1, 1, 0, st>>>(pat, row_lo, base);
  IGS_LAUNCH_CHECK("row_start_kernel");
  const int P = s.fs.p, Q = s.fs.k;
  igs_status r = IGS_ECAPACITY;
  bool done = false;
#define IGS_ASM_CASE(PP, QQ)                                                                    \
  if (!done && P == PP && Q == QQ) {                                                            \
    r = p->d == 3 ? launch3<PP, QQ>(p, s, pat, row_lo, row_hi, base, planes, values, buf, st)   \
                  : launch2<PP, QQ>(p, s, pat, row_lo, row_hi, base, planes, values, buf, st);  \
    done = true;                                                                                \
  }
  IGS_ASM_CASE(2, 2)
  IGS_ASM_CASE(3, 3)
  IGS_ASM_CASE(4, 4)
  IGS_ASM_CASE(5, 5)
  IGS_ASM_CASE(6, 6)
#undef IGS_ASM_CASE
  if (!done) return fail(IGS_ECAPACITY, "no fused assembly instantiation for this order / rule");
  return r;
}

}  // namespace igs
