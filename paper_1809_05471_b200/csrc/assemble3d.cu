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
//       asm_sweep<3> (one thread per (pair0, pair1)):
//         ring[m2][n2] += Σ_h W_z^{v2(h)} H_h  ->  CSR
//   2D: asm2_stage1 (x) -> HBM, asm_sweep<2> (y ring, chunked) -> CSR.
#include "fused.cuh"
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include "tma.cuh"

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
  int npl;                      // distinct coefficient planes
  int pl_list[kMaxBlocks];
  int b_ps[kMaxBlocks];         // block -> index into pl_list
  int g_b0[kMaxBlocks], g_nb[kMaxBlocks];  // blocks of group g: [g_b0, g_b0 + g_nb)
  int h_g0[kMaxBlocks], h_ng[kMaxBlocks];  // groups of stage-2 group h (3D)
  int half_b;                   // 3D stage 1: blocks [0, half_b) | [half_b, nb), whole
                                // groups, balanced by block count
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
      int ps = -1;
      for (int q = 0; q < P.npl; ++q)
        if (P.pl_list[q] == pl) ps = q;
      if (ps < 0) {
        ps = P.npl++;
        P.pl_list[ps] = pl;
      }
      P.b_ps[P.nb] = ps;
      P.b_plane[P.nb] = pl;
      P.b_v0[P.nb] = v[0];
      P.b_g[P.nb] = g;
      ++P.nb;
    }
  if (P.nb == 0) return false;
  // Renumber groups so each stage-2 group's groups are contiguous, then order
  // blocks by group (stable: the reference's block order within a group).
  int gperm[kMaxBlocks], ng_new = 0;
  if (d == 3) {
    for (int h = 0; h < P.nh; ++h) {
      P.h_g0[h] = ng_new;
      for (int g = 0; g < P.ng; ++g)
        if (P.g_h[g] == h) gperm[g] = ng_new++;
      P.h_ng[h] = ng_new - P.h_g0[h];
    }
  } else {
    for (int g = 0; g < P.ng; ++g) gperm[g] = g;
  }
  AsmPlan Q = P;
  for (int g = 0; g < P.ng; ++g) {
    Q.g_v1[gperm[g]] = P.g_v1[g];
    Q.g_h[gperm[g]] = P.g_h[g];
  }
  int nbo = 0;
  for (int gn = 0; gn < P.ng; ++gn) {
    Q.g_b0[gn] = nbo;
    for (int b = 0; b < P.nb; ++b)
      if (gperm[P.b_g[b]] == gn) {
        Q.b_plane[nbo] = P.b_plane[b];
        Q.b_v0[nbo] = P.b_v0[b];
        Q.b_ps[nbo] = P.b_ps[b];
        Q.b_g[nbo] = gn;
        ++nbo;
      }
    Q.g_nb[gn] = nbo - Q.g_b0[gn];
  }
  // two contiguous group ranges with ~nb/2 blocks each (stage-1 warp halves)
  Q.half_b = Q.nb;
  {
    int best = 1 << 30;
    for (int gn = 0; gn < Q.ng; ++gn) {
      const int end = Q.g_b0[gn] + Q.g_nb[gn];
      const int imb = std::abs(2 * end - Q.nb);
      if (end < Q.nb && imb < best) {
        best = imb;
        Q.half_b = end;
      }
    }
  }
  *plan = Q;
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
  int lz;             // z point layers per CTA
  int nplanes;        // planes in the TMA box (all planes of the field)
  int64_t z0, z1;     // global z points to contract: elements [e_lo, e_hi) of the row range
  int64_t NE;         // elements in H (e_hi - e_lo)
  int64_t zpl;        // global z point of the coefficient planes' first layer (slab origin)
};

__device__ __forceinline__ void dmma_a(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Sweep-blocked layout of the last-direction intermediate (H in 3D, G in
// 2D): [block of 128 slot pairs][element - e_lo][q][group][128], so one
// element of one sweep block is a contiguous Q·ngrp·128-double tile (one
// bulk copy).
constexpr int kSweepBlock = 128;
__host__ __device__ __forceinline__ int64_t sweep_offset(int64_t sp, int64_t e_loc, int q, int h, int64_t NE,
                                                         int Q, int ngrp) {
  return ((((sp / kSweepBlock) * NE + e_loc) * Q + q) * ngrp + h) * kSweepBlock + sp % kSweepBlock;
}

// Stage-1/2 tile plan: T x T rows in (x, y), their (T+P-1)-element support
// region, slots = T·(2P-1) band entries per direction.
// SYM: only the x-pairs n0 >= m0 (slots m·P + (n - m), the symmetric half of
// the band; three-pass path of a symmetric problem, mirrored in the z sweep).
template <int P, int Q, int T, bool SYM = false>
struct A3Cfg {
  static constexpr int W = SYM ? P : 2 * P - 1;  // slots per row: band width (or its symmetric half)
  static constexpr int OFF = SYM ? 0 : P - 1;    // slot offset of the diagonal (n = m)
  // slot positions per row: a 7-wide band is padded to 8 so every MMA slot
  // tile is exactly one row (its k-range is then exactly the row's P elements)
  static constexpr int SR = W == 7 ? 8 : W;
  static constexpr int PT = T * SR;          // slot positions per tile per direction
  static constexpr int PTP = (PT + 7) & ~7;  // padded to MMA tiles
  static constexpr int ER = T + P - 1;       // elements in the support region
  static constexpr int XR = ER * Q;          // points in the region (TMA box width)
  static constexpr int XRP = (XR + 7) & ~7;  // ... padded to MMA tiles (y rows)
  static constexpr int XK = (XR + 3) & ~3;   // ... padded to k-steps (x)
  static constexpr int NT = 512, NW = 16;
  // Row pitches ≡ 4 (mod 16) doubles: a fragment load that walks 4 rows x 8
  // consecutive doubles (or 8 rows x 4) then hits every bank once per half-warp.
  static constexpr int pitch4(int n) { return ((n + 11) / 16) * 16 + 4; }
  static constexpr int SP = pitch4(PTP);     // rows over slots: W0 tables, G
  static constexpr int YP = pitch4(XRP);     // rows over y points: W1 tables (transposed)
  static constexpr int W0T = 4 * XK * SP;    // W0[v][x][s0]
  static constexpr int W1T = 4 * PTP * YP;   // W1[v][s1][y]
  // + 4 doubles of zero tail: the last row's k-step padding (x in [XR, XK))
  static constexpr size_t fdoubles(int npl) { return ((size_t)npl * XRP * XR + 4 + 15) & ~size_t(15); }
  static constexpr size_t smem(int npl, int ng) {
    return (fdoubles(npl) + (size_t)ng * XRP * SP + W0T + W1T) * sizeof(double) + 16;
  }
};

// Dense band tables of one direction over the tile's region:
//   W[v][x][s] = w(x)·B^θ_{n}(x)·B^η_{m}(x)  for slot s = (m - a)·W + (n - m + P - 1),
// v = θ + 2η; zero where x is outside the mesh/region or (m, n) outside the
// support of x's element (same product order as _Core.w_matrix).
// transposed = true stores [v][s][x] (row pitch YP) for the stage-2 A operand.
template <int P, int Q, int T, bool TRANSPOSED, bool SYM = false>
__device__ void fill_band_table(double* Wt, const TabArgs& t, int dir, int a_row, int64_t x_first) {
  using C = A3Cfg<P, Q, T, SYM>;
  constexpr int W = C::W;
  constexpr int NX = TRANSPOSED ? C::XRP : C::XK;
  constexpr int NS = TRANSPOSED ? C::PTP : C::SP;
  constexpr int PITCH = TRANSPOSED ? C::YP : C::SP;
  constexpr int ROWS = TRANSPOSED ? C::PTP : C::XK;
  constexpr int TOT = 4 * ROWS * PITCH;
  const int64_t Nf = t.N[dir];
  for (int i = threadIdx.x; i < TOT; i += blockDim.x) {
    const int col = i % PITCH, row = (i / PITCH) % ROWS, v = i / (PITCH * ROWS);
    const int xl = TRANSPOSED ? col : row, sl = TRANSPOSED ? row : col;
    double val = 0.0;
    if (xl < C::XR && xl < NX && sl < C::PT && sl < NS && sl % C::SR < W) {
      const int64_t x = x_first + xl;
      const int64_t m = a_row + sl / C::SR, n = m + sl % C::SR - C::OFF;
      if (x >= 0 && x < t.X[dir] && m < Nf && n >= 0 && n < Nf) {
        const int64_t e = x / Q;
        const int64_t jn = n - e, jm = m - e;
        const int th = v & 1, et = v >> 1;
        if (jn >= 0 && jn < P && jm >= 0 && jm < P && th <= t.md[dir] && et <= t.md[dir]) {
          const double w = t.wts[dir][x];
          const double bn = t.vals[dir][((int64_t)th * P + jn) * t.X[dir] + x];
          const double bm = t.vals[dir][((int64_t)et * P + jm) * t.X[dir] + x];
          val = (w * bn) * bm;
        }
      }
    }
    Wt[i] = val;
  }
}

// k-steps (of 4 points) of the region that touch the tile rows behind slot
// tile `st`: row r (tile-relative) is supported by region elements [r, r+P-1].
template <int P, int Q, int T, bool SYM = false>
__host__ __device__ constexpr void slot_tile_ksteps(int st, int kmax, int& k_lo, int& k_hi) {
  constexpr int SR = A3Cfg<P, Q, T, SYM>::SR;
  const int r_lo = (st * 8) / SR;
  const int r_hi = (st * 8 + 7) / SR < T - 1 ? (st * 8 + 7) / SR : T - 1;
  k_lo = (r_lo * Q) / 4;
  k_hi = ((r_hi + P) * Q + 3) / 4 < kmax ? ((r_hi + P) * Q + 3) / 4 : kmax;
}
// shortest k-step range over the slot tiles (equal to the longest: no predicates)
template <int P, int Q, int T>
constexpr int min_ksteps(int ntiles, int kmax) {
  int m = 1 << 30;
  for (int st = 0; st < ntiles; ++st) {
    int lo = 0, hi = 0;
    slot_tile_ksteps<P, Q, T>(st, kmax, lo, hi);
    if (hi - lo < m) m = hi - lo;
  }
  return m;
}
// longest k-step range over the slot tiles (static unroll bound)
template <int P, int Q, int T, bool SYM = false>
constexpr int max_ksteps(int ntiles, int kmax) {
  int m = 1;
  for (int st = 0; st < ntiles; ++st) {
    int lo = 0, hi = 0;
    slot_tile_ksteps<P, Q, T, SYM>(st, kmax, lo, hi);
    if (hi - lo > m) m = hi - lo;
  }
  return m;
}

// Per (tile of T x T rows, chunk of z point layers), for every layer, as
// dense banded GEMMs (DMMA m8n8k4, accumulators in registers, no scatter):
//   stage 1 (x):  G_g[y][s0] = Σ_{b∈g} Σ_x F_b[y][x] · W0^{v0(b)}[x][s0]       (M=y  N=s0 K=x)
//   stage 2 (y):  H_h[s1][s0] = Σ_{g∈h} Σ_y W1^{v1(g)}[s1][y] · G_g[y][s0]     (M=s1 N=s0 K=y)
// Each warp task owns one output tile for all groups (balanced); k-steps
// that cannot touch the task's rows are skipped.  H goes straight from the
// MMA fragments to HBM; the next layer's coefficient region is fetched by TMA
// while stage 2 runs.
template <int P, int Q, int T>
__global__ void __launch_bounds__(512, 1)
    asm3_stage12(const Asm3Args a, const __grid_constant__ CUtensorMap fmap) {
  using C = A3Cfg<P, Q, T>;
  constexpr int PT = C::PT, PTP = C::PTP, XR = C::XR, XRP = C::XRP, XK = C::XK;
  constexpr int NT = C::NT, NW = C::NW, SP = C::SP, YP = C::YP, W = C::W;
  constexpr int KL1 = max_ksteps<P, Q, T>(PTP / 8, XK / 4), KL2 = max_ksteps<P, Q, T>(PTP / 8, XRP / 4);
  constexpr bool kFullK1 = KL1 == min_ksteps<P, Q, T>(PTP / 8, XK / 4);
  constexpr int NYP = (XRP / 8 + 1) / 2;  // pairs of y tiles
  constexpr bool kFullK2 = KL2 == min_ksteps<P, Q, T>(PTP / 8, XRP / 4);
  extern __shared__ __align__(128) double sm[];
  const AsmPlan& pl = a.plan;
  const int ng = pl.ng, nh = pl.nh;
  const size_t fsz = C::fdoubles(a.nplanes);
  double* Fs = sm;                   // [n_planes][XRP y][XR x]   (TMA box)
  double* Gs = Fs + fsz;             // [ng][XRP y][SP]
  double* W0 = Gs + (size_t)ng * XRP * SP;  // [4][XK x][SP]
  double* W1 = W0 + C::W0T;                  // [4][PTP s1][YP]
  uint64_t* bar = reinterpret_cast<uint64_t*>(W1 + C::W1T);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, m4 = lane & 3;
  const int t0 = blockIdx.x % a.nt0, t1 = blockIdx.x / a.nt0;
  const int64_t z_lo = a.z0 + (int64_t)blockIdx.y * a.lz;
  const int64_t z_hi = min64(a.z1, z_lo + a.lz);
  const int a0 = t0 * T, a1 = t1 * T;                     // first rows of the tile
  const int xb0 = (a0 - (P - 1)) * Q, xb1 = (a1 - (P - 1)) * Q;  // first region points (may be < 0)
  const unsigned fbytes = (unsigned)((size_t)a.nplanes * XRP * XR * sizeof(double));
  for (size_t i = (size_t)a.nplanes * XRP * XR + tid; i < fsz; i += NT) Fs[i] = 0.0;  // k-step tail
  if (tid == 0) {
    dev::mbar_init(bar, 1);
    dev::fence_mbar_init();
  }
  dev::fence_proxy_async();
  __syncthreads();
  if (tid == 0 && z_lo < z_hi) {
    dev::mbar_expect_tx(bar, fbytes);
    dev::tma_load_4d(Fs, &fmap, bar, xb0, xb1, (int)(z_lo - a.zpl), 0);
  }
  fill_band_table<P, Q, T, false>(W0, a.tab, 0, a0, xb0);
  fill_band_table<P, Q, T, true>(W1, a.tab, 1, a1, xb1);
  __syncthreads();
  unsigned phase = 0;
  for (int64_t x2 = z_lo; x2 < z_hi; ++x2, phase ^= 1) {
    dev::mbar_wait(bar, phase);
    // ---- stage 1: task = (pair of y tiles, s0 tile, half of the blocks) --------
    // Both y tiles share every W0 fragment (shared-memory traffic is the
    // stage's bound); the block halves are whole groups.  Blocks are ordered
    // by group: the accumulators are stored and reset after a group's last
    // block (static block index: plan reads are constant-bank immediates).
    for (int t = warp; t < NYP * (PTP / 8) * 2; t += NW) {
      const int half = t & 1, st = (t >> 1) % (PTP / 8), yp = (t >> 1) / (PTP / 8);
      int k_lo, k_hi;
      slot_tile_ksteps<P, Q, T>(st, XK / 4, k_lo, k_hi);
      const bool y1ok = 2 * yp + 1 < XRP / 8;
      const int y0 = 2 * yp * 8 + g8, y1 = y1ok ? y0 + 8 : y0;
      const double* F0 = Fs + y0 * XR + m4 + k_lo * 4;
      const double* F1 = Fs + y1 * XR + m4 + k_lo * 4;
      const double* Wk = W0 + (m4 + k_lo * 4) * SP + st * 8 + g8;
      const int b_lo = half ? pl.half_b : 0, b_hi = half ? pl.nb : pl.half_b;
      double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll
      for (int b = 0; b < kMaxBlocks; ++b) {
        if (b < b_lo) continue;
        if (b >= b_hi) break;
        const int po = pl.b_plane[b] * (XRP * XR);
        const double* Wb = Wk + pl.b_v0[b] * (XK * SP);
#pragma unroll
        for (int kk = 0; kk < KL1; ++kk)
          if (kFullK1 || k_lo + kk < k_hi) {
            const double w = Wb[kk * 4 * SP];
            dmma_a(c0[0], c0[1], F0[po + kk * 4], w);
            dmma_a(c1[0], c1[1], F1[po + kk * 4], w);
          }
        if (b + 1 == pl.nb || pl.b_g[b + 1] != pl.b_g[b]) {
          double* Gd = Gs + (pl.b_g[b] * XRP + y0) * SP + st * 8 + 2 * m4;
          *reinterpret_cast<double2*>(Gd) = make_double2(c0[0], c0[1]);
          if (y1ok) *reinterpret_cast<double2*>(Gd + 8 * SP) = make_double2(c1[0], c1[1]);
          c0[0] = c0[1] = c1[0] = c1[1] = 0.0;
        }
      }
    }
    __syncthreads();
    // F is consumed: fetch the next layer's region while stage 2 runs
    if (tid == 0 && x2 + 1 < z_hi) {
      dev::fence_proxy_async();
      dev::mbar_expect_tx(bar, fbytes);
      dev::tma_load_4d(Fs, &fmap, bar, xb0, xb1, (int)(x2 + 1 - a.zpl), 0);
    }
    // ---- stage 2: task = (s1 tile, s0 tile), all stage-2 groups ----------------
    for (int t = warp; t < (PTP / 8) * (PTP / 8); t += NW) {
      const int mt = t / (PTP / 8), st = t % (PTP / 8);
      int k_lo, k_hi;
      slot_tile_ksteps<P, Q, T>(mt, XRP / 4, k_lo, k_hi);
      constexpr int SR = C::SR;
      const int s1 = mt * 8 + g8;  // slot position (row s1 / SR, offset s1 % SR)
      const int64_t gs1 = (int64_t)(a1 + s1 / SR) * W + s1 % SR;
      const bool row_ok = s1 < PT && s1 % SR < W && gs1 < a.NS1;
      const int s0 = st * 8 + 2 * m4;
      const int64_t gs0 = (int64_t)(a0 + s0 / SR) * W + s0 % SR;
      const int64_t gs0b = (int64_t)(a0 + (s0 + 1) / SR) * W + (s0 + 1) % SR;
      const bool ok0 = row_ok && s0 < PT && s0 % SR < W && gs0 < a.NS0;
      const bool ok1 = row_ok && s0 + 1 < PT && (s0 + 1) % SR < W && gs0b < a.NS0;
      const int64_t e_loc = (x2 - a.z0) / Q;
      const int qz = (int)((x2 - a.z0) % Q);
      const int64_t off0 = sweep_offset(gs1 * a.NS0 + gs0, e_loc, qz, 0, a.NE, Q, nh);
      const int64_t off1 = sweep_offset(gs1 * a.NS0 + gs0b, e_loc, qz, 0, a.NE, Q, nh);
      const double* Wk = W1 + s1 * YP + m4 + k_lo * 4;
      const double* Gk = Gs + (m4 + k_lo * 4) * SP + st * 8 + g8;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int g = 0; g < kMaxBlocks; ++g) {
        if (g >= pl.ng) break;
        const double* Wg = Wk + pl.g_v1[g] * (PTP * YP);
        const double* Gg = Gk + g * (XRP * SP);
#pragma unroll
        for (int kk = 0; kk < KL2; ++kk)
          if (kFullK2 || k_lo + kk < k_hi) dmma_a(d0, d1, Wg[kk * 4], Gg[kk * 4 * SP]);
        if (g + 1 == pl.ng || pl.g_h[g + 1] != pl.g_h[g]) {
          const int hoff = pl.g_h[g] * kSweepBlock;
          if (ok0) a.H[off0 + hoff] = d0;
          if (ok1) a.H[off1 + hoff] = d1;
          d0 = d1 = 0.0;
        }
      }
    }
    __syncthreads();
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
  const double* w2g;              // [K][Q][P][P][4] weights of the swept direction
  int e_lo, e_hi;                 // elements swept (H holds their points from e_lo·Q)
  int64_t NE;                     // elements held by H (sweep-blocked layout)
  int chunk;                      // elements per thread chunk (rows written per chunk)
  int ngrp;                       // groups summed per point (3D: nh, 2D: ng)
  int vmap[4];                    // group holding variant v = θ + 2η of the swept direction (-1: none)
};

// Per element record of the swept (last) direction, computed once: the
// separable factors of W^{θ+2η}[jn][jm](q) = (w·B^θ_jn)(q) · B^η_jm(q),
// [q][wB^0 | wB^1 | B^0 | B^1][P padded to even], then the CSR metadata of row m2 = e (row
// start, width, first column).
template <int P, int Q, int D>
__global__ void asm_wlast_kernel(const Asm3bArgs a, double* w2g) {
  constexpr int PP = (P + 1) & ~1, NWT = Q * 4 * PP, NWR = NWT + 4, L = D - 1;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)a.tab.K[L] * NWR) return;
  const int e2 = (int)(i / NWR), r = (int)(i % NWR);
  if (r >= NWT) {  // row metadata of row m2 = e2: CSR row start, width, first column
    const int64_t rp2 = a.pat.rp[L][e2];
    const int64_t v = r == NWT ? rp2 : r == NWT + 1 ? a.pat.rp[L][e2 + 1] - rp2 : r == NWT + 2 ? a.pat.cl[L][rp2] : 0;
    reinterpret_cast<int64_t*>(w2g)[i] = v;
    return;
  }
  const int j = r % PP, f = (r / PP) % 4, q = r / (4 * PP);
  const int lvl = f & 1;
  if (j >= P) {
    w2g[i] = 0.0;
    return;
  }
  const int64_t x = (int64_t)e2 * Q + q;
  const double b = lvl > a.tab.md[L] ? 0.0 : a.tab.vals[L][((int64_t)lvl * P + j) * a.tab.X[L] + x];
  w2g[i] = f < 2 ? a.tab.wts[L][x] * b : b;
}

// Last-direction pipeline: shared-memory ring of NS3 element stages, each
// filled by two bulk copies (the block's H tile and the element weights)
// D3 = NS3 - 1 elements ahead.  One element ahead is the measured optimum:
// deeper rings (or L2 prefetch further ahead) put more concurrent streams on
// the DRAM and run slower (C3: D3 = 2 -> 1 saves 0.06 ms).
constexpr int NS3 = 2, D3 = NS3 - 1, NT3 = kSweepBlock;
template <int P, int Q>
struct S3Cfg {
  static constexpr int PP = (P + 1) & ~1;     // factor row pitch (16-byte rows)
  static constexpr int NWT = Q * 4 * PP;      // separable weight factors per element
  static constexpr int NWR = NWT + 4;         // + row metadata (3 int64, padded)
  static constexpr int HST = Q * 4 * NT3;     // H values per stage [q][group <= 4][thread]
  static constexpr size_t SMEM = (size_t)NS3 * (HST + NWR) * sizeof(double) + NS3 * sizeof(uint64_t);
};

// Last-direction sweep (3D stage 3, 2D stage 2).  Block = (chunk of
// elements, 128 consecutive slot pairs (slot0[, slot1])); each thread sweeps
// the last direction for its pair with a ring of P rows x (2P-1) cols in
// registers.  An element's H values for the whole block are one contiguous
// tile of the sweep-blocked layout, fetched with the element's weights by
// one thread (cp.async.bulk + mbarrier) D3 elements ahead.  A chunk starts
// P-1 elements early (its first rows are then complete) and writes the rows
// of its own elements (the last chunk also the trailing P-1 rows).  2D is
// 3D with a trivial middle direction.
// SYMX (3D three-pass path of a symmetric problem, whole matrix): the x slots
// hold only n0 >= m0 (s0 = m0·P + (n0 - m0)); a pair with n0 > m0 writes each
// value to its own row and, mirrored, to row (n0, n1, n2) at column
// (m0, m1, m2) — every CSR entry exactly once.
template <int P, int Q, int D, bool SYMX = false>
__global__ void __launch_bounds__(NT3, P <= 4 ? 3 : 1) asm_sweep(const Asm3bArgs a) {
  using C = S3Cfg<P, Q>;
  constexpr int W = 2 * P - 1, NWT = C::NWT, NWR = C::NWR, PP = C::PP, L = D - 1;
  constexpr int WX = SYMX ? P : W, OFFX = SYMX ? 0 : P - 1;
  static_assert(!SYMX || D == 3, "mirrored sweep: 3D only");
  static_assert(NWT % 2 == 0, "16-byte table chunks");
  extern __shared__ __align__(16) double s3[];
  double* hst = s3;                    // [NS3][Q][ngrp][NT3]
  double* w2s = s3 + NS3 * C::HST;     // [NS3][NWR]: factors [Q][4][P] + row metadata
  uint64_t* bars = reinterpret_cast<uint64_t*>(w2s + NS3 * NWR);
  int64_t* zrt = reinterpret_cast<int64_t*>(bars + NS3);  // SYMX: [N2][3] z-row table
  const int nh = a.ngrp;
  const int tid = threadIdx.x;
  const int64_t npairs = a.NS0 * a.NS1;
  const int64_t nbsp = (npairs + NT3 - 1) / NT3;
  const int chunk_id = (int)(blockIdx.x / nbsp);
  const int64_t sb = blockIdx.x % nbsp;
  const int64_t sp = sb * NT3 + tid;
  const int64_t s0 = sp % a.NS0, s1 = sp / a.NS0;
  const int64_t N0 = a.tab.N[0], N1 = D == 3 ? a.tab.N[1] : 1, N2 = a.tab.N[L];
  const int64_t m0 = s0 / WX, n0 = m0 + (s0 % WX) - OFFX;
  const int64_t m1 = D == 3 ? s1 / W : 0, n1 = D == 3 ? m1 + (s1 % W) - (P - 1) : 0;
  const bool valid = sp < npairs && n0 >= 0 && n0 < N0 && n1 >= 0 && n1 < N1 && m0 < N0 && m1 < N1;
  // CSR geometry of this thread's (row, column) pairs in the first directions
  int64_t w0 = 1, w1 = 1, rp0 = 0, rp1 = 0, r0 = 0, r1 = 0, P0 = 1, P1 = 1;
  if (valid) {
    rp0 = a.pat.rp[0][m0];
    w0 = a.pat.rp[0][m0 + 1] - rp0;
    P0 = a.pat.rp[0][N0];
    r0 = n0 - a.pat.cl[0][rp0];
    if (D == 3) {
      rp1 = a.pat.rp[1][m1];
      w1 = a.pat.rp[1][m1 + 1] - rp1;
      P1 = a.pat.rp[1][N1];
      r1 = n1 - a.pat.cl[1][rp1];
    }
  }
  // mirror geometry: row (n0, n1, ·), column (m0, m1, ·)
  const bool mir = SYMX && valid && n0 > m0;
  int64_t w0n = 1, w1n = 1, rp0n = 0, rp1n = 0, r0n = 0, r1n = 0;
  if (mir) {
    rp0n = a.pat.rp[0][n0];
    w0n = a.pat.rp[0][n0 + 1] - rp0n;
    r0n = m0 - a.pat.cl[0][rp0n];
    rp1n = a.pat.rp[1][n1];
    w1n = a.pat.rp[1][n1 + 1] - rp1n;
    r1n = m1 - a.pat.cl[1][rp1n];
  }
  double ring[P][W];
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k < W; ++k) ring[r][k] = 0.0;
  const int K2 = a.tab.K[L];
  // this block's chunk: rows [c_lo, c_hi) (+ trailing rows), elements from c_lo - P + 1
  const int c_lo = a.e_lo + chunk_id * a.chunk;
  const int c_hi = min(a.e_hi, c_lo + a.chunk);
  const int e_lo = max(a.e_lo, c_lo - (P - 1)), e_hi = c_hi;
  const int64_t base = *a.base;
  // meta = {rp2, w2, lo2} of row m2 (from the element record in shared
  // memory, or from the pattern for the trailing rows)
  auto flush = [&](int64_t m2, const double* row, const int64_t* meta) {
    if (m2 < c_lo || (m2 >= c_hi && c_hi != K2)) return;
    const int64_t rp2 = meta[0], w2 = meta[1], lo2 = meta[2];
    const int64_t m = m0 + N0 * (m1 + N1 * m2);
    if (m < a.row_lo || m >= a.row_hi) return;
    const int64_t start = rp0 * w1 * w2 + P0 * rp1 * w2 + P0 * P1 * rp2 - base;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int64_t n2 = m2 + k - (P - 1);
      if (n2 >= 0 && n2 < N2) a.values[start + (n2 - lo2) * w0 * w1 + r1 * w0 + r0] = row[k];
    }
    if (mir) {
      // (SYMX runs whole-matrix ranges only: every mirrored row is in range)
      if (m2 >= 2 * (P - 1) && m2 + 2 * P - 1 <= N2) {
        // every row n2 within P-1 of m2 is an interior z row (width W, first
        // column n2 - (P-1), row starts W apart): the mirror offsets are affine in k
        const int64_t ww = w0n * w1n;
        const int64_t rz = zrt[3 * (P - 1)] + (m2 - 2 * (P - 1)) * W;  // row start of n2 = m2 - (P-1)
        double* vm = a.values + ((rp0n * w1n + P0 * rp1n) * W + P0 * P1 * rz - base + 2 * (P - 1) * ww +
                                 r1n * w0n + r0n);
        const int64_t step = P0 * P1 * W - ww;
#pragma unroll
        for (int k = 0; k < W; ++k) vm[k * step] = row[k];
      } else
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int64_t n2 = m2 + k - (P - 1);
        if (n2 < 0 || n2 >= N2) continue;
        const int64_t rp2n = zrt[3 * n2], w2n = zrt[3 * n2 + 1], lo2n = zrt[3 * n2 + 2];
        const int64_t startn = rp0n * w1n * w2n + P0 * rp1n * w2n + P0 * P1 * rp2n - base;
        a.values[startn + (m2 - lo2n) * w0n * w1n + r1n * w0n + r0n] = row[k];
      }
    }
  };
  const unsigned htile = (unsigned)(Q * nh * NT3 * sizeof(double));
  const unsigned wbytes = (unsigned)(NWR * sizeof(double));
  const double* hblock = a.H + sb * a.NE * Q * nh * NT3;
  auto issue = [&](int e2) {  // one thread
    if (e2 >= e_hi) return;
    const int stg = (e2 - e_lo) % NS3;
    dev::mbar_expect_tx(bars + stg, htile + wbytes);
    dev::bulk_load(hst + stg * C::HST, hblock + (int64_t)(e2 - a.e_lo) * Q * nh * NT3, htile, bars + stg);
    dev::bulk_load(w2s + stg * NWR, a.w2g + (int64_t)e2 * NWR, wbytes, bars + stg);
  };
  if (tid < NS3) dev::mbar_init(bars + tid, 1);
  dev::fence_mbar_init();
  if constexpr (SYMX) {
    // z-row table of the mirrored rows: [row start, width, first column]
    const int64_t* rpz = a.pat.rp[L];
    const int64_t* clz = a.pat.cl[L];
    for (int64_t r = tid; r < N2; r += NT3) {
      const int64_t rs = rpz[r];
      zrt[3 * r] = rs;
      zrt[3 * r + 1] = rpz[r + 1] - rs;
      zrt[3 * r + 2] = clz[rs];
    }
  }
  __syncthreads();
  if (tid == 0)
    for (int e = 0; e < D3; ++e) issue(e_lo + e);
  for (int eb = e_lo; eb < e_hi; eb += P) {
#pragma unroll
    for (int r = 0; r < P; ++r) {  // ring row of element e2 is static: r
      const int e2 = eb + r;
      if (e2 >= e_hi) break;
      // stage (e2 + D3 - e_lo) % NS3 was last read for element e2 - 1,
      // finished by every thread before this barrier
      __syncthreads();
      if (tid == 0) {
        dev::fence_proxy_async();
        issue(e2 + D3);
      }
      const int stg = (e2 - e_lo) % NS3;
      dev::mbar_wait(bars + stg, (unsigned)(((e2 - e_lo) / NS3) & 1));
      const double* hcol = hst + stg * C::HST + tid;
      const double* wst = w2s + stg * NWR;
      // Σ_{θ,η} (wB^θ_jn)(B^η_jm) H_{θ+2η}: contract θ first (u_η[jn]),
      // then η into the ring (P·P·2 + 4P FMAs, 4P broadcast factors per q);
      // p >= 5 keeps the point loop rolled (instruction-cache footprint)
#pragma unroll(P >= 5 ? 1 : Q)
      for (int q = 0; q < Q; ++q) {
        double hv[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) hv[v] = a.vmap[v] >= 0 ? hcol[(q * nh + a.vmap[v]) * NT3] : 0.0;
        double fb[4][P];
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
          for (int j = 0; j < P; j += 2) {
            if (j + 1 < P) {
              const double2 t = *reinterpret_cast<const double2*>(wst + (q * 4 + f) * PP + j);
              fb[f][j] = t.x;
              fb[f][j + 1] = t.y;
            } else {
              fb[f][j] = wst[(q * 4 + f) * PP + j];
            }
          }
        double u0[P], u1[P];
#pragma unroll
        for (int jn = 0; jn < P; ++jn) {
          u0[jn] = fma(fb[1][jn], hv[1], fb[0][jn] * hv[0]);
          u1[jn] = fma(fb[1][jn], hv[3], fb[0][jn] * hv[2]);
        }
#pragma unroll
        for (int jm = 0; jm < P; ++jm)
#pragma unroll
          for (int jn = 0; jn < P; ++jn) {
            double& acc = ring[(r + jm) % P][jn - jm + P - 1];
            acc = fma(fb[3][jm], u1[jn], fma(fb[2][jm], u0[jn], acc));
          }
      }
      // row m2 = e2 is final: write its 2P-1 columns, recycle the ring row
      if (valid) flush(e2, ring[r], reinterpret_cast<const int64_t*>(wst + NWT));
#pragma unroll
      for (int k = 0; k < W; ++k) ring[r][k] = 0.0;
    }
  }
  // trailing rows m2 in [K2, K2 + P - 1) (their last element is K2 - 1)
  if (valid && e_hi == K2) {
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const int64_t m2 = K2 - 1 + t;
      const int slot = (int)((m2 - e_lo) % P);
#pragma unroll
      const int64_t rp2 = a.pat.rp[L][m2];
      const int64_t meta[3] = {rp2, a.pat.rp[L][m2 + 1] - rp2, a.pat.cl[L][rp2]};
#pragma unroll
      for (int s = 0; s < P; ++s)
        if (s == slot) flush(m2, ring[s], meta);
    }
  }
}

// ---- 3D three-pass path (orders whose stage-1/2 tile would be < 4 rows) ---
//
// At p >= 5 the fused stage-1/2 kernel only fits 2 x 2 (p = 5) or 1 x 1
// (p = 6) row tiles: every tile re-reads and re-contracts a (T+p-1)^2 region
// for T^2 rows (9x / 36x redundant) and its MMA tiles are nearly empty.  The
// three-pass path splits the two contractions (the reference's recursion,
// sumfac.py:200-213, one direction per pass):
//   pass A  asm2_stage1 over the rows (y, z) of a chunk of z layers:
//           G_g[(z,y)][s0] = Σ_{b∈g} Σ_x F_b W0^{v0(b)}            (DMMA, -> HBM chunk)
//   pass B  asm_ysweep: one thread per (s0, z, stage-2 group h) sweeps y with
//           the ring of P rows x (2P-1) columns of asm_sweep, exact band
//           sparsity on DFMA:  H_h[s1][s0] = Σ_{g∈h} Σ_y W1^{v1(g)} G_g  -> HBM
//   pass C  asm_sweep<3> (z), as for the two-pass path.
struct AsmYArgs {
  TabArgs tab;
  const double* G;      // chunk, sweep-blocked [NS0 blocks][layer·K1 + e1][Q][ng][128]
  double* H;            // sweep-blocked [pair blocks][e2 - e_lo][Q][nh][128]
  const double* w1g;    // per y element: separable factors [Q][wB^0 | wB^1 | B^0 | B^1][PP] (+ 4 unused)
  int64_t NS0;
  int64_t NE_G;         // layers in the chunk x K1
  int64_t zrel0;        // z point of the chunk's first layer relative to H's first point
  int64_t NE_H;
  int ng, nh;
  int h_g0[4], h_ng[4];
  int vmap[4][4];       // [h][v1]: group (relative to h_g0[h]) holding y variant v1, -1: none
};

// Pipeline of the y sweep: NSY element stages, NSY - 1 elements ahead (the
// per-stage tiles are small — Q bulk copies of hng·1 KB — so the copy
// latency, not the DRAM stream count, is what the ring has to cover).
constexpr int NSY = 2, DY = NSY - 1;
template <int P, int Q>
struct SYCfg {
  using C = S3Cfg<P, Q>;
  static constexpr size_t SMEM = (size_t)NSY * (C::HST + C::NWR) * sizeof(double) + NSY * sizeof(uint64_t);
};

// TH / ET: the stage-2 group has y variants with a trial (θ) / test (η)
// derivative; absent ones are compiled out (u_η = Σ_θ (wB^θ) G_{θ+2η},
// ring += Σ_η B^η u_η).
template <int P, int Q, bool TH, bool ET>
__device__ __forceinline__ void ysweep_body(const AsmYArgs& a, double* s3) {
  using C = S3Cfg<P, Q>;
  constexpr int W = 2 * P - 1, NWR = C::NWR, PP = C::PP;
  double* hst = s3;                    // [NSY][Q][hng][NT3]
  double* w2s = s3 + NSY * C::HST;     // [NSY][NWR]
  uint64_t* bars = reinterpret_cast<uint64_t*>(w2s + NSY * NWR);
  const int tid = threadIdx.x;
  // h is the slowest grid index: co-resident CTAs then run the same
  // specialisation (h fastest measured 2x slower: instruction-cache misses)
  const int64_t sb = blockIdx.x;
  const int zl = blockIdx.y, h = blockIdx.z;
  const int hng = a.h_ng[h], g0 = a.h_g0[h];
  const int64_t s0 = sb * NT3 + tid;
  const bool valid = s0 < a.NS0;
  const int K1 = a.tab.K[1];
  const int64_t zrel = a.zrel0 + zl;
  const int64_t ez = zrel / Q;
  const int qz = (int)(zrel % Q);
  int vm[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) vm[v] = a.vmap[h][v];
  double ring[P][W];
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k < W; ++k) ring[r][k] = 0.0;
  // row m1 is final: its 2P-1 slots s1 = m1·W + k of this thread's s0
  // sweep_offset(sp) = (sp / 128)·S + c + sp % 128 with S = NE·Q·nh·128 and
  // c = ((ez·Q + qz)·nh + h)·128; consecutive slots advance sp by NS0
  const int64_t hS = a.NE_H * Q * a.nh * kSweepBlock;
  double* const hc = a.H + ((ez * Q + qz) * a.nh + h) * kSweepBlock;
  const int ns_blk = (int)(a.NS0 / kSweepBlock), ns_rem = (int)(a.NS0 % kSweepBlock);
  auto flush = [&](int64_t m1, const double* row) {
    const int64_t sp0 = (m1 * W) * a.NS0 + s0;
    int64_t blk = sp0 / kSweepBlock;
    int lo = (int)(sp0 % kSweepBlock);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      hc[blk * hS + lo] = row[k];
      lo += ns_rem;
      const int carry = lo >= kSweepBlock ? 1 : 0;
      lo -= carry * kSweepBlock;
      blk += ns_blk + carry;
    }
  };
  const unsigned qbytes = (unsigned)(hng * NT3 * sizeof(double));
  const unsigned wbytes = (unsigned)(NWR * sizeof(double));
  const double* gblock = a.G + ((sb * a.NE_G + (int64_t)zl * K1) * Q * a.ng + g0) * NT3;
  auto issue = [&](int e1) {  // one thread
    if (e1 >= K1) return;
    const int stg = e1 % NSY;
    dev::mbar_expect_tx(bars + stg, Q * qbytes + wbytes);
#pragma unroll
    for (int q = 0; q < Q; ++q)
      dev::bulk_load(hst + stg * C::HST + q * hng * NT3, gblock + ((int64_t)e1 * Q + q) * a.ng * NT3, qbytes,
                     bars + stg);
    dev::bulk_load(w2s + stg * NWR, a.w1g + (int64_t)e1 * NWR, wbytes, bars + stg);
  };
  if (tid < NSY) dev::mbar_init(bars + tid, 1);
  dev::fence_mbar_init();
  __syncthreads();
  if (tid == 0)
    for (int e = 0; e < DY; ++e) issue(e);
  for (int eb = 0; eb < K1; eb += P) {
#pragma unroll
    for (int r = 0; r < P; ++r) {  // ring row of element e1 is static: r
      const int e1 = eb + r;
      if (e1 >= K1) break;
      __syncthreads();  // stage (e1 + DY) % NSY was last read for element e1 - 1
      if (tid == 0) {
        dev::fence_proxy_async();
        issue(e1 + DY);
      }
      const int stg = e1 % NSY;
      dev::mbar_wait(bars + stg, (unsigned)((e1 / NSY) & 1));
      const double* hcol = hst + stg * C::HST + tid;
      const double* wst = w2s + stg * NWR;
      // (the point loop stays rolled: P·Q unrolled copies of the update
      // overflow the instruction cache — `no_inst` was the top stall)
#pragma unroll 1
      for (int q = 0; q < Q; ++q) {
        double hv[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const bool used = (TH || !(v & 1)) && (ET || !(v & 2));
          hv[v] = used && vm[v] >= 0 ? hcol[(q * hng + vm[v]) * NT3] : 0.0;
        }
        double fb[4][P];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          if ((f == 1 && !TH) || (f == 3 && !ET)) continue;
#pragma unroll
          for (int j = 0; j < P; j += 2) {
            if (j + 1 < P) {
              const double2 t = *reinterpret_cast<const double2*>(wst + (q * 4 + f) * PP + j);
              fb[f][j] = t.x;
              fb[f][j + 1] = t.y;
            } else {
              fb[f][j] = wst[(q * 4 + f) * PP + j];
            }
          }
        }
        double u0[P], u1[P];
#pragma unroll
        for (int jn = 0; jn < P; ++jn) {
          u0[jn] = TH ? fma(fb[1][jn], hv[1], fb[0][jn] * hv[0]) : fb[0][jn] * hv[0];
          if (ET) u1[jn] = TH ? fma(fb[1][jn], hv[3], fb[0][jn] * hv[2]) : fb[0][jn] * hv[2];
        }
#pragma unroll
        for (int jm = 0; jm < P; ++jm)
#pragma unroll
          for (int jn = 0; jn < P; ++jn) {
            double& acc = ring[(r + jm) % P][jn - jm + P - 1];
            if (ET) acc = fma(fb[3][jm], u1[jn], fma(fb[2][jm], u0[jn], acc));
            else acc = fma(fb[2][jm], u0[jn], acc);
          }
      }
      if (valid) flush(e1, ring[r]);
#pragma unroll
      for (int k = 0; k < W; ++k) ring[r][k] = 0.0;
    }
  }
  // trailing rows m1 in [K1, K1 + P - 1)
  if (valid) {
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const int64_t m1 = K1 - 1 + t;
      const int slot = (int)(m1 % P);
#pragma unroll
      for (int s = 0; s < P; ++s)
        if (s == slot) flush(m1, ring[s]);
    }
  }
}

template <int P, int Q>
__global__ void __launch_bounds__(NT3, 2) asm_ysweep(const AsmYArgs a) {
  extern __shared__ __align__(16) double s3y[];
  const int h = blockIdx.z;
  const bool th = a.vmap[h][1] >= 0 || a.vmap[h][3] >= 0;
  const bool et = a.vmap[h][2] >= 0 || a.vmap[h][3] >= 0;
  if (th && et) ysweep_body<P, Q, true, true>(a, s3y);
  else if (th) ysweep_body<P, Q, true, false>(a, s3y);
  else if (et) ysweep_body<P, Q, false, true>(a, s3y);
  else ysweep_body<P, Q, false, false>(a, s3y);
}

// ---------------------------------------------------------------- 2D -------

struct Asm2Args {
  AsmPlan plan;
  TabArgs tab;
  double* G;       // sweep-blocked [NS0 blocks][K1][Q][ng][128]
  int64_t NS0;
  int64_t NE;      // elements of the last direction (K1)
  int nt0;         // row tiles in x
  int yc;          // y points per CTA (multiple of the TMA box height YS)
  const double* Wg;  // [nt0][W0T] band tables, built once per assembly (asm2_tables_kernel)
  int64_t X1;      // rows (y points) to contract: 2D the y points; 3D three-pass a chunk of
                   // z layers flattened with y (row = zl·X1d + y, NE = layers·K1)
  int64_t ytma0;   // TMA row of row 0 (3D three-pass: the chunk's first layer; 2D: 0)
};

// The 2D tiles' band tables, one block per row tile, built once per
// assembly: the stage-1 CTAs (several per tile, one per y chunk) then
// bulk-copy theirs instead of recomputing it.
template <int P, int Q, int T, bool SYM = false>
__global__ void asm2_tables_kernel(const TabArgs tab, double* Wg) {
  using C = A3Cfg<P, Q, T, SYM>;
  const int a0 = blockIdx.x * T;
  fill_band_table<P, Q, T, false, SYM>(Wg + (size_t)blockIdx.x * C::W0T, tab, 0, a0, (a0 - (P - 1)) * Q);
}

// 2D stage 1 as a dense banded GEMM on DMMA (the 3D stage-1 structure):
// one CTA per (T-row tile in x, chunk of y points); the tile's band table
// W0[v][x][slot] is built once and reused for every y block; coefficient
// boxes of A2_YS y rows x the tile's x region (all planes) stream in by
// TMA, double-buffered.  G_g[y][s0] = Σ_{b∈g} Σ_x F_b[y][x] W0^{v0(b)}[x][s0].
constexpr int A2_YS = 64, A2_NT = 512, A2_NW = 16;
template <int P, int Q, int T, int YS = A2_YS>
struct A2Cfg {
  using B = A3Cfg<P, Q, T>;
  static constexpr size_t fbox(int npl) { return ((size_t)npl * YS * B::XR + 4 + 15) & ~size_t(15); }
  static constexpr size_t smem(int npl) { return (2 * fbox(npl) + B::W0T) * sizeof(double) + 32; }
};

template <int P, int Q, int T, int YS = A2_YS>
__global__ void __launch_bounds__(A2_NT) asm2_stage1(const Asm2Args a, const __grid_constant__ CUtensorMap fmap,
                                                     int nplanes) {
  using C = A3Cfg<P, Q, T>;
  using C2 = A2Cfg<P, Q, T, YS>;
  constexpr int A2_YS = YS;  // (shadows the 2D default inside this kernel)
  constexpr int PT = C::PT, PTP = C::PTP, XR = C::XR, XK = C::XK, SP = C::SP, W = C::W, SR = C::SR;
  constexpr int KL = max_ksteps<P, Q, T>(PTP / 8, XK / 4);
  constexpr int NYB = A2_YS / 8, NST = PTP / 8;
  extern __shared__ __align__(128) double sm[];
  const AsmPlan& pl = a.plan;
  const size_t fb = C2::fbox(nplanes);
  double* Fs = sm;                 // [2][nplanes][A2_YS][XR]
  double* W0 = Fs + 2 * fb;        // [4][XK][SP]
  uint64_t* bar = reinterpret_cast<uint64_t*>(W0 + C::W0T);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, m4 = lane & 3;
  const int a0 = (blockIdx.x % a.nt0) * T;
  const int xb0 = (a0 - (P - 1)) * Q;
  const int64_t X1 = a.X1;
  const int64_t y_lo = (int64_t)(blockIdx.x / a.nt0) * a.yc;
  const int64_t y_hi = min64(X1, y_lo + a.yc);
  const int nstage = (int)((y_hi - y_lo + A2_YS - 1) / A2_YS);
  const unsigned fbytes = (unsigned)((size_t)nplanes * A2_YS * XR * sizeof(double));
  for (int b = 0; b < 2; ++b)
    for (size_t i = (size_t)nplanes * A2_YS * XR + tid; i < fb; i += A2_NT) Fs[b * fb + i] = 0.0;
  if (tid < 3) dev::mbar_init(bar + tid, 1);
  dev::fence_mbar_init();
  dev::fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    if (a.Wg) {
      constexpr unsigned wbytes = (unsigned)(C::W0T * sizeof(double));
      dev::mbar_expect_tx(bar + 2, wbytes);
      dev::bulk_load(W0, a.Wg + (size_t)(blockIdx.x % a.nt0) * C::W0T, wbytes, bar + 2);
    }
    for (int i = 0; i < 2 && i < nstage; ++i) {
      dev::mbar_expect_tx(bar + i, fbytes);
      dev::tma_load_4d(Fs + i * fb, &fmap, bar + i, xb0, (int)(a.ytma0 + y_lo + i * A2_YS), 0, 0);
    }
  }
  if (a.Wg) {
    dev::mbar_wait(bar + 2, 0u);
  } else {
    fill_band_table<P, Q, T, false>(W0, a.tab, 0, a0, xb0);
    __syncthreads();
  }
  for (int i = 0; i < nstage; ++i) {
    const int buf = i & 1;
    dev::mbar_wait(bar + buf, (unsigned)((i >> 1) & 1));
    const double* Fb0 = Fs + buf * fb;
    const int64_t y0 = y_lo + (int64_t)i * A2_YS;
    for (int t = warp; t < NYB * NST; t += A2_NW) {
      const int yb = t / NST, st = t % NST;
      int k_lo, k_hi;
      slot_tile_ksteps<P, Q, T>(st, XK / 4, k_lo, k_hi);
      const double* Fy = Fb0 + (yb * 8 + g8) * XR + m4 + k_lo * 4;
      const double* Wk = W0 + (m4 + k_lo * 4) * SP + st * 8 + g8;
      const int64_t y = y0 + yb * 8 + g8;
      const int s = st * 8 + 2 * m4;
      const int64_t gs0 = (int64_t)(a0 + s / SR) * W + s % SR;
      const int64_t gs0b = (int64_t)(a0 + (s + 1) / SR) * W + (s + 1) % SR;
      const bool ok0 = y < y_hi && s < PT && s % SR < W && gs0 < a.NS0;
      const bool ok1 = y < y_hi && s + 1 < PT && (s + 1) % SR < W && gs0b < a.NS0;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int b = 0; b < kMaxBlocks; ++b) {
        if (b >= pl.nb) break;
        const double* Fb = Fy + pl.b_plane[b] * (A2_YS * XR);
        const double* Wb = Wk + pl.b_v0[b] * (XK * SP);
#pragma unroll
        for (int kk = 0; kk < KL; ++kk)
          if (k_lo + kk < k_hi) dmma_a(d0, d1, Fb[kk * 4], Wb[kk * 4 * SP]);
        if (b + 1 == pl.nb || pl.b_g[b + 1] != pl.b_g[b]) {
          const int gq = (int)(y % Q), h = pl.b_g[b];
          if (ok0) a.G[sweep_offset(gs0, y / Q, gq, h, a.NE, Q, pl.ng)] = d0;
          if (ok1) a.G[sweep_offset(gs0b, y / Q, gq, h, a.NE, Q, pl.ng)] = d1;
          d0 = d1 = 0.0;
        }
      }
    }
    __syncthreads();
    if (tid == 0 && i + 2 < nstage) {
      dev::fence_proxy_async();
      dev::mbar_expect_tx(bar + buf, fbytes);
      dev::tma_load_4d(Fs + buf * fb, &fmap, bar + buf, xb0, (int)(a.ytma0 + y0 + 2 * A2_YS), 0, 0);
    }
  }
}

// Pass A kernel of the three-pass path: asm2_stage1's banded GEMM with
//   * TMA boxes of 16 rows (the 7-plane regions of p = 5, 6 then fit twice),
//     row pitch XB ≡ 4 or 12 (mod 16) doubles so the A-fragment loads (8
//     rows x 4 columns) are bank-conflict-free (the plain region width 54 /
//     50 gave 35 % conflict wavefronts);
//   * one warp per (slot tile, half of the blocks — whole groups) for both y
//     tiles of the box: every warp has a task in every stage (12-14 tasks on
//     16 warps left a quarter of the CTA idle at the stage barrier) and each
//     W fragment feeds two DMMAs (3 fragment loads per 2 MMAs).
template <int P, int Q, int T, bool SYM = false>
struct AXCfg {
  using B = A3Cfg<P, Q, T, SYM>;
  static constexpr int YS = 16;
  static constexpr int xb() {
    int b = B::XK;  // >= the region width, covers the k-step tail
    while (b % 16 != 4 && b % 16 != 12) b += 2;
    return b;
  }
  static constexpr int XB = xb();
  static constexpr int NTASK = (B::PTP / 8) * 2;  // (slot tile, half of the blocks), both y tiles
  static constexpr int NW = NTASK < 32 ? NTASK : 32;
  static constexpr int NT = NW * 32;
  static constexpr size_t fbox(int npl) { return ((size_t)npl * YS * XB + 4 + 15) & ~size_t(15); }
  static constexpr size_t smem(int npl) { return (2 * fbox(npl) + B::W0T) * sizeof(double) + 32; }
  static_assert(XB <= 256 && XB >= B::XK, "TMA box / k-step tail");
};

template <int P, int Q, int T, bool SYM = false>
__global__ void __launch_bounds__(AXCfg<P, Q, T, SYM>::NT) asm3_xpass(const Asm2Args a,
                                                                       const __grid_constant__ CUtensorMap fmap,
                                                                       int nplanes) {
  using C = A3Cfg<P, Q, T, SYM>;
  using CX = AXCfg<P, Q, T, SYM>;
  constexpr int PT = C::PT, PTP = C::PTP, XK = C::XK, SP = C::SP, W = C::W, SR = C::SR;
  constexpr int YS = CX::YS, XB = CX::XB, NT = CX::NT, NW = CX::NW;
  constexpr int KL = max_ksteps<P, Q, T, SYM>(PTP / 8, XK / 4);
  constexpr int NST = PTP / 8;
  extern __shared__ __align__(128) double sm[];
  const AsmPlan& pl = a.plan;
  const size_t fb = CX::fbox(nplanes);
  double* Fs = sm;                 // [2][nplanes][YS][XB]
  double* W0 = Fs + 2 * fb;        // [4][XK][SP]
  uint64_t* bar = reinterpret_cast<uint64_t*>(W0 + C::W0T);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, m4 = lane & 3;
  const int a0 = (blockIdx.x % a.nt0) * T;
  const int xb0 = (a0 - (P - 1)) * Q;
  const int64_t X1 = a.X1;
  const int64_t y_lo = (int64_t)(blockIdx.x / a.nt0) * a.yc;
  const int64_t y_hi = min64(X1, y_lo + a.yc);
  const int nstage = (int)((y_hi - y_lo + YS - 1) / YS);
  const unsigned fbytes = (unsigned)((size_t)nplanes * YS * XB * sizeof(double));
  for (int b = 0; b < 2; ++b)
    for (size_t i = (size_t)nplanes * YS * XB + tid; i < fb; i += NT) Fs[b * fb + i] = 0.0;
  if (tid < 3) dev::mbar_init(bar + tid, 1);
  dev::fence_mbar_init();
  dev::fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    constexpr unsigned wbytes = (unsigned)(C::W0T * sizeof(double));
    dev::mbar_expect_tx(bar + 2, wbytes);
    dev::bulk_load(W0, a.Wg + (size_t)(blockIdx.x % a.nt0) * C::W0T, wbytes, bar + 2);
    for (int i = 0; i < 2 && i < nstage; ++i) {
      dev::mbar_expect_tx(bar + i, fbytes);
      dev::tma_load_4d(Fs + i * fb, &fmap, bar + i, xb0, (int)(a.ytma0 + y_lo + i * YS), 0, 0);
    }
  }
  dev::mbar_wait(bar + 2, 0u);
  for (int i = 0; i < nstage; ++i) {
    const int buf = i & 1;
    dev::mbar_wait(bar + buf, (unsigned)((i >> 1) & 1));
    const double* Fb0 = Fs + buf * fb;
    const int64_t y0 = y_lo + (int64_t)i * YS;
    for (int t = warp; t < CX::NTASK; t += NW) {
      const int half = t & 1, st = t >> 1;
      int k_lo, k_hi;
      slot_tile_ksteps<P, Q, T, SYM>(st, XK / 4, k_lo, k_hi);
      const double* Fy = Fb0 + g8 * XB + m4 + k_lo * 4;  // y tile 0; tile 1 at + 8·XB
      const double* Wk = W0 + (m4 + k_lo * 4) * SP + st * 8 + g8;
      const int s = st * 8 + 2 * m4;
      const int64_t gs0 = (int64_t)(a0 + s / SR) * W + s % SR;
      const int64_t gs0b = (int64_t)(a0 + (s + 1) / SR) * W + (s + 1) % SR;
      const bool sok0 = s < PT && s % SR < W && gs0 < a.NS0;
      const bool sok1 = s + 1 < PT && (s + 1) % SR < W && gs0b < a.NS0;
      // G offsets of group 0 (sweep-blocked; groups advance by 128 doubles), per y tile
      int64_t off0[2], off1[2];
      bool yok[2];
#pragma unroll
      for (int jy = 0; jy < 2; ++jy) {
        const int64_t y = y0 + jy * 8 + g8;
        yok[jy] = y < y_hi;
        off0[jy] = sweep_offset(gs0, y / Q, (int)(y % Q), 0, a.NE, Q, pl.ng);
        off1[jy] = sweep_offset(gs0b, y / Q, (int)(y % Q), 0, a.NE, Q, pl.ng);
      }
      const int b_lo = half ? pl.half_b : 0, b_hi = half ? pl.nb : pl.half_b;
      double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll
      for (int b = 0; b < kMaxBlocks; ++b) {
        if (b < b_lo) continue;
        if (b >= b_hi) break;
        const double* Fb = Fy + pl.b_plane[b] * (YS * XB);
        const double* Wb = Wk + pl.b_v0[b] * (XK * SP);
#pragma unroll
        for (int kk = 0; kk < KL; ++kk)
          if (k_lo + kk < k_hi) {
            const double w = Wb[kk * 4 * SP];
            dmma_a(c0[0], c0[1], Fb[kk * 4], w);
            dmma_a(c1[0], c1[1], Fb[kk * 4 + 8 * XB], w);
          }
        if (b + 1 == pl.nb || pl.b_g[b + 1] != pl.b_g[b]) {
          const int hoff = pl.b_g[b] * kSweepBlock;
          if (sok0 && yok[0]) a.G[off0[0] + hoff] = c0[0];
          if (sok1 && yok[0]) a.G[off1[0] + hoff] = c0[1];
          if (sok0 && yok[1]) a.G[off0[1] + hoff] = c1[0];
          if (sok1 && yok[1]) a.G[off1[1] + hoff] = c1[1];
          c0[0] = c0[1] = c1[0] = c1[1] = 0.0;
        }
      }
    }
    __syncthreads();
    if (tid == 0 && i + 2 < nstage) {
      dev::fence_proxy_async();
      dev::mbar_expect_tx(bar + buf, fbytes);
      dev::tma_load_4d(Fs + buf * fb, &fmap, bar + buf, xb0, (int)(a.ytma0 + y0 + 2 * YS), 0, 0);
    }
  }
}

// ---- host side ----------------------------------------------------------------

// Row tile per direction of the 3D stage-1/2 kernel: the largest of 4, 2, 1
// whose shared-memory plan fits (0 = none).
template <int P>
constexpr int kWideTile = P == 2 ? 10 : P == 3 ? 6 : 0;

template <int P>
int asm3_tile(const AsmPlan& pl, int nplanes) {
  // low orders: wider tiles so both stages have >= 16 warp tasks (and, for
  // p = 3, a region of whole MMA row tiles); else the largest of 4, 2, 1
  constexpr int wide = kWideTile<P>;
  // (the TMA box is XR points wide: its rows must be 16-byte multiples, which
  // rules out 1-row tiles at odd p)
  if constexpr (wide > 0)
    if (A3Cfg<P, P, wide>::smem(nplanes, pl.ng) <= 232448 && A3Cfg<P, P, wide>::XR % 2 == 0) return wide;
  if (A3Cfg<P, P, 4>::smem(nplanes, pl.ng) <= 232448 && A3Cfg<P, P, 4>::XR % 2 == 0) return 4;
  if (A3Cfg<P, P, 2>::smem(nplanes, pl.ng) <= 232448 && A3Cfg<P, P, 2>::XR % 2 == 0) return 2;
  if (A3Cfg<P, P, 1>::smem(nplanes, pl.ng) <= 232448 && A3Cfg<P, P, 1>::XR % 2 == 0) return 1;
  return 0;
}

int asm3_tile_for(int P, const AsmPlan& pl, int nplanes) {
  switch (P) {
    case 2: return asm3_tile<2>(pl, nplanes);
    case 3: return asm3_tile<3>(pl, nplanes);
    case 4: return asm3_tile<4>(pl, nplanes);
    case 5: return asm3_tile<5>(pl, nplanes);
    case 6: return asm3_tile<6>(pl, nplanes);
    default: return 0;
  }
}

// row tile of the 2D stage-1 kernel: the largest of 8, 4, 2, 1 that fits
template <int P>
int asm2_tile(int nplanes) {
  // (TMA box rows of XR points must be 16-byte multiples)
  if (A2Cfg<P, P, 8>::smem(nplanes) <= 232448 && A3Cfg<P, P, 8>::XR % 2 == 0) return 8;
  if (A2Cfg<P, P, 4>::smem(nplanes) <= 232448 && A3Cfg<P, P, 4>::XR % 2 == 0) return 4;
  if (A2Cfg<P, P, 2>::smem(nplanes) <= 232448 && A3Cfg<P, P, 2>::XR % 2 == 0) return 2;
  if (A2Cfg<P, P, 1>::smem(nplanes) <= 232448 && A3Cfg<P, P, 1>::XR % 2 == 0) return 1;
  return 0;
}

// Upper bound over the row tiles T of the band-table store (bytes).
template <int P>
size_t asm2_tables_bytes(int64_t nfn0) {
  const size_t t8 = (size_t)ceil_div(nfn0, 8) * A3Cfg<P, P, 8>::W0T;
  const size_t t6 = (size_t)ceil_div(nfn0, 6) * A3Cfg<P, P, 6>::W0T;  // x-pass kernel (p >= 5)
  const size_t t4 = (size_t)ceil_div(nfn0, 4) * A3Cfg<P, P, 4>::W0T;
  const size_t t2 = (size_t)ceil_div(nfn0, 2) * A3Cfg<P, P, 2>::W0T;
  const size_t t1 = (size_t)nfn0 * A3Cfg<P, P, 1>::W0T;
  size_t m = t8 > t4 ? t8 : t4;
  m = m > t6 ? m : t6;
  m = m > t2 ? m : t2;
  m = m > t1 ? m : t1;
  return m * sizeof(double);
}

size_t asm2_tables_bytes_for(int P, int64_t nfn0) {
  switch (P) {
    case 2: return asm2_tables_bytes<2>(nfn0);
    case 3: return asm2_tables_bytes<3>(nfn0);
    case 4: return asm2_tables_bytes<4>(nfn0);
    case 5: return asm2_tables_bytes<5>(nfn0);
    case 6: return asm2_tables_bytes<6>(nfn0);
    default: return 0;
  }
}

int asm2_tile_for(int P, int nplanes) {
  switch (P) {
    case 2: return asm2_tile<2>(nplanes);
    case 3: return asm2_tile<3>(nplanes);
    case 4: return asm2_tile<4>(nplanes);
    case 5: return asm2_tile<5>(nplanes);
    case 6: return asm2_tile<6>(nplanes);
    default: return 0;
  }
}

struct AsmShape {
  FusedShape fs;
  AsmPlan plan;
  int64_t zpts;  // z points held by the coefficient planes (slab or grid)
  int nplanes;
};

bool three_pass_available(const AsmShape& s);

bool asm_shape(const igs_problem* p, const Dims& D, AsmShape* out) {
  AsmShape s;
  if (p->d != 2 && p->d != 3) return false;
  if ((p->slab_lo || p->slab_hi) && p->d != 3) return false;  // slab assembly: 3D fused only
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
  s.zpts = (p->slab_lo || p->slab_hi) ? (int64_t)(p->slab_hi - p->slab_lo) * s.fs.k : s.fs.npt[d - 1];
  s.nplanes = p->n_planes;
  // tables must hold the derivative levels the blocks use
  for (int k = 0; k < d; ++k)
    if (p->trial[k].max_deriv < 1) {
      for (int b = 0; b < s.plan.nb; ++b)
        if (s.plan.b_v0[b] != 0) return false;
    }
  if (s.fs.p < 2 || s.fs.p > 6 || s.fs.k != s.fs.p) return false;
  // a stage-1/2 tile must fit, or the three-pass path serves the order
  if (d == 3 && asm3_tile_for(s.fs.p, s.plan, p->n_planes) == 0 && !three_pass_available(s)) return false;
  if (d == 2 && asm2_tile_for(s.fs.p, p->n_planes) == 0) return false;
  // TMA: 16-byte aligned rows and plane stride
  if ((s.fs.npt[0] * 8) % 16 != 0 || (p->plane_stride * 8) % 16 != 0 || p->n_planes > 256) return false;
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

#include "asm3_sym.cuh"
#include "asm2_sym.cuh"

// The one-pass symmetric kernel serves this problem (3D, p <= 4, A = Aᵀ).
bool sym_eligible(const igs_problem* p, const AsmShape& s) {
  // p = 3 keeps the two-pass path (measured faster: the 5-wide band does not
  // fill the 8-wide MMA tiles of the one-pass kernel)
  return s.fs.d == 3 && (s.fs.p == 2 || s.fs.p == 4) && problem_symmetric(p) &&
         sym_fits_for(s.fs.p, s.plan, p->n_planes, s.fs.nfn[2]);
}

// 3D three-pass path (p >= 5): pass-A row tile (TMA boxes of 16 rows), z
// layers per G chunk (G chunk <= ~1.5 GB) and the workspace behind H and the
// z records: [y records][G chunk][pass-A band tables].
constexpr int A3P_YS = 16;
struct ThreePass {
  bool on;
  int T;                // pass-A row tile in x
  int64_t nzc;          // z layers per chunk
  size_t w1_doubles, g_doubles, wg_doubles;
};

template <int P>
int three_pass_tile(int nplanes) {
  if (AXCfg<P, P, 6>::smem(nplanes) <= 232448) return 6;
  if (AXCfg<P, P, 4>::smem(nplanes) <= 232448) return 4;
  if (AXCfg<P, P, 2>::smem(nplanes) <= 232448) return 2;
  // (a 1-row tile starts its TMA box at x point (t - P + 1)·P: odd, i.e. not
  // 16-byte aligned, for odd p and odd t)
  if (P % 2 == 0 && AXCfg<P, P, 1>::smem(nplanes) <= 232448) return 1;
  return 0;
}

template <int P>
size_t three_pass_table_doubles(int T, int64_t nfn0) {
  switch (T) {
    case 6: return (size_t)ceil_div(nfn0, 6) * A3Cfg<P, P, 6>::W0T;
    case 4: return (size_t)ceil_div(nfn0, 4) * A3Cfg<P, P, 4>::W0T;
    case 2: return (size_t)ceil_div(nfn0, 2) * A3Cfg<P, P, 2>::W0T;
    default: return (size_t)nfn0 * A3Cfg<P, P, 1>::W0T;
  }
}

ThreePass three_pass_plan(const AsmShape& s) {
  ThreePass t{};
  if (s.fs.d != 3 || s.fs.p < 3) return t;
  for (int h = 0; h < s.plan.nh; ++h)
    if (s.plan.h_ng[h] > 4) return t;
  if (s.plan.nh > 4) return t;
  t.T = s.fs.p == 3 ? three_pass_tile<3>(s.nplanes) : s.fs.p == 4 ? three_pass_tile<4>(s.nplanes)
        : s.fs.p == 5 ? three_pass_tile<5>(s.nplanes) : three_pass_tile<6>(s.nplanes);
  if (t.T == 0) return t;
  const int W = 2 * s.fs.p - 1;
  const size_t s0pad = (size_t)ceil_div(s.fs.nfn[0] * W, (int64_t)kSweepBlock) * kSweepBlock;
  const size_t per_layer = s0pad * s.fs.npt[1] * s.plan.ng;  // doubles of G per z layer
  int64_t nzc = (int64_t)(187500000 / per_layer);            // ~1.5 GB
  if (nzc < 1) nzc = 1;
  if (nzc > s.zpts) nzc = s.zpts;
  t.nzc = nzc;
  t.g_doubles = per_layer * nzc;
  const int PP = (s.fs.p + 1) & ~1;
  t.w1_doubles = ((size_t)s.fs.nel[1] * (s.fs.k * 4 * PP + 4) + 1) & ~size_t(1);
  t.wg_doubles = s.fs.p == 3   ? three_pass_table_doubles<3>(t.T, s.fs.nfn[0])
                 : s.fs.p == 4 ? three_pass_table_doubles<4>(t.T, s.fs.nfn[0])
                 : s.fs.p == 5 ? three_pass_table_doubles<5>(t.T, s.fs.nfn[0])
                               : three_pass_table_doubles<6>(t.T, s.fs.nfn[0]);
  t.on = true;
  return t;
}

bool three_pass_available(const AsmShape& s) { return three_pass_plan(s).on; }

size_t asm_workspace(const AsmShape& s) {
  const int W = 2 * s.fs.p - 1;
  auto padded = [](int64_t n) { return (size_t)ceil_div(n, (int64_t)kSweepBlock) * kSweepBlock; };
  if (s.fs.d == 3) {
    const ThreePass tp = three_pass_plan(s);
    const size_t extra = tp.on ? (tp.w1_doubles + tp.g_doubles + tp.wg_doubles + 8) * sizeof(double) : 0;
    return padded((s.fs.nfn[1] * W) * (s.fs.nfn[0] * W)) * s.zpts * s.plan.nh * sizeof(double) +
           (size_t)s.fs.nel[2] * (s.fs.k * 4 * (s.fs.p + 1) + 4) * sizeof(double) + 512 + extra;
  }
  return padded(s.fs.nfn[0] * W) * s.fs.npt[1] * s.plan.ng * sizeof(double) +
         ((size_t)s.fs.nel[1] * (s.fs.k * 4 * (s.fs.p + 1) + 4) + 2) * sizeof(double) +
         asm2_tables_bytes_for(s.fs.p, s.fs.nfn[0]) + 512;
}

// z elements the row range needs (rows of DoF layers [m2a, m2b] are summed
// over elements [m2a - P + 1, m2b]) and the slab origin of the planes.
struct ZRange {
  int e_lo, e_hi;   // elements to contract
  int sl, sh;       // elements held by the coefficient planes
};

igs_status z_range(const igs_problem* p, const AsmShape& s, int64_t row_lo, int64_t row_hi, ZRange* z) {
  const int P = s.fs.p, K2 = (int)s.fs.nel[2];
  const int64_t layer = s.fs.nfn[0] * s.fs.nfn[1];
  const int64_t m2a = row_lo / layer, m2b = (row_hi - 1) / layer;
  z->e_lo = (int)max64(0, m2a - P + 1);
  z->e_hi = (int)min64(K2, m2b + 1);
  const bool slab = p->slab_lo || p->slab_hi;
  z->sl = slab ? p->slab_lo : 0;
  z->sh = slab ? p->slab_hi : K2;
  if (z->e_lo < z->sl || z->e_hi > z->sh)
    return fail(IGS_EARG, "row range needs coefficient elements outside the slab (elements " +
                              std::to_string(z->e_lo) + ".." + std::to_string(z->e_hi) + ")");
  return IGS_OK;
}

template <int P, int Q, int T>
igs_status launch3_stage12(const igs_problem* p, const AsmShape& s, const ZRange& z, const double* planes,
                           double* H, cudaStream_t st) {
  using C = A3Cfg<P, Q, T>;
  Asm3Args a{};
  a.plan = s.plan;
  a.tab = tab_args(p);
  a.planes = planes;
  a.pstride = p->plane_stride;
  a.H = H;
  a.NS0 = s.fs.nfn[0] * C::W;
  a.NS1 = s.fs.nfn[1] * C::W;
  a.nt0 = (int)ceil_div(s.fs.nfn[0], T);
  a.nt1 = (int)ceil_div(s.fs.nfn[1], T);
  a.nplanes = p->n_planes;
  size_t smem = C::smem(a.nplanes, s.plan.ng);
  if (smem > 232448) return fail(IGS_ECAPACITY, "fused assembly tile does not fit shared memory");
  if (((uintptr_t)planes & 15) != 0) return fail(IGS_EARG, "coefficient planes must be 16-byte aligned");
  CUtensorMap fmap;
  {
    const int64_t dims[4] = {s.fs.npt[0], s.fs.npt[1], (int64_t)(z.sh - z.sl) * Q, p->n_planes};
    const unsigned box[4] = {(unsigned)C::XR, (unsigned)C::XRP, 1u, (unsigned)p->n_planes};
    IGS_TRY(planes_tensor_map(&fmap, planes, dims, p->plane_stride, box));
  }
  a.z0 = (int64_t)z.e_lo * Q;
  a.z1 = (int64_t)z.e_hi * Q;
  a.NE = z.e_hi - z.e_lo;
  a.zpl = (int64_t)z.sl * Q;
  // z chunks: the fewest (each CTA refills its band tables) whose CTAs fill
  // >= 97 % of the last wave at one CTA per SM (C3: 289 tiles -> 1 chunk)
  const int64_t tiles = (int64_t)a.nt0 * a.nt1;
  int64_t nz = 1;
  {
    double best = -1.0;
    for (int n = 1; n <= 16; ++n) {
      const double w = n * (double)tiles / 148.0;
      const double eff = w / std::ceil(w);
      if (eff >= 0.97) {
        nz = n;
        break;
      }
      if (eff > best + 1e-9) {
        best = eff;
        nz = n;
      }
    }
  }
  if (nz > a.z1 - a.z0) nz = a.z1 - a.z0;
  if (nz < 1) nz = 1;
  a.lz = (int)ceil_div(a.z1 - a.z0, nz);
  if (a.lz < 1) a.lz = 1;
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm3_stage12<P, Q, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem),
                     "smem attribute"));
  dim3 grid((unsigned)tiles, (unsigned)ceil_div(a.z1 - a.z0, a.lz));
  asm3_stage12<P, Q, T><<<grid, C::NT, smem, st>>>(a, fmap);
  IGS_LAUNCH_CHECK("asm3_stage12");
  return IGS_OK;
}

// Pass A of the three-pass path for one chunk of z layers [zc0, zc0 + nz):
// asm2_stage1 over the chunk's rows (layer-major, y fastest).
template <int P, int Q, int T, bool SYM = false>
igs_status launch3_passA(const igs_problem* p, const AsmShape& s, const CUtensorMap& fmap, const double* Wg,
                         double* G, int64_t ytma0, int64_t nz, cudaStream_t st) {
  using C = A3Cfg<P, Q, T, SYM>;
  Asm2Args a{};
  a.plan = s.plan;
  a.tab = tab_args(p);
  a.G = G;
  a.NS0 = s.fs.nfn[0] * C::W;
  a.NE = nz * s.fs.nel[1];
  a.X1 = nz * s.fs.npt[1];
  a.ytma0 = ytma0;
  a.nt0 = (int)ceil_div(s.fs.nfn[0], T);
  a.Wg = Wg;
  using CX = AXCfg<P, Q, T, SYM>;
  const size_t smem = CX::smem(p->n_planes);
  static std::atomic<int> res_cache[17];
  const int npl_key = p->n_planes < 0 ? 0 : (p->n_planes > 16 ? 16 : p->n_planes);
  int resident = res_cache[npl_key].load(std::memory_order_relaxed);
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm3_xpass<P, Q, T, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem),
                     "smem attribute"));
  if (resident <= 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, asm3_xpass<P, Q, T, SYM>, CX::NT, smem) !=
            cudaSuccess ||
        resident < 1) {
      cudaGetLastError();
      resident = 1;
    }
    res_cache[npl_key].store(resident, std::memory_order_relaxed);
  }
  // rows per CTA (whole TMA boxes): minimise waves x (boxes per CTA + 2: the
  // CTA's table copy and pipeline fill)
  const int64_t slots = 148 * (int64_t)resident, nbox = ceil_div(a.X1, (int64_t)A3P_YS);
  int64_t per_best = nbox;
  {
    int64_t best = -1;
    for (int64_t per = 1; per <= nbox && per <= 4096; ++per) {
      const int64_t ctas = a.nt0 * ceil_div(nbox, per);
      const int64_t cost = ceil_div(ctas, slots) * (per + 2);
      if (best < 0 || cost < best) {
        best = cost;
        per_best = per;
      }
    }
  }
  a.yc = (int)(per_best * A3P_YS);
  const int64_t nyc = ceil_div(a.X1, (int64_t)a.yc);
  asm3_xpass<P, Q, T, SYM><<<(unsigned)(a.nt0 * nyc), CX::NT, smem, st>>>(a, fmap, p->n_planes);
  IGS_LAUNCH_CHECK("asm3_xpass");
  return IGS_OK;
}

template <int P, int Q, int T, bool SYM>
igs_status launch3_three_pass_T(const igs_problem* p, const AsmShape& s, const ThreePass& tp, const ZRange& z,
                                TensorPat pat, const double* planes, double* H, double* extra,
                                cudaStream_t st) {
  using C = A3Cfg<P, Q, T, SYM>;
  constexpr int W = C::W;  // x slots per row (the symmetric half for SYM)
  if (((uintptr_t)planes & 15) != 0) return fail(IGS_EARG, "coefficient planes must be 16-byte aligned");
  double* w1g = extra;
  double* G = w1g + tp.w1_doubles;
  double* Wg = G + tp.g_doubles;
  const int64_t ny = s.fs.npt[1];
  CUtensorMap fmap;
  {
    // rows = (layer of the held planes, y) flattened
    const int64_t dims[4] = {s.fs.npt[0], ny * (int64_t)(z.sh - z.sl) * Q, 1, p->n_planes};
    const unsigned box[4] = {(unsigned)AXCfg<P, Q, T, SYM>::XB, (unsigned)A3P_YS, 1u, (unsigned)p->n_planes};
    IGS_TRY(planes_tensor_map(&fmap, planes, dims, p->plane_stride, box));
  }
  const TabArgs tab = tab_args(p);
  const int nt0 = (int)ceil_div(s.fs.nfn[0], T);
  asm2_tables_kernel<P, Q, T, SYM><<<(unsigned)nt0, 256, 0, st>>>(tab, Wg);
  IGS_LAUNCH_CHECK("asm2_tables_kernel");
  {
    Asm3bArgs b{};
    b.tab = tab;
    b.pat = pat;
    const int64_t n = (int64_t)tab.K[1] * S3Cfg<P, Q>::NWR;
    asm_wlast_kernel<P, Q, 2><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(b, w1g);
    IGS_LAUNCH_CHECK("asm_wlast_kernel (y)");
  }
  AsmYArgs y{};
  y.tab = tab;
  y.G = G;
  y.H = H;
  y.w1g = w1g;
  y.NS0 = s.fs.nfn[0] * W;
  y.NE_H = z.e_hi - z.e_lo;
  y.ng = s.plan.ng;
  y.nh = s.plan.nh;
  for (int h = 0; h < 4; ++h)
    for (int v = 0; v < 4; ++v) y.vmap[h][v] = -1;
  for (int h = 0; h < s.plan.nh; ++h) {
    y.h_g0[h] = s.plan.h_g0[h];
    y.h_ng[h] = s.plan.h_ng[h];
    for (int g = s.plan.h_g0[h]; g < s.plan.h_g0[h] + s.plan.h_ng[h]; ++g)
      y.vmap[h][s.plan.g_v1[g]] = g - s.plan.h_g0[h];
  }
  constexpr size_t smem3 = SYCfg<P, Q>::SMEM;
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm_ysweep<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem3),
                     "smem attribute"));
  const int64_t z0 = (int64_t)z.e_lo * Q, z1 = (int64_t)z.e_hi * Q, zpl = (int64_t)z.sl * Q;
  const unsigned nbs0 = (unsigned)ceil_div(y.NS0, (int64_t)kSweepBlock);
  for (int64_t zc = z0; zc < z1; zc += tp.nzc) {
    const int64_t nz = min64(tp.nzc, z1 - zc);
    IGS_TRY((launch3_passA<P, Q, T, SYM>(p, s, fmap, Wg, G, (zc - zpl) * ny, nz, st)));
    y.NE_G = nz * s.fs.nel[1];
    y.zrel0 = zc - z0;
    dim3 grid(nbs0, (unsigned)nz, (unsigned)s.plan.nh);
    asm_ysweep<P, Q><<<grid, NT3, smem3, st>>>(y);
    IGS_LAUNCH_CHECK("asm_ysweep");
  }
  return IGS_OK;
}

template <int P, int Q>
igs_status launch3_three_pass(const igs_problem* p, const AsmShape& s, const ThreePass& tp, const ZRange& z,
                              TensorPat pat, const double* planes, double* H, double* extra, cudaStream_t st,
                              bool sym) {
  if constexpr (P >= 3) {
    if (sym) switch (tp.T) {
      case 6: return launch3_three_pass_T<P, Q, 6, true>(p, s, tp, z, pat, planes, H, extra, st);
      case 4: return launch3_three_pass_T<P, Q, 4, true>(p, s, tp, z, pat, planes, H, extra, st);
      case 2: return launch3_three_pass_T<P, Q, 2, true>(p, s, tp, z, pat, planes, H, extra, st);
      case 1: return launch3_three_pass_T<P, Q, 1, true>(p, s, tp, z, pat, planes, H, extra, st);
      default: break;
    }
    else switch (tp.T) {
      case 6: return launch3_three_pass_T<P, Q, 6, false>(p, s, tp, z, pat, planes, H, extra, st);
      case 4: return launch3_three_pass_T<P, Q, 4, false>(p, s, tp, z, pat, planes, H, extra, st);
      case 2: return launch3_three_pass_T<P, Q, 2, false>(p, s, tp, z, pat, planes, H, extra, st);
      case 1: return launch3_three_pass_T<P, Q, 1, false>(p, s, tp, z, pat, planes, H, extra, st);
      default: break;
    }
  }
  return fail(IGS_ECAPACITY, "no three-pass assembly for this order");
}

template <int P, int Q>
igs_status launch3(const igs_problem* p, const AsmShape& s, TensorPat pat, int64_t row_lo, int64_t row_hi,
                   const int64_t* base, const double* planes, double* values, double* H, cudaStream_t st,
                   bool kernel_only, bool two_pass, bool force3) {
  if (row_hi <= row_lo) return IGS_OK;
  ZRange z;
  IGS_TRY(z_range(p, s, row_lo, row_hi, &z));
  const int tile = asm3_tile<P>(s.plan, p->n_planes);
  constexpr int W = 2 * P - 1;
  // p >= 5: x and y contractions as separate passes (G chunks through HBM)
  // unless IGS_FLAG_TWO_PASS asks for the fused stage-1/2 kernel
  const ThreePass tp = three_pass_plan(s);
  if (tile == 0 && !tp.on) return fail(IGS_ECAPACITY, "fused assembly tile does not fit shared memory");
  // A = Aᵀ (whole matrix, whole-grid planes): only the x-pairs n0 >= m0 go
  // through the passes; the z sweep writes each value and its mirror
  const bool sym_whole = problem_symmetric(p) && !(p->slab_lo || p->slab_hi) && row_lo == 0 && s.fs.nfn[2] <= 4096 &&
                         row_hi == s.fs.nfn[0] * s.fs.nfn[1] * s.fs.nfn[2];
  // p = 3: the symmetric three-pass path beats the stage-1/2 kernel (0.83 vs
  // 1.02 ms at 64^3 M+K; its 5-wide band wastes the 8-wide MMA tiles of both
  // stages); p = 4 keeps the one-pass / stage-1/2 kernels (three-pass 1.99 ms
  // vs 1.50 ms: G and H through HBM); IGS_FLAG_THREE_PASS forces it
  const bool three = tp.on && (tile < 4 || force3 || (P == 3 && sym_whole)) && (!two_pass || tile == 0);
  const bool symx = three && sym_whole;
  struct {
    int64_t NS0, NS1;
  } a{s.fs.nfn[0] * (symx ? P : W), s.fs.nfn[1] * W};
  if (three) {
    const int64_t nbh = ceil_div(a.NS0 * a.NS1, (int64_t)kSweepBlock);
    double* extra = H + (size_t)nbh * kSweepBlock * (z.sh - z.sl) * Q * s.plan.nh +
                    (size_t)s.fs.nel[2] * (Q * 4 * (P + 1) + 4);
    IGS_TRY((launch3_three_pass<P, Q>(p, s, tp, z, pat, planes, H, extra, st, symx)));
  } else {
    if constexpr (kWideTile<P> > 0) {
      if (tile == kWideTile<P>) IGS_TRY((launch3_stage12<P, Q, kWideTile<P>>(p, s, z, planes, H, st)));
    }
    if (tile == 4) IGS_TRY((launch3_stage12<P, Q, 4>(p, s, z, planes, H, st)));
    else if (tile == 2) IGS_TRY((launch3_stage12<P, Q, 2>(p, s, z, planes, H, st)));
    else if (tile == 1) IGS_TRY((launch3_stage12<P, Q, 1>(p, s, z, planes, H, st)));
  }
  if (kernel_only) return IGS_OK;  // measurement: the dominant kernel alone
  const TabArgs tab = tab_args(p);
  Asm3bArgs b{};
  b.plan = s.plan;
  b.tab = tab;
  b.H = H;
  b.NS0 = a.NS0;
  b.NS1 = a.NS1;
  b.pat = pat;
  b.row_lo = row_lo;
  b.row_hi = row_hi;
  b.values = values;
  b.base = base;
  // stage-3 weights after H in the workspace (H sized for the slab / grid)
  const int64_t nbsp = ceil_div(a.NS0 * a.NS1, (int64_t)kSweepBlock);
  double* w2g = H + (size_t)nbsp * kSweepBlock * (z.sh - z.sl) * Q * s.plan.nh;
  b.w2g = w2g;
  b.e_lo = z.e_lo;
  b.e_hi = z.e_hi;
  b.chunk = z.e_hi - z.e_lo;
  b.ngrp = s.plan.nh;
  for (int v = 0; v < 4; ++v) b.vmap[v] = -1;
  for (int h = 0; h < s.plan.nh; ++h) b.vmap[s.plan.h_v2[h]] = h;
  {
    const int64_t n = (int64_t)tab.K[2] * S3Cfg<P, Q>::NWR;
    asm_wlast_kernel<P, Q, 3><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(b, w2g);
    IGS_LAUNCH_CHECK("asm_wlast_kernel");
  }
  b.NE = z.e_hi - z.e_lo;
  constexpr size_t smem3 = S3Cfg<P, Q>::SMEM;
  if constexpr (P >= 3) {
    if (symx) {
      const size_t smem3s = smem3 + 3 * (size_t)s.fs.nfn[2] * sizeof(int64_t);  // + z-row table
      IGS_TRY(cuda_check(cudaFuncSetAttribute(asm_sweep<P, Q, 3, true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3s),
                         "smem attribute"));
      asm_sweep<P, Q, 3, true><<<(unsigned)nbsp, NT3, smem3s, st>>>(b);
      IGS_LAUNCH_CHECK("asm_sweep<3, sym>");
      return IGS_OK;
    }
  }
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm_sweep<P, Q, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem3),
                     "smem attribute"));
  asm_sweep<P, Q, 3><<<(unsigned)nbsp, NT3, smem3, st>>>(b);
  IGS_LAUNCH_CHECK("asm_sweep<3>");
  return IGS_OK;
}

template <int P, int Q, int T>
igs_status launch2_stage1(const igs_problem* p, const AsmShape& s, const double* planes, double* G,
                          cudaStream_t st) {
  using C = A3Cfg<P, Q, T>;
  Asm2Args a{};
  a.plan = s.plan;
  a.tab = tab_args(p);
  a.G = G;
  a.NS0 = s.fs.nfn[0] * C::W;
  a.NE = s.fs.nel[1];
  a.X1 = s.fs.npt[1];
  a.ytma0 = 0;
  a.nt0 = (int)ceil_div(s.fs.nfn[0], T);
  const size_t smem = A2Cfg<P, Q, T>::smem(p->n_planes);
  if (((uintptr_t)planes & 15) != 0) return fail(IGS_EARG, "coefficient planes must be 16-byte aligned");
  CUtensorMap fmap;
  {
    const int64_t dims[4] = {s.fs.npt[0], s.fs.npt[1], 1, p->n_planes};
    const unsigned box[4] = {(unsigned)C::XR, (unsigned)A2_YS, 1u, (unsigned)p->n_planes};
    IGS_TRY(planes_tensor_map(&fmap, planes, dims, p->plane_stride, box));
  }
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm2_stage1<P, Q, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem),
                     "smem attribute"));
  // y chunks of whole TMA boxes: minimise waves x (boxes per CTA + 1 for the
  // CTA's prologue), the waves counted against the measured residency
  static std::atomic<int> res_cache[17];  // residency per plane count (the smem size), queried once
  const int npl_key = p->n_planes < 0 ? 0 : (p->n_planes > 16 ? 16 : p->n_planes);
  int resident = res_cache[npl_key].load(std::memory_order_relaxed);
  if (resident <= 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, asm2_stage1<P, Q, T>, A2_NT, smem) !=
            cudaSuccess ||
        resident < 1) {
      cudaGetLastError();
      resident = 1;
    }
    res_cache[npl_key].store(resident, std::memory_order_relaxed);
  }
  const int64_t slots = 148 * (int64_t)resident, nbox = ceil_div(s.fs.npt[1], (int64_t)A2_YS);
  int64_t yc = nbox * A2_YS;
  {
    int64_t best = -1;
    for (int64_t per = 1; per <= nbox; ++per) {  // boxes per CTA
      const int64_t ctas = a.nt0 * ceil_div(nbox, per);
      const int64_t cost = ceil_div(ctas, slots) * (per + 1);
      if (best < 0 || cost < best) {
        best = cost;
        yc = per * A2_YS;
      }
    }
  }
  a.yc = (int)yc;
  const int64_t nyc = ceil_div(s.fs.npt[1], yc);
  // band tables after the G region and the last-direction element records
  const int64_t nbsp = ceil_div(a.NS0, (int64_t)kSweepBlock);
  double* Wg = G + (size_t)nbsp * kSweepBlock * s.fs.npt[1] * s.plan.ng +
               (((size_t)s.fs.nel[1] * S3Cfg<P, Q>::NWR + 1) & ~size_t(1));
  // GPU-filling grids share one table per tile (built once); small grids
  // (launch-bound, e.g. C1) fill it in the CTA and skip the extra launch
  if (nyc >= 4 && a.nt0 * nyc >= 2 * 148) {
    asm2_tables_kernel<P, Q, T><<<(unsigned)a.nt0, 256, 0, st>>>(a.tab, Wg);
    IGS_LAUNCH_CHECK("asm2_tables_kernel");
    a.Wg = Wg;
  }
  asm2_stage1<P, Q, T><<<(unsigned)(a.nt0 * nyc), A2_NT, smem, st>>>(a, fmap, p->n_planes);
  IGS_LAUNCH_CHECK("asm2_stage1");
  return IGS_OK;
}

// 2D x pass through asm3_xpass (one "layer": the rows are the y points).
template <int P, int Q, int T>
igs_status launch2_xpass(const igs_problem* p, const AsmShape& s, const double* planes, double* G,
                         cudaStream_t st) {
  using C = A3Cfg<P, Q, T>;
  if (((uintptr_t)planes & 15) != 0) return fail(IGS_EARG, "coefficient planes must be 16-byte aligned");
  CUtensorMap fmap;
  {
    const int64_t dims[4] = {s.fs.npt[0], s.fs.npt[1], 1, p->n_planes};
    const unsigned box[4] = {(unsigned)AXCfg<P, Q, T>::XB, (unsigned)A3P_YS, 1u, (unsigned)p->n_planes};
    IGS_TRY(planes_tensor_map(&fmap, planes, dims, p->plane_stride, box));
  }
  // band tables behind the G region and the last-direction element records (as launch2_stage1)
  const int64_t nbsp = ceil_div(s.fs.nfn[0] * C::W, (int64_t)kSweepBlock);
  double* Wg = G + (size_t)nbsp * kSweepBlock * s.fs.npt[1] * s.plan.ng +
               (((size_t)s.fs.nel[1] * S3Cfg<P, Q>::NWR + 1) & ~size_t(1));
  const int nt0 = (int)ceil_div(s.fs.nfn[0], T);
  asm2_tables_kernel<P, Q, T><<<(unsigned)nt0, 256, 0, st>>>(tab_args(p), Wg);
  IGS_LAUNCH_CHECK("asm2_tables_kernel");
  return launch3_passA<P, Q, T>(p, s, fmap, Wg, G, 0, 1, st);
}

template <int P, int Q>
igs_status launch2(const igs_problem* p, const AsmShape& s, TensorPat pat, int64_t row_lo, int64_t row_hi,
                   const int64_t* base, const double* planes, double* values, double* G, cudaStream_t st,
                   bool kernel_only) {
  constexpr int W = 2 * P - 1;
  bool xdone = false;
  if constexpr (P >= 5) {
    // p >= 5: the 16-row-box x-pass kernel of the 3D three-pass path fits a
    // wider x tile than asm2_stage1's 64-row boxes (p = 6: 4 rows instead of 2)
    const int tx = three_pass_tile<P>(p->n_planes);
    if (tx > asm2_tile<P>(p->n_planes)) {
      switch (tx) {
        case 6: IGS_TRY((launch2_xpass<P, Q, 6>(p, s, planes, G, st))); break;
        case 4: IGS_TRY((launch2_xpass<P, Q, 4>(p, s, planes, G, st))); break;
        default: IGS_TRY((launch2_xpass<P, Q, 2>(p, s, planes, G, st))); break;
      }
      xdone = true;
    }
  }
  if (!xdone) switch (asm2_tile<P>(p->n_planes)) {
    case 8: IGS_TRY((launch2_stage1<P, Q, 8>(p, s, planes, G, st))); break;
    case 4: IGS_TRY((launch2_stage1<P, Q, 4>(p, s, planes, G, st))); break;
    case 2: IGS_TRY((launch2_stage1<P, Q, 2>(p, s, planes, G, st))); break;
    case 1: IGS_TRY((launch2_stage1<P, Q, 1>(p, s, planes, G, st))); break;
    default: return fail(IGS_ECAPACITY, "2D assembly tile does not fit shared memory");
  }
  if (kernel_only) return IGS_OK;  // measurement: the dominant kernel alone
  struct {
    int64_t NS0;
  } a{s.fs.nfn[0] * W};
  const TabArgs tab = tab_args(p);
  Asm3bArgs b{};
  b.plan = s.plan;
  b.tab = tab;
  b.H = G;
  b.NS0 = a.NS0;
  b.NS1 = 1;
  b.pat = pat;
  b.row_lo = row_lo;
  b.row_hi = row_hi;
  b.base = base;
  b.values = values;
  const int K1 = (int)s.fs.nel[1];
  const int64_t nbsp = ceil_div(a.NS0, (int64_t)kSweepBlock);
  double* wlg = G + (size_t)nbsp * kSweepBlock * s.fs.npt[1] * s.plan.ng;
  b.NE = K1;
  b.w2g = wlg;
  b.e_lo = 0;
  b.e_hi = K1;
  // chunks of >= 2(P-1) elements (each re-sweeps P-1 elements ahead of it):
  // minimise waves x (chunk + P - 1), the waves counted against the sweep
  // kernel's measured residency
  static const int resident = [] {
    constexpr size_t sm3 = S3Cfg<P, Q>::SMEM;
    int n = 1;
    if (cudaFuncSetAttribute(asm_sweep<P, Q, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, asm_sweep<P, Q, 2>, NT3, sm3) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 1;
    }
    return n;
  }();
  const int64_t slots = 148 * (int64_t)resident;
  int chunk = K1;
  {
    int64_t best = -1;
    for (int c = 2 * (P - 1); c <= K1; ++c) {
      const int64_t blocks = nbsp * ceil_div(K1, c);
      const int64_t cost = ceil_div(blocks, slots) * (c + P - 1);
      if (best < 0 || cost < best) {
        best = cost;
        chunk = c;
      }
    }
    if (chunk > K1) chunk = K1;
    if (chunk < 1) chunk = 1;
  }
  b.chunk = chunk;
  if (s.plan.ng > 4) return fail(IGS_ECAPACITY, "2D fused assembly sums at most 4 variant groups");
  b.ngrp = s.plan.ng;
  for (int v = 0; v < 4; ++v) b.vmap[v] = -1;
  for (int g = 0; g < s.plan.ng; ++g) b.vmap[s.plan.g_v1[g]] = g;
  {
    const int64_t n = (int64_t)K1 * S3Cfg<P, Q>::NWR;
    asm_wlast_kernel<P, Q, 2><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(b, wlg);
    IGS_LAUNCH_CHECK("asm_wlast_kernel");
  }
  constexpr size_t smem3 = S3Cfg<P, Q>::SMEM;
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm_sweep<P, Q, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem3),
                     "smem attribute"));
  asm_sweep<P, Q, 2><<<(unsigned)(nbsp * ceil_div(K1, chunk)), NT3, smem3, st>>>(b);
  IGS_LAUNCH_CHECK("asm_sweep<2>");
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

size_t fused_assemble_workspace(const igs_problem* p, const Dims& D, int flags) {
  AsmShape s;
  if (!asm_shape(p, D, &s)) return 0;
  // whole-grid coefficients: the one-pass kernel covers every row range and
  // needs only the row-offset scalar; a slab may need the two-kernel path
  const bool slab = p->slab_lo || p->slab_hi;
  if (!slab && !(flags & (IGS_FLAG_TWO_PASS | IGS_FLAG_THREE_PASS)) && sym_eligible(p, s)) return 512;
  return asm_workspace(s);
}

igs_status fused_assemble(const igs_problem* p, const Dims& D, const int64_t* const* rowptr1d,
                          const int64_t* const* cols1d, int64_t row_lo, int64_t row_hi,
                          const double* planes, double* values, void* ws, size_t ws_bytes,
                          cudaStream_t st, int flags) {
  AsmShape s;
  if (!asm_shape(p, D, &s)) return fail(IGS_ECAPACITY, "no fused assembly");
  if (ws_bytes < 512 || !ws) return fail(IGS_EWORKSPACE, "workspace too small for the fused assembly");
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
  const int P = s.fs.p, Q = s.fs.k;
  const bool ko = (flags & IGS_FLAG_KERNEL_ONLY) != 0;
  if (row_hi <= row_lo) return IGS_OK;
  // 2D, whole matrix: the one-pass symmetric kernel (values start at row 0)
  if (!(flags & IGS_FLAG_TWO_PASS) && sym2_eligible(p, s, row_lo, row_hi)) {
    igs_status r = IGS_ECAPACITY;
    switch (P) {
      case 2: r = launch2_sym<2>(p, s, pat, planes, values, st); break;
      case 3: r = launch2_sym<3>(p, s, pat, planes, values, st); break;
      case 4: r = launch2_sym<4>(p, s, pat, planes, values, st); break;
      case 5: r = launch2_sym<5>(p, s, pat, planes, values, st); break;
      default: break;
    }
    if (r != IGS_ECAPACITY) return r;
  }
  // the CSR offset of row_lo (device scalar in the workspace, written by a
  // one-thread kernel; the one-pass kernel needs none for ranges at row 0)
  bool base_set = false;
  auto set_base = [&]() -> igs_status {
    if (base_set) return IGS_OK;
    base_set = true;
    row_start_kernel<<<1, 1, 0, st>>>(pat, row_lo, base);
    IGS_LAUNCH_CHECK("row_start_kernel");
    return IGS_OK;
  };
  if (sym_eligible(p, s) && !(flags & (IGS_FLAG_TWO_PASS | IGS_FLAG_THREE_PASS))) {
    const bool slab = p->slab_lo || p->slab_hi;
    const int sl = slab ? p->slab_lo : 0, sh = slab ? p->slab_hi : (int)s.fs.nel[2];
    if (row_lo != 0) IGS_TRY(set_base());
    const int64_t* sb = row_lo != 0 ? base : nullptr;
    igs_status r = IGS_ECAPACITY;
    switch (P) {
      case 2: r = launch3_sym<2>(p, s, pat, row_lo, row_hi, sb, planes, values, sl, sh, st); break;
      case 4: r = launch3_sym<4>(p, s, pat, row_lo, row_hi, sb, planes, values, sl, sh, st); break;
      default: break;
    }
    if (r != IGS_ECAPACITY) return r;  // else: the slab lacks the kernel's halo, two-pass below
  }
  if (ws_bytes < asm_workspace(s)) return fail(IGS_EWORKSPACE, "workspace too small for the fused assembly");
  IGS_TRY(set_base());
  igs_status r = IGS_ECAPACITY;
  bool done = false;
#define IGS_ASM_CASE(PP, QQ)                                                                    \
  if (!done && P == PP && Q == QQ) {                                                            \
    r = p->d == 3 ? launch3<PP, QQ>(p, s, pat, row_lo, row_hi, base, planes, values, buf, st, ko,   \
                                     (flags & IGS_FLAG_TWO_PASS) != 0,                           \
                                     (flags & IGS_FLAG_THREE_PASS) != 0)                          \
                  : launch2<PP, QQ>(p, s, pat, row_lo, row_hi, base, planes, values, buf, st, ko);  \
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
