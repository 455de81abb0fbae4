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
  double* scratch;            // per-item boxes
  int64_t box;                // doubles per box
};

template <int P, int Q, int EX, int EY, bool MASS, bool STIFF>
struct Cfg {
  static constexpr int FX = EX + P - 1, FY = EY + P - 1;
  static constexpr int FXP = FX;             // row pitch of [n1][n0] arrays
  static constexpr int TX = EX * Q, TY = EY * Q;
  static constexpr int NT = TY * EX;         // one (line, element) task per thread
  static constexpr int NA = STIFF ? 2 : 1;   // z variants carried (val, der)
  static constexpr int NV = STIFF ? 3 : 1;   // (y,z) variants carried: 00, 10, 01
  static constexpr int XR = P * FY * FXP;
  static constexpr int AA = NA * FY * FXP;
  static constexpr int CC = NV * TY * FXP;   // C, then R (aliased)
  static constexpr int RP = NV * TY * EX * P;
  static constexpr int SS = NA * FY * FXP;
  static constexpr int YR = P * FY * FXP;
  static constexpr int TBX = EX * 2 * Q * P;
  static constexpr int TBY = EY * 2 * Q * P;
  static constexpr int TBZ = 2 * Q * P;
  static constexpr int WW = TX + TY + Q;
  static constexpr int TOTAL = XR + AA + CC + RP + SS + YR + TBX + TBY + TBZ + WW;
  static constexpr size_t SMEM = (size_t)TOTAL * sizeof(double);
};

template <int P, int Q, int EX, int EY, bool MASS, bool STIFF>
__global__ void __launch_bounds__(Cfg<P, Q, EX, EY, MASS, STIFF>::NT)
    apply3d_kernel(const ApplyArgs a) {
  using C = Cfg<P, Q, EX, EY, MASS, STIFF>;
  constexpr int FX = C::FX, FY = C::FY, FXP = C::FXP, TX = C::TX, TY = C::TY, NT = C::NT;
  constexpr int NA = C::NA, NV = C::NV;
  extern __shared__ double sm[];
  double* Xr = sm;                 // [P][FY][FXP]
  double* Aa = Xr + C::XR;         // [NA][FY][FXP]
  double* Cc = Aa + C::AA;         // [NV][TY][FXP]   (R aliases it)
  double* Rp = Cc + C::CC;         // [NV][TY][EX][P]
  double* Ss = Rp + C::RP;         // [NA][FY][FXP]
  double* Yr = Ss + C::SS;         // [P][FY][FXP]
  double* Tx = Yr + C::YR;         // [EX][2][Q][P]
  double* Ty = Tx + C::TBX;        // [EY][2][Q][P]
  double* Tz = Ty + C::TBY;        // [2][Q][P]
  double* Wx = Tz + C::TBZ;        // [TX]
  double* Wy = Wx + TX;            // [TY]
  double* Wz = Wy + TY;            // [Q]

  const int tid = threadIdx.x;
  const int item = blockIdx.x;
  const int tx = item % a.ntx;
  const int ty = (item / a.ntx) % a.nty;
  const int tz = item / (a.ntx * a.nty);
  const int ex0 = tx * EX, ey0 = ty * EY;
  const int z0 = tz * a.ez;
  const int z1 = min(a.K2, z0 + a.ez);
  double* box = a.scratch + (int64_t)item * a.box;

  // ---- prologue: x/y tables + weights of the tile, zeroed y ring ------------
  for (int i = tid; i < C::TBX; i += NT) {
    int j = i % P, q = (i / P) % Q, v = (i / (P * Q)) % 2, e = i / (2 * P * Q);
    int ge = ex0 + e;
    Tx[i] = ge < a.K0 ? a.vals[0][((int64_t)v * P + j) * a.xtab[0] + (int64_t)ge * Q + q] : 0.0;
  }
  for (int i = tid; i < C::TBY; i += NT) {
    int j = i % P, q = (i / P) % Q, v = (i / (P * Q)) % 2, e = i / (2 * P * Q);
    int ge = ey0 + e;
    Ty[i] = ge < a.K1 ? a.vals[1][((int64_t)v * P + j) * a.xtab[1] + (int64_t)ge * Q + q] : 0.0;
  }
  for (int i = tid; i < TX; i += NT) {
    int64_t g = (int64_t)ex0 * Q + i;
    Wx[i] = g < a.X0 ? a.wts[0][g] : 0.0;
  }
  for (int i = tid; i < TY; i += NT) {
    int64_t g = (int64_t)ey0 * Q + i;
    Wy[i] = g < a.X1 ? a.wts[1][g] : 0.0;
  }
  for (int i = tid; i < C::YR; i += NT) Yr[i] = 0.0;

  auto load_layer = [&](int n2) {
    double* dst = Xr + (n2 % P) * FY * FXP;
    for (int i = tid; i < FY * FX; i += NT) {
      int n0 = i % FX, n1 = i / FX;
      int64_t g0 = (int64_t)ex0 + n0, g1 = (int64_t)ey0 + n1;
      double v = 0.0;
      if (g0 < a.N0 && g1 < a.N1 && n2 < a.N2) v = __ldg(a.x + ((int64_t)n2 * a.N1 + g1) * a.N0 + g0);
      dst[n1 * FXP + n0] = v;
    }
  };
  for (int l = 0; l < P; ++l) load_layer(z0 + l);

  // Line task of this thread in the X phase: (line q1, element ex).
  const int t_q1 = tid / EX, t_ex = tid % EX;
  const bool t_valid = (ex0 + t_ex) < a.K0 && (ey0 + t_q1 / Q) < a.K1;

  const double* Fc = MASS ? a.planes + (int64_t)a.pl_c * a.pstride : nullptr;
  const double* Fa00 = STIFF ? a.planes + (int64_t)a.pl_a[0][0] * a.pstride : nullptr;
  const double* Fa11 = STIFF ? a.planes + (int64_t)a.pl_a[1][1] * a.pstride : nullptr;
  const double* Fa22 = STIFF ? a.planes + (int64_t)a.pl_a[2][2] * a.pstride : nullptr;
  const double* Fa01 = STIFF ? a.planes + (int64_t)a.pl_a[0][1] * a.pstride : nullptr;
  const double* Fa02 = STIFF ? a.planes + (int64_t)a.pl_a[0][2] * a.pstride : nullptr;
  const double* Fa12 = STIFF ? a.planes + (int64_t)a.pl_a[1][2] * a.pstride : nullptr;

  for (int e2 = z0; e2 < z1; ++e2) {
    // z tables and weights of this element layer
    const int gz = e2 + a.z_el_off;
    for (int i = tid; i < C::TBZ; i += NT) {
      int j = i % P, q = (i / P) % Q, v = i / (P * Q);
      Tz[i] = a.vals[2][((int64_t)v * P + j) * a.xtab[2] + (int64_t)gz * Q + q];
    }
    for (int i = tid; i < Q; i += NT) Wz[i] = a.wts[2][(int64_t)gz * Q + i];
    __syncthreads();

    for (int q2 = 0; q2 < Q; ++q2) {
      // ---- Z: contract the P active x layers to point layer q2 -------------
      for (int i = tid; i < FY * FX; i += NT) {
        int n0 = i % FX, n1 = i / FX;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          double xv = Xr[((e2 + j) % P) * FY * FXP + n1 * FXP + n0];
          a0 = fma(Tz[(0 * Q + q2) * P + j], xv, a0);
          if (STIFF) a1 = fma(Tz[(1 * Q + q2) * P + j], xv, a1);
        }
        Aa[n1 * FXP + n0] = a0;
        if (STIFF) Aa[FY * FXP + n1 * FXP + n0] = a1;
      }
      __syncthreads();
      // ---- Y: contract y functions to y points -----------------------------
      for (int i = tid; i < TY * FX; i += NT) {
        int n0 = i % FX, q1 = i / FX;
        int ey = q1 / Q, ql = q1 % Q;
        const double* T0 = Ty + ((ey * 2 + 0) * Q + ql) * P;
        const double* T1 = Ty + ((ey * 2 + 1) * Q + ql) * P;
        double c00 = 0.0, c10 = 0.0, c01 = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          double a0 = Aa[(ey + j) * FXP + n0];
          c00 = fma(T0[j], a0, c00);
          if (STIFF) {
            c10 = fma(T1[j], a0, c10);
            c01 = fma(T0[j], Aa[FY * FXP + (ey + j) * FXP + n0], c01);
          }
        }
        Cc[q1 * FXP + n0] = c00;
        if (STIFF) {
          Cc[TY * FXP + q1 * FXP + n0] = c10;
          Cc[2 * TY * FXP + q1 * FXP + n0] = c01;
        }
      }
      __syncthreads();
      // ---- X + pointwise + X^T partials (one line segment per thread) -------
      {
        double p00[P], p10[P], p01[P];
#pragma unroll
        for (int j = 0; j < P; ++j) p00[j] = p10[j] = p01[j] = 0.0;
        if (t_valid) {
          double c00[P], c10[P], c01[P];
#pragma unroll
          for (int j = 0; j < P; ++j) {
            c00[j] = Cc[t_q1 * FXP + t_ex + j];
            if (STIFF) {
              c10[j] = Cc[TY * FXP + t_q1 * FXP + t_ex + j];
              c01[j] = Cc[2 * TY * FXP + t_q1 * FXP + t_ex + j];
            }
          }
          const int64_t zq = (int64_t)(e2 - 0) * Q + q2;  // slab-local point layer
          const int64_t fo = (zq * a.X1 + (int64_t)ey0 * Q + t_q1) * a.X0 + (int64_t)(ex0 + t_ex) * Q;
          const double wyz = Wz[q2] * Wy[t_q1];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const double* T0 = Tx + ((t_ex * 2 + 0) * Q + q) * P;
            const double* T1 = Tx + ((t_ex * 2 + 1) * Q + q) * P;
            double u = 0.0, ux = 0.0, uy = 0.0, uz = 0.0;
#pragma unroll
            for (int j = 0; j < P; ++j) {
              double b0 = T0[j];
              if (MASS) u = fma(b0, c00[j], u);
              if (STIFF) {
                ux = fma(T1[j], c00[j], ux);
                uy = fma(b0, c10[j], uy);
                uz = fma(b0, c01[j], uz);
              }
            }
            const double w = wyz * Wx[t_ex * Q + q];
            double g0 = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
            if (MASS) g0 = w * (__ldg(Fc + fo + q) * u);
            if (STIFF) {
              double f00 = __ldg(Fa00 + fo + q), f11 = __ldg(Fa11 + fo + q), f22 = __ldg(Fa22 + fo + q);
              double f01 = __ldg(Fa01 + fo + q), f02 = __ldg(Fa02 + fo + q), f12 = __ldg(Fa12 + fo + q);
              gx = w * fma(f00, ux, fma(f01, uy, f02 * uz));
              gy = w * fma(f01, ux, fma(f11, uy, f12 * uz));
              gz = w * fma(f02, ux, fma(f12, uy, f22 * uz));
            }
#pragma unroll
            for (int j = 0; j < P; ++j) {
              double b0 = T0[j];
              if (STIFF) {
                p00[j] = fma(T1[j], gx, p00[j]);
                p10[j] = fma(b0, gy, p10[j]);
                p01[j] = fma(b0, gz, p01[j]);
              }
              if (MASS) p00[j] = fma(b0, g0, p00[j]);
            }
          }
        }
        double* r = Rp + (t_q1 * EX + t_ex) * P;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          r[j] = p00[j];
          if (STIFF) {
            r[TY * EX * P + j] = p10[j];
            r[2 * TY * EX * P + j] = p01[j];
          }
        }
      }
      __syncthreads();
      // ---- X^T: overlap-add the element partials into R (aliases C) --------
      for (int i = tid; i < TY * FX; i += NT) {
        int n0 = i % FX, q1 = i / FX;
        int s_lo = n0 - (EX - 1) > 0 ? n0 - (EX - 1) : 0;
        int s_hi = n0 < P - 1 ? n0 : P - 1;
        double r00 = 0.0, r10 = 0.0, r01 = 0.0;
        for (int s = s_lo; s <= s_hi; ++s) {
          int o = (q1 * EX + (n0 - s)) * P + s;
          r00 += Rp[o];
          if (STIFF) {
            r10 += Rp[TY * EX * P + o];
            r01 += Rp[2 * TY * EX * P + o];
          }
        }
        Cc[q1 * FXP + n0] = r00;
        if (STIFF) {
          Cc[TY * FXP + q1 * FXP + n0] = r10;
          Cc[2 * TY * FXP + q1 * FXP + n0] = r01;
        }
      }
      __syncthreads();
      // ---- Y^T + Z^T: test back in y, then accumulate into the y ring -------
      for (int i = tid; i < FY * FX; i += NT) {
        int n0 = i % FX, n1 = i / FX;
        int e_lo = n1 - (P - 1) > 0 ? n1 - (P - 1) : 0;
        int e_hi = n1 < EY - 1 ? n1 : EY - 1;
        double s0 = 0.0, s1 = 0.0;
        for (int ey = e_lo; ey <= e_hi; ++ey) {
          int j = n1 - ey;
#pragma unroll
          for (int ql = 0; ql < Q; ++ql) {
            int q1 = ey * Q + ql;
            double b0 = Ty[((ey * 2 + 0) * Q + ql) * P + j];
            s0 = fma(b0, Cc[q1 * FXP + n0], s0);
            if (STIFF) {
              s0 = fma(Ty[((ey * 2 + 1) * Q + ql) * P + j], Cc[TY * FXP + q1 * FXP + n0], s0);
              s1 = fma(b0, Cc[2 * TY * FXP + q1 * FXP + n0], s1);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < P; ++j) {
          double* yr = Yr + ((e2 + j) % P) * FY * FXP + n1 * FXP + n0;
          double v = fma(Tz[(0 * Q + q2) * P + j], s0, *yr);
          if (STIFF) v = fma(Tz[(1 * Q + q2) * P + j], s1, v);
          *yr = v;
        }
      }
      __syncthreads();
    }
    // ---- DoF layer e2 is complete for this chunk: flush, recycle the slots -
    {
      double* yr = Yr + (e2 % P) * FY * FXP;
      double* dst = box + (int64_t)(e2 - z0) * FY * FX;
      for (int i = tid; i < FY * FX; i += NT) {
        int n0 = i % FX, n1 = i / FX;
        dst[i] = yr[n1 * FXP + n0];
        yr[n1 * FXP + n0] = 0.0;
      }
    }
    load_layer(e2 + P);
    __syncthreads();
  }
  // trailing P-1 layers [z1, z1 + P - 1)
  for (int l = z1; l < z1 + P - 1; ++l) {
    double* yr = Yr + (l % P) * FY * FXP;
    double* dst = box + (int64_t)(l - z0) * FY * FX;
    for (int i = tid; i < FY * FX; i += NT) {
      int n0 = i % FX, n1 = i / FX;
      dst[i] = yr[n1 * FXP + n0];
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
__global__ void apply_reduce_kernel(const ReduceArgs r) {
  const int64_t total = r.N0 * r.N1 * r.N2;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t n0 = g % r.N0, n1 = (g / r.N0) % r.N1, n2 = g / (r.N0 * r.N1);
    int tx_hi = (int)min64(r.ntx - 1, n0 / r.EX);
    int ty_hi = (int)min64(r.nty - 1, n1 / r.EY);
    int tz_hi = (int)min64(r.nch - 1, n2 / r.ez);
    // first tiles whose boxes can still reach n (box extent FX / FY / ez+P-1)
    int tx_lo = n0 >= r.FX ? (int)((n0 - r.FX) / r.EX + 1) : 0;
    int ty_lo = n1 >= r.FY ? (int)((n1 - r.FY) / r.EY + 1) : 0;
    int64_t zspan = (int64_t)r.ez + r.P - 1;
    int tz_lo = n2 >= zspan ? (int)((n2 - zspan) / r.ez + 1) : 0;
    double s = 0.0;
    for (int tz = tz_lo; tz <= tz_hi; ++tz) {
      int64_t z0 = (int64_t)tz * r.ez;
      int64_t z1 = min64(r.K2, z0 + r.ez);
      if (n2 >= z1 + r.P - 1 || n2 < z0) continue;
      for (int ty = ty_lo; ty <= ty_hi; ++ty) {
        int64_t l1 = n1 - (int64_t)ty * r.EY;
        if (l1 >= r.FY) continue;
        for (int tx = tx_lo; tx <= tx_hi; ++tx) {
          int64_t l0 = n0 - (int64_t)tx * r.EX;
          if (l0 >= r.FX) continue;
          int64_t item = ((int64_t)tz * r.nty + ty) * r.ntx + tx;
          s += r.scratch[item * r.box + ((n2 - z0) * r.FY + l1) * r.FX + l0];
        }
      }
    }
    r.y[g] = r.accumulate ? r.y[g] + s : s;
  }
}

// ---- instantiation table ----------------------------------------------------

struct Launch {
  int EX, EY, NT;
  size_t smem;
  void (*kernel)(ApplyArgs);
};

template <int P, int Q, int EX, int EY, bool MASS, bool STIFF>
Launch make_launch() {
  using C = Cfg<P, Q, EX, EY, MASS, STIFF>;
  return Launch{EX, EY, C::NT, C::SMEM, &apply3d_kernel<P, Q, EX, EY, MASS, STIFF>};
}

// Tile shapes per order: NT = EX·EY·Q threads, shared memory < 113 KB so
// two CTAs fit on an SM where possible.
template <bool MASS, bool STIFF>
bool pick(int P, int Q, Launch* L) {
  if (P != Q) return false;
  switch (P) {
    case 2: *L = make_launch<2, 2, 8, 16, MASS, STIFF>(); return true;
    case 3: *L = make_launch<3, 3, 8, 8, MASS, STIFF>(); return true;
    case 4: *L = make_launch<4, 4, 8, 8, MASS, STIFF>(); return true;
    case 5: *L = make_launch<5, 5, 8, 6, MASS, STIFF>(); return true;
    case 6: *L = make_launch<6, 6, 8, 8, MASS, STIFF>(); return true;
    case 7: *L = make_launch<7, 7, 8, 4, MASS, STIFF>(); return true;
    case 8: *L = make_launch<8, 8, 8, 4, MASS, STIFF>(); return true;
    default: return false;
  }
}

bool pick_launch(const FusedShape& s, Launch* L) {
  if (s.d != 3) return false;
  if (s.mass && s.stiff) return pick<true, true>(s.p, s.k, L);
  if (s.stiff) return pick<false, true>(s.p, s.k, L);
  if (s.mass) return pick<true, false>(s.p, s.k, L);
  return false;
}

struct Tiling {
  int ntx, nty, nch, ez;
  int64_t box;
};

Tiling tiling(const FusedShape& s, const Launch& L) {
  Tiling t;
  t.ntx = (int)ceil_div(s.nel[0], L.EX);
  t.nty = (int)ceil_div(s.nel[1], L.EY);
  // z chunks: enough work items for ~8 waves of 2 CTAs per SM, chunks of at
  // least P-1 layers so each DoF sees at most two chunks.
  int K2 = (int)s.nel[2];
  int64_t tiles = (int64_t)t.ntx * t.nty;
  int want = (int)ceil_div(148 * 2 * 8, tiles);
  int ez = (int)ceil_div(K2, want > 0 ? want : 1);
  if (ez < s.p - 1) ez = s.p - 1;
  if (ez < 1) ez = 1;
  if (ez > K2) ez = K2;
  t.ez = ez;
  t.nch = (int)ceil_div(K2, ez);
  int FX = L.EX + s.p - 1, FY = L.EY + s.p - 1;
  t.box = (int64_t)(ez + s.p - 1) * FY * FX;
  return t;
}

}  // namespace

bool fused_apply_supported(const igs_problem* p, const Dims& D) {
  FusedShape s;
  if (!fused_shape(p, D, &s)) return false;
  Launch L;
  return pick_launch(s, &L);
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
  if (!fused_shape(p, D, &s) || !pick_launch(s, &L)) return fail(IGS_ECAPACITY, "no fused apply");
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
  a.ntx = t.ntx; a.nty = t.nty; a.nch = t.nch; a.ez = t.ez;
  a.scratch = reinterpret_cast<double*>(ws);
  a.box = t.box;
  IGS_TRY(cuda_check(cudaFuncSetAttribute(L.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)L.smem), "smem attribute"));
  unsigned grid = (unsigned)(t.ntx * t.nty * t.nch);
  L.kernel<<<grid, L.NT, L.smem, st>>>(a);
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
  int64_t total = r.N0 * r.N1 * r.N2;
  int64_t g = ceil_div(total, 256);
  if (g > 148 * 16) g = 148 * 16;
  apply_reduce_kernel<<<(unsigned)g, 256, 0, st>>>(r);
  IGS_LAUNCH_CHECK("apply_reduce_kernel");
  return IGS_OK;
}

}  // namespace igs
