// K3s2 — one-pass symmetric 2D assembly (Alg. 1 fused over both directions),
// included by assemble3d.cu inside its anonymous namespace after
// asm3_sym.cuh (it shares sym_keep / sym_mirror and the z-factor layout).
//
// Same sums as the reference's _Core.block_values (sumfac.py:200-213) with
// W_δ = w·B^θ_n·B^η_m (_Core.w_matrix, sumfac.py:163-198), for a symmetric
// problem (A = Aᵀ): a CTA forms only the x-pairs (m0, n0 = m0 + o0), o0 >= 0,
// and writes each value to its row and, for o0 > 0 (or o0 = 0, o1 > 0),
// mirrored to the transposed entry.
//
// One CTA = T0 rows in x (a strip), sweeping y over its chunk of y rows,
// one MMA m-tile of 8 y points per phase:
//   TMA      coefficient region of the strip (all planes, (T0+P-1)·Q x points
//            x 8 y points), double-buffered, two phases ahead;
//   stage 1  G_g[y][s0] = Σ_{b∈g} Σ_x F_b[y][x] W0^{v0(b)}[x][s0]    DMMA (M=y, N=s0, K=x)
//            one warp per n-tile of 8 slots, its band-table fragments held
//            in registers for the whole sweep (no table in shared memory);
//   stage 3  one thread per x-pair: the y contraction of the 8 points into
//            the element matrix E[jm][jn] (registers, DFMA: u_η[jn] =
//            Σ_θ (w·B^θ_jn) G_{θ+2η}, E += B^η_jm u_η); at the element's last
//            point E's rows go into the pending rows (shared memory, one slot
//            per y row mod P) and row e is final -> CSR (+ mirrors).
// Stage-3 warps work on phase k-1 while the stage-1 warps work on phase k
// (G double-buffered, one barrier per phase).  Nothing but the CSR values
// reaches HBM (the two-kernel path writes G to HBM and sweeps it again).
//
// Rows: a chunk owns y rows [r_lo, r_hi) and contracts elements
// [r_lo - P + 1, r_hi) (its first P-1 elements only complete rows it owns);
// every CSR entry is written by exactly one thread (the pair with
// m0 <= n0, at row min-by-sym_keep), so the whole-matrix assembly needs no
// halo beyond those P-1 elements.  Row ranges other than the whole matrix use
// the two-kernel path.

// Measurement / debugging variants (tools/build_variant.sh; wrong values):
// 1 skips the stage-1 MMAs, 2 stage 3, 3 the CSR stores.  The library builds 0.
#ifndef IGS_SYM2_EXP
#define IGS_SYM2_EXP 0
#endif

template <int P>
struct Sym2Tile;
template <> struct Sym2Tile<2> { static constexpr int T0 = 48; };
template <> struct Sym2Tile<3> { static constexpr int T0 = 32; };
template <> struct Sym2Tile<4> { static constexpr int T0 = 24; };
template <> struct Sym2Tile<5> { static constexpr int T0 = 19; };

template <int P, int T0>
struct Sym2Cfg {
  static constexpr int Q = P;
  static constexpr int W = 2 * P - 1;
  static constexpr int NS0 = T0 * P;                 // symmetric x slots = stage-3 pairs
  static constexpr int NST0 = (NS0 + 7) / 8;         // stage-1 n-tiles = stage-1 warps
  static constexpr int NW3 = (NS0 + 31) / 32;        // stage-3 warps
  static constexpr int NW = NW3 + NST0, NT = 32 * NW;
  static constexpr int NS3 = NW3 * 32;               // pair pitch of the pending rows
  static constexpr int ER0 = T0 + P - 1, XR0 = ER0 * Q;
  static constexpr int YT = 8;                       // y points per phase
  // TMA box width: >= XR0 + 1 (the box starts at the even x point at or
  // below the region: a TMA box must start 16-byte aligned), a multiple of 4
  // doubles, pitch ≡ 4 or 12 (mod 16) doubles so the A-fragment loads (8 rows
  // x 4 columns) hit distinct banks
  static constexpr int box0() {
    int b = (XR0 + (Q & 1) + 3) & ~3;
    while (b % 16 != 4 && b % 16 != 12) b += 4;
    return b;
  }
  static constexpr int XB0 = box0();
  static constexpr int pitch4(int n) { return ((n + 11) / 16) * 16 + 4; }
  static constexpr int SPG = pitch4(NS0);            // G row pitch
  // k-step range of n-tile st (x points of its rows' supports)
  static constexpr int k0_lo(int st) { return ((8 * st) / P) * Q / 4; }
  static constexpr int r0_hi(int st) { return (8 * st + 7) / P < T0 - 1 ? (8 * st + 7) / P : T0 - 1; }
  static constexpr int k0_hi(int st) { return ((r0_hi(st) + P) * Q + 3) / 4; }
  static constexpr int ks0() {
    int m = 1;
    for (int st = 0; st < NST0; ++st) m = k0_hi(st) - k0_lo(st) > m ? k0_hi(st) - k0_lo(st) : m;
    return m;
  }
  static constexpr int KS0 = ks0();
  static constexpr int PP = (P + 1) & ~1;            // y factor row (16-byte rows)
  static constexpr int FZP = 4 * PP;                 // y factors per point: wB^0 | wB^1 | B^0 | B^1
  // shared memory (doubles): F buffers (+ a zero tail the widest k-range may
  // read past the last row), G buffers, pending rows, y factors per point of
  // the chunk, then the y-row table (3 int64 per row) and the barriers
  static constexpr size_t fbuf(int npl) {
    return ((size_t)npl * YT * XB0 + (size_t)KS0 * 4 + 4 + 15) & ~size_t(15);
  }
  static constexpr size_t GS = (size_t)4 * YT * SPG;
  static constexpr size_t PS = (size_t)P * W * NS3;
  static constexpr size_t smem(int npl, int npts, int yrows) {
    return (2 * fbuf(npl) + 2 * GS + PS + (size_t)npts * FZP + 3 * (size_t)yrows) * sizeof(double) + 64;
  }
  static_assert(XB0 <= 256, "TMA box");
};

struct Sym2Args {
  TabArgs tab;
  TensorPat pat;
  double* values;
  int nt0;               // strips in x
  int nplanes;
  int K1;                // elements in y
  int rows_per_chunk;    // y rows per chunk (grid.y)
  int max_pts;           // capacity of the per-point y-factor table
  int yrows;             // capacity of the y-row table
  int vmap[4];           // stage-1 group holding y variant v = θ + 2η (-1: none)
  int nb;                // stage-1 blocks (group order)
  int b_plane[kMaxBlocks], b_v0[kMaxBlocks], b_g[kMaxBlocks];
  unsigned b_end;        // bit b: last block of its group
};

template <int P, int T0>
__global__ void __launch_bounds__(Sym2Cfg<P, T0>::NT, 1)
    asm2_sym(const Sym2Args a, const __grid_constant__ CUtensorMap fmap) {
  using C = Sym2Cfg<P, T0>;
  constexpr int Q = C::Q, W = C::W, NS0 = C::NS0, NW3 = C::NW3, NS3 = C::NS3;
  constexpr int XB0 = C::XB0, SPG = C::SPG, KS0 = C::KS0, PP = C::PP, FZP = C::FZP, YT = C::YT, NT = C::NT;
  extern __shared__ __align__(128) double sm[];
  const size_t fb = C::fbuf(a.nplanes);
  double* Fs = sm;                                   // [2][npl][YT][XB0] (+ zero tails)
  double* Gs = Fs + 2 * fb;                          // [2][4][YT][SPG]
  double* PD = Gs + 2 * C::GS;                       // [P][W][NS3] pending rows (slot = y row mod P)
  double* FZs = PD + C::PS;                          // [pts][FZP]
  int64_t* YR = reinterpret_cast<int64_t*>(FZs + (size_t)a.max_pts * FZP);  // [yrows][3]
  uint64_t* bar = reinterpret_cast<uint64_t*>(YR + 3 * (size_t)a.yrows);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, m4 = lane & 3;
  const int a0 = blockIdx.x * T0;
  const int xb0 = (a0 - (P - 1)) * Q;    // first x point of the strip's region
  const int xbox = xb0 - (xb0 & 1);      // TMA box origin (even: 16-byte aligned)
  const int64_t N0 = a.tab.N[0], N1 = a.tab.N[1];
  // y rows owned by this chunk and the elements that complete them
  const int r_lo = blockIdx.y * a.rows_per_chunk;
  const int r_hi = (int)min64(N1, (int64_t)r_lo + a.rows_per_chunk);
  const int e_lo = max(0, r_lo - (P - 1));
  const int e_hi = min(a.K1, r_hi);
  const int npts = (e_hi - e_lo) * Q;
  const int nph = (npts + YT - 1) / YT;
  const int y_first = e_lo * Q;
  const unsigned fbytes = (unsigned)((size_t)a.nplanes * YT * XB0 * sizeof(double));

  // ---- prologue ---------------------------------------------------------------
  for (int b = 0; b < 2; ++b)
    for (size_t i = (size_t)a.nplanes * YT * XB0 + tid; i < fb; i += NT) Fs[b * fb + i] = 0.0;
  for (int i = tid; i < (int)C::PS; i += NT) PD[i] = 0.0;
  if (tid == 0) {
    dev::mbar_init(bar, 1);
    dev::mbar_init(bar + 1, 1);
    dev::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < 2 && i < nph; ++i) {
      dev::mbar_expect_tx(bar + i, fbytes);
      dev::tma_load_4d(Fs + i * fb, &fmap, bar + i, xbox, y_first + i * YT, 0, 0);
    }
  }
  // y factors of every point of the chunk: [wB^0 | wB^1 | B^0 | B^1][PP]
  for (int i = tid; i < npts * FZP; i += NT) {
    const int yl = i / FZP, r = i % FZP;
    const int j = r % PP, f = r / PP, lvl = f & 1;
    double v = 0.0;
    if (j < P && lvl <= a.tab.md[1]) {
      const int64_t y = (int64_t)y_first + yl;
      const double b = a.tab.vals[1][((int64_t)lvl * P + j) * a.tab.X[1] + y];
      v = f < 2 ? a.tab.wts[1][y] * b : b;
    }
    FZs[i] = v;
  }
  // y-row table over the rows written directly or mirrored: [rp1, width, lo]
  const int yr0 = max(0, r_lo - (P - 1));
  {
    const int yr1 = (int)min64(N1, (int64_t)r_hi + P - 1);
    const int64_t* rp1 = a.pat.rp[1];
    const int64_t* cl1 = a.pat.cl[1];
    for (int r = yr0 + tid; r < yr1; r += NT) {
      const int64_t rs = rp1[r];
      YR[3 * (r - yr0)] = rs;
      YR[3 * (r - yr0) + 1] = rp1[r + 1] - rs;
      YR[3 * (r - yr0) + 2] = cl1[rs];
    }
  }

  if (warp >= NW3) {
    // ================= stage-1 warps: one n-tile each ==========================
    const int st = warp - NW3;
    int klo = 0;
#pragma unroll
    for (int i = 0; i < C::NST0; ++i)
      if (i == st) klo = C::k0_lo(i);
    // band-table fragments of this n-tile, all four x variants, in registers:
    //   w0r[v][kk] = w(x)·B^θ_n(x)·B^η_m(x), x = region k-step klo + kk, lane m4;
    //   slot 8·st + g8 (m = a0 + slot / P, n = m + slot % P), v = θ + 2η
    double w0r[4][KS0];
    {
      const int s = 8 * st + g8;
      const int r = s / P, off = s % P;
      const int64_t m = a0 + r, n = m + off;
#pragma unroll
      for (int kk = 0; kk < KS0; ++kk) {
        const int64_t x = xb0 + (klo + kk) * 4 + m4;
        const bool in = s < NS0 && x >= 0 && x < a.tab.X[0] && m < N0 && n < N0;
        const int64_t e = x / Q;
        const int64_t jn = n - e, jm = m - e;
        const bool sup = in && jn >= 0 && jn < P && jm >= 0 && jm < P;
        double w = 0.0, b0n = 0.0, b1n = 0.0, b0m = 0.0, b1m = 0.0;
        if (sup) {
          w = a.tab.wts[0][x];
          b0n = a.tab.vals[0][jn * a.tab.X[0] + x];
          b0m = a.tab.vals[0][jm * a.tab.X[0] + x];
          if (a.tab.md[0] >= 1) {
            b1n = a.tab.vals[0][((int64_t)P + jn) * a.tab.X[0] + x];
            b1m = a.tab.vals[0][((int64_t)P + jm) * a.tab.X[0] + x];
          }
        }
        w0r[0][kk] = (w * b0n) * b0m;
        w0r[1][kk] = (w * b1n) * b0m;
        w0r[2][kk] = (w * b0n) * b1m;
        w0r[3][kk] = (w * b1n) * b1m;
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k <= nph; ++k) {
      if (k < nph) {
        dev::mbar_wait(bar + (k & 1), (unsigned)((k >> 1) & 1));
        const double* Fy = Fs + (k & 1) * fb + g8 * XB0 + (xb0 - xbox) + m4 + klo * 4;
        double* Gy = Gs + (k & 1) * C::GS + g8 * SPG + st * 8 + 2 * m4;
        const bool st_ok = st * 8 + 2 * m4 < NS0;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll 1
        for (int b = 0; b < a.nb; ++b) {
          const double* Fp = Fy + a.b_plane[b] * (YT * XB0);
          double f[KS0];
#pragma unroll
          for (int kk = 0; kk < KS0; ++kk) f[kk] = Fp[kk * 4];
          if (IGS_SYM2_EXP == 1) continue;
          switch (a.b_v0[b]) {
            case 0:
#pragma unroll
              for (int kk = 0; kk < KS0; ++kk) dmma_a(c0, c1, f[kk], w0r[0][kk]);
              break;
            case 1:
#pragma unroll
              for (int kk = 0; kk < KS0; ++kk) dmma_a(c0, c1, f[kk], w0r[1][kk]);
              break;
            case 2:
#pragma unroll
              for (int kk = 0; kk < KS0; ++kk) dmma_a(c0, c1, f[kk], w0r[2][kk]);
              break;
            default:
#pragma unroll
              for (int kk = 0; kk < KS0; ++kk) dmma_a(c0, c1, f[kk], w0r[3][kk]);
              break;
          }
          if ((a.b_end >> b) & 1) {
            if (st_ok) *reinterpret_cast<double2*>(Gy + a.b_g[b] * (YT * SPG)) = make_double2(c0, c1);
            c0 = c1 = 0.0;
          }
        }
      }
      __syncthreads();
      // F[k & 1] is consumed: fetch phase k + 2 behind the next phase
      if (tid == NW3 * 32 && k + 2 < nph) {
        dev::fence_proxy_async();
        dev::mbar_expect_tx(bar + (k & 1), fbytes);
        dev::tma_load_4d(Fs + (k & 1) * fb, &fmap, bar + (k & 1), xbox, y_first + (k + 2) * YT, 0, 0);
      }
    }
    return;
  }

  // ================= stage-3 warps: one x-pair per thread =======================
  const int s0 = tid;
  const int r0 = s0 / P, o0 = s0 % P;
  const int64_t m0 = a0 + r0, n0 = m0 + o0;
  const bool valid = s0 < NS0 && m0 < N0 && n0 < N0;
  // CSR addressing (2D): row (m0, m1) starts at rp0[m0]·w1(m1) + P0·rp1[m1];
  // entry (n0, n1) at + (n1 - lo1(m1))·w0(m0) + (n0 - lo0(m0)); the mirror
  // the same for row (n0, n1) with the roles of m and n exchanged
  const int64_t* rp0 = a.pat.rp[0];
  const int64_t P0 = rp0[N0];
  int64_t rs0m = 0, rs0n = 0;
  int w0m = 0, w0n = 0, dm = 0, dn = 0;
  if (valid) {
    rs0m = rp0[m0];
    w0m = (int)(rp0[m0 + 1] - rs0m);
    dm = (int)(n0 - a.pat.cl[0][rs0m]);  // column n0 in row m0
    rs0n = rp0[n0];
    w0n = (int)(rp0[n0 + 1] - rs0n);
    dn = (int)(m0 - a.pat.cl[0][rs0n]);  // column m0 in row n0
  }
  unsigned keepm = 0, mirm = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    keepm |= (valid && sym_keep(o0, k - (P - 1), 0) ? 1u : 0u) << k;
    mirm |= (valid && sym_mirror(o0, k - (P - 1), 0) ? 1u : 0u) << k;
  }
  double* pd = PD + s0;  // this pair's pending rows: pd[(slot·W + k)·NS3]
  auto store_row = [&](int m1, const double (&row)[W]) {
    if (!valid || m1 < r_lo || m1 >= r_hi || IGS_SYM2_EXP == 3) return;
    const int64_t* ym = YR + 3 * (m1 - yr0);
    const int64_t dbase = rs0m * ym[1] + P0 * ym[0] + dm - ym[2] * w0m;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int n1 = m1 + k - (P - 1);
      if (n1 < 0 || n1 >= N1) continue;
      if (keepm & (1u << k)) a.values[dbase + (int64_t)n1 * w0m] = row[k];
      if (mirm & (1u << k)) {
        const int64_t* yn = YR + 3 * (n1 - yr0);
        a.values[rs0n * yn[1] + P0 * yn[0] + (m1 - yn[2]) * w0n + dn] = row[k];
      }
    }
  };
  __syncthreads();
  double E[P][P];
#pragma unroll
  for (int i = 0; i < P; ++i)
#pragma unroll
    for (int j = 0; j < P; ++j) E[i][j] = 0.0;
#pragma unroll 1
  for (int k = 0; k <= nph; ++k) {
    if (k >= 1 && IGS_SYM2_EXP != 2) {
      const int ph = k - 1;
      const double* Gb = Gs + (ph & 1) * C::GS + s0;
#pragma unroll 1
      for (int i = 0; i < YT; ++i) {
        const int yl = ph * YT + i;
        if (yl >= npts) break;
        const int qs = yl % Q, es = e_lo + yl / Q;
        double hv[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) hv[v] = a.vmap[v] >= 0 ? Gb[(a.vmap[v] * YT + i) * SPG] : 0.0;
        const double* fq = FZs + (size_t)yl * FZP;
        double u0[P], u1[P];
#pragma unroll
        for (int jn = 0; jn < P; ++jn) {
          const double wb0 = fq[jn], wb1 = fq[PP + jn];
          u0[jn] = fma(wb1, hv[1], wb0 * hv[0]);
          u1[jn] = fma(wb1, hv[3], wb0 * hv[2]);
        }
#pragma unroll
        for (int jm = 0; jm < P; ++jm) {
          const double b0 = fq[2 * PP + jm], b1 = fq[3 * PP + jm];
#pragma unroll
          for (int jn = 0; jn < P; ++jn) E[jm][jn] = fma(b1, u1[jn], fma(b0, u0[jn], E[jm][jn]));
        }
        if (qs == Q - 1) {
          // element es done: E's rows into the pending rows es .. es+P-1
#pragma unroll
          for (int jm = 0; jm < P; ++jm) {
            const int sl = (es + jm) % P;
#pragma unroll
            for (int jn = 0; jn < P; ++jn) {
              double* q = pd + (size_t)(sl * W + jn - jm + P - 1) * NS3;
              *q += E[jm][jn];
              E[jm][jn] = 0.0;
            }
          }
          // row es is final (and, after the last element, rows es+1 .. es+P-1)
          const int nfin = es == a.K1 - 1 ? P : 1;
#pragma unroll 1
          for (int t = 0; t < nfin; ++t) {
            const int sl = (es + t) % P;
            double row[W];
#pragma unroll
            for (int kx = 0; kx < W; ++kx) {
              double* q = pd + (size_t)(sl * W + kx) * NS3;
              row[kx] = *q;
              *q = 0.0;
            }
            store_row(es + t, row);
          }
        }
      }
    }
    __syncthreads();
  }
}

// ---- host side -------------------------------------------------------------

template <int P>
bool sym2_fits(int nplanes, int ng) {
  using C = Sym2Cfg<P, Sym2Tile<P>::T0>;
  // worst-case chunk: capacity for the whole y range is checked at launch
  return ng <= 4 && C::smem(nplanes, 8 * P, 3 * P) <= 232448;
}

bool sym2_eligible(const igs_problem* p, const AsmShape& s, int64_t row_lo, int64_t row_hi) {
  if (s.fs.d != 2 || !problem_symmetric(p)) return false;
  if (p->slab_lo || p->slab_hi) return false;
  if (row_lo != 0 || row_hi != s.fs.nfn[0] * s.fs.nfn[1]) return false;  // whole matrix only
  switch (s.fs.p) {
    case 2: return sym2_fits<2>(p->n_planes, s.plan.ng);
    case 3: return sym2_fits<3>(p->n_planes, s.plan.ng);
    case 4: return sym2_fits<4>(p->n_planes, s.plan.ng);
    case 5: return sym2_fits<5>(p->n_planes, s.plan.ng);
    default: return false;
  }
}

template <int P>
igs_status launch2_sym(const igs_problem* p, const AsmShape& s, TensorPat pat, const double* planes,
                       double* values, cudaStream_t st) {
  constexpr int T0 = Sym2Tile<P>::T0;
  using C = Sym2Cfg<P, T0>;
  Sym2Args a{};
  a.tab = tab_args(p);
  a.pat = pat;
  a.values = values;
  a.nt0 = (int)ceil_div(s.fs.nfn[0], (int64_t)T0);
  a.nplanes = p->n_planes;
  a.K1 = (int)s.fs.nel[1];
  const int N1 = (int)s.fs.nfn[1];
  if (s.plan.ng > 4) return IGS_ECAPACITY;
  for (int v = 0; v < 4; ++v) a.vmap[v] = -1;
  for (int g = 0; g < s.plan.ng; ++g) a.vmap[s.plan.g_v1[g]] = g;
  a.nb = s.plan.nb;
  for (int b = 0; b < s.plan.nb; ++b) {
    a.b_plane[b] = s.plan.b_plane[b];
    a.b_v0[b] = s.plan.b_v0[b];
    a.b_g[b] = s.plan.b_g[b];
    if (b + 1 == s.plan.nb || s.plan.b_g[b + 1] != s.plan.b_g[b]) a.b_end |= 1u << b;
  }
  // y chunks: minimise waves x phases per chunk (rows + P - 1 lead elements),
  // one CTA per SM; the y-factor table bounds the chunk length
  int nch = 1;
  {
    double best = -1.0;
    for (int n = 1; n <= 64 && n <= N1; ++n) {
      const int rpc = (N1 + n - 1) / n;
      const double waves = std::ceil((double)a.nt0 * n / 148.0);
      const double cost = waves * std::ceil((double)(rpc + P - 1) * P / C::YT);
      if (best < 0 || cost < best - 1e-9) {
        best = cost;
        nch = n;
      }
    }
  }
  for (;;) {
    a.rows_per_chunk = (N1 + nch - 1) / nch;
    a.max_pts = (a.rows_per_chunk + P - 1) * P;
    a.yrows = a.rows_per_chunk + 2 * (P - 1);
    if (C::smem(a.nplanes, a.max_pts, a.yrows) <= 232448 || a.rows_per_chunk <= 1) break;
    ++nch;
  }
  nch = (N1 + a.rows_per_chunk - 1) / a.rows_per_chunk;
  const size_t smem = C::smem(a.nplanes, a.max_pts, a.yrows);
  if (smem > 232448) return IGS_ECAPACITY;
  if (((uintptr_t)planes & 15) != 0) return IGS_ECAPACITY;
  CUtensorMap fmap;
  {
    const int64_t dims[4] = {s.fs.npt[0], s.fs.npt[1], 1, p->n_planes};
    const unsigned box[4] = {(unsigned)C::XB0, (unsigned)C::YT, 1u, (unsigned)p->n_planes};
    IGS_TRY(planes_tensor_map(&fmap, planes, dims, p->plane_stride, box));
  }
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm2_sym<P, T0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem),
                     "smem attribute"));
  dim3 grid((unsigned)a.nt0, (unsigned)nch);
  asm2_sym<P, T0><<<grid, C::NT, smem, st>>>(a, fmap);
  IGS_LAUNCH_CHECK("asm2_sym");
  return IGS_OK;
}
