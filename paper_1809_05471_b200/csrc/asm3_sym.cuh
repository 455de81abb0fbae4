// K3s — one-pass symmetric 3D assembly (Alg. 1 fused over all three
// directions), included by assemble3d.cu inside its anonymous namespace.
//
// For a symmetric problem (trial == test, θ-set == η-set, F_{η,θ} = F_{θ,η};
// every BASELINE assembly) A = Aᵀ, so a CTA only forms the 1D x-pairs
// (m0, n0 = m0 + o0) with o0 >= 0 and writes every value twice: to its own
// row m and, for o0 > 0, mirrored to row n (column m).  Every entry of the
// CSR is written exactly once (o0 = 0 pairs cover all (o1, o2) directly).
//
// One CTA = T0 x T1 rows in (x, y), sweeping the z direction (all of it, or
// a chunk of rows) point layer by point layer:
//   TMA      coefficient region of the tile, all planes, (T+P-1)·Q points per
//            direction (the next layer is fetched as soon as stage 1 has
//            consumed the buffer, behind stages 2 and 3);
//   stage 1  G_g[y][s0] = Σ_{b∈g} Σ_x F_b[y][x] W0^{v0(b)}[x][s0]     DMMA (M=y, N=s0, K=x)
//   stage 2  H_h[s1][s0] = Σ_{g∈h} Σ_y W1^{v1(g)}[s1][y] G_g[y][s0]   DMMA (M=s1, N=s0, K=y)
//   stage 3  per thread = one (s0, s1) pair: the z contraction of the point
//            layer into the element matrix E[jm][jn] (registers); after the
//            element's last layer, row m2 = e is final -> CSR (+ mirror), and
//            the pending rows e+1 .. e+P-1 (shared memory) take E's rows.
// Nothing but the CSR values leaves the SM: G, H and the pending rows stay
// on chip (the two-kernel path writes H to HBM and reads it back).
//
// Slots: s0 = r0·P + o0 (o0 = n0 - m0 in [0, P)), s1 = r1·SR1 + (o1 + P - 1)
// (o1 in [-(P-1), P-1], rows padded to SR1 slots); tables are band tables
// restricted to the k-steps each MMA tile can touch.

// Measurement-only variants (tools/build_variant.sh; wrong values): 1 drops
// stage 3, 2 stage 2, 3 stage 1 of the phase loop, 4 the CSR stores of the
// finished rows.  The library builds 0.
#ifndef IGS_SYM_EXP
#define IGS_SYM_EXP 0
#endif
// Where stage 3 runs in a phase (measurement variants): 0 first, 1 last,
// 2 first on half the warps and last on the others (the library: each SMSP
// then mixes stage-3 FMA work with the other warps' DMMA work).
#ifndef IGS_SYM_S3_ORDER
#define IGS_SYM_S3_ORDER 2
#endif

template <int P, int T0, int T1>
struct SymCfg {
  static constexpr int Q = P;
  static constexpr int W = 2 * P - 1;
  static constexpr int NS0 = T0 * P;                 // symmetric x slots
  static constexpr int NST0 = (NS0 + 7) / 8;         // stage-1 / stage-2 n-tiles
  static constexpr int SR1 = W == 7 ? 8 : W;         // y slot positions per row
  static constexpr int NS1 = T1 * SR1;
  static constexpr int NMT1 = (NS1 + 7) / 8;         // stage-2 m-tiles
  static constexpr int NS1C = T1 * W;                // compact y slots (stage 3)
  static constexpr int NPAIR = NS0 * NS1C;           // pairs = stage-3 threads
  static constexpr int ER0 = T0 + P - 1, ER1 = T1 + P - 1;
  static constexpr int XR0 = ER0 * Q, XR1 = ER1 * Q;
  // TMA box width: >= XR0, a multiple of 4 doubles, pitch ≡ 4 or 12 (mod 16)
  // doubles so the A-fragment loads (8 rows x 4 columns) hit distinct banks
  static constexpr int box0() {
    int b = (XR0 + 3) & ~3;
    while (b % 16 != 4 && b % 16 != 12) b += 4;
    return b;
  }
  static constexpr int XB0 = box0();
  static constexpr int XRP1 = (XR1 + 7) & ~7;        // y rows of the stage-1 M tiles
  static constexpr int NYT = XRP1 / 8;
  static constexpr int NT = 512, NW = 16;
  static constexpr int pitch4(int n) { return ((n + 11) / 16) * 16 + 4; }
  static constexpr int SPG = pitch4(NS0);            // G row pitch
  static constexpr int HP = ((NS0 + 1) & ~1) + 4;   // H row pitch (even: double2 stores)
  // k-step range of stage-1 n-tile st (x points of its rows' supports)
  static constexpr int k0_lo(int st) { return ((8 * st) / P) * Q / 4; }
  static constexpr int r0_hi(int st) { return (8 * st + 7) / P < T0 - 1 ? (8 * st + 7) / P : T0 - 1; }
  static constexpr int k0_hi(int st) { return ((r0_hi(st) + P) * Q + 3) / 4; }
  static constexpr int ks0() {
    int m = 1;
    for (int st = 0; st < NST0; ++st) m = k0_hi(st) - k0_lo(st) > m ? k0_hi(st) - k0_lo(st) : m;
    return m;
  }
  static constexpr int KS0 = ks0();
  // k-step range of stage-2 m-tile mt (y points of its rows' supports)
  static constexpr int k1_lo(int mt) { return ((8 * mt) / SR1) * Q / 4; }
  static constexpr int r1_hi(int mt) { return (8 * mt + 7) / SR1 < T1 - 1 ? (8 * mt + 7) / SR1 : T1 - 1; }
  static constexpr int k1_hi(int mt) { return ((r1_hi(mt) + P) * Q + 3) / 4; }
  static constexpr int ks1() {
    int m = 1;
    for (int mt = 0; mt < NMT1; ++mt) m = k1_hi(mt) - k1_lo(mt) > m ? k1_hi(mt) - k1_lo(mt) : m;
    return m;
  }
  static constexpr int KS1 = ks1();
  static constexpr int w1p() {
    int b = KS1 * 4;
    while (b % 16 != 4 && b % 16 != 12) b += 4;
    return b;
  }
  static constexpr int W1P = w1p();                  // stage-2 A rows: pitch ≡ 4 or 12 (mod 16)
  static constexpr int PP = (P + 1) & ~1;            // z factor row (16-byte rows)
  static constexpr int FZ = Q * 4 * PP;              // z factors per element
  // shared memory plan (doubles)
  static constexpr size_t fbuf(int npl) { return ((size_t)npl * XR1 * XB0 + (size_t)(XRP1 - XR1 + 1) * XB0 + 15) & ~size_t(15); }
  static constexpr int W0R = 12;                     // stage-1 B rows: 8 slots, pitch ≡ 12 (mod 16)
  static constexpr size_t W0C = (size_t)4 * NST0 * KS0 * 4 * W0R;
  static constexpr size_t W1C = (size_t)4 * NMT1 * 8 * W1P;
  static constexpr size_t HS = (size_t)4 * NS1C * HP;
  static constexpr int FZL = (FZ + 31) / 32;        // z factors per lane of the prefetching warp
  // + z-row table: 3 int64 per DoF row of the chunk's sweep (zrows rows)
  static constexpr int NPEND = (P - 1) * (2 * P - 2) - (P - 1) * (P - 2) / 2;  // pending z values per pair
  static constexpr size_t smem(int npl, int ng, int zrows = 0) {
    return (fbuf(npl) + 2 * (size_t)ng * XRP1 * SPG + W0C + W1C + 2 * HS + 2 * FZ + 3 * (size_t)zrows) *
               sizeof(double) + 32;
  }
  static_assert(XR1 <= 256 && XB0 <= 256, "TMA box");
};

struct SymArgs {
  AsmPlan plan;
  TabArgs tab;
  TensorPat pat;
  double* values;
  const int64_t* base;   // CSR offset of row_lo (device scalar; null: row_lo = 0, offset 0)
  int64_t row_lo, row_hi;
  int nt0;               // tiles in x
  int nplanes;
  int64_t zpl;           // global z point of the planes' first layer
  int K2;                // elements in z
  int rows_per_chunk;    // z DoF rows written per chunk (grid.y)
  int m2a, m2b;          // z DoF rows of the range: [m2a, m2b)
  int zrows;             // capacity of the z-row table (rows_per_chunk + 6P)
  int hsplit;            // stage-2 groups [0, hsplit) | [hsplit, ng) (whole stage-2 groups)
  int vmap[4];           // stage-2 group holding z variant v = θ + 2η (-1: none)
  // compact plan for the kernel's runtime loops
  int b_plane[kMaxBlocks], b_v0[kMaxBlocks], b_g[kMaxBlocks];  // stage-1 blocks (group order)
  int nb1, half_b1;       // stage-1 blocks, split into two halves at a group boundary
  int g_v1[kMaxBlocks], g_h[kMaxBlocks];                       // per stage-1 group
  int g_src[kMaxBlocks];  // G buffer stage 2 reads for group g (groups with identical
                          // (plane, x variant) block sets share one stage-1 result)
  unsigned b_end, g_end;  // bit b: last block of its group; bit g: last group of its stage-2 group
};

// Band table of one direction for a tile, restricted per MMA tile:
//   TRANS = false (stage 1, B operand):  Wt[v][st][kk·4 + m][j] over x = region
//             k-step (k0_lo(st) + kk), slot s0 = 8·st + j  (symmetric slots)
//   TRANS = true  (stage 2, A operand):  Wt[v][mt][j][kk·4 + m] over y = region
//             k-step (k1_lo(mt) + kk), slot s1 = 8·mt + j
// value w(x)·B^θ_n(x)·B^η_m(x), v = θ + 2η, zero outside the supports.
template <int P, int T0, int T1, bool TRANS>
__device__ void sym_fill_table(double* Wt, const TabArgs& t, int dir, int a_row, int64_t x_first) {
  using C = SymCfg<P, T0, T1>;
  constexpr int Q = C::Q;
  constexpr int NTL = TRANS ? C::NMT1 : C::NST0;
  constexpr int KS = TRANS ? C::KS1 : C::KS0;
  constexpr int ROW = TRANS ? C::W1P : C::W0R;         // innermost pitch
  constexpr int TOT = 4 * NTL * (TRANS ? 8 * C::W1P : KS * 4 * C::W0R);
  const int64_t Nf = t.N[dir];
  for (int i = threadIdx.x; i < TOT; i += blockDim.x) {
    int v, tl, j, kx;
    if (TRANS) {
      kx = i % ROW;
      j = (i / ROW) % 8;
      tl = (i / (ROW * 8)) % NTL;
      v = i / (ROW * 8 * NTL);
    } else {
      j = i % ROW;
      kx = (i / ROW) % (KS * 4);
      tl = (i / (ROW * KS * 4)) % NTL;
      v = i / (ROW * KS * 4 * NTL);
    }
    double val = 0.0;
    const int s = 8 * tl + j;
    int r, m_off;  // tile row, n - m
    bool ok;
    if (TRANS) {
      r = s / C::SR1;
      m_off = s % C::SR1 - (P - 1);
      ok = r < T1 && s % C::SR1 < C::W && kx < KS * 4;
    } else {
      r = s / P;
      m_off = s % P;
      ok = r < T0 && j < 8;
    }
    if (ok) {
      const int klo = TRANS ? C::k1_lo(tl) : C::k0_lo(tl);
      const int64_t x = x_first + klo * 4 + kx;
      const int64_t m = a_row + r, n = m + m_off;
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

// z factors of element e: [q][wB^0 | wB^1 | B^0 | B^1][PP], entry i
template <int P>
__device__ __forceinline__ double sym_fz_value(const TabArgs& t, int e, int i) {
  constexpr int Q = P, PP = (P + 1) & ~1;
  if (i >= Q * 4 * PP) return 0.0;
  const int j = i % PP, f = (i / PP) % 4, q = i / (4 * PP);
  const int lvl = f & 1;
  if (j >= P || lvl > t.md[2]) return 0.0;
  const int64_t x = (int64_t)e * Q + q;
  const double b = t.vals[2][((int64_t)lvl * P + j) * t.X[2] + x];
  return f < 2 ? t.wts[2][x] * b : b;
}
template <int P>
__device__ void sym_fill_fz(double* fz, const TabArgs& t, int e, int tid, int nthr) {
  constexpr int FZ = P * 4 * ((P + 1) & ~1);
  for (int i = tid; i < FZ; i += nthr) fz[i] = sym_fz_value<P>(t, e, i);
}

// Write row m2's 2P-1 columns (ring[0]) to its CSR row, and the mirrors
// (o0 > 0) to the rows n = (n0, n1, n2) at column m.
// Which copies of pair value (o0, o1, o2) = (n - m) a CTA writes: o0 > 0 both
// the entry and its mirror; o0 = 0 (the pair is its own mirror class) only
// the lexicographically non-negative (o1, o2), mirrored when positive, so
// A = Aᵀ holds bit for bit.
__device__ __forceinline__ bool sym_keep(int o0, int o1, int o2) {
  return o0 > 0 || o1 > 0 || (o1 == 0 && o2 >= 0);
}
__device__ __forceinline__ bool sym_mirror(int o0, int o1, int o2) {
  return o0 > 0 || o1 > 0 || (o1 == 0 && o2 > 0);
}

// Pending z rows of a pair between elements: after element e, rows e+1+a
// (age a = 0 .. P-2) hold the contributions of elements <= e, columns
// k = n2 - m2 + P - 1 in [0, 2P-3-a].  Stored in shared memory per pair.
template <int P>
struct Pend {
  static constexpr int off(int a) { return a * (2 * P - 2) - a * (a - 1) / 2; }
  static constexpr int len(int a) { return 2 * P - 2 - a; }
  static constexpr int N = off(P - 1);
};

// Write row m2's 2P-1 values (ROW[k], k = n2 - m2 + P - 1) to its CSR row and
// the mirrors to rows n.  Fast path (uniform per element): every row within
// P-1 of m2 is an interior row (1D width 2P-1) inside the written range, so
// the offsets are affine in k; else the general path through the z-row table.
#define IGS_SYM_STORE(M2, ROW)                                                               \
  do {                                                                                       \
    const int m2_ = (M2);                                                                    \
    if (valid) {                                                                             \
      const int64_t* zm = ZR + 3 * (m2_ - zr0);                                              \
      if (m2_ >= fw_lo && m2_ < fw_hi) {                                                     \
        double* vd = a.values + (zm[0] + dBase);                                             \
        double* vm = a.values + (zm[0] + mBase);                                             \
        _Pragma("unroll") for (int k = 0; k < W; ++k) {                                      \
          if (keepm & (1u << k)) vd[(int64_t)k * dD] = ROW[k];                               \
          if (mirm & (1u << k)) vm[(int64_t)k * mStep] = ROW[k];                             \
        }                                                                                    \
      } else {                                                                               \
        const bool dir_ok = m2_ >= r_lo && m2_ < r_hi;                                       \
        const int64_t mrow = m_flat0 + layer * m2_;                                          \
        const int64_t dstart = dA * zm[1] + zm[0] - zm[2] * dD + dC;                         \
        _Pragma("unroll") for (int k = 0; k < W; ++k) {                                      \
          const int n2 = m2_ + k - (P - 1);                                                  \
          if (n2 < 0 || n2 >= N2) continue;                                                  \
          if ((keepm & (1u << k)) && dir_ok && mrow >= a.row_lo && mrow < a.row_hi)          \
            a.values[dstart + (int64_t)n2 * dD] = ROW[k];                                    \
          if ((mirm & (1u << k)) && n2 >= r_lo && n2 < r_hi) {                               \
            const int64_t nrow = n_flat0 + layer * n2;                                       \
            if (nrow >= a.row_lo && nrow < a.row_hi) {                                       \
              const int64_t* zn = ZR + 3 * (n2 - zr0);                                       \
              a.values[mA * zn[1] + zn[0] + (m2_ - zn[2]) * mD + mC] = ROW[k];               \
            }                                                                                \
          }                                                                                  \
        }                                                                                    \
      }                                                                                      \
    }                                                                                        \
  } while (0)

// TMEM (tcgen05) helpers: the pending z rows live in tensor memory, one
// private 32-column slice of its lane per thread (warp w owns lanes
// 32·(w % 4) .. +31; warps w, w+4, w+8, w+12 take column groups 0..3).
// issue only: tcgen05.wait::ld before the registers are used
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");  // the previous store has landed
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

template <int P, int T0, int T1>
__global__ void __launch_bounds__(512, 1)
    asm3_sym(const SymArgs a, const __grid_constant__ CUtensorMap fmap) {
  using C = SymCfg<P, T0, T1>;
  using PD = Pend<P>;
  constexpr int Q = C::Q, W = C::W, NS0 = C::NS0, NST0 = C::NST0, SR1 = C::SR1, NMT1 = C::NMT1;
  constexpr int XB0 = C::XB0, XR1 = C::XR1, XRP1 = C::XRP1, NYT = C::NYT, SPG = C::SPG, HP = C::HP;
  constexpr int KS0 = C::KS0, W0R = C::W0R, KS1 = C::KS1, W1P = C::W1P, PP = C::PP, FZ = C::FZ;
  constexpr int NT = C::NT, NW = C::NW, NPAIR = C::NPAIR, NPW = (NPAIR + 31) / 32;
  static_assert(2 * PD::N <= 32 && 2 * P * P <= 32, "pending rows and E fit 32-column TMEM slices");
  static_assert(NPAIR <= NT, "one pair per thread");
  extern __shared__ __align__(128) double sm[];
  const int ng = a.plan.ng;
  const size_t fb = C::fbuf(a.nplanes);
  const size_t gsz = (size_t)ng * XRP1 * SPG;
  double* Fs = sm;                                   // [npl][XR1][XB0] (+ zero tail)
  double* Gs = Fs + fb;                              // [2][ng][XRP1][SPG]
  double* W0 = Gs + 2 * gsz;                         // [4][NST0][KS0·4][W0R]
  double* W1 = W0 + C::W0C;                          // [4][NMT1][8][W1P]
  double* Hs = W1 + C::W1C;                          // [2][4][NS1C][HP]
  double* FZs = Hs + 2 * C::HS;                      // [2][FZ]
  int64_t* ZR = reinterpret_cast<int64_t*>(FZs + 2 * FZ);  // [zrows][3]
  uint64_t* bar = reinterpret_cast<uint64_t*>(ZR + 3 * (size_t)a.zrows);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, m4 = lane & 3;
  const int t0 = blockIdx.x % a.nt0, t1 = blockIdx.x / a.nt0;
  const int a0 = t0 * T0, a1 = t1 * T1;
  const int xb0 = (a0 - (P - 1)) * Q, xb1 = (a1 - (P - 1)) * Q;
  // z rows written by this chunk, and the elements that complete the rows
  // whose values (direct or mirrored) land in them
  const int r_lo = a.m2a + blockIdx.y * a.rows_per_chunk;
  const int r_hi = min(a.m2b, r_lo + a.rows_per_chunk);
  const int e_lo = max(0, r_lo - 2 * (P - 1));
  const int e_hi = min(a.K2, r_hi + P - 1);
  const int64_t N0 = a.tab.N[0], N1 = a.tab.N[1], N2 = a.tab.N[2];
  const int64_t layer = N0 * N1;
  const unsigned fbytes = (unsigned)((size_t)a.nplanes * XR1 * XB0 * sizeof(double));
  const int nz = (e_hi - e_lo) * Q;

  // ---- prologue: TMEM, zeroed shared memory, tables, barrier, first layer ---
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
                     dev::smem_u32(tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  for (size_t i = tid; i < fb + 2 * gsz; i += NT) sm[i] = 0.0;
  for (int i = tid; i < 2 * (int)C::HS; i += NT) Hs[i] = 0.0;
  if (tid == 0) {
    dev::mbar_init(bar, 1);
    dev::fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // per thread 64 TMEM columns of its lane: [0, 32) pending rows, [32, 64)
  // the element matrix E[jm][jn] being accumulated (registers only in stage 3)
  const uint32_t taddr = *tmem_holder + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
  dev::fence_proxy_async();
  __syncthreads();
  if (tid == 0 && nz > 0) {
    dev::mbar_expect_tx(bar, fbytes);
    dev::tma_load_4d(Fs, &fmap, bar, xb0, xb1, (int)((int64_t)e_lo * Q - a.zpl), 0);
  }
  sym_fill_table<P, T0, T1, false>(W0, a.tab, 0, a0, xb0);
  sym_fill_table<P, T0, T1, true>(W1, a.tab, 1, a1, xb1);
  if (e_lo < e_hi) sym_fill_fz<P>(FZs, a.tab, e_lo, tid, NT);
  if (warp < NPW) {  // pending rows start at zero
    uint32_t z[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) z[i] = 0u;
    tmem_st32(taddr, z);
    tmem_st32(taddr + 32, z);
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }

  // ---- this thread's (s0, s1) pair and its CSR addressing ------------------
  const int s0 = tid % NS0, s1c = tid / NS0;
  const int r0 = s0 / P, o0 = s0 % P, r1 = s1c / W, o1 = s1c % W - (P - 1);
  const int64_t m0 = a0 + r0, n0 = m0 + o0, m1 = a1 + r1, n1 = m1 + o1;
  const bool valid = tid < NPAIR && m0 < N0 && n0 < N0 && m1 < N1 && n1 >= 0 && n1 < N1 &&
                     (o0 > 0 || o1 >= 0);  // o0 = 0, o1 < 0: the mirror of another pair
  unsigned keepm = 0, mirm = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    keepm |= (valid && sym_keep(o0, o1, k - (P - 1)) ? 1u : 0u) << k;
    mirm |= (valid && sym_mirror(o0, o1, k - (P - 1)) ? 1u : 0u) << k;
  }
  // row m: start = (rp0[m0]·w1 + P0·rp1[m1])·w2 + P0·P1·rp2[m2]; entry offset
  // (n2 - lo2)·w0·w1 + (n1 - lo1)·w0 + (n0 - lo0); the mirror the same for
  // row n with the roles of m and n exchanged
  int64_t dA = 0, mA = 0;
  int dD = 0, dC = 0, mD = 0, mC = 0;
  const int64_t* rp0 = a.pat.rp[0];
  const int64_t* rp1 = a.pat.rp[1];
  const int64_t P0 = rp0[N0], P1 = rp1[N1], P01 = P0 * P1;
  if (valid) {
    const int64_t w0m = rp0[m0 + 1] - rp0[m0], w1m = rp1[m1 + 1] - rp1[m1];
    dA = rp0[m0] * w1m + P0 * rp1[m1];
    dD = (int)(w0m * w1m);
    dC = (int)((n1 - a.pat.cl[1][rp1[m1]]) * w0m + (n0 - a.pat.cl[0][rp0[m0]]));
    const int64_t w0n = rp0[n0 + 1] - rp0[n0], w1n = rp1[n1 + 1] - rp1[n1];
    mA = rp0[n0] * w1n + P0 * rp1[n1];
    mD = (int)(w0n * w1n);
    mC = (int)((m1 - a.pat.cl[1][rp1[n1]]) * w0n + (m0 - a.pat.cl[0][rp0[n0]]));
  }
  // fast-path offsets (interior z rows: width W, lo2 = m2 - P + 1):
  //   direct  zm0 + dA·W + dC + k·dD
  //   mirror  zm0 + mA·W + mC + P01·W·(k - P + 1) + (2P - 2 - k)·mD
  const int64_t dBase = dA * W + dC;
  const int64_t mBase = mA * W + mC + (int64_t)(2 * P - 2) * mD - P01 * W * (P - 1);
  const int64_t mStep = P01 * W - mD;
  const int64_t base = a.base ? *a.base : 0;
  const int64_t m_flat0 = m0 + N0 * m1, n_flat0 = n0 + N0 * n1;
  // z-row table of the rows this chunk completes or mirrors into
  const int zr0 = max(0, e_lo - (P - 1));
  const int zr1 = min((int)N2, e_hi + 2 * (P - 1));
  {
    const int64_t* rp2 = a.pat.rp[2];
    const int64_t* cl2 = a.pat.cl[2];
    for (int r = zr0 + tid; r < zr1; r += NT) {
      const int64_t rs = rp2[r];
      ZR[3 * (r - zr0)] = P01 * rs - base;
      ZR[3 * (r - zr0) + 1] = rp2[r + 1] - rs;
      ZR[3 * (r - zr0) + 2] = cl2[rs];
    }
  }
  // fast rows: all rows within P-1 interior, in [r_lo, r_hi) and in whole
  // layers of [row_lo, row_hi)
  const int lay_lo = (int)((a.row_lo + layer - 1) / layer), lay_hi = (int)(a.row_hi / layer);
  const int fw_lo = max(max(2 * (P - 1), r_lo + P - 1), lay_lo + P - 1);
  const int fw_hi = min(min(a.K2 - P + 1, r_hi - P + 1), lay_hi - P + 1);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // stage-1 tasks: (y tile, n-tile, half of the blocks); warp w runs on SMSP
  // w % 4, so each SMSP gets one y tile's tasks
  const int nt1 = 2 * NYT * NST0;
  // stage-2 tasks: (m-tile, n-tile, half of the stage-2 groups); halves
  // alternate across SMSPs so each SMSP gets both
  const int nt2 = NMT1 * NST0 * 2;
  unsigned ph = 0u;
  double fzr[C::FZL];

  // stage 1 of point layer iz (F in smem) into G buffer gb
  auto stage1 = [&](double* Gb) {
    for (int t = warp; t < nt1; t += NW) {
      const int yt = t % NYT, st = (t / NYT) % NST0, half = t / (NYT * NST0);
      const int b_lo = half ? a.half_b1 : 0, b_hi = half ? a.nb1 : a.half_b1;
      int klo = 0;
#pragma unroll
      for (int i = 0; i < NST0; ++i)
        if (i == st) klo = C::k0_lo(i);
      const double* Fy = Fs + (yt * 8 + g8) * XB0 + m4 + klo * 4;
      const double* Wk = W0 + (st * KS0 * 4 + m4) * W0R + g8;
      double* Gy = Gb + (yt * 8 + g8) * SPG + st * 8 + 2 * m4;
      const bool st_ok = st * 8 + 2 * m4 < NS0;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll 1
      for (int b = b_lo; b < b_hi; ++b) {
        const double* Fp = Fy + a.b_plane[b] * (XR1 * XB0);
        const double* Wv = Wk + a.b_v0[b] * (NST0 * KS0 * 4 * W0R);
        double f[KS0], w[KS0];
#pragma unroll
        for (int kk = 0; kk < KS0; ++kk) {
          f[kk] = Fp[kk * 4];
          w[kk] = Wv[kk * 4 * W0R];
        }
#pragma unroll
        for (int kk = 0; kk < KS0; ++kk) dmma_a(c0, c1, f[kk], w[kk]);
        if ((a.b_end >> b) & 1) {
          if (st_ok) *reinterpret_cast<double2*>(Gy + a.b_g[b] * (XRP1 * SPG)) = make_double2(c0, c1);
          c0 = c1 = 0.0;
        }
      }
    }
  };
  if (nz > 0) {
    dev::mbar_wait(bar, ph);
    ph ^= 1u;
    stage1(Gs);
  }
  __syncthreads();
  if (tid == 0 && nz > 1) {
    dev::fence_proxy_async();
    dev::mbar_expect_tx(bar, fbytes);
    dev::tma_load_4d(Fs, &fmap, bar, xb0, xb1, (int)((int64_t)e_lo * Q + 1 - a.zpl), 0);
  }

  // stage 3 of layer k-1: this thread's pair, point layer -> E; element end
  // -> row out, pending rows (TMEM) updated
  auto stage3 = [&](int k) {
    if (k >= 1 && warp < NPW) {
      const int z = k - 1, es = e_lo + z / Q, qs = z % Q;
      const double* fq = FZs + ((es - e_lo) & 1) * FZ + qs * 4 * PP;
      const double* hcol = Hs + (z & 1) * C::HS + s1c * HP + s0;
      uint32_t er[32];
      tmem_ld32(taddr + 32, er);  // E of this element so far, in flight during the smem loads
      double hv[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) hv[v] = a.vmap[v] >= 0 ? hcol[a.vmap[v] * (C::NS1C * HP)] : 0.0;
      double fbv[4][P];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int j = 0; j < P; j += 2) {
          if (j + 1 < P) {
            const double2 tt = *reinterpret_cast<const double2*>(fq + f * PP + j);
            fbv[f][j] = tt.x;
            fbv[f][j + 1] = tt.y;
          } else {
            fbv[f][j] = fq[f * PP + j];
          }
        }
      // Σ_{θ,η} (w·B^θ_jn)(B^η_jm) H_{θ+2η}: θ first (u_η[jn]), then η
      tmem_wait_ld();
      double E[P][P];
#pragma unroll
      for (int jm = 0; jm < P; ++jm)
#pragma unroll
        for (int jn = 0; jn < P; ++jn) E[jm][jn] = u2d(er[2 * (jm * P + jn)], er[2 * (jm * P + jn) + 1]);
      double u0[P], u1[P];
#pragma unroll
      for (int jn = 0; jn < P; ++jn) {
        u0[jn] = fma(fbv[1][jn], hv[1], fbv[0][jn] * hv[0]);
        u1[jn] = fma(fbv[1][jn], hv[3], fbv[0][jn] * hv[2]);
      }
#pragma unroll
      for (int jm = 0; jm < P; ++jm)
#pragma unroll
        for (int jn = 0; jn < P; ++jn) E[jm][jn] = fma(fbv[3][jm], u1[jn], fma(fbv[2][jm], u0[jn], E[jm][jn]));
      if (qs == Q - 1) {
        // element es done: row es is final; the pending rows move up one age
        uint32_t rr[32];
        tmem_ld32(taddr, rr);
        tmem_wait_ld();
        double row[W];
#pragma unroll
        for (int kx = 0; kx < W; ++kx) {
          double v = kx < PD::len(0) ? u2d(rr[2 * (PD::off(0) + kx)], rr[2 * (PD::off(0) + kx) + 1]) : 0.0;
          if (kx >= P - 1) v += E[0][kx - (P - 1)];
          row[kx] = v;
        }
        // age ag <- age ag+1 + E[ag+1] (row es+1+ag, kx = jn + P - 2 - ag)
#pragma unroll
        for (int ag = 0; ag < P - 1; ++ag) {
#pragma unroll
          for (int kx = 0; kx < PD::len(ag); ++kx) {
            const int src = PD::off(ag + 1) + kx;
            double v = (ag + 1 < P - 1 && kx < PD::len(ag + 1)) ? u2d(rr[2 * src], rr[2 * src + 1]) : 0.0;
            const int jn = kx - (P - 2 - ag);
            if (jn >= 0 && jn < P) v += E[ag + 1][jn];
            const int dst = PD::off(ag) + kx;
            rr[2 * dst] = (uint32_t)__double2loint(v);
            rr[2 * dst + 1] = (uint32_t)__double2hiint(v);
          }
        }
        tmem_st32(taddr, rr);
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
          for (int j = 0; j < P; ++j) E[i][j] = 0.0;
#if IGS_SYM_EXP != 4
        IGS_SYM_STORE(es, row);
#endif
      }
#pragma unroll
      for (int jm = 0; jm < P; ++jm)
#pragma unroll
        for (int jn = 0; jn < P; ++jn) {
          er[2 * (jm * P + jn)] = (uint32_t)__double2loint(E[jm][jn]);
          er[2 * (jm * P + jn) + 1] = (uint32_t)__double2hiint(E[jm][jn]);
        }
      tmem_st32(taddr + 32, er);
    }
  };

  // ---- one phase per point layer k: stage 3 of k-1, stage 2 of k, stage 1
  // of k+1 (G, H double-buffered), one barrier --------------------------------
#pragma unroll 1
  for (int k = 0; k <= nz; ++k) {
    // ---- stage 3 of layer k-1 ------------------------------------------------
#if IGS_SYM_EXP != 1 && IGS_SYM_S3_ORDER == 0
    stage3(k);
#elif IGS_SYM_S3_ORDER == 2
    if (((warp >> 2) & 1) == 0) stage3(k);
#endif
    // next element's z factors: loaded at the first layer of an element (in
    // stage 3 terms), stored one phase later (the other buffer's last reader,
    // the previous element's stage 3, finished two barriers before)
    if (warp == NW - 1 && k >= 1) {
      const int z = k - 1, es = e_lo + z / Q, qs = z % Q;
      if (es + 1 < e_hi) {
        if (qs == 0) {
#pragma unroll
          for (int i = 0; i < C::FZL; ++i) fzr[i] = sym_fz_value<P>(a.tab, es + 1, lane + 32 * i);
        } else if (qs == 1) {
          double* dst = FZs + ((es + 1 - e_lo) & 1) * FZ;
#pragma unroll
          for (int i = 0; i < C::FZL; ++i)
            if (lane + 32 * i < FZ) dst[lane + 32 * i] = fzr[i];
        }
      }
    }
    // ---- stage 2 of layer k: G[k&1] -> H[k&1] ---------------------------------
    if (k < nz && IGS_SYM_EXP != 2) {
      const double* Gb = Gs + (k & 1) * gsz;
      double* Hb = Hs + (k & 1) * C::HS;
      for (int t = warp; t < nt2; t += NW) {
        const bool by8 = nt2 % 8 == 0;
        const int hh = by8 ? (t >> 2) & 1 : t & 1;
        const int rest = by8 ? (t & 3) | ((t >> 3) << 2) : t >> 1;
        const int mt = rest / NST0, st = rest % NST0;
        const int g_lo = hh ? a.hsplit : 0, g_hi = hh ? ng : a.hsplit;
        const int s1 = mt * 8 + g8;
        const int rr1 = s1 / SR1, oo1 = s1 % SR1;
        const int sc = 8 * st + 2 * m4;
        const bool h_ok = rr1 < T1 && oo1 < W && sc < NS0;
        double* Hd = Hb + (rr1 * W + oo1) * HP + sc;
        const double* Wk = W1 + (mt * 8 + g8) * W1P + m4;
        int klo = 0;
#pragma unroll
        for (int i = 0; i < NMT1; ++i)
          if (i == mt) klo = C::k1_lo(i);
        const double* Gk = Gb + (klo * 4 + m4) * SPG + 8 * st + g8;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll 1
        for (int g = g_lo; g < g_hi; ++g) {
          const double* Wg = Wk + a.g_v1[g] * (NMT1 * 8 * W1P);
          const double* Gg = Gk + a.g_src[g] * (XRP1 * SPG);
          double wv[KS1], gv[KS1];
#pragma unroll
          for (int kk = 0; kk < KS1; ++kk) {
            wv[kk] = Wg[kk * 4];
            gv[kk] = Gg[kk * 4 * SPG];
          }
#pragma unroll
          for (int kk = 0; kk < KS1; ++kk) dmma_a(d0, d1, wv[kk], gv[kk]);
          if ((a.g_end >> g) & 1) {
            if (h_ok) *reinterpret_cast<double2*>(Hd + a.g_h[g] * (C::NS1C * HP)) = make_double2(d0, d1);
            d0 = d1 = 0.0;
          }
        }
      }
    }
    // ---- stage 1 of layer k+1: F -> G[(k+1)&1] ---------------------------------
    if (k + 1 < nz) {
      dev::mbar_wait(bar, ph);
      ph ^= 1u;
#if IGS_SYM_EXP != 3
      stage1(Gs + ((k + 1) & 1) * gsz);
#endif
    }
#if IGS_SYM_S3_ORDER == 1
    stage3(k);
#elif IGS_SYM_S3_ORDER == 2
    if (((warp >> 2) & 1) == 1) stage3(k);
#endif
    __syncthreads();
    // F is consumed: fetch layer k+2 behind the next phase's stages 3 and 2
    if (tid == 0 && k + 2 < nz) {
      dev::fence_proxy_async();
      dev::mbar_expect_tx(bar, fbytes);
      dev::tma_load_4d(Fs, &fmap, bar, xb0, xb1, (int)((int64_t)e_lo * Q + k + 2 - a.zpl), 0);
    }
  }
  // trailing rows K2 + ag (age ag after the last element)
  if (e_hi == a.K2 && e_lo < e_hi && warp < NPW) {
    uint32_t rr[32];
    tmem_ld32(taddr, rr);
    tmem_wait_ld();
#pragma unroll
    for (int ag = 0; ag < P - 1; ++ag) {
      double row[W];
#pragma unroll
      for (int kx = 0; kx < W; ++kx)
        row[kx] = kx < PD::len(ag) ? u2d(rr[2 * (PD::off(ag) + kx)], rr[2 * (PD::off(ag) + kx) + 1]) : 0.0;
      IGS_SYM_STORE(a.K2 + ag, row);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(*tmem_holder));
  }
}

#undef IGS_SYM_STORE

// ---- host side -------------------------------------------------------------

// Tile of the symmetric kernel per order: about NT pairs (one per thread).
template <int P> struct SymTile;
template <> struct SymTile<2> { static constexpr int T0 = 8, T1 = 10; };
template <> struct SymTile<3> { static constexpr int T0 = 5, T1 = 6; };
template <> struct SymTile<4> { static constexpr int T0 = 4, T1 = 4; };

// A = Aᵀ structurally: same bases/tables for trial and test, θ-set == η-set,
// F_{η,θ} and F_{θ,η} the same plane (or both zero).
bool problem_symmetric(const igs_problem* p) {
  if (p->n_theta != p->n_eta) return false;
  for (int j = 0; j < p->n_theta; ++j)
    for (int k = 0; k < p->d; ++k)
      if (p->theta[j][k] != p->eta[j][k]) return false;
  for (int i = 0; i < p->n_eta; ++i)
    for (int j = 0; j < p->n_theta; ++j)
      if (p->plane_of[i][j] != p->plane_of[j][i]) return false;
  return true;
}

template <int P>
bool sym_fits(const AsmPlan& pl, int nplanes, int64_t zrows) {
  using C = SymCfg<P, SymTile<P>::T0, SymTile<P>::T1>;
  return pl.nh <= 4 && C::smem(nplanes, pl.ng, (int)zrows) <= 232448;
}

// zrows: DoF rows of the last direction (the z-row table holds at most
// min(rows, 1024) + 6P of them)
bool sym_fits_for(int P, const AsmPlan& pl, int nplanes, int64_t rows) {
  const int64_t zr = (rows < 1024 ? rows : 1024) + 6 * P;
  switch (P) {
    case 2: return sym_fits<2>(pl, nplanes, zr);
    case 3: return sym_fits<3>(pl, nplanes, zr);
    case 4: return sym_fits<4>(pl, nplanes, zr);
    default: return false;
  }
}

// Launch over z DoF rows [m2a, m2b) (whole layers); the coefficient planes
// hold elements [z.sl, z.sh).  Returns IGS_ECAPACITY (caller falls back)
// when a chunk needs elements outside the slab.
template <int P>
igs_status launch3_sym(const igs_problem* p, const AsmShape& s, TensorPat pat, int64_t row_lo, int64_t row_hi,
                       const int64_t* base, const double* planes, double* values, int sl, int sh,
                       cudaStream_t st) {
  constexpr int T0 = SymTile<P>::T0, T1 = SymTile<P>::T1;
  using C = SymCfg<P, T0, T1>;
  const int K2 = (int)s.fs.nel[2];
  const int64_t layer = s.fs.nfn[0] * s.fs.nfn[1];
  SymArgs a{};
  a.plan = s.plan;
  a.tab = tab_args(p);
  a.pat = pat;
  a.values = values;
  a.base = base;
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  a.nt0 = (int)ceil_div(s.fs.nfn[0], T0);
  const int nt1 = (int)ceil_div(s.fs.nfn[1], T1);
  a.nplanes = p->n_planes;
  a.zpl = (int64_t)sl * P;
  a.K2 = K2;
  // z DoF layers touched by the range; partial layers are cut by the
  // kernel's flat-row checks
  a.m2a = (int)(row_lo / layer);
  a.m2b = (int)((row_hi + layer - 1) / layer);
  // stage-2 group halves: whole stage-2 groups, balanced by group count
  {
    int best = 1 << 30;
    a.hsplit = s.plan.ng;
    for (int h = 1; h <= s.plan.nh; ++h) {
      const int end = h < s.plan.nh ? s.plan.h_g0[h] : s.plan.ng;
      const int imb = std::abs(2 * end - s.plan.ng);
      if (imb < best) {
        best = imb;
        a.hsplit = end;
      }
    }
  }
  for (int v = 0; v < 4; ++v) a.vmap[v] = -1;
  for (int h = 0; h < s.plan.nh; ++h) a.vmap[s.plan.h_v2[h]] = h;
  // stage-1 groups whose blocks read the same (plane, x variant) set compute
  // the same G (3D M+K: the two a12 blocks, θ/η = e2/e3 and e3/e2, both use
  // the x variant 0): contract it once, let stage 2 read it for both
  {
    auto key = [&](int g) {
      int k[kMaxBlocks], n = 0;
      for (int b = s.plan.g_b0[g]; b < s.plan.g_b0[g] + s.plan.g_nb[g]; ++b)
        k[n++] = s.plan.b_plane[b] * 4 + s.plan.b_v0[b];
      std::sort(k, k + n);
      long long h = n;
      for (int i = 0; i < n; ++i) h = h * 1031 + k[i];
      return h;
    };
    for (int g = 0; g < s.plan.ng; ++g) {
      a.g_src[g] = g;
      for (int q = 0; q < g; ++q)
        if (a.g_src[q] == q && key(q) == key(g)) {
          a.g_src[g] = q;
          break;
        }
    }
    int nb = 0;
    for (int b = 0; b < s.plan.nb; ++b) {
      const int g = s.plan.b_g[b];
      if (a.g_src[g] != g) continue;
      a.b_plane[nb] = s.plan.b_plane[b];
      a.b_v0[nb] = s.plan.b_v0[b];
      a.b_g[nb] = g;
      ++nb;
    }
    a.nb1 = nb;
    for (int b = 0; b < nb; ++b)
      if (b + 1 == nb || a.b_g[b + 1] != a.b_g[b]) a.b_end |= 1u << b;
    // halves at a group boundary, balanced by block count
    a.half_b1 = nb;
    int best = 1 << 30;
    for (int b = 0; b + 1 < nb; ++b)
      if ((a.b_end >> b) & 1) {
        const int imb = std::abs(2 * (b + 1) - nb);
        if (imb < best) {
          best = imb;
          a.half_b1 = b + 1;
        }
      }
  }
  for (int g = 0; g < s.plan.ng; ++g) {
    a.g_v1[g] = s.plan.g_v1[g];
    a.g_h[g] = s.plan.g_h[g];
    if (g + 1 == s.plan.ng || s.plan.g_h[g + 1] != s.plan.g_h[g]) a.g_end |= 1u << g;
  }
  // z chunks: minimise waves x elements swept per chunk (rows + 3(P-1) lead)
  const int rows = a.m2b - a.m2a;
  const int64_t tiles = (int64_t)a.nt0 * nt1;
  int nch = 1;
  {
    double best = -1.0;
    for (int n = 1; n <= 16 && n <= rows; ++n) {
      const int rpc = (rows + n - 1) / n;
      const double waves = std::ceil((double)tiles * n / 148.0);
      const double cost = waves * (rpc + 3 * (P - 1));
      if (best < 0 || cost < best - 1e-9) {
        best = cost;
        nch = n;
      }
    }
  }
  a.rows_per_chunk = (rows + nch - 1) / nch;
  if (a.rows_per_chunk > 1024) a.rows_per_chunk = 1024;  // bounds the z-row table
  nch = (rows + a.rows_per_chunk - 1) / a.rows_per_chunk;
  a.zrows = a.rows_per_chunk + 6 * P;
  // every chunk's elements must be in the planes
  {
    const int e_need_lo = std::max(0, a.m2a - 2 * (P - 1));
    const int e_need_hi = std::min(K2, a.m2b + P - 1);
    if (e_need_lo < sl || e_need_hi > sh) return IGS_ECAPACITY;
  }
  const size_t smem = C::smem(a.nplanes, s.plan.ng, a.zrows);
  if (smem > 232448) return IGS_ECAPACITY;
  CUtensorMap fmap;
  {
    const int64_t dims[4] = {s.fs.npt[0], s.fs.npt[1], (int64_t)(sh - sl) * P, p->n_planes};
    const unsigned box[4] = {(unsigned)C::XB0, (unsigned)C::XR1, 1u, (unsigned)p->n_planes};
    IGS_TRY(planes_tensor_map(&fmap, planes, dims, p->plane_stride, box));
  }
  IGS_TRY(cuda_check(cudaFuncSetAttribute(asm3_sym<P, T0, T1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem),
                     "smem attribute"));
  dim3 grid((unsigned)tiles, (unsigned)nch);
  asm3_sym<P, T0, T1><<<grid, C::NT, smem, st>>>(a, fmap);
  IGS_LAUNCH_CHECK("asm3_sym");
  return IGS_OK;
}
