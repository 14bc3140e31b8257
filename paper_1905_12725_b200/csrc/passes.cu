// passes.cu — the five FFT passes of one DBFFT operator application.
//
//   I1 (z inverse, xi_z terms)  ->  I2 (y inverse, xi_x/xi_y terms)  ->  X (x C2R, contraction
//   C(x):eps or K(x):G, x R2C, xi_x fold)  ->  F2 (y forward, xi_y fold)  ->  F3 (z forward,
//   divergence, fused <p, Kp>)
//
// implements f = -d:F(C:F^-1(s.u)) (P:118 Eq. lineqf, positive form R3) with the gradient s
// / g (R2) applied per axis right before that axis is transformed ("deferred
// gradient") and the divergence d folded per axis right after ("early divergence"),
// so fewer than 2c fields cross the y and z sweeps (52 H / 66 H complex moves).
#include "passes.cuh"

#include <algorithm>

namespace {

// ------------------------------------------------------------------------------------------------
// Column passes
// ------------------------------------------------------------------------------------------------
struct ColAt {
  const ColGeom* g;
  int outer, pos, kx;
  DBF_DEV long long in_idx(int f) const {
    long long p = (long long)(pos >> g->in_psh) * g->in_pcs + (long long)(pos & ((1 << g->in_psh) - 1)) * g->in_ps;
    return f * g->in_fs + outer * g->in_os + p + kx;
  }
  DBF_DEV long long out_idx(int f) const {
    long long p = (long long)(pos >> g->out_psh) * g->out_pcs + (long long)(pos & ((1 << g->out_psh) - 1)) * g->out_ps;
    return f * g->out_fs + outer * g->out_os + p + kx;
  }
  DBF_DEV cplx in(int f) const { return __ldg(g->in + in_idx(f)); }
};

template <int KIND>
struct ColOp;

// z inverse, small strain.  outer = ky, pos = kz.
template <>
struct ColOp<COL_I1S> {
  static constexpr bool INV = true;
  static constexpr int NOUT = 5;
  DBF_DEV static int nterms(int) { return 1; }
  DBF_DEV static cplx load(const ColAt& a, int o, int) {
    const double xx = __ldg(a.g->fq.xx + a.kx), xy = __ldg(a.g->fq.xy + a.outer), xz = __ldg(a.g->fq.xz + a.pos);
    switch (o) {
      case 0: return a.in(0);
      case 1: return a.in(1);
      case 2: return cimul(a.in(2), xz);                                               // eps_zz
      case 3: { cplx u0 = a.in(0), u2 = a.in(2); return cimul(make_double2(xz * u0.x + xx * u2.x, xz * u0.y + xx * u2.y), 0.5); }  // eps_xz
      default: { cplx u1 = a.in(1), u2 = a.in(2); return cimul(make_double2(xz * u1.x + xy * u2.x, xz * u1.y + xy * u2.y), 0.5); }  // eps_yz
    }
  }
  DBF_DEV static cplx post(const ColAt&, int, int) { return make_double2(1.0, 0.0); }
};

template <>
struct ColOp<COL_I1F> {
  static constexpr bool INV = true;
  static constexpr int NOUT = 6;
  DBF_DEV static int nterms(int) { return 1; }
  DBF_DEV static cplx load(const ColAt& a, int o, int) {
    if (o < 3) return a.in(o);
    return cimul(a.in(o - 3), __ldg(a.g->fq.xz + a.pos));  // G_iz = i xi_z u_i
  }
  DBF_DEV static cplx post(const ColAt&, int, int) { return make_double2(1.0, 0.0); }
};

// y inverse, small strain.  outer = z, pos = ky.  in: {u_x, u_y, eps_zz, eps_xz, eps_yz}
// out (Voigt): {xx, yy, zz, yz, xz, xy}
template <>
struct ColOp<COL_I2S> {
  static constexpr bool INV = true;
  static constexpr int NOUT = 6;
  DBF_DEV static int nterms(int) { return 1; }
  DBF_DEV static cplx load(const ColAt& a, int o, int) {
    const double xx = __ldg(a.g->fq.xx + a.kx), xy = __ldg(a.g->fq.xy + a.pos);
    switch (o) {
      case 0: return cimul(a.in(0), xx);
      case 1: return cimul(a.in(1), xy);
      case 2: return a.in(2);
      case 3: return a.in(4);
      case 4: return a.in(3);
      default: { cplx u0 = a.in(0), u1 = a.in(1); return cimul(make_double2(xy * u0.x + xx * u1.x, xy * u0.y + xx * u1.y), 0.5); }
    }
  }
  DBF_DEV static cplx post(const ColAt&, int, int) { return make_double2(1.0, 0.0); }
};

// y inverse, finite strain.  in: {u_0,u_1,u_2, G_0z,G_1z,G_2z}; out o = 3i+j:
// j=0: u_i (x derivative applied in the x pass), j=1: i xi_y u_i, j=2: G_iz.
template <>
struct ColOp<COL_I2F> {
  static constexpr bool INV = true;
  static constexpr int NOUT = 9;
  DBF_DEV static int nterms(int) { return 1; }
  DBF_DEV static cplx load(const ColAt& a, int o, int) {
    const int i = o / 3, j = o % 3;
    if (j == 0) return a.in(i);
    if (j == 1) return cimul(a.in(i), __ldg(a.g->fq.xy + a.pos));
    return a.in(3 + i);
  }
  DBF_DEV static cplx post(const ColAt&, int, int) { return make_double2(1.0, 0.0); }
};

template <>
struct ColOp<COL_F2S> {
  static constexpr bool INV = false;
  static constexpr int NOUT = 6;
  DBF_DEV static int nterms(int) { return 1; }
  DBF_DEV static cplx load(const ColAt& a, int o, int) { return a.in(o); }
  DBF_DEV static cplx post(const ColAt&, int, int) { return make_double2(1.0, 0.0); }
};

// y forward, finite strain.  in o=3i+j: {g_i (xi_x folded), P_iy, P_iz};  out: g_i (+ -i xi_y P_iy), P_iz
template <>
struct ColOp<COL_F2F> {
  static constexpr bool INV = false;
  static constexpr int NOUT = 6;
  DBF_DEV static int nterms(int o) { return o < 3 ? 2 : 1; }
  DBF_DEV static cplx load(const ColAt& a, int o, int t) {
    if (o < 3) return a.in(3 * o + t);
    return a.in(3 * (o - 3) + 2);
  }
  DBF_DEV static cplx post(const ColAt& a, int o, int t) {
    if (o < 3 && t == 1) return make_double2(0.0, -__ldg(a.g->fq.xy + a.pos));
    return make_double2(1.0, 0.0);
  }
};

// z forward + divergence, small strain.  outer = ky, pos = kz.  in Voigt sigma:
// f_x = Z(-i(xi_x s_xx + xi_y s_xy)) - i xi_z Z(s_xz), etc.  (R3 sign)
template <>
struct ColOp<COL_F3S> {
  static constexpr bool INV = false;
  static constexpr int NOUT = 3;
  DBF_DEV static int nterms(int) { return 2; }
  DBF_DEV static cplx load(const ColAt& a, int o, int t) {
    const double xx = __ldg(a.g->fq.xx + a.kx), xy = __ldg(a.g->fq.xy + a.outer);
    // (first, second) in-plane components and the z component of row o
    const int fa = (o == 0) ? 0 : (o == 1) ? 5 : 4;   // s_ox
    const int fb = (o == 0) ? 5 : (o == 1) ? 1 : 3;   // s_oy
    const int fz = (o == 0) ? 4 : (o == 1) ? 3 : 2;   // s_oz
    if (t == 1) return a.in(fz);
    cplx sa = a.in(fa), sb = a.in(fb);
    return cimul(make_double2(xx * sa.x + xy * sb.x, xx * sa.y + xy * sb.y), -1.0);
  }
  DBF_DEV static cplx post(const ColAt& a, int, int t) {
    if (t == 1) return make_double2(0.0, -__ldg(a.g->fq.xz + a.pos));
    return make_double2(1.0, 0.0);
  }
};

template <>
struct ColOp<COL_F3F> {
  static constexpr bool INV = false;
  static constexpr int NOUT = 3;
  DBF_DEV static int nterms(int) { return 2; }
  DBF_DEV static cplx load(const ColAt& a, int o, int t) { return a.in(t == 0 ? o : 3 + o); }
  DBF_DEV static cplx post(const ColAt& a, int, int t) {
    if (t == 1) return make_double2(0.0, -__ldg(a.g->fq.xz + a.pos));
    return make_double2(1.0, 0.0);
  }
};

template <>
struct ColOp<COL_ZI3> {
  static constexpr bool INV = true;
  static constexpr int NOUT = 3;
  DBF_DEV static int nterms(int) { return 1; }
  DBF_DEV static cplx load(const ColAt& a, int o, int) { return a.in(o); }
  DBF_DEV static cplx post(const ColAt&, int, int) { return make_double2(1.0, 0.0); }
};
template <>
struct ColOp<COL_YI3> : ColOp<COL_ZI3> {};

template <int KIND>
struct ColTwo {  // does any output of this pass sum two transformed terms?
  static constexpr bool value = (KIND == COL_F2F || KIND == COL_F3S || KIND == COL_F3F);
};

template <int N, int KIND>
__global__ void __launch_bounds__(256, 3) col_pass_kernel(ColGeom g) {
  typedef ColOp<KIND> Op;
  constexpr int TPC = N / 8;        // threads per column
  constexpr int COLS = 256 / TPC;   // columns per CTA
  constexpr bool TWO = ColTwo<KIND>::value;
  extern __shared__ cplx col_smem[];
  cplx* sbuf = col_smem;                 // FFT exchange, N * COLS
  cplx* sacc = col_smem + N * COLS;      // first-term results of two-term outputs (TWO only)
  const int t = threadIdx.x;
  const int c = t % COLS;
  const int gq = t / COLS;
  const long long col = (long long)blockIdx.x * COLS + c;
  const bool valid = col < g.ncols;
  ColAt at;
  at.g = &g;
  at.outer = valid ? (int)(col / g.n1h) : 0;
  at.kx = valid ? (int)(col % g.n1h) : 0;
  const double wdot = (at.kx == 0 || 2 * at.kx == g.n1) ? 1.0 : 2.0;
  double dot = 0.0;
  IdxCols<COLS> idx{c};
#pragma unroll 1
  for (int o = 0; o < Op::NOUT; ++o) {
    const int nt = Op::nterms(o);
#pragma unroll 1
    for (int term = 0; term < nt; ++term) {
      cplx a[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        at.pos = gq + s * (N / 8);
        a[s] = valid ? Op::load(at, o, term) : make_double2(0.0, 0.0);
      }
      fft_cta<N, Op::INV>(a, sbuf, gq, idx, g.tw);
      const bool last = (term + 1 == nt);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        at.pos = gq + s * (N / 8);
        cplx v = cmul(Op::post(at, o, term), a[s]);
        if (TWO && term > 0) v = cadd(v, sacc[idx(at.pos)]);
        if (!last) {
          if (TWO) sacc[idx(at.pos)] = v;  // own positions only: no barrier needed
        } else if (valid) {
          const long long oi = at.out_idx(o);
          g.out[oi] = v;
          if (g.dotp) {
            cplx p = __ldg(g.dotp + oi);
            dot += wdot * (p.x * v.x + p.y * v.y);
          }
        }
      }
    }
  }
  if (g.dotp) {
    __shared__ double red[8];
    dot = warp_sum(dot);
    if ((t & 31) == 0) red[t >> 5] = dot;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
      g.partials[blockIdx.x] = s;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// X pass: per CTA LPAR lines; per line the C fields are C2R'd in pairs (z = a + i b trick),
// the per-voxel operation runs on the real fields in shared memory, and the results are R2C'd
// in pairs and untangled: A_k = (Z_k + conj Z_{N-k})/2, B_k = (Z_k - conj Z_{N-k})/(2i).
// ------------------------------------------------------------------------------------------------
template <int KIND>
struct XTraits;
template <> struct XTraits<X_K_SMALL_PHASE> { static constexpr int CIN = 6, COUT = 6, NRED = 9; static constexpr bool FIN = false; };
template <> struct XTraits<X_K_J2> { static constexpr int CIN = 6, COUT = 6, NRED = 9; static constexpr bool FIN = false; };
template <> struct XTraits<X_K_FIN_TAN> { static constexpr int CIN = 9, COUT = 9, NRED = 9; static constexpr bool FIN = true; };
template <> struct XTraits<X_K_FIN_NH> { static constexpr int CIN = 9, COUT = 9, NRED = 9; static constexpr bool FIN = true; };
template <> struct XTraits<X_RHS_SMALL_PHASE> { static constexpr int CIN = 0, COUT = 6, NRED = 9; static constexpr bool FIN = false; };
template <> struct XTraits<X_CONST_FIN> { static constexpr int CIN = 9, COUT = 9, NRED = 10; static constexpr bool FIN = true; };
template <> struct XTraits<X_CONST_J2> { static constexpr int CIN = 6, COUT = 6, NRED = 10; static constexpr bool FIN = false; };
template <> struct XTraits<X_REAL_OUT> { static constexpr int CIN = 9, COUT = 0, NRED = 0; static constexpr bool FIN = false; };

DBF_DEV int sym9(int i, int j) {
  if (i > j) { int t = i; i = j; j = t; }
  return i * 9 - i * (i - 1) / 2 + (j - i);
}

// Voigt index (xx,yy,zz,yz,xz,xy) -> row-major 3x3 entry
__device__ __constant__ int c_row9_of_voigt[6] = {0, 4, 8, 5, 2, 1};

// streaming load of per-voxel data (read once per launch: do not allocate in L1)
DBF_DEV double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// small-strain contraction: sigma_I = sum_J C[I][J] gamma_J, gamma = (e0,e1,e2,2e3,2e4,2e5)
DBF_DEV void voigt_contract_full(const double* __restrict__ C36, const double* e, double* s) {
  const double g[6] = {e[0], e[1], e[2], 2.0 * e[3], 2.0 * e[4], 2.0 * e[5]};
#pragma unroll
  for (int I = 0; I < 6; ++I) {
    double acc = 0.0;
#pragma unroll
    for (int J = 0; J < 6; ++J) acc = fma(__ldg(C36 + 6 * I + J), g[J], acc);
    s[I] = acc;
  }
}

// Neo-Hookean (R14): P = mu (F - F^-T) + lam lnJ F^-T; returns J, F^-1 (row-major) and
// c1 = mu - lam lnJ, so that the tangent acts as K:G = mu G + c1 (Fi G Fi)^T + lam tr(Fi G) Fi^T.
DBF_DEV double neo_hookean(const double* F, double mu, double kappa, double* P, double* Fi, double* c1_out) {
  const double lam = kappa - 2.0 * mu / 3.0;
  const double c00 = F[4] * F[8] - F[5] * F[7];
  const double c01 = F[5] * F[6] - F[3] * F[8];
  const double c02 = F[3] * F[7] - F[4] * F[6];
  const double J = F[0] * c00 + F[1] * c01 + F[2] * c02;
  const double iJ = 1.0 / J;
  Fi[0] = c00 * iJ;
  Fi[3] = c01 * iJ;
  Fi[6] = c02 * iJ;
  Fi[1] = (F[2] * F[7] - F[1] * F[8]) * iJ;
  Fi[4] = (F[0] * F[8] - F[2] * F[6]) * iJ;
  Fi[7] = (F[1] * F[6] - F[0] * F[7]) * iJ;
  Fi[2] = (F[1] * F[5] - F[2] * F[4]) * iJ;
  Fi[5] = (F[2] * F[3] - F[0] * F[5]) * iJ;
  Fi[8] = (F[0] * F[4] - F[1] * F[3]) * iJ;
  const double lnJ = log(J);
  *c1_out = mu - lam * lnJ;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) P[3 * i + j] = mu * F[3 * i + j] + (lam * lnJ - mu) * Fi[3 * j + i];
  return J;
}

// full 9x9 tangent (upper triangle, 45) from (Fi, c1, mu, lam):
// K_ijkl = mu d_ik d_jl + c1 Fi_li Fi_jk + lam Fi_ji Fi_lk
DBF_DEV void nh_tangent45(const double* Fi, double c1, double mu, double lam, double* K45) {
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    const int i = a / 3, j = a % 3;
#pragma unroll
    for (int b = a; b < 9; ++b) {
      const int k = b / 3, l = b % 3;
      double v = c1 * Fi[3 * l + i] * Fi[3 * j + k] + lam * Fi[3 * j + i] * Fi[3 * l + k];
      if (i == k && j == l) v += mu;
      K45[a * 9 - a * (a - 1) / 2 + (b - a)] = v;
    }
  }
}

// matrix-free neo-Hookean tangent: P = mu G + c1 (Fi G Fi)^T + lam tr(Fi G) Fi^T
DBF_DEV void nh_apply(const double* Fi, double c1, double mu, double lam, const double* G, double* P) {
  double A[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) A[3 * i + k] = Fi[3 * i] * G[k] + Fi[3 * i + 1] * G[3 + k] + Fi[3 * i + 2] * G[6 + k];
  const double tr = A[0] + A[4] + A[8];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const double B_il = A[3 * i] * Fi[l] + A[3 * i + 1] * Fi[3 + l] + A[3 * i + 2] * Fi[6 + l];
      // P_li += c1 B_il ; P_ij = mu G_ij + lam tr Fi_ji
      P[3 * l + i] = mu * G[3 * l + i] + c1 * B_il + lam * tr * Fi[3 * i + l];
    }
}

// J2 Perzyna return map (R16).  eps, epsp: Voigt tensor components.  Outputs sigma, the plastic
// strain, and the compact algorithmic tangent (theta, thetabar, n = s_tr/|s_tr|):
//   C_alg = kappa 1x1 + 2 mu theta I_dev - 2 mu thetabar n x n.
DBF_DEV void j2_update(const double* eps, const double* epsp, const double* prm, double dt,
                       double* sig, double* tc /*8: theta, thetabar, n[6]*/, double* epsp_new) {
  const double E = prm[0], nu = prm[1], sy = prm[2], nexp = prm[3], edot0 = prm[4];
  const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = E / (2.0 * (1.0 + nu));
  const double kappa = lam + 2.0 * mu / 3.0;
  double ee[6];
#pragma unroll
  for (int I = 0; I < 6; ++I) ee[I] = eps[I] - epsp[I];
  const double tr = ee[0] + ee[1] + ee[2];
  double s[6];
#pragma unroll
  for (int I = 0; I < 6; ++I) s[I] = 2.0 * mu * (ee[I] - (I < 3 ? tr / 3.0 : 0.0));
  const double ss = s[0] * s[0] + s[1] * s[1] + s[2] * s[2] + 2.0 * (s[3] * s[3] + s[4] * s[4] + s[5] * s[5]);
  const double svm = sqrt(1.5 * ss);
  double theta = 1.0, thetabar = 0.0, dp = 0.0;
  double nn[6] = {0, 0, 0, 0, 0, 0};
  if (svm > sy) {
    // g(x) = svm - 3 mu rdt x^n - sy (1 + x) = 0, x = (dp / rdt)^(1/n); safeguarded Newton
    const double rdt = edot0 * dt, m3 = 3.0 * mu * rdt;
    double lo = 0.0, hi = svm / sy - 1.0, x = 0.5 * hi;
    for (int it = 0; it < 200; ++it) {
      const double xn1 = pow(x, nexp - 1.0);
      const double gx = svm - m3 * xn1 * x - sy * (1.0 + x);
      if (gx > 0) lo = x; else hi = x;
      const double dg = -m3 * nexp * xn1 - sy;
      double xn = x - gx / dg;
      if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
      if (fabs(xn - x) <= 1e-16 * x || hi - lo <= 1e-16 * hi) { x = xn; break; }
      x = xn;
    }
    dp = rdt * pow(x, nexp);
    theta = 1.0 - 3.0 * mu * dp / svm;
    const double Hp = (dp > 0) ? sy / (nexp * rdt) * pow(dp / rdt, 1.0 / nexp - 1.0) : 0.0;
    thetabar = 1.0 / (1.0 + Hp / (3.0 * mu)) - (1.0 - theta);
    const double is = 1.0 / sqrt(ss);
#pragma unroll
    for (int I = 0; I < 6; ++I) nn[I] = s[I] * is;
  }
#pragma unroll
  for (int I = 0; I < 6; ++I) {
    sig[I] = theta * s[I] + (I < 3 ? kappa * tr : 0.0);
    epsp_new[I] = epsp[I] + (svm > sy ? dp * 1.5 * s[I] / svm : 0.0);
    tc[2 + I] = nn[I];
  }
  tc[0] = theta;
  tc[1] = thetabar;
}

// sigma = C_alg : e with the compact J2 tangent (Voigt tensor components)
DBF_DEV void j2_apply(const double* tc, double kappa, double mu, const double* e, double* s) {
  const double tr = e[0] + e[1] + e[2];
  const double ne = tc[2] * e[0] + tc[3] * e[1] + tc[4] * e[2] + 2.0 * (tc[5] * e[3] + tc[6] * e[4] + tc[7] * e[5]);
  const double a = 2.0 * mu * tc[0], b = 2.0 * mu * tc[1] * ne;
#pragma unroll
  for (int I = 0; I < 6; ++I) s[I] = a * (e[I] - (I < 3 ? tr / 3.0 : 0.0)) - b * tc[2 + I] + (I < 3 ? kappa * tr : 0.0);
}

DBF_DEV void j2_moduli(const double* prm, double* kappa, double* mu) {
  const double E = prm[0], nu = prm[1];
  const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  *mu = E / (2.0 * (1.0 + nu));
  *kappa = lam + 2.0 * (*mu) / 3.0;
}

template <int KIND>
DBF_DEV void x_voxel(const XGeom& g, long long v, double* G, double* P, double* red) {
  if (KIND == X_K_SMALL_PHASE || KIND == X_RHS_SMALL_PHASE || KIND == X_K_J2) {
    double e6[6];
#pragma unroll
    for (int I = 0; I < 6; ++I)
      e6[I] = (KIND == X_RHS_SMALL_PHASE ? 0.0 : G[I]) + (g.e ? __ldg(g.e + c_row9_of_voigt[I]) : 0.0);
    const int ph = __ldg(g.phase + v);
    double s[6];
    if (KIND == X_K_J2) {
      double tc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) tc[k] = ld_stream(g.tan + (long long)k * g.nvox + v);
      double kappa, mu;
      j2_moduli(g.ptable + 36 * ph, &kappa, &mu);
      j2_apply(tc, kappa, mu, e6, s);
    } else {
      voigt_contract_full(g.ptable + 36 * ph, e6, s);
    }
    const double sg = (KIND == X_RHS_SMALL_PHASE) ? -1.0 : 1.0;
#pragma unroll
    for (int I = 0; I < 6; ++I) {
      P[I] = sg * s[I];
      red[c_row9_of_voigt[I]] += s[I];
    }
  } else if (KIND == X_K_FIN_TAN) {
    double e9[9], K[45];
#pragma unroll
    for (int k = 0; k < 45; ++k) K[k] = ld_stream(g.tan + (long long)k * g.nvox + v);
#pragma unroll
    for (int a = 0; a < 9; ++a) e9[a] = G[a] + (g.e ? __ldg(g.e + a) : 0.0);
#pragma unroll
    for (int a = 0; a < 9; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < 9; ++b) acc = fma(K[sym9(a, b)], e9[b], acc);
      P[a] = acc;
      red[a] += acc;
    }
  } else if (KIND == X_K_FIN_NH) {
    double Fi[9], e9[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Fi[k] = ld_stream(g.tan + (long long)k * g.nvox + v);
    const double c1 = ld_stream(g.tan + 9 * g.nvox + v);
    const int ph = __ldg(g.phase + v);
    const double mu = __ldg(g.ptable + 36 * ph), lam = __ldg(g.ptable + 36 * ph + 1) - 2.0 * mu / 3.0;
#pragma unroll
    for (int a = 0; a < 9; ++a) e9[a] = G[a] + (g.e ? __ldg(g.e + a) : 0.0);
    nh_apply(Fi, c1, mu, lam, e9, P);
#pragma unroll
    for (int a = 0; a < 9; ++a) red[a] += P[a];
  } else if (KIND == X_CONST_FIN) {
    double F[9], Pv[9], Fi[9], c1;
    double mx = 0.0;
#pragma unroll
    for (int a = 0; a < 9; ++a) {
      const double d = (g.has_in ? G[a] : 0.0) + __ldg(g.e + a);
      mx = fmax(mx, fabs(d));
      F[a] = g.F[(long long)a * g.nvox + v] + d;
      g.F[(long long)a * g.nvox + v] = F[a];
    }
    const int ph = __ldg(g.phase + v);
    const double mu = __ldg(g.ptable + 36 * ph), kappa = __ldg(g.ptable + 36 * ph + 1);
    const double J = neo_hookean(F, mu, kappa, Pv, Fi, &c1);
    if (!(J > 0.0)) atomicMin(g.bad, (int)min(v, (long long)0x7fffffff));
    if (g.tmode == 1) {
#pragma unroll
      for (int k = 0; k < 9; ++k) g.tan[(long long)k * g.nvox + v] = Fi[k];
      g.tan[9 * g.nvox + v] = c1;
    } else {
      double K45[45];
      nh_tangent45(Fi, c1, mu, kappa - 2.0 * mu / 3.0, K45);
#pragma unroll
      for (int k = 0; k < 45; ++k) g.tan[(long long)k * g.nvox + v] = K45[k];
    }
#pragma unroll
    for (int a = 0; a < 9; ++a) {
      P[a] = -Pv[a];
      red[a] += Pv[a];
    }
    red[9] = fmax(red[9], mx);
  } else if (KIND == X_CONST_J2) {
    double eps[6], ep[6], s[6], tc[8], epn[6];
    double mx = 0.0;
#pragma unroll
    for (int I = 0; I < 6; ++I) {
      const double d = (g.has_in ? G[I] : 0.0) + __ldg(g.e + c_row9_of_voigt[I]);
      mx = fmax(mx, fabs(d));
      eps[I] = g.F[(long long)I * g.nvox + v] + d;
      g.F[(long long)I * g.nvox + v] = eps[I];
      ep[I] = __ldg(g.epsp_c + (long long)I * g.nvox + v);
    }
    const int ph = __ldg(g.phase + v);
    j2_update(eps, ep, g.ptable + 36 * ph, g.dt, s, tc, epn);
#pragma unroll
    for (int k = 0; k < 8; ++k) g.tan[(long long)k * g.nvox + v] = tc[k];
#pragma unroll
    for (int I = 0; I < 6; ++I) {
      g.epsp_t[(long long)I * g.nvox + v] = epn[I];
      P[I] = -s[I];
      red[c_row9_of_voigt[I]] += s[I];
    }
    red[9] = fmax(red[9], mx);
  }
}

// XOR swizzle inside 8-element groups: conflict-free radix-8 scatter/gather, no padding, so
// the exchange buffer of a field pair is exactly the pair's two real slots (in place).
struct IdxSwz {
  int base;
  DBF_DEV int operator()(int pos) const { return base + (pos ^ ((pos >> 3) & 7)); }
};

template <int N1, int KIND>
struct XCfg {
  typedef XTraits<KIND> T;
  static constexpr int C = (T::CIN > T::COUT) ? T::CIN : T::COUT;
  static constexpr int CS = (C + 1) & ~1;          // real slots per line (even)
  static constexpr int TPJ = N1 / 8;
  static constexpr int NP = CS / 2;
  static constexpr int PERLINE = TPJ * NP;
  static constexpr int LRAW = 192 / PERLINE;
  static constexpr int LPAR = LRAW >= 64 ? 64 : LRAW >= 32 ? 32 : LRAW >= 16 ? 16 : LRAW >= 8 ? 8 : LRAW >= 4 ? 4 : LRAW >= 2 ? 2 : 1;
  static constexpr int THREADS = LPAR * PERLINE;
  static constexpr size_t SMEM = sizeof(double) * LPAR * CS * N1;
  static constexpr int MINB = (THREADS <= 192) ? 3 : 2;
};

// X pass.  Persistent: each CTA loops over groups of LPAR lines.  Per line the C fields are
// C2R'd in pairs (z = a + i b), the per-voxel operation runs on the real fields in shared
// memory, and results are R2C'd in pairs and untangled:
//   A_k = (Z_k + conj Z_{N-k})/2,  B_k = (Z_k - conj Z_{N-k})/(2i).
template <int N1, int KIND>
__global__ void __launch_bounds__(XCfg<N1, KIND>::THREADS, XCfg<N1, KIND>::MINB) x_pass_kernel(XGeom g, int nf_real) {
  typedef XCfg<N1, KIND> CF;
  typedef XTraits<KIND> T;
  constexpr int C = CF::C, CS = CF::CS, TPJ = CF::TPJ, NP = CF::NP, LPAR = CF::LPAR;
  extern __shared__ double real[];
  cplx* cx = reinterpret_cast<cplx*>(real);
  const int t = threadIdx.x;
  const int job = t / TPJ, gq = t % TPJ;
  const int l = job / NP, p = job % NP;
  const int fa = 2 * p, fb = 2 * p + 1;
  IdxSwz idx{(l * CS + fa) * (N1 / 2)};  // complex view of slots fa, fb of line l
  const int cin = (KIND == X_REAL_OUT) ? nf_real : T::CIN;
  const bool do_in = (T::CIN > 0) && (cin > 0) && ((KIND != X_CONST_FIN && KIND != X_CONST_J2) || g.has_in);
  const long long ngroups = (g.nlines + LPAR - 1) / LPAR;
  double red[T::NRED > 0 ? T::NRED : 1];
#pragma unroll
  for (int r = 0; r < (T::NRED > 0 ? T::NRED : 1); ++r) red[r] = 0.0;

  for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const long long line = grp * LPAR + l;
    const bool lvalid = line < g.nlines;
    // ------------------------------------------------------------ inverse (C2R) of pairs
    if (do_in) {
      cplx a[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int k = gq + s * TPJ;
        const bool lo = (2 * k <= N1);
        const int kk = lo ? k : N1 - k;
        cplx A = make_double2(0, 0), B = make_double2(0, 0);
        if (lvalid && fa < cin) {
          const long long base = line * g.n1h + kk;
          A = __ldg(g.in + fa * g.fs_in + base);
          if (fb < cin) B = __ldg(g.in + fb * g.fs_in + base);
          if (T::FIN) {  // G_ix = i xi_x u_i for the j = 0 slots (deferred gradient)
            const double xx = __ldg(g.xix + kk);
            if (fa % 3 == 0) A = cimul(A, xx);
            if (fb % 3 == 0 && fb < cin) B = cimul(B, xx);
          }
          if (kk == 0 || 2 * kk == N1) { A.y = 0.0; B.y = 0.0; }  // Hermitian part (C2R)
        }
        // Y_k = A_k + i B_k (k <= N/2);  conj(A_{N-k}) + i conj(B_{N-k}) otherwise
        a[s] = lo ? make_double2(A.x - B.y, A.y + B.x) : make_double2(A.x + B.y, B.x - A.y);
      }
      fft_cta<N1, true>(a, cx, gq, idx, g.tw);
      __syncthreads();  // exchange reads done before the slots are overwritten with reals
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int m = gq + s * TPJ;
        real[(l * CS + fa) * N1 + m] = a[s].x;
        real[(l * CS + fb) * N1 + m] = a[s].y;
      }
    }
    __syncthreads();

    if (KIND == X_REAL_OUT) {
      for (int vv = t; vv < LPAR * N1; vv += CF::THREADS) {
        const int l2 = vv / N1, x = vv % N1;
        const long long ln = grp * LPAR + l2;
        if (ln >= g.nlines) continue;
        for (int f = 0; f < nf_real; ++f) g.real_out[(long long)f * g.nvox + ln * N1 + x] = real[(l2 * CS + f) * N1 + x];
      }
      __syncthreads();
      continue;
    }

    // ------------------------------------------------------------ per-voxel operation
    for (int vv = t; vv < LPAR * N1; vv += CF::THREADS) {
      const int l2 = vv / N1, x = vv % N1;
      const long long ln = grp * LPAR + l2;
      if (ln >= g.nlines) continue;
      double G[C], P[C];
#pragma unroll
      for (int f = 0; f < C; ++f) G[f] = (f < T::CIN && do_in) ? real[(l2 * CS + f) * N1 + x] : 0.0;
      x_voxel<KIND>(g, ln * N1 + x, G, P, red);
#pragma unroll
      for (int f = 0; f < T::COUT; ++f) real[(l2 * CS + f) * N1 + x] = P[f];
    }
    __syncthreads();

    // ------------------------------------------------------------ forward (R2C) of pairs
    {
      constexpr int COUT = T::COUT;
      cplx a[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int m = gq + s * TPJ;
        const double ra = (fa < COUT) ? real[(l * CS + fa) * N1 + m] : 0.0;
        const double rb = (fb < COUT) ? real[(l * CS + fb) * N1 + m] : 0.0;
        a[s] = make_double2(ra, rb);
      }
      fft_cta<N1, false>(a, cx, gq, idx, g.tw);
      __syncthreads();
#pragma unroll
      for (int s = 0; s < 8; ++s) cx[idx(gq + s * TPJ)] = a[s];
      __syncthreads();
      if (lvalid && fa < COUT) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const int k = gq + s * TPJ;
          if (2 * k > N1) continue;
          const cplx Z = a[s];
          const cplx Zn = cx[idx((N1 - k) & (N1 - 1))];
          cplx A = make_double2(0.5 * (Z.x + Zn.x), 0.5 * (Z.y - Zn.y));
          cplx B = make_double2(0.5 * (Z.y + Zn.y), -0.5 * (Z.x - Zn.x));
          A = cscale(A, g.inv_n);
          B = cscale(B, g.inv_n);
          if (T::FIN) {  // fold -i xi_x P_ix into the j = 0 slots (early divergence)
            const double xx = __ldg(g.xix + k);
            if (fa % 3 == 0) A = cimul(A, -xx);
            if (fb % 3 == 0) B = cimul(B, -xx);
          }
          const long long base = line * g.n1h + k;
          g.out[fa * g.fs_out + base] = A;
          if (fb < COUT) g.out[fb * g.fs_out + base] = B;
        }
      }
      __syncthreads();  // slots are reused by the next group
    }
  }

  if (T::NRED > 0) {
    // block reduction -> partials[block][nred] (sums; slot 9 of the const kinds is a max)
    __shared__ double sred[(CF::THREADS + 31) / 32][10];
    constexpr int nw = (CF::THREADS + 31) / 32;
#pragma unroll
    for (int r = 0; r < T::NRED; ++r) {
      const bool is_max = (r == 9);
      double v = is_max ? warp_max(red[r]) : warp_sum(red[r]);
      if ((t & 31) == 0) sred[t >> 5][r] = v;
    }
    __syncthreads();
    if (t < T::NRED) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s = (t == 9) ? fmax(s, sred[w][t]) : s + sred[w][t];
      g.partials[(long long)blockIdx.x * g.nred + t] = s;
    }
  }
}

// mean tangent from the stored per-voxel tangent -> partials[block][nk]
template <int MODE>  // 0: full 45 (finite), 1: compact NH (finite, 45 out), 2: compact J2 (21 out)
__global__ void __launch_bounds__(256) k_mean_tangent(XGeom g, double* partials) {
  constexpr int NK = (MODE == 2) ? 21 : 45;
  double acc[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) acc[k] = 0.0;
  for (long long v = (long long)blockIdx.x * 256 + threadIdx.x; v < g.nvox; v += (long long)gridDim.x * 256) {
    if (MODE == 0) {
#pragma unroll
      for (int k = 0; k < 45; ++k) acc[k] += __ldg(g.tan + (long long)k * g.nvox + v);
    } else if (MODE == 1) {
      double Fi[9], K45[45];
#pragma unroll
      for (int k = 0; k < 9; ++k) Fi[k] = __ldg(g.tan + (long long)k * g.nvox + v);
      const double c1 = __ldg(g.tan + 9 * g.nvox + v);
      const int ph = __ldg(g.phase + v);
      const double mu = __ldg(g.ptable + 36 * ph), lam = __ldg(g.ptable + 36 * ph + 1) - 2.0 * mu / 3.0;
      nh_tangent45(Fi, c1, mu, lam, K45);
#pragma unroll
      for (int k = 0; k < 45; ++k) acc[k] += K45[k];
    } else {
      double tc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) tc[k] = __ldg(g.tan + (long long)k * g.nvox + v);
      const int ph = __ldg(g.phase + v);
      double kappa, mu;
      j2_moduli(g.ptable + 36 * ph, &kappa, &mu);
#pragma unroll
      for (int I = 0; I < 6; ++I)
#pragma unroll
        for (int J = I; J < 6; ++J) {
          const double idev = (I < 3 && J < 3) ? ((I == J ? 1.0 : 0.0) - 1.0 / 3.0) : ((I == J) ? 0.5 : 0.0);
          acc[I * 6 - I * (I - 1) / 2 + (J - I)] += ((I < 3 && J < 3) ? kappa : 0.0) + 2.0 * mu * tc[0] * idev -
                                                    2.0 * mu * tc[1] * tc[2 + I] * tc[2 + J];
        }
    }
  }
  __shared__ double red[8][NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    double s = warp_sum(acc[k]);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NK) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    partials[(long long)blockIdx.x * NK + threadIdx.x] = s;
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------------------------
int col_grid(int N, long long ncols) {
  const int cols = 256 / (N / 8);
  return (int)((ncols + cols - 1) / cols);
}

template <int N, int KIND>
static cudaError_t launch_col_k(const ColGeom& g, cudaStream_t s) {
  constexpr int COLS = 256 / (N / 8);
  constexpr size_t smem = sizeof(cplx) * N * COLS * (ColTwo<KIND>::value ? 2 : 1);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(col_pass_kernel<N, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  col_pass_kernel<N, KIND><<<col_grid(N, g.ncols), 256, smem, s>>>(g);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_col_n(int kind, const ColGeom& g, cudaStream_t s) {
  switch (kind) {
    case COL_I1S: return launch_col_k<N, COL_I1S>(g, s);
    case COL_I1F: return launch_col_k<N, COL_I1F>(g, s);
    case COL_I2S: return launch_col_k<N, COL_I2S>(g, s);
    case COL_I2F: return launch_col_k<N, COL_I2F>(g, s);
    case COL_F2S: return launch_col_k<N, COL_F2S>(g, s);
    case COL_F2F: return launch_col_k<N, COL_F2F>(g, s);
    case COL_F3S: return launch_col_k<N, COL_F3S>(g, s);
    case COL_F3F: return launch_col_k<N, COL_F3F>(g, s);
    case COL_ZI3: return launch_col_k<N, COL_ZI3>(g, s);
    case COL_YI3: return launch_col_k<N, COL_YI3>(g, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_col(int kind, int N, const ColGeom& g, cudaStream_t s) {
  switch (N) {
    case 8: return launch_col_n<8>(kind, g, s);
    case 16: return launch_col_n<16>(kind, g, s);
    case 32: return launch_col_n<32>(kind, g, s);
    case 64: return launch_col_n<64>(kind, g, s);
    case 128: return launch_col_n<128>(kind, g, s);
    case 256: return launch_col_n<256>(kind, g, s);
    case 512: return launch_col_n<512>(kind, g, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int N1, int KIND>
static cudaError_t launch_x_k(const XGeom& g, cudaStream_t s, int* grid_out, int nf_real) {
  typedef XCfg<N1, KIND> CF;
  static int max_grid = 0;  // per template instance: resident CTAs on the whole device
  if (max_grid == 0) {
    cudaError_t e = cudaFuncSetAttribute(x_pass_kernel<N1, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    if (e != cudaSuccess) return e;
    int nb = 0, dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, x_pass_kernel<N1, KIND>, CF::THREADS, CF::SMEM);
    if (e != cudaSuccess) return e;
    max_grid = std::max(1, nb) * nsm;
  }
  const long long ngroups = (g.nlines + CF::LPAR - 1) / CF::LPAR;
  const int grid = (int)std::min<long long>(ngroups, max_grid);
  if (grid_out) *grid_out = grid;
  x_pass_kernel<N1, KIND><<<grid, CF::THREADS, CF::SMEM, s>>>(g, nf_real);
  return cudaGetLastError();
}

template <int N1>
static cudaError_t launch_x_n(int kind, const XGeom& g, cudaStream_t s, int* grid_out) {
  switch (kind) {
    case X_K_SMALL_PHASE: return launch_x_k<N1, X_K_SMALL_PHASE>(g, s, grid_out, 0);
    case X_K_J2: return launch_x_k<N1, X_K_J2>(g, s, grid_out, 0);
    case X_K_FIN_TAN: return launch_x_k<N1, X_K_FIN_TAN>(g, s, grid_out, 0);
    case X_K_FIN_NH: return launch_x_k<N1, X_K_FIN_NH>(g, s, grid_out, 0);
    case X_RHS_SMALL_PHASE: return launch_x_k<N1, X_RHS_SMALL_PHASE>(g, s, grid_out, 0);
    case X_CONST_FIN: return launch_x_k<N1, X_CONST_FIN>(g, s, grid_out, 0);
    case X_CONST_J2: return launch_x_k<N1, X_CONST_J2>(g, s, grid_out, 0);
    default: break;
  }
  if (kind >= X_REAL_OUT) return launch_x_k<N1, X_REAL_OUT>(g, s, grid_out, kind - X_REAL_OUT);
  return cudaErrorInvalidValue;
}

// kind X_REAL_OUT + nf selects a real-output transform of nf fields (1..9)
cudaError_t launch_x(int kind, int N1, const XGeom& g, cudaStream_t s, int* grid_out) {
  switch (N1) {
    case 8: return launch_x_n<8>(kind, g, s, grid_out);
    case 16: return launch_x_n<16>(kind, g, s, grid_out);
    case 32: return launch_x_n<32>(kind, g, s, grid_out);
    case 64: return launch_x_n<64>(kind, g, s, grid_out);
    case 128: return launch_x_n<128>(kind, g, s, grid_out);
    case 256: return launch_x_n<256>(kind, g, s, grid_out);
    case 512: return launch_x_n<512>(kind, g, s, grid_out);
    default: return cudaErrorInvalidValue;
  }
}

// upper bound of the X-pass grid (= number of line groups) for partial-buffer sizing
int x_grid(int kind, int N1, long long nlines) {
  (void)kind;
  (void)N1;
  return (int)std::min<long long>(nlines, 148LL * 32);
}

cudaError_t launch_mean_tangent(int mode, const XGeom& g, double* partials, int nblk, cudaStream_t s) {
  if (mode == 0) k_mean_tangent<0><<<nblk, 256, 0, s>>>(g, partials);
  else if (mode == 1) k_mean_tangent<1><<<nblk, 256, 0, s>>>(g, partials);
  else k_mean_tangent<2><<<nblk, 256, 0, s>>>(g, partials);
  return cudaGetLastError();
}
