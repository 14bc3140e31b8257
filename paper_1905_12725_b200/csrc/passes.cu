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

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

// Per-device one-time initialisation (kernel attributes, occupancy-derived grids): a process may
// hold contexts on several devices, each call runs with its ctx's device current (dbfft.cu).
namespace {
constexpr int kMaxDevices = 64;
struct DevOnce {
  std::once_flag flag[kMaxDevices];
  cudaError_t err[kMaxDevices] = {};
  int val[kMaxDevices] = {};
};
int current_device() {
  int d = 0;
  return cudaGetDevice(&d) == cudaSuccess ? d : -1;
}
template <class F>
cudaError_t dev_once(DevOnce& o, F init, int* val = nullptr) {
  const int d = current_device();
  if (d < 0 || d >= kMaxDevices) return cudaErrorInvalidDevice;
  std::call_once(o.flag[d], [&] { o.err[d] = init(o.val[d]); });
  if (val) *val = o.val[d];
  return o.err[d];
}
}  // namespace

// opt-in (DBFFT_PDL=1): measured on B200 (tools/ab_pdl.sh, back to back) it shortened the small
// solves (c1 0.135 -> 0.133, c2 0.121 -> 0.119 ms per PCG iteration) but slowed c3 (0.419 -> 0.433)
// and the c4 bench (5.07e9 -> 4.89e9): the early-scheduled dependent CTAs cost more in the
// predecessor's tail than the launch latency they hide
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("DBFFT_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

int num_sms() {
  static DevOnce once;
  int n = 0;
  dev_once(once, [](int& v) { return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device()); }, &n);
  return n > 0 ? n : 148;
}

#ifndef DBF_X_MINB
#define DBF_X_MINB 3
#endif
#ifndef DBF_X_P16_256
#define DBF_X_P16_256 0x11  // pass_X kinds (bit = XKind) that run radix-16 FFTs (16 points per thread) at N1 <= 256
#endif
#ifndef DBF_XWS
#define DBF_XWS 0  // 1: warp-specialised pass_X for the neo-Hookean apply kind at N1 = 256
#endif
#ifndef DBF_XWS_NV
#define DBF_XWS_NV 2  // its voxel warps per CTA
#endif
#ifndef DBF_XWS_MINB
#define DBF_XWS_MINB 3
#endif
#ifndef DBF_XWS_MAXREG
#define DBF_XWS_MAXREG 0  // > 0: register cap instead of the CTAs-per-SM bound
#endif
#ifndef DBF_X_MINB_J2P16
#define DBF_X_MINB_J2P16 3  // CTAs per SM of the radix-16 J2 apply kind
#endif
#ifndef DBF_X_P16_512
#define DBF_X_P16_512 0x11  // ... at N1 = 512
#endif
#ifndef DBF_X_LRAW
#define DBF_X_LRAW 192  // target threads per pass_X CTA (lines per CTA = DBF_X_LRAW / threads per line)
#endif
#ifndef DBF_X_LRAWJ2
#define DBF_X_LRAWJ2 DBF_X_LRAW  // the J2 apply kind
#endif
#ifndef DBF_X_MINB_NOTAN_J2
#define DBF_X_MINB_NOTAN_J2 DBF_X_MINB_NOTAN
#endif
#ifndef DBF_X_LRAW16
#define DBF_X_LRAW16 96  // the radix-16 kinds: 2 lines (96 threads) per CTA, ~50 KB shared memory, 4 CTAs/SM
                         // (256^3 small 0.618 -> 0.550 ms, 128^3 0.098 -> 0.084 against 4 lines / 192)
#endif
#ifndef DBF_X_LRAW9
#define DBF_X_LRAW9 DBF_X_LRAW  // the same for the 9-field (finite-strain) kinds
#endif
#ifndef DBF_X_STAGE_SPEC
#define DBF_X_STAGE_SPEC 1  // pass_X: stage the input spectra too (else only the per-voxel data)
#endif
#ifndef DBF_X_STAGE_TAN_J2
#define DBF_X_STAGE_TAN_J2 0  // pass_X J2 kind: stage the 8 per-voxel tangent doubles (1), or load
                              // them in the voxel loop and run 4 CTAs/SM (0; B200 512^3: 7.89 -> 7.08 ms)
#endif
#ifndef DBF_X_STAGE_TAN_NH
#define DBF_X_STAGE_TAN_NH 0  // pass_X compact neo-Hookean kind: stage the 10 per-voxel tangent doubles (1),
                              // or load them in the voxel loop at 4 CTAs/SM (0; B200 256^3: 1.120 -> 1.098 ms)
#endif
#ifndef DBF_X_MINB_CONST
#define DBF_X_MINB_CONST 3  // CTAs per SM of the constitutive-update kinds (Newton residual)
#endif
#ifndef DBF_X_MINB_NOTAN
#define DBF_X_MINB_NOTAN 4  // CTAs per SM of the pass_X kinds that load their tangent in the voxel loop
#endif
#ifndef DBF_X_STAGE_IN
#define DBF_X_STAGE_IN 1
#endif
#ifndef DBF_X_PREFETCH
#define DBF_X_PREFETCH 1  // pass_X: bulk L2 prefetch of the next line group's per-voxel tangent rows
#endif
#ifndef DBF_X_L1PF
#define DBF_X_L1PF 0  // 1: neo-Hookean apply prefetches its line's tangent rows to L1 (CCTL.E.PF1) while the C2R runs (256^3: 0.926 -> 0.928 ms, no gain)
#endif
#ifndef DBF_X_TBATCH
#define DBF_X_TBATCH 0  // neo-Hookean apply: both voxels' tangent rows loaded before either contraction
#endif
#ifndef DBF_X_TPIPE
#define DBF_X_TPIPE 0  // 1: software-pipelined tangent loads across voxels (spilled: 256^3 0.911 -> 1.015 ms)
#endif
#ifndef DBF_X_PACK
#define DBF_X_PACK 0  // 1: finite-strain apply kinds pair the 9 fields of two lines into 9 FFT jobs (B200 256^3: 0.990 -> 1.058 ms, slower)
#endif
#ifndef DBF_COL_MINB
#define DBF_COL_MINB 4
#endif
// (the 168-register cap of these 288-thread kernels is the hardware's: 9 warps put 3 on one SM
// sub-partition of 16 K registers; __maxnreg__(208) fails to launch)
#ifndef DBF_COL_XINPLACE
#define DBF_COL_XINPLACE 0  // 1: TMA column passes run their FFT exchanges inside the output tile's own staging slots (no 32 KB exchange buffer, 60 KB of L1 instead of 28): parity green, 4-10 % slower (256^3 finite I1 0.257 -> 0.282, F2 0.432 -> 0.471 ms)
#endif
#ifndef DBF_UPD_TAB
#define DBF_UPD_TAB 0  // the fused F3 + residual update with the stage table (and a 2-slot ring to fit)
#endif
#ifndef DBF_COL_TAB512
#define DBF_COL_TAB512 0  // stage-table twiddles in the N = 512 TMA column passes too
#endif
namespace {

// ------------------------------------------------------------------------------------------------
// Column passes
// ------------------------------------------------------------------------------------------------
struct ColAt {
  const ColGeom* g;
  int outer, pos, kx;
  double xxk, xyo;  // xi_x(kx) and xi_y(outer) of the column (set with kx / outer; y passes: xyo unused)
  double xp;        // xi along the pass's FFT axis at `pos` (z passes: xi_z, y passes: xi_y)
  DBF_DEV void set_col(int o, int k) {
    outer = o;
    kx = k;
    xxk = __ldg(g->fq.xx + k);
    xyo = __ldg(g->fq.xy + (o < g->n_xy ? o : 0));
  }
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

// Each pass is a list of NT "terms".  Term j FFTs one pre-weighted combination of one or two
// input fields (raw values loaded first, so the next term's loads can be issued before the
// current FFT: software pipelining in registers) and adds post-weight x FFT into output o.
struct TermInfo {
  int o;       // output field
  int first;   // first term of output o
  int last;    // last term of output o (store)
  int f0, f1;  // input fields (f1 < 0: single field)
};

template <int KIND>
struct ColOp;

// z inverse, small strain.  outer = ky, pos = kz.  out {u_x, u_y, eps_zz, eps_xz, eps_yz}
template <>
struct ColOp<COL_I1S> {
  static constexpr bool INV = true;
  static constexpr int NT = 5, MAXIN = 2;
  DBF_DEV static TermInfo term(int j) {
    switch (j) {
      case 0: return {0, 1, 1, 0, -1};
      case 1: return {1, 1, 1, 1, -1};
      case 2: return {2, 1, 1, 2, -1};
      case 3: return {3, 1, 1, 0, 2};
      default: return {4, 1, 1, 1, 2};
    }
  }
  DBF_DEV static cplx pre(const ColAt& a, int j, cplx r0, cplx r1) {
    const double xz = a.xp;
    switch (j) {
      case 0: case 1: return r0;
      case 2: return cimul(r0, xz);  // eps_zz
      case 3: { const double xx = a.xxk; return cimul(make_double2(xz * r0.x + xx * r1.x, xz * r0.y + xx * r1.y), 0.5); }
      default: { const double xy = a.xyo; return cimul(make_double2(xz * r0.x + xy * r1.x, xz * r0.y + xy * r1.y), 0.5); }
    }
  }
  DBF_DEV static cplx post(const ColAt&, int) { return make_double2(1.0, 0.0); }
};

// z inverse, finite strain: u_i, G_iz = i xi_z u_i
template <>
struct ColOp<COL_I1F> {
  static constexpr bool INV = true;
  static constexpr int NT = 6, MAXIN = 1;
  DBF_DEV static TermInfo term(int j) { return {j, 1, 1, j < 3 ? j : j - 3, -1}; }
  DBF_DEV static cplx pre(const ColAt& a, int j, cplx r0, cplx) { return j < 3 ? r0 : cimul(r0, a.xp); }
  DBF_DEV static cplx post(const ColAt&, int) { return make_double2(1.0, 0.0); }
};

// y inverse, small strain.  outer = z, pos = ky.  in: {u_x, u_y, eps_zz, eps_xz, eps_yz}
// out (Voigt): {xx, yy, zz, yz, xz, xy}
template <>
struct ColOp<COL_I2S> {
  static constexpr bool INV = true;
  static constexpr int NT = 6, MAXIN = 2;
  DBF_DEV static TermInfo term(int j) {
    switch (j) {
      case 0: return {0, 1, 1, 0, -1};
      case 1: return {1, 1, 1, 1, -1};
      case 2: return {2, 1, 1, 2, -1};
      case 3: return {3, 1, 1, 4, -1};
      case 4: return {4, 1, 1, 3, -1};
      default: return {5, 1, 1, 0, 1};
    }
  }
  DBF_DEV static cplx pre(const ColAt& a, int j, cplx r0, cplx r1) {
    switch (j) {
      case 0: return cimul(r0, a.xxk);
      case 1: return cimul(r0, a.xp);
      case 5: { const double xx = a.xxk, xy = a.xp;
                return cimul(make_double2(xy * r0.x + xx * r1.x, xy * r0.y + xx * r1.y), 0.5); }
      default: return r0;
    }
  }
  DBF_DEV static cplx post(const ColAt&, int) { return make_double2(1.0, 0.0); }
};

// y inverse, finite strain.  in: {u_0,u_1,u_2, G_0z,G_1z,G_2z}; out o = 3i+j:
// j=0: G_ix = i xi_x u_i (post-weight: xi_x is constant along a y column), j=1: G_iy = i xi_y u_i,
// j=2: G_iz.
template <>
struct ColOp<COL_I2F> {
  static constexpr bool INV = true;
  static constexpr int NT = 9, MAXIN = 1;
  DBF_DEV static TermInfo term(int j) {
    const int i = j / 3, jj = j % 3;
    return {j, 1, 1, jj == 2 ? 3 + i : i, -1};
  }
  DBF_DEV static cplx pre(const ColAt& a, int j, cplx r0, cplx) { return (j % 3 == 1) ? cimul(r0, a.xp) : r0; }
  DBF_DEV static cplx post(const ColAt& a, int j) {
    return (j % 3 == 0) ? make_double2(0.0, a.xxk) : make_double2(1.0, 0.0);
  }
};

template <>
struct ColOp<COL_F2S> {
  static constexpr bool INV = false;
  static constexpr int NT = 6, MAXIN = 1;
  DBF_DEV static TermInfo term(int j) { return {j, 1, 1, j, -1}; }
  DBF_DEV static cplx pre(const ColAt&, int, cplx r0, cplx) { return r0; }
  DBF_DEV static cplx post(const ColAt&, int) { return make_double2(1.0, 0.0); }
};

// y forward, finite strain.  in o=3i+j: {P_ix, P_iy, P_iz};  out: g_i = -i xi_x P_ix - i xi_y P_iy, P_iz
template <>
struct ColOp<COL_F2F> {
  static constexpr bool INV = false;
  static constexpr int NT = 9, MAXIN = 1;
  DBF_DEV static TermInfo term(int j) {
    if (j < 6) return {j / 2, (j & 1) == 0, (j & 1) == 1, 3 * (j / 2) + (j & 1), -1};
    return {j - 3, 1, 1, 3 * (j - 6) + 2, -1};
  }
  DBF_DEV static cplx pre(const ColAt& a, int j, cplx r0, cplx) {
    return (j < 6 && (j & 1) == 0) ? cimul(r0, -a.xxk) : r0;
  }
  DBF_DEV static cplx post(const ColAt& a, int j) {
    if (j < 6 && (j & 1)) return make_double2(0.0, -a.xp);
    return make_double2(1.0, 0.0);
  }
};

// z forward + divergence, small strain.  outer = ky, pos = kz.  in Voigt sigma:
// f_x = Z(-i(xi_x s_xx + xi_y s_xy)) - i xi_z Z(s_xz), etc.  (R3 sign)
template <>
struct ColOp<COL_F3S> {
  static constexpr bool INV = false;
  static constexpr int NT = 6, MAXIN = 2;
  DBF_DEV static TermInfo term(int j) {
    const int o = j / 2;
    const int fa = (o == 0) ? 0 : (o == 1) ? 5 : 4;  // s_ox
    const int fb = (o == 0) ? 5 : (o == 1) ? 1 : 3;  // s_oy
    const int fz = (o == 0) ? 4 : (o == 1) ? 3 : 2;  // s_oz
    if ((j & 1) == 0) return {o, 1, 0, fa, fb};
    return {o, 0, 1, fz, -1};
  }
  DBF_DEV static cplx pre(const ColAt& a, int j, cplx r0, cplx r1) {
    if (j & 1) return r0;
    const double xx = a.xxk, xy = a.xyo;
    return cimul(make_double2(xx * r0.x + xy * r1.x, xx * r0.y + xy * r1.y), -1.0);
  }
  DBF_DEV static cplx post(const ColAt& a, int j) {
    if (j & 1) return make_double2(0.0, -a.xp);
    return make_double2(1.0, 0.0);
  }
};

template <>
struct ColOp<COL_F3F> {
  static constexpr bool INV = false;
  static constexpr int NT = 6, MAXIN = 1;
  DBF_DEV static TermInfo term(int j) {
    const int o = j / 2;
    if ((j & 1) == 0) return {o, 1, 0, o, -1};
    return {o, 0, 1, 3 + o, -1};
  }
  DBF_DEV static cplx pre(const ColAt&, int, cplx r0, cplx) { return r0; }
  DBF_DEV static cplx post(const ColAt& a, int j) {
    if (j & 1) return make_double2(0.0, -a.xp);
    return make_double2(1.0, 0.0);
  }
};

template <>
struct ColOp<COL_ZI3> {
  static constexpr bool INV = true;
  static constexpr int NT = 3, MAXIN = 1;
  DBF_DEV static TermInfo term(int j) { return {j, 1, 1, j, -1}; }
  DBF_DEV static cplx pre(const ColAt&, int, cplx r0, cplx) { return r0; }
  DBF_DEV static cplx post(const ColAt&, int) { return make_double2(1.0, 0.0); }
};
template <>
struct ColOp<COL_YI3> : ColOp<COL_ZI3> {};

// plain transforms of NF fields (no weights): residual monitors
template <int NF, bool INVERSE>
struct ColPlain {
  static constexpr bool INV = INVERSE;
  static constexpr int NT = NF, MAXIN = 1;
  DBF_DEV static TermInfo term(int j) { return {j, 1, 1, j, -1}; }
  DBF_DEV static cplx pre(const ColAt&, int, cplx r0, cplx) { return r0; }
  DBF_DEV static cplx post(const ColAt&, int) { return make_double2(1.0, 0.0); }
};
template <> struct ColOp<COL_ZI6> : ColPlain<6, true> {};
template <> struct ColOp<COL_YI6> : ColPlain<6, true> {};
template <> struct ColOp<COL_ZF3> : ColPlain<3, false> {};
template <> struct ColOp<COL_YF3> : ColPlain<3, false> {};
template <> struct ColOp<COL_ZF6> : ColPlain<6, false> {};
template <> struct ColOp<COL_YF6> : ColPlain<6, false> {};

template <int KIND>
struct ColTwo {  // does any output of this pass sum two transformed terms?
  static constexpr bool value = (KIND == COL_F2F || KIND == COL_F3S || KIND == COL_F3F);
};

// Column-pass CTA geometry: 256 threads; a column's length-N FFT is done by N/8 threads
// (8 points each); columns are kx-contiguous so each warp load is 128-byte row segments.
// Odd N (the paper's 63^3 grids): OddPlan<N>::P points per thread, mixed radix.
template <int N>
struct ColCfg {
  static constexpr bool ODD = (N & 1) != 0;
  static constexpr int P = PtsPerThread<N>::value;  // points per thread
  static constexpr int TPC = N / P;
  static constexpr int COLS = 256 / TPC;
  static constexpr int THREADS = COLS * TPC;
};

// the in-CTA FFT of a column pass / X pair: radix-8 (powers of two) or mixed radix (odd N)
template <int N, bool INV, class IDX, class SYNC>
DBF_DEV void fft_col(cplx (&a)[ColCfg<N>::P], cplx* sbuf, int g, const IDX& idx, const cplx* __restrict__ tw, const SYNC& sync) {
  if constexpr (ColCfg<N>::ODD) fft_odd<N, INV>(a, sbuf, g, idx, tw, sync);
  else fft_cta<N, INV>(a, sbuf, g, idx, tw, sync);
}

// single-term passes pipeline the next term's loads in registers (2 CTAs/SM); two-term
// passes keep the first term in shared memory and run without prefetch (3 CTAs/SM)
template <int KIND>
struct ColPref {
  static constexpr bool value = !ColTwo<KIND>::value && ColOp<KIND>::MAXIN == 1;
  static constexpr int MINB = ColTwo<KIND>::value ? 3 : 2;
};

template <int N, int KIND>
__global__ void __launch_bounds__(256, ColCfg<N>::ODD ? 1 : ColPref<KIND>::MINB) col_pass_kernel(ColGeom g) {
  DBF_PDL_ENTRY_BIG();
  if (g.cg_stop0 && (*g.cg_stop0 | *g.cg_stop1)) return;  // PCG stopped: nothing to compute
  typedef ColOp<KIND> Op;
  typedef ColCfg<N> CF;
  constexpr int P = CF::P, TPC = CF::TPC, COLS = CF::COLS;
  constexpr bool TWO = ColTwo<KIND>::value;
  constexpr bool PREF = ColPref<KIND>::value;
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
  at.set_col(valid ? (int)(col / g.n1h) : 0, valid ? (int)(col % g.n1h) : 0);
  IdxCols<COLS> idx{c};
  cplx r0[PREF ? P : 1];
  if (PREF) {
    const TermInfo ti = Op::term(0);
#pragma unroll
    for (int s = 0; s < P; ++s) {
      at.pos = gq + s * TPC;
      at.xp = __ldg(g.fpos + at.pos);
      r0[PREF ? s : 0] = valid ? at.in(ti.f0) : make_double2(0.0, 0.0);
    }
  }
#pragma unroll 1
  for (int j = 0; j < Op::NT; ++j) {
    const TermInfo ti = Op::term(j);
    cplx a[P];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      at.pos = gq + s * TPC;
      at.xp = __ldg(g.fpos + at.pos);
      if (PREF) {
        a[s] = Op::pre(at, j, r0[PREF ? s : 0], r0[PREF ? s : 0]);
      } else {
        const cplx v0 = valid ? at.in(ti.f0) : make_double2(0.0, 0.0);
        const cplx v1 = (valid && ti.f1 >= 0) ? at.in(ti.f1) : make_double2(0.0, 0.0);
        a[s] = Op::pre(at, j, v0, v1);
      }
    }
    if (PREF && j + 1 < Op::NT) {  // issue the next term's loads; they fly during this FFT
      const TermInfo tn = Op::term(j + 1);
#pragma unroll
      for (int s = 0; s < P; ++s) {
        at.pos = gq + s * TPC;
        at.xp = __ldg(g.fpos + at.pos);
        r0[PREF ? s : 0] = valid ? at.in(tn.f0) : make_double2(0.0, 0.0);
      }
    }
    fft_col<N, Op::INV>(a, sbuf, gq, idx, g.tw, SyncCtaDefault{});
#pragma unroll
    for (int s = 0; s < P; ++s) {
      at.pos = gq + s * TPC;
      at.xp = __ldg(g.fpos + at.pos);
      cplx v = cmul(Op::post(at, j), a[s]);
      if (TWO && !ti.first) v = cadd(v, sacc[idx(at.pos)]);
      if (!ti.last) {
        if (TWO) sacc[idx(at.pos)] = v;  // own positions only: no barrier needed
      } else if (valid) {
        g.out[at.out_idx(ti.o)] = v;
      }
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
template <> struct XTraits<X_REAL_IN> { static constexpr int CIN = 0, COUT = 9, NRED = 0; static constexpr bool FIN = false; };

DBF_DEV int sym9(int i, int j) {
  if (i > j) { int t = i; i = j; j = t; }
  return i * 9 - i * (i - 1) / 2 + (j - i);
}

// Voigt index (xx,yy,zz,yz,xz,xy) -> row-major 3x3 entry
// (a compile-time function: with the loops unrolled every index folds to a constant, so the
// per-thread accumulators red[] stay in registers — a __constant__ table index put red[] in local
// memory: 28 % of the J2 pass_X stall samples at 512^3)
DBF_DEV constexpr int row9_of_voigt(int I) { return I == 0 ? 0 : I == 1 ? 4 : I == 2 ? 8 : I == 3 ? 5 : I == 4 ? 2 : 1; }

// streaming load of per-voxel data (read once per launch: do not allocate in L1)
DBF_DEV double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// small-strain contraction: sigma_I = sum_J C[I][J] gamma_J, gamma = (e0,e1,e2,2e3,2e4,2e5); the
// stiffness is symmetric, so its 21 upper-triangle entries are loaded (not 36)
DBF_DEV void voigt_contract_full(const double* __restrict__ C36, const double* e, double* s) {
  const double g[6] = {e[0], e[1], e[2], 2.0 * e[3], 2.0 * e[4], 2.0 * e[5]};
  double c[6][6];
#pragma unroll
  for (int I = 0; I < 6; ++I)
#pragma unroll
    for (int J = I; J < 6; ++J) c[I][J] = c[J][I] = __ldg(C36 + 6 * I + J);
#pragma unroll
  for (int I = 0; I < 6; ++I) {
    double acc = 0.0;
#pragma unroll
    for (int J = 0; J < 6; ++J) acc = fma(c[I][J], g[J], acc);
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
  const double sy = prm[2], nexp = prm[3], edot0 = prm[4];
  const double mu = prm[5], kappa = prm[6];  // per-phase moduli from set_phases (no divisions here)
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
    // x^(n-1) by binary powering when the rate exponent is an integer (c5: n = 20), else pow
    const int ni = (int)nexp;
    const bool nint = (double)ni == nexp && ni >= 1 && ni <= 64;
    auto xpow_n1 = [&](double b) {
      if (!nint) return pow(b, nexp - 1.0);
      double r = 1.0;
      for (int e = ni - 1; e; e >>= 1, b *= b)
        if (e & 1) r *= b;
      return r;
    };
    double lo = 0.0, hi = svm / sy - 1.0, x = 0.5 * hi;
    for (int it = 0; it < 200; ++it) {
      const double xn1 = xpow_n1(x);
      const double gx = svm - m3 * xn1 * x - sy * (1.0 + x);
      if (gx > 0) lo = x; else hi = x;
      const double dg = -m3 * nexp * xn1 - sy;
      double xn = x - gx / dg;
      if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
      if (fabs(xn - x) <= 1e-16 * x || hi - lo <= 1e-16 * hi) { x = xn; break; }
      x = xn;
    }
    const double xn1 = xpow_n1(x);
    dp = rdt * x * xn1;  // rdt x^n
    theta = 1.0 - 3.0 * mu * dp / svm;
    // H' = d(sy (1 + x))/d(dp) = sy/(n rdt) (dp/rdt)^(1/n - 1) = sy/(n rdt) x^(1 - n)
    const double Hp = (dp > 0) ? sy / (nexp * rdt) / xn1 : 0.0;
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
  // (tr / 3 kept as a division: a hoisted tr * (1/3) made ptxas spill 184 bytes in the J2 pass_X)
  for (int I = 0; I < 6; ++I) s[I] = a * (e[I] - (I < 3 ? tr / 3.0 : 0.0)) - b * tc[2 + I] + (I < 3 ? kappa * tr : 0.0);
}

// shear and bulk moduli of a J2 phase: computed once per phase on the host (set_phases:
// lam = E nu / ((1 + nu)(1 - 2 nu)), mu = E / (2 (1 + nu)), kappa = lam + 2 mu / 3), not three
// fp64 divisions per voxel
DBF_DEV void j2_moduli(const double* prm, double* kappa, double* mu) {
  *mu = __ldg(prm + 5);
  *kappa = __ldg(prm + 6);
}

// Per-voxel material data of the apply kinds come either from global memory (tp = tan + v,
// ts = nvox) or from the CTA's shared-memory stage filled by bulk async copies (ts = N1).
// xd: the apply kinds accumulate grad p : sigma of the voxel, so <p_u, K p_u> = sum / N (Parseval:
// the operator's Hermitian form in real space, sigma including the macro part; FIN_NH accumulates
// the 1/(2N)-scaled P)
template <int KIND>
DBF_DEV void x_voxel(const XGeom& g, long long v, double* G, double* P, double* red, const double* tp, long long ts, int ph,
                     double& xd, const double* se, const double* tpre = nullptr) {
  if (KIND == X_K_SMALL_PHASE || KIND == X_RHS_SMALL_PHASE || KIND == X_K_J2) {
    double e6[6];
#pragma unroll
    for (int I = 0; I < 6; ++I)
      e6[I] = (KIND == X_RHS_SMALL_PHASE ? 0.0 : G[I]) + (se ? se[row9_of_voigt(I)] : 0.0);
    double s[6];
    if (KIND == X_K_J2) {
      double tc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) tc[k] = tp[k * ts];
      double kappa, mu;
      j2_moduli(g.ptable + 36 * ph, &kappa, &mu);
      j2_apply(tc, kappa, mu, e6, s);
    } else {
      voigt_contract_full(g.ptable + 36 * ph, e6, s);
    }
    if (KIND != X_RHS_SMALL_PHASE)
      xd += G[0] * s[0] + G[1] * s[1] + G[2] * s[2] + 2.0 * (G[3] * s[3] + G[4] * s[4] + G[5] * s[5]);
    const double sg = (KIND == X_RHS_SMALL_PHASE) ? -g.oscale : g.oscale;
#pragma unroll
    for (int I = 0; I < 6; ++I) {
      P[I] = sg * s[I];
      // the apply kinds read <sigma> off the R2C's k = 0 outputs instead (XDcRed)
      if (KIND == X_RHS_SMALL_PHASE) red[row9_of_voigt(I)] += s[I];
    }
  } else if (KIND == X_K_FIN_TAN) {
    double e9[9], K[45];
#pragma unroll
    for (int k = 0; k < 45; ++k) K[k] = ld_stream(tp + k * ts);
#pragma unroll
    for (int a = 0; a < 9; ++a) e9[a] = G[a] + (se ? se[a] : 0.0);
#pragma unroll
    for (int a = 0; a < 9; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < 9; ++b) acc = fma(K[sym9(a, b)], e9[b], acc);
      P[a] = acc * g.oscale;
      red[a] += acc;
      xd += G[a] * acc;
    }
  } else if (KIND == X_K_FIN_NH) {
    double Fi[9], e9[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Fi[k] = tpre ? tpre[k] : tp[k * ts];
    const double c1 = tpre ? tpre[9] : tp[9 * ts];
    // lam = kappa - 2 mu / 3 per phase from set_phases (ptable[3]): no fp64 division per voxel
    const double mu = __ldg(g.ptable + 36 * ph), lam = __ldg(g.ptable + 36 * ph + 3);
#pragma unroll
    for (int a = 0; a < 9; ++a) e9[a] = G[a] + (se ? se[a] : 0.0);
    nh_apply(Fi, c1 * g.oscale, mu * g.oscale, lam * g.oscale, e9, P);  // P x 1/(2N): exact for powers of 2
#pragma unroll
    for (int a = 0; a < 9; ++a) xd += G[a] * P[a];
  } else if (KIND == X_CONST_FIN) {
    double F[9], Pv[9], Fi[9], c1;
    double mx = 0.0;
#pragma unroll
    for (int a = 0; a < 9; ++a) {
      const double d = (g.has_in ? G[a] : 0.0) + se[a];
      mx = fmax(mx, fabs(d));
      F[a] = g.F[(long long)a * g.nvox + v] + d;
      g.F[(long long)a * g.nvox + v] = F[a];
    }
    const int ph = __ldg(g.phase + v);
    if (__ldg(g.ptable + 36 * ph + 2) != 0.0) {  // Saint Venant-Kirchhoff phase (full tangent storage)
      const double mu = __ldg(g.ptable + 36 * ph), lam = __ldg(g.ptable + 36 * ph + 1);
      double S[9], K45[45];
      svk_stress(F, mu, lam, Pv, S);
      svk_tangent45(F, S, mu, lam, K45);
#pragma unroll
      for (int k = 0; k < 45; ++k) g.tan[(long long)k * g.nvox + v] = K45[k];
#pragma unroll
      for (int a = 0; a < 9; ++a) {
        P[a] = -g.oscale * Pv[a];
        red[a] += Pv[a];
      }
      red[9] = fmax(red[9], mx);
      return;
    }
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
      P[a] = -g.oscale * Pv[a];
      red[a] += Pv[a];
    }
    red[9] = fmax(red[9], mx);
  } else if (KIND == X_CONST_J2) {
    double eps[6], ep[6], s[6], tc[8], epn[6];
    double mx = 0.0;
#pragma unroll
    for (int I = 0; I < 6; ++I) {
      const double d = (g.has_in ? G[I] : 0.0) + se[row9_of_voigt(I)];
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
      P[I] = -g.oscale * s[I];
      red[row9_of_voigt(I)] += s[I];
    }
    red[9] = fmax(red[9], mx);
  }
}

// Real slots of pass_X: field c (line-major: c = l CS + f) at position x; the two fields of a pair
// (c = 2q, 2q + 1) are interleaved, so a pair job's reals are one complex array (its FFT's own
// input / output, 16-byte accesses) and a voxel reads a line's fields as CS/2 16-byte loads
// (ILV = false: field-major slots c N1 + x, the layout the 6-field kinds keep — interleaving
// raised their register pressure into spills, 256^3 small pass_X 0.759 -> 0.780 ms)
template <int N1, bool ILV = true>
DBF_DEV int x_slot(int c, int x) {
  return ILV ? (((c >> 1) * N1 + x) << 1) + (c & 1) : c * N1 + x;
}

// XOR swizzle inside 8-element groups: conflict-free radix-8 scatter/gather, no padding, so
// the exchange buffer of a field pair is exactly the pair's two real slots (in place).
struct IdxSwz {
  int base;
  DBF_DEV int operator()(int pos) const { return base + (pos ^ ((pos >> 3) & 7)); }
};

// pass_X FFT of one field pair: radix-8 with CTA-wide exchange barriers (P = 8) or radix-16
// with warp-local exchanges (P = 16, the pair's threads share a warp)
struct IdxPlain {
  int base;
  DBF_DEV int operator()(int pos) const { return base + pos; }
};
template <int N1, int P>
DBF_DEV int x_idx(int base, int pos) {
  return (N1 & 1) ? IdxPlain{base}(pos) : P == 16 ? IdxGrp{base}(pos) : IdxSwz{base}(pos);
}
// exchange sync of one pair job (N1 / P threads): the warp when the job fits in one; a named
// barrier of the job's warps when it spans several (N1 = 512: 64 threads, ids 1 + job); the CTA
// barrier otherwise (odd lengths: jobs of 3 threads straddle warps)
template <int N1, int P>
DBF_DEV void x_jobsync(int job) {
  constexpr int TPJ = N1 / P;
  if (TPJ <= 32 && 32 % TPJ == 0) __syncwarp();
  else if (TPJ % 32 == 0) asm volatile("bar.sync %0, %1;" ::"r"(1 + job), "r"(TPJ) : "memory");
  else __syncthreads();
}
template <int N1, int P>
struct XSync {
  int job;
  DBF_DEV void operator()() const { x_jobsync<N1, P>(job); }
};
template <int N1, int P, bool INV, bool TAB>
DBF_DEV void x_fft(cplx (&a)[P], cplx* cx, int gq, int base, const cplx* __restrict__ tw, int job) {
  if constexpr ((N1 & 1) != 0) {
    fft_odd<N1, INV>(a, cx, gq, IdxPlain{base}, tw, XSync<N1, P>{job});
  } else if constexpr (P == 16) {
    fft_sub<N1, 16, INV>(a, cx, gq, IdxGrp{base}, tw, XSync<N1, 16>{job});
  } else {
    fft_cta<N1, INV, IdxSwz, XSync<N1, 8>, TAB>(a, cx, gq, IdxSwz{base}, tw, XSync<N1, 8>{job});  // TAB: stage table
  }
}

// Z[N-k] of the R2C untangle for the thread's outputs k = gq + s TPJ: held by job thread
// (TPJ - gq) % TPJ in slot 7 - s (gq > 0) or by this thread in slot (8 - s) % 8 (gq = 0),
// fetched with shuffles inside the job's warp segment (TPJ <= 32, P = 8).
template <int TPJ>
DBF_DEV void x_partner(const cplx (&a)[8], cplx (&zn)[8], int gq) {
  const int src = (TPJ - gq) & (TPJ - 1);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const cplx v = a[7 - s];
    cplx r;
    r.x = __shfl_sync(0xffffffffu, v.x, src, TPJ);
    r.y = __shfl_sync(0xffffffffu, v.y, src, TPJ);
    zn[s] = (gq == 0) ? a[(8 - s) & 7] : r;
  }
}

// pass_X line positions k = gq + s TPJ (TPJ PX = N1): k <= N1/2 ("lo", stored half spectrum)
// is static except at s = PX/2, where only gq = 0 (k = N1/2) qualifies
template <int N1, int PX, int TPJ>
DBF_DEV bool x_lo(int s, int gq) {
  if (TPJ * PX != N1 || (N1 & 1)) return 2 * (gq + s * TPJ) <= N1;
  return s < PX / 2 || (s == PX / 2 && gq == 0);
}
// apply kinds reduce <out> from the R2C DC (sums over the line), no per-voxel accumulators
template <int KIND>
struct XDcRed {
  static constexpr bool value = (KIND == X_K_SMALL_PHASE || KIND == X_K_J2 || KIND == X_K_FIN_TAN || KIND == X_K_FIN_NH);
};
// reduction slot (row-major 3x3) of output field f: Voigt components at small strain
template <int KIND>
DBF_DEV int x_red_slot(int f) {
  if (XTraits<KIND>::FIN) return f;
  return f == 0 ? 0 : f == 1 ? 4 : f == 2 ? 8 : f == 3 ? 5 : f == 4 ? 2 : 1;
}

// Which apply kinds stream their inputs through the shared-memory stage (bulk async copies)
template <int KIND>
struct XStage {
  static constexpr bool IN = DBF_X_STAGE_IN && (KIND == X_K_SMALL_PHASE || KIND == X_K_J2 || KIND == X_K_FIN_TAN || KIND == X_K_FIN_NH);
  static constexpr int NTAN = (KIND == X_K_J2) ? (DBF_X_STAGE_TAN_J2 ? 8 : 0) : (KIND == X_K_FIN_NH) ? (DBF_X_STAGE_TAN_NH ? 10 : 0) : 0;  // staged per-voxel doubles
  static constexpr bool PH = (KIND == X_K_SMALL_PHASE || KIND == X_K_J2 || KIND == X_K_FIN_NH);
};

template <int N1, int KIND>
struct XCfg {
  typedef XTraits<KIND> T;
  typedef XStage<KIND> S;
  static constexpr int C = (T::CIN > T::COUT) ? T::CIN : T::COUT;
  // PACK (an odd field count, 9): the fields of LPAR (even) lines are numbered line-major and
  // paired consecutively — the 18 fields of two lines make 9 pair FFTs, one pair spanning the two
  // lines, instead of 2 x 5 pairs with an empty slot each (10 % less FFT work, and the voxel loop
  // of 512 voxels over 288 threads idles less than 256 voxels over 160)
  static constexpr bool PACK = DBF_X_PACK && (C & 1) && (N1 & 1) == 0 && (KIND == X_K_FIN_NH || KIND == X_K_FIN_TAN);
  static constexpr int CS = PACK ? C : (C + 1) & ~1;  // real slots per line
  // FFT points per thread: radix-16 stages with warp-local exchanges (16) for the kinds in the
  // P16 masks (bit = kind; N1 <= 256 and N1 = 512 separately), else radix-8 (8)
  static constexpr unsigned P16M = (N1 <= 256) ? DBF_X_P16_256 : DBF_X_P16_512;
  static constexpr bool P16 = (N1 & 1) == 0 && N1 >= 32 && KIND < 32 && ((P16M >> KIND) & 1u);
  static constexpr int PX = (N1 & 1) ? PtsPerThread<N1>::value : P16 ? 16 : 8;
  static constexpr int TPJ = N1 / PX;              // threads per pair FFT (divides 32: warp-local)
  static constexpr int NP = CS / 2;
  static constexpr int PERLINE = TPJ * NP;
  // PACK: 64/TPJ lines (at least 2) so that the CTA is whole warps (the untangle shuffles)
  static constexpr int LRAW = PACK ? (TPJ >= 32 ? 2 : 64 / TPJ) : (C == 9 ? DBF_X_LRAW9 : P16 ? DBF_X_LRAW16 : KIND == X_K_J2 ? DBF_X_LRAWJ2 : DBF_X_LRAW) / PERLINE;
  static constexpr int LPAR = LRAW >= 64 ? 64 : LRAW >= 32 ? 32 : LRAW >= 16 ? 16 : LRAW >= 8 ? 8 : LRAW >= 4 ? 4 : LRAW >= 2 ? 2 : 1;
  static constexpr int NJOB = PACK ? LPAR * C / 2 : LPAR * NP;  // pair FFT jobs per line group
  static constexpr int THREADS = NJOB * TPJ;
  static_assert(!PACK || THREADS % 32 == 0, "packed pass_X CTAs are whole warps");
  static constexpr int N1H = N1 / 2 + 1;
  static constexpr size_t SLOTS = sizeof(double) * LPAR * CS * N1;
  // bulk-copy staging needs 16-byte rows: powers of two only (odd lines load directly)
  static constexpr bool STG = S::IN && (N1 & 1) == 0;
  static constexpr bool STG_SPEC = STG && DBF_X_STAGE_SPEC;
  static constexpr size_t ST_IN = STG_SPEC ? sizeof(cplx) * LPAR * T::CIN * N1H : 0;
  static constexpr size_t ST_TAN = STG ? sizeof(double) * LPAR * S::NTAN * N1 : 0;
  // PH2: only phase ids staged (no tangent rows): two buffers, group g+1's copy issued when group g
  // starts (a whole group of lead time instead of the R2C + C2R)
  // (6-field kinds only: the 9-field neo-Hookean pass measured 0.5 % slower with it)
  static constexpr bool PH2 = STG && S::PH && S::NTAN == 0 && C != 9;
  static constexpr size_t ST_PH1 = (STG && S::PH) ? ((sizeof(uint16_t) * LPAR * N1 + 15) & ~size_t(15)) : 0;
  static constexpr size_t ST_PH = PH2 ? 2 * ST_PH1 : ST_PH1;
  // stage-ordered twiddles (N1 - 1) in shared memory for the 9-field kinds (B200 256^3 finite
  // pass_X 1.099 -> 0.990 ms); the 6-field small-strain kinds measured a little slower with it
  static constexpr bool TAB = (N1 & 1) == 0 && C == 9 && PX == 8;  // (the table is the radix-8 plan's)
  static constexpr size_t ST_TW = TAB ? sizeof(cplx) * N1 : 0;
  static constexpr bool ILV = C == 9;  // pair-interleaved real slots (x_slot)
  static constexpr size_t SMEM = SLOTS + ST_IN + ST_TAN + ST_PH + 32 + ST_TW;  // + 3 mbarriers (+ pad)
  // (CTAs of more than 256 threads — the 9-field kinds at n1 = 512 — take 2 per SM: at 4 their
  // 320 threads were capped at 48 registers and spilled 424 bytes)
  static constexpr int MINB = PACK ? (THREADS <= 160 ? DBF_X_MINB_NOTAN : THREADS <= 320 ? 2 : 1)
                               : (THREADS > 256) ? 2
                               : (KIND == X_K_J2 && P16) ? DBF_X_MINB_J2P16
                               : (KIND == X_K_J2 && !DBF_X_STAGE_TAN_J2) ? DBF_X_MINB_NOTAN_J2
                               : (KIND == X_K_FIN_NH && !DBF_X_STAGE_TAN_NH) ? DBF_X_MINB_NOTAN
                               : (KIND == X_CONST_FIN || KIND == X_CONST_J2) ? DBF_X_MINB_CONST
                               : (THREADS <= 192) ? DBF_X_MINB : 2;
};

// per-voxel tangent arrays an apply kind reads in its voxel loop from global memory (L2-prefetched
// one line group ahead)
template <int KIND>
struct XPref {
  static constexpr int NTAN = DBF_X_PREFETCH ? ((KIND == X_K_FIN_NH) ? (DBF_X_STAGE_TAN_NH ? 0 : 10)
                                              : (KIND == X_K_J2) ? (DBF_X_STAGE_TAN_J2 ? 0 : 8)
                                              : (KIND == X_K_FIN_TAN) ? 45 : 0) : 0;
};
DBF_DEV void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p) : "memory"); }
DBF_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- bulk async copy (TMA engine) + mbarrier helpers ------------------------------------------
DBF_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
DBF_DEV void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
DBF_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
DBF_DEV bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
DBF_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
DBF_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
DBF_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
DBF_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// pencil decomposition: offset of line kx k (0..n1/2) in the kx-chunked layout of XGeom.kch
// (chunk c = min(k / kch, npy - 1): the Nyquist sits in slot kch of the last chunk)
DBF_DEV long long x_koff(const XGeom& g, int k, long long pcs) {
  if (g.kch == 0) return k;
  const int c = min(k / g.kch, g.npy - 1);
  return (long long)c * pcs + (k - c * g.kch);
}

// issue the stage copies of line group `grp` (one elected thread)
template <int N1, int KIND>
DBF_DEV void x_issue_in(const XGeom& g, long long grp, cplx* st_in, uint64_t* bar) {
  typedef XCfg<N1, KIND> CF;
  constexpr int CIN = XTraits<KIND>::CIN;
  long long l0 = grp * CF::LPAR;
  const int nl = (int)min((long long)CF::LPAR, g.nlines - l0);
  const uint32_t row = sizeof(cplx) * CF::N1H;
  mbar_expect_tx(bar, row * CIN * nl);
  for (int l = 0; l < nl; ++l)
    for (int f = 0; f < CIN; ++f) {
      cplx* dst = st_in + (l * CIN + f) * CF::N1H;
      const cplx* src = g.in + f * g.fs_in + (l0 + l) * g.kxp;
      if (g.kch == 0) {
        bulk_g2s(dst, src, row, bar);
      } else {  // pencil: one copy per kx chunk (the last one carries the Nyquist)
        for (int c = 0; c < g.npy; ++c)
          bulk_g2s(dst + c * g.kch, src + c * g.kpcs_in, (uint32_t)sizeof(cplx) * (g.kch + (c == g.npy - 1 ? 1 : 0)), bar);
      }
    }
}
template <int N1, int KIND>
DBF_DEV void x_issue_tan(const XGeom& g, long long grp, double* st_tan, uint16_t* st_ph, uint64_t* bar) {
  typedef XCfg<N1, KIND> CF;
  typedef XStage<KIND> S;
  const long long l0 = grp * CF::LPAR;
  const int nl = (int)min((long long)CF::LPAR, g.nlines - l0);
  const long long v0 = l0 * N1;
  const uint32_t trow = sizeof(double) * N1 * nl;  // LPAR lines are contiguous voxels
  const uint32_t prow = sizeof(uint16_t) * N1 * nl;
  const uint32_t pbytes = S::PH ? ((prow + 15) & ~15u) : 0;
  mbar_expect_tx(bar, trow * S::NTAN + pbytes);
  for (int k = 0; k < S::NTAN; ++k) bulk_g2s(st_tan + k * (CF::LPAR * N1), g.tan + (long long)k * g.nvox + v0, trow, bar);
  if (S::PH) bulk_g2s(st_ph, g.phase + v0, pbytes, bar);
}

// X pass.  Persistent: each CTA loops over groups of LPAR lines.  Per line the C fields are
// C2R'd in pairs (z = a + i b), the per-voxel operation runs on the real fields in shared
// memory, and results are R2C'd in pairs and untangled:
//   A_k = (Z_k + conj Z_{N-k})/2,  B_k = (Z_k - conj Z_{N-k})/(2i).
// Apply kinds stream group i+1's spectra and per-voxel data into a shared-memory stage with
// bulk async copies (cp.async.bulk -> TMA engine, mbarrier completion) while group i computes.
template <int N1, int KIND>
__global__ void __launch_bounds__(XCfg<N1, KIND>::THREADS, XCfg<N1, KIND>::MINB) x_pass_kernel(XGeom g, int nf_real) {
  DBF_PDL_ENTRY_BIG();
  if (g.stop0 && (*g.stop0 | *g.stop1)) return;  // PCG stopped: nothing to compute
  typedef XCfg<N1, KIND> CF;
  typedef XTraits<KIND> T;
  typedef XStage<KIND> S;
  constexpr int C = CF::C, CS = CF::CS, TPJ = CF::TPJ, NP = CF::NP, LPAR = CF::LPAR, PX = CF::PX;
  constexpr bool SIN = CF::STG;  // stage per-voxel data (and the spectra: SSP) with bulk copies
  constexpr bool SSP = CF::STG_SPEC;
  extern __shared__ __align__(16) double real[];
  cplx* cx = reinterpret_cast<cplx*>(real);
  unsigned char* sb = reinterpret_cast<unsigned char*>(real);
  cplx* st_in = reinterpret_cast<cplx*>(sb + CF::SLOTS);
  double* st_tan = reinterpret_cast<double*>(sb + CF::SLOTS + CF::ST_IN);
  uint16_t* st_ph = reinterpret_cast<uint16_t*>(sb + CF::SLOTS + CF::ST_IN + CF::ST_TAN);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + CF::SLOTS + CF::ST_IN + CF::ST_TAN + CF::ST_PH);
  cplx* stab = reinterpret_cast<cplx*>(bars + 4);
  // odd lengths keep the plain W_N table (mixed-radix fft_odd); CF::TAB kinds the stage table
  const cplx* twx = CF::TAB ? stab : g.tw;
  if constexpr (CF::TAB) {
    for (int i = threadIdx.x; i < N1 - 1; i += CF::THREADS) stab[i] = __ldg(g.tw + N1 + i);
    __syncthreads();
  }
  const int t = threadIdx.x;
  const int job = t / TPJ, gq = t % TPJ;
  // the job's two fields: slots ca, cb of the line group (line-major, CS per line); without PACK
  // both lie in one line, with PACK a pair may span two lines
  const int ca = 2 * job, cb = 2 * job + 1;
  const int la = ca / CS, fa = ca % CS, lb = cb / CS, fb = cb % CS;
  const int jbase = (ca * N1) / 2;  // complex view of the job's two slots (its FFT exchange buffer)
  const int cin = (KIND == X_REAL_OUT) ? nf_real : T::CIN;
  const int cout_rt = (KIND == X_REAL_IN) ? nf_real : T::COUT;  // spectral outputs written
  const bool do_in = (T::CIN > 0) && (cin > 0) && ((KIND != X_CONST_FIN && KIND != X_CONST_J2) || g.has_in);
  const long long ngroups = (g.nlines + LPAR - 1) / LPAR;
  // apply kinds: <sigma> / <dP> from the k = 0 outputs of the R2C (one owner thread per field)
  constexpr bool DCRED = XDcRed<KIND>::value;
  __shared__ double s_dc[DCRED ? LPAR : 1][10];  // per line slot of the CTA: one owner thread per entry
  __shared__ double s_e[9];  // the macro block (read by every voxel; one load per CTA, not per voxel)
  if (DCRED)
    for (int i = t; i < 10 * LPAR; i += CF::THREADS) s_dc[i / 10][i % 10] = 0.0;
  if (g.e && t < 9) s_e[t] = g.e[t];
  __syncthreads();
  double xdot = 0.0;  // apply kinds: sum (G + e) : sigma over the CTA's voxels
  double red[T::NRED > 0 ? T::NRED : 1];
#pragma unroll
  for (int r = 0; r < (T::NRED > 0 ? T::NRED : 1); ++r) red[r] = 0.0;
  constexpr bool STAGE_TAN = (S::NTAN > 0 || S::PH);
  if (SIN) {
    if (t == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_init(&bars[2], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0 && (long long)blockIdx.x < ngroups) {
      if (SSP) x_issue_in<N1, KIND>(g, blockIdx.x, st_in, &bars[0]);
      if (STAGE_TAN) x_issue_tan<N1, KIND>(g, blockIdx.x, st_tan, st_ph, &bars[1]);
    }
  }
  uint32_t it = 0;

  for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    // PH2: this group's phase ids are in buffer it & 1 (barrier 1 + (it & 1)); the next group's go
    // to the other buffer now — its last reader, group it - 1, finished its voxel loop
    uint16_t* ph_cur = CF::PH2 ? st_ph + (it & 1) * (CF::ST_PH1 / sizeof(uint16_t)) : st_ph;
    if (CF::PH2 && t == 0 && grp + gridDim.x < ngroups) {
      fence_proxy_async();  // the buffer's generic-proxy reads (group it - 1) before the async write
      x_issue_tan<N1, KIND>(g, grp + gridDim.x, st_tan, st_ph + ((it + 1) & 1) * (CF::ST_PH1 / sizeof(uint16_t)),
                            &bars[1 + ((it + 1) & 1)]);
    }
    const long long linea = grp * LPAR + la, lineb = grp * LPAR + lb;
    // per-voxel data read in the voxel loop straight from global memory: the next group's rows
    // go to L2 now (bulk prefetch), so the voxel loop's loads hit L2 instead of HBM
    if (XPref<KIND>::NTAN > 0 && t == 0 && grp + gridDim.x < ngroups) {
      const long long v1 = (grp + gridDim.x) * LPAR * N1;
      const uint32_t bytes = (uint32_t)(sizeof(double) * N1 * min((long long)LPAR, g.nlines - (grp + gridDim.x) * LPAR));
#pragma unroll 1
      for (int k = 0; k < XPref<KIND>::NTAN; ++k) prefetch_l2(g.tan + (long long)k * g.nvox + v1, bytes);
    }
    // this group's rows (L2-resident since the previous group's prefetch) go on to L1 while the C2R
    // runs: the voxel loop's 10 loads per voxel then wait for an L1 hit, not an L2 round trip
    if constexpr (DBF_X_L1PF && KIND == X_K_FIN_NH && S::NTAN == 0 && LPAR == 1 && (N1 % 16) == 0) {
      constexpr int LPR = N1 / 16;  // 128-byte lines per tangent row of one voxel line
      const long long v0 = grp * N1;
      for (int i = t; i < 10 * LPR; i += CF::THREADS) prefetch_l1(g.tan + (long long)(i / LPR) * g.nvox + v0 + (i % LPR) * 16);
      if (!S::PH && t < (N1 + 63) / 64) prefetch_l1(g.phase + v0 + t * 64);
    }
    const bool va = linea < g.nlines, vb = lineb < g.nlines;
    const long long nxt = grp + gridDim.x;
    // ------------------------------------------------------------ inverse (C2R) of pairs
    if (do_in) {
      if (SSP) mbar_wait(&bars[0], it & 1);
      cplx a[PX];
#pragma unroll
      for (int s = 0; s < PX; ++s) {
        const int k = gq + s * TPJ;
        const bool lo = x_lo<N1, PX, TPJ>(s, gq);
        const int kk = lo ? k : N1 - k;
        cplx A = make_double2(0, 0), B = make_double2(0, 0);
        if (va && fa < cin) A = SSP ? st_in[(la * T::CIN + fa) * CF::N1H + kk] : __ldg(g.in + fa * g.fs_in + linea * g.kxp + x_koff(g, kk, g.kpcs_in));
        if (vb && fb < cin) B = SSP ? st_in[(lb * T::CIN + fb) * CF::N1H + kk] : __ldg(g.in + fb * g.fs_in + lineb * g.kxp + x_koff(g, kk, g.kpcs_in));
        if (kk == 0 || 2 * kk == N1) { A.y = 0.0; B.y = 0.0; }  // Hermitian part (C2R)
        // Y_k = A_k + i B_k (k <= N/2);  conj(A_{N-k}) + i conj(B_{N-k}) otherwise
        a[s] = lo ? make_double2(A.x - B.y, A.y + B.x) : make_double2(A.x + B.y, B.x - A.y);
      }
      x_fft<N1, PX, true, CF::TAB>(a, cx, gq, jbase, twx, job);
      x_jobsync<N1, PX>(job);  // the job's exchange reads are done before its slots become reals
#pragma unroll
      for (int s = 0; s < PX; ++s) {
        const int m = gq + s * TPJ;
        if (CF::ILV) {
          cx[jbase + m] = a[s];  // the pair's reals interleaved (fa, fb) at position m
        } else {
          real[ca * N1 + m] = a[s].x;
          real[cb * N1 + m] = a[s].y;
        }
      }
    }
    __syncthreads();
    // everyone has read the input stage (before its C2R): refill it with the next group's
    // spectra here, behind the barrier the voxel loop needs anyway (no barrier of its own)
    if (SSP && do_in && t == 0 && nxt < ngroups) {
      fence_proxy_async();
      x_issue_in<N1, KIND>(g, nxt, st_in, &bars[0]);
    }

    if (KIND == X_REAL_OUT) {
      for (int vv = t; vv < LPAR * N1; vv += CF::THREADS) {
        const int l2 = vv / N1, x = vv % N1;
        const long long ln = grp * LPAR + l2;
        if (ln >= g.nlines) continue;
        for (int f = 0; f < nf_real; ++f) g.real_out[(long long)f * g.nvox + ln * N1 + x] = real[x_slot<N1, CF::ILV>(l2 * CS + f, x)];
      }
      __syncthreads();
      continue;
    }
    if (KIND == X_REAL_IN) {  // real fields -> slots, pre-scaled by 1/(2N) like the voxel outputs
      for (int vv = t; vv < LPAR * N1; vv += CF::THREADS) {
        const int l2 = vv / N1, x = vv % N1;
        const long long ln = grp * LPAR + l2;
        for (int f = 0; f < CS; ++f)
          real[x_slot<N1, CF::ILV>(l2 * CS + f, x)] =
              (ln < g.nlines && f < nf_real) ? g.oscale * __ldg(g.real_in + (long long)g.real_map[f] * g.nvox + ln * N1 + x) : 0.0;
      }
    }

    // ------------------------------------------------------------ per-voxel operation
    if (SIN && STAGE_TAN) {
      if (CF::PH2) mbar_wait(&bars[1 + (it & 1)], (it >> 1) & 1);
      else mbar_wait(&bars[1], it & 1);
    }
    // neo-Hookean apply: the next voxel's tangent row is loaded while this voxel computes
    // TBATCH (neo-Hookean apply, at most 2 voxels per thread and group): the tangent rows of both of
    // the thread's voxels are loaded before either is contracted, so their L2 latencies overlap
    constexpr bool TBATCH = DBF_X_TBATCH && KIND == X_K_FIN_NH && S::NTAN == 0 && LPAR * N1 <= 2 * CF::THREADS;
    if constexpr (TBATCH) {
      double tq[2][10];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int vv = t + r * CF::THREADS;
        const long long v = (grp * LPAR) * N1 + vv;
        if (vv < LPAR * N1 && v < g.nvox)
#pragma unroll
          for (int k = 0; k < 10; ++k) tq[r][k] = __ldg(g.tan + (long long)k * g.nvox + v);
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int vv = t + r * CF::THREADS;
        const int l2 = vv / N1, x = vv % N1;
        const long long ln = grp * LPAR + l2;
        if (vv >= LPAR * N1 || ln >= g.nlines) continue;
        double G[CS], P[CS];
#pragma unroll
        for (int q = 0; q < CS / 2; ++q) {
          const cplx v2 = cx[(l2 * (CS / 2) + q) * N1 + x];
          G[2 * q] = v2.x;
          G[2 * q + 1] = (2 * q + 1 < T::CIN) ? v2.y : 0.0;
        }
        const long long v = ln * N1 + x;
        x_voxel<KIND>(g, v, G, P, red, nullptr, 0, S::PH ? (int)ph_cur[vv] : (int)__ldg(g.phase + v), xdot, g.e ? s_e : nullptr, tq[r]);
#pragma unroll
        for (int q = 0; q < CS / 2; ++q)
          if (2 * q < T::COUT) cx[(l2 * (CS / 2) + q) * N1 + x] = make_double2(P[2 * q], 2 * q + 1 < T::COUT ? P[2 * q + 1] : 0.0);
      }
    }
    constexpr bool TPIPE = DBF_X_TPIPE && KIND == X_K_FIN_NH && S::NTAN == 0;
    double tnext[TPIPE ? 10 : 1];
    if (TPIPE && t < LPAR * N1) {
      const long long v0 = (grp * LPAR) * N1 + t;
      if (v0 < g.nvox)
#pragma unroll
        for (int k = 0; k < 10; ++k) tnext[TPIPE ? k : 0] = __ldg(g.tan + (long long)k * g.nvox + v0);
    }
    for (int vv = t; KIND != X_REAL_IN && !TBATCH && vv < LPAR * N1; vv += CF::THREADS) {
      const int l2 = vv / N1, x = vv % N1;
      const long long ln = grp * LPAR + l2;
      if (ln >= g.nlines) continue;
      double tcur[TPIPE ? 10 : 1];
      if (TPIPE) {
#pragma unroll
        for (int k = 0; k < 10; ++k) tcur[TPIPE ? k : 0] = tnext[TPIPE ? k : 0];
        const int vn = vv + CF::THREADS;
        const long long v1 = (grp * LPAR) * N1 + vn;
        if (vn < LPAR * N1 && v1 < g.nvox)
#pragma unroll
          for (int k = 0; k < 10; ++k) tnext[TPIPE ? k : 0] = __ldg(g.tan + (long long)k * g.nvox + v1);
      }
      double G[CS], P[CS];
      if constexpr (CS % 2 == 0 && C == 9) {  // a line's pairs: one 16-byte load per field pair
                                             // (the 6-field kinds spilled with it: scalar)
#pragma unroll
        for (int q = 0; q < CS / 2; ++q) {
          const cplx v2 = cx[(l2 * (CS / 2) + q) * N1 + x];
          G[2 * q] = (2 * q < T::CIN && do_in) ? v2.x : 0.0;
          G[2 * q + 1] = (2 * q + 1 < T::CIN && do_in) ? v2.y : 0.0;
        }
      } else {
#pragma unroll
        for (int f = 0; f < CS; ++f) G[f] = (f < T::CIN && do_in) ? real[x_slot<N1, CF::ILV>(l2 * CS + f, x)] : 0.0;
      }
      const long long v = ln * N1 + x;
      const double* tp;
      long long ts;
      int ph;
      if (SIN && STAGE_TAN) {
        tp = (S::NTAN > 0) ? st_tan + vv : (g.tan ? g.tan + v : nullptr);
        ts = (S::NTAN > 0) ? (long long)LPAR * N1 : g.nvox;
        ph = S::PH ? (int)ph_cur[vv] : 0;
      } else {
        tp = g.tan ? g.tan + v : nullptr;
        ts = g.nvox;
        ph = (KIND == X_K_FIN_TAN || KIND == X_REAL_OUT) ? 0 : (int)__ldg(g.phase + v);
      }
      x_voxel<KIND>(g, v, G, P, red, tp, ts, ph, xdot, g.e ? s_e : nullptr, TPIPE ? tcur : nullptr);
      if constexpr (CS % 2 == 0 && C == 9) {
#pragma unroll
        for (int q = 0; q < CS / 2; ++q)
          if (2 * q < T::COUT) cx[(l2 * (CS / 2) + q) * N1 + x] = make_double2(P[2 * q], 2 * q + 1 < T::COUT ? P[2 * q + 1] : 0.0);
      } else {
#pragma unroll
        for (int f = 0; f < T::COUT; ++f) real[x_slot<N1, CF::ILV>(l2 * CS + f, x)] = P[f];
      }
    }
    __syncthreads();
    if (SIN && STAGE_TAN && !CF::PH2 && t == 0 && nxt < ngroups) {
      fence_proxy_async();
      x_issue_tan<N1, KIND>(g, nxt, st_tan, st_ph, &bars[1]);
    }

    // ------------------------------------------------------------ forward (R2C) of pairs
    {
      constexpr int COUT = T::COUT;
      cplx a[PX];
#pragma unroll
      for (int s = 0; s < PX; ++s) {
        const int m = gq + s * TPJ;
        const cplx v2 = CF::ILV ? cx[jbase + m] : make_double2(real[ca * N1 + m], real[cb * N1 + m]);
        a[s] = make_double2(fa < COUT ? v2.x : 0.0, fb < COUT ? v2.y : 0.0);
      }
      x_fft<N1, PX, false, CF::TAB>(a, cx, gq, jbase, twx, job);
      constexpr bool SHFL = (PX == 8 && TPJ <= 32);
      cplx zn[PX];
      if constexpr (SHFL) {
        x_partner<TPJ>(a, zn, gq);
      } else {
        x_jobsync<N1, PX>(job);
#pragma unroll
        for (int s = 0; s < PX; ++s) cx[x_idx<N1, PX>(jbase, gq + s * TPJ)] = a[s];
        x_jobsync<N1, PX>(job);
#pragma unroll
        for (int s = 0; s < PX; ++s) zn[s] = cx[x_idx<N1, PX>(jbase, (N1 - (gq + s * TPJ)) % N1)];
      }
      const bool sta = va && fa < cout_rt, stb = vb && fb < cout_rt;
      if (sta || stb) {
#pragma unroll
        for (int s = 0; s < PX; ++s) {
          const int k = gq + s * TPJ;
          if (!x_lo<N1, PX, TPJ>(s, gq)) continue;
          const cplx Z = a[s];
          const cplx Zn = zn[s];
          // 2x the spectra of the pair: with the voxel outputs scaled by 1/(2N) this is the
          // mean-normalised spectrum (R5)
          const cplx A = make_double2(Z.x + Zn.x, Z.y - Zn.y);
          const cplx B = make_double2(Z.y + Zn.y, Zn.x - Z.x);
          if (DCRED && s == 0 && gq == 0) {  // k = 0: the line sums of the pair (<sigma> / <dP>)
            const double dcs = 0.5 / g.oscale;  // undo the exact 1/(2N) of the voxel outputs
            if (sta) s_dc[DCRED ? la : 0][x_red_slot<KIND>(fa)] += dcs * A.x;
            if (stb && fb < COUT) s_dc[DCRED ? lb : 0][x_red_slot<KIND>(fb)] += dcs * B.x;
          }
          const long long ko = x_koff(g, k, g.kpcs_out);
          if (sta) g.out[fa * g.fs_out + linea * g.kxp + ko] = A;
          if (stb) g.out[fb * g.fs_out + lineb * g.kxp + ko] = B;
          if (g.kch > 0 && 2 * k == N1)  // pencil: the padding slot kch of the other kx chunks stays 0
            for (int c = 0; c + 1 < g.npy; ++c) {
              if (sta) g.out[c * g.kpcs_out + fa * g.fs_out + linea * g.kxp + g.kch] = make_double2(0.0, 0.0);
              if (stb) g.out[c * g.kpcs_out + fb * g.fs_out + lineb * g.kxp + g.kch] = make_double2(0.0, 0.0);
            }
        }
      }
      // no barrier here: a job's R2C and the next group's C2R touch only the job's own two slots
      // (their reals and FFT exchange), the voxel loop and the real-field kinds that read every
      // slot sit behind the unconditional barrier after the C2R
    }
  }

  // block reductions in a fixed order (deterministic); warp shuffles only for full warps
  // (odd line lengths give a partial last warp)
  constexpr int nw = (CF::THREADS + 31) / 32;
  constexpr bool FULLW = (CF::THREADS % 32) == 0;
  __shared__ double sred[FULLW ? nw : CF::THREADS];
  auto block_red = [&](double v, bool is_max) -> double {  // result valid in thread 0
    __syncthreads();
    if (FULLW) {
      v = is_max ? warp_max(v) : warp_sum(v);
      if ((t & 31) == 0) sred[t >> 5] = v;
    } else {
      sred[t] = v;
    }
    __syncthreads();
    double s = 0.0;
    if (t == 0)
      for (int w = 0; w < (FULLW ? nw : CF::THREADS); ++w) s = is_max ? fmax(s, sred[w]) : s + sred[w];
    return s;
  };
  DBF_PDL_EXIT();
  if (DCRED) {
    const double xs = block_red(xdot, false);
    if (t < T::NRED) {
      double s = 0.0;
      for (int q = 0; q < (DCRED ? LPAR : 1); ++q) s += s_dc[q][t];
      g.partials[(long long)blockIdx.x * g.nred + t] = s;
    }
    // slot 9: sum grad p : sigma (unscaled; FIN_NH summed the exactly 1/(2N)-scaled P)
    if (t == 0) g.partials[(long long)blockIdx.x * g.nred + 9] = (KIND == X_K_FIN_NH) ? xs / g.oscale : xs;
  } else if (T::NRED > 0) {
    // partials[block][nred] (sums; slot 9 of the const kinds is a max)
#pragma unroll
    for (int r = 0; r < T::NRED; ++r) {
      const double s = block_red(red[r], r == 9);
      if (t == 0) g.partials[(long long)blockIdx.x * g.nred + r] = s;
    }
  }
}


// ------------------------------------------------------------------------------------------------
// Warp-specialised pass_X (neo-Hookean apply kind, N1 = 256: one warp per field-pair FFT job).
// NFW = 5 FFT warps and NVW voxel warps per CTA, one line at a time, two slot buffers: while the
// voxel warps contract line i in buffer i&1, the FFT warps C2R line i+1 into the other buffer and
// then R2C line i once the voxel warps signal it — the hand-offs are mbarriers (FULL[b]: C2R done,
// DONE[b]: voxel op done), so neither role waits at a CTA barrier (the line-group design stalls
// ~20 % of its samples after its two __syncthreads per line).  The input spectra of the next line
// are bulk-copied into one stage buffer right after the FFT warps have read the current one (a
// named barrier of the FFT warps only); per-voxel tangent rows are L2-prefetched one line ahead.
// ------------------------------------------------------------------------------------------------
template <int N1>
struct XwsCfg {
  typedef XCfg<N1, X_K_FIN_NH> CF;
  static constexpr int NFW = CF::NP;  // pair jobs of a line (TPJ = 32: one warp each)
  static constexpr int NVW = DBF_XWS_NV;
  static constexpr int THREADS = (NFW + NVW) * 32;
  static constexpr int CS = CF::CS, N1H = CF::N1H;
  static constexpr size_t SLOTS = sizeof(double) * 2 * CS * N1;
  static constexpr size_t ST_IN = sizeof(cplx) * 9 * N1H;
  static constexpr size_t SMEM = SLOTS + ST_IN + sizeof(cplx) * N1 + 8 * sizeof(uint64_t);
  static_assert(CF::TPJ == 32 && CF::LPAR == 1 && CF::ILV && CF::TAB, "warp-specialised pass_X: N1 = 256 layout");
};

template <int N1>
#if DBF_XWS_MAXREG > 0
__global__ void __maxnreg__(DBF_XWS_MAXREG) x_pass_ws_kernel(XGeom g) {
#else
__global__ void __launch_bounds__(XwsCfg<N1>::THREADS, DBF_XWS_MINB) x_pass_ws_kernel(XGeom g) {
#endif
  if (g.stop0 && (*g.stop0 | *g.stop1)) return;  // PCG stopped: nothing to compute
  constexpr int KIND = X_K_FIN_NH;
  typedef XwsCfg<N1> W;
  typedef typename W::CF CF;
  constexpr int CS = W::CS, PX = CF::PX, TPJ = CF::TPJ, NFW = W::NFW, NVW = W::NVW;
  extern __shared__ __align__(16) double real[];
  unsigned char* sb = reinterpret_cast<unsigned char*>(real);
  cplx* st_in = reinterpret_cast<cplx*>(sb + W::SLOTS);
  cplx* stab = reinterpret_cast<cplx*>(sb + W::SLOTS + W::ST_IN);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + W::SLOTS + W::ST_IN + sizeof(cplx) * N1);
  uint64_t* bstage = bars;      // input stage filled
  uint64_t* bfull = bars + 1;   // [2] C2R of the buffer's line done (NFW arrivals)
  uint64_t* bdone = bars + 3;   // [2] voxel op of the buffer's line done (NVW arrivals)
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  __shared__ double s_dc[10];
  __shared__ double s_e[9];
  for (int i = t; i < N1 - 1; i += W::THREADS) stab[i] = __ldg(g.tw + N1 + i);
  if (t < 10) s_dc[t] = 0.0;
  if (g.e && t < 9) s_e[t] = g.e[t];
  const long long nmine = (g.nlines > (long long)blockIdx.x) ? (g.nlines - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (t == 0) {
    mbar_init(bstage, 1);
    mbar_init(&bfull[0], NFW);
    mbar_init(&bfull[1], NFW);
    mbar_init(&bdone[0], NVW);
    mbar_init(&bdone[1], NVW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0 && nmine > 0) x_issue_in<N1, KIND>(g, blockIdx.x, st_in, bstage);
  double xdot = 0.0;
  double red[10];
#pragma unroll
  for (int r = 0; r < 10; ++r) red[r] = 0.0;

  if (warp < NFW) {
    // ------------------------------------------------------------------ FFT warps
    const int job = warp, gq = lane;
    const int fa = 2 * job, fb = 2 * job + 1;
    const int jbase = (fa * N1) / 2;
    auto c2r = [&](long long i) {  // line i of this CTA -> buffer i & 1
      const long long line = blockIdx.x + i * gridDim.x;
      cplx* cx = reinterpret_cast<cplx*>(real + (i & 1) * CS * N1);
      mbar_wait(bstage, (uint32_t)(i & 1));
      cplx a[PX];
#pragma unroll
      for (int s = 0; s < PX; ++s) {
        const int k = gq + s * TPJ;
        const bool lo = x_lo<N1, PX, TPJ>(s, gq);
        const int kk = lo ? k : N1 - k;
        cplx A = st_in[fa * W::N1H + kk];
        cplx B = (fb < 9) ? st_in[fb * W::N1H + kk] : make_double2(0, 0);
        if (kk == 0 || 2 * kk == N1) { A.y = 0.0; B.y = 0.0; }
        a[s] = lo ? make_double2(A.x - B.y, A.y + B.x) : make_double2(A.x + B.y, B.x - A.y);
      }
      // every FFT warp has its inputs in registers: the stage takes the next line's spectra now
      asm volatile("bar.sync 1, %0;" ::"n"(NFW * 32) : "memory");
      if (t == 0 && i + 1 < nmine) {
        fence_proxy_async();
        x_issue_in<N1, KIND>(g, line + gridDim.x, st_in, bstage);
      }
      x_fft<N1, PX, true, true>(a, cx, gq, jbase, stab, job);
      __syncwarp();
#pragma unroll
      for (int s = 0; s < PX; ++s) cx[jbase + gq + s * TPJ] = a[s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bfull[i & 1]);
    };
    auto r2c = [&](long long i) {
      const long long line = blockIdx.x + i * gridDim.x;
      cplx* cx = reinterpret_cast<cplx*>(real + (i & 1) * CS * N1);
      mbar_wait(&bdone[i & 1], (uint32_t)((i >> 1) & 1));
      cplx a[PX];
#pragma unroll
      for (int s = 0; s < PX; ++s) {
        const cplx v2 = cx[jbase + gq + s * TPJ];
        a[s] = make_double2(v2.x, fb < 9 ? v2.y : 0.0);
      }
      x_fft<N1, PX, false, true>(a, cx, gq, jbase, stab, job);
      cplx zn[PX];
      x_partner<TPJ>(a, zn, gq);
#pragma unroll
      for (int s = 0; s < PX; ++s) {
        const int k = gq + s * TPJ;
        if (!x_lo<N1, PX, TPJ>(s, gq)) continue;
        const cplx Z = a[s], Zn = zn[s];
        const cplx A = make_double2(Z.x + Zn.x, Z.y - Zn.y);
        const cplx B = make_double2(Z.y + Zn.y, Zn.x - Z.x);
        if (s == 0 && gq == 0) {  // k = 0: the line sums of the pair (<dP>)
          const double dcs = 0.5 / g.oscale;
          s_dc[fa] += dcs * A.x;
          if (fb < 9) s_dc[fb] += dcs * B.x;
        }
        const long long ko = x_koff(g, k, g.kpcs_out);
        g.out[fa * g.fs_out + line * g.kxp + ko] = A;
        if (fb < 9) g.out[fb * g.fs_out + line * g.kxp + ko] = B;
        if (g.kch > 0 && 2 * k == N1)
          for (int c = 0; c + 1 < g.npy; ++c) {
            g.out[c * g.kpcs_out + fa * g.fs_out + line * g.kxp + g.kch] = make_double2(0.0, 0.0);
            if (fb < 9) g.out[c * g.kpcs_out + fb * g.fs_out + line * g.kxp + g.kch] = make_double2(0.0, 0.0);
          }
      }
      __syncwarp();  // the job's slots are read (exchange + untangle) before the next C2R writes them
    };
    if (nmine > 0) c2r(0);
    for (long long i = 0; i < nmine; ++i) {
      if (i + 1 < nmine) c2r(i + 1);
      r2c(i);
    }
  } else {
    // ------------------------------------------------------------------ voxel warps
    const int vt = t - NFW * 32;
    for (long long i = 0; i < nmine; ++i) {
      const long long line = blockIdx.x + i * gridDim.x;
      if (vt == 0 && i + 1 < nmine) {  // the next line's tangent rows and phase ids -> L2
        const long long v1 = (line + gridDim.x) * N1;
#pragma unroll 1
        for (int k = 0; k < 10; ++k) prefetch_l2(g.tan + (long long)k * g.nvox + v1, sizeof(double) * N1);
        prefetch_l2(g.phase + v1, sizeof(uint16_t) * N1);
      }
      const cplx* cx = reinterpret_cast<const cplx*>(real + (i & 1) * CS * N1);
      double* rw = real + (i & 1) * CS * N1;
      mbar_wait(&bfull[i & 1], (uint32_t)((i >> 1) & 1));
      for (int x = vt; x < N1; x += NVW * 32) {
        double G[CS], P[CS];
#pragma unroll
        for (int q = 0; q < CS / 2; ++q) {
          const cplx v2 = cx[q * N1 + x];
          G[2 * q] = v2.x;
          G[2 * q + 1] = (2 * q + 1 < 9) ? v2.y : 0.0;
        }
        const long long v = line * N1 + x;
        const int ph = (int)__ldg(g.phase + v);
        x_voxel<KIND>(g, v, G, P, red, g.tan + v, g.nvox, ph, xdot, g.e ? s_e : nullptr);
#pragma unroll
        for (int q = 0; q < CS / 2; ++q)
          reinterpret_cast<cplx*>(rw)[q * N1 + x] = make_double2(P[2 * q], 2 * q + 1 < 9 ? P[2 * q + 1] : 0.0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bdone[i & 1]);
    }
  }
  // block reductions in a fixed order (deterministic)
  __shared__ double sred[W::THREADS / 32];
  __syncthreads();
  double v = warp_sum(xdot);
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  if (t < 9) {
    g.partials[(long long)blockIdx.x * g.nred + t] = s_dc[t];
  } else if (t == 9) {
    double s = 0.0;
    for (int w = 0; w < W::THREADS / 32; ++w) s += sred[w];
    g.partials[(long long)blockIdx.x * g.nred + 9] = s / g.oscale;  // FIN_NH summed the 1/(2N)-scaled P
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
      const double mu = __ldg(g.ptable + 36 * ph), lam = __ldg(g.ptable + 36 * ph + 3);
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

// per-voxel tangent as a full 3x3x3x3 array (DBFFT_FIELD_TANGENT): out[(9 a + b) nv + (v - v0)],
// a = 3i + j, b = 3k + l, for voxels v0 <= v < v0 + nv.  MODE 0: stored 45-entry upper triangle
// (finite); 1: compact neo-Hookean (F^-1, c1); 2: compact J2 (theta, thetabar, n); 3: linear phase
// stiffness (Voigt 6x6 of tensor components, ptable)
template <int MODE>
__global__ void __launch_bounds__(256) k_tangent81(XGeom g, long long v0, long long nv, double* __restrict__ out) {
  const int vo[9] = {0, 5, 4, 5, 1, 3, 4, 3, 2};  // row-major entry -> Voigt index
  for (long long e = (long long)blockIdx.x * 256 + threadIdx.x; e < nv; e += (long long)gridDim.x * 256) {
    const long long v = v0 + e;
    double* o = out + e;
    if (MODE == 0 || MODE == 1) {
      double K45[45];
      if (MODE == 0) {
#pragma unroll
        for (int k = 0; k < 45; ++k) K45[k] = g.tan[(long long)k * g.nvox + v];
      } else {
        double Fi[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) Fi[k] = g.tan[(long long)k * g.nvox + v];
        const int ph = g.phase[v];
        const double mu = g.ptable[36 * ph], lam = g.ptable[36 * ph + 3];
        nh_tangent45(Fi, g.tan[9 * g.nvox + v], mu, lam, K45);
      }
#pragma unroll
      for (int a = 0; a < 9; ++a)
#pragma unroll
        for (int b = 0; b < 9; ++b) o[(long long)(9 * a + b) * nv] = K45[sym9(a, b)];
    } else if (MODE == 2) {
      // C_alg = kappa 1 x 1 + 2 mu theta I_dev - 2 mu thetabar n x n   (R16, j2_update)
      double tc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) tc[k] = g.tan[(long long)k * g.nvox + v];
      double kappa, mu;
      j2_moduli(g.ptable + 36 * g.phase[v], &kappa, &mu);
#pragma unroll
      for (int a = 0; a < 9; ++a)
#pragma unroll
        for (int b = 0; b < 9; ++b) {
          const int i = a / 3, j = a % 3, k = b / 3, l = b % 3;
          const double idev = 0.5 * ((i == k && j == l) + (i == l && j == k)) - ((i == j && k == l) ? 1.0 / 3.0 : 0.0);
          o[(long long)(9 * a + b) * nv] = ((i == j && k == l) ? kappa : 0.0) + 2.0 * mu * tc[0] * idev -
                                          2.0 * mu * tc[1] * tc[2 + vo[a]] * tc[2 + vo[b]];
        }
    } else {
      const double* C = g.ptable + 36 * g.phase[v];
#pragma unroll
      for (int a = 0; a < 9; ++a)
#pragma unroll
        for (int b = 0; b < 9; ++b) o[(long long)(9 * a + b) * nv] = C[6 * vo[a] + vo[b]];
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Column passes, TMA pipeline.  Persistent, one CTA per SM:
// warp 8 (one elected lane) streams 32 KB tiles — KC = 2048/N kx-columns x N positions of ONE
// field, 128-byte rows — into an R-slot shared-memory ring with cp.async.bulk.tensor
// (mbarrier complete_tx); warps 0-7 FFT the columns (a column's N/8 threads share one warp, so
// every exchange is warp-local), apply the pass's pre/post weights, and write each finished
// output tile into a staging buffer that one thread sends back with a TMA store.  A pass is a
// static "program": the order in which input fields are loaded and the order of its terms, chosen
// so that ring slots are released in load order (FIFO) — see c_prog.
// Main tiles cover kx in [0, n1/2) in KC-column blocks of one outer index; tail tiles carry the
// Nyquist column kx = n1/2 of KC consecutive outer indices (no compute is spent on padding).
// ------------------------------------------------------------------------------------------------
struct TProg {
  int nl;                 // loads per tile
  signed char ld[12];     // load i: input field (0..15) or dot-vector field (16 + f)
  int nt;                 // terms
  signed char j[10];      // ColOp term index
  signed char la[10], lb[10], ldot[10];  // load indices of the term's inputs / dot vector (-1: none)
  signed char rel[10];    // loads released (cumulative, FIFO) once the term is done
  signed char acc[10];    // register accumulator of a two-term output
};

#define DBF_PLAIN3 {3, {0, 1, 2}, 3, {0, 1, 2}, {0, 1, 2}, {-1, -1, -1}, {-1, -1, -1}, {1, 2, 3}, {0, 0, 0}}
#define DBF_PLAIN6                                                                                               \
  {6, {0, 1, 2, 3, 4, 5}, 6, {0, 1, 2, 3, 4, 5}, {0, 1, 2, 3, 4, 5}, {-1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1}, \
   {1, 2, 3, 4, 5, 6}, {0, 0, 0, 0, 0, 0}}
// index: 2*kind + dot (one table: host copy for the liveness check, constant-bank copy for the kernel)
#define DBF_COL_PROGS \
    /* COL_I1S: loads u0, u2, u1; terms 0, 2, 3{0,2}, 1, 4{1,2} */ \
    {3, {0, 2, 1}, 5, {0, 2, 3, 1, 4}, {0, 1, 0, 2, 2}, {-1, -1, 1, -1, 1}, {-1, -1, -1, -1, -1}, {0, 0, 1, 1, 3}, {0, 0, 0, 0, 0}}, \
    {0}, \
    /* COL_I1F: u_i then i xi_z u_i from the same load */ \
    {3, {0, 1, 2}, 6, {0, 3, 1, 4, 2, 5}, {0, 0, 1, 1, 2, 2}, {-1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1}, {0, 1, 1, 2, 2, 3}, {0, 0, 0, 0, 0, 0}}, \
    {0}, \
    /* COL_I2S: loads 0,1,2,4,3; terms 0, 1, 5{0,1}, 2, 3{4}, 4{3} */ \
    {5, {0, 1, 2, 4, 3}, 6, {0, 1, 5, 2, 3, 4}, {0, 1, 0, 2, 3, 4}, {-1, -1, 1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1}, {0, 0, 2, 3, 4, 5}, {0, 0, 0, 0, 0, 0}}, \
    {0}, \
    /* COL_I2F: loads u0, G0z, u1, G1z, u2, G2z */ \
    {6, {0, 3, 1, 4, 2, 5}, 9, {0, 1, 2, 3, 4, 5, 6, 7, 8}, {0, 0, 1, 2, 2, 3, 4, 4, 5}, {-1, -1, -1, -1, -1, -1, -1, -1, -1}, \
     {-1, -1, -1, -1, -1, -1, -1, -1, -1}, {0, 1, 2, 2, 3, 4, 4, 5, 6}, {0, 0, 0, 0, 0, 0, 0, 0, 0}}, \
    {0}, \
    /* COL_F2S */ \
    {6, {0, 1, 2, 3, 4, 5}, 6, {0, 1, 2, 3, 4, 5}, {0, 1, 2, 3, 4, 5}, {-1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1}, {1, 2, 3, 4, 5, 6}, {0, 0, 0, 0, 0, 0}}, \
    {0}, \
    /* COL_F2F: term j reads field ld[j] */ \
    {9, {0, 1, 3, 4, 6, 7, 2, 5, 8}, 9, {0, 1, 2, 3, 4, 5, 6, 7, 8}, {0, 1, 2, 3, 4, 5, 6, 7, 8}, {-1, -1, -1, -1, -1, -1, -1, -1, -1}, \
     {-1, -1, -1, -1, -1, -1, -1, -1, -1}, {1, 2, 3, 4, 5, 6, 7, 8, 9}, {0, 0, 0, 0, 0, 0, 0, 0, 0}}, \
    {0}, \
    /* COL_F3S: loads 0,5,1,4,3,2; terms j0{0,5} j2{5,1} j1{4} j3{3} j4{4,3} j5{2} */ \
    {6, {0, 5, 1, 4, 3, 2}, 6, {0, 2, 1, 3, 4, 5}, {0, 1, 3, 4, 3, 5}, {1, 2, -1, -1, 4, -1}, {-1, -1, -1, -1, -1, -1}, {1, 3, 3, 3, 5, 6}, {0, 1, 0, 1, 0, 0}}, \
    /* COL_F3S + <p, f>: p_o loaded right before the term that stores output o */ \
    {9, {0, 5, 1, 4, 16, 3, 17, 2, 18}, 6, {0, 2, 1, 3, 4, 5}, {0, 1, 3, 5, 3, 7}, {1, 2, -1, -1, 5, -1}, {-1, -1, 4, 6, -1, 8}, {1, 3, 3, 3, 7, 9}, {0, 1, 0, 1, 0, 0}}, \
    /* COL_F3F */ \
    {6, {0, 3, 1, 4, 2, 5}, 6, {0, 1, 2, 3, 4, 5}, {0, 1, 2, 3, 4, 5}, {-1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1}, {1, 2, 3, 4, 5, 6}, {0, 0, 0, 0, 0, 0}}, \
    {9, {0, 3, 16, 1, 4, 17, 2, 5, 18}, 6, {0, 1, 2, 3, 4, 5}, {0, 1, 3, 4, 6, 7}, {-1, -1, -1, -1, -1, -1}, {-1, 2, -1, 5, -1, 8}, {1, 3, 4, 6, 7, 9}, {0, 0, 0, 0, 0, 0}}, \
    /* COL_ZI3, COL_YI3 */ \
    DBF_PLAIN3, {0}, DBF_PLAIN3, {0}, \
    /* COL_ZI6, COL_YI6, COL_ZF3, COL_YF3, COL_ZF6, COL_YF6 */ \
    DBF_PLAIN6, {0}, DBF_PLAIN6, {0}, DBF_PLAIN3, {0}, DBF_PLAIN3, {0}, DBF_PLAIN6, {0}, DBF_PLAIN6, {0},

__device__ __constant__ TProg c_prog[2 * COL_NKINDS] = {DBF_COL_PROGS};
static const TProg kColProgHost[2 * COL_NKINDS] = {DBF_COL_PROGS};

struct ColTiles {
  int n_outer;   // outer indices
  int nkb;       // main kx blocks per outer (n1/2 / KC)
  int n_main;    // n_outer * nkb
  int n_tiles;   // n_main + ceil(n_outer / KC)
  int tail_cols; // outer indices per tail box: min(KC, n_outer)
};

template <int N>
struct TmaCfg {
  static constexpr int KC = 2048 / N;          // columns per tile (32 KB of complex128)
  static constexpr int TPC = N / 8;            // threads per column (8 points each)
  static constexpr int CONS = 256;             // consumer threads (8 warps)
  static constexpr int THREADS = CONS + 32;    // + producer warp
  static constexpr int TILE = 32768;           // bytes per ring slot / staging buffer
  static constexpr int SW = KC < 8 ? KC : 8;   // sub-tile width in columns (TMA box rows of 16 SW bytes)
  // twiddles from the stage-ordered table in shared memory (B200 256^3 finite apply_K 2.71 -> 2.43
  // ms); at N = 512 the product-of-table-entries twiddles stayed faster for I1 / I2 (2.55 / 6.15 ms
  // vs 2.78 / 7.15 ms with the table)
  static constexpr bool TAB = N <= 256 || DBF_COL_TAB512;
};
// per pass: the small-strain F2 (a plain 6 -> 6 transform, the fastest pass at 5.1 TB/s) ran
// slower with the table (256^3: 0.318 -> 0.343 ms) and keeps the products
template <int N, int KIND>
struct ColTab {
  static constexpr bool value = TmaCfg<N>::TAB && KIND != COL_F2S;
  // xi at the thread's positions hoisted into registers (not where the 168-register cap of the
  // 288-thread CTA would spill: the two-accumulator small-strain F3 at N = 512)
  static constexpr bool HOIST = !(KIND == COL_F3S && N == 512);
};

// cplx offset of (pos, column c) inside a main tile: KC/8 sub-tiles of [N][8], 128B swizzle
template <int N>
DBF_DEV int tma_moff(int pos, int c) {
  constexpr int SW = TmaCfg<N>::SW;  // columns per sub-tile row: 8 (128B swizzle) or 4 (64B)
  if (SW == 8) return (c >> 3) * (N * 8) + pos * 8 + ((c & 7) ^ (pos & 7));
  return (c / SW) * (N * SW) + pos * SW + ((c % SW) ^ ((pos >> 1) & 3));
}
// exchange sync of one column's N/8 threads: the warp, or a named barrier when a column spans
// two warps (N = 512: 64 threads, ids 2..5)
struct SyncCol {
  int id, nthreads;
  DBF_DEV void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }
};
// tail tile: [KC][N] unswizzled
template <int N>
DBF_DEV int tma_toff(int pos, int c) { return c * N + pos; }
// FFT exchange index inside a staging tile: column c keeps to its own 16-byte slots of the tile
// layout (so a warp never touches another column's), positions XOR-swizzled as in IdxSwz — the
// slot's bank group depends on pos & 7 only, in both layouts, so scatter and gather stay
// conflict-free
template <int N>
struct IdxTile {
  int cb, sh, sw, sm;  // per tile and column: base, log2 row pitch, swizzle term and mask (tail tiles: 0)
  DBF_DEV IdxTile(int c, bool tail) {
    constexpr int SW = TmaCfg<N>::SW;
    cb = tail ? c * N : (c / SW) * (N * SW);
    sh = tail ? 0 : (SW == 8 ? 3 : 2);
    sw = tail ? 0 : c % SW;
    sm = tail ? 0 : SW - 1;
  }
  DBF_DEV int operator()(int pos) const {
    const int p = pos ^ ((pos >> 3) & 7);
    return cb + (p << sh) + (sw ^ ((TmaCfg<N>::SW == 8 ? p : (p >> 1)) & sm));
  }
};

DBF_DEV void tma_load5(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(smem_u32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)) : "memory");
}
DBF_DEV void tma_store5(const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4, const void* src) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
               ::"l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(src)) : "memory");
}
DBF_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int K>
DBF_DEV void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K) : "memory"); }
DBF_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
DBF_DEV void cons_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

struct TmaMaps {
  CUtensorMap in_m, in_t, out_m, out_t, dot_m, dot_t;
};

template <int N, int KIND, bool DOT, int R, bool UPD = false>
__global__ void __launch_bounds__(TmaCfg<N>::THREADS, 1) col_tma_kernel(const __grid_constant__ TmaMaps maps, ColGeom g, ColTiles tl) {
  if (!DBF_PDL_LATE) DBF_PDL_ENTRY_BIG();
  typedef ColOp<KIND> Op;
  typedef TmaCfg<N> CF;
  constexpr bool TAB = ColTab<N, KIND>::value && (!UPD || DBF_UPD_TAB);
  if (!DBF_PDL_LATE && g.cg_stop0 && (*g.cg_stop0 | *g.cg_stop1)) return;  // PCG stopped (UPD: r stays as it is)
  constexpr int KC = CF::KC, TPC = CF::TPC;
  constexpr int S = UPD ? 3 : 2;  // staging buffers (UPD: r_0, r_1 of a tile stay readable until r_2)
  extern __shared__ __align__(1024) unsigned char tsm[];
  // 1024-byte alignment of the ring (128B swizzle atoms)
  // (offset arithmetic on the shared array keeps the shared address space: LDS/STS, not LD/ST)
  unsigned char* base = tsm + ((1024u - (smem_u32(tsm) & 1023u)) & 1023u);
  // XIN: the exchanges of a term run inside the staging buffer its output goes to (free since the
  // barrier of the previous output: the store two outputs back has been read), so there is no
  // separate exchange buffer; the fused update reads earlier staging buffers and keeps one
  constexpr bool XIN = DBF_COL_XINPLACE && !UPD;
  cplx* ring = reinterpret_cast<cplx*>(base);
  cplx* stg = reinterpret_cast<cplx*>(base + R * CF::TILE);
  cplx* xb = reinterpret_cast<cplx*>(base + (R + S) * CF::TILE);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (R + S + (XIN ? 0 : 1)) * CF::TILE);
  uint64_t* empty = full + R;
  cplx* stab = reinterpret_cast<cplx*>(empty + R);  // stage-ordered twiddles (N - 1), copied once
  const TProg& pg = c_prog[2 * KIND + (DOT ? 1 : 0)];
  const int t = threadIdx.x;
  const int warp = t >> 5;
  if (t == 0) {
    for (int i = 0; i < R; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CF::CONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TAB)
    for (int i = t; i < N - 1; i += CF::THREADS) stab[i] = __ldg(g.tw + N + i);
  __syncthreads();
  if (DBF_PDL_LATE) {  // the prologue above touched only constant tables: wait for the predecessor here
    DBF_PDL_ENTRY_BIG();
    if (g.cg_stop0 && (*g.cg_stop0 | *g.cg_stop1)) return;
  }
  const int nl = pg.nl;

  if (warp == CF::CONS / 32) {
    // ------------------------------------------------------------------ producer
    if ((t & 31) == 0) {
      uint32_t seq = 0;
      for (int tile = blockIdx.x; tile < tl.n_tiles; tile += gridDim.x) {
        const bool tail = tile >= tl.n_main;
        const int outer = tail ? (tile - tl.n_main) * KC : tile / tl.nkb;
        const int kb = tail ? 0 : tile % tl.nkb;
        for (int i = 0; i < nl; ++i, ++seq) {
          const int slot = seq % R;
          const uint32_t round = seq / R;
          if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
          const int ld = pg.ld[i];
          const bool isdot = ld >= 16;
          const int f = ld & 15;
          mbar_expect_tx(&full[slot], tail ? 16u * N * tl.tail_cols : (uint32_t)CF::TILE);
          cplx* dst = ring + slot * (CF::TILE / 16);
          if (tail) {
            tma_load5(dst, isdot ? &maps.dot_t : &maps.in_t, 2 * (g.n1h - 1), 0, 0, outer, f, &full[slot]);
          } else {
#pragma unroll
            for (int sb = 0; sb < KC / CF::SW; ++sb)
              tma_load5(dst + sb * N * CF::SW, isdot ? &maps.dot_m : &maps.in_m, 2 * (kb * KC + sb * CF::SW), 0, 0, outer, f,
                        &full[slot]);
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int c = t / TPC;   // column of the tile
  const int gq = t % TPC;  // position group
  const int lane = t & 31;
  cplx* xcol = xb + c * N;  // this column's FFT exchange buffer
  double xpos[ColTab<N, KIND>::HOIST ? 8 : 1];  // xi along the FFT axis at this thread's positions (every tile)
  if (ColTab<N, KIND>::HOIST)
#pragma unroll
    for (int s = 0; s < 8; ++s) xpos[ColTab<N, KIND>::HOIST ? s : 0] = __ldg(g.fpos + gq + s * TPC);
  double acc_rz = 0.0, acc_rr = 0.0;  // UPD: partial <r, M r>, <r, r>
  const double alpha = UPD ? *g.cg_alpha : 0.0;
  __shared__ double sprec[UPD ? 36 : 1];  // M's coefficients (device memory -> shared, once)
  if (UPD) {
    for (int i = t; i < 36; i += CF::CONS) sprec[i] = g.precq[i];
    cons_sync();
  }
  uint32_t nout = 0;        // output tiles written (staging rotation)
  uint32_t it = 0;
  for (int tile = blockIdx.x; tile < tl.n_tiles; tile += gridDim.x, ++it) {
    const bool tail = tile >= tl.n_main;
    ColAt at;
    at.g = &g;
    const int outer = tail ? (tile - tl.n_main) * KC + c : tile / tl.nkb;
    const bool valid = outer < tl.n_outer;
    at.set_col(valid ? outer : 0, tail ? g.n1h - 1 : (tile % tl.nkb) * KC + c);
    const double wdot = (at.kx + g.kx0 == 0 || 2 * (at.kx + g.kx0) == g.n1) ? 1.0 : 2.0;
    const uint32_t sbase = it * nl;
    int released = 0;
    constexpr int NACC = (KIND == COL_F3S) ? 2 : 1;  // pending two-term outputs
    cplx acc0[8], acc1[NACC > 1 ? 8 : 1];
#pragma unroll 1
    for (int k = 0; k < pg.nt; ++k) {
      const int j = pg.j[k];
      const TermInfo ti = Op::term(j);
      const int la = pg.la[k], lb = pg.lb[k];
      const uint32_t qa = sbase + la;
      mbar_wait(&full[qa % R], (qa / R) & 1);
      const cplx* sa = ring + (qa % R) * (CF::TILE / 16);
      const cplx* sbp = sa;
      if (lb >= 0) {
        const uint32_t qb = sbase + lb;
        mbar_wait(&full[qb % R], (qb / R) & 1);
        sbp = ring + (qb % R) * (CF::TILE / 16);
      }
      cplx a[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        at.pos = gq + s * TPC;
        at.xp = ColTab<N, KIND>::HOIST ? xpos[ColTab<N, KIND>::HOIST ? s : 0] : __ldg(g.fpos + at.pos);
        const int o = tail ? tma_toff<N>(at.pos, c) : tma_moff<N>(at.pos, c);
        const cplx v0 = sa[o];
        const cplx v1 = (lb >= 0) ? sbp[o] : v0;
        a[s] = Op::pre(at, j, v0, v1);
      }
      cplx* so = stg + (nout % S) * (CF::TILE / 16);
      if constexpr (XIN) {
        const IdxTile<N> ix(c, tail);
        if constexpr (TPC <= 32) {
          fft_cta<N, Op::INV, IdxTile<N>, SyncWarp, TAB>(a, so, gq, ix, TAB ? stab : g.tw, SyncWarp{});
          SyncWarp{}();  // the column's last gathers are done before its outputs overwrite the slots
        } else {
          fft_cta<N, Op::INV, IdxTile<N>, SyncCol, TAB>(a, so, gq, ix, TAB ? stab : g.tw, SyncCol{2 + c, TPC});
          SyncCol{2 + c, TPC}();
        }
      } else if constexpr (TPC <= 32) fft_cta<N, Op::INV, IdxSwz, SyncWarp, TAB>(a, xcol, gq, IdxSwz{0}, TAB ? stab : g.tw, SyncWarp{});
      else fft_cta<N, Op::INV, IdxSwz, SyncCol, TAB>(a, xcol, gq, IdxSwz{0}, TAB ? stab : g.tw, SyncCol{2 + c, TPC});
      const int ai = pg.acc[k];
      const int ld = pg.ldot[k];
      const cplx* sd = nullptr;
      if (DOT && ti.last && ld >= 0) {
        const uint32_t qd = sbase + ld;
        mbar_wait(&full[qd % R], (qd / R) & 1);
        sd = ring + (qd % R) * (CF::TILE / 16);
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        at.pos = gq + s * TPC;
        at.xp = ColTab<N, KIND>::HOIST ? xpos[ColTab<N, KIND>::HOIST ? s : 0] : __ldg(g.fpos + at.pos);
        cplx v = cmul(Op::post(at, j), a[s]);
        if (ColTwo<KIND>::value && !ti.first) v = cadd(v, (NACC > 1 && ai) ? acc1[NACC > 1 ? s : 0] : acc0[s]);
        if (ColTwo<KIND>::value && !ti.last) {
          if (NACC > 1 && ai) acc1[NACC > 1 ? s : 0] = v;
          else acc0[s] = v;
        } else {
          const int o = tail ? tma_toff<N>(at.pos, c) : tma_moff<N>(at.pos, c);
          if (UPD) {  // r_o -= alpha q_o (the F3 output is q = K p); the tile's r is staged in sd
            const cplx rr = sd[o];
            v = make_double2(fma(-alpha, v.x, rr.x), fma(-alpha, v.y, rr.y));
            if (ti.o == 2 && valid) {  // r_0, r_1 are in the previous two staging buffers
              const cplx r3[3] = {stg[((nout + S - 2) % S) * (CF::TILE / 16) + o], stg[((nout + S - 1) % S) * (CF::TILE / 16) + o], v};
              const double xz = __ldg(g.fq.xz + at.pos);
              cplx z3[3] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
              if (!(at.xxk == 0.0 && at.xyo == 0.0 && xz == 0.0)) prec_apply(sprec, at.xxk, at.xyo, xz, r3, z3);
#pragma unroll
              for (int q = 0; q < 3; ++q) {
                acc_rz += wdot * (r3[q].x * z3[q].x + r3[q].y * z3[q].y);
                acc_rr += wdot * (r3[q].x * r3[q].x + r3[q].y * r3[q].y);
              }
            }
          }
          so[o] = v;
        }
      }
      // release the ring slots this term finished (FIFO): all lanes of the warp are done
      const int rel = pg.rel[k];
      __syncwarp();
      if (lane == 0)
        for (int i = released; i < rel; ++i) mbar_arrive(&empty[(sbase + i) % R]);
      released = rel;
      if (ti.last) {
        // every consumer wrote its part of the output tile; the store S-1 outputs ago is done
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (t == 0) bulk_wait_read<S - 2>();  // staging[(nout + 1) % S] is free for the next output
        cons_sync();
        if (t == 0) {
          if (tail) tma_store5(&maps.out_t, 2 * (g.n1h - 1), 0, 0, (tile - tl.n_main) * KC, ti.o, so);
          else tma_store5(&maps.out_m, 2 * ((tile % tl.nkb) * KC), 0, 0, tile / tl.nkb, ti.o, so);
          if (!tail && KC > CF::SW) {
#pragma unroll
            for (int sb = 1; sb < KC / CF::SW; ++sb)
              tma_store5(&maps.out_m, 2 * ((tile % tl.nkb) * KC + sb * CF::SW), 0, 0, tile / tl.nkb, ti.o, so + sb * N * CF::SW);
          }
          bulk_commit();
        }
        ++nout;
      }
    }
  }
  DBF_PDL_EXIT();
  if (t == 0) bulk_wait_all();
  if (UPD) {
    __shared__ double red2[8][2];
    acc_rz = warp_sum(acc_rz);
    acc_rr = warp_sum(acc_rr);
    if (lane == 0) {
      red2[warp][0] = acc_rz;
      red2[warp][1] = acc_rr;
    }
    cons_sync();
    if (t < 2) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red2[w][t];
      g.partials[2 * blockIdx.x + t] = s;
    }
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------------------------
template <int N>
static int col_cols() { return ColCfg<N>::COLS; }

int col_grid(int N, long long ncols) {
  int cols;
  switch (N) {
    case 8: cols = col_cols<8>(); break;
    case 16: cols = col_cols<16>(); break;
    case 32: cols = col_cols<32>(); break;
    case 64: cols = col_cols<64>(); break;
    case 128: cols = col_cols<128>(); break;
    case 256: cols = col_cols<256>(); break;
    case 15: cols = col_cols<15>(); break;
    case 21: cols = col_cols<21>(); break;
    case 27: cols = col_cols<27>(); break;
    case 63: cols = col_cols<63>(); break;
    default: cols = col_cols<512>(); break;
  }
  return (int)((ncols + cols - 1) / cols);
}

template <int N, int KIND>
static cudaError_t launch_col_k(const ColGeom& g, cudaStream_t s) {
  constexpr int COLS = ColCfg<N>::COLS;
  constexpr size_t smem = sizeof(cplx) * N * COLS * (ColTwo<KIND>::value ? 2 : 1);
  static DevOnce once;
  cudaError_t e = dev_once(once, [](int&) {
    return cudaFuncSetAttribute(col_pass_kernel<N, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  return launch_k(col_pass_kernel<N, KIND>, col_grid(N, g.ncols), ColCfg<N>::THREADS, smem, s, g);
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
    case COL_ZI6: return launch_col_k<N, COL_ZI6>(g, s);
    case COL_YI6: return launch_col_k<N, COL_YI6>(g, s);
    case COL_ZF3: return launch_col_k<N, COL_ZF3>(g, s);
    case COL_YF3: return launch_col_k<N, COL_YF3>(g, s);
    case COL_ZF6: return launch_col_k<N, COL_ZF6>(g, s);
    case COL_YF6: return launch_col_k<N, COL_YF6>(g, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---- TMA column passes: tensor maps + dispatch ------------------------------------------------
#ifndef DBF_COL_TMA
#define DBF_COL_TMA 1
#endif
#ifndef DBF_TMA_PROMO
#define DBF_TMA_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
#ifndef DBF_RING2_SMALL
#define DBF_RING2_SMALL 0  // 2-deep ring for the small-strain I1 / F2 too (slower: 256^3 I1S 0.319 -> 0.381 ms)
#endif
#ifndef DBF_RING2_FIN
#define DBF_RING2_FIN 1  // 2-deep ring for the finite-strain I1 (F2F went back to 3 with the 128-byte
                         // pitch: 256^3 0.447 -> 0.433 ms; I1F 0.257 with 2 vs 0.271 with 3)
#endif
#ifndef DBF_REG512_MASK
#define DBF_REG512_MASK 0  // bit k: column kind k at N = 512 takes the register-pipelined kernel
#endif
#ifndef DBF_COL_R
#define DBF_COL_R 3
#endif

static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// fields of the pass's input / output buffers (tensor-map bounds)
static const int kColNfIn[COL_NKINDS] = {3, 3, 5, 6, 6, 9, 6, 6, 3, 3, 6, 6, 3, 3, 6, 6};
static const int kColNfOut[COL_NKINDS] = {5, 6, 6, 9, 6, 6, 3, 3, 3, 3, 6, 6, 3, 3, 6, 6};

// 5D view [field][outer][pos_hi][pos_lo][kx re/im] of a column-pass operand (complex strides)
static bool col_map(CUtensorMap* m, const void* ptr, int N, int n1h, int psh, long long ps, long long pcs, int n_outer,
                    long long os, int nf, long long fs, bool tail, int KC) {
  auto enc = tma_encoder();
  if (!enc || !ptr) return false;
  long long L = 1LL << psh;
  if (L >= N) {  // plain layout: re-express as chunks of <= 256 positions
    L = N > 256 ? 256 : N;
    pcs = L * ps;
  } else if (L > 256) {
    return false;
  }
  if (N / L > 256) return false;
  cuuint64_t dims[5] = {(cuuint64_t)(2 * n1h), (cuuint64_t)L, (cuuint64_t)(N / L), (cuuint64_t)n_outer, (cuuint64_t)nf};
  cuuint64_t strides[4] = {(cuuint64_t)(ps * 16), (cuuint64_t)(pcs * 16), (cuuint64_t)(os * 16), (cuuint64_t)(fs * 16)};
  const int SW = KC < 8 ? KC : 8;
  cuuint32_t box[5] = {tail ? 2u : (cuuint32_t)(2 * SW), (cuuint32_t)L, (cuuint32_t)(N / L), tail ? (cuuint32_t)std::min(KC, n_outer) : 1u, 1u};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   tail ? CU_TENSOR_MAP_SWIZZLE_NONE : (SW == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
                   DBF_TMA_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}


template <int N>
static bool col_tma_tiles(const ColGeom& g, ColTiles* tl) {
  constexpr int KC = TmaCfg<N>::KC;
  if (!DBF_COL_TMA || (g.n1h - 1) % KC != 0 || g.n1h - 1 < KC) return false;
  tl->n_outer = (int)(g.ncols / g.n1h);
  tl->nkb = (g.n1h - 1) / KC;
  tl->n_main = tl->n_outer * tl->nkb;
  tl->n_tiles = tl->n_main + (tl->n_outer + KC - 1) / KC;
  tl->tail_cols = std::min(KC, tl->n_outer);
  return true;
}

// ring slots a program needs: term k may use loads up to max(la, lb, ldot) while only rel[k-1]
// have been released (FIFO), so R must exceed that span or producer and consumers deadlock
static int col_prog_span(const TProg& p) {
  int span = 1, released = 0;
  for (int k = 0; k < p.nt; ++k) {
    int need = std::max<int>(p.la[k], std::max<int>(p.lb[k], p.ldot[k]));
    span = std::max(span, need - released + 1);
    released = p.rel[k];
  }
  return span;
}

template <int KIND, bool DOT>
struct ColRing {  // ring depth: 3 slots; small-strain F3 (two-term outputs from 6 inputs) takes 4
  // (B200: 512^3 3.35 -> 3.26 ms, 256^3 0.400 -> 0.392 ms; R = 4 everywhere was slower overall);
  // the finite-strain I1 runs faster with 2 (256^3: 0.319 -> 0.300 ms; I2 was slower with 2, and F2
  // too once the intermediate rows were 128-byte aligned)
  static constexpr int R = (KIND == COL_F3S) ? 4
                           : ((DBF_RING2_FIN && KIND == COL_I1F) || (DBF_RING2_SMALL && (KIND == COL_I1S || KIND == COL_F2S))) ? 2
                           : DBF_COL_R;
};
// ring depth of a launch: the fused F3 + residual update (3 staging buffers) takes 2 slots — its
// program's live span is 2 — and the small-strain F3 3 (span 2) when the stage twiddle table is
// in shared memory, so that everything fits 227 KB
template <int N, int KIND, bool DOT, bool UPD>
struct ColRingL {
  static constexpr bool TAB = ColTab<N, KIND>::value && (!UPD || DBF_UPD_TAB);
  static constexpr int R = UPD ? (TAB ? 2 : 3) : (KIND == COL_F3S && TAB) ? 3 : ColRing<KIND, DOT>::R;
};

template <int N, int KIND, bool DOT, bool UPD = false>
static cudaError_t launch_col_tma_k(const TmaMaps& maps, const ColGeom& g, const ColTiles& tl, cudaStream_t s, int* grid_out) {
  constexpr int R = ColRingL<N, KIND, DOT, UPD>::R;
  constexpr size_t smem = (size_t)(R + (UPD ? 3 : 2) + ((DBF_COL_XINPLACE && !UPD) ? 0 : 1)) * TmaCfg<N>::TILE + 2 * R * sizeof(uint64_t) +
                          (ColRingL<N, KIND, DOT, UPD>::TAB ? sizeof(cplx) * N : 0) + 1024;
  static DevOnce once;
  cudaError_t e = dev_once(once, [](int&) {
    if (col_prog_span(kColProgHost[2 * KIND + (DOT ? 1 : 0)]) > R) return cudaErrorInvalidConfiguration;
    return cudaFuncSetAttribute(col_tma_kernel<N, KIND, DOT, R, UPD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  const int grid = std::min(tl.n_tiles, num_sms());
  if (grid_out) *grid_out = grid;
  return launch_k(col_tma_kernel<N, KIND, DOT, R, UPD>, grid, TmaCfg<N>::THREADS, smem, s, maps, g, tl);
}

// returns cudaErrorNotSupported when this geometry must take the register-pipelined kernel
template <int N>
static cudaError_t launch_col_tma(int kind, const ColGeom& g, cudaStream_t s, int* grid_out) {
  ColTiles tl;
  if (!col_tma_tiles<N>(g, &tl)) return cudaErrorNotSupported;
  constexpr int KC = TmaCfg<N>::KC;
  TmaMaps maps;
  memset(&maps, 0, sizeof(maps));
  const int nfi = kColNfIn[kind], nfo = kColNfOut[kind];
  bool ok = col_map(&maps.in_m, g.in, N, g.n1h, g.in_psh, g.in_ps, g.in_pcs, tl.n_outer, g.in_os, nfi, g.in_fs, false, KC) &&
            col_map(&maps.in_t, g.in, N, g.n1h, g.in_psh, g.in_ps, g.in_pcs, tl.n_outer, g.in_os, nfi, g.in_fs, true, KC) &&
            col_map(&maps.out_m, g.out, N, g.n1h, g.out_psh, g.out_ps, g.out_pcs, tl.n_outer, g.out_os, nfo, g.out_fs, false, KC) &&
            col_map(&maps.out_t, g.out, N, g.n1h, g.out_psh, g.out_ps, g.out_pcs, tl.n_outer, g.out_os, nfo, g.out_fs, true, KC);
  const bool dot = g.dotp != nullptr;
  if (ok && dot)
    ok = col_map(&maps.dot_m, g.dotp, N, g.n1h, g.out_psh, g.out_ps, g.out_pcs, tl.n_outer, g.out_os, 3, g.out_fs, false, KC) &&
         col_map(&maps.dot_t, g.dotp, N, g.n1h, g.out_psh, g.out_ps, g.out_pcs, tl.n_outer, g.out_os, 3, g.out_fs, true, KC);
  if (!ok) return cudaErrorNotSupported;
#define DBF_TK(K) \
  case K: return launch_col_tma_k<N, K, false>(maps, g, tl, s, grid_out);
  if (g.upd) {  // F3 fused with the PCG residual update (r through the ring)
    if (!dot || kind != COL_F3F) return cudaErrorInvalidValue;
    return launch_col_tma_k<N, COL_F3F, true, true>(maps, g, tl, s, grid_out);
  }
  if (dot) return cudaErrorInvalidValue;  // the ring-loaded operand exists only for the fused update
  switch (kind) {
    DBF_TK(COL_I1S) DBF_TK(COL_I1F) DBF_TK(COL_I2S) DBF_TK(COL_I2F) DBF_TK(COL_F2S) DBF_TK(COL_F2F) DBF_TK(COL_F3S)
    DBF_TK(COL_F3F) DBF_TK(COL_ZI3) DBF_TK(COL_YI3) DBF_TK(COL_ZI6) DBF_TK(COL_YI6) DBF_TK(COL_ZF3)
    DBF_TK(COL_YF3) DBF_TK(COL_ZF6) DBF_TK(COL_YF6)
    default: return cudaErrorInvalidValue;
  }
#undef DBF_TK
}

static cudaError_t launch_col_reg(int kind, int N, const ColGeom& g, cudaStream_t s) {
  switch (N) {
    case 8: return launch_col_n<8>(kind, g, s);
    case 16: return launch_col_n<16>(kind, g, s);
    case 32: return launch_col_n<32>(kind, g, s);
    case 64: return launch_col_n<64>(kind, g, s);
    case 128: return launch_col_n<128>(kind, g, s);
    case 256: return launch_col_n<256>(kind, g, s);
    case 512: return launch_col_n<512>(kind, g, s);
    case 15: return launch_col_n<15>(kind, g, s);
    case 21: return launch_col_n<21>(kind, g, s);
    case 27: return launch_col_n<27>(kind, g, s);
    case 63: return launch_col_n<63>(kind, g, s);
    default: return cudaErrorInvalidValue;
  }
}

bool col_upd_supported(int N, const ColGeom& g) {
  ColTiles tl;
  if (N == 512) return col_tma_tiles<512>(g, &tl);
  if (N == 256) return col_tma_tiles<256>(g, &tl);
  if (N == 128) return col_tma_tiles<128>(g, &tl);
  if (N == 64) return col_tma_tiles<64>(g, &tl);
  return false;
}

cudaError_t launch_col(int kind, int N, const ColGeom& g, cudaStream_t s, int* grid_out) {
  cudaError_t e = cudaErrorNotSupported;
  // N = 512 y-forward passes write rows 2 MB apart (the ky stride of [f][ky][z][kx] at 512^2): the
  // TMA store path ran them at 2.2 TB/s against 4 TB/s for direct stores (B200, kbench 512^3)
  const bool far_store = N == 512 && (kind == COL_F2S || kind == COL_F2F || kind == COL_YF3 || kind == COL_YF6 ||
                                       ((DBF_REG512_MASK >> kind) & 1));
  if (N == 512 && !far_store) e = launch_col_tma<512>(kind, g, s, grid_out);
  else if (N == 256) e = launch_col_tma<256>(kind, g, s, grid_out);
  else if (N == 128) e = launch_col_tma<128>(kind, g, s, grid_out);
  else if (N == 64) e = launch_col_tma<64>(kind, g, s, grid_out);
  if (e != cudaErrorNotSupported) return e;
  if (g.upd || g.dotp) return cudaErrorInvalidValue;  // the fused update exists on the TMA path only
  if (grid_out) *grid_out = col_grid(N, g.ncols);
  return launch_col_reg(kind, N, g, s);
}

template <int N1, int KIND>
static cudaError_t launch_x_k(const XGeom& g, cudaStream_t s, int* grid_out, int nf_real) {
  typedef XCfg<N1, KIND> CF;
  static DevOnce once;  // per template instance and device: resident CTAs on the whole device
  int max_grid = 0;
  cudaError_t e = dev_once(
      once,
      [](int& mg) {
        cudaError_t e2 = cudaFuncSetAttribute(x_pass_kernel<N1, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
        if (e2 != cudaSuccess) return e2;
        int nb = 0;
        e2 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, x_pass_kernel<N1, KIND>, CF::THREADS, CF::SMEM);
        mg = std::max(1, nb) * num_sms();
        return e2;
      },
      &max_grid);
  if (e != cudaSuccess) return e;
  const long long ngroups = (g.nlines + CF::LPAR - 1) / CF::LPAR;
  // never more CTAs than partial slots were allocated for (x_grid)
  const int grid = (int)std::min<long long>(std::min<long long>(ngroups, max_grid), x_grid(KIND, N1, g.nlines));
  if (grid_out) *grid_out = grid;
  return launch_k(x_pass_kernel<N1, KIND>, grid, CF::THREADS, CF::SMEM, s, g, nf_real);
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
  if (kind >= X_REAL_IN) return launch_x_k<N1, X_REAL_IN>(g, s, grid_out, kind - X_REAL_IN);
  if (kind >= X_REAL_OUT) return launch_x_k<N1, X_REAL_OUT>(g, s, grid_out, kind - X_REAL_OUT);
  return cudaErrorInvalidValue;
}

// kind X_REAL_OUT + nf selects a real-output transform of nf fields (1..9)
template <int N1>
static cudaError_t launch_x_ws(const XGeom& g, cudaStream_t s, int* grid_out) {
  typedef XwsCfg<N1> W;
  static DevOnce once;
  int max_grid = 0;
  cudaError_t e = dev_once(
      once,
      [](int& mg) {
        cudaError_t e2 = cudaFuncSetAttribute(x_pass_ws_kernel<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W::SMEM);
        if (e2 != cudaSuccess) return e2;
        int nb = 0;
        e2 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, x_pass_ws_kernel<N1>, W::THREADS, W::SMEM);
        mg = std::max(1, nb) * num_sms();
        return e2;
      },
      &max_grid);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<long long>(std::min<long long>(g.nlines, max_grid), x_grid(X_K_FIN_NH, N1, g.nlines));
  if (grid_out) *grid_out = grid;
  x_pass_ws_kernel<N1><<<grid, W::THREADS, W::SMEM, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_x(int kind, int N1, const XGeom& g, cudaStream_t s, int* grid_out) {
  if (DBF_XWS && kind == X_K_FIN_NH && N1 == 256 && g.in && g.out) return launch_x_ws<256>(g, s, grid_out);
  switch (N1) {
    case 8: return launch_x_n<8>(kind, g, s, grid_out);
    case 16: return launch_x_n<16>(kind, g, s, grid_out);
    case 32: return launch_x_n<32>(kind, g, s, grid_out);
    case 64: return launch_x_n<64>(kind, g, s, grid_out);
    case 128: return launch_x_n<128>(kind, g, s, grid_out);
    case 256: return launch_x_n<256>(kind, g, s, grid_out);
    case 512: return launch_x_n<512>(kind, g, s, grid_out);
    case 15: return launch_x_n<15>(kind, g, s, grid_out);
    case 21: return launch_x_n<21>(kind, g, s, grid_out);
    case 27: return launch_x_n<27>(kind, g, s, grid_out);
    case 63: return launch_x_n<63>(kind, g, s, grid_out);
    default: return cudaErrorInvalidValue;
  }
}

// upper bound of the X-pass grid (= number of line groups) for partial-buffer sizing
int x_grid(int kind, int N1, long long nlines) {
  (void)kind;
  (void)N1;
  return (int)std::min<long long>(nlines, 32LL * num_sms());  // <= 32 resident CTAs per SM
}

cudaError_t launch_tangent81(int mode, const XGeom& g, long long v0, long long nv, double* out, cudaStream_t s) {
  const int grid = (int)std::min<long long>((nv + 255) / 256, 8LL * num_sms());
  switch (mode) {
    case 0: k_tangent81<0><<<grid, 256, 0, s>>>(g, v0, nv, out); break;
    case 1: k_tangent81<1><<<grid, 256, 0, s>>>(g, v0, nv, out); break;
    case 2: k_tangent81<2><<<grid, 256, 0, s>>>(g, v0, nv, out); break;
    default: k_tangent81<3><<<grid, 256, 0, s>>>(g, v0, nv, out); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_mean_tangent(int mode, const XGeom& g, double* partials, int nblk, cudaStream_t s) {
  if (mode == 0) k_mean_tangent<0><<<nblk, 256, 0, s>>>(g, partials);
  else if (mode == 1) k_mean_tangent<1><<<nblk, 256, 0, s>>>(g, partials);
  else k_mean_tangent<2><<<nblk, 256, 0, s>>>(g, partials);
  return cudaGetLastError();
}
