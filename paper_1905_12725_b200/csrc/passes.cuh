// passes.cuh — geometry/parameter structs shared by the pass kernels and the host driver.
#pragma once
#include "common.cuh"

// Frequency tables (Eq. 1 with the Nyquist reading R1), device arrays.
struct Freq {
  const double* xx;  // [n1h]
  const double* xy;  // [n2]
  const double* xz;  // [n3]
};

// Column pass (FFT along z or y) geometry.  Field f, outer index o, position p, kx:
//   addr = f*fs + o*os + (p >> psh)*pcs + (p & (2^psh - 1))*ps + kx      (complex elements)
// psh/pcs express rank-blocked layouts of a distributed transpose (2^psh = N: plain).
struct ColGeom {
  const cplx* in;
  cplx* out;
  long long in_fs, in_os, in_ps, in_pcs;
  long long out_fs, out_os, out_ps, out_pcs;
  int in_psh, out_psh;   // log2 of the rank chunk along the FFT axis (log2 N: plain)
  int n1h;
  long long ncols;   // n_outer * n1h columns
  const cplx* tw;    // twiddles W_N[k], k < N, then the stage-ordered table (N - 1, powers of two)
  const double* fpos;  // xi along the FFT axis, indexed by position (z passes: xi_z, y passes: xi_y)
  Freq fq;
  // F3 fused with the PCG residual update (TMA path only): out = dotp = r, streamed through the
  // ring; r -= alpha q, partial <r, M r>, <r, r> per CTA into partials[2 blockIdx] (Hermitian
  // weights: kx = 0 and n1/2 count once); skipped once PCG stopped
  const cplx* dotp;
  double* partials;
  int n1;            // full x length
  int upd;
  const double* cg_alpha;
  // early exit (any column kind): inside the PCG loop the passes of an iteration return at once
  // when PCG has stopped (CgDev.converged / .breakdown; null: always run)
  const int* cg_stop0;   // CgDev.converged
  const int* cg_stop1;   // CgDev.breakdown
  const double* precq;   // preconditioner coefficients (prec_apply; 36 doubles, device)
  int n_xy;          // length of fq.xy (guards the per-column xi_y(outer) lookup of y passes)
  int kx0;           // global kx of local column 0 (pencil decomposition: the rank's kx block; else 0)
};

// Column pass kinds
enum ColKind {
  COL_I1S = 0,  // small strain, z inverse: u(3) -> {u_x, u_y, eps_zz, eps_xz, eps_yz}
  COL_I1F,      // finite strain, z inverse: u(3) -> {u_i, G_iz}
  COL_I2S,      // small strain, y inverse: 5 -> eps (Voigt 6)
  COL_I2F,      // finite strain, y inverse: 6 -> 9 (G_ix holds u_i until the x pass)
  COL_F2S,      // small strain, y forward: sigma (6) -> 6
  COL_F2F,      // finite strain, y forward: 9 -> {g_i, P_iz}
  COL_F3S,      // small strain, z forward + divergence: 6 -> f (3)
  COL_F3F,      // finite strain, z forward + divergence: 6 -> f (3)
  COL_ZI3,      // plain z inverse of a vector (3)
  COL_YI3,      // plain y inverse of a vector (3)
  COL_ZI6,      // plain z / y inverse and forward transforms of 3 or 6 fields (residual monitors)
  COL_YI6,
  COL_ZF3,
  COL_YF3,
  COL_ZF6,
  COL_YF6,
  COL_NKINDS
};

// X pass (lines along x: C2R -> per-voxel op -> R2C) voxel-op kinds
enum XKind {
  X_K_SMALL_PHASE = 0,  // sigma = C_phase : (eps + e)            (apply_K, linear)
  X_K_J2,               // sigma = C_alg(x) : (eps + e)           (apply_K, compact J2 tangent)
  X_K_FIN_TAN,          // dP = K(x) : (G + e), 45-entry K        (apply_K, finite strain)
  X_K_FIN_NH,           // dP = K(x) : (G + e), matrix-free K(F)  (apply_K, finite strain)
  X_RHS_SMALL_PHASE,    // -sigma = -C_phase : e                  (rhs of the linear system)
  X_CONST_FIN,          // F += G + dF; P, K (neo-Hookean); -P    (Newton residual)
  X_CONST_J2,           // eps += G + de; J2 return map; -sigma   (Newton residual)
  X_REAL_OUT,           // C2R only -> real fields (kind X_REAL_OUT + nf)
  X_NKINDS,
  X_REAL_IN = 32        // R2C only <- real fields [f][N] (kind X_REAL_IN + nf, nf <= 9)
};

struct XGeom {
  const cplx* in;       // [f][line][kx], line = z*n2 + y
  cplx* out;
  long long fs_in, fs_out;
  int n1h, n1;
  int kxp;              // line pitch of in / out (complex elements, >= n1h)
  long long nlines;
  const cplx* tw;       // twiddles W_{n1}
  const double* xix;    // xi_x [n1h]
  double inv_n;         // 1 / (n1 n2 n3)
  double oscale;        // 1 / (2N): voxel outputs are pre-scaled so the unnormalised pair R2C (x2) is F/N
  double* partials;     // per CTA reduction outputs [grid][nred]
  int nred;
  // materials / state (SoA, voxel index = line*n1 + x)
  const uint16_t* phase;
  const double* ptable;   // per phase: 36 doubles (linear Voigt 6x6 row-major) / params
  const double* e;        // 9 macro doubles (device) or null
  double* tan;            // tangent SoA [21 or 45][N]
  double* F;              // finite: F SoA [9][N]; J2: eps SoA [6][N]
  const double* epsp_c;   // J2 committed plastic strain [6][N]
  double* epsp_t;         // J2 trial plastic strain [6][N]
  double dt;
  long long nvox;
  double* real_out;       // X_REAL_OUT: [f][N]
  const double* real_in;  // X_REAL_IN: field f at real_in + real_map[f] * nvox
  int real_map[9];
  int* bad;               // first bad voxel flag (atomicMin on voxel index)
  int has_in;             // constitutive kinds: 0 = no C2R input (uniform increment only)
  int tmode;              // X_CONST_FIN: 0 = store the 45-entry tangent, 1 = compact (F^-1, c1)
  const int* stop0;       // PCG loop early exit (CgDev.converged / .breakdown), null: always run
  const int* stop1;
  // pencil decomposition (kch > 0): a line's kx arrive in npy chunks of kch columns (+ the Nyquist
  // in slot kch of the last chunk; slot kch of the others is padding, written 0), chunk c at
  // in + c * kpcs_in (out + c * kpcs_out); kch = 0: one contiguous row of n1h
  int kch, npy;
  long long kpcs_in, kpcs_out;
};

// host launchers (passes.cu)
// grid_out: CTAs launched (= per-CTA partial pairs written when upd is set)
cudaError_t launch_col(int kind, int N, const ColGeom& g, cudaStream_t s, int* grid_out = nullptr);
// can F3 on this geometry run fused with the PCG residual update (TMA column path)?
bool col_upd_supported(int N, const ColGeom& g);
cudaError_t launch_x(int kind, int N1, const XGeom& g, cudaStream_t s, int* grid_out);
int x_grid(int kind, int N1, long long nlines);
// streaming multiprocessors of the current device (cached per device)
int num_sms();
int col_grid(int N, long long ncols);
// per-voxel tangent, full 81 entries [81][nv] of voxels v0 .. v0+nv (mode 0: stored 45, 1: compact
// neo-Hookean, 2: compact J2, 3: linear phase table)
cudaError_t launch_tangent81(int mode, const XGeom& g, long long v0, long long nv, double* out, cudaStream_t s);
// mean tangent partials (mode 0: full 45, 1: compact neo-Hookean -> 45, 2: compact J2 -> 21)
cudaError_t launch_mean_tangent(int mode, const XGeom& g, double* partials, int nblk, cudaStream_t s);
