// dbfft.cu — C-ABI implementation and host driver (plan, buffers, PCG and Newton drivers).
//
// Host code only orchestrates: every arithmetic step of the hot path (gradient, FFTs,
// contraction, divergence, preconditioner, CG algebra, constitutive updates, reductions) runs
// in the kernels of passes.cu / cg.cu / this file.  The host does the O(1) macro algebra
// (9x9 macro-block inverse, preconditioner coefficients from Cbar) once per increment.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dbfft.h"
#include "cg.cuh"
#include "passes.cuh"

namespace {

enum Family { FAM_NONE = 0, FAM_LINEAR = 1, FAM_NEOHOOKE = 2, FAM_J2 = 3 };

enum ProfId { PK_I1 = 0, PK_I2, PK_X, PK_F2, PK_F3, PK_XCONST, PK_CGUPD, PK_CGDIR, PK_FIN, PK_OTHER, PK_COUNT };
const char* kProfNames[PK_COUNT] = {"pass_I1", "pass_I2", "pass_X", "pass_F2", "pass_F3", "pass_X_const",
                                    "cg_update", "cg_direction", "cg_finalize", "other"};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

std::string g_create_error;

}  // namespace

struct dbfft_ctx_s {
  int n1, n2, n3, n1h;
  double L[3];
  int kin;  // 6 or 9
  long long N, Hs;
  int device;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  // tables
  double *xix = nullptr, *xiy = nullptr, *xiz = nullptr;
  cplx *tw1 = nullptr, *tw2 = nullptr, *tw3 = nullptr;
  // vectors [3][Hs]
  cplx *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *b = nullptr, *u = nullptr, *u_c = nullptr;
  cplx *WA = nullptr, *WB = nullptr;
  // materials and state
  int family = FAM_NONE;
  int nph = 0;
  uint16_t* phase = nullptr;
  double* ptable = nullptr;
  std::vector<double> h_ptable;
  double *F = nullptr, *F_c = nullptr;      // finite: F [9][N]; J2: eps [6][N]
  double *epsp_c = nullptr, *epsp_t = nullptr;
  double* tan = nullptr;                    // [21|45][N]
  double Fbar[9], Fbar_c[9];                // macro strain / F (incl. stress-controlled comps)
  bool tangent_valid = false;
  int tmode = 1;                            // neo-Hookean tangent storage: 1 compact (F^-1, c1), 0 full 45
  // linear mean stiffness (Voigt 6x6) or current mean tangent (full 81)
  double Cbar[81];
  PrecQ prec;
  bool prec_valid = false;
  // CG
  CgDev* cg = nullptr;
  CgDev* h_cg = nullptr;      // pinned mirror
  double *part_x = nullptr, *part_f3 = nullptr, *part_cg = nullptr, *part_misc = nullptr;
  double* red_out = nullptr;  // [64]
  double* h_red = nullptr;    // pinned [64]
  double* e_dev = nullptr;    // [9] macro block for passes
  int* bad = nullptr;
  int* h_bad = nullptr;
  unsigned long long* counts = nullptr;
  double* tmp_real = nullptr;  // [9][N] scratch for get_field / eval_state
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<int, int>>> ev_pending;  // id, (start idx, stop idx)
  size_t ev_next = 0;
  double prof_ms[PK_COUNT];
  long long prof_n[PK_COUNT];
  long long nlaunch = 0;  // kernels launched by this ctx (always counted)
};

namespace {

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                          \
      return e_ == cudaErrorMemoryAllocation ? DBFFT_E_OOM : DBFFT_E_CUDA;                    \
    }                                                                                         \
  } while (0)

#define CKS(call)                                                                             \
  do {                                                                                        \
    dbfft_status s_ = (call);                                                                 \
    if (s_ != DBFFT_OK) return s_;                                                            \
  } while (0)

int ilog2(int n) {
  int k = 0;
  while ((1 << k) < n) ++k;
  return k;
}

bool is_pow2_in(int n) { return n >= 8 && n <= 512 && (n & (n - 1)) == 0; }

// ---------------------------------------------------------------- profiling helpers
struct ProfScope {
  dbfft_ctx ctx;
  int id;
  int i0 = -1;
  ProfScope(dbfft_ctx c, int k) : ctx(c), id(k) {
    ctx->nlaunch += 1;
    if (!ctx->prof) return;
    if (ctx->ev_next + 2 > ctx->ev_pool.size()) {
      for (int j = 0; j < 256; ++j) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
      }
    }
    i0 = (int)ctx->ev_next;
    ctx->ev_next += 2;
    cudaEventRecord(ctx->ev_pool[i0], ctx->stream);
  }
  ~ProfScope() {
    if (i0 < 0) return;
    cudaEventRecord(ctx->ev_pool[i0 + 1], ctx->stream);
    ctx->ev_pending.push_back({id, {i0, i0 + 1}});
  }
};

void prof_flush(dbfft_ctx ctx) {
  if (ctx->ev_pending.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->ev_pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev_pool[e.second.first], ctx->ev_pool[e.second.second]) == cudaSuccess) {
      ctx->prof_ms[e.first] += ms;
      ctx->prof_n[e.first] += 1;
    }
  }
  ctx->ev_pending.clear();
  ctx->ev_next = 0;
}

// ---------------------------------------------------------------- geometry builders
Freq freq(dbfft_ctx ctx) { return Freq{ctx->xix, ctx->xiy, ctx->xiz}; }

SpecGeom spec(dbfft_ctx ctx) {
  SpecGeom g;
  g.n1h = ctx->n1h;
  g.n2 = ctx->n2;
  g.n3 = ctx->n3;
  g.Hs = ctx->Hs;
  g.fq = freq(ctx);
  g.n1 = ctx->n1;
  return g;
}

// layouts (complex elements):
//   S  spectral [f][ky][kz][kx] : fs = Hs, ky stride n3*n1h, kz stride n1h
//   A  after z   [f][ky][z][kx]  : same strides as S
//   B  after y   [f][z][y][kx]   : fs = Hs, z stride n2*n1h, y stride n1h
ColGeom colgeom(dbfft_ctx ctx, bool zpass, const cplx* in, cplx* out, bool in_is_B, bool out_is_B) {
  ColGeom g;
  memset(&g, 0, sizeof(g));
  const long long n1h = ctx->n1h;
  g.in = in;
  g.out = out;
  g.in_fs = g.out_fs = ctx->Hs;
  g.n1h = ctx->n1h;
  g.n1 = ctx->n1;
  g.fq = freq(ctx);
  if (zpass) {  // outer = ky, pos = kz/z, both in S/A layout
    g.in_os = g.out_os = (long long)ctx->n3 * n1h;
    g.in_ps = g.out_ps = n1h;
    g.ncols = (long long)ctx->n2 * n1h;
    g.in_psh = g.out_psh = ilog2(ctx->n3);
    g.tw = ctx->tw3;
  } else {  // outer = z, pos = y/ky
    if (in_is_B) { g.in_os = (long long)ctx->n2 * n1h; g.in_ps = n1h; }
    else { g.in_os = n1h; g.in_ps = (long long)ctx->n3 * n1h; }
    if (out_is_B) { g.out_os = (long long)ctx->n2 * n1h; g.out_ps = n1h; }
    else { g.out_os = n1h; g.out_ps = (long long)ctx->n3 * n1h; }
    g.ncols = (long long)ctx->n3 * n1h;
    g.in_psh = g.out_psh = ilog2(ctx->n2);
    g.tw = ctx->tw2;
  }
  g.in_pcs = g.out_pcs = 0;
  return g;
}

XGeom xgeom(dbfft_ctx ctx, const cplx* in, cplx* out) {
  XGeom g;
  memset(&g, 0, sizeof(g));
  g.in = in;
  g.out = out;
  g.fs_in = g.fs_out = ctx->Hs;
  g.n1h = ctx->n1h;
  g.n1 = ctx->n1;
  g.nlines = (long long)ctx->n2 * ctx->n3;
  g.tw = ctx->tw1;
  g.xix = ctx->xix;
  g.inv_n = 1.0 / (double)ctx->N;
  g.partials = ctx->part_x;
  g.nred = 10;
  g.phase = ctx->phase;
  g.ptable = ctx->ptable;
  g.tan = ctx->tan;
  g.F = ctx->F;
  g.epsp_c = ctx->epsp_c;
  g.epsp_t = ctx->epsp_t;
  g.nvox = ctx->N;
  g.bad = ctx->bad;
  g.tmode = ctx->tmode;
  return g;
}

dbfft_status run_col(dbfft_ctx ctx, int kind, int prof_id, const ColGeom& g) {
  ProfScope ps(ctx, prof_id);
  const int N = (kind == COL_I1S || kind == COL_I1F || kind == COL_F3S || kind == COL_F3F || kind == COL_ZI3) ? ctx->n3 : ctx->n2;
  CK(launch_col(kind, N, g, ctx->stream));
  return DBFFT_OK;
}

dbfft_status run_x(dbfft_ctx ctx, int kind, int prof_id, const XGeom& g, int* grid) {
  ProfScope ps(ctx, prof_id);
  CK(launch_x(kind, ctx->n1, g, ctx->stream, grid));
  return DBFFT_OK;
}

// ---------------------------------------------------------------- host linear algebra
const int kVoigtI[6] = {0, 1, 2, 1, 0, 0};
const int kVoigtJ[6] = {0, 1, 2, 2, 2, 1};
int voigt_of(int i, int j) {
  if (i == j) return i;
  if ((i == 1 && j == 2) || (i == 2 && j == 1)) return 3;
  if ((i == 0 && j == 2) || (i == 2 && j == 0)) return 4;
  return 5;
}

// full C_ijkl (81) from a Voigt 6x6 of tensor entries
void voigt_to_full(const double* CV, double* C81) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) C81[((i * 3 + j) * 3 + k) * 3 + l] = CV[6 * voigt_of(i, j) + voigt_of(k, l)];
}

void iso_voigt(double E, double nu, double* CV) {
  const double lam = E * nu / ((1 + nu) * (1 - 2 * nu)), mu = E / (2 * (1 + nu));
  for (int a = 0; a < 36; ++a) CV[a] = 0.0;
  for (int I = 0; I < 3; ++I)
    for (int J = 0; J < 3; ++J) CV[6 * I + J] = lam + (I == J ? 2 * mu : 0.0);
  for (int I = 3; I < 6; ++I) CV[6 * I + I] = mu;
}

void cubic_voigt(double C11, double C12, double C44, const double* R, double* CV) {
  double C0[81], C[81];
  for (int a = 0; a < 81; ++a) C0[a] = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      C0[((a * 3 + a) * 3 + b) * 3 + b] = (a == b) ? C11 : C12;
      if (a != b) {
        C0[((a * 3 + b) * 3 + a) * 3 + b] = C44;
        C0[((a * 3 + b) * 3 + b) * 3 + a] = C44;
      }
    }
  // rotate index by index: C_ijkl = R_ia R_jb R_kc R_ld C0_abcd (four successive contractions)
  double T1[81], T2[81], T3[81];
  auto idx = [](int i, int j, int k, int l) { return ((i * 3 + j) * 3 + k) * 3 + l; };
  for (int i = 0; i < 3; ++i) for (int b = 0; b < 3; ++b) for (int c = 0; c < 3; ++c) for (int d = 0; d < 3; ++d) {
    double s = 0; for (int a = 0; a < 3; ++a) s += R[3 * i + a] * C0[idx(a, b, c, d)]; T1[idx(i, b, c, d)] = s; }
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) for (int c = 0; c < 3; ++c) for (int d = 0; d < 3; ++d) {
    double s = 0; for (int b = 0; b < 3; ++b) s += R[3 * j + b] * T1[idx(i, b, c, d)]; T2[idx(i, j, c, d)] = s; }
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) for (int k = 0; k < 3; ++k) for (int d = 0; d < 3; ++d) {
    double s = 0; for (int c = 0; c < 3; ++c) s += R[3 * k + c] * T2[idx(i, j, c, d)]; T3[idx(i, j, k, d)] = s; }
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) for (int k = 0; k < 3; ++k) for (int l = 0; l < 3; ++l) {
    double s = 0; for (int d = 0; d < 3; ++d) s += R[3 * l + d] * T3[idx(i, j, k, d)]; C[idx(i, j, k, l)] = s; }
  for (int I = 0; I < 6; ++I)
    for (int J = 0; J < 6; ++J) CV[6 * I + J] = C[idx(kVoigtI[I], kVoigtJ[I], kVoigtI[J], kVoigtJ[J])];
}

// preconditioner coefficients from a full C81: A_ik = sum_jl xi_j xi_l C_ijkl
PrecQ make_prec(const double* C81) {
  PrecQ q;
  const int mi[6] = {0, 1, 2, 1, 0, 0}, mk[6] = {0, 1, 2, 2, 2, 1};
  const int pj[6] = {0, 1, 2, 1, 0, 0}, pl[6] = {0, 1, 2, 2, 2, 1};
  auto C = [&](int i, int j, int k, int l) { return C81[((i * 3 + j) * 3 + k) * 3 + l]; };
  for (int m = 0; m < 6; ++m)
    for (int p = 0; p < 6; ++p) {
      const int i = mi[m], k = mk[m], j = pj[p], l = pl[p];
      q.Q[6 * m + p] = (j == l) ? C(i, j, k, l) : C(i, j, k, l) + C(i, l, k, j);
    }
  return q;
}

bool invert(std::vector<double>& A, int n) {  // Gauss-Jordan with partial pivoting, in place
  std::vector<double> I(n * n, 0.0);
  for (int i = 0; i < n; ++i) I[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (std::fabs(A[piv * n + c]) < 1e-300) return false;
    for (int k = 0; k < n; ++k) {
      std::swap(A[c * n + k], A[piv * n + k]);
      std::swap(I[c * n + k], I[piv * n + k]);
    }
    const double d = 1.0 / A[c * n + c];
    for (int k = 0; k < n; ++k) { A[c * n + k] *= d; I[c * n + k] *= d; }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = A[r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) { A[r * n + k] -= f * A[c * n + k]; I[r * n + k] -= f * I[c * n + k]; }
    }
  }
  A = I;
  return true;
}

// Minv (9x9 on row-major tensors) = sum_ab E_a (M^-1)_ab E_b^T, M_ab = E_a : C : E_b over an
// orthonormal basis of the stress-controlled subspace (R4).
bool macro_inverse(const double* C81, const uint8_t* mask, bool sym, double* Minv) {
  std::vector<std::vector<double>> B;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      if (!mask[3 * i + j]) continue;
      std::vector<double> E(9, 0.0);
      if (sym) {
        if (j < i) continue;
        if (i == j) E[3 * i + i] = 1.0;
        else E[3 * i + j] = E[3 * j + i] = 1.0 / std::sqrt(2.0);
      } else {
        E[3 * i + j] = 1.0;
      }
      B.push_back(E);
    }
  for (int a = 0; a < 81; ++a) Minv[a] = 0.0;
  const int m = (int)B.size();
  if (m == 0) return true;
  std::vector<double> M(m * m, 0.0);
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) {
      double s = 0.0;
      for (int u = 0; u < 9; ++u)
        for (int v = 0; v < 9; ++v) s += B[a][u] * C81[u * 9 + v] * B[b][v];
      M[a * m + b] = s;
    }
  if (!invert(M, m)) return false;
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b)
      for (int u = 0; u < 9; ++u)
        for (int v = 0; v < 9; ++v) Minv[u * 9 + v] += B[a][u] * M[a * m + b] * B[b][v];
  return true;
}

// ---------------------------------------------------------------- small pointwise kernels
__global__ void k_expand6(const double* __restrict__ v6, long long n, const double* macro9, double* __restrict__ out9) {
  const int row9_of_voigt[6] = {0, 4, 8, 5, 2, 1};
  (void)row9_of_voigt;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int vo[9] = {0, 5, 4, 5, 1, 3, 4, 3, 2};
    for (int a = 0; a < 9; ++a) out9[(long long)a * n + i] = v6[(long long)vo[a] * n + i] + (macro9 ? macro9[a] : 0.0);
  }
}

__global__ void k_stress_linear(const double* __restrict__ e9, const uint16_t* __restrict__ ph, const double* __restrict__ pt,
                                long long n, double* __restrict__ s9) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double* C = pt + 36 * ph[i];
    const int ri[6] = {0, 4, 8, 5, 2, 1};
    double g[6];
    for (int J = 0; J < 6; ++J) g[J] = e9[(long long)ri[J] * n + i] * (J < 3 ? 1.0 : 2.0);
    double s[6];
    for (int I = 0; I < 6; ++I) {
      double a = 0.0;
      for (int J = 0; J < 6; ++J) a += C[6 * I + J] * g[J];
      s[I] = a;
    }
    const int vo[9] = {0, 5, 4, 5, 1, 3, 4, 3, 2};
    for (int a = 0; a < 9; ++a) s9[(long long)a * n + i] = s[vo[a]];
  }
}

__global__ void k_stress_j2(const double* __restrict__ eps6, const double* __restrict__ ep6, const uint16_t* __restrict__ ph,
                            const double* __restrict__ pt, long long n, double* __restrict__ s9) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double* prm = pt + 36 * ph[i];
    const double E = prm[0], nu = prm[1];
    const double lam = E * nu / ((1 + nu) * (1 - 2 * nu)), mu = E / (2 * (1 + nu));
    double ee[6];
    for (int I = 0; I < 6; ++I) ee[I] = eps6[(long long)I * n + i] - ep6[(long long)I * n + i];
    const double tr = ee[0] + ee[1] + ee[2];
    double s[6];
    for (int I = 0; I < 6; ++I) s[I] = 2 * mu * ee[I] + (I < 3 ? lam * tr : 0.0);
    const int vo[9] = {0, 5, 4, 5, 1, 3, 4, 3, 2};
    for (int a = 0; a < 9; ++a) s9[(long long)a * n + i] = s[vo[a]];
  }
}

__global__ void k_stress_nh(const double* __restrict__ F9, const uint16_t* __restrict__ ph, const double* __restrict__ pt,
                            long long n, double* __restrict__ P9) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double F[9];
    for (int a = 0; a < 9; ++a) F[a] = F9[(long long)a * n + i];
    const double mu = pt[36 * ph[i]], kappa = pt[36 * ph[i] + 1];
    const double lam = kappa - 2.0 * mu / 3.0;
    const double c00 = F[4] * F[8] - F[5] * F[7], c01 = F[5] * F[6] - F[3] * F[8], c02 = F[3] * F[7] - F[4] * F[6];
    const double J = F[0] * c00 + F[1] * c01 + F[2] * c02;
    double FiT[9];  // F^-T = cof(F)/J
    FiT[0] = c00 / J; FiT[1] = c01 / J; FiT[2] = c02 / J;
    FiT[3] = (F[2] * F[7] - F[1] * F[8]) / J; FiT[4] = (F[0] * F[8] - F[2] * F[6]) / J; FiT[5] = (F[1] * F[6] - F[0] * F[7]) / J;
    FiT[6] = (F[1] * F[5] - F[2] * F[4]) / J; FiT[7] = (F[2] * F[3] - F[0] * F[5]) / J; FiT[8] = (F[0] * F[4] - F[1] * F[3]) / J;
    const double lnJ = log(J);
    for (int a = 0; a < 9; ++a) P9[(long long)a * n + i] = mu * F[a] + (lam * lnJ - mu) * FiT[a];
  }
}

__global__ void k_identity9(double* F9, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    for (int a = 0; a < 9; ++a) F9[(long long)a * n + i] = (a % 4 == 0) ? 1.0 : 0.0;
}

template <typename T>
dbfft_status dalloc(dbfft_ctx ctx, T** p, size_t count) {
  CK(cudaMalloc((void**)p, sizeof(T) * std::max<size_t>(count, 1)));
  return DBFFT_OK;
}

dbfft_status make_twiddles(dbfft_ctx ctx, int n, cplx** out) {
  std::vector<double2> h(n);
  for (int k = 0; k < n; ++k) {
    long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)k / (long double)n;
    h[k] = make_double2((double)cosl(a), (double)sinl(a));
  }
  CKS(dalloc(ctx, out, n));
  CK(cudaMemcpy(*out, h.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
  return DBFFT_OK;
}

// xi_a(k) = 2 pi kappa / L, Nyquist zero (R1)
std::vector<double> axis_xi(int n, double L, int count) {
  std::vector<double> v(count);
  for (int k = 0; k < count; ++k) {
    int kappa = (2 * k < n) ? k : k - n;
    if (2 * k == n) kappa = 0;
    v[k] = 2.0 * 3.14159265358979323846 * (double)kappa / L;
  }
  return v;
}

// ---------------------------------------------------------------- operator application
struct ApplyOut {
  int grid_x = 0, grid_f3 = 0;
};

// f = K(u) [+ e]; partials: part_x (DC of sigma), part_f3 (<u, f>)
dbfft_status apply_K_internal(dbfft_ctx ctx, const cplx* u, cplx* f, const double* e, bool dot, ApplyOut* ao) {
  const bool fin = ctx->kin == 9;
  int xkind;
  if (ctx->family == FAM_LINEAR) xkind = X_K_SMALL_PHASE;
  else if (ctx->family == FAM_J2) xkind = X_K_J2;
  else xkind = ctx->tmode ? X_K_FIN_NH : X_K_FIN_TAN;
  ColGeom g1 = colgeom(ctx, true, u, ctx->WA, false, false);
  CKS(run_col(ctx, fin ? COL_I1F : COL_I1S, PK_I1, g1));
  ColGeom g2 = colgeom(ctx, false, ctx->WA, ctx->WB, false, true);
  CKS(run_col(ctx, fin ? COL_I2F : COL_I2S, PK_I2, g2));
  XGeom gx = xgeom(ctx, ctx->WB, ctx->WB);
  gx.e = e;
  int gridx = 0;
  CKS(run_x(ctx, xkind, PK_X, gx, &gridx));
  ColGeom g4 = colgeom(ctx, false, ctx->WB, ctx->WA, true, false);
  CKS(run_col(ctx, fin ? COL_F2F : COL_F2S, PK_F2, g4));
  ColGeom g5 = colgeom(ctx, true, ctx->WA, f, false, false);
  if (dot) {
    g5.dotp = u;
    g5.partials = ctx->part_f3;
  }
  CKS(run_col(ctx, fin ? COL_F3F : COL_F3S, PK_F3, g5));
  if (ao) {
    ao->grid_x = gridx;
    ao->grid_f3 = col_grid(ctx->n3, g5.ncols);
  }
  return DBFFT_OK;
}

// forward tail of the rhs: WB holds -sigma spectra (from an X pass) -> F2 -> F3 -> out
dbfft_status forward_tail(dbfft_ctx ctx, cplx* out) {
  const bool fin = ctx->kin == 9;
  ColGeom g4 = colgeom(ctx, false, ctx->WB, ctx->WA, true, false);
  CKS(run_col(ctx, fin ? COL_F2F : COL_F2S, PK_F2, g4));
  ColGeom g5 = colgeom(ctx, true, ctx->WA, out, false, false);
  CKS(run_col(ctx, fin ? COL_F3F : COL_F3S, PK_F3, g5));
  return DBFFT_OK;
}

dbfft_status read_reduction(dbfft_ctx ctx, const double* partials, int nblk, int nred, double* host_out) {
  {
    ProfScope ps(ctx, PK_FIN);
    CK(launch_reduce(partials, nblk, nred, ctx->red_out, ctx->stream));
  }
  CK(cudaMemcpyAsync(ctx->h_red, ctx->red_out, sizeof(double) * nred, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  memcpy(host_out, ctx->h_red, sizeof(double) * nred);
  return DBFFT_OK;
}

void sym_fill(double* m) {
  m[3] = m[1];
  m[6] = m[2];
  m[7] = m[5];
}

// mean tangent -> Cbar (full 81), prec coefficients
dbfft_status refresh_mean_tangent(dbfft_ctx ctx) {
  const int nk = ctx->kin == 9 ? 45 : 21;
  const int nblk = cg_blocks();
  {
    ProfScope ps(ctx, PK_OTHER);
    const int mode = (ctx->family == FAM_J2) ? 2 : (ctx->tmode ? 1 : 0);
    CK(launch_mean_tangent(mode, xgeom(ctx, nullptr, nullptr), ctx->part_misc, nblk, ctx->stream));
  }
  double m[64];
  CKS(read_reduction(ctx, ctx->part_misc, nblk, nk, m));
  for (int k = 0; k < nk; ++k) m[k] /= (double)ctx->N;
  if (ctx->kin == 9) {
    for (int a = 0; a < 9; ++a)
      for (int b = 0; b < 9; ++b) {
        const int i = std::min(a, b), j = std::max(a, b);
        ctx->Cbar[9 * a + b] = m[i * 9 - i * (i - 1) / 2 + (j - i)];
      }
  } else {
    double CV[36];
    for (int I = 0; I < 6; ++I)
      for (int J = 0; J < 6; ++J) {
        const int i = std::min(I, J), j = std::max(I, J);
        CV[6 * I + J] = m[i * 6 - i * (i - 1) / 2 + (j - i)];
      }
    voigt_to_full(CV, ctx->Cbar);
  }
  ctx->prec = make_prec(ctx->Cbar);
  ctx->prec_valid = true;
  return DBFFT_OK;
}

// ---------------------------------------------------------------- PCG
// Solves A {x | xe} = {b | be} with x0 = 0.  Requires cg->msig0, cg->be, cg->mask, Minv_e set.
dbfft_status pcg(dbfft_ctx ctx, const dbfft_opts& o, const uint8_t* mask, int* iters_out) {
  SpecGeom sg = spec(ctx);
  const int nb = cg_blocks();
  CgDev* cg = ctx->cg;
  const bool macro = ctx->h_cg->macro != 0;
  const double* e_p = macro ? cg->pe : nullptr;
  (void)mask;
  CK(cudaMemsetAsync(ctx->x, 0, sizeof(cplx) * 3 * ctx->Hs, ctx->stream));
  CK(cudaMemcpyAsync(ctx->r, ctx->b, sizeof(cplx) * 3 * ctx->Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  {
    ProfScope ps(ctx, PK_CGDIR);
    CK(launch_cg_init(sg, ctx->prec, ctx->r, ctx->p, ctx->part_cg, nb, ctx->stream));
  }
  {
    ProfScope ps(ctx, PK_FIN);
    CK(launch_fin_init(cg, ctx->part_cg, nb, ctx->stream));
  }
  const int every = std::max(1, o.check_every);
  int restarts = 0;
  for (;;) {
    // poll
    CK(cudaMemcpyAsync(ctx->h_cg, cg, sizeof(CgDev), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    prof_flush(ctx);
    if (ctx->h_cg->breakdown) {
      ctx->err = "PCG breakdown: <p,Kp> <= 0 or NaN";
      *iters_out = ctx->h_cg->iters;
      return DBFFT_E_BREAKDOWN;
    }
    if (ctx->h_cg->converged == 2 || ctx->h_cg->iters >= o.max_cg) {
      *iters_out = ctx->h_cg->iters;
      ctx->err = "PCG did not converge within max_cg";
      return DBFFT_E_NOT_CONVERGED;
    }
    if (ctx->h_cg->converged == 1) {
      // true-residual confirmation (R7): r = b - A x
      ApplyOut ao;
      CKS(apply_K_internal(ctx, ctx->x, ctx->q, macro ? cg->xe : nullptr, false, &ao));
      {
        ProfScope ps(ctx, PK_CGUPD);
        CK(launch_true_residual(sg, ctx->b, ctx->q, ctx->r, ctx->part_cg, nb, ctx->stream));
      }
      {
        ProfScope ps(ctx, PK_FIN);
        CK(launch_fin_true(cg, ctx->part_cg, nb, ctx->part_x, ao.grid_x, 10, ctx->stream));
      }
      CK(cudaMemcpyAsync(ctx->h_cg, cg, sizeof(CgDev), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (ctx->h_cg->converged == 1 || restarts > 20) {
        *iters_out = ctx->h_cg->iters;
        return DBFFT_OK;
      }
      // restart from the true residual: z = M r, p = z
      ++restarts;
      {
        ProfScope ps(ctx, PK_CGDIR);
        CK(launch_cg_init(sg, ctx->prec, ctx->r, ctx->p, ctx->part_cg, nb, ctx->stream));
      }
      {
        ProfScope ps(ctx, PK_FIN);
        CK(launch_fin_init(cg, ctx->part_cg, nb, ctx->stream));
      }
      continue;
    }
    for (int k = 0; k < every; ++k) {
      ApplyOut ao;
      CKS(apply_K_internal(ctx, ctx->p, ctx->q, e_p, true, &ao));
      {
        ProfScope ps(ctx, PK_FIN);
        CK(launch_fin_alpha(cg, ctx->part_f3, ao.grid_f3, ctx->part_x, ao.grid_x, 10, ctx->stream));
      }
      {
        ProfScope ps(ctx, PK_CGUPD);
        CK(launch_cg_update(sg, ctx->prec, cg, ctx->x, ctx->p, ctx->r, ctx->q, ctx->part_cg, nb, ctx->stream));
      }
      {
        ProfScope ps(ctx, PK_FIN);
        CK(launch_fin_beta(cg, ctx->part_cg, nb, ctx->stream));
      }
      {
        ProfScope ps(ctx, PK_CGDIR);
        CK(launch_cg_direction(sg, ctx->prec, cg, ctx->p, ctx->r, ctx->stream));
      }
    }
  }
}

// set CgDev header fields on the host mirror and upload
dbfft_status cg_setup(dbfft_ctx ctx, const dbfft_opts& o, const uint8_t* mask, const double* msig0, const double* be) {
  CgDev* h = ctx->h_cg;
  memset(h, 0, sizeof(CgDev));
  h->tol_eq = o.tol_eq;
  h->tol_load = o.tol_load;
  h->inv_n = 1.0 / (double)ctx->N;
  h->sym = ctx->kin == 6 ? 1 : 0;
  h->max_iter = o.max_cg;
  int anym = 0;
  for (int a = 0; a < 9; ++a) {
    h->mask[a] = mask[a] ? 1.0 : 0.0;
    anym |= mask[a];
    h->msig0[a] = h->msig[a] = msig0[a];
    h->be[a] = h->re[a] = be[a];
  }
  h->macro = anym;
  if (!macro_inverse(ctx->Cbar, mask, ctx->kin == 6, h->Minv_e)) {
    ctx->err = "singular macro block (P Cbar P)";
    return DBFFT_E_INVALID_ARG;
  }
  CK(cudaMemcpyAsync(ctx->cg, h, sizeof(CgDev), cudaMemcpyHostToDevice, ctx->stream));
  return DBFFT_OK;
}

dbfft_status check_target(dbfft_ctx ctx, const double* target, const uint8_t* mask) {
  if (!target || !mask) {
    ctx->err = "null target or mask";
    return DBFFT_E_INVALID_ARG;
  }
  if (ctx->kin == 6) {
    for (int i = 0; i < 3; ++i)
      for (int j = i + 1; j < 3; ++j)
        if (mask[3 * i + j] != mask[3 * j + i] || target[3 * i + j] != target[3 * j + i]) {
          ctx->err = "small-strain target and mask must be symmetric";
          return DBFFT_E_INVALID_ARG;
        }
  }
  return DBFFT_OK;
}

dbfft_status finish_report(dbfft_ctx ctx, dbfft_report* rep, std::chrono::steady_clock::time_point t0) {
  if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return DBFFT_OK;
}

// ---------------------------------------------------------------- linear solve
dbfft_status solve_linear(dbfft_ctx ctx, const double* target, const uint8_t* mask, const dbfft_opts& o, dbfft_report* rep) {
  double epsU[9], sigf[9];
  for (int a = 0; a < 9; ++a) {
    epsU[a] = mask[a] ? 0.0 : target[a];
    sigf[a] = mask[a] ? target[a] : 0.0;
  }
  CK(cudaMemcpyAsync(ctx->e_dev, epsU, sizeof(double) * 9, cudaMemcpyHostToDevice, ctx->stream));
  // rhs b = d:F(C:eps_U) (P:118 right-hand side, R3) and <C:eps_U>
  XGeom gx = xgeom(ctx, nullptr, ctx->WB);
  gx.e = ctx->e_dev;
  int gridx = 0;
  CKS(run_x(ctx, X_RHS_SMALL_PHASE, PK_XCONST, gx, &gridx));
  CKS(forward_tail(ctx, ctx->b));
  double red[10];
  CKS(read_reduction(ctx, ctx->part_x, gridx, 10, red));
  double msig0[9], be[9];
  for (int a = 0; a < 9; ++a) msig0[a] = red[a] / (double)ctx->N;
  sym_fill(msig0);
  for (int a = 0; a < 9; ++a) be[a] = mask[a] ? sigf[a] - msig0[a] : 0.0;
  CKS(cg_setup(ctx, o, mask, msig0, be));
  int iters = 0;
  dbfft_status st = pcg(ctx, o, mask, &iters);
  if (rep) {
    rep->cg_iters = iters;
    rep->newton_iters = 0;
    rep->converged = st == DBFFT_OK;
    rep->eps_eq = ctx->h_cg->eps_eq;
    rep->eps_load = ctx->h_cg->eps_load;
    rep->bad_voxel = -1;
    for (int a = 0; a < 9; ++a) {
      rep->macro_strain[a] = epsU[a] + ctx->h_cg->xe[a];
      rep->macro_stress[a] = ctx->h_cg->msig[a];
    }
  }
  if (st != DBFFT_OK) return st;
  CK(cudaMemcpyAsync(ctx->u, ctx->x, sizeof(cplx) * 3 * ctx->Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->u_c, ctx->x, sizeof(cplx) * 3 * ctx->Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  for (int a = 0; a < 9; ++a) ctx->Fbar[a] = ctx->Fbar_c[a] = epsU[a] + ctx->h_cg->xe[a];
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

// ---------------------------------------------------------------- Newton
// constitutive pass: state += grad(du) + dF ; P, K ; b = F(div P) ; returns <P>, max|d|
dbfft_status constitutive(dbfft_ctx ctx, bool has_in, const double* dF_host, double dt, double* meanP, double* maxd) {
  const bool fin = ctx->kin == 9;
  CK(cudaMemcpyAsync(ctx->e_dev, dF_host, sizeof(double) * 9, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->bad, 0x7f, sizeof(int), ctx->stream));
  if (has_in) {
    ColGeom g1 = colgeom(ctx, true, ctx->x, ctx->WA, false, false);
    CKS(run_col(ctx, fin ? COL_I1F : COL_I1S, PK_I1, g1));
    ColGeom g2 = colgeom(ctx, false, ctx->WA, ctx->WB, false, true);
    CKS(run_col(ctx, fin ? COL_I2F : COL_I2S, PK_I2, g2));
  }
  XGeom gx = xgeom(ctx, ctx->WB, ctx->WB);
  gx.e = ctx->e_dev;
  gx.has_in = has_in ? 1 : 0;
  gx.dt = dt;
  int gridx = 0;
  CKS(run_x(ctx, fin ? X_CONST_FIN : X_CONST_J2, PK_XCONST, gx, &gridx));
  CKS(forward_tail(ctx, ctx->b));
  double red[10];
  CKS(read_reduction(ctx, ctx->part_x, gridx, 10, red));
  for (int a = 0; a < 9; ++a) meanP[a] = red[a] / (double)ctx->N;
  if (!fin) sym_fill(meanP);
  *maxd = red[9];
  CK(cudaMemcpy(ctx->h_bad, ctx->bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (*ctx->h_bad != 0x7f7f7f7f) {
    ctx->err = "det F <= 0 at voxel " + std::to_string(*ctx->h_bad);
    return DBFFT_E_MATERIAL;
  }
  ctx->tangent_valid = true;
  return DBFFT_OK;
}

dbfft_status rollback(dbfft_ctx ctx) {
  const int nf = ctx->kin == 9 ? 9 : 6;
  CK(cudaMemcpyAsync(ctx->u, ctx->u_c, sizeof(cplx) * 3 * ctx->Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->F, ctx->F_c, sizeof(double) * nf * ctx->N, cudaMemcpyDeviceToDevice, ctx->stream));
  memcpy(ctx->Fbar, ctx->Fbar_c, sizeof(ctx->Fbar));
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status solve_newton(dbfft_ctx ctx, const double* target, const uint8_t* mask, double dt, const dbfft_opts& o,
                          dbfft_report* rep) {
  const bool fin = ctx->kin == 9;
  const int nf = fin ? 9 : 6;
  // start from the committed state
  CK(cudaMemcpyAsync(ctx->u, ctx->u_c, sizeof(cplx) * 3 * ctx->Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->F, ctx->F_c, sizeof(double) * nf * ctx->N, cudaMemcpyDeviceToDevice, ctx->stream));
  double Fbar_new[9], dF[9], Pf[9];
  for (int a = 0; a < 9; ++a) {
    Fbar_new[a] = mask[a] ? ctx->Fbar_c[a] : target[a];   // F^0 = Fbar^{k+1} + grad u^k
    dF[a] = Fbar_new[a] - ctx->Fbar_c[a];
    Pf[a] = mask[a] ? target[a] : 0.0;
  }
  memcpy(ctx->Fbar, Fbar_new, sizeof(Fbar_new));
  double meanP[9], maxd = 0.0;
  dbfft_status st = constitutive(ctx, false, dF, dt, meanP, &maxd);
  int total_cg = 0, newton = 0;
  double last = 0.0;
  bool conv = false;
  while (st == DBFFT_OK) {
    if (newton == 0 || o.precond_refresh) {
      st = refresh_mean_tangent(ctx);
      if (st != DBFFT_OK) break;
    }
    double be[9];
    for (int a = 0; a < 9; ++a) be[a] = mask[a] ? Pf[a] - meanP[a] : 0.0;
    st = cg_setup(ctx, o, mask, meanP, be);
    if (st != DBFFT_OK) break;
    int iters = 0;
    st = pcg(ctx, o, mask, &iters);
    total_cg += iters;
    if (st != DBFFT_OK) break;
    // u += du ; Fbar_f += dF_f
    {
      ProfScope ps(ctx, PK_OTHER);
      CK(launch_axpy(spec(ctx), ctx->u, ctx->x, 1.0, ctx->stream));
    }
    double de[9];
    for (int a = 0; a < 9; ++a) {
      de[a] = mask[a] ? ctx->h_cg->xe[a] : 0.0;
      ctx->Fbar[a] += de[a];
    }
    st = constitutive(ctx, true, de, dt, meanP, &maxd);
    ++newton;
    last = maxd;
    if (st != DBFFT_OK) break;
    if (maxd < o.tol_newton) {
      conv = true;
      break;
    }
    if (newton >= o.max_newton) {
      st = DBFFT_E_NOT_CONVERGED;
      ctx->err = "Newton did not converge within max_newton";
      break;
    }
  }
  if (rep) {
    rep->cg_iters = total_cg;
    rep->newton_iters = newton;
    rep->converged = conv;
    rep->eps_eq = ctx->h_cg->eps_eq;
    rep->eps_load = ctx->h_cg->eps_load;
    rep->max_dgrad = last;
    rep->bad_voxel = (st == DBFFT_E_MATERIAL) ? (int64_t)*ctx->h_bad : -1;
    for (int a = 0; a < 9; ++a) {
      rep->macro_strain[a] = ctx->Fbar[a];
      rep->macro_stress[a] = meanP[a];
    }
  }
  if (st != DBFFT_OK) {
    rollback(ctx);
    return st;
  }
  // commit (state accepted)
  CK(cudaMemcpyAsync(ctx->u_c, ctx->u, sizeof(cplx) * 3 * ctx->Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->F_c, ctx->F, sizeof(double) * nf * ctx->N, cudaMemcpyDeviceToDevice, ctx->stream));
  if (!fin) CK(cudaMemcpyAsync(ctx->epsp_c, ctx->epsp_t, sizeof(double) * 6 * ctx->N, cudaMemcpyDeviceToDevice, ctx->stream));
  memcpy(ctx->Fbar_c, ctx->Fbar, sizeof(ctx->Fbar));
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

void free_all(dbfft_ctx ctx) {
  void* ptrs[] = {ctx->xix, ctx->xiy, ctx->xiz, ctx->tw1, ctx->tw2, ctx->tw3, ctx->x, ctx->r, ctx->p, ctx->q, ctx->b, ctx->u,
                  ctx->u_c, ctx->WA, ctx->WB, ctx->phase, ctx->ptable, ctx->F, ctx->F_c, ctx->epsp_c, ctx->epsp_t, ctx->tan,
                  ctx->cg, ctx->part_x, ctx->part_f3, ctx->part_cg, ctx->part_misc, ctx->red_out, ctx->e_dev, ctx->bad,
                  ctx->counts, ctx->tmp_real};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ctx->h_cg) cudaFreeHost(ctx->h_cg);
  if (ctx->h_red) cudaFreeHost(ctx->h_red);
  if (ctx->h_bad) cudaFreeHost(ctx->h_bad);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
}

dbfft_status free_state(dbfft_ctx ctx) {
  void** ptrs[] = {(void**)&ctx->F, (void**)&ctx->F_c, (void**)&ctx->epsp_c, (void**)&ctx->epsp_t, (void**)&ctx->tan};
  for (void** p : ptrs)
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
  return DBFFT_OK;
}

// real-field [9][N] temporary for outputs
dbfft_status ensure_tmp(dbfft_ctx ctx) {
  if (!ctx->tmp_real) CKS(dalloc(ctx, &ctx->tmp_real, 9 * ctx->N));
  return DBFFT_OK;
}

}  // namespace

// =================================================================================================
// C ABI
// =================================================================================================
extern "C" {

dbfft_opts dbfft_default_opts(void) {
  dbfft_opts o;
  o.tol_eq = 1e-10;
  o.tol_load = 1e-10;
  o.tol_newton = 1e-6;
  o.max_cg = 10000;
  o.max_newton = 25;
  o.check_every = 4;
  o.precond_refresh = 0;
  return o;
}

const char* dbfft_last_error(dbfft_ctx ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

dbfft_status dbfft_create(const int32_t n[3], const double L[3], int32_t kinematics, const dbfft_env* env, dbfft_ctx* out) {
  if (!n || !L || !out) {
    g_create_error = "null argument";
    return DBFFT_E_INVALID_ARG;
  }
  *out = nullptr;
  for (int a = 0; a < 3; ++a)
    if (!is_pow2_in(n[a]) || !(L[a] > 0)) {
      g_create_error = "grid dims must be powers of two in [8,512] and L > 0";
      return DBFFT_E_INVALID_GRID;
    }
  if (kinematics != 6 && kinematics != 9) {
    g_create_error = "kinematics must be 6 (small strain) or 9 (finite strain)";
    return DBFFT_E_INVALID_ARG;
  }
  if (env && env->world != 1) {
    g_create_error = "world > 1 not supported in this build (slab decomposition reserved)";
    return DBFFT_E_INVALID_ARG;
  }
  dbfft_ctx ctx = new dbfft_ctx_s();
  ctx->n1 = n[0];
  ctx->n2 = n[1];
  ctx->n3 = n[2];
  ctx->n1h = n[0] / 2 + 1;
  for (int a = 0; a < 3; ++a) ctx->L[a] = L[a];
  ctx->kin = kinematics;
  ctx->N = (long long)n[0] * n[1] * n[2];
  ctx->Hs = (long long)ctx->n1h * n[1] * n[2];
  memset(ctx->prof_ms, 0, sizeof(ctx->prof_ms));
  memset(ctx->prof_n, 0, sizeof(ctx->prof_n));
  for (int a = 0; a < 9; ++a) ctx->Fbar[a] = ctx->Fbar_c[a] = 0.0;
  auto fail = [&](dbfft_status s) {
    g_create_error = ctx->err;
    free_all(ctx);
    delete ctx;
    return s;
  };
  int dev = (env && env->device >= 0) ? env->device : -1;
  if (dev >= 0) {
    cudaError_t e = cudaSetDevice(dev);
    if (e != cudaSuccess) {
      ctx->err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
      return fail(DBFFT_E_CUDA);
    }
  }
  cudaGetDevice(&ctx->device);
  if (env && env->cuda_stream) {
    ctx->stream = (cudaStream_t)env->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      ctx->err = "cudaStreamCreate failed (no CUDA device?)";
      return fail(DBFFT_E_CUDA);
    }
    ctx->own_stream = true;
  }
  dbfft_status s;
  // frequency tables and twiddles
  std::vector<double> hx = axis_xi(ctx->n1, L[0], ctx->n1h), hy = axis_xi(ctx->n2, L[1], ctx->n2), hz = axis_xi(ctx->n3, L[2], ctx->n3);
  if ((s = dalloc(ctx, &ctx->xix, hx.size())) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->xiy, hy.size())) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->xiz, hz.size())) != DBFFT_OK) return fail(s);
  cudaMemcpy(ctx->xix, hx.data(), sizeof(double) * hx.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(ctx->xiy, hy.data(), sizeof(double) * hy.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(ctx->xiz, hz.data(), sizeof(double) * hz.size(), cudaMemcpyHostToDevice);
  if ((s = make_twiddles(ctx, ctx->n1, &ctx->tw1)) != DBFFT_OK) return fail(s);
  if ((s = make_twiddles(ctx, ctx->n2, &ctx->tw2)) != DBFFT_OK) return fail(s);
  if ((s = make_twiddles(ctx, ctx->n3, &ctx->tw3)) != DBFFT_OK) return fail(s);
  const size_t v3 = 3 * ctx->Hs;
  cplx** vecs[] = {&ctx->x, &ctx->r, &ctx->p, &ctx->q, &ctx->b, &ctx->u, &ctx->u_c};
  for (cplx** v : vecs)
    if ((s = dalloc(ctx, v, v3)) != DBFFT_OK) return fail(s);
  const int c = kinematics;
  if ((s = dalloc(ctx, &ctx->WA, (size_t)6 * ctx->Hs)) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->WB, (size_t)c * ctx->Hs)) != DBFFT_OK) return fail(s);
  cudaMemset(ctx->u, 0, sizeof(cplx) * v3);
  cudaMemset(ctx->u_c, 0, sizeof(cplx) * v3);
  if ((s = dalloc(ctx, &ctx->cg, 1)) != DBFFT_OK) return fail(s);
  // partial buffers
  const long long nlines = (long long)ctx->n2 * ctx->n3;
  int gx = 0;
  for (int k = 0; k < X_REAL_OUT; ++k) gx = std::max(gx, x_grid(k, ctx->n1, nlines));
  if ((s = dalloc(ctx, &ctx->part_x, (size_t)gx * 10)) != DBFFT_OK) return fail(s);
  const int gf3 = col_grid(ctx->n3, (long long)ctx->n2 * ctx->n1h);
  if ((s = dalloc(ctx, &ctx->part_f3, (size_t)gf3)) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->part_cg, (size_t)cg_blocks() * 2)) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->part_misc, (size_t)cg_blocks() * 45)) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->red_out, 64)) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->e_dev, 9)) != DBFFT_OK) return fail(s);
  if ((s = dalloc(ctx, &ctx->bad, 1)) != DBFFT_OK) return fail(s);
  if (cudaMallocHost(&ctx->h_cg, sizeof(CgDev)) != cudaSuccess || cudaMallocHost(&ctx->h_red, 64 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_bad, sizeof(int)) != cudaSuccess) {
    ctx->err = "cudaMallocHost failed";
    return fail(DBFFT_E_OOM);
  }
  memset(ctx->h_cg, 0, sizeof(CgDev));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    ctx->err = std::string("create: ") + cudaGetErrorString(e);
    return fail(DBFFT_E_CUDA);
  }
  *out = ctx;
  return DBFFT_OK;
}

dbfft_status dbfft_destroy(dbfft_ctx ctx) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_all(ctx);
  delete ctx;
  return DBFFT_OK;
}

dbfft_status dbfft_spectral_layout(dbfft_ctx ctx, int64_t shape[4], int64_t strides[4]) {
  if (!ctx || !shape || !strides) return DBFFT_E_INVALID_ARG;
  shape[0] = 3;
  shape[1] = ctx->n2;
  shape[2] = ctx->n3;
  shape[3] = ctx->n1h;
  strides[3] = 1;
  strides[2] = ctx->n1h;
  strides[1] = (int64_t)ctx->n3 * ctx->n1h;
  strides[0] = ctx->Hs;
  return DBFFT_OK;
}

dbfft_status dbfft_set_phases(dbfft_ctx ctx, const uint16_t* phase_id, int32_t on_device, int32_t n_phases, const dbfft_material* table) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (!phase_id || !table || n_phases <= 0 || n_phases > 65535) {
    ctx->err = "set_phases: bad arguments";
    return DBFFT_E_INVALID_ARG;
  }
  int fam = FAM_NONE;
  std::vector<double> pt(36 * (size_t)n_phases, 0.0);
  for (int k = 0; k < n_phases; ++k) {
    const dbfft_material& m = table[k];
    int f;
    double* d = pt.data() + 36 * k;
    switch (m.kind) {
      case DBFFT_MAT_ISO:
        if (!(m.p[0] > 0) || !(m.p[1] > -1.0 && m.p[1] < 0.5)) { ctx->err = "ISO: need E > 0, -1 < nu < 0.5"; return DBFFT_E_INVALID_ARG; }
        iso_voigt(m.p[0], m.p[1], d);
        f = FAM_LINEAR;
        break;
      case DBFFT_MAT_CUBIC:
        cubic_voigt(m.p[0], m.p[1], m.p[2], m.p + 3, d);
        f = FAM_LINEAR;
        break;
      case DBFFT_MAT_NEOHOOKE:
        if (!(m.p[0] > 0) || !(m.p[1] > 2.0 * m.p[0] / 3.0 - 1e300)) { ctx->err = "NEOHOOKE: need mu > 0"; return DBFFT_E_INVALID_ARG; }
        d[0] = m.p[0];
        d[1] = m.p[1];
        f = FAM_NEOHOOKE;
        break;
      case DBFFT_MAT_J2:
        if (!(m.p[0] > 0) || !(m.p[1] > -1.0 && m.p[1] < 0.5) || !(m.p[2] > 0) || !(m.p[3] > 0) || !(m.p[4] > 0)) {
          ctx->err = "J2: need E > 0, -1 < nu < 0.5, sigma_y, n, edot0 > 0";
          return DBFFT_E_INVALID_ARG;
        }
        for (int a = 0; a < 5; ++a) d[a] = m.p[a];
        f = FAM_J2;
        break;
      default:
        ctx->err = "unknown material kind";
        return DBFFT_E_INVALID_ARG;
    }
    if (fam != FAM_NONE && fam != f) {
      ctx->err = "all phases must belong to one material family";
      return DBFFT_E_INVALID_ARG;
    }
    fam = f;
  }
  if ((fam == FAM_NEOHOOKE) != (ctx->kin == 9)) {
    ctx->err = "NEOHOOKE requires a finite-strain context; ISO/CUBIC/J2 a small-strain one";
    return DBFFT_E_INVALID_ARG;
  }
  dbfft_status s;
  if (!ctx->phase && (s = dalloc(ctx, &ctx->phase, ctx->N)) != DBFFT_OK) return s;
  CK(cudaMemcpyAsync(ctx->phase, phase_id, sizeof(uint16_t) * ctx->N, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     ctx->stream));
  if (ctx->ptable) cudaFree(ctx->ptable);
  ctx->ptable = nullptr;
  if ((s = dalloc(ctx, &ctx->ptable, pt.size())) != DBFFT_OK) return s;
  CK(cudaMemcpyAsync(ctx->ptable, pt.data(), sizeof(double) * pt.size(), cudaMemcpyHostToDevice, ctx->stream));
  ctx->h_ptable = pt;
  ctx->nph = n_phases;
  // validate ids and count phases (for the linear mean stiffness)
  if (ctx->counts) cudaFree(ctx->counts);
  ctx->counts = nullptr;
  if ((s = dalloc(ctx, &ctx->counts, n_phases)) != DBFFT_OK) return s;
  CK(cudaMemsetAsync(ctx->counts, 0, sizeof(unsigned long long) * n_phases, ctx->stream));
  CK(cudaMemsetAsync(ctx->bad, 0, sizeof(int), ctx->stream));
  CK(launch_phase_hist(ctx->phase, ctx->N, ctx->counts, n_phases, ctx->bad, ctx->stream));
  std::vector<unsigned long long> cnt(n_phases);
  CK(cudaMemcpyAsync(cnt.data(), ctx->counts, sizeof(unsigned long long) * n_phases, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ctx->h_bad, ctx->bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (*ctx->h_bad) {
    ctx->err = "phase id >= n_phases";
    return DBFFT_E_INVALID_ARG;
  }
  ctx->family = fam;
  // state
  free_state(ctx);
  CK(cudaMemsetAsync(ctx->u, 0, sizeof(cplx) * 3 * ctx->Hs, ctx->stream));
  CK(cudaMemsetAsync(ctx->u_c, 0, sizeof(cplx) * 3 * ctx->Hs, ctx->stream));
  for (int a = 0; a < 9; ++a) ctx->Fbar[a] = ctx->Fbar_c[a] = (fam == FAM_NEOHOOKE && a % 4 == 0) ? 1.0 : 0.0;
  ctx->tangent_valid = false;
  if (fam == FAM_LINEAR) {
    double CV[36] = {0};
    for (int k = 0; k < n_phases; ++k)
      for (int a = 0; a < 36; ++a) CV[a] += (double)cnt[k] * pt[36 * k + a];
    for (int a = 0; a < 36; ++a) CV[a] /= (double)ctx->N;
    voigt_to_full(CV, ctx->Cbar);
    ctx->prec = make_prec(ctx->Cbar);
    ctx->prec_valid = true;
  } else {
    const int nf = fam == FAM_NEOHOOKE ? 9 : 6;
    const char* tm = getenv("DBFFT_TANGENT");
    ctx->tmode = (tm && strcmp(tm, "full") == 0) ? 0 : 1;
    const int nk = fam == FAM_NEOHOOKE ? (ctx->tmode ? 10 : 45) : 8;
    if ((s = dalloc(ctx, &ctx->F, (size_t)nf * ctx->N)) != DBFFT_OK) return s;
    if ((s = dalloc(ctx, &ctx->F_c, (size_t)nf * ctx->N)) != DBFFT_OK) return s;
    if ((s = dalloc(ctx, &ctx->tan, (size_t)nk * ctx->N)) != DBFFT_OK) return s;
    if (fam == FAM_NEOHOOKE) {
      k_identity9<<<1024, 256, 0, ctx->stream>>>(ctx->F_c, ctx->N);
    } else {
      CK(cudaMemsetAsync(ctx->F_c, 0, sizeof(double) * nf * ctx->N, ctx->stream));
      if ((s = dalloc(ctx, &ctx->epsp_c, (size_t)6 * ctx->N)) != DBFFT_OK) return s;
      if ((s = dalloc(ctx, &ctx->epsp_t, (size_t)6 * ctx->N)) != DBFFT_OK) return s;
      CK(cudaMemsetAsync(ctx->epsp_c, 0, sizeof(double) * 6 * ctx->N, ctx->stream));
      CK(cudaMemsetAsync(ctx->epsp_t, 0, sizeof(double) * 6 * ctx->N, ctx->stream));
    }
    CK(cudaMemcpyAsync(ctx->F, ctx->F_c, sizeof(double) * nf * ctx->N, cudaMemcpyDeviceToDevice, ctx->stream));
    // tangent at the undeformed state (so apply_K / precond are usable before a solve)
    double zero[9] = {0}, mp[9], mx;
    s = constitutive(ctx, false, zero, 1.0, mp, &mx);
    if (s != DBFFT_OK) return s;
    s = refresh_mean_tangent(ctx);
    if (s != DBFFT_OK) return s;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status dbfft_apply_K(dbfft_ctx ctx, const void* u_hat, void* f_hat) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (!u_hat || !f_hat || u_hat == f_hat) {
    ctx->err = "apply_K: null or aliased vectors";
    return DBFFT_E_INVALID_ARG;
  }
  if (ctx->family == FAM_NONE) {
    ctx->err = "apply_K before set_phases";
    return DBFFT_E_STATE;
  }
  return apply_K_internal(ctx, (const cplx*)u_hat, (cplx*)f_hat, nullptr, false, nullptr);
}

dbfft_status dbfft_apply_K_aug(dbfft_ctx ctx, const uint8_t mask[9], const void* u_hat, const double e_in[9], void* f_hat, double r_out[9]) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (!mask || !u_hat || !e_in || !f_hat || !r_out || u_hat == f_hat) {
    ctx->err = "apply_K_aug: bad arguments";
    return DBFFT_E_INVALID_ARG;
  }
  if (ctx->family == FAM_NONE) {
    ctx->err = "apply_K_aug before set_phases";
    return DBFFT_E_STATE;
  }
  double e[9];
  for (int a = 0; a < 9; ++a) e[a] = mask[a] ? e_in[a] : 0.0;
  CK(cudaMemcpyAsync(ctx->e_dev, e, sizeof(e), cudaMemcpyHostToDevice, ctx->stream));
  ApplyOut ao;
  CKS(apply_K_internal(ctx, (const cplx*)u_hat, (cplx*)f_hat, ctx->e_dev, false, &ao));
  double red[10];
  CKS(read_reduction(ctx, ctx->part_x, ao.grid_x, 10, red));
  for (int a = 0; a < 9; ++a) red[a] /= (double)ctx->N;
  if (ctx->kin == 6) sym_fill(red);
  for (int a = 0; a < 9; ++a) r_out[a] = mask[a] ? red[a] : 0.0;
  return DBFFT_OK;
}

dbfft_status dbfft_precond(dbfft_ctx ctx, const void* r_hat, void* z_hat) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (!r_hat || !z_hat) {
    ctx->err = "precond: null vectors";
    return DBFFT_E_INVALID_ARG;
  }
  if (!ctx->prec_valid) {
    ctx->err = "precond before set_phases";
    return DBFFT_E_STATE;
  }
  ProfScope ps(ctx, PK_OTHER);
  CK(launch_precond(spec(ctx), ctx->prec, (const cplx*)r_hat, (cplx*)z_hat, ctx->stream));
  return DBFFT_OK;
}

dbfft_status dbfft_eval_state(dbfft_ctx ctx, const double* field, int32_t on_device, double dt) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (ctx->family == FAM_NONE) {
    ctx->err = "eval_state before set_phases";
    return DBFFT_E_STATE;
  }
  if (ctx->family == FAM_LINEAR) return DBFFT_OK;
  if (!field) {
    ctx->err = "eval_state: null field";
    return DBFFT_E_INVALID_ARG;
  }
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (ctx->family == FAM_NEOHOOKE) {
    CK(cudaMemcpyAsync(ctx->F, field, sizeof(double) * 9 * ctx->N, kind, ctx->stream));
  } else {
    const int rowv[6] = {0, 4, 8, 5, 2, 1};
    for (int I = 0; I < 6; ++I)
      CK(cudaMemcpyAsync(ctx->F + (size_t)I * ctx->N, field + (size_t)rowv[I] * ctx->N, sizeof(double) * ctx->N, kind, ctx->stream));
  }
  double zero[9] = {0}, mp[9], mx;
  CKS(constitutive(ctx, false, zero, dt, mp, &mx));
  CKS(refresh_mean_tangent(ctx));
  return DBFFT_OK;
}

dbfft_status dbfft_solve_increment(dbfft_ctx ctx, const double target[9], const uint8_t mask[9], double dt, const dbfft_opts* opts,
                                   dbfft_report* report) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (ctx->family == FAM_NONE) {
    ctx->err = "solve_increment before set_phases";
    return DBFFT_E_STATE;
  }
  CKS(check_target(ctx, target, mask));
  dbfft_opts o = opts ? *opts : dbfft_default_opts();
  auto t0 = std::chrono::steady_clock::now();
  if (report) {
    memset(report, 0, sizeof(*report));
    report->bad_voxel = -1;
  }
  dbfft_status st = (ctx->family == FAM_LINEAR) ? solve_linear(ctx, target, mask, o, report) : solve_newton(ctx, target, mask, dt, o, report);
  prof_flush(ctx);
  if (report) report->status = st;
  finish_report(ctx, report, t0);
  return st;
}

dbfft_status dbfft_get_field(dbfft_ctx ctx, int32_t which, void* out, int32_t out_on_device) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  if (!out) {
    ctx->err = "get_field: null output";
    return DBFFT_E_INVALID_ARG;
  }
  if (ctx->family == FAM_NONE) {
    ctx->err = "get_field before set_phases";
    return DBFFT_E_STATE;
  }
  const cudaMemcpyKind k = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const long long N = ctx->N;
  CKS(ensure_tmp(ctx));
  switch (which) {
    case DBFFT_FIELD_U_HAT:
      CK(cudaMemcpyAsync(out, ctx->u_c, sizeof(cplx) * 3 * ctx->Hs, k, ctx->stream));
      break;
    case DBFFT_FIELD_U: {
      ColGeom g1 = colgeom(ctx, true, ctx->u_c, ctx->WA, false, false);
      CKS(run_col(ctx, COL_ZI3, PK_OTHER, g1));
      ColGeom g2 = colgeom(ctx, false, ctx->WA, ctx->WB, false, true);
      CKS(run_col(ctx, COL_YI3, PK_OTHER, g2));
      XGeom gx = xgeom(ctx, ctx->WB, nullptr);
      gx.real_out = ctx->tmp_real;
      CKS(run_x(ctx, X_REAL_OUT + 3, PK_OTHER, gx, nullptr));
      CK(cudaMemcpyAsync(out, ctx->tmp_real, sizeof(double) * 3 * N, k, ctx->stream));
      break;
    }
    case DBFFT_FIELD_STRAIN:
    case DBFFT_FIELD_STRESS: {
      double* strain9 = ctx->tmp_real;
      double* dst = (which == DBFFT_FIELD_STRAIN) ? strain9 : nullptr;
      double* tmp6 = nullptr;
      if (ctx->family == FAM_NEOHOOKE) {
        if (which == DBFFT_FIELD_STRAIN) {
          CK(cudaMemcpyAsync(out, ctx->F_c, sizeof(double) * 9 * N, k, ctx->stream));
        } else {
          k_stress_nh<<<1024, 256, 0, ctx->stream>>>(ctx->F_c, ctx->phase, ctx->ptable, N, ctx->tmp_real);
          CK(cudaGetLastError());
          CK(cudaMemcpyAsync(out, ctx->tmp_real, sizeof(double) * 9 * N, k, ctx->stream));
        }
        break;
      }
      if (ctx->family == FAM_J2) {
        if (which == DBFFT_FIELD_STRAIN) {
          k_expand6<<<1024, 256, 0, ctx->stream>>>(ctx->F_c, N, nullptr, ctx->tmp_real);
        } else {
          k_stress_j2<<<1024, 256, 0, ctx->stream>>>(ctx->F_c, ctx->epsp_c, ctx->phase, ctx->ptable, N, ctx->tmp_real);
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, ctx->tmp_real, sizeof(double) * 9 * N, k, ctx->stream));
        break;
      }
      // linear: eps = Ebar + sym grad u (Voigt 6 via the inverse passes), sigma = C:eps
      CKS(dalloc(ctx, &tmp6, 6 * N));
      ColGeom g1 = colgeom(ctx, true, ctx->u_c, ctx->WA, false, false);
      CKS(run_col(ctx, COL_I1S, PK_OTHER, g1));
      ColGeom g2 = colgeom(ctx, false, ctx->WA, ctx->WB, false, true);
      CKS(run_col(ctx, COL_I2S, PK_OTHER, g2));
      XGeom gx = xgeom(ctx, ctx->WB, nullptr);
      gx.real_out = tmp6;
      CKS(run_x(ctx, X_REAL_OUT + 6, PK_OTHER, gx, nullptr));
      CK(cudaMemcpyAsync(ctx->e_dev, ctx->Fbar_c, sizeof(double) * 9, cudaMemcpyHostToDevice, ctx->stream));
      k_expand6<<<1024, 256, 0, ctx->stream>>>(tmp6, N, ctx->e_dev, strain9);
      CK(cudaGetLastError());
      (void)dst;
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(tmp6);
      if (which == DBFFT_FIELD_STRAIN) {
        CK(cudaMemcpyAsync(out, strain9, sizeof(double) * 9 * N, k, ctx->stream));
      } else {
        double* sig = nullptr;
        CKS(dalloc(ctx, &sig, 9 * N));
        k_stress_linear<<<1024, 256, 0, ctx->stream>>>(strain9, ctx->phase, ctx->ptable, N, sig);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, sig, sizeof(double) * 9 * N, k, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        cudaFree(sig);
      }
      break;
    }
    default:
      ctx->err = "get_field: unknown field";
      return DBFFT_E_INVALID_ARG;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status dbfft_profile_enable(dbfft_ctx ctx, int32_t enable) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  prof_flush(ctx);
  ctx->prof = enable != 0;
  if (enable) {
    memset(ctx->prof_ms, 0, sizeof(ctx->prof_ms));
    memset(ctx->prof_n, 0, sizeof(ctx->prof_n));
  }
  return DBFFT_OK;
}

dbfft_status dbfft_profile_read(dbfft_ctx ctx, int32_t id, double* total_ms, int64_t* launches) {
  if (!ctx || id < 0 || id >= PK_COUNT) return DBFFT_E_INVALID_ARG;
  prof_flush(ctx);
  if (total_ms) *total_ms = ctx->prof_ms[id];
  if (launches) *launches = ctx->prof_n[id];
  return DBFFT_OK;
}

dbfft_status dbfft_launch_count(dbfft_ctx ctx, int64_t* count) {
  if (!ctx || !count) return DBFFT_E_INVALID_ARG;
  *count = ctx->nlaunch;
  return DBFFT_OK;
}

const char* dbfft_profile_name(int32_t id) { return (id >= 0 && id < PK_COUNT) ? kProfNames[id] : ""; }
int32_t dbfft_profile_count(void) { return PK_COUNT; }

}  // extern "C"
