// cg.cuh — device-resident PCG state and launchers (cg.cu).
#pragma once
#include "common.cuh"
#include "passes.cuh"

// Scalars of the preconditioned CG on the augmented system {u_hat | e}, kept
// on the device so an iteration needs no host round trip; the host polls `converged`.
struct CgDev {
  double rz, pq, alpha, beta, rr, rz_new;
  double eps_eq, eps_load;
  double tol_eq, tol_load;
  double inv_n;
  double xe[9], re[9], pe[9], qe[9], ze[9], be[9];
  double msig[9];      // tracked <sigma> of the current iterate (R7)
  double msig0[9];     // <sigma> at x = 0
  double dc[9];        // <sigma(p)> of the latest operator application
  double mask[9];      // 1 = stress controlled
  double Minv_e[81];   // (P Cbar P)^-1 on the stress-controlled subspace (R4), 9x9 row-major
  int converged, breakdown, iters, sym, macro, max_iter;
  int xphase;  // 1 between k_fin_alpha and k_fin_x: the direction kernel still owes x += alpha p
  int trace_cap;   // entries available at trace (0: no trace)
  double* trace;   // per-iteration (eps_eq, eps_load) of this PCG call: [0] initial, [k] after k
};

// spectral-point preconditioner coefficients: A_m(xi) = sum_p Q[m][p] q_p(xi),
// m over (xx,yy,zz,yz,xz,xy) of A = xi.Cbar.xi, q = (x x, y y, z z, y z, x z, x y) products.
struct PrecQ { double Q[36]; };

struct SpecGeom {
  int n1h, n2, n3;
  long long Hs;         // points per component
  Freq fq;              // xy already offset to the local ky slab (xx to the local kx block)
  int n1;
  int kx0;              // global kx of local column 0 (pencil decomposition; else 0)
};

cudaError_t launch_precond(const SpecGeom& g, const PrecQ* q, const cplx* r, cplx* z, cudaStream_t s);
cudaError_t launch_cg_init(const SpecGeom& g, const PrecQ* q, const cplx* r, cplx* p, double* partials, int nblk, cudaStream_t s);
cudaError_t launch_cg_update(const SpecGeom& g, const PrecQ* q, CgDev* cg, cplx* r, const cplx* qv,
                             double* partials, int nblk, cudaStream_t s);
cudaError_t launch_cg_direction(const SpecGeom& g, const PrecQ* q, const CgDev* cg, cplx* x, cplx* p, const cplx* r, cudaStream_t s,
                                int x_done = 0);
cudaError_t launch_cg_xupdate(const SpecGeom& g, const CgDev* cg, cplx* x, const cplx* p, int ctas_per_sm, cudaStream_t s);
// cond/set_cond: inside the device-side PCG loop (CUDA graph WHILE node) k_fin_x also sets the
// loop condition to "not converged and no breakdown"
cudaError_t launch_fin_x(CgDev* cg, cudaStream_t s, cudaGraphConditionalHandle cond = 0, int set_cond = 0);
cudaError_t launch_loop_cond(const CgDev* cg, cudaGraphConditionalHandle cond, cudaStream_t s);
cudaError_t launch_fin_init(CgDev* cg, const double* loc, cudaStream_t s);
cudaError_t launch_fin_alpha(CgDev* cg, const double* loc, cudaStream_t s);
cudaError_t launch_fin_beta(CgDev* cg, const double* loc, cudaStream_t s);
// one rank: CTA partials -> loc (x-pass slots 1..10 / CG slots 0..1) and the finalizer in one launch
cudaError_t launch_reduce_alpha(const double* partials, int nblk, double* loc, CgDev* cg, cudaStream_t s);
cudaError_t launch_reduce_beta(const double* partials, int nblk, double* loc, CgDev* cg, cudaStream_t s);
cudaError_t launch_true_residual(const SpecGeom& g, const cplx* b, const cplx* Ax, cplx* r, double* partials, int nblk, cudaStream_t s);
cudaError_t launch_fin_true(CgDev* cg, const double* loc, cudaStream_t s);
cudaError_t launch_allreduce_lb(double* const* v, int off, int P, int k, int is_max, cudaStream_t s);
cudaError_t launch_axpy(const SpecGeom& g, cplx* y, const cplx* x, double a, cudaStream_t s);
// out[k] = sum_j partials[j nred + k] (max over j for k == max_slot)
cudaError_t launch_reduce(const double* partials, int nblk, int nred, double* out, cudaStream_t s, int max_slot = -1);
cudaError_t launch_phase_hist(const uint16_t* ph, long long nvox, double* counts, int nphase, int* bad, cudaStream_t s);
cudaError_t launch_fill(double* p, long long n, double v, cudaStream_t s);
int cg_blocks();

// frequency of spectral point i of a SpecGeom layout [ky][kz][kx] (Eq. 1, R1), Hermitian weight
struct Pt {
  double xx, xy, xz;
  double w;
  bool null;
};

DBF_DEV Pt point(const SpecGeom& g, long long i) {
  const int kx = (int)(i % g.n1h);
  const long long rest = i / g.n1h;
  const int kz = (int)(rest % g.n3);
  const int ky = (int)(rest / g.n3);
  Pt p;
  p.xx = __ldg(g.fq.xx + kx);
  p.xy = __ldg(g.fq.xy + ky);
  p.xz = __ldg(g.fq.xz + kz);
  p.w = (kx + g.kx0 == 0 || 2 * (kx + g.kx0) == g.n1) ? 1.0 : 2.0;
  p.null = (p.xx == 0.0 && p.xy == 0.0 && p.xz == 0.0);
  return p;
}
