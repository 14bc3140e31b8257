// cg.cu — PCG vector algebra with the preconditioner applied on the fly.
//
// Vectors are half spectra [3][ky][kz][kx] (R6); inner products weight kx = 0 and kx = n1/2 by
// 1 and the other kx by 2, and take Re() (the full-spectrum Hermitian product, mean-normalised
// spectra so it equals the voxel-mean product by Parseval, R5/R7).  z = M(xi) r is never stored:
// M(xi) = [xi.Cbar.xi]^-1 is rebuilt per point from 36 coefficients (~70 flops) in the update
// and direction kernels (HBM-bound work, no table read).  Reductions are two-stage and
// deterministic: per-CTA partials in a fixed grid, then one CTA sums them in a fixed order.
#include "cg.cuh"

namespace {

constexpr int BLK = 256;
// grid-stride kernels run whole waves (a partial second wave — a 4-per-SM grid at 3 resident
// CTAs per SM — made k_cg_update 1.5x slower, B200 512^3): 3 CTAs of 256 per SM (<= 85
// registers, no spills); k_cg_direction holds 2 (94 registers; 3 would spill) and runs two
// full waves of them (measured a little faster than one).  Grids follow the device's SM count.
constexpr int MINB = 3;
int nblk() { return MINB * num_sms(); }
int nblk_dir() { return 4 * num_sms(); }


// z = A^-1 r with A = xi.Cbar.xi (symmetric 3x3), 0 on the null set Z (R4)
DBF_DEV void apply_M(const PrecQ& Q, const Pt& p, const cplx* r, cplx* z) {
  if (p.null) {
    z[0] = z[1] = z[2] = make_double2(0.0, 0.0);
    return;
  }
  prec_apply(Q.Q, p.xx, p.xy, p.xz, r, z);
}

DBF_DEV double cdot(cplx a, cplx b) { return a.x * b.x + a.y * b.y; }  // Re(conj(a) b)

// M's 36 coefficients live in device memory (updated when Cbar changes, so a captured CUDA graph
// of the PCG loop stays valid across solves); every CTA stages them in shared memory once
DBF_DEV void load_prec(PrecQ& sq, const PrecQ* __restrict__ q) {
  for (int i = threadIdx.x; i < 36; i += blockDim.x) sq.Q[i] = q->Q[i];
  __syncthreads();
}

template <int NV>
DBF_DEV void block_store(double (&v)[NV], double* partials) {
  __shared__ double red[BLK / 32][NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = warp_sum(v[k]);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < BLK / 32; ++w) s += red[w][threadIdx.x];
    partials[(long long)blockIdx.x * NV + threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(BLK, MINB) k_precond(SpecGeom g, const PrecQ* __restrict__ q, const cplx* __restrict__ r, cplx* __restrict__ z) {
  DBF_PDL_ENTRY();
  __shared__ PrecQ Q;
  load_prec(Q, q);
  for (long long i = (long long)blockIdx.x * BLK + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * BLK) {
    Pt p = point(g, i);
    cplx rv[3] = {__ldg(r + i), __ldg(r + g.Hs + i), __ldg(r + 2 * g.Hs + i)};
    cplx zv[3];
    apply_M(Q, p, rv, zv);
    z[i] = zv[0];
    z[g.Hs + i] = zv[1];
    z[2 * g.Hs + i] = zv[2];
  }
}

// p = M r ; partials (<r, p>, <r, r>)
__global__ void __launch_bounds__(BLK, MINB) k_cg_init(SpecGeom g, const PrecQ* __restrict__ q, const cplx* __restrict__ r, cplx* __restrict__ pv, double* partials) {
  DBF_PDL_ENTRY();
  __shared__ PrecQ Q;
  load_prec(Q, q);
  double acc[2] = {0.0, 0.0};
  for (long long i = (long long)blockIdx.x * BLK + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * BLK) {
    Pt p = point(g, i);
    cplx rv[3] = {__ldg(r + i), __ldg(r + g.Hs + i), __ldg(r + 2 * g.Hs + i)};
    cplx zv[3];
    apply_M(Q, p, rv, zv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      pv[c * g.Hs + i] = zv[c];
      acc[0] += p.w * cdot(rv[c], zv[c]);
      acc[1] += p.w * cdot(rv[c], rv[c]);
    }
  }
  block_store<2>(acc, partials);
}

// x += alpha p ; r -= alpha q ; z = M r ; partials (<r, z>, <r, r>)
// r -= alpha q, z = M r on the fly, partial <r,z>, <r,r> (x += alpha p is deferred to the
// direction kernel, which reads p anyway: 3 vector transfers here instead of 6)
__global__ void __launch_bounds__(BLK, MINB) k_cg_update(SpecGeom g, const PrecQ* __restrict__ pq, const CgDev* __restrict__ cg, cplx* __restrict__ r,
                                                   const cplx* __restrict__ qv, double* partials) {
  DBF_PDL_ENTRY_BIG();
  if (cg->converged | cg->breakdown) return;
  __shared__ PrecQ Q;
  load_prec(Q, pq);
  const double alpha = cg->alpha;
  double acc[2] = {0.0, 0.0};
  for (long long i = (long long)blockIdx.x * BLK + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * BLK) {
    cplx rv[3], qj[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // every load of the point in flight before any arithmetic
      rv[c] = r[c * g.Hs + i];
      qj[c] = __ldg(qv + c * g.Hs + i);
    }
    const Pt p = point(g, i);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      rv[c].x = fma(-alpha, qj[c].x, rv[c].x);
      rv[c].y = fma(-alpha, qj[c].y, rv[c].y);
      r[c * g.Hs + i] = rv[c];
    }
    cplx zv[3];
    apply_M(Q, p, rv, zv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      acc[0] += p.w * cdot(rv[c], zv[c]);
      acc[1] += p.w * cdot(rv[c], rv[c]);
    }
  }
  DBF_PDL_EXIT();
  block_store<2>(acc, partials);
}

// x += alpha p (owed since k_fin_alpha), then p = M r + beta p unless PCG has converged.  All
// loads of a point are issued before any arithmetic (5 vector transfers per iteration).
template <bool DO_X, bool DO_P>
DBF_DEV void cg_direction_body(const SpecGeom& g, const PrecQ& Q, double alpha, double beta, cplx* __restrict__ x,
                               cplx* __restrict__ pv, const cplx* __restrict__ r) {
  for (long long i = (long long)blockIdx.x * BLK + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * BLK) {
    cplx rv[3], pj[3], xj[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long j = c * g.Hs + i;
      pj[c] = pv[j];
      if (DO_P) rv[c] = __ldg(r + j);
      if (DO_X) xj[c] = x[j];
    }
    if (DO_X) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xj[c].x = fma(alpha, pj[c].x, xj[c].x);
        xj[c].y = fma(alpha, pj[c].y, xj[c].y);
        x[c * g.Hs + i] = xj[c];
      }
    }
    if (DO_P) {
      const Pt p = point(g, i);
      cplx zv[3];
      apply_M(Q, p, rv, zv);
#pragma unroll
      for (int c = 0; c < 3; ++c)
        pv[c * g.Hs + i] = make_double2(fma(beta, pj[c].x, zv[c].x), fma(beta, pj[c].y, zv[c].y));
    }
  }
}

__global__ void __launch_bounds__(BLK, 2) k_cg_direction(SpecGeom g, const PrecQ* __restrict__ q, const CgDev* __restrict__ cg, cplx* __restrict__ x,
                                                      cplx* __restrict__ pv, const cplx* __restrict__ r, int x_done) {
  DBF_PDL_ENTRY_BIG();
  if (cg->breakdown) return;
  __shared__ PrecQ Q;
  load_prec(Q, q);
  const bool do_x = cg->xphase != 0 && !x_done, do_p = cg->converged == 0;
  if (do_x && do_p) cg_direction_body<true, true>(g, Q, cg->alpha, cg->beta, x, pv, r);
  else if (do_p) cg_direction_body<false, true>(g, Q, cg->alpha, cg->beta, x, pv, r);
  else if (do_x) cg_direction_body<true, false>(g, Q, cg->alpha, cg->beta, x, pv, r);
}

// x += alpha p on a side stream, beside the forward passes of the same iteration (DBFFT_XOVERLAP=1):
// alpha is final since k_fin_alpha and p stays as it is until the direction kernel, which then runs
// with x_done = 1 (3 vector transfers instead of 5).  Same fma as cg_direction_body.
__global__ void __launch_bounds__(BLK, 2) k_cg_xupdate(SpecGeom g, const CgDev* __restrict__ cg, cplx* __restrict__ x, const cplx* __restrict__ pv) {
  DBF_PDL_ENTRY();
  if (cg->breakdown | (cg->xphase == 0)) return;
  const double alpha = cg->alpha;
  for (long long i = (long long)blockIdx.x * BLK + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * BLK) {
    cplx pj[3], xj[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      pj[c] = __ldg(pv + c * g.Hs + i);
      xj[c] = x[c * g.Hs + i];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xj[c].x = fma(alpha, pj[c].x, xj[c].x);
      xj[c].y = fma(alpha, pj[c].y, xj[c].y);
      x[c * g.Hs + i] = xj[c];
    }
  }
}

// end of a PCG iteration; inside the device-side loop (a CUDA graph WHILE node) it also decides
// whether the body runs again
__global__ void k_fin_x(CgDev* cg, cudaGraphConditionalHandle cond, int set_cond) {
  DBF_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  cg->xphase = 0;
  if (set_cond) cudaGraphSetConditional(cond, (cg->converged | cg->breakdown) ? 0u : 1u);
}

// entry of the device-side loop: run the body only if PCG has not stopped yet
__global__ void k_loop_cond(const CgDev* cg, cudaGraphConditionalHandle cond) {
  DBF_PDL_ENTRY();
  if (threadIdx.x == 0) cudaGraphSetConditional(cond, (cg->converged | cg->breakdown) ? 0u : 1u);
}

// r = b - Ax ; partial <r, r>
__global__ void __launch_bounds__(BLK, MINB) k_true_residual(SpecGeom g, const cplx* __restrict__ b, const cplx* __restrict__ ax,
                                                       cplx* __restrict__ r, double* partials) {
  DBF_PDL_ENTRY();
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * BLK + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * BLK) {
    Pt p = point(g, i);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long j = c * g.Hs + i;
      cplx bj = __ldg(b + j), aj = __ldg(ax + j);
      cplx rj = make_double2(bj.x - aj.x, bj.y - aj.y);
      r[j] = rj;
      acc[0] += p.w * cdot(rj, rj);
    }
  }
  block_store<1>(acc, partials);
}

__global__ void __launch_bounds__(BLK, MINB) k_axpy(SpecGeom g, cplx* __restrict__ y, const cplx* __restrict__ x, double a) {
  DBF_PDL_ENTRY();
  for (long long i = (long long)blockIdx.x * BLK + threadIdx.x; i < 3 * g.Hs; i += (long long)gridDim.x * BLK) {
    cplx xv = __ldg(x + i), yv = y[i];
    y[i] = make_double2(fma(a, xv.x, yv.x), fma(a, xv.y, yv.y));
  }
}

// ---- single-CTA finalizers ---------------------------------------------------------------------
// sum partials[j*nred + k] over j for k < nred into out[k] (slot max_slot, if >= 0, is a max)
// out[k] = sum (or max, k = max_slot) over the nblk CTA partials of slot k (nred <= 64), in a fixed
// order: thread-strided partial sums, warp shuffles, then the 8 warp results — one CTA barrier for
// all slots (a tree of 8 barriers per slot took ~10 us for the 10 slots of the x pass)
DBF_DEV void cta_reduce(const double* partials, int nblk, int nred, double* out, int max_slot) {
  __shared__ double red[BLK / 32][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < nred; ++k) {
    const bool is_max = (k == max_slot);
    double s = 0.0;
    for (int j = threadIdx.x; j < nblk; j += BLK) {
      const double v = partials[(long long)j * nred + k];
      s = is_max ? fmax(s, v) : s + v;
    }
    s = is_max ? warp_max(s) : warp_sum(s);
    if (lane == 0) red[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < nred) {
    const bool is_max = ((int)threadIdx.x == max_slot);
    double s = 0.0;
    for (int q = 0; q < BLK / 32; ++q) s = is_max ? fmax(s, red[q][threadIdx.x]) : s + red[q][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

DBF_DEV void sym9(double* m) {  // small strain: only 6 Voigt slots were accumulated
  m[3] = m[1];
  m[6] = m[2];
  m[7] = m[5];
}

DBF_DEV double norm9(const double* m) {
  double s = 0.0;
  for (int a = 0; a < 9; ++a) s += m[a] * m[a];
  return sqrt(s);
}

// The finalizers read small vectors already reduced over CTAs (k_reduce) and, with several
// ranks, over ranks (NCCL all-reduce or the loopback kernel below).

// loc = [<r,z>_u, <r,r>_u]
__global__ void k_fin_init(CgDev* cg, const double* loc) {
  DBF_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  for (int a = 0; a < 9; ++a) {
    double z = 0.0;
    for (int b = 0; b < 9; ++b) z += cg->Minv_e[9 * a + b] * cg->re[b];
    cg->ze[a] = z;
  }
  double rze = 0.0, ree = 0.0;
  for (int a = 0; a < 9; ++a) {
    cg->pe[a] = cg->ze[a];
    rze += cg->re[a] * cg->ze[a];
    ree += cg->re[a] * cg->re[a];
  }
  cg->rz = loc[0] + rze;
  cg->rr = loc[1];
  const double den = fmax(norm9(cg->msig), 1e-300);
  cg->eps_eq = sqrt(loc[1]) / den;
  cg->eps_load = cg->macro ? sqrt(ree) / den : 0.0;
  cg->converged = (cg->eps_eq <= cg->tol_eq && cg->eps_load <= cg->tol_load) ? 1 : 0;
  if (cg->trace && cg->iters == 0 && cg->trace_cap > 0) {  // restarts keep the history
    cg->trace[0] = cg->eps_eq;
    cg->trace[1] = cg->eps_load;
  }
  if (!(cg->rz == cg->rz)) cg->breakdown = 1;
}

// loc = [<p,q>_u, sum sigma(p) (9)]
DBF_DEV void fin_alpha_dev(CgDev* cg, const double* loc) {
  if (cg->converged | cg->breakdown) return;
  for (int a = 0; a < 9; ++a) cg->dc[a] = loc[1 + a] * cg->inv_n;
  if (cg->sym) sym9(cg->dc);
  // <p, A p> = <p_u, q_u> + p_e . q_e; <p_u, q_u> = (1/N) sum_x grad p_u : sigma(p) from the X pass
  // (loc[10], Parseval), so F3 does not re-read p
  double pq = loc[10] * cg->inv_n;
  for (int a = 0; a < 9; ++a) {
    cg->qe[a] = cg->mask[a] * cg->dc[a];
    pq += cg->pe[a] * cg->qe[a];
  }
  cg->pq = pq;
  if (!(pq > 0.0) || !(pq == pq)) {
    cg->breakdown = 1;
    return;
  }
  const double alpha = cg->rz / pq;
  cg->alpha = alpha;
  cg->xphase = 1;
  for (int a = 0; a < 9; ++a) {
    cg->xe[a] += alpha * cg->pe[a];
    cg->re[a] -= alpha * cg->qe[a];
    cg->msig[a] += alpha * cg->dc[a];
  }
  for (int a = 0; a < 9; ++a) {
    double z = 0.0;
    for (int b = 0; b < 9; ++b) z += cg->Minv_e[9 * a + b] * cg->re[b];
    cg->ze[a] = z;
  }
}
__global__ void k_fin_alpha(CgDev* cg, const double* loc) {
  DBF_PDL_ENTRY();
  if (threadIdx.x == 0) fin_alpha_dev(cg, loc);
}

// loc = [<r,z>_u, <r,r>_u]
DBF_DEV void fin_beta_dev(CgDev* cg, const double* loc) {
  if (cg->converged | cg->breakdown) return;
  double rze = 0.0, ree = 0.0;
  for (int a = 0; a < 9; ++a) {
    rze += cg->re[a] * cg->ze[a];
    ree += cg->re[a] * cg->re[a];
  }
  const double rz_new = loc[0] + rze;
  cg->rr = loc[1];
  cg->iters += 1;
  const double den = fmax(norm9(cg->msig), 1e-300);
  cg->eps_eq = sqrt(loc[1]) / den;
  cg->eps_load = cg->macro ? sqrt(ree) / den : 0.0;
  if (cg->trace && cg->iters < cg->trace_cap) {
    cg->trace[2 * cg->iters] = cg->eps_eq;
    cg->trace[2 * cg->iters + 1] = cg->eps_load;
  }
  if (!(rz_new == rz_new)) {
    cg->breakdown = 1;
    return;
  }
  if (cg->eps_eq <= cg->tol_eq && cg->eps_load <= cg->tol_load) {
    cg->converged = 1;
    return;
  }
  const double beta = rz_new / cg->rz;
  cg->beta = beta;
  cg->rz = rz_new;
  for (int a = 0; a < 9; ++a) cg->pe[a] = cg->ze[a] + beta * cg->pe[a];
  if (cg->iters >= cg->max_iter) cg->converged = 2;  // exhausted
}
__global__ void k_fin_beta(CgDev* cg, const double* loc) {
  DBF_PDL_ENTRY();
  if (threadIdx.x == 0) fin_beta_dev(cg, loc);
}

// true residual: r = b - Ax already formed.  loc = [<r,r>_u, sum sigma(x) (9)]
__global__ void k_fin_true(CgDev* cg, const double* loc) {
  DBF_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  for (int a = 0; a < 9; ++a) cg->dc[a] = loc[1 + a] * cg->inv_n;
  if (cg->sym) sym9(cg->dc);
  double ree = 0.0;
  for (int a = 0; a < 9; ++a) {
    cg->msig[a] = cg->msig0[a] + cg->dc[a];
    cg->re[a] = cg->be[a] - cg->mask[a] * cg->dc[a];
    ree += cg->re[a] * cg->re[a];
  }
  const double den = fmax(norm9(cg->msig), 1e-300);
  cg->rr = loc[0];
  cg->eps_eq = sqrt(loc[0]) / den;
  cg->eps_load = cg->macro ? sqrt(ree) / den : 0.0;
  cg->converged = (cg->eps_eq <= cg->tol_eq && cg->eps_load <= cg->tol_load) ? 1 : 0;
}

// loopback all-reduce over P virtual ranks of one process: v[r][off + j] <- op_r v[r][off + j]
// (v: the slabs' loc buffers, a device array uploaded once at creation)
__global__ void k_allreduce_lb(double* const* v, int off, int P, int k, int is_max) {
  DBF_PDL_ENTRY();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double s = v[0][off + j];
    for (int r = 1; r < P; ++r) s = is_max ? fmax(s, v[r][off + j]) : s + v[r][off + j];
    for (int r = 0; r < P; ++r) v[r][off + j] = s;
  }
}

__global__ void __launch_bounds__(BLK) k_reduce(const double* partials, int nblk, int nred, double* out, int max_slot) {
  DBF_PDL_ENTRY();
  __shared__ double s[64];
  cta_reduce(partials, nblk, nred, s, max_slot);
  if (threadIdx.x < nred) out[threadIdx.x] = s[threadIdx.x];
}
// one rank: the CTA reduction and the finalizer that consumes it in one launch (loc as for the pair)
__global__ void __launch_bounds__(BLK) k_reduce_alpha(const double* partials, int nblk, double* loc, CgDev* cg) {
  DBF_PDL_ENTRY();
  __shared__ double s[64];
  cta_reduce(partials, nblk, 10, s, -1);
  if (threadIdx.x < 10) loc[1 + threadIdx.x] = s[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) fin_alpha_dev(cg, loc);
}
__global__ void __launch_bounds__(BLK) k_reduce_beta(const double* partials, int nblk, double* loc, CgDev* cg) {
  DBF_PDL_ENTRY();
  __shared__ double s[64];
  cta_reduce(partials, nblk, 2, s, -1);
  if (threadIdx.x < 2) loc[threadIdx.x] = s[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) fin_beta_dev(cg, loc);
}

// phase counts: per-CTA shared-memory histogram (integer atomics), one global add per phase and
// CTA (a global atomic per voxel serialises on the few phase addresses: 19 ms at 256^3)
constexpr int HIST_SMEM = 4096;
__global__ void k_phase_hist(const uint16_t* __restrict__ ph, long long nvox, double* counts, int nphase, int* bad) {
  __shared__ unsigned int h[HIST_SMEM];
  const bool local = nphase <= HIST_SMEM;
  if (local)
    for (int i = threadIdx.x; i < nphase; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nvox; v += (long long)gridDim.x * blockDim.x) {
    const int p = ph[v];
    if (p >= nphase) atomicExch(bad, 1);
    else if (local) atomicAdd(h + p, 1u);
    else atomicAdd(counts + p, 1.0);  // integer-valued doubles: exact below 2^53
  }
  __syncthreads();
  if (local)
    for (int i = threadIdx.x; i < nphase; i += blockDim.x)
      if (h[i]) atomicAdd(counts + i, (double)h[i]);
}

__global__ void k_fill(double* p, long long n, double v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = v;
}

}  // namespace

int cg_blocks() { return nblk(); }

cudaError_t launch_precond(const SpecGeom& g, const PrecQ* q, const cplx* r, cplx* z, cudaStream_t s) {
  return launch_k(k_precond, nblk(), BLK, 0, s, g, q, r, z);
}
cudaError_t launch_cg_init(const SpecGeom& g, const PrecQ* q, const cplx* r, cplx* p, double* partials, int nblk, cudaStream_t s) {
  return launch_k(k_cg_init, nblk, BLK, 0, s, g, q, r, p, partials);
}
cudaError_t launch_cg_update(const SpecGeom& g, const PrecQ* q, CgDev* cg, cplx* r, const cplx* qv,
                             double* partials, int nblk, cudaStream_t s) {
  return launch_k(k_cg_update, nblk, BLK, 0, s, g, q, cg, r, qv, partials);
}
cudaError_t launch_cg_direction(const SpecGeom& g, const PrecQ* q, const CgDev* cg, cplx* x, cplx* p, const cplx* r, cudaStream_t s,
                                int x_done) {
  return launch_k(k_cg_direction, nblk_dir(), BLK, 0, s, g, q, cg, x, p, r, x_done);
}
cudaError_t launch_cg_xupdate(const SpecGeom& g, const CgDev* cg, cplx* x, const cplx* p, int ctas_per_sm, cudaStream_t s) {
  return launch_k(k_cg_xupdate, ctas_per_sm * num_sms(), BLK, 0, s, g, cg, x, p);
}
cudaError_t launch_fin_x(CgDev* cg, cudaStream_t s, cudaGraphConditionalHandle cond, int set_cond) {
  return launch_k(k_fin_x, 1, 32, 0, s, cg, cond, set_cond);
}
cudaError_t launch_loop_cond(const CgDev* cg, cudaGraphConditionalHandle cond, cudaStream_t s) {
  return launch_k(k_loop_cond, 1, 32, 0, s, cg, cond);
}
cudaError_t launch_fin_init(CgDev* cg, const double* loc, cudaStream_t s) {
  return launch_k(k_fin_init, 1, 32, 0, s, cg, loc);
}
cudaError_t launch_fin_alpha(CgDev* cg, const double* loc, cudaStream_t s) {
  return launch_k(k_fin_alpha, 1, 32, 0, s, cg, loc);
}
cudaError_t launch_fin_beta(CgDev* cg, const double* loc, cudaStream_t s) {
  return launch_k(k_fin_beta, 1, 32, 0, s, cg, loc);
}
cudaError_t launch_true_residual(const SpecGeom& g, const cplx* b, const cplx* Ax, cplx* r, double* partials, int nblk, cudaStream_t s) {
  return launch_k(k_true_residual, nblk, BLK, 0, s, g, b, Ax, r, partials);
}
cudaError_t launch_fin_true(CgDev* cg, const double* loc, cudaStream_t s) {
  return launch_k(k_fin_true, 1, 32, 0, s, cg, loc);
}
cudaError_t launch_allreduce_lb(double* const* v, int off, int P, int k, int is_max, cudaStream_t s) {
  return launch_k(k_allreduce_lb, 1, 64, 0, s, v, off, P, k, is_max);
}
cudaError_t launch_axpy(const SpecGeom& g, cplx* y, const cplx* x, double a, cudaStream_t s) {
  return launch_k(k_axpy, nblk(), BLK, 0, s, g, y, x, a);
}
cudaError_t launch_reduce_alpha(const double* partials, int nblk, double* loc, CgDev* cg, cudaStream_t s) {
  return launch_k(k_reduce_alpha, 1, BLK, 0, s, partials, nblk, loc, cg);
}
cudaError_t launch_reduce_beta(const double* partials, int nblk, double* loc, CgDev* cg, cudaStream_t s) {
  return launch_k(k_reduce_beta, 1, BLK, 0, s, partials, nblk, loc, cg);
}
cudaError_t launch_reduce(const double* partials, int nblk, int nred, double* out, cudaStream_t s, int max_slot) {
  return launch_k(k_reduce, 1, BLK, 0, s, partials, nblk, nred, out, max_slot);
}
cudaError_t launch_phase_hist(const uint16_t* ph, long long nvox, double* counts, int nphase, int* bad, cudaStream_t s) {
  k_phase_hist<<<nblk(), BLK, 0, s>>>(ph, nvox, counts, nphase, bad);
  return cudaGetLastError();
}
cudaError_t launch_fill(double* p, long long n, double v, cudaStream_t s) {
  k_fill<<<nblk(), BLK, 0, s>>>(p, n, v);
  return cudaGetLastError();
}
