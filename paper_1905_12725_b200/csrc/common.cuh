// common.cuh — device helpers shared by the DBFFT kernels (complex fp64, in-CTA FFT).
//
// FFT design (B200-first): every pass FFTs along ONE axis for a batch of
// lines held by one CTA.  A length-N transform is done by N/8 threads, each holding 8 points in
// registers (a[s] <-> position g + s*N/8).  Stages are radix-8 (then one radix-4 or radix-2
// stage when N is not a power of 8), Stockham order, exchanging through shared memory; the
// first stage loads straight from global memory and the last stage's registers go straight to
// global memory, so the fused pointwise pre/post operations (gradient, divergence, contraction)
// touch registers only.  Twiddles come from a table of W_N = exp(-2 pi i k/N) computed on the
// host in long double (accurate to 0.5 ulp), never from sincos recurrences.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DBF_DEV __device__ __forceinline__

typedef double2 cplx;

// Programmatic dependent launch (PDL, sm_90+): a kernel launched with launch_k() may be scheduled
// while its stream predecessor drains (launch latency and prologue overlap the predecessor's
// tail).  Every such kernel starts with DBF_PDL_ENTRY(): it lets its own successor launch early
// and waits — before touching any global data and in every CTA, so that its completion implies
// its predecessors' — until the predecessor grid has completed and its writes are visible.
DBF_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
DBF_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define DBF_PDL_ENTRY() \
  do {                  \
    pdl_trigger();      \
    pdl_wait();         \
  } while (0)
// DBF_PDL_LATE=1: the big kernels (passes, k_cg_update, k_cg_direction) let their successor launch
// only once a CTA has finished its main loop (DBF_PDL_EXIT), so that the successor's CTAs take
// an SM as this grid drains instead of queueing behind it from the start.
#ifndef DBF_PDL_LATE
#define DBF_PDL_LATE 0
#endif
#define DBF_PDL_ENTRY_BIG()            \
  do {                                 \
    if (!DBF_PDL_LATE) pdl_trigger();  \
    pdl_wait();                        \
  } while (0)
#define DBF_PDL_EXIT()               \
  do {                               \
    if (DBF_PDL_LATE) pdl_trigger(); \
  } while (0)

bool pdl_enabled();  // DBFFT_PDL=1 (default off, see passes.cu)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  if (!pdl_enabled()) {
    k<<<grid, block, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

DBF_DEV cplx cmk(double r, double i) { return make_double2(r, i); }
DBF_DEV cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
DBF_DEV cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
DBF_DEV cplx cmul(cplx a, cplx b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
DBF_DEV cplx cconj(cplx a) { return make_double2(a.x, -a.y); }
DBF_DEV cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
// i*s*a  (multiplication by the imaginary number i s)
DBF_DEV cplx cimul(cplx a, double s) { return make_double2(-a.y * s, a.x * s); }
// a + i*s*b
DBF_DEV cplx cfma_i(cplx a, double s, cplx b) { return make_double2(a.x - s * b.y, a.y + s * b.x); }

// ---------------------------------------------------------------------------------------------
// In-register DFTs.  INV = false: exp(-2 pi i jk/R); INV = true: exp(+2 pi i jk/R).
// ---------------------------------------------------------------------------------------------
template <bool INV>
DBF_DEV cplx mul_mi(cplx a) {  // forward: multiply by -i ; inverse: by +i
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
DBF_DEV void dft2(cplx& a, cplx& b) {
  cplx t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
DBF_DEV void dft4(cplx& x0, cplx& x1, cplx& x2, cplx& x3) {
  cplx t0 = cadd(x0, x2), t1 = csub(x0, x2);
  cplx t2 = cadd(x1, x3), t3 = mul_mi<INV>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

template <bool INV>
DBF_DEV void dft8(cplx* x) {
  const double h = 0.70710678118654752440;
  cplx e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
  cplx o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  // o_k *= W8^k
  o1 = INV ? make_double2(h * (o1.x - o1.y), h * (o1.x + o1.y)) : make_double2(h * (o1.x + o1.y), h * (o1.y - o1.x));
  o2 = mul_mi<INV>(o2);
  o3 = INV ? make_double2(-h * (o3.x + o3.y), h * (o3.x - o3.y)) : make_double2(h * (o3.y - o3.x), -h * (o3.x + o3.y));
  x[0] = cadd(e0, o0); x[4] = csub(e0, o0);
  x[1] = cadd(e1, o1); x[5] = csub(e1, o1);
  x[2] = cadd(e2, o2); x[6] = csub(e2, o2);
  x[3] = cadd(e3, o3); x[7] = csub(e3, o3);
}

// ---------------------------------------------------------------------------------------------
// Stage plan: radix-8 stages, then one radix-(N / 8^k) stage if N is not a power of 8.
// ---------------------------------------------------------------------------------------------
template <int N>
struct FftPlan {
  static constexpr int log2n = (N == 8) ? 3 : (N == 16) ? 4 : (N == 32) ? 5 : (N == 64) ? 6 : (N == 128) ? 7 : (N == 256) ? 8 : (N == 512) ? 9 : (N == 1024) ? 10 : -1;
  static_assert(log2n > 0, "unsupported FFT length");
  static constexpr int n8 = log2n / 3;                  // number of radix-8 stages
  static constexpr int last = 1 << (log2n - 3 * n8);    // 1, 2 or 4
  static constexpr int nstages = n8 + (last > 1 ? 1 : 0);
};

// a[m + M r] *= W^(r step) for r = 1..R-1.  Only W^step, W^2step, W^4step (and W^8step for
// R = 16) come from the table; the others are products of two or three table entries
// (<= 4 ulp), which keeps the L1 twiddle traffic at 3-4 loads per butterfly.
template <int N, int R, bool INV, int P>
DBF_DEV void twiddle_r(cplx (&a)[P], int m, int M, int step, const cplx* __restrict__ tw) {
  cplx w[R];
  auto ld = [&](int e) {
    cplx v = __ldg(tw + e);
    if (INV) v.y = -v.y;
    return v;
  };
  w[1] = ld(step);
  if (R >= 4) {
    w[2] = ld(2 * step);
    w[3] = cmul(w[1], w[2]);
  }
  if (R >= 8) {
    w[4] = ld(4 * step);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
  }
  if (R >= 16) {
    w[8] = ld(8 * step);
#pragma unroll
    for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
  }
#pragma unroll
  for (int r = 1; r < R; ++r) a[m + M * r] = cmul(a[m + M * r], w[r]);
}

// One Stockham stage of radix R on the register array a[8] (positions g + s*N/8), reading
// was already done; writes outputs to smem via idx(pos).  Ns = product of previous radices.
template <int N, int R, bool INV>
DBF_DEV void stage_compute(cplx (&a)[8], int g, int Ns, const cplx* __restrict__ tw) {
  constexpr int M = 8 / R;  // butterflies per thread
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int b = g + m * (N / 8);
    const int k = b % Ns;
    if (Ns > 1) twiddle_r<N, R, INV>(a, m, M, (N / (Ns * R)) * k, tw);
    if (R == 8) {
      dft8<INV>(a);
    } else if (R == 4) {
      dft4<INV>(a[m], a[m + M], a[m + 2 * M], a[m + 3 * M]);
    } else {
      dft2<INV>(a[m], a[m + M]);
    }
  }
}

// Stage-ordered twiddle table (powers of two): for every stage st >= 1 of FftPlan<N> (radix R,
// Ns = product of the earlier radices) and every k < Ns, the R-1 twiddles W_N^(r (N/(Ns R)) k),
// r = 1..R-1, each a correctly rounded table value (no products); N-1 entries in all.  The
// twiddles of a butterfly are then R-1 independent loads from one contiguous row.
template <int N, int R, bool INV, int P>
DBF_DEV void twiddle_tab(cplx (&a)[P], int m, int M, const cplx* __restrict__ ts) {
#pragma unroll
  for (int r = 1; r < R; ++r) {
    cplx w = ts[r - 1];
    if (INV) w.y = -w.y;
    a[m + M * r] = cmul(a[m + M * r], w);
  }
}

// Full in-CTA FFT.  On entry a[s] = x[g + s*N/8]; on exit a[s] = X[g + s*N/8].
// IDX(pos) maps a line position to a shared-memory slot (column interleave or padding).
// All threads of the CTA must call this (it contains __syncthreads()).
struct SyncCtaDefault {
  DBF_DEV void operator()() const { __syncthreads(); }
};

// TAB: `tw` is the stage-ordered table (stage_twiddles on the host) instead of W_N[k].
template <int N, int R, bool INV>
DBF_DEV void stage_compute_tab(cplx (&a)[8], int g, int Ns, const cplx* __restrict__ stab) {
  constexpr int M = 8 / R;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int b = g + m * (N / 8);
    const int k = b % Ns;
    if (Ns > 1) twiddle_tab<N, R, INV>(a, m, M, stab + k * (R - 1));
    if (R == 8) {
      dft8<INV>(a);
    } else if (R == 4) {
      dft4<INV>(a[m], a[m + M], a[m + 2 * M], a[m + 3 * M]);
    } else {
      dft2<INV>(a[m], a[m + M]);
    }
  }
}

template <int N, bool INV, class IDX, class SYNC = SyncCtaDefault, bool TAB = false>
DBF_DEV void fft_cta(cplx (&a)[8], cplx* sbuf, int g, const IDX& idx, const cplx* __restrict__ tw, const SYNC& sync = SYNC{}) {
  typedef FftPlan<N> P;
  int Ns = 1;
  int tbase = 0;  // TAB: offset of this stage's rows in the stage-ordered table
#pragma unroll
  for (int st = 0; st < P::nstages; ++st) {
    const bool is_last = (st == P::nstages - 1);
    const int R = (st < P::n8) ? 8 : P::last;
    if (st > 0) {
      // load a[s] = buf[g + s*N/8]
#pragma unroll
      for (int s = 0; s < 8; ++s) a[s] = sbuf[idx(g + s * (N / 8))];
    }
    if (TAB) {
      if (R == 8) stage_compute_tab<N, 8, INV>(a, g, Ns, tw + tbase);
      else if (R == 4) stage_compute_tab<N, 4, INV>(a, g, Ns, tw + tbase);
      else stage_compute_tab<N, 2, INV>(a, g, Ns, tw + tbase);
      if (Ns > 1) tbase += Ns * (R - 1);
    } else if (R == 8) stage_compute<N, 8, INV>(a, g, Ns, tw);
    else if (R == 4) stage_compute<N, 4, INV>(a, g, Ns, tw);
    else stage_compute<N, 2, INV>(a, g, Ns, tw);
    if (!is_last) {
      sync();  // the group finished reading the buffer
      const int M = 8 / R;
#pragma unroll
      for (int m = 0; m < 8 / 2; ++m) {
        if (m >= M) break;
        const int b = g + m * (N / 8);
        const int base = (b / Ns) * Ns * R + (b % Ns);
        for (int r = 0; r < R; ++r) sbuf[idx(base + r * Ns)] = a[m + M * r];
      }
      sync();
    }
    Ns *= R;
  }
}

// Column interleave: element (pos, column c) at pos*COLS + c.
template <int COLS>
struct IdxCols {
  int c;
  DBF_DEV int operator()(int pos) const { return pos * COLS + c; }
};
// One line per buffer, one pad complex per 8 (bank-conflict-free radix-8 scatter).
struct IdxPad {
  int base;
  DBF_DEV int operator()(int pos) const { return base + pos + (pos >> 3); }
};

// ---------------------------------------------------------------------------------------------
// Warp/block reductions (deterministic order).
// ---------------------------------------------------------------------------------------------
DBF_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
DBF_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------------------------
// Sub-warp FFT (column passes): a length-N transform is owned by T = N/P threads of ONE warp
// (P points each, a[s] <-> position g + s*T), so every exchange needs only __syncwarp().
// Stages: radix-P (P = 16: DFT-16 as 4x4 in registers) while possible, then one radix-R stage.
// ---------------------------------------------------------------------------------------------
template <bool INV>
DBF_DEV cplx w16(int e) {  // W16^e, e in [0, 16)
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
  double c, s;
  switch (e & 15) {
    case 0: c = 1; s = 0; break;
    case 1: c = c1; s = s1; break;
    case 2: c = h; s = h; break;
    case 3: c = s1; s = c1; break;
    case 4: c = 0; s = 1; break;
    case 5: c = -s1; s = c1; break;
    case 6: c = -h; s = h; break;
    case 7: c = -c1; s = s1; break;
    case 8: c = -1; s = 0; break;
    case 9: c = -c1; s = -s1; break;
    case 10: c = -h; s = -h; break;
    case 11: c = -s1; s = -c1; break;
    case 12: c = 0; s = -1; break;
    case 13: c = s1; s = -c1; break;
    case 14: c = h; s = -h; break;
    default: c = c1; s = -s1; break;
  }
  return make_double2(c, INV ? s : -s);  // exp(-+ 2 pi i e / 16)
}

// x[n*st + off] for n = 0..15 -> X[k] in place (natural order), via 4 x 4
template <bool INV, int ST>
DBF_DEV void dft16s(cplx* x, int off) {
  cplx y[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    cplx v0 = x[off + ST * q], v1 = x[off + ST * (q + 4)], v2 = x[off + ST * (q + 8)], v3 = x[off + ST * (q + 12)];
    dft4<INV>(v0, v1, v2, v3);  // over n1: outputs k1 = 0..3
    y[4 * q + 0] = v0;
    y[4 * q + 1] = cmul(v1, w16<INV>(q));
    y[4 * q + 2] = cmul(v2, w16<INV>(2 * q));
    y[4 * q + 3] = cmul(v3, w16<INV>(3 * q));
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    cplx v0 = y[k1], v1 = y[4 + k1], v2 = y[8 + k1], v3 = y[12 + k1];
    dft4<INV>(v0, v1, v2, v3);  // over q: outputs k2
    x[off + ST * (k1)] = v0;
    x[off + ST * (k1 + 4)] = v1;
    x[off + ST * (k1 + 8)] = v2;
    x[off + ST * (k1 + 12)] = v3;
  }
}

template <int N, int P>
struct SubPlan {
  static constexpr int log2n = (N == 8) ? 3 : (N == 16) ? 4 : (N == 32) ? 5 : (N == 64) ? 6 : (N == 128) ? 7 : (N == 256) ? 8 : (N == 512) ? 9 : (N == 1024) ? 10 : -1;
  static constexpr int log2p = (P == 16) ? 4 : 3;
  static constexpr int nfull = log2n / log2p;
  static constexpr int last = 1 << (log2n - log2p * nfull);
  static constexpr int nstages = nfull + (last > 1 ? 1 : 0);
};

template <int N, int P, int R, bool INV>
DBF_DEV void sub_stage(cplx (&a)[P], int g, int Ns, const cplx* __restrict__ tw) {
  constexpr int T = N / P;
  constexpr int M = P / R;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int b = g + m * T;
    const int k = b % Ns;
    if (Ns > 1) twiddle_r<N, R, INV>(a, m, M, (N / (Ns * R)) * k, tw);
    if (R == 16) dft16s<INV, 1>(a, 0);
    else if (R == 8) {
      cplx t8[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) t8[r] = a[m + M * r];
      dft8<INV>(t8);
#pragma unroll
      for (int r = 0; r < 8; ++r) a[m + M * r] = t8[r];
    } else if (R == 4) dft4<INV>(a[m], a[m + M], a[m + 2 * M], a[m + 3 * M]);
    else dft2<INV>(a[m], a[m + M]);
  }
}

// All T threads of the group must call it; SYNC() orders the group's shared-memory exchange.
template <int N, int P, bool INV, class IDX, class SYNC>
DBF_DEV void fft_sub(cplx (&a)[P], cplx* sbuf, int g, const IDX& idx, const cplx* __restrict__ tw, const SYNC& sync) {
  typedef SubPlan<N, P> PL;
  constexpr int T = N / P;
  int Ns = 1;
#pragma unroll
  for (int st = 0; st < PL::nstages; ++st) {
    const bool is_last = (st == PL::nstages - 1);
    const int R = (st < PL::nfull) ? P : PL::last;
    if (st > 0) {
#pragma unroll
      for (int s = 0; s < P; ++s) a[s] = sbuf[idx(g + s * T)];
    }
    if (R == 16) sub_stage<N, P, (P >= 16 ? 16 : 2), INV>(a, g, Ns, tw);
    else if (R == 8) sub_stage<N, P, (P >= 8 ? 8 : 2), INV>(a, g, Ns, tw);
    else if (R == 4) sub_stage<N, P, 4, INV>(a, g, Ns, tw);
    else sub_stage<N, P, 2, INV>(a, g, Ns, tw);
    if (!is_last) {
      sync();  // the group finished reading the buffer
      const int M = P / R;
#pragma unroll
      for (int m = 0; m < P; ++m) {
        if (m >= M) break;
        const int b = g + m * T;
        const int base = (b / Ns) * Ns * R + (b % Ns);
        for (int r = 0; r < R; ++r) sbuf[idx(base + r * Ns)] = a[m + M * r];
      }
      sync();
    }
    Ns *= R;
  }
}

// per-group buffer of N complex, XOR swizzle of the low 3 bits by bits 4..6: conflict-free
// radix-16 scatter (positions 16 g + r) and gather (g + 16 s)
struct IdxGrp {
  int base;
  DBF_DEV int operator()(int pos) const { return base + (pos ^ ((pos >> 4) & 7)); }
};
struct SyncWarp {
  DBF_DEV void operator()() const { __syncwarp(); }
};
struct SyncCta {
  DBF_DEV void operator()() const { __syncthreads(); }
};

// ---------------------------------------------------------------------------------------------
// Saint Venant-Kirchhoff hyperelasticity (the paper's SS3.3 matrix and voids):
//   E = (F^T F - I)/2,  S = lam tr(E) I + 2 mu E,  P = F S,
//   K_ijkl = dP_ij/dF_kl = d_ik S_lj + lam F_ij F_kl + mu (F_il F_kj + (F F^T)_ik d_jl)
// (major symmetric).  F, P row-major 3x3; K45 = upper triangle of the 9x9 (a = 3i+j <= b = 3k+l).
// ---------------------------------------------------------------------------------------------
DBF_DEV void svk_stress(const double* F, double mu, double lam, double* P, double* S) {
  double C[9];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) C[3 * p + q] = F[p] * F[q] + F[3 + p] * F[3 + q] + F[6 + p] * F[6 + q];
  const double trE = 0.5 * (C[0] + C[4] + C[8] - 3.0);
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) S[3 * p + q] = mu * (C[3 * p + q] - (p == q ? 1.0 : 0.0)) + (p == q ? lam * trE : 0.0);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) P[3 * i + j] = F[3 * i] * S[j] + F[3 * i + 1] * S[3 + j] + F[3 * i + 2] * S[6 + j];
}

DBF_DEV void svk_tangent45(const double* F, const double* S, double mu, double lam, double* K45) {
  double B[9];  // F F^T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) B[3 * i + k] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    const int i = a / 3, j = a % 3;
#pragma unroll
    for (int b = a; b < 9; ++b) {
      const int k = b / 3, l = b % 3;
      double v = lam * F[3 * i + j] * F[3 * k + l] + mu * F[3 * i + l] * F[3 * k + j];
      if (i == k) v += S[3 * l + j];
      if (j == l) v += mu * B[3 * i + k];
      K45[a * 9 - a * (a - 1) / 2 + (b - a)] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Mixed-radix FFT for the odd grids of the paper (N = 15, 21, 27, 63 = 3^2 7; Eq. 1 without a
// Nyquist frequency).  Same Stockham scheme as fft_cta: T = N/P threads per
// transform, thread g owns positions g + s T (s < P); stage radices R in {3, 5, 7} with R | P,
// so a thread runs P/R butterflies per stage; exchanges through shared memory via IDX/SYNC.
// ---------------------------------------------------------------------------------------------
template <int N>
struct OddPlan {  // points per thread and the radix sequence (product = N)
  static constexpr int P = (N == 15) ? 15 : (N == 21) ? 21 : (N == 27) ? 9 : (N == 63) ? 21 : 0;
  static constexpr int NST = (N == 15) ? 2 : (N == 21) ? 2 : (N == 27) ? 3 : (N == 63) ? 3 : 0;
  DBF_DEV static constexpr int radix(int st) {
    return (N == 15) ? (st == 0 ? 3 : 5) : (N == 21) ? (st == 0 ? 3 : 7) : (N == 27) ? 3 : (st < 2 ? 3 : 7);
  }
  static_assert(P > 0, "unsupported odd FFT length");
};

// cos / sin of 2 pi e / R (R = 3, 5, 7), correctly rounded literals (constant-folded when unrolled)
template <int R>
DBF_DEV void w_root(int e, double& cs, double& sn) {
  cs = 1.0;
  sn = 0.0;
  if (R == 3) { const double c[3] = {1.000000000000000000000e+00, -5.000000000000000000000e-01, -5.000000000000000000000e-01}; const double s[3] = {0.000000000000000000000e+00, 8.660254037844385965883e-01, -8.660254037844385965883e-01}; cs = c[e]; sn = s[e]; }
  if (R == 5) { const double c[5] = {1.000000000000000000000e+00, 3.090169943749474512629e-01, -8.090169943749474512629e-01, -8.090169943749474512629e-01, 3.090169943749474512629e-01}; const double s[5] = {0.000000000000000000000e+00, 9.510565162951535311819e-01, 5.877852522924731371035e-01, -5.877852522924731371035e-01, -9.510565162951535311819e-01}; cs = c[e]; sn = s[e]; }
  if (R == 7) { const double c[7] = {1.000000000000000000000e+00, 6.234898018587334833640e-01, -2.225209339563143928764e-01, -9.009688679024191459987e-01, -9.009688679024191459987e-01, -2.225209339563143928764e-01, 6.234898018587334833640e-01}; const double s[7] = {0.000000000000000000000e+00, 7.818314824680298036341e-01, 9.749279121818236193420e-01, 4.338837391175581204017e-01, -4.338837391175581204017e-01, -9.749279121818236193420e-01, -7.818314824680298036341e-01}; cs = c[e]; sn = s[e]; }
}

// points per thread of a column / X-pair FFT: 8 for powers of two, OddPlan<N>::P for odd N
template <int N, bool ODD = (N & 1) != 0>
struct PtsPerThread { static constexpr int value = 8; };
template <int N>
struct PtsPerThread<N, true> { static constexpr int value = OddPlan<N>::P; };

// y_k = sum_r x_r W_R^(rk), W_R = exp(-+2 pi i / R), in place on x[m + M r]
template <int R, bool INV, int P>
DBF_DEV void dft_small(cplx (&a)[P], int m, int M) {
  cplx x[R], y[R];
#pragma unroll
  for (int r = 0; r < R; ++r) x[r] = a[m + M * r];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    cplx acc = x[0];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const int e = (r * k) % R;
      if (e == 0) {
        acc = cadd(acc, x[r]);
      } else {
        double c, s;
        w_root<R>(e, c, s);
        const cplx w = make_double2(c, INV ? s : -s);
        acc = cadd(acc, cmul(x[r], w));
      }
    }
    y[k] = acc;
  }
#pragma unroll
  for (int k = 0; k < R; ++k) a[m + M * k] = y[k];
}

template <int N, int R, bool INV, int P>
DBF_DEV void odd_stage(cplx (&a)[P], int g, int Ns, const cplx* __restrict__ tw) {
  constexpr int T = N / P;
  constexpr int M = P / R;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int b = g + m * T;
    const int k = b % Ns;
    if (Ns > 1) {
      const int step = (N / (Ns * R)) * k;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cplx w = tw[(r * step) % N];
        if (INV) w.y = -w.y;
        a[m + M * r] = cmul(a[m + M * r], w);
      }
    }
    dft_small<R, INV>(a, m, M);
  }
}

template <int N, bool INV, class IDX, class SYNC>
DBF_DEV void fft_odd(cplx (&a)[OddPlan<N>::P], cplx* sbuf, int g, const IDX& idx, const cplx* __restrict__ tw, const SYNC& sync) {
  typedef OddPlan<N> PL;
  constexpr int P = PL::P, T = N / P;
  int Ns = 1;
#pragma unroll
  for (int st = 0; st < PL::NST; ++st) {
    const int R = PL::radix(st);
    if (st > 0) {
#pragma unroll
      for (int s = 0; s < P; ++s) a[s] = sbuf[idx(g + s * T)];
    }
    if (R == 3) odd_stage<N, 3, INV>(a, g, Ns, tw);
    else if (R == 5) odd_stage<N, 5, INV>(a, g, Ns, tw);
    else odd_stage<N, 7, INV>(a, g, Ns, tw);
    if (st < PL::NST - 1) {
      sync();
      const int M = P / R;
#pragma unroll
      for (int m = 0; m < P; ++m) {
        if (m >= M) break;
        const int b = g + m * T;
        const int base = (b / Ns) * Ns * R + (b % Ns);
#pragma unroll
        for (int r = 0; r < 7; ++r)
          if (r < R) sbuf[idx(base + r * Ns)] = a[m + M * r];
      }
      sync();
    }
    Ns *= R;
  }
}

// ---------------------------------------------------------------------------------------------
// Preconditioner at one frequency (Eqs. pred2/pred3): z = A^-1 r, A = xi . Cbar . xi,
// A_m = sum_k Q36[6m + k] q_k(xi) with q = (xx xx, yy yy, zz zz, yy zz, xx zz, xx yy) products;
// inverse by cofactors.  Callers handle the null set (xi = 0: z = 0).
// ---------------------------------------------------------------------------------------------
DBF_DEV void prec_apply(const double* Q36, double xx, double xy, double xz, const cplx* r, cplx* z) {
  const double q[6] = {xx * xx, xy * xy, xz * xz, xy * xz, xx * xz, xx * xy};
  double A[6];
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) a = fma(Q36[6 * m + k], q[k], a);
    A[m] = a;
  }
  // A = [[A0, A5, A4], [A5, A1, A3], [A4, A3, A2]]
  const double c00 = A[1] * A[2] - A[3] * A[3];
  const double c01 = A[4] * A[3] - A[5] * A[2];
  const double c02 = A[5] * A[3] - A[1] * A[4];
  const double c11 = A[0] * A[2] - A[4] * A[4];
  const double c12 = A[5] * A[4] - A[0] * A[3];
  const double c22 = A[0] * A[1] - A[5] * A[5];
  const double id = 1.0 / (A[0] * c00 + A[5] * c01 + A[4] * c02);
  z[0] = make_double2((c00 * r[0].x + c01 * r[1].x + c02 * r[2].x) * id, (c00 * r[0].y + c01 * r[1].y + c02 * r[2].y) * id);
  z[1] = make_double2((c01 * r[0].x + c11 * r[1].x + c12 * r[2].x) * id, (c01 * r[0].y + c11 * r[1].y + c12 * r[2].y) * id);
  z[2] = make_double2((c02 * r[0].x + c12 * r[1].x + c22 * r[2].x) * id, (c02 * r[0].y + c12 * r[1].y + c22 * r[2].y) * id);
}
