// dbfft.cu — C-ABI implementation and host driver (plan, slabs, exchanges, PCG and Newton).
//
// Host code only orchestrates: every arithmetic step of the hot path (gradient, FFTs,
// contraction, divergence, preconditioner, CG algebra, constitutive updates, reductions) runs
// in the kernels of passes.cu / cg.cu / this file.  The host does the O(1) macro algebra
// (9x9 macro-block inverse, preconditioner coefficients from Cbar) once per increment.
//
// Distribution: real space in z-slabs, spectral space in ky-slabs.  The z pass
// I1 writes its output already blocked by destination rank ([dest][f][ky_loc][z_loc][kx]), one
// exchange moves the blocks, the y pass I2 reads them in place (rank-chunked addressing); F2
// writes [dest][f][ky_loc][z_loc][kx] and the second exchange feeds F3.  Inner products are
// per-rank partial sums followed by an all-reduce of <= 10 doubles.  Exchanges and all-reduces
// use NCCL (dlopen'd at run time) across processes, or the in-process loopback (P virtual ranks
// on one device, device-to-device copies) that tests the same kernels and layouts on one GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

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
#include "monitors.cuh"
#include "peer.cuh"

namespace {

enum Family { FAM_NONE = 0, FAM_LINEAR = 1, FAM_NEOHOOKE = 2, FAM_J2 = 3 };

enum ProfId { PK_I1 = 0, PK_I2, PK_X, PK_F2, PK_F3, PK_XCONST, PK_CGUPD, PK_CGDIR, PK_FIN, PK_OTHER, PK_XCHG, PK_COUNT };
const char* kProfNames[PK_COUNT] = {"pass_I1", "pass_I2", "pass_X", "pass_F2", "pass_F3", "pass_X_const",
                                    "cg_update", "cg_direction", "cg_finalize", "other", "exchange"};

std::string g_create_error;

// ---------------------------------------------------------------- NCCL, loaded on demand
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl g_nccl;

bool nccl_load(std::string* err) {
  if (g_nccl.h) return true;
  const char* names[] = {getenv("DBFFT_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    if (!nm) continue;
    g_nccl.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) {
    *err = "cannot dlopen libnccl.so.2 (set DBFFT_NCCL_LIB)";
    return false;
  }
#define LD(field, sym) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(g_nccl.h, sym))
  LD(GetUniqueId, "ncclGetUniqueId");
  LD(CommInitRank, "ncclCommInitRank");
  LD(CommDestroy, "ncclCommDestroy");
  LD(AllReduce, "ncclAllReduce");
  LD(Send, "ncclSend");
  LD(Recv, "ncclRecv");
  LD(GroupStart, "ncclGroupStart");
  LD(GroupEnd, "ncclGroupEnd");
  LD(GetErrorString, "ncclGetErrorString");
#undef LD
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.Send || !g_nccl.Recv || !g_nccl.GroupStart ||
      !g_nccl.GroupEnd) {
    *err = "libnccl is missing required symbols";
    return false;
  }
  return true;
}

int ilog2(int n) {
  int k = 0;
  while ((1 << k) < n) ++k;
  return k;
}

// grid sizes with FFT kernels: powers of two 8..512, and the odd sizes 15, 21, 27, 63 (the
// paper's 63^3 cells, Eq. 1 without a Nyquist frequency)
bool is_pow2_in(int n) { return (n >= 8 && n <= 512 && (n & (n - 1)) == 0) || n == 15 || n == 21 || n == 27 || n == 63; }

}  // namespace

// one rank's share of the problem
struct Slab {
  int rank = 0;
  // spectral block: ky in [ky0, ky0 + nyl), all kz, local kx columns [0, nkx) = global kx0 + c;
  // real block: z in [z0, z0 + nzl), y in [y0, y0 + nyr), all x.  Pencil grid position (pa, pb),
  // rank = pb Py + pa (z-slabs: Py = 1, pa = 0, pb = rank, nyr = n2, kx0 = 0)
  int nyl = 0, nzl = 0, ky0 = 0, z0 = 0;
  int pa = 0, pb = 0, nyr = 0, y0 = 0, kx0 = 0;
  long long fsB = 0;      // field stride of the x-line layout B inside one kx chunk: nzl * nyr * kxp
  long long Hs = 0;       // complex points per field (= n1h * nyl * n3 = n1h * n2 * nzl)
  long long Hsp = 0;      // the same with the padded kx pitch of the intermediate layouts (kxp)
  long long Nloc = 0;     // voxels in the z-slab
  long long nlines = 0;   // x lines in the z-slab
  const double* xiy = nullptr;  // xi_y of the local ky slab (offset into the global table)
  cplx *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *b = nullptr, *u = nullptr, *u_c = nullptr;
  cplx *WA = nullptr, *WR = nullptr, *WB = nullptr;  // send, receive (== WA when P == 1), y-pass buffers
  // x-line layout B: the y-inverse and x passes store into WBX, the x and y-forward passes read WB.
  // Pencils (Py > 1) exchange WBX -> WB within the row group after each; slabs: WBX == WB.
  cplx* WBX = nullptr;
  // exchange targets: the I1-type passes store into WS1, their readers take WR; the F2-type into
  // WS2, read from WR2.  NCCL transport: WS1 = WS2 = WA, WR2 = WR.  Peer transport: WS1 / WS2 are
  // windows onto every rank's WR / WR2 (peer.cuh), WA stays local scratch.
  cplx *WS1 = nullptr, *WS2 = nullptr, *WR2 = nullptr;
  uint16_t* phase = nullptr;
  double* ptable = nullptr;
  size_t cap_ptable = 0, cap_counts = 0;  // capacities (doubles): set_phases reuses what fits
  int state_nf = 0, state_nk = 0;          // state / tangent fields allocated (0: none)
  double *F = nullptr, *F_c = nullptr, *epsp_c = nullptr, *epsp_t = nullptr, *tan = nullptr;
  CgDev* cg = nullptr;
  double *part_x = nullptr, *part_cg = nullptr, *part_misc = nullptr;
  double* loc = nullptr;   // [64] small reduced vectors (also the all-reduce buffers)
  double* e_dev = nullptr; // [9]
  int* bad = nullptr;
  double* counts = nullptr;
  double* tmp_real = nullptr;
};

struct dbfft_ctx_s {
  int n1, n2, n3, n1h;
  int kxp;  // kx pitch of the intermediate layouts (X1, B, X2): n1h, or rounded up to 8 (DBFFT_KX_PAD=1)
  double L[3];
  int kin;  // 6 or 9
  long long N;  // global voxels
  int P = 1, rank = 0, loopback = 0;
  // decomposition: Py x Pz rank grid (SURVEY 8(f3) pencils; Py = 1: z-slabs / ky-slabs).  Local
  // spectral kx columns nkx: n1/2 + 1 (Py = 1), else kxm + 1 (kxm = n1 / (2 Py) columns + the
  // Nyquist on the last row rank, a zero padding column on the others)
  int Py = 1, Pz = 1, nkx = 0, kxm = 0;
  int device;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // DBFFT_XOVERLAP=k (k CTAs per SM): x += alpha p runs on `side`, forked after alpha and joined
  // before the direction kernel (pcg_body)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int xoverlap = 0;
  // device allocations: the caller's allocator (e.g. torch's caching allocator) or cudaMalloc
  void* (*dev_alloc)(size_t, void*) = nullptr;
  void (*dev_free)(void*, void*) = nullptr;
  void* alloc_user = nullptr;
  std::string err;
  ncclComm_t comm = nullptr;
  // peer transport (env->transport = 1): exchange windows, flag window, barrier bookkeeping
  int peer = 0;
  PeerBuf pb1, pb2, pbf;
  long long xpcs = 0;            // chunk stride of the exchange layouts (complex elements)
  bool pending[2] = {false, false};  // a local read of WR / WR2 since the last device barrier
  std::vector<Slab> slabs;
  double** loc_ptrs = nullptr;  // device array of the slabs' loc pointers (loopback all-reduce)
  // tables (global)
  double *xix = nullptr, *xiy = nullptr, *xiz = nullptr;
  cplx *tw1 = nullptr, *tw2 = nullptr, *tw3 = nullptr;
  // materials
  int family = FAM_NONE;
  int nph = 0;
  int tmode = 1;  // neo-Hookean tangent storage: 1 compact (F^-1, c1), 0 full 45
  std::vector<double> h_ptable;
  double Fbar[9], Fbar_c[9];  // macro strain / F (incl. stress-controlled comps)
  double Cbar[81];
  PrecQ prec;                    // host copy of M's coefficients ...
  PrecQ* prec_dev = nullptr;     // ... and the device copy the kernels read
  bool prec_valid = false;
  // device-side PCG loop (CUDA graph with a WHILE node), one per parameter key, rebuilt when
  // set_phases reallocates the buffers baked into it (gen)
  struct LoopGraph {
    cudaGraphExec_t exec = nullptr;
    long long gen = -1;
    long long body_launches = 0;
  };
  LoopGraph loop[4], rounds[4];  // WHILE-node loop / host-polled round of check_every iterations
  long long gen = 0;
  int loop_fail = 0;             // 1: WHILE graph unavailable here, 2: round graphs too (eager)
  std::string loop_note;         // how the last PCG loop ran (dbfft_info)
  // preconditioner variants: reference medium of linear phases, initial tangent
  std::vector<double> h_counts;  // voxels per phase (global)
  int prec_medium = 0;           // medium the linear prec was built with (0 arithmetic, 1 harmonic, 2 Hill)
  double Cbar_init[81];          // mean tangent at the undeformed state (set_phases), policy 2
  long long n_incr = 0;          // committed increments since set_phases (policy 3)
  // residual trace of the last solve_increment (P:304 Fig. div): (eps_eq, eps_load) per iteration
  double* trace_dev = nullptr;
  int trace_cap = 0, trace_n = 0;
  CgDev* h_cg = nullptr;     // pinned mirror (slab 0)
  double* h_red = nullptr;   // pinned [64]
  int* h_bad = nullptr;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<int, int>>> ev_pending;
  size_t ev_next = 0;
  double prof_ms[PK_COUNT];
  long long prof_n[PK_COUNT];
  long long nlaunch = 0;
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

#define CKN(call)                                                                             \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) {                                                                  \
      ctx->err = std::string(#call) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r_) : "nccl error"); \
      return DBFFT_E_NCCL;                                                                    \
    }                                                                                         \
  } while (0)

// Every ABI call on a ctx runs with the ctx's device current (kernels, the per-device kernel
// attribute / occupancy caches of passes.cu, stream work) and restores the caller's device.
struct DevGuard {
  int prev = -1, dev;
  explicit DevGuard(int d) : dev(d) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};

// NVTX range (host timeline of a profiler: per pass launch, per solve / Newton iteration / PCG
// loop); header-only NVTX v3, a no-op unless a tool is attached
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// ---------------------------------------------------------------- profiling helpers
struct ProfScope {
  dbfft_ctx ctx;
  int id;
  int i0 = -1;
  Nvtx range;
  ProfScope(dbfft_ctx c, int k) : ctx(c), id(k), range(kProfNames[k]) {
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
SpecGeom spec(dbfft_ctx ctx, const Slab& s) {
  SpecGeom g;
  g.n1h = ctx->nkx;
  g.n2 = s.nyl;
  g.n3 = ctx->n3;
  g.Hs = s.Hs;
  g.fq = Freq{ctx->xix + s.kx0, s.xiy, ctx->xiz};
  g.n1 = ctx->n1;
  g.kx0 = s.kx0;
  return g;
}

ColGeom colbase(dbfft_ctx ctx, const Slab& s, const cplx* in, cplx* out) {
  ColGeom g;
  memset(&g, 0, sizeof(g));
  g.in = in;
  g.out = out;
  g.n1h = ctx->nkx;  // local kx columns
  g.n1 = ctx->n1;
  g.kx0 = s.kx0;
  return g;
}

// layouts (complex elements, per rank; P = 1 reduces every one of them to the plain layouts):
//   S  spectral  [f][kyl][kz][kxl]                      fs = Hs   (kx dense, nkx: the API layout)
//   X1 I1 -> I2  [b'][f][kyl][zl][kxl]  (sender: b' = destination column rank, receiver: source)
//   B  y <-> x   [a'][f][zl][yr][kxl]   (pencils: a' = destination / source row rank, chunk
//                                        nf fsB; slabs: one chunk [f][zl][y][kx], fs = Hsp)
//   X2 F2 -> F3  [b'][f][kyl][zl][kxl]
// X1, B, X2 rows have the padded kx pitch kxp; X1 / X2 chunk sizes nf * nyl * nzl * kxp.
// chunk stride of the rank-chunked exchange layouts X1 / X2: dense, or the granularity-padded
// chunk of the peer windows
long long xpcs(dbfft_ctx ctx, const Slab& s, int nf) {
  return ctx->peer ? ctx->xpcs : (long long)nf * s.nyl * s.nzl * ctx->kxp;
}
// chunk stride of the B layout for nf fields (pencils; unused with one chunk)
long long bpcs(dbfft_ctx ctx, const Slab& s, int nf) { return ctx->Py > 1 ? (long long)nf * s.fsB : 0; }

ColGeom geom_I1(dbfft_ctx ctx, const Slab& s, const cplx* in, cplx* out, int nf) {
  ColGeom g = colbase(ctx, s, in, out);
  const long long nkx = ctx->nkx;
  const long long kxp = ctx->kxp;
  g.in_fs = s.Hs; g.in_os = (long long)ctx->n3 * nkx; g.in_ps = nkx; g.in_psh = ilog2(ctx->n3); g.in_pcs = 0;
  g.out_fs = (long long)s.nyl * s.nzl * kxp; g.out_os = (long long)s.nzl * kxp; g.out_ps = kxp;
  g.out_psh = ilog2(s.nzl); g.out_pcs = xpcs(ctx, s, nf);
  g.ncols = (long long)s.nyl * nkx;
  g.tw = ctx->tw3;
  g.fpos = ctx->xiz;
  g.fq = Freq{ctx->xix + s.kx0, s.xiy, ctx->xiz};
  g.n_xy = s.nyl;
  return g;
}
// nf_out: fields the pass writes (the B layout's chunk stride)
ColGeom geom_I2(dbfft_ctx ctx, const Slab& s, const cplx* in, cplx* out, int nf_in, int nf_out) {
  ColGeom g = colbase(ctx, s, in, out);
  const long long nkx = ctx->nkx;
  const long long kxp = ctx->kxp;
  g.in_fs = (long long)s.nyl * s.nzl * kxp; g.in_os = kxp; g.in_ps = (long long)s.nzl * kxp;
  g.in_psh = ilog2(s.nyl); g.in_pcs = xpcs(ctx, s, nf_in);
  g.out_fs = s.fsB; g.out_os = (long long)s.nyr * kxp; g.out_ps = kxp; g.out_psh = ilog2(s.nyr); g.out_pcs = bpcs(ctx, s, nf_out);
  g.ncols = (long long)s.nzl * nkx;
  g.tw = ctx->tw2;
  g.fpos = ctx->xiy;
  g.fq = Freq{ctx->xix + s.kx0, ctx->xiy, ctx->xiz};
  g.n_xy = ctx->n2;
  return g;
}
// nf_in: fields in the B layout (its chunk stride)
ColGeom geom_F2(dbfft_ctx ctx, const Slab& s, const cplx* in, cplx* out, int nf_out, int nf_in) {
  ColGeom g = colbase(ctx, s, in, out);
  const long long nkx = ctx->nkx;
  const long long kxp = ctx->kxp;
  g.in_fs = s.fsB; g.in_os = (long long)s.nyr * kxp; g.in_ps = kxp; g.in_psh = ilog2(s.nyr); g.in_pcs = bpcs(ctx, s, nf_in);
  g.out_fs = (long long)s.nyl * s.nzl * kxp; g.out_os = kxp; g.out_ps = (long long)s.nzl * kxp;
  g.out_psh = ilog2(s.nyl); g.out_pcs = xpcs(ctx, s, nf_out);
  g.ncols = (long long)s.nzl * nkx;
  g.tw = ctx->tw2;
  g.fpos = ctx->xiy;
  g.fq = Freq{ctx->xix + s.kx0, ctx->xiy, ctx->xiz};
  g.n_xy = ctx->n2;
  return g;
}
ColGeom geom_F3(dbfft_ctx ctx, const Slab& s, const cplx* in, cplx* out, int nf_in) {
  ColGeom g = colbase(ctx, s, in, out);
  const long long nkx = ctx->nkx;
  const long long kxp = ctx->kxp;
  g.in_fs = (long long)s.nyl * s.nzl * kxp; g.in_os = (long long)s.nzl * kxp; g.in_ps = kxp;
  g.in_psh = ilog2(s.nzl); g.in_pcs = xpcs(ctx, s, nf_in);
  g.out_fs = s.Hs; g.out_os = (long long)ctx->n3 * nkx; g.out_ps = nkx; g.out_psh = ilog2(ctx->n3); g.out_pcs = 0;
  g.ncols = (long long)s.nyl * nkx;
  g.tw = ctx->tw3;
  g.fpos = ctx->xiz;
  g.fq = Freq{ctx->xix + s.kx0, s.xiy, ctx->xiz};
  g.n_xy = s.nyl;
  return g;
}

// nf_in / nf_out: fields of the B-layout input / output (pencils: their kx-chunk strides)
XGeom xgeom(dbfft_ctx ctx, const Slab& s, const cplx* in, cplx* out, int nf_in = 9, int nf_out = 9) {
  XGeom g;
  memset(&g, 0, sizeof(g));
  g.in = in;
  g.out = out;
  g.fs_in = g.fs_out = s.fsB;
  if (ctx->Py > 1) {
    g.kch = ctx->kxm;
    g.npy = ctx->Py;
    g.kpcs_in = bpcs(ctx, s, nf_in);
    g.kpcs_out = bpcs(ctx, s, nf_out);
  }
  g.n1h = ctx->n1h;
  g.kxp = ctx->kxp;
  g.n1 = ctx->n1;
  g.nlines = s.nlines;
  g.tw = ctx->tw1;
  g.xix = ctx->xix;
  g.inv_n = 1.0 / (double)ctx->N;
  g.oscale = 0.5 / (double)ctx->N;  // exact scaling when N is a power of two; odd grids round once (1 ulp)
  for (int f = 0; f < 9; ++f) g.real_map[f] = f;
  g.partials = s.part_x;
  g.nred = 10;
  g.phase = s.phase;
  g.ptable = s.ptable;
  g.tan = s.tan;
  g.F = s.F;
  g.epsp_c = s.epsp_c;
  g.epsp_t = s.epsp_t;
  g.nvox = s.Nloc;
  g.bad = s.bad;
  g.tmode = ctx->tmode;
  return g;
}

dbfft_status peer_barrier(dbfft_ctx ctx) {
  ProfScope ps(ctx, PK_XCHG);
  // the epoch is a device-side counter (a replayed CUDA graph issues the same launches)
  CK(launch_peer_barrier((unsigned*)ctx->pbf.recv[0], (char*)ctx->pbf.win[0], ctx->pbf.chunk, ctx->P, ctx->rank, ctx->stream));
  ctx->pending[0] = ctx->pending[1] = false;
  return DBFFT_OK;
}

dbfft_status run_col(dbfft_ctx ctx, int kind, int prof_id, const ColGeom& g, int N, int* grid = nullptr) {
  // peer transport across processes: a pass may store into a window only once every rank has
  // finished reading the receive buffers behind it, i.e. after a barrier that follows the last
  // read (all ranks issue the same pass sequence, so the local bookkeeping stands for all)
  const bool guard = ctx->peer && !ctx->loopback;
  if (guard) {
    const Slab& s = ctx->slabs[0];
    const int w = (g.out == s.WS1) ? 0 : (g.out == s.WS2) ? 1 : -1;
    if (w >= 0 && ctx->pending[w]) CKS(peer_barrier(ctx));
  }
  {
    ProfScope ps(ctx, prof_id);
    CK(launch_col(kind, N, g, ctx->stream, grid));
  }
  if (guard) {
    const Slab& s = ctx->slabs[0];
    if (g.in == s.WR) ctx->pending[0] = true;
    if (g.in == s.WR2) ctx->pending[1] = true;
  }
  return DBFFT_OK;
}

dbfft_status run_x(dbfft_ctx ctx, int kind, int prof_id, const XGeom& g, int* grid) {
  ProfScope ps(ctx, prof_id);
  CK(launch_x(kind, ctx->n1, g, ctx->stream, grid));
  return DBFFT_OK;
}

long long global_voxel(dbfft_ctx ctx, const Slab& s, long long v);

// ---------------------------------------------------------------- collectives
// rank of pencil-grid position (a, b) (z-slabs: a = 0, rank = b)
int grank(dbfft_ctx ctx, int a, int b) { return b * ctx->Py + a; }

// all-to-all of equal chunks within the column group (ranks with the same a): (a, b) sends
// WA[d*chunk] to (a, d), which stores it at WR[b*chunk] (z-slabs: all ranks, b = rank)
dbfft_status exchange(dbfft_ctx ctx, long long chunk) {
  if (ctx->Pz == 1) return DBFFT_OK;
  if (ctx->peer) {  // the pass already stored into the peers' receive buffers: wait until all have
    if (ctx->loopback) return DBFFT_OK;  // one stream orders the virtual ranks
    return peer_barrier(ctx);
  }
  ProfScope ps(ctx, PK_XCHG);
  const size_t bytes = sizeof(cplx) * chunk;
  if (ctx->loopback) {
    for (Slab& s : ctx->slabs)
      for (int d = 0; d < ctx->Pz; ++d)
        CK(cudaMemcpyAsync(ctx->slabs[grank(ctx, s.pa, d)].WR + (long long)s.pb * chunk, s.WA + (long long)d * chunk, bytes,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    return DBFFT_OK;
  }
  Slab& s = ctx->slabs[0];
  CK(cudaMemcpyAsync(s.WR + (long long)s.pb * chunk, s.WA + (long long)s.pb * chunk, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  CKN(g_nccl.GroupStart());
  for (int d = 0; d < ctx->Pz; ++d) {
    if (d == s.pb) continue;
    const int peer = grank(ctx, s.pa, d);
    CKN(g_nccl.Send(s.WA + (long long)d * chunk, 2 * chunk, ncclFloat64, peer, ctx->comm, ctx->stream));
    CKN(g_nccl.Recv(s.WR + (long long)d * chunk, 2 * chunk, ncclFloat64, peer, ctx->comm, ctx->stream));
  }
  CKN(g_nccl.GroupEnd());
  return DBFFT_OK;
}

// pencils: all-to-all of the x-line layout B within the row group (ranks with the same b): (a, b)
// sends WBX[d*chunk] (nf fields of kx block d) to (d, b), which stores it at WB[a*chunk] — after
// the y-inverse pass (kx blocks -> full x lines) and after the x pass (back).  No-op for slabs.
dbfft_status xchg_row(dbfft_ctx ctx, int nf) {
  if (ctx->Py == 1) return DBFFT_OK;
  ProfScope ps(ctx, PK_XCHG);
  const long long chunk = (long long)nf * ctx->slabs[0].fsB;
  const size_t bytes = sizeof(cplx) * chunk;
  if (ctx->loopback) {
    for (Slab& s : ctx->slabs)
      for (int d = 0; d < ctx->Py; ++d)
        CK(cudaMemcpyAsync(ctx->slabs[grank(ctx, d, s.pb)].WB + (long long)s.pa * chunk, s.WBX + (long long)d * chunk, bytes,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    return DBFFT_OK;
  }
  Slab& s = ctx->slabs[0];
  CK(cudaMemcpyAsync(s.WB + (long long)s.pa * chunk, s.WBX + (long long)s.pa * chunk, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  CKN(g_nccl.GroupStart());
  for (int d = 0; d < ctx->Py; ++d) {
    if (d == s.pa) continue;
    const int peer = grank(ctx, d, s.pb);
    CKN(g_nccl.Send(s.WBX + (long long)d * chunk, 2 * chunk, ncclFloat64, peer, ctx->comm, ctx->stream));
    CKN(g_nccl.Recv(s.WB + (long long)d * chunk, 2 * chunk, ncclFloat64, peer, ctx->comm, ctx->stream));
  }
  CKN(g_nccl.GroupEnd());
  return DBFFT_OK;
}
int nf_B(dbfft_ctx ctx) { return ctx->kin == 9 ? 9 : 6; }  // fields of the operator's x-line layout

// all-reduce of slab.loc[off .. off+k) over ranks (sum or max)
dbfft_status allreduce(dbfft_ctx ctx, int off, int k, bool is_max) {
  if (ctx->P == 1) return DBFFT_OK;
  ProfScope ps(ctx, PK_FIN);
  if (ctx->loopback) {  // loc_ptrs: the slabs' loc buffers (uploaded at creation)
    CK(launch_allreduce_lb(ctx->loc_ptrs, off, ctx->P, k, is_max ? 1 : 0, ctx->stream));
    return DBFFT_OK;
  }
  double* v = ctx->slabs[0].loc + off;
  CKN(g_nccl.AllReduce(v, v, k, ncclFloat64, is_max ? ncclMax : ncclSum, ctx->comm, ctx->stream));
  return DBFFT_OK;
}

// reduce CTA partials into slab.loc[off ..] (k values)
dbfft_status reduce_to(dbfft_ctx ctx, Slab& s, const double* partials, int nblk, int nred, int off, int max_slot = -1) {
  ProfScope ps(ctx, PK_FIN);
  CK(launch_reduce(partials, nblk, nred, s.loc + off, ctx->stream, max_slot));
  return DBFFT_OK;
}

// copy slab 0's loc[off .. off+k) to the host (all slabs hold the same values after allreduce)
dbfft_status read_loc(dbfft_ctx ctx, int off, int k, double* host) {
  CK(cudaMemcpyAsync(ctx->h_red, ctx->slabs[0].loc + off, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  memcpy(host, ctx->h_red, sizeof(double) * k);
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
  auto idx = [](int i, int j, int k, int l) { return ((i * 3 + j) * 3 + k) * 3 + l; };
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      C0[idx(a, a, b, b)] = (a == b) ? C11 : C12;
      if (a != b) {
        C0[idx(a, b, a, b)] = C44;
        C0[idx(a, b, b, a)] = C44;
      }
    }
  // rotate index by index: C_ijkl = R_ia R_jb R_kc R_ld C0_abcd (four successive contractions)
  double T1[81], T2[81], T3[81];
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

// M's coefficients from Cbar (host), then the device copy the kernels read (stream ordered: kernels
// queued before keep the previous M)
dbfft_status set_prec(dbfft_ctx ctx, const double* C81) {
  ctx->prec = make_prec(C81);
  CK(cudaMemcpyAsync(ctx->prec_dev, &ctx->prec, sizeof(PrecQ), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // the host copy may change again before a pageable copy ran
  ctx->prec_valid = true;
  return DBFFT_OK;
}

// Mandel 6x6 of a symmetric fourth-order tensor (w = 1 normal, sqrt 2 shear) and back
const double kMw[6] = {1.0, 1.0, 1.0, 1.4142135623730950488, 1.4142135623730950488, 1.4142135623730950488};
void full_to_mandel(const double* C81, double* M) {
  for (int I = 0; I < 6; ++I)
    for (int J = 0; J < 6; ++J)
      M[6 * I + J] = kMw[I] * kMw[J] * C81[((kVoigtI[I] * 3 + kVoigtJ[I]) * 3 + kVoigtI[J]) * 3 + kVoigtJ[J]];
}
void mandel_to_full(const double* M, double* C81) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) {
          const int I = voigt_of(i, j), J = voigt_of(k, l);
          C81[((i * 3 + j) * 3 + k) * 3 + l] = M[6 * I + J] / (kMw[I] * kMw[J]);
        }
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
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int vo[9] = {0, 5, 4, 5, 1, 3, 4, 3, 2};
    for (int a = 0; a < 9; ++a) out9[(long long)a * n + i] = v6[(long long)vo[a] * n + i] + (macro9 ? macro9[a] : 0.0);
  }
}

// in place allowed (e9 == s9): every voxel reads its 9 strains before writing its stresses
__global__ void k_stress_linear(const double* e9, const uint16_t* __restrict__ ph, const double* __restrict__ pt, long long n,
                                double* s9) {
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
    if (pt[36 * ph[i] + 2] != 0.0) {  // Saint Venant-Kirchhoff
      double P[9], S[9];
      svk_stress(F, pt[36 * ph[i]], pt[36 * ph[i] + 1], P, S);
      for (int a = 0; a < 9; ++a) P9[(long long)a * n + i] = P[a];
      continue;
    }
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
  const size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
  if (ctx->dev_alloc) {
    *p = static_cast<T*>(ctx->dev_alloc(bytes, ctx->alloc_user));
    if (!*p) {
      ctx->err = "env allocator returned NULL for " + std::to_string(bytes) + " bytes";
      return DBFFT_E_OOM;
    }
    return DBFFT_OK;
  }
  CK(cudaMalloc((void**)p, bytes));
  return DBFFT_OK;
}

void dfree(dbfft_ctx ctx, void* p) {
  if (!p) return;
  if (ctx->dev_free) ctx->dev_free(p, ctx->alloc_user);
  else cudaFree(p);
}

// W_n[k] = exp(-2 pi i k / n), k < n, from long double (0.5 ulp), followed for powers of two by the
// stage-ordered table of the radix-8 plan (common.cuh fft_cta TAB): for every stage with Ns > 1,
// rows k < Ns of the R-1 twiddles W_n^(r (n/(Ns R)) k) — each entry a table value, no products.
dbfft_status make_twiddles(dbfft_ctx ctx, int n, cplx** out) {
  std::vector<double2> h(2 * (size_t)n);
  auto W = [n](long long e) {
    long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)(e % n) / (long double)n;
    return make_double2((double)cosl(a), (double)sinl(a));
  };
  for (int k = 0; k < n; ++k) h[k] = W(k);
  if ((n & (n - 1)) == 0) {
    const int log2n = ilog2(n);
    const int n8 = log2n / 3, last = 1 << (log2n - 3 * n8);
    const int nst = n8 + (last > 1 ? 1 : 0);
    size_t o = n;
    int Ns = 1;
    for (int st = 0; st < nst; ++st) {
      const int R = st < n8 ? 8 : last;
      if (Ns > 1)
        for (int k = 0; k < Ns; ++k)
          for (int r = 1; r < R; ++r) h[o++] = W((long long)r * (n / (Ns * R)) * k);
      Ns *= R;
    }
  }
  CKS(dalloc(ctx, out, h.size()));
  CK(cudaMemcpy(*out, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
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
  std::vector<int> grid_x;  // X-pass CTAs per slab (partials to reduce)
};

int nf_I1(dbfft_ctx ctx) { return ctx->kin == 9 ? 6 : 5; }

// f = K(u) [+ e] on every slab; partials: part_x (DC of sigma, and <u, f> in slot 9) per slab.
// u / f select per-slab vectors, e_member the macro block inside each slab's CgDev.
typedef double Macro9[9];

// PCG-loop early exit: the passes of an iteration return at once once PCG has stopped
template <class G>
void guard_geom(G& g, const Slab& s);
template <>
void guard_geom(ColGeom& g, const Slab& s) {
  g.cg_stop0 = &s.cg->converged;
  g.cg_stop1 = &s.cg->breakdown;
}
template <>
void guard_geom(XGeom& g, const Slab& s) {
  g.stop0 = &s.cg->converged;
  g.stop1 = &s.cg->breakdown;
}

// guard: inside the PCG loop (early exit of every pass once PCG stopped)
dbfft_status apply_K_slabs(dbfft_ctx ctx, cplx* Slab::*u, cplx* Slab::*f, bool use_e, Macro9 CgDev::*e_member,
                           ApplyOut* ao, bool front_only = false, bool guard = false) {
  const bool fin = ctx->kin == 9;
  int xkind;
  if (ctx->family == FAM_LINEAR) xkind = X_K_SMALL_PHASE;
  else if (ctx->family == FAM_J2) xkind = X_K_J2;
  else xkind = ctx->tmode ? X_K_FIN_NH : X_K_FIN_TAN;
  const int nf1 = nf_I1(ctx);
  for (Slab& s : ctx->slabs) {
    ColGeom g = geom_I1(ctx, s, s.*u, s.WS1, nf1);
    if (guard) guard_geom(g, s);
    CKS(run_col(ctx, fin ? COL_I1F : COL_I1S, PK_I1, g, ctx->n3));
  }
  CKS(exchange(ctx, (long long)nf1 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
  const int nfb = nf_B(ctx);
  for (Slab& s : ctx->slabs) {
    ColGeom g = geom_I2(ctx, s, s.WR, s.WBX, nf1, nfb);
    if (guard) guard_geom(g, s);
    CKS(run_col(ctx, fin ? COL_I2F : COL_I2S, PK_I2, g, ctx->n2));
  }
  CKS(xchg_row(ctx, nfb));
  if (ao) ao->grid_x.assign(ctx->slabs.size(), 0);
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    Slab& s = ctx->slabs[k];
    XGeom gx = xgeom(ctx, s, s.WB, s.WBX, nfb, nfb);
    gx.e = use_e ? (const double*)(s.cg->*e_member) : nullptr;
    if (guard) guard_geom(gx, s);
    int gridx = 0;
    CKS(run_x(ctx, xkind, PK_X, gx, &gridx));
    if (ao) ao->grid_x[k] = gridx;
  }
  CKS(xchg_row(ctx, nfb));
  if (front_only) return DBFFT_OK;  // the caller runs the forward tail (PCG: F3 fused with r -= alpha q)
  for (Slab& s : ctx->slabs) {
    ColGeom g = geom_F2(ctx, s, s.WB, s.WS2, 6, nfb);
    if (guard) guard_geom(g, s);
    CKS(run_col(ctx, fin ? COL_F2F : COL_F2S, PK_F2, g, ctx->n2));
  }
  CKS(exchange(ctx, (long long)6 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
  for (Slab& s : ctx->slabs) {
    ColGeom g = geom_F3(ctx, s, s.WR2, s.*f, 6);
    if (guard) guard_geom(g, s);
    CKS(run_col(ctx, fin ? COL_F3F : COL_F3S, PK_F3, g, ctx->n3));
  }
  return DBFFT_OK;
}

// forward tail of the rhs: WB holds -sigma spectra (from an X pass) -> F2 -> F3 -> b
dbfft_status forward_tail(dbfft_ctx ctx) {
  const bool fin = ctx->kin == 9;
  CKS(xchg_row(ctx, nf_B(ctx)));  // the X pass before it stored into WBX
  for (Slab& s : ctx->slabs) CKS(run_col(ctx, fin ? COL_F2F : COL_F2S, PK_F2, geom_F2(ctx, s, s.WB, s.WS2, 6, nf_B(ctx)), ctx->n2));
  CKS(exchange(ctx, (long long)6 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
  for (Slab& s : ctx->slabs) CKS(run_col(ctx, fin ? COL_F3F : COL_F3S, PK_F3, geom_F3(ctx, s, s.WR2, s.b, 6), ctx->n3));
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
  const int mode = (ctx->family == FAM_J2) ? 2 : (ctx->tmode ? 1 : 0);
  for (Slab& s : ctx->slabs) {
    {
      ProfScope ps(ctx, PK_OTHER);
      CK(launch_mean_tangent(mode, xgeom(ctx, s, nullptr, nullptr), s.part_misc, nblk, ctx->stream));
    }
    CKS(reduce_to(ctx, s, s.part_misc, nblk, nk, 0));
  }
  CKS(allreduce(ctx, 0, nk, false));
  double m[64];
  CKS(read_loc(ctx, 0, nk, m));
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
  return set_prec(ctx, ctx->Cbar);
}

// X-pass reductions of every slab into loc[1..9] (sums) and loc[10] (max), all-reduced
dbfft_status reduce_x(dbfft_ctx ctx, const std::vector<int>& grids, double* host10, bool with_max) {
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    Slab& s = ctx->slabs[k];
    CKS(reduce_to(ctx, s, s.part_x, grids[k], 10, 1, 9));  // constitutive kinds: slot 9 = max |d|
  }
  CKS(allreduce(ctx, 1, 9, false));
  if (with_max) CKS(allreduce(ctx, 10, 1, true));
  CKS(read_loc(ctx, 1, 10, host10));
  return DBFFT_OK;
}

// ---------------------------------------------------------------- PCG
// Solves A {x | xe} = {b | be} with x0 = 0.  Requires CgDev (msig0, be, mask, Minv_e) set.
// loc layout: [0] <p,q> / <r,z> / <r,r>, [1] <r,r> (CG pairs), [1..9] DC sums, [10] max.
//
// The iterations run on the device: one CUDA graph per parameter key holds a WHILE node whose
// body is one PCG iteration; the body's last kernel sets the loop condition from CgDev
// (converged / breakdown / max_cg), so the host launches the loop once per solve and waits once —
// no host polls, no operator application after convergence, no per-solve re-capture (M's
// coefficients and every scalar live in device memory).  Fallbacks, in order, when a WHILE
// graph cannot be built here (e.g. collectives that cannot sit inside a conditional body) or
// while the per-kernel profiler records events: host-polled rounds of check_every iterations
// replayed from a plain graph, then eager launches; in both every pass of an iteration exits at
// once after convergence.
dbfft_status pcg_body(dbfft_ctx ctx, int every, bool macro, int nb, cudaGraphConditionalHandle cond);
bool pcg_fused(dbfft_ctx ctx);

struct GraphDel {
  cudaGraph_t g = nullptr;
  ~GraphDel() {
    if (g) cudaGraphDestroy(g);
  }
};

// end a capture whose issue failed; clears the sticky capture error
void abort_capture(dbfft_ctx ctx) {
  cudaGraph_t junk = nullptr;
  cudaStreamEndCapture(ctx->stream, &junk);
  if (junk) cudaGraphDestroy(junk);
  cudaGetLastError();
}

int loop_key(dbfft_ctx ctx, bool macro) { return (macro ? 1 : 0) | (pcg_fused(ctx) ? 2 : 0); }

// the device-side loop: [k_loop_cond] -> WHILE(cond) { one PCG iteration; k_fin_x sets cond }
dbfft_status build_loop_graph(dbfft_ctx ctx, bool macro, int nb, dbfft_ctx_s::LoopGraph* lg) {
  GraphDel g;
  CK(cudaGraphCreate(&g.g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g.g, 0, 0));
  CK(cudaStreamBeginCaptureToGraph(ctx->stream, g.g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  cudaError_t e = launch_loop_cond(ctx->slabs[0].cg, h, ctx->stream);
  cudaGraph_t cap = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(ctx->stream, &cap);
  CK(e);
  CK(e2);
  size_t nn = 0;
  CK(cudaGraphGetNodes(g.g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CK(cudaGraphGetNodes(g.g, nodes.data(), &nn));
  alignas(cudaGraphNodeParams) unsigned char cpbuf[sizeof(cudaGraphNodeParams)] = {};  // (no default ctor)
  cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cpbuf);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  CK(cudaGraphAddNode(&cn, g.g, nodes.data(), nn, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  const long long nl0 = ctx->nlaunch;
  // DBFFT_LOOP_UNROLL=k: k PCG iterations per evaluation of the WHILE condition (after convergence
  // the rest of a body exits pass by pass, as in the host-polled rounds); default 1
  int unroll = 1;
  if (const char* ue = getenv("DBFFT_LOOP_UNROLL")) unroll = std::min(8, std::max(1, atoi(ue)));
  const dbfft_status bst = pcg_body(ctx, unroll, macro, nb, h);
  if (bst != DBFFT_OK) {
    abort_capture(ctx);
    return bst;
  }
  e2 = cudaStreamEndCapture(ctx->stream, &cap);
  CK(e2);
  lg->body_launches = ctx->nlaunch - nl0;
  ctx->nlaunch = nl0;  // captured, not launched
  if (lg->exec) cudaGraphExecDestroy(lg->exec);
  lg->exec = nullptr;
  CK(cudaGraphInstantiate(&lg->exec, g.g, 0));
  lg->gen = ctx->gen;
  return DBFFT_OK;
}

// host-polled round: `every` PCG iterations captured into a plain graph (reused across solves)
dbfft_status build_round_graph(dbfft_ctx ctx, int every, bool macro, int nb, dbfft_ctx_s::LoopGraph* lg) {
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  const long long nl0 = ctx->nlaunch;
  const dbfft_status bst = pcg_body(ctx, every, macro, nb, 0);
  if (bst != DBFFT_OK) {
    abort_capture(ctx);
    return bst;
  }
  GraphDel g;
  CK(cudaStreamEndCapture(ctx->stream, &g.g));
  lg->body_launches = ctx->nlaunch - nl0;
  ctx->nlaunch = nl0;
  if (lg->exec) cudaGraphExecDestroy(lg->exec);
  lg->exec = nullptr;
  CK(cudaGraphInstantiate(&lg->exec, g.g, 0));
  lg->gen = ctx->gen;
  return DBFFT_OK;
}

// run PCG iterations until CgDev says stop (converged, breakdown or max_cg); h_cg is current on return
dbfft_status pcg_iterate(dbfft_ctx ctx, const dbfft_opts& o, bool macro, int nb) {
  const char* genv = getenv("DBFFT_GRAPHS");
  const bool graphs = !ctx->prof && !(genv && genv[0] == '0');
  const int key = loop_key(ctx, macro);
  const int it0 = ctx->h_cg->iters;
  // NCCL mode: a plain captured graph replayed per host-polled round is NCCL's supported graph
  // usage; collectives inside a WHILE body (replayed a data-dependent number of times within one
  // launch) are opt-in (DBFFT_NCCL_WHILE=1) until they have run on a multi-GPU node
  const char* nw = getenv("DBFFT_NCCL_WHILE");
  if (ctx->comm && !(nw && nw[0] == '1') && ctx->loop_fail == 0) {
    ctx->loop_fail = 1;
    ctx->loop_note = "NCCL mode: host-polled graph rounds (DBFFT_NCCL_WHILE=1 tries the WHILE graph)";
  }
  if (graphs && ctx->loop_fail == 0) {
    dbfft_ctx_s::LoopGraph& lg = ctx->loop[key];
    dbfft_status st = DBFFT_OK;
    if (!lg.exec || lg.gen != ctx->gen) st = build_loop_graph(ctx, macro, nb, &lg);
    if (st == DBFFT_OK) {
      Nvtx range("pcg_while_graph");
      CK(cudaGraphLaunch(lg.exec, ctx->stream));
      CK(cudaMemcpyAsync(ctx->h_cg, ctx->slabs[0].cg, sizeof(CgDev), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      ctx->nlaunch += 1 + lg.body_launches * std::max(1, ctx->h_cg->iters - it0);
      ctx->loop_note = "device-side WHILE graph";
      return DBFFT_OK;
    }
    // not available here: remember, fall back to host-polled rounds
    ctx->loop_fail = 1;
    ctx->loop_note = "WHILE graph unavailable (" + ctx->err + "); host-polled graph rounds";
    cudaGetLastError();
  }
  // profiler on: poll every iteration, so no launch is an early exit and the per-kernel event
  // times are those of real work
  const int every = ctx->prof ? 1 : std::max(1, o.check_every);
  for (;;) {
    CK(cudaMemcpyAsync(ctx->h_cg, ctx->slabs[0].cg, sizeof(CgDev), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    prof_flush(ctx);
    const CgDev* h = ctx->h_cg;
    if (h->converged || h->breakdown || h->iters >= o.max_cg) return DBFFT_OK;
    if (graphs && ctx->loop_fail < 2) {
      dbfft_ctx_s::LoopGraph& lg = ctx->rounds[key];
      dbfft_status st = DBFFT_OK;
      if (!lg.exec || lg.gen != ctx->gen || lg.body_launches == 0) st = build_round_graph(ctx, every, macro, nb, &lg);
      if (st == DBFFT_OK) {
        CK(cudaGraphLaunch(lg.exec, ctx->stream));
        ctx->nlaunch += lg.body_launches;
        if (ctx->loop_fail == 0 || ctx->loop_note.empty()) ctx->loop_note = "host-polled graph rounds";
        continue;
      }
      ctx->loop_fail = 2;
      ctx->loop_note += "; round graphs unavailable, eager";
      cudaGetLastError();
    } else if (!graphs) {
      ctx->loop_note = "eager (profiler on or DBFFT_GRAPHS=0)";
    }
    CKS(pcg_body(ctx, every, macro, nb, 0));
  }
}

dbfft_status pcg(dbfft_ctx ctx, const dbfft_opts& o, int* iters_out) {
  Nvtx range("pcg");
  const int nb = cg_blocks();
  const bool macro = ctx->h_cg->macro != 0;
  for (Slab& s : ctx->slabs) {
    CK(cudaMemsetAsync(s.x, 0, sizeof(cplx) * 3 * s.Hs, ctx->stream));
    CK(cudaMemcpyAsync(s.r, s.b, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  auto init_dir = [&]() -> dbfft_status {
    for (Slab& s : ctx->slabs) {
      {
        ProfScope ps(ctx, PK_CGDIR);
        CK(launch_cg_init(spec(ctx, s), ctx->prec_dev, s.r, s.p, s.part_cg, nb, ctx->stream));
      }
      CKS(reduce_to(ctx, s, s.part_cg, nb, 2, 0));
    }
    CKS(allreduce(ctx, 0, 2, false));
    for (Slab& s : ctx->slabs) {
      ProfScope ps(ctx, PK_FIN);
      CK(launch_fin_init(s.cg, s.loc, ctx->stream));
    }
    CK(cudaMemcpyAsync(ctx->h_cg, ctx->slabs[0].cg, sizeof(CgDev), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DBFFT_OK;
  };
  CKS(init_dir());
  int restarts = 0;
  for (;;) {
    CKS(pcg_iterate(ctx, o, macro, nb));  // h_cg current
    prof_flush(ctx);
    *iters_out = ctx->h_cg->iters;
    if (ctx->h_cg->breakdown) {
      ctx->err = "PCG breakdown: <p,Kp> <= 0 or NaN";
      return DBFFT_E_BREAKDOWN;
    }
    if (ctx->h_cg->converged != 1) {
      ctx->err = "PCG did not converge within max_cg";
      return DBFFT_E_NOT_CONVERGED;
    }
    // true-residual confirmation (R7): r = b - A x
    Nvtx range_tr("pcg_true_residual");
    ApplyOut ao;
    CKS(apply_K_slabs(ctx, &Slab::x, &Slab::q, macro, &CgDev::xe, &ao));
    for (size_t k = 0; k < ctx->slabs.size(); ++k) {
      Slab& s = ctx->slabs[k];
      {
        ProfScope ps(ctx, PK_CGUPD);
        CK(launch_true_residual(spec(ctx, s), s.b, s.q, s.r, s.part_cg, nb, ctx->stream));
      }
      CKS(reduce_to(ctx, s, s.part_cg, nb, 1, 0));
      CKS(reduce_to(ctx, s, s.part_x, ao.grid_x[k], 10, 1));
    }
    CKS(allreduce(ctx, 0, 10, false));
    for (Slab& s : ctx->slabs) {
      ProfScope ps(ctx, PK_FIN);
      CK(launch_fin_true(s.cg, s.loc, ctx->stream));
    }
    CK(cudaMemcpyAsync(ctx->h_cg, ctx->slabs[0].cg, sizeof(CgDev), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *iters_out = ctx->h_cg->iters;
    if (ctx->h_cg->converged == 1) return DBFFT_OK;
    // the restarted iterations count against max_cg (cg->iters carries over); a true residual
    // that stays above tolerance after the restart budget is a failure, not a success
    if (restarts >= 20 || ctx->h_cg->iters >= o.max_cg) {
      ctx->err = "PCG did not converge: true residual b - Ax above tolerance after " + std::to_string(restarts) +
                 " restarts (eps_eq " + std::to_string(ctx->h_cg->eps_eq) + ")";
      return DBFFT_E_NOT_CONVERGED;
    }
    ++restarts;  // restart from the true residual: z = M r, p = z
    CKS(init_dir());
  }
}

// F3 geometry of the fused PCG step: q = K p is never stored; r -= alpha q, <r, M r>, <r, r>
ColGeom geom_F3_update(dbfft_ctx ctx, Slab& s) {
  ColGeom g5 = geom_F3(ctx, s, s.WR2, s.r, 6);
  g5.dotp = s.r;
  g5.partials = s.part_cg;
  g5.upd = 1;
  g5.cg_alpha = &s.cg->alpha;
  g5.cg_stop0 = &s.cg->converged;
  g5.cg_stop1 = &s.cg->breakdown;
  g5.precq = ctx->prec_dev->Q;
  return g5;
}

bool pcg_fused(dbfft_ctx ctx) {
  const char* e = getenv("DBFFT_FUSED_UPDATE");
  // opt-in (DBFFT_FUSED_UPDATE=1): once the plain F3 took the stage twiddle table it ran faster
  // unfused (B200 c4 256^3, 2 steps: F3 + k_cg_update 79 + 56 ms vs the fused F3 154 ms; value
  // 5.03e9 vs 4.99e9).  Finite strain only: small strain's F3S program leaves no ring slot for r,
  // and a variant reading r straight from global memory was slower (c5 512^3: 8.6 vs 6.2 ms).
  if (!(e && e[0] == '1') || ctx->kin != 9) return false;
  for (Slab& s : ctx->slabs)
    if (!col_upd_supported(ctx->n3, geom_F3_update(ctx, s))) return false;
  return true;
}

// CTA partials of the x pass (alpha: slots 1..10 of loc) or of the residual update (beta: slots
// 0..1) -> loc, all-reduce over ranks, finalizer.  One rank: reduction and finalizer in one launch.
dbfft_status reduce_fin(dbfft_ctx ctx, const std::vector<int>& nblk, bool alpha) {
  if (ctx->P == 1) {
    Slab& s = ctx->slabs[0];
    ProfScope ps(ctx, PK_FIN);
    CK(alpha ? launch_reduce_alpha(s.part_x, nblk[0], s.loc, s.cg, ctx->stream)
             : launch_reduce_beta(s.part_cg, nblk[0], s.loc, s.cg, ctx->stream));
    return DBFFT_OK;
  }
  for (size_t j = 0; j < ctx->slabs.size(); ++j) {
    Slab& s = ctx->slabs[j];
    CKS(alpha ? reduce_to(ctx, s, s.part_x, nblk[j], 10, 1) : reduce_to(ctx, s, s.part_cg, nblk[j], 2, 0));
  }
  CKS(alpha ? allreduce(ctx, 1, 10, false) : allreduce(ctx, 0, 2, false));
  for (Slab& s : ctx->slabs) {
    ProfScope ps(ctx, PK_FIN);
    CK(alpha ? launch_fin_alpha(s.cg, s.loc, ctx->stream) : launch_fin_beta(s.cg, s.loc, ctx->stream));
  }
  return DBFFT_OK;
}

// end of an iteration: x += alpha p owed by the direction kernel is settled; slab 0's k_fin_x
// decides whether the device-side loop runs again (all slabs hold the same reduced scalars)
dbfft_status fin_x_all(dbfft_ctx ctx, cudaGraphConditionalHandle cond) {
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    ProfScope ps(ctx, PK_FIN);
    CK(launch_fin_x(ctx->slabs[k].cg, ctx->stream, cond, (cond && k == 0) ? 1 : 0));
  }
  return DBFFT_OK;
}

// one PCG iteration with the residual update fused into F3 (8 - 3 + 1 = 6 vector transfers of
// CG algebra per iteration instead of 8): I1 I2 X | alpha | F2 F3(r -= alpha q, <r,z>, <r,r>) |
// beta | direction (x += alpha p, p = z + beta p)
dbfft_status pcg_iteration_fused(dbfft_ctx ctx, bool macro, int nb, cudaGraphConditionalHandle cond) {
  const bool fin = ctx->kin == 9;
  ApplyOut ao;
  CKS(apply_K_slabs(ctx, &Slab::p, &Slab::q, macro, &CgDev::pe, &ao, true, true));
  CKS(reduce_fin(ctx, ao.grid_x, true));
  for (Slab& s : ctx->slabs) {
    ColGeom g = geom_F2(ctx, s, s.WB, s.WS2, 6, nf_B(ctx));
    guard_geom(g, s);
    CKS(run_col(ctx, fin ? COL_F2F : COL_F2S, PK_F2, g, ctx->n2));
  }
  CKS(exchange(ctx, (long long)6 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
  std::vector<int> g3(ctx->slabs.size(), 0);
  for (size_t j = 0; j < ctx->slabs.size(); ++j) {
    Slab& s = ctx->slabs[j];
    CKS(run_col(ctx, fin ? COL_F3F : COL_F3S, PK_F3, geom_F3_update(ctx, s), ctx->n3, &g3[j]));
  }
  CKS(reduce_fin(ctx, g3, false));
  for (Slab& s : ctx->slabs) {
    {
      ProfScope ps(ctx, PK_CGDIR);
      CK(launch_cg_direction(spec(ctx, s), ctx->prec_dev, s.cg, s.x, s.p, s.r, ctx->stream));
    }
  }
  return fin_x_all(ctx, cond);
}

dbfft_status pcg_body(dbfft_ctx ctx, int every, bool macro, int nb, cudaGraphConditionalHandle cond) {
  if (pcg_fused(ctx)) {
    for (int k = 0; k < every; ++k) CKS(pcg_iteration_fused(ctx, macro, nb, cond));
    return DBFFT_OK;
  }
  for (int k = 0; k < every; ++k) {
    ApplyOut ao;
    // <p, A p> comes from the X pass (slot 9: sum (grad p + p_e) : sigma, Parseval), so F3 does
    // not re-read p
    if (ctx->xoverlap) {
      // alpha right after the X pass; x += alpha p on the side stream beside F2 / F3 / the residual
      // update (joined before the direction kernel, which alone writes p)
      CKS(apply_K_slabs(ctx, &Slab::p, &Slab::q, macro, &CgDev::pe, &ao, true, true));
      CKS(reduce_fin(ctx, ao.grid_x, true));
      CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
      CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
      for (Slab& s : ctx->slabs) {
        ctx->nlaunch += 1;
        CK(launch_cg_xupdate(spec(ctx, s), s.cg, s.x, s.p, ctx->xoverlap, ctx->side));
      }
      CK(cudaEventRecord(ctx->ev_join, ctx->side));
      const bool fin = ctx->kin == 9;
      for (Slab& s : ctx->slabs) {
        ColGeom g = geom_F2(ctx, s, s.WB, s.WS2, 6, nf_B(ctx));
        guard_geom(g, s);
        CKS(run_col(ctx, fin ? COL_F2F : COL_F2S, PK_F2, g, ctx->n2));
      }
      CKS(exchange(ctx, (long long)6 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
      for (Slab& s : ctx->slabs) {
        ColGeom g = geom_F3(ctx, s, s.WR2, s.q, 6);
        guard_geom(g, s);
        CKS(run_col(ctx, fin ? COL_F3F : COL_F3S, PK_F3, g, ctx->n3));
      }
    } else {
      CKS(apply_K_slabs(ctx, &Slab::p, &Slab::q, macro, &CgDev::pe, &ao, false, true));
      CKS(reduce_fin(ctx, ao.grid_x, true));
    }
    for (Slab& s : ctx->slabs) {
      ProfScope ps(ctx, PK_CGUPD);
      CK(launch_cg_update(spec(ctx, s), ctx->prec_dev, s.cg, s.r, s.q, s.part_cg, nb, ctx->stream));
    }
    CKS(reduce_fin(ctx, std::vector<int>(ctx->slabs.size(), nb), false));
    if (ctx->xoverlap) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
    for (Slab& s : ctx->slabs) {
      {
        ProfScope ps(ctx, PK_CGDIR);
        CK(launch_cg_direction(spec(ctx, s), ctx->prec_dev, s.cg, s.x, s.p, s.r, ctx->stream, ctx->xoverlap ? 1 : 0));
      }
    }
    CKS(fin_x_all(ctx, cond));
  }
  return DBFFT_OK;
}

// set CgDev header fields on the host mirror and upload to every slab
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
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    h->trace = (k == 0 && ctx->trace_dev) ? ctx->trace_dev + 2 * (size_t)ctx->trace_n : nullptr;
    h->trace_cap = h->trace ? ctx->trace_cap - ctx->trace_n : 0;
    CK(cudaMemcpyAsync(ctx->slabs[k].cg, h, sizeof(CgDev), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // h is reused for the next slab
  }
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

dbfft_status upload_e(dbfft_ctx ctx, const double* host9) {
  for (Slab& s : ctx->slabs) CK(cudaMemcpyAsync(s.e_dev, host9, sizeof(double) * 9, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // host9 may be a stack array
  return DBFFT_OK;
}

dbfft_status copy_vec_all(dbfft_ctx ctx, cplx* Slab::*dst, cplx* Slab::*src) {
  for (Slab& s : ctx->slabs) CK(cudaMemcpyAsync(s.*dst, s.*src, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToDevice, ctx->stream));
  return DBFFT_OK;
}

// ---------------------------------------------------------------- linear solve
// Reference medium of the linear preconditioner from the phase counts.  0: the paper's
// arithmetic mean C = <C(x)>; 1: harmonic mean <C(x)^-1>^-1 (Reuss); 2: Hill, the mean of
// the two.  1 and 2 are the "new ad-hoc preconditioners" of P:394; every variant
// only changes M, never the solution.
dbfft_status linear_reference(dbfft_ctx ctx, int medium) {
  const int nph = ctx->nph;
  const double* pt = ctx->h_ptable.data();
  double CA[81] = {0}, CR[81] = {0};
  double CV[36] = {0};
  for (int k = 0; k < nph; ++k)
    for (int a = 0; a < 36; ++a) CV[a] += ctx->h_counts[k] * pt[36 * k + a];
  for (int a = 0; a < 36; ++a) CV[a] /= (double)ctx->N;
  voigt_to_full(CV, CA);
  if (medium != 0) {
    std::vector<double> S(36, 0.0);
    for (int k = 0; k < nph; ++k) {
      if (ctx->h_counts[k] == 0.0) continue;
      double C81[81], M[36];
      voigt_to_full(pt + 36 * k, C81);
      full_to_mandel(C81, M);
      std::vector<double> Mi(M, M + 36);
      if (!invert(Mi, 6)) {
        ctx->err = "harmonic reference medium: singular phase stiffness";
        return DBFFT_E_MATERIAL;
      }
      for (int a = 0; a < 36; ++a) S[a] += ctx->h_counts[k] * Mi[a];
    }
    for (int a = 0; a < 36; ++a) S[a] /= (double)ctx->N;
    if (!invert(S, 6)) {
      ctx->err = "harmonic reference medium: singular mean compliance";
      return DBFFT_E_MATERIAL;
    }
    mandel_to_full(S.data(), CR);
  }
  for (int a = 0; a < 81; ++a) ctx->Cbar[a] = medium == 0 ? CA[a] : medium == 1 ? CR[a] : 0.5 * (CA[a] + CR[a]);
  ctx->prec_medium = medium;
  return set_prec(ctx, ctx->Cbar);
}

dbfft_status check_opts(dbfft_ctx ctx, const dbfft_opts& o) {
  if (o.precond_refresh < 0 || o.precond_refresh > 3 || o.precond_period < 1 || o.precond_medium < 0 || o.precond_medium > 2) {
    ctx->err = "opts: precond_refresh in 0..3, precond_period >= 1, precond_medium in 0..2";
    return DBFFT_E_INVALID_ARG;
  }
  if (o.precond_medium != 0 && ctx->family != FAM_LINEAR) {
    ctx->err = "opts: precond_medium 1/2 (harmonic / Hill reference medium) needs linear phases";
    return DBFFT_E_INVALID_ARG;
  }
  return DBFFT_OK;
}

dbfft_status solve_linear(dbfft_ctx ctx, const double* target, const uint8_t* mask, const dbfft_opts& o, dbfft_report* rep) {
  if (o.precond_medium != ctx->prec_medium) CKS(linear_reference(ctx, o.precond_medium));
  double epsU[9], sigf[9];
  for (int a = 0; a < 9; ++a) {
    epsU[a] = mask[a] ? 0.0 : target[a];
    sigf[a] = mask[a] ? target[a] : 0.0;
  }
  CKS(upload_e(ctx, epsU));
  // rhs b = d:F(C:eps_U) (P:118 right-hand side, R3) and <C:eps_U>
  std::vector<int> grids(ctx->slabs.size());
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    Slab& s = ctx->slabs[k];
    XGeom gx = xgeom(ctx, s, nullptr, s.WBX, 6, 6);
    gx.e = s.e_dev;
    CKS(run_x(ctx, X_RHS_SMALL_PHASE, PK_XCONST, gx, &grids[k]));
  }
  CKS(forward_tail(ctx));
  double red[10];
  CKS(reduce_x(ctx, grids, red, false));
  double msig0[9], be[9];
  for (int a = 0; a < 9; ++a) msig0[a] = red[a] / (double)ctx->N;
  sym_fill(msig0);
  for (int a = 0; a < 9; ++a) be[a] = mask[a] ? sigf[a] - msig0[a] : 0.0;
  CKS(cg_setup(ctx, o, mask, msig0, be));
  int iters = 0;
  dbfft_status st = pcg(ctx, o, &iters);
  ctx->trace_n = std::min(ctx->trace_cap, ctx->trace_n + iters + 1);
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
  CKS(copy_vec_all(ctx, &Slab::u, &Slab::x));
  CKS(copy_vec_all(ctx, &Slab::u_c, &Slab::x));
  for (int a = 0; a < 9; ++a) ctx->Fbar[a] = ctx->Fbar_c[a] = epsU[a] + ctx->h_cg->xe[a];
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

// ---------------------------------------------------------------- Newton
// constitutive pass: state += grad(du) + dF ; P, K ; b = F(div P) ; returns <P>, max|d|
dbfft_status constitutive(dbfft_ctx ctx, bool has_in, const double* dF_host, double dt, double* meanP, double* maxd) {
  Nvtx range("constitutive_update");
  const bool fin = ctx->kin == 9;
  CKS(upload_e(ctx, dF_host));
  for (Slab& s : ctx->slabs) CK(cudaMemsetAsync(s.bad, 0x7f, sizeof(int), ctx->stream));
  if (has_in) {
    const int nf1 = nf_I1(ctx);
    for (Slab& s : ctx->slabs) CKS(run_col(ctx, fin ? COL_I1F : COL_I1S, PK_I1, geom_I1(ctx, s, s.x, s.WS1, nf1), ctx->n3));
    CKS(exchange(ctx, (long long)nf1 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
    for (Slab& s : ctx->slabs)
      CKS(run_col(ctx, fin ? COL_I2F : COL_I2S, PK_I2, geom_I2(ctx, s, s.WR, s.WBX, nf1, nf_B(ctx)), ctx->n2));
    CKS(xchg_row(ctx, nf_B(ctx)));
  }
  std::vector<int> grids(ctx->slabs.size());
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    Slab& s = ctx->slabs[k];
    XGeom gx = xgeom(ctx, s, s.WB, s.WBX, nf_B(ctx), nf_B(ctx));
    gx.e = s.e_dev;
    gx.has_in = has_in ? 1 : 0;
    gx.dt = dt;
    CKS(run_x(ctx, fin ? X_CONST_FIN : X_CONST_J2, PK_XCONST, gx, &grids[k]));
  }
  CKS(forward_tail(ctx));
  double red[10];
  CKS(reduce_x(ctx, grids, red, true));
  for (int a = 0; a < 9; ++a) meanP[a] = red[a] / (double)ctx->N;
  if (!fin) sym_fill(meanP);
  *maxd = red[9];
  int bad = 0x7f7f7f7f;
  for (Slab& s : ctx->slabs) {
    CK(cudaMemcpy(ctx->h_bad, s.bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (*ctx->h_bad != 0x7f7f7f7f && bad == 0x7f7f7f7f) bad = (int)global_voxel(ctx, s, *ctx->h_bad);
  }
  if (bad != 0x7f7f7f7f) {
    *ctx->h_bad = bad;
    ctx->err = "det F <= 0 at voxel " + std::to_string(bad);
    return DBFFT_E_MATERIAL;
  }
  return DBFFT_OK;
}

int state_fields(dbfft_ctx ctx) { return ctx->kin == 9 ? 9 : 6; }

dbfft_status rollback(dbfft_ctx ctx) {
  const int nf = state_fields(ctx);
  for (Slab& s : ctx->slabs) {
    CK(cudaMemcpyAsync(s.u, s.u_c, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(s.F, s.F_c, sizeof(double) * nf * s.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  memcpy(ctx->Fbar, ctx->Fbar_c, sizeof(ctx->Fbar));
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status solve_newton(dbfft_ctx ctx, const double* target, const uint8_t* mask, double dt, const dbfft_opts& o,
                          dbfft_report* rep) {
  const bool fin = ctx->kin == 9;
  const int nf = state_fields(ctx);
  for (Slab& s : ctx->slabs) {  // start from the committed state
    CK(cudaMemcpyAsync(s.u, s.u_c, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(s.F, s.F_c, sizeof(double) * nf * s.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  double Fbar_new[9], dF[9], Pf[9];
  for (int a = 0; a < 9; ++a) {
    Fbar_new[a] = mask[a] ? ctx->Fbar_c[a] : target[a];  // F^0 = Fbar^{k+1} + grad u^k
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
    Nvtx range("newton_iteration");
    // preconditioner refresh policy ("computed at the beginning of the increment ... can be
    // recomputed once in a while"; "computed with the initial tangent stiffness")
    if (o.precond_refresh == 2) {
      if (newton == 0) {
        memcpy(ctx->Cbar, ctx->Cbar_init, sizeof(ctx->Cbar));
        st = set_prec(ctx, ctx->Cbar);
        if (st != DBFFT_OK) break;
      }
    } else if (o.precond_refresh == 1 || (newton == 0 && (o.precond_refresh == 0 || ctx->n_incr % o.precond_period == 0))) {
      st = refresh_mean_tangent(ctx);
      if (st != DBFFT_OK) break;
    }
    double be[9];
    for (int a = 0; a < 9; ++a) be[a] = mask[a] ? Pf[a] - meanP[a] : 0.0;
    st = cg_setup(ctx, o, mask, meanP, be);
    if (st != DBFFT_OK) break;
    int iters = 0;
    st = pcg(ctx, o, &iters);
    ctx->trace_n = std::min(ctx->trace_cap, ctx->trace_n + iters + 1);
    total_cg += iters;
    if (st != DBFFT_OK) break;
    for (Slab& s : ctx->slabs) {  // u += du
      ProfScope ps(ctx, PK_OTHER);
      CK(launch_axpy(spec(ctx, s), s.u, s.x, 1.0, ctx->stream));
    }
    double de[9];
    for (int a = 0; a < 9; ++a) {  // Fbar_f += dF_f
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
  for (Slab& s : ctx->slabs) {  // commit (state accepted)
    CK(cudaMemcpyAsync(s.u_c, s.u, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(s.F_c, s.F, sizeof(double) * nf * s.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
    if (!fin) CK(cudaMemcpyAsync(s.epsp_c, s.epsp_t, sizeof(double) * 6 * s.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  memcpy(ctx->Fbar_c, ctx->Fbar, sizeof(ctx->Fbar));
  ++ctx->n_incr;
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

void free_slab(dbfft_ctx ctx, Slab& s) {
  void* ptrs[] = {s.x, s.r, s.p, s.q, s.b, s.u, s.u_c, s.WA, s.WB, s.phase, s.ptable, s.F, s.F_c, s.epsp_c, s.epsp_t, s.tan,
                  s.cg, s.part_x, s.part_cg, s.part_misc, s.loc, s.e_dev, s.bad, s.counts, s.tmp_real};
  for (void* p : ptrs) dfree(ctx, p);
  if (!ctx->peer && s.WR && s.WR != s.WA) dfree(ctx, s.WR);
  if (s.WBX && s.WBX != s.WB) dfree(ctx, s.WBX);
}

void free_all(dbfft_ctx ctx) {
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);  // an external allocator may reuse the memory at once
  for (Slab& s : ctx->slabs) free_slab(ctx, s);
  peer_free(&ctx->pb1);
  peer_free(&ctx->pb2);
  peer_free(&ctx->pbf);
  for (auto* lg : {ctx->loop, ctx->rounds})
    for (int k = 0; k < 4; ++k)
      if (lg[k].exec) cudaGraphExecDestroy(lg[k].exec);
  void* ptrs[] = {ctx->xix, ctx->xiy, ctx->xiz, ctx->tw1, ctx->tw2, ctx->tw3, ctx->loc_ptrs, ctx->trace_dev, ctx->prec_dev};
  for (void* p : ptrs) dfree(ctx, p);
  if (ctx->h_cg) cudaFreeHost(ctx->h_cg);
  if (ctx->h_red) cudaFreeHost(ctx->h_red);
  if (ctx->h_bad) cudaFreeHost(ctx->h_bad);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(ctx->comm);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
}

void free_state(dbfft_ctx ctx, Slab& s) {
  double** ptrs[] = {&s.F, &s.F_c, &s.epsp_c, &s.epsp_t, &s.tan};
  for (double** p : ptrs) {
    dfree(ctx, *p);
    *p = nullptr;
  }
}

dbfft_status ensure_tmp(dbfft_ctx ctx, Slab& s) {
  if (!s.tmp_real) CKS(dalloc(ctx, &s.tmp_real, 9 * s.Nloc));
  return DBFFT_OK;
}

// A rank's real block [zl][yr][x] (nzl rows of nyr n1 contiguous elements) <-> its place in a
// global [z][y][x] array at (z0, y0, 0) (loopback API); z-slabs: one contiguous block
cudaError_t real_block_copy(dbfft_ctx ctx, const Slab& s, void* dst, const void* src, size_t esz, bool to_global, cudaMemcpyKind kind) {
  const size_t row = esz * (size_t)s.nyr * ctx->n1, plane = esz * (size_t)ctx->n1 * ctx->n2;
  const size_t goff = esz * ((size_t)s.z0 * ctx->n1 * ctx->n2 + (size_t)s.y0 * ctx->n1);
  if (to_global) return cudaMemcpy2DAsync((char*)dst + goff, plane, src, row, row, s.nzl, kind, ctx->stream);
  return cudaMemcpy2DAsync(dst, row, (const char*)src + goff, plane, row, s.nzl, kind, ctx->stream);
}
// global voxel index of the rank's local voxel v (line-major [zl][yr][x])
long long global_voxel(dbfft_ctx ctx, const Slab& s, long long v) {
  const long long rowv = (long long)s.nyr * ctx->n1;
  return ((long long)s.z0 + v / rowv) * ctx->n1 * ctx->n2 + (long long)s.y0 * ctx->n1 + v % rowv;
}

// Real fields: the loopback API exposes global [c][z][y][x] arrays; with NCCL each rank passes
// its own block [c][zl][yr][x] (z-slabs: [c][zl][y][x]).
dbfft_status scatter_real(dbfft_ctx ctx, const double* src, int on_device, int ncomp, const int* comp_map, double* Slab::*dst) {
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const long long Nsrc = ctx->loopback ? ctx->N : ctx->slabs[0].Nloc;
  for (Slab& s : ctx->slabs) {
    for (int c = 0; c < ncomp; ++c) {
      const int sc = comp_map ? comp_map[c] : c;
      if (ctx->loopback) CK(real_block_copy(ctx, s, s.*dst + (long long)c * s.Nloc, src + (long long)sc * Nsrc, sizeof(double), false, kind));
      else CK(cudaMemcpyAsync(s.*dst + (long long)c * s.Nloc, src + (long long)sc * Nsrc, sizeof(double) * s.Nloc, kind, ctx->stream));
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status gather_real(dbfft_ctx ctx, double* Slab::*srcm, int ncomp, double* out, int out_on_device) {
  const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const long long Ndst = ctx->loopback ? ctx->N : ctx->slabs[0].Nloc;
  for (Slab& s : ctx->slabs) {
    for (int c = 0; c < ncomp; ++c) {
      if (ctx->loopback) CK(real_block_copy(ctx, s, out + (long long)c * Ndst, s.*srcm + (long long)c * s.Nloc, sizeof(double), true, kind));
      else CK(cudaMemcpyAsync(out + (long long)c * Ndst, s.*srcm + (long long)c * s.Nloc, sizeof(double) * s.Nloc, kind, ctx->stream));
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

// spectral vectors [3][ky][kz][kx]: loopback API vectors are global [3][n2][n3][n1/2+1], a rank
// owns ky in [ky0, ky0 + nyl) and (pencils) the kx columns [kx0, kx0 + kxm) plus the Nyquist on
// the last row rank; its local layout [3][nyl][n3][nkx] keeps the padding column at zero
long long spec_cols(dbfft_ctx ctx, const Slab& s) {
  return ctx->Py == 1 ? ctx->n1h : ctx->kxm + (s.pa == ctx->Py - 1 ? 1 : 0);
}
dbfft_status spec_in(dbfft_ctx ctx, const cplx* src, cplx* Slab::*dst) {
  const long long Hs_glob = (long long)ctx->n1h * ctx->n2 * ctx->n3;
  for (Slab& s : ctx->slabs) {
    if (!ctx->loopback) {
      CK(cudaMemcpyAsync(s.*dst, src, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToDevice, ctx->stream));
      continue;
    }
    if (ctx->Py > 1) CK(cudaMemsetAsync(s.*dst, 0, sizeof(cplx) * 3 * s.Hs, ctx->stream));
    for (int c = 0; c < 3; ++c)
      CK(cudaMemcpy2DAsync(s.*dst + c * s.Hs, sizeof(cplx) * ctx->nkx, src + c * Hs_glob + (long long)s.ky0 * ctx->n3 * ctx->n1h + s.kx0,
                           sizeof(cplx) * ctx->n1h, sizeof(cplx) * spec_cols(ctx, s), (size_t)s.nyl * ctx->n3,
                           cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return DBFFT_OK;
}
dbfft_status spec_out(dbfft_ctx ctx, cplx* Slab::*srcm, cplx* dst, cudaMemcpyKind kind) {
  const long long Hs_glob = (long long)ctx->n1h * ctx->n2 * ctx->n3;
  for (Slab& s : ctx->slabs) {
    if (!ctx->loopback) {
      CK(cudaMemcpyAsync(dst, s.*srcm, sizeof(cplx) * 3 * s.Hs, kind, ctx->stream));
      continue;
    }
    for (int c = 0; c < 3; ++c)
      CK(cudaMemcpy2DAsync(dst + c * Hs_glob + (long long)s.ky0 * ctx->n3 * ctx->n1h + s.kx0, sizeof(cplx) * ctx->n1h,
                           s.*srcm + c * s.Hs, sizeof(cplx) * ctx->nkx, sizeof(cplx) * spec_cols(ctx, s), (size_t)s.nyl * ctx->n3,
                           kind, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status alloc_slab(dbfft_ctx ctx, Slab& s) {
  const size_t v3 = 3 * s.Hs;
  cplx** vecs[] = {&s.x, &s.r, &s.p, &s.q, &s.b, &s.u, &s.u_c};
  for (cplx** v : vecs) CKS(dalloc(ctx, v, v3));
  CK(cudaMemset(s.u, 0, sizeof(cplx) * v3));
  CK(cudaMemset(s.u_c, 0, sizeof(cplx) * v3));
  CKS(dalloc(ctx, &s.WA, (size_t)6 * s.Hsp));
  if (ctx->Pz == 1) s.WR = s.WA;
  else if (!ctx->peer) CKS(dalloc(ctx, &s.WR, (size_t)6 * s.Hsp));
  // peer transport: WR / WR2 / WS1 / WS2 are mapped by build_peer once all slabs exist
  s.WS1 = s.WS2 = s.WA;
  s.WR2 = s.WR;
  CKS(dalloc(ctx, &s.WB, (size_t)ctx->kin * s.Hsp));
  if (ctx->Py > 1) CKS(dalloc(ctx, &s.WBX, (size_t)ctx->kin * s.Hsp));
  else s.WBX = s.WB;
  CKS(dalloc(ctx, &s.cg, 1));
  int gx = 0;
  for (int k = 0; k < X_REAL_OUT; ++k) gx = std::max(gx, x_grid(k, ctx->n1, s.nlines));
  CKS(dalloc(ctx, &s.part_x, (size_t)gx * 10));
  CKS(dalloc(ctx, &s.part_cg, (size_t)cg_blocks() * 2));
  CKS(dalloc(ctx, &s.part_misc, (size_t)cg_blocks() * 45));
  CKS(dalloc(ctx, &s.loc, 64));
  CKS(dalloc(ctx, &s.e_dev, 9));
  CKS(dalloc(ctx, &s.bad, 1));
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
  o.precond_period = 1;
  o.precond_medium = 0;
  return o;
}

const char* dbfft_last_error(dbfft_ctx ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

dbfft_status dbfft_nccl_unique_id(void* out128) {
  if (!out128) return DBFFT_E_INVALID_ARG;
  std::string err;
  if (!nccl_load(&err)) {
    g_create_error = err;
    return DBFFT_E_NCCL;
  }
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) {
    g_create_error = "ncclGetUniqueId failed";
    return DBFFT_E_NCCL;
  }
  memcpy(out128, &id, sizeof(id));
  return DBFFT_OK;
}

// peer transport: the two exchange buffers as VMM windows over all ranks (peer.cuh), plus the
// barrier flags (NCCL mode only: loopback ranks share one stream)
static int g_peer_seq = 0;
static dbfft_status build_peer(dbfft_ctx ctx, const void* nccl_id) {
  std::string err;
  if (ctx->P > 32) {  // the barrier kernel runs one warp, one lane per rank
    ctx->err = "peer transport: at most 32 ranks";
    return DBFFT_E_INVALID_ARG;
  }
  const Slab& s0 = ctx->slabs[0];
  const size_t chunk = peer_chunk(sizeof(cplx) * 6 * (size_t)s0.nyl * s0.nzl * ctx->kxp, ctx->device, &err);
  const size_t fchunk = chunk ? peer_chunk(4096, ctx->device, &err) : 0;
  bool ok = chunk && fchunk;
  if (ok && ctx->loopback) {
    ok = peer_build_loopback(&ctx->pb1, ctx->P, chunk, ctx->device, true, false, &err) &&
         peer_build_loopback(&ctx->pb2, ctx->P, chunk, ctx->device, true, false, &err);
  } else if (ok) {
    // rendezvous tag: a hash of the job's NCCL unique id (equal on all ranks) + a per-process
    // sequence number (all ranks create their contexts in the same order)
    unsigned long long h = 1469598103934665603ull;
    const unsigned char* b = static_cast<const unsigned char*>(nccl_id);
    for (int i = 0; i < 128; ++i) h = (h ^ b[i]) * 1099511628211ull;
    char tag[64];
    snprintf(tag, sizeof(tag), "%016llx-%d", h, g_peer_seq++);
    ok = peer_build_ipc(&ctx->pbf, ctx->P, ctx->rank, fchunk, ctx->device, false, true, std::string(tag) + "-f", &err) &&
         peer_build_ipc(&ctx->pb1, ctx->P, ctx->rank, chunk, ctx->device, true, false, std::string(tag) + "-1", &err) &&
         peer_build_ipc(&ctx->pb2, ctx->P, ctx->rank, chunk, ctx->device, true, false, std::string(tag) + "-2", &err);
  }
  if (!ok) {
    ctx->err = err;
    return DBFFT_E_CUDA;
  }
  ctx->xpcs = (long long)(chunk / sizeof(cplx));
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    Slab& s = ctx->slabs[k];
    s.WR = reinterpret_cast<cplx*>(ctx->pb1.recv[k]);
    s.WS1 = reinterpret_cast<cplx*>(ctx->pb1.win[k]);
    s.WR2 = reinterpret_cast<cplx*>(ctx->pb2.recv[k]);
    s.WS2 = reinterpret_cast<cplx*>(ctx->pb2.win[k]);
  }
  return DBFFT_OK;
}

dbfft_status dbfft_create(const int32_t n[3], const double L[3], int32_t kinematics, const dbfft_env* env, dbfft_ctx* out) {
  if (!n || !L || !out) {
    g_create_error = "null argument";
    return DBFFT_E_INVALID_ARG;
  }
  *out = nullptr;
  for (int a = 0; a < 3; ++a)
    if (!is_pow2_in(n[a]) || !(L[a] > 0)) {
      g_create_error = "grid dims must be powers of two in [8,512] or one of 15, 21, 27, 63, and L > 0";
      return DBFFT_E_INVALID_GRID;
    }
  if (kinematics != 6 && kinematics != 9) {
    g_create_error = "kinematics must be 6 (small strain) or 9 (finite strain)";
    return DBFFT_E_INVALID_ARG;
  }
  const int P = env ? std::max(1, env->world) : 1;
  const int rank = env ? env->rank : 0;
  const int loopback = env ? env->loopback : 0;
  const int Py = (env && env->pencil_rows > 1) ? env->pencil_rows : 1;
  const int Pz = P / Py;
  if ((P & (P - 1)) != 0 || (Py & (Py - 1)) != 0 || Py > P || n[1] % Pz != 0 || n[2] % Pz != 0 || rank < 0 || rank >= P) {
    g_create_error = "world and pencil_rows must be powers of two, world / pencil_rows dividing n2 and n3 (S:48), 0 <= rank < world";
    return DBFFT_E_INVALID_GRID;
  }
  if (Py > 1 && (!is_pow2_in(n[0]) || (n[0] & (n[0] - 1)) != 0 || n[0] / 2 < Py || n[1] % Py != 0)) {
    g_create_error = "pencil_rows > 1: n1 a power of two with n1/2 >= pencil_rows, pencil_rows dividing n2";
    return DBFFT_E_INVALID_GRID;
  }
  if (Py > 1 && env && env->transport == DBFFT_TRANSPORT_PEER) {
    g_create_error = "pencil_rows > 1 runs on the NCCL transport (the peer windows are built for z-slabs)";
    return DBFFT_E_INVALID_ARG;
  }
  if (P > 1 && !loopback && !env->nccl_id) {
    g_create_error = "world > 1 needs env->nccl_id (dbfft_nccl_unique_id on rank 0, broadcast) or env->loopback";
    return DBFFT_E_INVALID_ARG;
  }
  dbfft_ctx ctx = new dbfft_ctx_s();
  ctx->n1 = n[0];
  ctx->n2 = n[1];
  ctx->n3 = n[2];
  ctx->n1h = n[0] / 2 + 1;
  {
    // 128-byte aligned rows (the local kx count rounded up to 8) in the intermediate layouts
    // X1, B, X2: a dense 129-column row starts 16 bytes off the 128-byte grid, so a 128-byte TMA
    // row touches 5 DRAM sectors (ncu: column-pass reads 8-12 % above the algorithmic bytes).
    // B200 (tools/ab_promo_pad.sh): 256^3 finite apply_K 2.319 -> 2.301 ms (I1 0.271 -> 0.260,
    // I2 0.426 -> 0.420), small 1.892 -> 1.876, 128^3 0.365 -> 0.362; but at n1 = 512 the
    // direct-store y-forward pass slows (2.90 -> 3.22 ms), so the default pads for n1 <= 256.
    // DBFFT_KX_PAD=1 / =0 forces either (the full GPU suite passes with both).
    const char* e = getenv("DBFFT_KX_PAD");
    const bool pad = e ? e[0] == '1' : n[0] <= 256;
    ctx->Py = Py;
    ctx->Pz = Pz;
    ctx->kxm = Py > 1 ? n[0] / (2 * Py) : 0;
    ctx->nkx = Py > 1 ? ctx->kxm + 1 : ctx->n1h;
    ctx->kxp = pad ? (ctx->nkx + 7) / 8 * 8 : ctx->nkx;
  }
  for (int a = 0; a < 3; ++a) ctx->L[a] = L[a];
  ctx->kin = kinematics;
  ctx->N = (long long)n[0] * n[1] * n[2];
  ctx->P = P;
  ctx->loopback = (P > 1 && loopback) ? 1 : 0;
  ctx->rank = ctx->loopback ? 0 : rank;
  ctx->peer = (P > 1 && env && env->transport == DBFFT_TRANSPORT_PEER) ? 1 : 0;
  if (env && (env->dev_alloc != nullptr) != (env->dev_free != nullptr)) {
    g_create_error = "env: dev_alloc and dev_free must be given together";
    delete ctx;
    return DBFFT_E_INVALID_ARG;
  }
  if (env) {
    ctx->dev_alloc = env->dev_alloc;
    ctx->dev_free = env->dev_free;
    ctx->alloc_user = env->alloc_user;
  }
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
    // a blocking stream: work a caller issues on the legacy default stream (NULL) is ordered
    // with the context's kernels, and events recorded there bracket them
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault) != cudaSuccess) {
      ctx->err = "cudaStreamCreate failed (no CUDA device?)";
      return fail(DBFFT_E_CUDA);
    }
    ctx->own_stream = true;
  }
  if (const char* xo = getenv("DBFFT_XOVERLAP")) {
    ctx->xoverlap = std::min(4, std::max(0, atoi(xo)));
    if (ctx->xoverlap && (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
                          cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                          cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess)) {
      ctx->err = "DBFFT_XOVERLAP: side stream / events could not be created";
      return fail(DBFFT_E_CUDA);
    }
  }
  dbfft_status s;
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
  // slabs: loopback holds all P virtual ranks, NCCL mode holds this rank's slab
  const int nslab = ctx->loopback ? P : 1;
  ctx->slabs.resize(nslab);
  for (int k = 0; k < nslab; ++k) {
    Slab& sl = ctx->slabs[k];
    sl.rank = ctx->loopback ? k : rank;
    sl.pa = sl.rank % Py;  // pencil grid position, rank = b Py + a
    sl.pb = sl.rank / Py;
    sl.nyl = n[1] / Pz;
    sl.nzl = n[2] / Pz;
    sl.ky0 = sl.pb * sl.nyl;
    sl.z0 = sl.pb * sl.nzl;
    sl.nyr = n[1] / Py;
    sl.y0 = sl.pa * sl.nyr;
    sl.kx0 = sl.pa * ctx->kxm;
    sl.Hs = (long long)ctx->nkx * sl.nyl * n[2];
    sl.Hsp = (long long)ctx->kxp * sl.nyl * n[2];
    sl.fsB = (long long)sl.nzl * sl.nyr * ctx->kxp;
    sl.Nloc = (long long)n[0] * sl.nyr * sl.nzl;
    sl.nlines = (long long)sl.nyr * sl.nzl;
    sl.xiy = ctx->xiy + sl.ky0;
    if ((s = alloc_slab(ctx, sl)) != DBFFT_OK) return fail(s);
  }
  if ((s = dalloc(ctx, &ctx->prec_dev, 1)) != DBFFT_OK) return fail(s);
  if (ctx->loopback) {  // the slabs' loc buffers for the loopback all-reduce kernel
    if ((s = dalloc(ctx, &ctx->loc_ptrs, P)) != DBFFT_OK) return fail(s);
    std::vector<double*> h(P);
    for (int r = 0; r < P; ++r) h[r] = ctx->slabs[r].loc;
    if (cudaMemcpy(ctx->loc_ptrs, h.data(), sizeof(double*) * P, cudaMemcpyHostToDevice) != cudaSuccess) {
      ctx->err = "create: loc pointer upload failed";
      return fail(DBFFT_E_CUDA);
    }
  }
  if (P > 1 && !ctx->loopback) {
    std::string err;
    if (!nccl_load(&err)) {
      ctx->err = err;
      return fail(DBFFT_E_NCCL);
    }
    ncclUniqueId id;
    memcpy(&id, env->nccl_id, sizeof(id));
    if (g_nccl.CommInitRank(&ctx->comm, P, id, rank) != ncclSuccess) {
      ctx->err = "ncclCommInitRank failed";
      return fail(DBFFT_E_NCCL);
    }
  }
  if (ctx->peer && (s = build_peer(ctx, env->nccl_id)) != DBFFT_OK) return fail(s);
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

dbfft_status dbfft_fd_allgather(const char* tag, int32_t rank, int32_t world, const int32_t* fds, int32_t nfd,
                                int32_t* out, int32_t timeout_ms) {
  if (!tag || !fds || !out || world < 1 || rank < 0 || rank >= world || nfd < 1 || nfd > 16 || timeout_ms < 0) {
    g_create_error = "fd_allgather: bad arguments";
    return DBFFT_E_INVALID_ARG;
  }
  std::string err;
  if (fd_allgather(tag, rank, world, fds, nfd, out, timeout_ms, &err) != 0) {
    g_create_error = err;
    return DBFFT_E_STATE;
  }
  return DBFFT_OK;
}

// ---------------------------------------------------------------- peer-window probe (tests)
__global__ void k_peer_fill(unsigned* win, size_t chunk_words, int P, unsigned base, int nwords) {
  for (int i = threadIdx.x; i < P * nwords; i += blockDim.x) {
    const int d = i / nwords;
    win[(size_t)d * chunk_words + i % nwords] = base + d;
  }
}

struct dbfft_peer_probe_s {
  PeerBuf b;
  int rank = 0, P = 1;
};

dbfft_status dbfft_peer_probe_open(const char* tag, int32_t rank, int32_t world, int32_t device, void** out) {
  if (!tag || !out || world < 1 || rank < 0 || rank >= world) {
    g_create_error = "peer_probe_open: bad arguments";
    return DBFFT_E_INVALID_ARG;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    g_create_error = "peer_probe_open: cudaSetDevice";
    return DBFFT_E_CUDA;
  }
  auto* pr = new dbfft_peer_probe_s();
  pr->rank = rank;
  pr->P = world;
  std::string err;
  const size_t chunk = peer_chunk(4096, device, &err);
  if (!chunk || !peer_build_ipc(&pr->b, world, rank, chunk, device, true, true, tag, &err)) {
    g_create_error = err;
    peer_free(&pr->b);
    delete pr;
    return DBFFT_E_CUDA;
  }
  // store 1000 rank + d into the first 1024 words of window chunk d (rank d's buffer, chunk rank)
  k_peer_fill<<<1, 256>>>(reinterpret_cast<unsigned*>(pr->b.win[0]), chunk / 4, world, 1000u * rank, 1024);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    g_create_error = "peer_probe_open: fill kernel failed";
    peer_free(&pr->b);
    delete pr;
    return DBFFT_E_CUDA;
  }
  *out = pr;
  return DBFFT_OK;
}

dbfft_status dbfft_peer_probe_check(void* h, int32_t* bad_words) {
  auto* pr = static_cast<dbfft_peer_probe_s*>(h);
  if (!pr || !bad_words) return DBFFT_E_INVALID_ARG;
  std::vector<unsigned> host(1024);
  int bad = 0;
  for (int src = 0; src < pr->P; ++src) {
    if (cudaMemcpy(host.data(), reinterpret_cast<char*>(pr->b.recv[0]) + (size_t)src * pr->b.chunk, 4096,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      return DBFFT_E_CUDA;
    for (unsigned w : host) bad += (w != 1000u * src + pr->rank);
  }
  *bad_words = bad;
  return DBFFT_OK;
}

dbfft_status dbfft_peer_probe_close(void* h) {
  auto* pr = static_cast<dbfft_peer_probe_s*>(h);
  if (!pr) return DBFFT_E_INVALID_ARG;
  cudaDeviceSynchronize();
  peer_free(&pr->b);
  delete pr;
  return DBFFT_OK;
}

dbfft_status dbfft_destroy(dbfft_ctx ctx) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_all(ctx);
  delete ctx;
  return DBFFT_OK;
}

dbfft_status dbfft_spectral_layout(dbfft_ctx ctx, int64_t shape[4], int64_t strides[4]) {
  if (!ctx || !shape || !strides) return DBFFT_E_INVALID_ARG;
  const int nyl = ctx->loopback ? ctx->n2 : ctx->slabs[0].nyl;  // loopback API vectors are global
  const int nkx = ctx->loopback ? ctx->n1h : ctx->nkx;          // NCCL pencils: the local kx block
  shape[0] = 3;
  shape[1] = nyl;
  shape[2] = ctx->n3;
  shape[3] = nkx;
  strides[3] = 1;
  strides[2] = nkx;
  strides[1] = (int64_t)ctx->n3 * nkx;
  strides[0] = (int64_t)nyl * ctx->n3 * nkx;
  return DBFFT_OK;
}

// captured PCG loops bake buffer pointers in: rebuild them only if set_phases moved one
static void bump_gen_if_moved(dbfft_ctx ctx, const std::vector<const void*>& before) {
  size_t i = 0;
  bool moved = false;
  for (Slab& sl : ctx->slabs)
    for (const void* q : {(const void*)sl.phase, (const void*)sl.ptable, (const void*)sl.counts, (const void*)sl.F,
                          (const void*)sl.F_c, (const void*)sl.tan, (const void*)sl.epsp_c, (const void*)sl.epsp_t})
      moved |= (i < before.size() ? before[i++] : nullptr) != q;
  if (moved) ++ctx->gen;
}

dbfft_status dbfft_set_phases(dbfft_ctx ctx, const uint16_t* phase_id, int32_t on_device, int32_t n_phases, const dbfft_material* table) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (!phase_id || !table || n_phases <= 0 || n_phases > 65535) {
    ctx->err = "set_phases: bad arguments";
    return DBFFT_E_INVALID_ARG;
  }
  int fam = FAM_NONE;
  bool has_svk = false;
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
        if (!(m.p[0] > 0)) { ctx->err = "NEOHOOKE: need mu > 0"; return DBFFT_E_INVALID_ARG; }
        d[0] = m.p[0];
        d[1] = m.p[1];
        d[2] = 0.0;  // model flag: neo-Hookean
        d[3] = m.p[1] - 2.0 * m.p[0] / 3.0;  // lam = kappa - 2 mu / 3 (R14), once per phase
        f = FAM_NEOHOOKE;
        break;
      case DBFFT_MAT_SVK:
        if (!(m.p[0] > 0) || !(m.p[1] > -1.0 && m.p[1] < 0.5)) { ctx->err = "SVK: need E > 0, -1 < nu < 0.5"; return DBFFT_E_INVALID_ARG; }
        d[0] = m.p[0] / (2.0 * (1.0 + m.p[1]));                         // mu
        d[1] = m.p[0] * m.p[1] / ((1.0 + m.p[1]) * (1.0 - 2.0 * m.p[1]));  // lam
        d[2] = 1.0;  // model flag: Saint Venant-Kirchhoff
        f = FAM_NEOHOOKE;  // finite-strain hyperelastic family
        has_svk = true;
        break;
      case DBFFT_MAT_J2:
        if (!(m.p[0] > 0) || !(m.p[1] > -1.0 && m.p[1] < 0.5) || !(m.p[2] > 0) || !(m.p[3] > 0) || !(m.p[4] > 0)) {
          ctx->err = "J2: need E > 0, -1 < nu < 0.5, sigma_y, n, edot0 > 0";
          return DBFFT_E_INVALID_ARG;
        }
        for (int a = 0; a < 5; ++a) d[a] = m.p[a];
        {  // shear and bulk moduli for the kernels (passes.cu j2_moduli / j2_update)
          const double E = m.p[0], nu = m.p[1];
          const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
          d[5] = E / (2.0 * (1.0 + nu));
          d[6] = lam + 2.0 * d[5] / 3.0;
        }
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
    ctx->err = "NEOHOOKE/SVK require a finite-strain context; ISO/CUBIC/J2 a small-strain one";
    return DBFFT_E_INVALID_ARG;
  }
  dbfft_status s;
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  // buffers are reused when they fit (pointers stable: the captured PCG loop graphs stay valid,
  // e.g. for a new load walk on the same grid); `gen` moves only if a pointer changed
  std::vector<const void*> before;
  for (Slab& sl : ctx->slabs)
    for (const void* q : {(const void*)sl.phase, (const void*)sl.ptable, (const void*)sl.counts, (const void*)sl.F,
                          (const void*)sl.F_c, (const void*)sl.tan, (const void*)sl.epsp_c, (const void*)sl.epsp_t})
      before.push_back(q);
  CK(cudaStreamSynchronize(ctx->stream));  // kernels still reading the old table / counts
  for (Slab& sl : ctx->slabs) {
    if (!sl.phase && (s = dalloc(ctx, &sl.phase, sl.Nloc)) != DBFFT_OK) return s;
    if (ctx->loopback) CK(real_block_copy(ctx, sl, sl.phase, phase_id, sizeof(uint16_t), false, kind));
    else CK(cudaMemcpyAsync(sl.phase, phase_id, sizeof(uint16_t) * sl.Nloc, kind, ctx->stream));
    if (sl.cap_ptable < pt.size()) {
      dfree(ctx, sl.ptable);
      sl.ptable = nullptr;
      if ((s = dalloc(ctx, &sl.ptable, pt.size())) != DBFFT_OK) return s;
      sl.cap_ptable = pt.size();
    }
    CK(cudaMemcpyAsync(sl.ptable, pt.data(), sizeof(double) * pt.size(), cudaMemcpyHostToDevice, ctx->stream));
    if (sl.cap_counts < (size_t)n_phases) {
      dfree(ctx, sl.counts);
      sl.counts = nullptr;
      if ((s = dalloc(ctx, &sl.counts, n_phases)) != DBFFT_OK) return s;
      sl.cap_counts = n_phases;
    }
    CK(cudaMemsetAsync(sl.counts, 0, sizeof(double) * n_phases, ctx->stream));
    CK(cudaMemsetAsync(sl.bad, 0, sizeof(int), ctx->stream));
    CK(launch_phase_hist(sl.phase, sl.Nloc, sl.counts, n_phases, sl.bad, ctx->stream));
  }
  for (Slab& sl : ctx->slabs) {
    CK(cudaMemcpyAsync(ctx->h_bad, sl.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_bad) {
      ctx->err = "phase id >= n_phases";
      return DBFFT_E_INVALID_ARG;
    }
  }
  // phase counts (for the linear mean stiffness) summed over ranks
  if (ctx->P > 1 && !ctx->loopback)
    CKN(g_nccl.AllReduce(ctx->slabs[0].counts, ctx->slabs[0].counts, n_phases, ncclFloat64, ncclSum, ctx->comm, ctx->stream));
  std::vector<double> cnt(n_phases, 0.0);
  for (Slab& sl : ctx->slabs) {
    std::vector<double> c(n_phases);
    CK(cudaMemcpyAsync(c.data(), sl.counts, sizeof(double) * n_phases, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < n_phases; ++k) cnt[k] += c[k];
  }
  ctx->h_ptable = pt;
  ctx->nph = n_phases;
  ctx->family = fam;
  {
    // per-voxel state of the new family: kept when the same fields are allocated already
    const char* tm = getenv("DBFFT_TANGENT");
    ctx->tmode = ((tm && strcmp(tm, "full") == 0) || has_svk) ? 0 : 1;
    const int nf = fam == FAM_NEOHOOKE ? 9 : fam == FAM_J2 ? 6 : 0;
    const int nk = fam == FAM_NEOHOOKE ? (ctx->tmode ? 10 : 45) : fam == FAM_J2 ? 8 : 0;
    for (Slab& sl : ctx->slabs) {
      if (sl.state_nf != nf || sl.state_nk != nk || (fam == FAM_J2) != (sl.epsp_c != nullptr)) {
        free_state(ctx, sl);
        sl.state_nf = sl.state_nk = 0;
      }
      CK(cudaMemsetAsync(sl.u, 0, sizeof(cplx) * 3 * sl.Hs, ctx->stream));
      CK(cudaMemsetAsync(sl.u_c, 0, sizeof(cplx) * 3 * sl.Hs, ctx->stream));
    }
  }
  for (int a = 0; a < 9; ++a) ctx->Fbar[a] = ctx->Fbar_c[a] = (fam == FAM_NEOHOOKE && a % 4 == 0) ? 1.0 : 0.0;
  ctx->h_counts = cnt;
  ctx->n_incr = 0;
  if (fam == FAM_LINEAR) {
    bump_gen_if_moved(ctx, before);
    CKS(linear_reference(ctx, 0));
  } else {
    // the matrix-free compact tangent is neo-Hookean's; SVK phases store the 45-entry tangent
    const int nf = fam == FAM_NEOHOOKE ? 9 : 6;
    const int nk = fam == FAM_NEOHOOKE ? (ctx->tmode ? 10 : 45) : 8;
    for (Slab& sl : ctx->slabs) {
      if (!sl.state_nf) {
        if ((s = dalloc(ctx, &sl.F, (size_t)nf * sl.Nloc)) != DBFFT_OK) return s;
        if ((s = dalloc(ctx, &sl.F_c, (size_t)nf * sl.Nloc)) != DBFFT_OK) return s;
        if ((s = dalloc(ctx, &sl.tan, (size_t)nk * sl.Nloc)) != DBFFT_OK) return s;
        if (fam == FAM_J2) {
          if ((s = dalloc(ctx, &sl.epsp_c, (size_t)6 * sl.Nloc)) != DBFFT_OK) return s;
          if ((s = dalloc(ctx, &sl.epsp_t, (size_t)6 * sl.Nloc)) != DBFFT_OK) return s;
        }
        sl.state_nf = nf;
        sl.state_nk = nk;
      }
      if (fam == FAM_NEOHOOKE) {
        k_identity9<<<1024, 256, 0, ctx->stream>>>(sl.F_c, sl.Nloc);
        CK(cudaGetLastError());
      } else {
        CK(cudaMemsetAsync(sl.F_c, 0, sizeof(double) * nf * sl.Nloc, ctx->stream));
        CK(cudaMemsetAsync(sl.epsp_c, 0, sizeof(double) * 6 * sl.Nloc, ctx->stream));
        CK(cudaMemsetAsync(sl.epsp_t, 0, sizeof(double) * 6 * sl.Nloc, ctx->stream));
      }
      CK(cudaMemcpyAsync(sl.F, sl.F_c, sizeof(double) * nf * sl.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // tangent at the undeformed state (so apply_K / precond are usable before a solve)
    double zero[9] = {0}, mp[9], mx;
    bump_gen_if_moved(ctx, before);
    s = constitutive(ctx, false, zero, 1.0, mp, &mx);
    if (s != DBFFT_OK) return s;
    s = refresh_mean_tangent(ctx);
    if (s != DBFFT_OK) return s;
    memcpy(ctx->Cbar_init, ctx->Cbar, sizeof(ctx->Cbar));  // refresh policy 2
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status dbfft_apply_K(dbfft_ctx ctx, const void* u_hat, void* f_hat) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (!u_hat || !f_hat || u_hat == f_hat) {
    ctx->err = "apply_K: null or aliased vectors";
    return DBFFT_E_INVALID_ARG;
  }
  if (ctx->family == FAM_NONE) {
    ctx->err = "apply_K before set_phases";
    return DBFFT_E_STATE;
  }
  if (!ctx->loopback) {  // zero-copy on the caller's vectors
    Slab& s = ctx->slabs[0];
    cplx* su = s.p;
    cplx* sf = s.q;
    s.p = (cplx*)u_hat;
    s.q = (cplx*)f_hat;
    dbfft_status st = apply_K_slabs(ctx, &Slab::p, &Slab::q, false, &CgDev::pe, nullptr);
    s.p = su;
    s.q = sf;
    return st;
  }
  CKS(spec_in(ctx, (const cplx*)u_hat, &Slab::p));
  CKS(apply_K_slabs(ctx, &Slab::p, &Slab::q, false, &CgDev::pe, nullptr));
  return spec_out(ctx, &Slab::q, (cplx*)f_hat, cudaMemcpyDeviceToDevice);
}

dbfft_status dbfft_apply_K_aug(dbfft_ctx ctx, const uint8_t mask[9], const void* u_hat, const double e_in[9], void* f_hat, double r_out[9]) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
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
  // the macro block travels in CgDev::pe of every slab
  for (Slab& s : ctx->slabs) CK(cudaMemcpyAsync(&s.cg->pe, e, sizeof(e), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CKS(spec_in(ctx, (const cplx*)u_hat, &Slab::p));
  ApplyOut ao;
  CKS(apply_K_slabs(ctx, &Slab::p, &Slab::q, true, &CgDev::pe, &ao));
  double red[10];
  CKS(reduce_x(ctx, ao.grid_x, red, false));
  for (int a = 0; a < 9; ++a) red[a] /= (double)ctx->N;
  if (ctx->kin == 6) sym_fill(red);
  for (int a = 0; a < 9; ++a) r_out[a] = mask[a] ? red[a] : 0.0;
  return spec_out(ctx, &Slab::q, (cplx*)f_hat, cudaMemcpyDeviceToDevice);
}

dbfft_status dbfft_precond(dbfft_ctx ctx, const void* r_hat, void* z_hat) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (!r_hat || !z_hat) {
    ctx->err = "precond: null vectors";
    return DBFFT_E_INVALID_ARG;
  }
  if (!ctx->prec_valid) {
    ctx->err = "precond before set_phases";
    return DBFFT_E_STATE;
  }
  CKS(spec_in(ctx, (const cplx*)r_hat, &Slab::r));
  for (Slab& s : ctx->slabs) {
    ProfScope ps(ctx, PK_OTHER);
    CK(launch_precond(spec(ctx, s), ctx->prec_dev, s.r, s.q, ctx->stream));
  }
  return spec_out(ctx, &Slab::q, (cplx*)z_hat, cudaMemcpyDeviceToDevice);
}

dbfft_status dbfft_eval_state(dbfft_ctx ctx, const double* field, int32_t on_device, double dt) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (ctx->family == FAM_NONE) {
    ctx->err = "eval_state before set_phases";
    return DBFFT_E_STATE;
  }
  if (ctx->family == FAM_LINEAR) return DBFFT_OK;
  if (!field) {
    ctx->err = "eval_state: null field";
    return DBFFT_E_INVALID_ARG;
  }
  if (ctx->family == FAM_NEOHOOKE) {
    CKS(scatter_real(ctx, field, on_device, 9, nullptr, &Slab::F));
  } else {
    const int rowv[6] = {0, 4, 8, 5, 2, 1};
    CKS(scatter_real(ctx, field, on_device, 6, rowv, &Slab::F));
  }
  double zero[9] = {0}, mp[9], mx;
  CKS(constitutive(ctx, false, zero, dt, mp, &mx));
  CKS(refresh_mean_tangent(ctx));
  return DBFFT_OK;
}

dbfft_status dbfft_solve_increment(dbfft_ctx ctx, const double target[9], const uint8_t mask[9], double dt, const dbfft_opts* opts,
                                   dbfft_report* report) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (ctx->family == FAM_NONE) {
    ctx->err = "solve_increment before set_phases";
    return DBFFT_E_STATE;
  }
  CKS(check_target(ctx, target, mask));
  dbfft_opts o = opts ? *opts : dbfft_default_opts();
  CKS(check_opts(ctx, o));
  if (!ctx->trace_dev) {
    ctx->trace_cap = 1 << 16;
    CKS(dalloc(ctx, &ctx->trace_dev, 2 * (size_t)ctx->trace_cap));
  }
  ctx->trace_n = 0;
  Nvtx range("dbfft_solve_increment");
  auto t0 = std::chrono::steady_clock::now();
  if (report) {
    memset(report, 0, sizeof(*report));
    report->bad_voxel = -1;
  }
  dbfft_status st = (ctx->family == FAM_LINEAR) ? solve_linear(ctx, target, mask, o, report) : solve_newton(ctx, target, mask, dt, o, report);
  prof_flush(ctx);
  if (report) {
    report->status = st;
    report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return st;
}

// committed strain (eps or F) / stress (sigma or P) -> every slab's tmp_real [9][Nloc], row-major 3x3
dbfft_status field_to_tmp(dbfft_ctx ctx, int which) {
  for (Slab& s : ctx->slabs) CKS(ensure_tmp(ctx, s));
  if (ctx->family == FAM_NEOHOOKE) {
    for (Slab& s : ctx->slabs) {
      ProfScope ps(ctx, PK_OTHER);
      if (which == DBFFT_FIELD_STRAIN) {
        CK(cudaMemcpyAsync(s.tmp_real, s.F_c, sizeof(double) * 9 * s.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
      } else {
        k_stress_nh<<<1024, 256, 0, ctx->stream>>>(s.F_c, s.phase, s.ptable, s.Nloc, s.tmp_real);
        CK(cudaGetLastError());
      }
    }
    return DBFFT_OK;
  }
  if (ctx->family == FAM_J2) {
    for (Slab& s : ctx->slabs) {
      ProfScope ps(ctx, PK_OTHER);
      if (which == DBFFT_FIELD_STRAIN) k_expand6<<<1024, 256, 0, ctx->stream>>>(s.F_c, s.Nloc, nullptr, s.tmp_real);
      else k_stress_j2<<<1024, 256, 0, ctx->stream>>>(s.F_c, s.epsp_c, s.phase, s.ptable, s.Nloc, s.tmp_real);
      CK(cudaGetLastError());
    }
    return DBFFT_OK;
  }
  // linear: eps = Ebar + sym grad u (Voigt 6 via the inverse passes), sigma = C:eps
  CKS(upload_e(ctx, ctx->Fbar_c));
  for (Slab& s : ctx->slabs) CKS(run_col(ctx, COL_I1S, PK_OTHER, geom_I1(ctx, s, s.u_c, s.WS1, 5), ctx->n3));
  CKS(exchange(ctx, (long long)5 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
  for (Slab& s : ctx->slabs) CKS(run_col(ctx, COL_I2S, PK_OTHER, geom_I2(ctx, s, s.WR, s.WBX, 5, 6), ctx->n2));
  CKS(xchg_row(ctx, 6));
  for (Slab& s : ctx->slabs) {
    double* tmp6 = reinterpret_cast<double*>(s.WA);  // 6 real fields fit in WA (6 complex fields)
    XGeom gx = xgeom(ctx, s, s.WB, nullptr, 6, 6);
    gx.real_out = tmp6;
    CKS(run_x(ctx, X_REAL_OUT + 6, PK_OTHER, gx, nullptr));
    ProfScope ps(ctx, PK_OTHER);
    k_expand6<<<1024, 256, 0, ctx->stream>>>(tmp6, s.Nloc, s.e_dev, s.tmp_real);
    CK(cudaGetLastError());
    if (which == DBFFT_FIELD_STRESS) {
      k_stress_linear<<<1024, 256, 0, ctx->stream>>>(s.tmp_real, s.phase, s.ptable, s.Nloc, s.tmp_real);
      CK(cudaGetLastError());
    }
  }
  return DBFFT_OK;
}

// ---------------------------------------------------------------- residual monitors
const int kRowMajorVoigt[6] = {0, 4, 8, 5, 2, 1};

// per-slab scalar (sum or max of monitor partials) combined over slabs and ranks
dbfft_status monitor_combine(dbfft_ctx ctx, std::vector<double>& per_slab, bool is_max, double* out) {
  for (size_t k = 0; k < ctx->slabs.size(); ++k)
    CK(cudaMemcpyAsync(ctx->slabs[k].loc + 60, &per_slab[k], sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CKS(allreduce(ctx, 60, 1, is_max));
  return read_loc(ctx, 60, 1, out);
}

dbfft_status partials_host(dbfft_ctx ctx, Slab& s, bool is_max, double* v) {
  const int nb = monitor_blocks();
  std::vector<double> h(nb);
  CK(cudaMemcpyAsync(h.data(), s.part_misc, sizeof(double) * nb, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double r = 0.0;
  for (int b = 0; b < nb; ++b) r = is_max ? std::max(r, h[b]) : r + h[b];
  *v = r;
  return DBFFT_OK;
}

// max over the field in tmp_real of |curl curl eps| (kinematics 6, symmetric) or |curl F| (rows,
// kinematics 9): forward transforms (X R2C, y, z), the spectral curl, inverse transforms, max
dbfft_status incompat_max(dbfft_ctx ctx, double* result) {
  const bool fin = ctx->kin == 9;
  std::vector<double> mx(ctx->slabs.size(), 0.0);
  const int nrow = fin ? 3 : 1, nf = fin ? 3 : 6;
  const long long chunk = (long long)nf * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp;
  for (int row = 0; row < nrow; ++row) {
    for (Slab& s : ctx->slabs) {
      XGeom gx = xgeom(ctx, s, nullptr, s.WBX, nf, nf);
      gx.real_in = s.tmp_real;
      for (int f = 0; f < nf; ++f) gx.real_map[f] = fin ? 3 * row + f : kRowMajorVoigt[f];
      CKS(run_x(ctx, X_REAL_IN + nf, PK_OTHER, gx, nullptr));
    }
    CKS(xchg_row(ctx, nf));
    for (Slab& s : ctx->slabs) CKS(run_col(ctx, fin ? COL_YF3 : COL_YF6, PK_OTHER, geom_F2(ctx, s, s.WB, s.WS2, nf, nf), ctx->n2));
    CKS(exchange(ctx, chunk));
    for (Slab& s : ctx->slabs) {
      CKS(run_col(ctx, fin ? COL_ZF3 : COL_ZF6, PK_OTHER, geom_F3(ctx, s, s.WR2, s.WB, nf), ctx->n3));
      ProfScope ps(ctx, PK_OTHER);
      CK(fin ? launch_curl3(spec(ctx, s), s.WB, ctx->stream) : launch_curlcurl6(spec(ctx, s), s.WB, ctx->stream));
    }
    for (Slab& s : ctx->slabs) CKS(run_col(ctx, fin ? COL_ZI3 : COL_ZI6, PK_OTHER, geom_I1(ctx, s, s.WB, s.WS1, nf), ctx->n3));
    CKS(exchange(ctx, chunk));
    for (Slab& s : ctx->slabs) CKS(run_col(ctx, fin ? COL_YI3 : COL_YI6, PK_OTHER, geom_I2(ctx, s, s.WR, s.WBX, nf, nf), ctx->n2));
    CKS(xchg_row(ctx, nf));
    for (size_t k = 0; k < ctx->slabs.size(); ++k) {
      Slab& s = ctx->slabs[k];
      double* out = reinterpret_cast<double*>(s.WA);
      XGeom gx = xgeom(ctx, s, s.WB, nullptr, nf, nf);
      gx.real_out = out;
      CKS(run_x(ctx, X_REAL_OUT + nf, PK_OTHER, gx, nullptr));
      {
        ProfScope ps(ctx, PK_OTHER);
        CK(launch_maxabs(out, (long long)nf * s.Nloc, s.part_misc, ctx->stream));
      }
      double m;
      CKS(partials_host(ctx, s, true, &m));
      mx[k] = std::max(mx[k], m);
    }
  }
  return monitor_combine(ctx, mx, true, result);
}

// ||div sigma||_L2 (Parseval over the half spectrum, R6) of the stress field in tmp_real, and its
// volume average <sigma> (row-major 9)
dbfft_status div_norm(dbfft_ctx ctx, double* norm, double* mean9) {
  const bool fin = ctx->kin == 9;
  const int nf = fin ? 9 : 6;
  std::vector<double> n2(ctx->slabs.size());
  for (int a = 0; a < 9; ++a) {
    std::vector<double> sum(ctx->slabs.size());
    for (size_t k = 0; k < ctx->slabs.size(); ++k) {
      Slab& s = ctx->slabs[k];
      {
        ProfScope ps(ctx, PK_OTHER);
        CK(launch_sum(s.tmp_real + (long long)a * s.Nloc, s.Nloc, s.part_misc, ctx->stream));
      }
      CKS(partials_host(ctx, s, false, &sum[k]));
    }
    CKS(monitor_combine(ctx, sum, false, &mean9[a]));
    mean9[a] /= (double)ctx->N;
  }
  for (Slab& s : ctx->slabs) {
    XGeom gx = xgeom(ctx, s, nullptr, s.WBX, nf, nf);
    gx.real_in = s.tmp_real;
    for (int f = 0; f < nf; ++f) gx.real_map[f] = fin ? f : kRowMajorVoigt[f];
    CKS(run_x(ctx, X_REAL_IN + nf, PK_OTHER, gx, nullptr));
  }
  CKS(xchg_row(ctx, nf));
  // the operator's forward tail: f = -i xi . sigma_hat (positive form, R3) into q
  for (Slab& s : ctx->slabs) CKS(run_col(ctx, fin ? COL_F2F : COL_F2S, PK_OTHER, geom_F2(ctx, s, s.WB, s.WS2, 6, nf), ctx->n2));
  CKS(exchange(ctx, (long long)6 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
  for (size_t k = 0; k < ctx->slabs.size(); ++k) {
    Slab& s = ctx->slabs[k];
    CKS(run_col(ctx, fin ? COL_F3F : COL_F3S, PK_OTHER, geom_F3(ctx, s, s.WR2, s.q, 6), ctx->n3));
    {
      ProfScope ps(ctx, PK_OTHER);
      CK(launch_specnorm2(spec(ctx, s), s.q, 3, s.part_misc, ctx->stream));
    }
    CKS(partials_host(ctx, s, false, &n2[k]));
  }
  double tot;
  CKS(monitor_combine(ctx, n2, false, &tot));
  *norm = std::sqrt(tot);
  return DBFFT_OK;
}

double frob9(const double* a) {
  double s = 0.0;
  for (int k = 0; k < 9; ++k) s += a[k] * a[k];
  return std::sqrt(s);
}

dbfft_status dbfft_get_field(dbfft_ctx ctx, int32_t which, void* out, int32_t out_on_device) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (!out) {
    ctx->err = "get_field: null output";
    return DBFFT_E_INVALID_ARG;
  }
  if (ctx->family == FAM_NONE) {
    ctx->err = "get_field before set_phases";
    return DBFFT_E_STATE;
  }
  const cudaMemcpyKind k = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  for (Slab& s : ctx->slabs) CKS(ensure_tmp(ctx, s));
  switch (which) {
    case DBFFT_FIELD_U_HAT:
      return spec_out(ctx, &Slab::u_c, (cplx*)out, k);
    case DBFFT_FIELD_U: {
      for (Slab& s : ctx->slabs) CKS(run_col(ctx, COL_ZI3, PK_OTHER, geom_I1(ctx, s, s.u_c, s.WS1, 3), ctx->n3));
      CKS(exchange(ctx, (long long)3 * ctx->slabs[0].nyl * ctx->slabs[0].nzl * ctx->kxp));
      for (Slab& s : ctx->slabs) CKS(run_col(ctx, COL_YI3, PK_OTHER, geom_I2(ctx, s, s.WR, s.WBX, 3, 3), ctx->n2));
      CKS(xchg_row(ctx, 3));
      for (Slab& s : ctx->slabs) {
        XGeom gx = xgeom(ctx, s, s.WB, nullptr, 3, 3);
        gx.real_out = s.tmp_real;
        CKS(run_x(ctx, X_REAL_OUT + 3, PK_OTHER, gx, nullptr));
      }
      return gather_real(ctx, &Slab::tmp_real, 3, (double*)out, out_on_device);
    }
    case DBFFT_FIELD_STRAIN:
    case DBFFT_FIELD_STRESS:
      CKS(field_to_tmp(ctx, which));
      return gather_real(ctx, &Slab::tmp_real, 9, (double*)out, out_on_device);
    case DBFFT_FIELD_TANGENT: {
      // the full 3x3x3x3 tangent of the current state, built per voxel from what apply_K reads,
      // in chunks through a device scratch of 81 x chunk doubles
      const int mode = ctx->family == FAM_LINEAR ? 3 : ctx->family == FAM_J2 ? 2 : (ctx->tmode ? 1 : 0);
      const long long Ndst = ctx->loopback ? ctx->N : ctx->slabs[0].Nloc;
      // (loopback pencils: one [yr][x] plane block per chunk, contiguous in the global array)
      const long long chunk = (ctx->loopback && ctx->Py > 1) ? (long long)ctx->slabs[0].nyr * ctx->n1
                                                             : std::min<long long>(ctx->slabs[0].Nloc, 1LL << 20);
      double* scratch = nullptr;
      CKS(dalloc(ctx, &scratch, 81 * (size_t)chunk));
      cudaError_t e = cudaSuccess;
      for (Slab& s : ctx->slabs) {
        for (long long v0 = 0; v0 < s.Nloc && e == cudaSuccess; v0 += chunk) {
          const long long off = ctx->loopback ? global_voxel(ctx, s, v0) - v0 : 0;
          const long long nv = std::min(chunk, s.Nloc - v0);
          e = launch_tangent81(mode, xgeom(ctx, s, nullptr, nullptr), v0, nv, scratch, ctx->stream);
          if (e == cudaSuccess)
            e = cudaMemcpy2DAsync((double*)out + off + v0, sizeof(double) * Ndst, scratch, sizeof(double) * nv,
                                  sizeof(double) * nv, 81, k, ctx->stream);
          if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // the scratch is reused
        }
      }
      dfree(ctx, scratch);
      CK(e);
      return DBFFT_OK;
    }
    default:
      ctx->err = "get_field: unknown field";
      return DBFFT_E_INVALID_ARG;
  }
}

dbfft_status dbfft_profile_enable(dbfft_ctx ctx, int32_t enable) {
  if (!ctx) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
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
  DevGuard dev_guard(ctx->device);
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

dbfft_status dbfft_info(dbfft_ctx ctx, char* buf, int32_t cap) {
  if (!ctx || !buf || cap <= 0) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  const char* tr = ctx->P == 1 ? "none" : ctx->peer ? "peer" : "nccl";
  std::string j = "{\"device\": " + std::to_string(ctx->device) + ", \"sms\": " + std::to_string(num_sms()) +
                  ", \"world\": " + std::to_string(ctx->P) + ", \"rank\": " + std::to_string(ctx->rank) +
                  ", \"loopback\": " + std::to_string(ctx->loopback) + ", \"decomposition\": \"" +
                  (ctx->Py > 1 ? "pencils " + std::to_string(ctx->Py) + "x" + std::to_string(ctx->Pz) : std::string("z-slabs")) +
                  "\", \"transport\": \"" + tr +
                  "\", \"nccl_comm\": " + (ctx->comm ? "true" : "false") + ", \"pcg_loop\": \"" + ctx->loop_note + "\"}";
  for (char& c : j)
    if (c == '\n') c = ' ';
  snprintf(buf, (size_t)cap, "%s", j.c_str());
  return (int)j.size() < cap ? DBFFT_OK : DBFFT_E_INVALID_ARG;
}
int32_t dbfft_profile_count(void) { return PK_COUNT; }

}  // extern "C"

dbfft_status dbfft_residuals(dbfft_ctx ctx, const double target[9], const uint8_t mask[9], double out[3]) {
  if (!ctx || !target || !mask || !out) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (ctx->family == FAM_NONE) {
    ctx->err = "residuals before set_phases";
    return DBFFT_E_STATE;
  }
  const bool fin = ctx->kin == 9;
  double msig[9], meps[9], nrm, mx;
  CKS(field_to_tmp(ctx, DBFFT_FIELD_STRESS));
  CKS(div_norm(ctx, &nrm, msig));
  CKS(field_to_tmp(ctx, DBFFT_FIELD_STRAIN));
  for (int a = 0; a < 9; ++a) meps[a] = ctx->Fbar_c[a];
  CKS(incompat_max(ctx, &mx));
  double ref[9];
  for (int a = 0; a < 9; ++a) ref[a] = meps[a] - ((fin && a % 4 == 0) ? 1.0 : 0.0);
  out[0] = nrm / std::max(frob9(msig), 1e-300);   // Eq. chedckeq
  out[1] = mx / std::max(frob9(ref), 1e-300);     // Eq. chedckcomp / P:330
  double de[9], te[9], ds[9];
  for (int a = 0; a < 9; ++a) {                   // Eq. chedckimp per control type
    de[a] = mask[a] ? 0.0 : meps[a] - target[a];
    te[a] = mask[a] ? 0.0 : target[a];
    ds[a] = mask[a] ? msig[a] - target[a] : 0.0;
  }
  const double te_n = frob9(te);
  out[2] = std::max(te_n > 0 ? frob9(de) / te_n : frob9(de), frob9(ds) / std::max(frob9(msig), 1e-300));
  return DBFFT_OK;
}

dbfft_status dbfft_incompatibility(dbfft_ctx ctx, const double* field, int32_t on_device, double* out) {
  if (!ctx || !field || !out) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  for (Slab& s : ctx->slabs) CKS(ensure_tmp(ctx, s));
  CKS(scatter_real(ctx, field, on_device, 9, nullptr, &Slab::tmp_real));
  return incompat_max(ctx, out);
}

// ---------------------------------------------------------------- checkpoint / resume
namespace {
struct CkptHeader {
  char magic[8];  // "DBFFTCK1"
  int32_t n[3], kin, family, P, rank, nph, tmode, pad;
  int64_t n_incr;
  double Fbar_c[9];
};

size_t ckpt_bytes(dbfft_ctx ctx) {
  size_t b = sizeof(CkptHeader);
  for (const Slab& s : ctx->slabs) {
    b += sizeof(cplx) * 3 * (size_t)s.Hs;
    if (ctx->family == FAM_NEOHOOKE || ctx->family == FAM_J2) b += sizeof(double) * state_fields(ctx) * (size_t)s.Nloc;
    if (ctx->family == FAM_J2) b += sizeof(double) * 6 * (size_t)s.Nloc;
  }
  return b;
}
}  // namespace

dbfft_status dbfft_checkpoint(dbfft_ctx ctx, void* buf, size_t* bytes) {
  if (!ctx || !bytes) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (ctx->family == FAM_NONE) {
    ctx->err = "checkpoint before set_phases";
    return DBFFT_E_STATE;
  }
  const size_t need = ckpt_bytes(ctx);
  if (!buf) {
    *bytes = need;
    return DBFFT_OK;
  }
  if (*bytes < need) {
    ctx->err = "checkpoint: buffer of " + std::to_string(*bytes) + " bytes, need " + std::to_string(need);
    *bytes = need;
    return DBFFT_E_INVALID_ARG;
  }
  *bytes = need;
  CkptHeader h;
  memset(&h, 0, sizeof(h));
  memcpy(h.magic, "DBFFTCK1", 8);
  h.n[0] = ctx->n1; h.n[1] = ctx->n2; h.n[2] = ctx->n3;
  h.kin = ctx->kin; h.family = ctx->family; h.P = ctx->P; h.rank = ctx->rank; h.nph = ctx->nph; h.tmode = ctx->tmode;
  h.n_incr = ctx->n_incr;
  memcpy(h.Fbar_c, ctx->Fbar_c, sizeof(h.Fbar_c));
  char* o = static_cast<char*>(buf);
  memcpy(o, &h, sizeof(h));
  o += sizeof(h);
  const int nf = state_fields(ctx);
  for (Slab& s : ctx->slabs) {
    CK(cudaMemcpyAsync(o, s.u_c, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToHost, ctx->stream));
    o += sizeof(cplx) * 3 * s.Hs;
    if (ctx->family == FAM_NEOHOOKE || ctx->family == FAM_J2) {
      CK(cudaMemcpyAsync(o, s.F_c, sizeof(double) * nf * s.Nloc, cudaMemcpyDeviceToHost, ctx->stream));
      o += sizeof(double) * nf * s.Nloc;
    }
    if (ctx->family == FAM_J2) {
      CK(cudaMemcpyAsync(o, s.epsp_c, sizeof(double) * 6 * s.Nloc, cudaMemcpyDeviceToHost, ctx->stream));
      o += sizeof(double) * 6 * s.Nloc;
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DBFFT_OK;
}

dbfft_status dbfft_restore(dbfft_ctx ctx, const void* buf, size_t bytes) {
  if (!ctx || !buf) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  if (ctx->family == FAM_NONE) {
    ctx->err = "restore before set_phases";
    return DBFFT_E_STATE;
  }
  CkptHeader h;
  if (bytes < sizeof(h)) {
    ctx->err = "restore: truncated checkpoint";
    return DBFFT_E_INVALID_ARG;
  }
  memcpy(&h, buf, sizeof(h));
  if (memcmp(h.magic, "DBFFTCK1", 8) != 0 || h.n[0] != ctx->n1 || h.n[1] != ctx->n2 || h.n[2] != ctx->n3 || h.kin != ctx->kin ||
      h.family != ctx->family || h.P != ctx->P || h.rank != ctx->rank || h.nph != ctx->nph || bytes != ckpt_bytes(ctx)) {
    ctx->err = "restore: checkpoint of another grid / kinematics / material family / decomposition, or wrong size";
    return DBFFT_E_INVALID_ARG;
  }
  const char* o = static_cast<const char*>(buf) + sizeof(h);
  const int nf = state_fields(ctx);
  for (Slab& s : ctx->slabs) {
    CK(cudaMemcpyAsync(s.u_c, o, sizeof(cplx) * 3 * s.Hs, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(s.u, s.u_c, sizeof(cplx) * 3 * s.Hs, cudaMemcpyDeviceToDevice, ctx->stream));
    o += sizeof(cplx) * 3 * s.Hs;
    if (ctx->family == FAM_NEOHOOKE || ctx->family == FAM_J2) {
      CK(cudaMemcpyAsync(s.F_c, o, sizeof(double) * nf * s.Nloc, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(s.F, s.F_c, sizeof(double) * nf * s.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
      o += sizeof(double) * nf * s.Nloc;
    }
    if (ctx->family == FAM_J2) {
      CK(cudaMemcpyAsync(s.epsp_c, o, sizeof(double) * 6 * s.Nloc, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(s.epsp_t, s.epsp_c, sizeof(double) * 6 * s.Nloc, cudaMemcpyDeviceToDevice, ctx->stream));
      o += sizeof(double) * 6 * s.Nloc;
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));  // the blob may be freed on return
  memcpy(ctx->Fbar_c, h.Fbar_c, sizeof(h.Fbar_c));
  memcpy(ctx->Fbar, h.Fbar_c, sizeof(h.Fbar_c));
  ctx->n_incr = h.n_incr;
  if (ctx->family != FAM_LINEAR) {  // tangent (and M) of the restored committed state, as after a commit
    double zero[9] = {0}, mp[9], mx;
    CKS(constitutive(ctx, false, zero, 1.0, mp, &mx));
    CKS(refresh_mean_tangent(ctx));
  }
  return DBFFT_OK;
}

dbfft_status dbfft_get_trace(dbfft_ctx ctx, double* out, int32_t cap, int32_t* n) {
  if (!ctx || !n || (cap > 0 && !out)) return DBFFT_E_INVALID_ARG;
  DevGuard dev_guard(ctx->device);
  *n = ctx->trace_n;
  const int m = std::min(cap, ctx->trace_n);
  if (m > 0) CK(cudaMemcpy(out, ctx->trace_dev, sizeof(double) * 2 * (size_t)m, cudaMemcpyDeviceToHost));
  return DBFFT_OK;
}
