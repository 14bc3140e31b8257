/* dbfft.h — C ABI of the B200-native DBFFT hot path.
 *
 * DBFFT (Lucarini & Segurado, arXiv 1905.12725; "P:<line>" = /root/reference/PAPER.md line)
 * solves the periodic cell problem with the Fourier displacement u_hat(xi) as the unknown.
 * This library implements, on one CUDA device (sm_100a) per process, the matrix-free operator
 *     K u_hat = -d_hat : F( C(x) : F^-1( s_hat . u_hat ) )                 (Eq. lineqf)
 * (symmetric gradient s_hat at small strain; full gradient g_hat at finite strain),
 * its mixed-control augmentation, the averaged-stiffness preconditioner
 * (Eqs. pred2/pred3), preconditioned CG and the Newton driver with per-voxel
 * constitutive updates.  Every call returns a dbfft_status; no C++ exception crosses
 * the ABI.  There is no CPU fallback: a call that cannot run on the GPU fails with DBFFT_E_CUDA.
 *
 * Conventions (SURVEY.md "Notation"; readings R1..R22 listed in DESIGN.md):
 *  - Grid n = {n1, n2, n3} voxels (x, y, z); each n_a a power of two in [8, 512].
 *    Cell lengths L = {L1, L2, L3} > 0.  Voxel (i,j,k) has centre ((i+1/2)L1/n1, ...).
 *  - Frequencies (Eq. 1) in FFT-native order, xi_a(k) = 2 pi kappa / L_a with
 *    kappa = k (k < n/2), k - n (k > n/2) and xi_a = 0 at the Nyquist index k = n/2 (R1).
 *  - Spectra are mean-normalised (R5): u_hat = F(u)/(n1 n2 n3), so u_hat(0) = <u>.
 *  - SPECTRAL VECTOR layout (device, complex128 = two doubles {re, im}):
 *        [3 components][ky = 0..n2-1][kz = 0..n3-1][kx = 0..n1/2]        (kx fastest)
 *    i.e. the half spectrum of a real field (R6).  H = (n1/2+1) n2 n3 points per component.
 *    dbfft_spectral_layout() returns the same as shape/strides (in complex elements).
 *    Inputs must be Hermitian-consistent on the kx = 0 and kx = n1/2 planes (true for any
 *    spectrum of a real field); the operator uses their Hermitian part.
 *  - REAL FIELD layout (host or device, double): [component][z][y][x] (x fastest).
 *    Second-order tensors have 9 components, row-major (c = 3 i + j).
 *  - Macro 3x3 quantities (targets, masks, e blocks, reports): 9 entries, row-major.
 *  - Ownership: the ctx owns all of its device memory (cudaMalloc, or the env allocator hooks
 *    below, e.g. torch's caching allocator).  Pointers passed in are
 *    borrowed for the duration of the call only; inputs are copied when retained.
 *  - Streams: all device work of a ctx is issued on env->cuda_stream (a cudaStream_t, e.g.
 *    torch.cuda.current_stream().cuda_stream) or on a ctx-owned stream if NULL.  Calls marked
 *    (async) return before the device work completes; the others synchronise that stream.
 *  - Distribution: with env->world = P > 1 (a power of two dividing n2 and n3)
 *    real space is split in z-slabs (rank r owns z in [r n3/P, (r+1) n3/P)) and spectral space
 *    in ky-slabs (ky in [r n2/P, (r+1) n2/P)).  Every call is collective over the P ranks.
 *    NCCL mode (env->loopback = 0): one process per GPU; rank 0 calls dbfft_nccl_unique_id and
 *    broadcasts the 128-byte id (e.g. via torch.distributed); each rank passes and receives
 *    only its own slab (spectral vectors [3][n2/P][kz][kx]; real fields [c][n3/P][y][x]).
 *    Loopback mode (env->loopback = 1): all P virtual ranks live in this process on one device
 *    and exchange through device copies (tests the distributed data path on one GPU); API
 *    arrays are then the global ones.  env->pencil_rows > 1 selects 2-D pencils instead of
 *    z-slabs (dbfft_env below: local blocks, padding column, exchanges).
 */
#ifndef DBFFT_H
#define DBFFT_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dbfft_ctx_s* dbfft_ctx;

typedef enum {
  DBFFT_OK = 0,
  DBFFT_E_INVALID_GRID = 1,  /* n_a not a power of two in [8,512], L_a <= 0, or world not a power
                                of two dividing n2 and n3                                 */
  DBFFT_E_INVALID_ARG = 2,   /* null pointer, unknown kind, phase id >= n_phases, bad parameters */
  DBFFT_E_STATE = 3,         /* call-order violation, e.g. apply_K before set_phases             */
  DBFFT_E_CUDA = 4,          /* CUDA error (message in dbfft_last_error)                          */
  DBFFT_E_NCCL = 5,          /* NCCL could not be loaded / initialised or a collective failed     */
  DBFFT_E_OOM = 6,           /* device allocation failed                                          */
  DBFFT_E_NOT_CONVERGED = 7, /* PCG max_cg or Newton max_newton exhausted; report filled; state
                                rolled back to the last commit                                   */
  DBFFT_E_BREAKDOWN = 8,     /* NaN/Inf or <p,Kp> <= 0 in PCG                                     */
  DBFFT_E_MATERIAL = 9       /* det F <= 0 at some voxel (report.bad_voxel)                       */
} dbfft_status;

typedef enum { DBFFT_SMALL_STRAIN = 6, DBFFT_FINITE_STRAIN = 9 } dbfft_kinematics;

typedef struct {
  int32_t rank, world;   /* this rank and the number of ranks P (1: single GPU)        */
  const void* nccl_id;   /* 128-byte ncclUniqueId (NCCL mode, world > 1), else NULL    */
  void* cuda_stream;     /* cudaStream_t, or NULL: ctx creates its own *blocking* stream,
                            ordered with the caller's legacy default stream              */
  int32_t device;        /* CUDA device ordinal (-1: current device)                   */
  int32_t loopback;      /* 1: all `world` ranks virtual in this process (testing)     */
  int32_t transport;     /* world > 1: how the two all-to-alls per operator application
                             move data.  DBFFT_TRANSPORT_NCCL: grouped
                            ncclSend/ncclRecv of the rank-chunked pass outputs.
                            DBFFT_TRANSPORT_PEER: the z-inverse and y-forward passes store
                            their chunk for rank d straight into rank d's receive buffer
                            through a CUDA VMM window (NVLink peer memory; one node), a
                            device barrier replaces the exchange.  All-reduces stay NCCL. */
  /* Device memory of the ctx (every buffer except the peer transport's CUDA VMM windows):
   * dev_alloc(bytes, alloc_user) returns device memory on `device` (NULL: DBFFT_E_OOM) and
   * dev_free(ptr, alloc_user) releases it — e.g. torch's caching allocator.  Both NULL: cudaMalloc
   * / cudaFree.  Called from the thread calling the ABI; frees happen after the ctx stream has
   * drained (destroy, set_phases). */
  void* (*dev_alloc)(size_t bytes, void* alloc_user);
  void (*dev_free)(void* ptr, void* alloc_user);
  void* alloc_user;
  /* Decomposition: 0 or 1 = z-slabs (above).  Py > 1 (a power of two,
   * Py <= n1/2, Py | n2): 2-D pencils on a Py x Pz grid, Pz = world / Py (Pz | n2, Pz | n3),
   * rank = b Py + a.  Rank (a, b) owns real z in [b n3/Pz, ...) x y in [a n2/Py, ...) (all x;
   * local real fields [c][n3/Pz][n2/Py][x]) and spectral ky in [b n2/Pz, ...) x kx in
   * [a kxm, (a+1) kxm) with kxm = n1/(2 Py), plus the Nyquist kx = n1/2 on a = Py - 1 (local
   * spectral vectors [3][n2/Pz][kz][kxm + 1]; column kxm is padding, kept 0, on a < Py - 1).
   * Per operator application 4 exchanges instead of 2: within the column group (same a) around
   * the z passes as for slabs, and within the row group (same b) after the y-inverse and after
   * the x pass (the x-line layout gathers / scatters the kx blocks).  NCCL transport only. */
  int32_t pencil_rows;
} dbfft_env;
enum { DBFFT_TRANSPORT_NCCL = 0, DBFFT_TRANSPORT_PEER = 1 };

/* Host helper of the peer transport's bootstrap: all-gather of nfd (1..16) file descriptors among
 * the `world` processes of one node over abstract Unix sockets (SCM_RIGHTS), rendezvous name
 * "dbfft-<tag>-<rank>".  out[src * nfd + i] receives a descriptor of process src's fds[i] (owned
 * by the caller; out[rank * nfd + i] = fds[i] itself).  DBFFT_E_INVALID_ARG on bad arguments,
 * DBFFT_E_STATE on a socket error or timeout (message in dbfft_last_error(NULL)).  (sync) */
dbfft_status dbfft_fd_allgather(const char* tag, int32_t rank, int32_t world, const int32_t* fds, int32_t nfd,
                                int32_t* out, int32_t timeout_ms);

/* Probe of the peer transport's cross-process windows (tests; no ctx, no NCCL): every process
 * builds an exchange buffer of `world` chunks exactly as dbfft_create does for
 * DBFFT_TRANSPORT_PEER (cuMemCreate, POSIX-fd export, dbfft_fd_allgather(tag), import, window
 * mapping), then stores 1000*rank + d into the first 1024 words of its window chunk d, i.e. into
 * rank d's buffer.  After a host barrier among the processes, _check counts the words of this
 * rank's buffer that differ from what rank src wrote into chunk src (0 = every window landed).
 * Several processes may share one GPU (no kernel waits on another process).  (sync) */
dbfft_status dbfft_peer_probe_open(const char* tag, int32_t rank, int32_t world, int32_t device, void** out);
dbfft_status dbfft_peer_probe_check(void* probe, int32_t* bad_words);
dbfft_status dbfft_peer_probe_close(void* probe);

/* NCCL bootstrap (rank 0): writes a 128-byte ncclUniqueId.  NCCL is loaded at run time
 * (dlopen libnccl.so.2, or $DBFFT_NCCL_LIB); DBFFT_E_NCCL if it cannot be loaded. */
dbfft_status dbfft_nccl_unique_id(void* out128);

/* Create a context for grid n (voxels) and cell lengths L.  Each n[a] is a power of
 * two in [8, 512] (Nyquist frequencies neglected, R1) or one of the odd sizes 15, 21, 27, 63
 * (Eq. 1 of P:41-43 verbatim, mixed-radix 3/5/7 FFTs; the paper's cells are 63^3).  world > 1
 * needs powers of two dividing n2 and n3.  DBFFT_E_INVALID_GRID otherwise.  (sync) */
dbfft_status dbfft_create(const int32_t n[3], const double L[3], int32_t kinematics,
                          const dbfft_env* env, dbfft_ctx* out);
dbfft_status dbfft_destroy(dbfft_ctx ctx);
/* Last error message of ctx (NULL ctx: last creation error); valid until the next call. */
const char* dbfft_last_error(dbfft_ctx ctx);
/* shape[4] = {3, n2, n3, n1/2+1}; strides[4] in complex elements. */
dbfft_status dbfft_spectral_layout(dbfft_ctx ctx, int64_t shape[4], int64_t strides[4]);

/* Material laws, one record per phase ("the behavior at a point x defined by the
 * constitutive equation of the phase occupying that point").  Parameters in p[]:
 *   DBFFT_MAT_ISO      : p = {E, nu}                      linear isotropic   small strain
 *   DBFFT_MAT_CUBIC    : p = {C11, C12, C44, R[9]}        cubic crystal, stiffness rotated
 *                        C'_ijkl = R_ia R_jb R_kc R_ld C_abcd, R row-major        small strain
 *   DBFFT_MAT_NEOHOOKE : p = {mu, kappa}                  compressible neo-Hookean (R14)   finite
 *   DBFFT_MAT_J2       : p = {E, nu, sigma_y, n, edot0}   J2 Perzyna overstress (R16)     small
 *   DBFFT_MAT_SVK      : p = {E, nu}                      Saint Venant-Kirchhoff:
 *                        S = lam tr(E) I + 2 mu E, E = (F^T F - I)/2, P = F S        finite
 * NEOHOOKE and SVK phases may be mixed (one finite-strain hyperelastic family); with any SVK
 * phase the 45-entry tangent is stored.
 * Linear kinds require no state; NEOHOOKE, SVK and J2 keep per-voxel state.
 * Tangent storage (implementation choice, same operator): NEOHOOKE keeps F^-1 and
 * c1 = mu - lam ln J per voxel and applies K:G = mu G + c1 (F^-1 G F^-1)^T + lam tr(F^-1 G) F^-T
 * matrix-free (80 B/voxel); environment DBFFT_TANGENT=full stores the 45 independent entries of
 * the 9x9 tangent instead (360 B/voxel).  J2 keeps (theta, thetabar, n) (64 B/voxel).          */
typedef enum {
  DBFFT_MAT_ISO = 1,
  DBFFT_MAT_CUBIC = 2,
  DBFFT_MAT_NEOHOOKE = 3,
  DBFFT_MAT_J2 = 4,
  DBFFT_MAT_SVK = 5
} dbfft_mat_kind;
typedef struct { int32_t kind; double p[36]; } dbfft_material;

/* Phase id per voxel ([z][y][x], uint16, host if on_device == 0 else device) and the per-phase
 * table (host, copied).  All phases must be of one family: linear (ISO/CUBIC), NEOHOOKE (finite
 * strain ctx) or J2.  Resets the mechanical state to the undeformed configuration.  (sync)  */
dbfft_status dbfft_set_phases(dbfft_ctx ctx, const uint16_t* phase_id, int32_t on_device,
                              int32_t n_phases, const dbfft_material* table);

/* f_hat = K u_hat with the current stiffness/tangent (positive form, R3).  u_hat, f_hat:
 * device spectral vectors (layout above), may not alias.  Output is 0 on the null set Z.
 * Nonlinear materials use the tangent of the last dbfft_eval_state / Newton iteration.  (async) */
dbfft_status dbfft_apply_K(dbfft_ctx ctx, const void* u_hat, void* f_hat);
/* Mixed-control augmented operator: the strain argument gains the macro block
 * e_in (host, 9, row-major; used on mask entries only) and r_out (host, 9) receives
 * P_mask <C:(F^-1(s.u) + e)> (the xi = 0 rows).  mask: host, 9 bytes, 1 = stress
 * controlled.  With mask all 0 this equals dbfft_apply_K and r_out = 0.  (sync)               */
dbfft_status dbfft_apply_K_aug(dbfft_ctx ctx, const uint8_t mask[9], const void* u_hat,
                               const double e_in[9], void* f_hat, double r_out[9]);
/* z_hat = M(xi) r_hat, M = [xi . Cbar . xi]^-1 off Z and 0 on Z (R4), Cbar the volume
 * average of the current stiffness/tangent.  Device vectors.  (async)         */
dbfft_status dbfft_precond(dbfft_ctx ctx, const void* r_hat, void* z_hat);
/* Evaluate the constitutive law at the real field `field` ([9][z][y][x] doubles: eps (small
 * strain, symmetric) or F (finite strain)), host or device, from the committed state, and
 * install the resulting tangent for apply_K / precond (no state is committed).  dt is used by
 * rate-dependent laws.  Linear materials: no-op.  (sync)                                    */
dbfft_status dbfft_eval_state(dbfft_ctx ctx, const double* field, int32_t on_device, double dt);

typedef struct {
  double tol_eq;       /* PCG stop: eps_eq = ||div sigma||_L2/||<sigma>||, default 1e-10 */
  double tol_load;     /* mixed control: ||P(<sigma> - sigma_bar)||/||<sigma>||, 1e-10  */
  double tol_newton;   /* Newton stop: max |grad du + dF_f|, default 1e-6               */
  int32_t max_cg;      /* default 10000                                                 */
  int32_t max_newton;  /* default 25                                                            */
  int32_t check_every; /* host convergence poll period in CG iterations (default 4)             */
  int32_t precond_refresh; /* mean-tangent refresh policy of M:
                              0: at the first Newton iterate of every increment (R12, default);
                              1: every Newton iteration; 2: never — the tangent of the undeformed
                              state computed by set_phases ("initial tangent"); 3: at the
                              first iterate of every precond_period-th increment ("once in a
                              while").  Linear phases: M is fixed, the policy is unused.   */
  int32_t precond_period;  /* policy 3 period in increments (>= 1, default 1)                     */
  int32_t precond_medium;  /* reference medium of M for linear phases: 0 arithmetic mean <C>
                              (Eq. pred3, default); 1 harmonic <C^-1>^-1; 2 Hill (mean of
                              0 and 1) — the ad-hoc preconditioners of P:394.  Nonlinear families
                              accept 0 only (DBFFT_E_INVALID_ARG otherwise).  Changes iteration
                              counts only: the solution is that of the same system.               */
} dbfft_opts;
dbfft_opts dbfft_default_opts(void);

typedef struct {
  int32_t converged, cg_iters, newton_iters, status;
  double eps_eq, eps_load, max_dgrad;
  double macro_strain[9];  /* <eps> (small strain) or <F> (finite strain), row-major          */
  double macro_stress[9];  /* <sigma> or <P>                                                    */
  int64_t bad_voxel;       /* first voxel with det F <= 0, else -1                              */
  double seconds;          /* device time of the call                                          */
} dbfft_report;

/* Advance one load increment to the TOTAL target.  mask[a] = 1: component a is stress
 * controlled (target is sigma or P); 0: strain controlled (eps or F) (IJ != ij).  Small
 * strain targets and masks must be symmetric.  Linear materials: one PCG solve of the
 * (augmented) system.  Nonlinear: Newton.  dt: increment duration.
 * On success the state is committed; on failure it is rolled back.  (sync)                   */
dbfft_status dbfft_solve_increment(dbfft_ctx ctx, const double target[9], const uint8_t mask[9],
                                   double dt, const dbfft_opts* opts, dbfft_report* report);

typedef enum {
  DBFFT_FIELD_U = 0,        /* fluctuation displacement u~(x): 3 x N doubles          */
  DBFFT_FIELD_STRAIN = 1,   /* eps (small) or F (finite): 9 x N doubles                        */
  DBFFT_FIELD_STRESS = 2,   /* sigma (small) or P (finite): 9 x N doubles                      */
  DBFFT_FIELD_U_HAT = 3,    /* u~_hat, spectral vector layout (3 x H complex)                  */
  DBFFT_FIELD_TANGENT = 4   /* the tangent apply_K uses, 81 x N doubles [(9a + b)][z][y][x] with
                               a = 3i + j, b = 3k + l: C_ijkl (small strain: the phase stiffness or
                               the J2 algorithmic tangent, P:204 / R16) or dP_ij/dF_kl (finite,
                               R14 / P:326), of the last Newton iterate / eval_state              */
} dbfft_field;
/* Copy a field of the committed state (TANGENT: of the current state) into `out` (host if
 * out_on_device == 0; loopback: the global array, NCCL: this rank's z-slab). (sync) */
dbfft_status dbfft_get_field(dbfft_ctx ctx, int32_t which, void* out, int32_t out_on_device);

/* Residual monitors of the committed state (SS3 of the paper; finite strain P:327-330):
 *   out[0] equilibrium   ||div sigma||_L2 / ||<sigma>||        (Eq. chedckeq; finite: P,
 *                        reference divergence)
 *   out[1] compatibility max|curl curl eps| / ||<eps>||         (Eq. chedckcomp; finite:
 *                        max|curl_0 F| / ||<F> - I||)
 *   out[2] loading       ||<eps> - eps_bar|| / ||eps_bar|| over the strain-controlled components
 *                        and ||<sigma> - sigma_bar|| / ||<sigma>|| over the stress-controlled ones
 *                        (Eq. chedckimp), the larger of the two
 * target/mask as in dbfft_solve_increment (row-major 3x3).  ||.||_L2 is the voxel-mean L2 norm
 * (Parseval on the mean-normalised half spectrum, R5/R6), ||.|| Frobenius, max over all
 * components and voxels.  Derivatives are the method's discrete ones (i xi, Eq. 1, R1).
 * Uses the context's work buffers; call between solves.  Errors: E_STATE before set_phases. */
dbfft_status dbfft_residuals(dbfft_ctx ctx, const double target[9], const uint8_t mask[9], double out[3]);

/* Unnormalised incompatibility of a given real tensor field field[9][n3][n2][n1] (row-major
 * 3x3 per voxel, host if on_device == 0; loopback: global array, NCCL: this rank's z-slab):
 * max|curl curl eps| for a small-strain context (the field's symmetric part is used),
 * max|curl F| (row-wise curl) for a finite-strain one.  Same derivatives as dbfft_residuals. */
dbfft_status dbfft_incompatibility(dbfft_ctx ctx, const double* field, int32_t on_device, double* out);

/* Residual history of the last dbfft_solve_increment (the paper's Fig. div): pairs
 * (eps_equilibrium, eps_loading) of Eq. chedckeq / chedckimp as the PCG tracks them (R7) — at the
 * start and after every iteration of every PCG solve (one per Newton iteration), concatenated in
 * order; a true-residual restart continues the same sequence.  *n = number of pairs recorded (at
 * most 65536); min(cap, *n) pairs are copied to out[2 cap] (host).  (sync) */
dbfft_status dbfft_get_trace(dbfft_ctx ctx, double* out, int32_t cap, int32_t* n);

/* Per-kernel device-time accounting: while enabled, CUDA events are recorded on the ctx stream
 * around every kernel launch and accumulated per kernel id (names via dbfft_profile_name). */
dbfft_status dbfft_profile_enable(dbfft_ctx ctx, int32_t enable);
dbfft_status dbfft_profile_read(dbfft_ctx ctx, int32_t kernel_id, double* total_ms, int64_t* launches);
const char* dbfft_profile_name(int32_t kernel_id);
/* Number of CUDA kernels this ctx has launched since creation (always counted). */
dbfft_status dbfft_launch_count(dbfft_ctx ctx, int64_t* count);
int32_t dbfft_profile_count(void);

/* Per-increment dump / resume of the committed state (host blob, layout private to this library
 * version, with a header checked on restore): the fluctuation spectrum u~_hat, the macro strain /
 * F, the per-voxel committed state (F or eps, and the J2 plastic strain) and the increment count
 * (preconditioner policy 3).  dbfft_checkpoint: buf NULL -> *bytes = size needed; else copies
 * (DBFFT_E_INVALID_ARG if *bytes is too small).  dbfft_restore: into a ctx of the same grid,
 * kinematics, material family and decomposition, after dbfft_set_phases with the same
 * microstructure; the next dbfft_solve_increment continues exactly where the dumped ctx would.
 * Loopback: all slabs; NCCL: this rank's slab.  (sync) */
dbfft_status dbfft_checkpoint(dbfft_ctx ctx, void* buf, size_t* bytes);
dbfft_status dbfft_restore(dbfft_ctx ctx, const void* buf, size_t bytes);

/* One-line JSON description of ctx (host): device and SM count, world / rank / loopback, the
 * transport of the two all-to-alls ("none" | "nccl" | "peer"), whether an NCCL communicator is
 * live, and how the last PCG loop ran ("device-side WHILE graph", host-polled graph rounds or
 * eager, with the reason of a fallback).  DBFFT_E_INVALID_ARG if it does not fit in cap bytes
 * (truncated, NUL-terminated).  (sync) */
dbfft_status dbfft_info(dbfft_ctx ctx, char* buf, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* DBFFT_H */
