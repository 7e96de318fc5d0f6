/*
 * heff.h -- C ABI of libheff: the B200 (sm_100a) two-site DMRG effective-Hamiltonian
 * matvec H_eff.psi and the Lanczos ground-state solver around it.
 *
 * What is computed (citations: lines of the paper text, /root/reference/PAPER.md).
 *   DMRG computes "dominant eigenvectors of very large Hermitian linear operators"
 *   (Sec. 6.2).  At a two-site window the operator is the product of
 *   the left environment, the two MPO tensors of Eq. (1)'s MPO form (Sec. 6.1,
 *   PAPER.md:666-672) and the right environment, contracted over all matching indices by
 *   ITensor's `*` (Sec. 4) with primes keeping the output legs apart
 *   (Sec. 2.6):
 *
 *     out[a',s1',s2',b'] = sum_{a,w,s1,w1,s2,w2,b}
 *          L[a',w,a] W1[w,s1',s1,w1] W2[w1,s2',s2,w2] R[b',w2,b] psi[a,s1,s2,b]     (D)
 *
 *   The output is returned un-primed in psi's layout.  libheff evaluates
 *   (D) exactly (up to rounding order) in the north_star's four steps
 *   L.psi -> .W1 -> .W2 -> .R (order A) on one GPU, and in the mirror order
 *   R.psi -> .W2 -> .W1 -> .L on a b'-shard (order B, reading R17).
 *
 * Layout: every tensor is dense, row-major (last index fastest), IEEE fp64:
 *   L  [mL][kL][mL]     W1 [kL][d1][d1][kM]    W2 [kM][d2][d2][kR]
 *   R  [nb][kR][mR]     rows b' in [b_lo, b_hi) of R (all mR rows when dist == NULL)
 *   psi, out  [mL][d1][d2][mR]   (a b'-shard [mL][d1][d2][nb] where stated)
 *
 * Pointers: every tensor pointer is a DEVICE pointer on the current CUDA device unless
 * the function name ends in _host.  Alignment: 8 B required; 16 B (and even row
 * lengths) enables the TMA-fed GEMM path, otherwise a plain-load path runs.
 *
 * Ownership: L, W1, W2 and R are BORROWED -- they must stay allocated and unmodified
 * for the plan's lifetime (W1/W2 are read once, at create, into the plan's device-side
 * two-site MPO; a sharded plan also keeps a row-reordered copy of its R shard).  The plan
 * owns its workspace (intermediates, Lanczos basis, gather buffer) and its NCCL
 * communicator.
 *
 * Streams: `heff_stream` is a cudaStream_t (NULL = legacy default stream).  heff_apply
 * is stream-ordered and returns before completion.  lanczos_ground blocks until done.
 *
 * Errors: functions return HEFF_OK (0) or a negative code; heff_last_error() gives a
 * thread-local message for the last failure.  There is no CPU fallback: a missing or
 * failing device is an error.
 *
 * Concurrency: one plan per host thread at a time, and a plan's calls on one stream at a
 * time (its GEMMs share one stream-K partial-tile workspace and one CTA ticket counter);
 * different plans, and the free functions on different host threads, may run
 * concurrently on different streams.
 */
#ifndef HEFF_H
#define HEFF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct heff_plan_s* heff_plan;
typedef void* heff_stream; /* cudaStream_t */

enum {
  HEFF_OK = 0,
  HEFF_EINVAL = -1,      /* null pointer, bad shape, aliasing, bad b-range      */
  HEFF_ENOMEM = -2,      /* device allocation failed                            */
  HEFF_ECUDA = -3,       /* CUDA runtime / driver error                         */
  HEFF_ENCCL = -4,       /* NCCL error (load, init or collective)               */
  HEFF_EZERO = -5,       /* lanczos start vector is zero          */
  HEFF_EUNSUPPORTED = -6, /* request outside what this build supports           */
  HEFF_ENOCONV = -7       /* an iterative decomposition did not converge          */
};

/* Dimensions: bond dims mL, mR; site dims d1, d2; MPO bond dims kL (L/W1), kM (W1/W2),
 * kR (W2/R).  All >= 1. */
typedef struct {
  int64_t mL, d1, d2, mR, kL, kM, kR;
} heff_dims;

/* Multi-GPU partition over the output right bond b' (R17).
 * This rank owns b' in [b_lo, b_hi); its R argument holds exactly those rows.
 * nccl_uid: 128-byte ncclUniqueId from heff_nccl_unique_id() on rank 0, broadcast by
 * the caller (torch.distributed).  nccl_uid == NULL gives a "virtual shard": the plan
 * computes its out-shard from a full psi with no communicator (heff_apply only). */
typedef struct {
  int nranks, rank;
  const unsigned char* nccl_uid;
  int64_t b_lo, b_hi;
} heff_dist;

/* Lanczos options (readings R11-R14).
 *   mode 0 (fixed): exactly max_iter matvecs unless an invariant subspace is hit;
 *   mode 1 (converge): stop when beta_j |y_j[last]| <= tol * hnorm_j, or at max_iter.
 *     Vectors of <= 2^20 doubles run up to 3 steps past that point before the host sees the
 *     scalars (HEFF_LANCZOS_BATCH=1 disables); the result is that of the stopping step.
 * alpha_out, beta_out, theta_out: optional HOST arrays of >= max_iter doubles receiving
 * the tridiagonal T_j and the lowest Ritz value after every step. */
typedef struct {
  int max_iter;
  int mode;
  double tol;
  double* alpha_out;
  double* beta_out;
  double* theta_out;
} heff_lanczos_opts;

/* Create a plan: validates dims, allocates workspace, builds the two-site MPO
 * Wc = sum_w1 W1 W2 as a CSR list ON THE DEVICE (no host copy, no synchronisation: the
 * set-up kernels are enqueued on `stream`, and every later call on another stream is
 * ordered after them by an event), and (dist with a uid) joins the NCCL communicator
 * (collective over all ranks).  Limits: kL d1 d2 <= 1600 and d1 d2 kR <= 1600 (the MPO
 * kernel's shared-memory tile narrows from 128 to 16 columns as k d^2 grows; HEFF_EUNSUPPORTED
 * beyond).  W1/W2 must be device pointers (HEFF_EINVAL otherwise). */
int heff_create(heff_plan* out, const heff_dims* dims, const double* L, const double* W1, const double* W2,
                const double* R, const heff_dist* dist, heff_stream stream);

/* Complex plans (ITensor's Dense{ComplexF64}/zgemm):
 * same as heff_create with L, W1, W2, R -- and later psi/out -- as interleaved complex
 * (re, im) fp64 arrays, 16-byte aligned.  (D) is evaluated without conjugation, so a
 * Hermitian H_eff needs environments built with the bra tensors conjugated.
 * heff_apply / heff_apply_host / lanczos_ground (Hermitian Lanczos, <v,w> = sum conj(v) w)
 * accept complex plans; sharding, U(1) sparsity, penalties and sums do not (EUNSUPPORTED). */
int heff_create_z(heff_plan* out, const heff_dims* dims, const double* L, const double* W1, const double* W2,
                  const double* R, const heff_dist* dist, heff_stream stream);

/* out = H_eff . psi  (D).  dist == NULL: psi, out are full [mL][d1][d2][mR].
 * Sharded plan: psi is the FULL vector, out is this rank's shard [mL][d1][d2][nb].
 * out must not alias psi.  Asynchronous on `stream`. */
int heff_apply(heff_plan p, const double* psi, double* out, heff_stream stream);

/* Gather-fused order-B matvec on a b'-sharded plan: psi is given
 * as the P = mR / nb shards of the blocked layout psi_blocked[P][mL*d1*d2][nb] (what an
 * all-gather of the shards produces) and GEMM_A reads every shard through its own TMA
 * descriptor -- no re-layout.  out = this plan's shard [mL][d1][d2][nb].  Requires
 * nb % 16 == 0, P <= 8, 16-byte alignment.  Asynchronous on `stream`. */
int heff_apply_blocked(heff_plan p, const double* psi_blocked, double* out, heff_stream stream);

/* Same as heff_apply with HOST psi / out (pageable or pinned); copies in and out on
 * `stream` and synchronises it.  The end-to-end entry point. */
int heff_apply_host(heff_plan p, const double* psi_host, double* out_host, heff_stream stream);

/* Lowest eigenpair of H_eff by Lanczos with full (CGS2) reorthogonalisation.
 * psi: in = start vector, out = normalised Ritz vector (device; the local shard
 * [mL][d1][d2][nb] on a communicating sharded plan, else the full vector).
 * energy: lowest Ritz value; iters_done: matvecs performed; resid_est:
 * beta_j |y_j[last]|.  Synchronous.  HEFF_EZERO if psi == 0 (psi is then left unchanged;
 * on plans without a communicator the test is made at the first scalar read-back, so the
 * call costs one host round trip less).  opts->theta_out == NULL in fixed mode: only the
 * breakdown test runs per step, and the last step's tridiagonal problem is solved once. */
int lanczos_ground(heff_plan p, double* psi, const heff_lanczos_opts* opts, double* energy, int* iters_done,
                   double* resid_est, heff_stream stream);

/* MPO sums ("loops over them internally as if they were summed"):
 * a composite plan whose matvec is sum_t H_eff^(t) psi over borrowed term plans (same
 * mL, d1, d2, mR; single-GPU, non-composite).  The terms must outlive the composite;
 * heff_destroy(composite) does not destroy them.  Usable with heff_apply,
 * heff_apply_host, lanczos_ground and heff_set_penalty. */
int heff_create_sum(heff_plan* out, const heff_plan* terms, int nterms);

/* Excited states by energy penalty: after this call every matvec of `p`
 * computes H_eff psi + weight * sum_i phi_i <phi_i|psi>.  phis: DEVICE array
 * [nphi][mL*d1*d2*mR] (copied; may be freed after the call).  nphi = 0 removes the
 * penalty.  Not supported on b'-sharded plans (HEFF_EUNSUPPORTED). */
int heff_set_penalty(heff_plan p, const double* phis, int nphi, double weight, heff_stream stream);

/* Destroys a plan: waits for the plan's last enqueued operation (a completion event
 * recorded by heff_apply / heff_apply_blocked / heff_set_penalty; the whole device if the
 * plan never ran), then returns its workspace blocks to the cache described at
 * heff_release_caches. */
int heff_destroy(heff_plan p);

/* Thread-local message describing the last failure on this thread ("" if none). */
const char* heff_last_error(void);

/* Device bytes the plan allocates for matvec workspace (excluding the Lanczos basis). */
size_t heff_workspace_bytes(const heff_dims* dims, const heff_dist* dist);

/* The layout map applied after the all-gather of b'-shards: src [P][rows][nb] ->
 * dst [rows][P*nb] (device pointers, no aliasing).  Exposed for tests and for callers
 * that gather shards themselves.  Asynchronous on `stream`. */
int heff_relayout_blocked(const double* src, double* dst, int64_t rows, int64_t nb, int P, heff_stream stream);

/* The Lanczos reduction kernels as a primitive (for kernel-level tests): *result (HOST) =
 * sum_i x[i] y[i] over n DEVICE doubles, with the same deterministic two-pass reduction
 * (per-block partials, fixed-order second pass) lanczos_ground uses.  Synchronous. */
int heff_dot(int64_t n, const double* x, const double* y, double* result, heff_stream stream);

/* Writes a fresh 128-byte ncclUniqueId (rank 0 calls this, then broadcasts it). */
int heff_nccl_unique_id(unsigned char uid[128]);

/* Tuning / test knobs.  HEFF_OPT_GEMM_PATH: 0 auto (small bonds: the fused one-launch
 * matvec kernel; otherwise the TMA DMMA GEMM where the operands allow it), 1 plain-load DMMA
 * GEMM, 2 TMA DMMA GEMM.
 * HEFF_OPT_LAST_KERNEL_COUNT (get only): kernels launched by the last heff_apply. */
enum { HEFF_OPT_GEMM_PATH = 1, HEFF_OPT_LAST_KERNEL_COUNT = 2, HEFF_OPT_MPO_NNZ = 3 };
int heff_set_option(heff_plan p, int option, int64_t value);
int heff_get_option(heff_plan p, int option, int64_t* value);

/* Kernel timing.  With HEFF_OPT_PROFILE = 1 every matvec (chunk) records CUDA events on
 * its launch stream around its first GEMM, the fused MPO kernel and its last GEMM, with
 * no host synchronisation.  heff_last_timings waits for them, returns the summed ms of
 * each of the three since the previous call (n_recorded = matvec chunks) and resets.
 * HEFF_OPT_TOTAL_LAUNCHES: kernels launched on this plan (set resets the counter). */
enum { HEFF_OPT_PROFILE = 4, HEFF_OPT_TOTAL_LAUNCHES = 5 };
int heff_last_timings(heff_plan p, float* ms_gemm_first, float* ms_mpo, float* ms_gemm_last, float* n_recorded);

/* The FP64 tensor-core GEMM of the hot path as a primitive: C[M][N] (+)= A[M][K] . op(B),
 * op(B) = B[K][N] (b_kmajor = 0, row pitch ldb) or B[N][K]^T (b_kmajor = 1).  Row-major
 * device pointers; accumulate != 0 adds into C; path as HEFF_OPT_GEMM_PATH.  Async. */
int heff_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb, int b_kmajor,
              double* C, int64_t ldc, int accumulate, int path, heff_stream stream);

/* Host-only (no device work): lowest eigenpair of the symmetric tridiagonal T with
 * diagonal alpha[0..j) and off-diagonal beta[0..j-1) by implicit-shift QL -- the solver
 * lanczos_ground runs on T_j.  y (optional, j doubles): unit eigenvector, largest-|.|
 * component positive (reading R14). */
int heff_tridiag_lowest(int j, const double* alpha, const double* beta, double* theta, double* y);

/* Host-only: the O(j) per-step check lanczos_ground runs after every step -- the lowest
 * eigenvalue of T_j by Sturm-sequence bisection to machine precision and |y_j[last]| of its
 * unit eigenvector by two steps of inverse iteration (tridiagonal LU with partial pivoting);
 * *ylast's sign is arbitrary.  The stopping test beta_j |y_j[last]| <= tol ||T_j|| and
 * theta_out use it; the returned energy and Ritz vector come from heff_tridiag_lowest.
 * Errors: HEFF_EINVAL (j < 1 or a null pointer). */
int heff_tridiag_lowest_check(int j, const double* alpha, const double* beta, double* theta, double* ylast);

/* ---- U(1) block sparsity (Sec. 7) -----------------
 * Declares conserved charges so heff_apply skips the GEMM k-blocks that are zero by
 * symmetry.  Conventions (reading R18): a bond index carries the total charge to
 * its left; L[a',w,a] = 0 unless qa[a'] - qa[a] = cL[w]; R[b',w,b] = 0 unless
 * qb[b'] - qb[b] = cR[w]; psi[a,s1,s2,b] = 0 unless qb[b] = qa[a] + qs1[s1] + qs2[s2]
 * (W1/W2 must conserve charge with channel charges cL -> cM -> cR).  qa (mL) and qb (mR)
 * are nondecreasing (sector-sorted bonds).  All arrays are HOST int arrays, copied.
 * Tensors stay dense; entries the declaration says are zero must be zero, otherwise the
 * result is undefined.  qn == NULL returns the plan to dense.  Single-GPU, unchunked
 * order-A plans only (HEFF_EUNSUPPORTED otherwise). */
typedef struct {
  const int* qa;
  const int* qb;
  const int* qs1;
  const int* qs2;
  const int* cL;
  const int* cM;
  const int* cR;
} heff_qn;
int heff_set_qn(heff_plan p, const heff_qn* qn);
enum { HEFF_OPT_SPARSE_KBLOCKS = 6 }; /* get: scheduled (tile, 16-wide k-block) products per matvec */

/* Gather-fused sharded Lanczos.  HEFF_OPT_FUSED_GATHER = 1 on a
 * communicating b'-sharded plan (default: env HEFF_FUSED_GATHER, else 0): lanczos_ground
 * keeps its Krylov basis in an NCCL symmetric-memory window (ncclMemAlloc +
 * ncclCommWindowRegister, collective on the first call) and every matvec's GEMM_A reads the
 * ranks' shards of v_j directly through their NVLink load/store pointers -- no ncclAllGather,
 * no re-layout.  Ordering: after writing its shard of v_j a rank releases a flag in every
 * rank's window; the matvec waits (acquire) for all flags (20 s bound -> HEFF_ENCCL).
 * get returns option | 2 * (the last lanczos_ground used the fused path).  Requires
 * nb % 16 == 0 and nranks <= 8; real, non-U(1) plans. */
enum { HEFF_OPT_FUSED_GATHER = 7 };

/* HEFF_OPT_LANCZOS_RESERVE = n (set only): allocate lanczos_ground's Krylov workspace for
 * n iterations now (synchronous), so later calls with max_iter <= n allocate nothing --
 * keeps cudaMalloc/cudaFree out of timed or latency-critical calls.  Collective for
 * gather-fused sharded plans (the symmetric window is registered on every rank). */
enum { HEFF_OPT_LANCZOS_RESERVE = 8 };

/* Communicating plans (dist with a uid).
 * HEFF_OPT_FORCE_ALLGATHER = 1: lanczos_ground runs the P > 1 exchange (ncclAllGather of
 *   the shard into the blocked buffer + the re-layout kernel) even on a 1-rank
 *   communicator, where it otherwise copies the shard (default: env HEFF_FORCE_ALLGATHER).
 * Failure detection: every host wait of lanczos_ground on a communicating plan
 *   polls the stream, ncclCommGetAsyncError and a no-progress timeout (env
 *   HEFF_NCCL_TIMEOUT_S, default 300 s without a Lanczos step completing); a gather-fused
 *   peer wait that times out (20 s) counts as an error too.  On error the plan calls
 *   ncclCommAbort -- so the peers' collectives fail instead of hanging -- and returns
 *   HEFF_ENCCL; the plan is then unusable (every later call returns HEFF_ENCCL; destroy it).
 * HEFF_OPT_COMM_STATE (get only): 1 live communicator, 0 none, -1 aborted. */
enum { HEFF_OPT_FORCE_ALLGATHER = 9, HEFF_OPT_COMM_STATE = 10 };

/* ---- Environment update --------------------------------------
 * After each local eigensolve a DMRG sweep moves the window one site and grows the
 * environment by that site (Sec. 6.2; SPEC ProjMPO):
 *   left:  Lout[a',w',a] = sum A[x',s',a'] L[x',w,x] W[w,s',s,w'] A[x,s,a]
 *          L [mi][kl][mi], A [mi][d][mo] (left-orthonormal site tensor), W [kl][d][d][kr]
 *          -> Lout [mo][kr][mo]
 *   right: Rout[b',w,b]  = sum B[b',s',y'] R[y',w',y] W[w,s',s,w'] B[b,s,y]
 *          R [mi][kr][mi], B [mo][d][mi] (right-orthonormal), W [kl][d][d][kr]
 *          -> Rout [mo][kl][mo]
 * Device pointers, row-major fp64; Lout/Rout must not alias the inputs.  Workspace
 * (about 2 mi k d mo doubles) lives in a per-thread arena that grows on demand and is
 * reused by later calls; the call synchronises `stream` before returning. */
typedef struct {
  int64_t mi, d, mo, kl, kr;
} heff_env_dims;
int heff_env_update_left(const heff_env_dims* dims, const double* L, const double* A, const double* W, double* Lout,
                         heff_stream stream);
int heff_env_update_right(const heff_env_dims* dims, const double* R, const double* B, const double* W, double* Rout,
                          heff_stream stream);

/* U(1) environment updates (NEXT-1 x NEXT-3): the same contraction with conserved charges
 * declared (reading R18) so both GEMMs skip the k-blocks that vanish by symmetry.  HOST int
 * arrays: q_in = charges of the incoming environment's bond (mi: x for left, y for right),
 * q_out = charges of the site tensor's new bond (mo: a for left, b for right), qs (d),
 * cl (kl) / cr (kr) = MPO channel charges of W's left / right bond.  The tensors must vanish
 * where the charges forbid (undefined result otherwise); bonds should be sector-sorted for
 * the schedule to pay off (the plain dense schedule is used when it does not). */
typedef struct {
  const int* q_in;
  const int* q_out;
  const int* qs;
  const int* cl;
  const int* cr;
} heff_env_qn;
int heff_env_update_left_qn(const heff_env_dims* dims, const double* L, const double* A, const double* W, double* Lout,
                            const heff_env_qn* qn, heff_stream stream);
int heff_env_update_right_qn(const heff_env_dims* dims, const double* R, const double* B, const double* W,
                             double* Rout, const heff_env_qn* qn, heff_stream stream);

/* ---- Two-site split ---------------------------------------------
 * After each local eigensolve a sweep splits the two-site wavefunction with a truncated SVD
 * (Sec. 5: "U,S,V = svd(W,(j,i);cutoff=1E-8,maxdim=10)"; Sec. 6.2,
 * PAPER.md:705-737).  psi is viewed as the matrix Psi[(a s1)][(s2 b)] of M = mL*d1 rows and
 * N = d2*mR columns (row-major, no copy) and factored Psi ~= U diag(s) V^T, keeping n values:
 *   dir 0 (moving right): Q = U [M][n] (left-orthonormal A[a][s1][k]),  C = diag(s) V^T [n][N]
 *   dir 1 (moving left):  Q = V^T [n][N] (right-orthonormal B[k][s2][b]), C = U diag(s) [M][n]
 * Truncation (readings R20-R22): n is the smallest count whose discarded weight
 * sum_{i>=n} s_i^2 <= cutoff * sum_i s_i^2, raised to mindim, capped at maxdim (<= 0:
 * unlimited); s_i <= 1e-12 s_1 are numerical zeros and never kept.  Each kept vector's sign
 * makes the largest-|.| entry of Q's vector positive (first on ties).
 * Arguments: psi, Q, S, C are DEVICE pointers (fp64; psi is not modified; Q and C are
 * written compactly with row pitch n resp. N -- allocate for n <= min(M, N, maxdim)).
 * S receives all min(M, N) singular values, descending.  n_kept, trunc_err (relative
 * discarded weight) and sweeps (Jacobi sweeps used; may be NULL) are HOST pointers.
 * trunc == NULL: cutoff 0, maxdim unlimited, mindim 1.  Errors: HEFF_EINVAL (bad sizes,
 * cutoff < 0, dir not 0/1), HEFF_EZERO (psi == 0), HEFF_ENOCONV (Jacobi sweep cap).
 * Workspace lives in a per-thread arena (about 4 M N + 2 n max(M, N) doubles, grown on
 * demand and kept for later calls).  Synchronous on `stream`. */
typedef struct {
  double cutoff;
  int64_t maxdim;
  int64_t mindim;
} heff_trunc;
int heff_svd_split(int64_t M, int64_t N, const double* psi, const heff_trunc* trunc, int dir, double* Q, double* S,
                   double* C, int64_t* n_kept, double* trunc_err, int* sweeps, heff_stream stream);

/* U(1) two-site split (NEXT-2 x NEXT-3, reading R24; block-sparse factorizations,
 * P:L1076-1085): qrow[M] / qcol[N] are HOST charge arrays of Psi's rows (a s1) and columns
 * (s2 b) -- for the R18 convention qrow = q(a) + q(s1), qcol = q(b) - q(s2).  Psi must vanish
 * where qrow[r] != qcol[c] (HEFF_EINVAL otherwise).  Every charge block is split by the dense
 * algorithm, one truncation (R20/R21) runs over the union of the blocks' values, and the new
 * bond is ordered by charge (ascending) then by descending value.  Outputs as heff_svd_split
 * plus Sk (DEVICE, n doubles: kept values in new-bond order) and qk (HOST, n ints: the new
 * bond's charges); S holds all blocks' values, descending, zero-padded to min(M, N); sweeps =
 * the most Jacobi sweeps any block needed.  Synchronous on `stream`. */
int heff_svd_split_qn(int64_t M, int64_t N, const double* psi, const int* qrow, const int* qcol,
                      const heff_trunc* trunc, int dir, double* Q, double* S, double* Sk, int* qk, double* C,
                      int64_t* n_kept, double* trunc_err, int* sweeps, heff_stream stream);

/* Frees the on-demand workspaces that heff_env_update_*, heff_gemm, heff_svd_split and
 * heff_svd_split_qn keep per host thread (and those of the U(1) split's worker threads),
 * and the workspace cache of destroyed plans on the current device (heff_destroy returns
 * a plan's intermediates, Krylov basis and staging buffers to a process-wide cache -- blocks
 * up to 4 GB, 16 GB in total -- that the next heff_create / lanczos_ground reuses: a DMRG
 * sweep builds one plan per bond); they are re-allocated by the next call.  Synchronises
 * the device. */
int heff_release_caches(void);

/* Host-only (no device work): the truncation rule heff_svd_split applies, on HOST values
 * s[0..k) (descending, non-negative).  n_kept / trunc_err as in heff_svd_split.
 * HEFF_EINVAL (not descending, negative, cutoff < 0), HEFF_EZERO (s[0] == 0). */
int heff_truncate_spectrum(const double* s, int64_t k, const heff_trunc* trunc, int64_t* n_kept, double* trunc_err);

#ifdef __cplusplus
}
#endif
#endif /* HEFF_H */
