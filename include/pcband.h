/*
 * pcband.h — C ABI of the B200-native compensated-Yee band solver (libpcband.so).
 *
 * Method: Jin & Xie, arXiv 2511.17107 ("PAPER.md" below; "P:123" = PAPER.md line 123).
 * The library computes, matrix-free on one GPU, in complex FP64,
 *
 *     Op(k) = A_c M_eps A_c^H + gamma(k) B^H B                     (display:kc_formulation)
 *
 * on an N^3 Bloch-shifted Yee grid, its FFT-diagonal preconditioner K_P^{-1}, and the
 * smallest eigenvalues omega^2 of Op(k) by block LOBPCG with soft locking.
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Complex numbers are interleaved (re, im) doubles (== cuDoubleComplex == torch.complex128).
 *  - A field is 3*N^3 complex values, component-major [c][z][y][x], x fastest (the Kronecker
 *    factor of axis 1 is the last one).  A block of ncols fields is column-major: column j starts at
 *    base + j*ld (ld in complex elements, ld >= 3*N^3).
 *  - Fourier coordinates: x = F3^H H, F_ij = w^{(i-1)(j-1)}/sqrt(N), w = exp(+2 pi i/N)
 *    (P:274), i.e. x = numpy.fft.fftn(H, norm="ortho") per component, modes m unshifted, same
 *    [c][m3][m2][m1] layout.
 *  - Device pointers (X, Y, R, P, evecs) are caller-owned CUDA device memory on the context's
 *    device; they must not alias each other.  Host pointers are noted as such.
 *  - stream arguments are cudaStream_t passed as void* (NULL = legacy default stream).  pc_apply /
 *    pc_precond / pc_apply_eps / pc_fft3 are asynchronous and stream-ordered; pc_bands is synchronous.
 *  - Calls on one context must be serialised by the caller (the workspace is per context).
 *    Different contexts share nothing and may be used concurrently.
 *
 * Errors: every int-returning call returns PC_OK (0) on success, a negative PC_E* code on failure
 * (no output written; message via pc_last_error(), thread-local), or PC_ENOTCONV (1) from pc_bands
 * when at least one k-point hit maxit (its best pairs are still returned, status[k] = 1;
 * SPEC "max_iter exceeded -> converged=false and best available pairs").
 */
#ifndef PCBAND_H
#define PCBAND_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pc_ctx pc_ctx; /* opaque, library-owned */

enum {
  PC_OK = 0,
  PC_ENOTCONV = 1,  /* pc_bands: some k-point did not reach tol within maxit                       */
  PC_EINVAL = -1,   /* bad argument: unsupported N, non-Hermitian eps1, singular A, bad sizes ...    */
  PC_ENOTPD = -2,   /* eps1 is not positive definite (P:69 requires HPD)                             */
  PC_ECUDA = -3,    /* a CUDA runtime error (message has the CUDA string)                            */
  PC_ENOMEM = -4,   /* device allocation failed                                                      */
  PC_ENUMERIC = -5  /* pc_bands: Rayleigh-Ritz breakdown that restarting could not repair            */
};

/* Discretisation of eps^{-1} (Section 3 of the paper). */
enum {
  PC_EPS_DIAGONAL = 0, /* M_ii = (eps_ii - 1) I_i + I, off-diagonal blocks 0      */
  PC_EPS_CROSSDOF = 1, /* off-diagonal eps_ij S_ij, S_ij = (I_i T_ij + T_ij I_j)/2      */
  PC_EPS_TRIVIAL = 2   /* off-diagonal eps_ij I_V (pointwise volume indicator)          */
};

enum { PC_SPACE_FOURIER = 0, PC_SPACE_REAL = 1 };
enum { PC_FFT_TO_FOURIER = 0 /* x = F3^H H */, PC_FFT_TO_REAL = 1 /* H = F3 x */ };

/* hpd_flags bits reported by pc_info (Assumptions 1-3; Props). */
enum {
  PC_HPD_ASSUMP1 = 1,    /* spec(eps1) in (0, 1]                      */
  PC_HPD_SDD = 2,        /* eps1 strictly diagonally dominant          */
  PC_HPD_ZERO_OFFD = 4,  /* at least one off-diagonal entry is zero    */
  PC_HPD_GUARANTEED = 8  /* Assump.1 and (SDD or zero off-diagonal): M_CrossDoF / M_Trivial HPD */
};

/*
 * pc_create — build a context for one (lattice, grid, eps1, geometry) problem.
 *   A[9]       host, row-major 3x3 whose COLUMNS are a_1, a_2, a_3: A[3*r+c] = (a_c)_r.
 *              Must be invertible; B = A^{-1} enters the shifted blocks (reading R3:
 *              Dhat_i = sum_j b_ji D_{1,j} + i k_i D_{0,i}).
 *   n          grid division N (h = 1/N), one of the sizes listed by pc_supported_n().
 *   eps1[18]   host, 3x3 complex row-major interleaved (re,im): the inverse permittivity inside
 *              Omega_1.  Must be Hermitian (|e_ij - conj e_ji| <= 1e-14 max|e|) -> else
 *              PC_EINVAL, and positive definite -> else PC_ENOTPD.  Violations of Assumptions 1-3
 *              only set pc_info flags ("hpd_report never blocks a run", SPEC).
 *   masks      host, uint8, 4*N^3: I_1, I_2, I_3, I_V, each [z][y][x], entries 0/1,
 *              sampled at the DoF locations (reading R6).  Copied to the device; not retained.
 *   eps_mode   PC_EPS_*.  PC_EPS_DIAGONAL with non-zero off-diagonal eps1 -> PC_EINVAL.
 *   gamma_override  > 0: use this penalty for every k; <= 0: the practical rule P:457-462.
 *   device     CUDA device ordinal.
 * On success *out receives the context (free with pc_destroy).
 */
int pc_create(pc_ctx **out, const double A[9], int n, const double eps1[18], const uint8_t *masks,
              int eps_mode, double gamma_override, int device);

/*
 * pc_apply — Y = Op(k) X for ncols columns (P:523-529 / display:matrixfree_finalform).
 *   space = PC_SPACE_FOURIER: X, Y are Fourier-coordinate fields; Y = K_A F3^H M F3 K_A^H X
 *           + gamma K_B X, computed as one inverse and one forward 3-D DFT per column with the
 *           curl symbol fused into the first pass and K_A + gamma K_B into the last.
 *   space = PC_SPACE_REAL: X, Y are real-space face fields H; Y = (A_c M A_c^H + gamma B^H B) X.
 *   k[3]  host, Bloch vector (Cartesian).  X, Y device, ld >= 3N^3, ncols >= 0
 *   (ncols = 0 is a no-op).  X and Y must not alias.
 */
int pc_apply(pc_ctx *ctx, const double k[3], const void *X, void *Y, int ncols, long long ld,
             int space, void *stream);

/*
 * pc_precond — P = K_P^{-1} R per Fourier mode, K_P = K_A K_A^H + gamma K_B
 * = |kappa|^2 I + (gamma - 1) conj(kappa) kappa^T, closed form
 * P = R/|kappa|^2 - (gamma-1)/(gamma |kappa|^4) conj(kappa)(kappa^T R); modes with
 * |kappa|^2 <= 1e-28 max|kappa|^2 pass through unchanged (reading R7).  Fourier coordinates only.
 * R, P device; P may equal R (in place).
 * With option "precond" = 1 the call returns instead the eps-weighted preconditioner (beyond the
 * paper, R16) T R = K_A^{+H} F3^H D^{-1} F3 K_A^+ R + Pi R / (gamma |kappa|^2), with
 * K_A^+ = K_A^H / |kappa|^2, Pi = conj(kappa) kappa^T / |kappa|^2 and D = diag(M_eps);
 * zero-symbol modes map to 0.  It uses the context workspace (ncols columns, grown on demand).
 */
int pc_precond(pc_ctx *ctx, const double k[3], const void *R, void *P, int ncols, long long ld,
               void *stream);

/*
 * pc_apply_eps — debug/parity entry: Y = M_eps E in real space, E edge fields.
 */
int pc_apply_eps(pc_ctx *ctx, const void *E, void *Y, int ncols, long long ld, void *stream);

/*
 * pc_fft3 — debug/parity entry: unitary 3-D DFT of each component.
 *   direction PC_FFT_TO_FOURIER: Y = F3^H X (numpy fftn, ortho); PC_FFT_TO_REAL: Y = F3 X.
 *   Y may equal X (in place).
 */
int pc_fft3(pc_ctx *ctx, const void *X, void *Y, int ncols, long long ld, int direction,
            void *stream);

/*
 * pc_bands — the nev smallest eigenvalues omega^2 of Op(k) at each of nk Bloch vectors
 * (kernel-compensation formulation P:254-262; LOBPCG with soft locking P:1055-1056).
 *   kpts     host, nk*3 Cartesian Bloch vectors.
 *   nev      number of eigenvalues (>= 1); block size = nev + guard (pc_set_option "guard",
 *            default 6, reading R14).
 *   tol      convergence when Res_j = ||Op x_j - w_j x_j|| / ||x_j|| <= tol for all j < nev
 *            (the paper uses 1e-5).
 *   maxit    iteration cap (SPEC default 500).
 *   seed     start block of k-point i is drawn from a counter-based generator keyed by
 *            (seed, i) — independent of how k-points are split across GPUs.
 *   omega2   host out, nk*nev, ascending per k.  At k = 0 exactly the 3-dimensional null space
 *            (constant fields) is deflated and the nev smallest positive eigenvalues
 *            are returned (reading R12).
 *   resid    host out (may be NULL), nk*nev final Res_j.
 *   iters    host out (may be NULL), nk iteration counts.
 *   status   host out (may be NULL), nk: 0 converged, 1 maxit reached.
 *   evecs    NULL, or device buffer of nk*nev columns (ld = 3N^3), k-major: Fourier-coordinate
 *            eigenvectors, unit 2-norm.
 * Returns PC_OK, PC_ENOTCONV, or a negative error.
 */
int pc_bands(pc_ctx *ctx, const double *kpts, int nk, int nev, double tol, int maxit,
             unsigned long long seed, double *omega2, double *resid, int *iters, int *status,
             void *evecs);

/*
 * pc_apply_multi / pc_precond_multi — several Bloch vectors in ONE launch (k as an
 * extra column dimension; at n <= 64 one k-point's block under-fills 148 SMs).  Column j of X / R is
 * processed with k = kpts[3*kcol[j] .. 3*kcol[j]+2]: pc_apply_multi computes Y_j = Op(k) X_j in Fourier
 * coordinates exactly as pc_apply (PC_SPACE_FOURIER), pc_precond_multi P_j = K_P(k)^{-1} R_j as
 * pc_precond (the paper's K_P^{-1}, whatever option "precond" says).  Per-k symbol tables,
 * penalties gamma(k) and pass-through thresholds (reading R7) live in a context buffer.
 *   kpts  host, nk*3 Cartesian Bloch vectors, 1 <= nk <= 16
 *   kcol  host, ncols ints in [0, nk)
 *   X, Y, R, P, ncols, ld, stream: as pc_apply / pc_precond.
 * Returns PC_EINVAL for nk out of range, a k index out of range, null pointers or aliasing X == Y.
 */
int pc_apply_multi(pc_ctx *ctx, const double *kpts, int nk, const int *kcol, const void *X, void *Y, int ncols,
                   long long ld, void *stream);
int pc_precond_multi(pc_ctx *ctx, const double *kpts, int nk, const int *kcol, const void *R, void *P, int ncols,
                     long long ld, void *stream);

/* Penalty gamma used for k (override if set, else P:457-462). */
double pc_gamma(const pc_ctx *ctx, const double k[3]);

/* hpd_flags: PC_HPD_* bits for eps1; ws_bytes_per_col: apply workspace bytes per column. */
int pc_info(const pc_ctx *ctx, int *hpd_flags, size_t *ws_bytes_per_col);

/*
 * pc_set_option — tuning knobs (return PC_EINVAL for unknown keys):
 *   "guard"        extra LOBPCG block columns beyond nev (default 6)
 *   "apply_chunk"  max columns per batched apply (default 0 = all at once)
 *   "profile"      1: time every kernel class with CUDA events (read with pc_stats), 0: off
 *   "drop_tol"     Rayleigh-Ritz rank threshold on the Jacobi-scaled mass Gram: Cholesky pivots / SVQB
 *                  eigenvalues below it (relative) are dropped and P restarts (default 1e-8; at 1e-12
 *                  an ill-conditioned basis let the Ritz coefficients grow and the solve diverge on
 *                  degenerate vacuum clusters from a Gaussian start)
 *   "kindex_offset" global index of kpts[0] in pc_bands (start-block seeds are keyed by it, so
 *                  results do not depend on how a k-path is split across GPUs; default 0)
 *   "start"        0: Gaussian start block; 1 (default): transverse plane waves of the b/2 modes
 *                  with the smallest |kappa|^2 (eigenvectors of K_P) plus a seeded Gaussian admixture
 *   "start_noise"  relative size of that admixture (default 1e-3)
 *   "start_precond" 1 (default): the admixture is K_P^{-1} of white noise (low modes only, small
 *                  residual); 0: white Gaussian noise
 *   "sticky_lock"  1: a locked column stays locked; 0 (default): it re-enters the search block if
 *                  its residual rises above tol again
 *   "gram_refresh" every n-th iteration forms the full Gram matrices instead of using
 *                  X^H X = I, X^H A X = Lambda (default 16; 0 = never)
 *   "xdev_tol"     if max_j | |X_j|^2 - 1 | exceeds this, the next Gram is formed in full from the
 *                  vectors (default 1e-10)
 *   "p_restart"    1 (default): drop the P block when the basis is numerically rank deficient
 *   "verbose"      1: per-iteration residuals on stderr
 *   "kbatch"       1 (default): pc_bands solves its k-points one after another; K in 2..16: in lock-step
 *                  batches of K: one multi-k operator apply and two host synchronisations per
 *                  LOBPCG iteration for the whole batch, each k-point's Gram / Rayleigh-Ritz / update on
 *                  its own stream; same results as kbatch 1 (the i-th k-point of a call is still keyed by
 *                  kindex_offset + i).  K x (nev + guard) <= 192; ignored with warm_start or precond = 1.
 *                  Pays at n <= 32 (C2: 104 vs 27 k-points/s), equal at n = 64 to concurrent contexts
 *   "warm_start"   1: start each k-point (k != 0) from the Ritz block of the previous pc_bands
 *                  k-point solved on this context (path continuation, not in the
 *                  paper); 0 (default): cold start.  Setting the option forgets the stored block.
 *   "w_guard"      guard columns that receive a search direction W (default 0: only the nev
 *                  wanted columns; -1: all b columns)
 *   "precond"      0 (default): LOBPCG and pc_precond use the paper's K_P^{-1};
 *                  1: the eps-weighted preconditioner (see pc_precond; beyond the paper): one extra
 *                  5-pass apply of the active W columns per iteration, ~40 % fewer iterations
 *   "precond_fuse" 1 (default): with precond = 1, pc_bands runs the preconditioner's last pass and the
 *                  next apply's first pass as one pass; 0: separately
 *   "fuse_xex"     1 (default): fused x-DFT + M_eps + x-DFT pass when eps_13 = eps_23 = 0 (or
 *                  Diagonal/Trivial mode); 0: 7-pass pipeline with the standalone stencil
 *   "plane_fuse"   1: at n = 128 the y-inverse, x-inverse + M_eps + x-forward and y-forward passes of
 *                  a z-plane-local medium run as one pass over thread-block clusters of 16 CTAs
 *                  (plane2.cu: 3 HBM passes per apply instead of 5; measured slower: 2.67 vs 1.93 ms
 *                  per 15 columns); 0 (default): the three passes
 *   "fuse_resid"   1 (default): both block updates + next residual + K_P^{-1} in one pass; 0: two
 *                  update launches and a separate residual pass
 *   "update_tmap"  1 (default): block-update kernel with TMA tensor-copy row tiles in a 2-stage
 *                  ring (update_tmap.cu); 0: per-thread cp.async tiles (update_all.cu)
 *   "gram_narrow"  1 (default): 8/16-column block shapes for narrow Gram products (tail iterations);
 *                  0: the wide shapes only (process-wide)
 *   "jacobi_tol"   rotation threshold of the Rayleigh-Ritz Jacobi sweeps, |a_pq| <= tol sqrt(|a_pp a_qq|)
 *                  (process-wide; default 1e-16)
 */
int pc_set_option(pc_ctx *ctx, const char *key, double value);

/*
 * pc_stats — cumulative per-kernel-class statistics since the last reset.  out: host,
 * 4*PC_NSTAT + 1 doubles: for class i (enum order below) out[4i] = timed launch groups,
 * out[4i+1] = CUDA-event milliseconds on the launching stream (only while option "profile" = 1),
 * out[4i+2] = algorithmic flops, out[4i+3] = algorithmic bytes (what the method must move, not
 * what the kernels moved); out[4*PC_NSTAT] = number of kernel launches.  reset != 0 clears them.
 */
enum {
  PC_STAT_FFT_Z_KAH = 0,   /* first inverse pass with K_A^H fused      */
  PC_STAT_FFT_MID = 1,     /* plain pencil passes                       */
  PC_STAT_EPS = 2,         /* real-space M_eps stencil                  */
  PC_STAT_FFT_Z_KA = 3,    /* last forward pass with K_A + gamma K_B    */
  PC_STAT_RESID = 4,       /* residual + K_P^{-1} + norms               */
  PC_STAT_GRAM = 5,        /* S^H [S AS] Gram products                  */
  PC_STAT_RR = 6,          /* on-device Rayleigh-Ritz                   */
  PC_STAT_UPDATE = 7,      /* block updates X, P, AX, AP                */
  PC_STAT_OTHER = 8,       /* init, reductions, copies                  */
  PC_NSTAT = 9
};
int pc_stats(pc_ctx *ctx, double *out, int reset);

/*
 * pc_debug_heevj — test entry for the on-device Jacobi eigensolver used by the Rayleigh-Ritz step:
 * A_host (n x n complex, column-major, Hermitian, 1 <= n <= 80) -> w_host ascending eigenvalues,
 * V_host (may be NULL) eigenvectors (column-major), *sweeps Jacobi sweeps used.  Synchronous,
 * current device.
 */
int pc_debug_heevj(const double *A_host, int n, double *w_host, double *V_host, int *sweeps);

/*
 * pc_debug_pass — test entry: one pencil pass of the pc_apply pipeline on ncols columns (device,
 * ld).  kind 0: plain unnormalised 1-D DFT along axis (0 x, 1 y, 2 z), sign dir (-1: e^{-},
 * +1: e^{+}), output scaled by scale; kind 1: u = scale * K_A^H X then e^{+} DFT along z, and
 * g = gamma (kappa . X) written to XH (N^3 complex per column, same ld); kind 2: e^{-} DFT s along
 * z of X then K_A s + conj(kappa) g with g read from XH (= gamma K_B xhat when XH holds the g of
 * kind 1 applied to xhat).  Synchronous.
 */
int pc_debug_pass(pc_ctx *ctx, const double k[3], int kind, int axis, int dir, const void *X, void *Y,
                  const void *XH, int ncols, long long ld, double scale);

/*
 * pc_history — residual history of the last k-point solved by pc_bands on this context: returns the
 * number of iterations R recorded; *block = b (columns); out (host, may be NULL) receives
 * min(R, cap) rows of b doubles Res_j, one row per LOBPCG iteration (row 0 = start
 * block after the first Rayleigh-Ritz step).  Used for the asymptotic damping factor theta.
 */
int pc_history(const pc_ctx *ctx, double *out, int cap, int *block);

/*
 * pc_bench_block — timing entry for the LOBPCG block kernels on random device data
 * in this context's workspace (overwrites any LOBPCG state): the shapes of one iteration with b X
 * columns, na W columns and nP P columns (nP <= na <= b, b + na + nP <= 80, 3b <= 80).  which = 0:
 * fused block update + residual + K_P^{-1} (one launch group as in pc_bands; 3: the TMA variant);
 * 1: Gram S^H [W P AW AP] + assembly (4: the TMA variant); 2: Gram S^H [W AW].  *ms = mean CUDA-event milliseconds per launch
 * group over reps (after one warm-up), on the context's stream.  Synchronous.
 */
int pc_bench_block(pc_ctx *ctx, int which, int b, int na, int nP, int reps, double *ms);

/* Supported grid sizes: writes up to cap values into sizes, returns how many exist. */
int pc_supported_n(int *sizes, int cap);

/* Free the context.  Its large device workspaces go to a process-wide per-device cache that later
 * contexts reuse (so create/destroy per problem avoids re-allocating ~16 GB at n = 128). */
void pc_destroy(pc_ctx *ctx);

/* Return the cached device blocks of `device` (all devices if device < 0) to the CUDA driver.  Only
 * blocks of destroyed contexts are cached; live contexts are unaffected.  Thread-safe. */
void pc_trim(int device);
const char *pc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PCBAND_H */
