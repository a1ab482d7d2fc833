// Internal interface between the host driver (pcband.cu) and the kernel translation units.
#pragma once
#include <algorithm>
#include "common.cuh"

#define PC_MAXCOLS 192  // column pointers per launch (Gram T side = [S AS] = 6b, b <= 32)

struct ColPtrs {
  const cplx* p[PC_MAXCOLS];
};
struct MutColPtrs {
  cplx* p[PC_MAXCOLS];
};

struct Sym3 {
  double B[9];  // row-major A^{-1}: B[3*a + i] = b_ai
  double k[3];
};

struct EpsCoef {
  double d[3];  // eps_ii - 1
  cplx e[3];    // eps_12, eps_13, eps_23
  int has[3];   // which off-diagonals are non-zero
};

#define PC_MAXK 16  // Bloch vectors per multi-k launch (pc_apply_multi / pc_precond_multi)

// Several k-points in one launch: column j uses the symbol table ktab + kcol[j] * 9N and the
// penalty / pass-through threshold of its k.
struct MultiK {
  int on = 0;
  unsigned char kcol[PC_MAXCOLS];
  double gamma[PC_MAXK], thr[PC_MAXK];
};

struct PassArgsH {
  const cplx* tw;    // tw[j] = exp(-2 pi i j / N)
  const cplx* ktab;  // symbol pieces, see pointwise.cu (multik: PC_MAXK consecutive 9N tables)
  double gamma;
  double scale;
  int z0 = 0, nz = 0;  // x/y passes: restrict to z-planes [z0, z0+nz) (nz = 0: all)
  double gamma2 = 0.0; // OP_KAGH: gamma of the apply that follows the preconditioner
  int kscale = 0;      // OP_KAG: output scaled by 1/|kappa|^2 per mode (0 where |kappa|^2 <= thr): the
  double thr = 0.0;    // last pass of the eps-weighted preconditioner (pcband.cu, precond_eps)
  MultiK mk;           // mk.on: per-column k (ktab, gamma, thr of k index mk.kcol[col])
};

// Persistent grids: 148 SMs x resident CTAs per SM.
int grid_cap(int ctas_per_sm);

// FFT passes ------------------------------------------------------------------------------
// kind: 0 plain (C=1), 1 inverse-z with K_A^H prologue (C=3), 2 forward-z with K_A+gamma K_B (C=3)
// in/out/xh: per-column pointers (xh only for kind 2: the apply's input x_hat), ncols <= PC_MAXCOLS.
int fft_supported(int n);
int fft_supported_list(int* sizes, int cap);
cudaError_t launch_fft_pass(int n, int axis, int dir, int kind, const ColPtrs& in, const MutColPtrs& out,
                            const ColPtrs& xh, int ncols, const PassArgsH& a, cudaStream_t st);

// fused x-inverse DFT + M_eps + x-forward DFT (media with eps_13 = eps_23 = 0 in CrossDoF mode; any
// Diagonal/Trivial medium): in -> out (must differ), output scaled by `scale`.
cudaError_t launch_xex(int n, int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, const uint8_t* mask,
                       const EpsCoef& ec, const cplx* tw, double scale, int z0, int nz, cudaStream_t st);

// fused xy-plane pass (plane2.cu, N = 128): y-inverse DFT, x-inverse DFT, M_eps (same media as
// launch_xex), x-forward DFT, y-forward DFT of every z-plane of every column, unnormalised, in -> out
// (must differ).  One thread-block cluster of 16 CTAs per z-plane (distributed shared memory).
bool plane2_supported(int n);
cudaError_t launch_plane2(int n, int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, const uint8_t* mask,
                          const EpsCoef& ec, const cplx* tw, cudaStream_t st);

// pointwise ---------------------------------------------------------------------------------
void launch_ktab(cplx* ktab, const cplx* tw, int n, const Sym3& s, cudaStream_t st);
void launch_precond(const ColPtrs& in, const MutColPtrs& out, int ncols, int n, const cplx* kt, double gamma,
                    double thr, cudaStream_t st, const MultiK* mk = nullptr);
void launch_eps(int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, int n, const uint8_t* mask,
                const EpsCoef& ec, cudaStream_t st);
int resid_grid(int n);
void launch_resid(const ColPtrs& X, const ColPtrs& AX, const MutColPtrs& W, const double* lam, int b, int n,
                  const cplx* kt, double gamma, double thr, int deflate0, double* partial, double* norms,
                  cudaStream_t st);
void launch_reduce_partial(const double* partial, int nb, int ncols, double* norms, cudaStream_t st);
void launch_randn(const MutColPtrs& X, int ncols, long long len, unsigned long long seed, int deflate_stride,
                  double scale, cudaStream_t st);
// plane-wave start block: per-CTA PW_T smallest |kappa|^2 (pw_grid() CTAs), then a host-built scatter
#define PW_T 16
struct PwEntry {
  int col, mode;
  double v[6];  // 3 complex components
};
int pw_grid();
void launch_kappa2_topk(const cplx* kt, int n, double thr, double* outv, int* outi, cudaStream_t st);
void launch_pw_scatter(const MutColPtrs& X, const PwEntry* e, int ne, int n3, cudaStream_t st);

// dense block algebra ------------------------------------------------------------------------
// G (p x q, column-major, ld p) = S^H T over rows [0, len): S p columns, T q columns.
size_t gram_partial_bytes(int p, int q);
// [G_M | G_A] (p x 2p) from Gp = S^H [W P AW AP] (p x 2c), S = [X W P], b = |X|, c = |W| + |P|,
// assuming X^H X = I, X^H A X = diag(lambda) (Ritz vectors of the previous Rayleigh-Ritz step).
void launch_gram_assemble(const cplx* Gp, const double* lam, int b, int c, cplx* G, cudaStream_t st);
void launch_gram(const ColPtrs& S, int p, const ColPtrs& T, int q, long long len, cplx* G, cplx* partial,
                 cudaStream_t st);
void set_gram_narrow(int v);  // 1 (default): 8/16-column T block shapes for narrow Grams (process-wide)
// Block update (r <= 32 output columns, C column-major ld = ldc):
//   Y1[:, c] = sum_{m in [split, p)} S[:, m] C[m, c]               (if Y1 != nullptr; columns with Y1->p[c] == nullptr skipped)
//   Y2[:, c] = sum_{m in [0, p)}     S[:, m] C[m, c] (+ add[:, c])
void launch_update(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                   const MutColPtrs& Y2, const ColPtrs* add, long long len, cudaStream_t st);

// Both block updates fused with the next residual (update_all.cu): for S and AS as in launch_update
// (Y1s/Y1a: P', AP' columns [split, p) only, null columns skipped; Y2s/Y2a: X', AX'), then
// R = AX' - X' diag(lam), W[:, c] = K_P^{-1} R[:, c] for W.p[c] != nullptr (mode 0 zeroed if deflate0),
// per-CTA |R_c|^2, |X'_c|^2 into partial[(c * grid + cta) * 2 + {0,1}].  r <= 32.  Returns the grid
// (<= max_grid) for launch_reduce_partial.
int launch_update_all(const ColPtrs& S, const ColPtrs& AS, int p, const cplx* C, int ldc, int r, int split,
                      const MutColPtrs& Y1s, const MutColPtrs& Y2s, const MutColPtrs& Y1a, const MutColPtrs& Y2a,
                      const MutColPtrs& W, const double* lam, int n, const cplx* kt, double gamma, double thr,
                      int deflate0, double* partial, int max_grid, cudaStream_t st);

// Same contract as launch_update_all with the row tiles streamed by TMA tensor copies (update_tmap.cu).
// The basis is given per block k (0: X, 1: W, 2: P) as a column range of one LOBPCG slot: s[k] / as[k]
// = column 0 of the S / AS slot (slot_cols[k] columns, column stride ld complex), box columns
// [c0[k], c0[k] + nc[k]) (nc[k] <= 32; 0 = block absent), crow[k][j] = row of C for box column j
// (-1: not in the basis).  Returns the grid, or -1 if the tensor maps cannot be encoded.
struct UtBlocks {
  const cplx* s[3];
  const cplx* as[3];
  int slot_cols[3];
  long long ld;
  int c0[3], nc[3];
  signed char crow[3][32];
};
bool update_tmap_supported(int n, int b);
int launch_update_tmap(const UtBlocks& blk, const cplx* C, int ldc, int r, const MutColPtrs& Y1s,
                       const MutColPtrs& Y2s, const MutColPtrs& Y1a, const MutColPtrs& Y2a, const MutColPtrs& W,
                       const double* lam, int n, const cplx* kt, double gamma, double thr, int deflate0,
                       double* partial, int max_grid, cudaStream_t st);

// Rayleigh-Ritz ------------------------------------------------------------------------------
// G = [G_M | G_A] (p x 2p, column-major ld p).  Outputs C (p x nb, ld p), lambda (nb), info[0] = rank,
// info[1] = sweeps of the last Jacobi.  Uses scratch (>= 4 p^2 complex).
void launch_rr(const cplx* G, int p, int nb, double drop_tol, cplx* C, double* lambda, int* info, cplx* scratch,
               cudaStream_t st);
void set_jacobi_tol(double t);  // tuning knob: Jacobi rotation threshold of the Rayleigh-Ritz step
// Dense Hermitian eigensolver (one-CTA Jacobi) for tests: A (n x n, ld n) -> w (n, ascending), V (n x n).
void launch_heevj(const cplx* A, int n, double* w, cplx* V, int* info, cudaStream_t st);
