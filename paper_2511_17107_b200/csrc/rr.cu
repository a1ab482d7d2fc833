// On-device Rayleigh-Ritz for LOBPCG: one CTA solves the small projected
// generalized Hermitian eigenproblem  G_A c = theta G_M c  (p <= RR_MAXN) by
//   1. symmetric scaling D = diag(G_M)^{-1/2};
//   2a. Cholesky D G_M D = L L^H (all pivots > drop_tol), H = L^{-1} D G_A D L^{-H}, T = D L^{-H};
//   2b. otherwise (rank-deficient basis): Jacobi D G_M D = V Sigma V^H, drop sigma < drop_tol
//       sigma_max (SVQB-style), T = D V_r Sigma_r^{-1/2}, H = T^H G_A T;
//   3. Jacobi eigendecomposition H = Q Theta Q^H, ascending;
//   4. C = T Q[:, :nb], lambda = Theta[:nb].
// Cyclic parallel Jacobi with a round-robin (tournament) pairing: per round np/2 disjoint complex
// rotations U = [[c, s e], [-s conj(e), c]] (e = a_pq/|a_pq|) are applied as 2x2 blocks
// U_i^H A_{ii'} U_{i'} (one barrier per round) and accumulated into V.
#include "kernels.h"

constexpr int RR_MAXN = 80;
#ifndef PC_RR_THREADS  // 512: a 1024-thread CTA needs a whole SM's registers and waits behind the
#define PC_RR_THREADS 512  // other streams' kernels (C3 with 2 contexts x kbatch 4 ran at half speed)
#endif
constexpr int RR_THREADS = PC_RR_THREADS;
#ifndef PC_RR_EARLY
#define PC_RR_EARLY 1
#endif

struct JacSm {
  int P[RR_MAXN / 2], Q[RR_MAXN / 2];
  double c[RR_MAXN / 2], s[RR_MAXN / 2];
  cplx e[RR_MAXN / 2];
};

DEV void tpair(int r, int i, int m, int& P, int& Q) {
  int a, b;
  if (i == 0) { a = 0; b = 1 + r % (m - 1); }
  else { a = 1 + (r + i) % (m - 1); b = 1 + (r - i + m - 1) % (m - 1); }
  P = min(a, b);
  Q = max(a, b);
}

// A, V column-major with leading dimension ld (= np).  A Hermitian n x n zero-padded to np (even).
// One round: the h = np/2 rotations (one thread each), one barrier, then the h^2 two-sided 2x2 block
// updates of A and the np*h row updates of V as one parallel loop, one barrier.  Stops after a sweep
// without rotations, or (PC_RR_EARLY) after a sweep whose largest relative off-diagonal |a_pq|^2 / |a_pp a_qq| was below max(1e-16, tol^2): cyclic
// Jacobi converges quadratically, so what that sweep leaves is O(1e-16) relative -- the sweep after it
// would only remove rotations at the rounding level.
DEV int jacobi_smem(cplx* A, cplx* V, int n, int np, int ld, JacSm& js, int max_sweeps, double rel_tol = 1e-16) {
  const int tid = threadIdx.x;
  const int h = np / 2;
  const double tol2 = rel_tol * rel_tol;
  const double stop2 = fmax(1e-16, tol2);
  int sweep = 0;
  for (; sweep < max_sweeps; sweep++) {
    int swept = 0;     // any rotation in this sweep (CTA-uniform)
    int big = 0;       // this thread saw a rotation with ratio^2 > stop2 in this sweep
    for (int r = 0; r < np - 1; r++) {
      int rot = 0;
      for (int i = tid; i < h; i += blockDim.x) {
        int P, Q;
        tpair(r, i, np, P, Q);
        double c = 1.0, s = 0.0;
        cplx e = mk(1.0, 0.0);
        if (Q < n) {
          // rotation zeroing a_pq with one reciprocal square root per quantity (no divisions by |a_pq|):
          // e = a_pq / |a_pq|, z = (a_qq - a_pp) / (2 |a_pq|), t = sign(z) / (|z| + sqrt(1 + z^2)),
          // c = 1 / sqrt(1 + t^2), s = t c
          const cplx apq = A[P + Q * ld];
          const double m2 = fma(apq.x, apq.x, apq.y * apq.y);
          const double app = A[P + P * ld].x, aqq = A[Q + Q * ld].x;
          const double dd = fabs(app * aqq);
          if (m2 > 0.0 && m2 > tol2 * dd) {
            const double rm = rsqrt(m2);
            const double z = 0.5 * (aqq - app) * rm;
            const double t = copysign(1.0, z) / (fabs(z) + sqrt(fma(z, z, 1.0)));
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
            e = mk(apq.x * rm, apq.y * rm);
            rot = 1;
            big |= !(m2 <= stop2 * dd);
          }
        }
        js.P[i] = P; js.Q[i] = Q; js.c[i] = c; js.s[i] = s; js.e[i] = e;
      }
      swept |= __syncthreads_or(rot);
      const int na = h * h, nitem = na + np * h;
      for (int it = tid; it < nitem; it += blockDim.x) {
        if (it < na) {
          const int i = it % h, i2 = it / h;
          const double c = js.c[i], s = js.s[i], c2 = js.c[i2], s2 = js.s[i2];
          if (s == 0.0 && s2 == 0.0) continue;
          const int P = js.P[i], Q = js.Q[i], P2 = js.P[i2], Q2 = js.Q[i2];
          const cplx e = js.e[i], e2 = js.e[i2];
          cplx m00 = A[P + P2 * ld], m01 = A[P + Q2 * ld], m10 = A[Q + P2 * ld], m11 = A[Q + Q2 * ld];
          // L = U_i^H M
          cplx se = s * e, sec = s * conjg(e);
          cplx l00 = c * m00 - cmul(se, m10), l01 = c * m01 - cmul(se, m11);
          cplx l10 = cmul(sec, m00) + c * m10, l11 = cmul(sec, m01) + c * m11;
          // R = L U_i2
          cplx se2 = s2 * e2, sec2 = s2 * conjg(e2);
          A[P + P2 * ld] = c2 * l00 - cmul(sec2, l01);
          A[P + Q2 * ld] = cmul(se2, l00) + c2 * l01;
          A[Q + P2 * ld] = c2 * l10 - cmul(sec2, l11);
          A[Q + Q2 * ld] = cmul(se2, l10) + c2 * l11;
        } else {
          const int iv = it - na, j = iv % np, i = iv / np;
          const double s = js.s[i];
          if (s == 0.0) continue;
          const double c = js.c[i];
          const int P = js.P[i], Q = js.Q[i];
          const cplx e = js.e[i];
          cplx a = V[j + P * ld], b = V[j + Q * ld];
          V[j + P * ld] = c * a - cmul(s * conjg(e), b);
          V[j + Q * ld] = cmul(s * e, a) + c * b;
        }
      }
      __syncthreads();
    }
    if (!swept) break;
    if (PC_RR_EARLY && !__syncthreads_or(big)) {
      sweep++;
      break;
    }
  }
  return sweep;
}

// Triangular solves with many right-hand sides, one warp per column c (lanes own rows lane + 32 q),
// column-sweep order without barriers: y_i = b_i / t_ii (dinv[i] = 1 / t_ii), broadcast from the owner
// lane, then b_m -= t_mi y_i for the rows still to solve.  T lower (forward, i = 0..p-1) or upper
// (backward, i = p-1..0), column-major in shared memory (ld), so a step reads T's column i: consecutive
// rows over the lanes.  B column c comes from bfun(m, c); yfun(i, c, y) stores y_i (owner lane).
constexpr int RR_RPL = (RR_MAXN + 31) / 32;
template <bool UPPER, class BF, class YF>
DEV void tri_solve_cols(const cplx* T, int ld, const double* dinv, int p, int ncol, BF bfun, YF yfun) {
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = threadIdx.x >> 5; c < ncol; c += nw) {
    cplx b[RR_RPL];
#pragma unroll
    for (int q = 0; q < RR_RPL; q++) {
      const int m = lane + 32 * q;
      b[q] = (m < p) ? bfun(m, c) : mk(0.0, 0.0);
    }
    for (int st = 0; st < p; st++) {
      const int i = UPPER ? p - 1 - st : st;
      const int qi = i >> 5, li = i & 31;
      cplx bi = b[0];
#pragma unroll
      for (int q = 1; q < RR_RPL; q++)
        if (qi == q) bi = b[q];
      cplx y = dinv[i] * bi;
      y.x = __shfl_sync(0xffffffffu, y.x, li);
      y.y = __shfl_sync(0xffffffffu, y.y, li);
      if (lane == li) yfun(i, c, y);
#pragma unroll
      for (int q = 0; q < RR_RPL; q++) {
        const int m = lane + 32 * q;
        if (UPPER ? (m < i) : (m > i && m < p)) b[q] = b[q] - cmul(T[m + i * ld], y);
      }
    }
  }
}

// rank[i] = position of w[i] in ascending order (ties by index); valid for i < n
DEV void rank_sort(const double* w, int n, int* order) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int r = 0;
    double wi = w[i];
    for (int j = 0; j < n; j++) r += (w[j] < wi) || (w[j] == wi && j < i);
    order[r] = i;
  }
}

// In-place Cholesky of the Hermitian n x n matrix in A (column-major, ld): lower triangle <- L with
// A = L L^H.  Returns false (uniformly across the CTA) when a pivot is <= tau.
DEV bool cholesky_smem(cplx* A, int n, int ld, double tau, int* flag) {
  const int tid = threadIdx.x;
  if (tid == 0) *flag = 1;
  __syncthreads();
  for (int j = 0; j < n; j++) {
    const double piv = A[j + j * ld].x;
    if (!(piv > tau)) {  // every thread sees the same pivot
      if (tid == 0) *flag = 0;
      __syncthreads();
      return false;
    }
    const double d = sqrt(piv);
    const double inv = 1.0 / d;
    for (int i = j + 1 + tid; i < n; i += blockDim.x) A[i + j * ld] = inv * A[i + j * ld];
    __syncthreads();
    if (tid == 0) A[j + j * ld] = mk(d, 0.0);
    // trailing update of the lower triangle: A[i][k] -= L[i][j] conj(L[k][j]), j < k <= i
    const int m = n - j - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e % m, k = j + 1 + e / m;
      if (k <= i) A[i + k * ld] = A[i + k * ld] - cmul(A[i + j * ld], conjg(A[k + j * ld]));
    }
    __syncthreads();
  }
  return true;
}

__global__ void __launch_bounds__(RR_THREADS) rr_kernel(const cplx* __restrict__ G, int p, int nb, double drop_tol,
                                                        cplx* Cout, double* lam, int* info, cplx* scratch,
                                                        double jtol) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const int np = (p + 1) & ~1, ld = np;
  cplx* A = reinterpret_cast<cplx*>(rsm);
  cplx* V = A + np * np;
  __shared__ JacSm js;
  __shared__ double dsc[RR_MAXN], sig[RR_MAXN], dinv[RR_MAXN];
  __shared__ int keep[RR_MAXN], order[RR_MAXN];
  __shared__ int rank_sh, chol_flag;
  const int tid = threadIdx.x;
#ifdef PC_RR_TIMING
  long long t_[8];
  int nt_ = 0;
#define RR_STAMP() do { if (tid == 0) t_[nt_] = clock64(); nt_++; } while (0)
#else
#define RR_STAMP() do { } while (0)
#endif
  RR_STAMP();
  const cplx* GM = G;
  const cplx* GA = G + (size_t)p * p;
  cplx* T = scratch;                                   // p x RR_MAXN
  cplx* U = scratch + (size_t)p * RR_MAXN;             // p x RR_MAXN
  cplx* Lg = scratch + (size_t)2 * p * RR_MAXN;        // p x p (Cholesky factor copy)

  // 1. scaling D = diag(G_M)^{-1/2}
  for (int i = tid; i < p; i += blockDim.x) {
    double d = GM[i + (size_t)i * p].x;
    dsc[i] = d > 0.0 ? 1.0 / sqrt(d) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < np * np; e += blockDim.x) {
    int i = e % np, j = e / np;
    cplx v = mk(0, 0);
    if (i < p && j < p) v = (dsc[i] * dsc[j]) * GM[i + (size_t)j * p];
    if (i == j && i < p) v.y = 0.0;
    A[e] = v;
  }
  __syncthreads();

  // 2a. fast path: Cholesky D G_M D = L L^H (pivots above drop_tol), H = L^{-1} D G_A D L^{-H}
  RR_STAMP();
  const bool chol = cholesky_smem(A, p, ld, drop_tol, &chol_flag);
  RR_STAMP();
  int r = p;
  int rp = np;
  if (chol) {
    // H = L^{-1} (D G_A D) L^{-H}: Z = L^{-1} (D G_A D) into V, then H^H = L^{-1} Z^H into T (global
    // scratch, p x p; H Hermitian, so T = H^H is symmetrised below like H)
    for (int i = tid; i < p; i += blockDim.x) dinv[i] = 1.0 / A[i + i * ld].x;
    __syncthreads();
    tri_solve_cols<false>(A, ld, dinv, p, p, [&](int m, int cc) { return (dsc[m] * dsc[cc]) * GA[m + (size_t)cc * p]; },
                          [&](int m, int cc, cplx v) { V[m + cc * ld] = v; });
    __syncthreads();
    tri_solve_cols<false>(A, ld, dinv, p, p, [&](int m, int cc) { return conjg(V[cc + m * ld]); },
                          [&](int m, int cc, cplx v) { T[m + (size_t)cc * p] = v; });
    __syncthreads();
    // keep L (global), A <- Hermitian part of H, V <- I
    for (int e = tid; e < p * p; e += blockDim.x) {
      int i = e % p, j = e / p;
      Lg[e] = (i >= j) ? A[i + j * ld] : mk(0, 0);
    }
    __syncthreads();
    for (int e = tid; e < np * np; e += blockDim.x) {
      int i = e % np, j = e / np;
      cplx v = mk(0, 0);
      if (i < p && j < p) {
        cplx a = T[i + (size_t)j * p], b = T[j + (size_t)i * p];
        v = mk(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
      }
      A[i + j * ld] = v;
    }
    __syncthreads();
    for (int e = tid; e < np * np; e += blockDim.x) {
      int i = e % np, j = e / np;
      V[i + j * ld] = mk(i == j ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
  } else {
    // 2b. robust path (rank deficient basis): Jacobi on D G_M D, drop sigma < drop_tol sigma_max
    for (int e = tid; e < np * np; e += blockDim.x) {
      int i = e % np, j = e / np;
      cplx v = mk(0, 0);
      if (i < p && j < p) v = (dsc[i] * dsc[j]) * GM[i + (size_t)j * p];
      if (i == j && i < p) v.y = 0.0;
      A[e] = v;
      V[e] = mk(i == j ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    jacobi_smem(A, V, p, np, ld, js, 40);
    for (int i = tid; i < p; i += blockDim.x) sig[i] = A[i + i * ld].x;
    __syncthreads();
    if (tid == 0) {
      double smax = 0.0;
      for (int i = 0; i < p; i++) smax = fmax(smax, sig[i]);
      int rr = 0;
      for (int i = 0; i < p; i++)
        if (sig[i] > drop_tol * smax) keep[rr++] = i;
      rank_sh = rr;
    }
    __syncthreads();
    r = rank_sh;
    // T = D V_r Sigma_r^{-1/2}
    for (int e = tid; e < p * r; e += blockDim.x) {
      int i = e % p, t = e / p;
      int kk = keep[t];
      T[i + (size_t)t * p] = (dsc[i] / sqrt(sig[kk])) * V[i + kk * ld];
    }
    __syncthreads();
    for (int e = tid; e < p * r; e += blockDim.x) {
      int i = e % p, t = e / p;
      cplx acc = mk(0, 0);
      for (int j = 0; j < p; j++) acc = cfma(GA[i + (size_t)j * p], T[j + (size_t)t * p], acc);
      U[i + (size_t)t * p] = acc;
    }
    __syncthreads();
    rp = (r + 1) & ~1;
    for (int e = tid; e < rp * rp; e += blockDim.x) {
      int i = e % rp, j = e / rp;
      cplx v = mk(0, 0);
      if (i < r && j < r)
        for (int k = 0; k < p; k++) v = v + cmulc(T[k + (size_t)i * p], U[k + (size_t)j * p]);
      A[i + j * rp] = v;
      V[i + j * rp] = mk(i == j ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    for (int e = tid; e < r * r; e += blockDim.x) {
      int i = e % r, j = e / r;
      if (i < j) {
        cplx a = A[i + j * rp], b = A[j + i * rp];
        cplx m = mk(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
        A[i + j * rp] = m;
        A[j + i * rp] = conjg(m);
      } else if (i == j) {
        A[i + i * rp].y = 0.0;
      }
    }
    __syncthreads();
  }
  // 3. eig of H (r x r, ld rp)
  RR_STAMP();
  int sw = jacobi_smem(A, V, r, rp, rp, js, 40, jtol);
  RR_STAMP();
  for (int i = tid; i < r; i += blockDim.x) sig[i] = A[i + i * rp].x;
  __syncthreads();
  rank_sort(sig, r, order);
  __syncthreads();
  const int nout = min(nb, r);
  if (chol) {
    // C = D L^{-H} Q_sel: L^H (upper) into A (eigenvalues are in sig), then backward substitution
    // L^H Y = Q_sel, written scaled by D straight to C
    for (int e = tid; e < p * p; e += blockDim.x) {
      int i = e % p, j = e / p;
      A[i + j * ld] = conjg(Lg[j + (size_t)i * p]);
    }
    for (int i = tid; i < p; i += blockDim.x) dinv[i] = 1.0 / Lg[i + (size_t)i * p].x;
    __syncthreads();
    tri_solve_cols<true>(A, ld, dinv, p, nout, [&](int m, int t) { return V[m + order[t] * rp]; },
                         [&](int m, int t, cplx v) { Cout[m + (size_t)t * p] = dsc[m] * v; });
  } else {
    for (int e = tid; e < p * nout; e += blockDim.x) {
      int i = e % p, t = e / p;
      int kk = order[t];
      cplx acc = mk(0, 0);
      for (int j = 0; j < r; j++) acc = cfma(T[i + (size_t)j * p], V[j + kk * rp], acc);
      Cout[i + (size_t)t * p] = acc;
    }
  }
  for (int t = tid; t < nout; t += blockDim.x) lam[t] = sig[order[t]];
  RR_STAMP();
  if (tid == 0) {
    info[0] = r;
    info[1] = sw;
    info[2] = chol ? 1 : 0;
    for (int i = 3; i < 8; i++) info[i] = 0;
#ifdef PC_RR_TIMING  // per-phase clock64 cycles: scaling, Cholesky, H formation, Jacobi, back substitution
    for (int i = 1; i < nt_ && i < 6; i++) info[3 + i - 1] = (int)(t_[i] - t_[i - 1]);
#endif
  }
}

// Rotation threshold of the Rayleigh-Ritz Jacobi: |a_pq| <= tol sqrt(|a_pp a_qq|) counts as zero (the
// eigenvalues it leaves out are O(tol^2) relative; eigenvectors O(tol)).  Process-wide tuning knob.
static double g_jacobi_tol = 1e-16;
void set_jacobi_tol(double t) { g_jacobi_tol = (t > 0.0 && t < 1e-6) ? t : 1e-16; }

void launch_rr(const cplx* G, int p, int nb, double drop_tol, cplx* C, double* lambda, int* info, cplx* scratch,
               cudaStream_t st) {
  const int np = (p + 1) & ~1;
  size_t smem = (size_t)2 * np * np * sizeof(cplx);
  smem_attr((const void*)rr_kernel, (int)(2 * RR_MAXN * RR_MAXN * sizeof(cplx)));
  rr_kernel<<<1, RR_THREADS, smem, st>>>(G, p, nb, drop_tol, C, lambda, info, scratch, g_jacobi_tol);
}

// Standalone Hermitian eigensolver (tests): w ascending, V columns in the same order.
__global__ void __launch_bounds__(RR_THREADS) heevj_kernel(const cplx* __restrict__ Ain, int n, double* w, cplx* Vout,
                                                           int* info) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const int np = (n + 1) & ~1, ld = np;
  cplx* A = reinterpret_cast<cplx*>(rsm);
  cplx* V = A + np * np;
  __shared__ JacSm js;
  __shared__ double sig[RR_MAXN];
  __shared__ int order[RR_MAXN];
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    int i = e % np, j = e / np;
    A[e] = (i < n && j < n) ? Ain[i + (size_t)j * n] : mk(0, 0);
    V[e] = mk(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  int sw = jacobi_smem(A, V, n, np, ld, js, 60);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sig[i] = A[i + i * ld].x;
  __syncthreads();
  rank_sort(sig, n, order);
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e % n, t = e / n;
    Vout[i + (size_t)t * n] = V[i + order[t] * ld];
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) w[t] = sig[order[t]];
  if (threadIdx.x == 0) info[0] = sw;
}

void launch_heevj(const cplx* A, int n, double* w, cplx* V, int* info, cudaStream_t st) {
  const int np = (n + 1) & ~1;
  size_t smem = (size_t)2 * np * np * sizeof(cplx);
  smem_attr((const void*)heevj_kernel, (int)(2 * RR_MAXN * RR_MAXN * sizeof(cplx)));
  heevj_kernel<<<1, RR_THREADS, smem, st>>>(A, n, w, V, info);
}
