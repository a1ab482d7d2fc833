// LOBPCG block update fused with the residual, the preconditioner and the NEXT iteration's Gram blocks
// (PAPER.md:1055-1064 LOBPCG, 530-548 K_P^{-1}).  For the Ritz coefficients C (p x b, S = [X W P]):
//   P'  = [W P] C_WP,    X'  = X C_X + P'                       (S phase)
//   AP' = [AW AP] C_WP,  AX' = AX C_X + AP'                     (AS phase)
//   R   = AX' - X' diag(lambda'),  W' = K_P^{-1} R              (residual phase; mode 0 zeroed at k = 0)
//   G1 += [X' W' P']^H [W' P' AP'],   G2 += (AX')^H W'          (Gram phase, this row tile)
// Everything the next Rayleigh-Ritz step needs except W'^H A W' (A W' does not exist before the next
// apply) follows from G1, G2 and X'^H X' = I, X'^H A X' = Lambda' (A Hermitian: X'^H A W' = (A X')^H W',
// P'^H A W' = (A P')^H W').  The Gram products ride on the update's row tiles while they are in shared
// memory, so the next iteration's Gram kernel does not re-read [X W P AX AW AP] from HBM: the update
// is HBM-bound and the Gram DMMA-bound, and the fused pass keeps both pipes busy.
//
// Row tile = UG_SEG consecutive Fourier modes x 3 components (24 rows), 6 warps: in the update phases
// warp w owns component w % 3 and output n-tile w / 3 (b <= 16 output columns); in the Gram phase the
// 8x8 output tiles of G1 and G2 are dealt to the warps in contiguous blocks.  Complex products use
// three real DMMAs per complex MAC (see gram.cu).  Partial Gram tiles and norm partials are written
// per CTA and reduced in a fixed order (deterministic).
#include "kernels.h"
#include "dmma.cuh"
#include "kp.cuh"

constexpr int UG_SEG = 8;           // modes per row tile
constexpr int UG_RP = 26;           // S/AS tile pitch in complex (24 rows + 2; 2 mod 8: conflict-free A fragments)
constexpr int UG_GP = 28;           // staging pitch (24 rows + 4; 4 mod 8: conflict-free Gram fragments)
constexpr int UG_WARPS = 6;
constexpr int UG_THREADS = 32 * UG_WARPS;
constexpr int UG_TPW = 4;           // Gram tiles per warp (max): 24 tiles covers b = 15, nw = 10

HD int ug_pitch4mod8(int p) {
  int x = p;
  while ((x & 7) != 4) x++;
  return x;
}

struct UgShape {
  int b, nw;            // X' columns (b <= 16), W'/P' columns (nw <= b)
  int xs, cax;          // staging: X' region padded to even width xs; AX' region start (even)
  int mt1, nt1, t1;     // G1 tiles: (b + 2 nw) x 3 nw
  int mt2, nt2, t;      // G2 tiles: b x nw; t = all tiles
};

UgShape ug_shape(int b, int nw) {
  UgShape s;
  s.b = b;
  s.nw = nw;
  s.xs = (b + 1) & ~1;
  s.cax = (s.xs + 3 * nw + 1) & ~1;
  s.mt1 = (s.xs + 2 * nw + 7) / 8;
  s.nt1 = (3 * nw + 7) / 8;
  s.t1 = s.mt1 * s.nt1;
  s.mt2 = (b + 7) / 8;
  s.nt2 = (nw + 7) / 8;
  s.t = s.t1 + s.mt2 * s.nt2;
  return s;
}

__global__ void __launch_bounds__(UG_THREADS, 2) update_gram_kernel(
    ColPtrs S, ColPtrs AS, int p, const cplx* __restrict__ C, int ldc, int split, UgShape sh, MutColPtrs Xo,
    MutColPtrs Po, MutColPtrs AXo, MutColPtrs APo, MutColPtrs Wo, const double* __restrict__ lam, int n,
    const cplx* __restrict__ kt, double gamma, double thr, int deflate0, double* __restrict__ npart,
    cplx* __restrict__ gpart) {
  extern __shared__ __align__(16) double ugsm[];
  const int b = sh.b, nw = sh.nw;
  const int n3 = n * n * n;
  const int pe = (p + 3) & ~3;
  const int PS = ug_pitch4mod8(pe);
  cplx* Buf = reinterpret_cast<cplx*>(ugsm);   // [2][pe][UG_RP]: 0 = S tile, 1 = AS tile
  cplx* Cs = Buf + 2 * pe * UG_RP;             // [16][PS]
  cplx* Gs = Cs + 16 * PS;                     // [cax + b][UG_GP]: X' | pad | W' | P' | AP' | pad | AX'
  const int cW = sh.xs, cP = cW + nw, cAP = cW + 2 * nw, cAX = sh.cax;
  // staging element (column col, row r) lives at col * UG_GP + (r ^ (col & 6)): the XOR keeps aligned
  // 4-row groups together (Gram fragments: rows 4k..4k+3 of columns 2j, 2j+1 conflict-free) and spreads
  // the update fragments' stores (columns c, c+2, c+4, c+6 of one row) over distinct banks
  auto GI = [](int col, int r) { return col * UG_GP + (r ^ (col & 6)); };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int e = tid; e < 16 * pe; e += UG_THREADS) {
    const int c = e / pe, m = e % pe;
    Cs[c * PS + m] = (c < b && m < p) ? C[(size_t)c * ldc + m] : mk(0, 0);
  }
  // padding columns of the staging area stay zero (they enter the Gram tiles as zero rows/columns)
  for (int e = tid; e < 3 * UG_SEG * ((cW - b) + (cAX - cAP - nw)); e += UG_THREADS) {
    const int k = e / (3 * UG_SEG), r = e % (3 * UG_SEG);
    const int col = (k < cW - b) ? b + k : cAP + nw + (k - (cW - b));
    Gs[GI(col, r)] = mk(0, 0);
  }
  const long long ntiles = (n3 + UG_SEG - 1) / UG_SEG;
  const cplx* dummy = S.p[0];
  auto load_tile = [&](int buf, const ColPtrs& src, long long t) {
    const long long m0 = t * UG_SEG;
    cplx* dst = Buf + buf * pe * UG_RP;
    for (int e = tid; e < 3 * UG_SEG * pe; e += UG_THREADS) {
      const int m = e / (3 * UG_SEG), rho = e % (3 * UG_SEG);
      const int seg = rho / UG_SEG, rr = rho % UG_SEG;
      const long long mode = m0 + rr;
      const bool ok = (m < p) && (mode < n3);
      cp_async16_zfill(&dst[m * UG_RP + rho],
                       ok ? (const void*)(src.p[m] + (long long)seg * n3 + mode) : (const void*)dummy, ok);
    }
    cp_async_commit();
  };

  // ---- update-phase ownership: component us, output n-tile unt; fragment rows = modes lane >> 2
  const int us = warp % 3, unt = warp / 3;
  const int umode = lane >> 2;
  double u1[2], u2[2], u3[2];
  auto kloop = [&](const cplx* Sc, int mlo, int mhi) {
#pragma unroll 3
    for (int m4 = mlo & ~3; m4 < mhi; m4 += 4) {
      const int mm = m4 + (lane & 3);
      const bool in = (mm >= mlo) && (mm < mhi);
      const cplx a = Sc[mm * UG_RP + us * UG_SEG + umode];
      cplx cv = Cs[(unt * 8 + (lane >> 2)) * PS + mm];
      if (!in) cv = mk(0, 0);
      dmma(u1[0], u1[1], a.x, cv.x);
      dmma(u2[0], u2[1], a.y, cv.y);
      dmma(u3[0], u3[1], a.x + a.y, cv.x + cv.y);
    }
  };
  auto uval = [&](int e) { return mk(u1[e] - u2[e], u3[e] - u1[e] - u2[e]); };
  // store the fragment's two columns c = unt*8 + 2 (lane & 3) + e to global (if Y.p[c]) and staging
  auto ustore = [&](const MutColPtrs& Y, int ncol, int gcol0, long long m0) {
    const long long mode = m0 + umode;
    const bool ok = mode < n3;
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const int c = unt * 8 + 2 * (lane & 3) + e;
      if (c < ncol) {
        const cplx v = ok ? uval(e) : mk(0, 0);
        if (ok && Y.p[c]) Y.p[c][(long long)us * n3 + mode] = v;
        Gs[GI(gcol0 + c, us * UG_SEG + umode)] = v;
      }
    }
  };

  // ---- residual-phase ownership: column rc, mode rm (8 consecutive threads share a column)
  const int rc = tid / UG_SEG, rm = tid % UG_SEG;
  const bool rown = rc < b;
  double nr = 0.0, nx = 0.0;

  // ---- Gram-phase ownership: contiguous block of tiles
  const int tpw = (sh.t + UG_WARPS - 1) / UG_WARPS;
  double g1[UG_TPW][2], g2[UG_TPW][2], g3[UG_TPW][2];
#pragma unroll
  for (int q = 0; q < UG_TPW; q++) g1[q][0] = g1[q][1] = g2[q][0] = g2[q][1] = g3[q][0] = g3[q][1] = 0.0;

  long long t = blockIdx.x;
  if (t < ntiles) {
    load_tile(0, S, t);
    load_tile(1, AS, t);
  }
  for (; t < ntiles; t += gridDim.x) {
    const long long m0 = t * UG_SEG;
    const bool more = t + gridDim.x < ntiles;
    // ---- S phase: P' then X' (same accumulators)
    cp_async_wait<1>();
    __syncthreads();
    u1[0] = u1[1] = u2[0] = u2[1] = u3[0] = u3[1] = 0.0;
    kloop(Buf, split, p);
    ustore(Po, nw, cP, m0);
    kloop(Buf, 0, split);
    ustore(Xo, b, 0, m0);
    __syncthreads();  // buffer 0 free
    if (more) load_tile(0, S, t + gridDim.x);
    // ---- AS phase: AP' then AX'
    if (more) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const cplx* Ab = Buf + pe * UG_RP;
    u1[0] = u1[1] = u2[0] = u2[1] = u3[0] = u3[1] = 0.0;
    kloop(Ab, split, p);
    ustore(APo, nw, cAP, m0);
    kloop(Ab, 0, split);
    ustore(AXo, b, cAX, m0);
    __syncthreads();  // buffer 1 free; X', P', AP', AX' staged
    if (more) load_tile(1, AS, t + gridDim.x);
    // ---- residual, preconditioner, norms
    if (rown) {
      const long long mode = m0 + rm;
      const bool ok = mode < n3;
      const double l = lam[rc];
      cplx rv[3];
#pragma unroll
      for (int s = 0; s < 3; s++) {
        const cplx x = Gs[GI(rc, s * UG_SEG + rm)];
        const cplx ax = Gs[GI(cAX + rc, s * UG_SEG + rm)];
        rv[s] = mk(ax.x - l * x.x, ax.y - l * x.y);
        nr += abs2(rv[s]);
        nx += abs2(x);
      }
      if (rc < nw) {
        if (ok) {
          const int mi = (int)mode;
          const int m1 = mi % n, m2 = (mi / n) % n, m3 = mi / (n * n);
          cplx k1, k2, k3;
          kappa_at(kt, n, m1, m2, m3, k1, k2, k3);
          kp_inv(k1, k2, k3, gamma, thr, rv[0], rv[1], rv[2]);
          if (deflate0 && mi == 0) rv[0] = rv[1] = rv[2] = mk(0, 0);
          cplx* w = Wo.p[rc];
#pragma unroll
          for (int s = 0; s < 3; s++) w[(long long)s * n3 + mi] = rv[s];
        } else {
          rv[0] = rv[1] = rv[2] = mk(0, 0);
        }
#pragma unroll
        for (int s = 0; s < 3; s++) Gs[GI(cW + rc, s * UG_SEG + rm)] = rv[s];
      }
    }
    __syncthreads();  // W' staged
    // ---- Gram phase: 6 k-steps of 4 rows; staging columns of this warp's tiles precomputed
    {
      int am[UG_TPW], bn[UG_TPW];
#pragma unroll
      for (int q = 0; q < UG_TPW; q++) {
        const int tt = warp * tpw + q;
        am[q] = bn[q] = -1;
        if (q < tpw && tt < sh.t) {
          int ca, cb, na_, nb_;
          if (tt < sh.t1) {
            const int mt = tt / sh.nt1, nt = tt % sh.nt1;
            ca = mt * 8; na_ = cW + 2 * nw;       // S' = X' pad W' P' from staging column 0
            cb = cW + nt * 8; nb_ = cW + 3 * nw;  // T' = W' P' AP'
          } else {
            const int t2 = tt - sh.t1, mt = t2 / sh.nt2, nt = t2 % sh.nt2;
            ca = cAX + mt * 8; na_ = cAX + b;     // AX'
            cb = cW + nt * 8; nb_ = cW + nw;      // W'
          }
          const int a_ = ca + (lane >> 2), b_ = cb + (lane >> 2);
          am[q] = (a_ < na_) ? a_ : -1;
          bn[q] = (b_ < nb_) ? b_ : -1;
        }
      }
#pragma unroll 1
      for (int k4 = 0; k4 < 3 * UG_SEG; k4 += 4) {
        const int row = k4 + (lane & 3);
#pragma unroll
        for (int q = 0; q < UG_TPW; q++) {
          if (q >= tpw) break;  // warp-uniform
          const cplx av = (am[q] >= 0) ? Gs[GI(am[q], row)] : mk(0, 0);
          const cplx bv = (bn[q] >= 0) ? Gs[GI(bn[q], row)] : mk(0, 0);
          dmma(g1[q][0], g1[q][1], av.x, bv.x);
          dmma(g2[q][0], g2[q][1], av.y, bv.y);
          dmma(g3[q][0], g3[q][1], av.x - av.y, bv.x + bv.y);
        }
      }
    }
  }
  cp_async_wait<0>();

  // ---- per-CTA Gram tiles: conj(S)^T T = (P1 + P2) + i (P3 - P1 + P2), entry (m, n) of tile tt
#pragma unroll
  for (int q = 0; q < UG_TPW; q++) {
    const int tt = warp * tpw + q;
    if (q >= tpw || tt >= sh.t) break;
    cplx* o = gpart + ((size_t)blockIdx.x * sh.t + tt) * 64;
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const int m = lane >> 2, nn = 2 * (lane & 3) + e;
      o[m * 8 + nn] = mk(g1[q][e] + g2[q][e], g3[q][e] - g1[q][e] + g2[q][e]);
    }
  }
  // ---- norms: the 8 threads of a column, fixed xor order
#pragma unroll
  for (int off = 1; off < UG_SEG; off <<= 1) {
    nr += __shfl_xor_sync(0xffffffffu, nr, off);
    nx += __shfl_xor_sync(0xffffffffu, nx, off);
  }
  if (rown && rm == 0) {
    npart[((long long)rc * gridDim.x + blockIdx.x) * 2 + 0] = nr;
    npart[((long long)rc * gridDim.x + blockIdx.x) * 2 + 1] = nx;
  }
}

// Fixed-order sum of the per-CTA Gram tiles: red[tt * 64 + e] = sum_cta gpart[(cta * t + tt) * 64 + e].
__global__ void ug_reduce_kernel(const cplx* __restrict__ gpart, int grid, int t, cplx* __restrict__ red) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= t * 64) return;
  cplx acc = mk(0, 0);
  for (int g = 0; g < grid; g++) acc = acc + gpart[(size_t)g * t * 64 + idx];
  red[idx] = acc;
}

bool update_gram_supported(int p, int b, int nw) {
  if (b > 16 || nw > b || nw < 1 || p > 80) return false;
  const UgShape sh = ug_shape(b, nw);
  return sh.t <= UG_WARPS * UG_TPW;
}

size_t update_gram_partial_bytes(int b, int nw) {
  return (size_t)148 * 4 * ug_shape(b, nw).t * 64 * sizeof(cplx);
}

int launch_update_gram(const ColPtrs& S, const ColPtrs& AS, int p, const cplx* C, int ldc, int b, int nw,
                       const MutColPtrs& Xo, const MutColPtrs& Po, const MutColPtrs& AXo, const MutColPtrs& APo,
                       const MutColPtrs& Wo, const double* lam, int n, const cplx* kt, double gamma, double thr,
                       int deflate0, double* npart, cplx* gpart, cplx* gred, int max_grid, cudaStream_t st) {
  const UgShape sh = ug_shape(b, nw);
  const int pe = (p + 3) & ~3;
  const size_t smem = (size_t)(2 * pe * UG_RP + 16 * ug_pitch4mod8(pe) + (sh.cax + b) * UG_GP) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(update_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, update_gram_kernel, UG_THREADS, smem);
  occ = std::max(1, std::min(occ, 4));
  const long long n3 = (long long)n * n * n;
  const long long ntiles = (n3 + UG_SEG - 1) / UG_SEG;
  const int grid = (int)std::min<long long>(std::min<long long>(ntiles, 148LL * occ), max_grid);
  update_gram_kernel<<<grid, UG_THREADS, smem, st>>>(S, AS, p, C, ldc, b, sh, Xo, Po, AXo, APo, Wo, lam, n, kt,
                                                    gamma, thr, deflate0, npart, gpart);
  ug_reduce_kernel<<<(sh.t * 64 + 255) / 256, 256, 0, st>>>(gpart, grid, sh.t, gred);
  return grid;
}

// Assemble [G_M | G_A] (p x 2p, column-major, ld p) for S = [X W_a P_a] (a = active subset of the nw
// W'/P' columns, P omitted when !haveP) from the fused Gram tiles red (G1, G2), Gww = W_a^H A W_a (na x na,
// ld na) and X^H X = I, X^H A X = diag(lam).
__global__ void ug_assemble_kernel(const cplx* __restrict__ red, UgShape sh, const int* __restrict__ act, int na,
                                   int haveP, const cplx* __restrict__ Gww, const double* __restrict__ lam,
                                   int p, cplx* __restrict__ G) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p * p) return;
  const int i = idx % p, j = idx / p;  // row i, column j
  const int b = sh.b, nw = sh.nw;
  // S index -> (kind 0 X / 1 W / 2 P, original column)
  auto kind_of = [&](int s, int& col) {
    if (s < b) { col = s; return 0; }
    if (s < b + na) { col = act[s - b]; return 1; }
    col = act[s - b - na];
    return 2;
  };
  auto g1 = [&](int r, int c) {  // G1 row r in [X' W' P'], column c in [W' P' AP']
    const int mt = r / 8, nt = c / 8;
    return red[((size_t)(mt * sh.nt1 + nt)) * 64 + (r % 8) * 8 + (c % 8)];
  };
  auto g2 = [&](int r, int c) {  // G2 row r in AX', column c in W'
    const int mt = r / 8, nt = c / 8;
    return red[((size_t)(sh.t1 + mt * sh.nt2 + nt)) * 64 + (r % 8) * 8 + (c % 8)];
  };
  int ci, cj;
  const int ki = kind_of(i, ci), kj = kind_of(j, cj);
  (void)haveP;
  // G_M(i, j) = s_i^H s_j
  cplx gm, ga;
  // index of a W'/P' column in G1's row space ([X' W' P']) and column space ([W' P' AP'])
  auto rowS = [&](int k, int c) { return k == 0 ? c : (k == 1 ? sh.xs + c : sh.xs + nw + c); };
  auto colT = [&](int k, int c) { return k == 1 ? c : nw + c; };  // k = 1 (W') or 2 (P')
  if (ki == 0 && kj == 0) {
    gm = mk(ci == cj ? 1.0 : 0.0, 0.0);
    ga = mk(ci == cj ? lam[ci] : 0.0, 0.0);
  } else if (kj != 0) {
    // column j is W or P: G1 has it in its column space
    gm = g1(rowS(ki, ci), colT(kj, cj));
    if (kj == 2) {
      ga = g1(rowS(ki, ci), 2 * nw + cj);                 // s_i^H A P'_c  (column AP')
    } else if (ki == 0) {
      ga = g2(ci, cj);                                     // X^H A W = (AX)^H W
    } else if (ki == 1) {
      ga = Gww[(size_t)(j - b) * na + (i - b)];            // W^H A W (small Gram, ld na)
    } else {
      ga = conjg(g1(rowS(1, cj), 2 * nw + ci));            // P^H A W = conj(W^H A P)^T
    }
  } else {
    // column j is X, row i is W or P: Hermitian mirror of (j, i)
    gm = conjg(g1(rowS(0, cj), colT(ki, ci)));
    ga = (ki == 1) ? conjg(g2(cj, ci)) : conjg(g1(rowS(0, cj), 2 * nw + ci));
  }
  G[(size_t)j * p + i] = gm;
  G[(size_t)p * p + (size_t)j * p + i] = ga;
}

void launch_ug_assemble(const cplx* red, int b, int nw, const int* act, int na, int haveP, const cplx* Gww,
                        const double* lam, int p, cplx* G, cudaStream_t st) {
  const UgShape sh = ug_shape(b, nw);
  ug_assemble_kernel<<<(p * p + 255) / 256, 256, 0, st>>>(red, sh, act, na, haveP, Gww, lam, p, G);
}
