// Tall-skinny complex FP64 block algebra of LOBPCG on the FP64 tensor pipe (DMMA, mma.sync
// m8n8k4 f64), used for the Rayleigh-Ritz Gram matrices and the block updates
// ("LOBPCG ... with soft locking"; Knyazev 2001).
//
// Complex products are done on the real interleaved view of the columns (a column of len complex
// numbers is 2*len doubles (re, im, re, im, ...)):
//   Gram   G = S^H T:   Re G_mn = sum_k' a[m][k'] b[k'][n],   Im G_mn = sum_k' a[m][k'] b~[k'][n]
//                       a = S view, b = T view, b~[2k] = Im T_k, b~[2k+1] = -Re T_k
//   Update Y = S C:     Re Y = sum_k' a[row][k'] br[k'][c],  Im Y = sum_k' a[row][k'] bi[k'][c]
//                       br[2m] = Re C_mc, br[2m+1] = -Im C_mc, bi[2m] = Im C_mc, bi[2m+1] = Re C_mc
// Reductions over rows are split across CTAs and summed in a fixed order (deterministic).
#include "kernels.h"

#include "dmma.cuh"

// [G_M | G_A] (p x 2p) for S = [X (b) | W (nw) | P (np)] from Gp = S^H [W P AW AP] (p x 2c, c = nw+np),
// using X^H X = I and X^H A X = diag(lambda) (X are the current Ritz vectors) and Hermitian symmetry.
__global__ void gram_assemble_kernel(const cplx* __restrict__ Gp, const double* __restrict__ lam, int b, int c,
                                     cplx* G) {
  const int p = b + c;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 2 * p * p) return;
  const int half = idx / (p * p), e = idx % (p * p);
  const int i = e % p, j = e / p;
  cplx v;
  if (i < b && j < b) {
    v = (i == j) ? mk(half ? lam[i] : 1.0, 0.0) : mk(0, 0);
  } else if (j >= b) {
    // [W P]^H [W P] and [W P]^H A [W P] are Hermitian: their strict lower triangles (not computed by
    // the Gram kernel) are the conjugates of the upper ones
    if (i >= b && i - b > j - b) v = conjg(Gp[(size_t)(half * c + (i - b)) * p + j]);
    else v = Gp[(size_t)(half * c + (j - b)) * p + i];
  } else {  // i >= b, j < b: conj of (j, i)
    v = conjg(Gp[(size_t)(half * c + (i - b)) * p + j]);
  }
  G[(size_t)half * p * p + e] = v;
}

void launch_gram_assemble(const cplx* Gp, const double* lam, int b, int c, cplx* G, cudaStream_t st) {
  const int p = b + c;
  gram_assemble_kernel<<<(2 * p * p + 255) / 256, 256, 0, st>>>(Gp, lam, b, c, G);
}

// ------------------------------------------------------------------------------------------
// Update: phase 1  acc = sum_{m in [split, p)} S[:, m] C[m, :]  -> Y1 (optional)
//         phase 2  acc += sum_{m in [0, split)} S[:, m] C[m, :] -> Y2 (+ Add)
// r <= 8 NT output columns.  CTA = 8 warps x 8 rows = 64-row tiles, persistent over row tiles with a
// 2-stage cp.async pipeline (tile t+1 streams in while tile t is multiplied).  S tile in smem as
// [m][row] (as streamed from HBM, conflict-free cp.async) with row pitch RP = 2 mod 8 complex; C as
// [c][m] with pitch PS = 4 mod 8 (conflict-free 16-B fragment loads).  Complex products with three real
// MMAs per m8n8k4 step of 4 complex m:  P1 = S_r C_r, P2 = S_i C_i, P3 = (S_r + S_i)(C_r + C_i),
// Re = P1 - P2, Im = P3 - P1 - P2.
// ------------------------------------------------------------------------------------------

HD int pitch2mod8(int p) {
  int x = p + 1;
  while ((x & 7) != 2) x++;
  return x;
}
HD int pitch4mod8(int p) {
  int x = p;
  while ((x & 7) != 4) x++;
  return x;
}

template <int NT, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) update_kernel(ColPtrs S, int p, const cplx* __restrict__ C, int ldc,
                                                           int r, int split, MutColPtrs Y1, int has_y1, MutColPtrs Y2,
                                                           ColPtrs Add, int has_add, long long len) {
  extern __shared__ __align__(16) double usm[];
  const int pe = (p + 3) & ~3;  // S columns padded to the k = 4 complex step
  const int PS = pitch4mod8(pe);
  constexpr int U_ROWS = 8 * WARPS, U_THREADS = 32 * WARPS;
  constexpr int RP = U_ROWS + 2;  // 2 mod 8
  cplx* Ss = reinterpret_cast<cplx*>(usm);   // [2][pe][RP]
  cplx* Cs = Ss + 2 * pe * RP;               // [NT*8][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int e = tid; e < NT * 8 * pe; e += U_THREADS) {
    int c = e / pe, m = e % pe;
    Cs[c * PS + m] = (c < r && m < p) ? C[(size_t)c * ldc + m] : mk(0, 0);
  }
  const long long ntiles = (len + U_ROWS - 1) / U_ROWS;
  const cplx* dummy = S.p[0];
  auto load_tile = [&](int stage, long long t) {
    const long long rbase = t * U_ROWS;
    cplx* dst = Ss + stage * pe * RP;
    for (int e = tid; e < U_ROWS * pe; e += U_THREADS) {
      int m = e / U_ROWS, rr = e % U_ROWS;
      long long row = rbase + rr;
      bool ok = (m < p) && (row < len);
      cp_async16_zfill(&dst[m * RP + rr], ok ? (const void*)(S.p[m] + row) : (const void*)dummy, ok);
    }
    cp_async_commit();
  };
  long long t = blockIdx.x;
  if (t < ntiles) load_tile(0, t);
  for (int i = 0; t < ntiles; t += gridDim.x, i++) {
    const int st = i & 1;
    if (t + gridDim.x < ntiles) {
      load_tile(st ^ 1, t + gridDim.x);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const long long rbase = t * U_ROWS;
    double p1[NT][2], p2[NT][2], p3[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; nt++) p1[nt][0] = p1[nt][1] = p2[nt][0] = p2[nt][1] = p3[nt][0] = p3[nt][1] = 0.0;
    const cplx* Sc = Ss + st * pe * RP;
    const int arow = warp * 8 + (lane >> 2);

    auto kloop = [&](int mlo, int mhi) {  // contributions of S columns m in [mlo, mhi)
#pragma unroll 2
      for (int m4 = mlo & ~3; m4 < mhi; m4 += 4) {  // one k4 step = 4 complex m
        const int mm = m4 + (lane & 3);
        const bool in = (mm >= mlo) && (mm < mhi);
        const cplx a = Sc[mm * RP + arow];
        const double as = a.x + a.y;
#pragma unroll
        for (int nt = 0; nt < NT; nt++) {
          cplx cv = Cs[(nt * 8 + (lane >> 2)) * PS + mm];
          if (!in) cv = mk(0, 0);
          dmma(p1[nt][0], p1[nt][1], a.x, cv.x);
          dmma(p2[nt][0], p2[nt][1], a.y, cv.y);
          dmma(p3[nt][0], p3[nt][1], as, cv.x + cv.y);
        }
      }
    };
    auto store = [&](const MutColPtrs& Y, bool add) {
      long long row = rbase + warp * 8 + (lane >> 2);
      if (row >= len) return;
#pragma unroll
      for (int nt = 0; nt < NT; nt++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          int c = nt * 8 + 2 * (lane & 3) + e;
          if (c < r && Y.p[c]) {
            cplx v = mk(p1[nt][e] - p2[nt][e], p3[nt][e] - p1[nt][e] - p2[nt][e]);
            if (add) v = v + Add.p[c][row];
            Y.p[c][row] = v;
          }
        }
    };
    kloop(split, p);
    if (has_y1) store(Y1, false);
    kloop(0, split);
    store(Y2, has_add != 0);
    __syncthreads();  // stage st is refilled by the next iteration's prefetch
  }
}

template <int NT, int WARPS>
static void run_update(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                       const MutColPtrs& Y2, const ColPtrs* add, long long len, cudaStream_t st) {
  constexpr int U_ROWS = 8 * WARPS;
  const int pe = (p + 3) & ~3, ps = pitch4mod8(pe);
  const size_t smem = (size_t)(2 * pe * (U_ROWS + 2) + NT * 8 * ps) * sizeof(cplx);
  smem_attr((const void*)update_kernel<NT, WARPS>, 220 * 1024);
  const long long ntiles = (len + U_ROWS - 1) / U_ROWS;
  const int occ = std::max(1, std::min(64 / WARPS, (int)((227 * 1024) / (smem + 1024))));
  const int grid = (int)std::min<long long>(ntiles, 148LL * occ);
  MutColPtrs y1 = Y1 ? *Y1 : MutColPtrs{};
  ColPtrs ad = add ? *add : ColPtrs{};
  update_kernel<NT, WARPS><<<grid, 32 * WARPS, smem, st>>>(S, p, C, ldc, r, split, y1, Y1 ? 1 : 0, Y2, ad,
                                                           add ? 1 : 0, len);
}

template <int WARPS>
static void launch_update_w(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                            const MutColPtrs& Y2, const ColPtrs* add, long long len, cudaStream_t st) {
  if (r <= 8) run_update<1, WARPS>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
  else if (r <= 16) run_update<2, WARPS>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
  else if (r <= 24) run_update<3, WARPS>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
  else run_update<4, WARPS>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
}

void launch_update(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                   const MutColPtrs& Y2, const ColPtrs* add, long long len, cudaStream_t st) {
  launch_update_w<4>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
}
