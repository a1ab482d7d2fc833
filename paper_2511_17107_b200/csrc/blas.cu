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

DEV void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

DEV void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

// ------------------------------------------------------------------------------------------
// Gram: partial[split][n][m] = sum over the split's rows of conj(S[r][m]) T[r][n]
// CTA output block BM x BN (complex) = (WARPS_M * WM * 8) x (WARPS_N * WN * 8); each warp owns
// WM x WN m8n8 tiles (real and imaginary accumulators).  Rows stream through a 2-stage cp.async
// pipeline in chunks of G_KC complex rows; the split-K partials are reduced in a fixed order.
// ------------------------------------------------------------------------------------------
constexpr int G_KC = 32, G_PITCH = 2 * G_KC + 4;

template <int WM, int WN, int WARPS_M, int WARPS_N>
struct GramCfg {
  static constexpr int BM = WARPS_M * WM * 8, BN = WARPS_N * WN * 8;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr size_t SMEM = 2 * (size_t)(BM + BN) * G_PITCH * sizeof(double);
};

template <int WM, int WN, int WARPS_M, int WARPS_N>
__global__ void __launch_bounds__(GramCfg<WM, WN, WARPS_M, WARPS_N>::THREADS)
gram_kernel(ColPtrs S, int p, ColPtrs T, int q, long long len, long long rows_per_split, int nmb, cplx* partial) {
  using Cfg = GramCfg<WM, WN, WARPS_M, WARPS_N>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, NTH = Cfg::THREADS;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                       // [2][BM][G_PITCH]
  double* Bs = gsm + 2 * BM * G_PITCH;    // [2][BN][G_PITCH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int mb = blockIdx.x % nmb, nb = blockIdx.x / nmb;
  const int m0 = mb * BM, n0 = nb * BN;
  const long long r0 = (long long)blockIdx.y * rows_per_split;
  const long long r1 = min(len, r0 + rows_per_split);

  double accR[WM][WN][2], accI[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; i++)
#pragma unroll
    for (int j = 0; j < WN; j++) accR[i][j][0] = accR[i][j][1] = accI[i][j][0] = accI[i][j][1] = 0.0;

  const cplx* dummy = S.p[0];
  auto load_chunk = [&](int stage, long long rbase) {
    for (int e = tid; e < (BM + BN) * G_KC; e += NTH) {
      int c = e / G_KC, r = e % G_KC;
      long long row = rbase + r;
      bool okr = row < r1;
      double* dst;
      const cplx* src = dummy;
      bool ok;
      if (c < BM) {
        int m = m0 + c;
        ok = okr && m < p;
        if (ok) src = S.p[m] + row;
        dst = As + (stage * BM + c) * G_PITCH + 2 * r;
      } else {
        int n = n0 + (c - BM);
        ok = okr && n < q;
        if (ok) src = T.p[n] + row;
        dst = Bs + (stage * BN + (c - BM)) * G_PITCH + 2 * r;
      }
      cp_async16_zfill(dst, src, ok);
    }
    cp_async_commit();
  };

  // warp tiles entirely outside [0, p) x [0, q) skip their MMAs (warp-uniform)
  const bool live = (m0 + wm * WM * 8 < p) && (n0 + wn * WN * 8 < q);
  const int nchunks = (r1 > r0) ? (int)((r1 - r0 + G_KC - 1) / G_KC) : 0;
  if (nchunks > 0) load_chunk(0, r0);
  for (int ch = 0; ch < nchunks; ch++) {
    const int st = ch & 1;
    if (ch + 1 < nchunks) {
      load_chunk(st ^ 1, r0 + (long long)(ch + 1) * G_KC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (live) {
      const double* A = As + st * BM * G_PITCH;
      const double* B = Bs + st * BN * G_PITCH;
#pragma unroll 4
      for (int s4 = 0; s4 < 2 * G_KC / 4; s4++) {
        const int kk = 4 * s4 + (lane & 3);
        double a[WM], b[WN], bi[WN];
#pragma unroll
        for (int mt = 0; mt < WM; mt++) a[mt] = A[(wm * WM * 8 + mt * 8 + (lane >> 2)) * G_PITCH + kk];
#pragma unroll
        for (int nt = 0; nt < WN; nt++) {
          b[nt] = B[(wn * WN * 8 + nt * 8 + (lane >> 2)) * G_PITCH + kk];
          double bx = __shfl_xor_sync(0xffffffffu, b[nt], 1);
          bi[nt] = (lane & 1) ? -bx : bx;
        }
#pragma unroll
        for (int mt = 0; mt < WM; mt++)
#pragma unroll
          for (int nt = 0; nt < WN; nt++) {
            dmma(accR[mt][nt][0], accR[mt][nt][1], a[mt], b[nt]);
            dmma(accI[mt][nt][0], accI[mt][nt][1], a[mt], bi[nt]);
          }
      }
    }
    __syncthreads();
  }

  cplx* out = partial + (size_t)blockIdx.y * p * q;
#pragma unroll
  for (int mt = 0; mt < WM; mt++)
#pragma unroll
    for (int nt = 0; nt < WN; nt++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        int m = m0 + wm * WM * 8 + mt * 8 + (lane >> 2);
        int n = n0 + wn * WN * 8 + nt * 8 + 2 * (lane & 3) + e;
        if (m < p && n < q) out[(size_t)n * p + m] = mk(accR[mt][nt][e], accI[mt][nt][e]);
      }
}

__global__ void gram_reduce_kernel(const cplx* partial, int nsplit, int pq, cplx* G) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= pq) return;
  cplx acc = mk(0, 0);
  for (int s = 0; s < nsplit; s++) acc = acc + partial[(size_t)s * pq + idx];
  G[idx] = acc;
}

size_t gram_partial_bytes(int p, int q) { return (size_t)2 * 148 * p * q * sizeof(cplx) + 4096; }

template <int WM, int WN, int WARPS_M, int WARPS_N>
static void run_gram(const ColPtrs& S, int p, const ColPtrs& T, int q, long long len, cplx* G, cplx* partial,
                     int ctas_per_sm, cudaStream_t st) {
  using Cfg = GramCfg<WM, WN, WARPS_M, WARPS_N>;
  auto kern = gram_kernel<WM, WN, WARPS_M, WARPS_N>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    attr = true;
  }
  const int nmb = (p + Cfg::BM - 1) / Cfg::BM, nnb = (q + Cfg::BN - 1) / Cfg::BN;
  const int nblk = nmb * nnb;
  int ns = std::max(1, (ctas_per_sm * 148 + nblk - 1) / nblk);
  ns = (int)std::max(1LL, std::min<long long>(ns, (len + 4 * G_KC - 1) / (4 * G_KC)));
  long long rps = (len + ns - 1) / ns;
  rps = (rps + G_KC - 1) / G_KC * G_KC;
  ns = (int)((len + rps - 1) / rps);
  kern<<<dim3(nblk, ns), Cfg::THREADS, Cfg::SMEM, st>>>(S, p, T, q, len, rps, nmb, partial);
  const int pq = p * q;
  gram_reduce_kernel<<<(pq + 255) / 256, 256, 0, st>>>(partial, ns, pq, G);
}

// Choose the CTA output block with the least padded area (ties: fewer blocks).
void launch_gram(const ColPtrs& S, int p, const ColPtrs& T, int q, long long len, cplx* G, cplx* partial,
                 cudaStream_t st) {
  struct Opt { int bm, bn; };
  const Opt opts[4] = {{48, 64}, {48, 48}, {32, 64}, {16, 32}};
  int best = 0;
  double best_cost = 1e300;
  for (int i = 0; i < 4; i++) {
    double area = (double)((p + opts[i].bm - 1) / opts[i].bm * opts[i].bm) * ((q + opts[i].bn - 1) / opts[i].bn * opts[i].bn);
    double cost = area * (1.0 + 0.02 * i);
    if (cost < best_cost) { best_cost = cost; best = i; }
  }
  switch (best) {
    case 0: run_gram<3, 2, 2, 4>(S, p, T, q, len, G, partial, 1, st); break;
    case 1: run_gram<3, 2, 2, 3>(S, p, T, q, len, G, partial, 2, st); break;
    case 2: run_gram<2, 2, 2, 4>(S, p, T, q, len, G, partial, 2, st); break;
    default: run_gram<2, 2, 1, 2>(S, p, T, q, len, G, partial, 4, st); break;
  }
}

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
    v = Gp[(size_t)(half * c + (j - b)) * p + i];
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
// [row][m] complex with pitch PS = 2 mod 8 (conflict-free fragments); C as [c][m], same pitch.
// ------------------------------------------------------------------------------------------
constexpr int U_ROWS = 64, U_THREADS = 256;

HD int pitch2mod8(int p) {
  int x = p + 1;
  while ((x & 7) != 2) x++;
  return x;
}

template <int NT>
__global__ void __launch_bounds__(U_THREADS) update_kernel(ColPtrs S, int p, const cplx* __restrict__ C, int ldc,
                                                           int r, int split, MutColPtrs Y1, int has_y1, MutColPtrs Y2,
                                                           ColPtrs Add, int has_add, long long len) {
  extern __shared__ __align__(16) double usm[];
  const int pe = (p + 1) & ~1;  // even number of S columns (k' multiple of 4)
  const int PS = pitch2mod8(pe);
  cplx* Ss = reinterpret_cast<cplx*>(usm);   // [2][U_ROWS][PS]
  cplx* Cs = Ss + 2 * U_ROWS * PS;           // [NT*8][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int e = tid; e < NT * 8 * pe; e += U_THREADS) {
    int c = e / pe, m = e % pe;
    Cs[c * PS + m] = (c < r && m < p) ? C[(size_t)c * ldc + m] : mk(0, 0);
  }
  const long long ntiles = (len + U_ROWS - 1) / U_ROWS;
  const cplx* dummy = S.p[0];
  auto load_tile = [&](int stage, long long t) {
    const long long rbase = t * U_ROWS;
    cplx* dst = Ss + stage * U_ROWS * PS;
    for (int e = tid; e < U_ROWS * pe; e += U_THREADS) {
      int m = e / U_ROWS, rr = e % U_ROWS;
      long long row = rbase + rr;
      bool ok = (m < p) && (row < len);
      cp_async16_zfill(&dst[rr * PS + m], ok ? (const void*)(S.p[m] + row) : (const void*)dummy, ok);
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
    double accR[NT][2], accI[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; nt++) accR[nt][0] = accR[nt][1] = accI[nt][0] = accI[nt][1] = 0.0;
    const double* Sd = reinterpret_cast<const double*>(Ss + st * U_ROWS * PS);
    const int arow = warp * 8 + (lane >> 2);

    auto kloop = [&](int mlo, int mhi) {  // contributions of S columns m in [mlo, mhi)
#pragma unroll 2
      for (int m2 = mlo & ~1; m2 < mhi; m2 += 2) {  // one k4 step = 2 complex m
        const int kk = 2 * m2 + (lane & 3);
        const double a = Sd[arow * 2 * PS + kk];
        const int mm = m2 + ((lane & 3) >> 1);
        const bool in = (mm >= mlo) && (mm < mhi);
#pragma unroll
        for (int nt = 0; nt < NT; nt++) {
          cplx cv = Cs[(nt * 8 + (lane >> 2)) * PS + mm];
          if (!in) cv = mk(0, 0);
          const double br = (lane & 1) ? -cv.y : cv.x;
          const double bi = (lane & 1) ? cv.x : cv.y;
          dmma(accR[nt][0], accR[nt][1], a, br);
          dmma(accI[nt][0], accI[nt][1], a, bi);
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
          if (c < r) {
            cplx v = mk(accR[nt][e], accI[nt][e]);
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

template <int NT>
static void run_update(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                       const MutColPtrs& Y2, const ColPtrs* add, long long len, cudaStream_t st) {
  const int pe = (p + 1) & ~1, ps = pitch2mod8(pe);
  const size_t smem = (size_t)(2 * U_ROWS * ps + NT * 8 * ps) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(update_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const long long ntiles = (len + U_ROWS - 1) / U_ROWS;
  const int occ = std::max(1, std::min(3, (int)((227 * 1024) / (smem + 1024))));
  const int grid = (int)std::min<long long>(ntiles, 148LL * occ);
  MutColPtrs y1 = Y1 ? *Y1 : MutColPtrs{};
  ColPtrs ad = add ? *add : ColPtrs{};
  update_kernel<NT><<<grid, U_THREADS, smem, st>>>(S, p, C, ldc, r, split, y1, Y1 ? 1 : 0, Y2, ad, add ? 1 : 0, len);
}

void launch_update(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                   const MutColPtrs& Y2, const ColPtrs* add, long long len, cudaStream_t st) {
  if (r <= 8) run_update<1>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
  else if (r <= 16) run_update<2>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
  else if (r <= 24) run_update<3>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
  else run_update<4>(S, p, C, ldc, r, split, Y1, Y2, add, len, st);
}
