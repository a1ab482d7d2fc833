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
// CTA output block 48 x 48 (complex), 6 warps as 2 (m) x 3 (n), warp tile 24 x 16 = 3 x 2 m8n8.
// ------------------------------------------------------------------------------------------
constexpr int G_BM = 48, G_BN = 48, G_KC = 32, G_PITCH = 2 * G_KC + 4, G_THREADS = 192;
constexpr size_t G_SMEM = 2 * (size_t)(G_BM + G_BN) * G_PITCH * sizeof(double);

__global__ void __launch_bounds__(G_THREADS) gram_kernel(ColPtrs S, int p, ColPtrs T, int q, long long len,
                                                         long long rows_per_split, int nmb, cplx* partial) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                                // [2][G_BM][G_PITCH]
  double* Bs = gsm + 2 * G_BM * G_PITCH;           // [2][G_BN][G_PITCH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % 2, wn = warp / 2;
  const int mb = blockIdx.x % nmb, nb = blockIdx.x / nmb;
  const int m0 = mb * G_BM, n0 = nb * G_BN;
  const long long r0 = (long long)blockIdx.y * rows_per_split;
  const long long r1 = min(len, r0 + rows_per_split);

  double accR[3][2][2], accI[3][2][2];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 2; j++) accR[i][j][0] = accR[i][j][1] = accI[i][j][0] = accI[i][j][1] = 0.0;

  const cplx* dummy = S.p[0];
  auto load_chunk = [&](int stage, long long rbase) {
    // (G_BM + G_BN) columns x G_KC complex rows
    for (int e = tid; e < (G_BM + G_BN) * G_KC; e += G_THREADS) {
      int c = e / G_KC, r = e % G_KC;
      long long row = rbase + r;
      bool okr = row < r1;
      double* dst;
      const cplx* src = dummy;
      bool ok;
      if (c < G_BM) {
        int m = m0 + c;
        ok = okr && m < p;
        if (ok) src = S.p[m] + row;
        dst = As + (stage * G_BM + c) * G_PITCH + 2 * r;
      } else {
        int n = n0 + (c - G_BM);
        ok = okr && n < q;
        if (ok) src = T.p[n] + row;
        dst = Bs + (stage * G_BN + (c - G_BM)) * G_PITCH + 2 * r;
      }
      cp_async16_zfill(dst, src, ok);
    }
    cp_async_commit();
  };

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
    const double* A = As + st * G_BM * G_PITCH;
    const double* B = Bs + st * G_BN * G_PITCH;
#pragma unroll 4
    for (int s4 = 0; s4 < 2 * G_KC / 4; s4++) {
      const int kk = 4 * s4 + (lane & 3);
      double a[3], b[2], bi[2];
#pragma unroll
      for (int mt = 0; mt < 3; mt++) a[mt] = A[(wm * 24 + mt * 8 + (lane >> 2)) * G_PITCH + kk];
#pragma unroll
      for (int nt = 0; nt < 2; nt++) {
        b[nt] = B[(wn * 16 + nt * 8 + (lane >> 2)) * G_PITCH + kk];
        double bx = __shfl_xor_sync(0xffffffffu, b[nt], 1);
        bi[nt] = (lane & 1) ? -bx : bx;
      }
#pragma unroll
      for (int mt = 0; mt < 3; mt++)
#pragma unroll
        for (int nt = 0; nt < 2; nt++) {
          dmma(accR[mt][nt][0], accR[mt][nt][1], a[mt], b[nt]);
          dmma(accI[mt][nt][0], accI[mt][nt][1], a[mt], bi[nt]);
        }
    }
    __syncthreads();
  }

  cplx* out = partial + (size_t)blockIdx.y * p * q;
#pragma unroll
  for (int mt = 0; mt < 3; mt++)
#pragma unroll
    for (int nt = 0; nt < 2; nt++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        int m = m0 + wm * 24 + mt * 8 + (lane >> 2);
        int n = n0 + wn * 16 + nt * 8 + 2 * (lane & 3) + e;
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

static int gram_nsplit(int p, int q, long long len) {
  int nblk = ((p + G_BM - 1) / G_BM) * ((q + G_BN - 1) / G_BN);
  int ns = std::max(1, (2 * 148 + nblk - 1) / nblk);
  long long maxs = (len + 4 * G_KC - 1) / (4 * G_KC);  // at least 4 chunks per split
  return (int)std::max(1LL, std::min<long long>(ns, maxs));
}

size_t gram_partial_bytes(int p, int q) { return (size_t)2 * 148 * p * q * sizeof(cplx) + 4096; }

void launch_gram(const ColPtrs& S, int p, const ColPtrs& T, int q, long long len, cplx* G, cplx* partial,
                 cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G_SMEM);
    attr = true;
  }
  int nmb = (p + G_BM - 1) / G_BM, nnb = (q + G_BN - 1) / G_BN;
  int ns = gram_nsplit(p, q, len);
  long long rps = (len + ns - 1) / ns;
  rps = (rps + G_KC - 1) / G_KC * G_KC;
  ns = (int)((len + rps - 1) / rps);
  gram_kernel<<<dim3(nmb * nnb, ns), G_THREADS, G_SMEM, st>>>(S, p, T, q, len, rps, nmb, partial);
  int pq = p * q;
  gram_reduce_kernel<<<(pq + 255) / 256, 256, 0, st>>>(partial, ns, pq, G);
}

// ------------------------------------------------------------------------------------------
// Update: phase 1  acc = sum_{m in [split, p)} S[:, m] C[m, :]  -> Y1 (optional)
//         phase 2  acc += sum_{m in [0, split)} S[:, m] C[m, :] -> Y2 (+ Add)
// r <= 32 output columns (4 n-tiles of 8), CTA = 8 warps x 8 rows = 64 rows, persistent over row tiles.
// S tile in smem as [row][m] complex with pitch PS = 2 mod 8 (conflict-free fragments); C as [c][m].
// ------------------------------------------------------------------------------------------
constexpr int U_ROWS = 64, U_THREADS = 256;

DEV int pitch2mod8(int p) {
  int x = p + 1;
  while ((x & 7) != 2) x++;
  return x;
}

__global__ void __launch_bounds__(U_THREADS) update_kernel(ColPtrs S, int p, const cplx* __restrict__ C, int ldc,
                                                           int r, int split, MutColPtrs Y1, int has_y1, MutColPtrs Y2,
                                                           ColPtrs Add, int has_add, long long len) {
  extern __shared__ __align__(16) double usm[];
  const int pe = (p + 1) & ~1;  // even number of S columns (k' multiple of 4)
  const int PS = pitch2mod8(pe);
  const int PC = pitch2mod8(pe);
  cplx* Ss = reinterpret_cast<cplx*>(usm);   // [U_ROWS][PS]
  cplx* Cs = Ss + U_ROWS * PS;               // [32][PC]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // C -> smem (zero padded to 32 columns x pe rows)
  for (int e = tid; e < 32 * pe; e += U_THREADS) {
    int c = e / pe, m = e % pe;
    Cs[c * PC + m] = (c < r && m < p) ? C[(size_t)c * ldc + m] : mk(0, 0);
  }
  const long long ntiles = (len + U_ROWS - 1) / U_ROWS;
  const cplx* dummy = S.p[0];
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long rbase = t * U_ROWS;
    __syncthreads();  // previous tile's smem reads done (and C staged on the first pass)
    for (int e = tid; e < U_ROWS * pe; e += U_THREADS) {
      int m = e / U_ROWS, rr = e % U_ROWS;
      long long row = rbase + rr;
      bool ok = (m < p) && (row < len);
      cp_async16_zfill(&Ss[rr * PS + m], ok ? (const void*)(S.p[m] + row) : (const void*)dummy, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();

    double accR[4][2], accI[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; nt++) accR[nt][0] = accR[nt][1] = accI[nt][0] = accI[nt][1] = 0.0;
    const double* Sd = reinterpret_cast<const double*>(Ss);
    const int arow = warp * 8 + (lane >> 2);

    auto kloop = [&](int mlo, int mhi) {  // contributions of S columns m in [mlo, mhi)
      for (int m2 = mlo & ~1; m2 < mhi; m2 += 2) {  // one k4 step = 2 complex m
        const int kk = 2 * m2 + (lane & 3);
        double a = Sd[arow * 2 * PS + kk];
        const int mm = m2 + ((lane & 3) >> 1);
        const bool in = (mm >= mlo) && (mm < mhi);
#pragma unroll
        for (int nt = 0; nt < 4; nt++) {
          cplx cv = Cs[(nt * 8 + (lane >> 2)) * PC + mm];
          if (!in) cv = mk(0, 0);
          double br = (lane & 1) ? -cv.y : cv.x;
          double bi = (lane & 1) ? cv.x : cv.y;
          dmma(accR[nt][0], accR[nt][1], a, br);
          dmma(accI[nt][0], accI[nt][1], a, bi);
        }
      }
    };
    auto store = [&](const MutColPtrs& Y, bool add) {
      long long row = rbase + warp * 8 + (lane >> 2);
      if (row >= len) return;
#pragma unroll
      for (int nt = 0; nt < 4; nt++)
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
  }
}

void launch_update(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                   const MutColPtrs& Y2, const ColPtrs* add, long long len, cudaStream_t st) {
  int pe = (p + 1) & ~1;
  int ps = pe + 1;
  while ((ps & 7) != 2) ps++;
  size_t smem = (size_t)(U_ROWS * ps + 32 * ps) * sizeof(cplx);
  static int attr_bytes = 0;
  if ((int)smem > attr_bytes) {
    cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_bytes = 200 * 1024;
  }
  long long ntiles = (len + U_ROWS - 1) / U_ROWS;
  int occ = smem <= 70 * 1024 ? 3 : (smem <= 110 * 1024 ? 2 : 1);
  int grid = (int)std::min<long long>(ntiles, 148LL * occ);
  MutColPtrs y1 = Y1 ? *Y1 : MutColPtrs{};
  ColPtrs ad = add ? *add : ColPtrs{};
  update_kernel<<<grid, U_THREADS, smem, st>>>(S, p, C, ldc, r, split, y1, Y1 ? 1 : 0, Y2, ad, add ? 1 : 0, len);
}
