// LOBPCG block update of the A-images fused with the next iteration's residual and preconditioner
// (PAPER.md:1055-1064, 530-548).  For the Ritz coefficients C of the current Rayleigh-Ritz step:
//   AP' = [AW AP] C_WP              (phase 1, optional output Y1)
//   AX' = [AX AW AP] C              (phase 2, output Y2; P' accumulators continue into X', see blas.cu)
//   R   = AX' - X' diag(lambda')    (X' was written by the S-update launched just before)
//   W   = K_P^{-1} R                (per Fourier mode; mode 0 zeroed when deflating k = 0)
//   partial sums of |R_c|^2 and |X'_c|^2 per CTA (reduced in a fixed order afterwards).
// Rows are tiled mode-aligned: a tile holds UR_SEG consecutive modes of each of the 3 components, so a
// thread owns the three components of its modes and applies K_P^{-1} in registers.  This removes the
// separate residual pass (one read of X', AX' and the launch).
#include "kernels.h"
#include "dmma.cuh"
#include "kp.cuh"

constexpr int UR_SEG = 32;               // modes per tile
constexpr int UR_ROWS = 3 * UR_SEG;      // rows per tile (3 components)
constexpr int UR_RP = UR_ROWS + 4;       // smem row pitch (complex), 4 mod 8: conflict-free fragments
constexpr int UR_THREADS = 256;          // warp w: modes [8 (w & 3), +8), n-tiles {w >> 2, +2, ...}

HD int ur_pitch2mod8(int p) {
  int x = p + 1;
  while ((x & 7) != 2) x++;
  return x;
}

template <int NT>
__global__ void __launch_bounds__(UR_THREADS) update_resid_kernel(
    ColPtrs S, int p, const cplx* __restrict__ C, int ldc, int r, int split, MutColPtrs Y1, int has_y1,
    MutColPtrs Y2, ColPtrs Xn, MutColPtrs Wout, const double* __restrict__ lam, int n, const cplx* __restrict__ kt,
    double gamma, double thr, int deflate0, double* partial) {
  constexpr int NTW = (NT + 1) / 2;
  extern __shared__ __align__(16) double ursm[];
  __shared__ double red[8][NTW][4][2][2];
  const int n3 = n * n * n;
  const int pe = (p + 1) & ~1;
  const int PS = ur_pitch2mod8(pe);
  cplx* Ss = reinterpret_cast<cplx*>(ursm);  // [2][pe][UR_RP]
  cplx* Cs = Ss + 2 * pe * UR_RP;            // [NT*8][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = warp & 3, ng = warp >> 2;

  for (int e = tid; e < NT * 8 * pe; e += UR_THREADS) {
    int c = e / pe, m = e % pe;
    Cs[c * PS + m] = (c < r && m < p) ? C[(size_t)c * ldc + m] : mk(0, 0);
  }
  const long long ntiles = (n3 + UR_SEG - 1) / UR_SEG;
  const cplx* dummy = S.p[0];
  auto load_tile = [&](int stage, long long t) {
    const long long m0 = t * UR_SEG;
    cplx* dst = Ss + stage * pe * UR_RP;
    for (int e = tid; e < UR_ROWS * pe; e += UR_THREADS) {
      const int m = e / UR_ROWS, rho = e % UR_ROWS;
      const int seg = rho / UR_SEG, rr = rho % UR_SEG;
      const long long mode = m0 + rr;
      const bool ok = (m < p) && (mode < n3);
      cp_async16_zfill(&dst[m * UR_RP + rho], ok ? (const void*)(S.p[m] + (long long)seg * n3 + mode) : (const void*)dummy,
                       ok);
    }
    cp_async_commit();
  };

  double nr[NTW][2], nx[NTW][2];
#pragma unroll
  for (int i = 0; i < NTW; i++) nr[i][0] = nr[i][1] = nx[i][0] = nx[i][1] = 0.0;

  long long t = blockIdx.x;
  if (t < ntiles) load_tile(0, t);
  for (int it = 0; t < ntiles; t += gridDim.x, it++) {
    const int st = it & 1;
    if (t + gridDim.x < ntiles) {
      load_tile(st ^ 1, t + gridDim.x);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const long long m0 = t * UR_SEG;
    const double* Sd = reinterpret_cast<const double*>(Ss + st * pe * UR_RP);
    const int lrow = 8 * rg + (lane >> 2);  // local mode of this thread's fragment rows
    double accR[3][NTW][2], accI[3][NTW][2];
#pragma unroll
    for (int s = 0; s < 3; s++)
#pragma unroll
      for (int i = 0; i < NTW; i++) accR[s][i][0] = accR[s][i][1] = accI[s][i][0] = accI[s][i][1] = 0.0;

    auto kloop = [&](int mlo, int mhi) {
#pragma unroll 2
      for (int m2 = mlo & ~1; m2 < mhi; m2 += 2) {
        const int mm = m2 + ((lane & 3) >> 1);
        const bool in = (mm >= mlo) && (mm < mhi);
        double a[3];
#pragma unroll
        for (int s = 0; s < 3; s++) a[s] = Sd[2 * (mm * UR_RP + s * UR_SEG + lrow) + (lane & 1)];
#pragma unroll
        for (int i = 0; i < NTW; i++) {
          const int nt = ng + 2 * i;
          if (nt >= NT) break;
          cplx cv = Cs[(nt * 8 + (lane >> 2)) * PS + mm];
          if (!in) cv = mk(0, 0);
          const double br = (lane & 1) ? -cv.y : cv.x;
          const double bi = (lane & 1) ? cv.x : cv.y;
#pragma unroll
          for (int s = 0; s < 3; s++) {
            dmma(accR[s][i][0], accR[s][i][1], a[s], br);
            dmma(accI[s][i][0], accI[s][i][1], a[s], bi);
          }
        }
      }
    };
    const long long mode = m0 + lrow;
    const bool mode_ok = mode < n3;
    auto store = [&](const MutColPtrs& Y) {
      if (!mode_ok) return;
#pragma unroll
      for (int i = 0; i < NTW; i++) {
        const int nt = ng + 2 * i;
        if (nt >= NT) break;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = nt * 8 + 2 * (lane & 3) + e;
          if (c < r && Y.p[c]) {
#pragma unroll
            for (int s = 0; s < 3; s++) Y.p[c][(long long)s * n3 + mode] = mk(accR[s][i][e], accI[s][i][e]);
          }
        }
      }
    };
    kloop(split, p);
    if (has_y1) store(Y1);
    kloop(0, split);
    store(Y2);
    // residual + preconditioner + norms
    if (mode_ok) {
      const int mi = (int)mode;
      const int m1 = mi % n, m2 = (mi / n) % n, m3 = mi / (n * n);
      cplx k1, k2, k3;
      kappa_at(kt, n, m1, m2, m3, k1, k2, k3);
#pragma unroll
      for (int i = 0; i < NTW; i++) {
        const int nt = ng + 2 * i;
        if (nt >= NT) break;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = nt * 8 + 2 * (lane & 3) + e;
          if (c >= r) continue;
          const double l = lam[c];
          cplx rv[3];
#pragma unroll
          for (int s = 0; s < 3; s++) {
            const cplx x = ldg(Xn.p[c] + (long long)s * n3 + mi);
            rv[s] = mk(accR[s][i][e] - l * x.x, accI[s][i][e] - l * x.y);
            nr[i][e] += abs2(rv[s]);
            nx[i][e] += abs2(x);
          }
          cplx* w = Wout.p[c];
          if (w) {
            kp_inv(k1, k2, k3, gamma, thr, rv[0], rv[1], rv[2]);
            if (deflate0 && mi == 0) rv[0] = rv[1] = rv[2] = mk(0, 0);
#pragma unroll
            for (int s = 0; s < 3; s++) w[(long long)s * n3 + mi] = rv[s];
          }
        }
      }
    }
    __syncthreads();  // stage st is refilled by the next iteration's prefetch
  }

  // deterministic reduction: lanes sharing (lane & 3) hold the same column -> xor over lane >> 2 bits
#pragma unroll
  for (int i = 0; i < NTW; i++)
#pragma unroll
    for (int e = 0; e < 2; e++) {
      double a = nr[i][e], b = nx[i][e];
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
      }
      if (lane < 4) {
        red[warp][i][lane][e][0] = a;
        red[warp][i][lane][e][1] = b;
      }
    }
  __syncthreads();
  for (int c = tid; c < r; c += UR_THREADS) {
    const int nt = c / 8, i = (nt - (nt & 1)) / 2, g = nt & 1;
    const int ln = (c % 8) / 2, e = c % 2;
    double a = 0, b = 0;
    for (int q = 0; q < 4; q++) {  // the four row-group warps of n-tile group g, fixed order
      a += red[q + 4 * g][i][ln][e][0];
      b += red[q + 4 * g][i][ln][e][1];
    }
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 0] = a;
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 1] = b;
  }
}

template <int NT>
static int run_update_resid(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                            const MutColPtrs& Y2, const ColPtrs& Xn, const MutColPtrs& W, const double* lam, int n,
                            const cplx* kt, double gamma, double thr, int deflate0, double* partial, int max_grid,
                            cudaStream_t st) {
  const int pe = (p + 1) & ~1, ps = ur_pitch2mod8(pe);
  const size_t smem = (size_t)(2 * pe * UR_RP + NT * 8 * ps) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(update_resid_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const long long n3 = (long long)n * n * n;
  const long long ntiles = (n3 + UR_SEG - 1) / UR_SEG;
  const int occ = std::max(1, std::min(3, (int)((227 * 1024) / (smem + 4096))));
  const int grid = (int)std::min<long long>(std::min<long long>(ntiles, 148LL * occ), max_grid);
  MutColPtrs y1 = Y1 ? *Y1 : MutColPtrs{};
  update_resid_kernel<NT><<<grid, UR_THREADS, smem, st>>>(S, p, C, ldc, r, split, y1, Y1 ? 1 : 0, Y2, Xn, W, lam, n, kt,
                                                           gamma, thr, deflate0, partial);
  return grid;
}

int launch_update_resid(const ColPtrs& S, int p, const cplx* C, int ldc, int r, int split, const MutColPtrs* Y1,
                        const MutColPtrs& Y2, const ColPtrs& Xn, const MutColPtrs& W, const double* lam, int n,
                        const cplx* kt, double gamma, double thr, int deflate0, double* partial, int max_grid,
                        cudaStream_t st) {
  if (r <= 8) return run_update_resid<1>(S, p, C, ldc, r, split, Y1, Y2, Xn, W, lam, n, kt, gamma, thr, deflate0, partial, max_grid, st);
  if (r <= 16) return run_update_resid<2>(S, p, C, ldc, r, split, Y1, Y2, Xn, W, lam, n, kt, gamma, thr, deflate0, partial, max_grid, st);
  if (r <= 24) return run_update_resid<3>(S, p, C, ldc, r, split, Y1, Y2, Xn, W, lam, n, kt, gamma, thr, deflate0, partial, max_grid, st);
  return run_update_resid<4>(S, p, C, ldc, r, split, Y1, Y2, Xn, W, lam, n, kt, gamma, thr, deflate0, partial, max_grid, st);
}
