// LOBPCG block updates of both S = [X W P] and AS = [AX AW AP] fused with the next iteration's
// residual and preconditioner.  For the Ritz coefficients C:
//   P'  = [W P] C_WP,    X'  = X C_X + P'                       (S phase: Y1s, Y2s)
//   AP' = [AW AP] C_WP,  AX' = AX C_X + AP'                     (AS phase: Y1a, Y2a)
//   R   = AX' - X' diag(lambda')      (X' kept in registers between the phases)
//   W   = K_P^{-1} R                  (per Fourier mode; mode 0 zeroed when deflating k = 0)
//   partial sums of |R_c|^2 and |X'_c|^2 per CTA (reduced in a fixed order afterwards).
// Rows are tiled mode-aligned: a tile holds UA_SEG consecutive modes of each of the 3 components, so
// a thread owns all components of its modes and applies K_P^{-1} in registers.  Compared with two
// update launches plus the residual pass this saves the re-read of X' and AX' and two launches.
// The S tile of row tile t+1 streams into one buffer while the AS tile of t is multiplied and vice
// versa.  Complex products use three real MMAs per complex MAC (see blas.cu).
#include "kernels.h"
#include "dmma.cuh"
#include "kp.cuh"

#ifndef PC_UA_SEG
#define PC_UA_SEG 16
#endif
constexpr int UA_SEG = PC_UA_SEG;        // modes per tile (multiple of 8)
constexpr int UA_RG = UA_SEG / 8;        // 8-mode row groups per component
constexpr int UA_ROWS = 3 * UA_SEG;      // rows per tile (3 components)
constexpr int UA_RP = UA_ROWS + 2;       // smem row pitch (complex), 2 mod 8
constexpr int UA_WARPS = 2 * UA_RG;      // warp w: modes [8 (w % UA_RG), +8), n-tiles {w / UA_RG, +2, ...}
constexpr int UA_THREADS = 32 * UA_WARPS;

HD int ua_pitch4mod8(int p) {
  int x = p;
  while ((x & 7) != 4) x++;
  return x;
}

template <int NT>
__global__ void __launch_bounds__(UA_THREADS, (NT <= 2) ? 512 / UA_THREADS : 1) update_all_kernel(
    ColPtrs S, ColPtrs AS, int p, const cplx* __restrict__ C, int ldc, int r, int split, MutColPtrs Y1s,
    MutColPtrs Y2s, MutColPtrs Y1a, MutColPtrs Y2a, MutColPtrs Wout, const double* __restrict__ lam, int n,
    const cplx* __restrict__ kt, double gamma, double thr, int deflate0, double* partial) {
  constexpr int NTW = (NT + 1) / 2;
  extern __shared__ __align__(16) double uasm[];
  __shared__ double red[UA_WARPS][NTW][4][2][2];
  const int n3 = n * n * n;
  const int pe = (p + 3) & ~3;
  const int PS = ua_pitch4mod8(pe);
  constexpr int RP = UA_RP;
  auto RI = [](int m, int rho) { return m * RP + rho; };
  cplx* Buf = reinterpret_cast<cplx*>(uasm);  // [2][pe][RP]: buffer 0 = S tiles, 1 = AS tiles
  cplx* Cs = Buf + 2 * pe * RP;               // [NT*8][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = warp % UA_RG, ng = warp / UA_RG;

  for (int e = tid; e < NT * 8 * pe; e += UA_THREADS) {
    int c = e / pe, m = e % pe;
    Cs[c * PS + m] = (c < r && m < p) ? C[(size_t)c * ldc + m] : mk(0, 0);
  }
  const long long ntiles = (n3 + UA_SEG - 1) / UA_SEG;
  const cplx* dummy = S.p[0];
  auto load_tile = [&](int buf, const ColPtrs& src, long long t) {
    const long long m0 = t * UA_SEG;
    cplx* dst = Buf + buf * pe * RP;
    for (int e = tid; e < UA_ROWS * pe; e += UA_THREADS) {
      const int m = e / UA_ROWS, rho = e % UA_ROWS;
      const int seg = rho / UA_SEG, rr = rho % UA_SEG;
      const long long mode = m0 + rr;
      const bool ok = (m < p) && (mode < n3);
      cp_async16_zfill(&dst[RI(m, rho)],
                       ok ? (const void*)(src.p[m] + (long long)seg * n3 + mode) : (const void*)dummy, ok);
    }
    cp_async_commit();
  };

  double nr[NTW][2], nx[NTW][2];
#pragma unroll
  for (int i = 0; i < NTW; i++) nr[i][0] = nr[i][1] = nx[i][0] = nx[i][1] = 0.0;

  const int lrow = 8 * rg + (lane >> 2);  // local mode of this thread's fragment rows
  double p1[3][NTW][2], p2[3][NTW][2], p3[3][NTW][2];
  auto zero = [&]() {
#pragma unroll
    for (int s = 0; s < 3; s++)
#pragma unroll
      for (int i = 0; i < NTW; i++)
#pragma unroll
        for (int e = 0; e < 2; e++) p1[s][i][e] = p2[s][i][e] = p3[s][i][e] = 0.0;
  };
  auto kloop = [&](const cplx* Sc, int mlo, int mhi) {
#pragma unroll 2
    for (int m4 = mlo & ~3; m4 < mhi; m4 += 4) {
      const int mm = m4 + (lane & 3);
      const bool in = (mm >= mlo) && (mm < mhi);
      cplx a[3];
#pragma unroll
      for (int s = 0; s < 3; s++) a[s] = Sc[RI(mm, s * UA_SEG + lrow)];
#pragma unroll
      for (int i = 0; i < NTW; i++) {
        const int nt = ng + 2 * i;
        if (nt >= NT) break;
        cplx cv = Cs[(nt * 8 + (lane >> 2)) * PS + mm];
        if (!in) cv = mk(0, 0);
        const double cs = cv.x + cv.y;
#ifdef PC_UA_NOMMA  // timing experiment: memory traffic only (results wrong)
        if (cs != 12345.0) continue;
#endif
#pragma unroll
        for (int s = 0; s < 3; s++) {
          dmma(p1[s][i][0], p1[s][i][1], a[s].x, cv.x);
          dmma(p2[s][i][0], p2[s][i][1], a[s].y, cv.y);
          dmma(p3[s][i][0], p3[s][i][1], a[s].x + a[s].y, cs);
        }
      }
    }
  };
  auto val = [&](int s, int i, int e) {
    return mk(p1[s][i][e] - p2[s][i][e], p3[s][i][e] - p1[s][i][e] - p2[s][i][e]);
  };
  cplx xs[3][NTW][2];

  long long t = blockIdx.x;
  if (t < ntiles) {
    load_tile(0, S, t);
    load_tile(1, AS, t);
  }
  for (; t < ntiles; t += gridDim.x) {
    const long long m0 = t * UA_SEG;
    const long long mode = m0 + lrow;
    const bool mode_ok = mode < n3;
    const bool more = t + gridDim.x < ntiles;
    auto store = [&](const MutColPtrs& Y, bool keep) {
#pragma unroll
      for (int i = 0; i < NTW; i++) {
        const int nt = ng + 2 * i;
        if (nt >= NT) break;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = nt * 8 + 2 * (lane & 3) + e;
#pragma unroll
          for (int s = 0; s < 3; s++) {
            const cplx v = val(s, i, e);
            if (keep) xs[s][i][e] = v;
            if (mode_ok && c < r && Y.p[c]) Y.p[c][(long long)s * n3 + mode] = v;
          }
        }
      }
    };
    // ---- S phase (buffer 0)
    cp_async_wait<1>();  // the S tile of t has landed (the AS tile may still stream)
    __syncthreads();
    zero();
    kloop(Buf, split, p);
    store(Y1s, false);
    kloop(Buf, 0, split);
    store(Y2s, true);
    __syncthreads();  // buffer 0 is free
    if (more) load_tile(0, S, t + gridDim.x);
    // ---- AS phase (buffer 1)
    if (more) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    zero();
    const cplx* Ac = Buf + pe * RP;
    kloop(Ac, split, p);
    store(Y1a, false);
    kloop(Ac, 0, split);
    store(Y2a, false);
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
            const cplx x = xs[s][i][e];
            const cplx ax = val(s, i, e);
            rv[s] = mk(ax.x - l * x.x, ax.y - l * x.y);
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
    __syncthreads();  // buffer 1 is free
    if (more) load_tile(1, AS, t + gridDim.x);
  }
  cp_async_wait<0>();

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
  for (int c = tid; c < r; c += UA_THREADS) {
    const int nt = c / 8, i = nt >> 1, g = nt & 1;
    const int ln = (c % 8) / 2, e = c % 2;
    double a = 0, b = 0;
    for (int q = 0; q < UA_RG; q++) {  // the row-group warps of n-tile group g, fixed order
      a += red[UA_RG * g + q][i][ln][e][0];
      b += red[UA_RG * g + q][i][ln][e][1];
    }
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 0] = a;
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 1] = b;
  }
}

template <int NT>
static int run_update_all(const ColPtrs& S, const ColPtrs& AS, int p, const cplx* C, int ldc, int r, int split,
                          const MutColPtrs& Y1s, const MutColPtrs& Y2s, const MutColPtrs& Y1a,
                          const MutColPtrs& Y2a, const MutColPtrs& W, const double* lam, int n, const cplx* kt,
                          double gamma, double thr, int deflate0, double* partial, int max_grid, cudaStream_t st) {
  const int pe = (p + 3) & ~3, ps = ua_pitch4mod8(pe);
  const size_t smem = (size_t)(2 * pe * UA_RP + NT * 8 * ps) * sizeof(cplx);
  auto kern = update_all_kernel<NT>;
  smem_attr((const void*)kern, 200 * 1024);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, UA_THREADS, smem);
  occ = std::max(1, std::min(8, occ));
  const long long n3 = (long long)n * n * n;
  const long long ntiles = (n3 + UA_SEG - 1) / UA_SEG;
  const int grid = (int)std::min<long long>(std::min<long long>(ntiles, (long long)grid_cap(occ)), max_grid);
  kern<<<grid, UA_THREADS, smem, st>>>(S, AS, p, C, ldc, r, split, Y1s, Y2s, Y1a, Y2a, W, lam, n, kt, gamma, thr,
                                       deflate0, partial);
  return grid;
}

int launch_update_all(const ColPtrs& S, const ColPtrs& AS, int p, const cplx* C, int ldc, int r, int split,
                      const MutColPtrs& Y1s, const MutColPtrs& Y2s, const MutColPtrs& Y1a, const MutColPtrs& Y2a,
                      const MutColPtrs& W, const double* lam, int n, const cplx* kt, double gamma, double thr,
                      int deflate0, double* partial, int max_grid, cudaStream_t st) {
#define PC_UA_ARGS S, AS, p, C, ldc, r, split, Y1s, Y2s, Y1a, Y2a, W, lam, n, kt, gamma, thr, deflate0, partial, max_grid, st
#define PC_UA(NT_) return run_update_all<NT_>(PC_UA_ARGS)
  if (r <= 8) PC_UA(1);
  if (r <= 16) PC_UA(2);
  if (r <= 24) PC_UA(3);
  PC_UA(4);
#undef PC_UA
#undef PC_UA_ARGS
}
