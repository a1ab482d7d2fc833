// Streaming variant of the fused LOBPCG update (same contract as launch_update_all, update_all.cu):
//   P'  = [W P] C_WP,    X'  = X C_X + P'                       (S phase)
//   AP' = [AW AP] C_WP,  AX' = AX C_X + AP'                     (AS phase)
//   R   = AX' - X' diag(lambda'),  W = K_P^{-1} R,  per-CTA |R_c|^2, |X'_c|^2
// (PAPER.md:1055-1064 LOBPCG; 530-548 K_P^{-1}).
//
// The update moves ~13 GB per iteration at n = 128 and does ~4 flop per byte, so it is HBM-bound; the
// shared-memory version stages each row tile with cp.async and synchronises the CTA twice per tile.
// Here every warp is independent: it owns 8 consecutive Fourier modes (all 3 components) and all output
// columns, and loads its DMMA A fragments straight from HBM -- for k-step (input columns m4..m4+3) lane
// (r, k) = (lane >> 2, lane & 3) needs S[m4 + k][component s][mode r], i.e. each warp load is four
// full 128-B lines.  The k-steps of a tile (S phase then AS phase) run through a register ring of
// UST_DEPTH k-steps of prefetch, so several KB per warp are in flight without any barrier.  C (the
// Ritz coefficients) sits in shared memory, loaded once.  Complex products use three real MMAs per
// complex MAC: P1 = a_r c_r, P2 = a_i c_i, P3 = (a_r + a_i)(c_r + c_i).
#include "kernels.h"
#include "dmma.cuh"
#include "kp.cuh"

constexpr int UST_WARPS = 4;
constexpr int UST_THREADS = 32 * UST_WARPS;
constexpr int UST_DEPTH = 4;  // k-steps in flight per warp

HD int ust_pitch4mod8(int p) {
  int x = p;
  while ((x & 7) != 4) x++;
  return x;
}

template <int NT>
__global__ void __launch_bounds__(UST_THREADS) update_stream_kernel(
    ColPtrs S, ColPtrs AS, int p, const cplx* __restrict__ C, int ldc, int r, int split, MutColPtrs Y1s,
    MutColPtrs Y2s, MutColPtrs Y1a, MutColPtrs Y2a, MutColPtrs Wout, const double* __restrict__ lam, int n,
    const cplx* __restrict__ kt, double gamma, double thr, int deflate0, double* partial) {
  extern __shared__ __align__(16) double ustsm[];
  __shared__ double red[UST_WARPS][NT][4][2][2];
  const int n3 = n * n * n;
  const int pe = (p + 3) & ~3;
  const int PS = ust_pitch4mod8(pe);
  cplx* Cs = reinterpret_cast<cplx*>(ustsm);  // [NT*8][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < NT * 8 * pe; e += UST_THREADS) {
    const int c = e / pe, m = e % pe;
    Cs[c * PS + m] = (c < r && m < p) ? C[(size_t)c * ldc + m] : mk(0, 0);
  }
  __syncthreads();

  // k-steps of one phase: first the [split, p) block (P' = [W P] C_WP), then [0, split) (adds X C_X)
  const int m4a = split & ~3;
  const int n1 = (p > split) ? (pe - m4a) / 4 : 0;
  const int n2 = (split + 3) / 4;
  const int nks = n1 + n2;    // k-steps per phase
  const int nq = 2 * nks;     // S phase then AS phase
  auto m4_of = [&](int q) {
    const int k = q % nks;
    return k < n1 ? m4a + 4 * k : 4 * (k - n1);
  };

  const int lr = lane >> 2, lk = lane & 3;
  double nr[NT][2], nx[NT][2];
#pragma unroll
  for (int i = 0; i < NT; i++) nr[i][0] = nr[i][1] = nx[i][0] = nx[i][1] = 0.0;

  const long long ntiles = (n3 + 7) / 8;
  const long long gw = (long long)blockIdx.x * UST_WARPS + warp, nwarps = (long long)gridDim.x * UST_WARPS;
  for (long long t = gw; t < ntiles; t += nwarps) {
    const long long mode = t * 8 + lr;   // this lane's A-fragment row and C-fragment row
    const bool mode_ok = mode < n3;
    // ---- register ring of A fragments: buf[d][s] = (S or AS)[m4(q) + lk][s][mode]
    cplx buf[UST_DEPTH][3];
    auto issue = [&](int d, int q) {
      if (q >= nq) return;
      const int m = m4_of(q) + lk;
      const bool ok = mode_ok && m < p;
      const cplx* col = ok ? ((q < nks) ? S.p[m] : AS.p[m]) : nullptr;  // direct param-bank reads
      const cplx* base = ok ? col + mode : nullptr;
#pragma unroll
      for (int s = 0; s < 3; s++) buf[d][s] = ok ? ldg(base + (long long)s * n3) : mk(0, 0);
    };
#pragma unroll
    for (int d = 0; d < UST_DEPTH; d++) issue(d, d);

    double p1[3][NT][2], p2[3][NT][2], p3[3][NT][2];
    cplx xs[3][NT][2];
    auto zero = [&]() {
#pragma unroll
      for (int s = 0; s < 3; s++)
#pragma unroll
        for (int i = 0; i < NT; i++) p1[s][i][0] = p1[s][i][1] = p2[s][i][0] = p2[s][i][1] = p3[s][i][0] = p3[s][i][1] = 0.0;
    };
    auto val = [&](int s, int i, int e) {
      return mk(p1[s][i][e] - p2[s][i][e], p3[s][i][e] - p1[s][i][e] - p2[s][i][e]);
    };
    auto store = [&](const MutColPtrs& Y, bool keep) {
#pragma unroll
      for (int i = 0; i < NT; i++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = i * 8 + 2 * lk + e;
#pragma unroll
          for (int s = 0; s < 3; s++) {
            const cplx v = val(s, i, e);
            if (keep) xs[s][i][e] = v;
            if (mode_ok && c < r && Y.p[c]) Y.p[c][(long long)s * n3 + mode] = v;
          }
        }
    };
    zero();
    // ---- the k-step stream of this tile
    for (int q0 = 0; q0 < nq; q0 += UST_DEPTH) {
#pragma unroll
      for (int d = 0; d < UST_DEPTH; d++) {
        const int q = q0 + d;
        if (q < nq) {
          const int k = q % nks;
          const bool ph1 = k < n1;
          const int mlo = ph1 ? split : 0, mhi = ph1 ? p : split;
          const int mm = m4_of(q) + lk;
          const bool in = (mm >= mlo) && (mm < mhi);
          cplx a[3];
#pragma unroll
          for (int s = 0; s < 3; s++) a[s] = buf[d][s];
          issue(d, q + UST_DEPTH);  // the slot is free again: prefetch UST_DEPTH k-steps ahead
#pragma unroll
          for (int i = 0; i < NT; i++) {
            cplx cv = Cs[(i * 8 + lr) * PS + mm];
            if (!in) cv = mk(0, 0);
            const double cs = cv.x + cv.y;
#pragma unroll
            for (int s = 0; s < 3; s++) {
              dmma(p1[s][i][0], p1[s][i][1], a[s].x, cv.x);
              dmma(p2[s][i][0], p2[s][i][1], a[s].y, cv.y);
              dmma(p3[s][i][0], p3[s][i][1], a[s].x + a[s].y, cs);
            }
          }
          // phase boundaries
          if (k == n1 - 1) {                                       // P' or AP'
            if (q < nks) store(Y1s, false);
            else store(Y1a, false);
          }
          if (k == nks - 1) {
            if (q < nks) {
              store(Y2s, true);                                    // X' (kept for the residual)
              zero();
            } else {
              store(Y2a, false);                                   // AX'
            }
          }
        }
      }
    }
    // ---- residual, preconditioner, norms (val() = AX', xs = X')
    if (mode_ok) {
      const int mi = (int)mode;
      const int m1 = mi % n, m2 = (mi / n) % n, m3 = mi / (n * n);
      cplx k1, k2, k3;
      kappa_at(kt, n, m1, m2, m3, k1, k2, k3);
#pragma unroll
      for (int i = 0; i < NT; i++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = i * 8 + 2 * lk + e;
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

  // deterministic reduction: lanes sharing lk hold the same columns -> xor over the lr bits, then warps
#pragma unroll
  for (int i = 0; i < NT; i++)
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
  for (int c = tid; c < r; c += UST_THREADS) {
    const int i = c / 8, ln = (c % 8) / 2, e = c % 2;
    double a = 0, b = 0;
    for (int w = 0; w < UST_WARPS; w++) {  // fixed order
      a += red[w][i][ln][e][0];
      b += red[w][i][ln][e][1];
    }
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 0] = a;
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 1] = b;
  }
}

template <int NT>
static int run_update_stream(const ColPtrs& S, const ColPtrs& AS, int p, const cplx* C, int ldc, int r, int split,
                             const MutColPtrs& Y1s, const MutColPtrs& Y2s, const MutColPtrs& Y1a,
                             const MutColPtrs& Y2a, const MutColPtrs& W, const double* lam, int n, const cplx* kt,
                             double gamma, double thr, int deflate0, double* partial, int max_grid,
                             cudaStream_t st) {
  const int pe = (p + 3) & ~3;
  const size_t smem = (size_t)NT * 8 * ust_pitch4mod8(pe) * sizeof(cplx);
  auto kern = update_stream_kernel<NT>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, UST_THREADS, smem);
  occ = std::max(1, occ);
  const long long n3 = (long long)n * n * n;
  const long long ntiles = (n3 + 7) / 8;
  const long long want = (ntiles + UST_WARPS - 1) / UST_WARPS;
  const int grid = (int)std::min<long long>(std::min<long long>(want, 148LL * occ), max_grid);
  kern<<<grid, UST_THREADS, smem, st>>>(S, AS, p, C, ldc, r, split, Y1s, Y2s, Y1a, Y2a, W, lam, n, kt, gamma, thr,
                                       deflate0, partial);
  return grid;
}

int launch_update_stream(const ColPtrs& S, const ColPtrs& AS, int p, const cplx* C, int ldc, int r, int split,
                         const MutColPtrs& Y1s, const MutColPtrs& Y2s, const MutColPtrs& Y1a, const MutColPtrs& Y2a,
                         const MutColPtrs& W, const double* lam, int n, const cplx* kt, double gamma, double thr,
                         int deflate0, double* partial, int max_grid, cudaStream_t st) {
#define PC_US(NT_)                                                                                          \
  return run_update_stream<NT_>(S, AS, p, C, ldc, r, split, Y1s, Y2s, Y1a, Y2a, W, lam, n, kt, gamma, thr, \
                                deflate0, partial, max_grid, st)
  if (r <= 8) PC_US(1);
  if (r <= 16) PC_US(2);
  if (r <= 24) PC_US(3);
  PC_US(4);
#undef PC_US
}
