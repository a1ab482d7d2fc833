// Gram products G = S^H T of LOBPCG (the Rayleigh-Ritz projections) on the FP64
// tensor pipe (DMMA mma.sync m8n8k4 f64).  Complex arithmetic with three real products per complex
// MAC (the k dimension of an m8n8k4 step is 4 complex rows):
//   P1 = S_r^T T_r,  P2 = S_i^T T_i,  P3 = (S_r - S_i)^T (T_r + T_i)
//   Re G = P1 + P2,  Im G = P3 - P1 + P2       (conj(S)^T T; 25% fewer MMAs than 4 real products)
// CTA output block BM x BN = (WARPS_M*WM*8) x (WARPS_N*WN*8) complex; each warp owns WM x WN m8n8
// tiles.  Rows stream through a STAGES-deep cp.async pipeline in chunks of KC complex rows.
// Split-K over rows; partials reduced in a fixed order (deterministic).
#include <type_traits>
#include "kernels.h"
#include "dmma.cuh"

template <int WM, int WN, int WARPS_M, int WARPS_N, int KC, int STAGES, int KS = 1>
struct GramCfg {
  static constexpr int BM = WARPS_M * WM * 8, BN = WARPS_N * WN * 8;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N * KS;  // KS warp groups split each chunk's rows
  static constexpr int PITCH = 2 * KC + 8;  // doubles per column, 8 mod 16: 16-B fragment loads conflict-free
  static constexpr size_t SMEM = (size_t)STAGES * (BM + BN) * PITCH * sizeof(double);
};

template <int WM, int WN, int WARPS_M, int WARPS_N, int KC, int STAGES, int KS>
__global__ void __launch_bounds__(GramCfg<WM, WN, WARPS_M, WARPS_N, KC, STAGES, KS>::THREADS)
gram_kernel(ColPtrs S, int p, ColPtrs T, int q, long long len, long long rows_per_split, int nmb, cplx* partial) {
  using Cfg = GramCfg<WM, WN, WARPS_M, WARPS_N, KC, STAGES, KS>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, NTH = Cfg::THREADS, PITCH = Cfg::PITCH;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                           // [STAGES][BM][PITCH]
  double* Bs = gsm + STAGES * BM * PITCH;     // [STAGES][BN][PITCH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kg = warp / (WARPS_M * WARPS_N);  // row group of this warp within a chunk
  const int wm = warp % WARPS_M, wn = (warp / WARPS_M) % WARPS_N;
  const int mb = blockIdx.x % nmb, nb = blockIdx.x / nmb;
  const int m0 = mb * BM, n0 = nb * BN;
  const long long r0 = (long long)blockIdx.y * rows_per_split;
  const long long r1 = min(len, r0 + rows_per_split);

  double p1[WM][WN][2], p2[WM][WN][2], p3[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; i++)
#pragma unroll
    for (int j = 0; j < WN; j++)
#pragma unroll
      for (int e = 0; e < 2; e++) p1[i][j][e] = p2[i][j][e] = p3[i][j][e] = 0.0;

  const cplx* dummy = S.p[0];
  auto load_chunk = [&](int stage, long long rbase) {
    for (int e = tid; e < (BM + BN) * KC; e += NTH) {
      const int c = e / KC, r = e % KC;
      const long long row = rbase + r;
      const bool okr = row < r1;
      double* dst;
      const cplx* src = dummy;
      bool ok;
      if (c < BM) {
        const int m = m0 + c;
        ok = okr && m < p;
        if (ok) src = S.p[m] + row;
        dst = As + (stage * BM + c) * PITCH + 2 * r;
      } else {
        const int n = n0 + (c - BM);
        ok = okr && n < q;
        if (ok) src = T.p[n] + row;
        dst = Bs + (stage * BN + (c - BM)) * PITCH + 2 * r;
      }
      cp_async16_zfill(dst, src, ok);
    }
  };

  // warp tiles entirely outside [0, p) x [0, q) skip their MMAs (warp-uniform)
  const bool live = (m0 + wm * WM * 8 < p) && (n0 + wn * WN * 8 < q);
  const int nchunks = (r1 > r0) ? (int)((r1 - r0 + KC - 1) / KC) : 0;
  // prologue: STAGES-1 chunks in flight (one commit group per chunk, empty groups allowed)
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nchunks) load_chunk(s, r0 + (long long)s * KC);
    cp_async_commit();
  }
  for (int ch = 0; ch < nchunks; ch++) {
    const int nx = ch + STAGES - 1;
    if (nx < nchunks) load_chunk(nx % STAGES, r0 + (long long)nx * KC);
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    __syncthreads();
    if (live) {
      const int st = ch % STAGES;
      const double* A = As + st * BM * PITCH;
      const double* B = Bs + st * BN * PITCH;
#pragma unroll 2
        for (int s4 = kg; s4 < KC / 4; s4 += KS) {
          const int kk = 2 * (4 * s4 + (lane & 3));  // complex row 4 s4 + (lane & 3), interleaved doubles
          double ar[WM], ai[WM], ad[WM], br[WN], bi[WN], bs[WN];
#pragma unroll
          for (int mt = 0; mt < WM; mt++) {
            const double2 v =
                *reinterpret_cast<const double2*>(&A[(wm * WM * 8 + mt * 8 + (lane >> 2)) * PITCH + kk]);
            ar[mt] = v.x;
            ai[mt] = v.y;
            ad[mt] = v.x - v.y;
          }
#pragma unroll
          for (int nt = 0; nt < WN; nt++) {
            const double2 v =
                *reinterpret_cast<const double2*>(&B[(wn * WN * 8 + nt * 8 + (lane >> 2)) * PITCH + kk]);
            br[nt] = v.x;
            bi[nt] = v.y;
            bs[nt] = v.x + v.y;
          }
#pragma unroll
          for (int mt = 0; mt < WM; mt++)
#pragma unroll
            for (int nt = 0; nt < WN; nt++) {
              dmma(p1[mt][nt][0], p1[mt][nt][1], ar[mt], br[nt]);
              dmma(p2[mt][nt][0], p2[mt][nt][1], ai[mt], bi[nt]);
              dmma(p3[mt][nt][0], p3[mt][nt][1], ad[mt], bs[nt]);
            }
        }
    }
    __syncthreads();  // the stage consumed here is refilled STAGES-1 iterations later
  }
  cp_async_wait<0>();

  if constexpr (KS > 1) {
    // fold the row groups' accumulators into group 0 through shared memory (fixed order)
    constexpr int NACC = WM * WN * 6;
    double* red = gsm;  // pipeline buffers are free now
    __syncthreads();
    const int wl = warp % (WARPS_M * WARPS_N);
    for (int g = 1; g < KS; g++) {
      if (kg == g) {
        double* dst = red + ((size_t)wl * 32 + lane) * NACC;
        int t = 0;
#pragma unroll
        for (int mt = 0; mt < WM; mt++)
#pragma unroll
          for (int nt = 0; nt < WN; nt++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
              dst[t++] = p1[mt][nt][e];
              dst[t++] = p2[mt][nt][e];
              dst[t++] = p3[mt][nt][e];
            }
      }
      __syncthreads();
      if (kg == 0) {
        const double* src = red + ((size_t)wl * 32 + lane) * NACC;
        int t = 0;
#pragma unroll
        for (int mt = 0; mt < WM; mt++)
#pragma unroll
          for (int nt = 0; nt < WN; nt++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
              p1[mt][nt][e] += src[t++];
              p2[mt][nt][e] += src[t++];
              p3[mt][nt][e] += src[t++];
            }
      }
      __syncthreads();
    }
    if (kg != 0) return;
  }

  cplx* out = partial + (size_t)blockIdx.y * p * q;
#pragma unroll
  for (int mt = 0; mt < WM; mt++)
#pragma unroll
    for (int nt = 0; nt < WN; nt++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int m = m0 + wm * WM * 8 + mt * 8 + (lane >> 2);
        const int n = n0 + wn * WN * 8 + nt * 8 + 2 * (lane & 3) + e;
        if (m < p && n < q) {
          const double re = p1[mt][nt][e] + p2[mt][nt][e];
          out[(size_t)n * p + m] = mk(re, p3[mt][nt][e] - p1[mt][nt][e] + p2[mt][nt][e]);
        }
      }
}

__global__ void gram_reduce_kernel(const cplx* partial, int nsplit, int pq, cplx* G) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= pq) return;
  cplx acc = mk(0, 0);
  for (int s = 0; s < nsplit; s++) acc = acc + partial[(size_t)s * pq + idx];
  G[idx] = acc;
}

#ifndef PC_GRAM40_KC  // rows per pipeline chunk / stages of the 40 x 40 Gram block (the C4 bench shape)
#define PC_GRAM40_KC 16
#endif
#ifndef PC_GRAM40_ST
#define PC_GRAM40_ST 4
#endif
int grid_cap(int ctas_per_sm) { return std::max(1, 148 * ctas_per_sm); }

static int g_gram_narrow = 1;  // pc_set_option "gram_narrow": the narrow-T block shapes (process-wide)
void set_gram_narrow(int v) { g_gram_narrow = v ? 1 : 0; }

size_t gram_partial_bytes(int p, int q) { return (size_t)4 * 148 * p * q * sizeof(cplx) + 4096; }

template <int WM, int WN, int WARPS_M, int WARPS_N, int KC, int STAGES, int KS = 1>
static void run_gram(const ColPtrs& S, int p, const ColPtrs& T, int q, long long len, cplx* G, cplx* partial,
                     cudaStream_t st) {
  using Cfg = GramCfg<WM, WN, WARPS_M, WARPS_N, KC, STAGES, KS>;
  static_assert(KS == 1 || (size_t)WARPS_M * WARPS_N * 32 * WM * WN * 6 * 8 <= Cfg::SMEM, "reduction buffer");
  auto kern = gram_kernel<WM, WN, WARPS_M, WARPS_N, KC, STAGES, KS>;
  smem_attr((const void*)kern, (int)Cfg::SMEM);
  static int ctas_per_sm = 0;
  if (!ctas_per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, kern, Cfg::THREADS, Cfg::SMEM);
    ctas_per_sm = std::max(1, ctas_per_sm);
  }
  const int nmb = (p + Cfg::BM - 1) / Cfg::BM, nnb = (q + Cfg::BN - 1) / Cfg::BN;
  const int nblk = nmb * nnb;
  int ns = std::max(1, (grid_cap(ctas_per_sm) + nblk - 1) / nblk);
  ns = std::min(ns, 4 * 148);
  ns = (int)std::max(1LL, std::min<long long>(ns, (len + 4 * KC - 1) / (4 * KC)));
  long long rps = (len + ns - 1) / ns;
  rps = (rps + KC - 1) / KC * KC;
  ns = (int)((len + rps - 1) / rps);
  kern<<<dim3(nblk, ns), Cfg::THREADS, Cfg::SMEM, st>>>(S, p, T, q, len, rps, nmb, partial);
  const int pq = p * q;
  gram_reduce_kernel<<<(pq + 255) / 256, 256, 0, st>>>(partial, ns, pq, G);
}

// Block shape: least padded output area (the DMMA pipe is the bound, padding is wasted MMAs), ties
// broken towards fewer CTA blocks per output.
void launch_gram(const ColPtrs& S, int p, const ColPtrs& T, int q, long long len, cplx* G, cplx* partial,
                 cudaStream_t st) {
  struct Opt { int bm, bn; };
  const Opt opts[] = {{48, 64}, {48, 48}, {32, 64}, {32, 32}, {40, 40}, {40, 64}, {64, 64}, {80, 64},
                      {80, 96}, {24, 32}, {48, 96}, {40, 24}, {24, 8}, {40, 8}, {24, 16}, {40, 16}};
  const int nopt = g_gram_narrow ? (int)(sizeof(opts) / sizeof(opts[0])) : 12;
  int best = 0;
  double best_cost = 1e300;
  for (int i = 0; i < nopt; i++) {
    const int nbm = (p + opts[i].bm - 1) / opts[i].bm, nbn = (q + opts[i].bn - 1) / opts[i].bn;
    const double area = (double)nbm * opts[i].bm * nbn * opts[i].bn;
    const double cost = area * (1.0 + 0.04 * (nbm * nbn - 1));
    if (cost < best_cost - 1e-9) { best_cost = cost; best = i; }
  }
  // KS = 2 (two warp groups per chunk, accumulators folded at the end) where the fold buffer fits
#define PC_GRAM_CASE(WM_, WN_, WAM, WAN, KC_, ST_)                                          \
  if (WM_ * WN_ <= 6 &&                                                                      \
      (size_t)WAM * WAN * 32 * WM_ * WN_ * 48 <=                                            \
                            GramCfg<WM_, WN_, WAM, WAN, KC_, ST_, 2>::SMEM)                  \
    run_gram<WM_, WN_, WAM, WAN, KC_, ST_, (WM_ * WN_ <= 6 &&             \
                                            WAM * WAN * 32 * WM_ * WN_ * 48 <=               \
                                            (int)GramCfg<WM_, WN_, WAM, WAN, KC_, ST_, 2>::SMEM) ? 2 : 1>( \
        S, p, T, q, len, G, partial, st);                                           \
  else                                                                                      \
    run_gram<WM_, WN_, WAM, WAN, KC_, ST_, 1>(S, p, T, q, len, G, partial, st);
  switch (best) {
    case 0: PC_GRAM_CASE(3, 2, 2, 4, 16, 3) break;
    case 1: PC_GRAM_CASE(3, 2, 2, 3, 16, 3) break;
    case 2: PC_GRAM_CASE(2, 2, 2, 4, 16, 3) break;
    case 3: PC_GRAM_CASE(2, 2, 2, 2, 16, 3) break;
    case 4: PC_GRAM_CASE(5, 1, 1, 5, PC_GRAM40_KC, PC_GRAM40_ST) break;
    case 5: PC_GRAM_CASE(5, 1, 1, 8, 16, 3) break;
    case 6: PC_GRAM_CASE(4, 2, 2, 4, 16, 3) break;
    case 7: PC_GRAM_CASE(5, 2, 2, 4, 16, 3) break;
    case 8: PC_GRAM_CASE(5, 3, 2, 4, 16, 2) break;
    case 9: PC_GRAM_CASE(3, 1, 1, 4, 16, 3) break;
    case 11: PC_GRAM_CASE(5, 1, 1, 3, 16, 3) break;
    // narrow T blocks (few active W/P columns in the tail of a solve): one or two 8-column warp tiles,
    // so the row chunks are split over 4 (2) warp groups instead
    case 12: run_gram<3, 1, 1, 1, 16, 3, 4>(S, p, T, q, len, G, partial, st); break;
    case 13: run_gram<5, 1, 1, 1, 16, 3, 4>(S, p, T, q, len, G, partial, st); break;
    case 14: run_gram<3, 1, 1, 2, 16, 3, 2>(S, p, T, q, len, G, partial, st); break;
    case 15: run_gram<5, 1, 1, 2, 16, 3, 2>(S, p, T, q, len, G, partial, st); break;
    default: PC_GRAM_CASE(3, 3, 2, 4, 16, 3) break;
  }
}
