// LOBPCG block updates fused with the next residual and K_P^{-1} (same contract as update_all.cu,
// PAPER.md:1055-1064, 530-548), with the row tiles streamed by TMA tensor copies.
//
//   P'  = [W P] C_WP,    X'  = X C_X + P'                       (S phase)
//   AP' = [AW AP] C_WP,  AX' = AX C_X + AP'                     (AS phase)
//   R   = AX' - X' diag(lambda'),  W' = K_P^{-1} R,  per-CTA |R_c|^2, |X'_c|^2
//
// Why: in update_all.cu the compute threads issue the loads (16-B cp.async) at phase boundaries and
// read the output column pointers from a parameter table with per-lane (divergent) indices; its
// DMMA work (~43 % of the pipe) and HBM stream (~4.2 TB/s) barely overlapped (ncu stalls: math pipe,
// shared loads, and the predicates of the stores).  Here one thread issues, per phase, three 4-D
// tensor copies (the X, W and P blocks of a slot: box = 16 modes x 3 components x a column range)
// into a 2-stage ring (3 CTAs = 12 warps per SM), the output columns are base + c * ld with a bit
// mask, and K_P^{-1} costs one division per mode: 3.09 -> 2.49 ms for the n = 128, b = 15 update
// (5.25 TB/s of algorithmic traffic, 80 % of the measured copy peak; tools/bench_block.py).
//
// Tensor view of a slot (b equally spaced columns of 3N^3 complex, column stride = ld):
//   dim0: 16 doubles (8 modes, re/im)  dim1: N^3/8 mode blocks (128 B)  dim2: 3 components (N^3*16 B)
//   dim3: columns (ld*16 B).  Box (16, 2, 3, nc) = 16 modes x 3 components x nc columns, landing in
// shared memory as [column][component][half][128 B] with the 128-B swizzle (16-B chunk j of 128-B row
// r at chunk j ^ (r & 7)), which makes the DMMA A-fragment loads (8 modes x 4 columns per quarter
// warp) conflict-free without padding.  A block starts at an even column (see PC_UT_ALIGN); columns of
// a box that are not in the basis (soft-locked columns between active ones) and the padding columns
// get zero rows of C.
#include <cuda.h>
#include <cudaTypedefs.h>
#include "kernels.h"
#include "dmma.cuh"
#include "kp.cuh"
#include "tma.cuh"

constexpr int UT_SEG = 16;              // modes per tile
// Warp w: modes [8 (w & 1), +8), n-tiles {w >> 1, + UtGeom<NT>::NG, ...}.  NG = 2 n-tile groups (4 warps)
// for b <= 16; for b > 16 one group per 8-column n-tile (6 warps at 168 registers, 2 CTAs/SM, for
// b = 17..24; 8 warps, 1 CTA/SM, for b = 25..32), so a warp holds one output tile (2 tiles per warp needed
// 255 registers with spills).  Measured: b = 22 5.82 -> 4.66 ms at n = 128, b = 26
// 31.2 -> 27.0 ms at n = 192.  PC_UT_NG2: the 4-warp layout for every b.
template <int NT>
struct UtGeom {
#ifdef PC_UT_NG2
  static constexpr int NG = 2;
#else
  static constexpr int NG = (NT <= 2) ? 2 : NT;
#endif
  static constexpr int THREADS = 64 * NG;
  static constexpr int NTW = (NT + NG - 1) / NG;  // n-tiles per warp
};
#ifndef PC_UT_STAGES
#define PC_UT_STAGES 2
#endif
#ifndef PC_UT_MINB
#define PC_UT_MINB 3
#endif
constexpr int UT_STAGES = PC_UT_STAGES;
#ifndef PC_UT_ALIGN
// block starts in columns: the tensor copies swizzle on absolute shared-memory address bits, so a box
// may start inside a 1024-B swizzle atom (parity-tested with 1, 2 and 4); even starts (1536 B) keep the
// basis at 36 stage columns for b = 15, 16 (40 with 4) and measured fastest (2.34 vs 2.50 ms)
#define PC_UT_ALIGN 2
#endif
#ifndef PC_UT_UNROLL
#define PC_UT_UNROLL 4
#endif
constexpr int UT_UNROLL = PC_UT_UNROLL;
constexpr int UT_COLB = 3 * UT_SEG * 16;  // bytes per column of a stage (768)

struct UtMaps {
  CUtensorMap m[6];   // S: X, W, P blocks; AS: AX, AW, AP blocks
  int c0[3];          // first slot column of each block's box
  int nc[3];          // columns per box (0: block absent)
  int off[3];         // stage column where each block lands (multiple of 4)
  int pe;             // stage columns (multiple of 4)
  int split;          // off[1]: columns [0, split) are X
  signed char crow[80];  // stage column -> row of C (-1: zero row)
};

DEV void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// stage element (column m, component s, local mode q) in complex (16-B) units
DEV int ut_idx(int m, int s, int q) {
  const int row = (m * 3 + s) * 2 + (q >> 3);
  return row * 8 + ((q & 7) ^ (row & 7));
}

// Outputs as strided column sets (the LOBPCG slots): column c of output o is base[o] + c * ld, written
// iff bit c of mask[o] is set (o: 0 P', 1 X', 2 AP', 3 AX', 4 W').  Column pointers are formed in
// registers: a per-lane pointer table would be read from the parameter space with divergent indices.
struct UtOut {
  cplx* base[5];
  unsigned mask[5];
  long long ld;
};

template <int NT>
__global__ void __launch_bounds__(UtGeom<NT>::THREADS, (NT <= 2) ? PC_UT_MINB : ((NT == 3 && UtGeom<NT>::NG == 3) ? 2 : 1)) update_tmap_kernel(
    const __grid_constant__ UtMaps mp, const cplx* __restrict__ C, int ldc, int r, const __grid_constant__ UtOut yo,
    const double* __restrict__ lam, int n, const cplx* __restrict__ kt, double gamma, double thr, int deflate0,
    double* partial) {
  constexpr int NTW = UtGeom<NT>::NTW, NG = UtGeom<NT>::NG, UT_THREADS = UtGeom<NT>::THREADS;
  extern __shared__ __align__(1024) unsigned char utsm_raw[];
  // dynamic shared memory is only guaranteed 16-B aligned: round the ring up to 1024 B
  cplx* Ring = reinterpret_cast<cplx*>((reinterpret_cast<uintptr_t>(utsm_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ double red[2 * NG][NTW][4][2][2];
  __shared__ __align__(8) unsigned long long full[UT_STAGES];
  const int n3 = n * n * n;
  const int pe = mp.pe, split = mp.split;
  const int stage_cplx = pe * UT_COLB / 16;
  const int PS = ((pe + 3) & ~7) + 4;  // 4 mod 8: conflict-free 16-B C fragments
  cplx* Cs = Ring + UT_STAGES * stage_cplx;  // [NT*8][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = warp & 1, ng = warp >> 1;

  for (int e = tid; e < NT * 8 * pe; e += UT_THREADS) {
    const int c = e / pe, m = e % pe;
    const int cr = mp.crow[m];
    Cs[c * PS + m] = (c < r && cr >= 0) ? C[(size_t)c * ldc + cr] : mk(0, 0);
  }
  // padding columns are never written by the tensor copies: zero them once (0 * NaN = NaN)
  for (int st = 0; st < UT_STAGES; st++) {
    cplx* sb = Ring + st * stage_cplx;
    for (int e = tid; e < pe * 48; e += UT_THREADS) {
      const int m = e / 48;
      bool pad = true;
#pragma unroll
      for (int k = 0; k < 3; k++)
        if (m >= mp.off[k] && m < mp.off[k] + mp.nc[k]) pad = false;
      if (pad) sb[m * 48 + e % 48] = mk(0, 0);
    }
  }
  unsigned txb = 0;
#pragma unroll
  for (int k = 0; k < 3; k++) txb += (unsigned)mp.nc[k] * UT_COLB;
  if (tid == 0) {
    for (int st = 0; st < UT_STAGES; st++) mbar_init(&full[st], 1);
  }
  fence_proxy_async();
  __syncthreads();

  const long long ntiles = (n3 + UT_SEG - 1) / UT_SEG;
  const long long my_tiles = (blockIdx.x < ntiles) ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nphase = 2 * my_tiles;
  // phase q: tile blockIdx.x + (q / 2) * gridDim.x, half q & 1 (0: S maps 0-2, 1: AS maps 3-5)
  auto issue = [&](long long q) {
    const int st = (int)(q % UT_STAGES);
    const long long t = blockIdx.x + (q >> 1) * (long long)gridDim.x;
    const int h = (int)(q & 1);
    cplx* dst = Ring + st * stage_cplx;
    mbar_arrive_expect_tx(&full[st], txb);
#pragma unroll
    for (int k = 0; k < 3; k++)
      if (mp.nc[k] > 0)
        tma_load_4d(dst + mp.off[k] * (UT_COLB / 16), &mp.m[3 * h + k], 0, (int)(2 * t), 0, mp.c0[k], &full[st]);
  };
  if (tid == 0)
    for (long long q = 0; q < UT_STAGES && q < nphase; q++) issue(q);

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
#pragma unroll UT_UNROLL
    for (int m4 = mlo; m4 < mhi; m4 += 4) {
      const int mm = m4 + (lane & 3);
      cplx a[3];
#pragma unroll
      for (int s = 0; s < 3; s++) a[s] = Sc[ut_idx(mm, s, lrow)];
#pragma unroll
      for (int i = 0; i < NTW; i++) {
        const int nt = ng + NG * i;
        if (nt >= NT) break;
        const cplx cv = Cs[(nt * 8 + (lane >> 2)) * PS + mm];
        const double cs = cv.x + cv.y;
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

  for (long long q = 0; q < nphase; q++) {
    const int st = (int)(q % UT_STAGES);
    const long long t = blockIdx.x + (q >> 1) * (long long)gridDim.x;
    const int h = (int)(q & 1);
    const long long mode = t * UT_SEG + lrow;
    const bool mode_ok = mode < n3;
    mbar_wait(&full[st], (unsigned)((q / UT_STAGES) & 1));
    const cplx* Sc = Ring + st * stage_cplx;
    auto store = [&](int o, bool keep) {
#pragma unroll
      for (int i = 0; i < NTW; i++) {
        const int nt = ng + NG * i;
        if (nt >= NT) break;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = nt * 8 + 2 * (lane & 3) + e;
          const bool wr = mode_ok && ((yo.mask[o] >> c) & 1u);
          cplx* y = yo.base[o] + (long long)c * yo.ld + mode;
#pragma unroll
          for (int s = 0; s < 3; s++) {
            const cplx v = val(s, i, e);
            if (keep) xs[s][i][e] = v;
            if (wr) y[(long long)s * n3] = v;
          }
        }
      }
    };
    zero();
    kloop(Sc, split, pe);
    if (h == 0) {
      store(0, false);
      kloop(Sc, 0, split);
      store(1, true);
    } else {
      store(2, false);
      kloop(Sc, 0, split);
      store(3, false);
    }
    __syncthreads();  // stage st is free
    if (tid == 0 && q + UT_STAGES < nphase) {
      fence_proxy_async();
      issue(q + UT_STAGES);
    }
    if (h == 1 && mode_ok) {  // residual + preconditioner + norms
      const int mi = (int)mode;
      const int m1 = mi % n, m2 = (mi / n) % n, m3 = mi / (n * n);
      cplx k1, k2, k3;
      kappa_at(kt, n, m1, m2, m3, k1, k2, k3);
      // K_P^{-1} per mode (kp.cuh): one division per mode, shared by the thread's columns
      const double k2n = abs2(k1) + abs2(k2) + abs2(k3);
      const bool pass = !(k2n > thr);
      const double inv = pass ? 1.0 : 1.0 / k2n;
      const double fk = pass ? 0.0 : (gamma - 1.0) / gamma * inv * inv;
      const bool zero0 = deflate0 && mi == 0;
#pragma unroll
      for (int i = 0; i < NTW; i++) {
        const int nt = ng + NG * i;
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
          if ((yo.mask[4] >> c) & 1u) {
            cplx kr = cmul(k1, rv[0]) + cmul(k2, rv[1]) + cmul(k3, rv[2]);
            kr = mk(fk * kr.x, fk * kr.y);
            rv[0] = inv * rv[0] - cmul(conjg(k1), kr);
            rv[1] = inv * rv[1] - cmul(conjg(k2), kr);
            rv[2] = inv * rv[2] - cmul(conjg(k3), kr);
            if (zero0) rv[0] = rv[1] = rv[2] = mk(0, 0);
            cplx* w = yo.base[4] + (long long)c * yo.ld + mi;
#pragma unroll
            for (int s = 0; s < 3; s++) w[(long long)s * n3] = rv[s];
          }
        }
      }
    }
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
  for (int c = tid; c < r; c += UT_THREADS) {
    const int nt = c / 8, i = nt / NG, g = nt % NG;
    const int ln = (c % 8) / 2, e = c % 2;
    double a = 0, b = 0;
    for (int q = 0; q < 2; q++) {  // the two row-group warps of n-tile group g, fixed order
      a += red[2 * g + q][i][ln][e][0];
      b += red[2 * g + q][i][ln][e][1];
    }
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 0] = a;
    partial[((long long)c * gridDim.x + blockIdx.x) * 2 + 1] = b;
  }
}

// ---- host side ------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool encode_slot(CUtensorMap* m, const cplx* base, int ncol_slot, long long ld, int n3, int box_cols) {
  if (!g_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[4] = {16, (cuuint64_t)n3 / 8, 3, (cuuint64_t)ncol_slot};
  const cuuint64_t strides[3] = {128, (cuuint64_t)n3 * 16, (cuuint64_t)ld * 16};
  const cuuint32_t box[4] = {16, 2, 3, (cuuint32_t)box_cols};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<cplx*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool update_tmap_supported(int n, int b) { return n % 2 == 0 && b <= 32; }

template <int NT>
static int run_update_tmap(const UtMaps& mp, const cplx* C, int ldc, int r, const UtOut& yo, const double* lam, int n, const cplx* kt, double gamma, double thr, int deflate0,
                           double* partial, int max_grid, cudaStream_t st) {
  const int PS = ((mp.pe + 3) & ~7) + 4;
  const size_t smem = 1024 + (size_t)UT_STAGES * mp.pe * UT_COLB + (size_t)NT * 8 * PS * sizeof(cplx);
  auto kern = update_tmap_kernel<NT>;
  smem_attr((const void*)kern, 200 * 1024);
  int occ = 0;
  constexpr int UT_THREADS = UtGeom<NT>::THREADS;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, UT_THREADS, smem);
  occ = std::max(1, std::min(8, occ));
  const long long n3 = (long long)n * n * n;
  const long long ntiles = (n3 + UT_SEG - 1) / UT_SEG;
  const int grid = (int)std::min<long long>(std::min<long long>(ntiles, (long long)grid_cap(occ)), max_grid);
  kern<<<grid, UT_THREADS, smem, st>>>(mp, C, ldc, r, yo, lam, n, kt, gamma, thr, deflate0, partial);
  return grid;
}

int launch_update_tmap(const UtBlocks& blk, const cplx* C, int ldc, int r, const MutColPtrs& Y1s,
                       const MutColPtrs& Y2s, const MutColPtrs& Y1a, const MutColPtrs& Y2a, const MutColPtrs& W,
                       const double* lam, int n, const cplx* kt, double gamma, double thr, int deflate0,
                       double* partial, int max_grid, cudaStream_t st) {
  const int n3 = n * n * n;
  UtMaps mp;
  memset(&mp, 0, sizeof(mp));
  for (int i = 0; i < 80; i++) mp.crow[i] = -1;
  int col = 0;
  for (int k = 0; k < 3; k++) {
    mp.off[k] = col;
    mp.c0[k] = blk.c0[k];
    mp.nc[k] = blk.nc[k];
    if (blk.nc[k] > 0) {
      if (!encode_slot(&mp.m[k], blk.s[k], blk.slot_cols[k], blk.ld, n3, blk.nc[k]) ||
          !encode_slot(&mp.m[3 + k], blk.as[k], blk.slot_cols[k], blk.ld, n3, blk.nc[k]))
        return -1;
      for (int j = 0; j < blk.nc[k]; j++) mp.crow[col + j] = blk.crow[k][j];
    }
    col += (blk.nc[k] + PC_UT_ALIGN - 1) / PC_UT_ALIGN * PC_UT_ALIGN;
    // the X block ends on a DMMA k-step (4 columns): phase 1 runs k over [split, pe) for P' and phase 2
    // over [0, split) for X C_X, so no k-step may straddle the split (W and P may start at any even column)
    if (k == 0) mp.split = col = (col + 3) & ~3;
  }
  mp.pe = std::max((col + 3) & ~3, 4);
  if (mp.pe > 80 || r > 32) return -1;
  UtOut yo;
  yo.ld = blk.ld;
  const MutColPtrs* outs[5] = {&Y1s, &Y2s, &Y1a, &Y2a, &W};
  for (int o = 0; o < 5; o++) {
    yo.mask[o] = 0;
    yo.base[o] = nullptr;
    for (int c = 0; c < r; c++) {
      cplx* q = outs[o]->p[c];
      if (!q) continue;
      if (!yo.base[o]) yo.base[o] = q - (long long)c * blk.ld;
      else if (q != yo.base[o] + (long long)c * blk.ld) return -1;  // not a strided column set
      yo.mask[o] |= 1u << c;
    }
    if (!yo.base[o]) yo.base[o] = outs[1]->p[0];  // unused (mask 0)
  }
  if (r <= 8) return run_update_tmap<1>(mp, C, ldc, r, yo, lam, n, kt, gamma, thr, deflate0,
                                        partial, max_grid, st);
  if (r <= 16) return run_update_tmap<2>(mp, C, ldc, r, yo, lam, n, kt, gamma, thr, deflate0,
                                         partial, max_grid, st);
  if (r <= 24) return run_update_tmap<3>(mp, C, ldc, r, yo, lam, n, kt, gamma, thr, deflate0,
                                         partial, max_grid, st);
  return run_update_tmap<4>(mp, C, ldc, r, yo, lam, n, kt, gamma, thr, deflate0, partial,
                            max_grid, st);
}
