// LOBPCG Gram blocks Gp = S^H T, S = [X W P], T = [W P AW AP] (the Rayleigh-Ritz projections,
// PAPER.md:1055-1056), with the row chunks streamed by TMA tensor copies (option gram_tmap, off).
//
// The five blocks X, W, P, AW, AP are column ranges of LOBPCG slots (b columns, stride ld).  One
// chunk of KC rows of all of them lands in shared memory as [column][KC rows], so S = columns
// [0, oAW) and T = columns [oW, end) of the same buffer: W and P are loaded once for both operands
// (gram.cu loads them twice).  Blocks start at even columns (128-B tensor-copy alignment).
// Measured (n = 128, 35 x 40 blocks, tools/bench_block.py): 2.37 ms at KC = 32 against 2.25 ms for
// gram.cu.  The [column][row] layout a tensor copy produces cannot be conflict-free for the DMMA
// fragments (two columns x four rows per quarter warp) unless the column pitch is 4 mod 8 complex
// (KC = 12, 20, 28), and those chunks are not 128-B aligned in HBM (KC = 20: 2.74 ms).
// Complex products: three real DMMAs per complex MAC (see gram.cu).  CTA = one 40 x 8*NT output
// block, KS*NT warps: warp (n-tile wn, row group kg) owns the 5 m-tiles of n-tile wn and the k-steps
// kg, kg + KS, ... of each chunk; the row groups are folded in a fixed order at the end, CTA
// partials are reduced in a fixed order by gt_reduce_kernel (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>
#include "kernels.h"
#include "dmma.cuh"
#include "tma.cuh"

#ifndef PC_GT_KC
#define PC_GT_KC 32
#endif
#ifndef PC_GT_KS
#define PC_GT_KS 2
#endif
constexpr int GT_KC = PC_GT_KC;              // complex rows per chunk
constexpr int GT_KS = PC_GT_KS;              // warp groups splitting the k-steps of a chunk
constexpr int GT_COLB = GT_KC * 16;          // bytes per column of a stage (320)
constexpr int GT_MT = 5;                     // m-tiles (S columns 0..39)
constexpr int GT_MAXC = 64;                  // buffer columns
#ifndef PC_GT_STAGES
#define PC_GT_STAGES 3
#endif
constexpr int GT_STAGES = PC_GT_STAGES;

struct GtMaps {
  CUtensorMap m[5];  // X, W, P, AW, AP slots
  int c0[5], nc[5], off[5];
  int ncol;          // buffer columns per stage (>= every column a fragment reads)
  int oT;            // first T column (= off[1])
};

DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <int NT>
__global__ void __launch_bounds__(32 * GT_KS * NT) gram_tmap_kernel(const __grid_constant__ GtMaps mp, long long len,
                                                            long long rows_per_split, double* __restrict__ partial) {
  constexpr int NTH = 32 * GT_KS * NT;
  extern __shared__ __align__(128) unsigned char gtsm_raw[];
  double* Ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(gtsm_raw) + 127) & ~(uintptr_t)127);
  __shared__ __align__(8) unsigned long long full[GT_STAGES];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wn = warp % NT, kg = warp / NT;
  const int ncol = mp.ncol;
  const int stage_d = ncol * (GT_COLB / 8);  // doubles per stage
  const long long r0 = (long long)blockIdx.x * rows_per_split;
  const long long r1 = min(len, r0 + rows_per_split);
  const int nchunks = (r1 > r0) ? (int)((r1 - r0 + GT_KC - 1) / GT_KC) : 0;

  // columns no block writes (padding) enter only discarded outputs; zero them anyway (finite data)
  for (int st = 0; st < GT_STAGES; st++)
    for (int e = tid; e < stage_d; e += NTH) {
      const int col = e / (GT_COLB / 8);
      bool pad = true;
#pragma unroll
      for (int k = 0; k < 5; k++)
        if (col >= mp.off[k] && col < mp.off[k] + mp.nc[k]) pad = false;
      if (pad) Ring[st * stage_d + e] = 0.0;
    }
  unsigned txb = 0;
#pragma unroll
  for (int k = 0; k < 5; k++) txb += (unsigned)mp.nc[k] * GT_COLB;
  if (tid == 0)
    for (int st = 0; st < GT_STAGES; st++) mbar_init(&full[st], 1);
  fence_proxy_async();
  __syncthreads();
  auto issue = [&](int ch) {
    const int st = ch % GT_STAGES;
    double* dst = Ring + st * stage_d;
    mbar_arrive_expect_tx(&full[st], txb);
    const int row2 = (int)(2 * (r0 + (long long)ch * GT_KC));
#pragma unroll
    for (int k = 0; k < 5; k++)
      if (mp.nc[k] > 0) tma_load_2d(dst + mp.off[k] * (GT_COLB / 8), &mp.m[k], row2, mp.c0[k], &full[st]);
  };
  if (tid == 0)
    for (int ch = 0; ch < GT_STAGES && ch < nchunks; ch++) issue(ch);

  double p1[GT_MT][2], p2[GT_MT][2], p3[GT_MT][2];
#pragma unroll
  for (int i = 0; i < GT_MT; i++) p1[i][0] = p1[i][1] = p2[i][0] = p2[i][1] = p3[i][0] = p3[i][1] = 0.0;
  const int bcol = mp.oT + wn * 8 + (lane >> 2);  // this lane's T column (B fragment n index)

  for (int ch = 0; ch < nchunks; ch++) {
    const int st = ch % GT_STAGES;
    mbar_wait(&full[st], (unsigned)((ch / GT_STAGES) & 1));
    const double* Sb = Ring + st * stage_d;
#pragma unroll
    for (int s4 = kg; s4 < GT_KC / 4; s4 += GT_KS) {
      const int kk = 2 * (4 * s4 + (lane & 3));  // interleaved doubles of complex row 4 s4 + (lane & 3)
      const double2 bv = *reinterpret_cast<const double2*>(Sb + bcol * (GT_COLB / 8) + kk);
      const double bs = bv.x + bv.y;
#pragma unroll
      for (int mt = 0; mt < GT_MT; mt++) {
        const double2 av = *reinterpret_cast<const double2*>(Sb + (mt * 8 + (lane >> 2)) * (GT_COLB / 8) + kk);
        dmma(p1[mt][0], p1[mt][1], av.x, bv.x);
        dmma(p2[mt][0], p2[mt][1], av.y, bv.y);
        dmma(p3[mt][0], p3[mt][1], av.x - av.y, bs);
      }
    }
    __syncthreads();  // stage st consumed by every warp
    if (tid == 0 && ch + GT_STAGES < nchunks) {
      fence_proxy_async();
      issue(ch + GT_STAGES);
    }
  }

  // fold row group 1 into row group 0 (fixed order), then write this CTA's 40 x 8 NT partial
  double* red = Ring;  // the ring is free now
  __syncthreads();
  if (GT_KS > 1 && kg == 1) {
    double* dst = red + ((size_t)wn * 32 + lane) * (GT_MT * 6);
#pragma unroll
    for (int mt = 0; mt < GT_MT; mt++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        dst[mt * 6 + e * 3 + 0] = p1[mt][e];
        dst[mt * 6 + e * 3 + 1] = p2[mt][e];
        dst[mt * 6 + e * 3 + 2] = p3[mt][e];
      }
  }
  __syncthreads();
  if (kg != 0) return;
  const double* src = red + ((size_t)wn * 32 + lane) * (GT_MT * 6);
  double* out = partial + (size_t)blockIdx.x * (GT_MT * 8) * (NT * 8) * 2;
#pragma unroll
  for (int mt = 0; mt < GT_MT; mt++)
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const double a1 = p1[mt][e] + (GT_KS > 1 ? src[mt * 6 + e * 3 + 0] : 0.0);
      const double a2 = p2[mt][e] + (GT_KS > 1 ? src[mt * 6 + e * 3 + 1] : 0.0);
      const double a3 = p3[mt][e] + (GT_KS > 1 ? src[mt * 6 + e * 3 + 2] : 0.0);
      const int m = mt * 8 + (lane >> 2), n = wn * 8 + 2 * (lane & 3) + e;
      out[((size_t)n * (GT_MT * 8) + m) * 2 + 0] = a1 + a2;
      out[((size_t)n * (GT_MT * 8) + m) * 2 + 1] = a3 - a1 + a2;
    }
}

// Sum of the CTA partials (fixed order) into Gp (p x q, column-major): Gp[tq][sp] = sum partial[n][m]
// with m = srow[sp] (buffer S column), n = tcol[tq] (buffer T column - oT).
struct GtIdx {
  signed char srow[80], tcol[80];
};
__global__ void gt_reduce_kernel(const double* __restrict__ partial, int nsplit, int ldm, int ldn, GtIdx ix, int p,
                                 int q, cplx* G) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p * q) return;
  const int sp = idx % p, tq = idx / p;
  const int m = ix.srow[sp], n = ix.tcol[tq];
  double re = 0.0, im = 0.0;
  const size_t blk = (size_t)ldm * ldn * 2;
  for (int s = 0; s < nsplit; s++) {
    const double* pp = partial + s * blk + ((size_t)n * ldm + m) * 2;
    re += pp[0];
    im += pp[1];
  }
  G[idx] = mk(re, im);
}

// ---- host side ------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode2 = nullptr;

static bool gt_encode(CUtensorMap* m, const cplx* base, int ncol_slot, long long ld, long long len, int box_cols) {
  if (!g_encode2) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    g_encode2 = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)(2 * len), (cuuint64_t)ncol_slot};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 16};
  const cuuint32_t box[2] = {2 * GT_KC, (cuuint32_t)box_cols};
  const cuuint32_t es[2] = {1, 1};
  return g_encode2(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<cplx*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t gram_tmap_partial_bytes() { return (size_t)4 * 148 * 40 * 40 * 16 + 4096; }

template <int NT>
static void run_gram_tmap(const GtMaps& mp, long long len, double* partial, const GtIdx& ix, int p, int q, cplx* G,
                          cudaStream_t st) {
  const size_t smem = 128 + (size_t)GT_STAGES * mp.ncol * GT_COLB;
  auto kern = gram_tmap_kernel<NT>;
  static int ctas_per_sm = 0;
  if (!ctas_per_sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, kern, 32 * GT_KS * NT, smem);
    ctas_per_sm = std::max(1, std::min(4, ctas_per_sm));
  }
  int ns = grid_cap(ctas_per_sm);
  ns = (int)std::max(1LL, std::min<long long>(ns, (len + 4 * GT_KC - 1) / (4 * GT_KC)));
  long long rps = (len + ns - 1) / ns;
  rps = (rps + GT_KC - 1) / GT_KC * GT_KC;
  ns = (int)((len + rps - 1) / rps);
  kern<<<ns, 32 * GT_KS * NT, smem, st>>>(mp, len, rps, partial);
  gt_reduce_kernel<<<(p * q + 127) / 128, 128, 0, st>>>(partial, ns, GT_MT * 8, NT * 8, ix, p, q, G);
}

int launch_gram_tmap(const GtBlocks& blk, long long len, cplx* G, cplx* partial, cudaStream_t st) {
  GtMaps mp;
  memset(&mp, 0, sizeof(mp));
  GtIdx ix;
  memset(&ix, -1, sizeof(ix));
  int col = 0;
  for (int k = 0; k < 5; k++) {
    mp.off[k] = col;
    mp.c0[k] = blk.c0[k];
    mp.nc[k] = blk.nc[k];
    if (blk.nc[k] > 0 && !gt_encode(&mp.m[k], blk.base[k], blk.slot_cols[k], blk.ld, len, blk.nc[k])) return -1;
    col += (blk.nc[k] + 1) & ~1;
  }
  mp.oT = mp.off[1];
  const int scount = mp.off[3];         // S = [X W P] buffer columns
  const int tcount = col - mp.oT;       // T = [W P AW AP] buffer columns
  const int ntile = (tcount + 7) / 8;
  mp.ncol = std::max(std::max(col, GT_MT * 8), mp.oT + 8 * ntile);
  if (scount > GT_MT * 8 || tcount > 40 || mp.ncol > GT_MAXC) return -1;
  // logical index maps: S rows (X 0..b-1, W b.., P ..) and T columns (W, P, AW, AP)
  int p = 0, q = 0;
  for (int k = 0; k < 3; k++)
    for (int j = 0; j < blk.nc[k]; j++)
      if (blk.lidx[k][j] >= 0) {
        ix.srow[blk.lidx[k][j]] = (signed char)(mp.off[k] + j);
        p = std::max(p, blk.lidx[k][j] + 1);
      }
  for (int k = 1; k < 5; k++)
    for (int j = 0; j < blk.nc[k]; j++)
      if (blk.tidx[k][j] >= 0) {
        ix.tcol[blk.tidx[k][j]] = (signed char)(mp.off[k] + j - mp.oT);
        q = std::max(q, blk.tidx[k][j] + 1);
      }
  if (p > 80 || q > 80) return -1;
  double* part = reinterpret_cast<double*>(partial);
  switch (ntile) {
    case 1: run_gram_tmap<1>(mp, len, part, ix, p, q, G, st); break;
    case 2: run_gram_tmap<2>(mp, len, part, ix, p, q, G, st); break;
    case 3: run_gram_tmap<3>(mp, len, part, ix, p, q, G, st); break;
    case 4: run_gram_tmap<4>(mp, len, part, ix, p, q, G, st); break;
    default: run_gram_tmap<5>(mp, len, part, ix, p, q, G, st); break;
  }
  return 0;
}
