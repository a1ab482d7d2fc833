// Fused xy-plane pass of pc_apply at N = 128, option plane_fuse = 1: one HBM round
// trip for the middle factor F_y F_x M_eps F_x^H F_y^H of Op in Fourier coordinates (
// M_eps of P:607-673, readings R4/R5) for media whose eps_1 couples only E^1 and E^2 (eps_13 = eps_23
// = 0, or Diagonal / Trivial mode).  Replaces the y-inverse pass, the fused x/M_eps/x pass and the
// y-forward pass (3 HBM round trips, 289 B per point per column) by one (97 B), so pc_apply moves
// 112 + 97 + 112 = 321 B per point per column (the §8(a) 3-pass floor is 336 B with x_hat re-read).
//
// One z-plane of one column (3 x 128 x 128 complex, 786 KB) is spread over a cluster of 16 CTAs of
// 108 KB shared memory each, so that two CTAs (of different planes) share an SM and one's HBM phases
// overlap the other's DFT phases (a round-1 8-CTA design with one 214-KB CTA per SM, its phases serialised,
// took 3.14 ms per 15 columns).  CTA q owns the x-slab x in [8q, 8q+8) and the y-rows [8q, 8q+8):
//   1. y-inverse DFT of its x-slab: the radix-16 first step reads HBM straight into registers (8 lanes
//      = one 128-B row segment), mid layout in Ty; the radix-8 second step PUSHES each output (c, y, x)
//      into the Tx row block of the CTA owning row y (distributed shared memory stores, 128-B runs),
//      plus the S_12 halo copies (E^1 of row y0-1, E^2 of row y0+8, MODE 1).
//   2. cluster barrier; x-inverse DFT of the 26 held rows, M_eps stencil (real space), x-forward DFT
//      whose second step pushes each output (c, y, x) into the Ty slab of the CTA owning column x.
//   3. cluster barrier; y-forward DFT, the second step writes HBM directly.
// No CTA reads another's shared memory: all exchange is by remote stores before a cluster barrier.
// Measured (C4, 15 columns): 2.67 ms against 1.93 ms for the y / xex / y passes it replaces; ncu: barrier
// stalls lead (3.8 per issue), 21 % warps active, FP64 pipe 22 %, DRAM 1.1 TB/s -- every CTA runs its
// load, DFT, exchange and store phases in sequence between two cluster barriers, and two CTAs per SM
// do not hide that.  Kept as the 3-pass candidate (option plane_fuse, default off).
// DFTs: 128 = 16 x 8 two-step Stockham with the register codelets of dft.cuh, twiddles from a
// transposed shared table (xex.cuh).  Unnormalised, as the passes it replaces.
#include <cooperative_groups.h>
#include "kernels.h"
#include "xex.cuh"

namespace cg = cooperative_groups;

namespace {
constexpr int N2 = 128;
constexpr int CL2 = 16;               // CTAs per cluster (one z-plane of one column)
constexpr int XB2 = N2 / CL2;         // x-slab width = y-rows per CTA (8)
constexpr int NT2 = 256;
constexpr int R1 = FftPlan<N2>::R1;   // 16
constexpr int R2 = FftPlan<N2>::R2;   // 8
constexpr int TXP = XRow<N2>::P;      // Tx row pitch (complex, odd; mid layout of xex.cuh)
// Tx rows: E^1 r = 0..8 (y0-1 .. y0+7), E^2 r = 0..8 (y0 .. y0+8), E^3 r = 0..7 (y0 .. y0+7)
constexpr int TXR = 26;
constexpr size_t TY_C = (size_t)3 * N2 * XB2;             // complex
constexpr size_t TX_C = (size_t)TXR * TXP;                // complex
constexpr int MKR = XB2 + 2;                              // mask rows y0-1 .. y0+8
constexpr size_t SMEM2 = (TY_C + TX_C + N2) * sizeof(cplx) + (size_t)MKR * N2;
static_assert(R1 == 16 && R2 == 8, "plane2 assumes 128 = 16 x 8");

DEV int rowc(int c) { return 9 * c; }  // first Tx row of component c
DEV int txrow(int c, int y, int y0) {  // Tx row of (component, global y) in the CTA owning y0
  return rowc(c) + (y - y0) + (c == 0 ? 1 : 0);
}
}  // namespace

template <int MODE>
__global__ void __launch_bounds__(NT2, 2)
plane2_kernel(ColPtrs in, MutColPtrs out, const uint8_t* __restrict__ mask, EpsCoef ec, const cplx* __restrict__ twg) {
  constexpr long long N3 = (long long)N2 * N2 * N2;
  extern __shared__ __align__(16) unsigned char p2sm[];
  cplx* Ty = reinterpret_cast<cplx*>(p2sm);       // [c][y][xl], y natural or mid
  cplx* Tx = Ty + TY_C;                            // [row][x]
  cplx* tw = Tx + TX_C;                            // transposed twiddles tw[k1 * R2 + j2]
  uint8_t* mk8 = reinterpret_cast<uint8_t*>(tw + N2);  // [r][x], r <-> y = y0 - 1 + r
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int z = blockIdx.x / CL2, col = blockIdx.y;
  const int x0 = q * XB2, y0 = q * XB2;
  const cplx* gin = in.p[col];
  cplx* gout = out.p[col];

  xrow_twiddles<N2>(tw, twg);
  for (int e = tid; e < MKR * (N2 / 16); e += NT2) {
    const int j = (e % (N2 / 16)) * 16, r = e / (N2 / 16);
    const int y = (y0 - 1 + r + N2) % N2;
    cp_async16(&mk8[r * N2 + j], mask + ((long long)z * N2 + y) * N2 + j);
  }
  cp_async_commit();
  __syncthreads();  // twiddle table complete before step 1 reads it

  // y-direction item of step 1: (c, xl, j2), xl fastest (8 lanes = one 128-B row segment)
  const int xl = tid % XB2, j2 = (tid / XB2) % R2, cc = tid / (XB2 * R2);  // 192 active threads
  const bool act1 = tid < 3 * XB2 * R2;

  // ---- 1. y-inverse DFT, step 1 straight from HBM
  if (act1) {
    cplx v[R1];
    const cplx* src = gin + cc * N3 + ((long long)z * N2) * N2 + x0 + xl;
#pragma unroll
    for (int j1 = 0; j1 < R1; j1++) v[j1] = ldg(src + (long long)(j2 + R2 * j1) * N2);
    Dft<R1, +1>::run(v);
#pragma unroll
    for (int k1 = 0; k1 < R1; k1++) {
      cplx wt = tw[k1 * R2 + j2];
      wt.y = -wt.y;
      Ty[(cc * N2 + k1 * R2 + j2) * XB2 + xl] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], wt);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // step 2: items (c, xl, k1); outputs y = k1 + 16 k2 pushed to the owner of row y
#pragma unroll
  for (int rnd = 0; rnd < 2; rnd++) {
    const int it = tid + rnd * NT2;
    if (it >= 3 * XB2 * R1) break;
    const int ixl = it % XB2, k1 = (it / XB2) % R1, c = it / (XB2 * R1);
    cplx v[R2];
#pragma unroll
    for (int jj = 0; jj < R2; jj++) v[jj] = Ty[(c * N2 + k1 * R2 + jj) * XB2 + ixl];
    Dft<R2, +1>::run(v);
#pragma unroll
    for (int k2 = 0; k2 < R2; k2++) {
      const int y = k1 + R1 * k2, d = y / XB2, yo = d * XB2;
      cplx* rt = cl.map_shared_rank(Tx, d);
      rt[txrow(c, y, yo) * TXP + x0 + ixl] = v[k2];
      if (MODE == 1) {
        if (c == 0 && (y % XB2) == XB2 - 1) {  // E^1 halo row y0-1 of the next row block
          cplx* rn = cl.map_shared_rank(Tx, (d + 1) % CL2);
          rn[(rowc(0) + 0) * TXP + x0 + ixl] = v[k2];
        }
        if (c == 1 && (y % XB2) == 0) {        // E^2 halo row y0+8 of the previous row block
          cplx* rp = cl.map_shared_rank(Tx, (d + CL2 - 1) % CL2);
          rp[(rowc(1) + XB2) * TXP + x0 + ixl] = v[k2];
        }
      }
    }
  }
  cl.sync();  // all row blocks complete; every Ty is free again

  // ---- 2. x-inverse DFT of the held rows (in place), M_eps, x-forward DFT pushed to the slab owners
  constexpr int NPEN = (MODE == 1) ? TXR : 3 * XB2;
  auto prow = [](int pen) {  // pencil -> Tx row (MODE != 1: only the 8 output rows per component)
    if (MODE == 1) return pen;
    const int c = pen / XB2;
    return rowc(c) + (c == 0 ? 1 : 0) + pen % XB2;
  };
  {
    auto ld = [&](int pen, int j) { return Tx[prow(pen) * TXP + j]; };
    xrow_step1<N2, +1, decltype(ld), decltype(prow), true>(Tx, tw, NPEN, ld, prow, true);
    xrow_step2<N2, +1>(Tx, NPEN, [&](int pen, int k, cplx v) { Tx[prow(pen) * TXP + k] = v; }, prow, true);
  }
  __syncthreads();
  constexpr int PPT = N2 * XB2 / NT2;  // 4 stencil points per thread and component
  cplx w[PPT][3];
#pragma unroll
  for (int t = 0; t < PPT; t++) {
    const int e = tid + t * NT2;
    const int x = e % N2, r = e / N2;   // output row y = y0 + r; mask row r + 1
    const uint8_t mp = mk8[(r + 1) * N2 + x];
    const double i1 = (mp & 1) ? 1.0 : 0.0, i2 = (mp & 2) ? 1.0 : 0.0, i3 = (mp & 4) ? 1.0 : 0.0;
    const cplx v1 = Tx[(rowc(0) + 1 + r) * TXP + x], v2 = Tx[(rowc(1) + r) * TXP + x],
               v3 = Tx[(rowc(2) + r) * TXP + x];
    cplx w1 = (1.0 + ec.d[0] * i1) * v1, w2 = (1.0 + ec.d[1] * i2) * v2, w3 = (1.0 + ec.d[2] * i3) * v3;
    if (MODE == 1) {
      const int xm = (x == 0) ? N2 - 1 : x - 1, xp = (x == N2 - 1) ? 0 : x + 1;
      // S_12 v2 (into w1): q in {x-1, x} x {y, y+1}, weight I1(p) + I2(q)
      cplx acc = mk(0, 0);
      const int qx[2] = {xm, x};
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int bb = 0; bb < 2; bb++) {
          const int xx = qx[a];
          const double wgt = i1 + ((mk8[(r + 1 + bb) * N2 + xx] & 2) ? 1.0 : 0.0);
          acc = acc + wgt * Tx[(rowc(1) + r + bb) * TXP + xx];
        }
      w1 = w1 + 0.125 * cmul(ec.e[0], acc);
      // S_12^T v1 (into w2): q in {x, x+1} x {y-1, y}, weight I1(q) + I2(p)
      cplx acc2 = mk(0, 0);
      const int qx2[2] = {x, xp};
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int bb = 0; bb < 2; bb++) {
          const int xx = qx2[a];
          const double wgt = i2 + ((mk8[(r + bb) * N2 + xx] & 1) ? 1.0 : 0.0);
          acc2 = acc2 + wgt * Tx[(rowc(0) + r + bb) * TXP + xx];
        }
      w2 = w2 + 0.125 * cmul(conjg(ec.e[0]), acc2);
    } else if (MODE == 2) {
      if (mp & 8) {
        w1 = w1 + cmul(ec.e[0], v2) + cmul(ec.e[1], v3);
        w2 = w2 + cmul(conjg(ec.e[0]), v1) + cmul(ec.e[2], v3);
        w3 = w3 + cmul(conjg(ec.e[1]), v1) + cmul(conjg(ec.e[2]), v2);
      }
    }
    w[t][0] = w1;
    w[t][1] = w2;
    w[t][2] = w3;
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < PPT; t++) {
    const int e = tid + t * NT2;
    const int x = e % N2, r = e / N2;
    Tx[(rowc(0) + 1 + r) * TXP + x] = w[t][0];
    Tx[(rowc(1) + r) * TXP + x] = w[t][1];
    Tx[(rowc(2) + r) * TXP + x] = w[t][2];
  }
  __syncthreads();
  {
    auto orow = [](int pen) {  // output pencil (c, r) -> Tx row
      const int c = pen / XB2;
      return rowc(c) + (c == 0 ? 1 : 0) + pen % XB2;
    };
    auto ld = [&](int pen, int j) { return Tx[orow(pen) * TXP + j]; };
    xrow_step1<N2, -1, decltype(ld), decltype(orow), true>(Tx, tw, 3 * XB2, ld, orow, true);
    xrow_step2<N2, -1>(Tx, 3 * XB2, [&](int pen, int k, cplx v) {
      const int c = pen / XB2, r = pen % XB2;
      cplx* rt = cl.map_shared_rank(Ty, k / XB2);
      rt[(c * N2 + y0 + r) * XB2 + (k % XB2)] = v;
    }, orow, false);
  }
  cl.sync();  // all x-slabs complete

  // ---- 3. y-forward DFT of the x-slab, straight to HBM
  cplx v[R1];
  if (act1) {
#pragma unroll
    for (int j1 = 0; j1 < R1; j1++) v[j1] = Ty[(cc * N2 + j2 + R2 * j1) * XB2 + xl];
    Dft<R1, -1>::run(v);
  }
  __syncthreads();
  if (act1) {
#pragma unroll
    for (int k1 = 0; k1 < R1; k1++) {
      const cplx wt = tw[k1 * R2 + j2];
      Ty[(cc * N2 + k1 * R2 + j2) * XB2 + xl] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], wt);
    }
  }
  __syncthreads();
#pragma unroll
  for (int rnd = 0; rnd < 2; rnd++) {
    const int it = tid + rnd * NT2;
    if (it >= 3 * XB2 * R1) break;
    const int ixl = it % XB2, k1 = (it / XB2) % R1, c = it / (XB2 * R1);
    cplx u[R2];
#pragma unroll
    for (int jj = 0; jj < R2; jj++) u[jj] = Ty[(c * N2 + k1 * R2 + jj) * XB2 + ixl];
    Dft<R2, -1>::run(u);
#pragma unroll
    for (int k2 = 0; k2 < R2; k2++)
      gout[c * N3 + ((long long)z * N2 + k1 + R1 * k2) * N2 + x0 + ixl] = u[k2];
  }
}

bool plane2_supported(int n) { return n == N2; }

cudaError_t launch_plane2(int n, int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, const uint8_t* mask,
                          const EpsCoef& ec, const cplx* tw, cudaStream_t st) {
  if (n != N2 || mode < 0 || mode > 2) return cudaErrorInvalidValue;
  auto run = [&](auto kern) -> cudaError_t {
    cudaError_t e = smem_attr((const void*)kern, (int)SMEM2);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL2 * N2, ncols);
    cfg.blockDim = dim3(NT2);
    cfg.dynamicSmemBytes = SMEM2;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, in, out, mask, ec, tw);
  };
  if (mode == 1) return run(plane2_kernel<1>);
  if (mode == 2) return run(plane2_kernel<2>);
  return run(plane2_kernel<0>);
}
