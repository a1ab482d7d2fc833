// Fused xy-plane pass of pc_apply at N = 128 (the middle factor F_y F_x M_eps
// F_x^H F_y^H of Op in Fourier coordinates; M_eps of P:607-673, readings R4/R5) for media whose eps_1
// couples only E^1 and E^2 (eps_13 = eps_23 = 0, or Diagonal / Trivial mode): one HBM round trip
// replaces the y-inverse pass, the fused x/M_eps/x pass and the y-forward pass (3 round trips).
//
// One z-plane of one column (3 components x 128 x 128, 786 KB) is spread over a cluster of 8 CTAs
// (distributed shared memory):
//   1. CTA q loads the x-slab x in [16q, 16q+16) of all y  -> Ty[c][y][xl]       (256-B HBM runs)
//   2. y-inverse DFT of its 48 (c, xl) pencils in shared memory
//   3. cluster barrier; CTA q pulls the y-rows [16q-1, 16q+16] of all x from the 8 slabs (DSMEM)
//      -> Tx[c][r][x]: E^1 with the row above, E^2 with the row below (the S_12 halo), E^3 without
//   4. x-inverse DFT, M_eps stencil (real space), x-forward DFT of its 16 output rows
//   5. cluster barrier; CTA q pulls its x-slab of all y back from the 8 row blocks (DSMEM) -> Ty
//   6. y-forward DFT, written straight to HBM; cluster barrier (peers done reading this CTA).
// All DFTs are the unnormalised two-step Stockham 128 = 16 x 8 of xex.cuh (register codelets,
// twiddles exp(-2 pi i j / N) from a shared table).  HBM traffic: 96 B per point per column + the
// z-plane mask (1 B per point per plane and column).
//
// Measured (option plane_fuse, off by default): 3.14 ms for a 15-column block against 1.98 ms for
// the three passes it replaces.  The pass moves ~1.1 KB of shared memory per point (four two-step
// DFTs, the stencil's neighbour reads, two DSMEM transposes), as much as the three separate passes
// together, but with 214 KB of shared memory per CTA it runs one CTA per SM and its phases (HBM
// load, DFTs, DSMEM exchanges, HBM store) do not overlap across planes.
#include <cooperative_groups.h>
#include "kernels.h"
#include "xex.cuh"

namespace cg = cooperative_groups;

constexpr int PL_N = 128;
constexpr int PL_CL = 8;                 // CTAs per cluster (one z-plane)
constexpr int PL_XB = PL_N / PL_CL;      // x-slab width / y-rows per CTA (16)
constexpr int PL_NT = 512;
constexpr int PL_RX = PL_XB + 2;         // Tx rows per component: y0 - 1 .. y0 + 16
constexpr int PL_P = XRow<PL_N>::P;      // Tx row pitch (odd; mid layout of xex.cuh)
constexpr size_t PL_TY = (size_t)3 * PL_N * PL_XB;   // complex
constexpr size_t PL_TX = (size_t)3 * PL_RX * PL_P;   // complex
constexpr size_t PL_SMEM = (PL_TY + PL_TX + PL_N) * sizeof(cplx) + (size_t)PL_RX * PL_N;

// y-direction DFT (sign DIR) of the 48 (c, xl) pencils of Ty[c][y][xl], two-step Stockham:
// step 1 over j = j2 + 8 j1 (16-point DFTs + twiddles W^{j2 k1}) to the mid position k1 * 8 + j2,
// step 2 (8-point DFTs) to natural k = k1 + 16 k2, in place or (LAST) straight to the store lambda.
template <int DIR, class Store>
DEV void pl_ydft(cplx* Ty, const cplx* tw, Store store) {
  constexpr int N = PL_N, XB = PL_XB, R1 = FftPlan<N>::R1, R2 = FftPlan<N>::R2;
  static_assert(R1 * R2 == N && 3 * R2 * XB <= PL_NT && 3 * R1 * XB <= 2 * PL_NT, "plane pass shape");
  const int tid = threadIdx.x;
  {
    const int xl = tid % XB, j2 = (tid / XB) % R2, c = tid / (XB * R2);
    const bool act = tid < 3 * R2 * XB;
    cplx v[R1];
    if (act) {
#pragma unroll
      for (int j1 = 0; j1 < R1; j1++) v[j1] = Ty[(c * N + j2 + R2 * j1) * XB + xl];
      Dft<R1, DIR>::run(v);
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int k1 = 0; k1 < R1; k1++) {
        cplx w = tw[(j2 * k1) % N];
        if (DIR > 0) w.y = -w.y;
        Ty[(c * N + k1 * R2 + j2) * XB + xl] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], w);
      }
    }
    __syncthreads();
  }
  cplx v[2][R2];
#pragma unroll
  for (int rnd = 0; rnd < 2; rnd++) {
    const int it = tid + rnd * PL_NT;
    const int xl = it % XB, k1 = (it / XB) % R1, c = it / (XB * R1);
    if (it < 3 * R1 * XB) {
#pragma unroll
      for (int j2 = 0; j2 < R2; j2++) v[rnd][j2] = Ty[(c * N + k1 * R2 + j2) * XB + xl];
    }
  }
  __syncthreads();
#pragma unroll
  for (int rnd = 0; rnd < 2; rnd++) {
    const int it = tid + rnd * PL_NT;
    const int xl = it % XB, k1 = (it / XB) % R1, c = it / (XB * R1);
    if (it < 3 * R1 * XB) {
      Dft<R2, DIR>::run(v[rnd]);
#pragma unroll
      for (int k2 = 0; k2 < R2; k2++) store(c, k1 + R1 * k2, xl, v[rnd][k2]);
    }
  }
}

// MODE: 0 diagonal, 1 CrossDoF with only eps_12, 2 trivial (as xex_kernel)
template <int MODE>
__global__ void __cluster_dims__(PL_CL, 1, 1) __launch_bounds__(PL_NT, 1)
plane_kernel(ColPtrs in, MutColPtrs out, const uint8_t* __restrict__ mask, EpsCoef ec,
             const cplx* __restrict__ twg) {
  constexpr int N = PL_N, XB = PL_XB, RX = PL_RX, P = PL_P, NT = PL_NT;
  constexpr long long N3 = (long long)N * N * N;
  extern __shared__ __align__(16) unsigned char plsm[];
  cplx* Ty = reinterpret_cast<cplx*>(plsm);
  cplx* Tx = Ty + PL_TY;
  cplx* tw = Tx + PL_TX;
  uint8_t* mk8 = reinterpret_cast<uint8_t*>(tw + N);  // [r][x], r <-> y = y0 - 1 + r
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int z = blockIdx.x / PL_CL, col = blockIdx.y;
  const int x0 = q * XB, y0 = q * XB;
  const cplx* gin = in.p[col];
  cplx* gout = out.p[col];

  // 1. x-slab of all y, the plane's mask rows y0-1 .. y0+16, twiddles
  for (int e = tid; e < 3 * N * XB; e += NT) {
    const int xl = e % XB, y = (e / XB) % N, c = e / (XB * N);
    cp_async16(&Ty[e], gin + c * N3 + ((long long)z * N + y) * N + x0 + xl);
  }
  for (int e = tid; e < RX * (N / 16); e += NT) {
    const int j = (e % (N / 16)) * 16, r = e / (N / 16);
    const int y = (y0 - 1 + r + N) % N;
    cp_async16(&mk8[r * N + j], mask + ((long long)z * N + y) * N + j);
  }
  cp_async_commit();
  for (int j = tid; j < N; j += NT) tw[j] = ldg(twg + j);
  cp_async_wait<0>();
  __syncthreads();

  // 2. y-inverse DFT
  pl_ydft<+1>(Ty, tw, [&](int c, int k, int xl, cplx v) { Ty[(c * N + k) * XB + xl] = v; });
  cl.sync();

  // 3. rows from the 8 slabs: pencil -> (component, row r); MODE 1 keeps the S_12 halo rows
  constexpr int NPEN = (MODE == 1) ? 3 * XB + 2 : 3 * XB;
  auto pen_row = [](int pen) {  // Tx row index c * RX + r
    if (MODE == 1) {
      if (pen < XB + 1) return pen;                                // E^1: r = 0 .. 16
      if (pen < 2 * XB + 2) return RX + 1 + (pen - (XB + 1));       // E^2: r = 1 .. 17
      return 2 * RX + 1 + (pen - (2 * XB + 2));                     // E^3: r = 1 .. 16
    }
    return (pen / XB) * RX + 1 + pen % XB;
  };
  for (int e = tid; e < NPEN * N; e += NT) {
    const int pen = e / N, x = e % N;
    const int row = pen_row(pen);
    const int c = row / RX, r = row % RX;
    const int y = (y0 - 1 + r + N) % N;
    const cplx* peer = cl.map_shared_rank(Ty, x / XB);
    Tx[row * P + x] = peer[(c * N + y) * XB + x % XB];
  }
  __syncthreads();

  // 4a. x-inverse DFT of the held rows
  xrow_step1<N, +1>(Tx, tw, NPEN, [&](int pen, int j) { return Tx[pen_row(pen) * P + j]; }, pen_row, true);
  xrow_step2<N, +1>(Tx, NPEN, [&](int pen, int k, cplx v) { Tx[pen_row(pen) * P + k] = v; }, pen_row, true);
  __syncthreads();

  // 4b. M_eps on the 16 output rows (r = 1 .. 16), registers first (the stencil reads neighbours)
  constexpr int PPT = (N * XB + NT - 1) / NT;
  cplx w[PPT][3];
#pragma unroll
  for (int t = 0; t < PPT; t++) {
    const int e = tid + t * NT;
    const int x = e % N, r = 1 + e / N;
    const uint8_t mp = mk8[r * N + x];
    const double i1 = (mp & 1) ? 1.0 : 0.0, i2 = (mp & 2) ? 1.0 : 0.0, i3 = (mp & 4) ? 1.0 : 0.0;
    const cplx v1 = Tx[(0 * RX + r) * P + x], v2 = Tx[(1 * RX + r) * P + x], v3 = Tx[(2 * RX + r) * P + x];
    cplx w1 = (1.0 + ec.d[0] * i1) * v1, w2 = (1.0 + ec.d[1] * i2) * v2, w3 = (1.0 + ec.d[2] * i3) * v3;
    if (MODE == 1) {
      const int xm = (x == 0) ? N - 1 : x - 1, xp = (x == N - 1) ? 0 : x + 1;
      // S_12 v2 (into w1): q in {x-1, x} x {y, y+1}, weight I1(p) + I2(q)
      cplx acc = mk(0, 0);
      const int qx[2] = {xm, x};
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int bb = 0; bb < 2; bb++) {
          const int rr = r + bb, xx = qx[a];
          const double wgt = i1 + ((mk8[rr * N + xx] & 2) ? 1.0 : 0.0);
          acc = acc + wgt * Tx[(1 * RX + rr) * P + xx];
        }
      w1 = w1 + 0.125 * cmul(ec.e[0], acc);
      // S_12^T v1 (into w2): q in {x, x+1} x {y-1, y}, weight I1(q) + I2(p)
      cplx acc2 = mk(0, 0);
      const int qx2[2] = {x, xp};
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int bb = 0; bb < 2; bb++) {
          const int rr = r - 1 + bb, xx = qx2[a];
          const double wgt = i2 + ((mk8[rr * N + xx] & 1) ? 1.0 : 0.0);
          acc2 = acc2 + wgt * Tx[(0 * RX + rr) * P + xx];
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
    const int e = tid + t * NT;
    const int x = e % N, r = 1 + e / N;
#pragma unroll
    for (int c = 0; c < 3; c++) Tx[(c * RX + r) * P + x] = w[t][c];
  }
  __syncthreads();

  // 4c. x-forward DFT of the 48 output rows, in place
  auto orow = [](int pen) { return (pen / XB) * RX + 1 + pen % XB; };
  xrow_step1<N, -1>(Tx, tw, 3 * XB, [&](int pen, int j) { return Tx[orow(pen) * P + j]; }, orow, true);
  xrow_step2<N, -1>(Tx, 3 * XB, [&](int pen, int k, cplx v) { Tx[orow(pen) * P + k] = v; }, orow, true);
  cl.sync();  // every CTA: rows transformed, and done reading the others' Ty (step 3)

  // 5. x-slab of all y back from the 8 row blocks
  for (int e = tid; e < 3 * N * XB; e += NT) {
    const int xl = e % XB, y = (e / XB) % N, c = e / (XB * N);
    const cplx* peer = cl.map_shared_rank(Tx, y / XB);
    Ty[e] = peer[(c * RX + 1 + y % XB) * P + x0 + xl];
  }
  __syncthreads();

  // 6. y-forward DFT straight to HBM
  pl_ydft<-1>(Ty, tw, [&](int c, int k, int xl, cplx v) { gout[c * N3 + ((long long)z * N + k) * N + x0 + xl] = v; });
  cl.sync();  // the other CTAs have finished reading this CTA's Tx (step 5)
}

bool plane_supported(int n) { return n == PL_N; }

cudaError_t launch_plane(int n, int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, const uint8_t* mask,
                         const EpsCoef& ec, const cplx* tw, cudaStream_t st) {
  if (n != PL_N || mode < 0 || mode > 2) return cudaErrorInvalidValue;
  auto run = [&](auto kern) -> cudaError_t {
    cudaError_t e = smem_attr((const void*)kern, (int)PL_SMEM);
    if (e != cudaSuccess) return e;
    kern<<<dim3(PL_CL * PL_N, ncols), PL_NT, PL_SMEM, st>>>(in, out, mask, ec, tw);
    return cudaGetLastError();
  };
  if (mode == 1) return run(plane_kernel<1>);
  if (mode == 2) return run(plane_kernel<2>);
  return run(plane_kernel<0>);
}
