// Instantiation of the FFT pass kernels for one grid size N (compiled once per N with
// -DPC_FFT_N=<N>, see Makefile) -- keeps the per-file compile time small and parallel.
#include "fft_pass.cuh"

#ifndef PC_FFT_N
#error "compile with -DPC_FFT_N=<N>"
#endif
#define PC_CAT2(a, b) a##b
#define PC_CAT(a, b) PC_CAT2(a, b)

template <int AXIS, int DIR, int OP, int C>
static cudaError_t run_one(const ColPtrs& in, const MutColPtrs& out, const ColPtrs& xh, int ncols,
                           const PassArgs& a, cudaStream_t st) {
  constexpr int N = PC_FFT_N;
  using Cfg = TileCfg<N, C>;
  auto kern = fft_pass_kernel<N, AXIS, DIR, OP, C>;
  cudaError_t e = smem_attr((const void*)kern, (int)Cfg::SMEM);
  if (e != cudaSuccess) return e;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::NT, Cfg::SMEM);
    if (occ < 1) occ = 1;
  }
  const int nzp = (AXIS != 2 && a.nz > 0) ? a.nz : N;
  const int ntiles = (N / Cfg::TP) * nzp * (C == 3 ? ncols : 3 * ncols);
  const int grid = Cfg::STAGES > 1 ? std::min(ntiles, occ * 148) : ntiles;
  kern<<<grid, Cfg::NT, Cfg::SMEM, st>>>(in, out, xh, a, ntiles);
  return cudaGetLastError();
}

cudaError_t PC_CAT(fft_launch_, PC_FFT_N)(int axis, int dir, int kind, const ColPtrs& in, const MutColPtrs& out,
                                          const ColPtrs& xh, int ncols, const PassArgs& a, cudaStream_t st) {
  if (kind == 1) return run_one<2, +1, OP_KAH, 3>(in, out, xh, ncols, a, st);
  if (kind == 2) return run_one<2, -1, OP_KAG, 3>(in, out, xh, ncols, a, st);
  if (kind == 3) return run_one<2, -1, OP_KAGH, 3>(in, out, xh, ncols, a, st);
  if (dir < 0) {
    if (axis == 0) return run_one<0, -1, OP_NONE, 1>(in, out, xh, ncols, a, st);
    if (axis == 1) return run_one<1, -1, OP_NONE, 1>(in, out, xh, ncols, a, st);
    return run_one<2, -1, OP_NONE, 1>(in, out, xh, ncols, a, st);
  }
  if (axis == 0) return run_one<0, +1, OP_NONE, 1>(in, out, xh, ncols, a, st);
  if (axis == 1) return run_one<1, +1, OP_NONE, 1>(in, out, xh, ncols, a, st);
  return run_one<2, +1, OP_NONE, 1>(in, out, xh, ncols, a, st);
}

#include "xex.cuh"

template <int MODE>
static cudaError_t run_xex(const ColPtrs& in, const MutColPtrs& out, int ncols, const uint8_t* mask, const EpsCoef& ec,
                           const cplx* tw, double scale, int z0, int nz, cudaStream_t st) {
  constexpr int N = PC_FFT_N;
  using Cfg = XexCfg<N>;
  auto kern = xex_kernel<N, MODE>;
  cudaError_t e = smem_attr((const void*)kern, (int)Cfg::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid((N / Cfg::TP) * (nz > 0 ? nz : N), ncols);
  kern<<<grid, Cfg::NT, Cfg::SMEM, st>>>(in, out, mask, ec, tw, scale, nz > 0 ? z0 : 0);
  return cudaGetLastError();
}

cudaError_t PC_CAT(xex_launch_, PC_FFT_N)(int mode, const ColPtrs& in, const MutColPtrs& out, int ncols,
                                          const uint8_t* mask, const EpsCoef& ec, const cplx* tw, double scale,
                                          int z0, int nz, cudaStream_t st) {
  if (mode == 1) return run_xex<1>(in, out, ncols, mask, ec, tw, scale, z0, nz, st);
  if (mode == 2) return run_xex<2>(in, out, ncols, mask, ec, tw, scale, z0, nz, st);
  return run_xex<0>(in, out, ncols, mask, ec, tw, scale, z0, nz, st);
}
