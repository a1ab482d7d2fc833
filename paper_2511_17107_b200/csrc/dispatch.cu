// Runtime dispatch of FFT passes over the compiled grid sizes.
#include "kernels.h"
#include "fft_sizes.h"

#define PC_DECL(N)                                                                                        \
  cudaError_t fft_launch_##N(int axis, int dir, int kind, const ColPtrs& in, const MutColPtrs& out,       \
                             const ColPtrs& xh, int ncols, const PassArgsH& a, cudaStream_t st);
PC_FFT_SIZES(PC_DECL)
#undef PC_DECL
#define PC_DECL2(N)                                                                                       \
  cudaError_t xex_launch_##N(int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, const uint8_t* mask, \
                             const EpsCoef& ec, const cplx* tw, double scale, int z0, int nz, cudaStream_t st);
PC_FFT_SIZES(PC_DECL2)
#undef PC_DECL2

int fft_supported(int n) {
#define PC_CASE(N) if (n == N) return 1;
  PC_FFT_SIZES(PC_CASE)
#undef PC_CASE
  return 0;
}

int fft_supported_list(int* sizes, int cap) {
  int cnt = 0;
#define PC_ADD(N) { if (sizes && cnt < cap) sizes[cnt] = N; cnt++; }
  PC_FFT_SIZES(PC_ADD)
#undef PC_ADD
  return cnt;
}

cudaError_t launch_fft_pass(int n, int axis, int dir, int kind, const ColPtrs& in, const MutColPtrs& out,
                            const ColPtrs& xh, int ncols, const PassArgsH& a, cudaStream_t st) {
  switch (n) {
#define PC_SW(N) case N: return fft_launch_##N(axis, dir, kind, in, out, xh, ncols, a, st);
    PC_FFT_SIZES(PC_SW)
#undef PC_SW
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_xex(int n, int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, const uint8_t* mask,
                       const EpsCoef& ec, const cplx* tw, double scale, int z0, int nz, cudaStream_t st) {
  switch (n) {
#define PC_SW2(N) case N: return xex_launch_##N(mode, in, out, ncols, mask, ec, tw, scale, z0, nz, st);
    PC_FFT_SIZES(PC_SW2)
#undef PC_SW2
    default: return cudaErrorInvalidValue;
  }
}
