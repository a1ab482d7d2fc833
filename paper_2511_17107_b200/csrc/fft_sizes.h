// Grid sizes N with compiled FFT kernels (must match FftPlan in fft_pass.cuh and the Makefile).
#pragma once
#define PC_FFT_SIZES(X) X(4) X(6) X(8) X(10) X(12) X(16) X(20) X(24) X(32) X(40) X(48) X(64) X(80) X(96) \
  X(100) X(120) X(128) X(160) X(192) X(240) X(256)
