// Small in-register DFT codelets, complex FP64.
//
//   Dft<R, DIR>::run(v):  v[k] <- sum_j v[j] W^{jk},  W = exp(DIR * 2 pi i / R)
//
// DIR = -1 is the e^{-} transform (F^H, numpy "fft"), DIR = +1 the e^{+} transform (F, numpy
// "ifft" without the 1/N), matching F_ij = w^{(i-1)(j-1)}, w = exp(+2 pi i/N) of PAPER.md:274.
// Composite sizes use the in-register four-step split R = P*Q with compile-time twiddles
// (tools/gen_twiddles.py), so trivial rotations (1, -1, +-i) cost no multiplies.
#pragma once
#include <type_traits>
#include "common.cuh"
#include "twiddles_gen.h"

template <int I, int N, class F>
DEV void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// v * W_R^E, W_R = exp(DIR 2 pi i / R)
template <int R, int E, int DIR>
DEV cplx twmul(cplx v) {
  constexpr int e = ((E % R) + R) % R;
  if constexpr (e == 0) {
    return v;
  } else if constexpr (2 * e == R) {
    return -v;
  } else if constexpr (4 * e == R) {
    return mul_i<DIR>(v);
  } else if constexpr (4 * e == 3 * R) {
    return mul_i<-DIR>(v);
  } else {
    constexpr double c = TwR<R>::c[e];
    constexpr double s = DIR * TwR<R>::s[e];
    return mk(fma(c, v.x, -s * v.y), fma(s, v.x, c * v.y));
  }
}

template <int R, int DIR>
struct Dft;

template <int DIR>
struct Dft<1, DIR> {
  static DEV void run(cplx*) {}
};

template <int DIR>
struct Dft<2, DIR> {
  static DEV void run(cplx* v) {
    cplx a = v[0] + v[1], b = v[0] - v[1];
    v[0] = a;
    v[1] = b;
  }
};

template <int DIR>
struct Dft<3, DIR> {
  static DEV void run(cplx* v) {
    constexpr double h = 0.8660254037844386;  // sin(2 pi/3)
    cplx t1 = v[1] + v[2];
    cplx t2 = mk(fma(-0.5, t1.x, v[0].x), fma(-0.5, t1.y, v[0].y));
    cplx d = v[1] - v[2];
    cplx t3 = mul_i<DIR>(mk(h * d.x, h * d.y));
    v[0] = v[0] + t1;
    v[1] = t2 + t3;
    v[2] = t2 - t3;
  }
};

template <int DIR>
struct Dft<4, DIR> {
  static DEV void run(cplx* v) {
    cplx a0 = v[0] + v[2], a1 = v[0] - v[2];
    cplx b0 = v[1] + v[3], b1 = mul_i<DIR>(v[1] - v[3]);
    v[0] = a0 + b0;
    v[2] = a0 - b0;
    v[1] = a1 + b1;
    v[3] = a1 - b1;
  }
};

// 5-point: direct evaluation with compile-time constants (used only for N with a factor 5).
template <int DIR>
struct Dft<5, DIR> {
  static DEV void run(cplx* v) {
    cplx o[5];
    static_for<0, 5>([&](auto K) {
      constexpr int k = decltype(K)::value;
      cplx acc = v[0];
      static_for<1, 5>([&](auto J) {
        constexpr int j = decltype(J)::value;
        acc = acc + twmul<5, j * k, DIR>(v[j]);
      });
      o[k] = acc;
    });
#pragma unroll
    for (int k = 0; k < 5; k++) v[k] = o[k];
  }
};

// Four-step split R = P * Q in registers:
//   X[k1 + P k2] = sum_{j2} W_Q^{j2 k2} W_R^{j2 k1} sum_{j1} x[j2 + Q j1] W_P^{j1 k1}
template <int P, int Q, int DIR>
DEV void dft_split(cplx* v) {
  constexpr int R = P * Q;
  cplx t[R];
  static_for<0, Q>([&](auto J2) {
    constexpr int j2 = decltype(J2)::value;
    cplx a[P];
#pragma unroll
    for (int j1 = 0; j1 < P; j1++) a[j1] = v[j2 + Q * j1];
    Dft<P, DIR>::run(a);
    static_for<0, P>([&](auto K1) {
      constexpr int k1 = decltype(K1)::value;
      t[j2 * P + k1] = twmul<R, j2 * k1, DIR>(a[k1]);
    });
  });
#pragma unroll
  for (int k1 = 0; k1 < P; k1++) {
    cplx c[Q];
#pragma unroll
    for (int j2 = 0; j2 < Q; j2++) c[j2] = t[j2 * P + k1];
    Dft<Q, DIR>::run(c);
#pragma unroll
    for (int k2 = 0; k2 < Q; k2++) v[k1 + P * k2] = c[k2];
  }
}

#define PC_SPLIT_DFT(R_, P_, Q_)                                      \
  template <int DIR>                                                  \
  struct Dft<R_, DIR> {                                               \
    static DEV void run(cplx* v) { dft_split<P_, Q_, DIR>(v); }       \
  };
PC_SPLIT_DFT(6, 2, 3)
PC_SPLIT_DFT(8, 2, 4)
PC_SPLIT_DFT(10, 2, 5)
PC_SPLIT_DFT(12, 4, 3)
PC_SPLIT_DFT(15, 3, 5)
PC_SPLIT_DFT(16, 4, 4)
#undef PC_SPLIT_DFT
