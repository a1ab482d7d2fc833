// Per-mode Fourier symbols and the K_P^{-1} closed form, shared by the residual kernels.
//   kappa_i(m) = sum_a ktab[(3 i + a) N + m_a]            (Dhat_i symbols, reading R3)
//   K_P^{-1} r = r/|k|^2 - (gamma-1)/(gamma |k|^4) conj(k) (k^T r)   (pass-through
//   when |k|^2 <= thr, reading R7)
#pragma once
#include "common.cuh"

DEV void kappa_at(const cplx* __restrict__ kt, int n, int m1, int m2, int m3, cplx& k1, cplx& k2, cplx& k3) {
  k1 = ldg(kt + 0 * n + m1) + ldg(kt + 1 * n + m2) + ldg(kt + 2 * n + m3);
  k2 = ldg(kt + 3 * n + m1) + ldg(kt + 4 * n + m2) + ldg(kt + 5 * n + m3);
  k3 = ldg(kt + 6 * n + m1) + ldg(kt + 7 * n + m2) + ldg(kt + 8 * n + m3);
}

DEV void kp_inv(cplx k1, cplx k2, cplx k3, double gamma, double thr, cplx& r1, cplx& r2, cplx& r3) {
  double k2n = abs2(k1) + abs2(k2) + abs2(k3);
  if (k2n <= thr) return;
  double inv = 1.0 / k2n;
  cplx kr = cmul(k1, r1) + cmul(k2, r2) + cmul(k3, r3);
  double f = (gamma - 1.0) / (gamma * k2n * k2n);
  kr = mk(f * kr.x, f * kr.y);
  r1 = inv * r1 - cmul(conjg(k1), kr);
  r2 = inv * r2 - cmul(conjg(k2), kr);
  r3 = inv * r3 - cmul(conjg(k3), kr);
}
