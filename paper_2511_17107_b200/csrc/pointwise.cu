// Pointwise / stencil kernels of libpcband:
//   * Fourier symbol tables for Dhat_i         (Lemma 2.1, reading R3)
//   * K_P^{-1} preconditioner                    (reading R7)
//   * real-space M_eps stencil                   (readings R4/R5)
//   * LOBPCG residual R = AX - X Lambda, Res_j norms fused with K_P^{-1}
//   * counter-based Gaussian start block, deterministic column reductions
#include "kernels.h"

// ------------------------------------------------------------------------------------------
// Symbol tables: ktab[(3 i + a) N + m] = b_ai lambda_1(m) + [a == i] i k_i lambda_0(m)
//   lambda_1(m) = (1 - W^m)/h, lambda_0(m) = (1 + W^m)/2, W = exp(-2 pi i/N)
// (eigenvalues of D_1, D_0 from their first rows by Lemma 2.1 with w = exp(+2 pi i/N)).
// kappa_i(m) = sum_a ktab[(3 i + a) N + m_a].
// ------------------------------------------------------------------------------------------
__global__ void ktab_kernel(cplx* ktab, const cplx* tw, int n, Sym3 s) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 9 * n) return;
  int m = idx % n, a = (idx / n) % 3, i = idx / (3 * n);
  cplx w = tw[m];
  cplx l1 = mk((double)n * (1.0 - w.x), (double)n * (-w.y));
  cplx l0 = mk(0.5 * (1.0 + w.x), 0.5 * w.y);
  double b = s.B[3 * a + i];  // b_ai = (A^{-1})_{ai}
  cplx v = mk(b * l1.x, b * l1.y);
  if (a == i) v = v + mk(-s.k[i] * l0.y, s.k[i] * l0.x);
  ktab[idx] = v;
}

void launch_ktab(cplx* ktab, const cplx* tw, int n, const Sym3& s, cudaStream_t st) {
  int tot = 9 * n;
  ktab_kernel<<<(tot + 127) / 128, 128, 0, st>>>(ktab, tw, n, s);
}

#include "kp.cuh"  // kappa_at, kp_inv

__global__ void precond_kernel(ColPtrs in, MutColPtrs out, int n, const cplx* __restrict__ kt0, double gamma,
                               double thr, MultiK mk) {
  const int col = blockIdx.y;
  const cplx* kt = kt0;
  if (mk.on) {  // per-column k (multi-k launch)
    kt = kt0 + (size_t)mk.kcol[col] * 9 * n;
    gamma = mk.gamma[mk.kcol[col]];
    thr = mk.thr[mk.kcol[col]];
  }
  const cplx* R = in.p[col];
  cplx* P = out.p[col];
  const int n3 = n * n * n;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n3; idx += gridDim.x * blockDim.x) {
    int m1 = idx % n, m2 = (idx / n) % n, m3 = idx / (n * n);
    cplx k1, k2, k3;
    kappa_at(kt, n, m1, m2, m3, k1, k2, k3);
    cplx r1 = ldg(R + idx), r2 = ldg(R + n3 + idx), r3 = ldg(R + 2 * n3 + idx);
    kp_inv(k1, k2, k3, gamma, thr, r1, r2, r3);
    P[idx] = r1;
    P[n3 + idx] = r2;
    P[2 * n3 + idx] = r3;
  }
}

void launch_precond(const ColPtrs& in, const MutColPtrs& out, int ncols, int n, const cplx* kt, double gamma,
                    double thr, cudaStream_t st, const MultiK* mk) {
  long long n3 = (long long)n * n * n;
  int gx = (int)std::min<long long>((n3 + 255) / 256, 148LL * 8);
  MultiK m;
  if (mk) m = *mk;
  precond_kernel<<<dim3(gx, ncols), 256, 0, st>>>(in, out, n, kt, gamma, thr, m);
}

// ------------------------------------------------------------------------------------------
// M_eps stencil (real space), one thread per grid point, all three components.
//   w_i = v_i + (eps_ii - 1) I_i v_i + off-diagonal terms:
//   CROSSDOF: eps_ij S_ij v_j with S_ij = (I_i T_ij + T_ij I_j)/2 written out as
//     (S_12 v2)(p) = 1/8 sum_{a in {-1,0}, b in {0,1}} (I1(p) + I2(q)) v2(q),  q = p + (a, b, 0)
//     (S_13 v3)(p) = 1/8 sum_{a in {-1,0}, c in {0,1}} (I1(p) + I3(q)) v3(q),  q = p + (a, 0, c)
//     (S_23 v3)(p) = 1/8 sum_{b in {-1,0}, c in {0,1}} (I2(p) + I3(q)) v3(q),  q = p + (0, b, c)
//   and the transposes with mirrored offsets, e.g.
//     (S_12^T v1)(p) = 1/8 sum_{a in {0,1}, b in {-1,0}} (I1(q) + I2(p)) v1(q).
//   TRIVIAL: eps_ij I_V(p) v_j(p).
// Mask byte per point: bit0 I1, bit1 I2, bit2 I3, bit3 I_V.
// ------------------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(256) eps_kernel(ColPtrs in, MutColPtrs out, int n, const uint8_t* __restrict__ mask,
                                                  EpsCoef ec) {
  const int col = blockIdx.y;
  const cplx* V = in.p[col];
  cplx* Wo = out.p[col];
  const int n3 = n * n * n;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n3; idx += gridDim.x * blockDim.x) {
    const int x = idx % n, y = (idx / n) % n, z = idx / (n * n);
    const int xm = (x == 0 ? n - 1 : x - 1), xp = (x == n - 1 ? 0 : x + 1);
    const int ym = (y == 0 ? n - 1 : y - 1), yp = (y == n - 1 ? 0 : y + 1);
    const int zm = (z == 0 ? n - 1 : z - 1), zp = (z == n - 1 ? 0 : z + 1);
    auto at = [&](int xx, int yy, int zz) { return (zz * n + yy) * n + xx; };
    const uint8_t mp = __ldg(mask + idx);
    const double i1 = (mp & 1) ? 1.0 : 0.0, i2 = (mp & 2) ? 1.0 : 0.0, i3 = (mp & 4) ? 1.0 : 0.0;
    cplx v1 = ldg(V + idx), v2 = ldg(V + n3 + idx), v3 = ldg(V + 2 * n3 + idx);
    cplx w1 = (1.0 + ec.d[0] * i1) * v1;
    cplx w2 = (1.0 + ec.d[1] * i2) * v2;
    cplx w3 = (1.0 + ec.d[2] * i3) * v3;
    if (MODE == 1) {  // CROSSDOF
      if (ec.has[0]) {  // eps_12: S_12 v2 into w1, S_12^T v1 into w2
        cplx acc = mk(0, 0);
        const int qs[4] = {at(xm, y, z), at(xm, yp, z), at(x, y, z), at(x, yp, z)};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          int q = qs[t];
          double wgt = i1 + ((__ldg(mask + q) & 2) ? 1.0 : 0.0);
          acc = acc + wgt * ldg(V + n3 + q);
        }
        w1 = w1 + 0.125 * cmul(ec.e[0], acc);
        cplx acc2 = mk(0, 0);
        const int qt[4] = {at(x, ym, z), at(x, y, z), at(xp, ym, z), at(xp, y, z)};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          int q = qt[t];
          double wgt = i2 + ((__ldg(mask + q) & 1) ? 1.0 : 0.0);
          acc2 = acc2 + wgt * ldg(V + q);
        }
        w2 = w2 + 0.125 * cmul(conjg(ec.e[0]), acc2);
      }
      if (ec.has[1]) {  // eps_13: S_13 v3 into w1, S_13^T v1 into w3
        cplx acc = mk(0, 0);
        const int qs[4] = {at(xm, y, z), at(xm, y, zp), at(x, y, z), at(x, y, zp)};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          int q = qs[t];
          double wgt = i1 + ((__ldg(mask + q) & 4) ? 1.0 : 0.0);
          acc = acc + wgt * ldg(V + 2 * n3 + q);
        }
        w1 = w1 + 0.125 * cmul(ec.e[1], acc);
        cplx acc2 = mk(0, 0);
        const int qt[4] = {at(x, y, zm), at(x, y, z), at(xp, y, zm), at(xp, y, z)};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          int q = qt[t];
          double wgt = i3 + ((__ldg(mask + q) & 1) ? 1.0 : 0.0);
          acc2 = acc2 + wgt * ldg(V + q);
        }
        w3 = w3 + 0.125 * cmul(conjg(ec.e[1]), acc2);
      }
      if (ec.has[2]) {  // eps_23: S_23 v3 into w2, S_23^T v2 into w3
        cplx acc = mk(0, 0);
        const int qs[4] = {at(x, ym, z), at(x, ym, zp), at(x, y, z), at(x, y, zp)};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          int q = qs[t];
          double wgt = i2 + ((__ldg(mask + q) & 4) ? 1.0 : 0.0);
          acc = acc + wgt * ldg(V + 2 * n3 + q);
        }
        w2 = w2 + 0.125 * cmul(ec.e[2], acc);
        cplx acc2 = mk(0, 0);
        const int qt[4] = {at(x, y, zm), at(x, y, z), at(x, yp, zm), at(x, yp, z)};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          int q = qt[t];
          double wgt = i3 + ((__ldg(mask + q) & 2) ? 1.0 : 0.0);
          acc2 = acc2 + wgt * ldg(V + n3 + q);
        }
        w3 = w3 + 0.125 * cmul(conjg(ec.e[2]), acc2);
      }
    } else if (MODE == 2) {  // TRIVIAL
      if (mp & 8) {
        w1 = w1 + cmul(ec.e[0], v2) + cmul(ec.e[1], v3);
        w2 = w2 + cmul(conjg(ec.e[0]), v1) + cmul(ec.e[2], v3);
        w3 = w3 + cmul(conjg(ec.e[1]), v1) + cmul(conjg(ec.e[2]), v2);
      }
    }
    Wo[idx] = w1;
    Wo[n3 + idx] = w2;
    Wo[2 * n3 + idx] = w3;
  }
}

void launch_eps(int mode, const ColPtrs& in, const MutColPtrs& out, int ncols, int n, const uint8_t* mask,
                const EpsCoef& ec, cudaStream_t st) {
  long long n3 = (long long)n * n * n;
  int gx = (int)std::min<long long>((n3 + 255) / 256, 148LL * 8);
  dim3 g(gx, ncols);
  if (mode == 1) eps_kernel<1><<<g, 256, 0, st>>>(in, out, n, mask, ec);
  else if (mode == 2) eps_kernel<2><<<g, 256, 0, st>>>(in, out, n, mask, ec);
  else eps_kernel<0><<<g, 256, 0, st>>>(in, out, n, mask, ec);
}

// ------------------------------------------------------------------------------------------
// LOBPCG residual: for column j < b:  R = AX_j - lambda_j X_j;  W_j = K_P^{-1} R
// (mode 0 zeroed when deflating the k = 0 null space); partial sums of |R|^2 and |X|^2 per CTA.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) resid_kernel(ColPtrs X, ColPtrs AX, MutColPtrs W, const double* __restrict__ lam,
                                                    int n, const cplx* __restrict__ kt, double gamma, double thr,
                                                    int deflate0, double* partial) {
  const int j = blockIdx.y;
  const cplx* x = X.p[j];
  const cplx* ax = AX.p[j];
  cplx* w = W.p[j];
  const double l = lam[j];
  const int n3 = n * n * n;
  double rn = 0.0, xn = 0.0;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n3; idx += gridDim.x * blockDim.x) {
    int m1 = idx % n, m2 = (idx / n) % n, m3 = idx / (n * n);
    cplx x1 = ldg(x + idx), x2 = ldg(x + n3 + idx), x3 = ldg(x + 2 * n3 + idx);
    cplx r1 = ldg(ax + idx) - l * x1, r2 = ldg(ax + n3 + idx) - l * x2, r3 = ldg(ax + 2 * n3 + idx) - l * x3;
    rn += abs2(r1) + abs2(r2) + abs2(r3);
    xn += abs2(x1) + abs2(x2) + abs2(x3);
    if (w) {
      cplx k1, k2, k3;
      kappa_at(kt, n, m1, m2, m3, k1, k2, k3);
      kp_inv(k1, k2, k3, gamma, thr, r1, r2, r3);
      if (deflate0 && idx == 0) r1 = r2 = r3 = mk(0, 0);
      w[idx] = r1;
      w[n3 + idx] = r2;
      w[2 * n3 + idx] = r3;
    }
  }
  // deterministic block reduction
  __shared__ double sr[256], sx[256];
  sr[threadIdx.x] = rn;
  sx[threadIdx.x] = xn;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sr[threadIdx.x] += sr[threadIdx.x + s];
      sx[threadIdx.x] += sx[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[(j * gridDim.x + blockIdx.x) * 2 + 0] = sr[0];
    partial[(j * gridDim.x + blockIdx.x) * 2 + 1] = sx[0];
  }
}

// out[j*2 + t] = sum_b partial[(j*nb + b)*2 + t]  (fixed order)
__global__ void reduce_partial_kernel(const double* partial, int nb, int ncols, double* out) {
  int j = blockIdx.x;
  __shared__ double s0[256], s1[256];
  double a = 0, c = 0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    a += partial[(j * nb + b) * 2 + 0];
    c += partial[(j * nb + b) * 2 + 1];
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = c;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s0[threadIdx.x] += s0[threadIdx.x + s];
      s1[threadIdx.x] += s1[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[j * 2 + 0] = s0[0];
    out[j * 2 + 1] = s1[0];
  }
}

int resid_grid(int n) {
  long long n3 = (long long)n * n * n;
  return (int)std::min<long long>((n3 + 255) / 256, 148LL * 4);
}

void launch_resid(const ColPtrs& X, const ColPtrs& AX, const MutColPtrs& W, const double* lam, int b, int n,
                  const cplx* kt, double gamma, double thr, int deflate0, double* partial, double* norms,
                  cudaStream_t st) {
  int gx = resid_grid(n);
  resid_kernel<<<dim3(gx, b), 256, 0, st>>>(X, AX, W, lam, n, kt, gamma, thr, deflate0, partial);
  reduce_partial_kernel<<<b, 256, 0, st>>>(partial, gx, b, norms);
}

void launch_reduce_partial(const double* partial, int nb, int ncols, double* norms, cudaStream_t st) {
  reduce_partial_kernel<<<ncols, 256, 0, st>>>(partial, nb, ncols, norms);
}

// ------------------------------------------------------------------------------------------
// Start block: complex Gaussian from a counter-based generator (splitmix64 of (seed, column,
// index)) -- the same numbers for a k-point whatever GPU or rank solves it.
// ------------------------------------------------------------------------------------------
DEV unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void randn_kernel(MutColPtrs X, long long len, unsigned long long seed, int deflate_stride, double scale) {
  const int j = blockIdx.y;
  cplx* x = X.p[j];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long h1 = splitmix64(seed ^ splitmix64(((unsigned long long)j << 40) ^ (unsigned long long)i));
    unsigned long long h2 = splitmix64(h1);
    double u1 = ((h1 >> 11) + 1) * (1.0 / 9007199254740993.0);  // (0, 1]
    double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
    double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    cplx v = mk(scale * r * cs, scale * r * sn);
    if (deflate_stride > 0 && (i % deflate_stride) == 0) v = mk(0, 0);  // zero Fourier mode 0
    x[i] = v;
  }
}

void launch_randn(const MutColPtrs& X, int ncols, long long len, unsigned long long seed, int deflate_stride,
                  double scale, cudaStream_t st) {
  randn_kernel<<<dim3(148 * 4, ncols), 256, 0, st>>>(X, len, seed, deflate_stride, scale);
}

// ------------------------------------------------------------------------------------------
// Plane-wave start block support: the PW_T smallest |kappa(m)|^2 per CTA (the low-lying modes of
// K_P = K_A K_A^H + gamma K_B, whose transverse plane waves are the vacuum
// eigenvectors).  Modes with |kappa|^2 <= thr (the k = 0 null mode) are skipped.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kappa2_topk_kernel(const cplx* __restrict__ kt, int n, double thr,
                                                          double* outv, int* outi) {
  const int n3 = n * n * n;
  double v[PW_T];
  int id[PW_T];
#pragma unroll
  for (int t = 0; t < PW_T; t++) { v[t] = 1e300; id[t] = -1; }
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n3; idx += gridDim.x * blockDim.x) {
    int m1 = idx % n, m2 = (idx / n) % n, m3 = idx / (n * n);
    cplx k1, k2, k3;
    kappa_at(kt, n, m1, m2, m3, k1, k2, k3);
    double q = abs2(k1) + abs2(k2) + abs2(k3);
    if (q <= thr || !(q < v[PW_T - 1])) continue;
    // insertion into the sorted list (fully unrolled: registers, no local memory)
    double cv = q;
    int ci = idx;
#pragma unroll
    for (int t = 0; t < PW_T; t++) {
      if (cv < v[t]) {
        double tv = v[t]; int ti = id[t];
        v[t] = cv; id[t] = ci;
        cv = tv; ci = ti;
      }
    }
  }
  // block merge: PW_T rounds of argmin over the thread list heads
  __shared__ double sv[256];
  __shared__ int st[256];
  int head = 0;
  for (int r = 0; r < PW_T; r++) {
    double hv = 1e300;
#pragma unroll
    for (int t = 0; t < PW_T; t++)
      if (t == head) hv = v[t];
    sv[threadIdx.x] = hv;
    st[threadIdx.x] = threadIdx.x;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        double a = sv[threadIdx.x], b = sv[threadIdx.x + s];
        if (b < a || (b == a && st[threadIdx.x + s] < st[threadIdx.x])) {
          sv[threadIdx.x] = b;
          st[threadIdx.x] = st[threadIdx.x + s];
        }
      }
      __syncthreads();
    }
    const int win = st[0];
    const double wv = sv[0];
    if (threadIdx.x == win) {
      int wid = -1;
#pragma unroll
      for (int t = 0; t < PW_T; t++)
        if (t == head) wid = id[t];
      outv[blockIdx.x * PW_T + r] = wv;
      outi[blockIdx.x * PW_T + r] = wid;
      head++;
    }
    __syncthreads();
  }
}

int pw_grid() { return 148 * 2; }

void launch_kappa2_topk(const cplx* kt, int n, double thr, double* outv, int* outi, cudaStream_t st) {
  kappa2_topk_kernel<<<pw_grid(), 256, 0, st>>>(kt, n, thr, outv, outi);
}

// X[col][c * N^3 + mode] += val  for a short host-built list (plane-wave start vectors)
__global__ void pw_scatter_kernel(MutColPtrs X, const PwEntry* __restrict__ e, int ne, int n3) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ne) return;
  PwEntry q = e[t];
  cplx* x = X.p[q.col];
  for (int c = 0; c < 3; c++) {
    cplx v = x[(long long)c * n3 + q.mode];
    x[(long long)c * n3 + q.mode] = mk(v.x + q.v[2 * c], v.y + q.v[2 * c + 1]);
  }
}

void launch_pw_scatter(const MutColPtrs& X, const PwEntry* e, int ne, int n3, cudaStream_t st) {
  if (ne > 0) pw_scatter_kernel<<<(ne + 127) / 128, 128, 0, st>>>(X, e, ne, n3);
}
