// Fused "x-inverse FFT + M_eps + x-forward FFT" pass of pc_apply (PAPER.md:523-529 middle factor
// F3^H M_eps F3, with M_eps of P:607-673) for media whose eps_1 couples only E^1 and E^2
// (eps_13 = eps_23 = 0: isotropic, diagonal, and the pseudochiral tensor of P:1083-1087), so that
// the CrossDoF stencil S_12 (readings R4/R5: (x-1|x) x (y|y+1) and (x|x+1) x (y-1|y) averages) is
// local to a z-plane.  A CTA owns TP consecutive y-rows of one z-plane for all three components plus
// one halo row on each side (only S_12 needs them), so the real-space field between the two x-passes
// never goes to HBM: the pass reads the y-transformed block once and writes the x-transformed
// M_eps-product once (96 B per point per column + 2 halo rows per TP).
#pragma once
#include "fft_pass.cuh"

// Two-step Stockham FFT of npen length-N pencils held in shared memory at addr(pencil, j).
// Step B runs in rounds of complete pencils so the in-place write never clobbers unread input.
template <int N, int DIR, class Addr>
DEV void smem_fft(cplx* s, const cplx* tw, int npen, Addr addr) {
  constexpr int R1 = FftPlan<N>::R1, R2 = FftPlan<N>::R2;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int it = tid; it < npen * R2; it += nt) {
    const int pen = it % npen, j2 = it / npen;
    cplx v[R1];
#pragma unroll
    for (int j1 = 0; j1 < R1; j1++) v[j1] = s[addr(pen, j2 + R2 * j1)];
    Dft<R1, DIR>::run(v);
#pragma unroll
    for (int k1 = 0; k1 < R1; k1++) {
      cplx w = tw[(j2 * k1) % N];
      if (DIR > 0) w.y = -w.y;
      s[addr(pen, j2 + R2 * k1)] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], w);
    }
  }
  __syncthreads();
  const int ppr = nt / R1 > 0 ? nt / R1 : 1;
  for (int p0 = 0; p0 < npen; p0 += ppr) {
    const int pen = p0 + tid % ppr, k1 = tid / ppr;
    const bool act = (tid < ppr * R1) && pen < npen;
    cplx v[R2];
    if (act) {
#pragma unroll
      for (int j2 = 0; j2 < R2; j2++) v[j2] = s[addr(pen, R2 * k1 + j2)];
      Dft<R2, DIR>::run(v);
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int k2 = 0; k2 < R2; k2++) s[addr(pen, k1 + R1 * k2)] = v[k2];
    }
    __syncthreads();
  }
}

template <int N>
struct XexCfg {
  static constexpr int TP = pow2_div(N, 8);   // output rows per tile
  static constexpr int RP = TP + 2;           // rows held (1 halo row each side)
  static constexpr int NP1 = N + 1;           // row pitch in complex (odd: conflict-free fragments)
  static constexpr int NT = 256;
  static constexpr int PPT = (N * TP + NT - 1) / NT;  // stencil points per thread
  static constexpr size_t SMEM = (size_t)3 * RP * NP1 * sizeof(cplx) + (size_t)N * sizeof(cplx) + (size_t)RP * N;
};

// MODE: 0 diagonal, 1 crossdof with only eps_12, 2 trivial
template <int N, int MODE>
__global__ void __launch_bounds__(XexCfg<N>::NT, 3)
xex_kernel(ColPtrs in, MutColPtrs out, const uint8_t* __restrict__ mask, EpsCoef ec, const cplx* __restrict__ twg,
           double scale, int zoff) {
  using Cfg = XexCfg<N>;
  constexpr int TP = Cfg::TP, RP = Cfg::RP, NP1 = Cfg::NP1, NT = Cfg::NT, PPT = Cfg::PPT;
  constexpr int N3 = N * N * N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* s = reinterpret_cast<cplx*>(smem_raw);  // [c][row][j] = (c*RP + row)*NP1 + j (rows as in HBM)
  cplx* tw = s + 3 * RP * NP1;
  uint8_t* mk8 = reinterpret_cast<uint8_t*>(tw + N);  // [row][x]
  const int tid = threadIdx.x;
  const int z = zoff + blockIdx.x / (N / TP), y0 = (blockIdx.x % (N / TP)) * TP;
  const int col = blockIdx.y;
  const cplx* gin = in.p[col];
  cplx* gout = out.p[col];

  // Rows held per component (smem row r <-> y = y0 - 1 + r): S_12^T v1 needs E^1 at y0-1 (r = 0),
  // S_12 v2 needs E^2 at y0+TP (r = TP+1); E^3 and the pointwise modes need only r = 1..TP.
  // pencil list: component 0 rows [lo0, lo0+n0), component 1 rows [1, 1+n1), component 2 rows [1, 1+TP)
  constexpr int n0 = (MODE == 1) ? TP + 1 : TP, lo0 = (MODE == 1) ? 0 : 1;
  constexpr int n1 = (MODE == 1) ? TP + 1 : TP;
  constexpr int NPEN = n0 + n1 + TP;
  auto pen_row = [&](int pen, int& c, int& r) {
    if (pen < n0) { c = 0; r = lo0 + pen; }
    else if (pen < n0 + n1) { c = 1; r = 1 + pen - n0; }
    else { c = 2; r = 1 + pen - n0 - n1; }
  };
  for (int e = tid; e < NPEN * N; e += NT) {
    const int j = e % N;
    int c, r;
    pen_row(e / N, c, r);
    const int y = (y0 - 1 + r + N) % N;
    cp_async16(&s[(c * RP + r) * NP1 + j], gin + (long long)c * N3 + ((long long)z * N + y) * N + j);
  }
  if constexpr (N % 16 == 0) {
    for (int e = tid; e < RP * (N / 16); e += NT) {
      const int j = (e % (N / 16)) * 16, r = e / (N / 16);
      const int y = (y0 - 1 + r + N) % N;
      cp_async16(&mk8[r * N + j], mask + ((long long)z * N + y) * N + j);
    }
  } else {
    for (int e = tid; e < RP * N; e += NT) {
      const int j = e % N, r = e / N;
      const int y = (y0 - 1 + r + N) % N;
      mk8[e] = __ldg(mask + ((long long)z * N + y) * N + j);
    }
  }
  cp_async_commit();
  for (int j = tid; j < N; j += NT) tw[j] = ldg(twg + j);
  cp_async_wait<0>();
  __syncthreads();

  // inverse x-DFT of the held rows
  smem_fft<N, +1>(s, tw, NPEN, [&](int pen, int j) {
    int c, r;
    pen_row(pen, c, r);
    return (c * RP + r) * NP1 + j;
  });

  // M_eps on the TP output rows (registers first: the stencil reads neighbours)
  cplx w[PPT][3];
#pragma unroll
  for (int t = 0; t < PPT; t++) {
    const int e = tid + t * NT;
    if (e >= N * TP) break;
    const int x = e % N, r = 1 + e / N;
    const uint8_t mp = mk8[r * N + x];
    const double i1 = (mp & 1) ? 1.0 : 0.0, i2 = (mp & 2) ? 1.0 : 0.0, i3 = (mp & 4) ? 1.0 : 0.0;
    const cplx v1 = s[(0 * RP + r) * NP1 + x], v2 = s[(1 * RP + r) * NP1 + x], v3 = s[(2 * RP + r) * NP1 + x];
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
          acc = acc + wgt * s[(1 * RP + rr) * NP1 + xx];
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
          acc2 = acc2 + wgt * s[(0 * RP + rr) * NP1 + xx];
        }
      w2 = w2 + 0.125 * cmul(conjg(ec.e[0]), acc2);
    } else if (MODE == 2) {
      if (mp & 8) {
        w1 = w1 + cmul(ec.e[0], v2) + cmul(ec.e[1], v3);
        w2 = w2 + cmul(conjg(ec.e[0]), v1) + cmul(ec.e[2], v3);
        w3 = w3 + cmul(conjg(ec.e[1]), v1) + cmul(conjg(ec.e[2]), v2);
      }
    }
    w[t][0] = scale * w1;
    w[t][1] = scale * w2;
    w[t][2] = scale * w3;
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < PPT; t++) {
    const int e = tid + t * NT;
    if (e >= N * TP) break;
    const int x = e % N, r = 1 + e / N;
#pragma unroll
    for (int c = 0; c < 3; c++) s[(c * RP + r) * NP1 + x] = w[t][c];
  }
  __syncthreads();

  // forward x-DFT of the TP output rows
  smem_fft<N, -1>(s, tw, 3 * TP, [&](int pen, int j) { return ((pen / TP) * RP + 1 + pen % TP) * NP1 + j; });

  for (int e = tid; e < 3 * TP * N; e += NT) {
    const int j = e % N, r = (e / N) % TP, c = e / (N * TP);
    gout[(long long)c * N3 + ((long long)z * N + y0 + r) * N + j] = s[(c * RP + 1 + r) * NP1 + j];
  }
}
