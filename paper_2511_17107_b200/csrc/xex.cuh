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

// Row pencils of length N = R1 * R2 (two-step Stockham).  Shared rows have pitch P (odd).  Two index
// layouts inside a row: "natural" j (0..N-1) and "mid" j2 * S1 + k1 (after the first step: R2 DFTs of
// size R1 over j = j2 + R2 j1, twiddled), S1 = R1 rounded up to odd, so that lanes with consecutive j2
// (first step) and lanes with consecutive k1 (second step) both hit distinct banks.
template <int N>
struct XRow {
  static constexpr int R1 = FftPlan<N>::R1, R2 = FftPlan<N>::R2;
  static constexpr int S1 = (R1 % 2 == 0) ? R1 + 1 : R1;
  static constexpr int L = ((R2 - 1) * S1 + R1 > N) ? (R2 - 1) * S1 + R1 : N;
  static constexpr int P = (L % 2 == 1) ? L : L + 1;
};

// Tile shape: N <= 128: 4 output rows, 128 threads, 4 CTAs/SM; larger N: 8 rows, 256 threads, 2 CTAs/SM.
// (At n = 128 the 4 x 128 shape was slower while the pass was shared-memory bound; after the round-2
// shared-memory cuts it is 10 % faster, profiles/r02_experiments/xex_shape_after_cuts.txt.)  The
// PC_XEX_TP / PC_XEX_NT / PC_XEX_MINB macros override for every N (variant builds).
template <int N>
struct XexCfg {
#ifdef PC_XEX_TP
  static constexpr int TP = pow2_div(N, PC_XEX_TP);   // output rows per tile
#else
  static constexpr int TP = pow2_div(N, N <= 128 ? 4 : 8);
#endif
  static constexpr int RP = TP + 2;           // rows held (1 halo row each side)
  static constexpr int P = XRow<N>::P;        // row pitch in complex
#ifdef PC_XEX_NT
  static constexpr int NT = PC_XEX_NT;
#else
  static constexpr int NT = N <= 128 ? 128 : 256;
#endif
#ifdef PC_XEX_MINB
  static constexpr int MINB = PC_XEX_MINB;
#else
  static constexpr int MINB = N <= 128 ? 4 : 2;
#endif
  static constexpr int PPT = (N * TP + NT - 1) / NT;  // stencil points per thread
  static constexpr size_t SMEM = (size_t)3 * RP * P * sizeof(cplx) + (size_t)N * sizeof(cplx) + (size_t)RP * N;
};

// First Stockham step for npen rows: R2 DFTs of size R1 (input stride R2) + twiddles, result in the
// mid layout of the row.  Input element j of pencil pen comes from load(pen, j) (global or shared).
// Thread item = (pen, j2) with j2 fastest: R2 lanes read R2 consecutive inputs of one pencil.
// TT: tw is the transposed table tw[k1 R2 + j2] = W_N^{j2 k1} (xrow_twiddles), so that the R2 lanes of
// one pencil read consecutive twiddles (the natural table tw[(j2 k1) % N] is a stride-k1 read: up to
// 8-way bank conflicts on the 16-B loads).
template <int N>
DEV void xrow_twiddles(cplx* tw, const cplx* __restrict__ twg) {
  constexpr int R2 = XRow<N>::R2;
  for (int j = threadIdx.x; j < N; j += blockDim.x) tw[j] = ldg(twg + ((j % R2) * (j / R2)) % N);
}

#ifndef PC_XEX_TWREC
#define PC_XEX_TWREC 1
#endif
template <int N, int DIR, class Load, class Row, bool TT = false>
DEV void xrow_step1(cplx* s, const cplx* tw, int npen, Load load, Row row, bool sync_inplace) {
  using X = XRow<N>;
  constexpr int R1 = X::R1, R2 = X::R2, S1 = X::S1, P = X::P;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = nt / R2;  // pencils per round
  for (int p0 = 0; p0 < npen; p0 += per) {
    const int pen = p0 + tid / R2, j2 = tid % R2;
    const bool act = (tid < per * R2) && pen < npen;
    cplx v[R1];
    if (act) {
#pragma unroll
      for (int j1 = 0; j1 < R1; j1++) v[j1] = load(pen, j2 + R2 * j1);
      Dft<R1, DIR>::run(v);
    }
    if (sync_inplace) __syncthreads();
    if (act) {
      cplx* d = s + row(pen) * P + j2 * S1;
      if constexpr (TT && PC_XEX_TWREC && R1 % 4 == 0 && R1 >= 8) {
        // twiddles W^{j2 k1}, k1 = 4a + b, from two table reads (W^{j2}, W^{4 j2}) and at most 3 + R1/4
        // products (<= 4 roundings each): the 16-B twiddle reads were as many shared-memory wavefronts
        // as the data of this step
        cplx w1 = tw[1 * R2 + j2], w4 = tw[4 * R2 + j2];
        if (DIR > 0) {
          w1.y = -w1.y;
          w4.y = -w4.y;
        }
        const cplx w2 = cmul(w1, w1), w3 = cmul(w2, w1);
        cplx wa = mk(1.0, 0.0);
#pragma unroll
        for (int a = 0; a < R1 / 4; a++) {
          if (a == 1) wa = w4;
          if (a > 1) wa = cmul(wa, w4);
#pragma unroll
          for (int b = 0; b < 4; b++) {
            const int k1 = 4 * a + b;
            cplx w = (b == 0) ? wa : (b == 1) ? w1 : (b == 2) ? w2 : w3;
            if (a > 0 && b > 0) w = cmul(wa, w);
            d[k1] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], w);
          }
        }
      } else {
#pragma unroll
        for (int k1 = 0; k1 < R1; k1++) {
          cplx w = TT ? tw[k1 * R2 + j2] : tw[(j2 * k1) % N];
          if (DIR > 0) w.y = -w.y;
          d[k1] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], w);
        }
      }
    }
    if (sync_inplace) __syncthreads();
  }
}

// Second step: R1 DFTs of size R2 from the mid layout; output k = k1 + R1 k2 goes to store(pen, k, v).
// Thread item = (pen, k1) with k1 fastest.  sync_inplace: the store writes the same shared rows.
template <int N, int DIR, class Store, class Row>
DEV void xrow_step2(const cplx* s, int npen, Store store, Row row, bool sync_inplace) {
  using X = XRow<N>;
  constexpr int R1 = X::R1, R2 = X::R2, S1 = X::S1, P = X::P;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = nt / R1;
  for (int p0 = 0; p0 < npen; p0 += per) {
    const int pen = p0 + tid / R1, k1 = tid % R1;
    const bool act = (tid < per * R1) && pen < npen;
    cplx v[R2];
    if (act) {
      const cplx* src = s + row(pen) * P + k1;
#pragma unroll
      for (int j2 = 0; j2 < R2; j2++) v[j2] = src[j2 * S1];
      Dft<R2, DIR>::run(v);
    }
    if (sync_inplace) __syncthreads();
    if (act) {
#pragma unroll
      for (int k2 = 0; k2 < R2; k2++) store(pen, k1 + R1 * k2, v[k2]);
    }
    if (sync_inplace) __syncthreads();
  }
}

// MODE: 0 diagonal, 1 crossdof with only eps_12, 2 trivial
#ifndef PC_XEX_COLS
#define PC_XEX_COLS 1
#endif
template <int N, int MODE>
__global__ void __launch_bounds__(XexCfg<N>::NT, XexCfg<N>::MINB)
xex_kernel(ColPtrs in, MutColPtrs out, const uint8_t* __restrict__ mask, EpsCoef ec, const cplx* __restrict__ twg,
           double scale, int zoff) {
  using Cfg = XexCfg<N>;
  constexpr int TP = Cfg::TP, RP = Cfg::RP, P = Cfg::P, NT = Cfg::NT, PPT = Cfg::PPT;
  constexpr int N3 = N * N * N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* s = reinterpret_cast<cplx*>(smem_raw);  // row (c*RP + r) at s + row * P
  cplx* tw = s + 3 * RP * P;
  uint8_t* mk8 = reinterpret_cast<uint8_t*>(tw + N);  // [row][x]
  const int tid = threadIdx.x;
  const int z = zoff + blockIdx.x / (N / TP), y0 = (blockIdx.x % (N / TP)) * TP;
  const int col = blockIdx.y;
  const cplx* gin = in.p[col];
  cplx* gout = out.p[col];

  // Rows held per component (smem row r <-> y = y0 - 1 + r, r = 0 .. TP+1).  Only S_12 needs the halo
  // rows (E^1 at y0-1, E^2 at y0+TP).  MODE 1 holds only the halo rows S_12 reads: E^1 rows r = 0..TP, E^2 rows r = 1..TP+1, E^3 rows
  // r = 1..TP (3 TP + 2 pencils instead of 3 TP + 6).
  constexpr int NPEN = (MODE == 1) ? 3 * TP + 2 : 3 * TP;
  auto prow = [](int pen) {
    if (MODE != 1) return (pen / TP) * RP + 1 + pen % TP;
    if (pen <= TP) return pen;
    if (pen <= 2 * TP + 1) return RP + (pen - TP);
    return 2 * RP + 1 + (pen - 2 * TP - 2);
  };
  auto grow = [&](int row) {  // global offset of smem row
    const int c = row / RP, r = row % RP;
    const int y = (y0 - 1 + r + N) % N;
    return (long long)c * N3 + ((long long)z * N + y) * N;
  };
  if constexpr (N % 16 == 0) {
    for (int e = tid; e < RP * (N / 16); e += NT) {
      const int j = (e % (N / 16)) * 16, r = e / (N / 16);
      const int y = (y0 - 1 + r + N) % N;
      cp_async16(&mk8[r * N + j], mask + ((long long)z * N + y) * N + j);
    }
    cp_async_commit();
  } else {
    for (int e = tid; e < RP * N; e += NT) {
      const int j = e % N, r = e / N;
      const int y = (y0 - 1 + r + N) % N;
      mk8[e] = __ldg(mask + ((long long)z * N + y) * N + j);
    }
  }
  xrow_twiddles<N>(tw, twg);
  __syncthreads();

  // inverse x-DFT of the held rows: first step straight from HBM (R2 lanes read R2 consecutive complex)
  auto gload = [&](int pen, int j) { return ldg(gin + grow(prow(pen)) + j); };
  xrow_step1<N, +1, decltype(gload), decltype(prow), true>(s, tw, NPEN, gload, prow, false);
  __syncthreads();
  xrow_step2<N, +1>(s, NPEN, [&](int pen, int k, cplx v) { s[prow(pen) * P + k] = v; }, prow, true);
  if constexpr (N % 16 == 0) cp_async_wait<0>();
  __syncthreads();

  // M_eps on the TP output rows (registers first: the stencil reads neighbours).  COLS: each thread
  // takes PPT consecutive rows of one x, so the rows its stencils share are read from shared memory once
  // (6 instead of 9 field reads per point in MODE 1).
  constexpr bool COLS = PC_XEX_COLS && NT % N == 0 && PPT * NT == N * TP;
  auto spt = [&](int t, int& x, int& r) {
    if (COLS) {
      x = tid % N;
      r = 1 + (tid / N) * PPT + t;
      return true;
    }
    const int e = tid + t * NT;
    x = e % N;
    r = 1 + e / N;
    return e < N * TP;
  };
  cplx w[PPT][3];
#pragma unroll
  for (int t = 0; t < PPT; t++) {
    int x, r;
    if (!spt(t, x, r)) break;
    const uint8_t mp = mk8[r * N + x];
    const double i1 = (mp & 1) ? 1.0 : 0.0, i2 = (mp & 2) ? 1.0 : 0.0, i3 = (mp & 4) ? 1.0 : 0.0;
    const cplx v1 = s[(0 * RP + r) * P + x], v2 = s[(1 * RP + r) * P + x], v3 = s[(2 * RP + r) * P + x];
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
          acc = acc + wgt * s[(1 * RP + rr) * P + xx];
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
          acc2 = acc2 + wgt * s[(0 * RP + rr) * P + xx];
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
    int x, r;
    if (!spt(t, x, r)) break;
#pragma unroll
    for (int c = 0; c < 3; c++) s[(c * RP + r) * P + x] = w[t][c];
  }
  __syncthreads();

  // forward x-DFT of the TP output rows; the last step writes HBM directly (R1 consecutive complex)
  auto orow = [](int pen) { return (pen / TP) * RP + 1 + pen % TP; };
  auto sload = [&](int pen, int j) { return s[orow(pen) * P + j]; };
  xrow_step1<N, -1, decltype(sload), decltype(orow), true>(s, tw, 3 * TP, sload, orow, true);
  xrow_step2<N, -1>(s, 3 * TP, [&](int pen, int k, cplx v) {
    const int c = pen / TP, r = pen % TP;
    gout[(long long)c * N3 + ((long long)z * N + y0 + r) * N + k] = v;
  }, orow, false);
}
