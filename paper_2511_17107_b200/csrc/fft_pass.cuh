// One pencil pass of the batched 3-component 3-D FFT (complex FP64), with the operator's
// Fourier-symbol work fused into the first / last pass of pc_apply.
//
// A CTA owns a tile of TP pencils of length N along AXIS (0 = x, 1 = y, 2 = z) for C components
// (C = 3 when the fused symbol op needs all field components of a mode).  The tile is staged
// HBM -> shared memory with cp.async (16 B per complex, coalesced: TP consecutive x for the y/z
// passes, TP whole rows for the x pass), transformed in shared memory by a two-step Stockham
// split N = R1 * R2 (register codelets + one twiddle stage), and written back coalesced.
//
// Shared layout SI(c, j, p): y/z passes [c][j][p] (pitch TP+1), x pass [c][p][j] (pitch N+1) so that the
// cp.async tile writes are contiguous like the HBM rows; odd pitches keep the FFT steps conflict-free.
//
// OP_KAH   (prologue): u = scale * (xhat x conj(kappa))   = K_A^H xhat
//          and the scalar g = gamma (kappa . xhat) of the penalty term to xh.p[col] (N^3 per column)
// OP_KAG   (epilogue): y = kappa x s + conj(kappa) g  = K_A s + gamma K_B xhat
//          with g read back from xh.p[col] (one complex per mode instead of re-reading the 3 components
//          of xhat: 32 B per point per column of HBM traffic instead of 48)
// OP_KAGH  (eps-weighted preconditioner + apply, DESIGN R16): the last pass of the preconditioner and the
//          first pass of the following apply on its output, in one HBM round trip per tile: forward z-DFT,
//          W = (kappa x s + conj(kappa) g) / |kappa|^2 (stored to out), then u = scale (W x conj(kappa)) and
//          g' = gamma2 (kappa . W) (g' over g in xh.p[col]), inverse z-DFT of u stored to xh.p[OUT2 + col].
// with kappa_i(m) = sum_a ktab[(3 i + a) N + m_a]  (Dhat_i symbols, reading R3).
#pragma once
#include <type_traits>
#include "kernels.h"
#include "dft.cuh"

enum { OP_NONE = 0, OP_KAH = 1, OP_KAG = 2, OP_KAGH = 3 };
constexpr int OP_KAGH_OUT2 = 96;  // OP_KAGH: xh.p[OP_KAGH_OUT2 + col] = second output column (ncols <= 96)

template <int N>
struct FftPlan;
// R1 >= R2 preferred: the thread count is TP * R1.
#define PC_PLAN(N_, R1_, R2_) \
  template <>                 \
  struct FftPlan<N_> {        \
    static constexpr int R1 = R1_, R2 = R2_; \
  };
PC_PLAN(4, 2, 2)
PC_PLAN(6, 3, 2)
PC_PLAN(8, 4, 2)
PC_PLAN(10, 5, 2)
PC_PLAN(12, 4, 3)
PC_PLAN(16, 4, 4)
PC_PLAN(20, 5, 4)
PC_PLAN(24, 6, 4)
PC_PLAN(32, 8, 4)
PC_PLAN(40, 8, 5)
PC_PLAN(48, 8, 6)
PC_PLAN(64, 8, 8)
PC_PLAN(80, 10, 8)
PC_PLAN(96, 12, 8)
PC_PLAN(100, 10, 10)
PC_PLAN(120, 15, 8)
PC_PLAN(128, 16, 8)
PC_PLAN(160, 16, 10)
PC_PLAN(192, 16, 12)
PC_PLAN(240, 16, 15)
PC_PLAN(256, 16, 16)
#undef PC_PLAN

// largest power of two dividing n, capped
constexpr int pow2_div(int n, int cap) {
  int t = 1;
  while (t < cap && n % (2 * t) == 0) t *= 2;
  return t;
}
#ifndef PC_ZTP
#define PC_ZTP 8
#endif
template <int N, int C>
struct TileCfg {
  static constexpr int TP = pow2_div(N, C == 3 ? PC_ZTP : 16);
  // C = 3 (the symbol-fused z passes): rows of TP >= 8 complex are whole 128-B bank sweeps, so the
  // [c][j][p] layout needs no padding; the space goes to the z-pieces of the symbol table
  static constexpr int TPP = (C == 3 && TP >= 8) ? TP : TP + 1;
  static constexpr int NT = TP * FftPlan<N>::R1;
  // x pass: [c][p][j] with pitch N+1 (tile rows contiguous as in HBM: conflict-free cp.async writes);
  // y/z passes: [c][j][p] with pitch TP+1.  Both odd pitches: conflict-free 16-B fragment accesses.
  // (C = 3 tiles are z-pass tiles only: N * TPP, which keeps the symbol passes at 56 KB = 4 CTAs/SM)
#ifndef PC_ZSPAN_TIGHT
#define PC_ZSPAN_TIGHT 1
#endif
  static constexpr int SPAN =
      (C == 3 && PC_ZSPAN_TIGHT) ? N * TPP : (TP * (N + 1) > N * TPP) ? TP * (N + 1) : N * TPP;
  // C = 1: persistent CTAs with a 2-stage prefetch pipeline; C = 3 (fused symbol passes, 3x the tile):
  // one tile per CTA and higher occupancy instead
#ifndef PC_C3_STAGES
#define PC_C3_STAGES 1
#endif
  static constexpr int STAGES = (C == 1) ? 2 : PC_C3_STAGES;
  static constexpr int KTZ = (C == 3) ? 3 * N : 0;  // ktab z-pieces [3 comps][N]
  static constexpr size_t SMEM = (size_t)STAGES * C * SPAN * sizeof(cplx) + (size_t)(N + KTZ) * sizeof(cplx);
};

// PassArgs: tw[j] = exp(-2 pi i j/N); ktab = [3 comps][3 axes][N] symbol pieces (OP_KAH/OP_KAG);
// gamma (OP_KAG); scale (OP_KAH: folded 1/N^3; OP_NONE: applied at store if != 1).
typedef PassArgsH PassArgs;


// Tile geometry: element (c, j, p) of tile t -> offset within one column, and its mode triple.
template <int N, int AXIS, int TP>
struct TileMap {
  int base;   // offset of (j=0, p=0)
  int sj, sp; // strides of j and p
  int fixed_a, fixed_b;
  DEV TileMap(int t, int qoff = 0) {
    constexpr int NT_ = N / TP;
    int q = t / NT_ + (AXIS == 2 ? 0 : qoff), r = (t % NT_) * TP;
    if (AXIS == 2) {        // pencils along z, tile = TP consecutive x at fixed y = q
      base = q * N + r; sj = N * N; sp = 1; fixed_a = q; fixed_b = r;
    } else if (AXIS == 1) { // pencils along y, tile = TP consecutive x at fixed z = q
      base = q * N * N + r; sj = N; sp = 1; fixed_a = q; fixed_b = r;
    } else {                // pencils along x, tile = TP consecutive rows y at fixed z = q
      base = q * N * N + r * N; sj = 1; sp = N; fixed_a = q; fixed_b = r;
    }
  }
  DEV int off(int j, int p) const { return base + j * sj + p * sp; }
  // mode indices (m1 = x, m2 = y, m3 = z) of element (j, p)
  DEV void modes(int j, int p, int& m1, int& m2, int& m3) const {
    if (AXIS == 2) { m3 = j; m2 = fixed_a; m1 = fixed_b + p; }
    else if (AXIS == 1) { m2 = j; m3 = fixed_a; m1 = fixed_b + p; }
    else { m1 = j; m3 = fixed_a; m2 = fixed_b + p; }
  }
};

// Persistent, double-buffered pass: CTA b processes tiles b, b + G, b + 2G, ...; the next tile streams
// into the other shared-memory stage (cp.async) while the current one is transformed and written.
// Tile index t -> (tile in volume t % TPV, column/component t / TPV).
#ifndef PC_KAG_PREFETCH
#define PC_KAG_PREFETCH 0  // 1: last pass loads g before the DFTs (see fft_pass_kernel)
#endif
#ifndef PC_FFT_TWREC
#define PC_FFT_TWREC 1  // symbol passes: step-A twiddles from two table reads and products (0: one read per k1)
#endif
#ifndef PC_FFT_BOUNDS
#define PC_FFT_BOUNDS 1
#endif
// N <= 128: plain passes at most 85 registers so that 3 persistent CTAs of 256 threads fit an SM (86
// registers left 2: the y pass at n = 128 ran 5 % slower); symbol passes at most 128 (4 CTAs of 128
// threads).  Larger N: no minimum (0 = unspecified; the caps spill there).
#if PC_FFT_BOUNDS
#define PC_FFT_LB(N_, OP_, ...) __launch_bounds__((__VA_ARGS__), ((N_) <= 128) ? ((OP_) != OP_NONE ? 4 : 3) : 0)
#else
#define PC_FFT_LB(N_, OP_, ...) __launch_bounds__((__VA_ARGS__))
#endif
template <int N, int AXIS, int DIR, int OP, int C>
__global__ void PC_FFT_LB(N, OP, TileCfg<N, C>::NT)
fft_pass_kernel(ColPtrs in, MutColPtrs out, ColPtrs xh, PassArgs a, int ntiles) {
  constexpr int R1 = FftPlan<N>::R1, R2 = FftPlan<N>::R2;
  static_assert(R1 * R2 == N, "bad plan");
  static_assert(C == 1 || AXIS == 2, "3-component tiles are z-pass tiles");
  constexpr int TP = TileCfg<N, C>::TP, TPP = TileCfg<N, C>::TPP, NT = TileCfg<N, C>::NT;
  constexpr int SPAN = TileCfg<N, C>::SPAN;
  constexpr int N3 = N * N * N;
  const int TPV = (N / TP) * ((AXIS != 2 && a.nz > 0) ? a.nz : N);  // tiles per component volume (z-range)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* tw = reinterpret_cast<cplx*>(smem_raw);
  cplx* ktz = tw + N;                             // [3][N]: ktab[(3 i + 2) N + m3] (C = 3 only)
  cplx* stage_base = ktz + TileCfg<N, C>::KTZ;    // [STAGES][C * SPAN]
  constexpr int ST = TileCfg<N, C>::STAGES;
  auto SI = [](int c, int j, int p) { return AXIS == 0 ? (c * TP + p) * (N + 1) + j : (c * N + j) * TPP + p; };
  const int tid = threadIdx.x;

  auto load_tile = [&](int t, cplx* s) {
    const TileMap<N, AXIS, TP> tm(t % TPV, a.z0);
    const int cc = t / TPV;
    const int col = (C == 3) ? cc : cc / 3, comp0 = (C == 3) ? 0 : cc % 3;
    const cplx* gin = in.p[col] + (long long)comp0 * N3;
    for (int e = tid; e < C * N * TP; e += NT) {
      int c, j, p;
      if (AXIS == 0) { j = e % N; p = (e / N) % TP; c = e / (N * TP); }
      else { p = e % TP; j = (e / TP) % N; c = e / (TP * N); }
      cp_async16(&s[SI(c, j, p)], gin + (long long)c * N3 + tm.off(j, p));
    }
  };

  for (int j = tid; j < N; j += NT) tw[j] = ldg(a.tw + j);
  // symbol table of a column (multi-k launches: per-column k)
  auto ktab_of = [&](int col) { return a.mk.on ? a.ktab + (size_t)a.mk.kcol[col] * 9 * N : a.ktab; };
  int kt_col = -1;  // column whose z-pieces are in ktz
  if constexpr (C == 3) {
    if (blockIdx.x < ntiles) {
      kt_col = (int)blockIdx.x / TPV;
      const cplx* kt0 = ktab_of(kt_col);
      for (int e = tid; e < 3 * N; e += NT) cp_async16(&ktz[e], kt0 + (3 * (e / N) + 2) * N + e % N);
    }
  }
  int t = blockIdx.x;
  if (t < ntiles) load_tile(t, stage_base);
  cp_async_commit();
  for (int it = 0; t < ntiles; t += gridDim.x, it++) {
    cplx* s = stage_base + (it % ST) * C * SPAN;
    if (ST > 1 && t + (int)gridDim.x < ntiles) load_tile(t + gridDim.x, stage_base + ((it + 1) % ST) * C * SPAN);
    cp_async_commit();
    const TileMap<N, AXIS, TP> tm(t % TPV, a.z0);
    // symbol passes: the (x, y) pieces of kappa are per-thread constants (see the prologue); their loads
    // are issued before the tile wait so the latency overlaps it
    cplx kxy[3];
    const cplx* kt = a.ktab;
    double gam = a.gamma, thr = a.thr;
    if constexpr (C == 3) {
      const int tcol = t / TPV;
      kt = ktab_of(tcol);
      if (a.mk.on) {
        gam = a.mk.gamma[a.mk.kcol[tcol]];
        thr = a.mk.thr[a.mk.kcol[tcol]];
        if (tcol != kt_col) {  // persistent CTA moved to another column's tile: its k's z-pieces
          __syncthreads();
          for (int e = tid; e < 3 * N; e += NT) cp_async16(&ktz[e], kt + (3 * (e / N) + 2) * N + e % N);
          cp_async_commit();
          cp_async_wait<0>();
          kt_col = tcol;
        }
      }
      int m1, m2, m3;
      tm.modes(0, tid % TP, m1, m2, m3);
#pragma unroll
      for (int i = 0; i < 3; i++) kxy[i] = ldg(kt + 3 * i * N + m1) + ldg(kt + (3 * i + 1) * N + m2);
    }
#if PC_KAG_PREFETCH
    // OP_KAG: the penalty scalars g of this thread's elements are loaded before the DFTs (registers),
    // so their latency overlaps the transform instead of the epilogue
    cplx gpre[(OP == OP_KAG) ? (N * TP) / NT : 1];
    if constexpr (OP == OP_KAG) {
      const int cc0 = t / TPV;
      const cplx* gkx0 = xh.p[(C == 3) ? cc0 : cc0 / 3];
#pragma unroll
      for (int q = 0; q < (N * TP) / NT; q++) gpre[q] = ldg(gkx0 + tm.off(tid / TP + q * (NT / TP), tid % TP));
    }
#endif
    cp_async_wait<1>();
    __syncthreads();

    const int cc = t / TPV;
    const int col = (C == 3) ? cc : cc / 3, comp0 = (C == 3) ? 0 : cc % 3;
    cplx* gout = out.p[col] + (long long)comp0 * N3;

    // ---- prologue: u = scale * (xhat x conj(kappa))
    // Symbol-fused passes run along z (AXIS 2): a thread's elements share x = fixed_b + (tid % TP) and
    // y = fixed_a, so kappa_i = [ktab_i,x(m1) + ktab_i,y(m2)] (per-thread constant) + ktab_i,z(m3); the
    // EPT z-pieces are loaded together (unrolled) so their latencies overlap.
    static_assert(OP == OP_NONE || (AXIS == 2 && NT % TP == 0 && (N * TP) % NT == 0), "symbol pass layout");
    constexpr int EPT = (N * TP) / NT;
    if constexpr (OP == OP_KAH) {
      const int p = tid % TP;
      cplx* gkx = const_cast<cplx*>(xh.p[col]);
#pragma unroll
      for (int q = 0; q < EPT; q++) {
        const int j = tid / TP + q * (NT / TP);
        const cplx k1 = kxy[0] + ktz[j], k2 = kxy[1] + ktz[N + j], k3 = kxy[2] + ktz[2 * N + j];
        cplx x1 = s[SI(0, j, p)], x2 = s[SI(1, j, p)], x3 = s[SI(2, j, p)];
        // (x x conj k)_1 = x2 ck3 - x3 ck2, _2 = x3 ck1 - x1 ck3, _3 = x1 ck2 - x2 ck1
        cplx u1 = cmul(x2, conjg(k3)) - cmul(x3, conjg(k2));
        cplx u2 = cmul(x3, conjg(k1)) - cmul(x1, conjg(k3));
        cplx u3 = cmul(x1, conjg(k2)) - cmul(x2, conjg(k1));
        // kappa . xhat (no conjugation: K_B = conj(kappa) kappa^T), kept for the last pass
        const cplx kx = cmul(k1, x1) + cmul(k2, x2) + cmul(k3, x3);
        gkx[tm.off(j, p)] = gam * kx;
        s[SI(0, j, p)] = a.scale * u1;
        s[SI(1, j, p)] = a.scale * u2;
        s[SI(2, j, p)] = a.scale * u3;
      }
      __syncthreads();
    }

    // ---- steps A + B (two-step Stockham, in place in the tile)
    auto dft = [&](auto dirc) {
      constexpr int D = decltype(dirc)::value;
      // step A: R2 DFTs of size R1 (stride R2) + twiddle W_N^{j2 k1}; in place
      for (int i = tid; i < C * TP * R2; i += NT) {
        int p = i % TP, j2 = (i / TP) % R2, c = i / (TP * R2);
        cplx v[R1];
#pragma unroll
        for (int j1 = 0; j1 < R1; j1++) v[j1] = s[SI(c, j2 + R2 * j1, p)];
        Dft<R1, D>::run(v);
        if constexpr (PC_FFT_TWREC && C == 3 && R1 % 4 == 0 && R1 >= 8) {
          // W^{j2 k1}, k1 = 4a + b, from two table reads and <= 4 products (as xrow_step1): the
          // per-k1 reads of the table were up to 4-way bank conflicts (lanes with different j2).
          // Symbol passes only: under the 80-register bound of the plain passes the extra registers
          // spill (y pass 0.98 -> 1.13 ms per 15 columns)
          cplx w1 = tw[j2], w4 = tw[(4 * j2) % N];
          if (D > 0) {
            w1.y = -w1.y;
            w4.y = -w4.y;
          }
          const cplx w2 = cmul(w1, w1), w3 = cmul(w2, w1);
          cplx wa = mk(1.0, 0.0);
#pragma unroll
          for (int a4 = 0; a4 < R1 / 4; a4++) {
            if (a4 == 1) wa = w4;
            if (a4 > 1) wa = cmul(wa, w4);
#pragma unroll
            for (int b4 = 0; b4 < 4; b4++) {
              const int k1 = 4 * a4 + b4;
              cplx w = (b4 == 0) ? wa : (b4 == 1) ? w1 : (b4 == 2) ? w2 : w3;
              if (a4 > 0 && b4 > 0) w = cmul(wa, w);
              s[SI(c, j2 + R2 * k1, p)] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], w);
            }
          }
        } else {
#pragma unroll
          for (int k1 = 0; k1 < R1; k1++) {
            cplx w = tw[(j2 * k1) % N];
            if (D > 0) w.y = -w.y;
            s[SI(c, j2 + R2 * k1, p)] = (k1 == 0 || j2 == 0) ? v[k1] : cmul(v[k1], w);
          }
        }
      }
      __syncthreads();
      // step B: R1 DFTs of size R2 (contiguous blocks) -> natural order k1 + R1 k2
      {
        const int p = tid % TP, k1 = tid / TP;  // NT = TP * R1: one item per thread per component
#pragma unroll 1
        for (int c = 0; c < C; c++) {
          cplx v[R2];
#pragma unroll
          for (int j2 = 0; j2 < R2; j2++) v[j2] = s[SI(c, R2 * k1 + j2, p)];
          Dft<R2, D>::run(v);
          __syncthreads();
#pragma unroll
          for (int k2 = 0; k2 < R2; k2++) s[SI(c, k1 + R1 * k2, p)] = v[k2];
        }
      }
      __syncthreads();
    };
    dft(std::integral_constant<int, DIR>{});

    // ---- store (with fused epilogue)
    if constexpr (OP == OP_KAGH) {
      cplx* gkx = const_cast<cplx*>(xh.p[col]);
      cplx* gout2 = const_cast<cplx*>(xh.p[OP_KAGH_OUT2 + col]);
      const int p = tid % TP;
      cplx g[EPT];
#pragma unroll
      for (int q = 0; q < EPT; q++) g[q] = ldg(gkx + tm.off(tid / TP + q * (NT / TP), p));
#pragma unroll
      for (int q = 0; q < EPT; q++) {
        const int j = tid / TP + q * (NT / TP);
        const int o = tm.off(j, p);
        const cplx k1 = kxy[0] + ktz[j], k2 = kxy[1] + ktz[N + j], k3 = kxy[2] + ktz[2 * N + j];
        const cplx s1 = s[SI(0, j, p)], s2 = s[SI(1, j, p)], s3 = s[SI(2, j, p)];
        const double kk = k1.x * k1.x + k1.y * k1.y + k2.x * k2.x + k2.y * k2.y + k3.x * k3.x + k3.y * k3.y;
        const double inv = (kk > thr) ? 1.0 / kk : 0.0;
        const cplx w1 = inv * (cmul(k2, s3) - cmul(k3, s2) + cmul(conjg(k1), g[q]));
        const cplx w2 = inv * (cmul(k3, s1) - cmul(k1, s3) + cmul(conjg(k2), g[q]));
        const cplx w3 = inv * (cmul(k1, s2) - cmul(k2, s1) + cmul(conjg(k3), g[q]));
        gout[o] = w1;
        gout[N3 + o] = w2;
        gout[2 * N3 + o] = w3;
        // first pass of the apply on W: u = scale (W x conj kappa), g' = gamma2 (kappa . W)
        gkx[o] = a.gamma2 * (cmul(k1, w1) + cmul(k2, w2) + cmul(k3, w3));
        s[SI(0, j, p)] = a.scale * (cmul(w2, conjg(k3)) - cmul(w3, conjg(k2)));
        s[SI(1, j, p)] = a.scale * (cmul(w3, conjg(k1)) - cmul(w1, conjg(k3)));
        s[SI(2, j, p)] = a.scale * (cmul(w1, conjg(k2)) - cmul(w2, conjg(k1)));
      }
      __syncthreads();
      dft(std::integral_constant<int, +1>{});
      for (int e = tid; e < C * N * TP; e += NT) {
        const int p2 = e % TP, j = (e / TP) % N, c = e / (TP * N);
        gout2[(long long)c * N3 + tm.off(j, p2)] = s[SI(c, j, p2)];
      }
    } else if constexpr (OP == OP_KAG) {
      // same element ownership as the prologue; x_hat (the apply input) and the z-pieces of kappa are
      // loaded for all EPT elements first so the global latencies overlap
      const cplx* gkx = xh.p[col];
      const int p = tid % TP;
#if PC_KAG_PREFETCH
      const cplx* g = gpre;
      (void)gkx;
#else
      cplx g[EPT];
#pragma unroll
      for (int q = 0; q < EPT; q++) g[q] = ldg(gkx + tm.off(tid / TP + q * (NT / TP), p));
#endif
#pragma unroll
      for (int q = 0; q < EPT; q++) {
        const int j = tid / TP + q * (NT / TP);
        const int o = tm.off(j, p);
        const cplx k1 = kxy[0] + ktz[j], k2 = kxy[1] + ktz[N + j], k3 = kxy[2] + ktz[2 * N + j];
        const cplx s1 = s[SI(0, j, p)], s2 = s[SI(1, j, p)], s3 = s[SI(2, j, p)];
        cplx y1 = cmul(k2, s3) - cmul(k3, s2) + cmul(conjg(k1), g[q]);
        cplx y2 = cmul(k3, s1) - cmul(k1, s3) + cmul(conjg(k2), g[q]);
        cplx y3 = cmul(k1, s2) - cmul(k2, s1) + cmul(conjg(k3), g[q]);
        if (a.kscale) {
          const double kk = k1.x * k1.x + k1.y * k1.y + k2.x * k2.x + k2.y * k2.y + k3.x * k3.x + k3.y * k3.y;
          const double inv = (kk > thr) ? 1.0 / kk : 0.0;
          y1 = inv * y1;
          y2 = inv * y2;
          y3 = inv * y3;
        }
        gout[o] = y1;
        gout[N3 + o] = y2;
        gout[2 * N3 + o] = y3;
      }
    } else {
      const double sc = (OP == OP_NONE) ? a.scale : 1.0;  // OP_KAH applied it in the prologue
      for (int e = tid; e < C * N * TP; e += NT) {
        int c, j, p;
        if (AXIS == 0) { j = e % N; p = (e / N) % TP; c = e / (N * TP); }
        else { p = e % TP; j = (e / TP) % N; c = e / (TP * N); }
        cplx v = s[SI(c, j, p)];
        if (sc != 1.0) v = sc * v;
        gout[(long long)c * N3 + tm.off(j, p)] = v;
      }
    }
    __syncthreads();  // this stage is refilled by the prefetch issued in the next iteration
  }
  cp_async_wait<0>();
}
