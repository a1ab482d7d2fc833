// libpcband host side: context, C ABI (include/pcband.h) and the LOBPCG driver.
//
// Method: Jin & Xie, arXiv 2511.17107.  Per Bloch vector k the driver runs block LOBPCG
// with soft locking on Op(k) = A_c M A_c^H + gamma B^H B in Fourier coordinates
// (P:523-529), preconditioned by K_P^{-1}, until Res_j <= tol for the nev smallest pairs
// (P:1059-1064).  Everything on the data path runs in this library's kernels; the host only decides
// which columns are still active (one D2H of 2b doubles per iteration) and sequences launches.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pcband.h"
#include "kernels.h"

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
static thread_local std::string g_err;
static int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return set_err(e_ == cudaErrorMemoryAllocation ? PC_ENOMEM : PC_ECUDA,          \
                     std::string(#call) + ": " + cudaGetErrorString(e_));             \
  } while (0)
#define CHK(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ < 0) return rc_; \
  } while (0)

extern "C" const char* pc_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------------------------------
// context
// ------------------------------------------------------------------------------------------
// Process-wide cache of large device blocks: a destroyed context's workspace is kept and handed to the
// next context on the same device (pc_create/pc_destroy per problem then costs no cudaMalloc/cudaFree
// of the ~16 GB LOBPCG workspace).  pc_trim() returns the cached blocks to the driver; an allocation
// failure trims and retries once.
static std::mutex g_cache_mu;
static std::multimap<std::pair<int, size_t>, void*> g_cache;  // (device, bytes) -> block

static void* cache_take(size_t want, size_t* got) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.lower_bound({dev, want});
  if (it == g_cache.end() || it->first.first != dev || it->first.second > want + want / 4) return nullptr;
  void* p = it->second;
  *got = it->first.second;
  g_cache.erase(it);
  return p;
}
static void cache_put(void* p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache.insert({{dev, bytes}, p});
}
static void cache_trim(int dev) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto it = g_cache.begin(); it != g_cache.end();) {
    if (dev < 0 || it->first.first == dev) {
      cudaSetDevice(it->first.first);
      cudaFree(it->second);
      it = g_cache.erase(it);
    } else {
      ++it;
    }
  }
  cudaSetDevice(cur);
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t b) {
    if (b <= bytes) return PC_OK;
    release();
    size_t got = 0;
    if ((p = cache_take(b, &got)) != nullptr) {
      bytes = got;
      return PC_OK;
    }
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      cudaGetLastError();
      int dev = 0;
      cudaGetDevice(&dev);
      cache_trim(dev);
      e = cudaMalloc(&p, b);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return set_err(PC_ENOMEM, std::string("cudaMalloc(") + std::to_string(b) + "): " + cudaGetErrorString(e));
    }
    bytes = b;
    return PC_OK;
  }
  void release() {
    if (p) cache_put(p, bytes);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

extern "C" void pc_trim(int device) { cache_trim(device); }

// pinned host staging: [0, 2048) norms, [2048, 2056) info ints, [PIN_PWV..) top-k |kappa|^2,
// [PIN_PWI..) top-k mode ints, [PIN_PWE..) plane-wave scatter entries
enum { PIN_PWV = 4096, PIN_PWI = 4096 + 5120, PIN_PWE = 4096 + 5120 + 2560, PIN_DOUBLES = 16384 };

struct pc_ctx {
  int n = 0, device = 0, eps_mode = 1;
  long long n3 = 0, len = 0;  // N^3, 3 N^3
  double A[9], B[9];          // row-major; B = A^{-1}
  double eps[18];
  double gamma_override = 0.0;
  int hpd_flags = 0;
  EpsCoef ec;
  uint8_t* d_mask = nullptr;
  cplx* d_tw = nullptr;
  cplx* d_ktab = nullptr;
  double cur_k[3] = {NAN, NAN, NAN};
  double cur_gamma = 0.0, cur_thr = 0.0;
  DevBuf ws;          // apply workspace
  DevBuf kxws;        // apply workspace: gamma (kappa . xhat), N^3 per column (first pass -> last pass)
  int apply_chunk = 0;
  int guard = 6;  // block b = nev + guard (reading R14; measured optimum of the current kernels)
  double drop_tol = 1e-8;   // Rayleigh-Ritz rank threshold (scaled mass Gram); see DESIGN R14
  long long kindex_offset = 0;  // global index of kpts[0] (seeds independent of sharding)
  int verbose = 0;
  int p_restart = 1;  // drop the P block when the Rayleigh-Ritz basis is rank deficient
  int sticky_lock = 0;         // 1: locked columns stay locked (SciPy's activeMask &=); 0: may re-activate
  int gram_refresh = 16;       // every n-th iteration uses the full Gram (no X^H X = I assumption)
  int fuse_xex = 1;            // fused x-DFT + M_eps + x-DFT pass for z-plane-local media
  int plane_fuse = 0;          // 1, n = 128: one cluster pass for y/x DFTs + M_eps (plane2.cu; measured slower)
  int w_guard = 0;             // >= 0: only the first nev + w_guard columns get W; -1: all b columns
  int precond = 0;             // 0: K_P^{-1}; 1: eps-weighted K_P^{-1} (beyond the paper, see precond_eps)
  int precond_fuse = 1;        // precond = 1 in pc_bands: its last pass and the apply's first pass as one (OP_KAGH)
  EpsCoef ec_inv{};            // diagonal of M_eps inverted: 1/eps_ii - 1 on the masks I_i (precond = 1)
  int fuse_resid = 1;          // both block updates + residual + K_P^{-1} in one pass (update_all.cu)
  int update_tmap = 1;         // 1: update kernel with TMA tensor-copy row tiles (update_tmap.cu); 0: cp.async tiles
  int trim_locked = 1;         // W', P', AP' only for the columns active in this iteration (see solve_k)
  double xdev_tol = 1e-10;     // max | |X_j|^2 - 1 | above which the next Gram is formed in full
  int start_mode = 1;          // 0: Gaussian start block; 1: transverse plane waves of the lowest |kappa|^2
  int start_precond = 1;       // plane-wave start: Gaussian admixture through K_P^{-1} (see solve_k)
#ifndef PC_START_NOISE
#define PC_START_NOISE 1e-3
#endif
  double start_noise = PC_START_NOISE;  // plane-wave start: relative Gaussian admixture per column
  int warm_start = 0;          // 1: start from the previous k-point's Ritz vectors (same context, k != 0)
  int have_prev = 0, prev_slot = 0, prev_b = 0;
  DevBuf pwbuf;
  DevBuf mkbuf;  // symbol tables of a multi-k launch (PC_MAXK x 9N)
  int kbatch = 1;                // pc_bands: k-points solved in lock step per batch (solve_batch; 1 = solve_k)
  double* h_batch = nullptr;     // pinned norms / info of a batch
  size_t h_batch_n = 0;
  std::vector<cudaStream_t> bst; // per-k streams of a batch (the per-k Gram / Rayleigh-Ritz / update launches)
  std::vector<cudaEvent_t> bev;
  std::vector<double> hist;  // Res_j per iteration of the last solved k-point (row-major, hist_b per row)
  int hist_b = 0;
  // LOBPCG storage
  DevBuf lob, small, gpart, cbuf;
  double* h_pinned = nullptr;
  cudaStream_t stream = nullptr;
  // profiling
  int profile = 0;
  double stat_ms[PC_NSTAT] = {0};
  double stat_cnt[PC_NSTAT] = {0};
  double stat_flops[PC_NSTAT] = {0};
  double stat_bytes[PC_NSTAT] = {0};
  double launches = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> ev_pool;
};

// ---- profiling helpers (CUDA events on the launching stream) --------------------------------
static cudaEvent_t ev_get(pc_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
// Times one kernel class (CUDA events on the launching stream) and books its algorithmic work:
// nl kernel launches, flops and bytes that the method requires for this launch group.
struct Prof {
  pc_ctx* c;
  int stat;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  Prof(pc_ctx* c_, int s_, cudaStream_t st_, int nl = 1, double flops = 0.0, double bytes = 0.0)
      : c(c_), stat(s_), st(st_) {
    c->launches += nl;
    c->stat_flops[s_] += flops;
    c->stat_bytes[s_] += bytes;
    if (c->profile) {
      e0 = ev_get(c);
      cudaEventRecord(e0, st);
    }
  }
  ~Prof() {
    if (c->profile) {
      cudaEvent_t e1 = ev_get(c);
      cudaEventRecord(e1, st);
      c->pending.push_back({stat, {e0, e1}});
    }
  }
};
static void prof_flush(pc_ctx* c) {
  for (auto& pe : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(pe.second.second);
    cudaEventElapsedTime(&ms, pe.second.first, pe.second.second);
    c->stat_ms[pe.first] += ms;
    c->stat_cnt[pe.first] += 1;
    c->ev_pool.push_back(pe.second.first);
    c->ev_pool.push_back(pe.second.second);
  }
  c->pending.clear();
}

// ---- small host linear algebra -------------------------------------------------------------
static bool inv3(const double* a, double* b) {
  double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) + a[2] * (a[3] * a[7] - a[4] * a[6]);
  double sc = 0;
  for (int i = 0; i < 9; i++) sc = std::fmax(sc, std::fabs(a[i]));
  if (!(std::fabs(det) > 1e-12 * sc * sc * sc)) return false;
  b[0] = (a[4] * a[8] - a[5] * a[7]) / det;
  b[1] = (a[2] * a[7] - a[1] * a[8]) / det;
  b[2] = (a[1] * a[5] - a[2] * a[4]) / det;
  b[3] = (a[5] * a[6] - a[3] * a[8]) / det;
  b[4] = (a[0] * a[8] - a[2] * a[6]) / det;
  b[5] = (a[2] * a[3] - a[0] * a[5]) / det;
  b[6] = (a[3] * a[7] - a[4] * a[6]) / det;
  b[7] = (a[1] * a[6] - a[0] * a[7]) / det;
  b[8] = (a[0] * a[4] - a[1] * a[3]) / det;
  return true;
}

// eigenvalues of a 3x3 Hermitian matrix (complex Jacobi, host)
static void heev3(const double* e18, double* w) {
  double ar[3][3], ai[3][3];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      ar[i][j] = e18[2 * (3 * i + j)];
      ai[i][j] = e18[2 * (3 * i + j) + 1];
    }
  for (int sweep = 0; sweep < 50; sweep++) {
    double off = 0;
    for (int p = 0; p < 3; p++)
      for (int q = p + 1; q < 3; q++) off += ar[p][q] * ar[p][q] + ai[p][q] * ai[p][q];
    if (off < 1e-34) break;
    for (int p = 0; p < 3; p++)
      for (int q = p + 1; q < 3; q++) {
        double mag = std::hypot(ar[p][q], ai[p][q]);
        if (mag < 1e-300) continue;
        double z = (ar[q][q] - ar[p][p]) / (2 * mag);
        double t = (z >= 0 ? 1.0 : -1.0) / (std::fabs(z) + std::sqrt(1 + z * z));
        double c = 1 / std::sqrt(1 + t * t), s = t * c;
        double er = ar[p][q] / mag, ei = ai[p][q] / mag;
        // A <- U^H A U, U = [[c, s e], [-s conj e, c]] on (p, q)
        for (int j = 0; j < 3; j++) {  // rows
          double apr = ar[p][j], api = ai[p][j], aqr = ar[q][j], aqi = ai[q][j];
          ar[p][j] = c * apr - s * (er * aqr - ei * aqi);
          ai[p][j] = c * api - s * (er * aqi + ei * aqr);
          ar[q][j] = s * (er * apr + ei * api) + c * aqr;
          ai[q][j] = s * (er * api - ei * apr) + c * aqi;
        }
        for (int j = 0; j < 3; j++) {  // columns
          double apr = ar[j][p], api = ai[j][p], aqr = ar[j][q], aqi = ai[j][q];
          ar[j][p] = c * apr - s * (er * aqr + ei * aqi);
          ai[j][p] = c * api - s * (er * aqi - ei * aqr);
          ar[j][q] = s * (er * apr - ei * api) + c * aqr;
          ai[j][q] = s * (er * api + ei * apr) + c * aqi;
        }
      }
  }
  for (int i = 0; i < 3; i++) w[i] = ar[i][i];
}

// ------------------------------------------------------------------------------------------
// pc_create / destroy / info
// ------------------------------------------------------------------------------------------
extern "C" int pc_supported_n(int* sizes, int cap) { return fft_supported_list(sizes, cap); }

extern "C" int pc_create(pc_ctx** out, const double A[9], int n, const double eps1[18], const uint8_t* masks,
                         int eps_mode, double gamma_override, int device) {
  if (!out || !A || !eps1 || !masks) return set_err(PC_EINVAL, "pc_create: null argument");
  *out = nullptr;
  if (!fft_supported(n)) return set_err(PC_EINVAL, "pc_create: unsupported grid size n=" + std::to_string(n));
  if (eps_mode < 0 || eps_mode > 2) return set_err(PC_EINVAL, "pc_create: bad eps_mode");
  double B[9];
  if (!inv3(A, B)) return set_err(PC_EINVAL, "pc_create: lattice matrix A is singular");
  // Hermitian check
  double emax = 0;
  for (int i = 0; i < 18; i++) emax = std::fmax(emax, std::fabs(eps1[i]));
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      double dr = eps1[2 * (3 * i + j)] - eps1[2 * (3 * j + i)];
      double di = eps1[2 * (3 * i + j) + 1] + eps1[2 * (3 * j + i) + 1];
      if (std::hypot(dr, di) > 1e-14 * emax) return set_err(PC_EINVAL, "pc_create: eps1 is not Hermitian");
    }
  double w[3];
  heev3(eps1, w);
  double wmin = std::fmin(w[0], std::fmin(w[1], w[2])), wmax = std::fmax(w[0], std::fmax(w[1], w[2]));
  if (!(wmin > 0)) return set_err(PC_ENOTPD, "pc_create: eps1 is not positive definite");
  bool offd = false, zero_off = false;
  for (int i = 0; i < 3; i++)
    for (int j = i + 1; j < 3; j++) {
      bool z = eps1[2 * (3 * i + j)] == 0.0 && eps1[2 * (3 * i + j) + 1] == 0.0;
      offd |= !z;
      zero_off |= z;
    }
  if (eps_mode == PC_EPS_DIAGONAL && offd)
    return set_err(PC_EINVAL, "pc_create: PC_EPS_DIAGONAL needs a diagonal eps1");
  bool sdd = true;
  for (int i = 0; i < 3; i++) {
    double s = 0;
    for (int j = 0; j < 3; j++)
      if (j != i) s += std::hypot(eps1[2 * (3 * i + j)], eps1[2 * (3 * i + j) + 1]);
    if (!(eps1[2 * (3 * i + i)] > s)) sdd = false;
  }
  bool a1 = wmin > 0 && wmax <= 1.0 + 1e-15;

  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return set_err(PC_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  pc_ctx* c = new pc_ctx();
  c->n = n;
  c->device = device;
  c->eps_mode = eps_mode;
  c->n3 = (long long)n * n * n;
  c->len = 3 * c->n3;
  std::memcpy(c->A, A, sizeof(c->A));
  std::memcpy(c->B, B, sizeof(c->B));
  std::memcpy(c->eps, eps1, sizeof(c->eps));
  c->gamma_override = gamma_override;
  c->hpd_flags = (a1 ? PC_HPD_ASSUMP1 : 0) | (sdd ? PC_HPD_SDD : 0) | (zero_off ? PC_HPD_ZERO_OFFD : 0) |
                 ((a1 && (sdd || zero_off)) ? PC_HPD_GUARANTEED : 0);
  for (int i = 0; i < 3; i++) c->ec.d[i] = eps1[2 * (3 * i + i)] - 1.0;
  for (int i = 0; i < 3; i++) c->ec_inv.d[i] = 1.0 / eps1[2 * (3 * i + i)] - 1.0;  // eps_ii > 0 (HPD, checked below)
  const int od[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  for (int t = 0; t < 3; t++) {
    int i = od[t][0], j = od[t][1];
    c->ec.e[t] = mk(eps1[2 * (3 * i + j)], eps1[2 * (3 * i + j) + 1]);
    c->ec.has[t] = (c->ec.e[t].x != 0.0 || c->ec.e[t].y != 0.0) ? 1 : 0;
  }
  auto fail = [&](int code, const std::string& m) {
    pc_destroy(c);
    return set_err(code, m);
  };
  // masks: pack I1, I2, I3, IV into one byte per point
  std::vector<uint8_t> packed(c->n3);
  for (long long i = 0; i < c->n3; i++) {
    uint8_t b = 0;
    for (int f = 0; f < 4; f++)
      if (masks[f * c->n3 + i]) b |= (uint8_t)(1u << f);
    packed[i] = b;
  }
  // twiddles, symbol table and mask in one cached block (no cudaMalloc / cudaFree per context: a
  // cudaFree can stall for hundreds of ms while other contexts run)
  if (c->cbuf.ensure((size_t)10 * n * sizeof(cplx) + (size_t)c->n3 + 256) != PC_OK)
    return fail(PC_ENOMEM, "pc_create: table alloc");
  c->d_tw = c->cbuf.as<cplx>();
  c->d_ktab = c->d_tw + n;
  c->d_mask = reinterpret_cast<uint8_t*>(c->d_ktab + 9 * n);
  if (cudaMemcpy(c->d_mask, packed.data(), c->n3, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(PC_ECUDA, "pc_create: mask upload");
  // twiddles exp(-2 pi i j / N) in long double, rounded once
  std::vector<cplx> tw(n);
  const long double PI_L = 3.141592653589793238462643383279502884L;
  for (int j = 0; j < n; j++) {
    long double a = -2.0L * PI_L * (long double)j / (long double)n;
    tw[j] = mk((double)cosl(a), (double)sinl(a));
    if ((4 * j) % n == 0) {  // exact quarter turns
      int qd = (4 * j) / n;
      const double cs[4][2] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};
      tw[j] = mk(cs[qd][0], cs[qd][1]);
    }
  }
  cudaMemcpy(c->d_tw, tw.data(), n * sizeof(cplx), cudaMemcpyHostToDevice);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(PC_ECUDA, "pc_create: stream");
  if (cudaMallocHost(&c->h_pinned, PIN_DOUBLES * sizeof(double)) != cudaSuccess)
    return fail(PC_ENOMEM, "pc_create: pinned");
  *out = c;
  return PC_OK;
}

extern "C" void pc_destroy(pc_ctx* c) {
  if (!c) return;
  static const bool trace = getenv("PCBAND_TRACE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto s_ : c->bst) cudaStreamSynchronize(s_);  // batch streams (an error return can leave work queued)
  prof_flush(c);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  auto t1 = now();
  c->cbuf.release();
  auto t2 = now();
  c->ws.release();
  c->kxws.release();
  c->lob.release();
  c->small.release();
  c->gpart.release();
  c->pwbuf.release();
  c->mkbuf.release();
  auto t3 = now();
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  if (c->h_batch) cudaFreeHost(c->h_batch);
  for (auto s_ : c->bst) cudaStreamDestroy(s_);
  for (auto e_ : c->bev) cudaEventDestroy(e_);
  auto t4 = now();
  if (c->stream) cudaStreamDestroy(c->stream);
  auto t5 = now();
  if (trace) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[pcband] destroy: sync %.1f ms, tables %.1f, cache %.1f, freehost %.1f, stream %.1f\n",
            ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5));
  }
  delete c;
}

static double gamma_rule(const pc_ctx* c, const double k[3]) {
  if (c->gamma_override > 0) return c->gamma_override;
  // practical penalty
  const double fourpi2 = 4.0 * M_PI * M_PI;
  double nk = std::sqrt(k[0] * k[0] + k[1] * k[1] + k[2] * k[2]);
  if (nk == 0.0 || nk >= 1.0) return fourpi2;
  return fourpi2 / (nk * nk);
}

extern "C" double pc_gamma(const pc_ctx* c, const double k[3]) { return (c && k) ? gamma_rule(c, k) : NAN; }

extern "C" int pc_info(const pc_ctx* c, int* hpd_flags, size_t* ws_bytes_per_col) {
  if (!c) return set_err(PC_EINVAL, "pc_info: null ctx");
  if (hpd_flags) *hpd_flags = c->hpd_flags;
  if (ws_bytes_per_col) *ws_bytes_per_col = (size_t)c->len * sizeof(cplx);
  return PC_OK;
}

extern "C" int pc_set_option(pc_ctx* c, const char* key, double v) {
  if (!c || !key) return set_err(PC_EINVAL, "pc_set_option: null");
  std::string k(key);
  if (k == "guard") { if (v < 0 || v > 32) return set_err(PC_EINVAL, "guard out of range"); c->guard = (int)v; }
  else if (k == "apply_chunk") c->apply_chunk = (int)v;
  else if (k == "profile") c->profile = v != 0.0;
  else if (k == "drop_tol") c->drop_tol = v;
  else if (k == "kindex_offset") c->kindex_offset = (long long)v;
  else if (k == "verbose") c->verbose = (int)v;
  else if (k == "kbatch") {
    if (v < 1 || v > PC_MAXK) return set_err(PC_EINVAL, "kbatch: 1 .. 16");
    c->kbatch = (int)v;
  }
  else if (k == "p_restart") c->p_restart = (int)v;
  else if (k == "start") c->start_mode = (int)v;
  else if (k == "warm_start") {
    c->warm_start = (int)v;
    c->have_prev = 0;
  }
  else if (k == "sticky_lock") c->sticky_lock = (int)v;
  else if (k == "gram_refresh") c->gram_refresh = (int)v;
  else if (k == "fuse_xex") c->fuse_xex = (int)v;
  else if (k == "plane_fuse") c->plane_fuse = (int)v;
  else if (k == "w_guard") c->w_guard = (int)v;
  else if (k == "precond") c->precond = (int)v;
  else if (k == "precond_fuse") c->precond_fuse = (int)v;
  else if (k == "fuse_resid") c->fuse_resid = (int)v;
  else if (k == "trim_locked") c->trim_locked = (int)v;
  else if (k == "xdev_tol") c->xdev_tol = v;
  else if (k == "update_tmap") c->update_tmap = (int)v;
  else if (k == "jacobi_tol") set_jacobi_tol(v);
  else if (k == "gram_narrow") set_gram_narrow((int)v);
  else if (k == "start_noise") c->start_noise = v;
  else if (k == "start_precond") c->start_precond = (int)v;
  else return set_err(PC_EINVAL, "pc_set_option: unknown key " + k);
  return PC_OK;
}

extern "C" int pc_history(const pc_ctx* c, double* out, int cap, int* block) {
  if (!c) return set_err(PC_EINVAL, "pc_history: null ctx");
  const int b = c->hist_b;
  const int rows = b ? (int)(c->hist.size() / b) : 0;
  if (block) *block = b;
  if (out)
    for (int i = 0; i < std::min(rows, cap) * b; i++) out[i] = c->hist[i];
  return rows;
}

extern "C" int pc_stats(pc_ctx* c, double* out, int reset) {
  if (!c) return set_err(PC_EINVAL, "pc_stats: null ctx");
  cudaSetDevice(c->device);
  prof_flush(c);
  if (out) {
    for (int i = 0; i < PC_NSTAT; i++) {
      out[4 * i] = c->stat_cnt[i];
      out[4 * i + 1] = c->stat_ms[i];
      out[4 * i + 2] = c->stat_flops[i];
      out[4 * i + 3] = c->stat_bytes[i];
    }
    out[4 * PC_NSTAT] = c->launches;
  }
  if (reset) {
    for (int i = 0; i < PC_NSTAT; i++) c->stat_cnt[i] = c->stat_ms[i] = c->stat_flops[i] = c->stat_bytes[i] = 0;
    c->launches = 0;
  }
  return PC_OK;
}

// ------------------------------------------------------------------------------------------
// symbols for k (stream-ordered; cached while k is unchanged)
// ------------------------------------------------------------------------------------------
// |kappa|^2 <= 1e-28 max|kappa|^2 -> pass-through (reading R7); max bounded via the 1-D pieces
static double pass_threshold(const pc_ctx* c, const double k[3]) {
  double bound = 0;
  const double n = c->n;
  for (int i = 0; i < 3; i++) {
    double m = 0;
    for (int a = 0; a < 3; a++) m += std::fabs(c->B[3 * a + i]) * 2.0 * n;
    m += std::fabs(k[i]);
    bound += m * m;
  }
  return 1e-28 * bound;
}

// Symbol tables of nk Bloch vectors for one multi-k launch: mkbuf holds nk consecutive 9N
// tables, mk the per-k penalty and pass-through threshold; kcol (ncols entries) maps columns to k.
static int build_multik(pc_ctx* c, const double* kpts, int nk, const int* kcol, int ncols, MultiK& mk,
                        cudaStream_t st) {
  if (nk < 1 || nk > PC_MAXK) return set_err(PC_EINVAL, "multi-k: 1 <= nk <= 16");
  for (int j = 0; j < ncols; j++)
    if (kcol[j] < 0 || kcol[j] >= nk) return set_err(PC_EINVAL, "multi-k: k index out of range");
  const size_t tb = (size_t)9 * c->n * sizeof(cplx);
  if ((size_t)nk * tb > c->mkbuf.bytes) {
    cudaStreamSynchronize(st);
    CHK(c->mkbuf.ensure((size_t)PC_MAXK * tb));
  }
  mk.on = 1;
  for (int i = 0; i < nk; i++) {
    Sym3 s;
    std::memcpy(s.B, c->B, sizeof(s.B));
    for (int a = 0; a < 3; a++) s.k[a] = kpts[3 * i + a];
    c->launches += 1;
    launch_ktab(c->mkbuf.as<cplx>() + (size_t)i * 9 * c->n, c->d_tw, c->n, s, st);
    mk.gamma[i] = gamma_rule(c, kpts + 3 * i);
    mk.thr[i] = pass_threshold(c, kpts + 3 * i);
  }
  for (int j = 0; j < ncols; j++) mk.kcol[j] = (unsigned char)kcol[j];
  return PC_OK;
}
static void set_k(pc_ctx* c, const double k[3], cudaStream_t st) {
  c->cur_gamma = gamma_rule(c, k);
  if (k[0] == c->cur_k[0] && k[1] == c->cur_k[1] && k[2] == c->cur_k[2]) return;
  Sym3 s;
  std::memcpy(s.B, c->B, sizeof(s.B));
  for (int i = 0; i < 3; i++) s.k[i] = k[i];
  c->launches += 1;
  launch_ktab(c->d_ktab, c->d_tw, c->n, s, st);
  c->cur_thr = pass_threshold(c, k);
  for (int i = 0; i < 3; i++) c->cur_k[i] = k[i];
}

// ------------------------------------------------------------------------------------------
// apply
// ------------------------------------------------------------------------------------------
constexpr int OP_KAGH_OUT2_HOST = 96;  // = OP_KAGH_OUT2 in fft_pass.cuh (second output slots of xh)

// The operator the apply pipeline runs: Op = K_A M K_A^H + gamma K_B (the paper's), or, for
// the eps-weighted preconditioner, (1/|kappa|^2) (K_A D^{-1} K_A^H + K_B) with D = diag(M_eps) (precond_eps).
struct ApplyOp {
  int mode;            // PC_EPS_* of the middle factor
  const EpsCoef* ec;   // its coefficients
  int prec;            // 1: gamma = 1 and the last pass scales by 1/|kappa|^2
};
static ApplyOp paper_op(const pc_ctx* c) { return ApplyOp{c->eps_mode, &c->ec, 0}; }

static int fft_pass(pc_ctx* c, int axis, int dir, int kind, const ColPtrs& in, const MutColPtrs& out,
                    const ColPtrs& xh, int nc, double scale, cudaStream_t st, int z0 = 0, int nz = 0,
                    int prec = 0, double gamma2 = 0.0, const MultiK* mk = nullptr) {
  PassArgsH a;
  a.tw = c->d_tw;
  a.ktab = (mk && mk->on) ? c->mkbuf.as<cplx>() : c->d_ktab;
  if (mk && mk->on) a.mk = *mk;
  a.gamma = prec ? 1.0 : c->cur_gamma;
  a.scale = scale;
  a.z0 = z0;
  a.nz = nz;
  a.kscale = (prec && kind == 2) ? 1 : 0;
  a.thr = c->cur_thr;
  a.gamma2 = gamma2;
  cudaError_t e = launch_fft_pass(c->n, axis, dir, kind, in, out, xh, nc, a, st);
  if (e != cudaSuccess) return set_err(PC_ECUDA, std::string("fft pass: ") + cudaGetErrorString(e));
  return PC_OK;
}

static ColPtrs to_const(const MutColPtrs& m, int nc) {
  ColPtrs r;
  for (int i = 0; i < nc; i++) r.p[i] = m.p[i];
  return r;
}

// Fourier-space apply of nc <= PC_MAXCOLS columns: Y = Op X, ws = nc workspace columns.  mk: per-column k
// (multi-k launch; the symbol passes read each column's own table).
static int apply_fourier(pc_ctx* c, const ColPtrs& X, const MutColPtrs& Y, const MutColPtrs& WS, int nc,
                         cudaStream_t st, const ApplyOp* opp = nullptr, const MultiK* mk = nullptr) {
  const ApplyOp op = opp ? *opp : paper_op(c);
  const int n = c->n;
  const double inv_n3 = 1.0 / ((double)n * n * n);
  ColPtrs Yc = to_const(Y, nc), Wc = to_const(WS, nc), none{};
  // algorithmic work per pass: one read + one write of the 3-component field (96 B per point per
  // column; the last pass also reads x_hat: 144 B), 5 log2(N) flops per point per component
  const double pts = (double)c->n3 * nc;
  const double fl = 15.0 * std::log2((double)n) * pts;
  // gamma (kappa . xhat) per mode and column: written by the first pass, read by the last
  const size_t kxb = (size_t)nc * c->n3 * sizeof(cplx);
  if (kxb > c->kxws.bytes) {
    cudaStreamSynchronize(st);
    CHK(c->kxws.ensure(kxb));
  }
  ColPtrs KX;
  for (int j = 0; j < nc; j++) KX.p[j] = c->kxws.as<cplx>() + (size_t)j * c->n3;
  {
    Prof p(c, PC_STAT_FFT_Z_KAH, st, 1, fl + 38.0 * pts, 112.0 * pts);
    CHK(fft_pass(c, 2, +1, 1, X, Y, KX, nc, inv_n3, st, 0, 0, op.prec, 0.0, mk));
  }
  // z-plane-local media (eps_13 = eps_23 = 0 in CrossDoF; any Diagonal/Trivial medium): the x-passes
  // and the M_eps stencil run fused (x-inverse DFT + M_eps + x-forward DFT in one HBM round trip)
  const bool plane_local = c->fuse_xex && (op.mode != PC_EPS_CROSSDOF || (!op.ec->has[1] && !op.ec->has[2]));
  if (plane_local) {
    if (c->plane_fuse && plane2_supported(n)) {
      // one HBM round trip for y-inverse, x-inverse, M_eps, x-forward, y-forward (plane2.cu)
      Prof p(c, PC_STAT_EPS, st, 1, 4 * fl + 100.0 * pts, 97.0 * pts);
      cudaError_t e = launch_plane2(n, op.mode, Yc, WS, nc, c->d_mask, *op.ec, c->d_tw, st);
      if (e != cudaSuccess) return set_err(PC_ECUDA, std::string("plane pass: ") + cudaGetErrorString(e));
    } else {
      // y-inverse, (x-inverse + M_eps + x-forward) fused, y-forward
      {
        Prof p(c, PC_STAT_FFT_MID, st, 1, fl, 96.0 * pts);
        CHK(fft_pass(c, 1, +1, 0, Yc, Y, none, nc, 1.0, st));
      }
      {
        Prof p(c, PC_STAT_EPS, st, 1, 2 * fl + 100.0 * pts, 97.0 * pts);
        cudaError_t e = launch_xex(n, op.mode, Yc, WS, nc, c->d_mask, *op.ec, c->d_tw, 1.0, 0, 0, st);
        if (e != cudaSuccess) return set_err(PC_ECUDA, std::string("xex pass: ") + cudaGetErrorString(e));
      }
      {
        Prof p(c, PC_STAT_FFT_MID, st, 1, fl, 96.0 * pts);
        CHK(fft_pass(c, 1, -1, 0, Wc, WS, none, nc, 1.0, st));
      }
    }
    {
      Prof p(c, PC_STAT_FFT_Z_KA, st, 1, fl + 32.0 * pts, 112.0 * pts);
      CHK(fft_pass(c, 2, -1, 2, Wc, Y, KX, nc, 1.0, st, 0, 0, op.prec, 0.0, mk));
    }
    return PC_OK;
  }
  {
    Prof p(c, PC_STAT_FFT_MID, st, 2, 2 * fl, 2 * 96.0 * pts);
    CHK(fft_pass(c, 1, +1, 0, Yc, Y, none, nc, 1.0, st));
    CHK(fft_pass(c, 0, +1, 0, Yc, Y, none, nc, 1.0, st));
  }
  {
    Prof p(c, PC_STAT_EPS, st, 1, 100.0 * pts, 97.0 * pts);
    launch_eps(op.mode, Yc, WS, nc, n, c->d_mask, *op.ec, st);
  }
  {
    Prof p(c, PC_STAT_FFT_MID, st, 2, 2 * fl, 2 * 96.0 * pts);
    CHK(fft_pass(c, 0, -1, 0, Wc, WS, none, nc, 1.0, st));
    CHK(fft_pass(c, 1, -1, 0, Wc, WS, none, nc, 1.0, st));
  }
  {
    Prof p(c, PC_STAT_FFT_Z_KA, st, 1, fl + 32.0 * pts, 112.0 * pts);
    CHK(fft_pass(c, 2, -1, 2, Wc, Y, KX, nc, 1.0, st, 0, 0, op.prec, 0.0, mk));
  }
  return PC_OK;
}

// eps-weighted preconditioner (beyond the paper; option precond = 1).  The paper's K_P^{-1} inverts
// the vacuum symbol K_A K_A^H + gamma K_B.  This variant puts the inverse of M_eps's
// diagonal D = diag(m_i), m_i = (eps_ii - 1) I_i + 1, between the two curl halves:
//   T = (K_A / |kappa|^2) D^{-1} (K_A^H / |kappa|^2) + Pi / (gamma |kappa|^2),  Pi = conj(kappa) kappa^T / |kappa|^2,
// which is K_P^{-1} in vacuum (D = I) and the exact inverse for a homogeneous medium.  Given
// W0 = K_P^{-1} R (what the residual kernels write): K_A^H W0 = K_A^H R / |kappa|^2 and
// kappa^T W0 = kappa^T R / (gamma |kappa|^2), so T R = (1/|kappa|^2) (K_A D^{-1} K_A^H + K_B) W0 --
// the apply pipeline with D^{-1} in the middle, gamma = 1 and a 1/|kappa|^2 epilogue, in place on W.
// Modes with |kappa|^2 <= thr map to 0.
static int precond_eps(pc_ctx* c, const MutColPtrs& W, const MutColPtrs& WS, int nc, cudaStream_t st) {
  const ApplyOp op{PC_EPS_DIAGONAL, &c->ec_inv, 1};
  return apply_fourier(c, to_const(W, nc), W, WS, nc, st, &op);
}

// W <- T W (W = K_P^{-1} R on entry, see precond_eps) and AW = Op W in 9 passes instead of 10: the
// preconditioner's last pass and the apply's first pass run as one OP_KAGH pass.  Only for the 5-pass
// pipeline of z-plane-local media (else: returns 1 and the caller runs the two steps).
static int precond_apply_fused(pc_ctx* c, const MutColPtrs& W, const MutColPtrs& AW, const MutColPtrs& WS, int nc,
                               cudaStream_t st) {
  const bool plane_local = c->fuse_xex && (c->eps_mode != PC_EPS_CROSSDOF || (!c->ec.has[1] && !c->ec.has[2]));
  if (!plane_local || c->plane_fuse || nc > OP_KAGH_OUT2_HOST) return 1;
  const int n = c->n;
  const double inv_n3 = 1.0 / ((double)n * n * n);
  const size_t kxb = (size_t)nc * c->n3 * sizeof(cplx);
  if (kxb > c->kxws.bytes) {
    cudaStreamSynchronize(st);
    CHK(c->kxws.ensure(kxb));
  }
  ColPtrs KX, none{};
  for (int j = 0; j < nc; j++) KX.p[j] = c->kxws.as<cplx>() + (size_t)j * c->n3;
  const ColPtrs Wc = to_const(W, nc), AWc = to_const(AW, nc), WSc = to_const(WS, nc);
  const double pts = (double)c->n3 * nc;
  const double fl = 15.0 * std::log2((double)n) * pts;
  {
    Prof p(c, PC_STAT_FFT_Z_KAH, st, 1, fl + 38.0 * pts, 112.0 * pts);
    CHK(fft_pass(c, 2, +1, 1, Wc, AW, KX, nc, inv_n3, st, 0, 0, 1));
  }
  auto middle = [&](int mode, const EpsCoef& ec) -> int {
    {
      Prof p(c, PC_STAT_FFT_MID, st, 1, fl, 96.0 * pts);
      CHK(fft_pass(c, 1, +1, 0, AWc, AW, none, nc, 1.0, st));
    }
    {
      Prof p(c, PC_STAT_EPS, st, 1, 2 * fl + 100.0 * pts, 96.0 * pts);
      cudaError_t e = launch_xex(n, mode, AWc, WS, nc, c->d_mask, ec, c->d_tw, 1.0, 0, 0, st);
      if (e != cudaSuccess) return set_err(PC_ECUDA, std::string("xex pass: ") + cudaGetErrorString(e));
    }
    Prof p(c, PC_STAT_FFT_MID, st, 1, fl, 96.0 * pts);
    return fft_pass(c, 1, -1, 0, WSc, WS, none, nc, 1.0, st);
  };
  CHK(middle(PC_EPS_DIAGONAL, c->ec_inv));
  {
    // W = (K_A s + K_B W0)/|kappa|^2 -> W; u = K_A^H W / N^3 -> AW (scratch); g = gamma kappa.W -> KX
    ColPtrs X2 = KX;
    for (int j = 0; j < nc; j++) X2.p[OP_KAGH_OUT2_HOST + j] = AW.p[j];
    Prof p(c, PC_STAT_FFT_Z_KA, st, 1, 2 * fl + 80.0 * pts, 192.0 * pts);
    CHK(fft_pass(c, 2, -1, 3, WSc, W, X2, nc, inv_n3, st, 0, 0, 1, c->cur_gamma));
  }
  CHK(middle(c->eps_mode, c->ec));
  {
    Prof p(c, PC_STAT_FFT_Z_KA, st, 1, fl + 32.0 * pts, 112.0 * pts);
    CHK(fft_pass(c, 2, -1, 2, WSc, AW, KX, nc, 1.0, st));
  }
  return PC_OK;
}

// unitary 3-D DFT per component; dir = -1: F3^H (to Fourier), +1: F3 (to real).  Y may equal X.
static int fft3(pc_ctx* c, const ColPtrs& X, const MutColPtrs& Y, int nc, int dir, cudaStream_t st) {
  const double s = 1.0 / std::sqrt((double)c->n);
  ColPtrs Yc = to_const(Y, nc), none{};
  const double pts = (double)c->n3 * nc;
  Prof p(c, PC_STAT_FFT_MID, st, 3, 3 * 15.0 * std::log2((double)c->n) * pts, 3 * 96.0 * pts);
  CHK(fft_pass(c, 0, dir, 0, X, Y, none, nc, s, st));
  CHK(fft_pass(c, 1, dir, 0, Yc, Y, none, nc, s, st));
  CHK(fft_pass(c, 2, dir, 0, Yc, Y, none, nc, s, st));
  return PC_OK;
}

static int ensure_ws(pc_ctx* c, int cols) {
  size_t need = (size_t)cols * c->len * sizeof(cplx);
  if (need <= c->ws.bytes) return PC_OK;
  cudaDeviceSynchronize();
  return c->ws.ensure(need);
}

static int chunk_cols(pc_ctx* c, int ncols, int per_call_max) {
  int ch = std::min(ncols, per_call_max);
  if (c->apply_chunk > 0) ch = std::min(ch, c->apply_chunk);
  return std::max(ch, 1);
}

static int apply_cols(pc_ctx* c, const double k[3], const ColPtrs& X, const MutColPtrs& Y, int ncols, int space,
                      cudaStream_t st) {
  set_k(c, k, st);
  const int ch = chunk_cols(c, ncols, 64);
  const int nws = (space == PC_SPACE_REAL) ? 2 * ch : ch;
  CHK(ensure_ws(c, nws));
  cplx* ws = c->ws.as<cplx>();
  for (int j0 = 0; j0 < ncols; j0 += ch) {
    int nc = std::min(ch, ncols - j0);
    ColPtrs x;
    MutColPtrs y, w, w2;
    for (int j = 0; j < nc; j++) {
      x.p[j] = X.p[j0 + j];
      y.p[j] = Y.p[j0 + j];
      w.p[j] = ws + (size_t)j * c->len;
      w2.p[j] = ws + (size_t)(ch + j) * c->len;
    }
    if (space == PC_SPACE_FOURIER) {
      CHK(apply_fourier(c, x, y, w, nc, st));
    } else {
      CHK(fft3(c, x, w2, nc, -1, st));                 // xhat = F3^H H
      CHK(apply_fourier(c, to_const(w2, nc), y, w, nc, st));
      CHK(fft3(c, to_const(y, nc), y, nc, +1, st));    // back to real space
    }
  }
  return PC_OK;
}

static void block_ptrs(const void* base, long long ld, int j0, int nc, ColPtrs& out) {
  const cplx* b = reinterpret_cast<const cplx*>(base);
  for (int j = 0; j < nc; j++) out.p[j] = b + (size_t)(j0 + j) * ld;
}
static void block_ptrs(void* base, long long ld, int j0, int nc, MutColPtrs& out) {
  cplx* b = reinterpret_cast<cplx*>(base);
  for (int j = 0; j < nc; j++) out.p[j] = b + (size_t)(j0 + j) * ld;
}

static int check_block(pc_ctx* c, const void* X, const void* Y, int ncols, long long ld, const char* who) {
  if (!c) return set_err(PC_EINVAL, std::string(who) + ": null ctx");
  if (ncols < 0) return set_err(PC_EINVAL, std::string(who) + ": ncols < 0");
  if (ncols > 0 && (!X || !Y)) return set_err(PC_EINVAL, std::string(who) + ": null data pointer");
  if (ld < c->len) return set_err(PC_EINVAL, std::string(who) + ": ld < 3 N^3");
  return PC_OK;
}

extern "C" int pc_apply(pc_ctx* c, const double k[3], const void* X, void* Y, int ncols, long long ld, int space,
                        void* stream) {
  CHK(check_block(c, X, Y, ncols, ld, "pc_apply"));
  if (!k) return set_err(PC_EINVAL, "pc_apply: null k");
  if (space != PC_SPACE_FOURIER && space != PC_SPACE_REAL) return set_err(PC_EINVAL, "pc_apply: bad space");
  if (X == Y && ncols > 0) return set_err(PC_EINVAL, "pc_apply: X and Y alias");
  CU(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  for (int j0 = 0; j0 < ncols; j0 += PC_MAXCOLS) {
    int nc = std::min(PC_MAXCOLS, ncols - j0);
    ColPtrs x;
    MutColPtrs y;
    block_ptrs(X, ld, j0, nc, x);
    block_ptrs(Y, ld, j0, nc, y);
    CHK(apply_cols(c, k, x, y, nc, space, st));
  }
  CU(cudaGetLastError());
  return PC_OK;
}

extern "C" int pc_precond(pc_ctx* c, const double k[3], const void* R, void* P, int ncols, long long ld,
                          void* stream) {
  CHK(check_block(c, R, P, ncols, ld, "pc_precond"));
  if (!k) return set_err(PC_EINVAL, "pc_precond: null k");
  CU(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  set_k(c, k, st);
  for (int j0 = 0; j0 < ncols; j0 += PC_MAXCOLS) {
    int nc = std::min(PC_MAXCOLS, ncols - j0);
    ColPtrs r;
    MutColPtrs p;
    block_ptrs(R, ld, j0, nc, r);
    block_ptrs(P, ld, j0, nc, p);
    {
      Prof pf(c, PC_STAT_RESID, st, 1, 60.0 * c->n3 * nc, 96.0 * c->n3 * nc);
      launch_precond(r, p, nc, c->n, c->d_ktab, c->cur_gamma, c->cur_thr, st);
    }
    if (c->precond == 1) {
      CHK(ensure_ws(c, nc));
      MutColPtrs w;
      for (int j = 0; j < nc; j++) w.p[j] = c->ws.as<cplx>() + (size_t)j * c->len;
      CHK(precond_eps(c, p, w, nc, st));
    }
  }
  CU(cudaGetLastError());
  return PC_OK;
}

// Several Bloch vectors in one launch: column j of X is applied with k = kpts[kcol[j]].
extern "C" int pc_apply_multi(pc_ctx* c, const double* kpts, int nk, const int* kcol, const void* X, void* Y,
                              int ncols, long long ld, void* stream) {
  CHK(check_block(c, X, Y, ncols, ld, "pc_apply_multi"));
  if (!kpts || !kcol) return set_err(PC_EINVAL, "pc_apply_multi: null kpts/kcol");
  if (X == Y && ncols > 0) return set_err(PC_EINVAL, "pc_apply_multi: X and Y alias");
  CU(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int ch = chunk_cols(c, ncols, 64);
  CHK(ensure_ws(c, ch));
  for (int j0 = 0; j0 < ncols; j0 += ch) {
    const int nc = std::min(ch, ncols - j0);
    MultiK mk;
    CHK(build_multik(c, kpts, nk, kcol + j0, nc, mk, st));
    ColPtrs x;
    MutColPtrs y, w;
    block_ptrs(X, ld, j0, nc, x);
    block_ptrs(Y, ld, j0, nc, y);
    for (int j = 0; j < nc; j++) w.p[j] = c->ws.as<cplx>() + (size_t)j * c->len;
    CHK(apply_fourier(c, x, y, w, nc, st, nullptr, &mk));
  }
  CU(cudaGetLastError());
  return PC_OK;
}

extern "C" int pc_precond_multi(pc_ctx* c, const double* kpts, int nk, const int* kcol, const void* R, void* P,
                                int ncols, long long ld, void* stream) {
  CHK(check_block(c, R, P, ncols, ld, "pc_precond_multi"));
  if (!kpts || !kcol) return set_err(PC_EINVAL, "pc_precond_multi: null kpts/kcol");
  CU(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  for (int j0 = 0; j0 < ncols; j0 += PC_MAXCOLS) {
    const int nc = std::min(PC_MAXCOLS, ncols - j0);
    MultiK mk;
    CHK(build_multik(c, kpts, nk, kcol + j0, nc, mk, st));
    ColPtrs r;
    MutColPtrs p;
    block_ptrs(R, ld, j0, nc, r);
    block_ptrs(P, ld, j0, nc, p);
    Prof pf(c, PC_STAT_RESID, st, 1, 60.0 * c->n3 * nc, 96.0 * c->n3 * nc);
    launch_precond(r, p, nc, c->n, c->mkbuf.as<cplx>(), 0.0, 0.0, st, &mk);
  }
  CU(cudaGetLastError());
  return PC_OK;
}

extern "C" int pc_apply_eps(pc_ctx* c, const void* E, void* Y, int ncols, long long ld, void* stream) {
  CHK(check_block(c, E, Y, ncols, ld, "pc_apply_eps"));
  if (E == Y && ncols > 0) return set_err(PC_EINVAL, "pc_apply_eps: E and Y alias");
  CU(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  for (int j0 = 0; j0 < ncols; j0 += PC_MAXCOLS) {
    int nc = std::min(PC_MAXCOLS, ncols - j0);
    ColPtrs e;
    MutColPtrs y;
    block_ptrs(E, ld, j0, nc, e);
    block_ptrs(Y, ld, j0, nc, y);
    Prof pf(c, PC_STAT_EPS, st, 1, 100.0 * c->n3 * nc, 97.0 * c->n3 * nc);
    launch_eps(c->eps_mode, e, y, nc, c->n, c->d_mask, c->ec, st);
  }
  CU(cudaGetLastError());
  return PC_OK;
}

extern "C" int pc_fft3(pc_ctx* c, const void* X, void* Y, int ncols, long long ld, int direction, void* stream) {
  CHK(check_block(c, X, Y, ncols, ld, "pc_fft3"));
  if (direction != PC_FFT_TO_FOURIER && direction != PC_FFT_TO_REAL) return set_err(PC_EINVAL, "pc_fft3: direction");
  CU(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  for (int j0 = 0; j0 < ncols; j0 += PC_MAXCOLS) {
    int nc = std::min(PC_MAXCOLS, ncols - j0);
    ColPtrs x;
    MutColPtrs y;
    block_ptrs(X, ld, j0, nc, x);
    block_ptrs(Y, ld, j0, nc, y);
    CHK(fft3(c, x, y, nc, direction == PC_FFT_TO_FOURIER ? -1 : +1, st));
  }
  CU(cudaGetLastError());
  return PC_OK;
}

// debug entry: one FFT pass (kind 0 plain / 1 K_A^H-fused inverse z / 2 K_A+gamma K_B forward z)
extern "C" int pc_debug_pass(pc_ctx* c, const double k[3], int kind, int axis, int dir, const void* X, void* Y,
                             const void* XH, int ncols, long long ld, double scale) {
  CHK(check_block(c, X, Y, ncols, ld, "pc_debug_pass"));
  CU(cudaSetDevice(c->device));
  set_k(c, k, 0);
  ColPtrs x, xh;
  MutColPtrs y;
  block_ptrs(X, ld, 0, ncols, x);
  block_ptrs(Y, ld, 0, ncols, y);
  if (XH) block_ptrs(XH, ld, 0, ncols, xh);
  CHK(fft_pass(c, axis, dir, kind, x, y, xh, ncols, scale, 0));
  CU(cudaDeviceSynchronize());
  return PC_OK;
}

// debug entry used by the tests: dense Hermitian eigensolver on device (host in/out)
extern "C" int pc_debug_heevj(const double* A_host, int n, double* w_host, double* V_host, int* sweeps) {
  if (n < 1 || n > 80) return set_err(PC_EINVAL, "pc_debug_heevj: 1 <= n <= 80");
  cplx *dA, *dV;
  double* dw;
  int* di;
  CU(cudaMalloc(&dA, n * n * sizeof(cplx)));
  CU(cudaMalloc(&dV, n * n * sizeof(cplx)));
  CU(cudaMalloc(&dw, n * sizeof(double)));
  CU(cudaMalloc(&di, sizeof(int)));
  CU(cudaMemcpy(dA, A_host, n * n * sizeof(cplx), cudaMemcpyHostToDevice));
  launch_heevj(dA, n, dw, dV, di, 0);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(w_host, dw, n * sizeof(double), cudaMemcpyDeviceToHost));
  if (V_host) CU(cudaMemcpy(V_host, dV, n * n * sizeof(cplx), cudaMemcpyDeviceToHost));
  if (sweeps) CU(cudaMemcpy(sweeps, di, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(dA);
  cudaFree(dV);
  cudaFree(dw);
  cudaFree(di);
  return PC_OK;
}

// Kernel timing entry for the LOBPCG block kernels on random data (tools/bench_block.py): the shapes
// of one iteration with b X columns, na W columns and nP P columns on this context's grid.
// which = 0: fused update (+ residual, K_P^{-1}); 1: Gram S^H [W P AW AP] (+ assembly); 2: Gram
// S^H [W AW]; 3: TMA update.  ms = mean milliseconds per launch group over reps (CUDA events on the context stream).
extern "C" int pc_bench_block(pc_ctx* c, int which, int b, int na, int nP, int reps, double* ms) {
  if (!c || !ms || b < 1 || na < 0 || nP < 0 || nP > na || na > b || reps < 1)
    return set_err(PC_EINVAL, "pc_bench_block: bad arguments");
  const int p = b + na + nP;
  if (3 * b > 80 || p > 80) return set_err(PC_EINVAL, "pc_bench_block: p <= 80");
  CU(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  const long long len = c->len;
  {
    const double k[3] = {0.5, 0.3, 0.2};
    set_k(c, k, st);
  }
  CHK(c->lob.ensure(10 * (size_t)b * len * sizeof(cplx)));
  cplx* base = c->lob.as<cplx>();
  auto col = [&](int slot, int j) { return base + ((size_t)slot * b + j) * len; };
  MutColPtrs all;
  for (int j = 0; j < 8 && j * b < PC_MAXCOLS; j++) {
    int nc = std::min(b, PC_MAXCOLS - j * b);
    for (int t = 0; t < nc; t++) all.p[t] = col(j, t);
    launch_randn(all, nc, len, 1234 + j, 0, 1.0, st);
  }
  const int rg = resid_grid(c->n);
  const size_t nG = (size_t)p * 2 * p;
  CHK(c->small.ensure((2 * nG + (size_t)p * b) * sizeof(cplx) + (size_t)(b + rg * b * 2) * sizeof(double) + 64));
  CHK(c->gpart.ensure(gram_partial_bytes(p, 2 * p)));
  cplx* dG = c->small.as<cplx>();
  cplx* dGp = dG + nG;
  cplx* dC = dGp + nG;
  double* dLam = reinterpret_cast<double*>(dC + (size_t)p * b);
  double* dPart = dLam + b;
  {
    MutColPtrs cm;
    cm.p[0] = dC;
    launch_randn(cm, 1, (long long)p * b, 99, 0, 0.1, st);
    cudaMemsetAsync(dLam, 0, b * sizeof(double), st);
  }
  // S = [X(slot 0) W(slot 8) P(slot 4)], AS = [AX(1) AW(9) AP(5)]; outputs X' 2, AX' 3, P' 6, AP' 7, W 8
  ColPtrs S, AS;
  for (int j = 0; j < b; j++) { S.p[j] = col(0, j); AS.p[j] = col(1, j); }
  for (int j = 0; j < na; j++) { S.p[b + j] = col(8, j); AS.p[b + j] = col(9, j); }
  for (int j = 0; j < nP; j++) { S.p[b + na + j] = col(4, j); AS.p[b + na + j] = col(5, j); }
  MutColPtrs Y1, Y2, Y1a, Y2a, W;
  for (int j = 0; j < b; j++) {
    Y2.p[j] = col(2, j);
    Y2a.p[j] = col(3, j);
    Y1.p[j] = j < na ? col(6, j) : nullptr;
    Y1a.p[j] = j < na ? col(7, j) : nullptr;
    W.p[j] = j < na ? col(8, j) : nullptr;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double tot = 0.0;
  for (int r = -1; r < reps; r++) {  // r = -1: warm-up
    cudaEventRecord(e0, st);
    if (which == 0) {
      // W is read (S) and overwritten tile by tile, as in pc_bands
      const int g = launch_update_all(S, AS, p, dC, p, b, b, Y1, Y2, Y1a, Y2a, W, dLam, c->n, c->d_ktab,
                                      1.0, 0.0, 0, dPart, rg, st);
      launch_reduce_partial(dPart, g, b, dLam + 0 * b, st);
    } else if (which == 3) {
      UtBlocks blk;
      memset(&blk, 0, sizeof(blk));
      blk.ld = len;
      const int slotS[3] = {0, 8, 4}, slotA[3] = {1, 9, 5}, cnt[3] = {b, na, nP}, rowoff[3] = {0, b, b + na};
      for (int kb = 0; kb < 3; kb++) {
        if (!cnt[kb]) continue;
        blk.s[kb] = col(slotS[kb], 0);
        blk.as[kb] = col(slotA[kb], 0);
        blk.slot_cols[kb] = b;
        blk.c0[kb] = 0;
        blk.nc[kb] = cnt[kb];
        for (int j = 0; j < 32; j++) blk.crow[kb][j] = j < cnt[kb] ? (signed char)(rowoff[kb] + j) : -1;
      }
      const int g = launch_update_tmap(blk, dC, p, b, Y1, Y2, Y1a, Y2a, W, dLam, c->n, c->d_ktab, 1.0, 0.0, 0,
                                       dPart, rg, st);
      if (g < 0) return set_err(PC_ECUDA, "pc_bench_block: tensor map encoding failed");
      launch_reduce_partial(dPart, g, b, dLam + 0 * b, st);
    } else if (which == 1) {
      ColPtrs T;
      const int cw = na + nP;
      for (int t = 0; t < cw; t++) T.p[t] = S.p[b + t];
      for (int t = 0; t < cw; t++) T.p[cw + t] = AS.p[b + t];
      launch_gram(S, p, T, 2 * cw, len, dGp, c->gpart.as<cplx>(), st);
      launch_gram_assemble(dGp, dLam, b, cw, dG, st);
    } else {
      ColPtrs T;
      for (int t = 0; t < na; t++) T.p[t] = S.p[b + t];
      for (int t = 0; t < na; t++) T.p[na + t] = AS.p[b + t];
      launch_gram(S, p, T, 2 * na, len, dGp, c->gpart.as<cplx>(), st);
    }
    cudaEventRecord(e1, st);
    CU(cudaEventSynchronize(e1));
    float m = 0.f;
    cudaEventElapsedTime(&m, e0, e1);
    if (r >= 0) tot += m;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CU(cudaGetLastError());
  *ms = tot / reps;
  return PC_OK;
}

// ------------------------------------------------------------------------------------------
// LOBPCG (pc_bands)
// ------------------------------------------------------------------------------------------
__global__ void normalize_copy_kernel(ColPtrs X, const double* norms, MutColPtrs Y, long long len) {
  const int j = blockIdx.y;
  const double s = 1.0 / sqrt(norms[2 * j + 1]);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
    Y.p[j][i] = s * X.p[j][i];
}

// Adds unit transverse plane waves to the b start columns: modes in ascending |kappa|^2 (ties by
// index), two polarisations u with kappa^T u = 0 (so K_B u = 0) per mode.
static int plane_wave_start(pc_ctx* c, const MutColPtrs& x0, int b, cudaStream_t st, const cplx* ktab = nullptr,
                            double thr = -1.0) {
  if (!ktab) ktab = c->d_ktab;
  if (thr < 0.0) thr = c->cur_thr;
  const int G = pw_grid(), n = c->n;
  CHK(c->pwbuf.ensure((size_t)G * PW_T * (sizeof(double) + sizeof(int)) + 64 * sizeof(PwEntry) +
                      9 * n * sizeof(cplx) + 256));
  double* dv = c->pwbuf.as<double>();
  int* di = reinterpret_cast<int*>(dv + G * PW_T);
  PwEntry* de = reinterpret_cast<PwEntry*>(di + G * PW_T + 8);
  launch_kappa2_topk(ktab, n, thr, dv, di, st);
  double* hv = c->h_pinned + PIN_PWV;
  int* hi = reinterpret_cast<int*>(c->h_pinned + PIN_PWI);
  PwEntry* he = reinterpret_cast<PwEntry*>(c->h_pinned + PIN_PWE);
  std::vector<cplx> kt(9 * n);
  cudaMemcpyAsync(hv, dv, G * PW_T * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hi, di, G * PW_T * sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(kt.data(), ktab, 9 * n * sizeof(cplx), cudaMemcpyDeviceToHost, st);
  CU(cudaStreamSynchronize(st));
  std::vector<std::pair<double, int>> cand;
  for (int t = 0; t < G * PW_T; t++)
    if (hi[t] >= 0) cand.push_back({hv[t], hi[t]});
  std::sort(cand.begin(), cand.end());
  int ne = 0;
  for (size_t q = 0; q < cand.size() && ne < b; q++) {
    const int m = cand[q].second;
    const int m1 = m % n, m2 = (m / n) % n, m3 = m / (n * n);
    cplx kap[3];
    for (int i = 0; i < 3; i++)
      kap[i] = kt[(3 * i) * n + m1] + kt[(3 * i + 1) * n + m2] + kt[(3 * i + 2) * n + m3];
    // a = conj(kappa)/|kappa|;  u1 = e - a (a^H e) for the unit axis least aligned with a;  u2 = conj(a x u1)
    double kn = std::sqrt(abs2(kap[0]) + abs2(kap[1]) + abs2(kap[2]));
    cplx a[3] = {conjg(kap[0]), conjg(kap[1]), conjg(kap[2])};
    for (int i = 0; i < 3; i++) a[i] = (1.0 / kn) * a[i];
    int ax = 0;
    for (int i = 1; i < 3; i++)
      if (abs2(a[i]) < abs2(a[ax])) ax = i;
    cplx u1[3] = {mk(0, 0), mk(0, 0), mk(0, 0)};
    u1[ax] = mk(1, 0);
    cplx ahe = conjg(a[ax]);  // a^H e
    for (int i = 0; i < 3; i++) u1[i] = u1[i] - cmul(a[i], ahe);
    double u1n = std::sqrt(abs2(u1[0]) + abs2(u1[1]) + abs2(u1[2]));
    for (int i = 0; i < 3; i++) u1[i] = (1.0 / u1n) * u1[i];
    cplx u2[3] = {conjg(cmul(a[1], u1[2]) - cmul(a[2], u1[1])), conjg(cmul(a[2], u1[0]) - cmul(a[0], u1[2])),
                  conjg(cmul(a[0], u1[1]) - cmul(a[1], u1[0]))};
    double u2n = std::sqrt(abs2(u2[0]) + abs2(u2[1]) + abs2(u2[2]));
    for (int i = 0; i < 3; i++) u2[i] = (1.0 / u2n) * u2[i];
    const cplx* us[2] = {u1, u2};
    for (int pol = 0; pol < 2 && ne < b; pol++, ne++) {
      he[ne].col = ne;
      he[ne].mode = m;
      for (int i = 0; i < 3; i++) {
        he[ne].v[2 * i] = us[pol][i].x;
        he[ne].v[2 * i + 1] = us[pol][i].y;
      }
    }
  }
  cudaMemcpyAsync(de, he, ne * sizeof(PwEntry), cudaMemcpyHostToDevice, st);
  launch_pw_scatter(x0, de, ne, (int)c->n3, st);
  return PC_OK;
}

static unsigned long long mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static int solve_k(pc_ctx* c, const double k[3], int kidx, int nev, double tol, int maxit, unsigned long long seed,
                   double* omega2, double* resid, int* iters, int* status, cplx* evec_out) {
  cudaStream_t st = c->stream;
  const int b = nev + c->guard;
  const long long len = c->len;
  const int maxp = 3 * b;
  set_k(c, k, st);
  const bool deflate = (k[0] == 0.0 && k[1] == 0.0 && k[2] == 0.0);

  // ---- storage: 10 b columns + apply workspace b columns
  const size_t colb = (size_t)len * sizeof(cplx);
  CHK(c->lob.ensure(10 * (size_t)b * colb));
  CHK(ensure_ws(c, b));
  cplx* base = c->lob.as<cplx>();
  auto col = [&](int slot, int j) { return base + ((size_t)slot * b + j) * len; };
  enum { XA = 0, AXA, XB, AXB, PA, APA, PB, APB, WW, AWW };
  int sX = XA, sAX = AXA, sXn = XB, sAXn = AXB, sP = PA, sAP = APA, sPn = PB, sAPn = APB;
  // small device buffers: G (maxp x 2maxp), Gp (maxp x 2maxp), C (maxp x b), rr scratch, lam, norms,
  // residual partials, info
  const size_t nG = (size_t)maxp * 2 * maxp, nC = (size_t)maxp * b, nScr = (size_t)3 * 80 * 80;
  const int rg = resid_grid(c->n);
  size_t small_bytes = (2 * nG + nC + nScr) * sizeof(cplx) + (size_t)(b + 2 * b + rg * b * 2) * sizeof(double) +
                       (size_t)8 * sizeof(int) + 64;
  CHK(c->small.ensure(small_bytes));
  CHK(c->gpart.ensure(gram_partial_bytes(maxp, 2 * maxp)));
  // only the first nw columns ever get a search direction W (option w_guard; -1: all b)
  const int nw = (c->w_guard >= 0) ? std::min(b, nev + c->w_guard) : b;
  cplx* dG = c->small.as<cplx>();
  cplx* dGp = dG + nG;
  cplx* dC = dGp + nG;
  cplx* dScr = dC + nC;
  double* dLam = reinterpret_cast<double*>(dScr + nScr);
  double* dNorm = dLam + b;
  double* dPart = dNorm + 2 * b;
  int* dInfo = reinterpret_cast<int*>(dPart + (size_t)rg * b * 2);
  bool force_full = false;  // next Gram from the vectors in full (X^H X = I no longer trusted)
  double* hN = c->h_pinned;                 // 2b norms
  int* hInfo = reinterpret_cast<int*>(c->h_pinned + 2048);
  MutColPtrs wsp;
  for (int j = 0; j < b; j++) wsp.p[j] = c->ws.as<cplx>() + (size_t)j * len;

  auto mcols = [&](int slot, const std::vector<int>& js, MutColPtrs& m, int off) {
    for (size_t t = 0; t < js.size(); t++) m.p[off + t] = col(slot, js[t]);
  };
  auto ccols = [&](int slot, const std::vector<int>& js, ColPtrs& m, int off) {
    for (size_t t = 0; t < js.size(); t++) m.p[off + t] = col(slot, js[t]);
  };
  std::vector<int> all(b);
  for (int j = 0; j < b; j++) all[j] = j;

  auto apply_list = [&](int src, int dst, const std::vector<int>& js) -> int {
    ColPtrs x;
    MutColPtrs y;
    ccols(src, js, x, 0);
    mcols(dst, js, y, 0);
    MutColPtrs w;
    for (size_t t = 0; t < js.size(); t++) w.p[t] = wsp.p[t];
    return apply_fourier(c, x, y, w, (int)js.size(), st);
  };
  auto precond_list = [&](int slot, const std::vector<int>& js) -> int {  // W <- T R from W = K_P^{-1} R
    MutColPtrs y;
    mcols(slot, js, y, 0);
    MutColPtrs w;
    for (size_t t = 0; t < js.size(); t++) w.p[t] = wsp.p[t];
    return precond_eps(c, y, w, (int)js.size(), st);
  };
  auto rr = [&](int p) -> int {
    {
      Prof pf(c, PC_STAT_RR, st, 1, 16.0 * 8.0 * 8.0 * (double)p * p * p, 0.0);
      launch_rr(dG, p, b, c->drop_tol, dC, dLam, dInfo, dScr, st);
    }
    cudaMemcpyAsync(hInfo, dInfo, 8 * sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    // a launch rejected on its configuration is not reported by the synchronisation: check it too
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(PC_ECUDA, std::string("rayleigh-ritz: ") + cudaGetErrorString(e));
    return hInfo[0];  // rank
  };

  // ---- start block X0, AX0, Rayleigh-Ritz on span(X0).
  // start 0: counter-based Gaussian columns.  start 1 (default): transverse plane waves of the
  // b/2 Fourier modes with the smallest |kappa(m)|^2 -- the eigenvectors of K_P, i.e.
  // of the vacuum operator -- plus a small seeded Gaussian admixture (reading R14: the paper does
  // not state its start block).
  // warm start (not in the paper): the previous k-point's Ritz vectors on this context
  const bool warm = c->warm_start && c->have_prev && c->prev_b == b && !deflate;
  c->have_prev = 0;  // set again only by a completed solve
  if (warm) {
    Prof pf(c, PC_STAT_OTHER, st, 1, 0.0, 32.0 * len * b);
    if (c->prev_slot != sX)
      CU(cudaMemcpyAsync(col(sX, 0), col(c->prev_slot, 0), (size_t)b * colb, cudaMemcpyDeviceToDevice, st));
  } else {
    const bool pw = c->start_mode == 1;
    // start_precond: the admixture is K_P^{-1} g (g white, scaled by 4 pi^2 so that its lowest modes keep
    // the white admixture's amplitude): every low mode is seeded (degenerate and spurious gamma-modes
    // are found), but without the white noise's high-|kappa| content, whose residual (~ noise x max
    // |kappa|^2 ~ 1e4 at n = 128) the first iterations otherwise spend their time removing
    const bool pre = pw && c->start_precond && c->start_noise > 0.0;
    const double noise = pw ? c->start_noise / std::sqrt((double)len) * (pre ? 4.0 * M_PI * M_PI : 1.0) : 1.0;
    Prof pf(c, PC_STAT_OTHER, st, pw ? (pre ? 4 : 3) : 1, 0.0, 16.0 * len * b);
    MutColPtrs x0;
    mcols(sX, all, x0, 0);
    launch_randn(x0, b, len, mix64(seed + 0x100000001ull * (unsigned long long)kidx), deflate ? (int)c->n3 : 0,
                 noise, st);
    if (pre) {
      ColPtrs xi;
      ccols(sX, all, xi, 0);
      launch_precond(xi, x0, b, c->n, c->d_ktab, c->cur_gamma, c->cur_thr, st);
    }
    if (pw) CHK(plane_wave_start(c, x0, b, st));
  }
  CHK(apply_list(sX, sAX, all));
  {
    ColPtrs S, T;
    ccols(sX, all, S, 0);
    ccols(sX, all, T, 0);
    ccols(sAX, all, T, b);
    Prof pf(c, PC_STAT_GRAM, st, 2, 8.0 * len * b * 2 * b, 16.0 * len * 2 * b);
    launch_gram(S, b, T, 2 * b, len, dG, c->gpart.as<cplx>(), st);
  }
  int rank = rr(b);
  if (rank < b) return set_err(PC_ENUMERIC, "pc_bands: start block is rank deficient");
  {
    Prof pf(c, PC_STAT_UPDATE, st, 2, 2 * 8.0 * len * b * b, 2 * 16.0 * len * 2 * b);
    ColPtrs S;
    MutColPtrs Y;
    ccols(sX, all, S, 0);
    mcols(sXn, all, Y, 0);
    launch_update(S, b, dC, b, b, b, nullptr, Y, nullptr, len, st);
    ccols(sAX, all, S, 0);
    mcols(sAXn, all, Y, 0);
    launch_update(S, b, dC, b, b, b, nullptr, Y, nullptr, len, st);
  }
  std::swap(sX, sXn);
  std::swap(sAX, sAXn);

  // P / AP slots: the update's TMA boxes span [first, last] active column, so a column that never got a
  // P' in this solve (locked from the start) can sit inside a box; C's zero row for it does not cancel a
  // non-finite leftover of an earlier solve (0 * NaN), so those slots start zeroed (4 b columns)
  for (int sl : {(int)PA, (int)APA, (int)PB, (int)APB}) CU(cudaMemsetAsync(col(sl, 0), 0, (size_t)b * colb, st));
  std::vector<char> active(b, 1);
  std::vector<double> res(b, 0.0);
  c->hist.clear();
  c->hist_b = b;
  bool haveP = false, resid_ready = false;
  int it = 0, conv = 0;
  // trim_locked: the update writes W', P', AP' only for the columns that are active in this iteration
  // (soft-locked columns skip 3 column writes each).  A locked column that re-activates (sticky_lock = 0)
  // gets its W from one residual pass and enters without a P column.
  const bool trim = c->trim_locked != 0;
  std::vector<char> hasW(b, 0), hasP(b, 0);
  for (;; it++) {
    // residuals of every column; W = K_P^{-1} R only for the columns that can receive a search direction
    if (!resid_ready) {
      Prof pf(c, PC_STAT_RESID, st, 2, 84.0 * c->n3 * b, 16.0 * len * (2 * b + nw));
      ColPtrs X, AX;
      MutColPtrs W;
      ccols(sX, all, X, 0);
      ccols(sAX, all, AX, 0);
      mcols(WW, all, W, 0);
      for (int j = nw; j < b; j++) W.p[j] = nullptr;
      launch_resid(X, AX, W, dLam, b, c->n, c->d_ktab, c->cur_gamma, c->cur_thr, deflate ? 1 : 0, dPart, dNorm, st);
      for (int j = 0; j < b; j++) hasW[j] = j < nw;
    }
    cudaMemcpyAsync(hN, dNorm, 2 * b * sizeof(double), cudaMemcpyDeviceToHost, st);
    {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) return set_err(PC_ECUDA, std::string("lobpcg: ") + cudaGetErrorString(e));
    }
    if (c->profile) prof_flush(c);
    conv = 1;
    double xdev = 0.0;  // X^H X = I is assumed by the Gram assembly; its diagonal is measured here
    for (int j = 0; j < b; j++) xdev = std::max(xdev, std::fabs(hN[2 * j + 1] - 1.0));
    force_full = !(xdev <= c->xdev_tol);
    for (int j = 0; j < b; j++) res[j] = std::sqrt(hN[2 * j]) / std::sqrt(hN[2 * j + 1]);
    for (int j = 0; j < b; j++)
      if (!std::isfinite(res[j]))
        return set_err(PC_ENUMERIC, "pc_bands: non-finite residual at iteration " + std::to_string(it) +
                                        " (column " + std::to_string(j) + ")");
    const int wlim = nw;
    for (int j = 0; j < b; j++) {
      c->hist.push_back(res[j]);
      // soft locking: a converged column leaves the search block (no W, P); with sticky_lock = 0 it
      // re-enters if its residual rises above tol again
      if (!(res[j] > tol)) active[j] = 0;
      else if (!c->sticky_lock) active[j] = 1;
      // guard columns beyond nev + w_guard never get a search direction (they ride along in X and P)
      if (j >= wlim) active[j] = 0;
      if (j < nev && !(res[j] <= tol)) conv = 0;
    }
    if (c->verbose) {
      fprintf(stderr, "[pcband] k%d it %d rank %d chol %d sweeps %d |X|-1 %.1e rr-cycles %d %d %d %d %d res:",
              kidx, it, rank, hInfo[2], hInfo[1], xdev, hInfo[3], hInfo[4], hInfo[5], hInfo[6], hInfo[7]);
      for (int j = 0; j < b; j++) fprintf(stderr, " %.2e%s", res[j], active[j] ? "" : "*");
      fprintf(stderr, "\n");
    }
    // Ritz pairs not trusted (X^H X drifted from I): one more step with a full Gram, which
    // re-orthonormalises X, before the convergence test may stop the solve
    if (force_full && it < maxit) {
      conv = 0;
      bool any = false;
      for (int j = 0; j < wlim; j++) any |= active[j] != 0;
      if (!any)  // every search column is locked: re-open them for this step (W from one residual pass)
        for (int j = 0; j < wlim; j++) active[j] = 1;
    }
    if (conv || it >= maxit) break;
    std::vector<int> act;
    for (int j = 0; j < b; j++)
      if (active[j]) act.push_back(j);
    const int na = (int)act.size();
    if (na == 0) break;
    std::vector<int> actP, miss;
    for (int j : act) {
      if (!trim || hasP[j]) actP.push_back(j);
      if (!hasW[j]) miss.push_back(j);
    }
    if (!miss.empty()) {  // re-activated columns: W = K_P^{-1} (AX - X Lambda) for them only
      Prof pf(c, PC_STAT_RESID, st, 2, 84.0 * c->n3 * b, 16.0 * len * (2 * b + (double)miss.size()));
      ColPtrs X, AX;
      MutColPtrs W;
      ccols(sX, all, X, 0);
      ccols(sAX, all, AX, 0);
      for (int j = 0; j < b; j++) W.p[j] = nullptr;
      for (int j : miss) W.p[j] = col(WW, j);
      launch_resid(X, AX, W, dLam, b, c->n, c->d_ktab, c->cur_gamma, c->cur_thr, deflate ? 1 : 0, dPart, dNorm, st);
      for (int j : miss) hasW[j] = 1;
    }
    const int nP = (int)actP.size();
    int pa = 1;  // 0: W preconditioned and AW applied by the fused 9-pass sequence
    if (c->precond == 1 && c->precond_fuse) {
      MutColPtrs y, ay, w;
      mcols(WW, act, y, 0);
      mcols(AWW, act, ay, 0);
      for (size_t t = 0; t < act.size(); t++) w.p[t] = wsp.p[t];
      pa = precond_apply_fused(c, y, ay, w, na, st);
      if (pa < 0) return pa;
    }
    if (pa) {
      if (c->precond == 1) CHK(precond_list(WW, act));
      CHK(apply_list(WW, AWW, act));
    }
    int p = 0;
    for (int attempt = 0; attempt < 2; attempt++) {
      p = b + na + (haveP ? nP : 0);
      const int cw = p - b;  // |W| + |P|
      ColPtrs S, T;
      ccols(sX, all, S, 0);
      ccols(WW, act, S, b);
      if (haveP) ccols(sP, actP, S, b + na);
      const bool full = force_full || (c->gram_refresh > 0 && (it % c->gram_refresh) == c->gram_refresh - 1);
      if (full) {  // periodic full Gram S^H [S AS]: no assumption on X (guards against drift)
        for (int t = 0; t < p; t++) T.p[t] = S.p[t];
        ccols(sAX, all, T, p);
        ccols(AWW, act, T, p + b);
        if (haveP) ccols(sAP, actP, T, p + b + na);
        Prof pf(c, PC_STAT_GRAM, st, 2, 8.0 * len * p * 2 * p, 16.0 * len * 2 * p);
        launch_gram(S, p, T, 2 * p, len, dG, c->gpart.as<cplx>(), st);
      } else {
        // only the blocks that are not known: S^H [W P AW AP]; X^H X = I and X^H A X = Lambda hold for
        // the Ritz vectors X of the previous step, the rest follows by Hermitian symmetry
        for (int t = 0; t < cw; t++) T.p[t] = S.p[b + t];
        ccols(AWW, act, T, cw);
        if (haveP) ccols(sAP, actP, T, cw + na);
        Prof pf(c, PC_STAT_GRAM, st, 3, 8.0 * len * p * 2 * cw, 16.0 * len * (p + cw));
        launch_gram(S, p, T, 2 * cw, len, dGp, c->gpart.as<cplx>(), st);
        launch_gram_assemble(dGp, dLam, b, cw, dG, st);
      }
      rank = rr(p);
      if (rank < 0) return rank;
      if (rank >= p || (rank >= b && !c->p_restart)) break;
      if (rank >= b && !haveP) break;
      if (!haveP) return set_err(PC_ENUMERIC, "pc_bands: Rayleigh-Ritz basis collapsed (rank " +
                                                  std::to_string(rank) + " < " + std::to_string(b) + ")");
      haveP = false;  // restart without the P block
    }
    // updates: P' = [W P] C_wp (phase 1), X' = S C (phase 2); same for A-images.  P' only for the
    // columns that can receive W (the others never use P).
    {
      ColPtrs S, AS;
      MutColPtrs Y1, Y2, Y1a, Y2a;
      ccols(sX, all, S, 0);
      ccols(WW, act, S, b);
      if (haveP) ccols(sP, actP, S, b + na);
      ccols(sAX, all, AS, 0);
      ccols(AWW, act, AS, b);
      if (haveP) ccols(sAP, actP, AS, b + na);
      mcols(sPn, all, Y1, 0);
      mcols(sXn, all, Y2, 0);
      mcols(sAPn, all, Y1a, 0);
      mcols(sAXn, all, Y2a, 0);
      std::vector<char> wr(b, 0);  // columns that get W', P', AP' from this update
      for (int j = 0; j < nw; j++) wr[j] = 1;
      if (trim) {
        for (int j = 0; j < b; j++) wr[j] = 0;
        for (int j : act) wr[j] = 1;
      }
      for (int j = 0; j < b; j++) {
        if (!wr[j]) Y1.p[j] = Y1a.p[j] = nullptr;
        hasP[j] = wr[j];
      }
      if (c->fuse_resid) {
        // both updates + the next residual R = AX' - X' Lambda', W = K_P^{-1} R (each row tile's W is
        // read into shared memory by the S phase before the same CTA overwrites it), |R|^2, |X'|^2
        Prof pf(c, PC_STAT_UPDATE, st, 2, 2 * 8.0 * len * p * b + 84.0 * c->n3 * b,
                16.0 * len * (2 * p + 2 * (b + nw) + nw));
        MutColPtrs W;
        mcols(WW, all, W, 0);
        for (int j = 0; j < b; j++) {
          if (!wr[j]) W.p[j] = nullptr;
          hasW[j] = wr[j];
        }
        int g = -1;
        if (c->update_tmap && update_tmap_supported(c->n, b)) {
          // basis blocks as column ranges of the X, W and P slots (holes = soft-locked columns)
          UtBlocks blk;
          memset(&blk, 0, sizeof(blk));
          blk.ld = len;
          const int slotS[3] = {sX, WW, sP}, slotA[3] = {sAX, AWW, sAP};
          const std::vector<int>* lists[3] = {&all, &act, &actP};
          const int rowoff[3] = {0, b, b + na};
          for (int kb = 0; kb < 3; kb++) {
            const std::vector<int>& L = *lists[kb];
            if (L.empty() || (kb == 2 && !haveP)) continue;
            blk.s[kb] = col(slotS[kb], 0);
            blk.as[kb] = col(slotA[kb], 0);
            blk.slot_cols[kb] = b;
            blk.c0[kb] = L.front();
            blk.nc[kb] = L.back() - L.front() + 1;
            for (int j = 0; j < 32; j++) blk.crow[kb][j] = -1;
            for (size_t t = 0; t < L.size(); t++) blk.crow[kb][L[t] - L.front()] = (signed char)(rowoff[kb] + t);
          }
          g = launch_update_tmap(blk, dC, p, b, Y1, Y2, Y1a, Y2a, W, dLam, c->n, c->d_ktab, c->cur_gamma,
                                 c->cur_thr, deflate ? 1 : 0, dPart, rg, st);
        }
        if (g < 0)
          g = launch_update_all(S, AS, p, dC, p, b, b, Y1, Y2, Y1a, Y2a, W, dLam, c->n, c->d_ktab, c->cur_gamma,
                                c->cur_thr, deflate ? 1 : 0, dPart, rg, st);
        launch_reduce_partial(dPart, g, b, dNorm, st);
        resid_ready = true;
      } else {
        Prof pf(c, PC_STAT_UPDATE, st, 2, 2 * 8.0 * len * p * b, 2 * 16.0 * len * (p + b + nw));
        launch_update(S, p, dC, p, b, b, &Y1, Y2, nullptr, len, st);
        launch_update(AS, p, dC, p, b, b, &Y1a, Y2a, nullptr, len, st);
      }
    }
    std::swap(sX, sXn);
    std::swap(sAX, sAXn);
    std::swap(sP, sPn);
    std::swap(sAP, sAPn);
    haveP = true;
  }
  // outputs
  c->have_prev = 1;
  c->prev_slot = sX;
  c->prev_b = b;
  cudaMemcpyAsync(hN + 2 * b, dLam, b * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (evec_out) {
    ColPtrs X;
    MutColPtrs Y;
    for (int j = 0; j < nev; j++) {
      X.p[j] = col(sX, j);
      Y.p[j] = evec_out + (size_t)j * len;
    }
    c->launches += 1;
    normalize_copy_kernel<<<dim3(148 * 2, nev), 256, 0, st>>>(X, dNorm, Y, len);
  }
  CU(cudaStreamSynchronize(st));
  CU(cudaGetLastError());
  if (c->profile) prof_flush(c);
  for (int j = 0; j < nev; j++) {
    omega2[j] = hN[2 * b + j];
    if (resid) resid[j] = res[j];
  }
  if (iters) *iters = it;
  if (status) *status = conv ? 0 : 1;
  return conv ? PC_OK : PC_ENOTCONV;
}


// ------------------------------------------------------------------------------------------
// Batched LOBPCG (k as an extra column dimension).  K k-points run the solve_k algorithm in
// lock step on one context: per iteration ONE host synchronisation for all residual norms and ONE for all
// Rayleigh-Ritz ranks (instead of two per k-point), and the operator applies of every k-point's active W
// columns run as ONE multi-k apply (per-column symbol tables, apply_fourier with MultiK); the Gram,
// Rayleigh-Ritz and update launches stay per k-point (their blocks are per k).  Same arithmetic as
// solve_k for each k-point (the multi-k apply computes each column exactly as a one-k apply), so the
// results equal K separate solves.  Not with warm_start or the eps-weighted preconditioner.
// ------------------------------------------------------------------------------------------
struct KSolve {
  cudaStream_t stm = nullptr;  // this k-point's stream
  double k[3];
  int kidx = 0;
  bool deflate = false;
  double gamma = 0.0, thr = 0.0;
  const cplx* kt = nullptr;
  cplx* base = nullptr;
  int sX, sAX, sXn, sAXn, sP, sAP, sPn, sAPn;
  cplx *dG, *dGp, *dC, *dScr;
  double *dLam, *dNorm, *dPart;
  int* dInfo;
  double* hN;
  int* hInfo;
  std::vector<char> active, hasW, hasP;
  std::vector<double> res;
  std::vector<int> act, actP;
  bool haveP = false, resid_ready = false, force_full = false, running = true;
  int it = 0, conv = 0, rank = 0, p = 0, na = 0, nP = 0;
};

static int solve_batch(pc_ctx* c, const double* kpts, int K, int kidx0, int nev, double tol, int maxit,
                       unsigned long long seed, double* omega2, double* resid, int* iters, int* status,
                       cplx* evec_out) {
  cudaStream_t st = c->stream;
  const int b = nev + c->guard;
  const long long len = c->len;
  const int maxp = 3 * b;
  if (K * b > PC_MAXCOLS) return set_err(PC_EINVAL, "pc_bands: kbatch x block > 192 columns");
  const size_t colb = (size_t)len * sizeof(cplx);
  CHK(c->lob.ensure((size_t)K * 10 * b * colb));
  CHK(ensure_ws(c, K * b));
  const size_t nG = (size_t)maxp * 2 * maxp, nC = (size_t)maxp * b, nScr = (size_t)3 * 80 * 80;
  const int rg = resid_grid(c->n);
  const size_t per_small = ((2 * nG + nC + nScr) * sizeof(cplx) + (size_t)(3 * b + rg * b * 2) * sizeof(double) +
                            8 * sizeof(int) + 255) / 256 * 256;
  CHK(c->small.ensure(per_small * K));
  const size_t gpb = (gram_partial_bytes(maxp, 2 * maxp) + 255) / 256 * 256;
  CHK(c->gpart.ensure(gpb * K));  // one Gram split-K partial buffer per k-point (per-k streams run concurrently)
  const size_t hper = 3 * (size_t)b + 8;  // doubles per k: 2b norms, b Ritz values, 8 ints (4 doubles) + pad
  if (c->h_batch_n < hper * K + (size_t)b) {
    if (c->h_batch) cudaFreeHost(c->h_batch);
    c->h_batch = nullptr;
    c->h_batch_n = 0;
    if (cudaMallocHost(&c->h_batch, (hper * PC_MAXK + b) * sizeof(double)) != cudaSuccess)
      return set_err(PC_ENOMEM, "pc_bands: pinned batch buffer");
    c->h_batch_n = hper * PC_MAXK + b;
  }
  const int nw = (c->w_guard >= 0) ? std::min(b, nev + c->w_guard) : b;
  const bool trim = c->trim_locked != 0;
  // per-k streams: k-point i's own launches run on bst[i], so those of different k-points overlap (at
  // n <= 64 one k-point's kernels fill a fraction of the GPU); the multi-k applies run on the context
  // stream between an event join and an event fork
  while ((int)c->bst.size() < K) {
    cudaStream_t s_;
    cudaEvent_t e_;
    if (cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking) != cudaSuccess) return set_err(PC_ECUDA, "batch streams");
    cudaEventCreateWithFlags(&e_, cudaEventDisableTiming);
    c->bst.push_back(s_);
    c->bev.push_back(e_);
  }
  cudaEvent_t ev_main = nullptr;
  if (c->bev.size() < (size_t)K + 1) {
    cudaEvent_t e_;
    cudaEventCreateWithFlags(&e_, cudaEventDisableTiming);
    c->bev.push_back(e_);
  }
  ev_main = c->bev[K];
  auto join = [&]() {  // context stream waits for every per-k stream
    for (int i = 0; i < K; i++) {
      cudaEventRecord(c->bev[i], c->bst[i]);
      cudaStreamWaitEvent(st, c->bev[i], 0);
    }
  };
  auto fork = [&]() {  // every per-k stream waits for the context stream
    cudaEventRecord(ev_main, st);
    for (int i = 0; i < K; i++) cudaStreamWaitEvent(c->bst[i], ev_main, 0);
  };
  // per-k symbol tables (multi-k buffer), penalties, thresholds
  MultiK mk;
  {
    std::vector<int> kc(K);
    for (int i = 0; i < K; i++) kc[i] = i;
    CHK(build_multik(c, kpts, K, kc.data(), K, mk, st));
  }
  fork();
  enum { XA = 0, AXA, XB, AXB, PA, APA, PB, APB, WW, AWW };
  std::vector<KSolve> ks(K);
  for (int i = 0; i < K; i++) {
    KSolve& s = ks[i];
    for (int a = 0; a < 3; a++) s.k[a] = kpts[3 * i + a];
    s.kidx = kidx0 + i;
    s.deflate = (s.k[0] == 0.0 && s.k[1] == 0.0 && s.k[2] == 0.0);
    s.gamma = mk.gamma[i];
    s.thr = mk.thr[i];
    s.kt = c->mkbuf.as<cplx>() + (size_t)i * 9 * c->n;
    s.stm = c->bst[i];
    s.base = c->lob.as<cplx>() + (size_t)i * 10 * b * len;
    s.sX = XA; s.sAX = AXA; s.sXn = XB; s.sAXn = AXB; s.sP = PA; s.sAP = APA; s.sPn = PB; s.sAPn = APB;
    char* sm = reinterpret_cast<char*>(c->small.p) + per_small * i;
    s.dG = reinterpret_cast<cplx*>(sm);
    s.dGp = s.dG + nG;
    s.dC = s.dGp + nG;
    s.dScr = s.dC + nC;
    s.dLam = reinterpret_cast<double*>(s.dScr + nScr);
    s.dNorm = s.dLam + b;
    s.dPart = s.dNorm + 2 * b;
    s.dInfo = reinterpret_cast<int*>(s.dPart + (size_t)rg * b * 2);
    s.hN = c->h_batch + hper * i;
    s.hInfo = reinterpret_cast<int*>(s.hN + 3 * b);
    s.active.assign(b, 1);
    s.hasW.assign(b, 0);
    s.hasP.assign(b, 0);
    s.res.assign(b, 0.0);
  }
  auto col = [&](const KSolve& s, int slot, int j) { return s.base + ((size_t)slot * b + j) * len; };
  auto gpart_of = [&](const KSolve& s) {
    return reinterpret_cast<cplx*>(reinterpret_cast<char*>(c->gpart.p) + gpb * (size_t)(&s - ks.data()));
  };
  std::vector<int> all(b);
  for (int j = 0; j < b; j++) all[j] = j;
  auto sync = [&](const char* what) -> int {
    join();
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(PC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    if (c->profile) prof_flush(c);
    return PC_OK;
  };
  auto rr_launch = [&](KSolve& s, int p) {
    {
      Prof pf(c, PC_STAT_RR, s.stm, 1, 16.0 * 8.0 * 8.0 * (double)p * p * p, 0.0);
      launch_rr(s.dG, p, b, c->drop_tol, s.dC, s.dLam, s.dInfo, s.dScr, s.stm);
    }
    cudaMemcpyAsync(s.hInfo, s.dInfo, 8 * sizeof(int), cudaMemcpyDeviceToHost, s.stm);
  };
  // one multi-k apply over a list of (k-state, source column, destination column)
  MutColPtrs wsp;
  for (int j = 0; j < K * b; j++) wsp.p[j] = c->ws.as<cplx>() + (size_t)j * len;
  auto apply_batch = [&](const std::vector<std::pair<const cplx*, cplx*>>& cols, const std::vector<int>& kof) -> int {
    if (cols.empty()) return PC_OK;
    ColPtrs x;
    MutColPtrs y;
    MultiK m = mk;
    for (size_t t = 0; t < cols.size(); t++) {
      x.p[t] = cols[t].first;
      y.p[t] = cols[t].second;
      m.kcol[t] = (unsigned char)kof[t];
    }
    join();
    const int rc = apply_fourier(c, x, y, wsp, (int)cols.size(), st, nullptr, &m);
    fork();
    return rc;
  };

  // ---- start blocks (as solve_k), their applies in one multi-k launch, Rayleigh-Ritz per k
  for (KSolve& s : ks) {
    const bool pw = c->start_mode == 1;
    const bool pre = pw && c->start_precond && c->start_noise > 0.0;
    const double noise = pw ? c->start_noise / std::sqrt((double)len) * (pre ? 4.0 * M_PI * M_PI : 1.0) : 1.0;
    Prof pf(c, PC_STAT_OTHER, s.stm, pw ? (pre ? 4 : 3) : 1, 0.0, 16.0 * len * b);
    MutColPtrs x0;
    for (int j = 0; j < b; j++) x0.p[j] = col(s, s.sX, j);
    launch_randn(x0, b, len, mix64(seed + 0x100000001ull * (unsigned long long)s.kidx), s.deflate ? (int)c->n3 : 0,
                 noise, s.stm);
    if (pre) {
      ColPtrs xi;
      for (int j = 0; j < b; j++) xi.p[j] = col(s, s.sX, j);
      launch_precond(xi, x0, b, c->n, s.kt, s.gamma, s.thr, s.stm);
    }
    if (pw) {
      CHK(plane_wave_start(c, x0, b, s.stm, s.kt, s.thr));
      CU(cudaStreamSynchronize(s.stm));  // the context's plane-wave scratch is reused by the next k-point
    }
  }
  {
    std::vector<std::pair<const cplx*, cplx*>> cols;
    std::vector<int> kof;
    for (int i = 0; i < K; i++)
      for (int j = 0; j < b; j++) {
        cols.push_back({col(ks[i], ks[i].sX, j), col(ks[i], ks[i].sAX, j)});
        kof.push_back(i);
      }
    CHK(apply_batch(cols, kof));
  }
  for (KSolve& s : ks) {
    ColPtrs S, T;
    for (int j = 0; j < b; j++) {
      S.p[j] = col(s, s.sX, j);
      T.p[j] = col(s, s.sX, j);
      T.p[b + j] = col(s, s.sAX, j);
    }
    {
      Prof pf(c, PC_STAT_GRAM, s.stm, 2, 8.0 * len * b * 2 * b, 16.0 * len * 2 * b);
      launch_gram(S, b, T, 2 * b, len, s.dG, gpart_of(s), s.stm);
    }
    rr_launch(s, b);
  }
  CHK(sync("rayleigh-ritz"));
  for (KSolve& s : ks) {
    s.rank = s.hInfo[0];
    if (s.rank < b) return set_err(PC_ENUMERIC, "pc_bands: start block is rank deficient");
    Prof pf(c, PC_STAT_UPDATE, s.stm, 2, 2 * 8.0 * len * b * b, 2 * 16.0 * len * 2 * b);
    ColPtrs S;
    MutColPtrs Y;
    for (int j = 0; j < b; j++) {
      S.p[j] = col(s, s.sX, j);
      Y.p[j] = col(s, s.sXn, j);
    }
    launch_update(S, b, s.dC, b, b, b, nullptr, Y, nullptr, len, s.stm);
    for (int j = 0; j < b; j++) {
      S.p[j] = col(s, s.sAX, j);
      Y.p[j] = col(s, s.sAXn, j);
    }
    launch_update(S, b, s.dC, b, b, b, nullptr, Y, nullptr, len, s.stm);
    std::swap(s.sX, s.sXn);
    std::swap(s.sAX, s.sAXn);
    for (int sl : {(int)PA, (int)APA, (int)PB, (int)APB})
      CU(cudaMemsetAsync(col(s, sl, 0), 0, (size_t)b * colb, s.stm));
  }

  auto resid_cols = [&](KSolve& s, const std::vector<int>& which) {
    ColPtrs X, AX;
    MutColPtrs W;
    for (int j = 0; j < b; j++) {
      X.p[j] = col(s, s.sX, j);
      AX.p[j] = col(s, s.sAX, j);
      W.p[j] = nullptr;
    }
    for (int j : which) W.p[j] = col(s, WW, j);
    Prof pf(c, PC_STAT_RESID, s.stm, 2, 84.0 * c->n3 * b, 16.0 * len * (2 * b + (double)which.size()));
    launch_resid(X, AX, W, s.dLam, b, c->n, s.kt, s.gamma, s.thr, s.deflate ? 1 : 0, s.dPart, s.dNorm, s.stm);
  };

  for (;;) {
    // residual norms of every running k-point: one synchronisation
    for (KSolve& s : ks) {
      if (!s.running) continue;
      if (!s.resid_ready) {
        std::vector<int> w0;
        for (int j = 0; j < nw; j++) w0.push_back(j);
        resid_cols(s, w0);
        for (int j = 0; j < b; j++) s.hasW[j] = j < nw;
      }
      cudaMemcpyAsync(s.hN, s.dNorm, 2 * b * sizeof(double), cudaMemcpyDeviceToHost, s.stm);
    }
    CHK(sync("lobpcg"));
    int nrun = 0;
    for (KSolve& s : ks) {
      if (!s.running) continue;
      s.conv = 1;
      double xdev = 0.0;
      for (int j = 0; j < b; j++) xdev = std::max(xdev, std::fabs(s.hN[2 * j + 1] - 1.0));
      s.force_full = !(xdev <= c->xdev_tol);
      for (int j = 0; j < b; j++) s.res[j] = std::sqrt(s.hN[2 * j]) / std::sqrt(s.hN[2 * j + 1]);
      for (int j = 0; j < b; j++)
        if (!std::isfinite(s.res[j]))
          return set_err(PC_ENUMERIC, "pc_bands: non-finite residual at iteration " + std::to_string(s.it));
      for (int j = 0; j < b; j++) {
        if (!(s.res[j] > tol)) s.active[j] = 0;
        else if (!c->sticky_lock) s.active[j] = 1;
        if (j >= nw) s.active[j] = 0;
        if (j < nev && !(s.res[j] <= tol)) s.conv = 0;
      }
      if (s.force_full && s.it < maxit) {
        s.conv = 0;
        bool any = false;
        for (int j = 0; j < nw; j++) any |= s.active[j] != 0;
        if (!any)
          for (int j = 0; j < nw; j++) s.active[j] = 1;
      }
      s.act.clear();
      for (int j = 0; j < b; j++)
        if (s.active[j]) s.act.push_back(j);
      if (s.conv || s.it >= maxit || s.act.empty()) {
        s.running = false;
        continue;
      }
      nrun++;
      s.na = (int)s.act.size();
      s.actP.clear();
      std::vector<int> miss;
      for (int j : s.act) {
        if (!trim || s.hasP[j]) s.actP.push_back(j);
        if (!s.hasW[j]) miss.push_back(j);
      }
      if (!miss.empty()) {
        resid_cols(s, miss);
        for (int j : miss) s.hasW[j] = 1;
      }
      s.nP = (int)s.actP.size();
    }
    if (nrun == 0) break;
    // A W for the active columns of every running k-point: one multi-k apply
    {
      std::vector<std::pair<const cplx*, cplx*>> cols;
      std::vector<int> kof;
      for (int i = 0; i < K; i++) {
        if (!ks[i].running) continue;
        for (int j : ks[i].act) {
          cols.push_back({col(ks[i], WW, j), col(ks[i], AWW, j)});
          kof.push_back(i);
        }
      }
      CHK(apply_batch(cols, kof));
    }
    // Grams and Rayleigh-Ritz of every running k-point: one synchronisation
    for (KSolve& s : ks) {
      if (!s.running) continue;
      s.p = b + s.na + (s.haveP ? s.nP : 0);
      const int cw = s.p - b;
      ColPtrs S, T;
      for (int j = 0; j < b; j++) S.p[j] = col(s, s.sX, j);
      for (int t = 0; t < s.na; t++) S.p[b + t] = col(s, WW, s.act[t]);
      if (s.haveP)
        for (int t = 0; t < s.nP; t++) S.p[b + s.na + t] = col(s, s.sP, s.actP[t]);
      const bool full = s.force_full || (c->gram_refresh > 0 && (s.it % c->gram_refresh) == c->gram_refresh - 1);
      if (full) {
        for (int t = 0; t < s.p; t++) T.p[t] = S.p[t];
        for (int j = 0; j < b; j++) T.p[s.p + j] = col(s, s.sAX, j);
        for (int t = 0; t < s.na; t++) T.p[s.p + b + t] = col(s, AWW, s.act[t]);
        if (s.haveP)
          for (int t = 0; t < s.nP; t++) T.p[s.p + b + s.na + t] = col(s, s.sAP, s.actP[t]);
        Prof pf(c, PC_STAT_GRAM, s.stm, 2, 8.0 * len * s.p * 2 * s.p, 16.0 * len * 2 * s.p);
        launch_gram(S, s.p, T, 2 * s.p, len, s.dG, gpart_of(s), s.stm);
      } else {
        for (int t = 0; t < cw; t++) T.p[t] = S.p[b + t];
        for (int t = 0; t < s.na; t++) T.p[cw + t] = col(s, AWW, s.act[t]);
        if (s.haveP)
          for (int t = 0; t < s.nP; t++) T.p[cw + s.na + t] = col(s, s.sAP, s.actP[t]);
        Prof pf(c, PC_STAT_GRAM, s.stm, 3, 8.0 * len * s.p * 2 * cw, 16.0 * len * (s.p + cw));
        launch_gram(S, s.p, T, 2 * cw, len, s.dGp, gpart_of(s), s.stm);
        launch_gram_assemble(s.dGp, s.dLam, b, cw, s.dG, s.stm);
      }
      rr_launch(s, s.p);
    }
    CHK(sync("rayleigh-ritz"));
    for (KSolve& s : ks) {
      if (!s.running) continue;
      s.rank = s.hInfo[0];
      // rank deficient with P: restart this k-point without the P block (rare; its own synchronisation)
      while (!(s.rank >= s.p || (s.rank >= b && !c->p_restart) || (s.rank >= b && !s.haveP))) {
        if (!s.haveP)
          return set_err(PC_ENUMERIC, "pc_bands: Rayleigh-Ritz basis collapsed (rank " + std::to_string(s.rank) +
                                          " < " + std::to_string(b) + ")");
        s.haveP = false;
        s.p = b + s.na;
        const int cw = s.na;
        ColPtrs S, T;
        for (int j = 0; j < b; j++) S.p[j] = col(s, s.sX, j);
        for (int t = 0; t < s.na; t++) {
          S.p[b + t] = col(s, WW, s.act[t]);
          T.p[t] = S.p[b + t];
          T.p[cw + t] = col(s, AWW, s.act[t]);
        }
        {
          Prof pf(c, PC_STAT_GRAM, s.stm, 3, 8.0 * len * s.p * 2 * cw, 16.0 * len * (s.p + cw));
          launch_gram(S, s.p, T, 2 * cw, len, s.dGp, gpart_of(s), s.stm);
          launch_gram_assemble(s.dGp, s.dLam, b, cw, s.dG, s.stm);
        }
        rr_launch(s, s.p);
        CHK(sync("rayleigh-ritz"));
        s.rank = s.hInfo[0];
      }
    }
    // updates (+ next residual, W = K_P^{-1} R) per k-point
    for (KSolve& s : ks) {
      if (!s.running) continue;
      std::vector<char> wr(b, 0);
      for (int j = 0; j < nw; j++) wr[j] = 1;
      if (trim) {
        for (int j = 0; j < b; j++) wr[j] = 0;
        for (int j : s.act) wr[j] = 1;
      }
      MutColPtrs Y1, Y2, Y1a, Y2a, W;
      for (int j = 0; j < b; j++) {
        Y1.p[j] = wr[j] ? col(s, s.sPn, j) : nullptr;
        Y2.p[j] = col(s, s.sXn, j);
        Y1a.p[j] = wr[j] ? col(s, s.sAPn, j) : nullptr;
        Y2a.p[j] = col(s, s.sAXn, j);
        W.p[j] = wr[j] ? col(s, WW, j) : nullptr;
        s.hasP[j] = wr[j];
        s.hasW[j] = wr[j];
      }
      Prof pf(c, PC_STAT_UPDATE, s.stm, 2, 2 * 8.0 * len * s.p * b + 84.0 * c->n3 * b,
              16.0 * len * (2 * s.p + 2 * (b + nw) + nw));
      int g = -1;
      if (c->update_tmap && update_tmap_supported(c->n, b)) {
        UtBlocks blk;
        memset(&blk, 0, sizeof(blk));
        blk.ld = len;
        const int slotS[3] = {s.sX, WW, s.sP}, slotA[3] = {s.sAX, AWW, s.sAP};
        const std::vector<int>* lists[3] = {&all, &s.act, &s.actP};
        const int rowoff[3] = {0, b, b + s.na};
        for (int kb = 0; kb < 3; kb++) {
          const std::vector<int>& L = *lists[kb];
          if (L.empty() || (kb == 2 && !s.haveP)) continue;
          blk.s[kb] = col(s, slotS[kb], 0);
          blk.as[kb] = col(s, slotA[kb], 0);
          blk.slot_cols[kb] = b;
          blk.c0[kb] = L.front();
          blk.nc[kb] = L.back() - L.front() + 1;
          for (int j = 0; j < 32; j++) blk.crow[kb][j] = -1;
          for (size_t t = 0; t < L.size(); t++) blk.crow[kb][L[t] - L.front()] = (signed char)(rowoff[kb] + t);
        }
        g = launch_update_tmap(blk, s.dC, s.p, b, Y1, Y2, Y1a, Y2a, W, s.dLam, c->n, s.kt, s.gamma, s.thr,
                               s.deflate ? 1 : 0, s.dPart, rg, s.stm);
      }
      if (g < 0) {
        ColPtrs S, AS;
        for (int j = 0; j < b; j++) {
          S.p[j] = col(s, s.sX, j);
          AS.p[j] = col(s, s.sAX, j);
        }
        for (int t = 0; t < s.na; t++) {
          S.p[b + t] = col(s, WW, s.act[t]);
          AS.p[b + t] = col(s, AWW, s.act[t]);
        }
        if (s.haveP)
          for (int t = 0; t < s.nP; t++) {
            S.p[b + s.na + t] = col(s, s.sP, s.actP[t]);
            AS.p[b + s.na + t] = col(s, s.sAP, s.actP[t]);
          }
        g = launch_update_all(S, AS, s.p, s.dC, s.p, b, b, Y1, Y2, Y1a, Y2a, W, s.dLam, c->n, s.kt, s.gamma, s.thr,
                              s.deflate ? 1 : 0, s.dPart, rg, s.stm);
      }
      launch_reduce_partial(s.dPart, g, b, s.dNorm, s.stm);
      s.resid_ready = true;
      std::swap(s.sX, s.sXn);
      std::swap(s.sAX, s.sAXn);
      std::swap(s.sP, s.sPn);
      std::swap(s.sAP, s.sAPn);
      s.haveP = true;
      s.it++;
    }
  }
  // outputs
  int rc = PC_OK;
  for (int i = 0; i < K; i++) {
    KSolve& s = ks[i];
    cudaMemcpyAsync(s.hN + 2 * b, s.dLam, b * sizeof(double), cudaMemcpyDeviceToHost, s.stm);
    if (evec_out) {
      ColPtrs X;
      MutColPtrs Y;
      for (int j = 0; j < nev; j++) {
        X.p[j] = col(s, s.sX, j);
        Y.p[j] = evec_out + ((size_t)i * nev + j) * len;
      }
      c->launches += 1;
      normalize_copy_kernel<<<dim3(148 * 2, nev), 256, 0, s.stm>>>(X, s.dNorm, Y, len);
    }
  }
  CHK(sync("lobpcg"));
  for (int i = 0; i < K; i++) {
    KSolve& s = ks[i];
    for (int j = 0; j < nev; j++) {
      omega2[(size_t)i * nev + j] = s.hN[2 * b + j];
      if (resid) resid[(size_t)i * nev + j] = s.res[j];
    }
    if (iters) iters[i] = s.it;
    if (status) status[i] = s.conv ? 0 : 1;
    if (!s.conv) rc = PC_ENOTCONV;
  }
  c->have_prev = 0;
  return rc;
}

extern "C" int pc_bands(pc_ctx* c, const double* kpts, int nk, int nev, double tol, int maxit,
                        unsigned long long seed, double* omega2, double* resid, int* iters, int* status, void* evecs) {
  if (!c || (!kpts && nk > 0) || (!omega2 && nk > 0)) return set_err(PC_EINVAL, "pc_bands: null argument");
  if (nk < 0 || nev < 1 || !(tol > 0) || maxit < 0) return set_err(PC_EINVAL, "pc_bands: bad sizes/tol");
  const int b = nev + c->guard;
  if (3 * b > 80) return set_err(PC_EINVAL, "pc_bands: nev + guard must be <= 26");
  CU(cudaSetDevice(c->device));
  int rc_all = PC_OK;
  if (c->kbatch > 1 && !c->warm_start && c->precond == 0) {
    // k-points in lock step, c->kbatch at a time
    for (int i0 = 0; i0 < nk; i0 += c->kbatch) {
      const int K = std::min(c->kbatch, nk - i0);
      int rc = solve_batch(c, kpts + 3 * i0, K, (int)(c->kindex_offset + i0), nev, tol, maxit, seed,
                           omega2 + (size_t)i0 * nev, resid ? resid + (size_t)i0 * nev : nullptr,
                           iters ? iters + i0 : nullptr, status ? status + i0 : nullptr,
                           evecs ? reinterpret_cast<cplx*>(evecs) + (size_t)i0 * nev * c->len : nullptr);
      if (rc < 0) {  // leave no batch work queued behind an error
        for (auto s_ : c->bst) cudaStreamSynchronize(s_);
        cudaStreamSynchronize(c->stream);
        return rc;
      }
      if (rc == PC_ENOTCONV) rc_all = PC_ENOTCONV;
    }
    return rc_all;
  }
  for (int i = 0; i < nk; i++) {
    cplx* ev = evecs ? reinterpret_cast<cplx*>(evecs) + (size_t)i * nev * c->len : nullptr;
    int st_i = 0, it_i = 0;
    int rc = solve_k(c, kpts + 3 * i, (int)(c->kindex_offset + i), nev, tol, maxit, seed, omega2 + (size_t)i * nev,
                     resid ? resid + (size_t)i * nev : nullptr, &it_i, &st_i, ev);
    if (rc < 0) return rc;
    if (iters) iters[i] = it_i;
    if (status) status[i] = st_i;
    if (rc == PC_ENOTCONV) rc_all = PC_ENOTCONV;
  }
  return rc_all;
}
