// Common device helpers for libpcband (complex FP64 on double2, error plumbing).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <mutex>
#include <map>
#include <utility>

#define DEV __device__ __forceinline__
#define HD __host__ __device__ __forceinline__

typedef double2 cplx;

// cudaFuncSetAttribute is a per-device setting: the dynamic shared-memory limit of `kern` is raised to
// `bytes` once per (kernel, current device) -- and again whenever a launch needs more than was set.
// (A process-wide "done" flag would leave the kernel without it on a second device used by another
// context, or below a later, larger request; such launches fail with cudaErrorInvalidValue.)
inline cudaError_t smem_attr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({kern, dev});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[{kern, dev}] = bytes;
  return e;
}

HD cplx mk(double r, double i) { return make_double2(r, i); }
HD cplx operator+(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
HD cplx operator-(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
HD cplx operator-(cplx a) { return mk(-a.x, -a.y); }
HD cplx operator*(double s, cplx a) { return mk(s * a.x, s * a.y); }
HD cplx cmul(cplx a, cplx b) { return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)); }
// conj(a) * b
HD cplx cmulc(cplx a, cplx b) { return mk(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x)); }
HD cplx conjg(cplx a) { return mk(a.x, -a.y); }
HD double abs2(cplx a) { return fma(a.x, a.x, a.y * a.y); }
// a + b*c
HD cplx cfma(cplx b, cplx c, cplx a) {
  return mk(fma(b.x, c.x, fma(-b.y, c.y, a.x)), fma(b.x, c.y, fma(b.y, c.x, a.y)));
}
// multiply by i^{dir} where dir = +1 (i) or -1 (-i)
template <int DIR> HD cplx mul_i(cplx a) { return DIR > 0 ? mk(-a.y, a.x) : mk(a.y, -a.x); }

// 16-byte global load/store of one complex (non-coherent read-only path for inputs)
DEV cplx ldg(const cplx* p) { return __ldg(p); }

// cp.async 16 B global -> shared (LDGSTS), bypassing L1
DEV void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
