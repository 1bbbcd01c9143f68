// api.cuh — host-side helpers shared by the C-ABI translation units (ib_api.cu, slab.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "ib_internal.cuh"

namespace ibk {

// Record msg as the thread's last error (ib_last_error) and return code.
int fail(int code, const std::string &msg);

#define CK(expr)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return ::ibk::fail(e_ == cudaErrorMemoryAllocation ? IB_ENOMEM : IB_ECUDA,    \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));      \
  } while (0)

template <class T>
inline cudaError_t dalloc(T **p, size_t count) {
  return cudaMalloc((void **)p, count * sizeof(T) > 0 ? count * sizeof(T) : 1);
}

inline void dfree(void *p) {
  if (p) cudaFree(p);
}

// Copy count elements from a host-or-device pointer to a host vector.
template <class T>
inline cudaError_t to_host(std::vector<T> &dst, const T *src, size_t count, cudaStream_t s) {
  dst.resize(count);
  if (!count) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(dst.data(), src, count * sizeof(T), cudaMemcpyDefault, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

inline cudaError_t copy_sync(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  if (!bytes) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

int count_nonfinite(ib_ctx *c, const double *d, size_t n, unsigned long long *out);
StructDev struct_dev(const ib_ctx *c);
void free_graph(ib_ctx *c);
Sym sym_of(const ib_ctx *c);
cudaError_t yfwd(ib_ctx *c, cudaStream_t s);
cudaError_t yinv(ib_ctx *c, cudaStream_t s);
cudaError_t xfwd(ib_ctx *c, int mode, const double *u, double *F, unsigned *rowflag,
                 double *r_out, cudaStream_t s);
cudaError_t xinv(ib_ctx *c, double *out, const long long *dev_n, long long n, long long *flag,
                 cudaStream_t s);
cudaError_t ensure_binned(ib_ctx *c, cudaStream_t s);

}  // namespace ibk
