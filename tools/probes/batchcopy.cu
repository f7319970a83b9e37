// Probe only: one copy through cudaMemcpyBatchAsync with cudaMemcpyAttributes.flags
// (cudaMemcpyFlagPreferOverlapWithCompute hint), stream-ordered source access.
#include <cuda_runtime.h>

extern "C" int batch_copy(void* dst, void* src, size_t bytes, unsigned flags, void* stream) {
  cudaMemcpyAttributes attr = {};
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  attr.flags = flags;
  size_t idx = 0, fail = 0;
  void* d[1] = {dst};
  void* s[1] = {src};
  size_t n[1] = {bytes};
  return (int)cudaMemcpyBatchAsync(d, s, n, 1, &attr, &idx, 1, &fail, (cudaStream_t)stream);
}
