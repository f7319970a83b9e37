// Probe only (not part of libppo_b200): SM-driven host-link copy -- a persistent kernel
// streams 16-byte vectors between device memory and mapped pinned host memory, to compare
// its link rate and its interference with compute against the copy engines.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void smcopy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

extern "C" int smcopy(const void* src, void* dst, size_t bytes, int blocks, int threads, void* stream) {
  smcopy_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, bytes / 16);
  return (int)cudaGetLastError();
}
