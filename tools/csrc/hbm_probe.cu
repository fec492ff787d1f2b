// hbm_probe.cu -- measurement aid for bench.py (NOT part of the product):
// a pure HBM read stream, to give read-only kernels (the reductions) a
// read-only roofline next to MEASURED_PEAKS.json's copy bandwidth.
//
// Persistent grid (blocks_per_sm x SMs), 512 threads, each thread issuing
// UNROLL independent 16-byte streaming loads per iteration; the XOR of
// everything is written per block so the loads cannot be elided.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr int kThreads = 512;
constexpr int kUnroll = 8;

__global__ void __launch_bounds__(kThreads) read_stream(const uint4* __restrict__ p, long long nv,
                                                        uint32_t* __restrict__ sink) {
  uint32_t acc = 0;
  const long long stride = static_cast<long long>(gridDim.x) * kThreads;
  long long i = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  for (; i + (kUnroll - 1) * stride < nv; i += kUnroll * stride) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < nv; i += stride) {
    const uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicXor(sink + blockIdx.x, acc);
}
}  // namespace

extern "C" int hbm_read_stream(const void* p, long long bytes, void* sink, int blocks,
                               void* stream) {
  if (!p || !sink || bytes < 16 || (reinterpret_cast<uintptr_t>(p) & 15) || blocks < 1) return 1;
  read_stream<<<blocks, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint4*>(p), bytes / 16, reinterpret_cast<uint32_t*>(sink));
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
