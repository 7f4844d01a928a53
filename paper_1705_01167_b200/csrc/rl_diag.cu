// Diagnostic: the random-gather ceiling the cast kernels are measured against.
// The cast path is a chain of scattered 32-byte-sector reads; this kernel
// issues the same kind of reads with no dependences between them (eight per
// thread in flight, one sector each, addresses from a hash), so its rate is
// the most the memory system delivers for scattered sectors out of a buffer
// of a given size: L2-resident for a few MB up to ~100 MB, HBM beyond.
#include <algorithm>

#include "rl_common.cuh"

namespace rl {

__device__ __forceinline__ uint32_t mix32(uint32_t h) {  // lowbias32
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}

constexpr int kGatherInFlight = 8;

__global__ void __launch_bounds__(256) k_gather(const uint4* __restrict__ buf, uint32_t nsec,
                                                uint32_t rounds, uint32_t seed,
                                                uint32_t* __restrict__ sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t h[kGatherInFlight];
#pragma unroll
  for (int u = 0; u < kGatherInFlight; u++) h[u] = mix32(t * kGatherInFlight + u + seed);
  uint32_t acc = 0;
  for (uint32_t r = 0; r < rounds; r++) {
#pragma unroll
    for (int u = 0; u < kGatherInFlight; u++) {
      h[u] = mix32(h[u]);
      const uint32_t s = uint32_t((uint64_t(h[u]) * nsec) >> 32);  // a 32-byte sector
      const uint4 v = __ldg(buf + 2 * size_t(s));
      acc ^= v.x ^ v.w;
    }
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);  // keeps the loads live
}

}  // namespace rl

using namespace rl;

extern "C" int rl_diag_gather(const void* buf, size_t bytes, size_t loads, void* stream,
                              double* ms, uint64_t* issued) {
  if (!buf || !ms || !issued || bytes < 32 || bytes / 32 > 0xffffffffull || loads == 0)
    return RL_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, per_sm = 0;
  RL_CK(cudaGetDevice(&dev));
  RL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather, 256, 0));
  const size_t threads = size_t(sm_count()) * size_t(std::max(per_sm, 1)) * 256;
  const uint32_t rounds =
      uint32_t(std::max<size_t>(1, loads / (threads * kGatherInFlight)));
  uint32_t* sink = nullptr;
  RL_TRY(scratch_alloc(reinterpret_cast<void**>(&sink), sizeof(uint32_t), st));
  cudaEvent_t e0, e1;
  RL_CK(cudaEventCreate(&e0));
  RL_CK(cudaEventCreate(&e1));
  const unsigned grid = unsigned(threads / 256);
  const uint32_t nsec = uint32_t(bytes / 32);
  k_gather<<<grid, 256, 0, st>>>(static_cast<const uint4*>(buf), nsec, 1, 7u, sink);  // warm-up
  RL_CK(cudaEventRecord(e0, st));
  k_gather<<<grid, 256, 0, st>>>(static_cast<const uint4*>(buf), nsec, rounds, 11u, sink);
  RL_CK(cudaEventRecord(e1, st));
  RL_CK(cudaEventSynchronize(e1));
  float f = 0.f;
  RL_CK(cudaEventElapsedTime(&f, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  RL_TRY(scratch_free(sink, st));
  RL_CK(cudaStreamSynchronize(st));
  *ms = double(f);
  *issued = uint64_t(threads) * kGatherInFlight * rounds;
  return RL_OK;
}
