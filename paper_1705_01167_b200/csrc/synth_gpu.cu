// Device twin of synth_free_queries (csrc/synth.c): the same per-query
// SplitMix64 stream and rejection rule, bit-identical output, so benchmarks can
// produce 100M-query workloads per GPU in milliseconds instead of seconds of
// host time per rank. Harness side only (inputs), not part of the C ABI.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__device__ __forceinline__ uint64_t sm_next(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double sm_uniform(uint64_t* s) {
  return (double)(sm_next(s) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ uint64_t sm_stream(uint64_t seed, uint64_t item) {
  uint64_t s = seed ^ 0x5851f42d4c957f2dull;
  uint64_t a = sm_next(&s);
  s = a + item * 0xd1b54a32d192ed03ull;
  (void)sm_next(&s);
  return s;
}

constexpr double kTwoPi = 6.283185307179586476925286766559;

__global__ void k_free_queries(const uint8_t* __restrict__ g, int w, int h, uint64_t seed,
                               uint64_t i0, uint64_t n, float* __restrict__ qx,
                               float* __restrict__ qy, float* __restrict__ qt) {
  const float fw = (float)w, fh = (float)h;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t s = sm_stream(seed, i0 + k);
    float x, y;
    int tries = 0;
    for (;;) {
      x = (float)(sm_uniform(&s) * w);
      y = (float)(sm_uniform(&s) * h);
      if (x >= fw) x = nextafterf(fw, 0.0f);
      if (y >= fh) y = nextafterf(fh, 0.0f);
      const int cx = (int)floor((double)x), cy = (int)floor((double)y);
      const bool occ = cx >= 0 && cy >= 0 && cx < w && cy < h && g[(size_t)cy * w + cx];
      if (!occ || ++tries >= 1000000) break;
    }
    float t = (float)(sm_uniform(&s) * kTwoPi);
    if ((double)t >= kTwoPi) t = nextafterf(t, 0.0f);
    qx[k] = x;
    qy[k] = y;
    qt[k] = t;
  }
}

}  // namespace

extern "C" int synth_free_queries_gpu(const uint8_t* grid_dev, int w, int h, uint64_t seed,
                                      uint64_t i0, uint64_t n, float* qx, float* qy, float* qt,
                                      void* stream) {
  if (n == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > uint64_t(sms) * 32) blocks = uint64_t(sms) * 32;
  k_free_queries<<<unsigned(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      grid_dev, w, h, seed, i0, n, qx, qy, qt);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
