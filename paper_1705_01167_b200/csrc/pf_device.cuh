// Device pieces of the particle-filter step shared by the motion, sensor and
// resampling kernels: the Philox4x32-10 counter generator, one particle's
// motion_update (proj/src/mcl.cpp:42-56) and an order-preserving integer key
// for the atomic max of the log-weights.
#pragma once
#include <cstdint>

#include "cddt_device.cuh"

namespace rl {

// Philox4x32-10 (Salmon et al., SC'11): counter (c0..c3), key (k0, k1).
struct U4 {
  uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// two uniforms in [0, 1) with 53 random bits each
__device__ __forceinline__ void philox_uniform2(uint64_t seed, uint32_t i, uint32_t draw,
                                                uint64_t iter, double& u0, double& u1) {
  const U4 r = philox4x32_10(U4{i, draw, uint32_t(iter), uint32_t(iter >> 32)}, uint32_t(seed),
                             uint32_t(seed >> 32));
  const uint64_t a = (uint64_t(r.y) << 32) | r.x, b = (uint64_t(r.w) << 32) | r.z;
  u0 = double(a >> 11) * 0x1.0p-53;
  u1 = double(b >> 11) * 0x1.0p-53;
}

constexpr uint32_t kResampleStream = 0xFFFFFFFFu;

// One step of motion_update for the odometry (dx, dy, dth) with noise
// standard deviations (st, sr): draws 0 and 1 of particle gi at iteration
// `iter` give three Box-Muller normals (rdx, rdy, rdth order, mcl.cpp:49-51).
struct MotionArgs {
  double dx, dy, dth, st, sr;
  uint64_t seed, iter, index_offset;
};

__device__ __forceinline__ void motion_one(const MotionArgs& m, uint32_t gi, double& x, double& y,
                                           double& t) {
  double a0, a1, b0, b1;
  philox_uniform2(m.seed, gi, 0, m.iter, a0, a1);
  philox_uniform2(m.seed, gi, 1, m.iter, b0, b1);
  // Box-Muller on (0, 1] x [0, 1)
  const double ra = sqrt(-2.0 * log(1.0 - a0)), rb = sqrt(-2.0 * log(1.0 - b0));
  double sa, ca, sb, cb;
  sincos(kTwoPi * a1, &sa, &ca);
  sincos(kTwoPi * b1, &sb, &cb);
  const double n0 = ra * ca, n1 = ra * sa, n2 = rb * cb;
  (void)sb;
  // motion_update (mcl.cpp:49-55)
  const double rdx = m.dx + m.st * n0, rdy = m.dy + m.st * n1, rdt = m.dth + m.sr * n2;
  double s, c;
  sincos(t, &s, &c);
  x += rdx * c - rdy * s;
  y += rdx * s + rdy * c;
  t = normalize_angle_2pi(t + rdt);
}

// Monotone map double -> u64 (total order for non-NaN values, -inf lowest
// among them), so a max over doubles is an integer atomicMax. Key 0 is below
// every encoded double and serves as the empty state.
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long u = __double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double order_key_value(unsigned long long k) {
  return __longlong_as_double((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k);
}

}  // namespace rl
