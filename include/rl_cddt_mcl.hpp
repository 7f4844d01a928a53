// rl_cddt_mcl.hpp — the reference's particle filter (rangelib::Mcl,
// proj/include/rangelib/mcl.hpp:101-127, proj/src/mcl.cpp:156-201) with the
// particles resident on the GPU and each step one call of the C ABI
// (rl_mcl_step: motion, fused sensor model, estimate, low-variance
// resampling). Same constructor arguments, same methods:
//
//   #include "rl_cddt_mcl.hpp"
//   rl_gpu::GpuCddtMethod m(grid, cfg, /*prune=*/false);
//   rl_gpu::GpuMcl filter(m, mcl_cfg);            // was: rangelib::Mcl filter(m, mcl_cfg)
//   filter.init_gaussian(x, y, theta, 2.0, 0.1);
//   rangelib::MclStepResult r = filter.step(dx, dy, dtheta, scan);
//
// Differences a caller can observe: motion noise and the resampling draw come
// from a counter-based generator (Philox4x32-10 keyed by MclConfig::seed;
// std::normal_distribution's stream is implementation-defined), and
// init_gaussian draws on the host with std::mt19937_64 as the reference does.
// An optional likelihood table T[m][e] (f32, zdim x zdim, host memory)
// replaces the analytic beam model. Header-only; needs the reference headers,
// the CUDA runtime and librl_cddt.so at link time.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>
#include <stdexcept>
#include <vector>

#include "rangelib/mcl.hpp"
#include "rl_cddt.h"
#include "rl_cddt_rangemethod.hpp"

namespace rl_gpu {

class GpuMcl {
 public:
  // Mcl::Mcl (mcl.cpp:156-163)
  GpuMcl(const GpuCddtMethod& method, const rangelib::MclConfig& cfg, const float* table = nullptr,
         int zdim = 0, double inv_res = 1.0)
      : method_(method), cfg_(cfg), init_rng_(cfg.seed), zdim_(zdim), inv_res_(inv_res) {
    if (cfg_.particle_count <= 0)
      throw std::invalid_argument("particle filter needs at least one particle");
    if (!(cfg_.beam.z_max > 0.0)) cfg_.beam.z_max = method_.max_range();
    n_ = size_t(cfg_.particle_count);
    alloc(&d_, 4 * n_ + size_t(cfg_.scan.beam_count));
    if (table) {
      alloc(&d_table_, size_t(zdim) * size_t(zdim));
      copy_in(d_table_, table, size_t(zdim) * size_t(zdim) * sizeof(float));
    }
    std::vector<double> init(4 * n_, 0.0);
    std::fill(init.begin() + 3 * n_, init.end(), 1.0 / double(n_));
    copy_in(d_, init.data(), init.size() * sizeof(double));
  }
  ~GpuMcl() {
    cudaFree(d_);
    cudaFree(d_table_);
  }
  GpuMcl(const GpuMcl&) = delete;
  GpuMcl& operator=(const GpuMcl&) = delete;

  // Mcl::init_gaussian (mcl.cpp:165-174), drawn on the host like the reference
  void init_gaussian(double x, double y, double theta, double sigma_xy, double sigma_theta) {
    std::normal_distribution<double> gxy(0.0, std::max(sigma_xy, 1e-12));
    std::normal_distribution<double> gth(0.0, std::max(sigma_theta, 1e-12));
    std::vector<double> h(4 * n_);
    for (size_t i = 0; i < n_; i++) {
      h[i] = x + gxy(init_rng_);
      h[n_ + i] = y + gxy(init_rng_);
      h[2 * n_ + i] = rangelib::normalize_angle_2pi(theta + gth(init_rng_));
      h[3 * n_ + i] = 1.0 / double(n_);
    }
    copy_in(d_, h.data(), h.size() * sizeof(double));
  }

  // Mcl::step (mcl.cpp:189-201): motion -> sensor -> estimate -> resample
  rangelib::MclStepResult step(double odo_dx, double odo_dy, double odo_dtheta,
                               const std::vector<double>& scan) {
    if (int(scan.size()) != cfg_.scan.beam_count)
      throw std::invalid_argument("scan length does not match beam count");  // mcl.cpp:61-62
    auto t0 = std::chrono::steady_clock::now();
    double* scan_d = d_ + 4 * n_;
    copy_in(scan_d, scan.data(), scan.size() * sizeof(double));
    const rl_motion_noise_t noise{cfg_.motion.trans_per_trans, cfg_.motion.trans_per_rot,
                                  cfg_.motion.rot_per_rot, cfg_.motion.rot_per_trans};
    const rangelib::BeamModelParams& b = cfg_.beam;
    const rl_beam_params_t bp{b.w_hit, b.w_short, b.w_max, b.w_rand, b.sigma_hit, b.lambda_short,
                              b.z_max};
    double est[3];
    const int st = rl_mcl_step(method_.handle(), d_, d_ + n_, d_ + 2 * n_, d_ + 3 * n_, n_,
                               odo_dx, odo_dy, odo_dtheta, scan_d, cfg_.scan.beam_count,
                               cfg_.scan.fov, &noise, &bp, d_table_, zdim_, inv_res_, cfg_.seed,
                               iteration_++, est, nullptr);
    if (st != RL_OK && st != RL_EDEGENERATE) throw_on(st);
    rangelib::MclStepResult r;
    r.estimate = {est[0], est[1], est[2]};
    r.degenerate = st == RL_EDEGENERATE;
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    last_ = r.estimate;
    return r;
  }

  // Mcl::estimate (mcl.cpp:176-187) as of the last step's sensor update
  rangelib::PoseEstimate estimate() const { return last_; }

  // Mcl::particles (mcl.hpp:116), copied to the host
  std::vector<rangelib::Particle> particles() const {
    std::vector<double> h(4 * n_);
    if (cudaMemcpy(h.data(), d_, h.size() * sizeof(double), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
      throw std::runtime_error("cudaMemcpy");
    std::vector<rangelib::Particle> p(n_);
    for (size_t i = 0; i < n_; i++) p[i] = {h[i], h[n_ + i], h[2 * n_ + i], h[3 * n_ + i]};
    return p;
  }

 private:
  template <class T>
  static void alloc(T** p, size_t count) {
    if (cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<size_t>(count, 1)) !=
        cudaSuccess)
      throw std::runtime_error("cudaMalloc");
  }
  static void copy_in(void* dst, const void* src, size_t bytes) {
    if (cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("cudaMemcpy");
  }

  const GpuCddtMethod& method_;
  rangelib::MclConfig cfg_;
  std::mt19937_64 init_rng_;
  size_t n_ = 0;
  double* d_ = nullptr;  // x[n] | y[n] | theta[n] | weight[n] | scan[beams]
  float* d_table_ = nullptr;
  int zdim_ = 0;
  double inv_res_ = 1.0;
  uint64_t iteration_ = 0;
  rangelib::PoseEstimate last_;
};

}  // namespace rl_gpu
