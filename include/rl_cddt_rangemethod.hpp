// rl_cddt_rangemethod.hpp — the reference-side binding of the C ABI.
//
// A rangelib::RangeMethod (proj/include/rangelib/methods.hpp:22-50) whose
// queries run on the GPU through include/rl_cddt.h. Existing callers of the
// reference — Mcl (proj/src/mcl.cpp:156-201), sensor_update (:58-120),
// run_batches (proj/src/bench.cpp:71-150), the CLI — take it unchanged:
//
//   #include "rl_cddt_rangemethod.hpp"
//   auto m = std::make_unique<rl_gpu::GpuCddtMethod>(grid, cfg, /*prune=*/true);
//   rangelib::Mcl mcl(*m, mcl_cfg);          // unchanged reference code
//
// Header-only; needs the reference headers on the include path and
// librl_cddt.so at link time. Status codes become the reference's exception
// types (std::invalid_argument, std::logic_error, std::out_of_range,
// rangelib::ParseError).
#pragma once

#include <chrono>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rangelib/grid.hpp"
#include "rangelib/methods.hpp"
#include "rangelib/raycast.hpp"
#include "rl_cddt.h"

namespace rl_gpu {

inline void throw_on(int status) {
  if (status == RL_OK || status == RL_EDEGENERATE) return;
  const std::string msg = rl_last_error();
  switch (status) {
    case RL_EINVAL: throw std::invalid_argument(msg);
    case RL_ELOGIC: throw std::logic_error(msg);
    case RL_ERANGE: throw std::out_of_range(msg);
    case RL_EPARSE: throw rangelib::ParseError(msg, 0);
    default: throw std::runtime_error(msg);
  }
}

class GpuCddtMethod final : public rangelib::RangeMethod {
 public:
  // make_method(cddt | pcddt, grid, cfg) (proj/src/methods.cpp:118-133)
  GpuCddtMethod(const rangelib::OccupancyGrid& grid, const rangelib::RangeMethodConfig& cfg,
                bool prune, int device = 0) {
    cfg.validate();
    auto t0 = std::chrono::steady_clock::now();
    std::vector<uint8_t> cells(size_t(grid.width()) * grid.height());
    for (int y = 0; y < grid.height(); y++)
      for (int x = 0; x < grid.width(); x++) cells[size_t(y) * grid.width() + x] = grid.at(x, y);
    throw_on(rl_cddt_create(cells.data(), grid.width(), grid.height(), grid.resolution(),
                            cfg.theta_disc, cfg.max_range, prune ? 1 : 0, device, &h_));
    rl_cddt_info_t info;
    throw_on(rl_cddt_info(h_, &info));
    max_range_ = info.max_range;
    theta_disc_ = info.theta_disc;
    pruned_ = info.pruned != 0;
    memory_ = size_t(info.memory_bytes);
    set_init_seconds(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  ~GpuCddtMethod() override { rl_cddt_destroy(h_); }
  GpuCddtMethod(const GpuCddtMethod&) = delete;
  GpuCddtMethod& operator=(const GpuCddtMethod&) = delete;

  const char* name() const override { return pruned_ ? "pcddt" : "cddt"; }

  double cast(const rangelib::RayQuery& q) const override {
    double r = 0.0;
    throw_on(rl_cddt_cast(h_, q.x, q.y, q.theta, &r));
    return r;
  }
  std::pair<double, double> cast_pair(const rangelib::RayQuery& q) const override {
    double f = 0.0, b = 0.0;
    throw_on(rl_cddt_cast_pair(h_, q.x, q.y, q.theta, &f, &b));
    return {f, b};
  }
  bool supports_paired_cast() const override { return true; }
  int direction_count() const override { return theta_disc_; }
  size_t memory_bytes() const override { return memory_; }

  // The batched extension the reference lacks: n f32 queries from host memory.
  void cast_batch(const float* x, const float* y, const float* theta, float* out, size_t n) const {
    throw_on(rl_cddt_cast_batch_host(h_, x, y, theta, out, n));
  }
  // run_batches' inner loop (proj/src/bench.cpp:86-106) as one call: out[i] = cast(q[i])
  void cast_many(const rangelib::RayQuery* q, size_t n, double* out) const {
    static_assert(sizeof(rangelib::RayQuery) == 3 * sizeof(double), "RayQuery is {x, y, theta}");
    throw_on(rl_cddt_cast_queries_host(h_, reinterpret_cast<const double*>(q), out, n));
  }
  // Cddt::set_occupancy (proj/src/cddt.cpp:332-377)
  void set_occupancy(int x, int y, bool occupied) {
    throw_on(rl_cddt_set_occupancy(h_, x, y, occupied ? 1 : 0));
  }
  rl_cddt* handle() const { return h_; }

 private:
  rl_cddt* h_ = nullptr;
  int theta_disc_ = 0;
  bool pruned_ = false;
  size_t memory_ = 0;
};

}  // namespace rl_gpu
