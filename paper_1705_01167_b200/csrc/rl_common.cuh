// Host-side plumbing shared by the CUDA translation units: error state,
// CUDA checks, device buffers, and the handle layout.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rl_cddt.h"
#include "cddt_device.cuh"

namespace rl {

void set_error(const char* fmt, ...);

// Exception-free CUDA check: records the message and returns RL_ECUDA.
#define RL_CK(call)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      ::rl::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));    \
      return e_ == cudaErrorMemoryAllocation ? RL_ENOMEM : RL_ECUDA;                         \
    }                                                                                        \
  } while (0)

#define RL_TRY(expr)          \
  do {                        \
    int st_ = (expr);         \
    if (st_ != RL_OK) return st_; \
  } while (0)

// Owning device allocation (cudaMalloc / cudaFree on the current device).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  int alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      set_error("cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
      return RL_ENOMEM;
    }
    n = count;
    return RL_OK;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Makes `dev` current for the lifetime of the guard.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace rl

namespace rl {
// checked builds: the device violation counter of `dev` (nullptr otherwise)
unsigned long long* check_counter(int dev);
}  // namespace rl

// The opaque handle (include/rl_cddt.h). Owns the device copy of the flags
// and the CSR structure on one device, plus host mirrors of the grid and
// membership (small: w*h bytes) that drive incremental edits.
struct rl_cddt {
  int dev = 0;
  bool counted = false;  // registered with the scratch pool (handle_opened)
  cudaStream_t stream = nullptr;
  int w = 0, h = 0, K = 0, S = 0;
  double max_range = 0.0, resolution = 0.05;
  bool pruned = false;
  double init_seconds = 0.0;

  std::vector<double> dcos, dsin;      // K, host glibc (cddt.cpp:30-42)
  std::vector<rl::SliceParam> slices;  // S
  uint64_t rows = 0, zero_points = 0;

  std::vector<uint8_t> grid_h;    // host mirror: occupancy
  std::vector<uint8_t> member_h;  // host mirror: membership
  bool mirror_stale = false;      // edits ran on the device since the mirrors were filled

  rl::DevBuf<uint8_t> flags;        // w*h
  rl::DevBuf<uint2> rowbits;        // row-major occupancy/clear bits for queries
  int wpr = 0;
  rl::DevBuf<uint32_t> row_off;     // rows+1
  rl::DevBuf<float> hints;          // rows x kHintFloats: row records (cddt_device.cuh)
  rl::DevBuf<float> zp;             // capacity >= zero_points
  rl::DevBuf<rl::SliceParam> d_slices;
  rl::DevBuf<double4> d_dirs;   // cos, sin, 1/cos, 1/sin
  rl::DevBuf<double4> d_pdirs;  // per direction: slice cos, slice sin, cos, sin (batch phase 1)
  rl::DevBuf<uint32_t> d_rbase;  // S slice row bases (batch phase 1)
  rl::DevBuf<double> d_scalar;      // scratch for single-query calls
  rl::DevBuf<uint8_t> ws;           // reusable workspace (sensor model reductions)
  rl::DevBuf<uint8_t> sensor_ctl;   // sensor_update's fused normalisation: {max key, ticket, flag}
  bool sensor_ctl_clean = false;    // its key and ticket are zero (every completed launch leaves them so)
  std::mutex mu;                    // serialises users of d_scalar / ws / pf_* / the handle stream
  rl::DevBuf<uint8_t> pf_ctl;       // fused PF step: {max key, ticket} | moments (zeroed when dirty)
  bool pf_ctl_clean = false;        // the max key is 0 (every completed step leaves it so)
  void* pf_host = nullptr;          // fused PF step: pinned host copy of the moments
  uint32_t* host_small = nullptr;   // 64 pinned bytes for small read-backs (flags, counts)
  rl::DevBuf<uint8_t> upd_ws;       // incremental edits: scratch
  rl::DevBuf<uint8_t> upd_up;       // incremental edits: the uploaded batch
  void* upd_host = nullptr;         // incremental edits: pinned staging for the uploads
  size_t upd_host_n = 0;
  rl::DevBuf<float> zp_spare;       // incremental edits: double buffer for zp
  rl::DevBuf<uint32_t> off_spare;   // incremental edits: double buffer for row_off
  // Slack rows (set by the first edit batch, rl_update.cu): row g owns
  // row_cap[g] slots of zp from row_off[g] (no longer monotone once rows move
  // to the append area) and stores row_len[g] points there, so later edit
  // batches merge only the rows they touch. Build, prune and load leave the
  // rows dense (gapped = false, no row_len / row_cap).
  bool gapped = false;
  uint64_t zp_slots = 0;            // slots in use (rows + append area used): zero_points when dense
  uint64_t slot_limit = 0;          // gapped: slots the append area may grow to (<= zp.n)
  rl::DevBuf<uint32_t> row_len;     // gapped: points per row
  rl::DevBuf<uint32_t> row_cap;     // gapped: slots per row
  rl::DevBuf<uint32_t> len_spare;   // incremental edits: double buffers for row_len / row_cap
  rl::DevBuf<uint32_t> cap_spare;
  rl::DevBuf<uint8_t> bkt;          // incremental edits: per-row delta buckets (zeroed counts)
  rl::DevBuf<uint32_t> estamp;      // incremental edits: per-cell (generation, edit) stamps
  rl::DevBuf<uint32_t> wstamp;      // incremental edits: per-cell dilation stamps
  uint32_t edit_gen = 0;

  rl::CddtView view() const {
    rl::CddtView v;
    v.flags = flags.p;
    v.rowbits = rowbits.p;
    v.wpr = wpr;
    v.row_off = row_off.p;
    v.zp = zp.p;
    v.hints = hints.p;
    v.slices = d_slices.p;
    v.dirs = d_dirs.p;
    v.pdirs = d_pdirs.p;
    v.rbase = d_rbase.p;
    v.w = w;
    v.h = h;
    v.K = K;
    v.S = S;
    v.max_range = max_range;
    v.chk = rl::check_counter(dev);
    v.n_rows = uint32_t(rows);
    v.n_zp = uint32_t(gapped ? zp_slots : zero_points);
    return v;
  }
};

namespace rl {
int sm_count();
inline cudaStream_t pick_stream(const rl_cddt* c, void* s) {
  return s ? static_cast<cudaStream_t>(s) : c->stream;
}
int finish(const rl_cddt* c, void* s);  // sync when the caller passed no stream
int refresh_query_bits(rl_cddt* c);     // rebuild the query occupancy bits from flags
int refresh_row_hints(rl_cddt* c);      // rebuild the row search hints from row_off / zp
int densify_rows(rl_cddt* c);           // slack rows back to dense CSR (rl_update.cu)
int refresh_mirrors(const rl_cddt* c);  // host grid/membership mirrors from the device flags
// stream-ordered scratch from the library's own per-device pool (rl_cddt.cu)
int scratch_alloc(void** p, size_t bytes, cudaStream_t st);
int scratch_free(void* p, cudaStream_t st);
void handle_opened(int dev);  // pool bookkeeping: live handles per device
void handle_closed(int dev);
// Structure changes (prune, set_occupancy*) rewrite arrays that casts already
// queued on caller streams may still read: wait for all work on the device
// first. Casts are asynchronous on any stream, so only a device-wide
// synchronisation orders them before the change.
inline int quiesce(const rl_cddt*) {
  RL_CK(cudaDeviceSynchronize());
  return RL_OK;
}
// 16 pinned u32 for small device->host read-backs (a pageable destination
// would add a staging copy to every synchronous step)
inline int host_small(rl_cddt* c, uint32_t** out) {
  if (!c->host_small) {
    const cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&c->host_small), 64);
    if (e != cudaSuccess) {
      c->host_small = nullptr;
      set_error("cudaMallocHost(64): %s", cudaGetErrorString(e));
      return RL_ENOMEM;
    }
  }
  *out = c->host_small;
  return RL_OK;
}
}  // namespace rl
