/*
 * rl_cddt.h — C ABI of the B200-native CDDT range method, beam sensor model
 * and particle-filter step.
 *
 * This is the drop-in boundary for the reference's range-method path
 * (rangelib, /root/reference/proj). Every entry point names the reference
 * interface it replaces (file:line relative to the reference tree). Plain
 * pointers and sizes only: no C++ or torch types cross this boundary, no
 * exceptions escape it. INTEGRATION.md shows the reference-side adapter
 * (a rangelib::RangeMethod subclass, include/rl_cddt_rangemethod.hpp; the
 * particle filter rl_gpu::GpuMcl, include/rl_cddt_mcl.hpp) and the ctypes binding.
 *
 * Conventions
 *  - Geometry is in pixel units, angles in radians counter-clockwise from +x,
 *    cell (x, y) at y * width + x (proj/include/rangelib/grid.hpp:12-16).
 *  - theta_disc is the number of discrete directions over the full circle,
 *    even and >= 4 (RangeMethodConfig, proj/include/rangelib/raycast.hpp:51-64).
 *  - Functions suffixed _batch take DEVICE pointers and run asynchronously on
 *    `stream` (a cudaStream_t; NULL = the handle's own stream, in which case
 *    the call also synchronises before returning). _host variants take host
 *    pointers and return when the results are in host memory.
 *  - Status codes mirror the reference's exceptions; the message of the last
 *    failure on the calling thread is available from rl_last_error().
 *  - Threading follows the reference's single-writer / many-reader contract
 *    (SPEC.md:341): casts (single, batched, from any thread or stream) may run
 *    concurrently on one handle; prune, set_occupancy* and deserialize-style
 *    structure changes need exclusive access; sensor/particle-filter calls on
 *    one handle are serialised internally.
 */
#ifndef RL_CDDT_H
#define RL_CDDT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RL_OK 0
#define RL_EINVAL 1      /* std::invalid_argument (bad theta_disc / max_range / sizes) */
#define RL_ELOGIC 2      /* std::logic_error: edit after prune (cddt.cpp:333) */
#define RL_ERANGE 3      /* std::out_of_range: edit outside the grid (cddt.cpp:334) */
#define RL_ECUDA 4       /* CUDA runtime failure */
#define RL_ENOMEM 5      /* device or host allocation failure */
#define RL_EDEGENERATE 6 /* sensor_update returned false: weights reset to uniform (mcl.cpp:114-117) */
#define RL_EPARSE 7      /* ParseError on a snapshot (cddt.cpp:502-579) */

typedef struct rl_cddt rl_cddt;

typedef struct {
  int32_t width, height, theta_disc, slice_count;
  int32_t pruned, device;
  double max_range, resolution;
  uint64_t rows;         /* bin rows over all slices (sum of SliceProjection::bin_count) */
  uint64_t zero_points;  /* Cddt::zero_point_count (cddt.hpp:193) */
  uint64_t memory_bytes; /* Cddt::memory_bytes accounting (cddt.hpp:200-203) */
  uint64_t device_bytes; /* bytes actually resident on the device for the structure */
  double init_seconds;   /* wall-clock build time, as make_method records (methods.cpp:118-133) */
} rl_cddt_info_t;

/* Message of the last failing call on this thread ("" if none). */
const char *rl_last_error(void);

/* Cddt::Cddt (proj/src/cddt.cpp:136-171) + Cddt::prune (cddt.cpp:281-330) when
 * prune != 0, i.e. make_method(cddt | pcddt, grid, cfg) (methods.cpp:118-133).
 * grid: width*height bytes, nonzero = occupied (host memory). max_range 0 =
 * grid diagonal (raycast.hpp:61-63). device: CUDA ordinal the structure lives on. */
int rl_cddt_create(const uint8_t *grid, int32_t width, int32_t height, double resolution,
                   int32_t theta_disc, double max_range, int32_t prune, int32_t device,
                   rl_cddt **out);
int rl_cddt_destroy(rl_cddt *c);

/* Cddt::prune (cddt.cpp:281-330). Idempotent. */
int rl_cddt_prune(rl_cddt *c);

int rl_cddt_info(const rl_cddt *c, rl_cddt_info_t *out);

/* Cddt::cast (cddt.cpp:271-273) / RangeMethod::cast (methods.hpp:27). */
int rl_cddt_cast(rl_cddt *c, double x, double y, double theta, double *out);

/* Cddt::cast_pair (cddt.cpp:275-279): ranges at theta and theta + pi. */
int rl_cddt_cast_pair(rl_cddt *c, double x, double y, double theta, double *out_fwd,
                      double *out_bwd);

/* Batched Cddt::cast over f32 queries (the batched replacement for the
 * per-query loop of run_batches, proj/src/bench.cpp:86-106). Device pointers.
 * hit_cell (optional): y*width+x of the occupied cell that settled the answer,
 * -1 when the result is max_range without a hit. */
int rl_cddt_cast_batch(rl_cddt *c, const float *x, const float *y, const float *theta,
                       float *out, int32_t *hit_cell, size_t n, void *stream);

/* Same in f64 (x, y, theta widened exactly), with the resolving zero point
 * (global row, index in row) as the reference's MarkSink sees it
 * (cddt.cpp:249, :259). Any of out/hit_cell/res_row/res_idx may be NULL. */
int rl_cddt_cast_batch_f64(rl_cddt *c, const double *x, const double *y, const double *theta,
                           double *out, int32_t *hit_cell, int64_t *res_row, int32_t *res_idx,
                           size_t n, void *stream);

/* Cddt::directional_cast (cddt.cpp:207-269) at explicit direction indices. */
int rl_cddt_directional_batch(rl_cddt *c, const double *x, const double *y, const int32_t *a,
                              double *out, size_t n, void *stream);

/* Host-memory batched casts (the per-query loop of run_batches, proj/src/bench.cpp:86-106,
 * over caller-owned arrays): host -> device copies, kernel and device -> host
 * copies pipelined in chunks over several streams. Page-locked (pinned or
 * registered) buffers are copied directly at full PCIe bandwidth. Pageable
 * buffers (plain vectors) of >= 2^20 queries are staged through a ring of pinned
 * buffers by a few host threads (RL_HOST_COPY_THREADS, default min(8, cores/2))
 * instead of the driver's synchronous bounce copy: about two thirds of the
 * pinned rate. Blocking: results are in `out` on return. */
int rl_cddt_cast_batch_host(rl_cddt *c, const float *x, const float *y, const float *theta,
                            float *out, size_t n);

/* The per-query loop of run_batches (proj/src/bench.cpp:86-106) over an array of
 * n RayQuery {double x, y, theta} (proj/include/rangelib/raycast.hpp:42-49) in
 * host memory, e.g. std::vector<RayQuery>::data(): out[i] = cast(queries[i]),
 * bit for bit. Chunks are pipelined over three streams; a pageable array is
 * staged through pinned buffers by host threads. Blocking. */
int rl_cddt_cast_queries_host(rl_cddt *c, const double *queries, double *out, size_t n);

/* Cddt::set_occupancy (cddt.cpp:332-377). */
int rl_cddt_set_occupancy(rl_cddt *c, int32_t x, int32_t y, int32_t occupied);

/* n edits applied in order with set_occupancy semantics; xy = n (x, y) pairs,
 * occupied = n flags (host memory). The structure afterwards equals a fresh
 * build of the edited grid (proj/tests/test_cddt.cpp:578-604). If edit k is
 * outside the grid, edits [0, k) are applied and RL_ERANGE is returned, as a
 * loop of set_occupancy calls would leave it. */
int rl_cddt_set_occupancy_batch(rl_cddt *c, const int32_t *xy, const uint8_t *occupied,
                                size_t n);

/* Copy the structure to host memory (any pointer may be NULL):
 *   slice_row_base[slice_count+1]  global row index of (slice, 0)
 *   row_off[rows+1]                CSR offsets into zp
 *   zp[zero_points]                concatenation of Cddt::bin(s, r).values()
 *   membership[w*h], grid[w*h]     0/1 bytes */
int rl_cddt_export(const rl_cddt *c, uint32_t *slice_row_base, uint64_t *row_off, float *zp,
                   uint8_t *membership, uint8_t *grid);

/* Snapshot I/O in the reference's binary format (serialize_cddt /
 * deserialize_cddt, cddt.cpp:458-579). rl_cddt_serialize writes at most cap
 * bytes and stores the full size in *size (call with buf NULL to query). */
int rl_cddt_serialize(const rl_cddt *c, uint8_t *buf, size_t cap, size_t *size);
int rl_cddt_deserialize(const uint8_t *buf, size_t n, int32_t device, rl_cddt **out);

/* oracle_cast (proj/src/raycast.cpp:9-16) on the handle's grid: the exact
 * distance to the first occupied cell along a continuous direction, clamped
 * to max_range. Device pointers. cos_t/sin_t (optional, both or neither) give
 * the direction per query — pass glibc cos/sin of the normalised angle for
 * bit parity with the reference; with NULL the device computes sincos(theta)
 * (within 1 ulp of glibc). */
int rl_exact_cast_batch(rl_cddt *c, const double *x, const double *y, const double *theta,
                        const double *cos_t, const double *sin_t, double *out, size_t n,
                        void *stream);

/* lut_build (proj/src/raycast.cpp:62-87) on the handle's grid and max_range:
 * entries[(i * height + y) * width + x] = clamp(llround(oracle_cast(x + 0.5,
 * y + 0.5, i * 2pi / theta_disc)), 0, 65535), written to device memory
 * (2 * width * height * theta_disc bytes). */
int rl_lut_build(rl_cddt *c, int32_t theta_disc, uint16_t *entries, void *stream);

/* simulate_scan (proj/src/mcl.cpp:144-154) for n poses at once on the
 * handle's grid: scan[i * nbeams + b] = clamp(oracle_cast(x_i, y_i, theta_i +
 * beam_offset(b), max_range) + noise, 0, max_range), beam_offset as
 * ScanSpec::beam_offset (mcl.hpp:42-51), noise ~ N(0, max(noise_sigma,
 * 1e-12)) from the counter generator (seed, stream_id, pose, beam) — the
 * reference's std::normal_distribution stream is implementation-defined.
 * cos_t/sin_t (optional, n * nbeams each) give each beam's direction as in
 * rl_exact_cast_batch. Device pointers. */
int rl_simulate_scans(rl_cddt *c, const double *x, const double *y, const double *theta,
                      size_t n, int32_t nbeams, double fov, double max_range,
                      double noise_sigma, uint64_t seed, uint64_t stream_id,
                      const double *cos_t, const double *sin_t, double *scan, void *stream);

/* Wait for all work queued on the handle's stream. */
int rl_cddt_sync(rl_cddt *c);

/* Diagnostic (no reference counterpart): the scattered-read ceiling the cast
 * kernels are measured against. Issues about `loads` independent 16-byte reads,
 * each in a random 32-byte sector of the device buffer `buf` (`bytes` long),
 * eight in flight per thread at full occupancy; returns the elapsed device
 * time (*ms) and the reads actually issued (*issued). Synchronous. */
int rl_diag_gather(const void *buf, size_t bytes, size_t loads, void *stream, double *ms,
                   uint64_t *issued);

/* Diagnostic (no reference counterpart): device bounds assertions of a
 * checked build (compiled with -DRL_CHECKED; compute-sanitizer stand-in).
 * *failures = violated assertions on `device` so far, *first_code = the site
 * of the first one (cddt_device.cuh RL_DCHECK codes). A regular build reports
 * 0 failures and first_code 0xFFFFFFFF. Synchronises the device. */
int rl_debug_checks(int32_t device, uint64_t *failures, uint32_t *first_code);

/* ---- beam sensor model and particle filter (proj/src/mcl.cpp) ---- */

/* BeamModelParams (proj/include/rangelib/mcl.hpp:32-40). */
typedef struct {
  double w_hit, w_short, w_max, w_rand, sigma_hit, lambda_short, z_max;
} rl_beam_params_t;

/* beam_likelihood (mcl.cpp:11-40) on the host, for building tables. */
double rl_beam_likelihood(const rl_beam_params_t *p, double expected, double measured);

/* Discretised likelihood table T[m][e] = float(beam_likelihood(e/inv_res,
 * m/inv_res)) for e, m in [0, zdim), written to host memory. */
int rl_beam_table(const rl_beam_params_t *p, int32_t zdim, double inv_res, float *table);

/* sensor_update (mcl.cpp:58-120), fused on the GPU: per particle, nbeams casts
 * at theta + beam_offset(b) (ScanSpec, mcl.hpp:42-51), likelihood per beam,
 * FP64 log-sum, max-subtract, exp, normalise. Device pointers:
 *   px, py, pt [n]  particle poses (f64, as rangelib::Particle, mcl.hpp:11-16)
 *   scan [nbeams]   measured ranges (f64)
 *   table           NULL = analytic beam_likelihood with *params; otherwise
 *                   zdim*zdim f32 T[m][e] indexed by clamp(iround(r*inv_res))
 *   logw, weight [n] outputs (f64); either may be NULL.
 * Returns RL_EDEGENERATE (weights set to 1/n) where the reference returns false. */
int rl_sensor_update(rl_cddt *c, const double *px, const double *py, const double *pt, size_t n,
                     const double *scan, int32_t nbeams, double fov, const rl_beam_params_t *params,
                     const float *table, int32_t zdim, double inv_res, double *logw, double *weight,
                     void *stream);

/* ---- particle-filter step (Mcl::step, mcl.cpp:189-201), stage by stage so a
 * multi-GPU driver can place its collectives between stages. All pointers are
 * device pointers; `stream` as above. Random numbers are counter-based
 * (Philox4x32-10 keyed by seed, counter = (particle index, draw, iteration)),
 * so a particle's noise does not depend on how particles are sharded. ---- */

/* MotionNoise (mcl.hpp:18-27). */
typedef struct {
  double trans_per_trans, trans_per_rot, rot_per_rot, rot_per_trans;
} rl_motion_noise_t;

/* motion_update (mcl.cpp:42-56): sigma_t = a|trans| + b|rot|, sigma_r =
 * c|rot| + d|trans| (floored at 1e-12), per particle three normals (rdx, rdy,
 * rdtheta) applied in the robot frame. index_offset is the global index of
 * particle 0 of this shard. */
int rl_motion_update(double *x, double *y, double *theta, size_t n, uint64_t index_offset,
                     double dx, double dy, double dtheta, const rl_motion_noise_t *noise,
                     uint64_t seed, uint64_t iteration, void *stream);

/* Log-weights only (the first half of sensor_update): logw[i] = sum over beams
 * of log likelihood, beams in order. Arguments as rl_sensor_update. */
int rl_sensor_logw(rl_cddt *c, const double *px, const double *py, const double *pt, size_t n,
                   const double *scan, int32_t nbeams, double fov, const rl_beam_params_t *params,
                   const float *table, int32_t zdim, double inv_res, double *logw, void *stream);

/* out[0] = max over logw[0, n) (device). */
int rl_pf_max(const double *logw, size_t n, double *out, void *stream);

/* w[i] = exp(logw[i] - *gmax); moments[0..9] = {sum w, sum w x, sum w y,
 * sum w cos t, sum w sin t, n, sum x, sum y, sum cos t, sum sin t} over this
 * shard (deterministic order). */
int rl_pf_weights(const double *logw, const double *gmax, const double *x, const double *y,
                  const double *theta, size_t n, double *w, double *moments, void *stream);

/* Normalise with the global sum moments[0] (mcl.cpp:108-119): w /= sum, or
 * w = 1/n_total and *degenerate = 1 when the sum is zero or not finite. */
int rl_pf_normalize(double *w, size_t n, const double *moments, uint64_t n_total,
                    int32_t *degenerate, void *stream);

/* resample_low_variance (mcl.cpp:122-142) over the full set (x, y, theta, w)
 * of n particles: r = U[0, 1/n) from the counter RNG, slot m takes the first
 * particle whose cumulative weight reaches r + m/n. Writes the slots
 * [out_begin, out_begin + out_count) with weight 1/n. */
int rl_resample_low_variance(const double *x, const double *y, const double *theta,
                             const double *w, size_t n, size_t out_begin, size_t out_count,
                             double *ox, double *oy, double *otheta, double *ow, uint64_t seed,
                             uint64_t iteration, void *stream);

/* Whole Mcl::step on one GPU: motion -> sensor -> estimate -> resample, with
 * the particle arrays updated in place. estimate (host, 3 doubles) receives
 * the weighted mean pose (Mcl::estimate, mcl.cpp:176-187) before resampling;
 * returns RL_EDEGENERATE when the weights were reset. */
int rl_mcl_step(rl_cddt *c, double *x, double *y, double *theta, double *w, size_t n,
                double odo_dx, double odo_dy, double odo_dtheta, const double *scan,
                int32_t nbeams, double fov, const rl_motion_noise_t *noise,
                const rl_beam_params_t *params, const float *table, int32_t zdim, double inv_res,
                uint64_t seed, uint64_t iteration, double *estimate, void *stream);

/* ---- asynchronous forms (no host synchronisation; for pipelined and
 * multi-GPU drivers). `stream` must be non-NULL; successive sensor /
 * particle-filter calls on one handle must use one stream (they share the
 * handle's workspace in stream order). ---- */

/* rl_sensor_update without the read-back: the degenerate flag (1 where the
 * reference's sensor_update returns false, mcl.cpp:114-117) is written to the
 * device int32 *degenerate. */
int rl_sensor_update_async(rl_cddt *c, const double *px, const double *py, const double *pt,
                           size_t n, const double *scan, int32_t nbeams, double fov,
                           const rl_beam_params_t *params, const float *table, int32_t zdim,
                           double inv_res, double *logw, double *weight, int32_t *degenerate,
                           void *stream);

/* rl_mcl_step without the read-back: the estimate (Mcl::estimate,
 * mcl.cpp:176-187, computed on the device) goes to the device buffer
 * estimate_dev = {x, y, theta, degenerate (0.0 / 1.0)}. */
int rl_mcl_step_async(rl_cddt *c, double *x, double *y, double *theta, double *w, size_t n,
                      double odo_dx, double odo_dy, double odo_dtheta, const double *scan,
                      int32_t nbeams, double fov, const rl_motion_noise_t *noise,
                      const rl_beam_params_t *params, const float *table, int32_t zdim,
                      double inv_res, uint64_t seed, uint64_t iteration, double *estimate_dev,
                      void *stream);

/* ---- the sharded Mcl::step (one process per GPU). Per step:
 *   rl_pf_shard_sensor -> all-reduce MAX(local_max) -> rl_pf_weights ->
 *   all-reduce SUM(moments) -> rl_pf_normalize -> rl_pf_estimate ->
 *   all-gather {x, y, theta, w} -> rl_resample_gathered
 * with no host synchronisation between the stages. ---- */

/* motion_update (mcl.cpp:42-56; skipped when noise is NULL) fused with the
 * sensor model's log-weights (mcl.cpp:64-103) for this rank's shard
 * (global indices [index_offset, index_offset + n)); *local_max (device) =
 * max over the shard's log-weights, -inf for an empty shard. */
int rl_pf_shard_sensor(rl_cddt *c, double *x, double *y, double *theta, size_t n,
                       uint64_t index_offset, double odo_dx, double odo_dy, double odo_dtheta,
                       const rl_motion_noise_t *noise, uint64_t seed, uint64_t iteration,
                       const double *scan, int32_t nbeams, double fov,
                       const rl_beam_params_t *params, const float *table, int32_t zdim,
                       double inv_res, double *logw, double *local_max, void *stream);

/* Mcl::estimate (mcl.cpp:176-187) from the all-reduced moments of
 * rl_pf_weights and the flag of rl_pf_normalize (may be NULL: not degenerate),
 * on the device: estimate_dev = {x, y, theta, degenerate}. */
int rl_pf_estimate(const double *moments, const int32_t *degenerate, uint64_t n_total,
                   double *estimate_dev, void *stream);

/* resample_low_variance (mcl.cpp:122-142) read straight from an all-gather
 * of per-rank shards: gathered = [world][4][n_local] doubles, rank-major, each
 * rank's block {x[n_local], y[n_local], theta[n_local], w[n_local]} (the
 * rank-concatenated output of ncclAllGather). Same comb and output slots as
 * rl_resample_low_variance over the concatenated set. */
int rl_resample_gathered(const double *gathered, size_t n_local, int32_t world, size_t out_begin,
                         size_t out_count, double *ox, double *oy, double *otheta, double *ow,
                         uint64_t seed, uint64_t iteration, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* RL_CDDT_H */
