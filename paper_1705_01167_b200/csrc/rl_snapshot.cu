// Binary snapshot in the reference's format: serialize_cddt / deserialize_cddt
// (proj/src/cddt.cpp:458-579). Little-endian: magic "CDDT", u32 version 1,
// u32 width, height, theta_disc, u8 pruned, u8 storage, 2 pad bytes, f64
// max_range, f64 resolution, occupancy bitmap, membership bitmap, then per
// slice u32 bin count and per bin u32 n + n ascending f32. Round-trips
// bit-exactly with the reference, so CPU-built (or CPU-pruned) structures
// load onto the GPU and GPU-built ones diff byte-for-byte against reference
// dumps.
#include <cmath>
#include <cstring>
#include <limits>

#include "rl_common.cuh"

namespace rl {
int init_geometry(rl_cddt* c);
int create_handle(int32_t device, rl_cddt** out, rl_cddt** keep);

namespace {

void put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; i++) b.push_back(uint8_t(v >> (8 * i)));
}
void put_f64(std::vector<uint8_t>& b, double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  for (int i = 0; i < 8; i++) b.push_back(uint8_t(u >> (8 * i)));
}

struct Reader {
  const uint8_t* b;
  size_t n, pos = 0;
  bool need(size_t k, const char* what) {
    if (pos + k > n) {
      set_error("cddt snapshot truncated reading %s (byte %zu)", what, pos);
      return false;
    }
    return true;
  }
  uint32_t u32() {
    uint32_t v = 0;
    for (int i = 0; i < 4; i++) v |= uint32_t(b[pos + i]) << (8 * i);
    pos += 4;
    return v;
  }
  double f64() {
    uint64_t u = 0;
    for (int i = 0; i < 8; i++) u |= uint64_t(b[pos + i]) << (8 * i);
    pos += 8;
    double v;
    std::memcpy(&v, &u, 8);
    return v;
  }
};

}  // namespace
}  // namespace rl

using namespace rl;

extern "C" {

int rl_cddt_serialize(const rl_cddt* c, uint8_t* buf, size_t cap, size_t* size) {
  if (!c || !size) return RL_EINVAL;
  const size_t wh = size_t(c->w) * c->h;
  std::vector<uint32_t> off32;
  std::vector<float> zp(c->zero_points);
  std::vector<uint64_t> off(c->rows + 1);
  RL_TRY(rl_cddt_export(c, nullptr, off.data(), zp.data(), nullptr, nullptr));
  {
    DeviceGuard guard(c->dev);
    RL_TRY(refresh_mirrors(c));  // the grid and membership bitmaps below
  }
  std::vector<uint8_t> out;
  out.reserve(64 + 2 * ((wh + 7) / 8) + 4 * c->zero_points + 4 * c->rows + 4 * c->S);
  out.push_back('C');
  out.push_back('D');
  out.push_back('D');
  out.push_back('T');
  put_u32(out, 1);
  put_u32(out, uint32_t(c->w));
  put_u32(out, uint32_t(c->h));
  put_u32(out, uint32_t(c->K));
  out.push_back(c->pruned ? 1 : 0);
  out.push_back(0);  // BinStorage::sorted_vector (both modes build identical bins)
  out.push_back(0);
  out.push_back(0);
  put_f64(out, c->max_range);
  put_f64(out, c->resolution);
  auto put_bitmap = [&](const std::vector<uint8_t>& cells) {
    std::vector<uint8_t> bits((wh + 7) / 8, 0);
    for (size_t i = 0; i < wh; i++)
      if (cells[i]) bits[i / 8] |= uint8_t(1u << (i % 8));
    out.insert(out.end(), bits.begin(), bits.end());
  };
  put_bitmap(c->grid_h);
  put_bitmap(c->member_h);
  uint64_t g = 0;
  for (int s = 0; s < c->S; s++) {
    put_u32(out, uint32_t(c->slices[s].bin_count));
    for (int r = 0; r < c->slices[s].bin_count; r++, g++) {
      const uint64_t a = off[g], b = off[g + 1];
      put_u32(out, uint32_t(b - a));
      const size_t at = out.size();
      out.resize(at + 4 * (b - a));
      if (b > a) std::memcpy(out.data() + at, zp.data() + a, 4 * (b - a));
    }
  }
  *size = out.size();
  if (buf && cap >= out.size()) std::memcpy(buf, out.data(), out.size());
  return RL_OK;
}

int rl_cddt_deserialize(const uint8_t* bytes, size_t n, int32_t device, rl_cddt** out) {
  if (!out) return RL_EINVAL;
  *out = nullptr;
  Reader r{bytes, bytes ? n : 0};
  if (!r.need(4, "magic")) return RL_EPARSE;
  if (bytes[0] != 'C' || bytes[1] != 'D' || bytes[2] != 'D' || bytes[3] != 'T') {
    set_error("cddt snapshot: bad magic (byte 0)");
    return RL_EPARSE;
  }
  r.pos = 4;
  if (!r.need(4, "version")) return RL_EPARSE;
  if (r.u32() != 1) {
    set_error("cddt snapshot: unsupported version (byte 4)");
    return RL_EPARSE;
  }
  if (!r.need(12, "header")) return RL_EPARSE;
  const uint32_t w = r.u32(), h = r.u32(), K = r.u32();
  if (w == 0 || h == 0 || w > (1u << 20) || h > (1u << 20)) {
    set_error("cddt snapshot: implausible grid size (byte 12)");
    return RL_EPARSE;
  }
  if (K < 4 || K % 2 != 0) {
    set_error("cddt snapshot: invalid direction count (byte 20)");
    return RL_EPARSE;
  }
  if (!r.need(4, "flags")) return RL_EPARSE;
  const uint8_t pruned = bytes[r.pos], storage = bytes[r.pos + 1];
  r.pos += 4;
  if (pruned > 1 || storage > 1) {
    set_error("cddt snapshot: bad flags (byte %zu)", r.pos - 4);
    return RL_EPARSE;
  }
  if (!r.need(16, "scalars")) return RL_EPARSE;
  const double max_range = r.f64(), resolution = r.f64();
  if (!(max_range > 0.0) || !(resolution > 0.0)) {
    set_error("cddt snapshot: bad scalar field (byte %zu)", r.pos - 16);
    return RL_EPARSE;
  }
  const size_t wh = size_t(w) * h, bm = (wh + 7) / 8;
  if (!r.need(bm, "occupancy bitmap")) return RL_EPARSE;
  std::vector<uint8_t> grid(wh), member(wh);
  for (size_t i = 0; i < wh; i++) grid[i] = (bytes[r.pos + i / 8] >> (i % 8)) & 1;
  r.pos += bm;
  if (!r.need(bm, "membership bitmap")) return RL_EPARSE;
  for (size_t i = 0; i < wh; i++) member[i] = (bytes[r.pos + i / 8] >> (i % 8)) & 1;
  r.pos += bm;

  DeviceGuard guard(device);
  rl_cddt* c = nullptr;
  RL_TRY(create_handle(device, out, &c));
  auto fail = [&](int st) {
    std::string msg = rl_last_error();
    rl_cddt_destroy(c);
    set_error("%s", msg.c_str());
    return st;
  };
  c->w = int(w);
  c->h = int(h);
  c->K = int(K);
  c->max_range = max_range;
  c->resolution = resolution;
  c->pruned = pruned != 0;
  c->grid_h = std::move(grid);
  c->member_h = std::move(member);
  int st = init_geometry(c);
  if (st) return fail(st);
  std::vector<uint32_t> off(c->rows + 1);
  std::vector<float> zp;
  uint64_t g = 0;
  for (int s = 0; s < c->S; s++) {
    if (!r.need(4, "bin count")) return fail(RL_EPARSE);
    const uint32_t nb = r.u32();
    if (int(nb) != c->slices[s].bin_count) {
      set_error("cddt snapshot: bin count mismatch (byte %zu)", r.pos - 4);
      return fail(RL_EPARSE);
    }
    for (uint32_t bi = 0; bi < nb; bi++, g++) {
      if (!r.need(4, "zero point count")) return fail(RL_EPARSE);
      const uint32_t k = r.u32();
      if (!r.need(size_t(k) * 4, "zero points")) return fail(RL_EPARSE);
      off[g] = uint32_t(zp.size());
      float prev = -std::numeric_limits<float>::infinity();
      for (uint32_t i = 0; i < k; i++) {
        float v;
        std::memcpy(&v, bytes + r.pos, 4);
        r.pos += 4;
        if (!(v >= prev)) {
          set_error("cddt snapshot: zero points out of order (byte %zu)", r.pos - 4);
          return fail(RL_EPARSE);
        }
        prev = v;
        zp.push_back(v);
      }
    }
  }
  off[c->rows] = uint32_t(zp.size());
  if (r.pos != n) {
    set_error("cddt snapshot: trailing bytes (byte %zu)", r.pos);
    return fail(RL_EPARSE);
  }
  c->zero_points = zp.size();
  c->zp_slots = zp.size();  // dense rows
  c->gapped = false;
  // flags: occupancy and membership from the snapshot, clear mask rebuilt
  // (deserialize_cddt rebuilds it too, cddt.cpp:576-577)
  std::vector<uint8_t> flags(wh, 0);
  for (int y = 0; y < c->h; y++)
    for (int x = 0; x < c->w; x++) {
      const size_t i = size_t(y) * c->w + x;
      bool any = false;
      for (int dy = -1; dy <= 1 && !any; dy++)
        for (int dx = -1; dx <= 1; dx++) {
          const int nx = x + dx, ny = y + dy;
          if (nx >= 0 && ny >= 0 && nx < c->w && ny < c->h && c->grid_h[size_t(ny) * c->w + nx]) {
            any = true;
            break;
          }
        }
      uint8_t f = 0;
      if (c->grid_h[i]) f |= kOcc;
      if (!any) f |= kClear;
      if (c->member_h[i]) f |= kMember;
      flags[i] = f;
    }
  if ((st = c->flags.alloc(wh)) || (st = c->row_off.alloc(c->rows + 1)) ||
      (st = c->zp.alloc(zp.size())))
    return fail(st);
  cudaError_t e = cudaMemcpy(c->flags.p, flags.data(), wh, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(c->row_off.p, off.data(), 4 * off.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !zp.empty())
    e = cudaMemcpy(c->zp.p, zp.data(), 4 * zp.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    set_error("cddt snapshot upload: %s", cudaGetErrorString(e));
    return fail(RL_ECUDA);
  }
  if ((st = refresh_query_bits(c))) return fail(st);
  if ((st = refresh_row_hints(c))) return fail(st);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return fail(RL_ECUDA);
  *out = c;
  return RL_OK;
}

}  // extern "C"
