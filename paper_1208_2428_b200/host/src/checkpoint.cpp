// Checkpoint / resume (see fhp_b200/checkpoint.hpp for the file layout).
#include "fhp_b200/checkpoint.hpp"

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>

namespace fhp_b200 {

namespace {

template <class T>
void put(std::vector<std::uint8_t>& out, std::size_t off, T v) {
  std::memcpy(out.data() + off, &v, sizeof v);  // little-endian host (x86-64 / aarch64)
}
template <class T>
T get(const std::vector<std::uint8_t>& in, std::size_t off) {
  T v;
  std::memcpy(&v, in.data() + off, sizeof v);
  return v;
}

}  // namespace

std::uint64_t fnv1a64(const std::uint8_t* p, std::size_t n) noexcept {
  std::uint64_t h = 0xCBF29CE484222325ull;
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

Checkpoint capture_checkpoint(const Engine& e, std::int64_t next_step, std::uint64_t seed,
                              double force_p, std::uint64_t swaps, const CollisionTable& table) {
  if (e.row_begin() != 0 || e.row_end() != e.height())
    throw std::invalid_argument("checkpoint: engine is a row strip; capture each strip's rows");
  Checkpoint c;
  c.width = e.width();
  c.height = e.height();
  c.next_step = next_step;
  c.seed = seed;
  c.force_p = force_p;
  c.swaps = swaps;
  c.table = table;
  c.state.resize(static_cast<std::size_t>(c.width) * c.height);
  e.download(c.state.data(), static_cast<std::size_t>(c.width));
  return c;
}

void restore_checkpoint(Engine& e, const Checkpoint& c) {
  if (e.width() != c.width || e.height() != c.height)
    throw std::invalid_argument("checkpoint: lattice size does not match the engine");
  std::vector<std::uint8_t> mask(c.state.size());
  for (std::size_t i = 0; i < mask.size(); ++i) mask[i] = c.state[i] >> 7;
  e.set_table(c.table);
  e.set_obstacles(mask.data(), static_cast<std::size_t>(c.width));
  e.upload(c.state.data(), static_cast<std::size_t>(c.width));
}

std::vector<std::uint8_t> serialize_checkpoint(const Checkpoint& c) {
  const std::size_t n = static_cast<std::size_t>(c.width) * c.height;
  if (c.state.size() != n) throw std::invalid_argument("checkpoint: state size != width * height");
  std::vector<std::uint8_t> out(kCheckpointHeader + n);
  std::memcpy(out.data(), kCheckpointMagic, 8);
  put<std::uint32_t>(out, 8, static_cast<std::uint32_t>(c.width));
  put<std::uint32_t>(out, 12, static_cast<std::uint32_t>(c.height));
  put<std::int64_t>(out, 16, c.next_step);
  put<std::uint64_t>(out, 24, c.seed);
  put<double>(out, 32, c.force_p);
  put<std::uint64_t>(out, 40, c.swaps);
  put<std::uint64_t>(out, 48, fnv1a64(c.state.data(), n));
  std::memcpy(out.data() + 56, c.table.entries.data(), 512);
  std::memcpy(out.data() + kCheckpointHeader, c.state.data(), n);
  return out;
}

Checkpoint parse_checkpoint(const std::vector<std::uint8_t>& in) {
  if (in.size() < kCheckpointHeader || std::memcmp(in.data(), kCheckpointMagic, 8) != 0)
    throw std::runtime_error("checkpoint: bad magic (expected FHPCKPT1)");
  Checkpoint c;
  c.width = static_cast<int>(get<std::uint32_t>(in, 8));
  c.height = static_cast<int>(get<std::uint32_t>(in, 12));
  if (c.width < 1 || c.height < 3) throw std::runtime_error("checkpoint: bad lattice size");
  const std::size_t n = static_cast<std::size_t>(c.width) * c.height;
  if (in.size() != kCheckpointHeader + n)
    throw std::runtime_error("checkpoint: file size does not match width * height");
  c.next_step = get<std::int64_t>(in, 16);
  c.seed = get<std::uint64_t>(in, 24);
  c.force_p = get<double>(in, 32);
  c.swaps = get<std::uint64_t>(in, 40);
  std::memcpy(c.table.entries.data(), in.data() + 56, 512);
  c.state.assign(in.begin() + kCheckpointHeader, in.end());
  if (fnv1a64(c.state.data(), n) != get<std::uint64_t>(in, 48))
    throw std::runtime_error("checkpoint: state digest mismatch (corrupt file)");
  return c;
}

void write_checkpoint_file(const std::string& path, const Checkpoint& c) {
  const auto bytes = serialize_checkpoint(c);
  const std::string tmp = path + ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) throw std::runtime_error("cannot write checkpoint " + tmp);
    f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!f) throw std::runtime_error("short write to checkpoint " + tmp);
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0)
    throw std::runtime_error("cannot rename checkpoint to " + path);
}

Checkpoint read_checkpoint_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open checkpoint " + path);
  std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  return parse_checkpoint(bytes);
}

}  // namespace fhp_b200
