// Host file formats of the hot path's inputs and outputs (SURVEY §8a A2, A3,
// A13), so a reference caller can hand the drop-in the same files:
//
//  * partition labels   partition_from_file / write_partition_labels
//                       (/root/reference/proj/src/graph.cpp:461-484, 624-628)
//  * vertex roles       load_roles / write_roles (graph.cpp:600-622)
//  * VIP vectors        write_vip_binary / load_vip_binary (vip.cpp:107-134)
//  * binary CSR writer  write_binary_csr (graph.cpp:553-563); the reader is
//                       vk_graph_load_vcsr (graph.cu)
//
// Text parsing follows the reference line by line: empty and '#' lines are
// skipped, each line's leading decimal digits are the value (std::from_chars,
// so trailing characters are ignored and a leading blank, sign or overflow is
// a format_error naming the file and line).
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "internal.cuh"

namespace vk {
namespace {

template <class T, class Check>
std::vector<T> read_codes(const char* path, const char* what_open, const char* what_bad, Check&& ok) {
  std::ifstream in(path);
  if (!in) raise(VK_ERR_IO, std::string(what_open) + path);
  std::vector<T> out;
  std::string line;
  std::size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty() || line[0] == '#') continue;
    std::uint64_t x = 0;
    using U = std::conditional_t<sizeof(T) <= 4, std::uint32_t, std::uint64_t>;
    U v = 0;
    auto [p, ec] = std::from_chars(line.data(), line.data() + line.size(), v);
    x = v;
    if (ec != std::errc() || !ok(x))
      raise(VK_ERR_FORMAT, std::string(path) + ":" + std::to_string(lineno) + ": " + what_bad);
    out.push_back(static_cast<T>(x));
  }
  return out;
}

template <class T>
void write_lines(const char* path, const T* v, std::uint64_t n) {
  std::FILE* f = std::fopen(path, "wb");
  if (!f) raise(VK_ERR_IO, std::string("cannot write ") + path);
  std::vector<char> buf;
  buf.reserve(1 << 20);
  char tmp[24];
  bool failed = false;
  for (std::uint64_t i = 0; i < n; ++i) {
    auto [e, ec] = std::to_chars(tmp, tmp + sizeof tmp, static_cast<std::uint64_t>(v[i]));
    buf.insert(buf.end(), tmp, e);
    buf.push_back('\n');
    if (buf.size() >= (1 << 20)) {
      failed |= std::fwrite(buf.data(), 1, buf.size(), f) != buf.size();
      buf.clear();
    }
  }
  failed |= std::fwrite(buf.data(), 1, buf.size(), f) != buf.size();
  failed |= std::fclose(f) != 0;
  if (failed) raise(VK_ERR_IO, std::string("write failed: ") + path);
}

}  // namespace
}  // namespace vk

using namespace vk;

extern "C" {

// graph.cpp:461-484 + PartitionMap::from_labels (graph.cpp:88-104)
int vk_partition_from_file(const char* path, uint32_t K, uint64_t n, uint32_t* part_of, uint32_t* K_out) {
  return guard([&] {
    if (!path || !part_of) raise(VK_ERR_PARAMETER, "null argument");
    const auto labels = read_codes<std::uint32_t>(path, "cannot open partition label file: ", "bad partition label",
                                                  [](std::uint64_t) { return true; });
    if (labels.size() != n)
      raise(VK_ERR_FORMAT, std::string(path) + ": expected " + std::to_string(n) + " labels, got " +
                               std::to_string(labels.size()));
    std::uint32_t mx = 0;
    for (std::uint32_t l : labels) mx = std::max(mx, l);
    if (K == 0) K = mx + 1;
    // from_labels: every label < K, every partition non-empty
    std::vector<std::uint8_t> seen(K, 0);
    for (std::uint64_t v = 0; v < n; ++v) {
      if (labels[v] >= K)
        raise(VK_ERR_FORMAT, "partition label " + std::to_string(labels[v]) + " out of range for K=" +
                                 std::to_string(K));
      seen[labels[v]] = 1;
    }
    for (std::uint32_t k = 0; k < K; ++k)
      if (!seen[k]) raise(VK_ERR_PARTITION, "partition " + std::to_string(k) + " is empty");
    std::memcpy(part_of, labels.data(), n * 4);
    if (K_out) *K_out = K;
  });
}

int vk_write_partition_labels(const char* path, const uint32_t* part_of, uint64_t n) {
  return guard([&] {
    if (!path || (!part_of && n)) raise(VK_ERR_PARAMETER, "null argument");
    write_lines(path, part_of, n);
  });
}

int vk_load_roles(const char* path, uint8_t** roles, uint64_t* n) {
  return guard([&] {
    if (!path || !roles || !n) raise(VK_ERR_PARAMETER, "null argument");
    const auto r = read_codes<std::uint8_t>(path, "cannot open roles file: ", "bad role code",
                                            [](std::uint64_t x) { return x <= 3; });
    auto* out = static_cast<std::uint8_t*>(std::malloc(std::max<std::size_t>(1, r.size())));
    if (!out) raise(VK_ERR_INTERNAL, "host allocation failed");
    std::memcpy(out, r.data(), r.size());
    *roles = out;
    *n = r.size();
  });
}

int vk_write_roles(const char* path, const uint8_t* roles, uint64_t n) {
  return guard([&] {
    if (!path || (!roles && n)) raise(VK_ERR_PARAMETER, "null argument");
    write_lines(path, roles, n);
  });
}

// vip.cpp:107-120: n little-endian f64 totals
int vk_write_vip_binary(const char* path, const double* total, uint64_t n) {
  return guard([&] {
    if (!path || (!total && n)) raise(VK_ERR_PARAMETER, "null argument");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) raise(VK_ERR_IO, std::string("cannot write ") + path);
    static_assert(sizeof(double) == 8, "f64");
    bool failed = std::fwrite(total, 8, n, f) != n;  // little-endian host (x86-64 / aarch64)
    failed |= std::fclose(f) != 0;
    if (failed) raise(VK_ERR_IO, std::string("write failed: ") + path);
  });
}

// vip.cpp:122-134: every whole 8-byte record; a trailing partial one is ignored
int vk_load_vip_binary(const char* path, double** values, uint64_t* n) {
  return guard([&] {
    if (!path || !values || !n) raise(VK_ERR_PARAMETER, "null argument");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) raise(VK_ERR_IO, std::string("cannot open ") + path);
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    const std::uint64_t cnt = size > 0 ? (std::uint64_t)size / 8 : 0;
    auto* out = static_cast<double*>(std::malloc(std::max<std::uint64_t>(1, cnt) * 8));
    if (!out) {
      std::fclose(f);
      raise(VK_ERR_INTERNAL, "host allocation failed");
    }
    const std::size_t got = cnt ? std::fread(out, 8, cnt, f) : 0;
    std::fclose(f);
    if (got != cnt) {
      std::free(out);
      raise(VK_ERR_IO, std::string("read failed: ") + path);
    }
    *values = out;
    *n = cnt;
  });
}

// graph.cpp:553-563: "VCSR", u32 1, u64 n, u64 m, (n+1) u64 offsets, m u64
// targets, little-endian
int vk_write_vcsr(const char* path, uint64_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt) {
  return guard([&] {
    if (!path || !off || (!tgt && m)) raise(VK_ERR_PARAMETER, "null argument");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) raise(VK_ERR_IO, std::string("cannot write ") + path);
    bool failed = false;
    const std::uint32_t version = 1;
    failed |= std::fwrite("VCSR", 1, 4, f) != 4;
    failed |= std::fwrite(&version, 4, 1, f) != 1;
    failed |= std::fwrite(&n, 8, 1, f) != 1;
    failed |= std::fwrite(&m, 8, 1, f) != 1;
    failed |= std::fwrite(off, 8, n + 1, f) != n + 1;
    std::vector<std::uint64_t> chunk(1 << 20);
    for (std::uint64_t i = 0; i < m && !failed; i += chunk.size()) {
      const std::uint64_t c = std::min<std::uint64_t>(chunk.size(), m - i);
      for (std::uint64_t j = 0; j < c; ++j) chunk[j] = tgt[i + j];
      failed |= std::fwrite(chunk.data(), 8, c, f) != c;
    }
    failed |= std::fclose(f) != 0;
    if (failed) raise(VK_ERR_IO, std::string("write failed: ") + path);
  });
}

}  // extern "C"
