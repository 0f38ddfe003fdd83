// CBM1 container (the reference's on-disk format, proj/include/cbm/io.hpp:44-57,
// proj/src/io.cpp:198-382): little-endian "CBM1", version 1, flags (bit 0 =
// normalized), two zero bytes, u64 n_rows, n_cols, alpha, nnz, then u32
// parent[m], u32 topo_order[m], u64 row_ptr[m+1], u32 col_idx[nnz],
// f64 values[nnz] and, when normalized, f64 row_scale[m]. Files written here
// load in the reference and vice versa; loading validates everything the
// reference validates, with the same messages (format errors -> EFORMAT).
#include <cmath>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "cbm_host.hpp"

namespace cbmb {

namespace {
constexpr char kMagic[4] = {'C', 'B', 'M', '1'};
constexpr uint8_t kVersion = 1;

template <typename T>
void put(std::vector<unsigned char>& b, T v) {
  unsigned char raw[sizeof(T)];
  std::memcpy(raw, &v, sizeof(T));  // little-endian host (x86-64, aarch64)
  b.insert(b.end(), raw, raw + sizeof(T));
}

struct Reader {
  const unsigned char* p;
  size_t left;
  void need(size_t n) const {
    if (left < n) throw format_error("truncated container");
  }
  template <typename T>
  T get() {
    need(sizeof(T));
    T v;
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    left -= sizeof(T);
    return v;
  }
};
}  // namespace

void save_cbm1(const HostCbm& c, const std::string& path) {
  const uint64_t m = c.n_rows, nnz = c.row_ptr.back();
  std::vector<unsigned char> b;
  b.reserve(40 + m * 8 + (m + 1) * 8 + nnz * 12 + (c.normalized ? m * 8 : 0));
  b.insert(b.end(), kMagic, kMagic + 4);
  put<uint8_t>(b, kVersion);
  put<uint8_t>(b, c.normalized ? 1 : 0);
  put<uint8_t>(b, 0);
  put<uint8_t>(b, 0);
  put<uint64_t>(b, c.n_rows);
  put<uint64_t>(b, c.n_cols);
  put<uint64_t>(b, c.alpha);
  put<uint64_t>(b, nnz);
  for (uint32_t v : c.parent) put<uint32_t>(b, v);
  for (uint32_t v : c.topo_order) put<uint32_t>(b, v);
  for (uint64_t v : c.row_ptr) put<uint64_t>(b, v);
  for (uint32_t v : c.col_idx) put<uint32_t>(b, v);
  for (float v : c.values) put<double>(b, double(v));
  if (c.normalized)
    for (float v : c.row_scale) put<double>(b, double(v));
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw format_error(path + ": cannot open for writing");
  out.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size()));
  if (!out) throw format_error(path + ": write failed");
}

HostCbm load_cbm1(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw format_error(path + ": cannot open file");
  const std::streamsize size = in.tellg();
  in.seekg(0);
  std::vector<unsigned char> buf(size_t(std::max<std::streamsize>(size, 0)));
  if (size > 0 && !in.read(reinterpret_cast<char*>(buf.data()), size))
    throw format_error(path + ": read failed");
  Reader r{buf.data(), buf.size()};
  r.need(4);
  if (std::memcmp(r.p, kMagic, 4) != 0) throw format_error("bad magic: not a CBM1 container");
  r.p += 4;
  r.left -= 4;
  if (r.get<uint8_t>() != kVersion) throw format_error("unsupported container version");
  const uint8_t flags = r.get<uint8_t>();
  if (flags > 1) throw format_error("unknown flag bits set");
  const bool normalized = flags & 1;
  const uint8_t z0 = r.get<uint8_t>(), z1 = r.get<uint8_t>();
  if (z0 != 0 || z1 != 0) throw format_error("reserved header bytes must be zero");
  const uint64_t m64 = r.get<uint64_t>(), n64 = r.get<uint64_t>();
  const uint64_t alpha = r.get<uint64_t>(), nnz = r.get<uint64_t>();
  if (m64 >= kVirtual || n64 >= kVirtual) throw format_error("container dimensions too large");
  const uint32_t m = uint32_t(m64), n = uint32_t(n64);
  if (normalized && m != n) throw format_error("normalized container must be square");
  const uint64_t expect = 8ull * m + 8ull * (m64 + 1) + 12ull * nnz + (normalized ? 8ull * m : 0);
  if (r.left != expect) throw format_error("container payload size mismatch");

  HostCbm c;
  c.n_rows = m;
  c.n_cols = n;
  c.alpha = alpha;
  c.normalized = normalized;
  c.parent.resize(m);
  for (auto& v : c.parent) v = r.get<uint32_t>();
  std::vector<uint32_t> stored_topo(m);
  for (auto& v : stored_topo) v = r.get<uint32_t>();
  c.row_ptr.resize(size_t(m) + 1);
  for (auto& v : c.row_ptr) v = r.get<uint64_t>();
  c.col_idx.resize(nnz);
  for (auto& v : c.col_idx) v = r.get<uint32_t>();
  std::vector<double> raw_values(nnz);
  for (auto& v : raw_values) v = r.get<double>();
  std::vector<double> raw_scale;
  if (normalized) {
    raw_scale.resize(m);
    for (auto& v : raw_scale) v = r.get<double>();
    for (double v : raw_scale)
      if (!std::isfinite(v) || v <= 0.0)
        throw format_error("row_scale entries must be positive and finite");
  }
  try {
    chain_from_parents(c);
    // CsrRealMatrix checks (csr.cpp:12-33, 69-82)
    if (c.row_ptr[0] != 0) throw invalid_argument("csr: row_ptr[0] must be 0");
    if (c.row_ptr.back() != nnz) throw invalid_argument("csr: row_ptr back must equal nnz");
    validate_csr(m, n, c.row_ptr.data(), c.col_idx.data());
    c.values.assign(raw_values.begin(), raw_values.end());
    for (float v : c.values)
      if (!std::isfinite(v)) throw invalid_argument("csr: values must be finite");
  } catch (const invalid_argument& e) {
    throw format_error(std::string("invalid container structure: ") + e.what());
  }
  if (c.topo_order != stored_topo) throw format_error("stored topological order is inconsistent");
  if (normalized) {
    c.row_scale.assign(raw_scale.begin(), raw_scale.end());
    for (uint64_t k = 0; k < nnz; ++k) {
      const double want = raw_scale[c.col_idx[k]];
      if (raw_values[k] != want && raw_values[k] != -want)
        throw format_error("delta values disagree with the column scales");
    }
  } else {
    for (double v : raw_values)
      if (v != 1.0 && v != -1.0) throw format_error("delta values must be +1 or -1");
  }
  return c;
}

}  // namespace cbmb
