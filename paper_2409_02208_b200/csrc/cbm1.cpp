// CBM1 container — the reference's on-disk format (proj/include/cbm/io.hpp:44-57):
// "CBM1", version 1, flags (bit 0 = normalized), two zero bytes, little-endian
// u64 n_rows, n_cols, alpha, nnz, then the sections u32 parent[m],
// u32 topo_order[m], u64 row_ptr[m+1], u32 col_idx[nnz], f64 values[nnz] and,
// when normalized, f64 row_scale[m]. Files interoperate with the reference's
// save_cbm / load_cbm (io.cpp:261-382) byte for byte.
//
// Reading: the file is memory-mapped; the header fixes every section's offset
// and the exact file size, the sections are decoded straight from the mapping
// into the host matrix and checked by all host threads at once. The reference
// validates sequentially; when an input breaks several rules the error
// reported here is still the one the reference reports first (its order:
// row scales, parent links, CSR structure row by row, finiteness, stored topo
// order, value pattern), with its message (format_error -> EFORMAT).
// Writing streams the sections through a fixed-size buffer instead of
// assembling the whole file in memory.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cbm_host.hpp"

namespace cbmb {

namespace {

constexpr unsigned char kTag[4] = {'C', 'B', 'M', '1'};
constexpr uint8_t kFormatVersion = 1;
constexpr uint64_t kHeaderBytes = 40;

// Section offsets of a container with the given header, relative to the file
// start; `end` is the only valid file size.
struct Sections {
  uint64_t parent, topo, row_ptr, col_idx, values, scale, end;
  Sections(uint64_t m, uint64_t nnz, bool normalized) {
    parent = kHeaderBytes;
    topo = parent + 4 * m;
    row_ptr = topo + 4 * m;
    col_idx = row_ptr + 8 * (m + 1);
    values = col_idx + 4 * nnz;
    scale = values + 8 * nnz;
    end = scale + (normalized ? 8 * m : 0);
  }
};

class MappedFile {
 public:
  explicit MappedFile(const std::string& path) {
    fd_ = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    if (fd_ < 0) throw format_error(path + ": cannot open file");
    struct stat st;
    if (::fstat(fd_, &st) != 0 || !S_ISREG(st.st_mode)) {
      ::close(fd_);
      throw format_error(path + ": cannot open file");
    }
    size_ = uint64_t(st.st_size);
    if (size_) {
      void* p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
      if (p == MAP_FAILED) {
        ::close(fd_);
        throw format_error(path + ": read failed");
      }
      ::madvise(p, size_, MADV_SEQUENTIAL | MADV_WILLNEED);
      base_ = static_cast<const unsigned char*>(p);
    }
  }
  ~MappedFile() {
    if (base_) ::munmap(const_cast<unsigned char*>(base_), size_);
    if (fd_ >= 0) ::close(fd_);
  }
  MappedFile(const MappedFile&) = delete;
  MappedFile& operator=(const MappedFile&) = delete;
  const unsigned char* data() const { return base_; }
  uint64_t size() const { return size_; }

 private:
  int fd_ = -1;
  const unsigned char* base_ = nullptr;
  uint64_t size_ = 0;
};

template <typename T>
T load_le(const unsigned char* p) {  // unaligned little-endian load (x86-64 / aarch64)
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

int host_threads() { return int(std::max(1u, std::thread::hardware_concurrency())); }

// Lowest index in [0, n) for which bad(i) holds (n if none), over all threads.
template <typename Pred>
uint64_t first_bad(uint64_t n, Pred bad) {
  std::atomic<uint64_t> best{n};
  parallel_for_chunks(size_t(n), host_threads(), [&](size_t lo, size_t hi, int) {
    for (size_t i = lo; i < hi && i < best.load(std::memory_order_relaxed); ++i)
      if (bad(i)) {
        uint64_t cur = best.load();
        while (i < cur && !best.compare_exchange_weak(cur, i)) {
        }
        return;
      }
  });
  return best.load();
}

// Copy a section of `count` little-endian T from the mapping, all threads.
template <typename T, typename U>
void decode(const unsigned char* src, uint64_t count, U* dst) {
  parallel_for_chunks(size_t(count), host_threads(), [&](size_t lo, size_t hi, int) {
    if constexpr (std::is_same_v<T, U>) {
      std::memcpy(dst + lo, src + lo * sizeof(T), (hi - lo) * sizeof(T));
    } else {
      for (size_t i = lo; i < hi; ++i) dst[i] = U(load_le<T>(src + i * sizeof(T)));
    }
  });
}

// The CSR structure rules of CsrRealMatrix (csr.cpp:12-33) for row r: the
// reference checks offsets, then column order, then the last column's range;
// 0 = fine, 1 = offsets decrease, 2 = not increasing, 3 = out of range.
int csr_row_defect(const HostCbm& c, uint64_t nnz, uint32_t r) {
  const uint64_t lo = c.row_ptr[r], hi = c.row_ptr[r + 1];
  if (lo > hi) return 1;
  // an offset past nnz: the reference scans on into the next rows' columns
  // (and past the array) until the order breaks; the order break inside the
  // array is what it reports, past it the offsets necessarily decrease later
  const uint64_t end = std::min(hi, nnz);
  for (uint64_t k = lo; k + 1 < end; ++k)
    if (c.col_idx[k] >= c.col_idx[k + 1]) return 2;
  if (hi > nnz) return 1;
  if (hi > lo && c.col_idx[hi - 1] >= c.n_cols) return 3;
  return 0;
}

}  // namespace

HostCbm load_cbm1(const std::string& path) {
  MappedFile f(path);
  const unsigned char* b = f.data();
  const uint64_t size = f.size();

  // ---- header (io.cpp:301-330 checks, in the reference's order) ----
  if (size < 4) throw format_error("truncated container");
  if (std::memcmp(b, kTag, 4) != 0) throw format_error("bad magic: not a CBM1 container");
  if (size < 5) throw format_error("truncated container");
  if (b[4] != kFormatVersion) throw format_error("unsupported container version");
  if (size < 6) throw format_error("truncated container");
  if (b[5] > 1) throw format_error("unknown flag bits set");
  const bool normalized = (b[5] & 1) != 0;
  if (size < 8) throw format_error("truncated container");
  if (b[6] != 0 || b[7] != 0) throw format_error("reserved header bytes must be zero");
  if (size < kHeaderBytes) throw format_error("truncated container");
  const uint64_t m64 = load_le<uint64_t>(b + 8), n64 = load_le<uint64_t>(b + 16);
  const uint64_t alpha = load_le<uint64_t>(b + 24), nnz = load_le<uint64_t>(b + 32);
  if (m64 >= kVirtual || n64 >= kVirtual) throw format_error("container dimensions too large");
  if (normalized && m64 != n64) throw format_error("normalized container must be square");
  // every section size follows from the header, so must the file size; a
  // header whose sizes overflow cannot describe this file either
  if (nnz > (uint64_t(1) << 60)) throw format_error("container payload size mismatch");
  const Sections sec(m64, nnz, normalized);
  if (sec.end != size) throw format_error("container payload size mismatch");

  const uint32_t m = uint32_t(m64);
  HostCbm c;
  c.n_rows = m;
  c.n_cols = uint32_t(n64);
  c.alpha = alpha;
  c.normalized = normalized;

  // ---- row scales first (io.cpp:346-352) ----
  if (normalized) {
    const unsigned char* s = b + sec.scale;
    if (first_bad(m, [&](uint64_t i) {
          const double v = load_le<double>(s + 8 * i);
          return !std::isfinite(v) || v <= 0.0;
        }) < m)
      throw format_error("row_scale entries must be positive and finite");
  }

  // ---- chain (CompressionChain::from_parents) and CSR structure ----
  c.parent.resize(m);
  decode<uint32_t>(b + sec.parent, m, c.parent.data());
  c.row_ptr.resize(size_t(m) + 1);
  decode<uint64_t>(b + sec.row_ptr, uint64_t(m) + 1, c.row_ptr.data());
  c.col_idx.resize(nnz);
  decode<uint32_t>(b + sec.col_idx, nnz, c.col_idx.data());
  c.values.resize(nnz);
  decode<double>(b + sec.values, nnz, c.values.data());   // f64 -> f32 (the f32 build)
  try {
    chain_from_parents(c);
    if (c.row_ptr[0] != 0) throw invalid_argument("csr: row_ptr[0] must be 0");
    if (c.row_ptr[m] != nnz) throw invalid_argument("csr: row_ptr back must equal nnz");
    const uint64_t r = first_bad(m, [&](uint64_t i) {
      return csr_row_defect(c, nnz, uint32_t(i)) != 0;
    });
    if (r < m) {
      switch (csr_row_defect(c, nnz, uint32_t(r))) {
        case 1: throw invalid_argument("csr: row_ptr must be non-decreasing");
        case 2:
          throw invalid_argument("csr: row " + std::to_string(r) + " is not strictly increasing");
        default:
          throw invalid_argument("csr: column index out of range in row " + std::to_string(r));
      }
    }
    if (first_bad(nnz, [&](uint64_t k) { return !std::isfinite(c.values[k]); }) < nnz)
      throw invalid_argument("csr: values must be finite");
  } catch (const invalid_argument& e) {
    throw format_error(std::string("invalid container structure: ") + e.what());
  }

  // ---- stored topological order must be the one the chain implies ----
  {
    const unsigned char* t = b + sec.topo;
    if (first_bad(m, [&](uint64_t i) { return load_le<uint32_t>(t + 4 * i) != c.topo_order[i]; }) < m)
      throw format_error("stored topological order is inconsistent");
  }

  // ---- value pattern, on the stored f64 values (io.cpp:369-380) ----
  const unsigned char* v = b + sec.values;
  if (normalized) {
    const unsigned char* s = b + sec.scale;
    if (first_bad(nnz, [&](uint64_t k) {
          const double want = load_le<double>(s + 8 * uint64_t(c.col_idx[k]));
          const double got = load_le<double>(v + 8 * k);
          return got != want && got != -want;
        }) < nnz)
      throw format_error("delta values disagree with the column scales");
    c.row_scale.resize(m);
    decode<double>(s, m, c.row_scale.data());
  } else {
    if (first_bad(nnz, [&](uint64_t k) {
          const double got = load_le<double>(v + 8 * k);
          return got != 1.0 && got != -1.0;
        }) < nnz)
      throw format_error("delta values must be +1 or -1");
  }
  return c;
}

namespace {

// Buffered little-endian section writer.
class SectionWriter {
 public:
  explicit SectionWriter(const std::string& path) : path_(path) {
    f_ = std::fopen(path.c_str(), "wb");
    if (!f_) throw format_error(path + ": cannot open for writing");
    buf_.reserve(kChunk);
  }
  ~SectionWriter() {
    if (f_) std::fclose(f_);
  }
  void bytes(const void* p, size_t n) {
    const auto* q = static_cast<const unsigned char*>(p);
    while (n) {
      const size_t take = std::min(n, kChunk - buf_.size());
      buf_.insert(buf_.end(), q, q + take);
      q += take;
      n -= take;
      if (buf_.size() == kChunk) flush();
    }
  }
  template <typename T, typename U>
  void array(const U* src, size_t n) {  // element-wise conversion U -> T
    if constexpr (std::is_same_v<T, U>) {
      bytes(src, n * sizeof(T));
    } else {
      T tmp[512];
      for (size_t i = 0; i < n; i += 512) {
        const size_t k = std::min<size_t>(512, n - i);
        for (size_t j = 0; j < k; ++j) tmp[j] = T(src[i + j]);
        bytes(tmp, k * sizeof(T));
      }
    }
  }
  void finish() {
    flush();
    const bool ok = std::fclose(f_) == 0;
    f_ = nullptr;
    if (!ok) throw format_error(path_ + ": write failed");
  }

 private:
  static constexpr size_t kChunk = size_t(1) << 22;
  void flush() {
    if (!buf_.empty() && std::fwrite(buf_.data(), 1, buf_.size(), f_) != buf_.size())
      throw format_error(path_ + ": write failed");
    buf_.clear();
  }
  std::string path_;
  std::FILE* f_ = nullptr;
  std::vector<unsigned char> buf_;
};

}  // namespace

void save_cbm1(const HostCbm& c, const std::string& path) {
  const uint64_t m = c.n_rows, nnz = c.row_ptr.back();
  unsigned char head[kHeaderBytes] = {};
  std::memcpy(head, kTag, 4);
  head[4] = kFormatVersion;
  head[5] = c.normalized ? 1 : 0;
  const uint64_t fields[4] = {c.n_rows, c.n_cols, c.alpha, nnz};
  std::memcpy(head + 8, fields, sizeof(fields));
  SectionWriter w(path);
  w.bytes(head, sizeof(head));
  w.array<uint32_t>(c.parent.data(), m);
  w.array<uint32_t>(c.topo_order.data(), m);
  w.array<uint64_t>(c.row_ptr.data(), m + 1);
  w.array<uint32_t>(c.col_idx.data(), nnz);
  w.array<double>(c.values.data(), nnz);
  if (c.normalized) w.array<double>(c.row_scale.data(), m);
  w.finish();
}

}  // namespace cbmb
