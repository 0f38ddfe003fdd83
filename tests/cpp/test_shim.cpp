// The reference-side shim (include/cbm_b200_shim.hpp) driven exactly like the
// reference's own kernel tests (proj/tests/test_kernels.cpp), with the
// reference's CbmMatrix / DenseMatrix types and builder. Built by
// `make -C oracle shim` into oracle/_ref/test_shim (needs the reference
// headers at build time); run on a GPU by tests/test_shim_gpu.py.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "cbm/builder.hpp"
#include "cbm/kernels.hpp"
#include "cbm_b200_shim.hpp"
#include "oracles.hpp"

using namespace cbm;
using namespace cbm::test;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, E)                                             \
  do {                                                                       \
    bool thrown = false;                                                     \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const E&) {                                                     \
      thrown = true;                                                         \
    }                                                                        \
    CHECK(thrown);                                                           \
  } while (0)

static CsrBinaryMatrix from_rows(index_t n_cols, const std::vector<std::vector<index_t>>& rows) {
  std::vector<std::pair<index_t, index_t>> e;
  for (std::size_t r = 0; r < rows.size(); ++r)
    for (index_t c : rows[r]) e.emplace_back(index_t(r), c);
  return CsrBinaryMatrix::from_coo(index_t(rows.size()), n_cols, std::move(e));
}

static bool bitwise(const DenseMatrix& a, const DenseMatrix& b) {
  return a.n_rows == b.n_rows && a.n_cols == b.n_cols &&
         std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(real_t)) == 0;
}

int main() {
  // test_kernels.cpp:45-54 identical rows
  {
    auto c = build_cbm(from_rows(3, {{0, 1}, {0, 1}}), 0);
    DenseMatrix v(3, 1, {2.0f, 3.0f, 5.0f});
    auto u = b200::spmv(b200::DeviceCbm(c), v);
    CHECK(u.at(0, 0) == 5.0f && u.at(1, 0) == 5.0f);
  }
  // :56-66 zero, identity, shape errors
  {
    auto zero = build_cbm(from_rows(3, {{}, {}, {}}), 0);
    DenseMatrix v(3, 1, {1.0f, 2.0f, 3.0f});
    for (real_t x : b200::spmv(b200::DeviceCbm(zero), v).data) CHECK(x == 0.0f);
    auto eye = build_cbm(from_rows(3, {{0}, {1}, {2}}), 0);
    b200::DeviceCbm deye(eye);
    CHECK(b200::spmv(deye, v) == v);
    CHECK_THROWS_AS(b200::spmv(deye, DenseMatrix(4, 1)), std::invalid_argument);
    CHECK_THROWS_AS(b200::spmv(deye, DenseMatrix(3, 2)), std::invalid_argument);
    CHECK_THROWS_AS(b200::spmm(deye, DenseMatrix(4, 2)), std::invalid_argument);
    DenseMatrix bad_out(2, 2), b(3, 2);
    CHECK_THROWS_AS(b200::spmm_into(deye, b, bad_out), std::invalid_argument);
  }
  // :68-73 identity operand densifies A
  {
    auto a = random_binary(12, 12, 0.3, 7);
    auto c = build_cbm(a, 0);
    CHECK(max_abs_diff(b200::spmm(c, DenseMatrix::identity(12)), densify_pattern(a)) == 0.0);
  }
  // :75-144 random instances, plain and normalized: the GPU equals spmm bit for bit
  for (std::uint64_t seed = 1; seed <= 30; ++seed) {
    UniformRng dims(seed * 7919);
    const index_t m = 1 + index_t(dims.below(16)), n = 1 + index_t(dims.below(16));
    const index_t p = 1 + index_t(dims.below(5));
    auto a = random_binary(m, n, 0.25, seed);
    auto b = random_dense(n, p, -1.0, 1.0, seed + 17);
    for (count_t alpha : {0, 1, 2, 4}) {
      auto c = build_cbm(a, alpha);
      CHECK(bitwise(b200::spmm(c, b), spmm(c, b)));
    }
  }
  for (std::uint64_t seed = 50; seed < 70; ++seed) {
    UniformRng dims(seed);
    const index_t n = 1 + index_t(dims.below(32)), p = 1 + index_t(dims.below(6));
    auto a = random_binary(n, n, 0.2, seed);
    auto b = random_dense(n, p, -1.0, 1.0, seed + 3);
    for (count_t alpha : {0, 2, 8}) {
      auto c = build_cbm_normalized(a, alpha);
      CHECK(bitwise(b200::spmm(c, b), spmm(c, b)));
    }
  }
  // :94-99 normalized two-node path
  {
    auto c = build_cbm_normalized(from_rows(2, {{1}, {0}}), 0);
    auto d = b200::spmm(c, DenseMatrix::identity(2));
    CHECK(bitwise(d, spmm(c, DenseMatrix::identity(2))));
  }
  // acceptance.cpp:175-190 community graph, larger operand, reused upload
  {
    auto a = community_graph(50, 40, 40, 1, 0xC0FFEE);
    auto c = build_cbm(a, 0);
    auto cn = build_cbm_normalized(a, 0);
    b200::DeviceCbm dc(c), dn(cn);
    b200::DeviceCbm fast(c, -1, /*order_faithful=*/false);
    for (index_t width : {1u, 7u, 64u, 130u}) {
      auto b = random_dense(a.n_cols, width, -1.0, 1.0, width);
      CHECK(bitwise(b200::spmm(dc, b), spmm(c, b)));
      CHECK(bitwise(b200::spmm(dn, b), spmm(cn, b)));
      // the fast mode on integer operands is exact too
      DenseMatrix bi(b.n_rows, b.n_cols);
      for (std::size_t i = 0; i < bi.data.size(); ++i) bi.data[i] = real_t(int(b.data[i] * 8));
      CHECK(bitwise(b200::spmm(fast, bi), spmm(c, bi)));
    }
  }
  // column-sharded multiply over several uploads (one per device in production)
  {
    auto a = community_graph(30, 40, 40, 1, 0xBEEF);
    auto c = build_cbm_normalized(a, 0);
    b200::DeviceCbm s0(c, 0), s1(c, 0), s2(c, 0);
    auto b = random_dense(a.n_cols, 100, -1.0, 1.0, 77);
    DenseMatrix out(c.n_rows, 100);
    b200::spmm_sharded_into({&s0, &s1, &s2}, b, out);
    CHECK(bitwise(out, spmm(c, b)));
    DenseMatrix bad(c.n_rows, 3);
    CHECK_THROWS_AS(b200::spmm_sharded_into({&s0, &s1}, DenseMatrix(4, 3), bad),
                    std::invalid_argument);
  }
  std::printf("test_shim: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
