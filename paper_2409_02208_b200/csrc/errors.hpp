// Exceptions used inside the library; the C ABI (capi.cpp) maps them onto
// CBM_B200_* status codes and never lets them cross the boundary.
#pragma once

#include <stdexcept>
#include <string>

namespace cbmb {

struct invalid_argument : std::invalid_argument {  // std::invalid_argument in the reference
  using std::invalid_argument::invalid_argument;
};
// a delta row that removes a column its parent lacks or adds one it has: the
// reference multiplies it (deltas + parent) but it has no full-row form, so
// paths that flatten or cut rows step aside for it
struct inconsistent_rows : invalid_argument {
  inconsistent_rows() : invalid_argument("delta rows are inconsistent with their parents' rows") {}
};
struct logic_error : std::logic_error {  // std::logic_error in the reference builder
  using std::logic_error::logic_error;
};
struct format_error : std::runtime_error {  // cbm::format_error (io.hpp:19-22)
  using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {  // CUDA failure, carries a CBM_B200_* code
  int code;
  cuda_error(const std::string& s, int c) : std::runtime_error(s), code(c) {}
};

}  // namespace cbmb
