// Hub-row panel (DESIGN.md §6 "Hub-row panel"): the longest rows of a
// power-law matrix taken off the streaming kernel and multiplied together on
// the tensor cores.
//
// cfg[4]'s 128 longest rows hold 18% of the entries and reference, between
// them, most of the columns, each column about 9 times. Gathered row by row
// those X rows cross the L2->SM link once per entry; as ONE 128-row tile of the
// dense-block kernel (dense_kernel.cu) each X row is loaded once and serves
// every hub row that holds it. The tile's chunk list (32 columns each, over
// the union of the hub rows' columns) is cut into pieces of consecutive chunks,
// one work unit per (piece, 128 features); each unit leaves a 128-row partial
// in a workspace and a fixed-order reduction forms Y[hub rows].
// Everything else stays on the streaming kernel, on a view of the CBM whose
// hub rows are empty (their children, if any, summed from their full rows).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/cbm_b200.h"
#include "dense_layout.hpp"

namespace cbmb {

inline constexpr uint32_t kHubPieceChunks = 32;  // chunks per piece (accumulation length)
inline constexpr uint32_t kHubFanIn = 64;        // partial rows combined per reduction step

struct HubPlan {
  bool on = false;
  std::vector<uint32_t> rows;      // the hub rows (<= kDenseRows), longest first
  uint64_t entries = 0;            // entries of the represented matrix in the hub rows
  uint64_t n_chunks = 0;           // chunks of kDenseK columns over the union of their columns
  uint32_t n_pieces = 0;           // consecutive chunk ranges (= tiles of the dense kernel)
  std::vector<uint32_t> tiles;     // per piece: piece * kDenseRows, kDenseRows, first chunk, chunks
  std::vector<uint32_t> meta;      // per chunk: kDenseMetaWords (dense_layout.hpp)
  // the rest of the matrix as a CBM view (same shape; hub rows empty)
  std::vector<uint32_t> rest_parent;
  std::vector<uint64_t> rest_row_ptr;
  std::vector<uint32_t> rest_col;
  std::vector<float> rest_val;
  // the hub rows alone as a (rows.size() x n_cols) view, every parent virtual
  // (narrow X, spmv: below the tensor path's minimum width)
  std::vector<uint32_t> hub_parent;
  std::vector<uint64_t> hub_row_ptr;
  std::vector<uint32_t> hub_col;
  std::vector<float> hub_val;
  std::vector<float> hub_row_scale;  // normalized: row_scale of the hub rows
};

// v: a validated view (plan_layout's checks). mode: 1 force, -1 auto (the
// cost rule in hub_layout.cpp). Returns on = false when the rule declines or
// some delta row has no full-row form.
HubPlan plan_hub(const cbm_b200_cbm_view& v, int mode, uint32_t num_sms);

}  // namespace cbmb
