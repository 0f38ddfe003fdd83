// Device layout of an uploaded CBM.
//
// The reference walks rows in DFS topological order per root branch
// (kernels.cpp:42-62). On the GPU the unit of work is an ITEM:
//   * ROW item   — one output row: its delta sum, + the parent's unscaled row,
//                  then (normalized) the row scale. ROW items are ordered by
//                  depth in the compression forest (roots first), ascending
//                  row id inside a level, so every parent precedes its
//                  children in ticket order.
//   * CHUNK item — a slice of a long delta row, summed on its own into a
//                  partial-sum slot (only when uploaded with order_faithful=0).
//   * MERGE item — the ordered sum of up to kFanIn earlier partials of the
//                  same row (a fixed tree, so results are deterministic).
// Order: all CHUNK items, then MERGE items level by level, then ROW items;
// every item depends only on items before it.
// Deltas are re-laid out in item order as one u32 each: column | sign << 31
// (the value is +-1, or +-row_scale[col] rebuilt bit-exactly on the fly).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/cbm_b200.h"

namespace cbmb {

inline constexpr uint32_t kInteriorBit = 0x80000000u;
inline constexpr uint32_t kSignBit = 0x80000000u;
inline constexpr uint32_t kNoItem = 0xFFFFFFFFu;
inline constexpr uint32_t kFanIn = 32;  // partials combined per MERGE / ROW item

struct Layout {
  uint32_t n_rows = 0, n_cols = 0;
  bool normalized = false;
  bool order_faithful = true;
  uint32_t n_items = 0;        // CHUNK + MERGE + ROW items
  uint32_t n_chunk_items = 0;  // items [0, n_chunk_items) produce partial sums
                               // (CHUNK then MERGE items)
  uint32_t n_merge_items = 0;
  uint32_t n_interior = 0;     // rows with children (scratch slots, normalized)
  uint32_t n_levels = 0, n_roots = 0, max_row_deltas = 0;
  uint64_t nnz = 0;
  std::vector<uint32_t> dptr;   // n_items + 1: item t owns dcol[dptr[t], dptr[t+1])
  std::vector<uint32_t> dcol;   // column | sign << 31
  // meta, 4 x u32 per item:
  //   [0] row | kInteriorBit (row has children -> publishes a ready flag)
  //   [1] ppos: item index of the parent's ROW item, or kNoItem
  //   [2] psrc: where the parent's unscaled row lives: its row id (plain) or
  //       its interior scratch slot (normalized)
  //   [3] first partial item summed after the own deltas (see pcnt)
  std::vector<uint32_t> meta;
  std::vector<uint32_t> pcnt;   // per item: number of partials [meta[3], meta[3]+pcnt)
  std::vector<uint32_t> oslot;  // per item: own scratch slot (normalized interior) or kNoItem
  std::vector<float> scale;     // row_scale (normalized)
  std::vector<uint32_t> level_ptr;  // ROW-item offsets of each level (relative to the ROW block)
};

// Validates the view like load_cbm (io.cpp:346-380) and builds the layout.
// Throws cbmb::invalid_argument with a reference-style message.
Layout plan_layout(const cbm_b200_cbm_view& v, bool order_faithful, uint32_t split_threshold,
                   uint32_t chunk);

}  // namespace cbmb
