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
  bool inconsistent = false;  // some delta row has no full-row form (nothing flattened)
  uint64_t nnz = 0;            // deltas of the uploaded CBM
  uint64_t nnz_effective = 0;  // deltas after flattening (what the kernel sums)
  uint32_t n_flattened = 0;    // rows summed directly instead of via their parent
  std::vector<uint32_t> dcol;   // column | sign << 31, in item order
  // rec, 8 x u32 per item (two uint4 loads on the device):
  //   [0] beg, [1] end   : the item owns dcol[beg, end)
  //   [2] row | kInteriorBit (row has children -> publishes a ready flag)
  //   [3] ppos  : item index of the parent's ROW item, or kNoItem
  //   [4] psrc  : where the parent's unscaled row lives: its row id (plain) or
  //               its interior scratch slot (normalized)
  //   [5] first : first partial item summed after the own deltas
  //   [6] cnt   : number of partials [first, first + cnt)
  //   [7] slot  : own interior scratch slot (normalized parents) or kNoItem
  std::vector<uint32_t> rec;
  std::vector<float> srow;      // per item: row_scale[row] (normalized)
  std::vector<float> scale;     // column scale (normalized): row_scale, or the view's col_scale
  std::vector<float> row_scale; // the rows' own scale (normalized)
  std::vector<uint32_t> item_beg;  // n_items + 1: delta prefix by item (kept on the host)
  uint32_t band_cols = 0;       // columns per band (0: the long rows' pieces are not banded)
  std::vector<uint32_t> order;  // processing order of the items (empty: item order)
  std::vector<uint32_t> level_ptr;  // ROW-item offsets of each level (relative to the ROW block)
};

// Validates the view like load_cbm (io.cpp:346-380) and builds the layout.
// Throws cbmb::invalid_argument with a reference-style message.
// warps_hint: resident warps of the target device (sizes the auto split).
// Full rows of every row, parents first; false if some delta row is
// inconsistent with its parent's row (layout.cpp).
bool reconstruct_full_rows(const cbm_b200_cbm_view& v, const std::vector<uint32_t>& bfs,
                           std::vector<uint64_t>& fptr, std::vector<uint32_t>& fcol);

// The structural checks alone (throws like plan_layout).
void validate_view(const cbm_b200_cbm_view& v);

Layout plan_layout(const cbm_b200_cbm_view& v, bool order_faithful, uint32_t split_threshold,
                   uint32_t chunk, uint32_t flatten_gain, uint32_t warps_hint);

}  // namespace cbmb
