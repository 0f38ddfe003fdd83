// Tiled device layout of an uploaded CBM (DESIGN.md §6 "Tiled path").
//
// The streaming kernel gathers every delta's X row from L2; on matrices whose
// rows fall into groups that reference a small common column set (community
// structure: cfg[0], cfg[3]) the same X rows are gathered hundreds of times.
// The tiled layout cuts the compression forest into ROW BLOCKS (whole trees,
// big trees split into subtrees) and lists, per block, its STAGED columns
// (referenced at least twice inside the block, the most referenced first, up
// to a capacity). One CTA per (block, column slab) copies those X rows into
// shared memory once and then sums every row of the block:
//   * staged deltas read shared memory (local index), cold deltas L2;
//   * parents inside the block are waited on with shared-memory flags (rows
//     are in depth order inside the block, claimed in order, so every wait
//     targets an earlier row of the same CTA: no deadlock, no grid sync);
//   * a subtree root whose parent lies in another block is FLATTENED (summed
//     from its full row), so blocks never wait on each other.
// Only the summation order changes (staged deltas first, then cold deltas,
// then the parent, as in kernels.cpp:27-62 otherwise): bit-exact on integer
// X, within the north_star tolerance otherwise. Default mode only.
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/cbm_b200.h"

namespace cbmb {

inline constexpr uint32_t kTileNone = 0xFFFFFFFFu;
// auto mode keeps the tiled path when at least this share of the deltas reads
// the shared-memory tile and each staged row serves at least this many deltas
inline constexpr double kTileMinStagedFrac = 0.6;
inline constexpr double kTileMinReuse = 8.0;

struct TileLayout {
  uint32_t n_blocks = 0, max_rows = 0, max_staged = 0, n_interior = 0, n_cut = 0, n_flat = 0;
  uint32_t row_cap = 0, stage_cap = 0;
  uint64_t n_deltas = 0, n_staged_deltas = 0, n_staged_cols = 0, n_entries = 0;
  uint64_t max_row_entries = 0;  // longest row (one warp sums a row: no splitting)
  uint64_t max_block_entries = 0;  // heaviest block (one CTA per block and slab)
  // per block: row0, nrows, st0, nst (tile rows [row0, row0+nrows), staged
  // columns tstage[st0, st0+nst)); blocks ordered by estimated work, largest first
  std::vector<uint32_t> block;
  // per tile row, 8 x u32: beg, mpos, mid, end, row, parent local index in the
  // block (or kTileNone), parent's interior slot, own interior slot (or kTileNone).
  // tdcol[beg, mpos): staged +1 deltas, [mpos, mid): staged -1 deltas (local
  // tile rows; each run padded to a multiple of 8 with the block's zero row),
  // [mid, end): cold deltas (column | sign << 31). beg is a multiple of 4.
  std::vector<uint32_t> row;
  std::vector<uint32_t> dcol;   // staged: local index | sign<<31; cold: column | sign<<31
  std::vector<float> dval;      // normalized: signed value +-row_scale[col] per delta
  std::vector<uint32_t> stage;  // staged global columns, per block ascending
  std::vector<uint32_t> work;   // per block (launch order): estimated work (kept on the host)
};

// rows_cap: rows per block (0 = auto); stage_cap: staged columns per block
// (0 = auto, 600); flatten_gain: as plan_layout (rows saving fewer entries are
// summed from their full row). The view must already be validated (plan_layout).
TileLayout plan_tiles(const cbm_b200_cbm_view& v, uint32_t rows_cap, uint32_t stage_cap,
                      uint32_t num_sms, uint32_t flatten_gain);

}  // namespace cbmb
