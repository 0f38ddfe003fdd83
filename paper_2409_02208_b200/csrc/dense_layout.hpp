// Dense-block layout (DESIGN.md §6 "Dense-block path"): the represented
// matrix (A, or A + I for a normalized CBM) cut into tiles of kDenseRows
// consecutive rows; in each tile the columns that enough of its rows share
// are gathered into chunks of kDenseK columns and multiplied on the tensor
// cores (tcgen05, tf32 split, dense_kernel.cu); every other entry is "cold"
// and summed by the streaming kernel on top of the tensor result.
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/cbm_b200.h"

namespace cbmb {

inline constexpr uint32_t kDenseRows = 128;  // rows per tile (the MMA's N)
inline constexpr uint32_t kDenseK = 32;      // columns per chunk (4 tf32 K-steps of 8)
inline constexpr uint32_t kDenseFeat = 128;  // features per work unit (the MMA's M)
inline constexpr uint32_t kDenseMaxChunks = 64;  // chunks per tile at most (load balance)
inline constexpr uint32_t kDenseMetaWords = 2 * kDenseK + kDenseRows;  // 768 B per chunk
inline constexpr double kDenseChunkCost = 150.0;  // gathers one chunk's time is worth (auto mode)

struct DenseLayout {
  bool ok = false;                // planned (consistent rows, not order-faithful)
  uint32_t n_tiles = 0;
  uint64_t n_chunks = 0;
  uint64_t dense_entries = 0;     // entries summed by the tensor cores
  uint64_t cold_entries = 0;      // entries left to the streaming kernel
  uint64_t padded_slots = 0;      // tile rows x chunk columns multiplied (incl. zeros)
  uint32_t min_count = 0;         // a column is dense in a tile with >= this many entries
  // per tile, in schedule order (heaviest first): row0, rows, first chunk, chunks
  std::vector<uint32_t> tiles;    // 4 x n_tiles
  // per chunk, kDenseMetaWords u32: its kDenseK columns (padding repeats a
  // real column), their scales (f32 bits; 1.0 for a binary matrix) and
  // kDenseRows row masks (bit k = the row has chunk column k)
  std::vector<uint32_t> meta;
  // the cold part as a CBM view: every parent virtual, values +1 or +s_col
  std::vector<uint32_t> cold_parent;
  std::vector<uint64_t> cold_row_ptr;
  std::vector<uint32_t> cold_col;
  std::vector<float> cold_val;
};

// Plans the dense-block layout of a validated CBM view. min_count = 0 picks
// the default (3: a column shared by >= 3 rows of a tile costs less as one
// loaded X row in a tensor-core chunk than as 3 gathers). Returns ok = false
// when some delta row is inconsistent with its parent (no full-row form).
DenseLayout plan_dense(const cbm_b200_cbm_view& v, uint32_t min_count);

}  // namespace cbmb
