/*
 * cbm_b200.h — C ABI of the B200-native CBM multiply (drop-in for the hot path
 * of arXiv 2409.02208's reference library, /root/reference/proj).
 *
 * Plain pointers and sizes only; no torch, no C++ types. Every entry point
 * names the reference interface it replaces (file:line under
 * /root/reference/proj). The reference-side C++ adapter that keeps the
 * reference signatures (cbm::spmm_into(const CbmMatrix&, ...)) is
 * include/cbm_b200_shim.hpp; INTEGRATION.md shows how a maintainer binds it.
 *
 * Error model (mirrors the reference's exceptions, kernels.cpp:11-14,107-109):
 * every int-returning call returns CBM_B200_OK or a status below and sets a
 * thread-local message readable with cbm_b200_last_error(). EINVAL carries the
 * reference's exact std::invalid_argument text ("spmm: inner dimensions
 * differ", "spmm: output has the wrong shape", ...).
 */
#ifndef CBM_B200_H_
#define CBM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CBM_B200_OK = 0,
  CBM_B200_EINVAL = 1,   /* std::invalid_argument in the reference */
  CBM_B200_ECUDA = 2,    /* CUDA runtime / launch failure */
  CBM_B200_ENOMEM = 3,   /* host or device allocation failure */
  CBM_B200_ELOGIC = 4,   /* std::logic_error in the reference (builder) */
  CBM_B200_EFORMAT = 5   /* cbm::format_error (bad or truncated CBM1 container) */
};

#define CBM_B200_VIRTUAL_PARENT 0xFFFFFFFFu /* kVirtualParent, types.hpp:19 */

/* Borrowed view of a pattern CSR matrix (CsrBinaryMatrix, csr.hpp:14-40):
 * row_ptr has n_rows+1 entries, columns strictly increasing per row. */
typedef struct cbm_b200_csr_view {
  uint32_t n_rows;
  uint32_t n_cols;
  const uint64_t* row_ptr;
  const uint32_t* col_idx;
} cbm_b200_csr_view;

/* Borrowed view of a built CBM (CbmMatrix, builder.hpp:66-74; f32 build,
 * real_t = float). values are +-1 (plain) or +-row_scale[col] (normalized),
 * exactly as build_cbm / build_cbm_normalized (builder.cpp:394-429) and
 * load_cbm (io.cpp:369-380) guarantee. topo_order may be NULL. */
typedef struct cbm_b200_cbm_view {
  uint32_t n_rows;
  uint32_t n_cols;
  uint64_t nnz;          /* delta_matrix.nnz() */
  uint64_t alpha;
  int32_t is_normalized;
  const uint32_t* parent;      /* chain.parent[n_rows] */
  const uint32_t* topo_order;  /* chain.topo_order[n_rows] or NULL */
  const uint64_t* row_ptr;     /* delta_matrix.row_ptr[n_rows+1] */
  const uint32_t* col_idx;     /* delta_matrix.col_idx[nnz] */
  const float* values;         /* delta_matrix.values[nnz] */
  const float* row_scale;      /* row_scale[n_rows] (normalized) or NULL */
  /* normalized only, optional: the per-COLUMN scale (n_cols entries) the
   * delta values are checked against (values = +-col_scale[col]) when the view
   * is a row block of a normalized matrix (a rectangular sub-CBM of the 2-D
   * multi-GPU partition); row_scale then scales the block's own
   * rows. NULL: square container, row_scale serves both (io.cpp:369-380). */
  const float* col_scale;
} cbm_b200_cbm_view;

/* ------------------------------------------------------------------------
 * Host construction (stays on the host, timed separately).
 * Replaces build_cbm (builder.hpp:99, builder.cpp:394-404) and
 * build_cbm_normalized (builder.hpp:104-106, builder.cpp:406-429). The result
 * is field-for-field identical to the reference builder's (same chain, same
 * delta matrix, same row_scale bits); see DESIGN.md §Builder.
 * degree_mode: 0 = DegreeMode::augmented, 1 = DegreeMode::original.
 * --------------------------------------------------------------------- */
typedef struct cbm_b200_host_cbm cbm_b200_host_cbm;

int cbm_b200_build(const cbm_b200_csr_view* a, uint64_t alpha, int32_t normalized,
                   int32_t degree_mode, int32_t threads, cbm_b200_host_cbm** out);
/* Same, choosing the arborescence algorithm: 0 = mergeable-heap Edmonds
 * (default, O(E log E)), 1 = the reference's round-synchronous contraction
 * restated (O(E * rounds)). Both return the reference's chain. */
int cbm_b200_build_ex(const cbm_b200_csr_view* a, uint64_t alpha, int32_t normalized,
                      int32_t degree_mode, int32_t threads, int32_t algo,
                      cbm_b200_host_cbm** out);
/* Borrowed view of a built CBM; valid until cbm_b200_host_free. */
int cbm_b200_host_view(const cbm_b200_host_cbm* c, cbm_b200_cbm_view* out);
/* chain.branch_ptr (builder.hpp:38-40): n_branches+1 entries. */
int cbm_b200_host_branches(const cbm_b200_host_cbm* c, const uint64_t** branch_ptr,
                           uint64_t* n_branches);
/* Build statistics: seconds per phase and the candidate-edge count. */
typedef struct cbm_b200_build_stats {
  double t_edges, t_arborescence, t_deltas, t_total;
  uint64_t candidate_edges;
  uint32_t rounds;
} cbm_b200_build_stats;
int cbm_b200_host_stats(const cbm_b200_host_cbm* c, cbm_b200_build_stats* out);
void cbm_b200_host_free(cbm_b200_host_cbm* c);

/* CBM1 container (io.hpp:44-57): load_cbm (io.cpp:293-382, same validation and
 * messages; f64 values narrowed to f32 like the f32 build) and save_cbm
 * (io.cpp:261-291). Files interoperate with the reference in both directions. */
int cbm_b200_load_cbm1(const char* path, cbm_b200_host_cbm** out);
int cbm_b200_save_cbm1(const cbm_b200_cbm_view* c, const char* path);

/* count_scalar_ops (kernels.hpp:22, kernels.cpp:66-68). */
int cbm_b200_count_ops(const cbm_b200_cbm_view* c, uint64_t* multiply_adds,
                       uint64_t* update_adds);

/* ------------------------------------------------------------------------
 * Device operator: the CBM uploaded once into the level-ordered device layout
 * (DESIGN.md §Layout). Immutable after upload and shareable: calls from any
 * thread are safe, and calls on distinct streams may run concurrently (each
 * stream gets its own per-call workspace; the reference's CbmMatrix is
 * likewise immutable and shareable).
 * --------------------------------------------------------------------- */
typedef struct cbm_b200_matrix cbm_b200_matrix;

typedef struct cbm_b200_options {
  int32_t device;            /* CUDA device ordinal (-1 = current) */
  int32_t order_faithful;    /* 1: every row summed in the reference's exact
                                order (bit-identical for ANY X); 0: rows longer
                                than split_threshold are split into chunks summed
                                in a fixed tree order (bit-exact on integer X,
                                ~1 ulp-level on Gaussian X) */
  uint32_t split_threshold;  /* deltas per row before splitting (0 = auto: a
                                power of two in [32, 1024], ~1/8 of a resident
                                warp's share of the deltas) */
  uint32_t chunk;            /* deltas per chunk (0 = auto: max(32, split/4)) */
  int32_t prescale;          /* normalized only: -1 auto, 0 off, 1 pre-scale X
                                by row_scale once per call (bit-identical
                                products, removes the per-delta FMUL) */
  int32_t kernel;            /* 0 auto (LDG.128-wide lanes when rows allow),
                                1 force scalar lanes (one float per lane) */
  int32_t max_segments;      /* column segments (32 lanes x V floats) per work
                                ticket: 0 auto (up to 4), 1 or 2 to cap */
  int32_t flatten_gain;      /* default mode only: a row whose CBM delta row
                                saves fewer than this many entries over its full
                                row is summed directly (no wait on its parent;
                                same value, CSR summation order). -1 = auto (16),
                                0 = keep every chain link */
  int32_t prefetch;          /* 1: bulk-prefetch a contiguous X that fits in
                                half of L2 before gathering; 0 (default): off
                                (measured neutral on cfg[0]/cfg[1]) */
  int32_t tile;              /* default mode only: tiled path: one
                                CTA per (row block, column slab) with the block's
                                re-used X rows staged in shared memory. -1 auto
                                (used when most deltas hit staged rows and each
                                staged row is re-used enough), 0 off, 1 force */
  uint32_t tile_rows;        /* rows per tile block (0 = auto, 64..512) */
  uint32_t tile_stage;       /* staged X rows per block (0 = auto, 600) */
  int32_t tile_vec;          /* floats per lane of a tile slab: 0 auto, 1, 2, 4 */
  int32_t dense;             /* default mode only: dense-block path:
                                the columns shared by >= dense_min rows of each
                                128-row tile multiplied on the tensor cores
                                (tcgen05, exact tf32 split), the remaining entries
                                by the streaming kernel on top. -1 auto (when the
                                cost model favours it), 0 off, 1 force */
  uint32_t dense_min;        /* entries per column per tile to count as shared
                                (0 = auto, 3) */
  int32_t hub;               /* default mode only: hub-row panel:
                                the longest rows of a power-law matrix (up to 128)
                                leave the streaming kernel and are multiplied as
                                one tile on the tensor cores, each X row loaded
                                once for all of them. -1 auto (when the cost rule
                                favours it), 0 off, 1 force */
} cbm_b200_options;

void cbm_b200_default_options(cbm_b200_options* opt);

/* Upload (the device counterpart of holding a CbmMatrix). Validates the
 * structure like load_cbm does (io.cpp:346-380): parent range/acyclicity,
 * row_ptr monotonicity, column range, value pattern. Host arrays are borrowed
 * only for the duration of the call. */
int cbm_b200_upload(const cbm_b200_cbm_view* c, const cbm_b200_options* opt,
                    cbm_b200_matrix** out);
void cbm_b200_free(cbm_b200_matrix* h);
/* Ship-pre-compressed path: a CBM1 container file straight to
 * the device — the file is memory-mapped and validated by all host threads
 * with load_cbm's rules and messages (io.cpp:293-382; EFORMAT), then uploaded
 * as cbm_b200_upload does. Equivalent to load_cbm1 + upload + host_free. */
int cbm_b200_upload_cbm1(const char* path, const cbm_b200_options* opt,
                         cbm_b200_matrix** out);

/* Y = A X on device memory (spmm_into, kernels.hpp:36-39, kernels.cpp:105-123).
 * X is x_rows x x_cols row-major with leading dimension ldx (floats); Y is
 * y_rows x y_cols with leading dimension ldy; Y is fully overwritten. A column
 * slab of a wider matrix is passed as (base + c0, ldx = full width); ldx must
 * be below 2^30 (EINVAL otherwise). Async on `stream` (a cudaStream_t; NULL =
 * legacy default stream). */
int cbm_b200_spmm(cbm_b200_matrix* h, const float* x, int64_t x_rows, int64_t x_cols,
                  int64_t ldx, float* y, int64_t y_rows, int64_t y_cols, int64_t ldy,
                  void* stream);

/* cbm_b200_spmm with epilogue flags: CBM_B200_RELU applies relu_inplace
 * (dense.cpp:51-54: v < 0 -> +0) to Y in the multiply's epilogue, as the
 * first GCN layer does (gcn.cpp:29-30). */
#define CBM_B200_RELU 1u
int cbm_b200_spmm_ex(cbm_b200_matrix* h, const float* x, int64_t x_rows, int64_t x_cols,
                     int64_t ldx, float* y, int64_t y_rows, int64_t y_cols, int64_t ldy,
                     uint32_t flags, void* stream);

/* Same with HOST buffers (the drop-in for spmm_into on DenseMatrix data):
 * H2D of X, the multiply, D2H of Y, then a stream synchronize. Pinned host
 * memory gives full-bandwidth copies; pageable memory works too. */
int cbm_b200_spmm_host(cbm_b200_matrix* h, const float* x, int64_t x_rows, int64_t x_cols,
                       float* y, int64_t y_rows, int64_t y_cols, void* stream);

/* Column sharding: every stage of the multiply acts on one
 * column (kernels.cpp:27-62), so device k of n multiplies the contiguous
 * column slab cbm_b200_column_slab(d, n, k) against a full replica of the
 * CBM; no collective is needed. Order-faithful handles give the single-device
 * bits; default-mode slabs may round differently (the kernel variant follows
 * the slab width) within the same tolerance. */
int cbm_b200_column_slab(int64_t d, int32_t world, int32_t rank, int64_t* lo, int64_t* hi);

/* Single-process multi-device spmm_into on HOST buffers: handles[k] (one
 * upload of the same CBM per device, distinct handles) multiplies column slab
 * k of X into slab k of Y; the devices' copies and kernels overlap; returns
 * when Y is complete. Shape errors as spmm_into. */
int cbm_b200_spmm_sharded(cbm_b200_matrix* const* handles, int32_t n_handles, const float* x,
                          int64_t x_rows, int64_t x_cols, float* y, int64_t y_rows,
                          int64_t y_cols);

/* u = A v (spmv_into, kernels.hpp:41-44, kernels.cpp:70-97): v is n_cols x 1. */
int cbm_b200_spmv(cbm_b200_matrix* h, const float* v, int64_t v_rows, int64_t v_cols,
                  float* u, int64_t u_rows, int64_t u_cols, void* stream);

/* C = A B on device memory with the reference's arithmetic (dense_matmul,
 * dense.hpp:48-50, dense.cpp:31-49): per output entry, ascending inner index,
 * zero lhs entries skipped, every product rounded before the add (no FMA) —
 * bit-identical to the reference. A is m x k, B k x n, C m x n, all packed
 * row-major. */
int cbm_b200_dense_matmul(const float* a, int64_t m, int64_t k, const float* b, int64_t n,
                          float* c, void* stream);

/* Fused all-gather + GEMM of the multi-GPU GCN: C = [A_0 | A_1 |
 * ... | A_{P-1}] B, where A_p is m x part_k[p] row-major (leading dimension
 * part_k[p]) and may be ANOTHER device's buffer mapped with cbm_b200_ipc_open,
 * so the tiles of the all-gathered operand are read over NVLink inside the
 * GEMM; C (m x n, leading dimension ldc) is written to every outs[o] (peer
 * buffers too), which fuses the result's gather. 1..8 parts and outputs.
 * ordered = 1: the reference's dense_matmul arithmetic over the concatenated
 * A (ascending k, zero lhs skipped, no FMA: bit-identical); 0: FFMA (part
 * widths multiples of 4). B is sum(part_k) x n packed. Async on `stream`. */
int cbm_b200_gemm_parts(const float* const* a_parts, const int64_t* part_k, int32_t n_parts,
                        int64_t m, const float* b, int64_t n, float* const* outs, int32_t n_outs,
                        int64_t ldc, int32_t ordered, void* stream);

/* CUDA IPC between the ranks of one node: export the allocation holding dptr
 * as a 64-byte handle plus dptr's byte offset inside it, map a peer's handle
 * (device = the caller's GPU, -1 = current; add the offset to the returned
 * base), unmap. A process cannot map its own handle. */
#define CBM_B200_IPC_HANDLE_BYTES 64
int cbm_b200_ipc_handle(const void* dptr, unsigned char* handle64, uint64_t* offset);
int cbm_b200_ipc_open(const unsigned char* handle64, int32_t device, void** dptr);
int cbm_b200_ipc_close(void* dptr);

/* Two-layer GCN inference out = A_hat relu(A_hat (X W0)) W1 (gcn_forward,
 * gcn.hpp:27-29, gcn.cpp:22-33) with a normalized uploaded adjacency: the two
 * GEMMs above, the ReLU fused into the first CBM product's epilogue. X is
 * n x f, W0 f x hid, W1 hid x classes, out n x classes (device, packed). */
int cbm_b200_gcn_forward(cbm_b200_matrix* h, const float* x, int64_t n, int64_t f,
                         const float* w0, int64_t hid, const float* w1, int64_t classes,
                         float* out, void* stream);

/* Pre-size the per-call workspace for up to d_max columns so later calls
 * never allocate (the device analogue of Property 3, kernels.hpp:36-39):
 * cbm_b200_reserve for the legacy default stream, cbm_b200_reserve_on for a
 * given stream. */
int cbm_b200_reserve(cbm_b200_matrix* h, int64_t d_max);
int cbm_b200_reserve_on(cbm_b200_matrix* h, int64_t d_max, void* stream);

typedef struct cbm_b200_info {
  uint32_t n_rows, n_cols;
  uint64_t nnz_delta;        /* delta entries of the uploaded CBM */
  uint64_t nnz_effective;    /* entries the kernel sums (after flattening) */
  uint32_t n_flattened;      /* rows summed directly instead of via their parent */
  uint32_t n_levels;         /* depth of the compression forest */
  uint32_t n_roots;
  uint32_t n_interior;       /* rows with at least one child */
  uint32_t n_items;          /* work items per column slab */
  uint32_t n_chunk_items;    /* split-row chunks per column slab */
  uint32_t max_row_deltas;
  uint64_t device_bytes;     /* structure bytes resident on the device */
  uint32_t launches_per_call;/* kernels launched by the last spmm call */
  int32_t is_normalized;
  int32_t order_faithful;
  int32_t tile_active;       /* multiplies with d >= 32 take the tiled path */
  uint32_t tile_blocks;      /* row blocks of the tiled layout (0: not planned) */
  uint32_t tile_max_rows, tile_max_staged, tile_cut_rows;
  uint64_t tile_deltas;      /* entries the tiled kernel sums (cut rows flattened) */
  uint64_t tile_staged_deltas; /* of which read from the shared-memory tile */
  uint64_t tile_staged_rows;   /* staged X rows over all blocks */
  int32_t dense_active;        /* multiplies with d >= 32 take the dense-block path */
  uint32_t dense_tiles;        /* 128-row tiles */
  uint64_t dense_chunks;       /* 32-column chunks multiplied on the tensor cores */
  uint64_t dense_entries;      /* entries summed by the tensor cores */
  uint64_t cold_entries;       /* entries summed by the streaming kernel */
  int32_t hub_active;          /* the hub-row panel takes the longest rows */
  uint32_t hub_rows;           /* rows in the panel */
  uint64_t hub_entries;        /* entries of those rows (summed by the tensor cores) */
  uint64_t hub_chunks;         /* 32-column chunks over the union of their columns */
} cbm_b200_info;
int cbm_b200_get_info(const cbm_b200_matrix* h, cbm_b200_info* out);

/* Thread-local message of the last failing call on this thread. */
const char* cbm_b200_last_error(void);

/* ------------------------------------------------------------------------
 * Seeded workload generators (bench / test infrastructure). Streams follow the
 * reference's UniformRng (prng.hpp:11-28: mt19937_64, unit() = 53-bit,
 * below(n) = modulo) so CPU and GPU runs see identical inputs.
 * --------------------------------------------------------------------- */
typedef struct cbm_b200_csr cbm_b200_csr;
/* kind: "community" (p = {n, communities, p_in, p_out}),
 *       "pa_triangle" (p = {n, m, p_triangle}),
 *       "clique_overlay" (p = {n, groups, k_min, k_max, zipf_s}),
 *       "random_binary" (p = {rows, cols, density}) — oracles.hpp:167-175. */
int cbm_b200_gen_graph(const char* kind, const double* params, int32_t n_params,
                       uint64_t seed, cbm_b200_csr** out);
int cbm_b200_csr_get(const cbm_b200_csr* a, cbm_b200_csr_view* out);
void cbm_b200_csr_free(cbm_b200_csr* a);
/* Host-only plan of the dense-block layout (no device): what an upload with
 * options.dense = 1 would multiply on the tensor cores. stats:
 * tiles, chunks, dense entries, cold entries, padded slots (tile rows x chunk
 * columns, zeros included), rows of the tallest tile. Validates the view like
 * load_cbm (io.cpp:346-380). */
int cbm_b200_plan_dense(const cbm_b200_cbm_view* c, uint32_t dense_min, uint64_t stats[6]);
/* Host-only: the hub-row panel an upload with options.hub = mode would build
 * (DESIGN.md §6). stats: active (0/1), rows in the panel, their entries, 32-column
 * chunks over the union of their columns, pieces, deltas left to the rest. */
int cbm_b200_plan_hub(const cbm_b200_cbm_view* c, int32_t mode, uint64_t stats[6]);

/* Dense fills: kind 0 = uniform [lo,hi) (random_dense, dense.cpp:56-62),
 * 1 = integers below(hi-lo+1)+lo, 2 = N(0,1) Box-Muller (lo/hi unused),
 * 3 = Glorot-uniform for a lo x hi (fan_in x fan_out) weight. */
int cbm_b200_gen_dense(int32_t kind, uint64_t rows, uint64_t cols, double lo, double hi,
                       uint64_t seed, float* out);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* CBM_B200_H_ */
