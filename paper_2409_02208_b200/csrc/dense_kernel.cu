// Dense-block path: the shared columns of each 128-row tile of
// the represented matrix (dense_layout.cpp) multiplied on the 5th-generation
// tensor cores. Per work unit (tile t, feature block of 128 columns of X):
//
//   D[f, r] = sum_k X'[col_k, f] * B[r, k]        (f: 128 features, r: 128 rows)
//
// with X' = X (binary) or fl(s_col * X) (normalized, the reference's per-product
// rounding, kernels.cpp:30-35) and B the tile's 0/1 pattern on the chunk
// columns. This is the transposed product Y_tile^T = X'^T B^T, so that:
//   * A operand = X'^T, written straight from registers into TMEM by the
//     producer warps (tcgen05.st; lane = feature, one column per K element):
//     the gathered X rows never touch shared memory;
//   * B operand = the 0/1 tile, expanded from bit masks into shared memory in
//     the 128-byte-swizzled K-major layout the MMA reads (1.0f / 0.0f);
//   * D accumulates in TMEM (fp32), double-buffered so the epilogue of one
//     unit overlaps the MMAs of the next.
// Exactness: kind::tf32 multiplies 19-bit operands, so each X' element is
// split into hi = X' with the low 13 mantissa bits cleared and lo = X' - hi
// (exact); D += A_hi B + A_lo B. B is exactly 0 or 1, integer X is exact in
// hi alone, and the lo term carries the rest to within 2^-21 relative.
// Sums run in a different order than the reference (default mode: bit-exact
// on integer X, <= 1e-5 normwise otherwise).
//
// Warp roles (30 warps, one CTA per SM, persistent over the units):
//   w0      MMA issuer (one elected lane) and TMEM owner (512 columns)
//   w1      metadata loader: each chunk's record (32 columns, their scales,
//           128 row masks; 768 B) copied into a 32-deep shared-memory ring
//           with cp.async, completion tracked by an mbarrier, so no role waits
//           on a dependent global load
//   w2-w5   B expanders: row masks -> swizzled 0/1 tiles (chunks g = e mod 4;
//           a 16-entry nibble table, one st.shared.v4 per 16 bytes)
//   w6-w17  X gatherers: warp i copies X row slices i, i+12, i+24 (512 B each)
//           of every chunk into one of 6 shared-memory slots with cp.async; a
//           warp sustains only a few rows in flight, so the gather bandwidth
//           comes from the number of gathering warps
//   w18-w25 two converter sets of four warps (one per TMEM lane quarter):
//           staged slice -> scale -> hi/lo split -> tcgen05.st into TMEM
//   w26-w29 epilogue: TMEM -> registers -> Y (unscaled; the streaming kernel
//           adds the cold entries and applies the row scale on top)
// Stages: 4 X'/B stages (64 TMEM columns + 16 KB smem each), 2 accumulators
// (128 TMEM columns each): 4 * 64 + 2 * 128 = 512 columns.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cuda_common.hpp"
#include "dense_layout.hpp"

namespace cbmb {

namespace {

// Role counts (measured defaults; overridable for A/B builds, `make alt`).
#ifndef DENSE_SETS
#define DENSE_SETS 2
#endif
#ifndef DENSE_EXPANDERS
#define DENSE_EXPANDERS 4
#endif
#ifndef DENSE_GATHERERS
#define DENSE_GATHERERS 12
#endif
constexpr int kStages = 4;
constexpr int kSets = DENSE_SETS;       // converter sets (set j owns chunks g = j mod kSets)
constexpr int kExpanders = DENSE_EXPANDERS;
constexpr int kGatherers = DENSE_GATHERERS; // cp.async gatherers: warp i copies rows i, i+G, i+2G... of every chunk
constexpr int kRowsPerGatherer = (kDenseK + kGatherers - 1) / kGatherers;
constexpr int kMeta = 32;      // metadata ring depth (chunks)
constexpr int kXSlots = 6;     // staged X' slices in shared memory (chunks in flight)
constexpr int kGatherAhead = 3;  // a gatherer's copy groups in flight behind the signalled chunk
constexpr int kMetaAhead = 8;    // the loader's record groups in flight
constexpr int kGath0 = 2 + kExpanders;       // first gatherer warp
constexpr int kProd0 = kGath0 + kGatherers;  // first converter warp
constexpr int kEpi0 = kProd0 + 4 * kSets;    // first epilogue warp
constexpr int kWarps = kEpi0 + 4;
static_assert(kWarps <= 32, "one CTA: at most 1024 threads");
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCol = 0;       // two accumulators: columns [0,128), [128,256)
constexpr uint32_t kStageCol = 256;   // stage s: [256 + 64 s, 256 + 64 s + 64): hi | lo
constexpr uint32_t kBBytes = kDenseRows * kDenseK * 4;  // 16 KB per B stage
constexpr uint32_t kXBytes = kDenseK * kDenseFeat * 4;   // 16 KB per staged X slice

struct DenseParams {
  const float* __restrict__ x;
  long long ldx;
  float* y;
  long long ldy;
  const float* __restrict__ scale;     // normalized: per-column scale, else null
  const uint4* __restrict__ tiles;     // row0, rows, first chunk, chunks
  const uint32_t* __restrict__ meta;   // kDenseMetaWords per chunk (dense_layout.hpp)
  uint32_t n_units;                    // tiles x feature blocks
  uint32_t n_fb;                       // feature blocks of kDenseFeat
  uint32_t d;
  unsigned long long* trace;  // dev only (CBM_B200_DENSE_TRACE): CTA 0's MMA-warp timeline
  uint32_t dbg;  // dev A/B only (CBM_B200_DENSE_DBG): 1 no X loads, 2 no MMAs, 4 no B fill,
                 // 8 no Y stores
};

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   saddr(b))
               : "memory");
}
// K-major operand, 128-byte rows, 128-byte swizzle (8-row groups 1024 B apart)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_byte_addr) {
  return uint64_t((smem_byte_addr & 0x3FFFF) >> 4) | (uint64_t(1) << 16) |
         (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#define R32(a)                                                                                   \
  "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]),        \
      "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]),          \
      "r"(a[15]), "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]),        \
      "r"(a[22]), "r"(a[23]), "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]),        \
      "r"(a[29]), "r"(a[30]), "r"(a[31])
#define W32(a)                                                                                   \
  "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),            \
      "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]),    \
      "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]),              \
      "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]), "=r"(a[25]),              \
      "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
#define ARGS32                                                                                   \
  "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, " \
  "%21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32}"

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " ARGS32 ";" ::"r"(taddr), R32(r)
               : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                   taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : W32(r)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// dev tool (CBM_B200_DENSE_TRACE): CTA 0's per-chunk timeline, 8 stamps per
// (role, chunk): roles 0 MMA, 1 loader, 2 expander 0, 3 gatherer 0, 4 converter
// set 0 / quarter 0, 5 epilogue quarter 0 (per unit)
constexpr uint32_t kTraceChunks = 2048;
#define DTRACE(role, g, k)                                                              \
  do {                                                                                  \
    if (p.trace && blockIdx.x == 0 && lane == 0 && (g) < kTraceChunks)                  \
      p.trace[(size_t(role) * kTraceChunks + (g)) * 8 + (k)] = clock64();               \
  } while (0)

struct __align__(16) DenseBars {
  uint64_t xfull[kStages], xempty[kStages], bfull[kStages];
  uint64_t accfull[2], accempty[2];
  uint64_t mfull[kMeta], mempty[kMeta];
  uint64_t sfull[kXSlots], sempty[kXSlots];
  uint32_t tmem_base;
  uint32_t pad[3];
  uint4 lut[16];   // the 4 floats (0.0 / 1.0) of each 4-bit mask nibble
};
constexpr uint32_t kMetaBytes = kDenseMetaWords * 4;

// Units are walked identically by every role: CTA b takes b, b + G, b + 2G...
__device__ __forceinline__ uint4 unit_tile(const DenseParams& p, uint32_t u, uint32_t& fb) {
  fb = u % p.n_fb;
  return p.tiles[u / p.n_fb];
}

// The CTA's chunk sequence (units b, b + G, ...; their chunks in order),
// restricted to the chunks g with g % stride == phase: lets a role that owns
// every stride-th chunk look one chunk ahead (prefetch) without replaying the
// unit walk by hand.
struct ChunkIter {
  uint32_t u, j, g;      // current unit, chunk within it, global chunk counter
  uint4 t;               // current unit's tile record
  uint32_t fb;
  bool done;
  __device__ void load(const DenseParams& p) {
    done = u >= p.n_units;
    if (!done) t = unit_tile(p, u, fb);
  }
  __device__ void init(const DenseParams& p, uint32_t phase, uint32_t stride) {
    u = blockIdx.x;
    j = 0;
    g = 0;
    load(p);
    skip(p, phase, stride);
  }
  // advance to the next position whose g matches (phase mod stride)
  __device__ void skip(const DenseParams& p, uint32_t phase, uint32_t stride) {
    while (!done) {
      if (j >= t.w) {
        u += gridDim.x;
        j = 0;
        load(p);
        continue;
      }
      if (g % stride == phase) return;
      ++j;
      ++g;
    }
  }
  __device__ void next(const DenseParams& p, uint32_t phase, uint32_t stride) {
    ++j;
    ++g;
    skip(p, phase, stride);
  }
};

template <bool NORM>
__global__ void __launch_bounds__(kThreads, 1) dense_kernel(const DenseParams p) {
  extern __shared__ __align__(1024) unsigned char dsmem[];
  // B stages at the first 1024-byte boundary (the swizzle is address-based)
  unsigned char* bstage = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  unsigned char* xslot = bstage + kStages * kBBytes;  // kXSlots x [32 columns][128 features]
  const uint32_t* meta_ring =
      reinterpret_cast<const uint32_t*>(xslot + kXSlots * kXBytes);
  DenseBars* bars = reinterpret_cast<DenseBars*>(reinterpret_cast<unsigned char*>(
                                                     const_cast<uint32_t*>(meta_ring)) +
                                                 kMeta * kMetaBytes);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(&bars->tmem_base)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  } else if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars->xfull[s], 4);
      mbar_init(&bars->xempty[s], 1);
      mbar_init(&bars->bfull[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bars->accfull[a], 1);
      mbar_init(&bars->accempty[a], 4);
    }
    for (int m = 0; m < kMeta; ++m) {
      mbar_init(&bars->mfull[m], 1);            // the loader's lane 0, once the record has landed
      mbar_init(&bars->mempty[m], 1 + kGatherers + 4);  // expander, gatherers, converter set
    }
    for (int q = 0; q < kXSlots; ++q) {
      mbar_init(&bars->sfull[q], kGatherers);   // one arrive per gatherer warp
      mbar_init(&bars->sempty[q], 4);           // the converter set's four warps
    }
    for (uint32_t q = 0; q < 16; ++q)
      bars->lut[q] = make_uint4(q & 1 ? 0x3F800000u : 0u, q & 2 ? 0x3F800000u : 0u,
                                q & 4 ? 0x3F800000u : 0u, q & 8 ? 0x3F800000u : 0u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = bars->tmem_base;
  const uint32_t G = gridDim.x;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    // instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kDenseRows >> 3) << 17) |
                           ((kDenseFeat >> 4) << 24);
    uint32_t g = 0, nacc = 0;
    for (uint32_t u = blockIdx.x; u < p.n_units; u += G) {
      uint32_t fb;
      const uint4 t = unit_tile(p, u, fb);
      if (t.w == 0) continue;
      const uint32_t a = nacc & 1;
      mbar_wait(&bars->accempty[a], ((nacc >> 1) & 1) ^ 1);
      tc_fence_after();
      // Two chunks per turn (kStages = 4: two stages in the MMAs, two being
      // filled): the issuing lane blocks ~830 cycles per chunk inside its eight
      // issues (the MMAs' real-data rate) and spends another ~400 in the operand
      // waits and the loop around them; issuing a pair back to back halves the
      // number of those gaps.
      for (uint32_t j = 0; j < t.w;) {
        const uint32_t n2 = (j + 1 < t.w && !(p.dbg & 256)) ? 2u : 1u;
        for (uint32_t q = 0; q < n2; ++q) {
          const uint32_t s = (g + q) % kStages, ph = ((g + q) / kStages) & 1;
          DTRACE(0, g + q, 0);
          mbar_wait(&bars->xfull[s], ph);
          DTRACE(0, g + q, 1);
          mbar_wait(&bars->bfull[s], ph);
          DTRACE(0, g + q, 2);
        }
        tc_fence_after();
        if (lane == 0 && !(p.dbg & 2)) {
          for (uint32_t q = 0; q < n2; ++q) {
            const uint32_t s = (g + q) % kStages;
            const uint64_t bdesc = sw128_desc(saddr(bstage + s * kBBytes));
#pragma unroll
            for (uint32_t piece = 0; piece < 2; ++piece)
#pragma unroll
              for (uint32_t ks = 0; ks < kDenseK / 8; ++ks)
                mma_tf32(tb + kAccCol + 128 * a, tb + kStageCol + 64 * s + 32 * piece + 8 * ks,
                         bdesc + 2 * ks, idesc, (j | q | piece | ks) != 0);
            // one commit frees the stage for both operand producers
            tc_commit(&bars->xempty[s]);
          }
          if (j + n2 == t.w) tc_commit(&bars->accfull[a]);
        } else if (lane == 0) {
          for (uint32_t q = 0; q < n2; ++q) mbar_arrive(&bars->xempty[(g + q) % kStages]);
          if (j + n2 == t.w) mbar_arrive(&bars->accfull[a]);
        }
        DTRACE(0, g, 3);
        __syncwarp();
        j += n2;
        g += n2;
      }
      ++nacc;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ metadata loader
    // One arrive per record, not one per lane (a few dozen mbarrier arrives per
    // chunk instead of ~450; measured neutral, kept for the shorter barrier
    // traffic). The warp commits one cp.async group per record and signals
    // record g - kMetaAhead once at most kMetaAhead newer groups are pending.
    ChunkIter it;
    it.init(p, 0, 1);
    uint32_t issued = 0;
    while (!it.done) {
      const uint32_t m = it.g % kMeta, ph = (it.g / kMeta) & 1;
      DTRACE(1, it.g, 0);
      mbar_wait(&bars->mempty[m], ph ^ 1);
      DTRACE(1, it.g, 1);
      const unsigned char* src =
          reinterpret_cast<const unsigned char*>(p.meta + size_t(it.t.z + it.j) * kDenseMetaWords);
      const uint32_t dst = saddr(meta_ring) + m * kMetaBytes;
      for (uint32_t o = 16 * lane; o < kMetaBytes; o += 512)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + o), "l"(src + o)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      ++issued;
      if (issued > kMetaAhead) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kMetaAhead) : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->mfull[(issued - 1 - kMetaAhead) % kMeta]);
      }
      DTRACE(1, it.g, 2);
      it.next(p, 0, 1);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    if (lane == 0)
      for (uint32_t k = issued > kMetaAhead ? issued - kMetaAhead : 0; k < issued; ++k)
        mbar_arrive(&bars->mfull[k % kMeta]);
  } else if (warp >= 2 && warp < 2 + kExpanders) {
    // ------------------------------------------------------------ B expanders
    const uint32_t e = warp - 2;
    ChunkIter it;
    it.init(p, e, kExpanders);
    while (!it.done) {
      const uint32_t s = it.g % kStages, ph = (it.g / kStages) & 1;
      const uint32_t m = it.g % kMeta, mph = (it.g / kMeta) & 1;
      if (e == 0) DTRACE(2, it.g, 0);
      mbar_wait(&bars->mfull[m], mph);
      if (e == 0) DTRACE(2, it.g, 1);
      const uint32_t* mk = meta_ring + m * kDenseMetaWords + 2 * kDenseK;
      uint32_t cur[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) cur[i] = mk[32 * i + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->mempty[m]);
      mbar_wait(&bars->xempty[s], ph ^ 1);   // the stage's MMAs are done: B may be overwritten
      if (e == 0) DTRACE(2, it.g, 2);
      // item = 32 k + lane: tile row r = 4 k + lane / 8, 16-byte chunk q of its
      // 128-byte line, stored at chunk q ^ (r & 7) (the 128-byte swizzle)
      const uint32_t q = lane & 7, rsub = lane >> 3;
      const uint32_t bs = saddr(bstage) + s * kBBytes;
      const uint32_t lut = saddr(&bars->lut[0]);
#pragma unroll
      for (uint32_t k = 0; k < (p.dbg & 4 ? 0u : 32u); ++k) {
        const uint32_t r = 4 * k + rsub;
        const uint32_t mask = __shfl_sync(0xFFFFFFFFu, cur[k >> 3], r & 31);
        uint4 v;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(lut + 16 * ((mask >> (4 * q)) & 15)));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                         bs + (r >> 3) * 1024 + (r & 7) * 128 + ((q ^ (r & 7)) << 4)),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->bfull[s]);
      if (e == 0) DTRACE(2, it.g, 3);
      it.next(p, e, kExpanders);
    }
  } else if (warp >= kGath0 && warp < kProd0) {
    // ------------------------------------------------------------ X gatherers
    // chunk g's 32 X row slices (128 features = 512 B each) copied into slot
    // g mod kXSlots with cp.async, one row slice per warp instruction; the
    // slot's mbarrier completes when every lane's copies have landed
    const uint32_t gi = warp - kGath0;
    ChunkIter it;
    it.init(p, 0, 1);
    uint32_t issued = 0;   // chunks whose copies this warp has committed (= it.g)
    while (!it.done) {
      const uint32_t q = it.g % kXSlots, qph = (it.g / kXSlots) & 1;
      const uint32_t m = it.g % kMeta, mph = (it.g / kMeta) & 1;
      if (gi == 0) DTRACE(3, it.g, 0);
      mbar_wait(&bars->mfull[m], mph);
      if (gi == 0) DTRACE(3, it.g, 1);
      uint32_t cols[kRowsPerGatherer];
#pragma unroll
      for (int r = 0; r < kRowsPerGatherer; ++r)
        cols[r] = gi + kGatherers * r < kDenseK
                      ? meta_ring[m * kDenseMetaWords + gi + kGatherers * r] : 0u;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->mempty[m]);
      mbar_wait(&bars->sempty[q], qph ^ 1);
      if (gi == 0) DTRACE(3, it.g, 2);
      const uint32_t f0 = it.fb * kDenseFeat + 4 * lane;      // this lane's 4 features
      const uint32_t dst = saddr(xslot) + q * kXBytes + 16 * lane;
      const bool full = f0 + 4 <= p.d && (p.ldx & 3) == 0 &&
                        (reinterpret_cast<uintptr_t>(p.x) & 15) == 0;
#pragma unroll
      for (int r = 0; r < kRowsPerGatherer; ++r) {
        const uint32_t k = gi + kGatherers * r;
        if (k >= kDenseK) break;
        const float* src = p.x + (long long)cols[r] * p.ldx + f0;
        if (p.dbg & 1) {
        } else if (full) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + k * 512),
                       "l"(src)
                       : "memory");
        } else {  // ragged feature edge or unaligned X: element copies, zeros past d
#pragma unroll
          for (uint32_t e = 0; e < 4; ++e) {
            const uint32_t sz = f0 + e < p.d ? 4u : 0u;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + k * 512 + 4 * e),
                         "l"(sz ? src + e : p.x), "r"(sz)
                         : "memory");
          }
        }
      }
      // one arrive per warp and slot (see the metadata loader): chunk
      // g - kGatherAhead is signalled once at most kGatherAhead newer groups pend
      asm volatile("cp.async.commit_group;" ::: "memory");
      ++issued;
      if (issued > kGatherAhead) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kGatherAhead) : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->sfull[(issued - 1 - kGatherAhead) % kXSlots]);
      }
      if (gi == 0) DTRACE(3, it.g, 3);
      it.next(p, 0, 1);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    if (lane == 0)
      for (uint32_t k = issued > kGatherAhead ? issued - kGatherAhead : 0; k < issued; ++k)
        mbar_arrive(&bars->sfull[k % kXSlots]);
  } else if (warp >= kProd0 && warp < kEpi0) {
    // ------------------------------------------------------------ X' converters
    // set j owns chunks g = j mod kSets: staged slice -> (scale) -> hi/lo split
    // -> TMEM (lane = feature)
    const uint32_t set = (warp - kProd0) / 4, quarter = warp & 3;
    ChunkIter it;
    it.init(p, set, kSets);
    while (!it.done) {
      const uint32_t s = it.g % kStages, ph = (it.g / kStages) & 1;
      const uint32_t m = it.g % kMeta, mph = (it.g / kMeta) & 1;
      const uint32_t q = it.g % kXSlots, qph = (it.g / kXSlots) & 1;
      const bool tr = set == 0 && quarter == 0;
      if (tr) DTRACE(4, it.g, 0);
      mbar_wait(&bars->mfull[m], mph);
      if (tr) DTRACE(4, it.g, 1);
      const float* sc = reinterpret_cast<const float*>(meta_ring + m * kDenseMetaWords + kDenseK);
      mbar_wait(&bars->sfull[q], qph);
      if (tr) DTRACE(4, it.g, 2);
      const float* xs = reinterpret_cast<const float*>(xslot + q * kXBytes) + quarter * 32 + lane;
      mbar_wait(&bars->xempty[s], ph ^ 1);
      if (tr) DTRACE(4, it.g, 3);
      tc_fence_after();
      const uint32_t taddr = tb + ((quarter * 32) << 16) + kStageCol + 64 * s;
#pragma unroll
      for (int part = 0; part < 4; ++part) {   // 8 columns at a time (register budget)
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float w = xs[(8 * part + k) * kDenseFeat];
          if constexpr (NORM) w = __fmul_rn(w, sc[8 * part + k]);
          hi[k] = __float_as_uint(w) & 0xFFFFE000u;
          lo[k] = __float_as_uint(__fsub_rn(w, __uint_as_float(hi[k])));
        }
        tmem_st8(taddr + 8 * part, hi);
        tmem_st8(taddr + 32 + 8 * part, lo);
      }
      __syncwarp();
      if (tr) DTRACE(4, it.g, 4);
      if (lane == 0) {
        mbar_arrive(&bars->sempty[q]);
        mbar_arrive(&bars->mempty[m]);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->xfull[s]);
      if (tr) DTRACE(4, it.g, 5);
      it.next(p, set, kSets);
    }
  } else if (warp >= kEpi0) {
    // ------------------------------------------------------------ epilogue
    const uint32_t quarter = warp & 3;
    uint32_t nacc = 0;
    for (uint32_t u = blockIdx.x; u < p.n_units; u += G) {
      uint32_t fb;
      const uint4 t = unit_tile(p, u, fb);
      const uint32_t f = fb * kDenseFeat + quarter * 32 + lane;
      const bool live = f < p.d;
      float* ybase = p.y + (long long)t.x * p.ldy + f;
      if (t.w == 0) {  // no shared columns: the dense part is zero
        if (live)
          for (uint32_t r = 0; r < t.y; ++r) __stcs(ybase + (long long)r * p.ldy, 0.f);
        continue;
      }
      const uint32_t a = nacc & 1;
      if (quarter == 0) DTRACE(5, nacc, 0);
      mbar_wait(&bars->accfull[a], (nacc >> 1) & 1);
      if (quarter == 0) DTRACE(5, nacc, 1);
      tc_fence_after();
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < kDenseRows; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tb + ((quarter * 32) << 16) + kAccCol + 128 * a + c0, r);
        if (c0 + 32 == kDenseRows) {  // accumulator drained: the MMA may reuse it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->accempty[a]);
        }
        if (live && !(p.dbg & 8)) {
#pragma unroll
          for (uint32_t j = 0; j < 32; ++j)
            if (c0 + j < t.y) __stcs(ybase + (long long)(c0 + j) * p.ldy, __uint_as_float(r[j]));
        }
      }
      if (quarter == 0) DTRACE(5, nacc, 2);
      ++nacc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// Hub panel: the pieces' partial rows are combined kHubFanIn at a time in
// ascending piece order (a fixed tree: deterministic), round-to-nearest adds.
// Group j of `in` (pieces [j F, j F + F)) becomes piece j of `out`; the last
// level (one group) writes Y[rows[r], :] = sum (*) row scale, optional ReLU.
// One thread per (group, hub row, float4).
__global__ void hub_reduce_kernel(const float* __restrict__ in, uint32_t n_pieces, uint32_t dpad,
                                  float* __restrict__ out, const uint32_t* __restrict__ rows,
                                  const float* __restrict__ srow, uint32_t n_rows, uint32_t d,
                                  float* __restrict__ y, long long ldy, uint32_t relu) {
  const uint32_t per_row = dpad / 4;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows * per_row) return;
  const uint32_t r = i / per_row, f = (i % per_row) * 4;
  const uint32_t g = blockIdx.y, p_lo = g * kHubFanIn;
  const uint32_t p_hi = min(n_pieces, p_lo + kHubFanIn);
  const size_t pstride = size_t(kDenseRows) * dpad;
  const float* src = in + size_t(r) * dpad + f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t p0 = p_lo; p0 < p_hi; p0 += 8) {
    float4 v[8];
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q)
      v[q] = p0 + q < p_hi ? __ldcs(reinterpret_cast<const float4*>(src + (p0 + q) * pstride))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
      acc.x = __fadd_rn(acc.x, v[q].x);
      acc.y = __fadd_rn(acc.y, v[q].y);
      acc.z = __fadd_rn(acc.z, v[q].z);
      acc.w = __fadd_rn(acc.w, v[q].w);
    }
  }
  if (out) {  // an inner level: piece g of the next level
    *reinterpret_cast<float4*>(out + (size_t(g) * kDenseRows + r) * dpad + f) = acc;
    return;
  }
  const float sc = srow ? srow[r] : 1.0f;
  float o[4] = {acc.x, acc.y, acc.z, acc.w};
  float* dst = y + (long long)rows[r] * ldy + f;
#pragma unroll
  for (uint32_t e = 0; e < 4; ++e) {
    if (f + e >= d) break;
    float w = srow ? __fmul_rn(o[e], sc) : o[e];
    if (relu && w < 0.0f) w = 0.0f;
    dst[e] = w;
  }
}

__global__ void hub_scatter_kernel(const float* __restrict__ src, uint32_t ld,
                                   const uint32_t* __restrict__ rows, uint32_t n, uint32_t d,
                                   float* __restrict__ y, long long ldy) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= uint64_t(n) * d) return;
  const uint32_t r = uint32_t(i / d), f = uint32_t(i % d);
  y[(long long)rows[r] * ldy + f] = src[size_t(r) * ld + f];
}

void dense_launch(DeviceMatrix* h, const uint32_t* tiles, const uint32_t* meta, uint32_t n_tiles,
                  const float* x, int64_t ldx, uint32_t d, float* y, int64_t ldy, cudaStream_t s);

}  // namespace

void dense_spmm(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y,
                int64_t ldy, cudaStream_t s) {
  dense_launch(h, h->dtiles, h->dmeta, h->dense.n_tiles, x, ldx, d, y, ldy, s);
}

void hub_spmm(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y, int64_t ldy,
              bool relu, float*& part, uint64_t& part_cap, cudaStream_t s) {
  const uint32_t dpad = (d + 3) & ~3u;
  // level 0: one 128-row partial per piece; level k: one per kHubFanIn of level k-1
  const uint64_t rows0 = uint64_t(h->hub_pieces) * kDenseRows;
  uint64_t total_rows = 0;
  for (uint32_t n = h->hub_pieces; n > 1; n = (n + kHubFanIn - 1) / kHubFanIn)
    total_rows += uint64_t(n) * kDenseRows;
  total_rows = std::max<uint64_t>(total_rows, rows0);
  grow(part, part_cap, total_rows * dpad, "workspace hub partials");
  // the pieces are the dense kernel's tiles: "rows" [128 p, 128 p + 128) of
  // the partial buffer, leading dimension dpad
  dense_launch(h, h->htiles, h->hmeta, h->hub_pieces, x, ldx, d, part, dpad, s);
  const uint32_t threads = h->hub_n_rows * (dpad / 4);
  float* in = part;
  for (uint32_t n = h->hub_pieces;;) {
    const uint32_t groups = (n + kHubFanIn - 1) / kHubFanIn;
    float* out = groups > 1 ? in + uint64_t(n) * kDenseRows * dpad : nullptr;
    hub_reduce_kernel<<<dim3((threads + 127) / 128, groups), 128, 0, s>>>(
        in, n, dpad, out, h->hrows, h->hsrow, h->hub_n_rows, d, y, ldy, relu ? 1u : 0u);
    ck(cudaGetLastError(), "hub_reduce launch");
    ++h->last_launches;
    if (groups == 1) break;
    in = out;
    n = groups;
  }
}

void hub_scatter(const float* src, uint32_t ld, const uint32_t* rows, uint32_t n, uint32_t d,
                 float* y, int64_t ldy, cudaStream_t s) {
  const uint64_t total = uint64_t(n) * d;
  if (total == 0) return;
  hub_scatter_kernel<<<unsigned((total + 255) / 256), 256, 0, s>>>(src, ld, rows, n, d, y, ldy);
  ck(cudaGetLastError(), "hub_scatter launch");
}

namespace {

void dense_launch(DeviceMatrix* h, const uint32_t* tiles, const uint32_t* meta, uint32_t n_tiles,
                  const float* x, int64_t ldx, uint32_t d, float* y, int64_t ldy, cudaStream_t s) {
  DenseParams p;
  p.x = x;
  p.ldx = ldx;
  p.y = y;
  p.ldy = ldy;
  p.scale = h->info.normalized ? h->scale : nullptr;
  p.tiles = reinterpret_cast<const uint4*>(tiles);
  p.meta = meta;
  p.n_fb = (d + kDenseFeat - 1) / kDenseFeat;
  p.d = d;
  p.dbg = 0;
  if (const char* e = std::getenv("CBM_B200_DENSE_DBG")) p.dbg = uint32_t(std::atoi(e));
  p.trace = nullptr;
  const char* trace_path = std::getenv("CBM_B200_DENSE_TRACE");
  if (trace_path) {
    ck(cudaMalloc(&p.trace, 6 * kTraceChunks * 8 * 8), "trace");
    ck(cudaMemsetAsync(p.trace, 0, 6 * kTraceChunks * 8 * 8, s), "trace");
  }
  const uint64_t units = uint64_t(n_tiles) * p.n_fb;
  if (units >= 0xFFFFFFFFull) throw invalid_argument("spmm: too many dense-block units");
  p.n_units = uint32_t(units);
  const size_t smem =
      1024 + kStages * kBBytes + kXSlots * kXBytes + kMeta * kMetaBytes + sizeof(DenseBars);
  const int grid = int(std::min<uint64_t>(units, uint64_t(h->num_sms)));
  if (grid == 0) return;
  if (h->info.normalized) {
    ck(cudaFuncSetAttribute(dense_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(smem)), "dense smem");
    dense_kernel<true><<<grid, kThreads, smem, s>>>(p);
  } else {
    ck(cudaFuncSetAttribute(dense_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(smem)), "dense smem");
    dense_kernel<false><<<grid, kThreads, smem, s>>>(p);
  }
  ck(cudaGetLastError(), "dense_kernel launch");
  if (trace_path) {  // dev tool: CTA 0's stamps, one line per (role, chunk)
    std::vector<unsigned long long> t(6 * kTraceChunks * 8);
    ck(cudaStreamSynchronize(s), "trace");
    ck(cudaMemcpy(t.data(), p.trace, t.size() * 8, cudaMemcpyDeviceToHost), "trace");
    cudaFree(p.trace);
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "call\n");
      for (uint32_t role = 0; role < 6; ++role)
        for (uint32_t g = 0; g < kTraceChunks; ++g) {
          const unsigned long long* q = &t[(size_t(role) * kTraceChunks + g) * 8];
          if (!q[0]) continue;
          std::fprintf(f, "%u %u %llu %llu %llu %llu %llu %llu\n", role, g, q[0], q[1], q[2], q[3],
                       q[4], q[5]);
        }
      std::fclose(f);
    }
  }
}

}  // namespace

}  // namespace cbmb
