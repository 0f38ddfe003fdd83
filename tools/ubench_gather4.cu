// Microbenchmark (dev tool): random X-row gathers on B200,
//   mode 0: cp.async (LDGSTS.128 per lane) into a per-warp shared-memory ring,
//           the streaming kernel's copy path (cbm_kernels.cu issue_group)
//   mode 1: TMA cp.async.bulk.tensor.2d tile::gather4 (one elected lane copies
//           four rows per instruction, completion on an mbarrier per ring group)
// Same ring geometry (G groups of 4 rows per warp), same residency (CTAs of 4
// warps, `ctas_per_sm` per SM), same consumer (each lane reads its float4s of
// every row back with LDS and sums them). Rows are row_f floats (128 = 512 B,
// 256 = 1 KB); the table is `table_mb` MB (64: L2-resident, 2048: HBM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_gather4 tools/ubench_gather4.cu
//   ./tools/ubench_gather4
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kWarps = 4;

// ---------------------------------------------------------------- mode 0
template <int RF4, int G>  // RF4: float4 per lane per row (row = 32 * RF4 float4)
__global__ void __launch_bounds__(kWarps * 32) cpa_gather(const float4* __restrict__ tab,
                                                          const uint32_t* __restrict__ idx,
                                                          int per_warp, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + warp;
  float4* ring = reinterpret_cast<float4*>(smem) + (size_t)warp * G * 4 * RF4 * 32;
  const uint32_t* my = idx + (size_t)gw * per_warp;
  auto issue = [&](int k) {  // rows k .. k+3 into group (k/4) % G
    const uint4 r = *reinterpret_cast<const uint4*>(my + k);
    const uint32_t rows[4] = {r.x, r.y, r.z, r.w};
    float4* dst = ring + (size_t)((k / 4) % G) * 4 * RF4 * 32;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < RF4; ++u)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(dst + (q * RF4 + u) * 32 + lane)),
                     "l"(tab + (size_t)rows[q] * (RF4 * 32) + u * 32 + lane)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int g = 0; g < G; ++g) issue(4 * g);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int k = 0; k < per_warp; k += 4) {
    asm volatile("cp.async.wait_group %0;" ::"n"(G - 1) : "memory");
    const float4* src = ring + (size_t)((k / 4) % G) * 4 * RF4 * 32;
#pragma unroll
    for (int q = 0; q < 4 * RF4; ++q) {
      const float4 v = src[q * 32 + lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    if (k + 4 * G < per_warp) issue(k + 4 * G);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  out[gw * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

// ---------------------------------------------------------------- mode 1
template <int RF4, int G>
__global__ void __launch_bounds__(kWarps * 32) tma_gather4(const __grid_constant__ CUtensorMap tmap,
                                                           const uint32_t* __restrict__ idx,
                                                           int per_warp, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + warp;
  constexpr uint32_t kRowBytes = RF4 * 32 * 16;
  float4* ring = reinterpret_cast<float4*>(smem) + (size_t)warp * G * 4 * RF4 * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * G * 4 * kRowBytes) + warp * G;
  if (lane == 0) {
    for (int g = 0; g < G; ++g) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bars + g)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint32_t* my = idx + (size_t)gw * per_warp;
  auto issue = [&](int k) {
    if (lane == 0) {
      const int g = (k / 4) % G;
      const uint4 r = *reinterpret_cast<const uint4*>(my + k);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bars + g)),
                   "r"(4 * kRowBytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(ring + (size_t)g * 4 * RF4 * 32)),
          "l"(&tmap), "r"(sa(bars + g)), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
          : "memory");
    }
  };
  for (int g = 0; g < G; ++g) issue(4 * g);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int k = 0; k < per_warp; k += 4) {
    const int g = (k / 4) % G;
    const uint32_t par = ((k / 4) / G) & 1;
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
            sa(bars + g)),
        "r"(par)
        : "memory");
    const float4* src = ring + (size_t)g * 4 * RF4 * 32;
#pragma unroll
    for (int q = 0; q < 4 * RF4; ++q) {
      const float4 v = src[q * 32 + lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    if (k + 4 * G < per_warp) issue(k + 4 * G);
  }
  out[gw * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

template <int RF4, int G>
void run(size_t table_mb, int ctas_per_sm, int sms, EncodeFn encode) {
  const int row_f = RF4 * 128;
  const size_t rows = table_mb * (1ull << 20) / (row_f * 4);
  const int per_warp = 4096;
  const int grid = sms * ctas_per_sm;
  const size_t nw = (size_t)grid * kWarps;
  float* tab;
  CK(cudaMalloc(&tab, rows * row_f * 4));
  {
    std::vector<float> h(rows * row_f);
    for (size_t i = 0; i < h.size(); ++i) h[i] = float((i / row_f) % 7) + 1.0f;  // row r holds (r % 7) + 1
    CK(cudaMemcpy(tab, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  }
  std::vector<uint32_t> hidx(nw * per_warp);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  std::vector<double> want(nw, 0.0);
  for (size_t i = 0; i < hidx.size(); ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    hidx[i] = uint32_t((s >> 33) % rows);
    want[i / per_warp] += double(hidx[i] % 7 + 1) * 4.0 * RF4;  // per lane: 4 * RF4 floats of every row
  }
  uint32_t* idx;
  CK(cudaMalloc(&idx, hidx.size() * 4));
  CK(cudaMemcpy(idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice));
  float* out;
  CK(cudaMalloc(&out, nw * 32 * 4));
  const size_t smem = (size_t)kWarps * G * 4 * row_f * 4 + kWarps * G * 8;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto check = [&](const char* what) {
    std::vector<float> h(nw * 32);
    CK(cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t w = 0; w < nw; ++w)
      for (int l = 0; l < 32; ++l)
        if (double(h[w * 32 + l]) != want[w]) ++bad;
    if (bad) std::printf("    %s: %zu lanes differ from the expected sums\n", what, bad);
  };
  const double bytes = double(nw) * per_warp * row_f * 4;
  for (int mode = 0; mode < 2; ++mode) {
    float best = 1e30f;
    bool ok = true;
    for (int rep = 0; rep < 5 && ok; ++rep) {
      CK(cudaMemset(out, 0, nw * 32 * 4));
      CK(cudaEventRecord(e0));
      if (mode == 0) {
        CK(cudaFuncSetAttribute(cpa_gather<RF4, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cpa_gather<RF4, G><<<grid, kWarps * 32, smem>>>(reinterpret_cast<const float4*>(tab), idx, per_warp, out);
      } else {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)row_f, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)row_f * 4};
        cuuint32_t box[2] = {(cuuint32_t)row_f, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          std::printf("    cuTensorMapEncodeTiled failed: %d\n", (int)r);
          ok = false;
          break;
        }
        CK(cudaFuncSetAttribute(tma_gather4<RF4, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        tma_gather4<RF4, G><<<grid, kWarps * 32, smem>>>(tm, idx, per_warp, out);
      }
      CK(cudaEventRecord(e1));
      cudaError_t e = cudaEventSynchronize(e1);
      if (e != cudaSuccess) {
        std::printf("    mode %d failed: %s\n", mode, cudaGetErrorString(e));
        std::exit(2);
      }
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;
    }
    if (!ok) continue;
    check(mode == 0 ? "cp.async" : "gather4");
    std::printf("  %-22s rows %4d B  table %5zu MB  G=%d (%2d rows in flight/warp)  %d CTAs/SM x 4 warps  smem/CTA %5.1f KB : %7.3f ms  %6.2f TB/s\n",
                mode == 0 ? "cp.async.cg 16B/lane" : "TMA tile::gather4", row_f * 4, table_mb, G, 4 * G,
                ctas_per_sm, smem / 1024.0, best, bytes / (best * 1e-3) / 1e12);
  }
  cudaFree(tab);
  cudaFree(idx);
  cudaFree(out);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
  if (!encode || q != cudaDriverEntryPointSuccess) {
    std::printf("cuTensorMapEncodeTiled not available\n");
    return 1;
  }
  std::printf("%s, %d SMs\n", prop.name, sms);
  for (size_t mb : {size_t(64), size_t(2048)}) {
    std::printf("table %zu MB (%s)\n", mb, mb <= 64 ? "L2-resident" : "HBM");
    run<1, 2>(mb, 5, sms, encode);   // 512 B rows, 8 rows in flight (the d <= 128 kernel's ring is 16)
    run<1, 4>(mb, 5, sms, encode);   // 512 B rows, 16 rows in flight
    run<2, 2>(mb, 5, sms, encode);   // 1 KB rows, 8 in flight (the d = 256 kernel: D = 8)
    run<2, 4>(mb, 3, sms, encode);   // 1 KB rows, 16 in flight (64 KB per CTA)
  }
  return 0;
}
