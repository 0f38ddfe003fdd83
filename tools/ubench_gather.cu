// Microbenchmark (dev tool): row-gather throughput on B200.
//   mode 0: LDG.128 per lane, PF rows in flight per warp (register staging)
//   mode 1: cp.async.bulk (one lane) into a per-warp smem ring of R slots
// Each warp gathers `per_warp` random rows of `row_bytes` from a table and sums them.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench_gather.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int PF>
__global__ void reg_gather(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                           int per_warp, int row_f4, float* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t* my = idx + (size_t)gw * per_warp;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int k = 0; k < per_warp; k += PF) {
    float4 v[PF];
#pragma unroll
    for (int q = 0; q < PF; ++q) v[q] = __ldg(tab + (size_t)my[k + q] * row_f4 + lane);
#pragma unroll
    for (int q = 0; q < PF; ++q) { acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w; }
  }
  out[gw * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

template <int R, bool SPIN>
__global__ void bulk_gather(const float* __restrict__ tab, const uint32_t* __restrict__ idx,
                            int per_warp, int row_bytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = blockDim.x / 32;
  float* ring = reinterpret_cast<float*>(sm) + (size_t)warp * R * (row_bytes / 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)nw * R * row_bytes) + warp * R;
  if (lane == 0) {
    for (int r = 0; r < R; ++r) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bars + r)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const uint32_t* my = idx + (size_t)gw * per_warp;
  uint32_t win = my[lane], nwin = my[32 + lane];   // indices [k0, k0+64) in registers
  int k0 = 0;
  auto issue = [&](int k) {
    const uint32_t o = k - k0;
    const uint32_t ia = __shfl_sync(0xffffffffu, win, o & 31), ib = __shfl_sync(0xffffffffu, nwin, o & 31);
    const uint32_t row = o < 32 ? ia : ib;
    if (lane == 0) {
      const int r = k % R;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bars + r)), "r"(row_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(ring + (size_t)r * (row_bytes / 4))), "l"(tab + (size_t)row * (row_bytes / 4)),
                   "r"(row_bytes), "r"(sa(bars + r)) : "memory");
    }
  };
  for (int k = 0; k < R && k < per_warp; ++k) issue(k);
  float acc = 0;
  for (int k = 0; k < per_warp; ++k) {
    const int r = k % R;
    const uint32_t par = (k / R) & 1;
    if (SPIN)
      asm volatile("{\n\t.reg .pred P1;\nT_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra T_%=;\n\t}" ::"r"(sa(bars + r)), "r"(par) : "memory");
    else
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(sa(bars + r)), "r"(par) : "memory");
    const float* src = ring + (size_t)r * (row_bytes / 4);
    for (int c = lane; c < row_bytes / 4; c += 32) acc += src[c];
    __syncwarp();
    if (k + R < per_warp) issue(k + R);
    if (k + 1 - k0 == 32) { k0 += 32; win = nwin; nwin = k0 + 32 + lane < per_warp ? my[k0 + 32 + lane] : 0; }
  }
  out[gw * 32 + lane] = acc;
}

template <int R>
__global__ void cpa_gather(const float* __restrict__ tab, const uint32_t* __restrict__ idx,
                           int per_warp, int row_bytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * R * 32;
  const uint32_t* my = idx + (size_t)gw * per_warp;
  uint32_t win = my[lane], nwin = my[32 + lane];
  int k0 = 0;
  auto issue = [&](int k) {
    if (k < per_warp) {
      const uint32_t o = k - k0;
      const uint32_t ia = __shfl_sync(0xffffffffu, win, o & 31), ib = __shfl_sync(0xffffffffu, nwin, o & 31);
      const uint32_t row = o < 32 ? ia : ib;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + (k % R) * 32 + lane);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(reinterpret_cast<const float4*>(tab) + (size_t)row * (row_bytes / 16) + lane) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int k = 0; k < R; ++k) issue(k);
  float acc = 0;
  for (int k = 0; k < per_warp; ++k) {
    asm volatile("cp.async.wait_group %0;" ::"n"(R - 1) : "memory");
    const float4 v = ring[(k % R) * 32 + lane];
    acc += v.x + v.y + v.z + v.w;
    issue(k + R);
    if (k + 1 - k0 == 32) { k0 += 32; win = nwin; nwin = k0 + 32 + lane < per_warp ? my[k0 + 32 + lane] : 0; }
  }
  out[gw * 32 + lane] = acc;
}

int main1(int argc, char** argv) {
  const int rows = 80000, row_bytes = argc > 1 ? atoi(argv[1]) : 512;
  const int per_warp = 256;
  float* tab; uint32_t* idx; float* out;
  cudaMalloc(&tab, (size_t)rows * row_bytes);
  cudaMemset(tab, 0, (size_t)rows * row_bytes);
  const int max_warps = 148 * 64;
  std::vector<uint32_t> h((size_t)max_warps * per_warp);
  srand(1);
  for (auto& v : h) v = rand() % rows;
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&out, (size_t)max_warps * 32 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto report = [&](const char* name, int warps, float ms) {
    const double bytes = double(warps) * per_warp * row_bytes;
    printf("%-34s warps=%6d  %8.1f us  %7.2f TB/s  %6.1f ns/row/warp\n", name, warps, ms * 1e3,
           bytes / (ms * 1e-3) / 1e12, ms * 1e6 / per_warp);
  };
  for (int wpsm : {4, 16, 20, 32}) {
    const int warps = 148 * wpsm;
    if (row_bytes == 512) {
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        reg_gather<8><<<warps / 4, 128>>>((const float4*)tab, idx, per_warp, row_bytes / 16, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      report("reg PF=8", warps, ms);
    }
    if (row_bytes == 512) {
      auto runc = [&](auto kern, int R) {
        const size_t smem = 4 * (size_t)R * 512;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float ms = 0;
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(a);
          kern<<<warps / 4, 128, smem>>>(tab, idx, per_warp, row_bytes, out);
          cudaEventRecord(b); cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        char nm[64]; snprintf(nm, sizeof nm, "cp.async R=%d", R);
        report(nm, warps, ms);
      };
      runc(cpa_gather<8>, 8); runc(cpa_gather<16>, 16); runc(cpa_gather<32>, 32);
    }
    for (int R : {4, 8, 16, 32}) {
      if (true) continue;
      const size_t smem = 4 * (size_t)R * (row_bytes + 8);
      if (smem * (wpsm / 4) > 220 * 1024) continue;
      auto run = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(a);
          kern<<<warps / 4, 128, smem>>>(tab, idx, per_warp, row_bytes, out);
          cudaEventRecord(b); cudaEventSynchronize(b);
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        char nm[64]; snprintf(nm, sizeof nm, "bulk R=%d row=%dB", R, row_bytes);
        report(nm, warps, ms);
      };
      if (R == 4) { run(bulk_gather<4, false>); run(bulk_gather<4, true>); }
      if (R == 16) { run(bulk_gather<16, false>); run(bulk_gather<16, true>); }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

// Double-buffered register ring: PF rows (U float4 per lane each) land in one
// register set while the other is summed (the consume/issue overlap of the
// CBM kernel without the shared-memory round trip).
template <int PF, int U>
__global__ void reg2_gather(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                            int per_warp, int row_f4, float* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t* my = idx + (size_t)gw * per_warp;
  float4 acc = make_float4(0, 0, 0, 0);
  float4 va[PF][U], vb[PF][U];
  uint32_t win = my[lane];
  auto load = [&](float4 (&v)[PF][U], int k) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const uint32_t r = __shfl_sync(0xffffffffu, win, (k + q) & 31);
#pragma unroll
      for (int u = 0; u < U; ++u) v[q][u] = __ldcg(tab + (size_t)r * row_f4 + u * 32 + lane);
    }
  };
  auto sum = [&](float4 (&v)[PF][U]) {
#pragma unroll
    for (int q = 0; q < PF; ++q)
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[q][u].x; acc.y += v[q][u].y; acc.z += v[q][u].z; acc.w += v[q][u].w; }
  };
  load(va, 0);
  for (int k = 0; k < per_warp; k += 2 * PF) {
    load(vb, k + PF);
    sum(va);
    if (((k + 2 * PF) & 31) == 0) win = k + 2 * PF + lane < per_warp ? my[k + 2 * PF + lane] : 0;
    if (k + 2 * PF < per_warp) load(va, k + 2 * PF);
    sum(vb);
  }
  out[gw * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

// cp.async ring of R slots of U segments, B slots per commit group, read back with LDS
template <int R, int U, int B>
__global__ void cpa2_gather(const float* __restrict__ tab, const uint32_t* __restrict__ idx,
                            int per_warp, int row_bytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * R * 32 * U;
  const uint32_t* my = idx + (size_t)gw * per_warp;
  uint32_t win = my[lane];
  constexpr int G = R / B;
  auto issue = [&](int k) {  // group of B rows starting at k
    if (k < per_warp) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const uint32_t row = __shfl_sync(0xffffffffu, win, (k + b) & 31);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + (((k + b) % R) * U + u) * 32 + lane);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                       "l"(reinterpret_cast<const float4*>(tab) + (size_t)row * (row_bytes / 16) + u * 32 + lane) : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int g = 0; g < G; ++g) issue(g * B);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int k = 0; k < per_warp; k += B) {
    asm volatile("cp.async.wait_group %0;" ::"n"(G - 1) : "memory");
    float4 v[B][U];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int u = 0; u < U; ++u) v[b][u] = ring[(((k + b) % R) * U + u) * 32 + lane];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[b][u].x; acc.y += v[b][u].y; acc.z += v[b][u].z; acc.w += v[b][u].w; }
    __syncwarp();
    if (((k + R) & 31) == 0) win = k + R + lane < per_warp ? my[k + R + lane] : 0;
    issue(k + R);
  }
  out[gw * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

int main2(int row_bytes) {
  const int rows = (40 << 20) / row_bytes, per_warp = 512;
  float* tab; uint32_t* idx; float* out;
  cudaMalloc(&tab, (size_t)rows * row_bytes);
  cudaMemset(tab, 0, (size_t)rows * row_bytes);
  const int max_warps = 148 * 64;
  std::vector<uint32_t> h((size_t)max_warps * per_warp);
  srand(1);
  for (auto& v : h) v = rand() % rows;
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&out, (size_t)max_warps * 32 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto report = [&](const char* name, int warps, float ms) {
    const double bytes = double(warps) * per_warp * row_bytes;
    printf("row=%5dB %-30s warps/SM=%3d  %8.1f us  %7.2f TB/s\n", row_bytes, name, warps / 148, ms * 1e3,
           bytes / (ms * 1e-3) / 1e12);
  };
  auto time = [&](auto launch) {
    float best = 1e30f;
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (it) best = ms < best ? ms : best;
    }
    return best;
  };
  for (int wpsm : {12, 16, 20, 24, 32}) {
    const int warps = 148 * wpsm;
    if (row_bytes == 512) {
      report("reg2 PF=4 U=1", warps, time([&] { reg2_gather<4, 1><<<warps / 4, 128>>>((const float4*)tab, idx, per_warp, row_bytes / 16, out); }));
      report("reg2 PF=8 U=1", warps, time([&] { reg2_gather<8, 1><<<warps / 4, 128>>>((const float4*)tab, idx, per_warp, row_bytes / 16, out); }));
      auto k = cpa2_gather<16, 1, 8>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16 * 512);
      if (wpsm <= 20) report("cp.async R=16 U=1 B=8", warps, time([&] { k<<<warps / 4, 128, 4 * 16 * 512>>>(tab, idx, per_warp, row_bytes, out); }));
    } else if (row_bytes == 2048) {
      report("reg2 PF=2 U=4", warps, time([&] { reg2_gather<2, 4><<<warps / 4, 128>>>((const float4*)tab, idx, per_warp, row_bytes / 16, out); }));
      report("reg2 PF=1 U=4", warps, time([&] { reg2_gather<1, 4><<<warps / 4, 128>>>((const float4*)tab, idx, per_warp, row_bytes / 16, out); }));
      auto k = cpa2_gather<4, 4, 2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4 * 2048);
      if (wpsm <= 20) report("cp.async R=4 U=4 B=2", warps, time([&] { k<<<warps / 4, 128, 4 * 4 * 2048>>>(tab, idx, per_warp, row_bytes, out); }));
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 2) return main2(atoi(argv[1]));
  return main1(argc, argv);
}
