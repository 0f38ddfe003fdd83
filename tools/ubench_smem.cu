// Shared-memory gather ceiling (dev tool): 16 warps per CTA, one CTA per SM,
// a 160 KB tile of 640 rows x 64 floats; each 16-lane group reads a random
// row (LDS.128 per lane) and accumulates, like the tiled kernel's staged loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_smem tools/ubench_smem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NT, int UNR>
__global__ void __launch_bounds__(NT, 1) gather(const uint32_t* __restrict__ idx, int steps, float* out) {
  extern __shared__ float4 tile[];  // 640 rows x 16 float4
  for (int i = threadIdx.x; i < 640 * 16; i += NT) tile[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 4, gl = lane & 15;
  const uint32_t* ix = idx + (blockIdx.x * (NT / 32) + warp) * 64;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int s = 0; s < steps; ++s) {
    const uint4* q = reinterpret_cast<const uint4*>(ix + ((s * 8) & 63));
    float4 v[UNR * 4];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint4 e = q[u * 2 + g];
      v[u * 4 + 0] = tile[e.x * 16 + gl];
      v[u * 4 + 1] = tile[e.y * 16 + gl];
      v[u * 4 + 2] = tile[e.z * 16 + gl];
      v[u * 4 + 3] = tile[e.w * 16 + gl];
    }
#pragma unroll
    for (int u = 0; u < UNR * 4; ++u) {
      acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
    }
  }
  if (acc.x == 12345.f) out[threadIdx.x] = acc.y + acc.z + acc.w;
}

template <int NT, int UNR>
void run(const uint32_t* idx, float* out, int sms) {
  const int smem = 640 * 16 * 16;
  cudaFuncSetAttribute(gather<NT, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int steps = 20000;
  gather<NT, UNR><<<sms, NT, smem>>>(idx, 10, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  gather<NT, UNR><<<sms, NT, smem>>>(idx, steps, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double bytes = double(sms) * NT / 32 * steps * UNR * 8 * 256;  // 8 deltas x 256 B per unroll step
  const double bpc = bytes / (ms * 1e-3) / sms / (clk * 1e3);
  printf("NT=%d UNR=%d: %.1f us, %.2f TB/s, %.1f B/clk/SM (max clock %d MHz)\n", NT, UNR, ms * 1e3,
         bytes / (ms * 1e-3) / 1e12, bpc, clk / 1000);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = sms * 32 * 64;
  uint32_t* h = new uint32_t[n];
  uint64_t st = 12345;
  for (int i = 0; i < n; ++i) { st = st * 6364136223846793005ull + 1442695040888963407ull; h[i] = uint32_t(st >> 33) % 640; }
  uint32_t* d; float* out;
  cudaMalloc(&d, n * 4); cudaMalloc(&out, 4096);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
  run<512, 1>(d, out, sms);
  run<512, 2>(d, out, sms);
  run<256, 2>(d, out, sms);
  run<1024, 1>(d, out, sms);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
