// Dev probe (not product code): tcgen05.mma issue rate from one thread with A in
// TMEM and B in 128B-swizzled shared memory, for the shapes the dense-block
// kernel could use. Prints cycles per MMA for kind::tf32 and kind::f16 (bf16)
// at N = 128 and 256 (M = 128, cta_group::1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_rate tools/umma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__device__ volatile int g_stop;

template <int KIND, int N, int CONT>   // KIND 0 = tf32, 1 = f16 (bf16); CONT 1 smem, 2 tmem traffic
__global__ void rate(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* b = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t dummy;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < N * 32; i += blockDim.x)
    reinterpret_cast<uint32_t*>(b)[i] = CONT == 20 ? (((i * 2654435761u) >> 13) & 1 ? 0x3F800000u : 0u) : 0u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&dummy)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  if (CONT == 20 && warp < 4) {   // A: pseudo-random tf32 values in every operand column
    for (int c = 256; c < 512; c += 8) {
      uint32_t r[8];
      for (int k = 0; k < 8; ++k)
        r[k] = (0x3F000000u + ((threadIdx.x * 40503u + (c + k) * 2654435761u) & 0x00FFE000u)) ^ ((c + k) & 1 ? 0x80000000u : 0u);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                       tb + ((32 * warp) << 16) + c),
                   "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  __shared__ __align__(16) float junk[4][32 * 64];
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp >= 4 && CONT == 1) {           // other warps: smem read/write traffic
    float acc = 0;
    const int w = warp & 3, l = threadIdx.x & 31;
    for (int it = 0; !stop && it < 1000000; ++it) {
      float4* q = reinterpret_cast<float4*>(junk[w]) + (it & 15) * 32 + l;
      float4 v = *q;
      acc += v.x;
      *q = make_float4(acc, v.y, v.z, v.w);
    }
    if (acc == 12345.f) out[0] = 1;
  } else if (warp >= 4 && CONT == 2) {    // other warps: TMEM stores into unused columns
    const int q = warp & 3;
    uint32_t r[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    for (int it = 0; !stop && it < 1000000; ++it)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                       tb + ((32 * q) << 16) + 480 + 8 * (it & 3)),
                   "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t bd = desc(smem_u32(b));
    const uint32_t acol = N == 256 ? 256 : 384;   // A columns after the accumulator
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      if (CONT >= 10 && (i & 1) == 0 && i) {   // CONT - 10 commits per 8 MMAs (dummy barrier)
#pragma unroll
        for (int c = 0; c < CONT - 10; ++c)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&dummy)));
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (i | ks) != 0;
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
                       "r"(tb + acol + 8 * ks), "l"(bd + 2 * ks), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
                       "r"(tb + acol + 8 * ks), "l"(bd + 2 * ks), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    unsigned long long t1 = clock64();
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&bar)), "r"(0));
    unsigned long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int KIND, int N, int CONT = 0>
void run(const char* name, int blocks, int threads = 128) {
  unsigned long long* d;
  cudaMalloc(&d, 2 * blocks * 8);
  const int iters = 2000;
  const size_t smem = 1024 + N * 128 + 64;
  cudaFuncSetAttribute(rate<KIND, N, CONT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  rate<KIND, N, CONT><<<blocks, threads, smem>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2 * 148];
  cudaMemcpy(h, d, 2 * blocks * 8, cudaMemcpyDeviceToHost);
  const double macs = 128.0 * N * (KIND == 0 ? 8 : 16);
  printf("%s blocks=%d err=%s: issue %.1f cyc/mma, complete %.1f cyc/mma, %.0f MAC/clk/SM\n", name, blocks,
         cudaGetErrorString(e), double(h[0]) / (iters * 4), double(h[1]) / (iters * 4),
         macs * iters * 4 / double(h[1]));
  cudaFree(d);
}

int main() {
  run<0, 128>("tf32 M128 N128 K8 ", 1);
  run<0, 256>("tf32 M128 N256 K8 ", 1);
  run<1, 128>("bf16 M128 N128 K16", 1);
  run<1, 256>("bf16 M128 N256 K16", 1);
  run<0, 128>("tf32 M128 N128 K8 ", 148);
  run<1, 256>("bf16 M128 N256 K16", 148);
  run<0, 128, 1>("tf32 N128 + smem traffic (12 warps)", 1, 512);
  run<0, 128, 2>("tf32 N128 + tmem st traffic (12 warps)", 1, 512);
  run<0, 128, 20>("tf32 N128, random A / 0-1 B data, 1 CTA", 1);
  run<0, 128, 20>("tf32 N128, random A / 0-1 B data, 148 CTAs", 148);
  run<1, 128, 20>("bf16 N128, random A / 0-1 B data, 148 CTAs", 148);
  run<0, 128, 11>("tf32 N128, 1 commit per 8 MMAs", 1);
  run<0, 128, 13>("tf32 N128, 3 commits per 8 MMAs", 1);
  return 0;
}
