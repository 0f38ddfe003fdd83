// Dev microbenchmark: GPU-side cost of launching the multiply's grid shape
// (740 CTAs x 128 threads, 44 KB dynamic smem) regular vs cooperative, each
// right after a large fill kernel (as in bench.py's L2 flush), timed with
// events like bench.py. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fill(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void empty_k(int* out) {
  extern __shared__ int sm[];
  __shared__ int s0;
  if (threadIdx.x == 0 && out) s0 = blockIdx.x, out[blockIdx.x] = s0 + (int)(size_t)sm;
}
__global__ void stamp_k(unsigned long long* t) {
  if (threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    t[blockIdx.x] = g;
  }
}

int main() {
  const size_t n = 64ull << 20;  // 256 MB
  float* buf;
  cudaMalloc(&buf, n * 4);
  int* out;
  cudaMalloc(&out, 1 << 20);
  const int grid = 740, threads = 128;
  for (int smem : {0, 44 * 1024}) {
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int coop = 0; coop < 2; ++coop) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float tot = 0;
      const int reps = 50;
      for (int r = 0; r < reps + 3; ++r) {
        fill<<<148 * 8, 512>>>(buf, n, float(r));
        cudaEventRecord(a);
        if (coop) {
          void* args[] = {&out};
          cudaLaunchCooperativeKernel((void*)empty_k, grid, threads, args, smem, 0);
        } else {
          empty_k<<<grid, threads, smem>>>(out);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) tot += ms;
      }
      printf("smem %5d coop %d: %.2f us per launch (after a fill)\n", smem, coop, tot / reps * 1e3);
    }
  }
  // back-to-back without fill
  for (int coop = 0; coop < 2; ++coop) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r < 53; ++r) {
      cudaEventRecord(a);
      if (coop) {
        void* args[] = {&out};
        cudaLaunchCooperativeKernel((void*)empty_k, grid, threads, args, 44 * 1024, 0);
      } else {
        empty_k<<<grid, threads, 44 * 1024>>>(out);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 3) tot += ms;
    }
    printf("no fill, smem 44K coop %d: %.2f us per launch\n", coop, tot / 50 * 1e3);
  }
  // events only, and grid-size sweep, after a fill
  for (int g : {0, 1, 148, 740, 1480}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r < 53; ++r) {
      fill<<<148 * 8, 512>>>(buf, n, float(r));
      cudaEventRecord(a);
      if (g) empty_k<<<g, threads, 0>>>(out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 3) tot += ms;
    }
    printf("after fill, grid %4d: %.2f us\n", g, tot / 50 * 1e3);
  }
  // kernel-to-kernel gap: stamp kernels back to back
  {
    unsigned long long* t;
    cudaMalloc(&t, 2 * 2048 * 8);
    for (int r = 0; r < 5; ++r) {
      fill<<<148 * 8, 512>>>(buf, n, float(r));
      stamp_k<<<740, 128>>>(t);
      stamp_k<<<740, 128>>>(t + 2048);
    }
    unsigned long long h[4096];
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long a0 = ~0ull, a1 = 0, b0 = ~0ull, b1 = 0;
    for (int i = 0; i < 740; ++i) {
      a0 = h[i] < a0 ? h[i] : a0; a1 = h[i] > a1 ? h[i] : a1;
      b0 = h[2048 + i] < b0 ? h[2048 + i] : b0; b1 = h[2048 + i] > b1 ? h[2048 + i] : b1;
    }
    printf("stamp kernel A: CTA start spread %.2f us; B first CTA - A last CTA = %.2f us\n",
           (a1 - a0) / 1e3, (double)(b0 - a1) / 1e3);
  }
  // launch through a 1-node CUDA graph (kernel node params updated per call)
  {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    empty_k<<<740, 128, 0, st>>>(out);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r < 53; ++r) {
      fill<<<148 * 8, 512, 0, st>>>(buf, n, float(r));
      cudaEventRecord(a, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 3) tot += ms;
    }
    printf("after fill, 1-node graph launch (grid 740): %.2f us\n", tot / 50 * 1e3);
    tot = 0;
    for (int r = 0; r < 53; ++r) {
      fill<<<148 * 8, 512, 0, st>>>(buf, n, float(r));
      cudaEventRecord(a, st);
      empty_k<<<740, 128, 0, st>>>(out);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 3) tot += ms;
    }
    printf("after fill, plain launch on a non-blocking stream (grid 740): %.2f us\n", tot / 50 * 1e3);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
