// Dev microbenchmark: host<->device copy rates for the host-buffer entry point
// (cfg[1] shape: 19,717 x 512 f32 = 40.4 MB each way), pinned host memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

int main() {
  const size_t rows = 19717, d = 512, bytes = rows * d * 4;
  float *hx, *hy, *dx, *dy;
  cudaMallocHost(&hx, bytes);
  cudaMallocHost(&hy, bytes);
  cudaMalloc(&dx, bytes);
  cudaMalloc(&dy, bytes);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* what, auto fn) {
    for (int w = 0; w < 2; ++w) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a, 0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(b, 0);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-44s %8.1f us  %6.1f GB/s (one direction bytes)\n", what, ms / reps * 1e3,
           bytes / (ms / reps * 1e-3) / 1e9);
  };
  timeit("H2D contiguous", [&] { cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s1); });
  timeit("D2H contiguous", [&] { cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, s2); });
  timeit("H2D + D2H concurrent", [&] {
    cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, s2);
  });
  for (int chunks : {2, 4, 8}) {
    const size_t cw = d / chunks;
    char name[64];
    snprintf(name, sizeof name, "H2D 2D column chunks x%d", chunks);
    timeit(name, [&] {
      for (int k = 0; k < chunks; ++k)
        cudaMemcpy2DAsync(dx + k * cw, d * 4, hx + k * cw, d * 4, cw * 4, rows,
                          cudaMemcpyHostToDevice, s1);
    });
    snprintf(name, sizeof name, "D2H 2D column chunks x%d", chunks);
    timeit(name, [&] {
      for (int k = 0; k < chunks; ++k)
        cudaMemcpy2DAsync(hy + k * cw, d * 4, dy + k * cw, d * 4, cw * 4, rows,
                          cudaMemcpyDeviceToHost, s2);
    });
    snprintf(name, sizeof name, "H2D row chunks x%d", chunks);
    const size_t rc = (rows + chunks - 1) / chunks;
    timeit(name, [&] {
      for (int k = 0; k < chunks; ++k) {
        const size_t r0 = k * rc, n = r0 + rc > rows ? rows - r0 : rc;
        cudaMemcpyAsync(dx + r0 * d, hx + r0 * d, n * d * 4, cudaMemcpyHostToDevice, s1);
      }
    });
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
