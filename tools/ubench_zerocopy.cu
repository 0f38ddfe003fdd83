// Zero-copy output over PCIe (dev tool): SM stores of a 40 MB result straight
// into pinned host memory, alone and concurrent with a 40 MB H2D DMA copy,
// against the copy-engine D2H.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_zerocopy tools/ubench_zerocopy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void store_rows(float4* __restrict__ dst, const float4* __restrict__ src, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t bytes = 19717ull * 512 * 4;
  const size_t n4 = bytes / 16;
  float *hx, *hy, *dx, *dy;
  cudaHostAlloc(&hx, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&hy, bytes, cudaHostAllocDefault);
  cudaMalloc(&dx, bytes);
  cudaMalloc(&dy, bytes);
  cudaMemset(dy, 0, bytes);
  cudaPointerAttributes at;
  cudaPointerGetAttributes(&at, hy);
  printf("pinned host: type %d devicePointer %p hostPointer %p (same=%d)\n", int(at.type), at.devicePointer, at.hostPointer, at.devicePointer == (void*)hy);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float ms;
  for (int grid : {148, 296, 592, 1184}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, s1);
      store_rows<<<grid, 256, 0, s1>>>((float4*)at.devicePointer, (const float4*)dy, n4);
      cudaEventRecord(b, s1);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("zero-copy store alone grid %4d: %8.1f us  %.1f GB/s\n", grid, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1);
    cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("D2H copy engine alone:          %8.1f us  %.1f GB/s\n", ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  // concurrent: H2D on s2 + zero-copy stores on s1
  for (int rep = 0; rep < 3; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(a, 0);
    cudaStreamWaitEvent(s1, a, 0); cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s2);
    store_rows<<<592, 256, 0, s1>>>((float4*)at.devicePointer, (const float4*)dy, n4);
    cudaEvent_t e1, e2; cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e1, s1); cudaEventRecord(e2, s2);
    cudaStreamWaitEvent(0, e1, 0); cudaStreamWaitEvent(0, e2, 0);
    cudaEventRecord(b, 0);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("H2D DMA + zero-copy stores:     %8.1f us  %.1f GB/s per direction\n", ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  for (int rep = 0; rep < 3; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(a, 0);
    cudaStreamWaitEvent(s1, a, 0); cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s2);
    cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, s1);
    cudaEvent_t e1, e2; cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e1, s1); cudaEventRecord(e2, s2);
    cudaStreamWaitEvent(0, e1, 0); cudaStreamWaitEvent(0, e2, 0);
    cudaEventRecord(b, 0);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("H2D DMA + D2H DMA:              %8.1f us  %.1f GB/s per direction\n", ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
