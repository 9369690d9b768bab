// Copy-engine probe: contiguous vs 2-D strided pinned-host copies, and H2D || D2H overlap.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t rows = 1 << 20, K = 256, total = rows * K * 8;  // c1: 1M rows x 256 cols (2 GiB)
  double *h, *h2, *d;
  cudaMallocHost(&h, total); cudaMallocHost(&h2, total); cudaMalloc(&d, total);
  cudaStream_t a, b; cudaStreamCreate(&a); cudaStreamCreate(&b);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  cudaMemcpy(d, h, total, cudaMemcpyHostToDevice);
  cudaEventRecord(e0, a); cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, a); cudaEventRecord(e1, a);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("H2D contiguous: %.1f GB/s\n", total / ms / 1e6);
  cudaEventRecord(e0, a); cudaMemcpyAsync(h, d, total, cudaMemcpyDeviceToHost, a); cudaEventRecord(e1, a);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("D2H contiguous: %.1f GB/s\n", total / ms / 1e6);
  for (size_t kc : {16, 32, 64, 128}) {
    cudaEventRecord(e0, a);
    for (size_t c = 0; c < K; c += kc)
      cudaMemcpy2DAsync(d + c * rows, kc * 8, h + c, K * 8, kc * 8, rows, cudaMemcpyHostToDevice, a);
    cudaEventRecord(e1, a); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("H2D 2-D rows of %4zu B: %.1f GB/s\n", kc * 8, total / ms / 1e6);
    cudaEventRecord(e0, a);
    for (size_t c = 0; c < K; c += kc)
      cudaMemcpy2DAsync(h + c, K * 8, d + c * rows, kc * 8, kc * 8, rows, cudaMemcpyDeviceToHost, a);
    cudaEventRecord(e1, a); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("D2H 2-D rows of %4zu B: %.1f GB/s\n", kc * 8, total / ms / 1e6);
  }
  // full duplex: H2D on a, D2H on b (different buffers)
  cudaDeviceSynchronize();
  cudaEventRecord(e0, 0);
  cudaMemcpyAsync(d, h, total / 2, cudaMemcpyHostToDevice, a);
  cudaMemcpyAsync(h2, (char*)d + total / 2, total / 2, cudaMemcpyDeviceToHost, b);
  cudaDeviceSynchronize(); cudaEventRecord(e1, 0); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("H2D || D2H contiguous (1 GiB each): %.1f GB/s aggregate\n", total / ms / 1e6);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
