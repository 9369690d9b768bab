// Zero-copy probe: SM-driven 2-D copies to/from mapped pinned host memory vs the
// copy engines, and kernel D2H concurrent with copy-engine H2D.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k2d(double2* __restrict__ dst, size_t dpitch, const double2* __restrict__ src, size_t spitch,
                    size_t wvec, size_t rows) {
  const size_t n = rows * wvec;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / wvec, v = i % wvec;
    dst[r * dpitch + v] = src[r * spitch + v];
  }
}

int main() {
  const size_t rows = 1 << 20, K = 256, total = rows * K * 8;
  double *h, *h2, *d, *d2;
  cudaHostAlloc(&h, total, cudaHostAllocMapped);
  cudaHostAlloc(&h2, total, cudaHostAllocMapped);
  cudaMalloc(&d, total); cudaMalloc(&d2, total);
  cudaMemset(d, 0, total);
  cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int blocks : {148, 296, 592, 1184}) {
    for (size_t kc : {32, 64, 128, 256}) {
      const size_t wvec = kc / 2;
      // D2H: device chunk (rows x kc, packed) -> host (rows x K, column offset 0)
      k2d<<<blocks, 512, 0, a>>>((double2*)h, K / 2, (const double2*)d, wvec, wvec, rows);
      cudaEventRecord(e0, a);
      for (size_t c = 0; c < K; c += kc)
        k2d<<<blocks, 512, 0, a>>>((double2*)(h + c), K / 2, (const double2*)(d + c * rows), wvec, wvec, rows);
      cudaEventRecord(e1, a); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      const float d2h = total / ms / 1e6;
      cudaEventRecord(e0, a);
      for (size_t c = 0; c < K; c += kc)
        k2d<<<blocks, 512, 0, a>>>((double2*)(d + c * rows), wvec, (const double2*)(h + c), K / 2, wvec, rows);
      cudaEventRecord(e1, a); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("blocks %5d rows %4zu B: kernel D2H %.1f GB/s  kernel H2D %.1f GB/s\n", blocks, kc * 8, d2h,
             total / ms / 1e6);
    }
  }
  // copy-engine H2D (2-D, 512 B rows) on a || kernel D2H (2-D, 512 B rows) on b
  for (int blocks : {148, 296}) {
    const size_t kc = 64, wvec = 32;
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    for (size_t c = 0; c < K; c += kc) {
      cudaMemcpy2DAsync(d + c * rows, kc * 8, h + c, K * 8, kc * 8, rows, cudaMemcpyHostToDevice, a);
      k2d<<<blocks, 512, 0, b>>>((double2*)(h2 + c), K / 2, (const double2*)(d2 + c * rows), wvec, wvec, rows);
    }
    cudaDeviceSynchronize(); cudaEventRecord(e1, 0); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("CE H2D || kernel D2H (blocks %d): %.1f GB/s aggregate (%.2f ms for 2 x %.2f GB)\n", blocks,
           2 * total / ms / 1e6, ms, total / 1e9);
  }
  {  // CE H2D || CE D2H, 2-D 512 B rows
    const size_t kc = 64;
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    for (size_t c = 0; c < K; c += kc) {
      cudaMemcpy2DAsync(d + c * rows, kc * 8, h + c, K * 8, kc * 8, rows, cudaMemcpyHostToDevice, a);
      cudaMemcpy2DAsync(h2 + c, K * 8, d2 + c * rows, kc * 8, kc * 8, rows, cudaMemcpyDeviceToHost, b);
    }
    cudaDeviceSynchronize(); cudaEventRecord(e1, 0); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("CE H2D || CE D2H 2-D 512 B: %.1f GB/s aggregate\n", 2 * total / ms / 1e6);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
