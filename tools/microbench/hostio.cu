// Host<->device column-chunk transfers for the numpy-path pipeline, c4 layout
// (rows = 2^20 * 16, K = 64 doubles per row = 512 B): copy engines (2-D) vs
// SM-driven zero-copy kernels over mapped pinned memory, alone and duplex
// (H2D of chunk c+1 concurrent with D2H of chunk c), for chunk widths
// kc = 8 / 16 / 32 / 64 columns (64 / 128 / 256 / 512 B row segments).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hostio hostio.cu
#include <cstdio>
#include <cuda_runtime.h>

// dst(rows x kc, packed) <- src(rows x K, columns c0..c0+kc)   (gather, H2D)
// or the reverse (scatter, D2H); one 16-byte vector per thread-iteration
__global__ void gather(double2* __restrict__ dst, const double2* __restrict__ src, size_t spitch2, size_t w2,
                       size_t rows) {
  const size_t n = rows * w2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / w2, v = i - r * w2;
    dst[i] = src[r * spitch2 + v];
  }
}
__global__ void scatter(double2* __restrict__ dst, size_t dpitch2, const double2* __restrict__ src, size_t w2,
                        size_t rows) {
  const size_t n = rows * w2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / w2, v = i - r * w2;
    dst[r * dpitch2 + v] = src[i];
  }
}

int main() {
  const size_t rows = (size_t)1 << 24, K = 64, total = rows * K * 8;
  double *hf, *hx, *d0, *d1;
  if (cudaHostAlloc(&hf, total, cudaHostAllocMapped) || cudaHostAlloc(&hx, total, cudaHostAllocMapped)) {
    printf("host alloc failed\n");
    return 1;
  }
  cudaMalloc(&d0, total);
  cudaMalloc(&d1, total);
  cudaMemset(d0, 0, total);
  cudaMemset(d1, 0, total);
  for (size_t i = 0; i < rows * K; i += 512) hf[i] = 1.0;
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto t_begin = [&] { cudaDeviceSynchronize(); cudaEventRecord(e0, 0); };
  auto t_end = [&] { cudaDeviceSynchronize(); cudaEventRecord(e1, 0); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); return ms; };
  const double gb = total / 1e9;
  for (size_t kc : {8, 16, 32, 64}) {
    const size_t nch = K / kc, w = kc * 8, w2 = kc / 2, cb = rows * kc;
    // copy engines, one direction
    t_begin();
    for (size_t c = 0; c < nch; ++c)
      cudaMemcpy2DAsync(d0 + c * cb, w, hf + c * kc, K * 8, w, rows, cudaMemcpyHostToDevice, a);
    const float ce_h2d = t_end();
    t_begin();
    for (size_t c = 0; c < nch; ++c)
      cudaMemcpy2DAsync(hx + c * kc, K * 8, d0 + c * cb, w, w, rows, cudaMemcpyDeviceToHost, a);
    const float ce_d2h = t_end();
    // copy engines, duplex (H2D chunk c+1 || D2H chunk c)
    t_begin();
    for (size_t c = 0; c < nch; ++c) {
      cudaMemcpy2DAsync(d0 + c * cb, w, hf + c * kc, K * 8, w, rows, cudaMemcpyHostToDevice, a);
      cudaMemcpy2DAsync(hx + c * kc, K * 8, d1 + c * cb, w, w, rows, cudaMemcpyDeviceToHost, b);
    }
    const float ce_dup = t_end();
    printf("kc %2zu (%3zu B): CE H2D %5.1f GB/s  CE D2H %5.1f GB/s  CE duplex %5.1f GB/s aggregate\n", kc, w,
           gb / ce_h2d * 1e3, gb / ce_d2h * 1e3, 2 * gb / ce_dup * 1e3);
    for (int blocks : {148, 296, 592}) {
      t_begin();
      for (size_t c = 0; c < nch; ++c)
        gather<<<blocks, 512, 0, a>>>((double2*)(d0 + c * cb), (const double2*)(hf + c * kc), K / 2, w2, rows);
      const float zh = t_end();
      t_begin();
      for (size_t c = 0; c < nch; ++c)
        scatter<<<blocks, 512, 0, a>>>((double2*)(hx + c * kc), K / 2, (const double2*)(d0 + c * cb), w2, rows);
      const float zd = t_end();
      t_begin();
      for (size_t c = 0; c < nch; ++c) {
        gather<<<blocks, 512, 0, a>>>((double2*)(d0 + c * cb), (const double2*)(hf + c * kc), K / 2, w2, rows);
        scatter<<<blocks, 512, 0, b>>>((double2*)(hx + c * kc), K / 2, (const double2*)(d1 + c * cb), w2, rows);
      }
      const float zdup = t_end();
      // mixed: copy-engine H2D || kernel D2H
      t_begin();
      for (size_t c = 0; c < nch; ++c) {
        cudaMemcpy2DAsync(d0 + c * cb, w, hf + c * kc, K * 8, w, rows, cudaMemcpyHostToDevice, a);
        scatter<<<blocks, 512, 0, b>>>((double2*)(hx + c * kc), K / 2, (const double2*)(d1 + c * cb), w2, rows);
      }
      const float mix = t_end();
      printf("   blocks %4d: ZC H2D %5.1f  ZC D2H %5.1f  ZC duplex %5.1f agg  CE-H2D||ZC-D2H %5.1f agg GB/s\n",
             blocks, gb / zh * 1e3, gb / zd * 1e3, 2 * gb / zdup * 1e3, 2 * gb / mix * 1e3);
    }
  }
  // contiguous full-width CE reference
  t_begin();
  cudaMemcpyAsync(d0, hf, total, cudaMemcpyHostToDevice, a);
  const float c1 = t_end();
  t_begin();
  cudaMemcpyAsync(hx, d0, total, cudaMemcpyDeviceToHost, a);
  const float c2 = t_end();
  t_begin();
  cudaMemcpyAsync(d0, hf, total, cudaMemcpyHostToDevice, a);
  cudaMemcpyAsync(hx, d1, total, cudaMemcpyDeviceToHost, b);
  const float c3 = t_end();
  printf("contiguous 8.6 GB: CE H2D %.1f  CE D2H %.1f  duplex %.1f GB/s aggregate\n", gb / c1 * 1e3, gb / c2 * 1e3,
         2 * gb / c3 * 1e3);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
