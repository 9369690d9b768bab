// Microbenchmark: do DMMA (tensor pipe) and DFMA (FP64 pipe) run concurrently on B200?
// Warps [0, nd) of each CTA issue DMMA m8n8k4, warps [nd, nd+nf) issue DFMA; the
// combined rate against either alone says whether a sweep could split its products
// between the two pipes.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix(double* out, int iters_d, int iters_f, int nd) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp < nd) {
    double acc[8][2];
    for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
    for (int it = 0; it < iters_d; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  } else {
    double acc[16];
    for (int i = 0; i < 16; ++i) acc[i] = i;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
    for (int it = 0; it < iters_f; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    for (int i = 0; i < 16; ++i) s += acc[i];
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case { int nd, nf, id, jf; };
  // iterations chosen so each side alone runs ~ the same time at its peak
  const Case cases[] = {{8, 0, 20000, 0}, {0, 8, 0, 40000}, {8, 8, 20000, 40000}, {4, 4, 20000, 40000},
                        {8, 4, 20000, 40000}, {4, 8, 20000, 40000}, {16, 0, 20000, 0}, {0, 16, 0, 40000}};
  for (const Case& c : cases) {
    const int grid = sms, block = 32 * (c.nd + c.nf);
    mix<<<grid, block>>>(out, 10, 10, c.nd);
    cudaEventRecord(e0);
    mix<<<grid, block>>>(out, c.id, c.jf, c.nd);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fd = 2.0 * 256 * 8 * (double)c.id * grid * c.nd;          // DMMA flops
    const double ff = 2.0 * 32 * 16 * (double)c.jf * grid * c.nf;          // DFMA flops
    printf("dmma warps %2d  dfma warps %2d : %7.3f ms  dmma %.2f + dfma %.2f = %.2f TFLOP/s\n", c.nd, c.nf, ms,
           fd / ms / 1e9, ff / ms / 1e9, (fd + ff) / ms / 1e9);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
