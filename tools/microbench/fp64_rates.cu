// Microbenchmark: FP64 issue rates on B200 (DMMA m8n8k4 / m16n8k4 vs DFMA) and
// L2 read bandwidth. Used once to choose the sweep kernels' FP64 path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma16_loop(double* out, int iters) {
  double acc[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = blockIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void l2_read(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i); s += v.x + v.y;
    }
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock_kHz=%d\n", sms, clk);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int grid = sms * bps, block = 32 * warps;
      dmma_loop<<<grid, block>>>(out, 100);
      cudaEventRecord(e0); dmma_loop<<<grid, block>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * grid * warps;
      printf("DMMA m8n8k4  warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", warps, bps, flops / ms / 1e9);
      dmma16_loop<<<grid, block>>>(out, 100);
      cudaEventRecord(e0); dmma16_loop<<<grid, block>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 512 * 4 * (double)iters * grid * warps;
      printf("DMMA m16n8k4 warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", warps, bps, flops / ms / 1e9);
      dfma_loop<<<grid, block>>>(out, 100);
      cudaEventRecord(e0); dfma_loop<<<grid, block>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * (double)iters * grid * block;
      printf("DFMA         warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", warps, bps, flops / ms / 1e9);
    }
  }
  // L2-resident read bandwidth: 32 MB buffer read repeatedly
  for (size_t mb : {32, 64, 96, 4096}) {
    size_t n = mb * (1 << 20) / 16; double2* p; cudaMalloc(&p, n * 16); cudaMemset(p, 0, n * 16);
    int reps = mb >= 1024 ? 2 : 20;
    l2_read<<<sms * 4, 512>>>(p, n, 1, out);
    cudaEventRecord(e0); l2_read<<<sms * 4, 512>>>(p, n, reps, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("read %4zu MB x%d: %.1f GB/s\n", mb, reps, (double)n * 16 * reps / ms / 1e6);
    cudaFree(p);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
