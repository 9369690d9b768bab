// DMMA.8x8x4 issue behaviour on B200: clocks per DMMA for one warp per SM sub-partition as a
// function of the number of independent accumulators (ILP), and for W warps per sub-partition.
// ILP = 1 is the dependent-issue latency; the pipe's rate is 16 clk per DMMA per sub-partition.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_latency dmma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k(double* out, long long* clk, int iters) {
  double c0[ILP], c1[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) c0[i] = c1[i] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < ILP; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0[i]), "+d"(c1[i])
                     : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int ILP>
void run(int warps, double* out, long long* clk) {
  const int iters = 2000;
  k<ILP><<<148, 32 * warps>>>(out, clk, iters);
  cudaDeviceSynchronize();
  k<ILP><<<148, 32 * warps>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  const double per_warp = (double)h / (iters * 8.0 * ILP);
  const double per_smsp = per_warp / ((warps + 3) / 4);
  printf("warps/SM=%2d (%d per sub-partition) ILP=%d: %.1f clk per DMMA per warp, %.1f clk per DMMA per sub-partition\n",
         warps, (warps + 3) / 4, ILP, per_warp, per_smsp);
}

int main() {
  double* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&clk, 8);
  for (int w : {4, 8, 16}) {
    run<1>(w, out, clk);
    run<2>(w, out, clk);
    run<3>(w, out, clk);
    run<4>(w, out, clk);
    run<8>(w, out, clk);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
