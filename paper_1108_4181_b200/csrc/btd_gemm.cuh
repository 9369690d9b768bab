// Indexed batched multi-term FP64 GEMM on DMMA tensor cores.
//
//   C_b = beta * Cin_b + sum_t alpha_t * A_{b,t} @ B_{b,t}     (b = 0..nbatch-1)
//
// Every operand of batch entry b lives at  base + (idx[b] + add) * stride
// (idx == nullptr means idx[b] = b), with a row stride `ld` (or a per-entry
// ld_arr[b]).  This one kernel carries every small product of Algorithm 2
// that is not on a sweep chain: the preprocessing products (ref
// _kernels.pyx:133-170 thomas_factor, dichotomy.py:172-236), the interface
// RHS assembly (dichotomy.py:239-276), the tree series sums and corrections of
// Algorithm 1 (dichotomy.py:279-295), and -- for block orders above 256 --
// the per-step sweep products themselves (mode 1, one launch per step).
//
// Tiling: CTA tile BM x BN, 4 warps in a 2x2 grid, BK = 16 k-slab staged in
// shared memory through registers (double-buffered).  A is stored [BM][24]
// (16B loads of (k,k+1) pairs, conflict-free for LDS.128), B is [16][BN+2]
// (LDS.64, conflict-free).
#pragma once
#include "btd_common.cuh"

namespace btd {

struct Opnd {
  const double* base;
  const int64_t* idx;     // per-entry index (nullable -> entry number)
  int64_t add;            // added to every index
  int64_t stride;         // elements per index unit
  int64_t ld;             // row stride
  const int64_t* ld_arr;  // per-entry row stride (nullable)
};

struct Term {
  Opnd A, B;
  int64_t k;              // reduction length
  const int64_t* k_arr;   // per-entry reduction length (nullable)
  double alpha;
};

struct GemmDesc {
  int64_t rows, cols;
  int nbatch;
  Opnd C;
  Opnd Cin;               // Cin.base == nullptr -> no addend
  double beta;
  int nterms;
  Term t[3];
};

BTD_DEVINL const double* opnd_ptr(const Opnd& o, int b) {
  const int64_t i = (o.idx ? o.idx[b] : (int64_t)b) + o.add;
  return o.base + i * o.stride;
}
BTD_DEVINL int64_t opnd_ld(const Opnd& o, int b) { return o.ld_arr ? o.ld_arr[b] : o.ld; }

template <int BM, int BN>
__global__ void __launch_bounds__(128) gemm_batched_kernel(GemmDesc d) {
  constexpr int BK = 16;
  constexpr int LDA = 24;          // doubles; 12 double2 == 4 (mod 8)
  constexpr int LDB = BN + 2;      // doubles; == 2 (mod 16)
  constexpr int WM = BM / 2, WN = BN / 2;
  constexpr int TM = WM / 8, TN = WN / 8;
  constexpr int AE = BM * BK / 128;  // A elements per thread per slab
  constexpr int BE = BK * BN / 128;  // B elements per thread per slab
  __shared__ __align__(16) double As[BM * LDA];
  __shared__ __align__(16) double Bs[BK * LDB];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;

  for (int b = blockIdx.z; b < d.nbatch; b += gridDim.z) {
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int ti = 0; ti < d.nterms; ++ti) {
      const Term& tm_ = d.t[ti];
      const double* A = opnd_ptr(tm_.A, b);
      const double* B = opnd_ptr(tm_.B, b);
      const int64_t lda = opnd_ld(tm_.A, b), ldb = opnd_ld(tm_.B, b);
      const int64_t K = tm_.k_arr ? tm_.k_arr[b] : tm_.k;
      const double alpha = tm_.alpha;
      double ra[AE], rb[BE];
      auto load_slab = [&](int64_t k0) {
#pragma unroll
        for (int i = 0; i < AE; ++i) {
          const int e = tid + i * 128;
          const int r = e / BK, kk = e % BK;
          const int64_t gr = row0 + r, gk = k0 + kk;
          ra[i] = (gr < d.rows && gk < K) ? alpha * A[gr * lda + gk] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < BE; ++i) {
          const int e = tid + i * 128;
          const int kk = e / BN, c = e % BN;
          const int64_t gk = k0 + kk, gc = col0 + c;
          rb[i] = (gk < K && gc < d.cols) ? B[gk * ldb + gc] : 0.0;
        }
      };
      auto store_slab = [&]() {
#pragma unroll
        for (int i = 0; i < AE; ++i) {
          const int e = tid + i * 128;
          As[(e / BK) * LDA + (e % BK)] = ra[i];
        }
#pragma unroll
        for (int i = 0; i < BE; ++i) {
          const int e = tid + i * 128;
          Bs[(e / BN) * LDB + (e % BN)] = rb[i];
        }
      };
      if (K <= 0) continue;
      load_slab(0);
      for (int64_t k0 = 0; k0 < K; k0 += BK) {
        __syncthreads();
        store_slab();
        __syncthreads();
        if (k0 + BK < K) load_slab(k0 + BK);
#pragma unroll
        for (int s = 0; s < BK / 8; ++s) {
          double2 a[TM];
          double b0[TN], b1[TN];
#pragma unroll
          for (int i = 0; i < TM; ++i)
            a[i] = *reinterpret_cast<const double2*>(&As[(wr * WM + i * 8 + g) * LDA + 8 * s + 2 * t]);
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            b0[j] = Bs[(8 * s + 2 * t) * LDB + wc * WN + j * 8 + g];
            b1[j] = Bs[(8 * s + 2 * t + 1) * LDB + wc * WN + j * 8 + g];
          }
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].x, b0[j]);
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].y, b1[j]);
        }
      }
      __syncthreads();
    }
    // epilogue
    double* C = const_cast<double*>(opnd_ptr(d.C, b));
    const int64_t ldc = opnd_ld(d.C, b);
    const double* Ci = d.Cin.base ? opnd_ptr(d.Cin, b) : nullptr;
    const int64_t ldci = d.Cin.base ? opnd_ld(d.Cin, b) : 0;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int64_t r = row0 + wr * WM + i * 8 + g;
          const int64_t c = col0 + wc * WN + j * 8 + 2 * t + v;
          if (r < d.rows && c < d.cols) {
            double val = acc[i][j][v];
            if (Ci) val += d.beta * Ci[r * ldci + c];
            C[r * ldc + c] = val;
          }
        }
  }
}

// Transpose a batch of square blocks: out[idx_o[b]] = in[idx_i[b]]^T.
__global__ void transpose_blocks_kernel(const double* in, const int64_t* idx_in, double* out,
                                        const int64_t* idx_out, int nb, int mp) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int b = blockIdx.z; b < nb; b += gridDim.z) {
    const double* src = in + idx_in[b] * (int64_t)mp * mp;
    double* dst = out + idx_out[b] * (int64_t)mp * mp;
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int r = by + i, c = bx + threadIdx.x;
      tile[i][threadIdx.x] = (r < mp && c < mp) ? src[(int64_t)r * mp + c] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int r = bx + i, c = by + threadIdx.x;
      if (r < mp && c < mp) dst[(int64_t)r * mp + c] = tile[threadIdx.x][i];
    }
    __syncthreads();
  }
}

}  // namespace btd
