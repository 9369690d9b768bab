// Batched Gauss-Jordan inversion with partial pivoting (preprocessing only).
//
// Pivot rule and singularity test follow the reference block LU
// (ref _kernels.pyx:35-63, _kernels_py.py:19-44): at column k the pivot is
// the first row i >= k maximising |a_ik| of the partially reduced matrix; the
// block is singular when that magnitude is <= RCOND * ||D||_inf with
// RCOND = 1e-13 and ||.||_inf the max absolute row sum of the ORIGINAL
// m x m block.  Gauss-Jordan visits exactly the same candidate values as the
// LU's elimination of the rows below the diagonal, so the same blocks fail.
// The solve phase then applies D^{-1} as a GEMM instead of LU triangular
// solves (hard part 4: 5 orders of headroom to the 1e-9 bar).
//
// One CTA per block; the augmented [D | I] (mp x 2mp) lives in shared memory
// when it fits (mp <= 64), else in a global workspace (L2-resident).  Only the
// leading m x m block is tested; padding rows/cols carry an identity.
#pragma once
#include "btd_common.cuh"

namespace btd {

struct InvDesc {
  const double* in;  const int64_t* idx_in;  int64_t add_in;
  double* out;       const int64_t* idx_out; int64_t add_out;
  double* ws;                       // global workspace [nbatch][mp][2mp] (when not smem)
  int nbatch, m, mp;
  int step;                         // sweep step recorded on failure
  const int32_t* active_until;      // entry b is checked only if step < active_until[b] (nullable)
  int32_t* fail_step;               // per slot: first failing step (-1 = none)
  const int64_t* fail_map;          // batch entry -> failure slot (nullable: identity)
  int32_t* fail_col;                // per entry: failing column of that step
  double rcond;
};

__global__ void __launch_bounds__(512) gj_inverse_kernel(InvDesc d, int use_smem) {
  extern __shared__ __align__(16) double smem_w[];
  __shared__ double red_v[16];
  __shared__ int red_i[16];
  __shared__ double s_piv;
  __shared__ int s_prow, s_fail;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int mp = d.mp, m = d.m, W2 = 2 * mp;
  for (int b = blockIdx.x; b < d.nbatch; b += gridDim.x) {
    const double* A = d.in + (d.idx_in ? d.idx_in[b] : (int64_t)b) * (int64_t)mp * mp + d.add_in * (int64_t)mp * mp;
    double* O = d.out + ((d.idx_out ? d.idx_out[b] : (int64_t)b) + d.add_out) * (int64_t)mp * mp;
    double* W = use_smem ? smem_w : d.ws + (int64_t)blockIdx.x * mp * W2;
    // init [D | I]; row abs sums of the leading m x m block
    double rs_max = 0.0;
    for (int r = warp; r < mp; r += nt / 32) {
      double s = 0.0;
      for (int c = lane; c < W2; c += 32) {
        double v = c < mp ? A[(int64_t)r * mp + c] : (c - mp == r ? 1.0 : 0.0);
        W[(int64_t)r * W2 + c] = v;
        if (r < m && c < m) s += fabs(v);
      }
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      rs_max = fmax(rs_max, s);
    }
    if (lane == 0) red_v[warp] = rs_max;
    __syncthreads();
    if (tid == 0) {
      double mx = 0.0;
      for (int w = 0; w < nt / 32; ++w) mx = fmax(mx, red_v[w]);
      s_piv = d.rcond * mx;  // tolerance
      s_fail = -1;
    }
    __syncthreads();
    const double tol = s_piv;
    const bool checked = !d.active_until || d.step < d.active_until[b];
    for (int k = 0; k < mp; ++k) {
      // pivot search: first max |W[i][k]|, i >= k
      double bv = -1.0;
      int bi = mp;
      for (int i = k + tid; i < mp; i += nt) {
        double v = fabs(W[(int64_t)i * W2 + k]);
        if (v > bv) { bv = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
      __syncthreads();
      if (tid == 0) {
        double v = red_v[0];
        int i = red_i[0];
        for (int w = 1; w < nt / 32; ++w)
          if (red_v[w] > v || (red_v[w] == v && red_i[w] < i)) { v = red_v[w]; i = red_i[w]; }
        s_prow = i;
        s_piv = W[(int64_t)i * W2 + k];
        if (k < m && v <= tol && s_fail < 0) s_fail = k;
      }
      __syncthreads();
      if (s_fail >= 0) break;
      const int p = s_prow;
      const double piv = s_piv;
      // swap rows k <-> p and normalise the pivot row
      for (int c = tid; c < W2; c += nt) {
        double vk = W[(int64_t)k * W2 + c], vp = W[(int64_t)p * W2 + c];
        if (p != k) W[(int64_t)p * W2 + c] = vk;
        W[(int64_t)k * W2 + c] = (p != k ? vp : vk) / piv;
      }
      __syncthreads();
      // eliminate column k from every other row (columns >= k only)
      const int ncols = W2 - k;
      for (int e = tid; e < mp * ncols; e += nt) {
        const int i = e / ncols, c = k + e % ncols;
        if (i == k) continue;
        const double f = W[(int64_t)i * W2 + k];
        if (c == k) continue;  // written last (below) so other threads still read f
        W[(int64_t)i * W2 + c] -= f * W[(int64_t)k * W2 + c];
      }
      __syncthreads();
      for (int i = tid; i < mp; i += nt)
        if (i != k) W[(int64_t)i * W2 + k] = 0.0;
      __syncthreads();
    }
    if (tid == 0 && checked && s_fail >= 0) {
      const int64_t slot = d.fail_map ? d.fail_map[b] : b;
      if (d.fail_step[slot] < 0) {
        d.fail_step[slot] = d.step;
        d.fail_col[slot] = s_fail;
      }
    }
    // D^{-1} = right half
    for (int e = tid; e < mp * mp; e += nt) {
      const int r = e / mp, c = e % mp;
      O[(int64_t)r * mp + c] = s_fail >= 0 ? 0.0 : W[(int64_t)r * W2 + mp + c];
    }
    __syncthreads();
  }
}

}  // namespace btd
