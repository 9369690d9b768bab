// Preprocessing inverse D^{-1} on thread-block clusters (replaces the one-CTA scalar
// Gauss-Jordan for block orders 128/256 and the cuSOLVER getrf/getrs route above 256).
//
// Pivot rule and singularity test are the reference block LU's (ref
// _kernels.pyx:35-63, _kernels_py.py:19-44): at column k the pivot is the FIRST
// row i >= k maximising |a_ik| of the partially reduced matrix, and the block is
// singular when that magnitude is <= RCOND * ||D||_inf (RCOND = 1e-13, max
// absolute row sum of the original m x m block).  Gauss-Jordan eliminates below
// AND above the pivot; the candidates below the diagonal see exactly the LU's
// values, so the same blocks fail at the same column.
//
// gjc_panel_kernel<CW, CS>: one cluster of CS CTAs runs the pivoted, in-place
// Gauss-Jordan on a panel of PW = CS*CW columns x all mp rows of the augmented
// matrix W = [D | I]; CTA r keeps columns [r*CW, (r+1)*CW) in shared memory.  Per
// pivot column: the owning CTA finds the pivot and publishes the (pre-swap) column
// in its shared memory; after one cluster barrier every CTA reads it through
// distributed shared memory (DSMEM), swaps rows k <-> p, scales the pivot row and
// eliminates its own columns.  The pivot column itself is replaced by the
// Gauss-Jordan column g (g_k = 1/p, g_i = -f_i/p), so that after the panel the
// panel holds T_K, the K-columns of the accumulated row transform T
// (T Pi W_rest = X + (T_K - E) X[K], X = Pi W_rest; verified against numpy).
//   * full mode (mp <= 256): the panel IS [D | I] (PW = 2 mp), loaded from D, and
//     the right half is D^{-1} at the end -- one launch per batch of blocks;
//   * panel mode (mp > 256): W lives in a global workspace; panels of PW = 32
//     columns alternate with gjc_update_kernel, the trailing rank-32 update
//     W_rest += (T_K - E) X[K] on the fp64 tensor cores (DMMA), after the panel's
//     row swaps.
#pragma once
#include <cooperative_groups.h>

#include "btd_common.cuh"

namespace btd {

struct GjcDesc {
  const double* in;  const int64_t* idx_in;  int64_t add_in;     // D blocks (mp x mp)
  double* out;       const int64_t* idx_out; int64_t add_out;    // D^{-1} blocks
  double* W;                   // panel mode: [nbatch][mp][2 mp] workspace
  int32_t* piv;                // panel mode: [nbatch][PW] pivot rows of the current panel
  double* tol;                 // panel mode: [nbatch] singularity threshold
  int32_t* dead;               // panel mode: [nbatch] entry failed (skip the rest)
  int nbatch, m, mp;
  int c0, k0, npiv, full;      // panel columns [c0, c0+PW), pivots k0..k0+npiv-1
  int step;                    // sweep step recorded on failure
  const int32_t* active_until;
  int32_t* fail_step;
  const int64_t* fail_map;
  int32_t* fail_col;
  double rcond;
};

constexpr int GJC_NT = 256;

template <int CW, int CS>
struct GjcSmem {
  static size_t bytes(int mp) {
    // W slice | fcol | 2 broadcast columns (+3 scalars each) | rk | ok | reductions
    return sizeof(double) * ((size_t)mp * CW + mp + 2 * ((size_t)mp + 4) + 2 * CW + 2 * (GJC_NT / 32));
  }
};

template <int CW, int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(GJC_NT) gjc_panel_kernel(GjcDesc d) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int mp = d.mp, m = d.m, W2 = 2 * mp;
  double* Wl = sm;                          // [mp][CW]
  double* fcol = Wl + (size_t)mp * CW;      // [mp]  swapped multipliers of this step
  double* bc = fcol + mp;                   // [2][mp + 4]: column, p, pv, fail
  double* rk = bc + 2 * (mp + 4);           // [CW]
  double* okr = rk + CW;                    // [CW]
  double* redv = okr + CW;                  // [NT/32]
  int* redi = reinterpret_cast<int*>(redv + GJC_NT / 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  if (b >= d.nbatch) return;  // whole clusters only (grid = nbatch * CS)
  const bool full = d.full != 0;
  if (!full && d.dead[b]) return;  // uniform over the cluster
  const int colbase = d.c0 + rank * CW;  // first global W column of this CTA
  const double* A = full ? d.in + ((d.idx_in ? d.idx_in[b] : (int64_t)b) + d.add_in) * (int64_t)mp * mp : nullptr;
  double* Wg = full ? nullptr : d.W + (int64_t)b * mp * W2;

  // ---- load the slice; full mode also computes the singularity threshold
  double rs_part = 0.0;  // unused in panel mode
  for (int e = tid; e < mp * CW; e += GJC_NT) {
    const int r = e / CW, c = e - r * CW, gc = colbase + c;
    double v;
    if (full) v = gc < mp ? A[(int64_t)r * mp + gc] : (gc - mp == r ? 1.0 : 0.0);
    else v = Wg[(int64_t)r * W2 + gc];
    Wl[e] = v;
  }
  double tol;
  if (full) {
    // row abs sums of the leading m x m block: each CTA sums its columns, the
    // partials meet through DSMEM
    __syncthreads();
    for (int r = tid; r < mp; r += GJC_NT) {
      double s = 0.0;
      for (int c = 0; c < CW; ++c)
        if (r < m && colbase + c < m) s += fabs(Wl[(size_t)r * CW + c]);
      fcol[r] = s;
    }
    cluster.sync();
    double mx = 0.0;
    for (int r = tid; r < m; r += GJC_NT) {
      double s = 0.0;
      for (int q = 0; q < CS; ++q) s += cluster.map_shared_rank(fcol, q)[r];
      mx = fmax(mx, s);
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) redv[warp] = mx;
    __syncthreads();
    mx = 0.0;
    for (int w = 0; w < GJC_NT / 32; ++w) mx = fmax(mx, redv[w]);
    tol = d.rcond * mx;
    cluster.sync();  // fcol is reused below
  } else {
    tol = d.tol[b];
    __syncthreads();
  }
  (void)rs_part;

  int fail = -1;
  for (int kk = 0; kk < d.npiv; ++kk) {
    const int k = d.k0 + kk;
    const int lk = k - d.c0;           // panel-local pivot column
    const int owner = lk / CW;
    double* myb = bc + (kk & 1) * (mp + 4);
    if (rank == owner) {
      const int lc = lk - owner * CW;
      double bv = -1.0;
      int bi = mp;
      for (int i = k + tid; i < mp; i += GJC_NT) {
        const double v = fabs(Wl[(size_t)i * CW + lc]);
        if (v > bv) { bv = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
      for (int i = tid; i < mp; i += GJC_NT) myb[i] = Wl[(size_t)i * CW + lc];
      __syncthreads();
      if (tid == 0) {
        double v = redv[0];
        int i = redi[0];
        for (int w = 1; w < GJC_NT / 32; ++w)
          if (redv[w] > v || (redv[w] == v && redi[w] < i)) { v = redv[w]; i = redi[w]; }
        myb[mp] = (double)i;
        myb[mp + 1] = Wl[(size_t)i * CW + lc];
        myb[mp + 2] = (k < m && v <= tol) ? 1.0 : 0.0;
      }
    }
    cluster.sync();
    const double* ob = cluster.map_shared_rank(myb, owner);
    const int p = (int)ob[mp];
    const double pv = ob[mp + 1];
    if (ob[mp + 2] != 0.0) { fail = k; break; }
    // swapped multipliers f (row p gets old row k's value, row k the pivot's)
    for (int i = tid; i < mp; i += GJC_NT) fcol[i] = ob[i];
    __syncthreads();
    if (tid == 0 && p != k) {
      const double t = fcol[k];
      fcol[k] = fcol[p];
      fcol[p] = t;
    }
    const double inv = 1.0 / pv;
    for (int c = tid; c < CW; c += GJC_NT) {
      okr[c] = Wl[(size_t)k * CW + c];
      rk[c] = Wl[(size_t)p * CW + c] * inv;
    }
    __syncthreads();
    for (int e = tid; e < mp * CW; e += GJC_NT) {
      const int i = e / CW, c = e - i * CW;
      if (i == k) { Wl[e] = rk[c]; continue; }
      const double src = i == p ? okr[c] : Wl[e];
      Wl[e] = fma(-fcol[i], rk[c], src);
    }
    __syncthreads();
    if (rank == owner) {  // in-place Gauss-Jordan column g
      const int lc = lk - owner * CW;
      for (int i = tid; i < mp; i += GJC_NT) Wl[(size_t)i * CW + lc] = i == k ? inv : -fcol[i] * inv;
      if (!full && tid == 0) d.piv[(int64_t)b * (CS * CW) + kk] = p;
    }
    __syncthreads();
  }

  if (fail >= 0) {
    if (rank == 0 && tid == 0) {
      const bool checked = !d.active_until || d.step < d.active_until[b];
      if (checked) {
        const int64_t slot = d.fail_map ? d.fail_map[b] : b;
        if (d.fail_step[slot] < 0) {
          d.fail_step[slot] = d.step;
          d.fail_col[slot] = fail;
        }
      }
      if (!full) d.dead[b] = 1;
    }
  }
  if (full) {
    double* O = d.out + ((d.idx_out ? d.idx_out[b] : (int64_t)b) + d.add_out) * (int64_t)mp * mp;
    for (int e = tid; e < mp * CW; e += GJC_NT) {
      const int r = e / CW, c = e - r * CW, gc = colbase + c;
      if (gc >= mp) O[(int64_t)r * mp + gc - mp] = fail >= 0 ? 0.0 : Wl[e];
    }
  } else if (fail < 0) {
    for (int e = tid; e < mp * CW; e += GJC_NT) {
      const int r = e / CW, c = e - r * CW;
      Wg[(int64_t)r * W2 + colbase + c] = Wl[e];
    }
  }
  cluster.sync();  // no CTA leaves while others may still read its shared memory
}

// W = [D | I] per batch entry (panel mode) + singularity threshold; clears `dead`.
__global__ void gjc_init_kernel(GjcDesc d) {
  __shared__ double red[32];
  const int mp = d.mp, W2 = 2 * mp;
  for (int b = blockIdx.x; b < d.nbatch; b += gridDim.x) {
    const double* A = d.in + ((d.idx_in ? d.idx_in[b] : (int64_t)b) + d.add_in) * (int64_t)mp * mp;
    double* Wg = d.W + (int64_t)b * mp * W2;
    double mx = 0.0;
    for (int r = threadIdx.x >> 5; r < mp; r += blockDim.x >> 5) {
      double s = 0.0;
      for (int c = threadIdx.x & 31; c < W2; c += 32) {
        const double v = c < mp ? A[(int64_t)r * mp + c] : (c - mp == r ? 1.0 : 0.0);
        Wg[(int64_t)r * W2 + c] = v;
        if (r < d.m && c < d.m) s += fabs(v);
      }
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      mx = fmax(mx, s);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
      d.tol[b] = d.rcond * v;
      d.dead[b] = 0;
    }
    __syncthreads();
  }
}

// D^{-1} = right half of W (zeros for failed entries).
__global__ void gjc_extract_kernel(GjcDesc d) {
  const int mp = d.mp, W2 = 2 * mp;
  const int64_t per = (int64_t)mp * mp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)d.nbatch * per;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / per);
    const int64_t rc = e - (int64_t)b * per;
    const int r = (int)(rc / mp), c = (int)(rc - (int64_t)r * mp);
    double* O = d.out + ((d.idx_out ? d.idx_out[b] : (int64_t)b) + d.add_out) * per;
    O[rc] = d.dead[b] ? 0.0 : d.W[(int64_t)b * mp * W2 + (int64_t)r * W2 + mp + c];
  }
}

// Trailing update after a panel (panel mode): for the columns [c0 + PW, 2 mp)
//   X = Pi W_rest (the panel's row swaps, in order),  W_rest <- X + (T_K - E) X[K]
// T_K = panel columns c0 .. c0+npiv-1 (written back by the panel kernel), E the unit
// columns at the pivot rows K = k0 .. k0+npiv-1.  One CTA per (entry, 32-column
// tile); the rank-npiv product runs on DMMA (m8n8k4): 8 warps, each a 16 x 16 tile
// of a 64-row block.  mp <= GJC_MAXMP.
constexpr int GJC_MAXMP = 4096;
template <int PW>
__global__ void __launch_bounds__(256) gjc_update_kernel(GjcDesc d, int ntiles) {
  constexpr int TN = 32, TMB = 64, LDX = TN + 2;
  __shared__ double Xk[PW][LDX];       // X[K] of this tile
  __shared__ double Xi[2 * PW][TN];    // source rows of the swapped positions
  __shared__ int pos[2 * PW], src[2 * PW];
  __shared__ int16_t rowmap[GJC_MAXMP];  // position -> index into Xi (-1: not swapped)
  __shared__ int npos;
  const int b = blockIdx.x / ntiles, tile = blockIdx.x - b * ntiles;
  if (b >= d.nbatch || d.dead[b]) return;
  const int mp = d.mp, W2 = 2 * mp, npiv = d.npiv, k0 = d.k0;
  const int cbeg = d.c0 + PW + tile * TN;
  if (cbeg >= W2) return;
  const int ncols = min(TN, W2 - cbeg);
  double* Wg = d.W + (int64_t)b * mp * W2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int r = tid; r < mp; r += 256) rowmap[r] = -1;
  if (tid == 0) {  // net source row of every position the swaps touch
    int n = 0;
    for (int kk = 0; kk < npiv; ++kk) {
      const int a = k0 + kk, p = d.piv[(int64_t)b * PW + kk];
      if (a == p) continue;
      int ia = -1, ip = -1;
      for (int j = 0; j < n; ++j) {
        if (pos[j] == a) ia = j;
        if (pos[j] == p) ip = j;
      }
      if (ia < 0) { pos[n] = a; src[n] = a; ia = n++; }
      if (ip < 0) { pos[n] = p; src[n] = p; ip = n++; }
      const int t = src[ia];
      src[ia] = src[ip];
      src[ip] = t;
    }
    npos = n;
  }
  __syncthreads();
  const int n = npos;
  for (int j = tid; j < n; j += 256) rowmap[pos[j]] = (int16_t)j;
  for (int e = tid; e < n * TN; e += 256) {
    const int j = e / TN, c = e - j * TN;
    Xi[j][c] = c < ncols ? Wg[(int64_t)src[j] * W2 + cbeg + c] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < PW * TN; e += 256) {
    const int kk = e / TN, c = e - kk * TN;
    double v = 0.0;
    if (kk < npiv && c < ncols) {
      const int r = k0 + kk, j = rowmap[r];
      v = j >= 0 ? Xi[j][c] : Wg[(int64_t)r * W2 + cbeg + c];
    }
    Xk[kk][c] = v;
  }
  __syncthreads();
  const int g = lane >> 2, t = lane & 3;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 16;
  for (int r0 = 0; r0 < mp; r0 += TMB) {
    double acc[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < PW; k4 += 4) {
      double a[2], bb[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = r0 + wr + i * 8 + g, kk = k4 + t;
        double v = 0.0;
        if (r < mp && kk < npiv) v = Wg[(int64_t)r * W2 + d.c0 + kk] - (r == k0 + kk ? 1.0 : 0.0);
        a[i] = v;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) bb[j] = Xk[k4 + t][wc + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
    // out = X + acc; X = Xi for swapped positions, else the row itself
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = r0 + wr + i * 8 + g;
      if (r >= mp) continue;
      const int jx = rowmap[r];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = wc + j * 8 + 2 * t + h;
          if (c >= ncols) continue;
          double* dst = Wg + (int64_t)r * W2 + cbeg + c;
          const double x = jx >= 0 ? Xi[jx][c] : *dst;
          *dst = x + acc[i][j][h];
        }
    }
  }
}

}  // namespace btd
