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
//   * full mode (mp = 128 / 256): the panel IS D (PW = mp), in-place Gauss-Jordan;
//     the slice then holds D^{-1} up to the column permutation of the row swaps,
//     undone by the store -- one launch per batch of blocks;
//   * panel mode (other orders > 64): W = D in a global workspace (in place, padded
//     to mp + 32 columns); panels of PW = 32 columns alternate with
//     gjc_update_kernel, the rank-32 update of every other column
//     W_rest += (T_K - E) X[K] on the fp64 tensor cores (DMMA) after the panel's row
//     swaps; gjc_extract_kernel undoes the column permutation.
#pragma once
#include <cooperative_groups.h>

#include "btd_common.cuh"

namespace btd {

struct GjcDesc {
  const double* in;  const int64_t* idx_in;  int64_t add_in;     // D blocks (mp x mp)
  double* out;       const int64_t* idx_out; int64_t add_out;    // D^{-1} blocks
  double* W;                   // panel mode: [nbatch][mp][mp + 32] workspace (D, inverted in place)
  int32_t* piv;                // panel mode: [nbatch][mp] pivot row of every column
  int32_t* colmap;             // panel mode: [nbatch][mp] output column of every W column
  unsigned long long* rsmax;   // panel mode: [nbatch] max row abs sum (bits of a nonnegative double)
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

template <int CW, int CS, int NT = GJC_NT>
struct GjcSmem {
  static constexpr int LDS = CW + 1;  // odd row stride: column reads are bank-conflict free
  static size_t bytes(int mp) {
    // W slice | fcol | 2 broadcast columns (+3 scalars each) | rk | ok | reduction | pivots + column map
    return sizeof(double) * ((size_t)mp * LDS + mp + 2 * ((size_t)mp + 4) + 2 * CW + 2 * (NT / 32)) +
           sizeof(int) * 2 * (size_t)mp;
  }
};

// Full mode: in-place Gauss-Jordan on D itself (PW = mp columns): after the last
// pivot the slice holds D^{-1} with its columns permuted by the row swaps, which
// the store undoes (the swaps, in reverse order, applied to the columns).
// Panel mode: the pivot columns end up as T_K (see the file comment).
// Per pivot the owning CTA PUSHES the pivot column and (p, pivot, fail) into every
// CTA's shared memory (DSMEM stores), so after the cluster barrier all reads are local.
template <int CW, int CS, int NT = GJC_NT>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(NT) gjc_panel_kernel(GjcDesc d) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int LDS = GjcSmem<CW, CS, NT>::LDS;
  extern __shared__ __align__(16) double sm[];
  const int mp = d.mp, m = d.m, LDW = mp + 32;
  double* Wl = sm;                          // [mp][LDS]
  double* fcol = Wl + (size_t)mp * LDS;     // [mp]  swapped multipliers of this step
  double* bc = fcol + mp;                   // [2][mp + 4]: column, p, pv, fail (written by the owner)
  double* rk = bc + 2 * (mp + 4);           // [CW]  new pivot row
  double* okr = rk + CW;                    // [CW]  old row k (moves to row p)
  double* redv = okr + CW;                  // [NT/32] cross-warp pivot search
  int* redi = reinterpret_cast<int*>(redv + NT / 32);
  int* piv_s = redi + 2 * (NT / 32);    // [mp] pivot row of every step (full mode)
  int* dest = piv_s + mp;                   // [mp]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  if (b >= d.nbatch) return;  // whole clusters only (grid = nbatch * CS)
  const bool full = d.full != 0;
  if (!full && d.dead[b]) return;  // uniform over the cluster
  const int colbase = d.c0 + rank * CW;  // first global W column of this CTA
  const double* A = full ? d.in + ((d.idx_in ? d.idx_in[b] : (int64_t)b) + d.add_in) * (int64_t)mp * mp : nullptr;
  double* Wg = full ? nullptr : d.W + (int64_t)b * mp * LDW;

  for (int e = tid; e < mp * CW; e += NT) {
    const int r = e / CW, c = e - r * CW, gc = colbase + c;
    Wl[r * LDS + c] = full ? A[(int64_t)r * mp + gc] : Wg[(int64_t)r * LDW + gc];
  }
  double tol;
  if (full) {
    // singularity threshold: max row abs sum of the leading m x m block; each CTA
    // sums its columns, the partials meet through DSMEM
    __syncthreads();
    for (int r = tid; r < mp; r += NT) {
      double sacc = 0.0;
      for (int c = 0; c < CW; ++c)
        if (r < m && colbase + c < m) sacc += fabs(Wl[r * LDS + c]);
      fcol[r] = sacc;
    }
    cluster.sync();
    double mx = 0.0;
    for (int r = tid; r < m; r += NT) {
      double sacc = 0.0;
      for (int q = 0; q < CS; ++q) sacc += cluster.map_shared_rank(fcol, q)[r];
      mx = fmax(mx, sacc);
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) redv[warp] = mx;
    __syncthreads();
    mx = 0.0;
    for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, redv[w]);
    tol = d.rcond * mx;
    cluster.sync();  // fcol / redv are reused below
  } else {
    tol = d.rcond * __longlong_as_double((long long)d.rsmax[b]);
    __syncthreads();
  }

  int fail = -1;
  for (int kk = 0; kk < d.npiv; ++kk) {
    const int k = d.k0 + kk;
    const int lk = k - d.c0;  // panel-local pivot column
    const int owner = lk / CW, lc = lk - owner * CW;
    const int boff = (kk & 1) * (mp + 4);
    if (rank == owner) {
      // pivot: first max |w_ik|, i >= k.  Short columns: every warp scans all rows (no
      // barrier); long ones: the warps split the rows and meet in shared memory.
      const bool split = mp > 256;
      double bv = -1.0;
      int bi = mp;
      for (int i = k + (split ? tid : lane); i < mp; i += (split ? NT : 32)) {
        const double v = fabs(Wl[i * LDS + lc]);
        if (v > bv) { bv = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (split) {
        if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
        __syncthreads();
        bv = redv[0];
        bi = redi[0];
        for (int w = 1; w < NT / 32; ++w)
          if (redv[w] > bv || (redv[w] == bv && redi[w] < bi)) { bv = redv[w]; bi = redi[w]; }
      }
      // push the (pre-swap) column and the pivot into every CTA of the cluster
      for (int e = tid; e < CS * mp; e += NT) {
        const int q = e / mp, i = e - q * mp;
        cluster.map_shared_rank(bc, q)[boff + i] = Wl[i * LDS + lc];
      }
      if (tid < CS) {
        double* rb = cluster.map_shared_rank(bc, tid) + boff;
        rb[mp] = (double)bi;
        rb[mp + 1] = Wl[bi * LDS + lc];
        rb[mp + 2] = (k < m && bv <= tol) ? 1.0 : 0.0;
      }
    }
    cluster.sync();
    const double* ob = bc + boff;
    const int p = (int)ob[mp];
    const double pv = ob[mp + 1];
    if (ob[mp + 2] != 0.0) { fail = k; break; }
    const double inv = 1.0 / pv;
    // swapped multipliers (row p holds old row k's value, row k the pivot's), the
    // new pivot row and the old row k
    for (int i = tid; i < mp; i += NT) fcol[i] = ob[i == k ? p : (i == p ? k : i)];
    for (int c = tid; c < CW; c += NT) {
      okr[c] = Wl[k * LDS + c];
      rk[c] = Wl[p * LDS + c] * inv;
    }
    if (tid == 0) piv_s[kk] = p;
    __syncthreads();
    for (int e = tid; e < mp * CW; e += NT) {
      const int i = e / CW, c = e - i * CW;
      double v;
      if (rank == owner && c == lc) v = i == k ? inv : -fcol[i] * inv;  // Gauss-Jordan column
      else if (i == k) v = rk[c];
      else v = fma(-fcol[i], rk[c], i == p ? okr[c] : Wl[i * LDS + c]);
      Wl[i * LDS + c] = v;
    }
    if (!full && rank == owner && tid == 0) d.piv[(int64_t)b * mp + k] = p;
    __syncthreads();
  }

  if (fail >= 0 && rank == 0 && tid == 0) {
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
  if (full) {
    // column j of the result holds column dest(j) of D^{-1}: undo the swaps in reverse order
    if (fail < 0 && tid == 0) {
      for (int j = 0; j < mp; ++j) dest[j] = j;  // dest[pos] = original column now at pos
      for (int kk = mp - 1; kk >= 0; --kk) {
        const int p = piv_s[kk];
        const int t = dest[kk];
        dest[kk] = dest[p];
        dest[p] = t;
      }
      for (int j = 0; j < mp; ++j) piv_s[dest[j]] = j;  // where each column goes
    }
    __syncthreads();
    double* O = d.out + ((d.idx_out ? d.idx_out[b] : (int64_t)b) + d.add_out) * (int64_t)mp * mp;
    for (int e = tid; e < mp * CW; e += NT) {
      const int r = e / CW, c = e - r * CW, gc = colbase + c;
      if (fail >= 0) O[(int64_t)r * mp + gc] = 0.0;
      else O[(int64_t)r * mp + piv_s[gc]] = Wl[r * LDS + c];
    }
  } else if (fail < 0) {
    for (int e = tid; e < mp * CW; e += NT) {
      const int r = e / CW, c = e - r * CW;
      Wg[(int64_t)r * LDW + colbase + c] = Wl[r * LDS + c];
    }
  }
  cluster.sync();  // no CTA leaves while others may still write into its shared memory
}

// Panel mode set-up: W = D (zero padding columns), max row abs sum of the leading
// m x m block (atomicMax on the bits: nonnegative doubles order like their bits).
// rsmax and dead are zeroed by the caller.  One warp per (entry, row).
__global__ void gjc_init_kernel(GjcDesc d) {
  const int mp = d.mp, LDW = mp + 32, lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < (int64_t)d.nbatch * mp;
       w += nw) {
    const int b = (int)(w / mp), r = (int)(w - (int64_t)b * mp);
    const double* A = d.in + ((d.idx_in ? d.idx_in[b] : (int64_t)b) + d.add_in) * (int64_t)mp * mp + (int64_t)r * mp;
    double* Wr = d.W + ((int64_t)b * mp + r) * LDW;
    double sacc = 0.0;
    for (int c = lane; c < LDW; c += 32) {
      const double v = c < mp ? A[c] : 0.0;
      Wr[c] = v;
      if (r < d.m && c < d.m) sacc += fabs(v);
    }
    for (int o = 16; o; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0 && r < d.m) atomicMax(d.rsmax + b, (unsigned long long)__double_as_longlong(sacc));
  }
}

// Output column of every W column: the row swaps of all pivots, in reverse order,
// applied to the columns (in-place Gauss-Jordan).  One thread per entry.
__global__ void gjc_colmap_kernel(GjcDesc d) {
  const int mp = d.mp;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < d.nbatch; b += gridDim.x * blockDim.x) {
    int32_t* pos = d.colmap + (int64_t)b * mp;  // first: pos[j] = W column found at output position j
    const int32_t* pv = d.piv + (int64_t)b * mp;
    for (int j = 0; j < mp; ++j) pos[j] = j;
    for (int k = mp - 1; k >= 0; --k) {
      const int p = pv[k];
      const int32_t t = pos[k];
      pos[k] = pos[p];
      pos[p] = t;
    }
  }
}

// D^{-1}[r][j] = W[r][colmap[j]] (zeros for failed entries).
__global__ void gjc_extract_kernel(GjcDesc d) {
  const int mp = d.mp, LDW = mp + 32;
  const int64_t per = (int64_t)mp * mp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)d.nbatch * per;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / per);
    const int64_t rc = e - (int64_t)b * per;
    const int r = (int)(rc / mp), j = (int)(rc - (int64_t)r * mp);
    double* O = d.out + ((d.idx_out ? d.idx_out[b] : (int64_t)b) + d.add_out) * per;
    O[rc] = d.dead[b] ? 0.0 : d.W[((int64_t)b * mp + r) * LDW + d.colmap[(int64_t)b * mp + j]];
  }
}

// Update after a panel (panel mode), every W column outside the panel window
// [c0, c0 + PW):  X = Pi W (the panel's row swaps, in order),  W <- X + (T_K - E) X[K]
// T_K = the panel's pivot columns (written back by the panel kernel), E the unit
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
  const int mp = d.mp, LDW = mp + 32, npiv = d.npiv, k0 = d.k0;
  const int cbeg = tile * TN;
  if (cbeg >= mp || (cbeg >= d.c0 && cbeg < d.c0 + PW)) return;  // the panel updated itself
  const int ncols = min(TN, mp - cbeg);
  double* Wg = d.W + (int64_t)b * mp * LDW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int r = tid; r < mp; r += 256) rowmap[r] = -1;
  if (tid == 0) {  // net source row of every position the swaps touch
    int n = 0;
    for (int kk = 0; kk < npiv; ++kk) {
      const int a = k0 + kk, p = d.piv[(int64_t)b * mp + a];
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
    Xi[j][c] = c < ncols ? Wg[(int64_t)src[j] * LDW + cbeg + c] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < PW * TN; e += 256) {
    const int kk = e / TN, c = e - kk * TN;
    double v = 0.0;
    if (kk < npiv && c < ncols) {
      const int r = k0 + kk, j = rowmap[r];
      v = j >= 0 ? Xi[j][c] : Wg[(int64_t)r * LDW + cbeg + c];
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
        if (r < mp && kk < npiv) v = Wg[(int64_t)r * LDW + d.c0 + kk] - (r == k0 + kk ? 1.0 : 0.0);
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
          double* dst = Wg + (int64_t)r * LDW + cbeg + c;
          const double x = jx >= 0 ? Xi[jx][c] : *dst;
          *dst = x + acc[i][j][h];
        }
    }
  }
}

}  // namespace btd
