// Fused Algorithm 1 (reduced interface solve) for small blocks, one cooperative launch.
//
// Reference: dichotomy.py:279-295 (reduced_solve) -- per tree node, in BFS order,
// x~_k = R_node f~[lo..hi] with the end corrections applied from the parent
// splits.  Written as   x~_k = z_node + E_node x~_{lo-1} + H_node x~_{hi+1},
// z_node = R_node f~[lo..hi]  (E, H precomputed at plan time).
//
// For M <= 32 the GEMM-per-level formulation is launch-latency-bound (a c4 plan has
// 592 ranges and 11 tree levels: ~25 dependent launches of tiny GEMMs).  Here:
//   phase 1: the series sums are cut into chunks of CH blocks; every (chunk,
//            16-column tile) item is one warp-level DMMA product (all independent);
//   grid sync;
//   phase 2: level by level, x~_k = sum of the node's chunk partials (fixed order,
//            deterministic) + E x~ + H x~, one grid sync per level.
#pragma once
#include <cooperative_groups.h>

#include "btd_common.cuh"

namespace btd {

struct TreeArgs {
  int nchunks, nlev;
  int64_t K;
  // chunks
  const int32_t* ch_node;
  const int32_t* ch_blk0;
  const int32_t* ch_nblk;
  // per node
  const int64_t* roff;
  const int64_t* rld;
  const int64_t* lo;
  const int64_t* k;
  const int32_t* zc_off;
  const int32_t* zc_cnt;
  const int64_t* xl;
  const int64_t* xh;
  const int32_t* has_e;
  const int32_t* has_h;
  // levels: nodes of level l are lv_nodes[lv_off[l] .. lv_off[l+1])
  const int32_t* lv_off;
  const int32_t* lv_nodes;
  const double* R;    // inverse rows
  const double* EH;   // [2*nodes][MP][MP]
  const double* ft;   // [nr][MP][K]
  double* partial;    // [nchunks][MP][K]
  double* xt;         // [nr+1][MP][K]
};

// acc(MP x 16) += A(MP x MP, global, row stride lda) @ B(MP x 16 cols from col0, global, row stride ldb)
template <int MP, int TM, int TN>
BTD_DEVINL void gmem_mma(double (&acc)[TM][TN][2], const double* __restrict__ A, int64_t lda,
                         const double* __restrict__ B, int64_t ldb, int64_t col0, int64_t K, int g, int t) {
#pragma unroll
  for (int s = 0; s < MP / 8; ++s) {
    double2 a[TM];
    double b0[TN], b1[TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) a[i] = ldg_cg2(A + (int64_t)(i * 8 + g) * lda + 8 * s + 2 * t);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t c = col0 + j * 8 + g;
      b0[j] = c < K ? __ldcg(B + (int64_t)(8 * s + 2 * t) * ldb + j * 8 + g) : 0.0;
      b1[j] = c < K ? __ldcg(B + (int64_t)(8 * s + 2 * t + 1) * ldb + j * 8 + g) : 0.0;
    }
    mma_k4<TM, TN, false>(acc, a, b0);
    mma_k4<TM, TN, true>(acc, a, b1);
  }
}

// One block's fragments for gmem_mma (A: MP x MP at lda; B: MP x 16 cols from col0),
// loaded ahead of use so a chunk's block products overlap their global loads.
template <int MP, int TM, int TN>
struct BlkFrag {
  double2 a[MP / 8][TM];
  double b0[MP / 8][TN], b1[MP / 8][TN];
  BTD_DEVINL void load(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
                       int64_t col0, int64_t K, int g, int t) {
#pragma unroll
    for (int s = 0; s < MP / 8; ++s) {
#pragma unroll
      for (int i = 0; i < TM; ++i) a[s][i] = ldg_cg2(A + (int64_t)(i * 8 + g) * lda + 8 * s + 2 * t);
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const bool in = col0 + j * 8 + g < K;
        b0[s][j] = in ? __ldcg(B + (int64_t)(8 * s + 2 * t) * ldb + j * 8 + g) : 0.0;
        b1[s][j] = in ? __ldcg(B + (int64_t)(8 * s + 2 * t + 1) * ldb + j * 8 + g) : 0.0;
      }
    }
  }
  BTD_DEVINL void mma(double (&acc)[TM][TN][2]) const {
#pragma unroll
    for (int s = 0; s < MP / 8; ++s) {
    mma_k4<TM, TN, false>(acc, a[s], b0[s]);
    mma_k4<TM, TN, true>(acc, a[s], b1[s]);
    }
  }
};

// acc = sum over nblk consecutive blocks e of R[:, e] (MP x MP at column e*MP of a
// row-major MP x ld array) times f~ block e (MP x 16 columns from col0; blocks
// MP*K apart) -- one chunk of a series sum, blocks added in order.
template <int MP, int TM, int TN>
BTD_DEVINL void chunk_series_sum(double (&acc)[TM][TN][2], const double* __restrict__ Rb, int64_t ld,
                                 const double* __restrict__ Fb, int nblk, int64_t K, int64_t col0, int g, int t) {
  const int64_t mpK = (int64_t)MP * K;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if constexpr (MP >= 32) {  // two fragment sets would not fit the register budget
    for (int e = 0; e < nblk; ++e) gmem_mma<MP, TM, TN>(acc, Rb + e * MP, ld, Fb + e * mpK, K, col0, K, g, t);
  } else {
    // block e+1's fragments are in flight while block e's products run (same order of sums)
    BlkFrag<MP, TM, TN> fa, fb;
    fa.load(Rb, ld, Fb, K, col0, K, g, t);
    int e = 0;
    for (; e + 1 < nblk; e += 2) {
      fb.load(Rb + (e + 1) * MP, ld, Fb + (e + 1) * mpK, K, col0, K, g, t);
      fa.mma(acc);
      if (e + 2 < nblk) fa.load(Rb + (e + 2) * MP, ld, Fb + (e + 2) * mpK, K, col0, K, g, t);
      fb.mma(acc);
    }
    if (e < nblk) fa.mma(acc);
  }
}

template <int TM, int TN>
BTD_DEVINL void acc_add_tile(double (&acc)[TM][TN][2], const double* __restrict__ P, int64_t K, int64_t col0, int g,
                             int t) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t c = col0 + j * 8 + 2 * t;
      const double* p = P + (int64_t)(i * 8 + g) * K + c;
      if (c < K) acc[i][j][0] += __ldcg(p);
      if (c + 1 < K) acc[i][j][1] += __ldcg(p + 1);
    }
}

// v = P tile (zeros outside the K columns), the loads acc_add_tile would issue
template <int TM, int TN>
BTD_DEVINL void acc_load_tile(double (&v)[TM][TN][2], const double* __restrict__ P, int64_t K, int64_t col0, int g,
                              int t) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t c = col0 + j * 8 + 2 * t;
      const double* p = P + (int64_t)(i * 8 + g) * K + c;
      v[i][j][0] = c < K ? __ldcg(p) : 0.0;
      v[i][j][1] = c + 1 < K ? __ldcg(p + 1) : 0.0;
    }
}

template <int TM, int TN>
BTD_DEVINL void acc_store_tile(const double (&acc)[TM][TN][2], double* __restrict__ P, int64_t K, int64_t col0,
                               int g, int t) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t c = col0 + j * 8 + 2 * t;
      double* p = P + (int64_t)(i * 8 + g) * K + c;
      if (c < K) __stcg(p, acc[i][j][0]);
      if (c + 1 < K) __stcg(p + 1, acc[i][j][1]);
    }
}

// One level item (node b, 16-column tile) with everything that does not depend on the previous
// level loaded BEFORE the grid barrier that completes it: the node's indices, its z tile and (for
// MP <= 16, register budget) the E / H fragments.  After the barrier only the x~ fragment loads,
// the DMMAs and the store remain on the level's critical path (c4: 11 levels, ~9 -> ~5 us each).
template <int MP, int TM, int TN>
struct LevelItem {
  static constexpr bool FRAG = MP <= 16;
  static constexpr int NS = MP / 8;
  bool have;
  int he, hh;
  int64_t col0, xl, xh, kk;
  double acc[TM][TN][2];
  double2 ea[FRAG ? NS : 1][TM], ha[FRAG ? NS : 1][TM];
  const double *E, *H;

  // indices and factor fragments of node b
  BTD_DEVINL void load_static(int b, int64_t c0, const int64_t* k, const int64_t* xlv, const int64_t* xhv,
                              const int32_t* has_e, const int32_t* has_h, const double* EH, int g, int t) {
    constexpr int64_t blk = (int64_t)MP * MP;
    col0 = c0;
    kk = k[b];
    he = has_e[b];
    hh = has_h[b];
    xl = he ? xlv[b] : 0;
    xh = hh ? xhv[b] : 0;
    E = EH + (2 * (int64_t)b) * blk;
    H = E + blk;
    if constexpr (FRAG) {
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          ea[s][i] = he ? ldg_cg2(E + (i * 8 + g) * MP + 8 * s + 2 * t) : make_double2(0.0, 0.0);
          ha[s][i] = hh ? ldg_cg2(H + (i * 8 + g) * MP + 8 * s + 2 * t) : make_double2(0.0, 0.0);
        }
    }
  }
  // acc += A x~[row] with A from the prefetched fragments (same order of sums as gmem_mma)
  BTD_DEVINL void frag_mma(const double2 (&af)[FRAG ? NS : 1][TM], const double* __restrict__ B, int64_t K, int g,
                           int t) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      double b0[TN], b1[TN];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const bool in = col0 + j * 8 + g < K;
        b0[j] = in ? __ldcg(B + (int64_t)(8 * s + 2 * t) * K + j * 8 + g) : 0.0;
        b1[j] = in ? __ldcg(B + (int64_t)(8 * s + 2 * t + 1) * K + j * 8 + g) : 0.0;
      }
      mma_k4<TM, TN, false>(acc, af[s], b0);
      mma_k4<TM, TN, true>(acc, af[s], b1);
    }
  }
  // x~_k = acc (= z) + E x~_{lo-1} + H x~_{hi+1}
  BTD_DEVINL void finish(double* xt, int64_t K, int g, int t) {
    const int64_t mpK = (int64_t)MP * K;
    if constexpr (FRAG) {
      if (he) frag_mma(ea, xt + xl * mpK + col0, K, g, t);
      if (hh) frag_mma(ha, xt + xh * mpK + col0, K, g, t);
    } else {
      if (he) gmem_mma<MP, TM, TN>(acc, E, MP, xt + xl * mpK + col0, K, col0, K, g, t);
      if (hh) gmem_mma<MP, TM, TN>(acc, H, MP, xt + xh * mpK + col0, K, col0, K, g, t);
    }
    acc_store_tile(acc, xt + kk * mpK, K, col0, g, t);
  }
};

// acc = sum of `ncnt` consecutive partial tiles (chunk order, loads U tiles ahead)
template <int MP, int TM, int TN>
BTD_DEVINL void sum_partials(double (&acc)[TM][TN][2], const double* __restrict__ P0, int ncnt, int64_t K,
                             int64_t col0, int g, int t) {
  const int64_t mpK = (int64_t)MP * K;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int c = 0;
  constexpr int U = MP <= 16 ? 4 : 2;  // loads in flight (register budget)
  for (; c + U <= ncnt; c += U) {
    double v[U][TM][TN][2];
#pragma unroll
    for (int u = 0; u < U; ++u) acc_load_tile(v[u], P0 + (int64_t)(c + u) * mpK, K, col0, g, t);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          acc[i][j][0] += v[u][i][j][0];
          acc[i][j][1] += v[u][i][j][1];
        }
  }
  for (; c < ncnt; ++c) acc_add_tile(acc, P0 + (int64_t)c * mpK, K, col0, g, t);
}

template <int MP>
__global__ void __launch_bounds__(256) tree_small_kernel(TreeArgs a) {
  namespace cg = cooperative_groups;
  constexpr int TM = MP / 8, TN = 2;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int64_t K = a.K, mpK = (int64_t)MP * K;
  const int ntile = (int)((K + 15) / 16);
  constexpr int64_t blk = (int64_t)MP * MP;

  // phase 1: chunk partial series sums  partial[c] = sum_blk R_b[:, blk] f~[lo_b + blk]
  for (int item = gw; item < a.nchunks * ntile; item += nw) {
    const int c = item / ntile;
    const int64_t col0 = (int64_t)(item % ntile) * 16;
    const int b = a.ch_node[c];
    double acc[TM][TN][2];
    chunk_series_sum<MP, TM, TN>(acc, a.R + a.roff[b] + (int64_t)a.ch_blk0[c] * MP, a.rld[b],
                                 a.ft + (a.lo[b] + a.ch_blk0[c]) * mpK + col0, a.ch_nblk[c], K, col0, g, t);
    acc_store_tile(acc, a.partial + (int64_t)c * mpK, K, col0, g, t);
  }
  // phase 2: levels.  A warp's first item of level l is prepared (indices, E / H fragments, and --
  // once the partials exist -- its z = sum of chunk partials) before the barrier that ends level l-1.
  LevelItem<MP, TM, TN> it;
  int itb = 0;
  auto prep_static = [&](int l) {
    const int n0 = a.lv_off[l], n1 = a.lv_off[l + 1];
    it.have = gw < (n1 - n0) * ntile;
    if (it.have) {
      itb = a.lv_nodes[n0 + gw / ntile];
      it.load_static(itb, (int64_t)(gw % ntile) * 16, a.k, a.xl, a.xh, a.has_e, a.has_h, a.EH, g, t);
    }
  };
  auto prep_z = [&]() {
    if (it.have)
      sum_partials<MP, TM, TN>(it.acc, a.partial + (int64_t)a.zc_off[itb] * mpK, a.zc_cnt[itb], K, it.col0, g, t);
  };
  if (a.nlev > 0) prep_static(0);
  grid.sync();
  if (a.nlev > 0) prep_z();
  for (int l = 0; l < a.nlev; ++l) {
    const int n0 = a.lv_off[l], n1 = a.lv_off[l + 1];
    if (it.have) it.finish(a.xt, K, g, t);
    for (int item = gw + nw; item < (n1 - n0) * ntile; item += nw) {  // further items of a wide level
      LevelItem<MP, TM, TN> o;
      const int b = a.lv_nodes[n0 + item / ntile];
      o.load_static(b, (int64_t)(item % ntile) * 16, a.k, a.xl, a.xh, a.has_e, a.has_h, a.EH, g, t);
      sum_partials<MP, TM, TN>(o.acc, a.partial + (int64_t)a.zc_off[b] * mpK, a.zc_cnt[b], K, o.col0, g, t);
      o.finish(a.xt, K, g, t);
    }
    if (l + 1 < a.nlev) {
      prep_static(l + 1);
      prep_z();
    }
    grid.sync();
  }
}


// ---------------------------------------------------------------------------
// Fused Algorithm 1 for a row-sharded plan (M <= 32, one rank of `world`).
// The rank's needed tree nodes split into nodes inside its own ranges (series
// sums computed here) and crossing nodes (each rank contributes the partial sum
// over its own ranges; the partials are all-gathered and added in rank order).
//   phase B (one cooperative launch, before the partials all-gather):
//     chunk partials of every inside node and of this rank's share of every
//     crossing node; grid sync; outputs: z_b (inside nodes) and part_out[c]
//     (crossing index c, zero when the rank owns none of its segment).
//   phase C (one cooperative launch, after it):
//     z_node(c) = sum_r part_all[r][c] (fixed rank order); grid sync; the levels
//     x~_k = z + E x~ + H x~ over this rank's needed nodes, one grid sync each.
// Same per-node arithmetic as the per-level GEMM path (ref dichotomy.py:279-295).
struct ShardTreeArgs {
  int nchunks, nout, ncross, nlev, world;
  int64_t K;
  const int64_t* ch_roff;  // chunk: first R element, R row stride, first f~ range, blocks
  const int64_t* ch_rld;
  const int64_t* ch_flo;
  const int32_t* ch_nblk;
  const int32_t* out_off;  // output o sums chunks [out_off, out_off + out_cnt)
  const int32_t* out_cnt;
  const int64_t* out_dst;  // >= 0: node index into z; < 0: -(1 + crossing index) into part_out
  const int64_t* cross_node;
  const int32_t* lv_off;
  const int32_t* lv_nodes;
  const int64_t* k;
  const int64_t* xl;
  const int64_t* xh;
  const int32_t* has_e;
  const int32_t* has_h;
  const double* R;
  const double* EH;
  const double* ft;
  double* partial;  // [nchunks][MP][K]
  double* z;        // [nodes][MP][K]
  double* xt;       // [nr+1][MP][K]
  double* part_out;        // [ncross][MP][K]
  const double* part_all;  // [world][ncross][MP][K]
};

template <int MP>
__global__ void __launch_bounds__(256) tree_shard_b_kernel(ShardTreeArgs a) {
  namespace cg = cooperative_groups;
  constexpr int TM = MP / 8, TN = 2;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int64_t K = a.K, mpK = (int64_t)MP * K;
  const int ntile = (int)((K + 15) / 16);
  for (int item = gw; item < a.nchunks * ntile; item += nw) {
    const int c = item / ntile;
    const int64_t col0 = (int64_t)(item % ntile) * 16;
    double acc[TM][TN][2];
    chunk_series_sum<MP, TM, TN>(acc, a.R + a.ch_roff[c], a.ch_rld[c], a.ft + a.ch_flo[c] * mpK + col0,
                                 a.ch_nblk[c], K, col0, g, t);
    acc_store_tile(acc, a.partial + (int64_t)c * mpK, K, col0, g, t);
  }
  grid.sync();
  for (int item = gw; item < a.nout * ntile; item += nw) {
    const int o = item / ntile;
    const int64_t col0 = (int64_t)(item % ntile) * 16;
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* P0 = a.partial + (int64_t)a.out_off[o] * mpK;
    for (int c = 0; c < a.out_cnt[o]; ++c) acc_add_tile(acc, P0 + (int64_t)c * mpK, K, col0, g, t);
    const int64_t d = a.out_dst[o];
    double* dst = d >= 0 ? a.z + d * mpK : a.part_out + (-1 - d) * mpK;
    acc_store_tile(acc, dst, K, col0, g, t);
  }
}

template <int MP>
__global__ void __launch_bounds__(256) tree_shard_c_kernel(ShardTreeArgs a) {
  namespace cg = cooperative_groups;
  constexpr int TM = MP / 8, TN = 2;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int64_t K = a.K, mpK = (int64_t)MP * K;
  const int ntile = (int)((K + 15) / 16);
  constexpr int64_t blk = (int64_t)MP * MP;
  if (a.ncross) {
    for (int item = gw; item < a.ncross * ntile; item += nw) {
      const int c = item / ntile;
      const int64_t col0 = (int64_t)(item % ntile) * 16;
      double acc[TM][TN][2];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int r = 0; r < a.world; ++r)
        acc_add_tile(acc, a.part_all + ((int64_t)r * a.ncross + c) * mpK, K, col0, g, t);
      acc_store_tile(acc, a.z + a.cross_node[c] * mpK, K, col0, g, t);
    }
    grid.sync();
  }
  // levels, a warp's first item of level l prepared before the barrier that ends level l-1 (as in
  // tree_small_kernel); z of a crossing node exists only after the barrier above
  LevelItem<MP, TM, TN> it;
  auto prep = [&](int l, bool with_z) {
    const int n0 = a.lv_off[l], n1 = a.lv_off[l + 1];
    it.have = gw < (n1 - n0) * ntile;
    if (it.have) {
      const int b = a.lv_nodes[n0 + gw / ntile];
      it.load_static(b, (int64_t)(gw % ntile) * 16, a.k, a.xl, a.xh, a.has_e, a.has_h, a.EH, g, t);
      if (with_z) acc_load_tile(it.acc, a.z + (int64_t)b * mpK, K, it.col0, g, t);
    }
  };
  if (a.nlev > 0) prep(0, true);
  for (int l = 0; l < a.nlev; ++l) {
    const int n0 = a.lv_off[l], n1 = a.lv_off[l + 1];
    if (it.have) it.finish(a.xt, K, g, t);
    for (int item = gw + nw; item < (n1 - n0) * ntile; item += nw) {
      LevelItem<MP, TM, TN> o;
      const int b = a.lv_nodes[n0 + item / ntile];
      o.load_static(b, (int64_t)(item % ntile) * 16, a.k, a.xl, a.xh, a.has_e, a.has_h, a.EH, g, t);
      acc_load_tile(o.acc, a.z + (int64_t)b * mpK, K, o.col0, g, t);
      o.finish(a.xt, K, g, t);
    }
    if (l + 1 < a.nlev) prep(l + 1, true);
    grid.sync();
  }
}

}  // namespace btd
