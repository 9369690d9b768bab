// Fused forward / backward block sweeps of Algorithm 2 (the per-RHS hot path).
//
// Reference path replaced (per range q, interior rows g = lo+1 .. hi-1):
//   W = thomas_solve(fact, f[lo+1:hi])        ref dichotomy.py:196-209, _kernels.pyx:173-194
//   base/carry of the interface RHS           ref dichotomy.py:239-263
//   x = U x~_q + V x~_{q+1} + W  (recovery)   ref dichotomy.py:345-355
// by two passes over the rows with factors precomputed at plan time:
//   forward :  y_j = Dinv_j f_g + AD_j y_{j-1}           (AD_j = Dinv_j A_j)
//              base_q = f_lo + sum_j Tb_j y_j           (Tb_j = B_lo S_0..S_{j-1}; = B_lo W[1])
//   backward:  x_j = y_j + G_j x~_q + S_j x_{j+1},  x_{nint} = x~_{q+1}
// which is the block LU of the interior with both boundary responses folded
// in (G = response to x~_q, S = D^{-1}B).  10 M^2 K flops and 5 M^2 + 4 M K
// doubles per row -- the SURVEY 8(d) algorithmic count.
//
// Work decomposition: one CTA per (range q, column tile of KT right-hand
// sides); the chain state (y or x, MP x KT) stays in shared memory for the
// whole range, factor fragments stream from HBM/L2 straight into registers
// (16-byte loads, PF pair-steps ahead), the next row's F tile is prefetched
// into a second shared buffer with cp.async.  Products are DMMA m8n8k4.
#pragma once
#include "btd_common.cuh"

namespace btd {

struct ChainArgs {
  const int64_t* lo;     // [nr] interface row of range q (may be >= n: padded range)
  const int32_t* nint;   // [nr] interior rows of range q inside [0, n)
  const int64_t* slot0;  // [nr] factor slot of interior row 0
  int nr;
  int m;                 // true block order (F/X rows per block)
  int64_t n, K;
  const double* F;
  double* X;
  const double* AD;      // factor pools: block s at ptr + s*MP*MP
  const double* Dinv;
  const double* Tb;
  const double* S;
  const double* G;
  double* base;          // fwd out: range q at base + q*base_stride ([MP][K] each)
  int64_t base_stride;
  const double* xt;      // bwd in:  [nr+1][MP][K], range q uses blocks q and q+1
};

// Forward sweep of a scalar-coupled plan (interior lower blocks A_g = a_g I).  A separate
// parameter struct: growing ChainArgs itself shifts ptxas' schedule of the register-capped
// general kernels (c2 forward sweep +2%, measured).
struct ChainArgsSc : ChainArgs {
  const double* Tbd;     // Tbd_j = Tb_j Dinv_j  (block s at ptr + s*MP*MP)
  const double* alpha;   // a_g per factor slot
};

// acc += A(warp rows, MP cols, global) @ Bs(MP x cols, smem, ld LDB)
template <int MP, int TM, int TN, int PF>
BTD_DEVINL void wgemm(double (&acc)[TM][TN][2], const double* __restrict__ A,
                      const double* __restrict__ Bs, int ldb, int g, int t) {
  constexpr int NS = MP / 8;
  constexpr int P = PF < NS ? PF : NS;
  double2 buf[P][TM];
#pragma unroll
  for (int s = 0; s < P; ++s)
#pragma unroll
    for (int i = 0; i < TM; ++i) buf[s][i] = ldg_cg2(A + (i * 8 + g) * MP + 8 * s + 2 * t);
#pragma unroll(NS <= 8 ? NS / P : 1)
  for (int s0 = 0; s0 < NS; s0 += P) {
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int s = s0 + u;
      double2 a[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = buf[u][i];
      if (s + P < NS) {
#pragma unroll
        for (int i = 0; i < TM; ++i) buf[u][i] = ldg_cg2(A + (i * 8 + g) * MP + 8 * (s + P) + 2 * t);
      }
      double b0[TN], b1[TN];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        b0[j] = Bs[(8 * s + 2 * t) * ldb + j * 8 + g];
        b1[j] = Bs[(8 * s + 2 * t + 1) * ldb + j * 8 + g];
      }
      mma_k4<TM, TN, false>(acc, a, b0);
      mma_k4<TM, TN, true>(acc, a, b1);
    }
  }
}

// acc1 += A1 @ Bs ; acc2 += A2 @ Bs  (shared B fragments)
template <int MP, int TM, int TN, int PF>
BTD_DEVINL void wgemm2(double (&acc1)[TM][TN][2], const double* __restrict__ A1,
                       double (&acc2)[TM][TN][2], const double* __restrict__ A2,
                       const double* __restrict__ Bs, int ldb, int g, int t) {
  constexpr int NS = MP / 8;
  constexpr int P = PF < NS ? PF : NS;
  double2 buf1[P][TM], buf2[P][TM];
#pragma unroll
  for (int s = 0; s < P; ++s)
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      buf1[s][i] = ldg_cg2(A1 + (i * 8 + g) * MP + 8 * s + 2 * t);
      buf2[s][i] = ldg_cg2(A2 + (i * 8 + g) * MP + 8 * s + 2 * t);
    }
#pragma unroll(NS <= 8 ? NS / P : 1)
  for (int s0 = 0; s0 < NS; s0 += P) {
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int s = s0 + u;
      double2 a1[TM], a2[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) { a1[i] = buf1[u][i]; a2[i] = buf2[u][i]; }
      if (s + P < NS) {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          buf1[u][i] = ldg_cg2(A1 + (i * 8 + g) * MP + 8 * (s + P) + 2 * t);
          buf2[u][i] = ldg_cg2(A2 + (i * 8 + g) * MP + 8 * (s + P) + 2 * t);
        }
      }
      double b0[TN], b1[TN];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        b0[j] = Bs[(8 * s + 2 * t) * ldb + j * 8 + g];
        b1[j] = Bs[(8 * s + 2 * t + 1) * ldb + j * 8 + g];
      }
      mma_k4<TM, TN, false>(acc1, a1, b0);
      mma_k4<TM, TN, false>(acc2, a2, b0);
      mma_k4<TM, TN, true>(acc1, a1, b1);
      mma_k4<TM, TN, true>(acc2, a2, b1);
    }
  }
}

template <int TM, int TN>
BTD_DEVINL void zero_acc(double (&acc)[TM][TN][2]) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// C-layout tile <-> global (rows r < rmax, cols c < K), row stride K.
// FULL: every row < rmax and column pair < K (block order == MP, K a multiple of the tile
// width, K even) -- no bounds checks, 16-byte accesses only.
template <int TM, int TN, bool FULL = false>
BTD_DEVINL void load_tile(double (&acc)[TM][TN][2], const double* __restrict__ P, int64_t K,
                          int r0, int64_t c0, int rmax, int g, int t, bool vec) {
  if constexpr (FULL) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(P + (int64_t)(r0 + i * 8 + g) * K + c0 + j * 8 + 2 * t));
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      }
    return;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int r = r0 + i * 8 + g;
      const int64_t c = c0 + j * 8 + 2 * t;
      double v0 = 0.0, v1 = 0.0;
      if (r < rmax) {
        const double* p = P + (int64_t)r * K + c;
        if (vec && c + 1 < K) {
          double2 v = __ldcs(reinterpret_cast<const double2*>(p));
          v0 = v.x; v1 = v.y;
        } else {
          if (c < K) v0 = __ldcs(p);
          if (c + 1 < K) v1 = __ldcs(p + 1);
        }
      }
      acc[i][j][0] = v0;
      acc[i][j][1] = v1;
    }
}

template <int TM, int TN, bool FULL = false>
BTD_DEVINL void store_tile(const double (&acc)[TM][TN][2], double* __restrict__ P, int64_t K,
                           int r0, int64_t c0, int rmax, int g, int t, bool vec) {
  if constexpr (FULL) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
        __stcg(reinterpret_cast<double2*>(P + (int64_t)(r0 + i * 8 + g) * K + c0 + j * 8 + 2 * t),
               make_double2(acc[i][j][0], acc[i][j][1]));
    return;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int r = r0 + i * 8 + g;
      const int64_t c = c0 + j * 8 + 2 * t;
      if (r >= rmax) continue;
      double* p = P + (int64_t)r * K + c;
      if (vec && c + 1 < K) {
        __stcg(reinterpret_cast<double2*>(p), make_double2(acc[i][j][0], acc[i][j][1]));
      } else {
        if (c < K) __stcg(p, acc[i][j][0]);
        if (c + 1 < K) __stcg(p + 1, acc[i][j][1]);
      }
    }
}

template <int TM, int TN>
BTD_DEVINL void store_smem(const double (&acc)[TM][TN][2], double* Ys, int ld, int r0, int c0, int g,
                           int t) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j)
      *reinterpret_cast<double2*>(&Ys[(r0 + i * 8 + g) * ld + c0 + j * 8 + 2 * t]) =
          make_double2(acc[i][j][0], acc[i][j][1]);
}

// Async copy of one (rows < rmax) x (KT cols from c0, < K) tile of a
// row-major [*, K] array into smem [MP][LD].  Rows/cols outside stay as they
// are (zeroed once at kernel start).
template <int MP, int KT, int LD, int NT>
BTD_DEVINL void cp_tile(double* Ys, const double* __restrict__ P, int64_t K, int64_t c0, int rmax,
                        bool vec) {
  const int tid = threadIdx.x;
  if (vec) {
    constexpr int CH = KT / 2;
    for (int e = tid; e < rmax * CH; e += NT) {
      const int r = e / CH, cc = (e % CH) * 2;
      if (c0 + cc < K) cp_async16(&Ys[r * LD + cc], P + (int64_t)r * K + c0 + cc);
    }
  } else {
    for (int e = tid; e < rmax * KT; e += NT) {
      const int r = e / KT, cc = e % KT;
      if (c0 + cc < K) cp_async8(&Ys[r * LD + cc], P + (int64_t)r * K + c0 + cc);
    }
  }
  cp_async_commit();
}

// Column-group variant of cp_tile: the NTG threads of one warp-column group copy
// columns [c0, c0 + W) into dst (already offset to the group's first column).
template <int W, int LD, int NTG>
BTD_DEVINL void cp_tile_cols(double* dst, const double* __restrict__ P, int64_t K, int64_t c0, int rmax, bool vec,
                             int gtid) {
  if (vec) {
    constexpr int CH = W / 2;
    for (int e = gtid; e < rmax * CH; e += NTG) {
      const int r = e / CH, cc = (e % CH) * 2;
      if (c0 + cc < K) cp_async16(&dst[r * LD + cc], P + (int64_t)r * K + c0 + cc);
    }
  } else {
    for (int e = gtid; e < rmax * W; e += NTG) {
      const int r = e / W, cc = e % W;
      if (c0 + cc < K) cp_async8(&dst[r * LD + cc], P + (int64_t)r * K + c0 + cc);
    }
  }
  cp_async_commit();
}

// Per-row barrier of a chain CTA.  Column tiles are independent chains, so with
// WC > 1 warp columns each column group (its WR warps) syncs on its own named
// barrier: the groups drift apart and one group's row epilogue (stores, F-tile
// refill, barrier) overlaps the other group's DMMAs instead of idling the pipe.
template <int WR, int WC>
BTD_DEVINL void group_sync(int wc) {
  if constexpr (WC == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wc), "r"(32 * WR) : "memory");
  }
}

template <int MP, int KT, int WR, int WC, int NF_ = -1, int NY_ = -1, int PF_ = -1>
struct ChainCfg {
  static constexpr int NW = WR * WC, NT = 32 * NW;
  static constexpr int RW = MP / WR, CW = KT / WC;
  static constexpr int TM = RW / 8, TN = CW / 8;
  static constexpr int LD = KT + 2;  // == 2 (mod 16) when KT % 16 == 0
  static constexpr int NS = MP / 8;  // pair steps per block product
  // factor-fragment prefetch distance (pair steps), one group ahead
  static constexpr int PF = PF_ > 0 ? (PF_ < NS ? PF_ : NS) : (NS < 4 ? NS : (TM >= 4 ? 2 : 4));
  static constexpr int GPS = NS / PF;  // groups per segment
  // cp.async ring depths: forward F tiles, backward y tiles (0 = register prefetch)
  // (measured on B200: deeper rings hurt the 16x16 one-warp tiles of c4)
  static constexpr int NF = NF_ >= 0 ? NF_ : (MP <= 16 ? 2 : (MP <= 64 ? 3 : 2));
  static constexpr int NY = NY_ >= 0 ? NY_ : (MP <= 16 ? 0 : (MP <= 64 ? 3 : 0));
  static constexpr int FWD_BUFS = 1 + NF;
  static constexpr int PD = 3;  // L2-prefetch distance (rows ahead) for factors and F / y tiles
  // only the memory-latency-bound small blocks profit (measured: c4 fwd -7%, c1/c2 +10-20%)
  static constexpr bool PREF = MP <= 32;
  static constexpr int BWD_BUFS = 2 + NY;
  static_assert(RW % 8 == 0 && CW % 8 == 0, "warp tile must be a multiple of 8x8");
  static_assert(NS % PF == 0, "prefetch groups must tile a segment");
  static_assert(NY != 1, "a one-deep y ring would read a tile before it is loaded");
};

// One prefetch group: PF pair steps of  acc += A_seg @ Bs, consuming the
// register ring `buf` and refilling it with the next group's fragments
// (`nxt` points at that group's first fragment; nullptr = stream end).
template <int MP, int TM, int TN, int PF>
BTD_DEVINL void group_mma(double (&acc)[TM][TN][2], double2 (&buf)[PF][TM], const double* __restrict__ nxt,
                          const double* __restrict__ Bs, int ldb, int s0, int g, int t) {
#pragma unroll
  for (int u = 0; u < PF; ++u) {
    double2 a[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) a[i] = buf[u][i];
    if (nxt) {
#pragma unroll
      for (int i = 0; i < TM; ++i) buf[u][i] = ldg_cg2(nxt + (i * 8 + g) * MP + 8 * u + 2 * t);
    }
    const int s = s0 + u;
    double b0[TN], b1[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      b0[j] = Bs[(8 * s + 2 * t) * ldb + j * 8 + g];
      b1[j] = Bs[(8 * s + 2 * t + 1) * ldb + j * 8 + g];
    }
    // all k-slot-0 products first, then k-slot-1: consecutive DMMAs are independent
    mma_k4<TM, TN, false>(acc, a, b0);
    mma_k4<TM, TN, true>(acc, a, b1);
  }
}

template <int MP, int TM, int PF>
BTD_DEVINL void group_load(double2 (&buf)[PF][TM], const double* __restrict__ p, int g, int t) {
#pragma unroll
  for (int u = 0; u < PF; ++u)
#pragma unroll
    for (int i = 0; i < TM; ++i) buf[u][i] = ldg_cg2(p + (i * 8 + g) * MP + 8 * u + 2 * t);
}


// Forward sweep.  Per interior row j, three segments stream through the same
// register ring:  seg0 acc += AD_j y_{j-1};  seg1 ser += Tb_{j-1} y_{j-1};
// seg2 acc += Dinv_j f_g.  (At j = 0, y_{-1} = 0 and seg1 reuses Tb_0.)
template <int MP, int KT, int WR, int WC, int NF_ = -1, int NY_ = -1, int PF_ = -1, int MINB_ = 1, int FULL_ = 0>
__global__ void __launch_bounds__(32 * WR * WC, MINB_) chain_fwd_kernel(ChainArgs a) {
  using Cfg = ChainCfg<MP, KT, WR, WC, NF_, NY_, PF_>;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, LD = Cfg::LD, NT = Cfg::NT, PF = Cfg::PF, GPS = Cfg::GPS;
  constexpr int NF = Cfg::NF;
  extern __shared__ __align__(16) double sm[];
  double* Ys = sm;
  double* Fs = sm + MP * LD;  // ring of NF F tiles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int r0 = wr * Cfg::RW, cw0 = wc * Cfg::CW;
  const int q = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * KT;
  const int64_t K = a.K;
  const bool vec = (K % 2) == 0;
  for (int e = tid; e < Cfg::FWD_BUFS * MP * LD; e += NT) sm[e] = 0.0;
  __syncthreads();

  const int64_t lo = a.lo[q];
  const int nint = a.nint[q];
  const int64_t slot0 = a.slot0[q];
  const int64_t blk = (int64_t)MP * MP;
  const int64_t rowK = (int64_t)a.m * K;

  double ser[TM][TN][2];
  if (lo < a.n)
    load_tile(ser, a.F + lo * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
  else
    zero_acc(ser);
  if (nint <= 0) {
    store_tile(ser, a.base + (int64_t)q * a.base_stride, K, r0, c0 + cw0, MP, g, t, vec);
    return;
  }
  // prologue: F rows 0 .. NF-2 in flight (one cp.async group per row, possibly empty)
#pragma unroll
  for (int r = 0; r < NF - 1; ++r) {
    if (r < nint)
      cp_tile<MP, KT, LD, NT>(Fs + r * MP * LD, a.F + (lo + 1 + r) * rowK, K, c0, a.m, vec);
    else
      cp_async_commit();
  }

  // factor-fragment stream, rows ascending: AD_j, Tb_{j-1} (row 0 reuses Tb_0 against y_{-1} = 0),
  // Dinv_j.  One row pointer into the AD blocks plus constant offsets to the Tb / Dinv pools.
  const double* frow = a.AD + slot0 * blk + r0 * MP;
  const int64_t tb_off = a.Tb - a.AD, dinv_off = a.Dinv - a.AD;
  int fseg = 0, fgrp = 0, frows = nint;
  bool frow0 = true;  // the stream is still in row 0 (its Tb segment uses Tb_0, not Tb_{-1})
  double2 buf[PF][TM];
  group_load<MP, TM, PF>(buf, frow, g, t);
  cp_async_wait<NF - 2>();
  __syncthreads();

  double acc[TM][TN][2];
  zero_acc(acc);
  for (int j = 0; j < nint; ++j) {
    const int64_t gr = lo + 1 + j;
    const double* Fcur = Fs + (j % NF) * MP * LD;
    if constexpr (Cfg::PREF) {  // L2 prefetch: row j+PD's factor blocks (this warp's rows), F tile
      const int jp = j + Cfg::PD;
      if (jp < nint) {
        const int64_t off = (slot0 + jp) * blk + r0 * MP;
        warp_prefetch_l2(a.AD + off, (int64_t)Cfg::RW * MP * 8, lane);
        warp_prefetch_l2(a.Tb + off - blk, (int64_t)Cfg::RW * MP * 8, lane);
        warp_prefetch_l2(a.Dinv + off, (int64_t)Cfg::RW * MP * 8, lane);
      }
      const int jf = j + NF - 1 + Cfg::PD;
      if (jf < nint && wc == 0) {
        const int rr = r0 + lane;
        if (lane < Cfg::RW && rr < a.m) prefetch_l2(a.F + (lo + 1 + jf) * rowK + (int64_t)rr * K + c0);
      }
    }
    // refill the slot freed by row j-1 with row j+NF-1
    if (j + NF - 1 < nint)
      cp_tile_cols<Cfg::CW, LD, 32 * WR>(Fs + ((j + NF - 1) % NF) * MP * LD + cw0, a.F + (gr + NF - 1) * rowK, K,
                                         c0 + cw0, a.m, vec, wr * 32 + lane);
    else
      cp_async_commit();
#pragma unroll 1
    for (int seg = 0; seg < 3; ++seg) {
#pragma unroll 1
      for (int grp = 0; grp < GPS; ++grp) {
        if (++fgrp == GPS) {  // advance the stream: next group, segment, row
          fgrp = 0;
          if (++fseg == 3) {
            fseg = 0;
            frow += blk;
            --frows;
            frow0 = false;
          }
        }
        const double* nx = nullptr;
        if (frows > 0)
          nx = frow + (fseg == 0 ? 0 : (fseg == 1 ? tb_off - (frow0 ? 0 : blk) : dinv_off)) + fgrp * 8 * PF;
        if (seg == 0)
          group_mma<MP, TM, TN, PF>(acc, buf, nx, Ys + cw0, LD, grp * PF, g, t);
        else if (seg == 1)
          group_mma<MP, TM, TN, PF>(ser, buf, nx, Ys + cw0, LD, grp * PF, g, t);
        else
          group_mma<MP, TM, TN, PF>(acc, buf, nx, Fcur + cw0, LD, grp * PF, g, t);
      }
    }
    group_sync<WR, WC>(wc);
    store_smem(acc, Ys, LD, r0, cw0, g, t);
    store_tile<TM, TN, FULL_ != 0>(acc, a.X + gr * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
    zero_acc(acc);
    cp_async_wait<NF - 2>();  // row j+1's F tile has landed
    group_sync<WR, WC>(wc);
  }
  cp_async_wait<0>();
  wgemm<MP, TM, TN, 2>(ser, a.Tb + (slot0 + nint - 1) * blk + r0 * MP, Ys + cw0, LD, g, t);
  store_tile(ser, a.base + (int64_t)q * a.base_stride, K, r0, c0 + cw0, MP, g, t, vec);
}

// Forward sweep of a scalar-coupled plan: every interior lower block is a_g I (5-point-stencil
// operators: BASELINE config 1, the Helmholtz subdomains of config 3), so AD_j = a_g Dinv_j and
//   y_j = Dinv_j u_j,  u_j = f_g + a_g y_{j-1},   base_q = f_lo + sum_j Tbd_j u_j  (Tbd_j = Tb_j Dinv_j)
// -- two block products per row instead of three (8 instead of 10 M^2 K flops per row and
// batch for the whole solve, one factor stream less).  The chain state in shared memory is u_j;
// per row two segments stream through the register ring (Dinv_j, Tbd_j against the same u_j);
// the epilogue stores y_j and forms u_{j+1} from the prefetched F tile.
template <int MP, int KT, int WR, int WC, int NF_ = -1, int NY_ = -1, int PF_ = -1, int MINB_ = 1, int FULL_ = 0>
__global__ void __launch_bounds__(32 * WR * WC, MINB_) chain_fwd_sc_kernel(ChainArgsSc a) {
  using Cfg = ChainCfg<MP, KT, WR, WC, 2, NY_, PF_>;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, LD = Cfg::LD, NT = Cfg::NT, PF = Cfg::PF, GPS = Cfg::GPS;
  constexpr int NF = 2;  // F tiles of rows j+1 (read in row j's epilogue) and j+2 (in flight)
  extern __shared__ __align__(16) double sm[];
  double* Us = sm;
  double* Fs = sm + MP * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int r0 = wr * Cfg::RW, cw0 = wc * Cfg::CW;
  const int q = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * KT;
  const int64_t K = a.K;
  const bool vec = (K % 2) == 0;
  for (int e = tid; e < (1 + NF) * MP * LD; e += NT) sm[e] = 0.0;
  __syncthreads();

  const int64_t lo = a.lo[q];
  const int nint = a.nint[q];
  const int64_t slot0 = a.slot0[q];
  const int64_t blk = (int64_t)MP * MP;
  const int64_t rowK = (int64_t)a.m * K;

  double ser[TM][TN][2];
  if (lo < a.n)
    load_tile(ser, a.F + lo * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
  else
    zero_acc(ser);
  if (nint <= 0) {
    store_tile(ser, a.base + (int64_t)q * a.base_stride, K, r0, c0 + cw0, MP, g, t, vec);
    return;
  }
  // u_0 = f of interior row 0 straight into the chain state; row 1's F tile into slot 1
  cp_tile<MP, KT, LD, NT>(Us, a.F + (lo + 1) * rowK, K, c0, a.m, vec);
  if (nint > 1)
    cp_tile<MP, KT, LD, NT>(Fs + MP * LD, a.F + (lo + 2) * rowK, K, c0, a.m, vec);
  else
    cp_async_commit();

  // factor-fragment stream, rows ascending: Dinv_j then Tbd_j
  const double* frow = a.Dinv + slot0 * blk + r0 * MP;
  const int64_t tbd_off = a.Tbd - a.Dinv;
  int fseg = 0, fgrp = 0, frows = nint;
  double2 buf[PF][TM];
  group_load<MP, TM, PF>(buf, frow, g, t);
  cp_async_wait<0>();
  __syncthreads();

  double acc[TM][TN][2];
  zero_acc(acc);
  for (int j = 0; j < nint; ++j) {
    const int64_t gr = lo + 1 + j;
    // row j+2's F tile into the slot row j's tile left (consumed in row j-1's epilogue)
    if (j + 2 < nint)
      cp_tile_cols<Cfg::CW, LD, 32 * WR>(Fs + (j % NF) * MP * LD + cw0, a.F + (gr + 2) * rowK, K, c0 + cw0, a.m, vec,
                                         wr * 32 + lane);
    else
      cp_async_commit();
    const double al = j + 1 < nint ? __ldg(a.alpha + slot0 + j + 1) : 0.0;
#pragma unroll 1
    for (int seg = 0; seg < 2; ++seg) {
#pragma unroll 1
      for (int grp = 0; grp < GPS; ++grp) {
        if (++fgrp == GPS) {  // advance the stream: next group, segment (Dinv -> Tbd), row
          fgrp = 0;
          if (++fseg == 2) {
            fseg = 0;
            frow += blk;
            --frows;
          }
        }
        const double* nx = frows > 0 ? frow + (fseg ? tbd_off : 0) + fgrp * 8 * PF : nullptr;
        if (seg == 0)
          group_mma<MP, TM, TN, PF>(acc, buf, nx, Us + cw0, LD, grp * PF, g, t);
        else
          group_mma<MP, TM, TN, PF>(ser, buf, nx, Us + cw0, LD, grp * PF, g, t);
      }
    }
    cp_async_wait<1>();  // this thread's part of row j+1's F tile has landed (issued a row ago)
    group_sync<WR, WC>(wc);  // ... and everyone's; all reads of u_j are done
    store_tile<TM, TN, FULL_ != 0>(acc, a.X + gr * rowK, K, r0, c0 + cw0, a.m, g, t, vec);  // y_j
    if (j + 1 < nint) {  // u_{j+1} = f_{g+1} + a_{g+1} y_j
      const double* Fn = Fs + ((j + 1) % NF) * MP * LD;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int c = 0; c < TN; ++c) {
          const int off = (r0 + i * 8 + g) * LD + cw0 + c * 8 + 2 * t;
          const double2 f = *reinterpret_cast<const double2*>(&Fn[off]);
          *reinterpret_cast<double2*>(&Us[off]) = make_double2(fma(al, acc[i][c][0], f.x), fma(al, acc[i][c][1], f.y));
        }
    }
    zero_acc(acc);
    group_sync<WR, WC>(wc);
  }
  cp_async_wait<0>();
  store_tile(ser, a.base + (int64_t)q * a.base_stride, K, r0, c0 + cw0, MP, g, t, vec);
}

// C-layout tile from a shared [MP][LD] tile
template <int TM, int TN>
BTD_DEVINL void load_smem(double (&acc)[TM][TN][2], const double* Ys, int ld, int r0, int c0, int g, int t) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(&Ys[(r0 + i * 8 + g) * ld + c0 + j * 8 + 2 * t]);
      acc[i][j][0] = v.x;
      acc[i][j][1] = v.y;
    }
}

// Backward sweep: per row j (descending) two segments through one ring:
// seg0 acc += G_j x~_q ; seg1 acc += S_j x_{j+1}, with acc initialised to y_j.
template <int MP, int KT, int WR, int WC, int NF_ = -1, int NY_ = -1, int PF_ = -1, int MINB_ = 1, int FULL_ = 0>
__global__ void __launch_bounds__(32 * WR * WC, MINB_) chain_bwd_kernel(ChainArgs a) {
  using Cfg = ChainCfg<MP, KT, WR, WC, NF_, NY_, PF_>;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, LD = Cfg::LD, NT = Cfg::NT, PF = Cfg::PF, GPS = Cfg::GPS;
  constexpr int NY = Cfg::NY;
  extern __shared__ __align__(16) double sm[];
  double* Xq = sm;
  double* Xn = sm + MP * LD;
  double* Ysr = sm + 2 * MP * LD;  // ring of NY y tiles (NY > 0)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int r0 = wr * Cfg::RW, cw0 = wc * Cfg::CW;
  const int q = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * KT;
  const int64_t K = a.K;
  const bool vec = (K % 2) == 0;
  for (int e = tid; e < Cfg::BWD_BUFS * MP * LD; e += NT) sm[e] = 0.0;
  __syncthreads();

  const int64_t lo = a.lo[q];
  const int nint = a.nint[q];
  const int64_t slot0 = a.slot0[q];
  const int64_t blk = (int64_t)MP * MP;
  const int64_t rowK = (int64_t)a.m * K;
  const int64_t xtK = (int64_t)MP * K;

  cp_tile<MP, KT, LD, NT>(Xq, a.xt + (int64_t)q * xtK, K, c0, MP, vec);
  cp_tile<MP, KT, LD, NT>(Xn, a.xt + (int64_t)(q + 1) * xtK, K, c0, MP, vec);
  if (lo < a.n) {  // x[lo] = x~_q  (ref dichotomy.py:351)
    double xq[TM][TN][2];
    load_tile(xq, a.xt + (int64_t)q * xtK, K, r0, c0 + cw0, MP, g, t, vec);
    store_tile(xq, a.X + lo * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
  }
  if (nint <= 0) {
    cp_async_wait<0>();
    return;
  }
  // rows run j = nint-1 .. 0 (step jj = nint-1-j); y tiles of steps 0..NY-2 in flight
  if constexpr (NY > 0) {
#pragma unroll
    for (int s_ = 0; s_ < NY - 1; ++s_) {
      if (s_ < nint)
        cp_tile<MP, KT, LD, NT>(Ysr + s_ * MP * LD, a.X + (lo + nint - s_) * rowK, K, c0, a.m, vec);
      else
        cp_async_commit();
    }
  }
  // factor-fragment stream, rows descending: G_j then S_j per row.  One row pointer into the G
  // blocks plus the constant G -> S distance (fewer live registers than a per-segment cursor).
  const double* frow = a.G + (slot0 + nint - 1) * blk + r0 * MP;
  const int64_t s_off = a.S - a.G;
  int fseg = 0, fgrp = 0, frows = nint;
  double2 buf[PF][TM];
  group_load<MP, TM, PF>(buf, frow, g, t);
  double y[TM][TN][2];
  if constexpr (NY == 0) load_tile(y, a.X + (lo + nint) * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
  cp_async_wait<(NY > 1 ? NY - 2 : 0)>();
  __syncthreads();
  for (int jj = 0; jj < nint; ++jj) {
    const int j = nint - 1 - jj;
    const int64_t gr = lo + 1 + j;
    if constexpr (Cfg::PREF) {  // L2 prefetch: row j-PD's G and S blocks (this warp's rows), y tile
      const int jp = j - Cfg::PD;
      if (jp >= 0) {
        const int64_t off = (slot0 + jp) * blk + r0 * MP;
        warp_prefetch_l2(a.G + off, (int64_t)Cfg::RW * MP * 8, lane);
        warp_prefetch_l2(a.S + off, (int64_t)Cfg::RW * MP * 8, lane);
        if (wc == 0) {
          const int rr = r0 + lane;
          if (lane < Cfg::RW && rr < a.m) prefetch_l2(a.X + (lo + 1 + jp) * rowK + (int64_t)rr * K + c0);
        }
      }
    }
    double acc[TM][TN][2];
    if constexpr (NY > 0) {
      load_smem(acc, Ysr + (jj % NY) * MP * LD, LD, r0, cw0, g, t);
      if (jj + NY - 1 < nint)
        cp_tile_cols<Cfg::CW, LD, 32 * WR>(Ysr + ((jj + NY - 1) % NY) * MP * LD + cw0, a.X + (gr - (NY - 1)) * rowK,
                                           K, c0 + cw0, a.m, vec, wr * 32 + lane);
      else
        cp_async_commit();
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int c = 0; c < TN; ++c) { acc[i][c][0] = y[i][c][0]; acc[i][c][1] = y[i][c][1]; }
      if (j > 0) load_tile<TM, TN, FULL_ != 0>(y, a.X + (gr - 1) * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
    }
#pragma unroll 1
    for (int seg = 0; seg < 2; ++seg) {
#pragma unroll 1
      for (int grp = 0; grp < GPS; ++grp) {
        if (++fgrp == GPS) {  // advance the stream: next group, segment (G -> S), row (down)
          fgrp = 0;
          if (++fseg == 2) {
            fseg = 0;
            frow -= blk;
            --frows;
          }
        }
        const double* nx = frows > 0 ? frow + (fseg ? s_off : 0) + fgrp * 8 * PF : nullptr;
        group_mma<MP, TM, TN, PF>(acc, buf, nx, (seg == 0 ? Xq : Xn) + cw0, LD, grp * PF, g, t);
      }
    }
    group_sync<WR, WC>(wc);
    store_smem(acc, Xn, LD, r0, cw0, g, t);
    store_tile<TM, TN, FULL_ != 0>(acc, a.X + gr * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
    if constexpr (NY > 1) cp_async_wait<NY - 2>();
    group_sync<WR, WC>(wc);
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// TMA-streamed sweeps for small blocks (MP <= 32, the memory-bound regime).
// One CTA per (range, KC = 16*NW columns), warp w owns columns [16w, 16w+16).
// Per row a ring stage holds the range's factor blocks (copied ONCE per CTA and
// shared by all warps) and the row's F (fwd) / y (bwd) tile, moved by
// cp.async.bulk (TMA) and completed on an mbarrier; NSTG rows are in flight.
template <int MP, int NW, int NSTG>
struct StreamCfg {
  static constexpr int KC = 16 * NW, LDT = KC + 2;
  static constexpr int NT = 32 * (NW + 1);  // NW consumer warps + 1 producer warp
  static constexpr int TM = MP / 8, TN = 2, NSP = MP / 8;
  static constexpr int BLK = MP * MP;
  static constexpr int TILE = MP * LDT;
  static constexpr int FWD_STAGE = TILE + 3 * BLK;  // F tile + AD, Tb, Dinv
  static constexpr int BWD_STAGE = TILE + 2 * BLK;  // y tile + G, S
  static constexpr size_t FWD_SMEM = (size_t)(TILE + NSTG * FWD_STAGE) * 8 + 2 * NSTG * 8;
  static constexpr size_t BWD_SMEM = (size_t)(2 * TILE + NSTG * BWD_STAGE) * 8 + 2 * NSTG * 8;
};

// acc += A(smem block, warp-all rows) @ B(smem tile, cols c0..c0+15)
template <int MP, int TM, int TN>
BTD_DEVINL void smem_mma(double (&acc)[TM][TN][2], const double* __restrict__ A, const double* __restrict__ B,
                         int ldb, int c0, int g, int t) {
#pragma unroll
  for (int s = 0; s < MP / 8; ++s) {
    double2 a[TM];
    double b0[TN], b1[TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) a[i] = *reinterpret_cast<const double2*>(&A[(i * 8 + g) * MP + 8 * s + 2 * t]);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      b0[j] = B[(8 * s + 2 * t) * ldb + c0 + j * 8 + g];
      b1[j] = B[(8 * s + 2 * t + 1) * ldb + c0 + j * 8 + g];
    }
    mma_k4<TM, TN, false>(acc, a, b0);
    mma_k4<TM, TN, true>(acc, a, b1);
  }
}

// issue one tile (rows < m, cols c0 .. c0+ncols of a row-major [*, K] array) as m row copies
BTD_DEVINL unsigned issue_tile(double* dst, int ldt, const double* src, int64_t K, int m, int ncols, uint64_t* bar,
                               int lane) {
  const unsigned rb = (unsigned)ncols * 8u;
  for (int r = lane; r < m; r += 32) bulk_g2s(dst + r * ldt, src + (int64_t)r * K, rb, bar);
  return rb * (unsigned)m;
}

// Warp-specialised streamed sweeps.  Warps split the CTA's columns, so a
// consumer warp's slice of the chain state (y / x) depends on its own columns
// only: no CTA barrier per row.  The producer warp refills ring slot s with row
// r once every consumer warp has released it (empty[s], count NW).
template <int MP, int NW, int NSTG>
__global__ void __launch_bounds__(32 * (NW + 1)) stream_fwd_kernel(ChainArgs a) {
  using C = StreamCfg<MP, NW, NSTG>;
  constexpr int TM = C::TM, TN = C::TN, LDT = C::LDT;
  extern __shared__ __align__(16) double sm[];
  double* Ys = sm;
  double* stg = sm + C::TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + NSTG * C::FWD_STAGE);
  uint64_t* empty = full + NSTG;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int q = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * C::KC;
  const int64_t K = a.K;
  const int ncols = (int)(K - c0 < C::KC ? K - c0 : C::KC);
  for (int e = tid; e < C::TILE + NSTG * C::FWD_STAGE; e += C::NT) sm[e] = 0.0;
  if (tid == 0) {
    for (int i = 0; i < NSTG; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t lo = a.lo[q];
  const int nint = a.nint[q];
  const int64_t slot0 = a.slot0[q];
  const int64_t rowK = (int64_t)a.m * K;
  constexpr int64_t blk = C::BLK;

  if (warp == NW) {  // ---- producer
    for (int j = 0; j < nint; ++j) {
      const int sl = j % NSTG;
      if (j >= NSTG) mbar_wait(&empty[sl], (unsigned)(((j / NSTG) - 1) & 1));
      double* st = stg + sl * C::FWD_STAGE;
      fence_proxy_async();
      if (lane == 0) mbar_expect_tx(&full[sl], (unsigned)(a.m * ncols * 8) + 3u * blk * 8u);
      __syncwarp();
      issue_tile(st, LDT, a.F + (lo + 1 + j) * rowK + c0, K, a.m, ncols, &full[sl], lane);
      if (lane == 0) {
        const int64_t s_ = slot0 + j;
        bulk_g2s(st + C::TILE, a.AD + s_ * blk, blk * 8, &full[sl]);
        bulk_g2s(st + C::TILE + blk, a.Tb + (j > 0 ? s_ - 1 : s_) * blk, blk * 8, &full[sl]);
        bulk_g2s(st + C::TILE + 2 * blk, a.Dinv + s_ * blk, blk * 8, &full[sl]);
      }
    }
    return;
  }
  // ---- consumers: warp owns columns [cw, cw+16) of the CTA tile
  const int cw = warp * 16;
  const bool vec = (K % 2) == 0;
  double ser[TM][TN][2];
  if (lo < a.n)
    load_tile(ser, a.F + lo * rowK, K, 0, c0 + cw, a.m, g, t, vec);
  else
    zero_acc(ser);
  double acc[TM][TN][2];
  for (int j = 0; j < nint; ++j) {
    const int sl = j % NSTG;
    const double* st = stg + sl * C::FWD_STAGE;
    mbar_wait(&full[sl], (unsigned)((j / NSTG) & 1));
    zero_acc(acc);
    smem_mma<MP, TM, TN>(acc, st + C::TILE + 2 * blk, st, LDT, cw, g, t);  // Dinv_j f_g
    smem_mma<MP, TM, TN>(acc, st + C::TILE, Ys, LDT, cw, g, t);            // AD_j y_{j-1}
    smem_mma<MP, TM, TN>(ser, st + C::TILE + blk, Ys, LDT, cw, g, t);      // Tb_{j-1} y_{j-1}
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sl]);
    store_smem(acc, Ys, LDT, 0, cw, g, t);
    store_tile(acc, a.X + (lo + 1 + j) * rowK, K, 0, c0 + cw, a.m, g, t, vec);
    __syncwarp();
  }
  if (nint > 0) wgemm<MP, TM, TN, 2>(ser, a.Tb + (slot0 + nint - 1) * blk, Ys + cw, LDT, g, t);
  store_tile(ser, a.base + (int64_t)q * a.base_stride, K, 0, c0 + cw, MP, g, t, vec);
}

template <int MP, int NW, int NSTG>
__global__ void __launch_bounds__(32 * (NW + 1)) stream_bwd_kernel(ChainArgs a) {
  using C = StreamCfg<MP, NW, NSTG>;
  constexpr int TM = C::TM, TN = C::TN, LDT = C::LDT;
  extern __shared__ __align__(16) double sm[];
  double* Xq = sm;
  double* Xn = sm + C::TILE;
  double* stg = sm + 2 * C::TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + NSTG * C::BWD_STAGE);
  uint64_t* empty = full + NSTG;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int q = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * C::KC;
  const int64_t K = a.K;
  const int ncols = (int)(K - c0 < C::KC ? K - c0 : C::KC);
  const bool vec = (K % 2) == 0;
  for (int e = tid; e < 2 * C::TILE + NSTG * C::BWD_STAGE; e += C::NT) sm[e] = 0.0;
  if (tid == 0) {
    for (int i = 0; i < NSTG; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t lo = a.lo[q];
  const int nint = a.nint[q];
  const int64_t slot0 = a.slot0[q];
  const int64_t rowK = (int64_t)a.m * K;
  const int64_t xtK = (int64_t)MP * K;
  constexpr int64_t blk = C::BLK;
  // x~_q, x~_{q+1} tiles (MP rows of the [nr+1][MP][K] buffer)
  for (int e = tid; e < MP * ncols; e += C::NT) {
    const int r = e / ncols, c = e % ncols;
    Xq[r * LDT + c] = a.xt[(int64_t)q * xtK + (int64_t)r * K + c0 + c];
    Xn[r * LDT + c] = a.xt[(int64_t)(q + 1) * xtK + (int64_t)r * K + c0 + c];
  }
  __syncthreads();
  if (warp == NW) {  // ---- producer: step jj handles row j = nint-1-jj
    for (int jj = 0; jj < nint; ++jj) {
      const int j = nint - 1 - jj;
      const int sl = jj % NSTG;
      if (jj >= NSTG) mbar_wait(&empty[sl], (unsigned)(((jj / NSTG) - 1) & 1));
      double* st = stg + sl * C::BWD_STAGE;
      fence_proxy_async();
      if (lane == 0) mbar_expect_tx(&full[sl], (unsigned)(a.m * ncols * 8) + 2u * blk * 8u);
      __syncwarp();
      issue_tile(st, LDT, a.X + (lo + 1 + j) * rowK + c0, K, a.m, ncols, &full[sl], lane);
      if (lane == 0) {
        const int64_t s_ = slot0 + j;
        bulk_g2s(st + C::TILE, a.G + s_ * blk, blk * 8, &full[sl]);
        bulk_g2s(st + C::TILE + blk, a.S + s_ * blk, blk * 8, &full[sl]);
      }
    }
    return;
  }
  const int cw = warp * 16;
  if (lo < a.n) {  // x[lo] = x~_q  (ref dichotomy.py:351)
    double xq[TM][TN][2];
    load_tile(xq, a.xt + (int64_t)q * xtK, K, 0, c0 + cw, MP, g, t, vec);
    store_tile(xq, a.X + lo * rowK, K, 0, c0 + cw, a.m, g, t, vec);
  }
  for (int jj = 0; jj < nint; ++jj) {
    const int j = nint - 1 - jj;
    const int sl = jj % NSTG;
    const double* st = stg + sl * C::BWD_STAGE;
    mbar_wait(&full[sl], (unsigned)((jj / NSTG) & 1));
    double acc[TM][TN][2];
    load_smem(acc, st, LDT, 0, cw, g, t);                                 // y_j
    smem_mma<MP, TM, TN>(acc, st + C::TILE, Xq, LDT, cw, g, t);        // + G_j x~_q
    smem_mma<MP, TM, TN>(acc, st + C::TILE + blk, Xn, LDT, cw, g, t);  // + S_j x_{j+1}
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sl]);
    store_smem(acc, Xn, LDT, 0, cw, g, t);
    store_tile(acc, a.X + (lo + 1 + j) * rowK, K, 0, c0 + cw, a.m, g, t, vec);
    __syncwarp();
  }
}

}  // namespace btd
