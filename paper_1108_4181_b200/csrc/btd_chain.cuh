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
  double* base;          // fwd out: [nr][MP][K]
  const double* xt;      // bwd in:  [nr+1][MP][K]
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
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          dmma(acc[i][j][0], acc[i][j][1], a[i].x, b0[j]);
          dmma(acc[i][j][0], acc[i][j][1], a[i].y, b1[j]);
        }
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
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          dmma(acc1[i][j][0], acc1[i][j][1], a1[i].x, b0[j]);
          dmma(acc1[i][j][0], acc1[i][j][1], a1[i].y, b1[j]);
          dmma(acc2[i][j][0], acc2[i][j][1], a2[i].x, b0[j]);
          dmma(acc2[i][j][0], acc2[i][j][1], a2[i].y, b1[j]);
        }
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
template <int TM, int TN>
BTD_DEVINL void load_tile(double (&acc)[TM][TN][2], const double* __restrict__ P, int64_t K,
                          int r0, int64_t c0, int rmax, int g, int t, bool vec) {
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

template <int TM, int TN>
BTD_DEVINL void store_tile(const double (&acc)[TM][TN][2], double* __restrict__ P, int64_t K,
                           int r0, int64_t c0, int rmax, int g, int t, bool vec) {
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

template <int MP, int KT, int WR, int WC>
struct ChainCfg {
  static constexpr int NW = WR * WC, NT = 32 * NW;
  static constexpr int RW = MP / WR, CW = KT / WC;
  static constexpr int TM = RW / 8, TN = CW / 8;
  static constexpr int LD = KT + 2;  // == 2 (mod 16) when KT % 16 == 0
  static constexpr int PF = MP >= 128 ? 2 : (MP >= 32 ? 2 : 1);
  static_assert(RW % 8 == 0 && CW % 8 == 0, "warp tile must be a multiple of 8x8");
};

template <int MP, int KT, int WR, int WC>
__global__ void __launch_bounds__(32 * WR * WC) chain_fwd_kernel(ChainArgs a) {
  using Cfg = ChainCfg<MP, KT, WR, WC>;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, LD = Cfg::LD, NT = Cfg::NT, PF = Cfg::PF;
  extern __shared__ __align__(16) double sm[];
  double* Ys = sm;
  double* Fs0 = sm + MP * LD;
  double* Fs1 = Fs0 + MP * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int r0 = wr * Cfg::RW, cw0 = wc * Cfg::CW;
  const int q = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * KT;
  const int64_t K = a.K;
  const bool vec = (K % 2) == 0;
  for (int e = tid; e < 3 * MP * LD; e += NT) sm[e] = 0.0;
  __syncthreads();

  const int64_t lo = a.lo[q];
  const int nint = a.nint[q];
  const int64_t slot0 = a.slot0[q];
  const int64_t blk = (int64_t)MP * MP;
  const int64_t rowK = (int64_t)a.m * K;  // elements per block row of F/X

  double ser[TM][TN][2];
  if (lo < a.n)
    load_tile(ser, a.F + lo * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
  else
    zero_acc(ser);

  if (nint > 0) {
    cp_tile<MP, KT, LD, NT>(Fs0, a.F + (lo + 1) * rowK, K, c0, a.m, vec);
    cp_async_wait_all();
  }
  __syncthreads();
  for (int j = 0; j < nint; ++j) {
    const int64_t gr = lo + 1 + j;
    double* Fcur = (j & 1) ? Fs1 : Fs0;
    double* Fnxt = (j & 1) ? Fs0 : Fs1;
    if (j + 1 < nint) cp_tile<MP, KT, LD, NT>(Fnxt, a.F + (gr + 1) * rowK, K, c0, a.m, vec);
    double acc[TM][TN][2];
    zero_acc(acc);
    const int64_t sl = slot0 + j;
    wgemm<MP, TM, TN, PF>(acc, a.Dinv + sl * blk + r0 * MP, Fcur + cw0, LD, g, t);
    if (j > 0)
      wgemm2<MP, TM, TN, PF>(acc, a.AD + sl * blk + r0 * MP, ser, a.Tb + (sl - 1) * blk + r0 * MP,
                             Ys + cw0, LD, g, t);
    __syncthreads();
    store_smem(acc, Ys, LD, r0, cw0, g, t);
    store_tile(acc, a.X + gr * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
    cp_async_wait_all();
    __syncthreads();
  }
  if (nint > 0)
    wgemm<MP, TM, TN, PF>(ser, a.Tb + (slot0 + nint - 1) * blk + r0 * MP, Ys + cw0, LD, g, t);
  store_tile(ser, a.base + (int64_t)q * MP * K, K, r0, c0 + cw0, MP, g, t, vec);
}

template <int MP, int KT, int WR, int WC>
__global__ void __launch_bounds__(32 * WR * WC) chain_bwd_kernel(ChainArgs a) {
  using Cfg = ChainCfg<MP, KT, WR, WC>;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, LD = Cfg::LD, NT = Cfg::NT, PF = Cfg::PF;
  extern __shared__ __align__(16) double sm[];
  double* Xq = sm;
  double* Xn = sm + MP * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int r0 = wr * Cfg::RW, cw0 = wc * Cfg::CW;
  const int q = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * KT;
  const int64_t K = a.K;
  const bool vec = (K % 2) == 0;
  for (int e = tid; e < 2 * MP * LD; e += NT) sm[e] = 0.0;
  __syncthreads();

  const int64_t lo = a.lo[q];
  const int nint = a.nint[q];
  const int64_t slot0 = a.slot0[q];
  const int64_t blk = (int64_t)MP * MP;
  const int64_t rowK = (int64_t)a.m * K;
  const int64_t xtK = (int64_t)MP * K;

  cp_tile<MP, KT, LD, NT>(Xq, a.xt + (int64_t)q * xtK, K, c0, MP, vec);
  cp_tile<MP, KT, LD, NT>(Xn, a.xt + (int64_t)(q + 1) * xtK, K, c0, MP, vec);
  double y[TM][TN][2];
  if (nint > 0) load_tile(y, a.X + (lo + nint) * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
  if (lo < a.n) {  // x[lo] = x~_q  (ref dichotomy.py:351)
    double xq[TM][TN][2];
    load_tile(xq, a.xt + (int64_t)q * xtK, K, r0, c0 + cw0, MP, g, t, vec);
    store_tile(xq, a.X + lo * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int j = nint - 1; j >= 0; --j) {
    const int64_t gr = lo + 1 + j;
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int jj = 0; jj < TN; ++jj) { acc[i][jj][0] = y[i][jj][0]; acc[i][jj][1] = y[i][jj][1]; }
    if (j > 0) load_tile(y, a.X + (gr - 1) * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
    const int64_t sl = slot0 + j;
    wgemm<MP, TM, TN, PF>(acc, a.G + sl * blk + r0 * MP, Xq + cw0, LD, g, t);
    wgemm<MP, TM, TN, PF>(acc, a.S + sl * blk + r0 * MP, Xn + cw0, LD, g, t);
    __syncthreads();
    store_smem(acc, Xn, LD, r0, cw0, g, t);
    store_tile(acc, a.X + gr * rowK, K, r0, c0 + cw0, a.m, g, t, vec);
    __syncthreads();
  }
}

}  // namespace btd
