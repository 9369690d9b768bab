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
// Tiling (gemm_pipe_kernel): CTA tile BM x BN, warps WGM x WGN, BK = 16 k-slabs in
// a STAGES-deep cp.async ring (zero-filled edges).  A is stored [BM][24] (16B loads
// of (k,k+1) pairs, conflict-free LDS.128), B is [16][BN+2] (LDS.64, conflict-free).
#pragma once
#include <cuda.h>

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
  // segmented split-K: grid.z enumerates (entry, k-chunk) pairs; partial sums go to
  // partial + z*rows*cols and a fixed-order reduction finishes C (deterministic)
  const int32_t* split_b;
  const int32_t* split_k;
  int64_t kchunk;
  double* partial;
  int nsplit_total;
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

// cp.async with zero fill: copies `src_bytes` (0..size) and zero-fills the rest
BTD_DEVINL void cp_async16_z(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes));
}
BTD_DEVINL void cp_async8_z(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes));
}

// Pipelined variant: STAGES-deep cp.async ring of (A: BM x 16, B: 16 x BN) slabs,
// warps WGM x WGN with 32x32 (or 16x16) warp tiles, DMMA m8n8k4.
template <int BM, int BN, int WGM, int WGN, int STAGES>
struct PipeCfg {
  static constexpr int NT = 32 * WGM * WGN;
  static constexpr int BK = 16;
  static constexpr int LDA = 24;       // A row pitch (doubles): 12 double2 == 4 (mod 8)
  static constexpr int LDB = BN + 2;   // B row pitch: == 2 (mod 16)
  static constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static constexpr int TM = WTM / 8, TN = WTN / 8;
  static constexpr int A_ELEMS = BM * LDA, B_ELEMS = BK * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE * sizeof(double);
};

template <int BM, int BN, int WGM, int WGN, int STAGES>
__global__ void __launch_bounds__(32 * WGM * WGN) gemm_pipe_kernel(GemmDesc d) {
  using C_ = PipeCfg<BM, BN, WGM, WGN, STAGES>;
  constexpr int NT = C_::NT, BK = C_::BK, LDA = C_::LDA, LDB = C_::LDB, TM = C_::TM, TN = C_::TN;
  extern __shared__ __align__(16) double smp[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / WGN, wn = warp % WGN;
  const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;

  const int nz = d.split_b ? d.nsplit_total : d.nbatch;
  for (int zz = blockIdx.z; zz < nz; zz += gridDim.z) {
    const int b = d.split_b ? d.split_b[zz] : zz;
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
      int64_t K = tm_.k_arr ? tm_.k_arr[b] : tm_.k;
      const double alpha = tm_.alpha;
      if (d.split_b) {  // this CTA's k-chunk: shift the operands, clip K
        const int64_t k0 = (int64_t)d.split_k[zz] * d.kchunk;
        A += k0;
        B += k0 * ldb;
        K = K - k0 < d.kchunk ? K - k0 : d.kchunk;
      }
      if (K <= 0) continue;
      const bool va = ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
      const bool vb = ((ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
      const int nk = (int)((K + BK - 1) / BK);
      auto load = [&](int kt, int slot) {
        double* As = smp + slot * C_::STAGE;
        double* Bs = As + C_::A_ELEMS;
        const int64_t k0 = (int64_t)kt * BK;
        // A: BM rows x 16 k  (8 chunks of 2 doubles per row)
        for (int e = tid; e < BM * 8; e += NT) {
          const int r = e >> 3, ch = (e & 7) * 2;
          const int64_t gr = row0 + r, gk = k0 + ch;
          double* dst = As + r * LDA + ch;
          const int64_t rem = (gr < d.rows) ? K - gk : 0;
          const double* src = (rem > 0) ? A + gr * lda + gk : A;
          if (va) {
            cp_async16_z(dst, src, rem >= 2 ? 16 : (rem == 1 ? 8 : 0));
          } else {
            cp_async8_z(dst, src, rem >= 1 ? 8 : 0);
            cp_async8_z(dst + 1, rem >= 2 ? src + 1 : src, rem >= 2 ? 8 : 0);
          }
        }
        // B: 16 k x BN cols
        for (int e = tid; e < BK * (BN / 2); e += NT) {
          const int kk = e / (BN / 2), ch = (e % (BN / 2)) * 2;
          const int64_t gk = k0 + kk, gc = col0 + ch;
          double* dst = Bs + kk * LDB + ch;
          const int64_t rem = (gk < K) ? d.cols - gc : 0;
          const double* src = (rem > 0) ? B + gk * ldb + gc : B;
          if (vb) {
            cp_async16_z(dst, src, rem >= 2 ? 16 : (rem == 1 ? 8 : 0));
          } else {
            cp_async8_z(dst, src, rem >= 1 ? 8 : 0);
            cp_async8_z(dst + 1, rem >= 2 ? src + 1 : src, rem >= 2 ? 8 : 0);
          }
        }
      };
#pragma unroll
      for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load(s, s);
        cp_async_commit();
      }
      for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (kt + STAGES - 1 < nk) load(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
        cp_async_commit();
        const double* As = smp + (kt % STAGES) * C_::STAGE;
        const double* Bs = As + C_::A_ELEMS;
#pragma unroll
        for (int s = 0; s < BK / 8; ++s) {
          double2 a[TM];
          double b0[TN], b1[TN];
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            a[i] = *reinterpret_cast<const double2*>(&As[(wm * C_::WTM + i * 8 + g) * LDA + 8 * s + 2 * t]);
            if (alpha != 1.0) { a[i].x *= alpha; a[i].y *= alpha; }
          }
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            b0[j] = Bs[(8 * s + 2 * t) * LDB + wn * C_::WTN + j * 8 + g];
            b1[j] = Bs[(8 * s + 2 * t + 1) * LDB + wn * C_::WTN + j * 8 + g];
          }
          mma_k4<TM, TN, false>(acc, a, b0);
          mma_k4<TM, TN, true>(acc, a, b1);
        }
      }
      cp_async_wait<0>();
      __syncthreads();
    }
    double* C = d.split_b ? d.partial + (int64_t)zz * d.rows * d.cols : const_cast<double*>(opnd_ptr(d.C, b));
    const int64_t ldc = d.split_b ? d.cols : opnd_ld(d.C, b);
    const double* Ci = (!d.split_b && d.Cin.base) ? opnd_ptr(d.Cin, b) : nullptr;
    const int64_t ldci = Ci ? opnd_ld(d.Cin, b) : 0;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int64_t r = row0 + wm * C_::WTM + i * 8 + g;
          const int64_t c = col0 + wn * C_::WTN + j * 8 + 2 * t + v;
          if (r < d.rows && c < d.cols) {
            double val = acc[i][j][v];
            if (Ci) val += d.beta * Ci[r * ldci + c];
            C[r * ldc + c] = val;
          }
        }
  }
}

// Warp-specialised variant for large aligned products (the mode-1 sweep steps of
// M = 2048, c3): one producer warp moves each (A: BM x 32, B: 32 x BN) k-slab with
// cp.async.bulk (TMA, one bulk copy per row segment) into an NSTG-deep smem ring
// completed on mbarriers; WGM x WGN consumer warps run DMMA on ready stages and
// release them with an arrive -- no CTA-wide barrier in the main loop, and the
// producer runs ahead across terms and batch entries.  Requires: rows % BM ==
// cols % BN == 0, every K (and split chunk) % 32 == 0, even row strides and
// 16-byte aligned operand rows (checked on the host: ws_eligible).
template <int BM, int BN, int WGM, int WGN, int NSTG>
struct WsCfg {
  static constexpr int NWC = WGM * WGN, NT = 32 * (NWC + 1);
  static constexpr int BK = 32;
  static constexpr int LDA = BK + 8;   // 320 B rows: fragment LDS.128 conflict-free, 16B-aligned bulk dst
  static constexpr int LDB = BN + 2;   // == 2 (mod 16) doubles, 16B-aligned rows when BN % 16 == 14.. (BN=64: 528 B)
  static constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static constexpr int TM = WTM / 8, TN = WTN / 8;
  static constexpr int A_ELEMS = BM * LDA, B_ELEMS = BK * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr unsigned TX = (unsigned)(BM + BN) * BK * 8u;
  static constexpr size_t SMEM = (size_t)NSTG * STAGE * sizeof(double) + 2 * NSTG * sizeof(uint64_t);
  static_assert((LDB * 8) % 16 == 0 && (STAGE * 8) % 16 == 0, "bulk-copy destinations must be 16B aligned");
};

template <int BM, int BN, int WGM, int WGN, int NSTG>
__global__ void __launch_bounds__(32 * (WGM * WGN + 1), 1) gemm_ws_kernel(GemmDesc d) {
  using C_ = WsCfg<BM, BN, WGM, WGN, NSTG>;
  constexpr int BK = C_::BK, LDA = C_::LDA, LDB = C_::LDB, TM = C_::TM, TN = C_::TN, NWC = C_::NWC;
  extern __shared__ __align__(16) double smw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smw + NSTG * C_::STAGE);
  uint64_t* empty = full + NSTG;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;
  if (tid == 0) {
    for (int i = 0; i < NSTG; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NWC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int nz = d.split_b ? d.nsplit_total : d.nbatch;

  if (warp == NWC) {  // ---- producer warp
    int it = 0;
    for (int zz = blockIdx.z; zz < nz; zz += gridDim.z) {
      const int b = d.split_b ? d.split_b[zz] : zz;
      for (int ti = 0; ti < d.nterms; ++ti) {
        const Term& tm_ = d.t[ti];
        const double* A = opnd_ptr(tm_.A, b);
        const double* B = opnd_ptr(tm_.B, b);
        const int64_t lda = tm_.A.ld, ldb = tm_.B.ld;
        int64_t K = tm_.k_arr ? tm_.k_arr[b] : tm_.k;
        if (d.split_b) {
          const int64_t k0 = (int64_t)d.split_k[zz] * d.kchunk;
          A += k0;
          B += k0 * ldb;
          K = K - k0 < d.kchunk ? K - k0 : d.kchunk;
        }
        const int nk = K > 0 ? (int)(K / BK) : 0;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int sl = it % NSTG;
          if (it >= NSTG) mbar_wait(&empty[sl], (unsigned)(((it / NSTG) - 1) & 1));
          double* As = smw + sl * C_::STAGE;
          double* Bs = As + C_::A_ELEMS;
          fence_proxy_async();
          if (lane == 0) mbar_expect_tx(&full[sl], C_::TX);
          __syncwarp();
          const double* Ak = A + row0 * lda + (int64_t)kt * BK;
          for (int r = lane; r < BM; r += 32) bulk_g2s(As + r * LDA, Ak + r * lda, BK * 8, &full[sl]);
          const double* Bk = B + ((int64_t)kt * BK) * ldb + col0;
          for (int r = lane; r < BK; r += 32) bulk_g2s(Bs + r * LDB, Bk + r * ldb, BN * 8, &full[sl]);
        }
      }
    }
    return;
  }
  // ---- consumer warps
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / WGN, wn = warp % WGN;
  int it = 0;
  for (int zz = blockIdx.z; zz < nz; zz += gridDim.z) {
    const int b = d.split_b ? d.split_b[zz] : zz;
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int ti = 0; ti < d.nterms; ++ti) {
      const Term& tm_ = d.t[ti];
      int64_t K = tm_.k_arr ? tm_.k_arr[b] : tm_.k;
      if (d.split_b) {
        const int64_t k0 = (int64_t)d.split_k[zz] * d.kchunk;
        K = K - k0 < d.kchunk ? K - k0 : d.kchunk;
      }
      const int nk = K > 0 ? (int)(K / BK) : 0;
      const bool neg = tm_.alpha != 1.0;
      const double alpha = tm_.alpha;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const int sl = it % NSTG;
        mbar_wait(&full[sl], (unsigned)((it / NSTG) & 1));
        const double* As = smw + sl * C_::STAGE;
        const double* Bs = As + C_::A_ELEMS;
#pragma unroll
        for (int s = 0; s < BK / 8; ++s) {
          double2 a[TM];
          double b0[TN], b1[TN];
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            a[i] = *reinterpret_cast<const double2*>(&As[(wm * C_::WTM + i * 8 + g) * LDA + 8 * s + 2 * t]);
            if (neg) { a[i].x *= alpha; a[i].y *= alpha; }
          }
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            b0[j] = Bs[(8 * s + 2 * t) * LDB + wn * C_::WTN + j * 8 + g];
            b1[j] = Bs[(8 * s + 2 * t + 1) * LDB + wn * C_::WTN + j * 8 + g];
          }
          mma_k4<TM, TN, false>(acc, a, b0);
          mma_k4<TM, TN, true>(acc, a, b1);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sl]);
      }
    }
    double* C = d.split_b ? d.partial + (int64_t)zz * d.rows * d.cols : const_cast<double*>(opnd_ptr(d.C, b));
    const int64_t ldc = d.split_b ? d.cols : opnd_ld(d.C, b);
    const double* Ci = (!d.split_b && d.Cin.base) ? opnd_ptr(d.Cin, b) : nullptr;
    const int64_t ldci = Ci ? opnd_ld(d.Cin, b) : 0;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t r = row0 + wm * C_::WTM + i * 8 + g;
        const int64_t c = col0 + wn * C_::WTN + j * 8 + 2 * t;
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (Ci) {
          const double2 ci = *reinterpret_cast<const double2*>(Ci + r * ldci + c);
          v.x += d.beta * ci.x;
          v.y += d.beta * ci.y;
        }
        *reinterpret_cast<double2*>(C + r * ldc + c) = v;
      }
  }
}

// TMA-2D variant (the one the large products use): the producer warp moves each
// k-slab with cp.async.bulk.tensor.2d through tensor maps over the operands'
// backing arrays (A: rows of the block pool / matrix, 128-byte boxes of 16 k-values;
// B: 128-byte boxes of 16 columns), 128-byte swizzled in shared memory, so a stage
// is 2 + BN/16 TMA instructions instead of BM + 32 row copies.  Consumers apply the
// swizzle (16-byte chunk c of row r lives at c ^ (r & 7)) in their fragment loads:
// LDS.128 A fragments and LDS.64 B fragments stay at the minimum wavefront count.
struct TmaOperands {
  CUtensorMap a[3], b[3];   // per term
  int64_t a_rpi[3], b_rpi[3];  // tensor rows per operand index unit (stride / ld)
};

template <int BM, int BN, int WGM, int WGN, int NSTG>
struct TmaCfg {
  static constexpr int NWC = WGM * WGN, NT = 32 * (NWC + 1);
  static constexpr int BK = 32;
  static constexpr int A_BOX = BM * 16, B_BOX = BK * 16;      // doubles per 128-byte-wide box
  static constexpr int A_ELEMS = 2 * A_BOX, B_ELEMS = (BN / 16) * B_BOX;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static constexpr int TM = WTM / 8, TN = WTN / 8;
  static constexpr unsigned TX = (unsigned)(BM + BN) * BK * 8u;
  static constexpr size_t SMEM = 1024 + (size_t)NSTG * STAGE * sizeof(double) + 2 * NSTG * sizeof(uint64_t);
  static_assert((A_BOX * 8) % 1024 == 0 && (B_BOX * 8) % 1024 == 0, "128B-swizzled boxes need 1 KB alignment");
  static_assert(WTN % 16 == 0, "B fragments assume 16-column-aligned warp tiles");
};

BTD_DEVINL void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

template <int BM, int BN, int WGM, int WGN, int NSTG>
__global__ void __launch_bounds__(32 * (WGM * WGN + 1), 1)
    gemm_tma_kernel(const __grid_constant__ TmaOperands ops, GemmDesc d) {
  using C_ = TmaCfg<BM, BN, WGM, WGN, NSTG>;
  constexpr int BK = C_::BK, TM = C_::TM, TN = C_::TN, NWC = C_::NWC;
  extern __shared__ __align__(16) double smt_raw[];
  double* smt = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smt_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smt + NSTG * C_::STAGE);
  uint64_t* empty = full + NSTG;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;
  if (tid == 0) {
    for (int i = 0; i < NSTG; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NWC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int nz = d.split_b ? d.nsplit_total : d.nbatch;

  if (warp == NWC) {  // ---- producer warp (one elected lane issues)
    if (lane == 0) {
      int it = 0;
      for (int zz = blockIdx.z; zz < nz; zz += gridDim.z) {
        const int b = d.split_b ? d.split_b[zz] : zz;
        for (int ti = 0; ti < d.nterms; ++ti) {
          const Term& tm_ = d.t[ti];
          const int64_t ai = (tm_.A.idx ? tm_.A.idx[b] : (int64_t)b) + tm_.A.add;
          const int64_t bi = (tm_.B.idx ? tm_.B.idx[b] : (int64_t)b) + tm_.B.add;
          int64_t K = tm_.k_arr ? tm_.k_arr[b] : tm_.k, k0 = 0;
          if (d.split_b) {
            k0 = (int64_t)d.split_k[zz] * d.kchunk;
            K = K - k0 < d.kchunk ? K - k0 : d.kchunk;
          }
          const int ya = (int)(ai * ops.a_rpi[ti] + row0);
          const int64_t yb0 = bi * ops.b_rpi[ti] + k0;
          const int nk = K > 0 ? (int)(K / BK) : 0;
          for (int kt = 0; kt < nk; ++kt, ++it) {
            const int sl = it % NSTG;
            if (it >= NSTG) mbar_wait(&empty[sl], (unsigned)(((it / NSTG) - 1) & 1));
            double* As = smt + sl * C_::STAGE;
            double* Bs = As + C_::A_ELEMS;
            fence_proxy_async();
            mbar_expect_tx(&full[sl], C_::TX);
            const int xk = (int)(k0 + (int64_t)kt * BK);
            tma_load_2d(As, &ops.a[ti], xk, ya, &full[sl]);
            tma_load_2d(As + C_::A_BOX, &ops.a[ti], xk + 16, ya, &full[sl]);
            const int yb = (int)(yb0 + (int64_t)kt * BK);
#pragma unroll
            for (int c = 0; c < BN / 16; ++c) tma_load_2d(Bs + c * C_::B_BOX, &ops.b[ti], (int)col0 + 16 * c, yb, &full[sl]);
          }
        }
      }
    }
    return;
  }
  // ---- consumer warps
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / WGN, wn = warp % WGN;
  int it = 0;
  for (int zz = blockIdx.z; zz < nz; zz += gridDim.z) {
    const int b = d.split_b ? d.split_b[zz] : zz;
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int ti = 0; ti < d.nterms; ++ti) {
      const Term& tm_ = d.t[ti];
      int64_t K = tm_.k_arr ? tm_.k_arr[b] : tm_.k;
      if (d.split_b) {
        const int64_t k0 = (int64_t)d.split_k[zz] * d.kchunk;
        K = K - k0 < d.kchunk ? K - k0 : d.kchunk;
      }
      const int nk = K > 0 ? (int)(K / BK) : 0;
      const bool neg = tm_.alpha != 1.0;
      const double alpha = tm_.alpha;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const int sl = it % NSTG;
        mbar_wait(&full[sl], (unsigned)((it / NSTG) & 1));
        const double* As = smt + sl * C_::STAGE;
        const double* Bs = As + C_::A_ELEMS;
#pragma unroll
        for (int s = 0; s < BK / 8; ++s) {
          // A(row, k = 8s + 2t .. +1): box s/2, 16B chunk (4s + t) % 8, swizzled ^ (row & 7) = ^ g
          const double* Ab = As + (s >> 1) * C_::A_BOX;
          const int ach = ((4 * s + t) & 7) ^ g;
          double2 a[TM];
          double b0[TN], b1[TN];
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            a[i] = *reinterpret_cast<const double2*>(Ab + (wm * C_::WTM + i * 8 + g) * 16 + ach * 2);
            if (neg) { a[i].x *= alpha; a[i].y *= alpha; }
          }
          // B(k, n): box n/16, row k (16 doubles), chunk (n % 16)/2 ^ (k & 7), element n % 2
          const int k_0 = 8 * s + 2 * t;
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            const int n = wn * C_::WTN + j * 8 + g;
            const double* Bb = Bs + (n >> 4) * C_::B_BOX;
            const int ch = (n & 15) >> 1, e = n & 1;
            b0[j] = Bb[k_0 * 16 + ((ch ^ (k_0 & 7)) << 1) + e];
            b1[j] = Bb[(k_0 + 1) * 16 + ((ch ^ ((k_0 + 1) & 7)) << 1) + e];
          }
          mma_k4<TM, TN, false>(acc, a, b0);
          mma_k4<TM, TN, true>(acc, a, b1);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sl]);
      }
    }
    double* C = d.split_b ? d.partial + (int64_t)zz * d.rows * d.cols : const_cast<double*>(opnd_ptr(d.C, b));
    const int64_t ldc = d.split_b ? d.cols : opnd_ld(d.C, b);
    const double* Ci = (!d.split_b && d.Cin.base) ? opnd_ptr(d.Cin, b) : nullptr;
    const int64_t ldci = Ci ? opnd_ld(d.Cin, b) : 0;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t r = row0 + wm * C_::WTM + i * 8 + g;
        const int64_t c = col0 + wn * C_::WTN + j * 8 + 2 * t;
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (Ci) {
          const double2 ci = *reinterpret_cast<const double2*>(Ci + r * ldci + c);
          v.x += d.beta * ci.x;
          v.y += d.beta * ci.y;
        }
        *reinterpret_cast<double2*>(C + r * ldc + c) = v;
      }
  }
}

// C_b = beta * Cin_b + sum_{z in [zoff_b, zoff_b + nz_b)} partial_z   (fixed order)
__global__ void splitk_reduce_kernel(const double* partial, const int32_t* zoff, const int32_t* zcnt, Opnd C, Opnd Cin,
                                     double beta, int64_t rows, int64_t cols, int nbatch) {
  const int64_t per = rows * cols;
  for (int b = blockIdx.y; b < nbatch; b += gridDim.y) {
    double* Cb = const_cast<double*>(opnd_ptr(C, b));
    const int64_t ldc = opnd_ld(C, b);
    const double* Ci = Cin.base ? opnd_ptr(Cin, b) : nullptr;
    const int64_t ldci = Ci ? opnd_ld(Cin, b) : 0;
    const double* P = partial + (int64_t)zoff[b] * per;
    const int n = zcnt[b];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = e / cols, c = e % cols;
      double v = 0.0;
      for (int z = 0; z < n; ++z) v += P[(int64_t)z * per + e];
      if (Ci) v += beta * Ci[r * ldci + c];
      Cb[r * ldc + c] = v;
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
