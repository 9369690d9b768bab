// Plan construction, solve orchestration and the C ABI (include/blocktri_b200.h).
//
// Algorithm 2 of arXiv 1108.4181 as implemented by the reference
// (/root/reference/pkg/src/blocktri/dichotomy.py), re-laid out for B200:
//
//  plan (once per matrix; ref dichotomy.py:318-338)
//    * the matrix is identity-padded to npad = P*L rows exactly as the
//      reference does (ref dichotomy.py:307-315, 328-330), so the device plan
//      has the reference's ranges, reduced system and partition tree;
//    * per range, a batched (over ranges) sweep over the L-1 interior rows:
//        D_j = C_g - A_g S_{j-1}           GEMM   (ref _kernels.pyx:163-168)
//        Dinv_j = D_j^{-1}                 Gauss-Jordan, reference pivot test
//        S_j = Dinv_j B_g, AD_j = Dinv_j A_g,
//        G_j = AD_j G_{j-1}  (left-boundary response, ref U of dichotomy.py:186-188)
//        Tb_j = B_lo S_0..S_{j-1}          (first-row transfer, gives B_lo W[1])
//      all in HBM: 5 blocks of mp x mp per interior row;
//    * reduced three-point system (ref dichotomy.py:212-236) from BU = B_lo U[1],
//      BV = B_lo V[1], G/S of the last interior row;
//    * inverse rows of every partition-tree node by transposed block sweeps
//      with unit right-hand sides (ref dichotomy.py:134-146, 298-304), then the
//      end corrections E = R[:, :M] A~, H = R[:, -M:] B~ of Algorithm 1.
//  solve (per K right-hand sides; ref dichotomy.py:358-390)
//    forward chain kernel -> interface RHS GEMM -> tree: z = R f~ (all nodes,
//    one launch) then one launch per tree level x~_k = z + E x~_{lo-1} +
//    H x~_{hi+1} -> backward chain kernel.  Block orders above 256 run the
//    sweeps as one batched GEMM launch per row step instead (mode 1).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "blocktri_b200.h"
#include "btd_chain.cuh"
#include "btd_gemm.cuh"
#include "btd_inv.cuh"
#include "btd_gjc.cuh"
#include "btd_band.cuh"
#include "btd_tree.cuh"

using namespace btd;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

struct BtdError {
  int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
  g_err = msg;
  throw BtdError{code};
}

void ck(cudaError_t e, const char* what, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %s (%s) at btd_api.cu:%d: %s", cudaGetErrorName(e),
             cudaGetErrorString(e), line, what);
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? BTD_ERR_OOM : BTD_ERR_CUDA, buf);
  }
}
#define CK(x) ck((x), #x, __LINE__)
#define CK_LAUNCH()                                   \
  do {                                                \
    g_launches.fetch_add(1, std::memory_order_relaxed); \
    ck(cudaGetLastError(), "kernel launch", __LINE__); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t b) {
    release();
    if (b == 0) b = 16;
    CK(cudaMalloc(&p, b));
    bytes = b;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  double* d() const { return static_cast<double*>(p); }
  int64_t* i64() const { return static_cast<int64_t*>(p); }
  int32_t* i32() const { return static_cast<int32_t*>(p); }
};

// Scalar-coupling probe: slot s = (range q, interior row j) -> is the row's lower block a I
// (exactly)?  alpha[s] = a; *bad set when any live slot's block is not.
__global__ void scalar_coupling_kernel(const double* Lw, const int64_t* lo, const int32_t* nint, int64_t cap, int mp,
                                       double* alpha, int* bad) {
  const int64_t s = blockIdx.x, q = s / cap, j = s % cap;
  if (j >= nint[q]) {
    if (threadIdx.x == 0) alpha[s] = 0.0;
    return;
  }
  const double* B = Lw + (lo[q] + j) * (int64_t)mp * mp;
  const double d = B[0];
  bool ok = true;
  for (int e = threadIdx.x; e < mp * mp; e += blockDim.x) {
    const double v = B[e];
    if (e / mp == e % mp ? !(v == d) : !(v == 0.0)) ok = false;
  }
  if (!ok) *bad = 1;
  if (threadIdx.x == 0) alpha[s] = d;
}

__global__ void pad_blocks_kernel(const double* src, int64_t nsrc, int m, double* dst, int64_t ndst,
                                  int mp, int diag_identity) {
  const int64_t total = ndst * mp * mp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / ((int64_t)mp * mp);
    const int r = (int)((e / mp) % mp), c = (int)(e % mp);
    double v;
    if (b < nsrc && r < m && c < m)
      v = src[(b * m + r) * m + c];
    else
      v = (diag_identity && r == c && (b >= nsrc || r >= m)) ? 1.0 : 0.0;
    dst[e] = v;
  }
}

__global__ void set_identity_kernel(double* dst, int mp) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < mp * mp; e += gridDim.x * blockDim.x)
    dst[e] = (e / mp == e % mp) ? 1.0 : 0.0;
}

// R_node[a][i*mp + c] = Y_i[c][a]  (ref dichotomy.py:145: y.transpose(2,0,1))
__global__ void assemble_rows_kernel(const double* Y, const int64_t* ynb0, const int64_t* roff, const int64_t* ld,
                                     const int64_t* size, const int64_t* eoff, int nnodes,
                                     int64_t total, int mp, double* R) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nnodes - 1;  // node with eoff[b] <= e < eoff[b+1]
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (eoff[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int64_t le = e - eoff[b];
    const int64_t s = size[b];
    const int64_t a = le / (s * mp), rest = le % (s * mp);
    const int64_t i = rest / mp, c = rest % mp;
    R[roff[b] + a * ld[b] + i * mp + c] = Y[(ynb0[b] + i) * (int64_t)mp * mp + c * mp + a];
  }
}

// row-major D (mp x mp) -> col-major copy of D (i.e. row-major D^T)

// cudaFuncSetAttribute is per device: remember which (kernel, device) pairs were set.
void set_smem_attr(const void* fn, size_t smem) {
  if (smem <= 48 * 1024) return;
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first == fn && d.second == dev) return;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  done.push_back({fn, dev});
}

Opnd mk(const double* base, const int64_t* idx, int64_t add, int64_t stride, int64_t ld,
        const int64_t* ld_arr = nullptr) {
  Opnd o;
  o.base = base;
  o.idx = idx;
  o.add = add;
  o.stride = stride;
  o.ld = ld;
  o.ld_arr = ld_arr;
  return o;
}
Opnd none() { return mk(nullptr, nullptr, 0, 0, 0); }
Term term(Opnd A, Opnd B, int64_t k, double alpha = 1.0, const int64_t* k_arr = nullptr) {
  Term t;
  t.A = A;
  t.B = B;
  t.k = k;
  t.k_arr = k_arr;
  t.alpha = alpha;
  return t;
}

// Segmented split-K maps for one batched GEMM (built at plan time).
struct SplitK {
  int ntotal = 0;
  int64_t kchunk = 0;
  const int32_t *sb = nullptr, *sk = nullptr, *zoff = nullptr, *zcnt = nullptr;
  double* partial = nullptr;
};

// Tensor maps for the TMA-2D GEMM: each operand's backing array seen as a 2-D
// [rows][ld] tensor (rows = index * stride / ld + row), 128-byte boxes, 128B swizzle.
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      fail(BTD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool encode_operand(CUtensorMap* map, const Opnd& o, int box_rows, int64_t* rpi) {
  if (o.ld < 16 || o.stride % o.ld) return false;
  *rpi = o.stride / o.ld;
  const cuuint64_t dims[2] = {(cuuint64_t)o.ld, (cuuint64_t)1 << 30};
  const cuuint64_t strides[1] = {(cuuint64_t)o.ld * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(o.base), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tma_operands(const GemmDesc& d, int bm, int bk, TmaOperands& ops) {
  for (int i = 0; i < d.nterms; ++i) {
    if (!encode_operand(&ops.a[i], d.t[i].A, bm, &ops.a_rpi[i])) return false;
    if (!encode_operand(&ops.b[i], d.t[i].B, bk, &ops.b_rpi[i])) return false;
    // int32 tensor coordinates: the rows any entry can reach stay below 2^30
  }
  return true;
}

// The warp-specialised TMA GEMM needs whole tiles, 32-multiple reductions, even
// row strides and 16-byte aligned rows for every operand (bulk copies, double2 epilogue).
bool ws_eligible(const GemmDesc& d, int bn) {
  if (d.rows % 128 || d.cols % bn) return false;
  auto ok = [](const Opnd& o) {
    return o.base && !o.ld_arr && (o.ld % 2) == 0 && (o.stride % 2) == 0 &&
           (reinterpret_cast<uintptr_t>(o.base) % 16) == 0;
  };
  for (int i = 0; i < d.nterms; ++i) {
    const Term& t = d.t[i];
    // with k_arr, t.k is a divisor of every per-entry reduction length (its granularity)
    if (t.k <= 0 || t.k % 32 || !ok(t.A) || !ok(t.B)) return false;
  }
  if (d.split_b) {
    if (d.kchunk % 32) return false;
  } else if (!ok(d.C) || (d.Cin.base && !ok(d.Cin))) {
    return false;
  }
  return true;
}

void launch_gemm(int64_t rows, int64_t cols, int nbatch, Opnd C, Opnd Cin, double beta,
                 std::initializer_list<Term> terms, cudaStream_t st, const SplitK* sp = nullptr) {
  if (nbatch <= 0 || rows <= 0 || cols <= 0) return;
  GemmDesc d;
  memset(&d, 0, sizeof d);
  if (sp && sp->ntotal > 0) {
    d.split_b = sp->sb;
    d.split_k = sp->sk;
    d.kchunk = sp->kchunk;
    d.partial = sp->partial;
    d.nsplit_total = sp->ntotal;
  }
  d.rows = rows;
  d.cols = cols;
  d.nbatch = nbatch;
  d.C = C;
  d.Cin = Cin;
  d.beta = beta;
  d.nterms = 0;
  for (const Term& t : terms) d.t[d.nterms++] = t;
  const int gz = std::min(d.split_b ? d.nsplit_total : nbatch, 65535);
  auto tiles = [&](int64_t bm, int64_t bn) { return ((rows + bm - 1) / bm) * ((cols + bn - 1) / bn) * gz; };
  static int ws_env = -1;
  if (ws_env < 0) {
    const char* e = getenv("BTD_GEMM_WS");
    ws_env = e ? atoi(e) : 1;
  }
  TmaOperands ops;
  if (ws_env == 1 && rows >= 128 && cols >= 64 && tiles(128, 64) >= 148 && ws_eligible(d, 64) &&
      make_tma_operands(d, 128, 32, ops)) {
    using C_ = TmaCfg<128, 64, 4, 2, 4>;
    set_smem_attr((const void*)gemm_tma_kernel<128, 64, 4, 2, 4>, C_::SMEM);
    dim3 grid((unsigned)(cols / 64), (unsigned)(rows / 128), gz);
    gemm_tma_kernel<128, 64, 4, 2, 4><<<grid, C_::NT, C_::SMEM, st>>>(ops, d);
  } else if (ws_env == 2 && rows >= 128 && cols >= 64 && tiles(128, 64) >= 148 && ws_eligible(d, 64)) {
    using C_ = WsCfg<128, 64, 4, 2, 3>;
    set_smem_attr((const void*)gemm_ws_kernel<128, 64, 4, 2, 3>, C_::SMEM);
    dim3 grid((unsigned)(cols / 64), (unsigned)(rows / 128), gz);
    gemm_ws_kernel<128, 64, 4, 2, 3><<<grid, C_::NT, C_::SMEM, st>>>(d);
  } else if (ws_env == 3 && rows >= 128 && cols >= 128 && tiles(128, 128) >= 120 && ws_eligible(d, 128)) {
    // one CTA per SM holds a 128 x 128 tile: 16 consumer warps of 32 x 32
    using C_ = WsCfg<128, 128, 4, 4, 3>;
    set_smem_attr((const void*)gemm_ws_kernel<128, 128, 4, 4, 3>, C_::SMEM);
    dim3 grid((unsigned)(cols / 128), (unsigned)(rows / 128), gz);
    gemm_ws_kernel<128, 128, 4, 4, 3><<<grid, C_::NT, C_::SMEM, st>>>(d);
  } else if (rows >= 128 && cols >= 64 && tiles(128, 64) >= 148) {
    using C_ = PipeCfg<128, 64, 4, 2, 3>;
    set_smem_attr((const void*)gemm_pipe_kernel<128, 64, 4, 2, 3>, C_::SMEM);
    dim3 grid((unsigned)((cols + 63) / 64), (unsigned)((rows + 127) / 128), gz);
    gemm_pipe_kernel<128, 64, 4, 2, 3><<<grid, C_::NT, C_::SMEM, st>>>(d);
  } else if (rows > 32 && cols > 32) {
    using C_ = PipeCfg<64, 64, 2, 2, 4>;
    set_smem_attr((const void*)gemm_pipe_kernel<64, 64, 2, 2, 4>, C_::SMEM);
    dim3 grid((unsigned)((cols + 63) / 64), (unsigned)((rows + 63) / 64), gz);
    gemm_pipe_kernel<64, 64, 2, 2, 4><<<grid, C_::NT, C_::SMEM, st>>>(d);
  } else {
    using C_ = PipeCfg<32, 32, 2, 2, 3>;
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32), gz);
    gemm_pipe_kernel<32, 32, 2, 2, 3><<<grid, C_::NT, C_::SMEM, st>>>(d);
  }
  CK_LAUNCH();
  if (d.split_b) {
    // enough CTAs to fill the GPU even for one or two entries (c1/c3 tree levels: 64 x 1-2
    // CTAs took 18-35 us per reduction)
    const int64_t per = rows * cols;
    const int64_t bx = std::max<int64_t>(64, 1184 / std::max(nbatch, 1));
    dim3 grid((unsigned)std::min<int64_t>((per + 255) / 256, bx), (unsigned)std::min(nbatch, 65535));
    splitk_reduce_kernel<<<grid, 256, 0, st>>>(sp->partial, sp->zoff, sp->zcnt, C, Cin, beta, rows, cols, nbatch);
    CK_LAUNCH();
  }
}

struct Node {
  int64_t lo, hi, k, level;
};

std::vector<Node> partition_tree(int64_t count, int64_t* depth) {
  // BFS, split k = lo + (hi-lo+1)//2  (ref dichotomy.py:28-57)
  std::vector<Node> out;
  std::vector<std::pair<int64_t, int64_t>> frontier{{0, count - 1}}, nxt;
  int64_t level = 0;
  while (!frontier.empty()) {
    nxt.clear();
    for (auto& f : frontier) {
      int64_t lo = f.first, hi = f.second, k = lo + (hi - lo + 1) / 2;
      out.push_back({lo, hi, k, level});
      if (k - 1 >= lo) nxt.push_back({lo, k - 1});
      if (k + 1 <= hi) nxt.push_back({k + 1, hi});
    }
    frontier.swap(nxt);
    ++level;
  }
  int64_t d = 0;
  while ((int64_t(1) << d) < count) ++d;
  *depth = d;
  return out;
}

}  // namespace

struct btd_plan {
  int device = 0;
  int64_t n = 0, m = 0, mp = 0, ranks = 0, split = 1, nr = 0, L = 0, npad = 0, cap = 0;
  int rank = 0, world = 1;
  int64_t q0 = 0, q1 = 0, nrl = 0;  // owned device ranges [q0, q1)
  int64_t R0 = 0, nl = 0, nloc = 0;  // first owned (padded) row, owned padded rows, owned true rows
  int mode = 0;
  int64_t blk = 0;
  bool finished = false;
  std::vector<int64_t> lo, slot0;  // per LOCAL range: interface row relative to R0, first factor slot
  std::vector<int32_t> nint;       // per LOCAL range: interior rows inside [0, n)
  std::vector<std::unique_ptr<DevBuf>> arrays;
  const int64_t* d_lo = nullptr;
  const int64_t* d_slot0 = nullptr;
  const int32_t* d_nint = nullptr;
  DevBuf pool;     // local factor blocks + global reduced blocks
  DevBuf contrib;  // [nrl][4][mp][mp]: C_lo - B_lo U[1],  A V_last,  A U_last,  B_lo V[1]
  // scalar-coupled plan (every interior lower block a_g I, m == mp, chain kernels): the forward
  // sweep runs y_j = Dinv_j (f_g + a_g y_{j-1}) with Tbd_j = Tb_j Dinv_j (chain_fwd_sc_kernel)
  int scoup = 0;
  int64_t off_Tbd = 0, off_al = 0;
  int64_t off_AD = 0, off_Dinv = 0, off_S = 0, off_G = 0, off_Tb = 0, off_Fc = 0, off_Bif = 0,
          off_BU = 0, off_BV = 0, off_Dt = 0, off_Rd = 0, off_Rl = 0, off_Ru = 0, off_RdT = 0,
          off_RlT = 0, off_RuT = 0, off_Z = 0, off_I = 0;
  // tree (global, identical on every rank)
  std::vector<Node> nodes;
  int64_t depth = 0;
  DevBuf Rrows, EH;
  const int64_t *d_roff = nullptr, *d_rld = nullptr, *d_nlo = nullptr;
  // nodes this rank needs (its own interfaces + dependency closure), z batch over them
  int nz = 0;
  const int64_t *z_id = nullptr, *z_roff = nullptr, *z_rld = nullptr, *z_nlo = nullptr;
  SplitK z_split;
  SplitK cross_split;              // crossing-node partial sums (sharded phase B)
  // mode 1: split-K maps of the per-row-step GEMMs when a step's batch is under one wave
  // (a sharded c3 rank owns 1-4 ranges: 32-128 output tiles), keyed by (entries, K)
  std::map<std::pair<int, int64_t>, SplitK> step_splits;
  bool host_concurrent = false;  // host pipeline with >1 compute stream: chunks fill the GPU together
  std::vector<int64_t> cross_kh;   // their reduction lengths (host)
  std::vector<int64_t> z_k;  // reduction length per z entry (host)
  const int64_t* z_kd = nullptr;  // ... (device)
  bool r_uniform = false;         // inverse rows stored with the common stride r_ld
  int64_t r_ld = 0;
  struct Level {
    int count = 0;
    const int64_t *c_idx = nullptr, *z_idx = nullptr, *e_idx = nullptr, *xl_idx = nullptr,
                  *h_idx = nullptr, *xh_idx = nullptr;
    const int64_t *e_k = nullptr, *h_k = nullptr;  // 0 where the correction block is zero
    SplitK split;
    bool copy_only = false;  // no node of the level has a correction (the root): x~_k = z
  };
  int64_t partial_elems_per_k = 0;  // split-K scratch: doubles per unit K
  DevBuf partial;
  // fused cooperative tree for a row-sharded plan (M <= 32, world > 1): phases B and C
  bool fused_shard = false;
  ShardTreeArgs sargs{};
  int shard_chunks = 0, shard_work_b = 0, shard_work_c = 0;
  // fused cooperative tree (M <= 32, single rank)
  bool fused_tree = false;
  TreeArgs targs{};
  int tree_chunks = 0;
  DevBuf tpartial;
  std::vector<Level> levels;
  // interface-RHS carry (local ranges whose last interior row exists)
  int ncarry = 0;
  const int64_t *carry_src = nullptr, *carry_fc = nullptr, *carry_row = nullptr;
  // sharded: carry of the last owned range (sent to the next rank)
  int ncarry_out = 0;
  const int64_t *cout_fc = nullptr, *cout_row = nullptr;
  // sharded: tree nodes whose segment crosses a rank boundary and that some rank needs;
  // this rank contributes partial series sums over its own ranges
  int ncross = 0;
  const int64_t *cross_node = nullptr, *cross_roff = nullptr, *cross_ld = nullptr, *cross_k = nullptr,
                *cross_lo = nullptr;
  // mode-1 per-step batches (local ranges)
  struct Step1 {
    int cnt = 0;
    int nx = 0, nt = 0;
    const int64_t *x_row = nullptr, *x_slot = nullptr, *x_q = nullptr;
    const int64_t *t_row = nullptr, *t_slot = nullptr, *t_q = nullptr;
  };
  std::vector<Step1> steps1;
  int nlive = 0;  // local ranges whose interface row is < n
  // scratch
  // per-solve scratch; two slots so the pipelined host path can run two column
  // chunks concurrently on two streams (fcopy: mode-1 staging of F aliasing X)
  struct Scratch {
    int64_t k = 0;
    DevBuf ft, zbuf, xt, partial, tpartial, fcopy;
    DevBuf ubuf;  // mode 1, scalar-coupled plan: u_j = f_g + a_g y_{j-1} of the live ranges, one row step
    cudaStream_t own = nullptr;  // graph replay stream
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaStream_t side = nullptr;  // mode 1: base-accumulation GEMMs beside the row steps
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  };
  static constexpr int kSlots = 4;  // host pipeline: chunk c solves in slot c % nstreams
  Scratch sc[kSlots];
  int cur = 0;
  Scratch& S() { return sc[cur]; }
  DevBuf hostio;
  int64_t hostio_k = 0;
  std::mutex mu;
  cudaStream_t last_stream = nullptr;
  cudaEvent_t ev_done = nullptr;  // recorded after every call on its stream (cross-stream ordering)
  int64_t factor_bytes = 0;
  // CUDA graphs of repeated solves: key (F, X, K) -> instantiated graph on the plan's stream
  struct GraphEntry {
    const double* F;
    double* X;
    int64_t K;
    int slot;
    int calls;
    cudaGraphExec_t exec;
    int64_t nkern;
  };
  std::vector<GraphEntry> graphs;
  // pipelined host path: copy-in / copy-out streams, double-buffered column chunks
  cudaStream_t s_in = nullptr, s_out = nullptr, s_c[kSlots - 1] = {};  // extra compute streams
  static constexpr int kHostBufs = 8;  // device chunk buffers of the host pipeline
  cudaEvent_t ev_h[kHostBufs][3] = {};
  DevBuf hchunk;  // kHostBufs x chunk elements
  int64_t hchunk_elems = 0;
  // cuSOLVER for block orders above 256 (preprocessing only)
  DevBuf gjc_aux;  // blocked Gauss-Jordan (block orders other than 128/256 above 64): pivots, tol, dead flags
  // profiling: 4 events per solve (before fwd, after fwd, after tree, after bwd)
  bool profiling = false;
  std::vector<cudaEvent_t> ev_free, ev_pending;
  double phase_ms[4] = {0, 0, 0, 0};
  int64_t nprof = 0;
  cudaEvent_t ev_get() {
    if (!ev_free.empty()) { cudaEvent_t e = ev_free.back(); ev_free.pop_back(); return e; }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  void ev_mark(cudaStream_t st) {
    if (!profiling) return;
    cudaEvent_t e = ev_get();
    CK(cudaEventRecord(e, st));
    ev_pending.push_back(e);
  }
  void ev_drain() {
    for (size_t i = 0; i + 3 < ev_pending.size(); i += 4) {
      float t[3];
      CK(cudaEventSynchronize(ev_pending[i + 3]));
      for (int p = 0; p < 3; ++p) CK(cudaEventElapsedTime(&t[p], ev_pending[i + p], ev_pending[i + p + 1]));
      phase_ms[0] += t[0]; phase_ms[1] += t[1]; phase_ms[2] += t[2]; phase_ms[3] += t[0] + t[1] + t[2];
      ++nprof;
    }
    for (auto e : ev_pending) ev_free.push_back(e);
    ev_pending.clear();
  }
  ~btd_plan() {
    for (auto e : ev_pending) cudaEventDestroy(e);
    for (auto e : ev_free) cudaEventDestroy(e);
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& x : sc) {
      if (x.own) cudaStreamDestroy(x.own);
      if (x.ev_in) cudaEventDestroy(x.ev_in);
      if (x.ev_out) cudaEventDestroy(x.ev_out);
      if (x.side) cudaStreamDestroy(x.side);
      if (x.ev_fork) cudaEventDestroy(x.ev_fork);
      if (x.ev_join) cudaEventDestroy(x.ev_join);
    }
    if (s_in) cudaStreamDestroy(s_in);
    if (ev_done) cudaEventDestroy(ev_done);
    if (s_out) cudaStreamDestroy(s_out);
    for (auto x : s_c)
      if (x) cudaStreamDestroy(x);
    for (auto& a : ev_h)
      for (auto& e : a)
        if (e) cudaEventDestroy(e);
  }
  template <class T>
  const T* upload(const std::vector<T>& v) {
    auto b = std::make_unique<DevBuf>();
    b->alloc(std::max<size_t>(v.size() * sizeof(T), 16));
    if (!v.empty()) CK(cudaMemcpy(b->p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    const T* p = static_cast<const T*>(b->p);
    arrays.push_back(std::move(b));
    return p;
  }
  double* P(int64_t off) const { return pool.d() + off * blk; }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    CK(cudaGetDevice(&prev));
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void launch_inv(btd_plan& pl, int nbatch, const double* in, const int64_t* idx_in, int64_t add_in,
                double* out, const int64_t* idx_out, int64_t add_out, int step, int32_t* fail_step,
                int32_t* fail_col, DevBuf& ws, cudaStream_t st, const int64_t* fail_map = nullptr) {
  if (nbatch <= 0) return;
  const int mp = (int)pl.mp;
  if (mp > 64) {
    GjcDesc g{};
    g.in = in; g.idx_in = idx_in; g.add_in = add_in;
    g.out = out; g.idx_out = idx_out; g.add_out = add_out;
    g.nbatch = nbatch; g.m = (int)pl.m; g.mp = mp;
    g.step = step; g.active_until = nullptr;
    g.fail_step = fail_step; g.fail_map = fail_map; g.fail_col = fail_col;
    g.rcond = 1e-13;  // ref _kernels.pyx:19
    if (mp == 128 || mp == 256) {
      // one cluster of 8 CTAs per block holds all of D in shared memory (in-place GJ)
      g.c0 = 0; g.k0 = 0; g.npiv = mp; g.full = 1;
      if (mp == 256) {
        const size_t smem = GjcSmem<32, 8>::bytes(mp);
        set_smem_attr((const void*)gjc_panel_kernel<32, 8>, smem);
        gjc_panel_kernel<32, 8><<<nbatch * 8, GJC_NT, smem, st>>>(g);
      } else {
        const size_t smem = GjcSmem<16, 8>::bytes(mp);
        set_smem_attr((const void*)gjc_panel_kernel<16, 8>, smem);
        gjc_panel_kernel<16, 8><<<nbatch * 8, GJC_NT, smem, st>>>(g);
      }
      CK_LAUNCH();
      return;
    }
    // blocked: D inverted in place in a workspace, 32-column panels on a 4-CTA cluster,
    // DMMA updates of the other columns
    if (mp > GJC_MAXMP) fail(BTD_ERR_UNSUPPORTED, "block order above 4096");
    constexpr int PW = 32;
    const size_t wbytes = (size_t)mp * (mp + PW) * sizeof(double);
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)nbatch, (size_t)(8ull << 30) / wbytes));
    if (ws.bytes < (size_t)chunk * wbytes) ws.alloc((size_t)chunk * wbytes);
    const size_t aux = (size_t)chunk * (2 * (size_t)mp * sizeof(int32_t) + sizeof(unsigned long long) + sizeof(int32_t));
    if (pl.gjc_aux.bytes < aux) pl.gjc_aux.alloc(aux);
    // long panels: 1024 threads per CTA (one CTA per SM anyway: the slice is ~150 KB)
    const size_t smem = GjcSmem<8, 4, 1024>::bytes(mp);
    set_smem_attr((const void*)gjc_panel_kernel<8, 4, 1024>, smem);
    for (int b0 = 0; b0 < nbatch; b0 += chunk) {
      GjcDesc c = g;
      c.nbatch = std::min(chunk, nbatch - b0);
      c.idx_in = idx_in ? idx_in + b0 : nullptr;
      c.add_in = idx_in ? add_in : add_in + b0;
      c.idx_out = idx_out ? idx_out + b0 : nullptr;
      c.add_out = idx_out ? add_out : add_out + b0;
      // fail_map entries are per batch entry: offset the map (or the identity) by b0
      c.fail_map = fail_map ? fail_map + b0 : nullptr;
      if (!fail_map && b0) {
        c.fail_step = fail_step + b0;
        c.fail_col = fail_col + b0;
      }
      c.W = ws.d();
      c.rsmax = reinterpret_cast<unsigned long long*>(pl.gjc_aux.p);
      c.dead = reinterpret_cast<int32_t*>(c.rsmax + chunk);
      c.piv = c.dead + chunk;
      c.colmap = c.piv + (size_t)chunk * mp;
      CK(cudaMemsetAsync(pl.gjc_aux.p, 0, (size_t)chunk * (sizeof(unsigned long long) + sizeof(int32_t)), st));
      gjc_init_kernel<<<1184, 256, 0, st>>>(c);
      CK_LAUNCH();
      c.full = 0;
      const int ntiles = (mp + 31) / 32;
      for (int k0 = 0; k0 < mp; k0 += PW) {
        c.c0 = k0; c.k0 = k0; c.npiv = std::min(PW, mp - k0);
        gjc_panel_kernel<8, 4, 1024><<<c.nbatch * 4, 1024, smem, st>>>(c);
        CK_LAUNCH();
        gjc_update_kernel<PW><<<c.nbatch * ntiles, 256, 0, st>>>(c, ntiles);
        CK_LAUNCH();
      }
      gjc_colmap_kernel<<<(c.nbatch + 127) / 128, 128, 0, st>>>(c);
      CK_LAUNCH();
      gjc_extract_kernel<<<1184, 256, 0, st>>>(c);
      CK_LAUNCH();
    }
    return;
  }
  InvDesc d;
  d.in = in;
  d.idx_in = idx_in;
  d.add_in = add_in;
  d.out = out;
  d.idx_out = idx_out;
  d.add_out = add_out;
  d.nbatch = nbatch;
  d.m = (int)pl.m;
  d.mp = mp;
  d.step = step;
  d.active_until = nullptr;
  d.fail_step = fail_step;
  d.fail_col = fail_col;
  d.fail_map = fail_map;
  d.rcond = 1e-13;  // ref _kernels.pyx:19
  const size_t wbytes = (size_t)mp * 2 * mp * sizeof(double);
  const int use_smem = mp <= 64;
  int grid = std::min(nbatch, 65535);
  if (!use_smem) {
    const size_t want = std::min<size_t>((size_t)nbatch, std::max<size_t>(1, (size_t)(4ull << 30) / wbytes));
    const size_t have = ws.bytes / wbytes;
    if (have < std::min<size_t>(want, 296)) ws.alloc(std::min<size_t>(want, 296) * wbytes);
    grid = (int)std::min<size_t>((size_t)grid, ws.bytes / wbytes);
  }
  d.ws = ws.d();
  const int nt = mp <= 16 ? 128 : (mp <= 64 ? 256 : 512);
  const size_t smem = use_smem ? wbytes : 0;
  if (use_smem) set_smem_attr((const void*)gj_inverse_kernel, smem);
  gj_inverse_kernel<<<grid, nt, smem, st>>>(d, use_smem);
  CK_LAUNCH();
}

// ---------------------------------------------------------------- chain kernels
template <int MP, int KT, int WR, int WC, int NF = -1, int NY = -1, int PF = -1, int MINB = 1, int FULL = 0>
void launch_chain_t(const ChainArgs& a, bool fwd, cudaStream_t st) {
  using Cfg = ChainCfg<MP, KT, WR, WC, NF, NY, PF>;
  const size_t smem = (size_t)(fwd ? Cfg::FWD_BUFS : Cfg::BWD_BUFS) * MP * Cfg::LD * sizeof(double);
  const int64_t ntile = (a.K + KT - 1) / KT;
  dim3 grid((unsigned)ntile, (unsigned)a.nr);
  if (fwd) {
    set_smem_attr((const void*)chain_fwd_kernel<MP, KT, WR, WC, NF, NY, PF, MINB, FULL>, smem);
    chain_fwd_kernel<MP, KT, WR, WC, NF, NY, PF, MINB, FULL><<<grid, Cfg::NT, smem, st>>>(a);
  } else {
    set_smem_attr((const void*)chain_bwd_kernel<MP, KT, WR, WC, NF, NY, PF, MINB, FULL>, smem);
    chain_bwd_kernel<MP, KT, WR, WC, NF, NY, PF, MINB, FULL><<<grid, Cfg::NT, smem, st>>>(a);
  }
  CK_LAUNCH();
}

// Forward sweep of a scalar-coupled plan (chain_fwd_sc_kernel): chain state + two F tiles.
template <int MP, int KT, int WR, int WC, int PF = -1, int MINB = 1>
void launch_chain_sc(const ChainArgsSc& a, cudaStream_t st) {
  using Cfg = ChainCfg<MP, KT, WR, WC, 2, -1, PF>;
  const size_t smem = (size_t)3 * MP * Cfg::LD * sizeof(double);
  dim3 grid((unsigned)((a.K + KT - 1) / KT), (unsigned)a.nr);
  if (a.m == MP && a.K % KT == 0 && a.K % 2 == 0) {
    set_smem_attr((const void*)chain_fwd_sc_kernel<MP, KT, WR, WC, 2, -1, PF, MINB, 1>, smem);
    chain_fwd_sc_kernel<MP, KT, WR, WC, 2, -1, PF, MINB, 1><<<grid, Cfg::NT, smem, st>>>(a);
  } else {
    set_smem_attr((const void*)chain_fwd_sc_kernel<MP, KT, WR, WC, 2, -1, PF, MINB, 0>, smem);
    chain_fwd_sc_kernel<MP, KT, WR, WC, 2, -1, PF, MINB, 0><<<grid, Cfg::NT, smem, st>>>(a);
  }
  CK_LAUNCH();
}

// Default shapes: a bounds-check-free variant when every tile is full (block order == MP,
// K a multiple of the column tile, K even).
template <int MP, int KT, int WR, int WC, int NF = -1, int NY = -1, int PF = -1>
void launch_chain_auto(const ChainArgs& a, bool fwd, cudaStream_t st) {
  if (a.m == MP && a.K % KT == 0 && a.K % 2 == 0)
    launch_chain_t<MP, KT, WR, WC, NF, NY, PF, 1, 1>(a, fwd, st);
  else
    launch_chain_t<MP, KT, WR, WC, NF, NY, PF, 1, 0>(a, fwd, st);
}

template <int MP, int NW, int NSTG>
void launch_stream_t(const ChainArgs& a, bool fwd, cudaStream_t st) {
  using C = StreamCfg<MP, NW, NSTG>;
  const size_t smem = fwd ? C::FWD_SMEM : C::BWD_SMEM;
  dim3 grid((unsigned)((a.K + C::KC - 1) / C::KC), (unsigned)a.nr);
  if (fwd) {
    set_smem_attr((const void*)stream_fwd_kernel<MP, NW, NSTG>, smem);
    stream_fwd_kernel<MP, NW, NSTG><<<grid, C::NT, smem, st>>>(a);
  } else {
    set_smem_attr((const void*)stream_bwd_kernel<MP, NW, NSTG>, smem);
    stream_bwd_kernel<MP, NW, NSTG><<<grid, C::NT, smem, st>>>(a);
  }
  CK_LAUNCH();
}

// Streamed (TMA bulk-copy) sweeps for MP <= 32: needs 16-byte aligned rows (even K).
bool launch_stream(int64_t mp, const ChainArgs& a, bool fwd, cudaStream_t st) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("BTD_STREAM");
    enabled = e ? atoi(e) : 1;
  }
  if (!enabled || mp > 32 || (a.K & 1) || (reinterpret_cast<uintptr_t>(a.F) & 15) ||
      (reinterpret_cast<uintptr_t>(a.X) & 15))
    return false;
  const bool wide = a.K > 32;
  switch (mp) {
    case 8: wide ? launch_stream_t<8, 4, 3>(a, fwd, st) : launch_stream_t<8, 2, 3>(a, fwd, st); break;
    case 16: wide ? launch_stream_t<16, 4, 3>(a, fwd, st) : launch_stream_t<16, 2, 3>(a, fwd, st); break;
    case 32: wide ? launch_stream_t<32, 4, 2>(a, fwd, st) : launch_stream_t<32, 2, 2>(a, fwd, st); break;
    default: return false;
  }
  return true;
}

// Chain-kernel configuration per padded block order (MP, KT, warp rows x warp cols).
// BTD_CHAIN_VARIANT selects alternatives for tuning experiments.
// True when a KT-column tiling of this batch fills less than one wave of 148 SMs.
bool under_wave(const ChainArgs& a, int kt) { return (int64_t)a.nr * ((a.K + kt - 1) / kt) < 148; }

struct ScPools { const double* Tbd; const double* alpha; };  // scalar-coupled plan: forward-sweep extras
void launch_chain_slice(int64_t mp, const ChainArgs& a, bool fwd, cudaStream_t st, const ScPools* sc);

// Sweep kernels index ranges by blockIdx.y (at most 65535): more ranges (ranks * split up to
// N) run as consecutive slices with the per-range arrays and outputs offset.
void launch_chain(int64_t mp, const ChainArgs& a, bool fwd, cudaStream_t st, const ScPools* sc = nullptr) {
  constexpr int kMaxY = 65535;
  for (int q0 = 0; q0 < a.nr; q0 += kMaxY) {
    ChainArgs s = a;
    s.nr = std::min(kMaxY, a.nr - q0);
    s.lo = a.lo + q0;
    s.nint = a.nint + q0;
    s.slot0 = a.slot0 + q0;
    if (a.base) s.base = a.base + (int64_t)q0 * a.base_stride;
    if (a.xt) s.xt = a.xt + (int64_t)q0 * mp * a.K;
    launch_chain_slice(mp, s, fwd, st, sc);
  }
}

void launch_chain_slice(int64_t mp, const ChainArgs& a0, bool fwd, cudaStream_t st, const ScPools* sc) {
  const ChainArgs& a = a0;
  if (a.nr <= 0) return;
  if (launch_stream(mp, a, fwd, st)) return;
  static int variant_f = -1, variant_b = -1;
  if (variant_f < 0) {
    const char* e = getenv("BTD_CHAIN_VARIANT");
    variant_f = e ? atoi(e) : 0;
    const char* eb = getenv("BTD_CHAIN_VARIANT_BWD");
    variant_b = eb ? atoi(eb) : variant_f;
  }
  const int variant = fwd ? variant_f : variant_b;
  if (fwd && sc) {  // scalar-coupled plan: the two-product forward sweep (same tile policy as below)
    ChainArgsSc as;
    static_cast<ChainArgs&>(as) = a0;
    as.Tbd = sc->Tbd;
    as.alpha = sc->alpha;
    static int scv = -1;
    if (scv < 0) {
      const char* e = getenv("BTD_SC_VARIANT");
      scv = e ? atoi(e) : 0;
    }
    switch (mp) {
      case 64:
        if (under_wave(a, 128)) launch_chain_sc<64, 32, 8, 1>(as, st);
        else launch_chain_sc<64, 128, 8, 2, 8>(as, st);
        return;
      case 128:
        if (under_wave(a, 64)) launch_chain_sc<128, 16, 16, 1>(as, st);
        else launch_chain_sc<128, 64, 16, 1>(as, st);
        return;
      case 256:
        if (scv == 1) launch_chain_sc<256, 32, 16, 1, 4>(as, st);
        else if (scv == 2) launch_chain_sc<256, 32, 32, 1>(as, st);
        else if (scv == 3) launch_chain_sc<256, 16, 16, 1, 4>(as, st);
        else if (scv == 4) launch_chain_sc<256, 32, 16, 1, 8>(as, st);
        else if (under_wave(a, 16)) launch_chain_sc<256, 8, 16, 1>(as, st);
        else launch_chain_sc<256, 16, 16, 1, 8>(as, st);
        return;
      default: fail(BTD_ERR_UNSUPPORTED, "scalar-coupled plan: no forward kernel for this block order");
    }
  }
  switch (mp) {
    case 8: launch_chain_t<8, 32, 1, 4>(a, fwd, st); break;
    case 16: launch_chain_t<16, 16, 1, 1>(a, fwd, st); break;
    case 32: launch_chain_t<32, 32, 2, 2>(a, fwd, st); break;
    case 64:
      if (variant == 2) launch_chain_t<64, 64, 8, 2, 2, 0>(a, fwd, st);
      else if (variant == 3) launch_chain_t<64, 64, 8, 2, 3, 0>(a, fwd, st);
      else if (variant == 4) launch_chain_t<64, 64, 8, 2, 2, 3>(a, fwd, st);
      else if (variant == 5) launch_chain_t<64, 128, 8, 2, 2, 0>(a, fwd, st);
      else if (variant == 6) launch_chain_t<64, 64, 4, 4>(a, fwd, st);
      else if (variant == 7) launch_chain_t<64, 32, 8, 2>(a, fwd, st);
      else if (variant == 8) launch_chain_t<64, 32, 8, 1>(a, fwd, st);
      else if (variant == 9) launch_chain_t<64, 32, 4, 2>(a, fwd, st);
      else if (variant == 10) launch_chain_t<64, 32, 8, 1, 2, 2>(a, fwd, st);
      else if (variant == 11) launch_chain_t<64, 32, 8, 1, 4, 4>(a, fwd, st);
      else if (variant == 12) launch_chain_t<64, 16, 8, 1>(a, fwd, st);
      else if (variant == 13) launch_chain_t<64, 32, 8, 1, 3, 0>(a, fwd, st);
      else if (variant == 14) launch_chain_t<64, 16, 4, 1>(a, fwd, st);
      else if (variant == 15) launch_chain_t<64, 128, 4, 4, 2, 0>(a, fwd, st);
      else if (variant == 16) launch_chain_t<64, 128, 8, 4, 2, 0>(a, fwd, st);
      else if (variant == 17) launch_chain_t<64, 64, 8, 2, 2, 0>(a, fwd, st);
      else if (variant == 18) launch_chain_t<64, 64, 4, 2, 2, 0>(a, fwd, st);
      else if (variant == 19) launch_chain_t<64, 64, 8, 1, 2, 0>(a, fwd, st);
      else if (variant == 20) launch_chain_t<64, 128, 8, 2, 2, 0, 8>(a, fwd, st);
      // measured best (c2, profiles/r01_chain_ab.txt): 128-column tiles of 2 x 8 warps with
      // per-column-group barriers in both directions (bwd 9.96 -> 9.54 ms vs 32-column tiles);
      // forward factor fragments 8 pair steps ahead (13.76 -> 13.66 ms).  Narrow batches
      // (host-pipeline chunks, small K) whose 128-column grid would leave SMs idle take
      // 32-column tiles: the sweep is a chain of L row steps, so its latency falls with
      // the work per CTA.
      else if (under_wave(a, 128)) launch_chain_auto<64, 32, 8, 1>(a, fwd, st);
      else if (fwd) launch_chain_auto<64, 128, 8, 2, 2, 0, 8>(a, fwd, st);
      else launch_chain_t<64, 128, 8, 2, 2, 0>(a, fwd, st);  // (the bounds-check-free variant is 7% slower here)
      break;
    case 128:
      if (variant == 1) launch_chain_t<128, 64, 16, 2>(a, fwd, st);
      else if (variant == 2) launch_chain_t<128, 64, 16, 1>(a, fwd, st);
      else if (variant == 3) launch_chain_t<128, 16, 16, 1>(a, fwd, st);
      else if (variant == 4) launch_chain_t<128, 32, 8, 1>(a, fwd, st);
      else if (variant == 5) launch_chain_t<128, 32, 16, 2>(a, fwd, st);
      else if (variant == 6) launch_chain_t<128, 32, 16, 1>(a, fwd, st);
      else if (variant == 7) launch_chain_t<128, 64, 16, 1, -1, -1, 8>(a, fwd, st);
      else if (variant == 8) launch_chain_t<128, 64, 16, 1, -1, -1, 16>(a, fwd, st);
      else if (under_wave(a, 64)) launch_chain_auto<128, 16, 16, 1>(a, fwd, st);  // narrow batches
      else launch_chain_auto<128, 64, 16, 1>(a, fwd, st);  // measured best on the c3dd interiors (+7%)
      break;
    case 256:
      if (variant == 1) launch_chain_t<256, 32, 16, 1>(a, fwd, st);
      else if (variant == 2) launch_chain_t<256, 16, 16, 1, 3, 0>(a, fwd, st);
      else if (variant == 3) launch_chain_t<256, 8, 16, 1>(a, fwd, st);
      else if (variant == 4) launch_chain_t<256, 16, 32, 1>(a, fwd, st);
      else if (variant == 5) launch_chain_t<256, 32, 32, 1>(a, fwd, st);
      else if (variant == 6) launch_chain_t<256, 32, 8, 2>(a, fwd, st);
      else if (variant == 7) launch_chain_t<256, 32, 16, 2>(a, fwd, st);
      else if (variant == 8) launch_chain_t<256, 64, 16, 2>(a, fwd, st);
      else if (variant == 9) launch_chain_t<256, 16, 16, 2>(a, fwd, st);
      else if (variant == 10) launch_chain_t<256, 32, 32, 1, -1, -1, 2>(a, fwd, st);
      else if (variant == 11) launch_chain_t<256, 16, 16, 1, -1, -1, 2>(a, fwd, st);
      else if (variant == 12) launch_chain_t<256, 16, 16, 1, -1, -1, 8>(a, fwd, st);
      else if (variant == 13) launch_chain_t<256, 32, 32, 1, -1, -1, 1>(a, fwd, st);
      else if (variant == 14) launch_chain_t<256, 16, 16, 1, 2, 3, 8>(a, fwd, st);
      else if (variant == 15) launch_chain_t<256, 16, 16, 1, 2, 2, 8>(a, fwd, st);
      else if (variant == 16) launch_chain_t<256, 32, 16, 1, 2, 0, 8>(a, fwd, st);
      else if (variant == 17) launch_chain_t<256, 16, 16, 1, 2, 3, 4>(a, fwd, st);
      // measured (c1, profiles/r01_chain_ab.txt): forward factor fragments 8 pair steps ahead
      // (13.08 -> 12.74 ms; 2 ahead: 17.1 ms), 32-warp CTAs backward (-4%).  Narrow batches
      // (host-pipeline chunks of 32 / 64 columns) take 8- / 16-column tiles so the chains
      // spread over all SMs.
      else if (fwd && under_wave(a, 16)) launch_chain_auto<256, 8, 16, 1>(a, fwd, st);
      else if (fwd) launch_chain_auto<256, 16, 16, 1, -1, -1, 8>(a, fwd, st);
      else if (under_wave(a, 16)) launch_chain_auto<256, 8, 16, 1>(a, fwd, st);
      else if (under_wave(a, 32)) launch_chain_auto<256, 16, 16, 1>(a, fwd, st);
      else launch_chain_auto<256, 32, 32, 1>(a, fwd, st);
      break;
    default: fail(BTD_ERR_UNSUPPORTED, "no chain kernel for this block order");
  }
}

int64_t pad_order(int64_t m, int mode) {
  if (mode == 1) return (m + 7) / 8 * 8;
  for (int64_t c : {8, 16, 32, 64, 128, 256})
    if (m <= c) return c;
  return (m + 7) / 8 * 8;
}

// ---------------------------------------------------------------- plan build, local part
// Ranges owned by this rank: [q0, q1).  The rank reads only its rows of the
// matrix and produces its factors plus the four reduced-system contributions
// per range; the tree part (build_finish) needs everyone's contributions.
//
// restore >= 0: metadata only (plan import, btd_plan_import); the factor pool is
// loaded from an exported image afterwards and `restore` is the image's sweep mode.
void build_local(btd_plan& pl, const double* diag, const double* lower, const double* upper, int flags,
                 cudaStream_t st, int64_t* err_row, int64_t* err_range, int restore = -1) {
  const int64_t n = pl.n, m = pl.m;
  int forced = -1;
  if (const char* e = getenv("BTD_FORCE_MODE")) forced = atoi(e);
  pl.mode = restore >= 0 ? restore : forced >= 0 ? forced : (m > 256 ? 1 : 0);
  pl.mp = pad_order(m, pl.mode);
  const int64_t mp = pl.mp, blk = mp * mp;
  pl.blk = blk;
  pl.nr = std::min<int64_t>(n, pl.ranks * std::max<int64_t>(1, pl.split));
  if (pl.world > 1 && pl.nr % pl.world != 0)
    fail(BTD_ERR_INVALID_ARG, "device ranges (ranks*split) must be a multiple of the world size");
  pl.L = (n + pl.nr - 1) / pl.nr;
  pl.npad = pl.L * pl.nr;
  pl.cap = pl.L - 1;
  pl.nrl = pl.nr / pl.world;
  pl.q0 = pl.rank * pl.nrl;
  pl.q1 = pl.q0 + pl.nrl;
  pl.R0 = pl.q0 * pl.L;
  pl.nl = pl.nrl * pl.L;
  pl.nloc = std::max<int64_t>(0, std::min<int64_t>(pl.nl, n - pl.R0));
  const int64_t nrl = pl.nrl, L = pl.L, cap = pl.cap, nl = pl.nl, R0 = pl.R0, nr = pl.nr;
  pl.lo.resize(nrl);
  pl.slot0.resize(nrl);
  pl.nint.resize(nrl);
  pl.nlive = 0;
  for (int64_t ql = 0; ql < nrl; ++ql) {
    const int64_t glo = (pl.q0 + ql) * L;
    pl.lo[ql] = ql * L;
    pl.slot0[ql] = ql * cap;
    pl.nint[ql] = (int32_t)std::max<int64_t>(0, std::min<int64_t>(L - 1, n - glo - 1));
    if (glo < n) pl.nlive++;
  }
  pl.d_lo = pl.upload(pl.lo);
  pl.d_slot0 = pl.upload(pl.slot0);
  pl.d_nint = pl.upload(pl.nint);

  // ---- local padded matrix rows [R0, R0+nl): [C | Lw | Uw], nl blocks each
  //      Lw[i] = lower[R0+i] (couples row R0+i+1 to R0+i), Uw[i] = upper[R0+i]; zero / identity past n
  DevBuf mat, tmp;
  if (restore < 0) {
    mat.alloc((size_t)3 * nl * blk * sizeof(double));
    const double* srcs[3] = {diag, lower, upper};
    const int64_t counts[3] = {std::max<int64_t>(0, std::min(nl, n - R0)), std::max<int64_t>(0, std::min(nl, n - 1 - R0)),
                               std::max<int64_t>(0, std::min(nl, n - 1 - R0))};
    const bool on_dev = flags & BTD_MATRIX_ON_DEVICE;
    if (!on_dev) tmp.alloc((size_t)nl * m * m * sizeof(double));
    for (int s = 0; s < 3; ++s) {
      const double* src = srcs[s] ? srcs[s] + (size_t)R0 * m * m : nullptr;
      const size_t bytes = (size_t)counts[s] * m * m * sizeof(double);
      if (!on_dev && bytes) {
        CK(cudaMemcpyAsync(tmp.p, src, bytes, cudaMemcpyHostToDevice, st));
        src = tmp.d();
      }
      pad_blocks_kernel<<<1184, 256, 0, st>>>(src, counts[s], (int)m, mat.d() + (size_t)s * nl * blk, nl, (int)mp,
                                             s == 0);
      CK_LAUNCH();
      if (!on_dev) CK(cudaStreamSynchronize(st));  // tmp reused
    }
  }
  tmp.release();
  const double* Cm = mat.d();
  const int64_t offL = nl, offU = 2 * nl;
  DevBuf sc_alpha;
  if (restore < 0) {
    static int sc_on = -1;
    if (sc_on < 0) {
      const char* e = getenv("BTD_SCALAR_COUPLING");
      sc_on = e ? atoi(e) : 1;
    }
    pl.scoup = 0;
    // chain kernels (mode 0, orders 64 / 128 / 256) and the GEMM-per-row sweep (mode 1)
    if (sc_on && m == mp && cap > 0 && nrl > 0 && ((pl.mode == 0 && mp >= 64) || pl.mode == 1)) {
      DevBuf bad;
      bad.alloc(sizeof(int));
      sc_alpha.alloc((size_t)nrl * cap * sizeof(double));
      CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
      scalar_coupling_kernel<<<(unsigned)(nrl * cap), 256, 0, st>>>(Cm + offL * blk, pl.d_lo, pl.d_nint, cap, (int)mp,
                                                                 sc_alpha.d(), static_cast<int*>(bad.p));
      CK_LAUNCH();
      int hbad = 1;
      CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      pl.scoup = hbad ? 0 : 1;
    }
  }

  // ---- pool layout: local factors, global reduced system, constants
  const int64_t nslot = nrl * cap;
  int64_t o = 0;
  auto take = [&](int64_t cnt) { int64_t r = o; o += cnt; return r; };
  pl.off_AD = take(nslot);
  pl.off_Dinv = take(nslot);
  pl.off_S = take(nslot);
  pl.off_G = take(nslot);
  pl.off_Tb = take(nslot);
  pl.off_Fc = take(nrl);
  pl.off_Bif = take(nrl);
  pl.off_BU = take(nrl);
  pl.off_BV = take(nrl);
  pl.off_Dt = take(nrl);
  pl.off_Rd = take(nr);
  pl.off_Rl = take(nr);
  pl.off_Ru = take(nr);
  pl.off_RdT = take(nr);
  pl.off_RlT = take(nr);
  pl.off_RuT = take(nr);
  pl.off_Z = take(1);
  pl.off_I = take(1);
  if (pl.scoup) {
    // mode 0: Tbd takes over the AD section once the build no longer needs AD (a scalar-coupled plan
    // never runs the general forward sweep: launch_chain_slice covers every shape with
    // chain_fwd_sc_kernel).  Mode 1 keeps Tb (its base accumulation is a GEMM of its own on y_j).
    pl.off_Tbd = pl.off_AD;
    pl.off_al = take((nslot + blk - 1) / blk);  // a_g per slot, as doubles inside the pool (plan images carry it)
  }
  pl.pool.alloc((size_t)o * blk * sizeof(double));
  CK(cudaMemsetAsync(pl.pool.p, 0, (size_t)o * blk * sizeof(double), st));
  set_identity_kernel<<<64, 256, 0, st>>>(pl.P(pl.off_I), (int)mp);
  CK_LAUNCH();
  pl.factor_bytes = (int64_t)o * blk * sizeof(double);

  if (restore < 0) {
  double* pool = pl.pool.d();
  const int64_t* lo_arr = pl.d_lo;
  const int64_t* slot_arr = pl.d_slot0;
  DevBuf ws, fail_step, fail_col;
  fail_step.alloc(sizeof(int32_t) * std::max<int64_t>(nrl, 1));
  fail_col.alloc(sizeof(int32_t) * std::max<int64_t>(nrl, 1));
  CK(cudaMemsetAsync(fail_step.p, 0xff, sizeof(int32_t) * std::max<int64_t>(nrl, 1), st));

  // Bif_q = upper[lo_q], Fc_q = lower[hi_q - 1]
  {
    std::vector<int64_t> src(2 * nrl), dst(2 * nrl);
    for (int64_t q = 0; q < nrl; ++q) {
      src[q] = offU + pl.lo[q];
      dst[q] = pl.off_Bif + q;
      src[nrl + q] = offL + (q + 1) * L - 1;
      dst[nrl + q] = pl.off_Fc + q;
    }
    launch_gemm(mp, mp, (int)(2 * nrl), mk(pool, pl.upload(dst), 0, blk, mp), mk(Cm, pl.upload(src), 0, blk, mp), 1.0,
                {}, st);
  }

  const int nb = (int)nrl;
  if (cap > 0 && nb > 0) {
    std::vector<int64_t> sa_c(2 * nrl), sa_a(2 * nrl), sa_b(2 * nrl), gt_c(2 * nrl), gt_a0(2 * nrl),
        gt_a(2 * nrl), gt_b(2 * nrl);
    for (int64_t q = 0; q < nrl; ++q) {
      const int64_t s0 = pl.slot0[q];
      sa_c[q] = pl.off_S + s0;
      sa_c[nrl + q] = pl.off_AD + s0;
      sa_a[q] = sa_a[nrl + q] = pl.off_Dinv + s0;
      sa_b[q] = offU + pl.lo[q] + 1;   // B_g = upper[g], g = lo+1+j
      sa_b[nrl + q] = offL + pl.lo[q];  // A_g = lower[g-1]
      gt_c[q] = pl.off_G + s0;
      gt_c[nrl + q] = pl.off_Tb + s0;
      gt_a0[q] = pl.off_AD + s0;          // G_0 = AD_0
      gt_a0[nrl + q] = pl.off_Bif + q;    // Tb_0 = B_lo
      gt_a[q] = pl.off_AD + s0;           // G_j = AD_j G_{j-1}
      gt_a[nrl + q] = pl.off_Tb + s0 - 1;  // Tb_j = Tb_{j-1} S_{j-1}
      gt_b[q] = pl.off_G + s0 - 1;
      gt_b[nrl + q] = pl.off_S + s0 - 1;
    }
    const int64_t *d_sa_c = pl.upload(sa_c), *d_sa_a = pl.upload(sa_a), *d_sa_b = pl.upload(sa_b),
                  *d_gt_c = pl.upload(gt_c), *d_gt_a0 = pl.upload(gt_a0), *d_gt_a = pl.upload(gt_a),
                  *d_gt_b = pl.upload(gt_b);
    for (int64_t j = 0; j < cap; ++j) {
      // D_j = C_g - A_g S_{j-1}     (ref _kernels.pyx:168)
      if (j == 0)
        launch_gemm(mp, mp, nb, mk(pool, nullptr, pl.off_Dt, blk, mp), mk(Cm, lo_arr, 1, blk, mp), 1.0, {}, st);
      else
        launch_gemm(mp, mp, nb, mk(pool, nullptr, pl.off_Dt, blk, mp), mk(Cm, lo_arr, 1 + j, blk, mp), 1.0,
                    {term(mk(Cm, lo_arr, offL + j, blk, mp), mk(pool, slot_arr, pl.off_S + j - 1, blk, mp), mp,
                          -1.0)},
                    st);
      launch_inv(pl, nb, pool, nullptr, pl.off_Dt, pool, slot_arr, pl.off_Dinv + j, (int)j, fail_step.i32(),
                 fail_col.i32(), ws, st);
      // S_j = Dinv_j B_g ; AD_j = Dinv_j A_g
      launch_gemm(mp, mp, 2 * nb, mk(pool, d_sa_c, j, blk, mp), none(), 0.0,
                  {term(mk(pool, d_sa_a, j, blk, mp), mk(Cm, d_sa_b, j, blk, mp), mp)}, st);
      // G_j, Tb_j
      if (j == 0)
        launch_gemm(mp, mp, 2 * nb, mk(pool, d_gt_c, 0, blk, mp), mk(pool, d_gt_a0, 0, blk, mp), 1.0, {}, st);
      else
        launch_gemm(mp, mp, 2 * nb, mk(pool, d_gt_c, j, blk, mp), none(), 0.0,
                    {term(mk(pool, d_gt_a, j, blk, mp), mk(pool, d_gt_b, j, blk, mp), mp)}, st);
      // BU_q += Tb_j G_j   (= B_lo U[1], ref dichotomy.py:232)
      launch_gemm(mp, mp, nb, mk(pool, nullptr, pl.off_BU, blk, mp),
                  j == 0 ? none() : mk(pool, nullptr, pl.off_BU, blk, mp), 1.0,
                  {term(mk(pool, slot_arr, pl.off_Tb + j, blk, mp), mk(pool, slot_arr, pl.off_G + j, blk, mp), mp)},
                  st);
    }
    // BV_q = Tb_{L-2} S_{L-2}  (= B_lo V[1])
    launch_gemm(mp, mp, nb, mk(pool, nullptr, pl.off_BV, blk, mp), none(), 0.0,
                {term(mk(pool, slot_arr, pl.off_Tb + cap - 1, blk, mp), mk(pool, slot_arr, pl.off_S + cap - 1, blk, mp),
                      mp)},
                st);
    if (pl.scoup) {  // Tbd_s = Tb_s Dinv_s for every slot, over AD (G_j = AD_j G_{j-1} is done); a_g beside it
      if (pl.mode == 0)
        launch_gemm(mp, mp, (int)nslot, mk(pool, nullptr, pl.off_Tbd, blk, mp), none(), 0.0,
                    {term(mk(pool, nullptr, pl.off_Tb, blk, mp), mk(pool, nullptr, pl.off_Dinv, blk, mp), mp)}, st);
      CK(cudaMemcpyAsync(pool + pl.off_al * blk, sc_alpha.p, (size_t)nslot * sizeof(double), cudaMemcpyDeviceToDevice,
                         st));
    }
  }

  // ---- range failures: first range (in order) wins, row local to its interior
  {
    std::vector<int32_t> fs(std::max<int64_t>(nrl, 1), -1);
    if (nrl) CK(cudaMemcpyAsync(fs.data(), fail_step.p, sizeof(int32_t) * nrl, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t q = 0; q < nrl; ++q)
      if (fs[q] >= 0) {
        *err_row = fs[q];
        *err_range = pl.q0 + q;
        char buf[160];
        snprintf(buf, sizeof buf, "block row %d: singular pivot (range %lld)", fs[q], (long long)(pl.q0 + q));
        fail(BTD_ERR_SINGULAR_PIVOT, buf);
      }
  }

  // ---- per-range contributions to the reduced system (ref dichotomy.py:212-236)
  //   c0 = C_lo - B_lo U[1]     (own diagonal)
  //   c1 = A_{hi} V[L-1]        (subtracted from the NEXT range's diagonal)
  //   c2 = A_{hi} U[L-1]        (the next range's lower coupling)
  //   c3 = B_lo V[1]            (own upper coupling)
  pl.contrib.alloc((size_t)std::max<int64_t>(nrl, 1) * 4 * blk * sizeof(double));
  if (nrl) {
    double* cb = pl.contrib.d();
    std::vector<int64_t> c0c(nrl), c0in(nrl), c0a(nrl), c1c(nrl), c1a(nrl), c1b(nrl), c2c(nrl), c2b(nrl),
        c3c(nrl), c3in(nrl);
    for (int64_t q = 0; q < nrl; ++q) {
      c0c[q] = 4 * q; c0in[q] = pl.lo[q]; c0a[q] = pl.off_BU + q;
      c1c[q] = 4 * q + 1; c1a[q] = pl.off_Fc + q;
      c1b[q] = cap > 0 ? pl.off_S + pl.slot0[q] + cap - 1 : pl.off_Z;
      c2c[q] = 4 * q + 2; c2b[q] = cap > 0 ? pl.off_G + pl.slot0[q] + cap - 1 : pl.off_I;
      c3c[q] = 4 * q + 3; c3in[q] = cap > 0 ? pl.off_BV + q : pl.off_Bif + q;
    }
    const int64_t* dI = nullptr;
    (void)dI;
    launch_gemm(mp, mp, nb, mk(cb, pl.upload(c0c), 0, blk, mp), mk(Cm, pl.upload(c0in), 0, blk, mp), 1.0,
                {term(mk(pool, pl.upload(c0a), 0, blk, mp), mk(pool + pl.off_I * blk, nullptr, 0, 0, mp), mp, -1.0)},
                st);
    const int64_t* d_c1a = pl.upload(c1a);
    launch_gemm(mp, mp, nb, mk(cb, pl.upload(c1c), 0, blk, mp), none(), 0.0,
                {term(mk(pool, d_c1a, 0, blk, mp), mk(pool, pl.upload(c1b), 0, blk, mp), mp)}, st);
    launch_gemm(mp, mp, nb, mk(cb, pl.upload(c2c), 0, blk, mp), none(), 0.0,
                {term(mk(pool, d_c1a, 0, blk, mp), mk(pool, pl.upload(c2b), 0, blk, mp), mp)}, st);
    launch_gemm(mp, mp, nb, mk(cb, pl.upload(c3c), 0, blk, mp), mk(pool, pl.upload(c3in), 0, blk, mp), 1.0, {}, st);
  }
  }  // restore < 0
  mat.release();

  // ---- solve-time local batches
  {
    // carry_q = Fc_q y_{q,last}: ranges whose last interior row lies inside [0, n)
    std::vector<int64_t> cs, cf, cr, of, orow;
    for (int64_t q = 0; q < nrl; ++q)
      if (cap > 0 && pl.nint[q] == cap && (pl.q0 + q + 1) * L <= n && pl.q0 + q + 1 < nr) {
        if (q + 1 < nrl) {
          cs.push_back(q); cf.push_back(pl.off_Fc + q); cr.push_back(pl.lo[q] + L - 1);
        } else {  // the next range belongs to the next rank
          of.push_back(pl.off_Fc + q); orow.push_back(pl.lo[q] + L - 1);
        }
      }
    pl.ncarry = (int)cs.size();
    pl.carry_src = pl.upload(cs); pl.carry_fc = pl.upload(cf); pl.carry_row = pl.upload(cr);
    pl.ncarry_out = (int)of.size();
    pl.cout_fc = pl.upload(of); pl.cout_row = pl.upload(orow);
    if (pl.world == 1 && pl.ncarry_out) fail(BTD_ERR_CUDA, "internal: boundary carry on a single-rank plan");
    if (pl.mode == 1) {
      pl.steps1.resize(cap);
      for (int64_t j = 0; j < cap; ++j) {
        std::vector<int64_t> xr, xs, xq, tr, ts, tq;
        int cnt = 0;
        for (int64_t q = 0; q < nrl; ++q) {
          if (pl.nint[q] > j) ++cnt;
          if (j < pl.nint[q] - 1) { xr.push_back(pl.lo[q] + 1 + j); xs.push_back(pl.slot0[q] + j); xq.push_back(q); }
          else if (j == pl.nint[q] - 1) { tr.push_back(pl.lo[q] + 1 + j); ts.push_back(pl.slot0[q] + j); tq.push_back(q); }
        }
        auto& s = pl.steps1[j];
        s.cnt = cnt; s.nx = (int)xq.size(); s.nt = (int)tq.size();
        s.x_row = pl.upload(xr); s.x_slot = pl.upload(xs); s.x_q = pl.upload(xq);
        s.t_row = pl.upload(tr); s.t_slot = pl.upload(ts); s.t_q = pl.upload(tq);
      }
    }
  }
  CK(cudaStreamSynchronize(st));
}

// Choose k-chunks so a tree launch fills >= 2 waves; record (entry, chunk) maps.
SplitK make_split(btd_plan& pl, const std::vector<int64_t>& kper, int64_t tiles_per_entry, int64_t& maxz) {
  SplitK sp;
  const int64_t want = 2 * 148;
  int64_t base = 0, kmax = 0;
  for (int64_t k : kper) { base += tiles_per_entry; kmax = std::max(kmax, k); }
  if (kper.empty() || base >= want * 2) return sp;
  // chunk: the largest multiple of 16 that still yields >= want CTAs in total (and >= 64 long)
  int64_t chunk = std::max<int64_t>(64, (kmax + 31) / 32 * 32);
  auto total = [&](int64_t ch) {
    int64_t t = 0;
    for (int64_t k : kper) t += (k + ch - 1) / ch;
    return t;
  };
  while (chunk > 64 && total(chunk) * tiles_per_entry < want) chunk = std::max<int64_t>(64, (chunk / 2 + 31) / 32 * 32);
  const int64_t nt = total(chunk);
  if (nt <= (int64_t)kper.size()) return sp;  // no entry split: plain launch
  std::vector<int32_t> sb, sk, zoff, zcnt;
  for (size_t b = 0; b < kper.size(); ++b) {
    const int64_t n = std::max<int64_t>(1, (kper[b] + chunk - 1) / chunk);
    zoff.push_back((int32_t)sb.size());
    zcnt.push_back((int32_t)n);
    for (int64_t c = 0; c < n; ++c) { sb.push_back((int32_t)b); sk.push_back((int32_t)c); }
  }
  sp.ntotal = (int)sb.size();
  sp.kchunk = chunk;
  sp.sb = pl.upload(sb); sp.sk = pl.upload(sk); sp.zoff = pl.upload(zoff); sp.zcnt = pl.upload(zcnt);
  maxz = std::max<int64_t>(maxz, sp.ntotal);
  return sp;
}

void build_splits(btd_plan& pl) {
  const int64_t mp = pl.mp;
  // tiles per entry for an (mp x K) output; K unknown at plan time: assume one column tile per 64
  const int64_t tiles = std::max<int64_t>(1, (mp + 63) / 64);
  int64_t maxz = 0;
  pl.z_split = make_split(pl, pl.z_k, tiles, maxz);
  pl.cross_split = make_split(pl, pl.cross_kh, tiles, maxz);
  for (auto& L_ : pl.levels) {
    std::vector<int64_t> kk(L_.count, mp);
    L_.split = make_split(pl, kk, tiles, maxz);
  }
  pl.partial_elems_per_k = maxz * mp;
}

// Index arrays for the many small launches of the tree build, sub-allocated from 4 MB pinned +
// device chunks and copied with cudaMemcpyAsync on the build stream.  (A cudaMalloc plus a
// blocking cudaMemcpy per array made plans of 20000 device ranges take ~20 s: the root's
// inverse rows are a sequential sweep over all ranges, a few launches per step.)
class StagedUploads {
 public:
  explicit StagedUploads(cudaStream_t st) : st_(st) {}
  StagedUploads(const StagedUploads&) = delete;
  StagedUploads& operator=(const StagedUploads&) = delete;
  ~StagedUploads() {
    cudaStreamSynchronize(st_);  // copies and the kernels reading them are done
    for (void* p : host_) cudaFreeHost(p);
    for (void* p : dev_) cudaFree(p);
  }
  template <class T>
  const T* put(const std::vector<T>& v) {
    const size_t bytes = (std::max<size_t>(v.size() * sizeof(T), 16) + 15) / 16 * 16;
    if (host_.empty() || off_ + bytes > cap_) {
      cap_ = std::max<size_t>(kChunk, bytes);
      void *h = nullptr, *d = nullptr;
      CK(cudaMallocHost(&h, cap_));
      host_.push_back(h);
      CK(cudaMalloc(&d, cap_));
      dev_.push_back(d);
      off_ = 0;
    }
    char* h = static_cast<char*>(host_.back()) + off_;
    char* d = static_cast<char*>(dev_.back()) + off_;
    if (!v.empty()) {
      memcpy(h, v.data(), v.size() * sizeof(T));
      CK(cudaMemcpyAsync(d, h, v.size() * sizeof(T), cudaMemcpyHostToDevice, st_));
    }
    off_ += bytes;
    return reinterpret_cast<const T*>(d);
  }

 private:
  static constexpr size_t kChunk = size_t(4) << 20;
  cudaStream_t st_;
  std::vector<void*> host_, dev_;
  size_t off_ = 0, cap_ = 0;
};

// ---------------------------------------------------------------- plan build, global part
// contrib_all: [nr][4][mp][mp] device, identical on every rank.
void build_finish(btd_plan& pl, const double* contrib_all, cudaStream_t st, int64_t* err_row, bool restore = false) {
  const int64_t mp = pl.mp, blk = pl.blk, nr = pl.nr;
  double* pool = pl.pool.d();
  const double* I = pool + pl.off_I * blk;
  // reduced system: Rd_q = c0_q - c1_{q-1}, Rl_{q-1} = c2_{q-1}, Ru_q = c3_q
  if (!restore) {
    std::vector<int64_t> d_c, d_in, d_a, l_c, l_in, u_c, u_in;
    for (int64_t q = 0; q < nr; ++q) {
      if (q >= 1) { d_c.push_back(pl.off_Rd + q); d_in.push_back(4 * q); d_a.push_back(4 * (q - 1) + 1); }
      if (q >= 1) { l_c.push_back(pl.off_Rl + q - 1); l_in.push_back(4 * (q - 1) + 2); }
      if (q + 1 < nr) { u_c.push_back(pl.off_Ru + q); u_in.push_back(4 * q + 3); }
    }
    launch_gemm(mp, mp, 1, mk(pool, nullptr, pl.off_Rd, blk, mp), mk(contrib_all, nullptr, 0, blk, mp), 1.0, {}, st);
    if (!d_c.empty()) {
      launch_gemm(mp, mp, (int)d_c.size(), mk(pool, pl.upload(d_c), 0, blk, mp), mk(contrib_all, pl.upload(d_in), 0, blk, mp),
                  1.0, {term(mk(contrib_all, pl.upload(d_a), 0, blk, mp), mk(I, nullptr, 0, 0, mp), mp, -1.0)}, st);
      launch_gemm(mp, mp, (int)l_c.size(), mk(pool, pl.upload(l_c), 0, blk, mp), mk(contrib_all, pl.upload(l_in), 0, blk, mp),
                  1.0, {}, st);
      launch_gemm(mp, mp, (int)u_c.size(), mk(pool, pl.upload(u_c), 0, blk, mp), mk(contrib_all, pl.upload(u_in), 0, blk, mp),
                  1.0, {}, st);
    }
    // transposed system T = R^T: diag Rd^T, lower Ru^T, upper Rl^T (ref core.py:137-143)
    std::vector<int64_t> ti, to;
    for (int64_t q = 0; q < nr; ++q) {
      ti.push_back(pl.off_Rd + q); to.push_back(pl.off_RdT + q);
      if (q + 1 < nr) {
        ti.push_back(pl.off_Rl + q); to.push_back(pl.off_RlT + q);
        ti.push_back(pl.off_Ru + q); to.push_back(pl.off_RuT + q);
      }
    }
    const int nb = (int)ti.size();
    dim3 grid((unsigned)((mp + 31) / 32), (unsigned)((mp + 31) / 32), std::min(nb, 65535));
    transpose_blocks_kernel<<<grid, dim3(32, 8), 0, st>>>(pool, pl.upload(ti), pool, pl.upload(to), nb, (int)mp);
    CK_LAUNCH();
  }

  // ---- partition tree inverse rows (ref dichotomy.py:134-146, 298-304)
  pl.nodes = partition_tree(nr, &pl.depth);
  const int nn = (int)pl.nodes.size();
  std::vector<int64_t> nb0(nn), sz(nn), roff(nn), rld(nn), eoff(nn + 1);
  int64_t tot = 0, rtot = 0;
  int64_t maxlevel = 0;
  // Large blocks store every node's rows with one common row stride (the widest
  // node), so the series-sum GEMM sees a plain strided operand (TMA tensor map).
  // (only while the padding costs at most 2 GB: deep trees keep the compact layout)
  int64_t maxsz = 0, sumsz = 0;
  for (int b = 0; b < nn; ++b) {
    maxsz = std::max<int64_t>(maxsz, pl.nodes[b].hi - pl.nodes[b].lo + 1);
    sumsz += pl.nodes[b].hi - pl.nodes[b].lo + 1;
  }
  pl.r_ld = maxsz * mp;
  pl.r_uniform = mp >= 128 && ((int64_t)nn * maxsz - sumsz) * blk * (int64_t)sizeof(double) <= (int64_t(2) << 30);
  int64_t ecount = 0;
  for (int b = 0; b < nn; ++b) {
    sz[b] = pl.nodes[b].hi - pl.nodes[b].lo + 1;
    nb0[b] = tot;
    tot += sz[b];
    rld[b] = pl.r_uniform ? pl.r_ld : sz[b] * mp;
    roff[b] = pl.r_uniform ? (int64_t)b * mp * pl.r_ld : rtot;
    eoff[b] = ecount;
    ecount += sz[b] * blk;
    rtot = pl.r_uniform ? (int64_t)(b + 1) * mp * pl.r_ld : rtot + sz[b] * blk;
    maxlevel = std::max(maxlevel, pl.nodes[b].level);
  }
  eoff[nn] = ecount;
  DevBuf tp, tfs, tfc, ws;
  double* T = nullptr;
  const int64_t tpY = 3 * tot;
  if (!restore) {
  const int64_t tpD = 0, tpS = tot, tpAD = 2 * tot, tpDt = 4 * tot;
  tp.alloc((size_t)(4 * tot + nn) * blk * sizeof(double));
  CK(cudaMemsetAsync(tp.p, 0, (size_t)(4 * tot + nn) * blk * sizeof(double), st));
  tfs.alloc(sizeof(int32_t) * nn);
  tfc.alloc(sizeof(int32_t) * nn);
  CK(cudaMemsetAsync(tfs.p, 0xff, sizeof(int32_t) * nn, st));
  T = tp.d();
  StagedUploads stg(st);
  for (int64_t lev = 0; lev <= maxlevel; ++lev) {
    std::vector<int> ids;
    int64_t smax = 0;
    for (int b = 0; b < nn; ++b)
      if (pl.nodes[b].level == lev) { ids.push_back(b); smax = std::max(smax, sz[b]); }
    for (int64_t i = 0; i < smax; ++i) {
      std::vector<int64_t> dt_c, dt_in, dt_a, dt_b, inv_in, inv_out, sc, sa, sb, ac, aa, ab, failidx;
      for (int b : ids) {
        if (sz[b] <= i) continue;
        const int64_t lo = pl.nodes[b].lo;
        dt_c.push_back(tpDt + b);
        dt_in.push_back(pl.off_RdT + lo + i);
        dt_a.push_back(i >= 1 ? pl.off_RuT + lo + i - 1 : pl.off_Z);
        dt_b.push_back(i >= 1 ? tpS + nb0[b] + i - 1 : 0);
        inv_in.push_back(tpDt + b);
        inv_out.push_back(tpD + nb0[b] + i);
        failidx.push_back(b);
        if (i + 1 < sz[b]) {  // S'_i = D'^{-1}_i T.upper = D'^{-1} Rl^T_{lo+i}
          sc.push_back(tpS + nb0[b] + i); sa.push_back(tpD + nb0[b] + i); sb.push_back(pl.off_RlT + lo + i);
        }
        if (i >= 1) {  // AD'_i = D'^{-1}_i T.lower[i-1] = D'^{-1} Ru^T_{lo+i-1}
          ac.push_back(tpAD + nb0[b] + i); aa.push_back(tpD + nb0[b] + i); ab.push_back(pl.off_RuT + lo + i - 1);
        }
      }
      const int cnt = (int)dt_c.size();
      if (i == 0)
        launch_gemm(mp, mp, cnt, mk(T, stg.put(dt_c), 0, blk, mp), mk(pool, stg.put(dt_in), 0, blk, mp), 1.0, {}, st);
      else
        launch_gemm(mp, mp, cnt, mk(T, stg.put(dt_c), 0, blk, mp), mk(pool, stg.put(dt_in), 0, blk, mp), 1.0,
                    {term(mk(pool, stg.put(dt_a), 0, blk, mp), mk(T, stg.put(dt_b), 0, blk, mp), mp, -1.0)}, st);
      launch_inv(pl, cnt, T, stg.put(inv_in), 0, T, stg.put(inv_out), 0, (int)i, tfs.i32(), tfc.i32(), ws, st,
                 stg.put(failidx));
      if (!sc.empty())
        launch_gemm(mp, mp, (int)sc.size(), mk(T, stg.put(sc), 0, blk, mp), none(), 0.0,
                    {term(mk(T, stg.put(sa), 0, blk, mp), mk(pool, stg.put(sb), 0, blk, mp), mp)}, st);
      if (!ac.empty())
        launch_gemm(mp, mp, (int)ac.size(), mk(T, stg.put(ac), 0, blk, mp), none(), 0.0,
                    {term(mk(T, stg.put(aa), 0, blk, mp), mk(pool, stg.put(ab), 0, blk, mp), mp)}, st);
    }
    // forward solve with unit RHS at kk = k - lo: y_kk = D'^{-1}_kk ; y_i = AD'_i y_{i-1}
    for (int64_t i = 0; i < smax; ++i) {
      std::vector<int64_t> cc, ci, gc, ga, gb;
      for (int b : ids) {
        const int64_t kk = pl.nodes[b].k - pl.nodes[b].lo;
        if (i >= sz[b]) continue;
        if (i == kk) { cc.push_back(tpY + nb0[b] + i); ci.push_back(tpD + nb0[b] + i); }
        else if (i > kk) { gc.push_back(tpY + nb0[b] + i); ga.push_back(tpAD + nb0[b] + i); gb.push_back(tpY + nb0[b] + i - 1); }
      }
      if (!cc.empty())
        launch_gemm(mp, mp, (int)cc.size(), mk(T, stg.put(cc), 0, blk, mp), mk(T, stg.put(ci), 0, blk, mp), 1.0, {}, st);
      if (!gc.empty())
        launch_gemm(mp, mp, (int)gc.size(), mk(T, stg.put(gc), 0, blk, mp), none(), 0.0,
                    {term(mk(T, stg.put(ga), 0, blk, mp), mk(T, stg.put(gb), 0, blk, mp), mp)}, st);
    }
    // backward: y_i += S'_i y_{i+1}
    for (int64_t i = smax - 2; i >= 0; --i) {
      std::vector<int64_t> c, a, bb;
      for (int b : ids) {
        if (i + 1 >= sz[b]) continue;
        c.push_back(tpY + nb0[b] + i); a.push_back(tpS + nb0[b] + i); bb.push_back(tpY + nb0[b] + i + 1);
      }
      if (!c.empty()) {
        const int64_t* dc = stg.put(c);
        launch_gemm(mp, mp, (int)c.size(), mk(T, dc, 0, blk, mp), mk(T, dc, 0, blk, mp), 1.0,
                    {term(mk(T, stg.put(a), 0, blk, mp), mk(T, stg.put(bb), 0, blk, mp), mp)}, st);
      }
    }
  }
  {  // tree failures: first node in BFS order (ref dichotomy.py:298-304 loop order)
    std::vector<int32_t> fs(nn);
    CK(cudaMemcpyAsync(fs.data(), tfs.p, sizeof(int32_t) * nn, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < nn; ++b)
      if (fs[b] >= 0) {
        *err_row = fs[b];
        char buf[160];
        snprintf(buf, sizeof buf, "block row %d: singular pivot (reduced system, tree node %d)", fs[b], b);
        fail(BTD_ERR_SINGULAR_PIVOT, buf);
      }
  }
  }  // !restore
  // R rows, then E = R[:, :mp] Rl_{lo-1}, H = R[:, -mp:] Ru_{hi}
  pl.Rrows.alloc((size_t)rtot * sizeof(double));
  if (!restore) {
    std::vector<int64_t> ynb0(nn);
    for (int b = 0; b < nn; ++b) ynb0[b] = tpY + nb0[b];
    if (pl.r_uniform) CK(cudaMemsetAsync(pl.Rrows.p, 0, (size_t)rtot * sizeof(double), st));
    assemble_rows_kernel<<<1184, 256, 0, st>>>(T, pl.upload(ynb0), pl.upload(roff), pl.upload(rld), pl.upload(sz),
                                              pl.upload(eoff), nn, ecount, (int)mp, pl.Rrows.d());
    CK_LAUNCH();
  }
  pl.d_roff = pl.upload(roff);
  pl.d_rld = pl.upload(rld);
  pl.EH.alloc((size_t)2 * nn * blk * sizeof(double));
  if (!restore) {
    CK(cudaMemsetAsync(pl.EH.p, 0, (size_t)2 * nn * blk * sizeof(double), st));
    std::vector<int64_t> ec, ea, eld, eb, hc, ha, hld, hb;
    for (int b = 0; b < nn; ++b) {
      const Node& nd = pl.nodes[b];
      if (nd.lo >= 1) { ec.push_back(2 * b); ea.push_back(roff[b]); eld.push_back(rld[b]); eb.push_back(pl.off_Rl + nd.lo - 1); }
      if (nd.hi <= nr - 2) {
        hc.push_back(2 * b + 1); ha.push_back(roff[b] + (sz[b] - 1) * mp); hld.push_back(rld[b]);
        hb.push_back(pl.off_Ru + nd.hi);
      }
    }
    if (!ec.empty())
      launch_gemm(mp, mp, (int)ec.size(), mk(pl.EH.d(), pl.upload(ec), 0, blk, mp), none(), 0.0,
                  {term(mk(pl.Rrows.d(), pl.upload(ea), 0, 1, 0, pl.upload(eld)), mk(pool, pl.upload(eb), 0, blk, mp), mp)},
                  st);
    if (!hc.empty())
      launch_gemm(mp, mp, (int)hc.size(), mk(pl.EH.d(), pl.upload(hc), 0, blk, mp), none(), 0.0,
                  {term(mk(pl.Rrows.d(), pl.upload(ha), 0, 1, 0, pl.upload(hld)), mk(pool, pl.upload(hb), 0, blk, mp), mp)},
                  st);
  }
  {  // solve-time batches over the nodes this rank needs
    // x~ needed for own interfaces q0..q1-1 and the right neighbour q1; node k needs x~_{lo-1}, x~_{hi+1}
    auto needed = [&](int64_t q0, int64_t q1) {
      std::vector<char> need(nr + 1, 0);
      for (int64_t q = q0; q <= std::min(q1, nr - 1); ++q) need[q] = 1;
      for (bool changed = true; changed;) {
        changed = false;
        for (int b = nn - 1; b >= 0; --b) {
          const Node& nd = pl.nodes[b];
          if (!need[nd.k]) continue;
          if (nd.lo >= 1 && !need[nd.lo - 1]) { need[nd.lo - 1] = 1; changed = true; }
          if (nd.hi + 1 <= nr - 1 && !need[nd.hi + 1]) { need[nd.hi + 1] = 1; changed = true; }
        }
      }
      return need;
    };
    const std::vector<char> need_k = needed(pl.q0, pl.q1);
    // crossing nodes: needed by some rank, segment not inside that rank's ranges (same list on every rank)
    std::vector<char> crossing(nn, 0);
    if (pl.world > 1) {
      for (int r = 0; r < pl.world; ++r) {
        const int64_t a0 = r * pl.nrl, a1 = (r + 1) * pl.nrl;
        const std::vector<char> nr_ = needed(a0, a1);
        for (int b = 0; b < nn; ++b)
          if (nr_[pl.nodes[b].k] && (pl.nodes[b].lo < a0 || pl.nodes[b].hi >= a1)) crossing[b] = 1;
      }
    }
    std::vector<int64_t> zid, zro, zrl, znl;
    for (int b = 0; b < nn; ++b)
      if (need_k[pl.nodes[b].k] && !crossing[b]) {
        zid.push_back(b); zro.push_back(roff[b]); zrl.push_back(rld[b]); znl.push_back(pl.nodes[b].lo);
      }
    pl.nz = (int)zid.size();
    pl.z_id = pl.upload(zid); pl.z_roff = pl.upload(zro); pl.z_rld = pl.upload(zrl); pl.z_nlo = pl.upload(znl);
    std::vector<int64_t> cn, cro, cld, ck, clo;
    for (int b = 0; b < nn; ++b) {
      if (!crossing[b]) continue;
      const Node& nd = pl.nodes[b];
      const int64_t a = std::max(nd.lo, pl.q0), e = std::min(nd.hi, pl.q1 - 1);
      cn.push_back(b);
      cld.push_back(rld[b]);
      if (a <= e) {
        cro.push_back(roff[b] + (a - nd.lo) * mp); ck.push_back((e - a + 1) * mp); clo.push_back(a);
      } else {
        cro.push_back(roff[b]); ck.push_back(0); clo.push_back(0);
      }
    }
    pl.ncross = (int)cn.size();
    pl.cross_node = pl.upload(cn); pl.cross_roff = pl.upload(cro); pl.cross_ld = pl.upload(cld);
    pl.cross_k = pl.upload(ck); pl.cross_lo = pl.upload(clo);
    pl.cross_kh = ck;
    std::vector<int64_t> nlo(nn);
    for (int b = 0; b < nn; ++b) nlo[b] = pl.nodes[b].lo;
    pl.d_nlo = pl.upload(nlo);
    pl.levels.assign(maxlevel + 1, btd_plan::Level());
    for (int64_t lev = 0; lev <= maxlevel; ++lev) {
      std::vector<int64_t> c, z, e, xl, h, xh, ek, hk;
      for (int b = 0; b < nn; ++b) {
        const Node& nd = pl.nodes[b];
        if (nd.level != lev || !need_k[nd.k]) continue;
        c.push_back(nd.k); z.push_back(b); e.push_back(2 * b); h.push_back(2 * b + 1);
        xl.push_back(nd.lo >= 1 ? nd.lo - 1 : nr);
        xh.push_back(nd.hi + 1 <= nr - 1 ? nd.hi + 1 : nr);
        ek.push_back(nd.lo >= 1 ? mp : 0);
        hk.push_back(nd.hi + 1 <= nr - 1 ? mp : 0);
      }
      auto& L_ = pl.levels[lev];
      L_.count = (int)c.size();
      L_.c_idx = pl.upload(c); L_.z_idx = pl.upload(z); L_.e_idx = pl.upload(e);
      L_.xl_idx = pl.upload(xl); L_.h_idx = pl.upload(h); L_.xh_idx = pl.upload(xh);
      L_.e_k = pl.upload(ek); L_.h_k = pl.upload(hk);
      L_.copy_only = std::all_of(ek.begin(), ek.end(), [](int64_t v) { return v == 0; }) &&
                     std::all_of(hk.begin(), hk.end(), [](int64_t v) { return v == 0; });
    }
    // split-K plans: enough CTAs (>= 2 waves) for the series sums and the level corrections
    pl.z_k.clear();
    for (int b = 0; b < nn; ++b)
      if (need_k[pl.nodes[b].k] && !crossing[b]) pl.z_k.push_back(sz[b] * mp);
    pl.z_kd = pl.upload(pl.z_k);
    build_splits(pl);
    // fused cooperative tree for small blocks on a single rank
    const char* ft_env = getenv("BTD_FUSED_TREE");
    if (pl.mode == 0 && mp <= 32 && pl.world == 1 && (!ft_env || atoi(ft_env))) {
      constexpr int CH = 16;
      std::vector<int32_t> chn, chb, chc, zco(nn, 0), zcc(nn, 0), he(nn, 0), hh(nn, 0), lvo, lvn;
      std::vector<int64_t> klist(nn), xlv(nn), xhv(nn);
      for (int b = 0; b < nn; ++b) {
        const Node& nd = pl.nodes[b];
        klist[b] = nd.k;
        xlv[b] = nd.lo >= 1 ? nd.lo - 1 : nr;
        xhv[b] = nd.hi + 1 <= nr - 1 ? nd.hi + 1 : nr;
        he[b] = nd.lo >= 1;
        hh[b] = nd.hi + 1 <= nr - 1;
        if (!need_k[nd.k]) continue;
        zco[b] = (int32_t)chn.size();
        for (int64_t b0 = 0; b0 < sz[b]; b0 += CH) {
          chn.push_back(b); chb.push_back((int32_t)b0); chc.push_back((int32_t)std::min<int64_t>(CH, sz[b] - b0));
        }
        zcc[b] = (int32_t)chn.size() - zco[b];
      }
      for (int64_t lev = 0; lev <= maxlevel; ++lev) {
        lvo.push_back((int32_t)lvn.size());
        for (int b = 0; b < nn; ++b)
          if (pl.nodes[b].level == lev && need_k[pl.nodes[b].k]) lvn.push_back(b);
      }
      lvo.push_back((int32_t)lvn.size());
      TreeArgs& ta = pl.targs;
      ta.nchunks = (int)chn.size();
      ta.nlev = (int)maxlevel + 1;
      ta.ch_node = pl.upload(chn); ta.ch_blk0 = pl.upload(chb); ta.ch_nblk = pl.upload(chc);
      ta.roff = pl.upload(roff); ta.rld = pl.upload(rld); ta.lo = pl.d_nlo ? pl.d_nlo : nullptr;
      ta.k = pl.upload(klist); ta.zc_off = pl.upload(zco); ta.zc_cnt = pl.upload(zcc);
      ta.xl = pl.upload(xlv); ta.xh = pl.upload(xhv); ta.has_e = pl.upload(he); ta.has_h = pl.upload(hh);
      ta.lv_off = pl.upload(lvo); ta.lv_nodes = pl.upload(lvn);
      pl.tree_chunks = ta.nchunks;
      pl.fused_tree = true;
    }
    if (pl.mode == 0 && mp <= 32 && (!ft_env || atoi(ft_env))) {  // (a world-1 shard plan uses it too)
      constexpr int CH = 16;
      std::vector<int64_t> cro_, crld_, cflo_, odst, klist(nn), xlv(nn), xhv(nn);
      std::vector<int32_t> cnb_, ooff, ocnt, he(nn, 0), hh(nn, 0), lvo, lvn;
      auto add_out = [&](int64_t dst, int64_t r0, int64_t ld, int64_t f0, int64_t nblk) {
        ooff.push_back((int32_t)cro_.size());
        for (int64_t b0 = 0; b0 < nblk; b0 += CH) {
          cro_.push_back(r0 + b0 * mp); crld_.push_back(ld); cflo_.push_back(f0 + b0);
          cnb_.push_back((int32_t)std::min<int64_t>(CH, nblk - b0));
        }
        ocnt.push_back((int32_t)cro_.size() - ooff.back());
        odst.push_back(dst);
      };
      for (int b = 0; b < nn; ++b)  // nodes inside this rank: full series sums
        if (need_k[pl.nodes[b].k] && !crossing[b]) add_out(b, roff[b], rld[b], pl.nodes[b].lo, sz[b]);
      int64_t ci = 0;
      for (int b = 0; b < nn; ++b) {  // crossing nodes: this rank's share (same order as cross_node)
        if (!crossing[b]) continue;
        const Node& nd = pl.nodes[b];
        const int64_t a = std::max(nd.lo, pl.q0), e = std::min(nd.hi, pl.q1 - 1);
        add_out(-1 - ci, roff[b] + std::max<int64_t>(0, a - nd.lo) * mp, rld[b], a, a <= e ? e - a + 1 : 0);
        ++ci;
      }
      for (int b = 0; b < nn; ++b) {
        const Node& nd = pl.nodes[b];
        klist[b] = nd.k;
        xlv[b] = nd.lo >= 1 ? nd.lo - 1 : nr;
        xhv[b] = nd.hi + 1 <= nr - 1 ? nd.hi + 1 : nr;
        he[b] = nd.lo >= 1;
        hh[b] = nd.hi + 1 <= nr - 1;
      }
      for (int64_t lev = 0; lev <= maxlevel; ++lev) {
        lvo.push_back((int32_t)lvn.size());
        for (int b = 0; b < nn; ++b)
          if (pl.nodes[b].level == lev && need_k[pl.nodes[b].k]) lvn.push_back(b);
      }
      lvo.push_back((int32_t)lvn.size());
      ShardTreeArgs& sa = pl.sargs;
      sa.nchunks = (int)cro_.size();
      sa.nout = (int)odst.size();
      sa.ncross = pl.ncross;
      sa.nlev = (int)maxlevel + 1;
      sa.world = pl.world;
      sa.ch_roff = pl.upload(cro_); sa.ch_rld = pl.upload(crld_); sa.ch_flo = pl.upload(cflo_);
      sa.ch_nblk = pl.upload(cnb_);
      sa.out_off = pl.upload(ooff); sa.out_cnt = pl.upload(ocnt); sa.out_dst = pl.upload(odst);
      sa.cross_node = pl.cross_node;
      sa.lv_off = pl.upload(lvo); sa.lv_nodes = pl.upload(lvn);
      sa.k = pl.upload(klist); sa.xl = pl.upload(xlv); sa.xh = pl.upload(xhv);
      sa.has_e = pl.upload(he); sa.has_h = pl.upload(hh);
      int maxlev = 0;
      for (size_t l = 0; l + 1 < lvo.size(); ++l) maxlev = std::max(maxlev, lvo[l + 1] - lvo[l]);
      pl.shard_chunks = std::max(sa.nchunks, 1);
      pl.shard_work_b = std::max(sa.nchunks, sa.nout);
      pl.shard_work_c = std::max(pl.ncross, maxlev);
      pl.fused_shard = true;
    }
  }
  CK(cudaStreamSynchronize(st));
  pl.factor_bytes += (int64_t)(rtot + 2 * nn * blk) * sizeof(double);
  pl.finished = true;
}

// ---------------------------------------------------------------- solve
void ensure_scratch(btd_plan& pl, int64_t K) {
  auto& S = pl.S();
  if (S.k == K) return;
  std::vector<btd_plan::GraphEntry> keep;  // graphs of this slot point at the old buffers
  for (auto& g : pl.graphs)
    if (g.slot == pl.cur) { if (g.exec) cudaGraphExecDestroy(g.exec); } else keep.push_back(g);
  pl.graphs.swap(keep);
  const int64_t mpK = pl.mp * K;
  S.ft.alloc((size_t)pl.nr * mpK * sizeof(double));
  S.zbuf.alloc((size_t)pl.nodes.size() * mpK * sizeof(double));
  S.xt.alloc((size_t)(pl.nr + 1) * mpK * sizeof(double));
  CK(cudaMemset(S.xt.p, 0, (size_t)(pl.nr + 1) * mpK * sizeof(double)));
  CK(cudaMemset(S.ft.p, 0, (size_t)pl.nr * mpK * sizeof(double)));
  if (pl.fused_tree || pl.fused_shard)
    S.tpartial.alloc((size_t)std::max({pl.tree_chunks, pl.shard_chunks, 1}) * pl.mp * K * sizeof(double));
  size_t pbytes = (size_t)pl.partial_elems_per_k * K * sizeof(double);
  if (pl.mode == 1) {  // split-K maps for row steps whose batch is under one wave
    for (const auto& st1 : pl.steps1)
      for (int cnt : {st1.cnt, st1.nx, st1.nt}) {
        const int64_t tiles = ((pl.m + 127) / 128) * ((K + 63) / 64);
        if (cnt <= 0 || cnt * tiles >= 148) continue;
        auto it = pl.step_splits.find({cnt, K});
        if (it == pl.step_splits.end()) {  // (maps are per plan; the partials buffer is per slot)
          int64_t maxz = 0;
          it = pl.step_splits.emplace(std::make_pair(cnt, K),
                                      make_split(pl, std::vector<int64_t>(cnt, pl.mp), tiles, maxz)).first;
        }
        pbytes = std::max(pbytes, (size_t)it->second.ntotal * pl.mp * K * sizeof(double));
      }
  }
  if (pbytes) S.partial.alloc(pbytes);
  if (pl.mode == 1 && pl.scoup) S.ubuf.alloc((size_t)std::max<int64_t>(pl.nrl, 1) * pl.m * K * sizeof(double));
  S.k = K;
}


const SplitK* step_split(btd_plan& pl, int cnt, int64_t K);

ChainArgs chain_args(btd_plan& pl, const double* F, double* X, int64_t K, double* base, int64_t base_stride) {
  const int64_t blk = pl.blk;
  double* pool = pl.pool.d();
  ChainArgs a;
  a.lo = pl.d_lo; a.nint = pl.d_nint; a.slot0 = pl.d_slot0; a.nr = (int)pl.nrl;
  a.m = (int)pl.m; a.n = pl.nloc; a.K = K; a.F = F; a.X = X;
  a.AD = pool + pl.off_AD * blk; a.Dinv = pool + pl.off_Dinv * blk; a.Tb = pool + pl.off_Tb * blk;
  a.S = pool + pl.off_S * blk; a.G = pool + pl.off_G * blk;
  a.base = base; a.base_stride = base_stride;
  a.xt = pl.S().xt.d() + pl.q0 * pl.mp * K;
  return a;
}

}  // namespace
namespace btd {
// Mode 1, scalar-coupled plan: u_b = F[lo_b + 1 + j] + a_{slot0_b + j} X[lo_b + j] for the live ranges b
__global__ void sc_axpy_kernel(double* U, const double* F, const double* X, const int64_t* lo, const int64_t* slot0,
                               const double* alpha, int64_t j, int64_t mK) {
  const int b = blockIdx.y;
  const double a = alpha[slot0[b] + j];
  const double* f = F + (lo[b] + 1 + j) * mK;
  const double* y = X + (lo[b] + j) * mK;
  double* u = U + (int64_t)b * mK;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mK; e += (int64_t)gridDim.x * blockDim.x)
    u[e] = fma(a, y[e], f[e]);
}
}  // namespace btd
namespace {

// Forward sweeps of the owned ranges: y rows into X, base_q into base (+ q*base_stride)
void solve_forward(btd_plan& pl, const double* F, double* X, int64_t K, double* base, int64_t base_stride,
                   cudaStream_t st) {
  const int64_t mp = pl.mp, m = pl.m, blk = pl.blk;
  const int64_t mK = m * K;
  double* pool = pl.pool.d();
  if (pl.mode == 0) {  // each CTA owns its (rows, columns): in-place F == X is safe
    const ScPools scp{pool + pl.off_Tbd * blk, pool + pl.off_al * blk};
    launch_chain(mp, chain_args(pl, F, X, K, base, base_stride), true, st, pl.scoup ? &scp : nullptr);
    return;
  }
  // mode 1: a step's GEMM reads all of F[g] as its reduction operand while other
  // CTAs write X[g]; stage F when the caller solves in place.
  const size_t fbytes = (size_t)pl.nloc * mK * sizeof(double);
  const char *f0 = (const char*)F, *x0 = (const char*)X;
  if (fbytes && f0 < x0 + fbytes && x0 < f0 + fbytes) {
    auto& fc = pl.S().fcopy;
    if (fc.bytes < fbytes) fc.alloc(fbytes);
    CK(cudaMemcpyAsync(fc.p, F, fbytes, cudaMemcpyDeviceToDevice, st));
    F = fc.d();
  }
  // mode 1: base_q = F[lo_q] (rows < m; pad rows stay 0), then one GEMM launch per row step.
  // base += Tb_j y_j only reads y_j, like row j+1's product: without split-K (whose partials
  // buffer is shared) it runs on a side stream beside the next row step, so the two
  // launches' CTAs pack into fewer waves (joined before the interface RHS).
  launch_gemm(m, K, pl.nlive, mk(base, nullptr, 0, base_stride, K), mk(F, pl.d_lo, 0, mK, K), 1.0, {}, st);
  auto& S = pl.S();
  const bool fork = pl.cap > 1 && pl.steps1[0].cnt > 0 && !step_split(pl, pl.steps1[0].cnt, K);
  if (fork && !S.side) {
    CK(cudaStreamCreateWithFlags(&S.side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&S.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.ev_join, cudaEventDisableTiming));
  }
  bool forked = false;
  for (int64_t j = 0; j < pl.cap; ++j) {
    const auto& s = pl.steps1[j];
    if (s.cnt == 0) break;
    const SplitK* ssp = step_split(pl, s.cnt, K);  // few ranges (sharded): split the reductions
    if (j == 0) {
      launch_gemm(m, K, s.cnt, mk(X, pl.d_lo, 1, mK, K), none(), 0.0,
                  {term(mk(pool, pl.d_slot0, pl.off_Dinv, blk, mp), mk(F, pl.d_lo, 1, mK, K), m)}, st, ssp);
    } else if (pl.scoup) {  // y_j = Dinv_j (f_g + a_g y_{j-1}): one product per row step instead of two
      double* U = S.ubuf.d();
      dim3 grid((unsigned)std::min<int64_t>((mK + 255) / 256, 296), (unsigned)s.cnt);
      btd::sc_axpy_kernel<<<grid, 256, 0, st>>>(U, F, X, pl.d_lo, pl.d_slot0, pool + pl.off_al * blk, j, mK);
      CK_LAUNCH();
      launch_gemm(m, K, s.cnt, mk(X, pl.d_lo, 1 + j, mK, K), none(), 0.0,
                  {term(mk(pool, pl.d_slot0, pl.off_Dinv + j, blk, mp), mk(U, nullptr, 0, mK, K), m)}, st, ssp);
    } else
      launch_gemm(m, K, s.cnt, mk(X, pl.d_lo, 1 + j, mK, K), none(), 0.0,
                  {term(mk(pool, pl.d_slot0, pl.off_Dinv + j, blk, mp), mk(F, pl.d_lo, 1 + j, mK, K), m),
                   term(mk(pool, pl.d_slot0, pl.off_AD + j, blk, mp), mk(X, pl.d_lo, j, mK, K), m)},
                  st, ssp);
    cudaStream_t tst = st;
    if (fork && !ssp) {
      CK(cudaEventRecord(S.ev_fork, st));
      CK(cudaStreamWaitEvent(S.side, S.ev_fork, 0));
      tst = S.side;
      forked = true;
    } else if (forked) {  // a split step (ragged ranges): finish the side's base updates first
      CK(cudaEventRecord(S.ev_join, S.side));
      CK(cudaStreamWaitEvent(st, S.ev_join, 0));
      forked = false;
    }
    launch_gemm(mp, K, s.cnt, mk(base, nullptr, 0, base_stride, K), mk(base, nullptr, 0, base_stride, K), 1.0,
                {term(mk(pool, pl.d_slot0, pl.off_Tb + j, blk, mp), mk(X, pl.d_lo, 1 + j, mK, K), m)}, tst,
                ssp);
  }
  if (forked) {
    CK(cudaEventRecord(S.ev_join, S.side));
    CK(cudaStreamWaitEvent(st, S.ev_join, 0));
  }
}

// z_node = R_node f~[lo..hi] for the needed nodes: reduction length size * mp per node
Term z_term(btd_plan& pl, double* ft, int64_t K) {
  const int64_t mpK = pl.mp * K;
  if (pl.r_uniform)  // node rows at b * mp * r_ld with stride r_ld: a plain strided operand
    return term(mk(pl.Rrows.d(), pl.z_id, 0, pl.mp * pl.r_ld, pl.r_ld), mk(ft, pl.z_nlo, 0, mpK, K), pl.mp, 1.0,
                pl.z_kd);
  return term(mk(pl.Rrows.d(), pl.z_roff, 0, 1, 0, pl.z_rld), mk(ft, pl.z_nlo, 0, mpK, K), 0, 1.0, pl.z_kd);
}

// split-K maps with the current scratch slot's partial buffer
const SplitK* split_with(const SplitK& sp, btd_plan& pl) {
  static thread_local SplitK tmp;
  tmp = sp;
  tmp.partial = pl.S().partial.d();
  return &tmp;
}

// split-K map for a mode-1 row-step GEMM of `cnt` entries (nullptr: plain launch)
const SplitK* step_split(btd_plan& pl, int cnt, int64_t K) {
  if (pl.host_concurrent) return nullptr;  // concurrent chunk solves already fill the GPU
  auto it = pl.step_splits.find({cnt, K});
  if (it == pl.step_splits.end() || it->second.ntotal == 0) return nullptr;
  return split_with(it->second, pl);
}

// dst[dst_idx[b]] = src[src_idx[b]], blocks of `per` doubles
}  // namespace
namespace btd {  // (::btd: launch lists attribute it to this library)
__global__ void copy_blocks_kernel(double* dst, const int64_t* dst_idx, const double* src, const int64_t* src_idx,
                                   int count, int64_t per) {
  for (int b = blockIdx.y; b < count; b += gridDim.y) {
    double* d = dst + dst_idx[b] * per;
    const double* sp = src + src_idx[b] * per;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x)
      d[e] = sp[e];
  }
}
}  // namespace btd
namespace {

// Algorithm 1, level part: x~_k = z_node + E x~_{lo-1} + H x~_{hi+1}, level by level.
void solve_levels(btd_plan& pl, int64_t K, cudaStream_t st) {
  const int64_t mp = pl.mp, blk = pl.blk, mpK = mp * K;
  double* xt = pl.S().xt.d();
  double* z = pl.S().zbuf.d();
  for (const auto& lev : pl.levels) {
    if (lev.count <= 0) continue;
    if (lev.copy_only) {  // the root level: x~_k = z_root, a copy, not a GEMM + split-K reduction
      dim3 grid((unsigned)std::min<int64_t>((mpK + 255) / 256, 592), (unsigned)std::min(lev.count, 65535));
      btd::copy_blocks_kernel<<<grid, 256, 0, st>>>(xt, lev.c_idx, z, lev.z_idx, lev.count, mpK);
      CK_LAUNCH();
      continue;
    }
    launch_gemm(mp, K, lev.count, mk(xt, lev.c_idx, 0, mpK, K), mk(z, lev.z_idx, 0, mpK, K), 1.0,
                {term(mk(pl.EH.d(), lev.e_idx, 0, blk, mp), mk(xt, lev.xl_idx, 0, mpK, K), mp, 1.0, lev.e_k),
                 term(mk(pl.EH.d(), lev.h_idx, 0, blk, mp), mk(xt, lev.xh_idx, 0, mpK, K), mp, 1.0, lev.h_k)},
                st, split_with(lev.split, pl));
  }
}

template <int MP>
void launch_tree_small(btd_plan& pl, int64_t K, cudaStream_t st) {
  int max_blocks = 0, nsm = 0, dev = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks, tree_small_kernel<MP>, 256, 0));
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  TreeArgs ta = pl.targs;
  ta.K = K;
  ta.R = pl.Rrows.d();
  ta.EH = pl.EH.d();
  ta.ft = pl.S().ft.d();
  ta.partial = pl.S().tpartial.d();
  ta.xt = pl.S().xt.d();
  const int ntile = (int)((K + 15) / 16);
  const int64_t work = (int64_t)std::max(ta.nchunks, 1) * ntile;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)max_blocks * nsm, (work + 7) / 8));
  void* args[] = {&ta};
  CK(cudaLaunchCooperativeKernel((const void*)tree_small_kernel<MP>, dim3(grid), dim3(256), args, 0, st));
  CK_LAUNCH();
}

// Sharded fused tree: phase B (series sums + crossing partials) or C (crossing sums + levels).
template <int MP>
void launch_tree_shard(btd_plan& pl, int64_t K, bool phase_b, double* part_out, const double* part_all,
                       cudaStream_t st) {
  const void* fn = phase_b ? (const void*)tree_shard_b_kernel<MP> : (const void*)tree_shard_c_kernel<MP>;
  int max_blocks = 0, nsm = 0, dev = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks, fn, 256, 0));
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  ShardTreeArgs sa = pl.sargs;
  sa.K = K;
  sa.R = pl.Rrows.d();
  sa.EH = pl.EH.d();
  sa.ft = pl.S().ft.d();
  sa.partial = pl.S().tpartial.d();
  sa.z = pl.S().zbuf.d();
  sa.xt = pl.S().xt.d();
  sa.part_out = part_out;
  sa.part_all = part_all;
  const int ntile = (int)((K + 15) / 16);
  const int64_t work = (int64_t)std::max(phase_b ? pl.shard_work_b : pl.shard_work_c, 1) * ntile;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)max_blocks * nsm, (work + 7) / 8));
  void* args[] = {&sa};
  CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, 0, st));
  CK_LAUNCH();
}

void tree_shard(btd_plan& pl, int64_t K, bool phase_b, double* part_out, const double* part_all,
                cudaStream_t st) {
  switch (pl.mp) {
    case 8: launch_tree_shard<8>(pl, K, phase_b, part_out, part_all, st); break;
    case 16: launch_tree_shard<16>(pl, K, phase_b, part_out, part_all, st); break;
    case 32: launch_tree_shard<32>(pl, K, phase_b, part_out, part_all, st); break;
    default: fail(BTD_ERR_UNSUPPORTED, "fused shard tree: block order > 32");
  }
}

// Algorithm 1 on the interface system: z = R f~ (all needed nodes), then the levels.
void solve_tree(btd_plan& pl, int64_t K, cudaStream_t st) {
  const int64_t mp = pl.mp, mpK = mp * K;
  if (pl.fused_tree) {
    switch (mp) {
      case 8: launch_tree_small<8>(pl, K, st); return;
      case 16: launch_tree_small<16>(pl, K, st); return;
      case 32: launch_tree_small<32>(pl, K, st); return;
      default: break;
    }
  }
  launch_gemm(mp, K, pl.nz, mk(pl.S().zbuf.d(), pl.z_id, 0, mpK, K), none(), 0.0, {z_term(pl, pl.S().ft.d(), K)},
              st, split_with(pl.z_split, pl));
  solve_levels(pl, K, st);
}

// Backward sweeps of the owned ranges (x~ known), x[lo_q] = x~_q.
void solve_backward(btd_plan& pl, const double* F, double* X, int64_t K, cudaStream_t st) {
  const int64_t mp = pl.mp, m = pl.m, blk = pl.blk, mpK = mp * K, mK = m * K;
  double* pool = pl.pool.d();
  double* xt = pl.S().xt.d() + pl.q0 * mpK;
  if (pl.mode == 0) {
    launch_chain(mp, chain_args(pl, F, X, K, nullptr, 0), false, st);
    return;
  }
  launch_gemm(m, K, pl.nlive, mk(X, pl.d_lo, 0, mK, K), mk(xt, nullptr, 0, mpK, K), 1.0, {}, st);
  for (int64_t j = pl.cap - 1; j >= 0; --j) {
    const auto& s = pl.steps1[j];
    // x_j = y_j + G_j x~_q + S_j x_{j+1}   (x_{j+1} an interior row)
    launch_gemm(m, K, s.nx, mk(X, s.x_row, 0, mK, K), mk(X, s.x_row, 0, mK, K), 1.0,
                {term(mk(pool, s.x_slot, pl.off_G, blk, mp), mk(xt, s.x_q, 0, mpK, K), mp),
                 term(mk(pool, s.x_slot, pl.off_S, blk, mp), mk(X, s.x_row, 1, mK, K), m)},
                st, step_split(pl, s.nx, K));
    // last interior row: x_{j+1} = x~_{q+1}
    launch_gemm(m, K, s.nt, mk(X, s.t_row, 0, mK, K), mk(X, s.t_row, 0, mK, K), 1.0,
                {term(mk(pool, s.t_slot, pl.off_G, blk, mp), mk(xt, s.t_q, 0, mpK, K), mp),
                 term(mk(pool, s.t_slot, pl.off_S, blk, mp), mk(xt, s.t_q, 1, mpK, K), mp)},
                st, step_split(pl, s.nt, K));
  }
}

// Single-device solve: forward -> interface RHS -> tree -> backward.
void solve_device(btd_plan& pl, const double* F, double* X, int64_t K, cudaStream_t st) {
  const int64_t mp = pl.mp, m = pl.m, blk = pl.blk, mpK = mp * K, mK = m * K;
  double* ft = pl.S().ft.d();
  pl.ev_mark(st);
  solve_forward(pl, F, X, K, ft, mpK, st);
  pl.ev_mark(st);
  // f~_{q+1} += Fc_q y_{q,last}   (ref dichotomy.py:239-276)
  launch_gemm(mp, K, pl.ncarry, mk(ft, pl.carry_src, 1, mpK, K), mk(ft, pl.carry_src, 1, mpK, K), 1.0,
              {term(mk(pl.pool.d(), pl.carry_fc, 0, blk, mp), mk(X, pl.carry_row, 0, mK, K), m)}, st);
  solve_tree(pl, K, st);
  pl.ev_mark(st);
  solve_backward(pl, F, X, K, st);
  pl.ev_mark(st);
}

// Repeated (F, X, K) solves replay a CUDA graph of the whole launch sequence
// (captured on the plan's own stream at the second call, after the first call
// has set kernel attributes and scratch); the caller's stream is joined with events.
void solve_graphed(btd_plan& pl, const double* F, double* X, int64_t K, cudaStream_t st) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("BTD_GRAPHS");
    enabled = e ? atoi(e) : 1;
  }
  if (!enabled || pl.profiling) {
    solve_device(pl, F, X, K, st);
    return;
  }
  btd_plan::GraphEntry* ge = nullptr;
  for (auto& g : pl.graphs)
    if (g.F == F && g.X == X && g.K == K && g.slot == pl.cur) ge = &g;
  if (!ge) {
    if (pl.graphs.size() >= 24) {  // bounded cache (host pipeline: up to kHostBufs x kSlots keys)
      if (pl.graphs.front().exec) cudaGraphExecDestroy(pl.graphs.front().exec);
      pl.graphs.erase(pl.graphs.begin());
    }
    pl.graphs.push_back({F, X, K, pl.cur, 0, nullptr, 0});
    ge = &pl.graphs.back();
  }
  if (++ge->calls < 2) {
    solve_device(pl, F, X, K, st);
    return;
  }
  auto& S = pl.S();
  if (!S.own) {
    CK(cudaStreamCreateWithFlags(&S.own, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&S.ev_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.ev_out, cudaEventDisableTiming));
  }
  if (!ge->exec) {
    cudaGraph_t graph;
    const int64_t l0 = g_launches.load();
    CK(cudaStreamBeginCapture(S.own, cudaStreamCaptureModeThreadLocal));
    try {
      solve_device(pl, F, X, K, S.own);
    } catch (...) {
      cudaStreamEndCapture(S.own, &graph);
      throw;
    }
    CK(cudaStreamEndCapture(S.own, &graph));
    ge->nkern = g_launches.load() - l0;
    g_launches.fetch_sub(ge->nkern);  // counted when the graph runs, not when captured
    CK(cudaGraphInstantiate(&ge->exec, graph, 0));
    CK(cudaGraphDestroy(graph));
  }
  CK(cudaEventRecord(S.ev_in, st));
  CK(cudaStreamWaitEvent(S.own, S.ev_in, 0));
  CK(cudaGraphLaunch(ge->exec, S.own));
  g_launches.fetch_add(ge->nkern);
  CK(cudaEventRecord(S.ev_out, S.own));
  CK(cudaStreamWaitEvent(st, S.ev_out, 0));
}

// Sharded phase A: local sweeps (base into f~), internal carries, and the carry of
// the last owned range for the next rank (carry_out: mp x K, zero if none).
void solve_shard_a(btd_plan& pl, const double* F, double* X, int64_t K, double* carry_out, cudaStream_t st) {
  const int64_t mp = pl.mp, m = pl.m, blk = pl.blk, mpK = mp * K, mK = m * K;
  double* ft = pl.S().ft.d() + pl.q0 * mpK;
  CK(cudaMemsetAsync(carry_out, 0, (size_t)mpK * sizeof(double), st));
  pl.ev_mark(st);
  solve_forward(pl, F, X, K, ft, mpK, st);
  pl.ev_mark(st);
  launch_gemm(mp, K, pl.ncarry, mk(ft, pl.carry_src, 1, mpK, K), mk(ft, pl.carry_src, 1, mpK, K), 1.0,
              {term(mk(pl.pool.d(), pl.carry_fc, 0, blk, mp), mk(X, pl.carry_row, 0, mK, K), m)}, st);
  launch_gemm(mp, K, pl.ncarry_out, mk(carry_out, nullptr, 0, mpK, K), none(), 0.0,
              {term(mk(pl.pool.d(), pl.cout_fc, 0, blk, mp), mk(X, pl.cout_row, 0, mK, K), m)}, st);
}

}  // namespace
namespace btd {  // (::btd: launch lists attribute it to this library)
__global__ void add_block_kernel(double* dst, const double* src, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] += src[e];
}
}  // namespace btd
namespace {

// z_b = sum over ranks (fixed order) of the partial series sums of crossing node c
}  // namespace
namespace btd {  // (::btd: launch lists attribute it to this library)
__global__ void sum_ranks_kernel(const double* part_all, int world, int ncross, int64_t per, const int64_t* node,
                                 double* z) {
  for (int c = blockIdx.y; c < ncross; c += gridDim.y) {
    double* zb = z + node[c] * per;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x) {
      double v = 0.0;
      for (int r = 0; r < world; ++r) v += part_all[((int64_t)r * ncross + c) * per + e];
      zb[e] = v;
    }
  }
}
}  // namespace btd
namespace {

// Sharded phase B: finish f~ of the first owned range with the previous rank's carry,
// local series sums of nodes inside this rank, partial sums of crossing nodes.
void solve_shard_b(btd_plan& pl, const double* carry_all, double* partial_out, int64_t K, cudaStream_t st) {
  const int64_t mp = pl.mp, mpK = mp * K;
  double* ft = pl.S().ft.d();
  if (pl.rank >= 1) {
    btd::add_block_kernel<<<64, 256, 0, st>>>(ft + pl.q0 * mpK, carry_all + (int64_t)(pl.rank - 1) * mpK, mpK);
    CK_LAUNCH();
  }
  if (pl.fused_shard) {
    tree_shard(pl, K, true, partial_out, nullptr, st);
    return;
  }
  launch_gemm(mp, K, pl.nz, mk(pl.S().zbuf.d(), pl.z_id, 0, mpK, K), none(), 0.0,
              {z_term(pl, ft, K)}, st,
              split_with(pl.z_split, pl));
  launch_gemm(mp, K, pl.ncross, mk(partial_out, nullptr, 0, mpK, K), none(), 0.0,
              {term(mk(pl.Rrows.d(), pl.cross_roff, 0, 1, 0, pl.cross_ld), mk(ft, pl.cross_lo, 0, mpK, K), 0, 1.0,
                    pl.cross_k)},
              st, split_with(pl.cross_split, pl));
}

// Sharded phase C: crossing-node sums, tree levels, local recovery.
void solve_shard_c(btd_plan& pl, const double* partial_all, const double* F, double* X, int64_t K, cudaStream_t st) {
  const int64_t mp = pl.mp, mpK = mp * K;
  if (pl.fused_shard) {
    tree_shard(pl, K, false, nullptr, partial_all, st);
    pl.ev_mark(st);
    solve_backward(pl, F, X, K, st);
    pl.ev_mark(st);
    return;
  }
  if (pl.ncross) {
    dim3 grid((unsigned)std::min<int64_t>((mpK + 255) / 256, 64), (unsigned)std::min(pl.ncross, 65535));
    btd::sum_ranks_kernel<<<grid, 256, 0, st>>>(partial_all, pl.world, pl.ncross, mpK, pl.cross_node, pl.S().zbuf.d());
    CK_LAUNCH();
  }
  solve_levels(pl, K, st);
  pl.ev_mark(st);
  solve_backward(pl, F, X, K, st);
  pl.ev_mark(st);
}

int guarded(btd_plan* pl, void* stream, const std::function<void(cudaStream_t)>& fn) {
  g_err.clear();
  if (!pl) { g_err = "NULL plan"; return BTD_ERR_INVALID_ARG; }
  try {
    DeviceGuard dg(pl->device);
    std::lock_guard<std::mutex> lk(pl->mu);
    cudaStream_t st = (cudaStream_t)stream;
    // The plan's scratch is shared by its solves: a call on another stream than the
    // previous one is ordered after it ON THE DEVICE (event wait, no host block).
    if (!pl->ev_done) CK(cudaEventCreateWithFlags(&pl->ev_done, cudaEventDisableTiming));
    if (pl->last_stream != st && pl->sc[0].k) CK(cudaStreamWaitEvent(st, pl->ev_done, 0));
    pl->last_stream = st;
    fn(st);
    CK(cudaEventRecord(pl->ev_done, st));
  } catch (const BtdError& e) {
    return e.code;
  }
  return BTD_OK;
}

int create_impl(const double* diag, const double* lower, const double* upper, int64_t n, int64_t m, int64_t ranks,
                int64_t split, int rank, int world, int device, int flags, void* stream, btd_plan** out_plan,
                int64_t* err_info) {
  g_err.clear();
  if (err_info) { err_info[0] = -1; err_info[1] = -1; }
  if (!out_plan) { g_err = "out_plan is NULL"; return BTD_ERR_INVALID_ARG; }
  *out_plan = nullptr;
  if (n < 1 || m < 1) { g_err = "need n >= 1 and m >= 1"; return BTD_ERR_DIMENSION; }
  if (ranks < 1 || ranks > n) {
    char buf[128];
    snprintf(buf, sizeof buf, "ranks=%lld outside [1, N=%lld]", (long long)ranks, (long long)n);
    g_err = buf;
    return BTD_ERR_INVALID_RANKS;  // ref dichotomy.py:326-327
  }
  if (world < 1 || rank < 0 || rank >= world) { g_err = "bad rank/world"; return BTD_ERR_INVALID_ARG; }
  if (!diag || (n > 1 && (!lower || !upper))) { g_err = "NULL matrix pointer"; return BTD_ERR_INVALID_ARG; }
  auto* pl = new btd_plan();
  pl->device = device;
  pl->n = n; pl->m = m; pl->ranks = ranks; pl->split = std::max<int64_t>(1, split);
  pl->rank = rank; pl->world = world;
  int64_t row = -1, rng = -1;
  try {
    DeviceGuard dg(device);
    cudaStream_t st = (cudaStream_t)stream;
    build_local(*pl, diag, lower, upper, flags, st, &row, &rng);
    if (world == 1) build_finish(*pl, pl->contrib.d(), st, &row);
  } catch (const BtdError& e) {
    if (err_info) { err_info[0] = row; err_info[1] = rng; }
    delete pl;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    delete pl;
    return BTD_ERR_CUDA;
  }
  *out_plan = pl;
  return BTD_OK;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

int btd_version(void) { return 1; }

int btd_band_to_blocktri(const double* bands, int64_t n, int64_t d, int64_t m, double* diag, double* lower,
                         double* upper, void* stream) {
  g_err.clear();
  if (n < 1 || d < 0 || m < 1) { g_err = "band: need n >= 1, d >= 0, m >= 1"; return BTD_ERR_DIMENSION; }
  if (m < d) { g_err = "band: block order smaller than the half-bandwidth"; return BTD_ERR_DIMENSION; }
  const int64_t nb = (n + m - 1) / m;
  if (!bands || !diag || (nb > 1 && (!lower || !upper))) { g_err = "band: NULL pointer"; return BTD_ERR_INVALID_ARG; }
  try {
    const int64_t total = (3 * nb - 2) * m * m;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    band_to_blocks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(bands, n, d, m, nb, diag, lower, upper);
    CK_LAUNCH();
  } catch (const BtdError& e) {
    return e.code;
  }
  return BTD_OK;
}

int btd_blocktri_apply(const double* diag, const double* lower, const double* upper, int64_t n, int64_t m,
                       const double* x, double* y, int64_t k, void* stream) {
  g_err.clear();
  if (n < 1 || m < 1 || k < 1) { g_err = "apply: need n, m, k >= 1"; return BTD_ERR_DIMENSION; }
  if (!diag || !x || !y || (n > 1 && (!lower || !upper))) { g_err = "apply: NULL pointer"; return BTD_ERR_INVALID_ARG; }
  try {
    const int64_t total = n * m * k;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    blocktri_apply_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(diag, lower, upper, n, m, k, x, y);
    CK_LAUNCH();
  } catch (const BtdError& e) {
    return e.code;
  }
  return BTD_OK;
}

int btd_csr_spmm(const int64_t* rowptr, const int64_t* col, const double* val, int64_t nrows, int64_t k,
                 const double* x, double alpha, double beta, double* y, void* stream) {
  g_err.clear();
  if (nrows < 0 || k < 1) { g_err = "spmm: bad dimensions"; return BTD_ERR_DIMENSION; }
  if (nrows == 0) return BTD_OK;
  if (!rowptr || !y) { g_err = "spmm: NULL pointer"; return BTD_ERR_INVALID_ARG; }
  try {
    const int64_t total = nrows * k;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    csr_spmm_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(rowptr, col, val, nrows, k, x, alpha, beta, y);
    CK_LAUNCH();
  } catch (const BtdError& e) {
    return e.code;
  }
  return BTD_OK;
}

int btd_band_from_probes(const double* y, int64_t n, int64_t d, int64_t ldy, double* bands, void* stream) {
  g_err.clear();
  if (n < 1 || d < 0) { g_err = "band: need n >= 1 and d >= 0"; return BTD_ERR_DIMENSION; }
  if (2 * d + 1 > n) { g_err = "band: 2d+1 exceeds the operator order"; return BTD_ERR_DIMENSION; }
  if (ldy < 2 * d + 1) { g_err = "band: ldy < 2d+1"; return BTD_ERR_INVALID_ARG; }
  if (!y || !bands) { g_err = "band: NULL pointer"; return BTD_ERR_INVALID_ARG; }
  try {
    const int64_t total = (2 * d + 1) * n;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    band_from_probes_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(y, n, d, ldy, bands);
    CK_LAUNCH();
  } catch (const BtdError& e) {
    return e.code;
  }
  return BTD_OK;
}
int btd_copy_columns(double* host, int64_t rows, int64_t K, int64_t c0, int64_t kc, double* dev, int to_device,
                     void* stream) {
  if (!host || !dev || rows < 0 || kc < 1 || c0 < 0 || c0 + kc > K) {
    g_err = "btd_copy_columns: bad arguments";
    return BTD_ERR_INVALID_ARG;
  }
  if (rows == 0) return BTD_OK;
  const size_t w = (size_t)kc * sizeof(double), hp = (size_t)K * sizeof(double);
  const cudaError_t e =
      to_device ? cudaMemcpy2DAsync(dev, w, host + c0, hp, w, (size_t)rows, cudaMemcpyHostToDevice, (cudaStream_t)stream)
                : cudaMemcpy2DAsync(host + c0, hp, dev, w, w, (size_t)rows, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    g_err = std::string("btd_copy_columns: ") + cudaGetErrorString(e);
    return BTD_ERR_CUDA;
  }
  return BTD_OK;
}
int btd_host_pin(void* ptr, int64_t nbytes, int* was_pinned) {
  if (was_pinned) *was_pinned = 0;
  if (!ptr || nbytes < 0) { g_err = "btd_host_pin: bad arguments"; return BTD_ERR_INVALID_ARG; }
  if (nbytes == 0) return BTD_OK;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) == cudaSuccess && a.type == cudaMemoryTypeHost) {
    if (was_pinned) *was_pinned = 1;
    return BTD_OK;
  }
  cudaGetLastError();
  const cudaError_t e = cudaHostRegister(ptr, (size_t)nbytes, cudaHostRegisterDefault);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    if (was_pinned) *was_pinned = 1;
    return BTD_OK;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    g_err = std::string("btd_host_pin: ") + cudaGetErrorString(e);
    return BTD_ERR_CUDA;
  }
  return BTD_OK;
}
int btd_host_is_pinned(const void* ptr) {
  if (!ptr) return 0;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return a.type == cudaMemoryTypeHost ? 1 : 0;
}
int btd_host_unpin(void* ptr) {
  if (!ptr) return BTD_ERR_INVALID_ARG;
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    g_err = std::string("btd_host_unpin: ") + cudaGetErrorString(e);
    return BTD_ERR_CUDA;
  }
  return BTD_OK;
}
int btd_host_alloc(int64_t nbytes, void** out) {
  if (!out || nbytes < 1) { g_err = "btd_host_alloc: bad arguments"; return BTD_ERR_INVALID_ARG; }
  const cudaError_t e = cudaHostAlloc(out, (size_t)nbytes, cudaHostAllocDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    g_err = std::string("btd_host_alloc: ") + cudaGetErrorString(e);
    return BTD_ERR_OOM;
  }
  return BTD_OK;
}
int btd_host_free(void* ptr) {
  if (!ptr) return BTD_OK;
  return cudaFreeHost(ptr) == cudaSuccess ? BTD_OK : BTD_ERR_CUDA;
}
int64_t btd_launch_count(void) { return g_launches.load(); }
const char* btd_last_error(void) { return g_err.c_str(); }

int btd_plan_create(const double* diag, const double* lower, const double* upper, int64_t n, int64_t m,
                    int64_t ranks, int64_t split, int device, int flags, void* stream, btd_plan** out_plan,
                    int64_t* err_row) {
  int64_t info[2] = {-1, -1};
  const int rc = create_impl(diag, lower, upper, n, m, ranks, split, 0, 1, device, flags, stream, out_plan, info);
  if (err_row) *err_row = info[0];
  return rc;
}

int btd_plan_create_shard(const double* diag, const double* lower, const double* upper, int64_t n, int64_t m,
                          int64_t ranks, int64_t split, int rank, int world, int device, int flags, void* stream,
                          btd_plan** out_plan, int64_t* err_info) {
  return create_impl(diag, lower, upper, n, m, ranks, split, rank, world, device, flags, stream, out_plan, err_info);
}

int btd_shard_contrib(btd_plan* pl, double* dst, int64_t* nelems, void* stream) {
  if (!pl || !nelems) return BTD_ERR_INVALID_ARG;
  *nelems = pl->nrl * 4 * pl->blk;
  if (!dst) return BTD_OK;
  return guarded(pl, stream, [&](cudaStream_t st) {
    CK(cudaMemcpyAsync(dst, pl->contrib.p, (size_t)(*nelems) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  });
}

int btd_shard_finish(btd_plan* pl, const double* contrib_all, void* stream, int64_t* err_row) {
  if (err_row) *err_row = -1;
  if (!pl || !contrib_all) return BTD_ERR_INVALID_ARG;
  if (pl->finished) return BTD_OK;
  int64_t row = -1;
  const int rc = guarded(pl, stream, [&](cudaStream_t st) { build_finish(*pl, contrib_all, st, &row); });
  if (err_row) *err_row = row;
  return rc;
}

int btd_shard_exchange_size(const btd_plan* pl, int64_t k, int64_t* n_carry, int64_t* n_partial) {
  if (!pl || !n_carry || !n_partial) return BTD_ERR_INVALID_ARG;
  *n_carry = pl->mp * k;
  *n_partial = (int64_t)pl->ncross * pl->mp * k;
  return BTD_OK;
}

int btd_shard_solve_a(btd_plan* pl, const double* f_local, double* x_local, int64_t k, double* carry_out,
                      void* stream) {
  if (!pl || !pl->finished || (pl->nloc > 0 && (!f_local || !x_local)) || !carry_out || k < 1) {
    g_err = "btd_shard_solve_a: bad argument or unfinished plan";
    return BTD_ERR_INVALID_ARG;
  }
  return guarded(pl, stream, [&](cudaStream_t st) {
    ensure_scratch(*pl, k);
    solve_shard_a(*pl, f_local, x_local, k, carry_out, st);
  });
}

int btd_shard_solve_b(btd_plan* pl, const double* carry_all, double* partial_out, int64_t k, void* stream) {
  if (!pl || !pl->finished || !carry_all || (pl->ncross && !partial_out) || k < 1) {
    g_err = "btd_shard_solve_b: bad argument or unfinished plan";
    return BTD_ERR_INVALID_ARG;
  }
  return guarded(pl, stream, [&](cudaStream_t st) {
    ensure_scratch(*pl, k);
    solve_shard_b(*pl, carry_all, partial_out, k, st);
  });
}

int btd_shard_solve_c(btd_plan* pl, const double* partial_all, const double* f_local, double* x_local, int64_t k,
                      void* stream) {
  if (!pl || !pl->finished || (pl->ncross && !partial_all) || (pl->nloc > 0 && !x_local) || k < 1) {
    g_err = "btd_shard_solve_c: bad argument or unfinished plan";
    return BTD_ERR_INVALID_ARG;
  }
  return guarded(pl, stream, [&](cudaStream_t st) {
    ensure_scratch(*pl, k);
    solve_shard_c(*pl, partial_all, f_local, x_local, k, st);
  });
}

int btd_plan_solve(btd_plan* pl, const double* f, double* x, int64_t k, void* stream) {
  if (!pl || !f || !x) { g_err = "NULL argument"; return BTD_ERR_INVALID_ARG; }
  if (k < 1) { g_err = "k must be >= 1"; return BTD_ERR_DIMENSION; }
  if (pl->world != 1) { g_err = "sharded plan: use btd_shard_solve_a/b/c"; return BTD_ERR_INVALID_ARG; }
  return guarded(pl, stream, [&](cudaStream_t st) {
    ensure_scratch(*pl, k);
    solve_graphed(*pl, f, x, k, st);
  });
}

// Host-memory solve (the reference's numpy-in / numpy-out contract).  Columns are
// independent, so the K columns run as equal chunks through a pipeline:
// H2D of chunk c+1 (2-D strided copy out of the (n, m, k) layout) || solve of chunk c
// || D2H of chunk c-1, with two device chunk buffers.  A narrow chunk does not fill
// the GPU (c1: 64 columns = 72 chain CTAs), so consecutive chunks solve on two
// compute streams with their own scratch slots.  Needs pinned host memory to
// overlap (pageable memory still works, synchronously).
int btd_plan_solve_host(btd_plan* pl, const double* f_host, double* x_host, int64_t k, void* stream) {
  if (!pl || !f_host || !x_host) { g_err = "NULL argument"; return BTD_ERR_INVALID_ARG; }
  if (k < 1) { g_err = "k must be >= 1"; return BTD_ERR_DIMENSION; }
  if (pl->world != 1) { g_err = "sharded plan: use btd_shard_solve_a/b/c"; return BTD_ERR_INVALID_ARG; }
  return guarded(pl, stream, [&](cudaStream_t st) {
    // Column chunk plan.  Copies run on one H2D and one D2H stream (full duplex); the
    // D2H pipe starts after H2D(chunk 0) + solve(chunk 0) and then streams, so chunks
    // are narrow (>= 32 columns: >= 256 B rows still copy at full PCIe rate).  A
    // narrow chunk's solve is latency-bound (each range is one chain of L steps
    // whatever the width), so consecutive chunks solve concurrently on up to
    // kSlots compute streams, each with its own scratch slot.
    static int maxch = -1;
    if (maxch < 0) {
      const char* e = getenv("BTD_HOST_CHUNKS");
      maxch = e ? std::max(1, std::min(btd_plan::kHostBufs, atoi(e))) : btd_plan::kHostBufs;
    }
    // measured (profiles/r01_host_pipeline.txt): 32-column chunks of a 256-column
    // solve lose more to per-chunk solve latency than they gain in fill time
    static int64_t minw_env = -1;
    if (minw_env < 0) {
      const char* e = getenv("BTD_HOST_MINW");
      minw_env = e ? std::max(2, atoi(e)) : 0;
    }
    // mode 1 (blocks > 256): the solve outweighs the copies; narrow chunks only thin out its
    // GEMM batches (c3: 32-column chunks 8.2k, one 128-column chunk 8.4k RHS/s end to end)
    const int64_t minw = minw_env ? minw_env : (pl->mode == 1 ? 128 : (k >= 256 ? 64 : 32));
    int64_t kc = k;
    for (int64_t nch = maxch; nch >= 2; --nch)
      if (k % nch == 0 && (k / nch) % 2 == 0 && k / nch >= minw) { kc = k / nch; break; }
    // Chunk widths.  The copy pipes idle for one chunk's H2D + solve at the start and
    // one chunk's solve + D2H at the end, so the first and last chunks are half as
    // wide when that keeps >= 256-byte row segments (narrower 2-D copies lose rate:
    // tools/microbench/hostio.cu, profiles/r02_hostio.txt): c1 256 = 32+64+64+64+32.
    std::vector<int64_t> widths;
    {
      static int halves = -1;
      if (halves < 0) halves = getenv("BTD_HOST_HALF_ENDS") ? atoi(getenv("BTD_HOST_HALF_ENDS")) : 1;
      const int64_t n0 = k / kc;
      if (halves && n0 >= 2 && kc % 4 == 0 && kc / 2 >= 32 && pl->mode == 0) {
        widths.push_back(kc / 2);
        for (int64_t c = 1; c < n0; ++c) widths.push_back(kc);
        widths.push_back(kc / 2);
      } else {
        widths.assign((size_t)n0, kc);
      }
    }
    const int64_t nch = (int64_t)widths.size(), rows = pl->n * pl->m;
    const size_t celems = (size_t)rows * kc;
    // concurrent solves: not with the cooperative tree kernel (two partially-resident
    // cooperative grids could wait on each other) or while phase profiling (per-solve
    // phase events are single-stream)
    static int slots_env = -1;
    if (slots_env < 0) {
      const char* e = getenv("BTD_HOST_SLOTS");
      slots_env = e ? std::max(1, std::min(btd_plan::kSlots, atoi(e))) : btd_plan::kSlots;
    }
    const int nstr = (pl->fused_tree || pl->profiling) ? 1 : (int)std::min<int64_t>(nch, slots_env);
    if (pl->hostio_k != k) {
      for (auto& g : pl->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
      pl->graphs.clear();
      pl->hostio_k = k;
    }
    // up to kHostBufs chunks in flight: the H2D of chunk c waits only for the D2H of
    // chunk c - kHostBufs (with two buffers the pipeline serialises in/solve/out)
    const int nbuf = (int)std::min<int64_t>(nch, btd_plan::kHostBufs);
    if ((int64_t)celems * nbuf > pl->hchunk_elems) {
      pl->hchunk.alloc(celems * nbuf * sizeof(double));
      pl->hchunk_elems = (int64_t)celems * nbuf;
      for (auto& g : pl->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
      pl->graphs.clear();
    }
    if (!pl->s_in) {
      CK(cudaStreamCreateWithFlags(&pl->s_in, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&pl->s_out, cudaStreamNonBlocking));
      for (auto& x : pl->s_c) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
      for (auto& a : pl->ev_h)
        for (auto& e : a) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    struct SlotReset {
      btd_plan* p;
      ~SlotReset() { p->cur = 0; p->host_concurrent = false; }
    } reset{pl};
    pl->host_concurrent = nstr > 1;
    for (int sl = 0; sl < nstr; ++sl) {
      pl->cur = sl;
      ensure_scratch(*pl, kc);
    }
    const cudaStream_t cs[btd_plan::kSlots] = {st, pl->s_c[0], pl->s_c[1], pl->s_c[2]};
    cudaEvent_t start;
    CK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CK(cudaEventRecord(start, st));
    CK(cudaStreamWaitEvent(pl->s_in, start, 0));
    for (int i = 1; i < nstr; ++i) CK(cudaStreamWaitEvent(cs[i], start, 0));
    const size_t hpitch = (size_t)k * sizeof(double);
    // BTD_HOST_TRACE=1: per-chunk timeline (H2D / solve / D2H start+end) on stderr
    static int trace = -1;
    if (trace < 0) trace = getenv("BTD_HOST_TRACE") ? atoi(getenv("BTD_HOST_TRACE")) : 0;
    std::vector<cudaEvent_t> tev;
    auto tmark = [&](cudaStream_t s) {
      if (!trace) return;
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      CK(cudaEventRecord(e, s));
      tev.push_back(e);
    };
    tmark(st);
    int64_t col = 0;
    for (int64_t c = 0; c < nch; ++c) {
      const int b = (int)(c % nbuf), sl = (int)(c % nstr);
      const int64_t wc = widths[(size_t)c];
      const size_t wbytes = (size_t)wc * sizeof(double);
      const cudaStream_t cst = cs[sl];
      double* dbuf = pl->hchunk.d() + (size_t)b * celems;
      cudaEvent_t in_done = pl->ev_h[b][0], comp_done = pl->ev_h[b][1], out_done = pl->ev_h[b][2];
      if (c >= nbuf) CK(cudaStreamWaitEvent(pl->s_in, out_done, 0));  // buffer b free again
      tmark(pl->s_in);
      CK(cudaMemcpy2DAsync(dbuf, wbytes, f_host + col, hpitch, wbytes, rows, cudaMemcpyHostToDevice, pl->s_in));
      CK(cudaEventRecord(in_done, pl->s_in));
      tmark(pl->s_in);
      CK(cudaStreamWaitEvent(cst, in_done, 0));
      pl->cur = sl;
      tmark(cst);
      solve_graphed(*pl, dbuf, dbuf, wc, cst);
      CK(cudaEventRecord(comp_done, cst));
      tmark(cst);
      CK(cudaStreamWaitEvent(pl->s_out, comp_done, 0));
      tmark(pl->s_out);
      CK(cudaMemcpy2DAsync(x_host + col, hpitch, dbuf, wbytes, wbytes, rows, cudaMemcpyDeviceToHost, pl->s_out));
      CK(cudaEventRecord(out_done, pl->s_out));
      tmark(pl->s_out);
      col += wc;
    }
    pl->cur = 0;
    CK(cudaStreamSynchronize(pl->s_out));
    for (int i = 1; i < nstr; ++i) CK(cudaStreamSynchronize(cs[i]));
    CK(cudaStreamSynchronize(st));
    cudaEventDestroy(start);
    if (trace) {
      float ms[6];
      fprintf(stderr, "[btd host] k=%lld chunks=%lld streams=%d\n", (long long)k, (long long)nch, nstr);
      for (int64_t c = 0; c < nch; ++c) {
        for (int i = 0; i < 6; ++i) CK(cudaEventElapsedTime(&ms[i], tev[0], tev[1 + 6 * c + i]));
        fprintf(stderr, "  chunk %lld w=%lld  h2d %7.2f-%7.2f  solve %7.2f-%7.2f  d2h %7.2f-%7.2f\n", (long long)c,
                (long long)widths[(size_t)c], ms[0], ms[1], ms[2], ms[3], ms[4], ms[5]);
      }
      for (auto e : tev) cudaEventDestroy(e);
    }
  });
}

// ---- plan image: header + factor pool + inverse rows + E/H blocks (device bytes).
// The metadata (ranges, tree, batches) is recomputed from the header on import;
// the factors are the output of the expensive sequential preprocessing.
namespace {
constexpr int64_t kImageMagic = 0x314e414c50445442LL;  // "BTDPLAN1" little-endian
constexpr int64_t kImageVersion = 1;
struct ImageHeader {
  int64_t magic, version, n, m, ranks, split, rank, world, mode, mp, pool_bytes, rrows_bytes, eh_bytes;
};
}  // namespace

int btd_plan_export(btd_plan* pl, void* dst, int64_t* nbytes, void* stream) {
  if (!pl || !nbytes) { g_err = "btd_plan_export: NULL argument"; return BTD_ERR_INVALID_ARG; }
  if (!pl->finished) { g_err = "btd_plan_export: plan not finished"; return BTD_ERR_INVALID_ARG; }
  const int64_t need = (int64_t)(sizeof(ImageHeader) + pl->pool.bytes + pl->Rrows.bytes + pl->EH.bytes);
  if (!dst) { *nbytes = need; return BTD_OK; }
  if (*nbytes < need) { g_err = "btd_plan_export: destination too small"; return BTD_ERR_INVALID_ARG; }
  *nbytes = need;
  return guarded(pl, stream, [&](cudaStream_t st) {
    // mode field: sweep mode in the low byte, the scalar-coupling flag (extra pool sections) above it
    ImageHeader h{kImageMagic, kImageVersion, pl->n, pl->m, pl->ranks, pl->split, pl->rank, pl->world,
                  pl->mode | (pl->scoup << 8), pl->mp, (int64_t)pl->pool.bytes, (int64_t)pl->Rrows.bytes, (int64_t)pl->EH.bytes};
    char* out = static_cast<char*>(dst);
    memcpy(out, &h, sizeof h);
    out += sizeof h;
    CK(cudaMemcpyAsync(out, pl->pool.p, pl->pool.bytes, cudaMemcpyDeviceToHost, st));
    out += pl->pool.bytes;
    CK(cudaMemcpyAsync(out, pl->Rrows.p, pl->Rrows.bytes, cudaMemcpyDeviceToHost, st));
    out += pl->Rrows.bytes;
    CK(cudaMemcpyAsync(out, pl->EH.p, pl->EH.bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int btd_plan_import(const void* src, int64_t nbytes, int device, void* stream, btd_plan** out_plan) {
  g_err.clear();
  if (!src || !out_plan) { g_err = "btd_plan_import: NULL argument"; return BTD_ERR_INVALID_ARG; }
  *out_plan = nullptr;
  ImageHeader h;
  if (nbytes < (int64_t)sizeof h) { g_err = "plan image: truncated header"; return BTD_ERR_INVALID_ARG; }
  memcpy(&h, src, sizeof h);
  if (h.magic != kImageMagic) { g_err = "plan image: bad magic"; return BTD_ERR_INVALID_ARG; }
  if (h.version != kImageVersion) { g_err = "plan image: unsupported version"; return BTD_ERR_UNSUPPORTED; }
  if (h.n < 1 || h.m < 1 || h.ranks < 1 || h.ranks > h.n || h.split < 1 || h.world < 1 || h.rank < 0 ||
      h.rank >= h.world || ((h.mode & 0xff) != 0 && (h.mode & 0xff) != 1) || (h.mode >> 8) < 0 || (h.mode >> 8) > 1 ||
      h.pool_bytes < 0 || h.rrows_bytes < 0 || h.eh_bytes < 0 ||
      nbytes != (int64_t)sizeof h + h.pool_bytes + h.rrows_bytes + h.eh_bytes) {
    g_err = "plan image: inconsistent header or size";
    return BTD_ERR_INVALID_ARG;
  }
  auto* pl = new btd_plan();
  pl->device = device;
  pl->n = h.n; pl->m = h.m; pl->ranks = h.ranks; pl->split = h.split;
  pl->rank = (int)h.rank; pl->world = (int)h.world;
  try {
    DeviceGuard dg(device);
    cudaStream_t st = (cudaStream_t)stream;
    int64_t row = -1, rng = -1;
    pl->scoup = (int)(h.mode >> 8);
    build_local(*pl, nullptr, nullptr, nullptr, 0, st, &row, &rng, (int)(h.mode & 0xff));
    if (pl->mp != h.mp || (int64_t)pl->pool.bytes != h.pool_bytes) fail(BTD_ERR_INVALID_ARG, "plan image: pool layout mismatch");
    const char* in = static_cast<const char*>(src) + sizeof h;
    CK(cudaMemcpyAsync(pl->pool.p, in, h.pool_bytes, cudaMemcpyHostToDevice, st));
    in += h.pool_bytes;
    build_finish(*pl, nullptr, st, &row, true);
    if ((int64_t)pl->Rrows.bytes != h.rrows_bytes || (int64_t)pl->EH.bytes != h.eh_bytes)
      fail(BTD_ERR_INVALID_ARG, "plan image: tree layout mismatch");
    CK(cudaMemcpyAsync(pl->Rrows.p, in, h.rrows_bytes, cudaMemcpyHostToDevice, st));
    in += h.rrows_bytes;
    CK(cudaMemcpyAsync(pl->EH.p, in, h.eh_bytes, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  } catch (const BtdError& e) {
    delete pl;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    delete pl;
    return BTD_ERR_CUDA;
  }
  *out_plan = pl;
  return BTD_OK;
}

int btd_plan_destroy(btd_plan* pl) {
  if (!pl) return BTD_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(pl->device);
  cudaDeviceSynchronize();
  delete pl;
  if (prev >= 0) cudaSetDevice(prev);
  return BTD_OK;
}

int btd_plan_set_profiling(btd_plan* pl, int enable) {
  if (!pl) return BTD_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(pl->mu);
  pl->profiling = enable != 0;
  return BTD_OK;
}

int btd_plan_phase_times(btd_plan* pl, double* ms_out, int64_t* nsolves, int reset) {
  if (!pl || !ms_out) return BTD_ERR_INVALID_ARG;
  try {
    DeviceGuard dg(pl->device);
    std::lock_guard<std::mutex> lk(pl->mu);
    pl->ev_drain();
    for (int i = 0; i < 4; ++i) ms_out[i] = pl->phase_ms[i];
    if (nsolves) *nsolves = pl->nprof;
    if (reset) {
      for (double& v : pl->phase_ms) v = 0;
      pl->nprof = 0;
    }
  } catch (const BtdError& e) {
    return e.code;
  }
  return BTD_OK;
}

int btd_plan_query(const btd_plan* pl, btd_plan_info* info) {
  if (!pl || !info) return BTD_ERR_INVALID_ARG;
  memset(info, 0, sizeof *info);
  info->n = pl->n; info->m = pl->m; info->mp = pl->mp; info->ranks = pl->ranks; info->split = pl->split;
  info->nranges = pl->nr; info->L = pl->L; info->tree_nodes = (int64_t)pl->nodes.size();
  info->tree_depth = pl->depth; info->factor_bytes = pl->factor_bytes;
  info->row_lo = pl->R0; info->row_hi = pl->R0 + pl->nloc;
  info->device = pl->device; info->mode = pl->mode;
  info->rank = pl->rank; info->world = pl->world; info->range_lo = pl->q0; info->range_hi = pl->q1;
  info->scalar_coupling = pl->scoup;
  return BTD_OK;
}

}  // extern "C"
