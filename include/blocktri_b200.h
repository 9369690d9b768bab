/*
 * blocktri_b200.h -- C ABI of the B200-native many-RHS block-tridiagonal
 * dichotomy solver (arXiv 1108.4181, Algorithm 2).
 *
 * This is the drop-in boundary for the reference path
 *   blocktri.dichotomy.plan_build(p_matrix, ranks) -> DichotomyPlan
 *       (/root/reference/pkg/src/blocktri/dichotomy.py:318-338)
 *   blocktri.dichotomy.plan_solve(plan, f_batch)   -> X
 *       (/root/reference/pkg/src/blocktri/dichotomy.py:358-390)
 * The reference has no FFI of its own (pure Python + a Cython kernel module,
 * _kernels.pyx:111-194); these entry points are what its dichotomy module
 * binds through ctypes.  Plain pointers and sizes only.
 *
 * Storage convention (ref core.py:1-10, 84-90): row i of the operator reads
 *   -lower[i-1] x_{i-1} + diag[i] x_i - upper[i] x_{i+1} = f_i
 * diag is (n,m,m), lower/upper are (n-1,m,m), all row-major float64;
 * right-hand sides / solutions are (n,m,k) row-major float64.
 */
#ifndef BLOCKTRI_B200_H
#define BLOCKTRI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python host maps them to the reference exception
 * classes (ref errors.py): 1 -> DimensionMismatch, 2 -> SingularPivot(row),
 * 3 -> InvalidRankCount; the rest -> DeviceError. */
enum {
  BTD_OK = 0,
  BTD_ERR_DIMENSION = 1,
  BTD_ERR_SINGULAR_PIVOT = 2,
  BTD_ERR_INVALID_RANKS = 3,
  BTD_ERR_CUDA = 4,
  BTD_ERR_NCCL = 5,
  BTD_ERR_OOM = 6,
  BTD_ERR_INVALID_ARG = 7,
  BTD_ERR_UNSUPPORTED = 8
};

/* flags for btd_plan_create */
enum {
  BTD_MATRIX_ON_DEVICE = 1 /* diag/lower/upper are device pointers on `device` */
};

typedef struct btd_plan btd_plan;

typedef struct btd_plan_info {
  int64_t n, m, mp;          /* block rows, block order, padded order (multiple of 8) */
  int64_t ranks;             /* reference P (ranges of the Algorithm-2 partition) */
  int64_t split;             /* device sub-ranges per reference range (1 = exact ref. partition) */
  int64_t nranges;           /* device ranges actually used (= ranks*split clamped to n) */
  int64_t L;                 /* uniform range length; the last range may be shorter */
  int64_t tree_nodes, tree_depth;
  int64_t factor_bytes;      /* HBM held by the plan */
  int64_t row_lo, row_hi;    /* block rows owned by this plan (sharded plans) */
  int32_t device;
  int32_t mode;              /* 0 = fused chain kernels, 1 = per-step GEMM sweep (large m) */
  int32_t rank, world;       /* shard of a row-sharded plan (0, 1 when not sharded) */
  int64_t range_lo, range_hi;/* device ranges owned by this shard */
  int64_t scalar_coupling;   /* 1: every interior lower block is a scalar multiple of I (5-point-stencil
                              * operators); the forward sweep then runs y_j = Dinv_j (f_j + a_j y_{j-1}):
                              * 8 instead of 10 M^2 K flops per row and batch.  BTD_SCALAR_COUPLING=0 disables. */
} btd_plan_info;

/* Algorithm 2 step 1 (ref dichotomy.py:318-338): validate 1 <= ranks <= n
 * (BTD_ERR_INVALID_RANKS), partition rows into ranges K_q = q*L with
 * L = ceil(n / (ranks*split)), factor every range's interior sweep, assemble
 * the reduced interface system (Eq. 7) and the inverse rows of its partition
 * tree.  On BTD_ERR_SINGULAR_PIVOT *err_row holds the row local to the
 * factored submatrix, exactly as the reference's SingularPivot.row.
 * `stream` is a cudaStream_t (NULL = legacy default stream). */
int btd_plan_create(const double* diag, const double* lower, const double* upper,
                    int64_t n, int64_t m, int64_t ranks, int64_t split,
                    int device, int flags, void* stream,
                    btd_plan** out_plan, int64_t* err_row);

/* Algorithm 2 step 2 (ref dichotomy.py:358-390) on DEVICE buffers:
 * f, x are (n,m,k) float64 on the plan's device; x may alias f.
 * Stream-ordered; returns once enqueued.  No block factorization.
 * Threading: the plan is read-only after creation and calls are thread-safe.
 * Its solve scratch is shared, so solves on one plan issued on different
 * streams are ordered on the device (the later call's stream waits on an event
 * of the earlier one; the host never blocks).  Independent concurrent solves
 * of one matrix use one plan per stream, or btd_plan_solve_host, which runs
 * its column chunks on up to four internal streams at once. */
int btd_plan_solve(btd_plan* plan, const double* f, double* x, int64_t k, void* stream);

/* Same on HOST buffers (the reference's numpy-in / numpy-out contract): copies
 * f to the device, solves, copies x back, synchronizes `stream`. */
int btd_plan_solve_host(btd_plan* plan, const double* f_host, double* x_host, int64_t k,
                        void* stream);

int btd_plan_destroy(btd_plan* plan);
int btd_plan_query(const btd_plan* plan, btd_plan_info* info);

/* ---- plan images (replaces ref io.py:125-203 write_plan/read_plan, DPLN) --
 * btd_plan_export copies a finished plan (single or shard) into host memory:
 * a 104-byte header (magic "BTDPLAN1", version, n, m, ranks, split, rank,
 * world, sweep mode, padded order, three section sizes) followed by the raw
 * device factor pool, the tree inverse rows and the E/H correction blocks.
 * Call with dst = NULL to get the size in *nbytes.  btd_plan_import rebuilds
 * the plan on `device` from such an image without redoing the preprocessing
 * (the matrix is not needed; binding to a matrix is the caller's fingerprint
 * check, as in ref io.py:157-160).  Errors: BTD_ERR_INVALID_ARG for a
 * malformed image, BTD_ERR_UNSUPPORTED for another image version. */
int btd_plan_export(btd_plan* plan, void* dst, int64_t* nbytes, void* stream);

/* ---- band route (ref bands.py) ---------------------
 * Band storage: bands[k*n + j] = a(j + k - d, j), k = 0..2d (ref bands.py:18-41).
 * btd_band_to_blocktri replaces ref bands.py:120-157 band_as_blocktrid: block
 *   order m >= d, nb = ceil(n/m) blocks; writes diag (nb,m,m), lower/upper
 *   (nb-1,m,m) with the reference's signs and identity padding.  Device pointers.
 *   BTD_ERR_DIMENSION when m < d (ref BlockTooSmall) or n < 1.
 * btd_band_from_probes replaces ref bands.py:94-117 probing_build (+ the
 *   symmetrization at bands.py:73-84): y = A * P, P the n x (2d+1) class-probe
 *   matrix P[i][c] = (i mod (2d+1) == c), row-major with leading dimension ldy;
 *   writes the symmetrized band (B + B^T)/2.  BTD_ERR_DIMENSION when 2d+1 > n
 *   (ref BandTooWide).  Device pointers; both are stream-ordered. */
int btd_band_to_blocktri(const double* bands, int64_t n, int64_t d, int64_t m, double* diag, double* lower,
                         double* upper, void* stream);
int btd_band_from_probes(const double* y, int64_t n, int64_t d, int64_t ldy, double* bands, void* stream);

/* ---- operators around the path (Schur DD) -----------
 * btd_blocktri_apply: y = P x with P block tridiagonal (ref core.py:118-127
 *   BlockTriMatrix.apply; used by ref schur.py:191-195 BlocktriOperator.apply),
 *   x, y (n, m, k) row-major on the device.
 * btd_csr_spmm: y = alpha * S x + beta * y, S in CSR (int64 row pointers and
 *   column indices), x (ncols, k), y (nrows, k) row-major on the device (the
 *   interface couplings A_iG, A_iG^T, A_GG of ref schur.py:198-310). */
int btd_blocktri_apply(const double* diag, const double* lower, const double* upper, int64_t n, int64_t m,
                       const double* x, double* y, int64_t k, void* stream);
int btd_csr_spmm(const int64_t* rowptr, const int64_t* col, const double* val, int64_t nrows, int64_t k,
                 const double* x, double alpha, double beta, double* y, void* stream);
int btd_plan_import(const void* src, int64_t nbytes, int device, void* stream, btd_plan** out_plan);

/* ---- row-sharded (multi-GPU) plans and solves --------------------------
 * The ranges (ranks*split of them, a multiple of `world`) are split
 * contiguously over `world` processes, one GPU each; rank r owns ranges
 * [r*P/world, (r+1)*P/world) and their block rows.  The reference's
 * distributed solve (harness.py:147-216: local sweep, exchange of the
 * interface pairs, reduced solve, local recovery) maps to:
 *   plan:  btd_plan_create_shard (local factors + this shard's four
 *          reduced-system contributions per range) -> caller all-gathers the
 *          contributions (btd_shard_contrib) -> btd_shard_finish (reduced
 *          system + partition tree, identical on every rank);
 *   solve: btd_shard_solve_a (local sweeps; emits the carry of its last range,
 *          n_carry doubles) -> caller all-gathers the carries ->
 *          btd_shard_solve_b (interface RHS of its ranges; partial series sums
 *          R_node f~ over its own ranges for the tree nodes whose segment
 *          crosses a rank boundary, n_partial doubles) -> caller all-gathers
 *          the partials -> btd_shard_solve_c (sums them in rank order, tree
 *          levels for the nodes it needs, local recovery).
 *   This is the paper's "sum of a series over distributed data": per solve a
 *   rank exchanges M*K + (#crossing nodes)*M*K doubles, not the reference
 *   harness's all-gather of every range's pair.
 * f_local / x_local hold the shard's rows [row_lo, row_hi) (btd_plan_query).
 * err_info[0] = SingularPivot row, err_info[1] = failing global range. */
int btd_plan_create_shard(const double* diag, const double* lower, const double* upper,
                          int64_t n, int64_t m, int64_t ranks, int64_t split, int rank, int world,
                          int device, int flags, void* stream, btd_plan** out_plan,
                          int64_t* err_info);
/* copies this shard's contributions ([ranges][4][mp][mp] doubles) to device
 * buffer dst (dst == NULL: only report *nelems) */
int btd_shard_contrib(btd_plan* plan, double* dst, int64_t* nelems, void* stream);
int btd_shard_finish(btd_plan* plan, const double* contrib_all, void* stream, int64_t* err_row);
int btd_shard_exchange_size(const btd_plan* plan, int64_t k, int64_t* n_carry, int64_t* n_partial);
int btd_shard_solve_a(btd_plan* plan, const double* f_local, double* x_local, int64_t k,
                      double* carry_out, void* stream);
int btd_shard_solve_b(btd_plan* plan, const double* carry_all, double* partial_out, int64_t k,
                      void* stream);
int btd_shard_solve_c(btd_plan* plan, const double* partial_all, const double* f_local,
                      double* x_local, int64_t k, void* stream);

/* Per-phase device timing of solves (CUDA events recorded on the solve
 * stream between the forward sweep, the interface/tree phase and the backward
 * sweep).  ms_out[0..3] = forward, interface+tree, backward, total, summed
 * over the solves since the last reset; *nsolves = how many. */
int btd_plan_set_profiling(btd_plan* plan, int enable);
int btd_plan_phase_times(btd_plan* plan, double* ms_out, int64_t* nsolves, int reset);

/* Column-chunk copy between an (rows, K) host array and a dense (rows, kc)
 * device chunk, stream-ordered (cudaMemcpy2DAsync; the per-rank host pipeline
 * of the sharded solve, ShardedPlan.solve_host).  to_device = 1: host columns
 * [c0, c0+kc) -> device; 0: device -> host columns.  Host memory should be
 * pinned to overlap with compute.  (The reference ranks exchange and solve on
 * numpy arrays in host memory, harness.py:147-216; this moves a rank's rows
 * in column chunks so the copies overlap its solve.) */
int btd_copy_columns(double* host, int64_t rows, int64_t K, int64_t c0, int64_t kc, double* dev, int to_device,
                     void* stream);

/* Host memory for the numpy path (ref dichotomy.py:358-390 takes and returns
 * host arrays).  The pipelined btd_plan_solve_host overlaps its copies with the
 * solve only on page-locked memory:
 *   btd_host_pin    page-locks an existing host range (cudaHostRegister);
 *                   *was_pinned = 1 (and nothing is done) when it already is;
 *   btd_host_unpin  undoes btd_host_pin;
 *   btd_host_alloc / btd_host_free  page-locked allocations (solution arrays). */
int btd_host_pin(void* ptr, int64_t nbytes, int* was_pinned);
int btd_host_is_pinned(const void* ptr);  /* 1 when ptr lies in page-locked memory, else 0 */
int btd_host_unpin(void* ptr);
int btd_host_alloc(int64_t nbytes, void** out);
int btd_host_free(void* ptr);

/* Kernel launches issued by this library since load (the bench's
 * gpu_launches evidence) and the last error text. */
int64_t btd_launch_count(void);
const char* btd_last_error(void);
int btd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKTRI_B200_H */
