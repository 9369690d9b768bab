// Band route: band storage <-> block-tridiagonal blocks,
// and band recovery from probe responses.  Pure data movement / one add per
// entry: HBM-bound, every output element computed by one thread from at most
// two gathered inputs (no staging needed; the outputs are written coalesced).
//
// Band storage (ref bands.py:18-41): bands[k][j] = a(j + k - d, j), k = 0..2d.
#pragma once
#include <cstdint>

namespace btd {

// band_as_blocktrid (ref bands.py:120-157): block order m >= d, nb = ceil(n/m)
// blocks; diag[b] = a(bm+r, bm+c), lower[b] = -a((b+1)m+r, bm+c),
// upper[b] = -a(bm+r, (b+1)m+c); padding rows g >= n get diag 1.  Entries
// outside the band stay +0.0 (in-band zeros become -0.0 on the couplings,
// like the reference's `-v`).
__global__ void band_to_blocks_kernel(const double* __restrict__ bands, int64_t n, int64_t d, int64_t m,
                                      int64_t nb, double* __restrict__ diag, double* __restrict__ lower,
                                      double* __restrict__ upper) {
  const int64_t mm = m * m, nd = nb * mm, nc = (nb - 1) * mm, total = nd + 2 * nc;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t which, b, rc;
    if (e < nd) { which = 0; b = e / mm; rc = e % mm; }
    else if (e < nd + nc) { which = 1; b = (e - nd) / mm; rc = (e - nd) % mm; }
    else { which = 2; b = (e - nd - nc) / mm; rc = (e - nd - nc) % mm; }
    const int64_t r = rc / m, c = rc % m;
    const int64_t i = (which == 1 ? b + 1 : b) * m + r;
    const int64_t j = (which == 2 ? b + 1 : b) * m + c;
    const int64_t off = i - j;
    double v = 0.0;
    if (i < n && j < n && off >= -d && off <= d) {
      const double a = bands[(d + off) * n + j];
      v = which == 0 ? a : -a;
    } else if (which == 0 && i == j && i >= n) {
      v = 1.0;
    }
    double* out = which == 0 ? diag : which == 1 ? lower : upper;
    out[b * mm + rc] = v;
  }
}

// probing_build + symmetrized (ref bands.py:94-117, 73-84): y is the n x w
// response matrix (row-major, leading dimension ldy) to the w = 2d+1 class probes
// p_c = [i mod w == c].  raw(k, j) = y[j + k - d][j mod w]; the result is
// 0.5 * (raw(k, j) + raw(2d - k, j + k - d)) = 0.5 * (y[j+off][j mod w] + y[j][(j+off) mod w])
// for 0 <= j, j + off < n (off = k - d), else 0.
__global__ void band_from_probes_kernel(const double* __restrict__ y, int64_t n, int64_t d, int64_t ldy,
                                        double* __restrict__ bands) {
  const int64_t w = 2 * d + 1, total = w * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / n, j = e % n, off = k - d, i = j + off;
    double v = 0.0;
    if (i >= 0 && i < n) v = 0.5 * (y[i * ldy + j % w] + y[j * ldy + i % w]);
    bands[e] = v;
  }
}

}  // namespace btd

namespace btd {

// Operator application around the path (Schur DD, ref schur.py:168-195, core.py:118-127):
// y_i = C_i x_i - A_i x_{i-1} - B_i x_{i+1}, blocks (n, m, m) / (n-1, m, m), x, y (n, m, k).
// One thread per output entry; the three block rows it reads come from L1/L2.
// Used for apply_full / residuals, not on the solve path.
__global__ void blocktri_apply_kernel(const double* __restrict__ C, const double* __restrict__ A,
                                      const double* __restrict__ B, int64_t n, int64_t m, int64_t k,
                                      const double* __restrict__ x, double* __restrict__ y) {
  const int64_t total = n * m * k, mk = m * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / mk, r = (e % mk) / k, c = e % k;
    const double* cr = C + (i * m + r) * m;
    const double* xi = x + i * mk + c;
    double s = 0.0;
    for (int64_t j = 0; j < m; ++j) s += cr[j] * xi[j * k];
    if (i > 0) {
      const double* ar = A + ((i - 1) * m + r) * m;
      const double* xp = x + (i - 1) * mk + c;
      for (int64_t j = 0; j < m; ++j) s -= ar[j] * xp[j * k];
    }
    if (i + 1 < n) {
      const double* br = B + (i * m + r) * m;
      const double* xn = x + (i + 1) * mk + c;
      for (int64_t j = 0; j < m; ++j) s -= br[j] * xn[j * k];
    }
    y[e] = s;
  }
}

// CSR sparse x dense (k columns, row-major): y = alpha * S x + beta * y.  Interface
// couplings have a handful of entries per row; one thread per (row, column).
__global__ void csr_spmm_kernel(const int64_t* __restrict__ rowptr, const int64_t* __restrict__ col,
                                const double* __restrict__ val, int64_t nrows, int64_t k,
                                const double* __restrict__ x, double alpha, double beta, double* __restrict__ y) {
  const int64_t total = nrows * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / k, c = e % k;
    double s = 0.0;
    for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) s += val[p] * x[col[p] * k + c];
    y[e] = beta == 0.0 ? alpha * s : alpha * s + beta * y[e];
  }
}

}  // namespace btd
