// Sparse pieces of the LOR V-cycle on the device (solvers.py:269-392,
// lor.py:61-123):
//   * CSR SpMV / residual for the LOR level matrices and the nodal
//     interpolation transfers P, P^T (scipy `A @ x` at solvers.py:381-382);
//   * sparse triangular solves for the ILU(0) smoother factors and the
//     coarse-level LU factors (SuperLU `.solve` at solvers.py:298-311, 376);
//   * permutation gathers/scatters (the first-touch ordering).
// SpMV sums each row sequentially in index order with round-to-nearest
// multiply-then-add, exactly like scipy's csr_matvec, so the V-cycle's
// residuals match the reference bit for bit.
//
// Triangular solves are "sync-free": one warp per row, rows claimed in
// dependency order from an atomic counter, each row waits (spins) only on
// the completion flags of the rows it reads.  Every row it waits on was
// claimed earlier by a running warp, so the solve cannot deadlock, and one
// launch replaces the reference's level-by-level dependency chain (449-1409
// levels at 36k-0.9M DoFs).
#include <algorithm>
#include <cstring>
#include <memory>

#include "fb_common.cuh"
#include "fb_internal.cuh"


struct fb_trisolve {
  int64_t n = 0;
  int lower = 1, unit = 0;
  fb::DevBuf<int> indptr, indices;
  fb::DevBuf<double> data;  // off-diagonal entries only
  fb::DevBuf<double> invdiag;
  fb::DevBuf<unsigned int> flags;  // per-row completion epoch
  fb::DevBuf<unsigned int> counter;
  mutable unsigned int epoch = 0;
  // level schedule
  int nlevels = 0;
  std::vector<int> level_ptr;  // host: offsets into level_rows
  fb::DevBuf<int> level_rows;
  mutable cudaGraphExec_t graph = nullptr;
  mutable const double* graph_b = nullptr;
  mutable double* graph_x = nullptr;
  mutable cudaStream_t graph_stream = nullptr;
  ~fb_trisolve() {
    if (graph) cudaGraphExecDestroy(graph);
  }
};

static int g_trisolve_mode = 1;      // 0 = sync-free, 1 = level-scheduled graph
static int g_trisolve_backoff = 64;  // ns between polls (sync-free mode)

namespace fb {

__global__ void csr_spmv_kernel(int64_t nrows, const int64_t* __restrict__ ip,
                                const int* __restrict__ ix, const double* __restrict__ v,
                                const double* __restrict__ x, const double* __restrict__ b,
                                double* __restrict__ y) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double acc = 0.0;
  const int64_t e = __ldg(ip + r + 1);
  // batches of 8 independent loads, summed sequentially in index order
  for (int64_t k = __ldg(ip + r); k < e; k += 8) {
    double a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = k + u < e;
      a[u] = ok ? __ldg(v + k + u) : 0.0;
      b[u] = ok ? __ldg(x + __ldg(ix + k + u)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k + u < e) acc = __dadd_rn(acc, __dmul_rn(a[u], b[u]));
  }
  y[r] = b ? __dsub_rn(__ldg(b + r), acc) : acc;
}

// LANES lanes per row: lanes take the row's entries in LANES-wide coalesced
// strides and the partial sums are combined in a fixed butterfly order
// (deterministic, not scipy's sequential order).  Used for the scale-mode
// levels, whose rows have ~27 entries.
template <int LANES>
__global__ void __launch_bounds__(256) csr_spmv_group_kernel(int64_t nrows,
                                                             const int64_t* __restrict__ ip,
                                                             const int* __restrict__ ix,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ x,
                                                             const double* __restrict__ b,
                                                             double* __restrict__ y) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / LANES;
  const int lane = threadIdx.x % LANES;
  const bool live = r < nrows;
  double acc = 0.0;
  if (live) {
    const int64_t e0 = __ldg(ip + r), e1 = __ldg(ip + r + 1);
    for (int64_t k = e0 + lane; k < e1; k += LANES)
      acc = fma(__ldg(v + k), __ldg(x + __ldg(ix + k)), acc);
  }
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (live && lane == 0) y[r] = b ? __ldg(b + r) - acc : acc;
}

// Several right-hand sides at once (NV vectors at a common stride, e.g. the
// components of a vector field sharing one scalar LOR level): each matrix
// entry and column index is loaded once for all NV products.  Per vector the
// entry order and the butterfly combine are those of csr_spmv_group_kernel<4>,
// so every result is bitwise the single-vector one.
template <int NV>
__global__ void __launch_bounds__(256) csr_spmv_group_multi_kernel(
    int64_t nrows, const int64_t* __restrict__ ip, const int* __restrict__ ix,
    const double* __restrict__ v, const double* __restrict__ x, const double* __restrict__ b,
    double* __restrict__ y, int64_t stride) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 4;
  const int lane = threadIdx.x % 4;
  const bool live = r < nrows;
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  if (live) {
    const int64_t e0 = __ldg(ip + r), e1 = __ldg(ip + r + 1);
    for (int64_t k = e0 + lane; k < e1; k += 4) {
      const double a = __ldg(v + k);
      const int c = __ldg(ix + k);
#pragma unroll
      for (int j = 0; j < NV; ++j) acc[j] = fma(a, __ldg(x + j * stride + c), acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  }
  if (live && lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j)
      y[j * stride + r] = b ? __ldg(b + j * stride + r) - acc[j] : acc[j];
  }
}

// y = A^T x for CSR A without a stored transpose is not deterministic in
// parallel; transposes are stored explicitly by the caller instead.

__global__ void trisolve_kernel(int64_t n, int lower, const int* __restrict__ ip,
                                const int* __restrict__ ix, const double* __restrict__ v,
                                const double* __restrict__ invdiag, const double* __restrict__ b,
                                double* x, volatile unsigned int* flags, unsigned int* counter,
                                unsigned int epoch, int backoff_ns) {
  const int lane = threadIdx.x & 31;
  int64_t k;
  if (lane == 0) k = atomicAdd(counter, 1u);
  k = __shfl_sync(0xffffffffu, k, 0);
  if (k >= n) return;
  const int64_t row = lower ? k : n - 1 - k;
  const int beg = ip[row], end = ip[row + 1];
  // lanes wait for their dependencies, then accumulate in a fixed order
  double part = 0.0;
  for (int j = beg + lane; j < end; j += 32) {
    const int col = ix[j];
    while (flags[col] != epoch) {
      if (backoff_ns > 0) __nanosleep(backoff_ns);
    }
    __threadfence();
    part = __dadd_rn(part, __dmul_rn(v[j], reinterpret_cast<volatile double*>(x)[col]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_down_sync(0xffffffffu, part, o));
  if (lane == 0) {
    const double r = __dsub_rn(b[row], part);
    x[row] = invdiag ? __dmul_rn(r, invdiag[row]) : r;
    __threadfence();
    flags[row] = epoch;
  }
}

// Level-scheduled variant: rows of one dependency level are independent;
// one thread per row, rows listed level by level (level_rows), one launch
// per level (captured once into a CUDA graph by the host code).
__global__ void trisolve_level_kernel(int nrows_level, const int* __restrict__ rows,
                                      const int* __restrict__ ip, const int* __restrict__ ix,
                                      const double* __restrict__ v,
                                      const double* __restrict__ invdiag,
                                      const double* __restrict__ b, double* __restrict__ x) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows_level) return;
  const int row = rows[t];
  double acc = 0.0;
  for (int k = ip[row]; k < ip[row + 1]; ++k) acc = __dadd_rn(acc, __dmul_rn(v[k], x[ix[k]]));
  const double r = __dsub_rn(b[row], acc);
  x[row] = invdiag ? __dmul_rn(r, invdiag[row]) : r;
}

__global__ void permute_gather_kernel(int64_t n, const int* __restrict__ idx,
                                      const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void permute_scatter_kernel(int64_t n, const int* __restrict__ idx,
                                       const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
}

}  // namespace fb

using namespace fb;

namespace {
int upload_csr32(int64_t nrows, int64_t nnz, const int64_t* indptr, const int64_t* indices,
                 DevBuf<int>& ip, DevBuf<int>& ix) {
  FB_REQUIRE(nnz < (int64_t(1) << 31), "CSR too large for int32 indexing");
  std::vector<int> a(nrows + 1), b(nnz);
  for (int64_t i = 0; i <= nrows; ++i) a[i] = int(indptr[i]);
  for (int64_t i = 0; i < nnz; ++i) b[i] = int(indices[i]);
  FB_TRY_CUDA(ip.upload(a.data(), nrows + 1));
  FB_TRY_CUDA(ix.upload(b.data(), nnz));
  return FB_OK;
}
}  // namespace

extern "C" {

int fb_csr_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* indptr,
                  const int64_t* indices, const double* data, fb_csr** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(nrows >= 0 && ncols >= 0 && nnz >= 0, "negative sizes");
  FB_REQUIRE(indptr != nullptr, "indptr is NULL");
  FB_REQUIRE(indptr[0] == 0 && indptr[nrows] == nnz, "indptr inconsistent with nnz");
  for (int64_t k = 0; k < nnz; ++k)
    FB_REQUIRE(indices[k] >= 0 && indices[k] < ncols, "column index out of range");
  std::unique_ptr<fb_csr> A(new fb_csr());
  A->nrows = nrows;
  A->ncols = ncols;
  A->nnz = nnz;
  FB_REQUIRE(ncols < (int64_t(1) << 31), "CSR too wide for int32 column indices");
  {
    std::vector<int> b(nnz);
    for (int64_t i = 0; i < nnz; ++i) b[i] = int(indices[i]);
    FB_TRY_CUDA(A->indices.upload(b.data(), nnz));
  }
  FB_TRY_CUDA(A->indptr.upload(indptr, nrows + 1));
  FB_TRY_CUDA(A->data.upload(data, nnz));
  *out = A.release();
  return FB_OK;
}

void fb_csr_destroy(fb_csr* A) { delete A; }

int fb_csr_spmv(const fb_csr* A, const double* x, double* y, void* stream) {
  FB_REQUIRE(A != nullptr, "matrix is NULL");
  if (A->nrows == 0) return FB_OK;
  if (A->warp_rows)
    csr_spmv_group_kernel<4><<<ceil_div(A->nrows * 4, 256), 256, 0, as_stream(stream)>>>(
        A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, nullptr, y);
  else
    csr_spmv_kernel<<<ceil_div(A->nrows, 128), 128, 0, as_stream(stream)>>>(
        A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, nullptr, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_csr_residual(const fb_csr* A, const double* b, const double* x, double* y, void* stream) {
  FB_REQUIRE(A != nullptr, "matrix is NULL");
  if (A->nrows == 0) return FB_OK;
  if (A->warp_rows)
    csr_spmv_group_kernel<4><<<ceil_div(A->nrows * 4, 256), 256, 0, as_stream(stream)>>>(
        A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, b, y);
  else
    csr_spmv_kernel<<<ceil_div(A->nrows, 128), 128, 0, as_stream(stream)>>>(
        A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, b, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

// y_j = b_j - A x_j (b == NULL: y_j = A x_j) for nv vectors at a common stride
int fb_csr_residual_multi(const fb_csr* A, int nv, const double* b, const double* x, double* y,
                          int64_t stride, void* stream) {
  FB_REQUIRE(A != nullptr, "matrix is NULL");
  FB_REQUIRE(nv >= 1 && nv <= 4, "nv must be 1..4");
  FB_REQUIRE(A->warp_rows, "multi-vector SpMV needs a device-assembled (4 lanes per row) matrix");
  if (A->nrows == 0) return FB_OK;
  const unsigned grid = unsigned(ceil_div(A->nrows * 4, 256));
  cudaStream_t st = as_stream(stream);
  switch (nv) {
    case 1: csr_spmv_group_multi_kernel<1><<<grid, 256, 0, st>>>(A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, b, y, stride); break;
    case 2: csr_spmv_group_multi_kernel<2><<<grid, 256, 0, st>>>(A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, b, y, stride); break;
    case 3: csr_spmv_group_multi_kernel<3><<<grid, 256, 0, st>>>(A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, b, y, stride); break;
    default: csr_spmv_group_multi_kernel<4><<<grid, 256, 0, st>>>(A->nrows, A->indptr.ptr, A->indices.ptr, A->data.ptr, x, b, y, stride); break;
  }
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_trisolve_create(int64_t n, const int64_t* indptr, const int64_t* indices,
                       const double* data, int lower, int unit_diag, fb_trisolve** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(n >= 0 && indptr != nullptr, "bad triangular matrix");
  std::unique_ptr<fb_trisolve> T(new fb_trisolve());
  T->n = n;
  T->lower = lower ? 1 : 0;
  T->unit = unit_diag ? 1 : 0;
  std::vector<int64_t> ip(n + 1, 0), ix;
  std::vector<double> vv, inv(n, 1.0);
  ix.reserve(indptr[n]);
  vv.reserve(indptr[n]);
  for (int64_t r = 0; r < n; ++r) {
    bool has_diag = false;
    for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k) {
      const int64_t c = indices[k];
      FB_REQUIRE(c >= 0 && c < n, "column index out of range");
      if (c == r) {
        has_diag = true;
        if (!unit_diag) {
          FB_REQUIRE(data[k] != 0.0, "zero pivot on the diagonal");
          inv[r] = 1.0 / data[k];
        }
        continue;
      }
      FB_REQUIRE(lower ? (c < r) : (c > r), "entry outside the triangle");
      ix.push_back(c);
      vv.push_back(data[k]);
    }
    FB_REQUIRE(unit_diag || has_diag, "missing diagonal entry");
    ip[r + 1] = int64_t(ix.size());
  }
  int rc = upload_csr32(n, int64_t(ix.size()), ip.data(), ix.data(), T->indptr, T->indices);
  if (rc != FB_OK) return rc;
  FB_TRY_CUDA(T->data.upload(vv.data(), int64_t(vv.size())));
  if (!unit_diag) FB_TRY_CUDA(T->invdiag.upload(inv.data(), n));
  {
    // dependency levels: level[r] = 1 + max level of the rows r reads
    std::vector<int> level(n, 0);
    int maxl = 0;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t r = lower ? k : n - 1 - k;
      int lv = 0;
      for (int64_t j = ip[r]; j < ip[r + 1]; ++j) lv = std::max(lv, level[ix[j]] + 1);
      level[r] = lv;
      maxl = std::max(maxl, lv);
    }
    T->nlevels = n > 0 ? maxl + 1 : 0;
    T->level_ptr.assign(T->nlevels + 1, 0);
    for (int64_t r = 0; r < n; ++r) T->level_ptr[level[r] + 1]++;
    for (int l = 0; l < T->nlevels; ++l) T->level_ptr[l + 1] += T->level_ptr[l];
    std::vector<int> rows(n), pos(T->level_ptr.begin(), T->level_ptr.end() - 1);
    for (int64_t r = 0; r < n; ++r) rows[pos[level[r]]++] = int(r);
    FB_TRY_CUDA(T->level_rows.upload(rows.data(), n));
  }
  FB_TRY_CUDA(T->flags.alloc(n > 0 ? n : 1));
  FB_TRY_CUDA(cudaMemset(T->flags.ptr, 0, sizeof(unsigned int) * (n > 0 ? n : 1)));
  FB_TRY_CUDA(T->counter.alloc(1));
  *out = T.release();
  return FB_OK;
}

void fb_trisolve_destroy(fb_trisolve* T) { delete T; }

static int trisolve_levels(const fb_trisolve* T, const double* b, double* x, cudaStream_t st) {
  for (int l = 0; l < T->nlevels; ++l) {
    const int cnt = T->level_ptr[l + 1] - T->level_ptr[l];
    trisolve_level_kernel<<<ceil_div(cnt, 128), 128, 0, st>>>(
        cnt, T->level_rows.ptr + T->level_ptr[l], T->indptr.ptr, T->indices.ptr, T->data.ptr,
        T->unit ? nullptr : T->invdiag.ptr, b, x);
  }
  return FB_OK;
}

int fb_trisolve_solve(const fb_trisolve* T, const double* b, double* x, void* stream) {
  FB_REQUIRE(T != nullptr, "solver is NULL");
  FB_REQUIRE(b != x, "in-place triangular solve is not supported");
  if (T->n == 0) return FB_OK;
  cudaStream_t st = as_stream(stream);
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  FB_TRY_CUDA(cudaStreamIsCapturing(st, &cap_status));
  if (cap_status == cudaStreamCaptureStatusActive) {
    // inside a caller's stream capture (the device-resident CG loop): the
    // level kernels themselves become nodes of the caller's graph (no nested
    // graph launch, no host-side epoch)
    trisolve_levels(T, b, x, st);
    launch_counter() += T->nlevels;
    FB_CHECK_LAUNCH();
    return FB_OK;
  }
  if (g_trisolve_mode == 1) {
    // one graph per (b, x, stream) binding; re-captured when the operands change
    if (!T->graph || T->graph_b != b || T->graph_x != x || T->graph_stream != st) {
      if (T->graph) cudaGraphExecDestroy(T->graph);
      T->graph = nullptr;
      cudaStream_t cap;
      FB_TRY_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t g;
      FB_TRY_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      trisolve_levels(T, b, x, cap);
      FB_TRY_CUDA(cudaStreamEndCapture(cap, &g));
      FB_TRY_CUDA(cudaGraphInstantiate(&T->graph, g, 0));
      cudaGraphDestroy(g);
      cudaStreamDestroy(cap);
      T->graph_b = b;
      T->graph_x = x;
      T->graph_stream = st;
    }
    FB_TRY_CUDA(cudaGraphLaunch(T->graph, st));
    launch_counter() += T->nlevels;
    return FB_OK;
  }
  T->epoch += 1;
  if (T->epoch == 0) {  // wrapped: reset the flags
    FB_TRY_CUDA(cudaMemsetAsync(T->flags.ptr, 0, sizeof(unsigned int) * T->n, st));
    T->epoch = 1;
  }
  FB_TRY_CUDA(cudaMemsetAsync(T->counter.ptr, 0, sizeof(unsigned int), st));
  const int64_t threads = T->n * 32;
  trisolve_kernel<<<ceil_div(threads, 256), 256, 0, st>>>(
      T->n, T->lower, T->indptr.ptr, T->indices.ptr, T->data.ptr,
      T->unit ? nullptr : T->invdiag.ptr, b, x, T->flags.ptr, T->counter.ptr, T->epoch,
      g_trisolve_backoff);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_trisolve_levels(const fb_trisolve* T) { return T ? T->nlevels : -1; }

int fb_set_trisolve_mode(int mode, int backoff_ns) {
  FB_REQUIRE(mode == 0 || mode == 1, "mode must be 0 (sync-free) or 1 (level graph)");
  g_trisolve_mode = mode;
  g_trisolve_backoff = backoff_ns;
  return FB_OK;
}

int fb_permute(int64_t n, const int* idx, const double* src, double* dst, int scatter,
               void* stream) {
  if (n <= 0) return FB_OK;
  if (scatter)
    permute_scatter_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, idx, src, dst);
  else
    permute_gather_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, idx, src, dst);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

// ILU(0) in place on a square CSR matrix with sorted column indices, IKJ
// variant (kernels/numba_backend.py:64-103 semantics): returns -1 on
// success, else the first row whose pivot magnitude fell below 1e-300.
int64_t fb_ilu0_factor_host(int64_t n, const int64_t* indptr, const int64_t* indices,
                            double* data) {
  std::vector<int64_t> dpos(n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t found = -1;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
      if (indices[k] == i) {
        found = k;
        break;
      }
    if (found < 0) return i;
    dpos[i] = found;
  }
  std::vector<int64_t> where(n, -1);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t rb = indptr[i], re = indptr[i + 1];
    for (int64_t k = rb; k < re; ++k) where[indices[k]] = k;
    for (int64_t k = rb; k < re; ++k) {
      const int64_t c = indices[k];
      if (c >= i) break;
      const double piv = data[dpos[c]];
      if (std::fabs(piv) < 1e-300) return c;
      const double l = data[k] / piv;
      data[k] = l;
      for (int64_t kk = dpos[c] + 1; kk < indptr[c + 1]; ++kk) {
        const int64_t t = where[indices[kk]];
        if (t >= 0) data[t] -= l * data[kk];
      }
    }
    for (int64_t k = rb; k < re; ++k) where[indices[k]] = -1;
    if (std::fabs(data[dpos[i]]) < 1e-300) return i;
  }
  return -1;
}

}  // extern "C"
