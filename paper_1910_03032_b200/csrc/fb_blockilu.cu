// Block-Jacobi ILU(0) smoother application on the device ("scale mode" of
// the LOR V-cycle, SURVEY.md 8(e')).
//
// The reference smooths every LOR level with ONE global ILU(0) in first-touch
// order (solvers.py:269-311); its triangular solves are a dependency chain of
// ~60 n levels (449-1409 at 36k-0.9M DoFs) -- inherently sequential on any
// device.  Here the level matrix is restricted to element-cube blocks (2^d
// elements per block, every DoF in its first-touch owner element's block,
// the reference's first-touch order kept inside each block) and factored
// block-wise on the host.  On the device ONE launch applies a whole smoother
// sweep: one CTA per block gathers its right-hand side through the
// permutation into shared memory, runs the forward (L then U) or transposed
// (U^T then L^T) triangular solves level by level inside shared memory, and
// scatters the result.  The chain per block is ~89 (p=4) - 131 (p=7) levels
// regardless of the problem size, and blocks never talk to each other, so the
// sweep also shards across GPUs with identical math.
#include <algorithm>
#include <memory>
#include <vector>

#include "fb_common.cuh"

namespace {

struct TriPart {
  fb::DevBuf<int> ip, ix;        // CSR (global new numbering), off-diagonal only
  fb::DevBuf<double> v;
  fb::DevBuf<double> invdiag;    // empty for unit diagonal
  fb::DevBuf<int> rows;          // rows of each block, grouped by level
  fb::DevBuf<int> grp;           // level-group row offsets into `rows`
  fb::DevBuf<int> blk_grp;       // (nblocks + 1) offsets into grp
};

}  // namespace

struct fb_blockilu {
  int64_t n = 0;
  int nblocks = 0;
  int max_block = 0;
  fb::DevBuf<int> block_ptr;  // (nblocks + 1) row offsets (new numbering)
  fb::DevBuf<int> new2old;    // new -> original DoF index
  TriPart L, U, Ut, Lt;       // forward: L (unit) then U; backward: U^T then L^T (unit)
};

namespace fb {

struct TriView {
  const int* ip;
  const int* ix;
  const double* v;
  const double* invdiag;
  const int* rows;
  const int* grp;
  const int* blk_grp;
};

__device__ __forceinline__ void block_tri(const TriView& T, int b, int bs, double* y) {
  const int g0 = T.blk_grp[b], g1 = T.blk_grp[b + 1];
  for (int g = g0; g < g1; ++g) {
    const int r0 = T.grp[g], r1 = T.grp[g + 1];
    for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) {
      const int row = T.rows[k];
      double acc = 0.0;
      for (int e = T.ip[row]; e < T.ip[row + 1]; ++e)
        acc = __dadd_rn(acc, __dmul_rn(T.v[e], y[T.ix[e] - bs]));
      const double r = __dsub_rn(y[row - bs], acc);
      y[row - bs] = T.invdiag ? __dmul_rn(r, T.invdiag[row]) : r;
    }
    __syncthreads();
  }
}

__global__ void block_ilu_kernel(const int* __restrict__ block_ptr,
                                 const int* __restrict__ new2old, TriView A, TriView B,
                                 const double* __restrict__ r, double* __restrict__ out) {
  extern __shared__ double y[];
  const int b = blockIdx.x;
  const int bs = block_ptr[b], be = block_ptr[b + 1];
  for (int i = threadIdx.x; i < be - bs; i += blockDim.x) y[i] = r[new2old[bs + i]];
  __syncthreads();
  block_tri(A, b, bs, y);
  block_tri(B, b, bs, y);
  for (int i = threadIdx.x; i < be - bs; i += blockDim.x) out[new2old[bs + i]] = y[i];
}

}  // namespace fb

using namespace fb;

namespace {

// Build one triangular part: strict off-diagonal CSR + inverse diagonal + the
// per-block level grouping of its rows.
int build_part(int64_t n, const std::vector<int>& bptr, const std::vector<int64_t>& ip,
               const std::vector<int64_t>& ix, const std::vector<double>& v, bool lower,
               bool unit, TriPart& P) {
  std::vector<int> oip(n + 1, 0), oix;
  std::vector<double> ov, inv(n, 1.0);
  oix.reserve(ix.size());
  ov.reserve(ix.size());
  for (int64_t r = 0; r < n; ++r) {
    for (int64_t k = ip[r]; k < ip[r + 1]; ++k) {
      const int64_t c = ix[k];
      if (c == r) {
        if (!unit) {
          FB_REQUIRE(v[k] != 0.0, "zero pivot in block ILU factor");
          inv[r] = 1.0 / v[k];
        }
        continue;
      }
      FB_REQUIRE(lower ? c < r : c > r, "entry outside the triangle");
      oix.push_back(int(c));
      ov.push_back(v[k]);
    }
    oip[r + 1] = int(oix.size());
  }
  // levels within each block
  const int nb = int(bptr.size()) - 1;
  std::vector<int> level(n, 0);
  std::vector<int> rows;
  std::vector<int> grp;
  std::vector<int> blk_grp(nb + 1, 0);
  rows.reserve(n);
  grp.push_back(0);
  for (int b = 0; b < nb; ++b) {
    const int bs = bptr[b], be = bptr[b + 1];
    int maxl = 0;
    for (int k = 0; k < be - bs; ++k) {
      const int r = lower ? bs + k : be - 1 - k;
      int lv = 0;
      for (int e = oip[r]; e < oip[r + 1]; ++e) {
        FB_REQUIRE(oix[e] >= bs && oix[e] < be, "block ILU factor couples two blocks");
        lv = std::max(lv, level[oix[e]] + 1);
      }
      level[r] = lv;
      maxl = std::max(maxl, lv);
    }
    std::vector<int> cnt(maxl + 2, 0);
    for (int r = bs; r < be; ++r) cnt[level[r] + 1]++;
    for (int l = 0; l <= maxl; ++l) cnt[l + 1] += cnt[l];
    const int base = int(rows.size());
    rows.resize(base + (be - bs));
    std::vector<int> pos(cnt.begin(), cnt.end() - 1);
    for (int r = bs; r < be; ++r) rows[base + pos[level[r]]++] = r;
    for (int l = 0; l <= maxl; ++l) grp.push_back(base + cnt[l + 1]);
    blk_grp[b + 1] = int(grp.size()) - 1;
  }
  FB_TRY_CUDA(P.ip.upload(oip.data(), n + 1));
  FB_TRY_CUDA(P.ix.upload(oix.data(), int64_t(oix.size())));
  FB_TRY_CUDA(P.v.upload(ov.data(), int64_t(ov.size())));
  if (!unit) FB_TRY_CUDA(P.invdiag.upload(inv.data(), n));
  FB_TRY_CUDA(P.rows.upload(rows.data(), int64_t(rows.size())));
  FB_TRY_CUDA(P.grp.upload(grp.data(), int64_t(grp.size())));
  FB_TRY_CUDA(P.blk_grp.upload(blk_grp.data(), nb + 1));
  return FB_OK;
}

void transpose_csr(int64_t n, const int64_t* ip, const int64_t* ix, const double* v,
                   std::vector<int64_t>& tip, std::vector<int64_t>& tix, std::vector<double>& tv) {
  tip.assign(n + 1, 0);
  const int64_t nnz = ip[n];
  for (int64_t k = 0; k < nnz; ++k) tip[ix[k] + 1]++;
  for (int64_t i = 0; i < n; ++i) tip[i + 1] += tip[i];
  tix.resize(nnz);
  tv.resize(nnz);
  std::vector<int64_t> pos(tip.begin(), tip.end() - 1);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = ip[r]; k < ip[r + 1]; ++k) {
      const int64_t p = pos[ix[k]]++;
      tix[p] = r;
      tv[p] = v[k];
    }
}

TriView view(const TriPart& P, bool unit) {
  return TriView{P.ip.ptr, P.ix.ptr, P.v.ptr, unit ? nullptr : P.invdiag.ptr,
                 P.rows.ptr, P.grp.ptr, P.blk_grp.ptr};
}

}  // namespace

extern "C" {

// F: the block-diagonal ILU(0) factor in the new (block-major) numbering, as
// CSR with sorted columns (strict lower part = L, unit diagonal implied;
// upper part incl. diagonal = U).  block_ptr: (nblocks+1) row offsets.
// new2old: new -> original DoF index.
int fb_blockilu_create(int64_t n, int nblocks, const int64_t* block_ptr,
                       const int64_t* new2old, const int64_t* indptr, const int64_t* indices,
                       const double* data, fb_blockilu** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(n >= 0 && nblocks >= 0 && block_ptr && new2old && indptr, "bad block ILU input");
  FB_REQUIRE(block_ptr[0] == 0 && block_ptr[nblocks] == n, "block_ptr must cover all rows");
  std::unique_ptr<fb_blockilu> B(new fb_blockilu());
  B->n = n;
  B->nblocks = nblocks;
  std::vector<int> bptr(nblocks + 1), n2o(n);
  for (int b = 0; b <= nblocks; ++b) bptr[b] = int(block_ptr[b]);
  for (int b = 0; b < nblocks; ++b) B->max_block = std::max(B->max_block, bptr[b + 1] - bptr[b]);
  for (int64_t i = 0; i < n; ++i) n2o[i] = int(new2old[i]);
  // split F into L (strict lower) and U (upper incl. diagonal)
  std::vector<int64_t> lip(n + 1, 0), lix, uip(n + 1, 0), uix;
  std::vector<double> lv, uv;
  for (int64_t r = 0; r < n; ++r) {
    for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k) {
      if (indices[k] < r) {
        lix.push_back(indices[k]);
        lv.push_back(data[k]);
      } else {
        uix.push_back(indices[k]);
        uv.push_back(data[k]);
      }
    }
    lip[r + 1] = int64_t(lix.size());
    uip[r + 1] = int64_t(uix.size());
  }
  std::vector<int64_t> tip, tix;
  std::vector<double> tv;
  int rc = build_part(n, bptr, lip, lix, lv, true, true, B->L);
  if (rc != FB_OK) return rc;
  rc = build_part(n, bptr, uip, uix, uv, false, false, B->U);
  if (rc != FB_OK) return rc;
  transpose_csr(n, uip.data(), uix.data(), uv.data(), tip, tix, tv);
  rc = build_part(n, bptr, tip, tix, tv, true, false, B->Ut);
  if (rc != FB_OK) return rc;
  transpose_csr(n, lip.data(), lix.data(), lv.data(), tip, tix, tv);
  rc = build_part(n, bptr, tip, tix, tv, false, true, B->Lt);
  if (rc != FB_OK) return rc;
  FB_TRY_CUDA(B->block_ptr.upload(bptr.data(), nblocks + 1));
  FB_TRY_CUDA(B->new2old.upload(n2o.data(), n));
  FB_REQUIRE(size_t(B->max_block) * 8 <= 200 * 1024, "block too large for shared memory");
  *out = B.release();
  return FB_OK;
}

void fb_blockilu_destroy(fb_blockilu* B) { delete B; }

// out = (LU)^-1 r (transpose=0) or (LU)^-T r (transpose=1), both in the
// original numbering.
int fb_blockilu_apply(const fb_blockilu* B, int transpose, const double* r, double* out,
                      void* stream) {
  FB_REQUIRE(B != nullptr, "smoother is NULL");
  FB_REQUIRE(r != out, "in-place smoother application is not supported");
  if (B->nblocks == 0) return FB_OK;
  const size_t smem = size_t(B->max_block) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    FB_TRY_CUDA(cudaFuncSetAttribute(block_ilu_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  const TriView a = transpose ? view(B->Ut, false) : view(B->L, true);
  const TriView b = transpose ? view(B->Lt, true) : view(B->U, false);
  block_ilu_kernel<<<B->nblocks, 64, smem, as_stream(stream)>>>(B->block_ptr.ptr,
                                                                 B->new2old.ptr, a, b, r, out);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

// Dense coarse solve: out = Ainv x with a stored dense inverse (row-major),
// one warp per row, fixed-order reduction.
__global__ void dense_mv_kernel(int64_t n, const double* __restrict__ M,
                                const double* __restrict__ x, double* __restrict__ y) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* m = M + row * n;
  double acc = 0.0;
  for (int64_t j = lane; j < n; j += 32) acc = fma(__ldg(m + j), __ldg(x + j), acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) y[row] = acc;
}

int fb_dense_mv(int64_t n, const double* M, const double* x, double* y, void* stream) {
  if (n <= 0) return FB_OK;
  dense_mv_kernel<<<ceil_div(n * 32, 256), 256, 0, as_stream(stream)>>>(n, M, x, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

}  // extern "C"
