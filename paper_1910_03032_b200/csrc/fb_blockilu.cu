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
#include <cstdlib>
#include <algorithm>
#include <memory>
#include <vector>

#include <cub/cub.cuh>

#include "fb_common.cuh"
#include "fb_internal.cuh"

namespace {

struct TriPart {
  fb::DevBuf<int64_t> ip;        // CSR (global new numbering), off-diagonal only
  fb::DevBuf<int> ix;
  fb::DevBuf<double> v;
  fb::DevBuf<double> invdiag;    // empty for unit diagonal
  fb::DevBuf<int> rows;          // rows of each block, grouped by level
  fb::DevBuf<int> grp;           // level-group row offsets into `rows`
  fb::DevBuf<int> blk_grp;       // (nblocks + 1) offsets into grp
  // padded row layout for the sweeps: row r's entries at r*width, values
  // and shared-memory byte offsets of the column inside the block (padding:
  // value 0 at offset 0, so sequential sums are unchanged)
  int width = 0;
  fb::DevBuf<double> ev;
  fb::DevBuf<unsigned short> eo;
  // level-packed layout (block_ilu_packed_kernel): one contiguous, 16-byte
  // aligned chunk per dependency level of every block
  //   [values E x f64 | inverse diagonal R x f64 (U parts) | local columns
  //    E x u16 | local rows R x u16 | row starts R x u16 | row lengths R x u16]
  // so a TMA bulk copy stages one level into a shared-memory ring
  fb::DevBuf<unsigned char> pk;
  fb::DevBuf<int64_t> loff;   // (levels + 1) byte offsets of the chunks
  fb::DevBuf<int> lne;        // entries per level
  int max_chunk = 0;
  int lev_group = 1;          // levels staged per bulk copy
  int max_group = 0;          // largest staged span (bytes)
  int64_t nnz = 0;            // strict-triangle entries (kept when the CSR is freed)
};

}  // namespace
namespace {
inline bool small_grid(const fb_blockilu* B);  // grids of a few waves (below)
}  // namespace

static int g_bilu_pipe = 2;  // 0: CSR sweep, 1: CSR + next-level loads, 2: padded rows for large blocks, else 1
static int g_bilu_lanes = 0;  // 0 = by block size
static int g_bilu_deep = 1;   // two-level lookahead for one-wave grids (0: off)
static int g_bilu_packed = 1; // level-packed TMA-ring sweep for blocks > 160 rows (0: off)

struct fb_blockilu {
  int64_t n = 0;
  int nblocks = 0;
  int max_block = 0;
  fb::DevBuf<int> block_ptr;  // (nblocks + 1) row offsets (new numbering)
  fb::DevBuf<int> new2old;    // new -> original DoF index
  TriPart L, U, Ut, Lt;       // forward: L (unit) then U; backward: U^T then L^T (unit)
  int ell_w = 0;              // padded-row width of all parts (0: CSR sweeps)
  int max_grp = 0;            // most level groups of one block over the four parts
};

static int build_ell(fb_blockilu* B);

namespace fb {

struct TriView {
  const double* ev;
  const unsigned short* eo;
  const int64_t* ip;
  const int* ix;
  const double* v;
  const double* invdiag;
  const int* rows;
  const int* grp;
  const int* blk_grp;
};

constexpr int kRowBuf = 13;  // strict triangle of a 27-point row: <= 13 entries

struct RowLoad {
  int c[kRowBuf];
  double a[kRowBuf];
  int n, row;
  int64_t e0;
  double inv;
};

__device__ __forceinline__ void bulk_prefetch_range(const void* p, int64_t bytes) {
  uintptr_t b = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + uintptr_t(bytes) + 15) & ~uintptr_t(15);
  while (b < e) {
    const uint32_t len = uint32_t((e - b) > (1u << 20) ? (1u << 20) : (e - b));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(len) : "memory");
    b += len;
  }
}

// Issue the loads of one row (position k of the block's level order); all
// addresses come from shared memory, so the loads of the next level are in
// flight while the current level computes.
__device__ __forceinline__ void row_issue(const TriView& T, const unsigned short* srow,
                                          const int* soff, int64_t ebase, int bs, int k,
                                          RowLoad& R) {
  const int lr = srow[k];
  R.row = bs + lr;
  R.e0 = ebase + soff[lr];
  R.n = soff[lr + 1] - soff[lr];
#pragma unroll
  for (int u = 0; u < kRowBuf; ++u) {
    const bool ok = u < R.n;
    R.c[u] = ok ? __ldg(T.ix + R.e0 + u) : bs;
    R.a[u] = ok ? __ldg(T.v + R.e0 + u) : 0.0;
  }
  R.inv = T.invdiag ? __ldg(T.invdiag + R.row) : 1.0;
}

__device__ __forceinline__ void row_finish(const TriView& T, const RowLoad& R, int bs, double* y) {
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < kRowBuf; ++u)
    if (u < R.n) acc = __dadd_rn(acc, __dmul_rn(R.a[u], y[R.c[u] - bs]));
  for (int u = kRowBuf; u < R.n; ++u)  // longer rows (not produced by 27-point LOR levels)
    acc = __dadd_rn(acc, __dmul_rn(__ldg(T.v + R.e0 + u), y[__ldg(T.ix + R.e0 + u) - bs]));
  const double r = __dsub_rn(y[R.row - bs], acc);
  y[R.row - bs] = T.invdiag ? __dmul_rn(r, R.inv) : r;
}

// Triangular solves of BPW = 32 / LPB blocks by ONE warp: lanes
// [j LPB, (j+1) LPB) own block j and walk its level groups in shared memory
// (__syncwarp between levels; the warp runs the longest schedule of its
// blocks).  Level-parallel rows are few per level (1.5 at p = 2, 7 at p = 4,
// 24 at p = 7), so several blocks share a warp's instruction stream.  The
// block's level groups, level-ordered local rows and entry offsets are staged
// in shared memory and its factor entries prefetched into L2; with PIPE the
// loads of level g+1 are issued before level g computes.  Every row's sum
// stays sequential in index order (bitwise the host sweep).
template <int LPB, int PIPE>
__device__ __forceinline__ void block_tri(const TriView& T, bool live, int b, int bs, int nb,
                                          double* y, int* sgrp, unsigned short* srow,
                                          int* soff) {
  const int t = threadIdx.x % LPB;
  int G = 0;
  int64_t ebase = 0;
  if (live) {
    const int g0 = T.blk_grp[b];
    G = T.blk_grp[b + 1] - g0;
    ebase = T.ip[bs];
    for (int i = t; i <= G; i += LPB) sgrp[i] = T.grp[g0 + i] - bs;
    for (int i = t; i < nb; i += LPB) srow[i] = (unsigned short)(T.rows[bs + i] - bs);
    for (int i = t; i <= nb; i += LPB) soff[i] = int(T.ip[bs + i] - ebase);
    if (t == 0) {
      const int64_t ne = T.ip[bs + nb] - ebase;
      bulk_prefetch_range(T.ix + ebase, ne * int64_t(sizeof(int)));
      bulk_prefetch_range(T.v + ebase, ne * int64_t(sizeof(double)));
    }
  }
  int Gmax = G;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Gmax = max(Gmax, __shfl_xor_sync(0xffffffffu, Gmax, o));
  __syncwarp();
  if constexpr (PIPE == 2) {
    // two levels ahead (small grids, one wave: latency, not occupancy, bounds
    // the sweep): rows of level g+2 load while level g computes
    RowLoad cur, n1, n2;
    if (G > 0 && t < sgrp[1] - sgrp[0]) row_issue(T, srow, soff, ebase, bs, sgrp[0] + t, cur);
    if (G > 1 && t < sgrp[2] - sgrp[1]) row_issue(T, srow, soff, ebase, bs, sgrp[1] + t, n1);
    for (int g = 0; g < Gmax; ++g) {
      if (g < G) {
        const int r0 = sgrp[g], r1 = sgrp[g + 1];
        const bool nx = g + 2 < G && t < sgrp[g + 3] - sgrp[g + 2];
        if (nx) row_issue(T, srow, soff, ebase, bs, sgrp[g + 2] + t, n2);
        if (t < r1 - r0) row_finish(T, cur, bs, y);
        for (int k = r0 + t + LPB; k < r1; k += LPB) {  // levels wider than LPB
          RowLoad w;
          row_issue(T, srow, soff, ebase, bs, k, w);
          row_finish(T, w, bs, y);
        }
        cur = n1;
        n1 = n2;
      }
      __syncwarp();
    }
  } else if constexpr (PIPE == 1) {
    RowLoad cur, nxt;
    if (G > 0 && t < sgrp[1] - sgrp[0]) row_issue(T, srow, soff, ebase, bs, sgrp[0] + t, cur);
    for (int g = 0; g < Gmax; ++g) {
      if (g < G) {
        const int r0 = sgrp[g], r1 = sgrp[g + 1];
        const bool nx = g + 1 < G && t < sgrp[g + 2] - r1;
        if (nx) row_issue(T, srow, soff, ebase, bs, r1 + t, nxt);
        if (t < r1 - r0) row_finish(T, cur, bs, y);
        for (int k = r0 + t + LPB; k < r1; k += LPB) {  // levels wider than LPB
          RowLoad w;
          row_issue(T, srow, soff, ebase, bs, k, w);
          row_finish(T, w, bs, y);
        }
        if (nx) cur = nxt;
      }
      __syncwarp();
    }
  } else {
    for (int g = 0; g < Gmax; ++g) {
      if (g < G) {
        const int r0 = sgrp[g], r1 = sgrp[g + 1];
        for (int k = r0 + t; k < r1; k += LPB) {
          RowLoad w;
          row_issue(T, srow, soff, ebase, bs, k, w);
          row_finish(T, w, bs, y);
        }
      }
      __syncwarp();
    }
  }
}

// Quad-row variant for blocks with several rows per level (p >= 4 levels):
// each row is split over 4 lanes (entries s, s+4, s+8, ... for sub-lane s),
// the partial sums are combined with two butterfly shuffles (fixed order,
// deterministic; not the sequential order of block_tri), and the next level's
// entries are loaded before the current level computes.
struct QuadLoad {
  int c[4];
  double a[4];
  int n, row;
  int64_t e0;
  double inv;
};

__device__ __forceinline__ void quad_issue(const TriView& T, const unsigned short* srow,
                                           const int* soff, int64_t ebase, int bs, int k, int s,
                                           QuadLoad& R) {
  const int lr = srow[k];
  R.row = bs + lr;
  R.e0 = ebase + soff[lr];
  R.n = soff[lr + 1] - soff[lr];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = s + 4 * u;
    const bool ok = i < R.n;
    R.c[u] = ok ? __ldg(T.ix + R.e0 + i) : bs;
    R.a[u] = ok ? __ldg(T.v + R.e0 + i) : 0.0;
  }
  R.inv = T.invdiag ? __ldg(T.invdiag + R.row) : 1.0;
}

__device__ __forceinline__ double quad_partial(const TriView& T, const QuadLoad& R, int bs, int s,
                                               const double* y) {
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) acc = fma(R.a[u], y[R.c[u] - bs], acc);
  for (int i = s + 16; i < R.n; i += 4)  // rows longer than 16 entries
    acc = fma(__ldg(T.v + R.e0 + i), y[__ldg(T.ix + R.e0 + i) - bs], acc);
  return acc;
}

template <int LPB>
__device__ __forceinline__ void block_tri_quad(const TriView& T, bool live, int b, int bs, int nb,
                                               double* y, int* sgrp, unsigned short* srow,
                                               int* soff) {
  constexpr int RPP = LPB / 4;  // rows per pass
  const int t = threadIdx.x % LPB, q = t >> 2, s = t & 3;
  const unsigned qmask = 0xFu << (threadIdx.x & ~3u);
  int G = 0;
  int64_t ebase = 0;
  if (live) {
    const int g0 = T.blk_grp[b];
    G = T.blk_grp[b + 1] - g0;
    ebase = T.ip[bs];
    for (int i = t; i <= G; i += LPB) sgrp[i] = T.grp[g0 + i] - bs;
    for (int i = t; i < nb; i += LPB) srow[i] = (unsigned short)(T.rows[bs + i] - bs);
    for (int i = t; i <= nb; i += LPB) soff[i] = int(T.ip[bs + i] - ebase);
    if (t == 0) {
      const int64_t ne = T.ip[bs + nb] - ebase;
      bulk_prefetch_range(T.ix + ebase, ne * int64_t(sizeof(int)));
      bulk_prefetch_range(T.v + ebase, ne * int64_t(sizeof(double)));
    }
  }
  int Gmax = G;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Gmax = max(Gmax, __shfl_xor_sync(0xffffffffu, Gmax, o));
  __syncwarp();
  QuadLoad cur, nxt;
  if (G > 0 && q < sgrp[1] - sgrp[0]) quad_issue(T, srow, soff, ebase, bs, sgrp[0] + q, s, cur);
  for (int g = 0; g < Gmax; ++g) {
    if (g < G) {
      const int r0 = sgrp[g], r1 = sgrp[g + 1];
      const bool nx = g + 1 < G && q < sgrp[g + 2] - r1;
      if (nx) quad_issue(T, srow, soff, ebase, bs, r1 + q, s, nxt);
      // quads are converged: every lane of a quad has the same q
      if (q < r1 - r0) {
        double acc = quad_partial(T, cur, bs, s, y);
        acc += __shfl_xor_sync(qmask, acc, 1);
        acc += __shfl_xor_sync(qmask, acc, 2);
        if (s == 0) {
          const double r = y[cur.row - bs] - acc;
          y[cur.row - bs] = T.invdiag ? r * cur.inv : r;
        }
      }
      for (int k = r0 + q + RPP; k < r1; k += RPP) {  // levels wider than one pass
        QuadLoad w;
        quad_issue(T, srow, soff, ebase, bs, k, s, w);
        double acc = quad_partial(T, w, bs, s, y);
        acc += __shfl_xor_sync(qmask, acc, 1);
        acc += __shfl_xor_sync(qmask, acc, 2);
        if (s == 0) {
          const double r = y[w.row - bs] - acc;
          y[w.row - bs] = T.invdiag ? r * w.inv : r;
        }
      }
      if (nx) cur = nxt;
    }
    __syncwarp();
  }
}

// One block's shared-memory region (bytes): y (8 B per row), the level-group
// offsets (max_grp + 1 ints: sized by the deepest block, not by its rows),
// the row entry offsets (CSR sweep only, 4 B per row) and the level-ordered
// local rows (2 B per row).  Smaller regions keep more blocks resident per SM
// (the sweeps are latency bound).  max_grp < 0: unknown, size by rows.
__host__ __device__ inline size_t block_ilu_smem(int max_block, int max_grp = -1) {
  const size_t g = size_t(max_grp >= 0 ? max_grp : max_block) + 1;
  return (size_t(max_block) * 14 + 4 * g + 4 + 15) / 16 * 16;
}
__host__ __device__ inline size_t block_ilu_ell_smem(int max_block, int max_grp = -1) {
  const size_t g = size_t(max_grp >= 0 ? max_grp : max_block) + 1;
  return (size_t(max_block) * 10 + 4 * g + 15) / 16 * 16;
}

template <int LPB, int PIPE>
__global__ void __launch_bounds__(32) block_ilu_kernel(const int* __restrict__ block_ptr,
                                                       int nblocks,
                                                       const int* __restrict__ new2old,
                                                       TriView A, TriView B,
                                                       const double* __restrict__ r,
                                                       double* __restrict__ out, int max_block,
                                                       int max_grp) {
  extern __shared__ double smem_d[];
  const int j = threadIdx.x / LPB, t = threadIdx.x % LPB;
  const size_t per = block_ilu_smem(max_block, max_grp) / 8;  // doubles per block region
  double* y = smem_d + j * per;
  int* sgrp = reinterpret_cast<int*>(y + max_block);
  int* soff = sgrp + max_grp + 1;
  unsigned short* srow = reinterpret_cast<unsigned short*>(soff + max_block + 1);
  const int b = blockIdx.x * (32 / LPB) + j;
  const bool live = b < nblocks;
  const int bs = live ? block_ptr[b] : 0, be = live ? block_ptr[b + 1] : 0;
  // new2old == nullptr: the level is numbered block-major already
  for (int i = t; i < be - bs; i += LPB) y[i] = r[new2old ? new2old[bs + i] : bs + i];
  __syncwarp();
  if constexpr (LPB >= 4 && !PIPE) {  // PIPE=false selects the quad-row sweep here
    block_tri_quad<LPB>(A, live, b, bs, be - bs, y, sgrp, srow, soff);
    block_tri_quad<LPB>(B, live, b, bs, be - bs, y, sgrp, srow, soff);
  } else {
    block_tri<LPB, PIPE>(A, live, b, bs, be - bs, y, sgrp, srow, soff);
    block_tri<LPB, PIPE>(B, live, b, bs, be - bs, y, sgrp, srow, soff);
  }
  for (int i = t; i < be - bs; i += LPB) out[new2old ? new2old[bs + i] : bs + i] = y[i];
}

// ---- padded-row (ELL) sweep: the production path -------------------------
// Same schedule as block_tri (one warp serves 32/LPB blocks, level groups in
// shared memory, next level's loads issued before the current level
// computes) but every row is W padded entries: values as double2 and
// shared-memory byte offsets as uint4 vector loads, no per-entry predicates
// or address arithmetic.  Padding is value 0 at offset 0, so each row's sum
// is still the sequential index-order sum (bitwise the CSR sweep).
template <int W>
struct EllRow {
  double a[W];
  unsigned int o[W / 2];  // two 16-bit byte offsets per word
  int row;
  double inv;
};

template <int W>
__device__ __forceinline__ void ell_issue(const TriView& T, const unsigned short* srow, int bs,
                                          int k, EllRow<W>& R) {
  R.row = bs + srow[k];
  const double2* va = reinterpret_cast<const double2*>(T.ev + int64_t(R.row) * W);
  const uint4* oa = reinterpret_cast<const uint4*>(T.eo + int64_t(R.row) * W);
#pragma unroll
  for (int u = 0; u < W / 2; ++u) {
    const double2 t = __ldg(va + u);
    R.a[2 * u] = t.x;
    R.a[2 * u + 1] = t.y;
  }
#pragma unroll
  for (int u = 0; u < W / 8; ++u) {
    const uint4 t = __ldg(oa + u);
    R.o[4 * u] = t.x;
    R.o[4 * u + 1] = t.y;
    R.o[4 * u + 2] = t.z;
    R.o[4 * u + 3] = t.w;
  }
  R.inv = T.invdiag ? __ldg(T.invdiag + R.row) : 1.0;
}

template <int W>
__device__ __forceinline__ void ell_finish(const TriView& T, const EllRow<W>& R, int bs,
                                           double* y) {
  const char* yb = reinterpret_cast<const char*>(y);
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < W; ++u) {
    const unsigned off = (u & 1) ? (R.o[u >> 1] >> 16) : (R.o[u >> 1] & 0xFFFFu);
    acc = __dadd_rn(acc, __dmul_rn(R.a[u], *reinterpret_cast<const double*>(yb + off)));
  }
  const double r = __dsub_rn(y[R.row - bs], acc);
  y[R.row - bs] = T.invdiag ? __dmul_rn(r, R.inv) : r;
}

template <int LPB, int W, int D = 1>
__device__ __forceinline__ void block_tri_ell(const TriView& T, bool live, int b, int bs, int nb,
                                              double* y, int* sgrp, unsigned short* srow) {
  const int t = threadIdx.x % LPB;
  int G = 0;
  if (live) {
    const int g0 = T.blk_grp[b];
    G = T.blk_grp[b + 1] - g0;
    for (int i = t; i <= G; i += LPB) sgrp[i] = T.grp[g0 + i] - bs;
    for (int i = t; i < nb; i += LPB) srow[i] = (unsigned short)(T.rows[bs + i] - bs);
    if (t == 0) {
      bulk_prefetch_range(T.ev + int64_t(bs) * W, int64_t(nb) * W * int64_t(sizeof(double)));
      bulk_prefetch_range(T.eo + int64_t(bs) * W, int64_t(nb) * W * int64_t(sizeof(unsigned short)));
    }
  }
  int Gmax = G;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Gmax = max(Gmax, __shfl_xor_sync(0xffffffffu, Gmax, o));
  __syncwarp();
  if constexpr (D == 2) {  // two levels ahead (see block_tri)
    EllRow<W> cur, n1, n2;
    if (G > 0 && t < sgrp[1] - sgrp[0]) ell_issue<W>(T, srow, bs, sgrp[0] + t, cur);
    if (G > 1 && t < sgrp[2] - sgrp[1]) ell_issue<W>(T, srow, bs, sgrp[1] + t, n1);
    for (int g = 0; g < Gmax; ++g) {
      if (g < G) {
        const int r0 = sgrp[g], r1 = sgrp[g + 1];
        const bool nx = g + 2 < G && t < sgrp[g + 3] - sgrp[g + 2];
        if (nx) ell_issue<W>(T, srow, bs, sgrp[g + 2] + t, n2);
        if (t < r1 - r0) ell_finish<W>(T, cur, bs, y);
        for (int k = r0 + t + LPB; k < r1; k += LPB) {
          EllRow<W> w;
          ell_issue<W>(T, srow, bs, k, w);
          ell_finish<W>(T, w, bs, y);
        }
        cur = n1;
        n1 = n2;
      }
      __syncwarp();
    }
    return;
  }
  EllRow<W> cur, nxt;
  if (G > 0 && t < sgrp[1] - sgrp[0]) ell_issue<W>(T, srow, bs, sgrp[0] + t, cur);
  for (int g = 0; g < Gmax; ++g) {
    if (g < G) {
      const int r0 = sgrp[g], r1 = sgrp[g + 1];
      const bool nx = g + 1 < G && t < sgrp[g + 2] - r1;
      if (nx) ell_issue<W>(T, srow, bs, r1 + t, nxt);
      if (t < r1 - r0) ell_finish<W>(T, cur, bs, y);
      for (int k = r0 + t + LPB; k < r1; k += LPB) {  // levels wider than LPB
        EllRow<W> w;
        ell_issue<W>(T, srow, bs, k, w);
        ell_finish<W>(T, w, bs, y);
      }
      if (nx) cur = nxt;
    }
    __syncwarp();
  }
}

template <int LPB, int W, int D = 1>
__global__ void __launch_bounds__(32) block_ilu_ell_kernel(const int* __restrict__ block_ptr,
                                                           int nblocks,
                                                           const int* __restrict__ new2old,
                                                           TriView A, TriView B,
                                                           const double* __restrict__ r,
                                                           double* __restrict__ out,
                                                           int max_block, int max_grp) {
  extern __shared__ double smem_d[];
  const int j = threadIdx.x / LPB, t = threadIdx.x % LPB;
  const size_t per = block_ilu_ell_smem(max_block, max_grp) / 8;  // doubles per block region
  double* y = smem_d + j * per;
  int* sgrp = reinterpret_cast<int*>(y + max_block);
  unsigned short* srow = reinterpret_cast<unsigned short*>(sgrp + max_grp + 1);
  const int b = blockIdx.x * (32 / LPB) + j;
  const bool live = b < nblocks;
  const int bs = live ? block_ptr[b] : 0, be = live ? block_ptr[b + 1] : 0;
  for (int i = t; i < be - bs; i += LPB) y[i] = r[new2old ? new2old[bs + i] : bs + i];
  __syncwarp();
  block_tri_ell<LPB, W, D>(A, live, b, bs, be - bs, y, sgrp, srow);
  block_tri_ell<LPB, W, D>(B, live, b, bs, be - bs, y, sgrp, srow);
  for (int i = t; i < be - bs; i += LPB) out[new2old ? new2old[bs + i] : bs + i] = y[i];
}


__global__ void ell_rowlen_kernel(int64_t n, const int64_t* __restrict__ ip, int* __restrict__ mx) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n) atomicMax(mx, int(ip[r + 1] - ip[r]));
}

__global__ void ell_fill_kernel(int64_t n, int nblocks, const int* __restrict__ bptr,
                                const int64_t* __restrict__ ip, const int* __restrict__ ix,
                                const double* __restrict__ v, int W, double* __restrict__ ev,
                                unsigned short* __restrict__ eo) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int lo = 0, hi = nblocks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bptr[mid] <= r) lo = mid; else hi = mid - 1;
  }
  const int bs = bptr[lo];
  const int64_t e0 = ip[r], len = ip[r + 1] - e0;
  for (int u = 0; u < W; ++u) {
    const bool ok = u < len;
    ev[r * W + u] = ok ? v[e0 + u] : 0.0;
    eo[r * W + u] = (unsigned short)(ok ? unsigned(ix[e0 + u] - bs) * 8u : 0u);
  }
}


// lanes per block: small blocks (p <= 2 levels, ~1.5 rows per dependency
// level) run the two-level-lookahead sweep with 4 lanes (8 blocks per warp),
// or on grids of a few waves (latency bound) the quad-row sweep with 16;
// larger blocks are smem-bound (18 B per row) and run one per warp.
// Measured with tools/vcycle_breakdown.py and tools/box_tgv.py against the
// round-1 choice (2 lanes, one level of lookahead): cfg3 p = 4 small-block
// sweeps 7.05 -> 4.87 ms per V-cycle, TGV 16^3 p = 5 227 -> 168-173 ms per step.
inline int small_block_lanes() {  // FB_BILU_SMALL_LANES=<2|4|8|16>: A/B runs (0: auto)
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("FB_BILU_SMALL_LANES");
    v = env ? atoi(env) : 0;
  }
  return v;
}
inline int block_ilu_lanes(const fb_blockilu* B) {
  if (B->max_block > 160) return 32;
  const int v = small_block_lanes();
  return v > 0 ? v : (small_grid(B) ? 16 : 4);
}
// shared memory of the widest launch (small blocks: up to 16 per warp)
inline size_t block_ilu_smem_max(int max_block) {
  return block_ilu_smem(max_block) * (max_block <= 160 ? 16 : 1);
}

template <int LPB, int PIPE>
int launch_block_ilu(const fb_blockilu* B, TriView a, TriView b, const double* r, double* out,
                     cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    FB_TRY_CUDA(cudaFuncSetAttribute(block_ilu_kernel<LPB, PIPE>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  constexpr int BPW = 32 / LPB;
  const size_t smem = block_ilu_smem(B->max_block, B->max_grp) * BPW;
  block_ilu_kernel<LPB, PIPE><<<(B->nblocks + BPW - 1) / BPW, 32, smem, st>>>(
      B->block_ptr.ptr, B->nblocks, B->new2old.ptr, a, b, r, out, B->max_block, B->max_grp);
  FB_CHECK_LAUNCH();
  return FB_OK;
}


// ---- device-side construction (structured "scale mode" levels) -----------
// The same factor and the same per-block level grouping as the host path
// (fb_blockilu_create), built from a device CSR without a host round trip:
// the finest LOR level of a 100M-DoF box has ~2.7G entries.

__global__ void bilu_row_block_kernel(int64_t n, int64_t nblocks, const int64_t* __restrict__ bptr,
                                      int* __restrict__ rb) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t lo = 0, hi = nblocks - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (bptr[mid] <= r) lo = mid; else hi = mid - 1;
  }
  rb[r] = int(lo);
}

__global__ void bilu_count_kernel(int64_t n, const int64_t* __restrict__ ip,
                                  const int* __restrict__ ix, const int64_t* __restrict__ bptr,
                                  const int* __restrict__ rb, int* __restrict__ cnt) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t bs = bptr[rb[r]], be = bptr[rb[r] + 1];
  int c = 0;
  for (int64_t k = ip[r]; k < ip[r + 1]; ++k) c += (ix[k] >= bs && ix[k] < be);
  cnt[r] = c;
}

__global__ void bilu_fill_kernel(int64_t n, const int64_t* __restrict__ ip,
                                 const int* __restrict__ ix, const double* __restrict__ v,
                                 const int64_t* __restrict__ bptr, const int* __restrict__ rb,
                                 const int64_t* __restrict__ fip, int* __restrict__ fix,
                                 double* __restrict__ fv, int64_t* __restrict__ dpos,
                                 unsigned long long* __restrict__ missing) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t bs = bptr[rb[r]], be = bptr[rb[r] + 1];
  int64_t o = fip[r], d = -1;
  for (int64_t k = ip[r]; k < ip[r + 1]; ++k) {
    const int c = ix[k];
    if (c < bs || c >= be) continue;
    if (c == r) d = o;
    fix[o] = c;
    fv[o] = v[k];
    ++o;
  }
  dpos[r] = d;
  if (d < 0) atomicMin(missing, (unsigned long long)r);
}

// ILU(0), IKJ order of numba_backend.py:64-103, one thread per block; every
// update is a separately rounded multiply and subtract, so the factor is
// bitwise the host/numba factor of the same matrix.
__global__ void bilu_factor_kernel(int64_t nblocks, const int64_t* __restrict__ bptr,
                                   const int64_t* __restrict__ fip, const int* __restrict__ fix,
                                   double* __restrict__ fv, const int64_t* __restrict__ dpos,
                                   unsigned long long* __restrict__ fail) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  for (int64_t i = bptr[b]; i < bptr[b + 1]; ++i) {
    const int64_t re = fip[i + 1];
    for (int64_t kk = fip[i]; kk < dpos[i]; ++kk) {
      const int k = fix[kk];
      const double piv = fv[dpos[k]];
      if (fabs(piv) < 1e-300) {
        atomicMin(fail, (unsigned long long)k);
        return;
      }
      const double l = __ddiv_rn(fv[kk], piv);
      fv[kk] = l;
      int64_t p1 = kk + 1, p2 = dpos[k] + 1;
      const int64_t e2 = fip[k + 1];
      while (p1 < re && p2 < e2) {
        const int c1 = fix[p1], c2 = fix[p2];
        if (c1 == c2) {
          fv[p1] = __dsub_rn(fv[p1], __dmul_rn(l, fv[p2]));
          ++p1;
          ++p2;
        } else if (c1 < c2) {
          ++p1;
        } else {
          ++p2;
        }
      }
    }
    if (fabs(fv[dpos[i]]) < 1e-300) {
      atomicMin(fail, (unsigned long long)i);
      return;
    }
  }
}

__global__ void bilu_split_count_kernel(int64_t n, const int64_t* __restrict__ fip,
                                        const int64_t* __restrict__ dpos, int* __restrict__ lc,
                                        int* __restrict__ uc) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  lc[r] = int(dpos[r] - fip[r]);
  uc[r] = int(fip[r + 1] - dpos[r] - 1);
}

__global__ void bilu_split_fill_kernel(int64_t n, const int64_t* __restrict__ fip,
                                       const int* __restrict__ fix, const double* __restrict__ fv,
                                       const int64_t* __restrict__ dpos,
                                       const int64_t* __restrict__ lip, int* __restrict__ lix,
                                       double* __restrict__ lv, const int64_t* __restrict__ uip,
                                       int* __restrict__ uix, double* __restrict__ uv,
                                       double* __restrict__ uinv) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t o = lip[r];
  for (int64_t k = fip[r]; k < dpos[r]; ++k, ++o) {
    lix[o] = fix[k];
    lv[o] = fv[k];
  }
  o = uip[r];
  for (int64_t k = dpos[r] + 1; k < fip[r + 1]; ++k, ++o) {
    uix[o] = fix[k];
    uv[o] = fv[k];
  }
  uinv[r] = 1.0 / fv[dpos[r]];
}

__global__ void csr_col_count_kernel(int64_t n, const int64_t* __restrict__ ip,
                                     const int* __restrict__ ix, int* __restrict__ cnt) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t k = ip[r]; k < ip[r + 1]; ++k) atomicAdd(cnt + ix[k], 1);
}

__global__ void csr_transpose_fill_kernel(int64_t n, const int64_t* __restrict__ ip,
                                          const int* __restrict__ ix, const double* __restrict__ v,
                                          const int64_t* __restrict__ tip, int* __restrict__ cur,
                                          int* __restrict__ tix, double* __restrict__ tv) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t k = ip[r]; k < ip[r + 1]; ++k) {
    const int c = ix[k];
    const int64_t pos = tip[c] + atomicAdd(cur + c, 1);
    tix[pos] = int(r);
    tv[pos] = v[k];
  }
}

// rows of the transpose were filled in arbitrary order: sort each by column
__global__ void csr_sort_rows_kernel(int64_t n, const int64_t* __restrict__ ip,
                                     int* __restrict__ ix, double* __restrict__ v) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t b = ip[r], e = ip[r + 1];
  for (int64_t i = b + 1; i < e; ++i) {
    const int c = ix[i];
    const double x = v[i];
    int64_t j = i - 1;
    while (j >= b && ix[j] > c) {
      ix[j + 1] = ix[j];
      v[j + 1] = v[j];
      --j;
    }
    ix[j + 1] = c;
    v[j + 1] = x;
  }
}

__global__ void bilu_levels_kernel(int64_t nblocks, const int64_t* __restrict__ bptr,
                                   const int64_t* __restrict__ ip, const int* __restrict__ ix,
                                   int lower, int* __restrict__ level, int* __restrict__ nlev) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  const int64_t bs = bptr[b], be = bptr[b + 1];
  int maxl = 0;
  for (int64_t k = 0; k < be - bs; ++k) {
    const int64_t r = lower ? bs + k : be - 1 - k;
    int lv = 0;
    for (int64_t e = ip[r]; e < ip[r + 1]; ++e) lv = max(lv, level[ix[e]] + 1);
    level[r] = lv;
    maxl = max(maxl, lv);
  }
  nlev[b] = maxl + 1;
}

__global__ void bilu_group_kernel(int64_t nblocks, int64_t n, const int64_t* __restrict__ bptr,
                                  const int* __restrict__ level, const int64_t* __restrict__ bg,
                                  int* __restrict__ grp, int* __restrict__ blk_grp,
                                  int* __restrict__ cur, int* __restrict__ rows) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b > nblocks) return;
  blk_grp[b] = int(bg[b]);
  if (b == nblocks) {
    grp[bg[b]] = int(n);
    return;
  }
  const int64_t bs = bptr[b], be = bptr[b + 1];
  const int64_t g0 = bg[b], L = bg[b + 1] - g0;
  for (int64_t l = 0; l < L; ++l) grp[g0 + l] = 0;
  for (int64_t r = bs; r < be; ++r) grp[g0 + level[r]]++;
  int off = int(bs);
  for (int64_t l = 0; l < L; ++l) {
    const int t = grp[g0 + l];
    grp[g0 + l] = off;
    cur[g0 + l] = off;
    off += t;
  }
  for (int64_t r = bs; r < be; ++r) rows[cur[g0 + level[r]]++] = int(r);
}
}  // namespace fb

using namespace fb;

namespace {

// Build one triangular part: strict off-diagonal CSR + inverse diagonal + the
// per-block level grouping of its rows.
int build_part(int64_t n, const std::vector<int>& bptr, const std::vector<int64_t>& ip,
               const std::vector<int64_t>& ix, const std::vector<double>& v, bool lower,
               bool unit, TriPart& P) {
  std::vector<int64_t> oip(n + 1, 0);
  std::vector<int> oix;
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
    oip[r + 1] = int64_t(oix.size());
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
      for (int64_t e = oip[r]; e < oip[r + 1]; ++e) {
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
  return TriView{P.ev.ptr, P.eo.ptr, P.ip.ptr, P.ix.ptr, P.v.ptr,
                 unit ? nullptr : P.invdiag.ptr, P.rows.ptr, P.grp.ptr, P.blk_grp.ptr};
}

}  // namespace

namespace {

template <int LPB, int W, int D = 1>
int launch_ell(const fb_blockilu* B, TriView a, TriView b, const double* r, double* out,
               cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    FB_TRY_CUDA(cudaFuncSetAttribute(block_ilu_ell_kernel<LPB, W, D>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  constexpr int BPW = 32 / LPB;
  const size_t smem = block_ilu_ell_smem(B->max_block, B->max_grp) * BPW;
  block_ilu_ell_kernel<LPB, W, D><<<(B->nblocks + BPW - 1) / BPW, 32, smem, st>>>(
      B->block_ptr.ptr, B->nblocks, B->new2old.ptr, a, b, r, out, B->max_block, B->max_grp);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

// one-warp sweeps of a grid that fits one wave (<= 8 blocks per SM): the
// level latency, not occupancy, bounds them, so load two levels ahead
inline bool small_grid(const fb_blockilu* B) {
  static int sms = 0;
  if (sms == 0) {
    const char* env = getenv("FB_BILU_DEEP");  // A/B switch for tools/box_profile.py
    if (env && env[0] == '0') g_bilu_deep = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  return g_bilu_deep != 0 && B->nblocks <= 8 * sms;
}

template <int W>
int launch_ell_w(const fb_blockilu* B, int lanes, TriView a, TriView b, const double* r,
                 double* out, cudaStream_t st) {
  if (lanes == 2) return launch_ell<2, W>(B, a, b, r, out, st);
  return small_grid(B) ? launch_ell<32, W, 2>(B, a, b, r, out, st)
                       : launch_ell<32, W>(B, a, b, r, out, st);
}

}  // namespace

// Convert the four triangular parts to the padded-row layout (all parts
// padded to one width, a multiple of 8) and drop their CSR arrays.
static int build_ell(fb_blockilu* B) {
  // measured (tools/box_profile.py): padded rows pay off for the large p = 7
  // blocks (~3000 rows, 24 rows per level); CSR rows are faster below
  if (B->max_block <= 1000) return FB_OK;
  if (B->max_block > 8191) return FB_OK;  // byte offsets must fit 16 bits
  TriPart* parts[4] = {&B->L, &B->U, &B->Ut, &B->Lt};
  DevBuf<int> mx;
  FB_TRY_CUDA(mx.alloc(1));
  FB_TRY_CUDA(cudaMemset(mx.ptr, 0, sizeof(int)));
  const int64_t n = B->n;
  for (TriPart* P : parts) {
    ell_rowlen_kernel<<<ceil_div(n, 256), 256>>>(n, P->ip.ptr, mx.ptr);
    FB_CHECK_LAUNCH();
  }
  int maxlen = 0;
  FB_TRY_CUDA(cudaMemcpy(&maxlen, mx.ptr, sizeof(int), cudaMemcpyDeviceToHost));
  const int W = maxlen <= 8 ? 8 : (maxlen <= 16 ? 16 : (maxlen <= 24 ? 24 : (maxlen <= 32 ? 32 : 0)));
  if (W == 0) return FB_OK;
  for (TriPart* P : parts) {
    FB_TRY_CUDA(P->ev.alloc(n * W));
    FB_TRY_CUDA(P->eo.alloc(n * W));
    ell_fill_kernel<<<ceil_div(n, 256), 256>>>(n, B->nblocks, B->block_ptr.ptr, P->ip.ptr,
                                               P->ix.ptr, P->v.ptr, W, P->ev.ptr, P->eo.ptr);
    FB_CHECK_LAUNCH();
    FB_TRY_CUDA(cudaDeviceSynchronize());
    P->width = W;
    P->nnz = P->ix.n;
    P->ix.reset();
    P->v.reset();
    P->ip.reset();
  }
  B->ell_w = W;
  return FB_OK;
}

// ---- level-packed sweep: a TMA ring of dependency levels ------------------
// The CSR / ELL sweeps load each level's rows with per-lane global loads one
// (or two) levels ahead, so every level waits out most of a memory latency:
// at cfg3 the fine-level sweep ran at ~25-35 % of HBM bandwidth with
// 89-131 levels per block.  Here each level of each block is ONE contiguous
// chunk (TriPart::pk), and one lane streams chunks NSLOT levels ahead into a
// shared-memory ring with cp.async.bulk (TMA) + an mbarrier per slot, so the
// lanes computing level g read everything from shared memory.  Each row is
// split over 1-4 lanes (packed_rows): deterministic, equal to the CSR sweep
// to rounding (not bitwise its sequential chain).
namespace {

struct PackView {
  const unsigned char* pk;
  const int64_t* loff;
  const int* lne;
  const int* grp;
  const int* blk_grp;
  int has_inv;
  int s4, s2;  // rows per level up to which 4 / 2 lanes share a row
};

__device__ __forceinline__ uint32_t psmem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void pk_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "PKW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra PKW_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void pk_copy(uint32_t dst, const void* src, uint32_t bytes,
                                        uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__host__ __device__ inline size_t packed_smem(int nslot, int max_chunk, int max_block,
                                              int max_grp) {
  return 128 + size_t(nslot) * size_t(max_chunk) + size_t(max_block) * 8 +
         size_t(max_grp + 1) * 12;
}

// One dependency level of a packed chunk: rows t < R, S lanes per row.
// Lane `sub` of a row accumulates entries sub, sub + S, ... with fma; the S
// partial sums are combined by xor shuffles in a fixed order, so the result
// is deterministic (not bitwise the sequential CSR chain).
template <int S, int NW>
__device__ __forceinline__ void packed_rows(const double* vals, const double* inv,
                                            const unsigned short* cols,
                                            const unsigned short* rows,
                                            const unsigned short* rst,
                                            const unsigned short* cnt, int R, int has_inv,
                                            double* y) {
  constexpr int LG = (S == 4) ? 2 : (S == 2) ? 1 : 0;
  constexpr int U = (kRowBuf + S - 1) / S;  // unrolled entries per lane
  const int lane = threadIdx.x;
  const int sub = lane & (S - 1);
  for (int t0 = 0; t0 < R; t0 += ((32 * NW) >> LG)) {
    const int t = t0 + (lane >> LG);
    const bool live = t < R;
    const int start = live ? rst[t] : 0, n = live ? cnt[t] : 0;
    // S <= 2 (wide levels): the row's own value and scale do not depend on
    // this level's sums -- load them up front, off the critical path (p = 7
    // sweep -5 %); with 4 lanes per row the redundant loads cost more (p = 4 +3 %)
    int row = 0;
    double yr = 0.0, iv = 1.0;
    constexpr bool HOIST = S <= 2 && NW == 2;  // large blocks only (p = 4 measured neutral-to-worse)
    if constexpr (HOIST) {
      row = live ? rows[t] : 0;
      yr = live ? y[row] : 0.0;
      iv = (live && has_inv) ? inv[t] : 1.0;
    }
    double av[U], yv[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int u = sub + k * S;
      const bool ok = u < n;
      av[k] = ok ? vals[start + u] : 0.0;
      yv[k] = ok ? y[cols[start + u]] : 0.0;
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < U; ++k) acc = fma(av[k], yv[k], acc);
    for (int u = sub + U * S; u < n; u += S)  // first-touch order: up to 26 lower neighbours
      acc = fma(vals[start + u], y[cols[start + u]], acc);
    if constexpr (S >= 2) acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if constexpr (S >= 4) acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (live && sub == 0) {
      if constexpr (!HOIST) {
        row = rows[t];
        yr = y[row];
        iv = has_inv ? inv[t] : 1.0;
      }
      const double res = yr - acc;
      y[row] = has_inv ? res * iv : res;
    }
  }
}

// Levels are staged K at a time (one bulk copy spans K consecutive chunks of
// the block; NSLOT spans in flight), so the mbarrier wait and the copy issue
// are paid once per K levels.
// one warp (NW = 1) or NW warps per block (wide levels of large blocks)
template <int NW>
__device__ __forceinline__ void pk_sync() {
  if constexpr (NW == 1) __syncwarp();
  else __syncthreads();
}

template <int NSLOT, int NW>
__device__ __forceinline__ void packed_tri(const PackView& T, int b, double* y, uint64_t* bars,
                                           unsigned char* ring, int slot_bytes, int K,
                                           int* soff, int* sR, int* sE, uint32_t& used) {
  const int lane = threadIdx.x;
  const int g0 = T.blk_grp[b], G = T.blk_grp[b + 1] - g0;
  const int NG = (G + K - 1) / K;
  pk_sync<NW>();
  // level chunk offsets relative to the block's first chunk (32-bit), base kept 64-bit
  const int64_t lbase = T.loff[g0];
  for (int i = lane; i <= G; i += 32 * NW) soff[i] = int(T.loff[g0 + i] - lbase);
  for (int i = lane; i < G; i += 32 * NW) {
    sR[i] = T.grp[g0 + i + 1] - T.grp[g0 + i];
    sE[i] = T.lne[g0 + i];
  }
  pk_sync<NW>();
  auto issue = [&](int j) {
    const uint32_t slot = (used + uint32_t(j)) % NSLOT;
    const int a = j * K, z = min(a + K, G);
    pk_copy(psmem_u32(ring + size_t(slot) * slot_bytes), T.pk + lbase + soff[a],
            uint32_t(soff[z] - soff[a]), psmem_u32(&bars[slot]));
  };
  if (lane == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int j = 0; j < NG && j < NSLOT; ++j) issue(j);
  }
  for (int j = 0; j < NG; ++j) {
    const uint32_t c = used + uint32_t(j), slot = c % NSLOT;
    pk_wait(psmem_u32(&bars[slot]), (c / NSLOT) & 1u);
    const unsigned char* sb = ring + size_t(slot) * slot_bytes;
    const int a = j * K, z = min(a + K, G);
    for (int g = a; g < z; ++g) {
      const unsigned char* ch = sb + (soff[g] - soff[a]);
      const int R = sR[g], E = sE[g];
      const double* vals = reinterpret_cast<const double*>(ch);
      const double* inv = vals + E;
      const unsigned short* cols =
          reinterpret_cast<const unsigned short*>(inv + (T.has_inv ? R : 0));
      const unsigned short* rows = cols + E;
      const unsigned short* rst = rows + R;  // per row: first entry, entry count
      const unsigned short* cnt = rst + R;
      // S lanes per row (levels are narrow: ~6 rows at p = 4), each summing
      // a strided share of the row's entries, combined by a fixed xor tree
      if (R <= T.s4 * NW) packed_rows<4, NW>(vals, inv, cols, rows, rst, cnt, R, T.has_inv, y);
      else if (R <= T.s2 * NW) packed_rows<2, NW>(vals, inv, cols, rows, rst, cnt, R, T.has_inv, y);
      else packed_rows<1, NW>(vals, inv, cols, rows, rst, cnt, R, T.has_inv, y);
      pk_sync<NW>();
    }
    if (lane == 0 && j + NSLOT < NG) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(j + NSLOT);
    }
  }
  used += uint32_t(NG);
}

template <int NSLOT, int NW>
__global__ void __launch_bounds__(32 * NW) block_ilu_packed_kernel(
    const int* __restrict__ block_ptr, const int* __restrict__ new2old, PackView A, PackView Bv,
    const double* __restrict__ r, double* __restrict__ out, int slot_bytes, int KA, int KB,
    int max_block, int max_grp, int add) {
  extern __shared__ __align__(16) unsigned char psm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(psm);
  unsigned char* ring = psm + 128;
  double* y = reinterpret_cast<double*>(ring + size_t(NSLOT) * slot_bytes);
  int* soff = reinterpret_cast<int*>(y + max_block);
  int* sR = reinterpret_cast<int*>(soff + max_grp + 1);
  int* sE = sR + max_grp + 1;
  const int lane = threadIdx.x;
  const int b = blockIdx.x;
  const int bs = block_ptr[b], nb = block_ptr[b + 1] - bs;
  if (lane == 0) {
    for (int i = 0; i < NSLOT; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(&bars[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = lane; i < nb; i += 32 * NW) y[i] = r[new2old ? new2old[bs + i] : bs + i];
  uint32_t used = 0;
  packed_tri<NSLOT, NW>(A, b, y, bars, ring, slot_bytes, KA, soff, sR, sE, used);
  packed_tri<NSLOT, NW>(Bv, b, y, bars, ring, slot_bytes, KB, soff, sR, sE, used);
  pk_sync<NW>();
  for (int i = lane; i < nb; i += 32 * NW) {
    const int o = new2old ? new2old[bs + i] : bs + i;
    out[o] = add ? __dadd_rn(y[i], out[o]) : y[i];  // add: out += M^-1 r (axpby rounding)
  }
}

__global__ void pack_count_kernel(int64_t nlev, const int* __restrict__ grp,
                                  const int* __restrict__ rows, const int64_t* __restrict__ ip,
                                  int has_inv, int64_t* __restrict__ size, int* __restrict__ lne,
                                  int* __restrict__ max_chunk) {
  const int64_t L = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (L > nlev) return;
  if (L == nlev) {
    size[L] = 0;
    return;
  }
  int64_t E = 0;
  for (int k = grp[L]; k < grp[L + 1]; ++k) E += ip[rows[k] + 1] - ip[rows[k]];
  const int64_t R = grp[L + 1] - grp[L];
  const int64_t bytes = (8 * E + (has_inv ? 8 * R : 0) + 2 * E + 6 * R + 15) / 16 * 16;
  lne[L] = int(E);
  size[L] = bytes;
  atomicMax(max_chunk, int(bytes));
}

__global__ void pack_fill_kernel(int64_t nlev, int nblocks, const int* __restrict__ bptr,
                                 const int* __restrict__ blk_grp, const int* __restrict__ grp,
                                 const int* __restrict__ rows, const int64_t* __restrict__ ip,
                                 const int* __restrict__ ix, const double* __restrict__ v,
                                 const double* __restrict__ invdiag,
                                 const int64_t* __restrict__ loff, const int* __restrict__ lne,
                                 unsigned char* __restrict__ pk) {
  const int64_t L = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (L >= nlev) return;
  int lo = 0, hi = nblocks - 1;  // block of level L
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (blk_grp[mid] <= L) lo = mid; else hi = mid - 1;
  }
  const int bs = bptr[lo];
  const int E = lne[L], R = grp[L + 1] - grp[L];
  unsigned char* ch = pk + loff[L];
  double* vals = reinterpret_cast<double*>(ch);
  double* inv = vals + E;
  unsigned short* cols = reinterpret_cast<unsigned short*>(inv + (invdiag ? R : 0));
  unsigned short* lrows = cols + E;
  unsigned short* rst = lrows + R;
  unsigned short* cnt = rst + R;
  int e = 0;
  for (int t = 0; t < R; ++t) {
    const int row = rows[grp[L] + t];
    const int64_t a = ip[row], z = ip[row + 1];
    rst[t] = (unsigned short)e;
    for (int64_t k = a; k < z; ++k, ++e) {
      vals[e] = v[k];
      cols[e] = (unsigned short)(ix[k] - bs);
    }
    if (invdiag) inv[t] = invdiag[row];
    lrows[t] = (unsigned short)(row - bs);
    cnt[t] = (unsigned short)(z - a);
  }
}

// largest span of K consecutive level chunks of one block
__global__ void pack_group_kernel(int64_t nlev, int nblocks, const int* __restrict__ blk_grp,
                                  const int64_t* __restrict__ loff, int K,
                                  int* __restrict__ max_span) {
  const int64_t L = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (L >= nlev) return;
  int lo = 0, hi = nblocks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (blk_grp[mid] <= L) lo = mid; else hi = mid - 1;
  }
  const int64_t g0 = blk_grp[lo], g1 = blk_grp[lo + 1];
  if ((L - g0) % K) return;
  const int64_t z = (L + K < g1) ? L + K : g1;
  atomicMax(max_span, int(loff[z] - loff[L]));
}

}  // namespace

constexpr int kPackSpanBudget = 4 * 1024;  // bytes per staged span (two in flight; measured 2-16 KB)

static int pack_span_budget() {  // FB_BILU_SPAN=<bytes>: A/B runs (tools/bilu_ab.py)
  const char* env = getenv("FB_BILU_SPAN");
  const int v = env ? atoi(env) : 0;
  return v > 0 ? v : kPackSpanBudget;
}

static int pack_slots() {  // FB_BILU_NSLOT=<2..4>: spans in flight per block (A/B runs)
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("FB_BILU_NSLOT");
    v = env ? atoi(env) : 2;
  }
  return v;
}

static int build_packed_part(fb_blockilu* B, TriPart& P, bool has_inv) {
  const int64_t nlev = P.grp.n - 1;
  if (nlev <= 0) return FB_OK;
  DevBuf<int64_t> size;
  DevBuf<int> mx;
  FB_TRY_CUDA(size.alloc(nlev + 1));
  FB_TRY_CUDA(P.lne.alloc(nlev));
  FB_TRY_CUDA(mx.alloc(1));
  FB_TRY_CUDA(cudaMemset(mx.ptr, 0, sizeof(int)));
  pack_count_kernel<<<ceil_div(nlev + 1, 256), 256>>>(nlev, P.grp.ptr, P.rows.ptr, P.ip.ptr,
                                                      has_inv ? 1 : 0, size.ptr, P.lne.ptr,
                                                      mx.ptr);
  FB_CHECK_LAUNCH();
  size_t tb = 0;
  FB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, size.ptr, size.ptr, nlev + 1));
  DevBuf<unsigned char> tmp;
  FB_TRY_CUDA(tmp.alloc(int64_t(tb)));
  FB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, size.ptr, size.ptr, nlev + 1));
  int64_t total = 0;
  FB_TRY_CUDA(cudaMemcpy(&total, size.ptr + nlev, sizeof(int64_t), cudaMemcpyDeviceToHost));
  FB_TRY_CUDA(cudaMemcpy(&P.max_chunk, mx.ptr, sizeof(int), cudaMemcpyDeviceToHost));
  FB_TRY_CUDA(P.pk.alloc(total));
  pack_fill_kernel<<<ceil_div(nlev, 128), 128>>>(nlev, B->nblocks, B->block_ptr.ptr,
                                                 P.blk_grp.ptr, P.grp.ptr, P.rows.ptr, P.ip.ptr,
                                                 P.ix.ptr, P.v.ptr,
                                                 has_inv ? P.invdiag.ptr : nullptr, size.ptr,
                                                 P.lne.ptr, P.pk.ptr);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(cudaDeviceSynchronize());
  P.loff.ptr = size.ptr;  // keep the offsets
  P.loff.n = size.n;
  size.ptr = nullptr;
  size.n = 0;
  // stage as many levels per copy as keep two spans within the budget
  for (int K : {8, 4, 2, 1}) {
    FB_TRY_CUDA(cudaMemset(mx.ptr, 0, sizeof(int)));
    pack_group_kernel<<<ceil_div(nlev, 256), 256>>>(nlev, B->nblocks, P.blk_grp.ptr, P.loff.ptr,
                                                    K, mx.ptr);
    FB_CHECK_LAUNCH();
    int span = 0;
    FB_TRY_CUDA(cudaMemcpy(&span, mx.ptr, sizeof(int), cudaMemcpyDeviceToHost));
    P.lev_group = K;
    P.max_group = span;
    if (span <= pack_span_budget()) break;
  }
  return FB_OK;
}

// Pack all four parts and drop their CSR arrays (the packed chunks replace
// them); blocks must be large (one block per warp) and fit 16-bit indices.
static int build_packed(fb_blockilu* B) {
  if (!g_bilu_packed || B->max_block <= 160 || B->max_block > 65535) return FB_OK;
  // grids of a few waves (one warp per block) stay on the CSR sweeps, whose
  // two-level lookahead suits them better (TGV-size levels)
  if (small_grid(B) || B->nblocks < 16 * 148) return FB_OK;
  TriPart* parts[4] = {&B->L, &B->U, &B->Ut, &B->Lt};
  const bool inv[4] = {false, true, true, false};
  for (int i = 0; i < 4; ++i) {
    parts[i]->nnz = parts[i]->ix.n;
    const int rc = build_packed_part(B, *parts[i], inv[i]);
    if (rc != FB_OK) return rc;
  }
  for (TriPart* P : parts) {
    P->ix.reset();
    P->v.reset();
  }
  return FB_OK;
}

template <int NSLOT, int NW>
static int launch_packed_w(const fb_blockilu* B, const TriPart& a, bool ua, const TriPart& b,
                           bool ub, const double* r, double* out, cudaStream_t st, int add) {
  const int sb = (std::max(a.max_group, b.max_group) + 15) / 16 * 16;
  const size_t smem = packed_smem(NSLOT, sb, B->max_block, B->max_grp);
  static size_t configured = 0;
  if (smem > configured) {
    FB_TRY_CUDA(cudaFuncSetAttribute(block_ilu_packed_kernel<NSLOT, NW>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    configured = smem;
  }
  // FB_BILU_S4 / FB_BILU_S2: level widths up to which rows are split over 4 / 2
  // lanes (A/B runs; defaults measured with tools/vcycle_breakdown.py)
  static const int s4 = getenv("FB_BILU_S4") ? atoi(getenv("FB_BILU_S4")) : 8;
  static const int s2 = getenv("FB_BILU_S2") ? atoi(getenv("FB_BILU_S2")) : 16;
  const PackView pa{a.pk.ptr, a.loff.ptr, a.lne.ptr, a.grp.ptr, a.blk_grp.ptr, ua ? 0 : 1, s4, s2};
  const PackView pb{b.pk.ptr, b.loff.ptr, b.lne.ptr, b.grp.ptr, b.blk_grp.ptr, ub ? 0 : 1, s4, s2};
  block_ilu_packed_kernel<NSLOT, NW><<<B->nblocks, 32 * NW, smem, st>>>(
      B->block_ptr.ptr, B->new2old.ptr, pa, pb, r, out, sb, a.lev_group, b.lev_group,
      B->max_block, B->max_grp, add);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

// warps per block: FB_BILU_NW=<1|2> (A/B runs), else by block size
template <int NSLOT>
static int launch_packed(const fb_blockilu* B, const TriPart& a, bool ua, const TriPart& b,
                         bool ub, const double* r, double* out, cudaStream_t st, int add = 0) {
  static const int nw_env = getenv("FB_BILU_NW") ? atoi(getenv("FB_BILU_NW")) : 0;
  // by the typical block (first-touch boundary blocks are larger than interior ones)
  const int nw = nw_env > 0 ? nw_env : (B->n / std::max(B->nblocks, 1) > 1024 ? 2 : 1);
  if (nw == 2) return launch_packed_w<NSLOT, 2>(B, a, ua, b, ub, r, out, st, add);
  return launch_packed_w<NSLOT, 1>(B, a, ua, b, ub, r, out, st, add);
}

extern "C" {

// F: the block-diagonal ILU(0) factor in the new (block-major) numbering, as
// CSR with sorted columns (strict lower part = L, unit diagonal implied;
// upper part incl. diagonal = U).  block_ptr: (nblocks+1) row offsets.
// deepest level schedule of one block over the four triangular parts
static int compute_max_grp(fb_blockilu* B) {
  int mg = 0;
  std::vector<int> h(size_t(B->nblocks) + 1);
  for (const TriPart* P : {&B->L, &B->U, &B->Ut, &B->Lt}) {
    if (P->blk_grp.n < B->nblocks + 1) continue;
    FB_TRY_CUDA(cudaMemcpy(h.data(), P->blk_grp.ptr, h.size() * sizeof(int),
                           cudaMemcpyDeviceToHost));
    for (int b = 0; b < B->nblocks; ++b) mg = std::max(mg, h[b + 1] - h[b]);
  }
  B->max_grp = mg;
  return FB_OK;
}

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
  FB_REQUIRE(block_ilu_smem_max(B->max_block) <= 200 * 1024 &&
                 B->max_block <= 65535,
             "block too large for shared memory");
  {
    const int rc_p = build_packed(B.get());
    if (rc_p != FB_OK) return rc_p;
  }
  if (g_bilu_pipe == 2 && !B->L.pk.ptr) {
    const int rc_ell = build_ell(B.get());
    if (rc_ell != FB_OK) return rc_ell;
  }
  {
    const int rc_g = compute_max_grp(B.get());
    if (rc_g != FB_OK) return rc_g;
  }
  *out = B.release();
  return FB_OK;
}

int fb_blockilu_info(const fb_blockilu* B, int64_t* n, int64_t* nnz_lower, int64_t* nnz_upper,
                     int* ell_width) {
  FB_REQUIRE(B != nullptr, "block ILU is NULL");
  if (n) *n = B->n;
  if (nnz_lower) *nnz_lower = B->L.nnz ? B->L.nnz : B->L.ix.n;  // strict lower (unit diagonal)
  if (nnz_upper) *nnz_upper = B->U.nnz ? B->U.nnz : B->U.ix.n;  // strict upper (+ inverse diagonal)
  if (ell_width) *ell_width = B->ell_w;
  return FB_OK;
}

int fb_blockilu_sweep_kind(const fb_blockilu* B) {
  FB_REQUIRE(B != nullptr, "block ILU is NULL");
  return B->L.pk.ptr ? 2 : (B->ell_w ? 1 : 0);
}

void fb_blockilu_destroy(fb_blockilu* B) {
  if (B) debug_canary_unregister(B->block_ptr.ptr);
  delete B;
}

// out = (LU)^-1 r (transpose=0) or (LU)^-T r (transpose=1), both in the
// original numbering.
int fb_blockilu_apply(const fb_blockilu* B, int transpose, const double* r, double* out,
                      void* stream) {
  FB_REQUIRE(B != nullptr, "smoother is NULL");
  FB_REQUIRE(r != out, "in-place smoother application is not supported");
  if (B->nblocks == 0) return FB_OK;
  const TriView a = transpose ? view(B->Ut, false) : view(B->L, true);
  const TriView b = transpose ? view(B->Lt, true) : view(B->U, false);
  cudaStream_t st = as_stream(stream);
  if (B->L.pk.ptr) {  // level-packed TMA-ring sweep
    const TriPart& pa = transpose ? B->Ut : B->L;
    const TriPart& pb = transpose ? B->Lt : B->U;
    const bool ua = !transpose, ub = transpose;  // unit diagonal: L and L^T
    switch (pack_slots()) {
      case 3: return launch_packed<3>(B, pa, ua, pb, ub, r, out, st);
      case 4: return launch_packed<4>(B, pa, ua, pb, ub, r, out, st);
      default: return launch_packed<2>(B, pa, ua, pb, ub, r, out, st);
    }
  }
  const int lanes = g_bilu_lanes ? g_bilu_lanes : block_ilu_lanes(B);
  if (B->ell_w) {
    const int l2 = lanes == 2 ? 2 : 32;
    switch (B->ell_w) {
      case 8: return launch_ell_w<8>(B, l2, a, b, r, out, st);
      case 16: return launch_ell_w<16>(B, l2, a, b, r, out, st);
      case 24: return launch_ell_w<24>(B, l2, a, b, r, out, st);
      default: return launch_ell_w<32>(B, l2, a, b, r, out, st);
    }
  }
  // small blocks: quad-row sweep (FB_BILU_SMALL_QUAD=0: the sequential-chain sweep, A/B runs)
  static const bool small_quad = !(getenv("FB_BILU_SMALL_QUAD") && getenv("FB_BILU_SMALL_QUAD")[0] == '0');
  const bool pipe = g_bilu_pipe >= 1 && !(small_quad && B->max_block <= 160 && lanes >= 4);
  // small blocks on grids of many waves: the sequential-chain sweep with two
  // levels of lookahead, 4 lanes per block (cfg3 p = 4: 5.45 -> 4.87 ms of
  // small-block sweeps per V-cycle against the quad-row sweep);
  // FB_BILU_SMALL_PIPE2=0 turns it off (A/B runs)
  static const bool pipe2 = !(getenv("FB_BILU_SMALL_PIPE2") && getenv("FB_BILU_SMALL_PIPE2")[0] == '0');
  if (pipe2 && B->max_block <= 160 && g_bilu_pipe >= 1 && !small_grid(B)) {
    if (lanes == 4) return launch_block_ilu<4, 2>(B, a, b, r, out, st);
    if (lanes == 8) return launch_block_ilu<8, 2>(B, a, b, r, out, st);
    if (lanes == 2) return launch_block_ilu<2, 2>(B, a, b, r, out, st);
  }
  switch (lanes) {
    case 2: return pipe ? launch_block_ilu<2, true>(B, a, b, r, out, st) : launch_block_ilu<2, false>(B, a, b, r, out, st);
    case 4: return pipe ? launch_block_ilu<4, true>(B, a, b, r, out, st) : launch_block_ilu<4, false>(B, a, b, r, out, st);
    case 8: return pipe ? launch_block_ilu<8, true>(B, a, b, r, out, st) : launch_block_ilu<8, false>(B, a, b, r, out, st);
    case 16: return pipe ? launch_block_ilu<16, true>(B, a, b, r, out, st) : launch_block_ilu<16, false>(B, a, b, r, out, st);
    default:
      if (pipe && small_grid(B)) return launch_block_ilu<32, 2>(B, a, b, r, out, st);
      return pipe ? launch_block_ilu<32, true>(B, a, b, r, out, st) : launch_block_ilu<32, false>(B, a, b, r, out, st);
  }
}

// out += (LU)^-1 r / (LU)^-T r, level-packed sweeps only (fb_blockilu_sweep_kind
// == 2): the smoother's correction added in the sweep's final store, with the
// rounding of a separate out = 1 * (M^-1 r) + 1 * out
int fb_blockilu_apply_add(const fb_blockilu* B, int transpose, const double* r, double* out,
                          void* stream) {
  FB_REQUIRE(B != nullptr, "smoother is NULL");
  FB_REQUIRE(r != out, "in-place smoother application is not supported");
  FB_REQUIRE(B->nblocks == 0 || B->L.pk.ptr, "add mode needs the level-packed sweep");
  if (B->nblocks == 0) return FB_OK;
  const TriPart& pa = transpose ? B->Ut : B->L;
  const TriPart& pb = transpose ? B->Lt : B->U;
  const bool ua = !transpose, ub = transpose;
  cudaStream_t st = as_stream(stream);
  switch (pack_slots()) {
    case 3: return launch_packed<3>(B, pa, ua, pb, ub, r, out, st, 1);
    case 4: return launch_packed<4>(B, pa, ua, pb, ub, r, out, st, 1);
    default: return launch_packed<2>(B, pa, ua, pb, ub, r, out, st, 1);
  }
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

namespace {

inline int grid_for(int64_t n, int t = 256) { return fb::ceil_div(n > 0 ? n : 1, t); }

// levels + per-block grouping of one triangular part (device)
int device_levels(int64_t n, int64_t nblocks, const int64_t* bptr, TriPart& P, bool lower,
                  cudaStream_t st) {
  DevBuf<int> level, nlev;
  DevBuf<int64_t> bg;
  FB_TRY_CUDA(level.alloc(n));
  FB_TRY_CUDA(nlev.alloc(nblocks + 1));
  FB_TRY_CUDA(bg.alloc(nblocks + 1));
  bilu_levels_kernel<<<grid_for(nblocks, 128), 128, 0, st>>>(nblocks, bptr, P.ip.ptr, P.ix.ptr,
                                                              lower ? 1 : 0, level.ptr, nlev.ptr);
  FB_CHECK_LAUNCH();
  int rc = exclusive_offsets(nlev.ptr, nblocks, bg.ptr, st);
  if (rc != FB_OK) return rc;
  int64_t ngroups = 0;
  FB_TRY_CUDA(cudaMemcpyAsync(&ngroups, bg.ptr + nblocks, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FB_TRY_CUDA(cudaStreamSynchronize(st));
  FB_REQUIRE(ngroups < (int64_t(1) << 31), "too many level groups");
  DevBuf<int> cur;
  FB_TRY_CUDA(P.grp.alloc(ngroups + 1));
  FB_TRY_CUDA(cur.alloc(ngroups + 1));
  FB_TRY_CUDA(P.blk_grp.alloc(nblocks + 1));
  FB_TRY_CUDA(P.rows.alloc(n));
  bilu_group_kernel<<<grid_for(nblocks + 1, 128), 128, 0, st>>>(nblocks, n, bptr, level.ptr, bg.ptr,
                                                                 P.grp.ptr, P.blk_grp.ptr, cur.ptr,
                                                                 P.rows.ptr);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(cudaStreamSynchronize(st));
  return FB_OK;
}

// transpose of a (block-local) CSR part on the device, rows sorted
int device_transpose(int64_t n, const TriPart& S, TriPart& T, cudaStream_t st) {
  DevBuf<int> cnt;
  FB_TRY_CUDA(cnt.alloc(n));
  FB_TRY_CUDA(cudaMemsetAsync(cnt.ptr, 0, n * sizeof(int), st));
  csr_col_count_kernel<<<grid_for(n), 256, 0, st>>>(n, S.ip.ptr, S.ix.ptr, cnt.ptr);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(T.ip.alloc(n + 1));
  int rc = exclusive_offsets(cnt.ptr, n, T.ip.ptr, st);
  if (rc != FB_OK) return rc;
  const int64_t nnz = S.ix.n;
  FB_TRY_CUDA(T.ix.alloc(nnz));
  FB_TRY_CUDA(T.v.alloc(nnz));
  FB_TRY_CUDA(cudaMemsetAsync(cnt.ptr, 0, n * sizeof(int), st));
  csr_transpose_fill_kernel<<<grid_for(n), 256, 0, st>>>(n, S.ip.ptr, S.ix.ptr, S.v.ptr, T.ip.ptr,
                                                          cnt.ptr, T.ix.ptr, T.v.ptr);
  FB_CHECK_LAUNCH();
  csr_sort_rows_kernel<<<grid_for(n), 256, 0, st>>>(n, T.ip.ptr, T.ix.ptr, T.v.ptr);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

}  // namespace

extern "C" int fb_blockilu_create_csr(const fb_csr* A, int64_t nblocks,
                                      const int64_t* block_ptr_host, int64_t* fail_row,
                                      fb_blockilu** out) {
  FB_REQUIRE(out != nullptr && fail_row != nullptr, "out is NULL");
  *out = nullptr;
  *fail_row = -1;
  FB_REQUIRE(A != nullptr && block_ptr_host != nullptr, "bad block ILU input");
  const int64_t n = A->nrows;
  FB_REQUIRE(A->ncols >= n, "block ILU needs ncols >= nrows (columns beyond the rows are ghosts)");
  FB_REQUIRE(nblocks >= 1 && block_ptr_host[0] == 0 && block_ptr_host[nblocks] == n,
             "block_ptr must cover all rows");
  std::unique_ptr<fb_blockilu> B(new fb_blockilu());
  B->n = n;
  B->nblocks = int(nblocks);
  for (int64_t b = 0; b < nblocks; ++b) {
    FB_REQUIRE(block_ptr_host[b + 1] >= block_ptr_host[b], "block_ptr must be non-decreasing");
    B->max_block = std::max<int64_t>(B->max_block, block_ptr_host[b + 1] - block_ptr_host[b]);
  }
  FB_REQUIRE(block_ilu_smem_max(B->max_block) <= 200 * 1024 &&
                 B->max_block <= 65535,
             "block too large for shared memory");
  cudaStream_t st = 0;
  DevBuf<int64_t> bptr64;
  FB_TRY_CUDA(bptr64.upload(block_ptr_host, nblocks + 1));
  {
    std::vector<int> b32(nblocks + 1);
    for (int64_t b = 0; b <= nblocks; ++b) b32[b] = int(block_ptr_host[b]);
    FB_TRY_CUDA(B->block_ptr.upload(b32.data(), nblocks + 1));
  }
  // block-diagonal part F of A
  DevBuf<int> rb, cnt;
  DevBuf<int64_t> fip, dpos;
  DevBuf<int> fix;
  DevBuf<double> fv;
  DevBuf<unsigned long long> flag;
  FB_TRY_CUDA(rb.alloc(n));
  FB_TRY_CUDA(cnt.alloc(n));
  FB_TRY_CUDA(flag.alloc(2));
  FB_TRY_CUDA(cudaMemsetAsync(flag.ptr, 0xff, 2 * sizeof(unsigned long long), st));
  bilu_row_block_kernel<<<grid_for(n), 256, 0, st>>>(n, nblocks, bptr64.ptr, rb.ptr);
  FB_CHECK_LAUNCH();
  bilu_count_kernel<<<grid_for(n), 256, 0, st>>>(n, A->indptr.ptr, A->indices.ptr, bptr64.ptr,
                                                  rb.ptr, cnt.ptr);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(fip.alloc(n + 1));
  int rc = exclusive_offsets(cnt.ptr, n, fip.ptr, st);
  if (rc != FB_OK) return rc;
  int64_t fnnz = 0;
  FB_TRY_CUDA(cudaMemcpy(&fnnz, fip.ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  FB_TRY_CUDA(fix.alloc(fnnz));
  FB_TRY_CUDA(fv.alloc(fnnz));
  FB_TRY_CUDA(dpos.alloc(n));
  bilu_fill_kernel<<<grid_for(n), 256, 0, st>>>(n, A->indptr.ptr, A->indices.ptr, A->data.ptr,
                                                 bptr64.ptr, rb.ptr, fip.ptr, fix.ptr, fv.ptr,
                                                 dpos.ptr, flag.ptr);
  FB_CHECK_LAUNCH();
  rb.reset();
  unsigned long long h[2];
  FB_TRY_CUDA(cudaMemcpy(h, flag.ptr, sizeof(h), cudaMemcpyDeviceToHost));
  if (h[0] != ~0ull) {  // a row without a stored diagonal: same outcome as the host factor
    *fail_row = int64_t(h[0]);
    return FB_OK;
  }
  bilu_factor_kernel<<<grid_for(nblocks, 64), 64, 0, st>>>(nblocks, bptr64.ptr, fip.ptr, fix.ptr,
                                                           fv.ptr, dpos.ptr, flag.ptr + 1);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(cudaMemcpy(h, flag.ptr, sizeof(h), cudaMemcpyDeviceToHost));
  if (h[1] != ~0ull) {
    *fail_row = int64_t(h[1]);
    return FB_OK;
  }
  // split: L strict lower (unit diagonal), U strict upper + inverse diagonal
  DevBuf<int> uc;
  FB_TRY_CUDA(uc.alloc(n));
  bilu_split_count_kernel<<<grid_for(n), 256, 0, st>>>(n, fip.ptr, dpos.ptr, cnt.ptr, uc.ptr);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(B->L.ip.alloc(n + 1));
  FB_TRY_CUDA(B->U.ip.alloc(n + 1));
  rc = exclusive_offsets(cnt.ptr, n, B->L.ip.ptr, st);
  if (rc != FB_OK) return rc;
  rc = exclusive_offsets(uc.ptr, n, B->U.ip.ptr, st);
  if (rc != FB_OK) return rc;
  int64_t lnnz = 0, unnz = 0;
  FB_TRY_CUDA(cudaMemcpy(&lnnz, B->L.ip.ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  FB_TRY_CUDA(cudaMemcpy(&unnz, B->U.ip.ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  FB_TRY_CUDA(B->L.ix.alloc(lnnz));
  FB_TRY_CUDA(B->L.v.alloc(lnnz));
  FB_TRY_CUDA(B->U.ix.alloc(unnz));
  FB_TRY_CUDA(B->U.v.alloc(unnz));
  FB_TRY_CUDA(B->U.invdiag.alloc(n));
  bilu_split_fill_kernel<<<grid_for(n), 256, 0, st>>>(n, fip.ptr, fix.ptr, fv.ptr, dpos.ptr,
                                                       B->L.ip.ptr, B->L.ix.ptr, B->L.v.ptr,
                                                       B->U.ip.ptr, B->U.ix.ptr, B->U.v.ptr,
                                                       B->U.invdiag.ptr);
  FB_CHECK_LAUNCH();
  fix.reset();
  fv.reset();
  fip.reset();
  dpos.reset();
  cnt.reset();
  uc.reset();
  // transposed factors for the backward sweep
  rc = device_transpose(n, B->U, B->Ut, st);
  if (rc != FB_OK) return rc;
  FB_TRY_CUDA(B->Ut.invdiag.alloc(n));
  FB_TRY_CUDA(cudaMemcpyAsync(B->Ut.invdiag.ptr, B->U.invdiag.ptr, n * sizeof(double),
                              cudaMemcpyDeviceToDevice, st));
  rc = device_transpose(n, B->L, B->Lt, st);
  if (rc != FB_OK) return rc;
  // level groups: forward L (lower), U (upper); backward U^T (lower), L^T (upper)
  rc = device_levels(n, nblocks, bptr64.ptr, B->L, true, st);
  if (rc != FB_OK) return rc;
  rc = device_levels(n, nblocks, bptr64.ptr, B->U, false, st);
  if (rc != FB_OK) return rc;
  rc = device_levels(n, nblocks, bptr64.ptr, B->Ut, true, st);
  if (rc != FB_OK) return rc;
  rc = device_levels(n, nblocks, bptr64.ptr, B->Lt, false, st);
  if (rc != FB_OK) return rc;
  FB_TRY_CUDA(cudaDeviceSynchronize());
  {
    const int rc_p = build_packed(B.get());
    if (rc_p != FB_OK) return rc_p;
  }
  if (g_bilu_pipe == 2 && !B->L.pk.ptr) {
    const int rc_ell = build_ell(B.get());
    if (rc_ell != FB_OK) return rc_ell;
  }
  debug_canary_register(B->block_ptr.ptr, int(nblocks + 1));  // FB_DEBUG_SYNC=1 only
  {
    const int rc_g = compute_max_grp(B.get());
    if (rc_g != FB_OK) return rc_g;
  }
  *out = B.release();  // new2old stays empty: the level is block-major already
  return FB_OK;
}

extern "C" int fb_set_blockilu_packed(int on) {
  g_bilu_packed = on ? 1 : 0;
  return FB_OK;
}

extern "C" int fb_set_blockilu_pipeline(int mode, int lanes) {
  FB_REQUIRE(lanes == 0 || lanes == 2 || lanes == 4 || lanes == 8 || lanes == 16 || lanes == 32,
             "lanes per block must be 0 (auto), 2, 4, 8, 16 or 32");
  FB_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0, 1 or 2");
  g_bilu_pipe = mode;
  g_bilu_lanes = lanes;
  return FB_OK;
}
