// C ABI: element restriction and sum-factorized operators.
//   fb_restriction_*  <- FESpace.gather / scatter_add   (fespace.py:282-292)
//   fb_operator_*     <- mfop Mass/Stiffness/Helmholtz/Gradient/Divergence
//                        (mfop.py:169-319)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "fb_common.cuh"
#include "fb_internal.cuh"
#include "sf3_fast.cuh"
#include "sf3_mixed.cuh"
#include "sf3_q1.cuh"
#include "sf_general.cuh"

namespace fb {

int build_factors_device(int dim, int64_t ne, const double* corners_dev, int nq,
                         const double* pts, const double* w1, int kind, double c, double nu,
                         double* fac_dev, int nfac, int64_t fstride, int lanes, cudaStream_t st);

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
bool debug_sync() {
  static const bool on = [] {
    const char* v = std::getenv("FB_DEBUG_SYNC");
    return v != nullptr && v[0] == '1';
  }();
  return on;
}

static std::vector<std::pair<const int*, std::vector<int>>> g_canaries;
void debug_canary_register(const int* p, int n) {
  if (!debug_sync()) return;
  std::vector<int> h(n);
  cudaMemcpy(h.data(), p, n * sizeof(int), cudaMemcpyDeviceToHost);
  g_canaries.push_back({p, h});
}
void debug_canary_unregister(const int* p) {
  for (size_t i = 0; i < g_canaries.size(); ++i)
    if (g_canaries[i].first == p) {
      g_canaries.erase(g_canaries.begin() + i);
      return;
    }
}
bool debug_canary_check(const char* where) {
  for (auto& c : g_canaries) {
    std::vector<int> h(c.second.size());
    cudaMemcpy(h.data(), c.first, h.size() * sizeof(int), cudaMemcpyDeviceToHost);
    if (h != c.second) {
      fprintf(stderr, "CANARY %p corrupted after launch at %s\n", (const void*)c.first, where);
      c.second = h;  // report once
      return false;
    }
  }
  return true;
}

int64_t& launch_counter() {
  static int64_t n = 0;
  return n;
}

// Deterministic E->L sum: y[row_dof[r]] = 0.0 + sum_{k in row r} S[ent[k]],
// entries in ascending flat-E order (bitwise np.bincount, fespace.py:288-292).
__global__ void scatter_rows_kernel(int64_t nrows, const int* __restrict__ row_dof,
                                    const int* __restrict__ off, const int* __restrict__ ent,
                                    const double* __restrict__ S, int64_t S_comp_stride,
                                    double* __restrict__ y, int64_t y_comp_stride) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int comp = blockIdx.y;
  const double* Sc = S + comp * S_comp_stride;
  const int b = __ldg(off + r), e = __ldg(off + r + 1);
  double acc = 0.0;
  for (int k = b; k < e; ++k) acc += __ldg(Sc + __ldg(ent + k));
  const int64_t dof = row_dof ? int64_t(__ldg(row_dof + r)) : r;
  y[comp * y_comp_stride + dof] = acc;
}

// Slot sum of the fused path: shared rows are grouped by multiplicity m and
// a class stores its contributions slot-major (contribution j of all its rows,
// then j+1, ...), so one thread per row reads its m slots as m coalesced
// loads and sums them in flat-E order -- the sequential sum, bitwise
// np.bincount -- and the destinations are ascending DoF ids.
struct SlotClasses {
  int n;
  int m[16];
  int64_t row[17], slot[16];
};

__global__ void __launch_bounds__(256) scatter_slots_kernel(SlotClasses K,
                                                            const int* __restrict__ row_dof,
                                                            const double* __restrict__ S,
                                                            int64_t S_comp_stride,
                                                            double* __restrict__ y,
                                                            int64_t y_comp_stride) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= K.row[K.n]) return;
  int c = 0;
  while (r >= K.row[c + 1]) ++c;
  const int comp = blockIdx.y;
  const int64_t k = r - K.row[c], nc = K.row[c + 1] - K.row[c];
  const double* __restrict__ Sc = S + comp * S_comp_stride + K.slot[c] + k;
  const int m = K.m[c];
  double v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = j < m ? __ldg(Sc + j * nc) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < m) acc += v[j];
  for (int j = 8; j < m; ++j) acc += __ldg(Sc + j * nc);
  y[comp * y_comp_stride + __ldg(row_dof + r)] = acc;
}

__global__ void gather_kernel(int64_t total, const int* __restrict__ map,
                              const double* __restrict__ x, double* __restrict__ xe) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < total) xe[i] = __ldg(x + __ldg(map + i));
}

}  // namespace fb

using namespace fb;

struct fb_restriction {
  int dim = 0, p = 0, n = 0, nloc = 0;
  int64_t ne = 0, ndofs = 0;
  DevBuf<int> map;
  DevBuf<int> full_off, full_ent;  // rows = all DoFs
  int split_ok = 0;
  int nb = 0;  // element-boundary positions per element
  int64_t nsrows = 0;
  DevBuf<int> s_row, s_off, s_ent;
  // class-major slot layout: shared rows grouped by multiplicity m; class c
  // holds rows [cls_row[c], cls_row[c+1]) and their slots at
  // cls_slot[c] + j * (rows in class) + k  (j = contribution rank in flat-E order)
  int ncls = 0;
  int cls_m[16] = {0};
  int64_t cls_row[17] = {0}, cls_slot[16] = {0};
  int nlocp = 0;           // per-element stride of map_pad (multiple of 4)
  DevBuf<int> map_pad;     // (ne, nlocp) for 16-byte bulk copies
  int nbp = 0;             // per-element stride of s_pos (multiple of 4)
  DevBuf<int> s_pos;       // (ne, nbp): transposed-CSR slot of each boundary contribution
};

struct fb_operator {
  int kind = 0, dim = 0, vdim = 1, nq = 0, nv = 0, np = 0, nfac = 0;
  int64_t fstride = 0;  // per-element factor stride (nfac * nq^dim rounded to even)
  const fb_restriction* rv = nullptr;
  const fb_restriction* rp = nullptr;
  bool fast = false;
  bool q1 = false;  // trilinear thread-per-element kernel, interleaved factors
  SF3Params fp;     // host copy of the fast-path parameters
  Q1Params qp;
  DevBuf<double> fac;
  DevBuf<double> mats;
  DevBuf<double> S;  // shared-entry buffer / E-vector scratch
  int64_t S_comp_stride = 0;
  int gen_kind = 0;
  size_t gen_smem = 0;
  bool mixed = false;  // fused 3D G / G^T / D kernel (sf3_mixed.cuh)
  SF3MParams mp;
};

extern "C" {
static int mixed_apply(const fb_operator* op, int mkind, const double* x, double* y, int part,
                       cudaStream_t st);
}

namespace fb {
bool mixed_supported(int nv, int np, int nq);
int launch_mixed(int nv, int np, int kind, const SF3MParams& P, cudaStream_t st);
}  // namespace fb

namespace {

bool position_interior(int dim, int n, int l) {
  for (int a = 0; a < dim; ++a) {
    const int c = l % n;
    l /= n;
    if (c == 0 || c == n - 1) return false;
  }
  return true;
}

// Barycentric differentiation matrix on arbitrary distinct points (the
// formula of basis.py:98-119, evaluated in C++).
void diff_matrix(const double* x, int n, double* D) {
  std::vector<double> w(n, 1.0);
  for (int j = 0; j < n; ++j) {
    double prod = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j) prod *= (x[j] - x[k]);
    w[j] = 1.0 / prod;
  }
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      D[i * n + j] = (w[j] / w[i]) / (x[i] - x[j]);
      s += D[i * n + j];
    }
    D[i * n + i] = -s;
  }
}

// shape of the last fused-kernel launch on this host thread (tests: prove the
// persistent multi-batch path ran; fb_last_fast_launch)
thread_local int g_last_grid = 0, g_last_nbatch = 0, g_last_ne = 0;
int g_fast_skip = 0;  // diagnostics only (fb_set_fast_skip): passes to skip

template <int N, int Q, int KIND, int NE, int NT, int MINB, int ZL>
int launch_fast_t(const fb_operator* op, const double* x, double* y, cudaStream_t st) {
  constexpr size_t smem = SF3Shape<N, Q, KIND, NE, ZL>::SMEM;
  // persistent grid: as many CTAs as can be resident at once
  static int resident = 0;
  if (resident == 0) {
    auto kern = sf3_fast_kernel<N, Q, KIND, NE, NT, MINB, ZL>;
    FB_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
    int dev = 0, sms = 0, per_sm = 0;
    FB_TRY_CUDA(cudaGetDevice(&dev));
    FB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    resident = sms * (per_sm > 0 ? per_sm : 1);
  }
  SF3Params p = op->fp;
  p.x = x;
  p.y = y;
  p.nbatch = ceil_div(op->rv->ne, NE);
  p.skip = g_fast_skip;
  const int grid = p.nbatch < resident ? p.nbatch : resident;
  g_last_grid = grid;
  g_last_nbatch = p.nbatch;
  g_last_ne = NE;
  sf3_fast_kernel<N, Q, KIND, NE, NT, MINB, ZL><<<grid, NT, smem, st>>>(p);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

template <int N, int Q, int NE, int NT, int MINB, int ZL = 0>
int launch_fast_kind(const fb_operator* op, const double* x, double* y, cudaStream_t st) {
  switch (op->kind) {
    case FB_MASS: return launch_fast_t<N, Q, kMass, NE, NT, MINB, ZL>(op, x, y, st);
    case FB_STIFFNESS: return launch_fast_t<N, Q, kStiff, NE, NT, MINB, ZL>(op, x, y, st);
    default: return launch_fast_t<N, Q, kHelm, NE, NT, MINB, ZL>(op, x, y, st);
  }
}

// (N, Q, elements per CTA, threads, min CTAs/SM) per degree; shared memory
// per CTA: double-buffered map/slot stage, gather buffer, 4 work buffers per
// element (34-52 KB); the grid is persistent (all CTAs resident).
// Runtime-selectable launch shapes (tuning): g_fast_cfg[p] picks a variant.
// p = 4 default (v7): 2 elements x 96 threads at 4 CTAs / SM -- the 5-CTA shape
// capped registers at 128 and spilled; 0.566 -> 0.545 ms (tools/tune_fast.py).
// p = 5, 6 defaults (v6): the z-line schedule (ZL = 3) with a register budget
// of 158 / 211 (no spills): p = 5 0.484 -> 0.451 ms, p = 6 0.419 -> 0.352 ms.
// Defaults measured with tools/tune_fast.py: p = 2, 3, 5, 6 stage their
// factor blocks in shared memory through the TMA engine (p = 3: +5 %, p = 4
// with the z-line schedule: +9 %, p = 5:
// +14 %, p = 2, 6: +1-2 %); at p = 7, 8 the extra 41-56 KB per CTA costs more
// occupancy than it saves.
static const int kFastCfgDefault[9] = {0, 0, 0, 5, 7, 6, 6, 0, 6};
static int g_fast_cfg[9] = {0, 0, 0, 5, 7, 6, 6, 0, 6};

int launch_fast(const fb_operator* op, const double* x, double* y, cudaStream_t st) {
  const int v = g_fast_cfg[op->rv->p < 9 ? op->rv->p : 0];
  switch (op->rv->p) {
    case 1: return launch_fast_kind<2, 3, 32, 288, 3>(op, x, y, st);  // (p=1 uses sf3_q1)
    case 2:
      if (v == 1) return launch_fast_kind<3, 4, 16, 256, 3, true>(op, x, y, st);
      if (v == 2) return launch_fast_kind<3, 4, 4, 64, 6, 3>(op, x, y, st);
      if (v == 3) return launch_fast_kind<3, 4, 4, 64, 8, 3>(op, x, y, st);
      if (v == 4) return launch_fast_kind<3, 4, 4, 64, 10, 3>(op, x, y, st);
      return launch_fast_kind<3, 4, 4, 64, 10, true>(op, x, y, st);
    case 3:
      if (v == 1) return launch_fast_kind<4, 5, 2, 64, 6, 3>(op, x, y, st);
      if (v == 2) return launch_fast_kind<4, 5, 4, 128, 3, 3>(op, x, y, st);
      if (v == 3) return launch_fast_kind<4, 5, 2, 64, 8, 3>(op, x, y, st);
      if (v == 4) return launch_fast_kind<4, 5, 2, 64, 10, 3>(op, x, y, st);
      if (v == 5) return launch_fast_kind<4, 5, 4, 128, 4, 3>(op, x, y, st);
      return launch_fast_kind<4, 5, 2, 64, 10, true>(op, x, y, st);
    case 4:
      if (v == 1) return launch_fast_kind<5, 6, 4, 160, 5>(op, x, y, st);
      if (v == 2) return launch_fast_kind<5, 6, 1, 64, 12>(op, x, y, st);
      if (v == 3) return launch_fast_kind<5, 6, 2, 96, 6, 2>(op, x, y, st);
      if (v == 4) return launch_fast_kind<5, 6, 1, 64, 6, 3>(op, x, y, st);
      if (v == 5) return launch_fast_kind<5, 6, 1, 64, 4, 3>(op, x, y, st);
      if (v == 6) return launch_fast_kind<5, 6, 2, 96, 5, 3>(op, x, y, st);
      if (v == 7) return launch_fast_kind<5, 6, 2, 96, 4, 3>(op, x, y, st);
      return launch_fast_kind<5, 6, 2, 96, 8>(op, x, y, st);
    case 5:
      if (v == 1) return launch_fast_kind<6, 7, 1, 64, 6, 3>(op, x, y, st);
      if (v == 2) return launch_fast_kind<6, 7, 1, 64, 4, 3>(op, x, y, st);
      if (v == 3) return launch_fast_kind<6, 7, 1, 64, 5, 3>(op, x, y, st);
      if (v == 4) return launch_fast_kind<6, 7, 1, 96, 3, 3>(op, x, y, st);
      if (v == 5) return launch_fast_kind<6, 7, 2, 128, 3, 2>(op, x, y, st);
      if (v == 6) return launch_fast_kind<6, 7, 2, 128, 3, 3>(op, x, y, st);
      if (v == 7) return launch_fast_kind<6, 7, 2, 96, 4, 3>(op, x, y, st);
      return launch_fast_kind<6, 7, 1, 64, 10>(op, x, y, st);
    case 6:
      if (v == 1) return launch_fast_kind<7, 8, 2, 128, 2, 3>(op, x, y, st);
      if (v == 2) return launch_fast_kind<7, 8, 2, 192, 4>(op, x, y, st);
      if (v == 3) return launch_fast_kind<7, 8, 1, 96, 5, 2>(op, x, y, st);
      if (v == 4) return launch_fast_kind<7, 8, 1, 128, 4, 2>(op, x, y, st);
      if (v == 5) return launch_fast_kind<7, 8, 1, 64, 6, 2>(op, x, y, st);
      if (v == 6) return launch_fast_kind<7, 8, 1, 64, 4, 3>(op, x, y, st);
      if (v == 7) return launch_fast_kind<7, 8, 1, 64, 3, 3>(op, x, y, st);
      return launch_fast_kind<7, 8, 1, 96, 8>(op, x, y, st);
    case 7:
      if (v == 1) return launch_fast_kind<8, 9, 1, 96, 3, 3>(op, x, y, st);
      if (v == 2) return launch_fast_kind<8, 9, 1, 160, 2, 3>(op, x, y, st);
      if (v == 3) return launch_fast_kind<8, 9, 1, 128, 3, 2>(op, x, y, st);
      if (v == 4) return launch_fast_kind<8, 9, 1, 192, 2, 2>(op, x, y, st);
      if (v == 5) return launch_fast_kind<8, 9, 1, 96, 3, 2>(op, x, y, st);
      if (v == 6) return launch_fast_kind<8, 9, 1, 128, 2, 3>(op, x, y, st);
      if (v == 7) return launch_fast_kind<8, 9, 1, 192, 2, 3>(op, x, y, st);
      return launch_fast_kind<8, 9, 1, 128, 4>(op, x, y, st);
    case 8:
      if (v == 1) return launch_fast_kind<9, 10, 1, 96, 2, 3>(op, x, y, st);
      if (v == 2) return launch_fast_kind<9, 10, 1, 160, 1, 3>(op, x, y, st);
      if (v == 3) return launch_fast_kind<9, 10, 1, 128, 2, 2>(op, x, y, st);
      if (v == 4) return launch_fast_kind<9, 10, 1, 192, 2, 2>(op, x, y, st);
      if (v == 5) return launch_fast_kind<9, 10, 1, 256, 1, 2>(op, x, y, st);
      if (v == 6) return launch_fast_kind<9, 10, 1, 128, 2, 3>(op, x, y, st);
      if (v == 7) return launch_fast_kind<9, 10, 1, 192, 1, 3>(op, x, y, st);
      return launch_fast_kind<9, 10, 1, 128, 4>(op, x, y, st);
    default: set_error("fast path not built for this degree"); return FB_ERR_UNSUPPORTED;
  }
}

int scatter_rows(const fb_restriction* r, bool split, const double* S, int64_t S_comp_stride,
                 double* y, int64_t y_comp_stride, int ncomp, cudaStream_t st) {
  const int64_t nrows = split ? r->nsrows : r->ndofs;
  if (nrows == 0) return FB_OK;
  if (split) {
    SlotClasses K;
    K.n = r->ncls;
    for (int c = 0; c < r->ncls; ++c) {
      K.m[c] = r->cls_m[c];
      K.slot[c] = r->cls_slot[c];
    }
    for (int c = 0; c <= r->ncls; ++c) K.row[c] = r->cls_row[c];
    dim3 grid(ceil_div(nrows, 256), ncomp);
    scatter_slots_kernel<<<grid, 256, 0, st>>>(K, r->s_row.ptr, S, S_comp_stride, y,
                                               y_comp_stride);
  } else {
    dim3 grid(ceil_div(nrows, 256), ncomp);
    scatter_rows_kernel<<<grid, 256, 0, st>>>(nrows, nullptr, r->full_off.ptr, r->full_ent.ptr,
                                              S, S_comp_stride, y, y_comp_stride);
  }
  FB_CHECK_LAUNCH();
  return FB_OK;
}

// AoS (ne, nq, k) -> element-blocked (ne, [k, nq] padded to fstride), or for
// lanes = 32 the interleaved, point-major layout [ne/32][nq][ktot][32].
void relayout(const double* src, int64_t ne, int nqd, int k, double* dst, int64_t fstride,
              int koff, int lanes = 0, int ktot = 0) {
  for (int64_t e = 0; e < ne; ++e)
    for (int c = 0; c < k; ++c)
      for (int q = 0; q < nqd; ++q) {
        const double v = src[(e * nqd + q) * k + c];
        if (lanes)
          dst[((e / lanes) * int64_t(nqd) + q) * int64_t(ktot) * lanes +
              int64_t(koff + c) * lanes + (e % lanes)] = v;
        else
          dst[e * fstride + int64_t(koff + c) * nqd + q] = v;
      }
}

bool use_q1(int kind, int dim, int p, int nq1, const fb_restriction* rv) {
  return kind <= FB_HELMHOLTZ && dim == 3 && p == 1 && nq1 == 3 && rv->split_ok;
}

int64_t factor_count(bool q1, int64_t ne, int nfac, int nqd, int64_t fstride) {
  return q1 ? (ne + 31) / 32 * 32 * int64_t(nfac) * nqd : ne * fstride;
}

}  // namespace

static int finish_operator(fb_operator* op, const double* points, const double* B,
                           const double* D, const double* Bp, const double* Dp) {
  const fb_restriction* rv = op->rv;
  const fb_restriction* rp = op->rp;
  const int kind = op->kind, dim = op->dim, nq1 = op->nq, vdim = op->vdim;
  const int64_t ne = rv->ne;

  // fast path: 3D square kinds, n_q = p + 2, p in 1..8, conforming split
  const int p = rv->p;
  op->fast = (kind <= FB_HELMHOLTZ) && dim == 3 && nq1 == p + 2 && p >= 1 && p <= 8 &&
             rv->split_ok;
  op->q1 = op->fast && use_q1(kind, dim, p, nq1, rv);
  if (op->q1) {
    Q1Params& qp = op->qp;
    std::memset(&qp, 0, sizeof(qp));
    for (int q = 0; q < 3; ++q)
      for (int i = 0; i < 2; ++i) qp.B[q][i] = B[q * 2 + i];
    std::vector<double> Dq(9);
    diff_matrix(points, 3, Dq.data());
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) qp.Dq[a][b] = Dq[a * 3 + b];
    FB_REQUIRE(rv->nlocp == 8 && rv->nbp == 8, "unexpected p=1 map layout");
    qp.map = rv->map_pad.ptr;
    qp.spos = rv->s_pos.ptr;
    qp.fac = op->fac.ptr;
    qp.ne = ne;
    qp.x_comp_stride = rv->ndofs;
    qp.S_comp_stride = ne * rv->nb;
    qp.vdim = vdim;
    op->S_comp_stride = ne * rv->nb;
    FB_TRY_CUDA(op->S.alloc(op->S_comp_stride * vdim));
    qp.S = op->S.ptr;
  } else if (op->fast) {
    SF3Params& fp = op->fp;
    std::memset(&fp, 0, sizeof(fp));
    const int n = rv->n;
    for (int q = 0; q < nq1; ++q)
      for (int i = 0; i < n; ++i) fp.B[q][i] = B[q * n + i];
    std::vector<double> Dq(nq1 * nq1);
    diff_matrix(points, nq1, Dq.data());
    for (int a = 0; a < nq1; ++a)
      for (int b = 0; b < nq1; ++b) fp.Dq[a][b] = Dq[a * nq1 + b];
    {  // even-odd forms (sf3_fast.cuh eo_lines) of B, B^T, Dq, Dq^T
      std::vector<double> Bt(size_t(n) * nq1), Dt(size_t(nq1) * nq1);
      for (int q = 0; q < nq1; ++q)
        for (int i = 0; i < n; ++i) Bt[i * nq1 + q] = B[q * n + i];
      for (int a = 0; a < nq1; ++a)
        for (int b = 0; b < nq1; ++b) Dt[b * nq1 + a] = Dq[a * nq1 + b];
      eo_fill(fp.eB, B, nq1, n);
      eo_fill(fp.eBt, Bt.data(), n, nq1);
      eo_fill(fp.eD, Dq.data(), nq1, nq1);
      eo_fill(fp.eDt, Dt.data(), nq1, nq1);
    }
    fp.map = rv->map_pad.ptr;
    fp.spos = rv->s_pos.ptr;
    fp.fac = op->fac.ptr;
    fp.ne = ne;
    fp.x_comp_stride = rv->ndofs;
    fp.S_comp_stride = ne * rv->nb;
    fp.vdim = vdim;
    op->S_comp_stride = ne * rv->nb;  // == number of transposed-CSR slots
    FB_TRY_CUDA(op->S.alloc(op->S_comp_stride * vdim));
    fp.S = op->S.ptr;
  } else if ((kind == FB_GRADIENT || kind == FB_DIVERGENCE) && dim == 3 && rp != nullptr &&
             mixed_supported(rv->n, rp->n, nq1) && rv->split_ok && rp->split_ok) {
    // fused mixed-degree path (K1g): even-odd forms of B_v, B_p, Dq and transposes
    op->mixed = true;
    SF3MParams& mp = op->mp;
    std::memset(&mp, 0, sizeof(mp));
    const int nv = rv->n, np = rp->n;
    std::vector<double> Dq(nq1 * nq1), Dt(nq1 * nq1), Bvt(size_t(nv) * nq1), Bpt(size_t(np) * nq1);
    diff_matrix(points, nq1, Dq.data());
    for (int a = 0; a < nq1; ++a)
      for (int b = 0; b < nq1; ++b) Dt[b * nq1 + a] = Dq[a * nq1 + b];
    for (int q = 0; q < nq1; ++q) {
      for (int i = 0; i < nv; ++i) Bvt[i * nq1 + q] = B[q * nv + i];
      for (int i = 0; i < np; ++i) Bpt[i * nq1 + q] = Bp[q * np + i];
    }
    eo_fill(mp.eBv, B, nq1, nv);
    eo_fill(mp.eBvt, Bvt.data(), nv, nq1);
    eo_fill(mp.eBp, Bp, nq1, np);
    eo_fill(mp.eBpt, Bpt.data(), np, nq1);
    eo_fill(mp.eD, Dq.data(), nq1, nq1);
    eo_fill(mp.eDt, Dt.data(), nq1, nq1);
    mp.fac = op->fac.ptr;
    mp.ne = ne;
    mp.fstride = op->fstride;
    const int64_t sv = ne * rv->nb, sp_ = ne * rp->nb;
    FB_TRY_CUDA(op->S.alloc(std::max(3 * sv, sp_)));
    mp.S = op->S.ptr;
  } else {
    // general path
    const int nv = rv->n, np = op->np;
    std::vector<double> mats(size_t(2) * nq1 * nv + size_t(2) * nq1 * np);
    std::memcpy(mats.data(), B, sizeof(double) * nq1 * nv);
    std::memcpy(mats.data() + nq1 * nv, D, sizeof(double) * nq1 * nv);
    if (np > 0) {
      std::memcpy(mats.data() + 2 * nq1 * nv, Bp, sizeof(double) * nq1 * np);
      std::memcpy(mats.data() + 2 * nq1 * nv + nq1 * np, Dp, sizeof(double) * nq1 * np);
    }
    FB_TRY_CUDA(op->mats.upload(mats.data(), int64_t(mats.size())));
    op->gen_smem = gen_smem_bytes(dim, nv, np, nq1);
    FB_REQUIRE(op->gen_smem <= 227 * 1024, "element too large for the general kernel");
    FB_TRY_CUDA(cudaFuncSetAttribute(sf_general_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(227 * 1024)));
    // E-vector scratch: largest of input/output E-vectors over components
    const int64_t nvl = rv->nloc, npl = rp ? rp->nloc : 0;
    int64_t need = 0;
    if (kind <= FB_HELMHOLTZ || kind == FB_CONVECTION || kind == FB_CURLCURL)
      need = int64_t(vdim) * ne * nvl;
    else if (kind == FB_GRADIENT) need = int64_t(dim) * ne * nvl + ne * npl;
    else need = ne * npl;
    FB_TRY_CUDA(op->S.alloc(need));
  }
  return FB_OK;
}

namespace fb {
const int* restriction_map(const fb_restriction* r) { return r->map.ptr; }
int restriction_nloc(const fb_restriction* r) { return r->nloc; }
int64_t restriction_ne(const fb_restriction* r) { return r->ne; }
int64_t restriction_ndofs(const fb_restriction* r) { return r->ndofs; }
}  // namespace fb

extern "C" {

const char* fb_last_error(void) { return g_last_error.c_str(); }
int fb_abi_version(void) { return 1; }
int64_t fb_launch_count(void) { return launch_counter(); }

int fb_restriction_create(int dim, int p, int64_t ne, int64_t ndofs,
                          const int64_t* element_dofs, fb_restriction** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3");
  FB_REQUIRE(p >= 1, "degree must be >= 1");
  FB_REQUIRE(ne >= 0 && ndofs >= 0, "negative sizes");
  FB_REQUIRE(ne == 0 || element_dofs != nullptr, "element_dofs is NULL");
  std::unique_ptr<fb_restriction> r(new fb_restriction());
  r->dim = dim;
  r->p = p;
  r->n = p + 1;
  r->nloc = dim == 2 ? r->n * r->n : r->n * r->n * r->n;
  r->ne = ne;
  r->ndofs = ndofs;
  const int nloc = r->nloc, n = r->n;
  const int64_t total = ne * nloc;
  FB_REQUIRE(total < (int64_t(1) << 31) && ndofs < (int64_t(1) << 31),
             "element map exceeds int32 indexing");
  std::vector<int> map(total);
  std::vector<int> count(ndofs + 1, 0);
  for (int64_t k = 0; k < total; ++k) {
    const int64_t d = element_dofs[k];
    FB_REQUIRE(d >= 0 && d < ndofs, "element_dofs entry out of range");
    map[k] = int(d);
    ++count[d];
  }
  // full transposed map: counting sort keeps ascending flat-E order
  std::vector<int> off(ndofs + 1, 0);
  for (int64_t i = 0; i < ndofs; ++i) off[i + 1] = off[i] + count[i];
  std::vector<int> ent(total);
  {
    std::vector<int> pos(off.begin(), off.end() - 1);
    for (int64_t k = 0; k < total; ++k) ent[pos[map[k]]++] = int(k);
  }
  // split mode: interior positions written directly when their DoF is unique
  std::vector<char> interior(nloc);
  std::vector<int> rank(nloc, -1);
  int nb = 0;
  for (int l = 0; l < nloc; ++l) {
    interior[l] = position_interior(dim, n, l);
    if (!interior[l]) rank[l] = nb++;
  }
  r->nb = nb;
  std::vector<char> direct(ndofs, 0);
  bool ok = true;
  for (int64_t e = 0; e < ne && ok; ++e)
    for (int l = 0; l < nloc; ++l)
      if (interior[l]) {
        const int d = map[e * nloc + l];
        if (count[d] != 1) {
          ok = false;
          break;
        }
        direct[d] = 1;
      }
  r->split_ok = ok ? 1 : 0;
  FB_TRY_CUDA(r->map.upload(map.data(), total));
  {
    r->nlocp = (nloc + 3) / 4 * 4;
    std::vector<int> mp(size_t(ne) * r->nlocp, 0);
    for (int64_t e = 0; e < ne; ++e)
      std::memcpy(mp.data() + e * r->nlocp, map.data() + e * nloc, sizeof(int) * nloc);
    FB_TRY_CUDA(r->map_pad.upload(mp.data(), int64_t(mp.size())));
  }
  FB_TRY_CUDA(r->full_off.upload(off.data(), ndofs + 1));
  FB_TRY_CUDA(r->full_ent.upload(ent.data(), total));
  if (ok) {
    // shared rows (element-boundary DoFs) grouped by multiplicity, ascending
    // DoF order inside a class
    int mult_max = 0;
    for (int64_t i = 0; i < ndofs; ++i)
      if (!direct[i]) mult_max = std::max(mult_max, count[i]);
    std::vector<int> cls_of_m(mult_max + 1, -1);
    int ncls = 0;
    // multiplicity 0: DoFs no element touches (ghost planes of a slab-local
    // space); their class has no slots and the sum writes 0.0 (np.bincount)
    for (int64_t i = 0; i < ndofs; ++i)
      if (!direct[i] && cls_of_m[count[i]] < 0) cls_of_m[count[i]] = 1;
    for (int m = 0; m <= mult_max; ++m)
      if (cls_of_m[m] > 0) cls_of_m[m] = ncls++;
    ok = ncls <= 16;
    if (ok) {
      r->ncls = ncls;
      std::vector<int64_t> ccount(ncls, 0);
      for (int m = 0; m <= mult_max; ++m)
        if (cls_of_m[m] >= 0) r->cls_m[cls_of_m[m]] = m;
      for (int64_t i = 0; i < ndofs; ++i)
        if (!direct[i]) ccount[cls_of_m[count[i]]]++;
      r->cls_row[0] = 0;
      int64_t slot = 0;
      for (int c = 0; c < ncls; ++c) {
        r->cls_row[c + 1] = r->cls_row[c] + ccount[c];
        r->cls_slot[c] = slot;
        slot += ccount[c] * r->cls_m[c];
      }
      std::vector<int> rows(r->cls_row[ncls]);
      std::vector<int64_t> rowpos(ndofs, -1);  // class-ordered row index
      std::vector<int64_t> fill(r->cls_row, r->cls_row + ncls);
      for (int64_t i = 0; i < ndofs; ++i)
        if (!direct[i]) {
          const int c = cls_of_m[count[i]];
          rowpos[i] = fill[c];
          rows[fill[c]++] = int(i);
        }
      // slot of every (element, boundary position) contribution; j-th
      // contribution of a row in ascending flat-E order (np.bincount order)
      r->nbp = (nb + 3) / 4 * 4;
      std::vector<int> spos(size_t(ne) * r->nbp, 0);
      std::vector<int> seen(ndofs, 0);
      for (int64_t e = 0; e < ne; ++e)
        for (int l = 0; l < nloc; ++l) {
          if (interior[l]) continue;
          const int d = map[e * nloc + l];
          const int c = cls_of_m[count[d]];
          const int64_t k = rowpos[d] - r->cls_row[c];
          const int64_t nc = r->cls_row[c + 1] - r->cls_row[c];
          spos[e * r->nbp + rank[l]] = int(r->cls_slot[c] + int64_t(seen[d]++) * nc + k);
        }
      r->nsrows = int64_t(rows.size());
      FB_TRY_CUDA(r->s_row.upload(rows.data(), r->nsrows));
      FB_TRY_CUDA(r->s_pos.upload(spos.data(), int64_t(spos.size())));
      r->s_ent.reset();
    }
    r->split_ok = ok ? 1 : 0;
  }
  *out = r.release();
  return FB_OK;
}

void fb_restriction_destroy(fb_restriction* r) { delete r; }
int64_t fb_restriction_ndofs(const fb_restriction* r) { return r ? r->ndofs : -1; }

int fb_restriction_gather(const fb_restriction* r, const double* x, double* xe, void* stream) {
  FB_REQUIRE(r != nullptr, "restriction is NULL");
  const int64_t total = r->ne * r->nloc;
  if (total == 0) return FB_OK;
  gather_kernel<<<ceil_div(total, 256), 256, 0, as_stream(stream)>>>(total, r->map.ptr, x, xe);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_restriction_scatter_add(const fb_restriction* r, const double* xe, double* y,
                               void* stream) {
  FB_REQUIRE(r != nullptr, "restriction is NULL");
  return scatter_rows(r, false, xe, 0, y, 0, 1, as_stream(stream));
}

int fb_operator_create(int kind, const fb_restriction* rv, const fb_restriction* rp, int vdim,
                       int nq1, const double* points, const double* B, const double* D,
                       const double* Bp, const double* Dp, const double* wdet,
                       const double* stiff, const double* grad, fb_operator** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(rv != nullptr, "space restriction is NULL");
  FB_REQUIRE(kind >= FB_MASS && kind <= FB_CURLCURL, "unknown operator kind");
  FB_REQUIRE(nq1 >= 1 && nq1 <= 32, "unsupported rule size");
  FB_REQUIRE(B != nullptr && D != nullptr && points != nullptr, "B/D/points are NULL");
  std::unique_ptr<fb_operator> op(new fb_operator());
  const int dim = rv->dim;
  op->kind = kind;
  op->dim = dim;
  op->vdim = vdim;
  op->nq = nq1;
  op->nv = rv->n;
  op->rv = rv;
  const int64_t ne = rv->ne;
  const int nqd = dim == 2 ? nq1 * nq1 : nq1 * nq1 * nq1;
  const int ksym = dim == 2 ? 3 : 6;
  std::vector<double> fac;
  if (kind <= FB_HELMHOLTZ) {
    FB_REQUIRE(vdim >= 1, "vdim must be >= 1");
    if (kind != FB_STIFFNESS) FB_REQUIRE(wdet != nullptr, "mass factor (wdet) required");
    if (kind != FB_MASS) FB_REQUIRE(stiff != nullptr, "stiffness factor required");
    op->nfac = (kind == FB_MASS) ? 1 : (kind == FB_STIFFNESS ? ksym : ksym + 1);
    op->fstride = (int64_t(op->nfac) * nqd + 1) / 2 * 2;
    const bool q1 = use_q1(kind, dim, rv->p, nq1, rv);
    const int lanes = q1 ? 32 : 0;
    fac.assign(size_t(factor_count(q1, ne, op->nfac, nqd, op->fstride)), 0.0);
    int koff = 0;
    if (kind != FB_STIFFNESS) {
      relayout(wdet, ne, nqd, 1, fac.data(), op->fstride, 0, lanes, op->nfac);
      koff = 1;
    }
    if (kind != FB_MASS)
      relayout(stiff, ne, nqd, ksym, fac.data(), op->fstride, koff, lanes, op->nfac);
  } else if (kind == FB_CURLCURL) {
    FB_REQUIRE(vdim == dim, "curl-curl expects a vector space with vdim == dim");
    FB_REQUIRE(grad != nullptr, "curl factor (nu wdet, Jinv) required");
    op->nfac = 1 + dim * dim;
    op->fstride = (int64_t(op->nfac) * nqd + 1) / 2 * 2;
    fac.assign(size_t(ne) * op->fstride, 0.0);
    relayout(grad, ne, nqd, 1 + dim * dim, fac.data(), op->fstride, 0);
  } else if (kind == FB_CONVECTION) {
    FB_REQUIRE(vdim == dim, "convection expects a vector space with vdim == dim");
    FB_REQUIRE(grad != nullptr, "gradient factor required");
    op->nfac = dim * dim;
    op->fstride = (int64_t(op->nfac) * nqd + 1) / 2 * 2;
    fac.assign(size_t(ne) * op->fstride, 0.0);
    relayout(grad, ne, nqd, dim * dim, fac.data(), op->fstride, 0);
  } else {
    FB_REQUIRE(rp != nullptr, "pressure restriction is NULL");
    FB_REQUIRE(rp->ne == ne && rp->dim == dim, "velocity/pressure spaces disagree");
    FB_REQUIRE(vdim == dim, "mixed operators expect vdim == dim");
    FB_REQUIRE(grad != nullptr && Bp != nullptr && Dp != nullptr, "gradient factor / Bp / Dp required");
    op->rp = rp;
    op->np = rp->n;
    op->nfac = dim * dim;
    op->fstride = (int64_t(op->nfac) * nqd + 1) / 2 * 2;
    fac.assign(size_t(ne) * op->fstride, 0.0);
    relayout(grad, ne, nqd, dim * dim, fac.data(), op->fstride, 0);
  }
  FB_TRY_CUDA(op->fac.upload(fac.data(), int64_t(fac.size())));
  int rc = finish_operator(op.get(), points, B, D, Bp, Dp);
  if (rc != FB_OK) return rc;
  *out = op.release();
  return FB_OK;
}

int fb_operator_create_geom(int kind, const fb_restriction* rv, const fb_restriction* rp,
                            int vdim, int nq1, const double* points, const double* weights,
                            const double* B, const double* D, const double* Bp,
                            const double* Dp, const double* corners, double c, double nu,
                            fb_operator** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(rv != nullptr, "space restriction is NULL");
  FB_REQUIRE(kind >= FB_MASS && kind <= FB_CURLCURL, "unknown operator kind");
  FB_REQUIRE(nq1 >= 1 && nq1 <= 32, "unsupported rule size");
  FB_REQUIRE(points && weights && B && D, "points/weights/B/D are NULL");
  FB_REQUIRE(rv->ne == 0 || corners != nullptr, "corners are NULL");
  std::unique_ptr<fb_operator> op(new fb_operator());
  const int dim = rv->dim;
  op->kind = kind;
  op->dim = dim;
  op->vdim = vdim;
  op->nq = nq1;
  op->nv = rv->n;
  op->rv = rv;
  const int64_t ne = rv->ne;
  const int nqd = dim == 2 ? nq1 * nq1 : nq1 * nq1 * nq1;
  const int ksym = dim == 2 ? 3 : 6;
  if (kind <= FB_HELMHOLTZ) {
    op->nfac = (kind == FB_MASS) ? 1 : (kind == FB_STIFFNESS ? ksym : ksym + 1);
  } else if (kind == FB_CONVECTION) {
    FB_REQUIRE(vdim == dim, "convection expects a vector space with vdim == dim");
    op->nfac = dim * dim;
  } else if (kind == FB_CURLCURL) {
    FB_REQUIRE(vdim == dim, "curl-curl expects a vector space with vdim == dim");
    op->nfac = 1 + dim * dim;
  } else {
    FB_REQUIRE(rp != nullptr && rp->ne == ne && rp->dim == dim, "pressure restriction mismatch");
    FB_REQUIRE(Bp != nullptr && Dp != nullptr, "Bp/Dp required");
    FB_REQUIRE(vdim == dim, "mixed operators expect vdim == dim");
    op->rp = rp;
    op->np = rp->n;
    op->nfac = dim * dim;
  }
  op->fstride = (int64_t(op->nfac) * nqd + 1) / 2 * 2;
  const bool q1 = use_q1(kind, dim, rv->p, nq1, rv);
  FB_TRY_CUDA(op->fac.alloc(factor_count(q1, ne, op->nfac, nqd, op->fstride)));
  FB_TRY_CUDA(cudaMemset(op->fac.ptr, 0, op->fac.bytes()));
  {
    DevBuf<double> cd;
    FB_TRY_CUDA(cd.upload(corners, ne * (int64_t(1) << dim) * dim));
    int rc = build_factors_device(dim, ne, cd.ptr, nq1, points, weights, kind, c, nu,
                                  op->fac.ptr, op->nfac, op->fstride, q1 ? 32 : 0, 0);
    if (rc != FB_OK) return rc;
    FB_TRY_CUDA(cudaDeviceSynchronize());
  }
  int rc = finish_operator(op.get(), points, B, D, Bp, Dp);
  if (rc != FB_OK) return rc;
  *out = op.release();
  return FB_OK;
}

/* Copy the operator's element-blocked factors (ne, K, nq^d) to host. */
int fb_operator_factors(const fb_operator* op, double* host_out, int64_t count) {
  FB_REQUIRE(op != nullptr, "operator is NULL");
  FB_REQUIRE(count == op->fac.n, "factor count mismatch");
  FB_TRY_CUDA(cudaMemcpy(host_out, op->fac.ptr, sizeof(double) * count, cudaMemcpyDeviceToHost));
  return FB_OK;
}

int64_t fb_operator_factor_count(const fb_operator* op) { return op ? op->fac.n : 0; }

int fb_set_fast_skip(int mask) {
  g_fast_skip = mask;
  return FB_OK;
}

int fb_last_fast_launch(int* grid, int* nbatch, int* elements_per_batch) {
  if (grid) *grid = g_last_grid;
  if (nbatch) *nbatch = g_last_nbatch;
  if (elements_per_batch) *elements_per_batch = g_last_ne;
  return FB_OK;
}

int fb_set_fast_config(int p, int variant) {
  FB_REQUIRE(p >= 1 && p <= 8 && variant >= -1 && variant <= 7, "bad fast-path config");
  g_fast_cfg[p] = variant < 0 ? kFastCfgDefault[p] : variant;
  return FB_OK;
}

void fb_operator_destroy(fb_operator* op) { delete op; }

int64_t fb_operator_device_bytes(const fb_operator* op) {
  if (!op) return 0;
  return int64_t(op->fac.bytes() + op->mats.bytes() + op->S.bytes());
}

int fb_operator_fast_path(const fb_operator* op) { return !op ? 0 : op->fast ? 1 : op->mixed ? 2 : 0; }

static int general_apply(const fb_operator* op, int gkind, const double* x, double* y,
                         cudaStream_t st) {
  const fb_restriction* rv = op->rv;
  const fb_restriction* rp = op->rp;
  SFGParams P;
  P.fac = op->fac.ptr;
  P.x = x;
  P.ye = op->S.ptr;
  P.mats = op->mats.ptr;
  P.ne = rv->ne;
  P.dim = op->dim;
  P.kind = gkind;
  P.nv = op->nv;
  P.np = op->np;
  P.nq = op->nq;
  P.nfac = op->nfac;
  P.fstride = op->fstride;
  int gy = 1;
  const fb_restriction* rin = rv;
  const fb_restriction* rout = rv;
  int ncomp_out = 1;
  if (gkind <= kgHelm || gkind == kgConv || gkind == kgCurl) {
    gy = op->vdim;
    ncomp_out = op->vdim;
    P.in_comp_stride = rv->ndofs;
  } else if (gkind == kgGrad) {
    rin = rp;
    ncomp_out = op->dim;
    P.in_comp_stride = 0;
  } else {  // div, gradT: velocity in, pressure out
    rout = rp;
    P.in_comp_stride = rv->ndofs;
  }
  P.map_in = rin->map.ptr;
  if (rv->ne == 0) return FB_OK;
  dim3 grid(unsigned(rv->ne), gy);
  sf_general_kernel<<<grid, 128, op->gen_smem, st>>>(P);
  FB_CHECK_LAUNCH();
  return scatter_rows(rout, false, op->S.ptr, rout->ne * rout->nloc, y, rout->ndofs,
                      ncomp_out, st);
}

int fb_operator_apply_part(const fb_operator* op, const double* x, double* y, int part,
                           void* stream) {
  FB_REQUIRE(op != nullptr, "operator is NULL");
  FB_REQUIRE(part >= 0 && part <= 2, "part must be 0 (all), 1 (element kernel), 2 (E->L sum)");
  cudaStream_t st = as_stream(stream);
  if (op->fast) {
    if (op->rv->ne > 0 && part != 2) {
      if (op->q1) {
        Q1Params qp = op->qp;
        qp.x = x;
        const int grid = ceil_div(op->rv->ne, kQ1Threads);
        static bool q1_configured = false;
        if (!q1_configured) {
          FB_TRY_CUDA(cudaFuncSetAttribute(sf3_q1_kernel<kMass>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kQ1Smem));
          FB_TRY_CUDA(cudaFuncSetAttribute(sf3_q1_kernel<kStiff>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kQ1Smem));
          FB_TRY_CUDA(cudaFuncSetAttribute(sf3_q1_kernel<kHelm>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kQ1Smem));
          q1_configured = true;
        }
        if (op->kind == FB_MASS) sf3_q1_kernel<kMass><<<grid, kQ1Threads, kQ1Smem, st>>>(qp);
        else if (op->kind == FB_STIFFNESS) sf3_q1_kernel<kStiff><<<grid, kQ1Threads, kQ1Smem, st>>>(qp);
        else sf3_q1_kernel<kHelm><<<grid, kQ1Threads, kQ1Smem, st>>>(qp);
        FB_CHECK_LAUNCH();
      } else {
        int rc = launch_fast(op, x, y, st);
        if (rc != FB_OK) return rc;
      }
    }
    if (part == 1) return FB_OK;
    return scatter_rows(op->rv, true, op->S.ptr, op->S_comp_stride, y, op->rv->ndofs,
                        op->vdim, st);
  }
  if (op->mixed)
    return mixed_apply(op, op->kind == FB_GRADIENT ? kMxGrad : kMxDiv, x, y, part, st);
  FB_REQUIRE(part == 0, "split apply is only available on the fused path");
  return fb_operator_apply(op, x, y, stream);
}

// fused mixed-degree apply: kernel (part != 2), then the output space's slot sum
static int mixed_apply(const fb_operator* op, int mkind, const double* x, double* y, int part,
                       cudaStream_t st) {
  const fb_restriction* rv = op->rv;
  const fb_restriction* rp = op->rp;
  const fb_restriction* rin = (mkind == kMxGrad) ? rp : rv;
  const fb_restriction* rout = (mkind == kMxGrad) ? rv : rp;
  SF3MParams P = op->mp;
  P.x = x;
  P.y = y;
  P.map_in = rin->map.ptr;
  P.map_out = rout->map.ptr;
  P.spos_out = rout->s_pos.ptr;
  P.nbp_out = rout->nbp;
  P.in_comp_stride = rin->ndofs;
  P.out_comp_stride = rout->ndofs;
  P.S_comp_stride = rv->ne * rout->nb;
  const int ncomp = (mkind == kMxGrad) ? 3 : 1;
  if (part != 2 && rv->ne > 0) {
    int rc = launch_mixed(rv->n, rp->n, mkind, P, st);
    if (rc != FB_OK) return rc;
  }
  if (part == 1) return FB_OK;
  return scatter_rows(rout, true, op->S.ptr, P.S_comp_stride, y, rout->ndofs, ncomp, st);
}

int fb_operator_apply(const fb_operator* op, const double* x, double* y, void* stream) {
  FB_REQUIRE(op != nullptr, "operator is NULL");
  cudaStream_t st = as_stream(stream);
  if (op->fast) return fb_operator_apply_part(op, x, y, 0, stream);
  if (op->mixed)
    return mixed_apply(op, op->kind == FB_GRADIENT ? kMxGrad : kMxDiv, x, y, 0, st);
  int gk = kgMass;
  switch (op->kind) {
    case FB_MASS: gk = kgMass; break;
    case FB_STIFFNESS: gk = kgStiff; break;
    case FB_HELMHOLTZ: gk = kgHelm; break;
    case FB_GRADIENT: gk = kgGrad; break;
    case FB_CONVECTION: gk = kgConv; break;
    case FB_CURLCURL: gk = kgCurl; break;
    default: gk = kgDiv; break;
  }
  return general_apply(op, gk, x, y, st);
}

int fb_operator_apply_transpose(const fb_operator* op, const double* x, double* y,
                                void* stream) {
  FB_REQUIRE(op != nullptr, "operator is NULL");
  FB_REQUIRE(op->kind == FB_GRADIENT, "apply_transpose is defined for the gradient only");
  if (op->mixed) return mixed_apply(op, kMxGradT, x, y, 0, as_stream(stream));
  return general_apply(op, kgGradT, x, y, as_stream(stream));
}

}  // extern "C"
