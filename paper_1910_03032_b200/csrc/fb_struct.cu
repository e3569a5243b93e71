// Structured-box setup and grid transfers on the device: the "scale mode"
// LOR V-cycle of SURVEY.md 8(e'), with the setup moved off the host
// (SURVEY.md 8(f) items 1-2).
//
// The reference builds every LOR level on the host: a Python/numpy Q1
// assembly on the nodal sub-cell mesh (lor.py:61-81, mfop.py:496-528), a
// COO->CSR conversion, SciPy nodal-interpolation matrices (lor.py:102-123)
// and a numba ILU(0) (numba_backend.py:64-103) -- 55-70 s at 1M DoFs, and
// out of reach at the 100M DoFs of cfg3.  For a structured box everything a
// level needs follows from the lattice:
//   * fb_lor_assemble_box: one thread per lattice point assembles its CSR row
//     of the Q1 (2-point Gauss) matrix on the nodal sub-cell mesh, summing the
//     row of each of its (up to 8) incident sub-cells; sub-cell vertices are
//     evaluated from the parent element's trilinear map, like
//     element_node_coords.  Columns are the 27-point lattice neighbours,
//     sorted by DoF id; constrained rows/columns are zeroed with a unit
//     diagonal (constrain_matrix, lor.py:84-99).
//   * fb_transfer_*: the nodal interpolation between two levels applied
//     matrix-free per fine element: prolongation writes each fine DoF once,
//     from its first-touch owner element (the row the reference's
//     nodal_interpolation builds from dof_owner_elem); restriction (P^T)
//     accumulates per-element contributions and sums them with the coarse
//     map's deterministic transposed-CSR E->L sum.  The same kernels serve
//     p-transfers (same mesh, p -> p') and h-transfers (Q1 on a mesh -> Q1 on
//     the 2x coarsened mesh) through per-axis weight tables.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include "fb_common.cuh"
#include "fb_internal.cuh"

struct fb_transfer {
  const fb_restriction* fine = nullptr;  // fine level map (ne, nf^3)
  const fb_restriction* hmap = nullptr;  // coarse DoFs of each fine element's parent (ne, nc^3)
  int nf = 0, nc = 0;
  int64_t ne = 0, counts[3] = {0, 0, 0};
  int64_t origin[3] = {0, 0, 0};  // global coordinates of local element (0,0,0)
  int periodic = 0;                // periodic axes (bitmask) and their global element counts
  int64_t gcounts[3] = {0, 0, 0};
  fb::DevBuf<double> W;   // (nw, nf, nc) weight tables
  fb::DevBuf<int> widx;   // per axis, per element coordinate: table index
  fb::DevBuf<double> E;   // (ne, nc^3) restriction contributions
};

namespace fb {

__global__ void counts_to_i64_kernel(const int* __restrict__ c, int64_t n, int64_t* __restrict__ o) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i <= n) o[i] = i < n ? int64_t(c[i]) : 0;
}

int exclusive_offsets(const int* counts, int64_t n, int64_t* offsets, cudaStream_t st) {
  counts_to_i64_kernel<<<ceil_div(n + 1, 256), 256, 0, st>>>(counts, n, offsets);
  FB_CHECK_LAUNCH();
  size_t bytes = 0;
  FB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, offsets, offsets, n + 1, st));
  DevBuf<unsigned char> tmp;
  FB_TRY_CUDA(tmp.alloc(int64_t(bytes)));
  FB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, bytes, offsets, offsets, n + 1, st));
  FB_TRY_CUDA(cudaStreamSynchronize(st));  // tmp is freed on return
  return FB_OK;
}

// ---- Q1 LOR assembly on the lattice -----------------------------------------

struct BoxParams {
  int p;
  int64_t nx, ny, nz;   // element counts
  int64_t Nx, Ny, Nz;   // lattice sizes (n_a p + 1)
  const double* corners;  // (ne, 8, 3)
  const int* lid;         // lattice -> DoF id, x fastest
  int kind, constrain;   // constrain: bitmask of constrained box faces (x-, x+, y-, y+, z-, z+)
  int periodic;          // bitmask of periodic axes (x 1, y 2, z 4): N = n p, indices wrap
  int64_t nrows;         // rows with id >= nrows are not assembled (other ranks own them)
  double nu, c;
  double nodes[17];
};

__device__ __forceinline__ bool on_box_boundary(const BoxParams& P, int64_t gx, int64_t gy,
                                                int64_t gz) {
  const int m = P.constrain;
  return ((m & 1) && gx == 0) || ((m & 2) && gx == P.Nx - 1) || ((m & 4) && gy == 0) ||
         ((m & 8) && gy == P.Ny - 1) || ((m & 16) && gz == 0) || ((m & 32) && gz == P.Nz - 1);
}

// physical position of lattice point (gx,gy,gz) through element (ex,ey,ez)
__device__ void lattice_point(const BoxParams& P, int64_t ex, int64_t ey, int64_t ez, int64_t gx,
                              int64_t gy, int64_t gz, double X[3]) {
  const double* C = P.corners + ((ez * P.ny + ey) * P.nx + ex) * 24;
  const double t[3] = {P.nodes[gx - ex * P.p], P.nodes[gy - ey * P.p], P.nodes[gz - ez * P.p]};
  X[0] = X[1] = X[2] = 0.0;
  for (int cc = 0; cc < 8; ++cc) {
    double s = 1.0;
    for (int a = 0; a < 3; ++a) s *= ((cc >> a) & 1) ? (1.0 + t[a]) / 2.0 : (1.0 - t[a]) / 2.0;
    for (int d = 0; d < 3; ++d) X[d] += s * C[cc * 3 + d];
  }
}

// row `vi` of the trilinear sub-cell matrix with vertices X (2-point Gauss)
__device__ void q1_row(const double X[8][3], int vi, int kind, double nu, double c, double K[8]) {
  const double g = 0.57735026918962576451;  // 1/sqrt(3)
  for (int w = 0; w < 8; ++w) K[w] = 0.0;
  for (int q = 0; q < 8; ++q) {
    const double xi[3] = {(q & 1) ? g : -g, (q & 2) ? g : -g, (q & 4) ? g : -g};
    double N[8], dN[8][3];
    for (int v = 0; v < 8; ++v) {
      double f[3], df[3];
      for (int a = 0; a < 3; ++a) {
        const bool hi = (v >> a) & 1;
        f[a] = hi ? (1.0 + xi[a]) / 2.0 : (1.0 - xi[a]) / 2.0;
        df[a] = hi ? 0.5 : -0.5;
      }
      N[v] = f[0] * f[1] * f[2];
      dN[v][0] = df[0] * f[1] * f[2];
      dN[v][1] = f[0] * df[1] * f[2];
      dN[v][2] = f[0] * f[1] * df[2];
    }
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int v = 0; v < 8; ++v)
      for (int d = 0; d < 3; ++d)
        for (int b = 0; b < 3; ++b) J[d][b] += dN[v][b] * X[v][d];
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double Ji[3][3];
    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    if (kind != FB_STIFFNESS) {
      const double wm = (kind == FB_HELMHOLTZ) ? c * det : det;
      for (int w = 0; w < 8; ++w) K[w] += N[vi] * wm * N[w];
    }
    if (kind != FB_MASS) {
      double Wm[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          Wm[a][b] = nu * det * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]);
      double gi[3];
      for (int b = 0; b < 3; ++b)
        gi[b] = dN[vi][0] * Wm[0][b] + dN[vi][1] * Wm[1][b] + dN[vi][2] * Wm[2][b];
      for (int w = 0; w < 8; ++w) K[w] += gi[0] * dN[w][0] + gi[1] * dN[w][1] + gi[2] * dN[w][2];
    }
  }
}

__device__ __forceinline__ int axis_span(int64_t g, int64_t N, bool per) {
  return per ? 3 : 1 + (g > 0) + (g < N - 1);
}

__global__ void lor_box_count_kernel(BoxParams P, int* __restrict__ cnt) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = P.Nx * P.Ny * P.Nz;
  if (t >= total) return;
  const int64_t gx = t % P.Nx, gy = (t / P.Nx) % P.Ny, gz = t / (P.Nx * P.Ny);
  const int row = P.lid[t];
  if (row >= 0 && row < P.nrows)
    cnt[row] = axis_span(gx, P.Nx, P.periodic & 1) * axis_span(gy, P.Ny, P.periodic & 2) *
               axis_span(gz, P.Nz, P.periodic & 4);
}

__global__ void __launch_bounds__(128) lor_box_fill_kernel(BoxParams P,
                                                           const int64_t* __restrict__ ip,
                                                           int* __restrict__ ix,
                                                           double* __restrict__ v) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = P.Nx * P.Ny * P.Nz;
  if (t >= total) return;
  if (P.lid[t] < 0 || P.lid[t] >= P.nrows) return;  // a row of another rank
  const int64_t g[3] = {t % P.Nx, (t / P.Nx) % P.Ny, t / (P.Nx * P.Ny)};
  const int64_t N[3] = {P.Nx, P.Ny, P.Nz};
  const int64_t ne_[3] = {P.nx, P.ny, P.nz};
  const bool brow = on_box_boundary(P, g[0], g[1], g[2]);
  double acc[27];
  for (int k = 0; k < 27; ++k) acc[k] = 0.0;
  if (!brow) {
    // incident sub-cells: min corner m = g - s, s in {0,1}^3, in ascending s
    for (int s = 0; s < 8; ++s) {
      int64_t m[3];
      bool ok = true;
      for (int a = 0; a < 3; ++a) {
        m[a] = g[a] - ((s >> a) & 1);
        if ((P.periodic >> a) & 1) {
          if (m[a] < 0) m[a] += N[a];  // the sub-cell of the last element (wrap)
        } else {
          ok = ok && m[a] >= 0 && m[a] <= N[a] - 2;
        }
      }
      if (!ok) continue;
      int64_t e[3];
      for (int a = 0; a < 3; ++a) e[a] = min(m[a] / P.p, ne_[a] - 1);
      double X[8][3];
      for (int w = 0; w < 8; ++w)
        lattice_point(P, e[0], e[1], e[2], m[0] + (w & 1), m[1] + ((w >> 1) & 1),
                      m[2] + ((w >> 2) & 1), X[w]);
      double K[8];
      q1_row(X, s, P.kind, P.nu, P.c, K);
      for (int w = 0; w < 8; ++w) {
        // neighbour offset of vertex w relative to g, in {-1,0,1}^3
        const int dx = (w & 1) - (s & 1), dy = ((w >> 1) & 1) - ((s >> 1) & 1),
                  dz = ((w >> 2) & 1) - ((s >> 2) & 1);
        acc[(dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)] += K[w];
      }
    }
  }
  // gather the row's (column, value) pairs and insertion-sort them by column
  int cols[27];
  double vals[27];
  int m = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int64_t hx = g[0] + dx, hy = g[1] + dy, hz = g[2] + dz;
        if (P.periodic & 1) hx = (hx + N[0]) % N[0];
        if (P.periodic & 2) hy = (hy + N[1]) % N[1];
        if (P.periodic & 4) hz = (hz + N[2]) % N[2];
        if (hx < 0 || hy < 0 || hz < 0 || hx >= N[0] || hy >= N[1] || hz >= N[2]) continue;
        const int col = P.lid[(hz * N[1] + hy) * N[0] + hx];
        double val = acc[(dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)];
        if (brow) val = (dx == 0 && dy == 0 && dz == 0) ? 1.0 : 0.0;
        else if (on_box_boundary(P, hx, hy, hz)) val = 0.0;
        int j = m - 1;
        while (j >= 0 && cols[j] > col) {
          cols[j + 1] = cols[j];
          vals[j + 1] = vals[j];
          --j;
        }
        cols[j + 1] = col;
        vals[j + 1] = val;
        ++m;
      }
  const int64_t base = ip[P.lid[t]];
  for (int k = 0; k < m; ++k) {
    ix[base + k] = cols[k];
    v[base + k] = vals[k];
  }
}

// ---- matrix-free nodal interpolation between levels -------------------------

struct TransferView {
  const int* fmap;   // (ne, nf^3)
  const int* hmap;   // (ne, nc^3)
  const double* W;   // (nw, nf, nc)
  const int* widx;   // [nx | ny | nz]
  int64_t nx, ny, nz;
  int64_t ox, oy, oz;
  int nf, nc;
  int periodic;
  int64_t gn[3];
  int add;  // prolongation: xf += P xc instead of xf = P xc
};

// fine element e: per-axis coordinates and weight tables
__device__ __forceinline__ void transfer_elem(const TransferView& T, int64_t e, int64_t ec[3],
                                              const double* Wa[3]) {
  ec[0] = e % T.nx;
  ec[1] = (e / T.nx) % T.ny;
  ec[2] = e / (T.nx * T.ny);
  const int64_t off[3] = {0, T.nx, T.nx + T.ny};
  for (int a = 0; a < 3; ++a) Wa[a] = T.W + int64_t(T.widx[off[a] + ec[a]]) * T.nf * T.nc;
  // ownership is decided in global element coordinates (slab-local levels)
  ec[0] += T.ox;
  ec[1] += T.oy;
  ec[2] += T.oz;
}

// first-touch ownership on a structured box: local lattice index 0 along an
// axis belongs to the lower neighbour unless the element is the first one
// (periodic axis: the last element's local index nf-1 is the first
// element's local 0 and belongs to it)
__device__ __forceinline__ bool owned_axis(const TransferView& T, int a, int64_t ec, int l) {
  if (l == 0 && ec != 0) return false;
  if (((T.periodic >> a) & 1) && ec == T.gn[a] - 1 && l == T.nf - 1) return false;
  return true;
}
__device__ __forceinline__ bool owned_local(const TransferView& T, const int64_t ec[3], int l0,
                                            int l1, int l2) {
  return owned_axis(T, 0, ec[0], l0) && owned_axis(T, 1, ec[1], l1) && owned_axis(T, 2, ec[2], l2);
}

// One warp per fine element, kTE elements per CTA.
constexpr int kTE = 4;

// NF / NC > 0: compile-time sizes of the common ladder pairs (fully unrolled
// contractions, constant index arithmetic); 0: runtime sizes.  Same
// summation order either way.
template <int NF, int NC>
__global__ void __launch_bounds__(32 * kTE) transfer_prolong_kernel(TransferView T, int64_t ne,
                                                                    const double* __restrict__ xc,
                                                                    double* __restrict__ xf) {
  // sized by the compile-time ladder pair for nf <= 5 (less shared memory per
  // warp keeps more elements' gathers in flight: p = 4 -> 2 restriction
  // 2.17 -> 1.7 ms at cfg3); nf > 5 keeps the full size (measured slower
  // with more resident warps) and runtime sizes the largest (nf <= 9, nc <= 5)
  __shared__ double xe_all[kTE][(NF > 0 && NF <= 5) ? NC * NC * NC : 125];
  __shared__ double w_all[kTE][3][(NF > 0 && NF <= 5) ? NF * NC : 9 * 5];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = int64_t(blockIdx.x) * kTE + wi;
  if (e >= ne) return;
  double* xe = xe_all[wi];
  auto& w = w_all[wi];
  int64_t ec[3];
  const double* Wa[3];
  transfer_elem(T, e, ec, Wa);
  const int nc = NC > 0 ? NC : T.nc, nf = NF > 0 ? NF : T.nf;
  const int nc3 = nc * nc * nc, nf3 = nf * nf * nf;
  for (int j = lane; j < nc3; j += 32) xe[j] = __ldg(xc + __ldg(T.hmap + e * nc3 + j));
  for (int j = lane; j < nf * nc; j += 32)
    for (int a = 0; a < 3; ++a) w[a][j] = __ldg(Wa[a] + j);
  __syncwarp();
  for (int l = lane; l < nf3; l += 32) {
    const int l0 = l % nf, l1 = (l / nf) % nf, l2 = l / (nf * nf);
    if (!owned_local(T, ec, l0, l1, l2)) continue;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < nc; ++c) {
      double ab = 0.0;
#pragma unroll
      for (int b = 0; b < nc; ++b) {
        double aa = 0.0;
#pragma unroll
        for (int a = 0; a < nc; ++a) aa += w[0][l0 * nc + a] * xe[(c * nc + b) * nc + a];
        ab += w[1][l1 * nc + b] * aa;
      }
      acc += w[2][l2 * nc + c] * ab;
    }
    {
      double* d = xf + __ldg(T.fmap + e * nf3 + l);
      *d = T.add ? __dadd_rn(acc, *d) : acc;
    }
  }
}

template <int NF, int NC>
__global__ void __launch_bounds__(32 * kTE) transfer_restrict_kernel(TransferView T, int64_t ne,
                                                                     const double* __restrict__ xf,
                                                                     double* __restrict__ E) {
  __shared__ double rf_all[kTE][(NF > 0 && NF <= 5) ? NF * NF * NF : 729];
  __shared__ double w_all[kTE][3][(NF > 0 && NF <= 5) ? NF * NC : 9 * 5];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = int64_t(blockIdx.x) * kTE + wi;
  if (e >= ne) return;
  double* rf = rf_all[wi];
  auto& w = w_all[wi];
  int64_t ec[3];
  const double* Wa[3];
  transfer_elem(T, e, ec, Wa);
  const int nc = NC > 0 ? NC : T.nc, nf = NF > 0 ? NF : T.nf;
  const int nc3 = nc * nc * nc, nf3 = nf * nf * nf;
  for (int l = lane; l < nf3; l += 32) {
    const int l0 = l % nf, l1 = (l / nf) % nf, l2 = l / (nf * nf);
    rf[l] = owned_local(T, ec, l0, l1, l2) ? __ldg(xf + __ldg(T.fmap + e * nf3 + l)) : 0.0;
  }
  for (int j = lane; j < nf * nc; j += 32)
    for (int a = 0; a < 3; ++a) w[a][j] = __ldg(Wa[a] + j);
  __syncwarp();
  for (int j = lane; j < nc3; j += 32) {
    const int j0 = j % nc, j1 = (j / nc) % nc, j2 = j / (nc * nc);
    double acc = 0.0;
#pragma unroll 1  // rolled: the fully unrolled nf^3 body thrashes the instruction cache at nf = 8
    for (int l2 = 0; l2 < nf; ++l2) {
      double s1 = 0.0;
#pragma unroll
      for (int l1 = 0; l1 < nf; ++l1) {
        double s0 = 0.0;
#pragma unroll
        for (int l0 = 0; l0 < nf; ++l0) s0 += w[0][l0 * nc + j0] * rf[(l2 * nf + l1) * nf + l0];
        s1 += w[1][l1 * nc + j1] * s0;
      }
      acc += w[2][l2 * nc + j2] * s1;
    }
    E[e * nc3 + j] = acc;
  }
}

// Sum-factorized variants for the wide pairs (nf >= 4: p = 3..8 fine
// levels), one axis per pass with the partial results in shared memory
// sized exactly for the pair: the same nested sums as the direct loops
// above (sum_c w2 (sum_b w1 (sum_a w0 x)) and its transpose), at
// nf nc (nc^2 + nc nf + nf^2) instead of nf^3 (nc^3 + nc^2 + nc) FMAs.
// Measured per cfg3 V-cycle: p = 7 (66^3) restriction 2.46 -> 1.52 ms,
// prolongation 2.22 -> 0.84 ms; p = 4 (116^3) 1.71 -> 1.25 and 1.41 -> 1.15 ms.
// nf = 2, 3 run one thread per element (transfer_q1_kernel,
// transfer_thread_kernel); the warp-per-element direct loops remain for
// runtime sizes.
template <int NF, int NC>
__global__ void __launch_bounds__(32 * kTE) transfer_prolong_sf_kernel(TransferView T, int64_t ne,
                                                                       const double* __restrict__ xc,
                                                                       double* __restrict__ xf) {
  static_assert(NF > 0 && NF <= 9 && NC > 0 && NC <= 5, "compile-time ladder pair");
  __shared__ double xe_all[kTE][NC * NC * NC];
  __shared__ double t1_all[kTE][NC * NC * NF];  // [c][b][l0]
  __shared__ double t2_all[kTE][NC * NF * NF];  // [c][l1][l0]
  __shared__ double w_all[kTE][3][NF * NC];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = int64_t(blockIdx.x) * kTE + wi;
  if (e >= ne) return;
  double* xe = xe_all[wi];
  double* t1 = t1_all[wi];
  double* t2 = t2_all[wi];
  auto& w = w_all[wi];
  int64_t ec[3];
  const double* Wa[3];
  transfer_elem(T, e, ec, Wa);
  constexpr int nc = NC, nf = NF, nc3 = NC * NC * NC, nf3 = NF * NF * NF;
  constexpr int NG = (nf3 + 31) / 32;
  int fm[NG];  // output map, loaded before the passes (off the store path)
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const int l = lane + 32 * i;
    fm[i] = l < nf3 ? __ldg(T.fmap + e * nf3 + l) : 0;
  }
#pragma unroll
  for (int j = lane; j < nc3; j += 32) xe[j] = __ldg(xc + __ldg(T.hmap + e * nc3 + j));
  for (int j = lane; j < nf * nc; j += 32)
    for (int a = 0; a < 3; ++a) w[a][j] = __ldg(Wa[a] + j);
  __syncwarp();
  for (int k = lane; k < nc * nc * nf; k += 32) {  // x: (c, b, l0)
    const int l0 = k % nf, cb = k / nf;
    double aa = 0.0;
#pragma unroll
    for (int a = 0; a < nc; ++a) aa += w[0][l0 * nc + a] * xe[cb * nc + a];
    t1[k] = aa;
  }
  __syncwarp();
  for (int k = lane; k < nc * nf * nf; k += 32) {  // y: (c, l1, l0)
    const int l0 = k % nf, l1 = (k / nf) % nf, c = k / (nf * nf);
    double ab = 0.0;
#pragma unroll
    for (int b = 0; b < nc; ++b) ab += w[1][l1 * nc + b] * t1[(c * nc + b) * nf + l0];
    t2[k] = ab;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NG; ++i) {  // z: (l2, l1, l0), owned fine DoFs only
    const int l = lane + 32 * i;
    if (l >= nf3) continue;
    const int l0 = l % nf, l1 = (l / nf) % nf, l2 = l / (nf * nf);
    if (!owned_local(T, ec, l0, l1, l2)) continue;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < nc; ++c) acc += w[2][l2 * nc + c] * t2[(c * nf + l1) * nf + l0];
    xf[fm[i]] = T.add ? __dadd_rn(acc, xf[fm[i]]) : acc;
  }
}

template <int NF, int NC>
__global__ void __launch_bounds__(32 * kTE) transfer_restrict_sf_kernel(TransferView T, int64_t ne,
                                                                        const double* __restrict__ xf,
                                                                        double* __restrict__ E) {
  static_assert(NF > 0 && NF <= 9 && NC > 0 && NC <= 5, "compile-time ladder pair");
  __shared__ double rf_all[kTE][NF * NF * NF];  // fine values, then [l2][j1][j0]
  __shared__ double u1_all[kTE][NF * NF * NC];  // [l2][l1][j0]
  __shared__ double w_all[kTE][3][NF * NC];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = int64_t(blockIdx.x) * kTE + wi;
  if (e >= ne) return;
  double* rf = rf_all[wi];
  double* u1 = u1_all[wi];
  auto& w = w_all[wi];
  int64_t ec[3];
  const double* Wa[3];
  transfer_elem(T, e, ec, Wa);
  constexpr int nc = NC, nf = NF, nc3 = NC * NC * NC, nf3 = NF * NF * NF;
  constexpr int NG = (nf3 + 31) / 32;  // map loads first, then the gathers (two latencies)
  int fm[NG];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const int l = lane + 32 * i;
    fm[i] = l < nf3 ? __ldg(T.fmap + e * nf3 + l) : 0;
  }
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const int l = lane + 32 * i;
    if (l < nf3) {
      const int l0 = l % nf, l1 = (l / nf) % nf, l2 = l / (nf * nf);
      rf[l] = owned_local(T, ec, l0, l1, l2) ? __ldg(xf + fm[i]) : 0.0;
    }
  }
  for (int j = lane; j < nf * nc; j += 32)
    for (int a = 0; a < 3; ++a) w[a][j] = __ldg(Wa[a] + j);
  __syncwarp();
  for (int k = lane; k < nf * nf * nc; k += 32) {  // x: (l2, l1, j0)
    const int j0 = k % nc, l21 = k / nc;
    double s0 = 0.0;
#pragma unroll
    for (int l0 = 0; l0 < nf; ++l0) s0 += w[0][l0 * nc + j0] * rf[l21 * nf + l0];
    u1[k] = s0;
  }
  __syncwarp();
  double* u2 = rf;  // rf is free now: [l2][j1][j0]
  for (int k = lane; k < nf * nc * nc; k += 32) {  // y: (l2, j1, j0)
    const int j0 = k % nc, j1 = (k / nc) % nc, l2 = k / (nc * nc);
    double s1 = 0.0;
#pragma unroll
    for (int l1 = 0; l1 < nf; ++l1) s1 += w[1][l1 * nc + j1] * u1[(l2 * nf + l1) * nc + j0];
    u2[k] = s1;
  }
  __syncwarp();
  for (int j = lane; j < nc3; j += 32) {  // z: (j2, j1, j0)
    const int j10 = j % (nc * nc), j2 = j / (nc * nc);
    double acc = 0.0;
#pragma unroll
    for (int l2 = 0; l2 < nf; ++l2) acc += w[2][l2 * nc + j2] * u2[l2 * nc * nc + j10];
    E[e * nc3 + j] = acc;
  }
}

// Q1 -> Q1 (the h-coarsened levels, nf = nc = 2): one thread per fine
// element (a warp per element left 24 of 32 lanes idle and one element's
// gather latency per warp), same nested sums as transfer_*_kernel.
template <bool PROLONG>
__global__ void __launch_bounds__(256) transfer_q1_kernel(TransferView T, int64_t ne,
                                                          const double* __restrict__ in,
                                                          double* __restrict__ out) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  int64_t ec[3];
  const double* Wa[3];
  transfer_elem(T, e, ec, Wa);
  double w[3][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 4; ++j) w[a][j] = __ldg(Wa[a] + j);
  const int4* fm = reinterpret_cast<const int4*>(T.fmap + e * 8);
  const int4 f0 = __ldg(fm), f1 = __ldg(fm + 1);
  const int fmap[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
  if constexpr (PROLONG) {
    const int4* hm = reinterpret_cast<const int4*>(T.hmap + e * 8);
    const int4 h0 = __ldg(hm), h1 = __ldg(hm + 1);
    const int hmap[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
    double xe[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) xe[j] = __ldg(in + hmap[j]);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      const int l0 = l & 1, l1 = (l >> 1) & 1, l2 = l >> 2;
      if (!owned_local(T, ec, l0, l1, l2)) continue;
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double ab = 0.0;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          double aa = 0.0;
#pragma unroll
          for (int a = 0; a < 2; ++a) aa += w[0][l0 * 2 + a] * xe[(c * 2 + b) * 2 + a];
          ab += w[1][l1 * 2 + b] * aa;
        }
        acc += w[2][l2 * 2 + c] * ab;
      }
      out[fmap[l]] = T.add ? __dadd_rn(acc, out[fmap[l]]) : acc;
    }
  } else {
    double rf[8];
#pragma unroll
    for (int l = 0; l < 8; ++l)
      rf[l] = owned_local(T, ec, l & 1, (l >> 1) & 1, l >> 2) ? __ldg(in + fmap[l]) : 0.0;
    double E[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int j0 = j & 1, j1 = (j >> 1) & 1, j2 = j >> 2;
      double acc = 0.0;
#pragma unroll
      for (int l2 = 0; l2 < 2; ++l2) {
        double s1 = 0.0;
#pragma unroll
        for (int l1 = 0; l1 < 2; ++l1) {
          double s0 = 0.0;
#pragma unroll
          for (int l0 = 0; l0 < 2; ++l0) s0 += w[0][l0 * 2 + j0] * rf[(l2 * 2 + l1) * 2 + l0];
          s1 += w[1][l1 * 2 + j1] * s0;
        }
        acc += w[2][l2 * 2 + j2] * s1;
      }
      E[j] = acc;
    }
    double2* o = reinterpret_cast<double2*>(out + e * 8);
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = make_double2(E[2 * j], E[2 * j + 1]);
  }
}

// Narrow pairs with nf = 3 (p = 2 -> 1): one thread per fine element as for
// Q1, same nested sums.
template <bool PROLONG, int NF, int NC>
__global__ void __launch_bounds__(256) transfer_thread_kernel(TransferView T, int64_t ne,
                                                              const double* __restrict__ in,
                                                              double* __restrict__ out) {
  constexpr int nf3 = NF * NF * NF, nc3 = NC * NC * NC;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  int64_t ec[3];
  const double* Wa[3];
  transfer_elem(T, e, ec, Wa);
  double w[3][NF * NC];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < NF * NC; ++j) w[a][j] = __ldg(Wa[a] + j);
  if constexpr (PROLONG) {
    double xe[nc3];
#pragma unroll
    for (int j = 0; j < nc3; ++j) xe[j] = __ldg(in + __ldg(T.hmap + e * nc3 + j));
#pragma unroll
    for (int l = 0; l < nf3; ++l) {
      const int l0 = l % NF, l1 = (l / NF) % NF, l2 = l / (NF * NF);
      if (!owned_local(T, ec, l0, l1, l2)) continue;
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double ab = 0.0;
#pragma unroll
        for (int b = 0; b < NC; ++b) {
          double aa = 0.0;
#pragma unroll
          for (int a = 0; a < NC; ++a) aa += w[0][l0 * NC + a] * xe[(c * NC + b) * NC + a];
          ab += w[1][l1 * NC + b] * aa;
        }
        acc += w[2][l2 * NC + c] * ab;
      }
      double* d = out + __ldg(T.fmap + e * nf3 + l);
      *d = T.add ? __dadd_rn(acc, *d) : acc;
    }
  } else {
    double rf[nf3];
#pragma unroll
    for (int l = 0; l < nf3; ++l) {
      const int l0 = l % NF, l1 = (l / NF) % NF, l2 = l / (NF * NF);
      rf[l] = owned_local(T, ec, l0, l1, l2) ? __ldg(in + __ldg(T.fmap + e * nf3 + l)) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < nc3; ++j) {
      const int j0 = j % NC, j1 = (j / NC) % NC, j2 = j / (NC * NC);
      double acc = 0.0;
#pragma unroll
      for (int l2 = 0; l2 < NF; ++l2) {
        double s1 = 0.0;
#pragma unroll
        for (int l1 = 0; l1 < NF; ++l1) {
          double s0 = 0.0;
#pragma unroll
          for (int l0 = 0; l0 < NF; ++l0) s0 += w[0][l0 * NC + j0] * rf[(l2 * NF + l1) * NF + l0];
          s1 += w[1][l1 * NC + j1] * s0;
        }
        acc += w[2][l2 * NC + j2] * s1;
      }
      out[e * nc3 + j] = acc;
    }
  }
}

}  // namespace fb

using namespace fb;

extern "C" {

int fb_lor_assemble_box_rows(int p, const int64_t* counts, const double* corners_dev,
                             const double* nodes, const int* lattice_ids_dev, int kind,
                             double nu, double c, int constrain_faces, int64_t nrows,
                             int64_t ncols, fb_csr** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(p >= 1 && p <= 16, "degree must be in [1, 16]");
  FB_REQUIRE(counts && corners_dev && nodes && lattice_ids_dev, "NULL argument");
  FB_REQUIRE(kind >= FB_MASS && kind <= FB_HELMHOLTZ, "unsupported LOR kind");
  FB_REQUIRE(counts[0] >= 1 && counts[1] >= 1 && counts[2] >= 1, "cell counts must be positive");
  BoxParams P{};
  P.p = p;
  P.nx = counts[0];
  P.ny = counts[1];
  P.nz = counts[2];
  P.periodic = (constrain_faces >> 6) & 7;  // bits 6-8: periodic x, y, z
  P.Nx = P.nx * p + ((P.periodic & 1) ? 0 : 1);
  P.Ny = P.ny * p + ((P.periodic & 2) ? 0 : 1);
  P.Nz = P.nz * p + ((P.periodic & 4) ? 0 : 1);
  P.corners = corners_dev;
  P.lid = lattice_ids_dev;
  P.kind = kind;
  P.constrain = constrain_faces & 63;
  P.nu = nu;
  P.c = c;
  for (int i = 0; i <= p; ++i) P.nodes[i] = nodes[i];
  const int64_t npts = P.Nx * P.Ny * P.Nz;
  FB_REQUIRE(npts < (int64_t(1) << 31), "lattice exceeds int32 DoF ids");
  const int64_t n = nrows < 0 ? npts : nrows;
  P.nrows = n;
  std::unique_ptr<fb_csr> A(new fb_csr());
  A->nrows = n;
  A->ncols = ncols < 0 ? npts : ncols;
  A->warp_rows = 1;
  cudaStream_t st = 0;
  DevBuf<int> cnt;
  FB_TRY_CUDA(cnt.alloc(n));
  lor_box_count_kernel<<<ceil_div(npts, 256), 256, 0, st>>>(P, cnt.ptr);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(A->indptr.alloc(n + 1));
  int rc = exclusive_offsets(cnt.ptr, n, A->indptr.ptr, st);
  if (rc != FB_OK) return rc;
  cnt.reset();
  FB_TRY_CUDA(cudaMemcpy(&A->nnz, A->indptr.ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  FB_TRY_CUDA(A->indices.alloc(A->nnz));
  FB_TRY_CUDA(A->data.alloc(A->nnz));
  lor_box_fill_kernel<<<ceil_div(npts, 128), 128, 0, st>>>(P, A->indptr.ptr, A->indices.ptr,
                                                           A->data.ptr);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(cudaDeviceSynchronize());
  *out = A.release();
  return FB_OK;
}

int fb_lor_assemble_box(int p, const int64_t* counts, const double* corners_dev,
                        const double* nodes, const int* lattice_ids_dev, int kind, double nu,
                        double c, int constrain_boundary, fb_csr** out) {
  return fb_lor_assemble_box_rows(p, counts, corners_dev, nodes, lattice_ids_dev, kind, nu, c,
                                  constrain_boundary ? 63 : 0, -1, -1, out);
}

int fb_csr_info(const fb_csr* A, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
  FB_REQUIRE(A != nullptr, "matrix is NULL");
  if (nrows) *nrows = A->nrows;
  if (ncols) *ncols = A->ncols;
  if (nnz) *nnz = A->nnz;
  return FB_OK;
}

int fb_csr_download(const fb_csr* A, int64_t* indptr, int64_t* indices, double* data) {
  FB_REQUIRE(A != nullptr && indptr && indices && data, "NULL argument");
  FB_TRY_CUDA(cudaMemcpy(indptr, A->indptr.ptr, (A->nrows + 1) * sizeof(int64_t),
                         cudaMemcpyDeviceToHost));
  std::vector<int> ix(A->nnz);
  if (A->nnz) {
    FB_TRY_CUDA(cudaMemcpy(ix.data(), A->indices.ptr, A->nnz * sizeof(int), cudaMemcpyDeviceToHost));
    FB_TRY_CUDA(cudaMemcpy(data, A->data.ptr, A->nnz * sizeof(double), cudaMemcpyDeviceToHost));
  }
  for (int64_t k = 0; k < A->nnz; ++k) indices[k] = ix[k];
  return FB_OK;
}

int fb_transfer_create(const fb_restriction* fine, const fb_restriction* hmap,
                       const int64_t* counts, int nw, const double* W, const int64_t* widx,
                       fb_transfer** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  FB_REQUIRE(fine && hmap && counts && W && widx && nw >= 1, "NULL argument");
  const int64_t ne = restriction_ne(fine);
  FB_REQUIRE(restriction_ne(hmap) == ne, "fine and coarse maps must list the same elements");
  FB_REQUIRE(counts[0] * counts[1] * counts[2] == ne, "counts do not match the element count");
  const int nf3 = restriction_nloc(fine), nc3 = restriction_nloc(hmap);
  int nf = 1, nc = 1;
  while (nf * nf * nf < nf3) ++nf;
  while (nc * nc * nc < nc3) ++nc;
  FB_REQUIRE(nf * nf * nf == nf3 && nc * nc * nc == nc3, "transfers need 3D tensor maps");
  FB_REQUIRE(nf <= 9 && nc <= 5, "transfer sizes beyond p = 8 -> 4 are not supported");
  std::unique_ptr<fb_transfer> T(new fb_transfer());
  T->fine = fine;
  T->hmap = hmap;
  T->nf = nf;
  T->nc = nc;
  T->ne = ne;
  for (int a = 0; a < 3; ++a) T->counts[a] = counts[a];
  const int64_t nidx = counts[0] + counts[1] + counts[2];
  std::vector<int> wi(nidx);
  for (int64_t i = 0; i < nidx; ++i) {
    FB_REQUIRE(widx[i] >= 0 && widx[i] < nw, "weight table index out of range");
    wi[i] = int(widx[i]);
  }
  FB_TRY_CUDA(T->widx.upload(wi.data(), nidx));
  FB_TRY_CUDA(T->W.upload(W, int64_t(nw) * nf * nc));
  FB_TRY_CUDA(T->E.alloc(ne * nc3));
  *out = T.release();
  return FB_OK;
}

void fb_transfer_destroy(fb_transfer* T) { delete T; }

// constrain_matrix (lor.py:84-99) for one DoF on a device CSR: row and
// column `dof` zeroed, unit diagonal (the pure-Neumann pin, solvers.py:361-362)
__global__ void csr_pin_kernel(int64_t n, const int64_t* __restrict__ ip,
                               const int* __restrict__ ix, double* __restrict__ v, int64_t dof) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t k = ip[r]; k < ip[r + 1]; ++k)
    if (r == dof || ix[k] == dof) v[k] = (r == dof && ix[k] == dof) ? 1.0 : 0.0;
}

int fb_csr_pin(fb_csr* A, int64_t dof) {
  FB_REQUIRE(A != nullptr && dof >= 0 && dof < A->ncols, "bad pin");  // a ghost column may be pinned
  if (A->nrows == 0) return FB_OK;
  csr_pin_kernel<<<ceil_div(A->nrows, 256), 256>>>(A->nrows, A->indptr.ptr, A->indices.ptr,
                                                   A->data.ptr, dof);
  FB_CHECK_LAUNCH();
  FB_TRY_CUDA(cudaDeviceSynchronize());
  return FB_OK;
}

int fb_transfer_set_periodic(fb_transfer* T, int axes, int64_t gnx, int64_t gny, int64_t gnz) {
  FB_REQUIRE(T != nullptr && axes >= 0 && axes <= 7, "bad periodic transfer setup");
  T->periodic = axes;
  T->gcounts[0] = gnx;
  T->gcounts[1] = gny;
  T->gcounts[2] = gnz;
  return FB_OK;
}

int fb_transfer_set_origin(fb_transfer* T, int64_t x0, int64_t y0, int64_t z0) {
  FB_REQUIRE(T != nullptr && x0 >= 0 && y0 >= 0 && z0 >= 0, "bad transfer origin");
  T->origin[0] = x0;
  T->origin[1] = y0;
  T->origin[2] = z0;
  return FB_OK;
}

__global__ void index_add_kernel(int64_t n, const int* __restrict__ idx,
                                 const double* __restrict__ v, double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[idx[i]] += v[i];
}

// y[idx[i]] += v[i] (indices distinct; halo partial sums on slab cut planes)
int fb_index_add(int64_t n, const int* idx, const double* v, double* y, void* stream) {
  if (n <= 0) return FB_OK;
  index_add_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, idx, v, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

static TransferView transfer_view(const fb_transfer* T) {
  return TransferView{restriction_map(T->fine), restriction_map(T->hmap), T->W.ptr, T->widx.ptr,
                      T->counts[0], T->counts[1], T->counts[2], T->origin[0], T->origin[1],
                      T->origin[2], T->nf, T->nc, T->periodic,
                      {T->gcounts[0], T->gcounts[1], T->gcounts[2]}, 0};
}

}  // extern "C"

template <bool PROLONG, int NF, int NC>
static int launch_transfer_t(const fb_transfer* T, const double* in, double* out,
                             cudaStream_t st, int add) {
  const dim3 grid(unsigned(ceil_div(T->ne, kTE))), block(32 * kTE);
  TransferView V = transfer_view(T);
  V.add = PROLONG ? add : 0;
  if constexpr (NF == 2 && NC == 2) {
    transfer_q1_kernel<PROLONG><<<unsigned(ceil_div(T->ne, 256)), 256, 0, st>>>(V,
                                                                               T->ne, in, out);
  } else if constexpr (NF == 3) {
    transfer_thread_kernel<PROLONG, NF, NC><<<unsigned(ceil_div(T->ne, 256)), 256, 0, st>>>(
        V, T->ne, in, out);
  } else if constexpr (NF >= 4) {
    if (PROLONG)
      transfer_prolong_sf_kernel<NF, NC><<<grid, block, 0, st>>>(V, T->ne, in, out);
    else
      transfer_restrict_sf_kernel<NF, NC><<<grid, block, 0, st>>>(V, T->ne, in, out);
  } else {
    if (PROLONG)
      transfer_prolong_kernel<NF, NC><<<grid, block, 0, st>>>(V, T->ne, in, out);
    else
      transfer_restrict_kernel<NF, NC><<<grid, block, 0, st>>>(V, T->ne, in, out);
  }
  FB_CHECK_LAUNCH();
  return FB_OK;
}

// the degree ladder p -> ceil(p/2) (p = 2..8) and the Q1 h-coarsening levels
template <bool PROLONG>
static int launch_transfer(const fb_transfer* T, const double* in, double* out, cudaStream_t st,
                           int add = 0) {
  switch (T->nf * 16 + T->nc) {
    case 2 * 16 + 2: return launch_transfer_t<PROLONG, 2, 2>(T, in, out, st, add);
    case 3 * 16 + 2: return launch_transfer_t<PROLONG, 3, 2>(T, in, out, st, add);
    case 4 * 16 + 3: return launch_transfer_t<PROLONG, 4, 3>(T, in, out, st, add);
    case 5 * 16 + 3: return launch_transfer_t<PROLONG, 5, 3>(T, in, out, st, add);
    case 6 * 16 + 4: return launch_transfer_t<PROLONG, 6, 4>(T, in, out, st, add);
    case 7 * 16 + 4: return launch_transfer_t<PROLONG, 7, 4>(T, in, out, st, add);
    case 8 * 16 + 5: return launch_transfer_t<PROLONG, 8, 5>(T, in, out, st, add);
    case 9 * 16 + 5: return launch_transfer_t<PROLONG, 9, 5>(T, in, out, st, add);
    default: return launch_transfer_t<PROLONG, 0, 0>(T, in, out, st, add);
  }
}

extern "C" {

// xf (fine L-vector) = P xc: every fine DoF written once, by its owner element
int fb_transfer_prolong(const fb_transfer* T, const double* xc, double* xf, void* stream) {
  FB_REQUIRE(T != nullptr, "transfer is NULL");
  if (T->ne == 0) return FB_OK;
  return launch_transfer<true>(T, xc, xf, as_stream(stream));
}

// xf += P xc (the V-cycle's coarse-grid correction without a temporary and an
// axpby pass; the same rounding as xf = 1 * (P xc) + 1 * xf)
int fb_transfer_prolong_add(const fb_transfer* T, const double* xc, double* xf, void* stream) {
  FB_REQUIRE(T != nullptr, "transfer is NULL");
  if (T->ne == 0) return FB_OK;
  return launch_transfer<true>(T, xc, xf, as_stream(stream), 1);
}

// xc (coarse L-vector) = P^T xf, deterministic (per-element contributions,
// then the coarse map's transposed-CSR sum)
int fb_transfer_restrict(const fb_transfer* T, const double* xf, double* xc, void* stream) {
  FB_REQUIRE(T != nullptr, "transfer is NULL");
  if (T->ne == 0) return FB_OK;
  const int rc = launch_transfer<false>(T, xf, T->E.ptr, as_stream(stream));
  if (rc != FB_OK) return rc;
  return fb_restriction_scatter_add(T->hmap, T->E.ptr, xc, stream);
}

}  // extern "C"
