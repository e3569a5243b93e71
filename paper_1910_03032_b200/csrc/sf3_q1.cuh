// Trilinear (p = 1, 3-point Gauss) operator kernel: one thread per element.
//
// At p = 1 an element has 8 DoFs and 27 quadrature points; the factor stream
// (7 x 27 doubles = 1.5 KB per element for Helmholtz) is ~95 % of the bytes.
// The line-per-thread scheme of sf3_fast.cuh gives each thread 2-3-point lines
// and drowns in index arithmetic here, so this kernel keeps the whole element
// on chip: U at the 27 points and the transposed accumulator V live in
// thread-private shared-memory columns ([q][thread], conflict free), the
// gradients and factors of one 3-point row live in registers.  Factors use an
// element-interleaved, point-major layout (groups of 32 elements,
// [group][27][K][32]) so every factor load of a warp is one fully used
// 256-byte segment and one 3-point row of a warp is one contiguous
// 3*K*256-byte run, streamed into L2 two rows ahead of its use (a whole-block
// prefetch would keep ~110 MB in flight and get evicted before use); map and
// slot rows are read as 16-byte vectors.  All 8 outputs of an element lie on the element boundary,
// so they go to their transposed-map slots (scatter_rows sums them in
// np.bincount order).  Same arithmetic as the general path: U = B(x)B(x)B x,
// G_m = Dq_m U, pointwise factors, V = f_u + sum Dq_m^T f_m, y = B^T(x)B^T(x)B^T V
// (mfop.py:56-95, 155-166, 225-244).
#pragma once

#include "fb_common.cuh"
#include "sf3_fast.cuh"

namespace fb {

struct Q1Params {
  const int* __restrict__ map;     // (ne, 8) int32
  const int* __restrict__ spos;    // (ne, 8) slots
  const double* __restrict__ fac;  // [ne/32][K][27][32]
  const double* __restrict__ x;
  double* __restrict__ S;
  int64_t ne;
  int64_t x_comp_stride, S_comp_stride;
  int vdim;
  double B[3][2];
  double Dq[3][3];
};

constexpr int kQ1Threads = 128;
constexpr int kQ1Smem = 2 * 27 * kQ1Threads * 8;  // 55 KB (dynamic)

template <int KIND>
__global__ void __launch_bounds__(kQ1Threads, 4) sf3_q1_kernel(const __grid_constant__ Q1Params P) {
  constexpr int NK = KindInfo<KIND>::NK;
  constexpr int T = kQ1Threads;
  // thread-private columns: su[q][tid] = U at point q, sv[q][tid] = V
  extern __shared__ double q1_smem[];
  double* su = q1_smem;
  double* sv = q1_smem + 27 * T;
  const int tid = threadIdx.x;
  const int64_t e = int64_t(blockIdx.x) * T + tid;
  if (e >= P.ne) return;  // no block-level barriers below
  const int lane = int(e & 31);
  const double* __restrict__ fblk = P.fac + (e >> 5) * (int64_t(NK) * 27 * 32);
  const double* __restrict__ f = fblk + lane;
  constexpr int64_t kRowBytes = int64_t(3) * NK * 32 * 8;  // one 3-point row of the warp
  // lane 0 streams rows 0 and 1 of the warp's factor block into L2 now, and
  // row cb+2 while row cb is computed
  const uint64_t fpol = l2_evict_first_policy();  // factors are read once: keep x resident
  if (lane == 0) bulk_prefetch_l2_hint(fblk, 2 * kRowBytes, fpol);
  double* U = su + tid;
  double* V = sv + tid;
  int m[8], sl[8];
  {
    const int4 a = __ldg(reinterpret_cast<const int4*>(P.map + e * 8));
    const int4 b = __ldg(reinterpret_cast<const int4*>(P.map + e * 8 + 4));
    m[0] = a.x; m[1] = a.y; m[2] = a.z; m[3] = a.w; m[4] = b.x; m[5] = b.y; m[6] = b.z; m[7] = b.w;
    const int4 c = __ldg(reinterpret_cast<const int4*>(P.spos + e * 8));
    const int4 d = __ldg(reinterpret_cast<const int4*>(P.spos + e * 8 + 4));
    sl[0] = c.x; sl[1] = c.y; sl[2] = c.z; sl[3] = c.w; sl[4] = d.x; sl[5] = d.y; sl[6] = d.z; sl[7] = d.w;
  }
  for (int comp = 0; comp < P.vdim; ++comp) {
    const double* __restrict__ x = P.x + comp * P.x_comp_stride;
    double* __restrict__ S = P.S + comp * P.S_comp_stride;
    {
      double xe[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) xe[l] = __ldg(x + m[l]);
      double t1[2][2][3];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int a = 0; a < 3; ++a)
            t1[k][j][a] = fma(P.B[a][0], xe[(k * 2 + j) * 2], P.B[a][1] * xe[(k * 2 + j) * 2 + 1]);
      double t2[2][3][3];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int a = 0; a < 3; ++a) t2[k][b][a] = fma(P.B[b][0], t1[k][0][a], P.B[b][1] * t1[k][1][a]);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int q = (c * 3 + b) * 3 + a;
            U[q * T] = fma(P.B[c][0], t2[0][b][a], P.B[c][1] * t2[1][b][a]);
            V[q * T] = 0.0;
          }
    }
    // pointwise stage, one 3-point x-row (c, b) at a time
#pragma unroll 1
    for (int cb = 0; cb < 9; ++cb) {
      const int c = cb / 3, b = cb - 3 * c;
      if (lane == 0 && comp == 0 && cb + 2 < 9)
        bulk_prefetch_l2_hint(fblk + (cb + 2) * 3 * NK * 32, kRowBytes, fpol);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int q = cb * 3 + a;
        const double* fq = f + q * NK * 32;
        if (KIND == kMass) {
          V[q * T] = ld_evict_first(fq, fpol) * U[q * T];
          continue;
        }
        constexpr int o = (KIND == kHelm) ? 1 : 0;
        const double w00 = ld_evict_first(fq + (o + 0) * 32, fpol);
        const double w01 = ld_evict_first(fq + (o + 1) * 32, fpol);
        const double w02 = ld_evict_first(fq + (o + 2) * 32, fpol);
        const double w11 = ld_evict_first(fq + (o + 3) * 32, fpol);
        const double w12 = ld_evict_first(fq + (o + 4) * 32, fpol);
        const double w22 = ld_evict_first(fq + (o + 5) * 32, fpol);
        const double wm = (KIND == kHelm) ? ld_evict_first(fq, fpol) : 0.0;
        double g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          g0 = fma(P.Dq[a][s], U[(cb * 3 + s) * T], g0);
          g1 = fma(P.Dq[b][s], U[((c * 3 + s) * 3 + a) * T], g1);
          g2 = fma(P.Dq[c][s], U[((s * 3 + b) * 3 + a) * T], g2);
        }
        const double f0 = w00 * g0 + w01 * g1 + w02 * g2;
        const double f1 = w01 * g0 + w11 * g1 + w12 * g2;
        const double f2 = w02 * g0 + w12 * g1 + w22 * g2;
        if (KIND == kHelm) V[q * T] += wm * U[q * T];
        // transposed derivatives along the three lines through q
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          V[(cb * 3 + s) * T] = fma(P.Dq[a][s], f0, V[(cb * 3 + s) * T]);
          V[((c * 3 + s) * 3 + a) * T] = fma(P.Dq[b][s], f1, V[((c * 3 + s) * 3 + a) * T]);
          V[((s * 3 + b) * 3 + a) * T] = fma(P.Dq[c][s], f2, V[((s * 3 + b) * 3 + a) * T]);
        }
      }
    }
    // transpose passes: z, y, x
    double t2[2][3][3];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          t2[k][b][a] = fma(P.B[0][k], V[(b * 3 + a) * T],
                            fma(P.B[1][k], V[((3 + b) * 3 + a) * T],
                                P.B[2][k] * V[((6 + b) * 3 + a) * T]));
    double t1[2][2][3];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          t1[k][j][a] = fma(P.B[0][j], t2[k][0][a], fma(P.B[1][j], t2[k][1][a], P.B[2][j] * t2[k][2][a]));
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double v = fma(P.B[0][i], t1[k][j][0], fma(P.B[1][i], t1[k][j][1], P.B[2][i] * t1[k][j][2]));
          S[sl[(k * 2 + j) * 2 + i]] = v;
        }
  }
}

}  // namespace fb
