// Fused mixed-degree operator kernel for 3D hexahedra:
// the weak gradient G (pressure -> velocity), its transpose G^T and the weak
// divergence D (velocity -> pressure) of the Stokes / projection solvers.
//
// Replaces, per element, the reference chains (mfop.py:247-319)
//   G  : gather q -> grads_p -> f_c = sum_m grad[c,m] g_m -> values_t_v -> scatter (3 comps)
//   G^T: gather v_c -> values_v -> g_m = sum_c grad[c,m] vals_c -> grads_t_p -> scatter
//   D  : gather u_c -> grads_v -> f = sum_c sum_m grad[c,m] g_m^c -> values_t_p -> scatter
// with ONE kernel per operator.  grad[c,m] = wdet * Jinv[m,c] (mfop.py:145-152),
// stored element-blocked (ne, 9, q^3).
//
// Same collocated scheme as sf3_fast.cuh: values at the Gauss points by three
// 1D interpolation passes (B_v or B_p, even-odd form), gradients by the
// collocated derivative Dq on the Gauss points (Dq B = D exactly for either
// space, since q = p_v + 2 points resolve both), transposes likewise.  One
// element per CTA iteration, persistent grid-stride loop; the element's
// result is stored by the coalesced output stage into the output space's
// transposed-map slots / interior DoFs, then the class-major slot sum
// (scatter_slots_kernel) finishes the E->L sum in np.bincount order.
#pragma once

#include "sf3_fast.cuh"

namespace fb {

enum MixedKind { kMxGrad = 0, kMxGradT = 1, kMxDiv = 2 };

struct SF3MParams {
  const int* __restrict__ map_in;    // (ne, NIN^3) input-space L->E map
  const int* __restrict__ map_out;   // (ne, NOUT^3) output-space L->E map
  const int* __restrict__ spos_out;  // (ne, nbp_out) slots of the output space
  const double* __restrict__ fac;    // (ne, fstride): grad[c,m] blocks of q^3
  const double* __restrict__ x;
  double* __restrict__ y;
  double* __restrict__ S;
  int64_t ne, fstride;
  int64_t in_comp_stride, out_comp_stride, S_comp_stride;
  int nbp_out;
  EOMat eBv, eBvt, eBp, eBpt, eD, eDt;
};

template <int NV, int NP, int Q>
struct SF3MShape {
  static constexpr int QP = SF3Pitch<Q>::QP;
  static constexpr int YP = SF3Pitch<Q>::YP;
  static constexpr int BUF = Q * YP + SF3Pitch<Q>::PAD;  // one q^3 work buffer
  static constexpr int NBUF = 7;
  static constexpr int NMAX = NV > NP ? NV : NP;
  static constexpr int SMEM = (NBUF * BUF + 2 * round_up(NMAX * NMAX * NMAX, 8)) * 8;  // bytes
};

// Lines of one direction: D0 x D1 lines of NI inputs -> NO outputs (or in
// place); in/out addresses u*s0 + w*s1 + t*st for line (u, w), position t.
template <int NI, int NO, int S, int D0, int D1, int NT>
__device__ __forceinline__ void mx_lines(const EOMat& M, const double* in, int is0, int is1,
                                         int ist, double* out, int os0, int os1, int ost) {
#pragma unroll 1
  for (int L = threadIdx.x; L < D0 * D1; L += NT) {
    const int u = L / D1, w = L - u * D1;
    const double* pi = in + u * is0 + w * is1;
    double v[1][NI], r[1][NO];
#pragma unroll
    for (int t = 0; t < NI; ++t) v[0][t] = pi[t * ist];
    eo_lines<NO, NI, S, 1>(M, v, r);
    double* po = out + u * os0 + w * os1;
#pragma unroll
    for (int t = 0; t < NO; ++t) po[t * ost] = r[0][t];
  }
}

// values at the Gauss points: x_e (NI^3, dense) -> U (Q^3 in a work buffer)
template <int NI, int Q, int NT>
__device__ __forceinline__ void mx_interp(const EOMat& M, const double* xe, double* t1, double* t2,
                                          double* U) {
  constexpr int QP = SF3Pitch<Q>::QP, YP = SF3Pitch<Q>::YP;
  // x-lines (k, j): xe[k][j][i] -> t1[k][j][a]
  mx_lines<NI, Q, 1, NI, NI, NT>(M, xe, NI * NI, NI, 1, t1, YP, QP, 1);
  __syncthreads();
  // y-lines (k, a): t1[k][j][a] -> t2[k][b][a]
  mx_lines<NI, Q, 1, NI, Q, NT>(M, t1, YP, 1, QP, t2, YP, 1, QP);
  __syncthreads();
  // z-lines (b, a): t2[k][b][a] -> U[c][b][a]
  mx_lines<NI, Q, 1, Q, Q, NT>(M, t2, QP, 1, YP, U, QP, 1, YP);
  __syncthreads();
}

// V (Q^3) -> element result (NO^3 dense) by B^T in z, y, x
template <int Q, int NO, int NT>
__device__ __forceinline__ void mx_interp_t(const EOMat& Mt, const double* V, double* t1, double* t2,
                                            double* out) {
  constexpr int QP = SF3Pitch<Q>::QP, YP = SF3Pitch<Q>::YP;
  mx_lines<Q, NO, 1, Q, Q, NT>(Mt, V, QP, 1, YP, t1, QP, 1, YP);  // z: (b,a) -> t1[k][b][a]
  __syncthreads();
  mx_lines<Q, NO, 1, NO, Q, NT>(Mt, t1, YP, 1, QP, t2, YP, 1, QP);  // y: (k,a) -> t2[k][j][a]
  __syncthreads();
  mx_lines<Q, NO, 1, NO, NO, NT>(Mt, t2, YP, QP, 1, out, NO * NO, NO, 1);  // x: (k,j) -> out
  __syncthreads();
}

// collocated gradient: U -> G0 (x), G1 (y), G2 (z)
template <int Q, int NT>
__device__ __forceinline__ void mx_grad(const EOMat& D, const double* U, double* G0, double* G1,
                                        double* G2) {
  constexpr int QP = SF3Pitch<Q>::QP, YP = SF3Pitch<Q>::YP;
  mx_lines<Q, Q, -1, Q, Q, NT>(D, U, YP, QP, 1, G0, YP, QP, 1);
  mx_lines<Q, Q, -1, Q, Q, NT>(D, U, YP, 1, QP, G1, YP, 1, QP);
  mx_lines<Q, Q, -1, Q, Q, NT>(D, U, QP, 1, YP, G2, QP, 1, YP);
  __syncthreads();
}

__device__ __forceinline__ double ld_fac(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int NV, int NP, int Q, int KIND, int NT>
__global__ void __launch_bounds__(NT) sf3_mixed_kernel(const __grid_constant__ SF3MParams P) {
  using Sh = SF3MShape<NV, NP, Q>;
  constexpr int QP = Sh::QP, YP = Sh::YP, BUF = Sh::BUF, Q3 = Q * Q * Q;
  constexpr int NIN = (KIND == kMxGrad) ? NP : NV;
  constexpr int NOUT = (KIND == kMxGrad) ? NV : NP;
  constexpr int NINL = NIN * NIN * NIN, NOUTL = NOUT * NOUT * NOUT;
  extern __shared__ __align__(16) double msm[];
  double* W[Sh::NBUF];
#pragma unroll
  for (int b = 0; b < Sh::NBUF; ++b) W[b] = msm + b * BUF;
  double* xe = msm + Sh::NBUF * BUF;                        // gathered input (dense)
  double* oe = xe + round_up(Sh::NMAX * Sh::NMAX * Sh::NMAX, 8);  // element result (dense)
  const int tid = threadIdx.x;
  auto pt_index = [](int qp) {
    const int c = qp / (Q * Q), r = qp - c * Q * Q;
    const int b = r / Q, a = r - b * Q;
    return c * YP + b * QP + a;
  };
  // element result -> interior DoFs (direct) / transposed-map slots; the
  // boundary rank of a local DoF follows its lattice position
  auto store = [&](int64_t e, double* y, double* S) {
#pragma unroll 2
    for (int l = tid; l < NOUTL; l += NT) {
      const int i = l % NOUT, j = (l / NOUT) % NOUT, k = l / (NOUT * NOUT);
      const bool inner =
          i > 0 && i < NOUT - 1 && j > 0 && j < NOUT - 1 && k > 0 && k < NOUT - 1;
      const double v = oe[l];
      if (inner) y[__ldg(P.map_out + e * NOUTL + l)] = 0.0 + v;  // bincount: 0.0 + contribution
      else S[__ldg(P.spos_out + e * P.nbp_out + boundary_rank3<NOUT>(k, j, i))] = v;
    }
  };
  auto gather = [&](int64_t e, const double* x) {
#pragma unroll 4
    for (int l = tid; l < NINL; l += NT) xe[l] = __ldg(x + __ldg(P.map_in + e * NINL + l));
    __syncthreads();
  };

#pragma unroll 1
  for (int64_t e = blockIdx.x; e < P.ne; e += gridDim.x) {
    const double* fe = P.fac + e * P.fstride;
    if constexpr (KIND == kMxGrad) {
      // q -> U -> (G0, G1, G2) -> per component f_c -> B_v^T -> store
      gather(e, P.x);
      mx_interp<NP, Q, NT>(P.eBp, xe, W[0], W[1], W[2]);
      mx_grad<Q, NT>(P.eD, W[2], W[3], W[4], W[5]);
#pragma unroll 1
      for (int c = 0; c < 3; ++c) {
        for (int qp = tid; qp < Q3; qp += NT) {
          const int ix = pt_index(qp);
          const double* f = fe + (c * 3) * Q3 + qp;
          W[2][ix] = ld_fac(f) * W[3][ix] + ld_fac(f + Q3) * W[4][ix] + ld_fac(f + 2 * Q3) * W[5][ix];
        }
        __syncthreads();
        mx_interp_t<Q, NV, NT>(P.eBvt, W[2], W[0], W[1], oe);
        store(e, P.y + c * P.out_comp_stride, P.S + c * P.S_comp_stride);
        __syncthreads();
      }
    } else if constexpr (KIND == kMxGradT) {
      // v_c -> values -> g_m += grad[c,m] vals_c -> sum_m Dq_m^T g_m -> B_p^T
#pragma unroll 1
      for (int c = 0; c < 3; ++c) {
        gather(e, P.x + c * P.in_comp_stride);
        mx_interp<NV, Q, NT>(P.eBv, xe, W[0], W[1], W[2]);
        for (int qp = tid; qp < Q3; qp += NT) {
          const int ix = pt_index(qp);
          const double u = W[2][ix];
          const double* f = fe + (c * 3) * Q3 + qp;
          const double t0 = ld_fac(f) * u, t1 = ld_fac(f + Q3) * u, t2 = ld_fac(f + 2 * Q3) * u;
          if (c == 0) {
            W[3][ix] = t0;
            W[4][ix] = t1;
            W[5][ix] = t2;
          } else {
            W[3][ix] = W[3][ix] + t0;
            W[4][ix] = W[4][ix] + t1;
            W[5][ix] = W[5][ix] + t2;
          }
        }
        __syncthreads();
      }
      // transposed derivatives in place: x-lines of g0, y-lines of g1, z-lines of g2
      mx_lines<Q, Q, -1, Q, Q, NT>(P.eDt, W[3], YP, QP, 1, W[3], YP, QP, 1);
      mx_lines<Q, Q, -1, Q, Q, NT>(P.eDt, W[4], YP, 1, QP, W[4], YP, 1, QP);
      mx_lines<Q, Q, -1, Q, Q, NT>(P.eDt, W[5], QP, 1, YP, W[5], QP, 1, YP);
      __syncthreads();
      for (int qp = tid; qp < Q3; qp += NT) {
        const int ix = pt_index(qp);
        W[2][ix] = (W[3][ix] + W[4][ix]) + W[5][ix];
      }
      __syncthreads();
      mx_interp_t<Q, NP, NT>(P.eBpt, W[2], W[0], W[1], oe);
      store(e, P.y, P.S);
      __syncthreads();
    } else {
      // u_c -> U -> (G0, G1, G2) -> acc += sum_m grad[c,m] G_m -> B_p^T
#pragma unroll 1
      for (int c = 0; c < 3; ++c) {
        gather(e, P.x + c * P.in_comp_stride);
        mx_interp<NV, Q, NT>(P.eBv, xe, W[0], W[1], W[2]);
        mx_grad<Q, NT>(P.eD, W[2], W[3], W[4], W[5]);
        for (int qp = tid; qp < Q3; qp += NT) {
          const int ix = pt_index(qp);
          const double* f = fe + (c * 3) * Q3 + qp;
          const double s = ld_fac(f) * W[3][ix] + ld_fac(f + Q3) * W[4][ix] +
                           ld_fac(f + 2 * Q3) * W[5][ix];
          W[6][ix] = (c == 0) ? s : W[6][ix] + s;
        }
        __syncthreads();
      }
      mx_interp_t<Q, NP, NT>(P.eBpt, W[6], W[0], W[2], oe);
      store(e, P.y, P.S);
      __syncthreads();
    }
  }
}

}  // namespace fb
