// Fused sum-factorized operator kernel for 3D hexahedra, sm_100a.
//
// Replaces, per element and component, the reference chain
//   FESpace.gather -> _TensorEval.values/grads -> _apply_sym (qpt scale)
//   -> _TensorEval.values_t/grads_t -> FESpace.scatter_add
// (mfop.py:187-244, 34-95, 155-166; fespace.py:282-292) with ONE kernel.
//
// Algorithm (collocated-gradient sum factorization):
//   forward   U  = (B (x) B (x) B) x_e               three 1D passes (x, y, z)
//             G_m = Dq_m U,  Dq = derivative matrix of the Lagrange basis on
//                   the rule points (exact for degree <= nq-1, so Dq B = D)
//   pointwise f_u = wdet*U, f_m = sum_n W_mn G_n     (7 factors / qpt, Helmholtz)
//   transpose V = f_u + sum_m Dq_m^T f_m;  y_e = (B^T (x) B^T (x) B^T) V
// MACs/element = 2(n^3 q + n^2 q^2 + n q^3) + 6 q^4 (stiffness/Helmholtz),
// versus 8 full 3-pass contractions in the reference.
//
// Thread mapping: "one 1D line per thread per pass".  Each pass assigns every
// thread whole lines along the contraction direction, loads the line into
// registers once and produces all outputs of that line, so a line of n
// inputs costs n shared loads for n*q DFMAs; the 1D matrices are kernel
// parameters (constant bank) and become direct DFMA operands.  Shared
// buffers use an odd x-pitch so lines along x (stride = pitch) are bank-
// conflict free for 8-byte accesses.  The z-line owner keeps U and G_z in
// registers across the pointwise stage.
//
// Memory: factors are element-blocked (ne, K, q^3) so a CTA's factor block is
// one contiguous range; thread 0 issues a bulk L2 prefetch of it at kernel
// entry so the HBM stream overlaps the gather and the forward passes.
// Output: element-interior DoFs (multiplicity 1) are written straight to y;
// element-boundary DoFs go to the shared-entry buffer S (ne, NB) and are
// summed by scatter_rows in ascending flat-E order (bitwise np.bincount).
#pragma once

#include "fb_common.cuh"

namespace fb {

constexpr int kMaxQ1 = 12;

enum SFKind { kMass = 0, kStiff = 1, kHelm = 2 };

struct SF3Params {
  const int* __restrict__ map;     // (ne, N^3) L->E map, int32
  const double* __restrict__ fac;  // (ne, K, Q^3) element-blocked factors
  const double* __restrict__ x;    // input L-vector (component)
  double* __restrict__ y;          // output L-vector (component): interior DoFs
  double* __restrict__ S;          // (ne, NB) element-boundary contributions
  int64_t ne;
  int64_t x_comp_stride;           // component strides (vdim > 1 via gridDim.y)
  int64_t S_comp_stride;
  int direct;                      // 1: interior DoFs written to y directly
  double B[kMaxQ1][kMaxQ1];        // B[q][i]  basis values at rule points
  double Dq[kMaxQ1][kMaxQ1];       // Dq[q][r] collocated derivative at rule points
};

template <int KIND>
struct KindInfo;
template <>
struct KindInfo<kMass> {
  static constexpr int NK = 1;
};
template <>
struct KindInfo<kStiff> {
  static constexpr int NK = 6;
};
template <>
struct KindInfo<kHelm> {
  static constexpr int NK = 7;
};

// rank of lattice position (k,j,i) among the element-boundary positions of
// an N^3 lattice, lexicographic order (matches the host table in fb_api.cu).
template <int N>
__device__ __forceinline__ int boundary_rank3(int k, int j, int i) {
  constexpr int mid = 4 * N - 4;  // boundary positions of an interior plane
  const int base = (k == 0) ? 0 : N * N + (k - 1) * mid;
  if (k == 0 || k == N - 1) return base + j * N + i;
  const int rb = (j == 0) ? 0 : N + (j - 1) * 2;
  if (j == 0 || j == N - 1) return base + rb + i;
  return base + rb + (i == 0 ? 0 : 1);
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* ptr, int64_t bytes) {
  uintptr_t b = reinterpret_cast<uintptr_t>(ptr) & ~uintptr_t(15);
  uintptr_t e = (reinterpret_cast<uintptr_t>(ptr) + uintptr_t(bytes) + 15) & ~uintptr_t(15);
  // one instruction moves at most a few MB; chunk at 1 MB
  while (b < e) {
    uint32_t len = uint32_t((e - b) > (1u << 20) ? (1u << 20) : (e - b));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(len) : "memory");
    b += len;
  }
}

template <int N, int Q, int KIND, int NE, int NT>
__global__ void __launch_bounds__(NT) sf3_fast_kernel(const __grid_constant__ SF3Params P) {
  constexpr int QP = Q | 1;            // odd x-pitch
  constexpr int BUF = Q * Q * QP;      // one q^3 buffer (padded)
  constexpr int NLOC = N * N * N;
  constexpr int Q2 = Q * Q;
  constexpr int Q3 = Q * Q * Q;
  constexpr int NK = KindInfo<KIND>::NK;
  constexpr int NB = (N <= 2) ? NLOC : NLOC - (N - 2) * (N - 2) * (N - 2);
  static_assert(NT >= NE * Q2, "z-line owners must be unique threads");
  static_assert(Q <= kMaxQ1, "Q too large");

  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int64_t e0 = int64_t(blockIdx.x) * NE;
  const int64_t ne = P.ne;
  const int comp = blockIdx.y;
  const double* __restrict__ x = P.x + comp * P.x_comp_stride;
  double* __restrict__ y = P.y + comp * P.x_comp_stride;
  double* __restrict__ S = P.S + comp * P.S_comp_stride;

  auto IX = [](int z, int yy, int xx) { return (z * Q + yy) * QP + xx; };

  if (tid == 0) {
    const int64_t nel = (ne - e0) < NE ? (ne - e0) : NE;
    bulk_prefetch_l2(P.fac + e0 * NK * Q3, nel * NK * Q3 * int64_t(sizeof(double)));
  }

  // ---- P0: gather x_e (L->E) ------------------------------------------
  for (int idx = tid; idx < NE * NLOC; idx += NT) {
    const int el = idx / NLOC, l = idx - el * NLOC;
    const int64_t e = e0 + el;
    double v = 0.0;
    if (e < ne) v = __ldg(x + __ldg(P.map + e * NLOC + l));
    const int i = l % N, j = (l / N) % N, k = l / (N * N);
    smem[el * 3 * BUF + IX(k, j, i)] = v;
  }
  __syncthreads();

  // ---- P1: x-lines (k,j): b0 -> b1 ------------------------------------
  for (int L = tid; L < NE * N * N; L += NT) {
    const int el = L / (N * N), r = L - el * N * N;
    const int k = r / N, j = r - k * N;
    const double* in = smem + el * 3 * BUF + IX(k, j, 0);
    double* out = smem + el * 3 * BUF + BUF + IX(k, j, 0);
    double v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = in[i];
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) acc = fma(P.B[a][i], v[i], acc);
      out[a] = acc;
    }
  }
  __syncthreads();

  // ---- P2: y-lines (k,a): b1 -> b2 ------------------------------------
  for (int L = tid; L < NE * N * Q; L += NT) {
    const int el = L / (N * Q), r = L - el * N * Q;
    const int k = r / Q, a = r - k * Q;
    const double* in = smem + el * 3 * BUF + BUF + IX(k, 0, a);
    double* out = smem + el * 3 * BUF + 2 * BUF + IX(k, 0, a);
    double v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = in[j * QP];
#pragma unroll
    for (int b = 0; b < Q; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) acc = fma(P.B[b][j], v[j], acc);
      out[b * QP] = acc;
    }
  }
  __syncthreads();

  // ---- P3: z-lines (b,a): b2 -> U (registers + b0) ----------------------
  const bool zown = tid < NE * Q2;
  const int zel = zown ? tid / Q2 : 0;
  const int zr = tid - zel * Q2;
  const int zb = zr / Q, za = zr - zb * Q;
  double* zbase = smem + zel * 3 * BUF;
  double u[Q];
  double g2[Q];
  if (zown) {
    double v[N];
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = zbase[2 * BUF + IX(k, zb, za)];
#pragma unroll
    for (int c = 0; c < Q; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc = fma(P.B[c][k], v[k], acc);
      u[c] = acc;
    }
    if (KIND != kMass) {
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < Q; ++r) acc = fma(P.Dq[c][r], u[r], acc);
        g2[c] = acc;
      }
#pragma unroll
      for (int c = 0; c < Q; ++c) zbase[IX(c, zb, za)] = u[c];
    }
  }
  if (KIND != kMass) {
    __syncthreads();
    // ---- P4: derivative lines: x (c,b) b0 -> b1; y (c,a) b0 -> b2 -------
    for (int L = tid; L < NE * 2 * Q2; L += NT) {
      const int el = L / (2 * Q2);
      int r = L - el * 2 * Q2;
      double* base = smem + el * 3 * BUF;
      if (r < Q2) {
        const int c = r / Q, b = r - c * Q;
        const double* in = base + IX(c, b, 0);
        double* out = base + BUF + IX(c, b, 0);
        double v[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) v[a] = in[a];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < Q; ++s) acc = fma(P.Dq[a][s], v[s], acc);
          out[a] = acc;
        }
      } else {
        r -= Q2;
        const int c = r / Q, a = r - c * Q;
        const double* in = base + IX(c, 0, a);
        double* out = base + 2 * BUF + IX(c, 0, a);
        double v[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) v[b] = in[b * QP];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < Q; ++s) acc = fma(P.Dq[b][s], v[s], acc);
          out[b * QP] = acc;
        }
      }
    }
  }
  __syncthreads();

  // ---- P5: quadrature-point factors (the z-line owner) -------------------
  {
    const int64_t e = e0 + zel;
    if (zown && e < ne) {
      const double* __restrict__ f = P.fac + e * NK * Q3 + zb * Q + za;
      if (KIND == kMass) {
#pragma unroll
        for (int c = 0; c < Q; ++c) u[c] = __ldg(f + c * Q2) * u[c];
        // transpose z-pass directly from registers: b0[k][zb][za], k < N
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < Q; ++c) acc = fma(P.B[c][k], u[c], acc);
          zbase[IX(k, zb, za)] = acc;
        }
      } else {
        constexpr int o = (KIND == kHelm) ? 1 : 0;
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double* fc = f + c * Q2;
          const double g0 = zbase[BUF + IX(c, zb, za)];
          const double g1 = zbase[2 * BUF + IX(c, zb, za)];
          const double w00 = __ldg(fc + (o + 0) * Q3), w01 = __ldg(fc + (o + 1) * Q3);
          const double w02 = __ldg(fc + (o + 2) * Q3), w11 = __ldg(fc + (o + 3) * Q3);
          const double w12 = __ldg(fc + (o + 4) * Q3), w22 = __ldg(fc + (o + 5) * Q3);
          const double f0 = w00 * g0 + w01 * g1 + w02 * g2[c];
          const double f1 = w01 * g0 + w11 * g1 + w12 * g2[c];
          const double f2 = w02 * g0 + w12 * g1 + w22 * g2[c];
          zbase[BUF + IX(c, zb, za)] = f0;
          zbase[2 * BUF + IX(c, zb, za)] = f1;
          g2[c] = f2;
          if (KIND == kHelm) u[c] = __ldg(fc) * u[c];
        }
        // V = f_u + Dq_z^T f_z, kept in b0
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double acc = (KIND == kHelm) ? u[c] : 0.0;
#pragma unroll
          for (int r = 0; r < Q; ++r) acc = fma(P.Dq[r][c], g2[r], acc);
          zbase[IX(c, zb, za)] = acc;
        }
      }
    }
  }
  __syncthreads();

  if (KIND != kMass) {
    // ---- P6: transposed derivative lines, in place: x (c,b) b1; y (c,a) b2
    for (int L = tid; L < NE * 2 * Q2; L += NT) {
      const int el = L / (2 * Q2);
      int r = L - el * 2 * Q2;
      double* base = smem + el * 3 * BUF;
      if (r < Q2) {
        const int c = r / Q, b = r - c * Q;
        double* io = base + BUF + IX(c, b, 0);
        double v[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) v[a] = io[a];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < Q; ++s) acc = fma(P.Dq[s][a], v[s], acc);
          io[a] = acc;
        }
      } else {
        r -= Q2;
        const int c = r / Q, a = r - c * Q;
        double* io = base + 2 * BUF + IX(c, 0, a);
        double v[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) v[b] = io[b * QP];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < Q; ++s) acc = fma(P.Dq[s][b], v[s], acc);
          io[b * QP] = acc;
        }
      }
    }
    __syncthreads();
    // ---- P7: transposed z-lines (b,a): (b0+b1+b2) -> b0[k<N]
    for (int L = tid; L < NE * Q2; L += NT) {
      const int el = L / Q2, r = L - el * Q2;
      const int b = r / Q, a = r - b * Q;
      double* base = smem + el * 3 * BUF;
      double v[Q];
#pragma unroll
      for (int c = 0; c < Q; ++c)
        v[c] = base[IX(c, b, a)] + base[BUF + IX(c, b, a)] + base[2 * BUF + IX(c, b, a)];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < Q; ++c) acc = fma(P.B[c][k], v[c], acc);
        base[IX(k, b, a)] = acc;
      }
    }
    __syncthreads();
  }

  // ---- P8: transposed y-lines (k,a): b0[k][b<Q][a] -> b1[k][j<N][a] ------
  for (int L = tid; L < NE * N * Q; L += NT) {
    const int el = L / (N * Q), r = L - el * N * Q;
    const int k = r / Q, a = r - k * Q;
    const double* in = smem + el * 3 * BUF + IX(k, 0, a);
    double* out = smem + el * 3 * BUF + BUF + IX(k, 0, a);
    double v[Q];
#pragma unroll
    for (int b = 0; b < Q; ++b) v[b] = in[b * QP];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < Q; ++b) acc = fma(P.B[b][j], v[b], acc);
      out[j * QP] = acc;
    }
  }
  __syncthreads();

  // ---- P9: transposed x-lines (k,j): b1[k][j][a<Q] -> y_e, then E->L ----
  for (int L = tid; L < NE * N * N; L += NT) {
    const int el = L / (N * N), r = L - el * N * N;
    const int k = r / N, j = r - k * N;
    const int64_t e = e0 + el;
    if (e >= ne) continue;
    const double* in = smem + el * 3 * BUF + BUF + IX(k, j, 0);
    double v[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) v[a] = in[a];
    const bool edge_line = (k == 0 || k == N - 1 || j == 0 || j == N - 1);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < Q; ++a) acc = fma(P.B[a][i], v[a], acc);
      const int l = (k * N + j) * N + i;
      if (P.direct) {
        if (!edge_line && i > 0 && i < N - 1) {
          // bincount semantics: 0.0 + contribution
          y[__ldg(P.map + e * NLOC + l)] = 0.0 + acc;
        } else {
          S[e * NB + boundary_rank3<N>(k, j, i)] = acc;
        }
      } else {
        S[e * NLOC + l] = acc;
      }
    }
  }
}

}  // namespace fb
