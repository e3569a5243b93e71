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
// Data movement (B200):
//   * at CTA entry one thread arms an mbarrier and issues a bulk async copy
//     (cp.async.bulk, the TMA 1D engine) of the CTA's L->E map block into
//     shared memory, plus a bulk L2 prefetch (cp.async.bulk.prefetch.L2) of
//     its element-blocked factor block (ne, K, q^3): the factor stream runs
//     HBM -> L2 while the CTA gathers and runs the forward passes.
//   * as soon as the map lands, every thread issues cp.async (LDGSTS) 8-byte
//     gathers x[map[l]] straight into the work buffer -- no register round
//     trip, all loads in flight at once.
//   * the pointwise stage reads the factors point-parallel from L2 (7 independent
//     loads per point); keeping them out of shared memory lets 3-6 CTAs share
//     an SM, which is what hides the shared-memory and FMA latencies.
//   * vector operators (vdim > 1) loop over components inside the CTA, so the
//     factors are read from HBM once per element, not once per component.
//
// Compute mapping: "one 1D line per thread per pass".  Each pass assigns
// threads whole lines along the contraction direction, loads the line into
// registers once and produces all outputs of that line (n loads for n*q
// DFMAs); the 1D matrices are kernel parameters.  The z-line owner keeps U
// and G_z in registers across the pointwise stage.
//
// Output: element-interior DoFs (multiplicity 1) are written straight to y;
// element-boundary DoFs go to the shared-entry buffer S (ne, NB) and are
// summed by scatter_rows in ascending flat-E order (bitwise np.bincount).
#pragma once

#include "fb_common.cuh"

namespace fb {

constexpr int kMaxQ1 = 12;

enum SFKind { kMass = 0, kStiff = 1, kHelm = 2 };

struct SF3Params {
  const int* __restrict__ map;     // (ne, NLOCP) L->E map, int32, padded per element
  const double* __restrict__ fac;  // (ne, FACP) element-blocked factors (K, q^3), padded
  const double* __restrict__ x;    // input L-vector (all components)
  double* __restrict__ y;          // output L-vector: interior DoFs
  double* __restrict__ S;          // (vdim, ne, NB) element-boundary contributions
  int64_t ne;
  int64_t x_comp_stride;           // component stride of x / y
  int64_t S_comp_stride;
  int vdim;
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

__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }

// Compile-time geometry of one instantiation.
template <int N, int Q, int KIND, int NE>
struct SF3Shape {
  static constexpr int QP = Q | 1;        // odd x-pitch
  static constexpr int BUF = Q * Q * QP;  // one q^3 buffer (padded)
  static constexpr int NLOC = N * N * N;
  static constexpr int NLOCP = round_up(NLOC, 4);
  static constexpr int Q2 = Q * Q;
  static constexpr int Q3 = Q * Q * Q;
  static constexpr int NK = KindInfo<KIND>::NK;
  static constexpr int FACP = round_up(NK * Q3, 2);
  static constexpr int NB = (N <= 2) ? NLOC : NLOC - (N - 2) * (N - 2) * (N - 2);
  // shared-memory plan (bytes): [mbarrier | map | work]
  static constexpr int OFF_MAP = 16;
  static constexpr int OFF_WORK = round_up(OFF_MAP + NE * NLOCP * 4, 16);
  static constexpr int NBUF = (KIND == kMass) ? 3 : 4;  // work buffers per element
  static constexpr int SMEM = OFF_WORK + NE * NBUF * BUF * 8;
};

// rank of lattice position (k,j,i) among the element-boundary positions of
// an N^3 lattice, lexicographic order (matches the host table in fb_ops.cu).
template <int N>
__device__ __forceinline__ int boundary_rank3(int k, int j, int i) {
  constexpr int mid = 4 * N - 4;  // boundary positions of an interior plane
  const int base = (k == 0) ? 0 : N * N + (k - 1) * mid;
  if (k == 0 || k == N - 1) return base + j * N + i;
  const int rb = (j == 0) ? 0 : N + (j - 1) * 2;
  if (j == 0 || j == N - 1) return base + rb + i;
  return base + rb + (i == 0 ? 0 : 1);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// 1D bulk async copy global -> shared (TMA engine), completion on `bar`.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* ptr, int64_t bytes) {
  uintptr_t b = reinterpret_cast<uintptr_t>(ptr) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(ptr) + uintptr_t(bytes) + 15) & ~uintptr_t(15);
  while (b < e) {
    const uint32_t len = uint32_t((e - b) > (1u << 20) ? (1u << 20) : (e - b));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(len) : "memory");
    b += len;
  }
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

template <int N, int Q, int KIND, int NE, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) sf3_fast_kernel(const __grid_constant__ SF3Params P) {
  using Sh = SF3Shape<N, Q, KIND, NE>;
  constexpr int QP = Sh::QP, BUF = Sh::BUF, NLOC = Sh::NLOC, NLOCP = Sh::NLOCP;
  constexpr int Q2 = Sh::Q2, Q3 = Sh::Q3, FACP = Sh::FACP, NB = Sh::NB, NBUF = Sh::NBUF;
  static_assert(Q <= kMaxQ1, "Q too large");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  const int* smap = reinterpret_cast<const int*>(smem_raw + Sh::OFF_MAP);
  double* smem = reinterpret_cast<double*>(smem_raw + Sh::OFF_WORK);

  const int tid = threadIdx.x;
  const int64_t e0 = int64_t(blockIdx.x) * NE;
  const int64_t ne = P.ne;
  const int nel = (ne - e0) < NE ? int(ne - e0) : NE;
  const uint32_t bar_map = smem_u32(&bars[0]);

  if (tid == 0) {
    mbar_init(bar_map, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t mbytes = uint32_t(nel) * NLOCP * 4u;
    mbar_expect_tx(bar_map, mbytes);
    bulk_g2s(smem_u32(smap), P.map + e0 * NLOCP, mbytes, bar_map);
    // factors stream HBM -> L2 while the CTA gathers and runs the forward passes
    bulk_prefetch_l2(P.fac + e0 * FACP, int64_t(nel) * FACP * 8);
  }

  auto IX = [](int z, int yy, int xx) { return (z * Q + yy) * QP + xx; };

  mbar_wait(bar_map, 0);

#pragma unroll 1
  for (int comp = 0; comp < P.vdim; ++comp) {
    const double* __restrict__ x = P.x + comp * P.x_comp_stride;
    double* __restrict__ y = P.y + comp * P.x_comp_stride;
    double* __restrict__ S = P.S + comp * P.S_comp_stride;
    if (comp > 0) __syncthreads();  // previous component done with b0

    // ---- P0: gather x_e (L->E) via cp.async -------------------------------
#pragma unroll 4
    for (int idx = tid; idx < nel * NLOC; idx += NT) {
      const int el = idx / NLOC, l = idx - el * NLOC;
      const int i = l % N, j = (l / N) % N, k = l / (N * N);
      cp_async8(smem_u32(smem + el * NBUF * BUF + IX(k, j, i)), x + smap[el * NLOCP + l]);
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- P1: x-lines (k,j): b0 -> b1 --------------------------------------
    #pragma unroll 1
    for (int L = tid; L < NE * N * N; L += NT) {
      const int el = L / (N * N), r = L - el * N * N;
      const int k = r / N, j = r - k * N;
      const double* in = smem + el * NBUF * BUF + IX(k, j, 0);
      double* out = smem + el * NBUF * BUF + BUF + IX(k, j, 0);
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

    // ---- P2: y-lines (k,a): b1 -> b2 --------------------------------------
    #pragma unroll 1
    for (int L = tid; L < NE * N * Q; L += NT) {
      const int el = L / (N * Q), r = L - el * N * Q;
      const int k = r / Q, a = r - k * Q;
      const double* in = smem + el * NBUF * BUF + BUF + IX(k, 0, a);
      double* out = smem + el * NBUF * BUF + 2 * BUF + IX(k, 0, a);
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

    // ---- P3: z-lines (b,a): b2 -> U (b0) and Gz = Dq_z U (b3) --------------
#pragma unroll 1
    for (int L = tid; L < NE * Q2; L += NT) {
      const int el = L / Q2, r = L - el * Q2;
      const int b = r / Q, a = r - b * Q;
      double* base = smem + el * NBUF * BUF;
      double v[N];
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = base[2 * BUF + IX(k, b, a)];
      double u[Q];
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) acc = fma(P.B[c][k], v[k], acc);
        u[c] = acc;
      }
      if (KIND == kMass) {
        // mass: scale by wdet and contract back along z right here
        const double* __restrict__ f = P.fac + (e0 + el) * FACP + b * Q + a;
#pragma unroll
        for (int c = 0; c < Q; ++c) u[c] = __ldg(f + c * Q2) * u[c];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < Q; ++c) acc = fma(P.B[c][k], u[c], acc);
          base[IX(k, b, a)] = acc;
        }
      } else {
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < Q; ++s) acc = fma(P.Dq[c][s], u[s], acc);
          base[3 * BUF + IX(c, b, a)] = acc;
          base[IX(c, b, a)] = u[c];
        }
      }
    }
    __syncthreads();

    if (KIND != kMass) {
      // ---- P4: derivative lines: x (c,b) b0 -> b1; y (c,a) b0 -> b2 -------
#pragma unroll 1
      for (int L = tid; L < NE * 2 * Q2; L += NT) {
        const int el = L / (2 * Q2);
        int r = L - el * 2 * Q2;
        double* base = smem + el * NBUF * BUF;
        const bool xl = r < Q2;
        if (!xl) r -= Q2;
        const int c = r / Q, t = r - c * Q;
        // x-line (c, b=t) stride 1;  y-line (c, a=t) stride QP
        const int st = xl ? 1 : QP;
        const double* in = base + (xl ? IX(c, t, 0) : IX(c, 0, t));
        double* out = base + (xl ? BUF : 2 * BUF) + (xl ? IX(c, t, 0) : IX(c, 0, t));
        double v[Q];
#pragma unroll
        for (int s = 0; s < Q; ++s) v[s] = in[s * st];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < Q; ++s) acc = fma(P.Dq[a][s], v[s], acc);
          out[a * st] = acc;
        }
      }
      __syncthreads();

      // ---- P5: pointwise quadrature-point factors (read from L2) -------------
      //   b0: U -> f_u,  b1: G0 -> f0,  b2: G1 -> f1,  b3: G2 -> f2
      constexpr int o = (KIND == kHelm) ? 1 : 0;
#pragma unroll 2
      for (int idx = tid; idx < NE * Q3; idx += NT) {
        const int el = idx / Q3, qp = idx - el * Q3;
        const int c = qp / Q2, ba = qp - c * Q2;
        const int b = ba / Q, a = ba - b * Q;
        double* base = smem + el * NBUF * BUF + IX(c, b, a);
        const double* __restrict__ f = P.fac + (e0 + el) * FACP + qp;
        const double w00 = __ldg(f + (o + 0) * Q3), w01 = __ldg(f + (o + 1) * Q3);
        const double w02 = __ldg(f + (o + 2) * Q3), w11 = __ldg(f + (o + 3) * Q3);
        const double w12 = __ldg(f + (o + 4) * Q3), w22 = __ldg(f + (o + 5) * Q3);
        const double wm = (KIND == kHelm) ? __ldg(f) : 0.0;
        const double g0 = base[BUF], g1 = base[2 * BUF], g2 = base[3 * BUF];
        base[BUF] = w00 * g0 + w01 * g1 + w02 * g2;
        base[2 * BUF] = w01 * g0 + w11 * g1 + w12 * g2;
        base[3 * BUF] = w02 * g0 + w12 * g1 + w22 * g2;
        if (KIND == kHelm) base[0] = wm * base[0];
      }
      __syncthreads();

      // ---- P6: transposed derivative lines, in place: x b1, y b2, z b3 -----
#pragma unroll 1
      for (int L = tid; L < NE * 3 * Q2; L += NT) {
        const int el = L / (3 * Q2);
        int r = L - el * 3 * Q2;
        const int dir = r / Q2;
        r -= dir * Q2;
        const int c = r / Q, t = r - c * Q;
        double* base = smem + el * NBUF * BUF;
        // x: line (c, b=t); y: line (c, a=t); z: line (b=c, a=t)
        const int st = dir == 0 ? 1 : (dir == 1 ? QP : Q * QP);
        double* io = base + (dir + 1) * BUF +
                     (dir == 0 ? IX(c, t, 0) : (dir == 1 ? IX(c, 0, t) : IX(0, c, t)));
        double v[Q];
#pragma unroll
        for (int s = 0; s < Q; ++s) v[s] = io[s * st];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < Q; ++s) acc = fma(P.Dq[s][a], v[s], acc);
          io[a * st] = acc;
        }
      }
      __syncthreads();

      // ---- P7: transposed z-lines (b,a): (b0+b1+b2+b3) -> b0[k<N] ---------
#pragma unroll 1
      for (int L = tid; L < NE * Q2; L += NT) {
        const int el = L / Q2, r = L - el * Q2;
        const int b = r / Q, a = r - b * Q;
        double* base = smem + el * NBUF * BUF;
        double v[Q];
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const int ix = IX(c, b, a);
          const double fu = (KIND == kHelm) ? base[ix] : 0.0;  // stiffness: no mass term
          v[c] = ((fu + base[BUF + ix]) + base[2 * BUF + ix]) + base[3 * BUF + ix];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < Q; ++c) acc = fma(P.B[c][k], v[c], acc);
          base[IX(k, b, a)] = acc;
        }
      }
    }
    __syncthreads();

    // ---- P8: transposed y-lines (k,a): b0[k][b<Q][a] -> b1[k][j<N][a] ------
    #pragma unroll 1
    for (int L = tid; L < NE * N * Q; L += NT) {
      const int el = L / (N * Q), r = L - el * N * Q;
      const int k = r / Q, a = r - k * Q;
      const double* in = smem + el * NBUF * BUF + IX(k, 0, a);
      double* out = smem + el * NBUF * BUF + BUF + IX(k, 0, a);
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
    #pragma unroll 1
    for (int L = tid; L < nel * N * N; L += NT) {
      const int el = L / (N * N), r = L - el * N * N;
      const int k = r / N, j = r - k * N;
      const int64_t e = e0 + el;
      const double* in = smem + el * NBUF * BUF + BUF + IX(k, j, 0);
      double v[Q];
#pragma unroll
      for (int a = 0; a < Q; ++a) v[a] = in[a];
      const bool edge_line = (k == 0 || k == N - 1 || j == 0 || j == N - 1);
      const int* mrow = smap + el * NLOCP + (k * N + j) * N;
      double* srow = S + e * NB;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) acc = fma(P.B[a][i], v[a], acc);
        if (!edge_line && i > 0 && i < N - 1) {
          y[mrow[i]] = 0.0 + acc;  // bincount semantics: 0.0 + contribution
        } else {
          srow[boundary_rank3<N>(k, j, i)] = acc;
        }
      }
    }
  }
}

}  // namespace fb
