// General sum-factorized operator kernel: any dimension (2/3), any degree,
// any rule size, and the mixed velocity/pressure operators.  One CTA per
// element; the 1D matrices live in shared memory and every 1D contraction
// is a block-wide pass.  It follows the reference's contraction structure
// literally (kernels/numba_backend.py:7-61 three-pass tensor application;
// mfop.py:56-95 values/grads/values_t/grads_t) so it doubles as the
// correctness path for shapes the fused fast kernel does not cover
// (2D, p > 10, n_q != p+2, gradient/divergence).  Its output is an E-vector
// that scatter_rows sums into the L-vector.
#pragma once

#include "fb_common.cuh"

namespace fb {

enum GenKind { kgMass = 0, kgStiff = 1, kgHelm = 2, kgGrad = 3, kgDiv = 4, kgGradT = 5, kgConv = 6, kgCurl = 7 };

struct SFGParams {
  const int* __restrict__ map_in;   // (ne, nin^dim)
  const double* __restrict__ fac;   // (ne, K, nq^dim) element-blocked
  const double* __restrict__ x;     // input L-vector (all components)
  double* __restrict__ ye;          // output E-vector (ncomp_out, ne, nout^dim)
  const double* __restrict__ mats;  // device: Bv Dv Bp Dp, each (nq, n) row-major
  int64_t ne;
  int64_t in_comp_stride;           // L-vector component stride of the input
  int dim, kind, nv, np, nq, nfac;
  int64_t fstride;
};

// out (+)= (M2 (x) M1 (x) M0) in, M_a row-major (qa x na), in dims (n2,n1,n0)
__device__ void gen_tensor(int dim, const double* in, int n0, int n1, int n2,
                           const double* M0, const double* M1, const double* M2, int q0,
                           int q1, int q2, double* out, bool accumulate, double* t0,
                           double* t1) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (dim == 2) {
    // t0[i][b] = sum_j M0[b][j] in[i][j]  (n1, q0)
    for (int idx = tid; idx < n1 * q0; idx += nt) {
      const int i = idx / q0, b = idx - i * q0;
      double acc = 0.0;
      for (int j = 0; j < n0; ++j) acc += M0[b * n0 + j] * in[i * n0 + j];
      t0[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < q1 * q0; idx += nt) {
      const int a = idx / q0, b = idx - a * q0;
      double acc = 0.0;
      for (int i = 0; i < n1; ++i) acc += M1[a * n1 + i] * t0[i * q0 + b];
      out[idx] = accumulate ? out[idx] + acc : acc;
    }
    __syncthreads();
    return;
  }
  for (int idx = tid; idx < n2 * n1 * q0; idx += nt) {
    const int ki = idx / q0, b = idx - ki * q0;
    double acc = 0.0;
    for (int j = 0; j < n0; ++j) acc += M0[b * n0 + j] * in[ki * n0 + j];
    t0[idx] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < n2 * q1 * q0; idx += nt) {
    const int k = idx / (q1 * q0), r = idx - k * q1 * q0;
    const int a = r / q0, b = r - a * q0;
    double acc = 0.0;
    for (int i = 0; i < n1; ++i) acc += M1[a * n1 + i] * t0[(k * n1 + i) * q0 + b];
    t1[idx] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < q2 * q1 * q0; idx += nt) {
    const int c = idx / (q1 * q0), ab = idx - c * q1 * q0;
    double acc = 0.0;
    for (int k = 0; k < n2; ++k) acc += M2[c * n2 + k] * t1[k * q1 * q0 + ab];
    out[idx] = accumulate ? out[idx] + acc : acc;
  }
  __syncthreads();
}

// grads: g_m = tensor with D in direction m, B elsewhere (mfop.py:64-76)
__device__ void gen_grads(int dim, const double* in, int n, const double* B, const double* D,
                          int q, double* const* g, double* t0, double* t1) {
  if (dim == 2) {
    gen_tensor(2, in, n, n, 1, D, B, nullptr, q, q, 1, g[0], false, t0, t1);
    gen_tensor(2, in, n, n, 1, B, D, nullptr, q, q, 1, g[1], false, t0, t1);
  } else {
    gen_tensor(3, in, n, n, n, D, B, B, q, q, q, g[0], false, t0, t1);
    gen_tensor(3, in, n, n, n, B, D, B, q, q, q, g[1], false, t0, t1);
    gen_tensor(3, in, n, n, n, B, B, D, q, q, q, g[2], false, t0, t1);
  }
}

// out (+)= sum_m grad-transpose of f_m (mfop.py:86-95); Bt/Dt are (n, q)
__device__ void gen_grads_t(int dim, double* const* f, int q, const double* Bt,
                            const double* Dt, int n, double* out, bool accumulate, double* t0,
                            double* t1) {
  if (dim == 2) {
    gen_tensor(2, f[0], q, q, 1, Dt, Bt, nullptr, n, n, 1, out, accumulate, t0, t1);
    gen_tensor(2, f[1], q, q, 1, Bt, Dt, nullptr, n, n, 1, out, true, t0, t1);
  } else {
    gen_tensor(3, f[0], q, q, q, Dt, Bt, Bt, n, n, n, out, accumulate, t0, t1);
    gen_tensor(3, f[1], q, q, q, Bt, Dt, Bt, n, n, n, out, true, t0, t1);
    gen_tensor(3, f[2], q, q, q, Bt, Bt, Dt, n, n, n, out, true, t0, t1);
  }
}

__device__ __forceinline__ void gen_values(int dim, const double* in, int n, const double* B,
                                           int q, double* out, bool acc, double* t0,
                                           double* t1) {
  gen_tensor(dim, in, n, n, dim == 3 ? n : 1, B, B, B, q, q, dim == 3 ? q : 1, out, acc, t0, t1);
}

__device__ __forceinline__ int ipow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// Shared-memory plan: matrices (8 of nq*nmax) + 10 buffers of E^dim,
// E = max(nv, np, nq).
__host__ __device__ inline size_t gen_smem_bytes(int dim, int nv, int np, int nq) {
  int E = nv > nq ? nv : nq;
  if (np > E) E = np;
  int Ed = E * E * (dim == 3 ? E : 1);
  int nmax = nv > np ? nv : np;
  return sizeof(double) * (size_t(8) * nq * nmax + size_t(10) * Ed);
}

__global__ void sf_general_kernel(const __grid_constant__ SFGParams P) {
  extern __shared__ double sm[];
  const int dim = P.dim, nv = P.nv, np = P.np, nq = P.nq;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t e = blockIdx.x;
  const int comp = blockIdx.y;
  int E = nv > nq ? nv : nq;
  if (np > E) E = np;
  const int Ed = ipow(E, dim);
  const int nmax = nv > np ? nv : np;
  // matrices: Bv Dv Bp Dp (nq x n) and BvT DvT BpT DpT (n x nq)
  double* Bv = sm;
  double* Dv = Bv + nq * nmax;
  double* Bp = Dv + nq * nmax;
  double* Dp = Bp + nq * nmax;
  double* BvT = Dp + nq * nmax;
  double* DvT = BvT + nq * nmax;
  double* BpT = DvT + nq * nmax;
  double* DpT = BpT + nq * nmax;
  double* buf = DpT + nq * nmax;
  double* xin = buf;
  double* vals = buf + Ed;
  double* g[3] = {buf + 2 * Ed, buf + 3 * Ed, buf + 4 * Ed};
  double* f[3] = {buf + 5 * Ed, buf + 6 * Ed, buf + 7 * Ed};
  double* t0 = buf + 8 * Ed;
  double* t1 = buf + 9 * Ed;
  double* out = vals;  // reused once vals are consumed

  const double* mats = P.mats;
  for (int idx = tid; idx < nq * nv; idx += nt) {
    const int qq = idx / nv, j = idx - qq * nv;
    Bv[idx] = mats[idx];
    Dv[idx] = mats[nq * nv + idx];
    BvT[j * nq + qq] = mats[idx];
    DvT[j * nq + qq] = mats[nq * nv + idx];
  }
  if (np > 0) {
    for (int idx = tid; idx < nq * np; idx += nt) {
      const int qq = idx / np, j = idx - qq * np;
      Bp[idx] = mats[2 * nq * nv + idx];
      Dp[idx] = mats[2 * nq * nv + nq * np + idx];
      BpT[j * nq + qq] = mats[2 * nq * nv + idx];
      DpT[j * nq + qq] = mats[2 * nq * nv + nq * np + idx];
    }
  }
  const int nqd = ipow(nq, dim);
  const int nvd = ipow(nv, dim);
  const int npd = np > 0 ? ipow(np, dim) : 0;
  const double* fe = P.fac + e * P.fstride;
  const int kind = P.kind;
  __syncthreads();

  if (kind <= kgHelm) {
    // square operator on component `comp` (mfop.py:187-244)
    const double* xc = P.x + comp * P.in_comp_stride;
    for (int l = tid; l < nvd; l += nt) xin[l] = xc[P.map_in[e * nvd + l]];
    __syncthreads();
    const bool has_mass = kind != kgStiff, has_stiff = kind != kgMass;
    if (has_mass) gen_values(dim, xin, nv, Bv, nq, vals, false, t0, t1);
    if (has_stiff) gen_grads(dim, xin, nv, Bv, Dv, nq, g, t0, t1);
    const int ks = has_mass && has_stiff ? 1 : 0;
    for (int qp = tid; qp < nqd; qp += nt) {
      if (has_mass) vals[qp] = vals[qp] * fe[qp];
      if (has_stiff) {
        if (dim == 2) {
          const double w00 = fe[(ks + 0) * nqd + qp], w01 = fe[(ks + 1) * nqd + qp],
                       w11 = fe[(ks + 2) * nqd + qp];
          const double a0 = g[0][qp], a1 = g[1][qp];
          f[0][qp] = w00 * a0 + w01 * a1;
          f[1][qp] = w01 * a0 + w11 * a1;
        } else {
          const double w00 = fe[(ks + 0) * nqd + qp], w01 = fe[(ks + 1) * nqd + qp],
                       w02 = fe[(ks + 2) * nqd + qp], w11 = fe[(ks + 3) * nqd + qp],
                       w12 = fe[(ks + 4) * nqd + qp], w22 = fe[(ks + 5) * nqd + qp];
          const double a0 = g[0][qp], a1 = g[1][qp], a2 = g[2][qp];
          f[0][qp] = w00 * a0 + w01 * a1 + w02 * a2;
          f[1][qp] = w01 * a0 + w11 * a1 + w12 * a2;
          f[2][qp] = w02 * a0 + w12 * a1 + w22 * a2;
        }
      }
    }
    __syncthreads();
    double* res = xin;  // x_e no longer needed
    if (has_mass) gen_values(dim, vals, nq, BvT, nv, res, false, t0, t1);
    if (has_stiff) gen_grads_t(dim, f, nq, BvT, DvT, nv, res, has_mass, t0, t1);
    double* ye = P.ye + (int64_t(comp) * P.ne + e) * nvd;
    for (int l = tid; l < nvd; l += nt) ye[l] = res[l];
    return;
  }

  if (kind == kgGrad) {
    // pressure -> velocity (mfop.py:265-275)
    for (int l = tid; l < npd; l += nt) xin[l] = P.x[P.map_in[e * npd + l]];
    __syncthreads();
    gen_grads(dim, xin, np, Bp, Dp, nq, g, t0, t1);
    for (int c = 0; c < dim; ++c) {
      for (int qp = tid; qp < nqd; qp += nt) {
        double s = fe[(c * dim + 0) * nqd + qp] * g[0][qp];
        for (int m = 1; m < dim; ++m) s = s + fe[(c * dim + m) * nqd + qp] * g[m][qp];
        f[0][qp] = s;
      }
      __syncthreads();
      gen_values(dim, f[0], nq, BvT, nv, out, false, t0, t1);
      double* ye = P.ye + (int64_t(c) * P.ne + e) * nvd;
      for (int l = tid; l < nvd; l += nt) ye[l] = out[l];
      __syncthreads();
    }
    return;
  }

  if (kind == kgConv) {
    // convection load, output component comp (mfop.py:341-358):
    //   conv_c = sum_k U_k sum_m (wdet Jinv[m,k]) dU_c/dxi_m,  y_c = B^T conv_c
    // factors are the gradient set fe[(k*dim + m)] = wdet Jinv[m,k]
    for (int k = 0; k < dim; ++k) {  // values of every component -> f[k]
      const double* xk = P.x + k * P.in_comp_stride;
      for (int l = tid; l < nvd; l += nt) xin[l] = xk[P.map_in[e * nvd + l]];
      __syncthreads();
      gen_values(dim, xin, nv, Bv, nq, f[k], false, t0, t1);
    }
    const double* xc = P.x + comp * P.in_comp_stride;
    for (int l = tid; l < nvd; l += nt) xin[l] = xc[P.map_in[e * nvd + l]];
    __syncthreads();
    gen_grads(dim, xin, nv, Bv, Dv, nq, g, t0, t1);
    for (int qp = tid; qp < nqd; qp += nt) {
      double s = 0.0;
      for (int k = 0; k < dim; ++k) {
        double gk = 0.0;
        for (int m = 0; m < dim; ++m) gk += fe[(k * dim + m) * nqd + qp] * g[m][qp];
        s += f[k][qp] * gk;
      }
      vals[qp] = s;
    }
    __syncthreads();
    gen_values(dim, vals, nq, BvT, nv, xin, false, t0, t1);
    double* ye = P.ye + (int64_t(comp) * P.ne + e) * nvd;
    for (int l = tid; l < nvd; l += nt) ye[l] = xin[l];
    return;
  }

  if (kind == kgCurl) {
    // curl-curl, output component comp (mfop.py:381-413); factors
    // fe[0] = nu wdet, fe[1 + m d + k] = Jinv[m][k].  om = nu wdet curl u is
    // accumulated component by component in f[], then fs_m = sum_b Jinv[m][b]
    // t_b with t = eps(., ., comp) om, and y_comp = grads_t(fs).
    const int nom = dim == 3 ? 3 : 1;
    for (int a = 0; a < nom; ++a)
      for (int qp = tid; qp < nqd; qp += nt) f[a][qp] = 0.0;
    for (int cc = 0; cc < dim; ++cc) {
      const double* xk = P.x + cc * P.in_comp_stride;
      for (int l = tid; l < nvd; l += nt) xin[l] = xk[P.map_in[e * nvd + l]];
      __syncthreads();
      gen_grads(dim, xin, nv, Bv, Dv, nq, g, t0, t1);
      for (int qp = tid; qp < nqd; qp += nt) {
        const double wd = fe[qp];
        double gp[3];
        for (int k = 0; k < dim; ++k) {
          double s = 0.0;
          for (int m = 0; m < dim; ++m) s += fe[(1 + m * dim + k) * nqd + qp] * g[m][qp];
          gp[k] = s;  // d u_cc / d x_k
        }
        if (dim == 2) {
          f[0][qp] += (cc == 1 ? wd * gp[0] : -wd * gp[1]);
        } else if (cc == 0) {
          f[1][qp] += wd * gp[2];
          f[2][qp] -= wd * gp[1];
        } else if (cc == 1) {
          f[0][qp] -= wd * gp[2];
          f[2][qp] += wd * gp[0];
        } else {
          f[0][qp] += wd * gp[1];
          f[1][qp] -= wd * gp[0];
        }
      }
      __syncthreads();
    }
    for (int qp = tid; qp < nqd; qp += nt) {
      double t[3] = {0.0, 0.0, 0.0};
      if (dim == 2) {
        if (comp == 0) t[1] = -f[0][qp]; else t[0] = f[0][qp];
      } else if (comp == 0) {
        t[2] = f[1][qp];
        t[1] = -f[2][qp];
      } else if (comp == 1) {
        t[0] = f[2][qp];
        t[2] = -f[0][qp];
      } else {
        t[1] = f[0][qp];
        t[0] = -f[1][qp];
      }
      for (int m = 0; m < dim; ++m) {
        double s = 0.0;
        for (int b = 0; b < dim; ++b) s += fe[(1 + m * dim + b) * nqd + qp] * t[b];
        g[m][qp] = s;
      }
    }
    __syncthreads();
    gen_grads_t(dim, g, nq, BvT, DvT, nv, xin, false, t0, t1);
    double* ye = P.ye + (int64_t(comp) * P.ne + e) * nvd;
    for (int l = tid; l < nvd; l += nt) ye[l] = xin[l];
    return;
  }

  if (kind == kgGradT) {
    // velocity -> pressure, G^T (mfop.py:277-288)
    for (int c = 0; c < dim; ++c) {
      const double* xc = P.x + c * P.in_comp_stride;
      for (int l = tid; l < nvd; l += nt) xin[l] = xc[P.map_in[e * nvd + l]];
      __syncthreads();
      gen_values(dim, xin, nv, Bv, nq, vals, false, t0, t1);
      for (int qp = tid; qp < nqd; qp += nt) {
        for (int m = 0; m < dim; ++m) {
          const double t = fe[(c * dim + m) * nqd + qp] * vals[qp];
          f[m][qp] = (c == 0) ? t : f[m][qp] + t;
        }
      }
      __syncthreads();
    }
    gen_grads_t(dim, f, nq, BpT, DpT, np, out, false, t0, t1);
    double* ye = P.ye + e * npd;
    for (int l = tid; l < npd; l += nt) ye[l] = out[l];
    return;
  }

  // kgDiv: velocity -> pressure (mfop.py:309-319)
  for (int c = 0; c < dim; ++c) {
    const double* xc = P.x + c * P.in_comp_stride;
    for (int l = tid; l < nvd; l += nt) xin[l] = xc[P.map_in[e * nvd + l]];
    __syncthreads();
    gen_grads(dim, xin, nv, Bv, Dv, nq, g, t0, t1);
    for (int qp = tid; qp < nqd; qp += nt) {
      double s = fe[(c * dim + 0) * nqd + qp] * g[0][qp];
      for (int m = 1; m < dim; ++m) s = s + fe[(c * dim + m) * nqd + qp] * g[m][qp];
      f[0][qp] = (c == 0) ? s : f[0][qp] + s;
    }
    __syncthreads();
  }
  gen_values(dim, f[0], nq, BpT, np, out, false, t0, t1);
  double* ye = P.ye + e * npd;
  for (int l = tid; l < npd; l += nt) ye[l] = out[l];
}

}  // namespace fb
