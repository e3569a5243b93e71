// Krylov vector kernels (solvers.py:108-254) and constrained-row masking
// (ConstrainedOperator, mfop.py:428-433).
//
// Reductions are deterministic: the first pass sums fixed 4096-entry chunks
// (256 threads x 16 strided entries, then a fixed shuffle tree), the second
// pass reduces the chunk partials in a fixed order in one block.  Updates
// use explicit round-to-nearest multiply-then-add (no FMA contraction) so
// `x += alpha * p` rounds exactly like numpy's two-step evaluation.
#include "fb_common.cuh"

namespace fb {

constexpr int kDotChunk = 4096;
constexpr int kDotThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = lane < NT / 32 ? red[lane] : 0.0;
    s = warp_sum(s);
  }
  return s;
}

__global__ void __launch_bounds__(kDotThreads) dot_partial_kernel(int64_t n, const double* __restrict__ x,
                                                      const double* __restrict__ y,
                                                      double* __restrict__ partial) {
  __shared__ double red[kDotThreads / 32];
  const int64_t base = int64_t(blockIdx.x) * kDotChunk;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kDotChunk / kDotThreads; ++k) {
    const int64_t i = base + threadIdx.x + int64_t(k) * kDotThreads;
    if (i < n) acc = __dadd_rn(acc, __dmul_rn(__ldg(x + i), __ldg(y + i)));
  }
  const double s = block_sum<kDotThreads>(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) dot_final_kernel(int64_t np, const double* __restrict__ partial,
                                             double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < np; i += 1024) acc += partial[i];
  const double s = block_sum<1024>(acc, red);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
}

__global__ void axpy_dev_kernel(int64_t n, const double* __restrict__ a, double sign,
                                const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const double al = a[0];
  if (i < n) {
    const double t = __dmul_rn(al, x[i]);
    y[i] = sign > 0 ? __dadd_rn(y[i], t) : __dsub_rn(y[i], t);
  }
}

// Fused PCG update (solvers.py:141-150): alpha = rz / pAp (0 when pAp <= 0,
// the loop then stops), x += alpha p and, unless this is a true-residual
// iteration, r -= alpha Ap -- one pass instead of three launches, with the
// reference's rounding (numpy: round(x + round(alpha * p))).
template <bool VEC>
__global__ void cg_update_kernel(int64_t n, const double* __restrict__ rz,
                                 const double* __restrict__ pAp, double* __restrict__ alpha_out,
                                 const double* __restrict__ p, const double* __restrict__ Ap,
                                 double* __restrict__ x, double* __restrict__ r, int update_r) {
  const double d = pAp[0];
  const double al = d > 0.0 ? __ddiv_rn(rz[0], d) : 0.0;
  const int64_t i0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * (VEC ? 2 : 1);
  if (i0 == 0) alpha_out[0] = al;
  if (VEC && i0 + 1 < n) {
    const double2 pv = *reinterpret_cast<const double2*>(p + i0);
    double2 xv = *reinterpret_cast<const double2*>(x + i0);
    xv.x = __dadd_rn(xv.x, __dmul_rn(al, pv.x));
    xv.y = __dadd_rn(xv.y, __dmul_rn(al, pv.y));
    *reinterpret_cast<double2*>(x + i0) = xv;
    if (update_r) {
      const double2 av = *reinterpret_cast<const double2*>(Ap + i0);
      double2 rv = *reinterpret_cast<const double2*>(r + i0);
      rv.x = __dsub_rn(rv.x, __dmul_rn(al, av.x));
      rv.y = __dsub_rn(rv.y, __dmul_rn(al, av.y));
      *reinterpret_cast<double2*>(r + i0) = rv;
    }
  } else if (i0 < n) {
    x[i0] = __dadd_rn(x[i0], __dmul_rn(al, p[i0]));
    if (update_r) r[i0] = __dsub_rn(r[i0], __dmul_rn(al, Ap[i0]));
  }
}

__global__ void scalar_div_kernel(const double* num, const double* den, double* out) {
  out[0] = __ddiv_rn(num[0], den[0]);
}

__global__ void xpby_ratio_kernel(int64_t n, const double* __restrict__ z,
                                  const double* __restrict__ num, const double* __restrict__ den,
                                  double* __restrict__ p) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const double beta = __ddiv_rn(num[0], den[0]);
  if (i < n) p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

__global__ void div_scalar_kernel(int64_t n, const double* __restrict__ x, double s,
                                  double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __ddiv_rn(x[i], s);
}

__global__ void shift_ratio_kernel(int64_t n, const double* __restrict__ x,
                                   const double* __restrict__ num, double den,
                                   double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const double m = __ddiv_rn(num[0], den);
  if (i < n) y[i] = __dsub_rn(x[i], m);
}

__global__ void scale_kernel(int64_t n, double a, const double* __restrict__ x,
                             double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dmul_rn(a, x[i]);
}

__global__ void safe_div_kernel(const double* num, const double* den, double* out) {
  out[0] = den[0] > 0.0 ? __ddiv_rn(num[0], den[0]) : 0.0;
}

__global__ void vmul_kernel(int64_t n, const double* __restrict__ d, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dmul_rn(d[i], x[i]);
}

__global__ void copy_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i];
}

__global__ void mask_zero_kernel(int64_t m, const int64_t* __restrict__ dofs,
                                 double* __restrict__ xi) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) xi[dofs[i]] = 0.0;
}

__global__ void mask_restore_kernel(int64_t m, const int64_t* __restrict__ dofs,
                                    const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) {
    const int64_t d = dofs[i];
    y[d] = x[d];
  }
}

}  // namespace fb

using namespace fb;

extern "C" {

int64_t fb_dot_partials(int64_t n) { return n <= 0 ? 1 : (n + kDotChunk - 1) / kDotChunk; }

int fb_dot(int64_t n, const double* x, const double* y, double* partial, double* result,
           void* stream) {
  cudaStream_t st = as_stream(stream);
  const int64_t np = fb_dot_partials(n);
  if (n > 0) {
    dot_partial_kernel<<<unsigned(np), kDotThreads, 0, st>>>(n, x, y, partial);
    FB_CHECK_LAUNCH();
  } else {
    FB_TRY_CUDA(cudaMemsetAsync(partial, 0, sizeof(double), st));
  }
  dot_final_kernel<<<1, 1024, 0, st>>>(np, partial, result);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream) {
  if (n <= 0) return FB_OK;
  axpby_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, a, x, b, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_axpy_dev(int64_t n, const double* a, int sign, const double* x, double* y, void* stream) {
  if (n <= 0) return FB_OK;
  axpy_dev_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, a, sign >= 0 ? 1.0 : -1.0,
                                                                    x, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_cg_update(int64_t n, const double* rz, const double* pAp, double* alpha_out,
                 const double* p, const double* Ap, double* x, double* r, int update_r,
                 void* stream) {
  FB_REQUIRE(n >= 0, "negative length");
  const bool aligned = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(Ap) |
                         reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r)) & 15) == 0;
  cudaStream_t st = as_stream(stream);
  if (aligned) {
    const int64_t pairs = n > 0 ? (n + 1) / 2 : 1;
    cg_update_kernel<true><<<ceil_div(pairs, 256), 256, 0, st>>>(n, rz, pAp, alpha_out, p, Ap, x,
                                                                 r, update_r);
  } else {
    cg_update_kernel<false><<<ceil_div(n > 0 ? n : 1, 256), 256, 0, st>>>(n, rz, pAp, alpha_out,
                                                                          p, Ap, x, r, update_r);
  }
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_scalar_div(const double* num, const double* den, double* out, void* stream) {
  scalar_div_kernel<<<1, 1, 0, as_stream(stream)>>>(num, den, out);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_xpby_ratio(int64_t n, const double* z, const double* num, const double* den, double* p,
                  void* stream) {
  if (n <= 0) return FB_OK;
  xpby_ratio_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, z, num, den, p);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_div_scalar(int64_t n, const double* x, double s, double* y, void* stream) {
  if (n <= 0) return FB_OK;
  div_scalar_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, x, s, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_shift_ratio(int64_t n, const double* x, const double* num, double den, double* y,
                   void* stream) {
  if (n <= 0) return FB_OK;
  shift_ratio_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, x, num, den, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_scale(int64_t n, double a, const double* x, double* y, void* stream) {
  if (n <= 0) return FB_OK;
  scale_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, a, x, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_safe_div(const double* num, const double* den, double* out, void* stream) {
  safe_div_kernel<<<1, 1, 0, as_stream(stream)>>>(num, den, out);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_vmul(int64_t n, const double* d, const double* x, double* y, void* stream) {
  if (n <= 0) return FB_OK;
  vmul_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, d, x, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_mask_copy_zero(const double* x, double* xi, int64_t n, const int64_t* dofs, int64_t m,
                      void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n > 0 && x != xi) {
    copy_kernel<<<ceil_div(n, 256), 256, 0, st>>>(n, x, xi);
    FB_CHECK_LAUNCH();
  }
  if (m > 0) {
    mask_zero_kernel<<<ceil_div(m, 256), 256, 0, st>>>(m, dofs, xi);
    FB_CHECK_LAUNCH();
  }
  return FB_OK;
}

int fb_mask_restore(const double* x, double* y, const int64_t* dofs, int64_t m, void* stream) {
  if (m <= 0) return FB_OK;
  mask_restore_kernel<<<ceil_div(m, 256), 256, 0, as_stream(stream)>>>(m, dofs, x, y);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

}  // extern "C"
