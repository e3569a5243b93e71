// Launchers of the fused mixed-degree kernel (sf3_mixed.cuh): the 3D weak
// gradient, its transpose and the weak divergence for Taylor-Hood
// (p_p = p_v - 1) and equal-order (p_p = p_v) pairs, p_v = 2..8, n_q = p_v + 2.
#include "sf3_mixed.cuh"

namespace fb {

template <int NV, int NP, int KIND>
int launch_mixed_t(const SF3MParams& P, cudaStream_t st) {
  constexpr int Q = NV + 1;
  constexpr int NT = (Q * Q > 64) ? 128 : 64;
  constexpr size_t smem = SF3MShape<NV, NP, Q>::SMEM;
  static int resident = 0;
  if (resident == 0) {
    auto kern = sf3_mixed_kernel<NV, NP, Q, KIND, NT>;
    FB_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
    int dev = 0, sms = 0, per_sm = 0;
    FB_TRY_CUDA(cudaGetDevice(&dev));
    FB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    resident = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t grid = P.ne < resident ? P.ne : resident;
  if (grid <= 0) return FB_OK;
  sf3_mixed_kernel<NV, NP, Q, KIND, NT><<<unsigned(grid), NT, smem, st>>>(P);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

template <int NV, int NP>
int launch_mixed_k(int kind, const SF3MParams& P, cudaStream_t st) {
  if (kind == kMxGrad) return launch_mixed_t<NV, NP, kMxGrad>(P, st);
  if (kind == kMxGradT) return launch_mixed_t<NV, NP, kMxGradT>(P, st);
  return launch_mixed_t<NV, NP, kMxDiv>(P, st);
}

bool mixed_supported(int nv, int np, int nq) {
  return nv >= 3 && nv <= 9 && nq == nv + 1 && (np == nv || np == nv - 1);
}

int launch_mixed(int nv, int np, int kind, const SF3MParams& P, cudaStream_t st) {
  const bool th = np == nv - 1;
  switch (nv) {
    case 3: return th ? launch_mixed_k<3, 2>(kind, P, st) : launch_mixed_k<3, 3>(kind, P, st);
    case 4: return th ? launch_mixed_k<4, 3>(kind, P, st) : launch_mixed_k<4, 4>(kind, P, st);
    case 5: return th ? launch_mixed_k<5, 4>(kind, P, st) : launch_mixed_k<5, 5>(kind, P, st);
    case 6: return th ? launch_mixed_k<6, 5>(kind, P, st) : launch_mixed_k<6, 6>(kind, P, st);
    case 7: return th ? launch_mixed_k<7, 6>(kind, P, st) : launch_mixed_k<7, 7>(kind, P, st);
    case 8: return th ? launch_mixed_k<8, 7>(kind, P, st) : launch_mixed_k<8, 8>(kind, P, st);
    case 9: return th ? launch_mixed_k<9, 8>(kind, P, st) : launch_mixed_k<9, 9>(kind, P, st);
    default: set_error("mixed fast path not built for this degree"); return FB_ERR_UNSUPPORTED;
  }
}

}  // namespace fb
