// Library-internal handle layouts shared between translation units.
#pragma once

#include "fb_common.cuh"

// CSR matrix on the device: 64-bit row offsets (the finest LOR level of a
// 100M-DoF box has ~2.7G entries), 32-bit column indices.
struct fb_csr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int warp_rows = 0;  // 1: 4 lanes per row, butterfly-order sums (device-assembled LOR levels);
                      // 0: one thread per row, scipy's sequential order
  fb::DevBuf<int64_t> indptr;
  fb::DevBuf<int> indices;
  fb::DevBuf<double> data;
};

namespace fb {
// read-only views of a restriction (defined in fb_ops.cu)
const int* restriction_map(const fb_restriction* r);
int restriction_nloc(const fb_restriction* r);
int64_t restriction_ne(const fb_restriction* r);
int64_t restriction_ndofs(const fb_restriction* r);

// exclusive prefix sum of n counts into n+1 offsets (device, CUB)
int exclusive_offsets(const int* counts, int64_t n, int64_t* offsets, cudaStream_t st);
}  // namespace fb
