// LOR matrix assembly on the host in C++ (lor.py:61-99 semantics).
//
// The nodal lattice of a degree-p element is split into p^d trilinear
// sub-cells whose vertices are the element's DoFs; the Q1 mass/stiffness/
// Helmholtz matrix of that refined mesh is assembled with the 2-point Gauss
// rule per direction (the reference assembles it through mfop.assemble on a
// refined FESpace, lor.py:61-81).  Rows are built directly in CSR form:
// the pattern of a row is the union of the DoFs of its incident sub-cells,
// values are summed over incident sub-cells in ascending sub-cell order.
// Constrained rows/columns are zeroed in-pattern with a unit diagonal
// (constrain_matrix, lor.py:84-99).  Replaces a numpy einsum + COO sort that
// needs ~64 doubles of temporaries per sub-cell (26 s and ~8 GB at 1M DoFs).
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fbb200.h"

namespace fb {
void set_error(const std::string& msg);
}

namespace {

struct Q1Rule {
  int d, nc, nq;
  std::vector<double> N, dN, w;  // N[q][c], dN[q][c][b], w[q]
  Q1Rule(int dim) : d(dim), nc(1 << dim), nq(1 << dim) {
    const double g = 1.0 / std::sqrt(3.0);
    const double pts[2] = {-g, g};
    N.assign(nq * nc, 1.0);
    dN.assign(nq * nc * d, 1.0);
    w.assign(nq, 1.0);
    for (int q = 0; q < nq; ++q) {
      double xi[3];
      for (int a = 0; a < d; ++a) xi[a] = pts[(q >> a) & 1];
      for (int c = 0; c < nc; ++c)
        for (int a = 0; a < d; ++a) {
          const int hi = (c >> a) & 1;
          const double val = hi ? (1.0 + xi[a]) / 2.0 : (1.0 - xi[a]) / 2.0;
          const double der = hi ? 0.5 : -0.5;
          N[q * nc + c] *= val;
          for (int b = 0; b < d; ++b) dN[(q * nc + c) * d + b] *= (a == b) ? der : val;
        }
    }
  }
};

// local (2^d x 2^d) matrix of one sub-cell with corners X (nc x d)
template <int DIM>
void local_matrix(const Q1Rule& R, const double* X, int kind, double nu, double c, double* K) {
  constexpr int d = DIM, nc = 1 << DIM;
  std::fill(K, K + nc * nc, 0.0);
  for (int q = 0; q < nc; ++q) {
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int cc = 0; cc < nc; ++cc)
      for (int dd = 0; dd < d; ++dd)
        for (int b = 0; b < d; ++b) J[dd][b] += R.dN[(q * nc + cc) * d + b] * X[cc * d + dd];
    double det, Ji[3][3];
    if (d == 2) {
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      Ji[0][0] = J[1][1] / det;
      Ji[0][1] = -J[0][1] / det;
      Ji[1][0] = -J[1][0] / det;
      Ji[1][1] = J[0][0] / det;
    } else {
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
            J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    }
    const double wdet = det * R.w[q];
    if (kind != FB_STIFFNESS) {
      const double wm = (kind == FB_HELMHOLTZ) ? c * wdet : wdet;
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j) K[i * nc + j] += R.N[q * nc + i] * wm * R.N[q * nc + j];
    }
    if (kind != FB_MASS) {
      double W[3][3];
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          double s = 0.0;
          for (int m = 0; m < d; ++m) s += Ji[a][m] * Ji[b][m];
          W[a][b] = nu * wdet * s;
        }
      for (int i = 0; i < nc; ++i) {
        double gi[3];
        for (int a = 0; a < d; ++a) gi[a] = R.dN[(q * nc + i) * d + a];
        for (int j = 0; j < nc; ++j) {
          double s = 0.0;
          for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) s += gi[a] * W[a][b] * R.dN[(q * nc + j) * d + b];
          K[i * nc + j] += s;
        }
      }
    }
  }
}

}  // namespace

extern "C" {

void fb_host_free(void* p) { std::free(p); }

int64_t fb_lor_assemble_host(int dim, int p, int64_t ne, int64_t ndofs, const int64_t* element_dofs,
                             const double* corners, const double* nodes, int kind, double nu,
                             double c, int64_t ncons, const int64_t* constrained,
                             int64_t** indptr_out, int64_t** indices_out, double** data_out) {
  if ((dim != 2 && dim != 3) || p < 1 || kind < FB_MASS || kind > FB_HELMHOLTZ) {
    fb::set_error("bad LOR assembly arguments");
    return -FB_ERR_ARG;
  }
  const int d = dim, n = p + 1, nc = 1 << d;
  const int nloc = d == 2 ? n * n : n * n * n;
  const int nsub = d == 2 ? p * p : p * p * p;
  // sub-cell local corner ids
  std::vector<int> sub(size_t(nsub) * nc);
  for (int s = 0; s < nsub; ++s) {
    const int i = s % p, j = (s / p) % p, k = d == 3 ? s / (p * p) : 0;
    const int base = i + n * (j + n * k);
    for (int cc = 0; cc < nc; ++cc) {
      const int off = (cc & 1) + n * ((cc >> 1) & 1) + (d == 3 ? n * n * ((cc >> 2) & 1) : 0);
      sub[s * nc + cc] = base + off;
    }
  }
  // nodal lattice positions in the reference cell -> multilinear weights
  std::vector<double> shp(size_t(nloc) * nc, 1.0);
  for (int l = 0; l < nloc; ++l) {
    const int li[3] = {l % n, (l / n) % n, l / (n * n)};
    for (int cc = 0; cc < nc; ++cc)
      for (int a = 0; a < d; ++a) {
        const double t = nodes[li[a]];
        shp[l * nc + cc] *= ((cc >> a) & 1) ? (1.0 + t) / 2.0 : (1.0 - t) / 2.0;
      }
  }
  const int64_t nsc = ne * nsub;  // sub-cells
  // incidence: row -> (sub-cell, local corner), ascending sub-cell
  std::vector<int64_t> cnt(ndofs + 1, 0);
  for (int64_t e = 0; e < ne; ++e)
    for (int s = 0; s < nsub; ++s)
      for (int cc = 0; cc < nc; ++cc) {
        const int64_t r = element_dofs[e * nloc + sub[s * nc + cc]];
        if (r < 0 || r >= ndofs) {
          fb::set_error("element_dofs entry out of range");
          return -FB_ERR_ARG;
        }
        ++cnt[r + 1];
      }
  for (int64_t r = 0; r < ndofs; ++r) cnt[r + 1] += cnt[r];
  std::vector<int64_t> inc(cnt[ndofs]);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t e = 0; e < ne; ++e)
      for (int s = 0; s < nsub; ++s)
        for (int cc = 0; cc < nc; ++cc) {
          const int64_t r = element_dofs[e * nloc + sub[s * nc + cc]];
          inc[pos[r]++] = (e * nsub + s) * nc + cc;
        }
  }
  std::vector<char> cons(ndofs, 0);
  for (int64_t i = 0; i < ncons; ++i) cons[constrained[i]] = 1;
  // pass 1: row patterns (union of the DoFs of the incident sub-cells),
  // row counts in parallel, then the columns in parallel
  std::vector<int64_t> ip(ndofs + 1, 0);
  auto row_cols = [&](int64_t r, std::vector<int64_t>& cols) {
    cols.clear();
    for (int64_t k = cnt[r]; k < cnt[r + 1]; ++k) {
      const int64_t sc = inc[k] / nc;
      const int64_t e = sc / nsub;
      const int s = int(sc % nsub);
      for (int cc = 0; cc < nc; ++cc) cols.push_back(element_dofs[e * nloc + sub[s * nc + cc]]);
    }
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
  };
#pragma omp parallel
  {
    std::vector<int64_t> cols;
#pragma omp for schedule(static)
    for (int64_t r = 0; r < ndofs; ++r) {
      row_cols(r, cols);
      ip[r + 1] = int64_t(cols.size());
    }
  }
  for (int64_t r = 0; r < ndofs; ++r) ip[r + 1] += ip[r];
  std::vector<int64_t> ix(ip[ndofs]);
#pragma omp parallel
  {
    std::vector<int64_t> cols;
#pragma omp for schedule(static)
    for (int64_t r = 0; r < ndofs; ++r) {
      row_cols(r, cols);
      std::copy(cols.begin(), cols.end(), ix.begin() + ip[r]);
    }
  }
  std::vector<int64_t>().swap(inc);
  // pass 2: local matrices computed in parallel per chunk of sub-cells, then
  // added in ascending sub-cell order (deterministic sums)
  std::vector<double> vv(ix.size(), 0.0);
  const Q1Rule R(d);
  const int64_t chunk = 1 << 16;
  std::vector<double> Kc(size_t(chunk) * nc * nc);
  std::vector<int64_t> dofc(size_t(chunk) * nc);
  for (int64_t c0 = 0; c0 < nsc; c0 += chunk) {
    const int64_t c1 = std::min(nsc, c0 + chunk);
#pragma omp parallel for schedule(static)
    for (int64_t sc = c0; sc < c1; ++sc) {
      const int64_t e = sc / nsub;
      const int s = int(sc % nsub);
      double X[8 * 3];
      for (int cc = 0; cc < nc; ++cc) {
        const int l = sub[s * nc + cc];
        dofc[(sc - c0) * nc + cc] = element_dofs[e * nloc + l];
        for (int dd = 0; dd < d; ++dd) {
          double x = 0.0;
          for (int c2 = 0; c2 < nc; ++c2) x += shp[l * nc + c2] * corners[(e * nc + c2) * d + dd];
          X[cc * d + dd] = x;
        }
      }
      double* K = &Kc[size_t(sc - c0) * nc * nc];
      if (d == 3) local_matrix<3>(R, X, kind, nu, c, K);
      else local_matrix<2>(R, X, kind, nu, c, K);
    }
    for (int64_t sc = c0; sc < c1; ++sc) {
      const int64_t* dof = &dofc[(sc - c0) * nc];
      const double* K = &Kc[size_t(sc - c0) * nc * nc];
      for (int i = 0; i < nc; ++i) {
        const int64_t r = dof[i];
        const int64_t* b = ix.data() + ip[r];
        const int64_t* en = ix.data() + ip[r + 1];
        for (int j = 0; j < nc; ++j) {
          const int64_t at = std::lower_bound(b, en, dof[j]) - ix.data();
          vv[at] += K[i * nc + j];
        }
      }
    }
  }
  for (int64_t r = 0; r < ndofs; ++r)
    for (int64_t a = ip[r]; a < ip[r + 1]; ++a) {
      if (cons[r]) vv[a] = (ix[a] == r) ? 1.0 : 0.0;
      else if (cons[ix[a]]) vv[a] = 0.0;
    }
  const int64_t nnz = ip[ndofs];
  *indptr_out = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (ndofs + 1)));
  *indices_out = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (nnz > 0 ? nnz : 1)));
  *data_out = static_cast<double*>(std::malloc(sizeof(double) * (nnz > 0 ? nnz : 1)));
  if (!*indptr_out || !*indices_out || !*data_out) {
    fb::set_error("host allocation failed");
    return -FB_ERR_OOM;
  }
  std::memcpy(*indptr_out, ip.data(), sizeof(int64_t) * (ndofs + 1));
  std::memcpy(*indices_out, ix.data(), sizeof(int64_t) * nnz);
  std::memcpy(*data_out, vv.data(), sizeof(double) * nnz);
  return nnz;
}

}  // extern "C"
