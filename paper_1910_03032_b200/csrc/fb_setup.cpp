// Host-side setup in C++: the reference's DoF numbering (fespace.py:71-217).
//
// DoFs are numbered entity by entity -- vertex classes, then edge interiors,
// then face interiors (3D), then element interiors -- each entity in order of
// first appearance during the element scan, with shared edges/faces read
// through the orientation of the element that first saw them.  The Python
// reference runs this as a per-element interpreter loop (85.9 s at 10M DoFs,
// SURVEY.md 2 row 5a); here it is one pass with hash tables.
#include <stdint.h>

#include <algorithm>
#include <array>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/fbb200.h"

namespace fb {
void set_error(const std::string& msg);
}

namespace {

struct Key4 {
  int64_t v[4];
  bool operator==(const Key4& o) const {
    return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2] && v[3] == o.v[3];
  }
};
struct Key4Hash {
  size_t operator()(const Key4& k) const {
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < 4; ++i) {
      h ^= uint64_t(k.v[i]) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    }
    return size_t(h);
  }
};

inline int corner_of(const int* bits, int d) {
  int c = 0;
  for (int a = 0; a < d; ++a) c += bits[a] << a;
  return c;
}

}  // namespace

extern "C" int64_t fb_number_dofs_host(int dim, int p, int64_t ne, int64_t nv,
                                       const int64_t* elems, int64_t* out, int64_t* num_edges,
                                       int64_t* num_faces) {
  if (dim != 2 && dim != 3) {
    fb::set_error("dim must be 2 or 3");
    return -FB_ERR_ARG;
  }
  if (p < 1) {
    fb::set_error("degree must be >= 1");
    return -FB_ERR_ARG;
  }
  const int d = dim, n = p + 1;
  const int ncorner = 1 << d;
  // local edge table: (axis a, fixed bits on the other axes)
  struct LEdge {
    int lo_bits[3], hi_bits[3];
  };
  std::vector<LEdge> ledges;
  if (d == 2) {
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        LEdge E{};
        E.lo_bits[1 - a] = b;
        E.lo_bits[a] = 0;
        std::copy(E.lo_bits, E.lo_bits + 3, E.hi_bits);
        E.hi_bits[a] = 1;
        ledges.push_back(E);
      }
  } else {
    for (int a = 0; a < 3; ++a) {
      int others[2], k = 0;
      for (int x = 0; x < 3; ++x)
        if (x != a) others[k++] = x;
      for (int b2 = 0; b2 < 2; ++b2)
        for (int b1 = 0; b1 < 2; ++b1) {
          LEdge E{};
          E.lo_bits[others[0]] = b1;
          E.lo_bits[others[1]] = b2;
          E.lo_bits[a] = 0;
          std::copy(E.lo_bits, E.lo_bits + 3, E.hi_bits);
          E.hi_bits[a] = 1;
          ledges.push_back(E);
        }
    }
  }
  const int nle = int(ledges.size());
  const int nloc1 = d == 2 ? n * n : n * n * n;
  if (p == 1) {
    // vertex DoFs only (fespace.py:76-82); entity counts are not needed
    for (int64_t k = 0; k < ne * nloc1; ++k) out[k] = elems[k];
    if (num_edges) *num_edges = -1;
    if (num_faces) *num_faces = -1;
    return nv;
  }
  const int nlf = d == 3 ? 6 : 0;

  std::unordered_map<uint64_t, int64_t> edge_id_of;
  edge_id_of.reserve(size_t(ne) * (d == 3 ? 3 : 2) + 16);
  std::vector<std::array<int64_t, 2>> edge_owner;
  std::vector<int64_t> eid(size_t(ne) * nle);
  std::vector<uint8_t> eflip(size_t(ne) * nle);
  std::unordered_map<Key4, int64_t, Key4Hash> face_id_of;
  std::vector<std::array<int64_t, 4>> face_owner;
  std::vector<int64_t> fid(size_t(ne) * nlf);
  std::vector<std::array<int, 6>> ftr(size_t(ne) * nlf);
  if (d == 3) face_id_of.reserve(size_t(ne) * 3 + 16);

  for (int64_t e = 0; e < ne; ++e) {
    const int64_t* conn = elems + e * ncorner;
    for (int le = 0; le < nle; ++le) {
      const int64_t va = conn[corner_of(ledges[le].lo_bits, d)];
      const int64_t vb = conn[corner_of(ledges[le].hi_bits, d)];
      const int64_t lo = std::min(va, vb), hi = std::max(va, vb);
      const uint64_t key = uint64_t(lo) * uint64_t(nv > 0 ? nv : 1) + uint64_t(hi);
      auto it = edge_id_of.find(key);
      int64_t id;
      if (it == edge_id_of.end()) {
        id = int64_t(edge_owner.size());
        edge_id_of.emplace(key, id);
        edge_owner.push_back({va, vb});
      } else {
        id = it->second;
      }
      eid[e * nle + le] = id;
      eflip[e * nle + le] = !(edge_owner[id][0] == va && edge_owner[id][1] == vb);
    }
    if (d == 3) {
      for (int f = 0; f < 6; ++f) {
        const int fa = f / 2, side = f % 2;
        int t[2], k = 0;
        for (int x = 0; x < 3; ++x)
          if (x != fa) t[k++] = x;
        std::array<int64_t, 4> ids;
        int m = 0;
        for (int j = 0; j < 2; ++j)
          for (int i = 0; i < 2; ++i) {
            int bits[3];
            bits[fa] = side;
            bits[t[0]] = i;
            bits[t[1]] = j;
            ids[m++] = conn[corner_of(bits, 3)];
          }
        Key4 key{{ids[0], ids[1], ids[2], ids[3]}};
        std::sort(key.v, key.v + 4);
        auto it = face_id_of.find(key);
        int64_t id;
        if (it == face_id_of.end()) {
          id = int64_t(face_owner.size());
          face_id_of.emplace(key, id);
          face_owner.push_back(ids);
        } else {
          id = it->second;
        }
        fid[e * nlf + f] = id;
        // owner-frame lattice positions of the owner's corners
        const auto& ow = face_owner[id];
        auto posof = [&](int64_t v, int* pp) {
          // first match, as a dict built from the owner tuple keeps the last
          // duplicate; faces of valid meshes have 4 distinct vertices
          int idx = -1;
          for (int c = 0; c < 4; ++c)
            if (ow[c] == v) idx = c;
          pp[0] = (idx == 1 || idx == 3) ? p : 0;
          pp[1] = (idx == 2 || idx == 3) ? p : 0;
          return idx >= 0;
        };
        int p0[2], p1[2], p2[2];
        if (!posof(ids[0], p0) || !posof(ids[1], p1) || !posof(ids[2], p2)) {
          fb::set_error("non-conforming face connectivity");
          return -FB_ERR_ARG;
        }
        const int ex0 = (p1[0] - p0[0]) / p, ex1 = (p1[1] - p0[1]) / p;
        const int ey0 = (p2[0] - p0[0]) / p, ey1 = (p2[1] - p0[1]) / p;
        if (std::abs(ex0) + std::abs(ex1) != 1 || std::abs(ey0) + std::abs(ey1) != 1) {
          fb::set_error("non-conforming face connectivity");
          return -FB_ERR_ARG;
        }
        ftr[e * nlf + f] = {p0[0], p0[1], ex0, ex1, ey0, ey1};
      }
    }
  }
  const int64_t n_edges = int64_t(edge_owner.size());
  const int64_t n_faces = int64_t(face_owner.size());
  if (num_edges) *num_edges = n_edges;
  if (num_faces) *num_faces = n_faces;
  const int nloc = d == 2 ? n * n : n * n * n;
  if (p == 1) {
    for (int64_t k = 0; k < ne * nloc; ++k) out[k] = elems[k];
    return nv;
  }
  const int64_t per_edge = p - 1, per_face = int64_t(p - 1) * (p - 1);
  const int64_t per_int = d == 2 ? per_face : per_face * (p - 1);
  const int64_t edge_base = nv;
  const int64_t face_base = edge_base + n_edges * per_edge;
  const int64_t int_base = face_base + n_faces * per_face;
  const int64_t ndofs = int_base + ne * per_int;

  for (int l = 0; l < nloc; ++l) {
    int pos[3] = {0, 0, 0};
    bool on_end[3] = {false, false, false};
    int n_int = 0;
    for (int a = 0; a < d; ++a) {
      int v = l;
      for (int s = 0; s < a; ++s) v /= n;
      pos[a] = v % n;
      on_end[a] = (pos[a] == 0 || pos[a] == p);
      if (!on_end[a]) ++n_int;
    }
    if (n_int == 0) {
      int bits[3];
      for (int a = 0; a < d; ++a) bits[a] = pos[a] / p;
      const int c = corner_of(bits, d);
      for (int64_t e = 0; e < ne; ++e) out[e * nloc + l] = elems[e * ncorner + c];
    } else if (n_int == 1) {
      int a = 0;
      while (on_end[a]) ++a;
      int le;
      if (d == 2) {
        le = a * 2 + pos[1 - a] / p;
      } else {
        int o[2], k = 0;
        for (int x = 0; x < 3; ++x)
          if (x != a) o[k++] = x;
        le = a * 4 + (pos[o[1]] / p) * 2 + (pos[o[0]] / p);
      }
      const int kpos = pos[a] - 1;
      for (int64_t e = 0; e < ne; ++e) {
        const int kk = eflip[e * nle + le] ? (p - 2 - kpos) : kpos;
        out[e * nloc + l] = edge_base + eid[e * nle + le] * per_edge + kk;
      }
    } else if (n_int == 2 && d == 3) {
      int fa = 0;
      while (!on_end[fa]) ++fa;
      const int side = pos[fa] / p;
      const int f = 2 * fa + side;
      int t[2], k = 0;
      for (int x = 0; x < 3; ++x)
        if (x != fa) t[k++] = x;
      const int s = pos[t[0]], tt = pos[t[1]];
      for (int64_t e = 0; e < ne; ++e) {
        const auto& tr = ftr[e * nlf + f];
        const int64_t S = tr[0] + int64_t(s) * tr[2] + int64_t(tt) * tr[4];
        const int64_t T = tr[1] + int64_t(s) * tr[3] + int64_t(tt) * tr[5];
        out[e * nloc + l] = face_base + fid[e * nlf + f] * per_face + (S - 1) + per_edge * (T - 1);
      }
    } else {
      int64_t idx = 0, stride = 1;
      for (int a = 0; a < d; ++a) {
        idx += int64_t(pos[a] - 1) * stride;
        stride *= (p - 1);
      }
      for (int64_t e = 0; e < ne; ++e) out[e * nloc + l] = int_base + e * per_int + idx;
    }
  }
  return ndofs;
}
