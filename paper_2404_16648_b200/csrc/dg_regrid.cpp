// dg_regrid.cpp -- NEXT-1 host regrid planner (PAPER.md:207-215
// §3.2.1; readings R37-R39 of DESIGN.md).
//
// From the current leaf list (level + integer anchor, Morton order) and one
// refinement indicator per leaf it produces the next leaf list (Morton order)
// and the transfer maps the device kernels consume (dg_amr_project_refine /
// dg_amr_project_coarsen / dg_copy_elements):
//
//   1. feature set  T0 = { e : eta_e > refine_above }
//   2. buffer       T  = T0 dilated by B rounds; one round = a face-neighbour
//                  sweep along x, then along y (then z) of the grown set (R37)
//   3. refine       every leaf of T below max_level -> 2^dim children, then the
//                  2:1 face balance ripple (coarser neighbours refined, R15)
//   4. coarsen      finest level first: a family whose 2^dim children are all
//                  still leaves, all with eta < coarsen_below and none in T,
//                  merges into its parent unless the parent would touch a leaf
//                  two levels finer (R38)
//   5. output       new leaves in Morton order (R27); every new leaf is an old
//                  leaf (copy), a child of a refined old leaf, or the parent of
//                  a coarsened old family (one level per regrid).
//
// Plain integer work on hash maps; independent of oracle/regrid.py.
#include <cuda_runtime.h>  // dg_internal.h uses __host__ __device__

#include <algorithm>
#include <cstdint>
#include <unordered_map>
#include <vector>

#include "dg_internal.h"

namespace dgi {

namespace {

inline uint64_t lkey(int l, int a0, int a1, int a2) {
  return ((uint64_t)l << 60) | ((uint64_t)a0 << 40) | ((uint64_t)a1 << 20) | (uint64_t)a2;
}

struct Leaf {
  int l;
  int a[3];
};

struct Forest {
  int dim, max_level;
  int root[3];
  int periodic[3];
  std::unordered_map<uint64_t, int> idx;  // leaf key -> slot in `leaves`
  std::vector<Leaf> leaves;
  std::vector<char> alive;

  bool is_leaf(int l, const int* a) const { return idx.count(lkey(l, a[0], a[1], a[2])) != 0; }
  int find(int l, const int* a) const {
    auto it = idx.find(lkey(l, a[0], a[1], a[2]));
    return it == idx.end() ? -1 : it->second;
  }
  int add(int l, const int* a) {
    Leaf f{l, {a[0], a[1], a[2]}};
    leaves.push_back(f);
    alive.push_back(1);
    const int s = (int)leaves.size() - 1;
    idx[lkey(l, a[0], a[1], a[2])] = s;
    return s;
  }
  void kill(int s) {
    const Leaf& f = leaves[s];
    idx.erase(lkey(f.l, f.a[0], f.a[1], f.a[2]));
    alive[s] = 0;
  }
  // cell across face (d, sgn) of cell (l, a) at level l; false at a wall
  bool across(int l, const int* a, int d, int sgn, int* out) const {
    for (int t = 0; t < 3; ++t) out[t] = a[t];
    const int64_t ext = (int64_t)root[d] << l;
    int64_t m = (int64_t)a[d] + sgn;
    if (m < 0 || m >= ext) {
      if (!periodic[d]) return false;
      m = (m + ext) % ext;
    }
    out[d] = (int)m;
    return true;
  }
  // level of the leaf containing cell (l, c), or -1 if that cell is subdivided
  int containing(int l, const int* c) const {
    for (int k = l; k >= 0; --k) {
      const int sh = l - k;
      int b[3] = {c[0] >> sh, c[1] >> sh, c[2] >> sh};
      if (is_leaf(k, b)) return k;
    }
    return -1;
  }
  // leaves of the (balanced) forest across face (d, sgn) of leaf s
  void face_neighbours(int s, int d, int sgn, std::vector<int>& out) const {
    const Leaf& f = leaves[s];
    int nb[3];
    if (!across(f.l, f.a, d, sgn, nb)) return;
    int j = find(f.l, nb);
    if (j >= 0) {
      out.push_back(j);
      return;
    }
    if (f.l > 0) {
      int up[3] = {nb[0] >> 1, nb[1] >> 1, nb[2] >> 1};
      j = find(f.l - 1, up);
      if (j >= 0) {
        out.push_back(j);
        return;
      }
    }
    // finer: the 2^(dim-1) children of the neighbour cell on the shared face
    const int nsub = 1 << (dim - 1);
    for (int b = 0; b < nsub; ++b) {
      int c[3] = {2 * nb[0], 2 * nb[1], 2 * nb[2]};
      if (sgn < 0) c[d] += 1;
      int k = 0;
      for (int t = 0; t < dim; ++t)
        if (t != d) c[t] += (b >> k++) & 1;
      j = find(f.l + 1, c);
      if (j >= 0) out.push_back(j);
    }
  }
};

uint64_t morton(const Leaf& f, int dim, int max_level) {
  uint64_t key = 0;
  int fine[3];
  for (int d = 0; d < 3; ++d) fine[d] = d < dim ? (f.a[d] << (max_level - f.l)) : 0;
  for (int bit = 0; bit < 20; ++bit)
    for (int d = 0; d < dim; ++d) key |= (uint64_t)((fine[d] >> bit) & 1) << (bit * dim + d);
  return key;
}

}  // namespace

int regrid_plan(const RegridIn& in, RegridOut& out, const char** why) {
  const int dim = in.dim;
  const int64_t E = in.n;
  Forest F;
  F.dim = dim;
  F.max_level = in.max_level;
  for (int d = 0; d < 3; ++d) {
    F.root[d] = d < dim ? in.root[d] : 1;
    F.periodic[d] = d < dim ? in.periodic[d] : 0;
  }
  F.leaves.reserve((size_t)E * 2);
  F.idx.reserve((size_t)E * 4);
  for (int64_t e = 0; e < E; ++e) {
    int a[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) a[d] = in.anchor[e * dim + d];
    F.add(in.level[e], a);
  }
  std::unordered_map<uint64_t, int> old_idx(F.idx);  // old leaves by key (kept after they die)
  auto old_of = [&](int l, int a0, int a1, int a2) -> int {
    auto it = old_idx.find(lkey(l, a0, a1, a2));
    return it == old_idx.end() ? -1 : it->second;
  };
  // 1-2: feature set and buffer (slots 0..E-1 are the old leaves)
  std::vector<char> inT((size_t)E, 0);
  std::vector<int> cur;
  for (int64_t e = 0; e < E; ++e)
    if (in.eta[e] > in.refine_above) {
      inT[e] = 1;
      cur.push_back((int)e);
    }
  std::vector<int> nb;
  for (int r = 0; r < in.buffer; ++r)
    for (int d = 0; d < dim; ++d) {
      std::vector<int> add;
      for (int s : cur)
        for (int sg = -1; sg <= 1; sg += 2) {
          nb.clear();
          F.face_neighbours(s, d, sg, nb);
          for (int j : nb)
            if (!inT[j]) {
              inT[j] = 1;
              add.push_back(j);
            }
        }
      cur.insert(cur.end(), add.begin(), add.end());
    }
  // 3: refine T below max_level, then the balance ripple
  const int nch = 1 << dim;
  std::vector<char> refined((size_t)E, 0);
  std::vector<int> work;
  auto split = [&](int s) {
    const Leaf f = F.leaves[s];
    F.kill(s);
    if (s < E) refined[s] = 1;
    for (int b = 0; b < nch; ++b) {
      int c[3] = {2 * f.a[0] + (b & 1), dim > 1 ? 2 * f.a[1] + ((b >> 1) & 1) : 0,
                  dim > 2 ? 2 * f.a[2] + ((b >> 2) & 1) : 0};
      if (dim == 2) c[2] = 0;
      work.push_back(F.add(f.l + 1, c));
    }
  };
  for (int64_t e = 0; e < E; ++e)
    if (inT[e] && F.leaves[e].l < in.max_level) split((int)e);
  while (!work.empty()) {
    const int s = work.back();
    work.pop_back();
    if (!F.alive[s]) continue;
    const Leaf f = F.leaves[s];
    for (int d = 0; d < dim; ++d)
      for (int sg = -1; sg <= 1; sg += 2) {
        int c[3];
        if (!F.across(f.l, f.a, d, sg, c)) continue;
        for (;;) {
          const int lc = F.containing(f.l, c);
          if (lc < 0 || lc >= f.l - 1) break;
          const int sh = f.l - lc;
          int up[3] = {c[0] >> sh, c[1] >> sh, c[2] >> sh};
          const int j = F.find(lc, up);
          if (j < 0) break;
          if (F.leaves[j].l >= in.max_level) {
            *why = "regrid: balance ripple exceeds max_level";
            return -1;
          }
          split(j);
        }
      }
  }
  // 4: coarsening, finest level first
  std::vector<char> coarsened((size_t)E, 0);
  for (int l = in.max_level; l >= 1; --l) {
    for (int64_t e = 0; e < E; ++e) {
      const Leaf& f = F.leaves[e];
      if (f.l != l || !F.alive[e] || coarsened[e]) continue;
      bool first = true;
      for (int d = 0; d < dim; ++d) first = first && (f.a[d] & 1) == 0;
      if (!first) continue;
      // the family: all children alive old leaves, tagged, not in T
      int kids[8];
      bool ok = true;
      for (int b = 0; b < nch && ok; ++b) {
        int c[3] = {f.a[0] + (b & 1), dim > 1 ? f.a[1] + ((b >> 1) & 1) : 0, dim > 2 ? f.a[2] + ((b >> 2) & 1) : 0};
        const int j = F.find(l, c);
        ok = j >= 0 && j < E && F.alive[j] && !inT[j] && in.eta[j] < in.coarsen_below;
        kids[b] = j;
      }
      if (!ok) continue;
      // balance: no leaf finer than l may touch the parent's faces
      int P[3] = {f.a[0] >> 1, f.a[1] >> 1, f.a[2] >> 1};
      for (int d = 0; d < dim && ok; ++d)
        for (int sg = -1; sg <= 1 && ok; sg += 2) {
          int nbc[3];
          if (!F.across(l - 1, P, d, sg, nbc)) continue;
          if (F.containing(l - 1, nbc) >= 0) continue;  // a leaf at level <= l-1
          const int nsub = 1 << (dim - 1);
          for (int b = 0; b < nsub && ok; ++b) {
            int c[3] = {2 * nbc[0], 2 * nbc[1], 2 * nbc[2]};
            if (sg < 0) c[d] += 1;
            int k = 0;
            for (int t = 0; t < dim; ++t)
              if (t != d) c[t] += (b >> k++) & 1;
            ok = F.is_leaf(l, c);
          }
        }
      if (!ok) continue;
      for (int b = 0; b < nch; ++b) {
        F.kill(kids[b]);
        coarsened[kids[b]] = 1;
      }
      F.add(l - 1, P);
    }
  }
  // 5: output in Morton order and the transfer maps
  std::vector<int> live;
  for (size_t s = 0; s < F.leaves.size(); ++s)
    if (F.alive[s]) live.push_back((int)s);
  std::vector<std::pair<uint64_t, int>> ord;
  ord.reserve(live.size());
  for (int s : live) ord.emplace_back(morton(F.leaves[s], dim, in.max_level), s);
  std::sort(ord.begin(), ord.end());
  const int64_t En = (int64_t)ord.size();
  out.level.assign((size_t)En, 0);
  out.anchor.assign((size_t)En * dim, 0);
  out.refine_parent.clear();
  out.refine_child0.clear();
  out.coarsen_child0.clear();
  out.coarsen_parent.clear();
  out.copy_src.clear();
  out.copy_dst.clear();
  for (int64_t i = 0; i < En; ++i) {
    const Leaf& f = F.leaves[ord[i].second];
    out.level[i] = (int8_t)f.l;
    for (int d = 0; d < dim; ++d) out.anchor[i * dim + d] = f.a[d];
  }
  for (int64_t i = 0; i < En; ++i) {
    const int s = ord[i].second;
    if (s < E) {  // unchanged old leaf
      out.copy_src.push_back(s);
      out.copy_dst.push_back((int32_t)i);
      continue;
    }
    const Leaf& f = F.leaves[s];
    // child of a refined old leaf?
    bool first = true;
    for (int d = 0; d < dim; ++d) first = first && (f.a[d] & 1) == 0;
    const int parent_old = f.l > 0 ? old_of(f.l - 1, f.a[0] >> 1, f.a[1] >> 1, f.a[2] >> 1) : -1;
    if (parent_old >= 0 && refined[parent_old]) {
      if (first) {
        out.refine_parent.push_back(parent_old);
        out.refine_child0.push_back((int32_t)i);
      }
      continue;
    }
    // parent of a coarsened old family: its first child is an old leaf
    const int c0[3] = {2 * f.a[0], dim > 1 ? 2 * f.a[1] : 0, dim > 2 ? 2 * f.a[2] : 0};
    const int j0 = old_of(f.l + 1, c0[0], c0[1], c0[2]);
    if (j0 < 0 || !coarsened[j0]) {
      *why = "regrid: internal error (new leaf of unknown origin)";
      return -1;
    }
    // the old family must be consecutive in the old order for the coarsen kernel
    for (int b = 1; b < nch; ++b) {
      if (old_of(f.l + 1, c0[0] + (b & 1), dim > 1 ? c0[1] + ((b >> 1) & 1) : 0,
                 dim > 2 ? c0[2] + ((b >> 2) & 1) : 0) != j0 + b) {
        *why = "regrid: the old mesh is not in Morton order (siblings not consecutive)";
        return -2;
      }
    }
    out.coarsen_child0.push_back(j0);
    out.coarsen_parent.push_back((int32_t)i);
  }
  return 0;
}

}  // namespace dgi
