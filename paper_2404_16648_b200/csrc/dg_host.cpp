// dg_host.cpp -- libdg host runtime: C ABI (include/dg.h), operator set,
// connectivity build, device tables, argument checking and kernel dispatch.
//
// Independent of oracle/: the 1D operators here are built in long double by
// a different route (Newton on P_N', the classical closed-form D, P_b as the
// interpolation matrix, R_b = 1/2 M^-1 P_b^T M with M from the Legendre
// Vandermonde), and the connectivity is derived from per-element face
// descriptors rather than from the oracle's face-list pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dg.h"
#include "dg_internal.h"

using dgi::ElemDesc;

namespace {

thread_local std::string g_err;

dg_status fail(dg_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

dg_status cuda_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) return fail(DG_ERR_OOM, "%s: %s", where, cudaGetErrorString(e));
  return fail(DG_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CUDA_TRY(call, where)                      \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

typedef long double LD;

// Legendre P_N and P_N' at x (recurrences P_{k+1} = ((2k+1)xP_k - kP_{k-1})/(k+1),
// P'_{k+1} = P'_{k-1} + (2k+1) P_k).
void legendre(int N, LD x, LD* P, LD* dP) {
  LD p0 = 1, p1 = x, d0 = 0, d1 = 1;
  if (N == 0) { *P = 1; *dP = 0; return; }
  for (int k = 1; k < N; ++k) {
    LD p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    LD d2 = d0 + (2 * k + 1) * p1;
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  *P = p1;
  *dP = d1;
}

struct Basis {
  int N;
  std::vector<double> x, w, D, P[2], R[2];
  std::vector<LD> xl;  // nodes in long double
  std::vector<LD> Dl;  // D in long double (source of the even-odd split)
};

// Gauss-Jordan inverse (long double).
std::vector<LD> inverse(std::vector<LD> a, int n) {
  std::vector<LD> b(n * n, 0);
  for (int i = 0; i < n; ++i) b[i * n + i] = 1;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (fabsl(a[r * n + c]) > fabsl(a[piv * n + c])) piv = r;
    for (int k = 0; k < n; ++k) { std::swap(a[c * n + k], a[piv * n + k]); std::swap(b[c * n + k], b[piv * n + k]); }
    LD d = a[c * n + c];
    for (int k = 0; k < n; ++k) { a[c * n + k] /= d; b[c * n + k] /= d; }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      LD f = a[r * n + c];
      for (int k = 0; k < n; ++k) { a[r * n + k] -= f * a[c * n + k]; b[r * n + k] -= f * b[c * n + k]; }
    }
  }
  return b;
}

Basis make_basis(int N) {
  const int n1 = N + 1;
  std::vector<LD> x(n1);
  x[0] = -1;
  x[N] = 1;
  // interior LGL nodes: roots of P_N' by Newton with P_N'' from Legendre's ODE
  for (int i = 1; i < N; ++i) {
    LD xi = -cosl(3.141592653589793238462643383279502884L * i / N);
    for (int it = 0; it < 100; ++it) {
      LD P, dP;
      legendre(N, xi, &P, &dP);
      LD d2P = (2 * xi * dP - (LD)N * (N + 1) * P) / (1 - xi * xi);
      LD dx = dP / d2P;
      xi -= dx;
      if (fabsl(dx) < 1e-19L) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i < n1 / 2; ++i) {  // exact symmetry
    LD s = (x[N - i] - x[i]) / 2;
    x[i] = -s;
    x[N - i] = s;
  }
  if (N % 2 == 0) x[N / 2] = 0;
  std::vector<LD> PN(n1), w(n1);
  for (int i = 0; i < n1; ++i) {
    LD dP;
    legendre(N, x[i], &PN[i], &dP);
    w[i] = 2.0L / ((LD)N * (N + 1) * PN[i] * PN[i]);
  }
  Basis b;
  b.N = N;
  b.x.resize(n1);
  b.w.resize(n1);
  b.D.resize(n1 * n1);
  b.Dl.resize(n1 * n1);
  b.xl.assign(x.begin(), x.begin() + n1);
  for (int i = 0; i < n1; ++i) {
    b.x[i] = (double)x[i];
    b.w[i] = (double)w[i];
  }
  // classical LGL differentiation matrix
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      LD v;
      if (i != j) v = (PN[i] / PN[j]) / (x[i] - x[j]);
      else if (i == 0) v = -(LD)N * (N + 1) / 4;
      else if (i == N) v = (LD)N * (N + 1) / 4;
      else v = 0;
      b.D[i * n1 + j] = (double)v;
      b.Dl[i * n1 + j] = v;
    }
  // exact mass matrix M = V^-T diag(2/(2k+1)) V^-1, V_ik = P_k(x_i)
  std::vector<LD> V(n1 * n1);
  for (int i = 0; i < n1; ++i)
    for (int k = 0; k < n1; ++k) {
      LD P, dP;
      legendre(k, x[i], &P, &dP);
      V[i * n1 + k] = P;
    }
  std::vector<LD> Vi = inverse(V, n1);
  std::vector<LD> M(n1 * n1, 0), Minv(n1 * n1, 0);
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      LD s = 0, t = 0;
      for (int k = 0; k < n1; ++k) {
        s += Vi[k * n1 + i] * (2.0L / (2 * k + 1)) * Vi[k * n1 + j];
        t += V[i * n1 + k] * ((2 * k + 1) / 2.0L) * V[j * n1 + k];
      }
      M[i * n1 + j] = s;
      Minv[i * n1 + j] = t;
    }
  for (int bb = 0; bb < 2; ++bb) {
    // P_b: L2 projection face -> mortar of a degree-N polynomial = interpolation
    std::vector<LD> Pb(n1 * n1);
    for (int k = 0; k < n1; ++k) {
      LD t = bb == 0 ? (x[k] - 1) / 2 : (x[k] + 1) / 2;
      for (int j = 0; j < n1; ++j) {
        LD l = 1;
        for (int m = 0; m < n1; ++m)
          if (m != j) l *= (t - x[m]) / (x[j] - x[m]);
        Pb[k * n1 + j] = l;
      }
    }
    // R_b = 1/2 M^-1 S_b^T with S_b = M P_b  =>  R_b = 1/2 M^-1 P_b^T M
    std::vector<LD> T(n1 * n1, 0);
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        LD s = 0;
        for (int k = 0; k < n1; ++k) s += Pb[k * n1 + i] * M[k * n1 + j];
        T[i * n1 + j] = s;  // (P^T M)_ij
      }
    b.P[bb].resize(n1 * n1);
    b.R[bb].resize(n1 * n1);
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        LD s = 0;
        for (int k = 0; k < n1; ++k) s += Minv[i * n1 + k] * T[k * n1 + j];
        b.R[bb][i * n1 + j] = (double)(s / 2);
        b.P[bb][i * n1 + j] = (double)Pb[i * n1 + j];
      }
  }
  return b;
}

}  // namespace

struct dg_ctx {
  dg_params p;
  int dim, N, n1, Np, F;
  int64_t stride;
  Basis basis;
  std::vector<double> ops;  // OpsLayout
  std::vector<long> rowoff;
  int64_t n_rows_expected;
  // host mesh
  bool have_mesh = false;
  int64_t n_elem = 0;
  std::vector<ElemDesc> desc;
  std::vector<int32_t> nbrow;  // [E][8]: background row of the element across each face (-1 if none)
  std::vector<int32_t> mort;
  std::vector<int32_t> conf, nonconf, bnd;
  std::vector<int8_t> lev;    // current leaf list (regrid planner input)
  std::vector<int32_t> anc;   // [E][dim]
  // NEXT-4 partition (n_parts == 1: whole mesh): kernels compute rows [0, n_elem); state
  // arrays hold n_rows = n_elem + halo rows (remote elements the kernels read)
  int64_t n_rows = 0;
  int32_t n_parts = 1, part = 0;
  int64_t gbegin = 0;
  std::vector<int64_t> send_count, recv_count;
  std::vector<int32_t> send_idx;
  std::vector<int64_t> fsend_count, frecv_count;  // face-trace exchange: (element, face) pairs per peer
  std::vector<int32_t> fsend, frecv;
  // device tables
  bool on_device = false;
  ElemDesc* d_desc = nullptr;
  int32_t* d_nbrow = nullptr;
  int32_t* d_mort = nullptr;
  int32_t* d_mortbg = nullptr;
  int32_t* d_mort_owner = nullptr;  // [n_mort][16] record of each local coarse face (k_mortar_h4; see upload_tables)
  double* d_mlift = nullptr;        // [n_mort][F][Nf] coarse-side lift values (k_mortar_h4 -> k_stage_h4)
  int64_t n_mort = 0;
  double* d_ops = nullptr;
  double* d_bg = nullptr;   // (rho_bar, Theta_bar, P_bar) as given
  double* d_bg4 = nullptr;  // + 1/Theta_bar, 32-B rows (kernel layout)
  int64_t bg_rows = 0;
  double De[dgi::kMaxH * dgi::kMaxH] = {0}, Do[dgi::kMaxH * dgi::kMaxH] = {0};
  double eos_c[dgi::kEosTerms] = {0};
  double* d_partial = nullptr;
  double* d_jac = nullptr;
  unsigned long long* d_check = nullptr;  // dg_check_state counters (4)
  // scratch for *_host variants
  double* d_scratch[3] = {nullptr, nullptr, nullptr};
  int64_t launches = 0;
  int32_t ncmode = 0;  // NEXT-3: 2:1 face treatment (0 mortar, 1 pointwise interpolation)
  bool has_nc = false;  // some local element has a 2:1 face (set at upload; selects the stage kernel)
  int h4_amr = 2;  // env DG_H4_AMR at dg_create, 3D N = 4 meshes with 2:1 faces: 0 generic tile kernel,
                   // 1 k_stage_h4 with its inline mortar steps, 2 (default) mortar pre-pass (k_mortar_h4) +
                   // k_stage_h4 (c4 RK3 step 2.02 -> 1.79 ms)
  double mu = 0.0;     // NEXT-3: artificial viscosity (0: off)
  double* d_sig = nullptr;   // viscous scratch: gradients (dim rows per element) and V
  double* d_visc = nullptr;
  int64_t visc_rows = 0;
};

namespace {

void free_device(dg_ctx* c) {
  cudaFree(c->d_desc);
  cudaFree(c->d_nbrow);
  c->d_nbrow = nullptr;
  cudaFree(c->d_mort);
  cudaFree(c->d_mortbg);
  c->d_mortbg = nullptr;
  cudaFree(c->d_mort_owner);
  c->d_mort_owner = nullptr;
  cudaFree(c->d_mlift);
  c->d_mlift = nullptr;
  c->n_mort = 0;
  cudaFree(c->d_partial);
  for (auto& s : c->d_scratch) {
    cudaFree(s);
    s = nullptr;
  }
  c->d_desc = nullptr;
  c->d_mort = nullptr;
  c->d_partial = nullptr;
  c->on_device = false;
}

dg_status build_mesh(dg_ctx* c, int64_t n, const int8_t* level, const int32_t* anchor) {
  const dg_params& p = c->p;
  const int dim = c->dim;
  if (n < 1 || !level || !anchor) return fail(DG_ERR_ARG, "mesh: n_leaves < 1 or null array");
  if (n > (int64_t)INT32_MAX / 8) return fail(DG_ERR_ARG, "mesh: too many leaves");
  c->have_mesh = false;
  auto key = [](int l, int a0, int a1, int a2) -> uint64_t {
    return ((uint64_t)l << 60) | ((uint64_t)a0 << 40) | ((uint64_t)a1 << 20) | (uint64_t)a2;
  };
  std::unordered_map<uint64_t, int32_t> leaf;
  leaf.reserve((size_t)n * 2);
  std::vector<int> A((size_t)n * 3, 0), L((size_t)n);
  for (int64_t e = 0; e < n; ++e) {
    int l = level[e];
    if (l < 0 || l > p.max_level) return fail(DG_ERR_MESH, "mesh: leaf %lld level %d outside 0..%d", (long long)e, l, p.max_level);
    L[e] = l;
    for (int d = 0; d < dim; ++d) {
      int a = anchor[e * dim + d];
      if (a < 0 || (int64_t)a >= ((int64_t)p.root[d] << l))
        return fail(DG_ERR_MESH, "mesh: leaf %lld anchor out of range on axis %d", (long long)e, d);
      A[e * 3 + d] = a;
    }
    if (!leaf.emplace(key(l, A[e * 3], A[e * 3 + 1], A[e * 3 + 2]), (int32_t)e).second)
      return fail(DG_ERR_MESH, "mesh: duplicate leaf %lld", (long long)e);
  }
  for (int64_t e = 0; e < n; ++e)
    for (int up = 1; up <= L[e]; ++up)
      if (leaf.count(key(L[e] - up, A[e * 3] >> up, A[e * 3 + 1] >> up, A[e * 3 + 2] >> up)))
        return fail(DG_ERR_MESH, "mesh: leaf %lld overlaps an ancestor leaf", (long long)e);
  {
    unsigned __int128 vol = 0, dom = 1;
    for (int d = 0; d < dim; ++d) dom *= (unsigned __int128)p.root[d] << p.max_level;
    for (int64_t e = 0; e < n; ++e) vol += (unsigned __int128)1 << (dim * (p.max_level - L[e]));
    if (vol != dom) return fail(DG_ERR_MESH, "mesh: leaves do not tile the domain (gap)");
  }
  const int nsub = 1 << (dim - 1);
  std::vector<ElemDesc> desc((size_t)n);
  std::vector<int32_t> mort;
  for (int64_t e = 0; e < n; ++e) {
    ElemDesc& D = desc[e];
    const int l = L[e];
    int info = l << 24;
    for (int f = 0; f < 6; ++f) D.nbr[f] = -1;
    for (int f = 0; f < 2 * dim; ++f) {
      const int d = f >> 1, s = (f & 1) ? 1 : -1;
      int nb[3] = {A[e * 3], A[e * 3 + 1], A[e * 3 + 2]};
      const int64_t ext = (int64_t)p.root[d] << l;
      int64_t m = (int64_t)nb[d] + s;
      if (m < 0 || m >= ext) {
        if (!p.periodic[d]) {
          info |= dgi::kWall << (2 * f);
          continue;
        }
        m = (m + ext) % ext;
      }
      nb[d] = (int)m;
      auto it = leaf.find(key(l, nb[0], nb[1], nb[2]));
      if (it != leaf.end()) {
        D.nbr[f] = it->second;  // kConf == 0
        continue;
      }
      if (l > 0) {
        auto jt = leaf.find(key(l - 1, nb[0] >> 1, nb[1] >> 1, nb[2] >> 1));
        if (jt != leaf.end()) {
          int bsub = 0, k = 0;
          for (int t = 0; t < dim; ++t)
            if (t != d) bsub |= (A[e * 3 + t] & 1) << k++;
          D.nbr[f] = jt->second;
          info |= dgi::kFine << (2 * f);
          info |= bsub << (12 + 2 * f);
          continue;
        }
      }
      if (l + 1 > p.max_level)
        return fail(DG_ERR_UNBALANCED, "mesh: leaf %lld face %d: neighbour more than one level coarser", (long long)e, f);
      int32_t kids[4];
      for (int b = 0; b < nsub; ++b) {
        int c3[3] = {2 * nb[0], 2 * nb[1], 2 * nb[2]};
        if (s < 0) c3[d] += 1;
        int k = 0;
        for (int t = 0; t < dim; ++t)
          if (t != d) c3[t] += (b >> k++) & 1;
        auto kt = leaf.find(key(l + 1, c3[0], c3[1], c3[2]));
        if (kt == leaf.end())
          return fail(DG_ERR_UNBALANCED, "mesh: leaf %lld face %d: 2:1 balance violated", (long long)e, f);
        kids[b] = kt->second;
      }
      D.nbr[f] = (int32_t)(mort.size() / nsub);
      for (int b = 0; b < nsub; ++b) mort.push_back(kids[b]);
      info |= dgi::kCoarse << (2 * f);
    }
    D.info = info;
    D.bgrow = (int32_t)(c->rowoff[l] + (int64_t)A[e * 3 + c->dim - 1] * c->n1);
  }
  // canonical face lists from the descriptors (R29)
  c->conf.clear();
  c->nonconf.clear();
  c->bnd.clear();
  for (int64_t e = 0; e < n; ++e) {
    for (int f = 0; f < 2 * dim; ++f) {
      int k = dgi::face_kind(desc[e].info, f);
      if (k == dgi::kWall) {
        c->bnd.push_back((int32_t)e);
        c->bnd.push_back(f);
      } else if (k == dgi::kConf && (f & 1)) {
        c->conf.insert(c->conf.end(), {(int32_t)e, f, desc[e].nbr[f], f - 1});
      } else if (k == dgi::kCoarse) {
        c->nonconf.push_back((int32_t)e);
        c->nonconf.push_back(f);
        for (int b = 0; b < nsub; ++b) {
          c->nonconf.push_back(mort[(size_t)desc[e].nbr[f] * nsub + b]);
          c->nonconf.push_back(f ^ 1);
        }
      }
    }
  }
  // background row of the conforming neighbour / coarse element across each face (kernels
  // read it with the descriptor instead of chasing the neighbour's descriptor)
  std::vector<int32_t> nbrow((size_t)n * 8, -1);
  for (int64_t e = 0; e < n; ++e)
    for (int f = 0; f < 2 * c->dim; ++f) {
      const int k = dgi::face_kind(desc[e].info, f);
      if (k == dgi::kConf || k == dgi::kFine) nbrow[(size_t)e * 8 + f] = desc[desc[e].nbr[f]].bgrow;
    }
  c->desc.swap(desc);
  c->nbrow.swap(nbrow);
  c->mort.swap(mort);
  c->lev.assign(level, level + n);
  c->anc.assign(anchor, anchor + n * dim);
  c->n_elem = n;
  c->n_rows = n;
  c->n_parts = 1;
  c->part = 0;
  c->gbegin = 0;
  c->send_count.clear();
  c->recv_count.clear();
  c->send_idx.clear();
  c->have_mesh = true;
  return DG_OK;
}

// NEXT-4: restrict a built (global) mesh to part `part` of `np` contiguous Morton ranges
// (space-filling-curve partition) plus its halo.  Face neighbours are mutual
// (conforming pairs, coarse face <-> its fine elements), so the rows part r sends to part k
// are exactly the rows k lists as its halo from r, both in global order.
dg_status build_part(dg_ctx* c, int np, int part) {
  const int64_t n = c->n_elem;
  const int dim = c->dim, nsub = 1 << (dim - 1);
  if (np < 1 || part < 0 || part >= np) return fail(DG_ERR_ARG, "partition: part %d of %d", part, np);
  // cut k (first leaf of part k) = the SFC position n k / np (R40), moved forward past any leaf whose
  // predecessor is its sibling (same level >= 1, same parent: anchor >> 1 on every axis), so that
  // no family of sibling leaves -- consecutive in Morton order (R27), the unit of a coarsening --
  // is split between parts (P:183 SFC partition)
  auto siblings = [&](int64_t x, int64_t y) {
    if (c->lev[x] != c->lev[y] || c->lev[x] == 0) return false;
    for (int d = 0; d < dim; ++d)
      if ((c->anc[(size_t)x * dim + d] >> 1) != (c->anc[(size_t)y * dim + d] >> 1)) return false;
    return true;
  };
  std::vector<int64_t> bnd((size_t)np + 1);
  bnd[0] = 0;
  bnd[np] = n;
  for (int k = 1; k < np; ++k) {
    int64_t g = std::max(n * k / np, bnd[k - 1]);
    while (g > 0 && g < n && siblings(g - 1, g)) ++g;
    bnd[k] = g;
  }
  const int64_t b = bnd[part], e = bnd[part + 1], nl = e - b;
  if (nl < 1) return fail(DG_ERR_ARG, "partition: part %d of %d is empty (%lld leaves)", part, np, (long long)n);
  auto owner = [&](int64_t g) { return (int)(std::upper_bound(bnd.begin(), bnd.end(), g) - bnd.begin()) - 1; };
  const std::vector<ElemDesc>& G = c->desc;
  auto each_nbr = [&](int64_t g, auto&& fn) {
    for (int f = 0; f < 2 * dim; ++f) {
      const int k = dgi::face_kind(G[g].info, f);
      if (k == dgi::kConf || k == dgi::kFine) fn((int64_t)G[g].nbr[f]);
      else if (k == dgi::kCoarse)
        for (int s = 0; s < nsub; ++s) fn((int64_t)c->mort[(size_t)G[g].nbr[f] * nsub + s]);
    }
  };
  std::vector<std::vector<int64_t>> need((size_t)np), give((size_t)np);
  std::vector<char> needed((size_t)n, 0);
  std::vector<int> seen((size_t)np, -1);
  for (int64_t g = b; g < e; ++g)
    each_nbr(g, [&](int64_t h) {
      const int k = owner(h);
      if (k == part) return;
      if (!needed[h]) {
        needed[h] = 1;
        need[k].push_back(h);
      }
      if (seen[k] != (int)(g - b)) {
        seen[k] = (int)(g - b);
        give[k].push_back(g);
      }
    });
  std::vector<int32_t> lidx((size_t)n, -1);
  for (int64_t g = b; g < e; ++g) lidx[g] = (int32_t)(g - b);
  int64_t pos = nl;
  for (int k = 0; k < np; ++k) {
    std::sort(need[k].begin(), need[k].end());
    for (int64_t h : need[k]) lidx[h] = (int32_t)pos++;
  }
  const int64_t nrows = pos;
  std::vector<ElemDesc> d2((size_t)nrows);
  std::vector<int32_t> m2, nb2((size_t)nl * 8);
  for (int64_t g = b; g < e; ++g) {
    ElemDesc D = G[g];
    for (int f = 0; f < 2 * dim; ++f) {
      const int k = dgi::face_kind(G[g].info, f);
      if (k == dgi::kConf || k == dgi::kFine) {
        D.nbr[f] = lidx[G[g].nbr[f]];
      } else if (k == dgi::kCoarse) {
        D.nbr[f] = (int32_t)(m2.size() / nsub);
        for (int s = 0; s < nsub; ++s) m2.push_back(lidx[c->mort[(size_t)G[g].nbr[f] * nsub + s]]);
      }
    }
    d2[g - b] = D;
    std::copy(c->nbrow.begin() + g * 8, c->nbrow.begin() + g * 8 + 8, nb2.begin() + (g - b) * 8);
  }
  for (int k = 0; k < np; ++k)
    for (int64_t h : need[k]) {
      ElemDesc D = G[h];  // halo rows: only bgrow / level are read (mortar fine elements)
      for (int f = 0; f < 6; ++f) D.nbr[f] = -1;
      d2[lidx[h]] = D;
    }
  c->send_count.assign((size_t)np, 0);
  c->recv_count.assign((size_t)np, 0);
  c->send_idx.clear();
  for (int k = 0; k < np; ++k) {
    c->send_count[k] = (int64_t)give[k].size();
    c->recv_count[k] = (int64_t)need[k].size();
    for (int64_t g : give[k]) c->send_idx.push_back((int32_t)(g - b));
  }
  // face-trace exchange: the kernels read only the face nodes of a remote element that touch
  // this part, so per peer the (element, face) pairs whose neighbours lie in the other part
  // (same predicate and order -- element, then face, ascending -- on both sides)
  auto faces_to = [&](int64_t g, int f, int k) {
    const int kind = dgi::face_kind(G[g].info, f);
    if (kind == dgi::kConf || kind == dgi::kFine) return owner(G[g].nbr[f]) == k;
    if (kind == dgi::kCoarse)
      for (int s = 0; s < nsub; ++s)
        if (owner(c->mort[(size_t)G[g].nbr[f] * nsub + s]) == k) return true;
    return false;
  };
  c->fsend_count.assign((size_t)np, 0);
  c->frecv_count.assign((size_t)np, 0);
  c->fsend.clear();
  c->frecv.clear();
  for (int k = 0; k < np; ++k) {
    for (int64_t g : give[k])
      for (int f = 0; f < 2 * dim; ++f)
        if (faces_to(g, f, k)) {
          c->fsend.push_back((int32_t)(g - b));
          c->fsend.push_back(f);
          c->fsend_count[k]++;
        }
    for (int64_t h : need[k])
      for (int f = 0; f < 2 * dim; ++f)
        if (faces_to(h, f, part)) {
          c->frecv.push_back(lidx[h]);
          c->frecv.push_back(f);
          c->frecv_count[k]++;
        }
  }
  c->desc.swap(d2);
  c->nbrow.swap(nb2);
  c->mort.swap(m2);
  c->n_elem = nl;
  c->n_rows = nrows;
  c->n_parts = np;
  c->part = part;
  c->gbegin = b;
  return DG_OK;
}

dg_status check_ready(const dg_ctx* c) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh || !c->on_device) return fail(DG_ERR_MESH, "no mesh uploaded");
  if (!c->d_bg) return fail(DG_ERR_STATE, "no background table set");
  return DG_OK;
}

bool overlaps(const void* a, const void* b, size_t bytes) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + bytes && y < x + bytes;
}

// Debug phase clocks of the stage kernel (env DG_PHASE_PROF=1): a device
// buffer of kProfSlots counters shared by all contexts; read with
// dg_debug_phase_clocks (not part of the ABI in dg.h).
unsigned long long* g_prof = nullptr;
unsigned long long* debug_prof_buffer() {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = std::getenv("DG_PHASE_PROF");
    enabled = (e && e[0] == '1') ? 1 : 0;
    if (enabled && cudaMalloc(&g_prof, sizeof(unsigned long long) * dgi::kProfSlots) == cudaSuccess)
      cudaMemset(g_prof, 0, sizeof(unsigned long long) * dgi::kProfSlots);
    else
      g_prof = nullptr;
  }
  return g_prof;
}

// the stage kernel moves whole element rows with cp.async.bulk (16-B granules)
bool misaligned(const void* p) { return ((uintptr_t)p & 15) != 0; }

// Kernel arguments of one stage / RHS launch over the local elements (or the n_list listed ones).
dgi::StageArgs stage_args(const dg_ctx* c, int mode, int stage, double dt, const double* q_n, const double* q_in,
                          double* out, int64_t n_list = -1, const int32_t* list = nullptr);

dgi::StageArgs stage_args(const dg_ctx* c, int mode, int stage, double dt, const double* q_n, const double* q_in,
                          double* out, int64_t n_list, const int32_t* list) {
  dgi::StageArgs a;
  std::memset(&a, 0, sizeof a);
  a.q_in = q_in;
  a.q_n = q_n;
  a.out = out;
  a.desc = c->d_desc;
  a.nbrow = c->d_nbrow;
  a.mort = c->d_mort;
  a.mortbg = c->d_mortbg;
  a.bg4 = c->d_bg4;
  a.ops = c->d_ops;
  a.n_elem = n_list >= 0 ? n_list : c->n_elem;
  a.list = n_list >= 0 ? list : nullptr;
  a.stride = c->stride;
  a.gamma = c->p.gamma;
  a.g = c->p.g;
  a.w0inv = 1.0 / c->basis.w[0];
  a.dt = dt;
  const double B[3] = {1.0, 1.0 / 4.0, 2.0 / 3.0};
  a.rk_b = B[stage];
  a.stage = stage;
  a.mode = mode;
  a.ncmode = c->ncmode;
  a.amr = (c->has_nc && c->h4_amr == 0) ? 1 : 0;  // 1: the generic tile kernel for this mesh
  a.has_nc = c->has_nc ? 1 : 0;
  a.mort_owner = c->d_mort_owner;
  a.mlift = (c->has_nc && c->h4_amr == 2) ? c->d_mlift : nullptr;  // non-null: pre-pass + k_stage_h4
  a.n_mort = c->n_mort;
  std::memcpy(a.De, c->De, sizeof a.De);
  std::memcpy(a.Do, c->Do, sizeof a.Do);
  std::memcpy(a.eos_c, c->eos_c, sizeof a.eos_c);
  a.prof = debug_prof_buffer();
  return a;
}

dg_status stage_launch(dg_ctx* c, int mode, int stage, double dt, const double* q_n, const double* q_in,
                       double* out, void* stream, int64_t n_list = -1, const int32_t* list = nullptr) {
  dgi::StageArgs a = stage_args(c, mode, stage, dt, q_n, q_in, out, n_list, list);
  // viscosity needs the halo's gradients (not exchanged): checked here, where the work runs, so
  // set_viscosity followed by mesh_upload_part cannot slip past dg_set_viscosity's check
  if (c->mu > 0.0 && n_list >= 0) return fail(DG_ERR_UNSUPPORTED, "element-list launch with viscosity");
  if (n_list == 0) return DG_OK;
  if (c->mu > 0.0 && c->n_parts > 1)
    return fail(DG_ERR_UNSUPPORTED, "viscosity on a partitioned mesh (gradients of halo rows are not exchanged)");
  if (c->mu > 0.0) {  // NEXT-3: V = mu div grad u'(q_in) before the stage overwrites anything
    if (c->visc_rows != c->n_rows) {
      cudaFree(c->d_sig);
      cudaFree(c->d_visc);
      c->d_sig = c->d_visc = nullptr;
      c->visc_rows = 0;
      CUDA_TRY(cudaMalloc(&c->d_sig, sizeof(double) * c->dim * c->n_rows * c->stride), "viscous scratch alloc");
      CUDA_TRY(cudaMalloc(&c->d_visc, sizeof(double) * c->n_rows * c->stride), "viscous scratch alloc");
      c->visc_rows = c->n_rows;
    }
    int ev = dgi::launch_visc(c->dim, c->N, q_in, c->d_sig, c->d_visc, c->d_desc, c->d_mort, c->d_bg, c->d_ops,
                              c->n_elem, c->stride, c->mu, stream);
    c->launches += 2;
    if (ev != cudaSuccess) return cuda_fail((cudaError_t)ev, "viscous kernels launch");
  }
  int e = dgi::launch_stage(c->dim, c->N, a, stream);
  c->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "stage kernel launch");
  if (c->mu > 0.0) {  // out += (RK stage: b_s dt; RHS: 1) V
    const double coef = mode == 1 ? a.rk_b * dt : 1.0;
    int ev = dgi::launch_axpy_rows(out, c->d_visc, coef, c->n_elem, c->stride, c->F * c->Np, stream);
    c->launches++;
    if (ev != cudaSuccess) return cuda_fail((cudaError_t)ev, "viscous axpy launch");
  }
  return DG_OK;
}

}  // namespace

extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }

dg_status dg_create(const dg_params* p, dg_ctx** out) {
  if (!p || !out) return fail(DG_ERR_ARG, "null argument");
  *out = nullptr;
  if (p->dim != 2 && p->dim != 3) return fail(DG_ERR_UNSUPPORTED, "dim %d not supported", p->dim);
  if (p->order < 1 || p->order > dgi::kMaxOrder) return fail(DG_ERR_UNSUPPORTED, "order %d not in 1..8", p->order);
  if (!dgi::supported(p->dim, p->order)) return fail(DG_ERR_UNSUPPORTED, "dim %d order %d not compiled", p->dim, p->order);
  if (p->max_level < 0 || p->max_level > dgi::kMaxLevel) return fail(DG_ERR_ARG, "max_level %d not in 0..8", p->max_level);
  for (int d = 0; d < p->dim; ++d) {
    if (p->root[d] < 1 || ((int64_t)p->root[d] << p->max_level) >= (1 << 20))
      return fail(DG_ERR_ARG, "root[%d] = %d out of range", d, p->root[d]);
    if (!(p->hi[d] > p->lo[d]) || !std::isfinite(p->hi[d] - p->lo[d])) return fail(DG_ERR_ARG, "empty domain on axis %d", d);
    if (p->periodic[d] != 0 && p->periodic[d] != 1) return fail(DG_ERR_ARG, "periodic[%d] must be 0 or 1", d);
  }
  if (!(p->gamma > 1.0) || !(p->p0 > 0) || !(p->R > 0) || !std::isfinite(p->g))
    return fail(DG_ERR_ARG, "bad physical constants");
  dg_ctx* c = new dg_ctx;
  c->p = *p;
  {
    const char* v = std::getenv("DG_H4_AMR");
    c->h4_amr = v ? std::atoi(v) : 2;
  }
  c->dim = p->dim;
  c->N = p->order;
  c->n1 = p->order + 1;
  c->Np = c->dim == 2 ? c->n1 * c->n1 : c->n1 * c->n1 * c->n1;
  c->F = c->dim + 2;
  c->stride = ((int64_t)c->F * c->Np + 15) / 16 * 16;
  c->basis = make_basis(c->N);
  const int n1 = c->n1;
  c->ops.assign(dgi::OpsLayout::size(n1), 0.0);
  std::copy(c->basis.D.begin(), c->basis.D.end(), c->ops.begin());
  for (int b = 0; b < 2; ++b) {
    std::copy(c->basis.P[b].begin(), c->basis.P[b].end(), c->ops.begin() + dgi::OpsLayout::P(n1, b));
    std::copy(c->basis.R[b].begin(), c->basis.R[b].end(), c->ops.begin() + dgi::OpsLayout::R(n1, b));
  }
  std::copy(c->basis.w.begin(), c->basis.w.end(), c->ops.begin() + dgi::OpsLayout::W(n1));
  // pointwise-interpolation matrices I_b[j][k] = l_k(2 x_j + (b ? -1 : 1)) (long double Lagrange)
  for (int b = 0; b < 2; ++b)
    for (int j = 0; j < n1; ++j) {
      const LD xi = 2 * (LD)c->basis.xl[j] + (b ? -1 : 1);
      for (int k = 0; k < n1; ++k) {
        LD l = 1;
        for (int m = 0; m < n1; ++m)
          if (m != k) l *= (xi - c->basis.xl[m]) / (c->basis.xl[k] - c->basis.xl[m]);
        c->ops[dgi::OpsLayout::I(n1, b) + j * n1 + k] = (double)l;
      }
    }
  for (int l = 0; l <= dgi::kMaxLevel; ++l)
    for (int d = 0; d < 3; ++d) {
      double h = d < c->dim ? (p->hi[d] - p->lo[d]) / ((double)p->root[d] * std::ldexp(1.0, l)) : 1.0;
      c->ops[dgi::OpsLayout::H(n1) + 3 * l + d] = 2.0 / h;
    }
  // even-odd split of D (centro-antisymmetric: D[N-i][N-j] = -D[i][j]), from long double
  {
    const int N = c->N, H = n1 / 2;
    const auto& D = c->basis.Dl;
    for (int i = 0; i < H; ++i) {
      for (int m = 0; m < H; ++m) {
        c->De[i * dgi::kMaxH + m] = (double)((D[i * n1 + m] + D[i * n1 + N - m]) / 2);
        c->Do[i * dgi::kMaxH + m] = (double)((D[i * n1 + m] - D[i * n1 + N - m]) / 2);
      }
      if (n1 & 1) c->De[i * dgi::kMaxH + H] = (double)D[i * n1 + H];
    }
    if (n1 & 1)
      for (int m = 0; m < H; ++m) c->Do[H * dgi::kMaxH + m] = (double)D[H * n1 + m];
  }
  // binomial coefficients C(gamma, k+1) of (1+x)^gamma - 1 = x sum_k C(gamma,k+1) x^k (reading R2)
  {
    LD ck = 1;
    for (int k = 0; k < dgi::kEosTerms; ++k) {
      ck = ck * ((LD)p->gamma - k) / (k + 1);
      c->eos_c[k] = (double)ck;
    }
  }
  c->rowoff.assign(p->max_level + 2, 0);
  for (int l = 0; l <= p->max_level; ++l)
    c->rowoff[l + 1] = c->rowoff[l] + ((long)p->root[c->dim - 1] << l) * n1;
  c->n_rows_expected = c->rowoff[p->max_level + 1];
  *out = c;
  return DG_OK;
}

void dg_destroy(dg_ctx* c) {
  if (!c) return;
  free_device(c);
  cudaFree(c->d_sig);
  cudaFree(c->d_visc);
  cudaFree(c->d_ops);
  cudaFree(c->d_bg);
  cudaFree(c->d_bg4);
  cudaFree(c->d_jac);
  cudaFree(c->d_check);
  delete c;
}

dg_status dg_mesh_build(dg_ctx* c, int64_t n, const int8_t* level, const int32_t* anchor) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  c->on_device = false;
  return build_mesh(c, n, level, anchor);
}

static dg_status upload_tables(dg_ctx* c, cudaStream_t s) {
  const int nsub = 1 << (c->dim - 1);
  CUDA_TRY(cudaMalloc(&c->d_desc, sizeof(ElemDesc) * c->n_rows), "mesh upload: alloc");
  CUDA_TRY(cudaMalloc(&c->d_nbrow, sizeof(int32_t) * 8 * c->n_elem), "mesh upload: alloc");
  CUDA_TRY(cudaMalloc(&c->d_mort, sizeof(int32_t) * std::max<size_t>(c->mort.size(), nsub)), "mesh upload: alloc");
  CUDA_TRY(cudaMalloc(&c->d_mortbg, sizeof(int32_t) * std::max<size_t>(c->mort.size(), nsub)), "mesh upload: alloc");
  CUDA_TRY(cudaMalloc(&c->d_partial, sizeof(double) * c->n_elem * c->F), "mesh upload: alloc");
  if (!c->d_ops) CUDA_TRY(cudaMalloc(&c->d_ops, sizeof(double) * c->ops.size()), "mesh upload: alloc");
  if (!c->d_jac) CUDA_TRY(cudaMalloc(&c->d_jac, sizeof(double) * (dgi::kMaxLevel + 1)), "mesh upload: alloc");
  double jac[dgi::kMaxLevel + 1];
  for (int l = 0; l <= dgi::kMaxLevel; ++l) {
    double J = 1.0;
    for (int d = 0; d < c->dim; ++d) J *= 0.5 * ((c->p.hi[d] - c->p.lo[d]) / ((double)c->p.root[d] * std::ldexp(1.0, l)));
    jac[l] = J;
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_desc, c->desc.data(), sizeof(ElemDesc) * c->n_rows, cudaMemcpyHostToDevice, s), "mesh upload: copy");
  c->has_nc = false;
  for (int64_t e = 0; e < c->n_elem && !c->has_nc; ++e)
    for (int f = 0; f < 2 * c->dim; ++f) {
      const int k = dgi::face_kind(c->desc[e].info, f);
      if (k == dgi::kCoarse || k == dgi::kFine) c->has_nc = true;
    }
  CUDA_TRY(cudaMemcpyAsync(c->d_nbrow, c->nbrow.data(), sizeof(int32_t) * 8 * c->n_elem, cudaMemcpyHostToDevice, s), "mesh upload: copy");
  if (!c->mort.empty())
    CUDA_TRY(cudaMemcpyAsync(c->d_mort, c->mort.data(), sizeof(int32_t) * c->mort.size(), cudaMemcpyHostToDevice, s), "mesh upload: copy");
  std::vector<int32_t> mortbg(c->mort.size());
  for (size_t i = 0; i < c->mort.size(); ++i) mortbg[i] = c->desc[c->mort[i]].bgrow;
  if (!mortbg.empty())
    CUDA_TRY(cudaMemcpyAsync(c->d_mortbg, mortbg.data(), sizeof(int32_t) * mortbg.size(), cudaMemcpyHostToDevice, s),
             "mesh upload: copy");
  // coarse-face owners of the local mortar slots, and the slots' lift buffer (3D N = 4: the mortar
  // pre-pass of k_stage_h4)
  c->n_mort = (int64_t)(c->mort.size() / nsub);
  // one 64-B record per slot: element, face, its info word and background row, the slot's fine
  // elements and their background rows (everything the pre-pass needs to issue a face's loads)
  std::vector<int32_t> owner((size_t)16 * c->n_mort, -1);
  if (c->dim == 3)
    for (int64_t e = 0; e < c->n_elem; ++e)
      for (int f = 0; f < 2 * c->dim; ++f)
        if (dgi::face_kind(c->desc[e].info, f) == dgi::kCoarse) {
          int32_t* r = owner.data() + (size_t)16 * c->desc[e].nbr[f];
          r[0] = (int32_t)e;
          r[1] = f;
          r[2] = c->desc[e].info;
          r[3] = c->desc[e].bgrow;
          for (int b = 0; b < nsub; ++b) {
            r[4 + b] = c->mort[(size_t)c->desc[e].nbr[f] * nsub + b];
            r[8 + b] = mortbg[(size_t)c->desc[e].nbr[f] * nsub + b];
          }
        }
  if (c->n_mort > 0 && c->dim == 3 && c->N == 4) {
    CUDA_TRY(cudaMalloc(&c->d_mort_owner, sizeof(int32_t) * owner.size()), "mesh upload: alloc");
    CUDA_TRY(cudaMalloc(&c->d_mlift, sizeof(double) * c->n_mort * c->F * (c->Np / c->n1)), "mesh upload: alloc");
    CUDA_TRY(cudaMemcpyAsync(c->d_mort_owner, owner.data(), sizeof(int32_t) * owner.size(), cudaMemcpyHostToDevice, s),
             "mesh upload: copy");
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_ops, c->ops.data(), sizeof(double) * c->ops.size(), cudaMemcpyHostToDevice, s), "mesh upload: copy");
  CUDA_TRY(cudaMemcpyAsync(c->d_jac, jac, sizeof jac, cudaMemcpyHostToDevice, s), "mesh upload: copy");
  CUDA_TRY(cudaStreamSynchronize(s), "mesh upload: sync");
  c->on_device = true;
  return DG_OK;
}

dg_status dg_mesh_upload(dg_ctx* c, int64_t n, const int8_t* level, const int32_t* anchor, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamSynchronize(s), "mesh upload: sync");
  free_device(c);
  dg_status st = build_mesh(c, n, level, anchor);
  if (st != DG_OK) return st;
  return upload_tables(c, s);
}

dg_status dg_mesh_build_part(dg_ctx* c, int64_t n, const int8_t* level, const int32_t* anchor, int32_t n_parts,
                             int32_t part) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  c->on_device = false;
  dg_status st = build_mesh(c, n, level, anchor);
  if (st != DG_OK) return st;
  st = build_part(c, n_parts, part);
  if (st != DG_OK) c->have_mesh = false;
  return st;
}

dg_status dg_mesh_upload_part(dg_ctx* c, int64_t n, const int8_t* level, const int32_t* anchor, int32_t n_parts,
                              int32_t part, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamSynchronize(s), "mesh upload: sync");
  free_device(c);
  dg_status st = dg_mesh_build_part(c, n, level, anchor, n_parts, part);
  if (st != DG_OK) return st;
  return upload_tables(c, s);
}

dg_status dg_part_info(const dg_ctx* c, int32_t* n_parts, int32_t* part, int64_t* n_local, int64_t* n_halo,
                       int64_t* global_begin) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh) return fail(DG_ERR_MESH, "no mesh built");
  if (n_parts) *n_parts = c->n_parts;
  if (part) *part = c->part;
  if (n_local) *n_local = c->n_elem;
  if (n_halo) *n_halo = c->n_rows - c->n_elem;
  if (global_begin) *global_begin = c->gbegin;
  return DG_OK;
}

dg_status dg_part_exchange_lists(const dg_ctx* c, int64_t* send_count, int64_t* recv_count, int32_t* send_idx) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh) return fail(DG_ERR_MESH, "no mesh built");
  for (int k = 0; k < c->n_parts; ++k) {
    if (send_count) send_count[k] = c->n_parts > 1 ? c->send_count[k] : 0;
    if (recv_count) recv_count[k] = c->n_parts > 1 ? c->recv_count[k] : 0;
  }
  if (send_idx && !c->send_idx.empty()) std::memcpy(send_idx, c->send_idx.data(), sizeof(int32_t) * c->send_idx.size());
  return DG_OK;
}

dg_status dg_mesh_face_counts(const dg_ctx* c, int64_t* nc, int64_t* nn, int64_t* nb) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh) return fail(DG_ERR_MESH, "no mesh built");
  const int w = 2 + 2 * (1 << (c->dim - 1));
  if (nc) *nc = (int64_t)c->conf.size() / 4;
  if (nn) *nn = (int64_t)c->nonconf.size() / w;
  if (nb) *nb = (int64_t)c->bnd.size() / 2;
  return DG_OK;
}

dg_status dg_mesh_faces(const dg_ctx* c, int32_t* conf, int32_t* nonconf, int32_t* bnd) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh) return fail(DG_ERR_MESH, "no mesh built");
  if (conf) std::copy(c->conf.begin(), c->conf.end(), conf);
  if (nonconf) std::copy(c->nonconf.begin(), c->nonconf.end(), nonconf);
  if (bnd) std::copy(c->bnd.begin(), c->bnd.end(), bnd);
  return DG_OK;
}

dg_status dg_state_layout(const dg_ctx* c, int64_t* n_elem, int32_t* n_fields, int32_t* n_nodes, int64_t* stride) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (n_elem) *n_elem = c->have_mesh ? c->n_rows : 0;
  if (n_fields) *n_fields = c->F;
  if (n_nodes) *n_nodes = c->Np;
  if (stride) *stride = c->stride;
  return DG_OK;
}

dg_status dg_state_alloc(const dg_ctx* c, double** out, void* stream) {
  if (!c || !out) return fail(DG_ERR_ARG, "null argument");
  if (!c->have_mesh) return fail(DG_ERR_MESH, "no mesh built");
  CUDA_TRY(cudaMallocAsync((void**)out, sizeof(double) * c->n_rows * c->stride, (cudaStream_t)stream), "state alloc");
  return DG_OK;
}

dg_status dg_state_free(double* q, void* stream) {
  if (!q) return DG_OK;
  CUDA_TRY(cudaFreeAsync(q, (cudaStream_t)stream), "state free");
  return DG_OK;
}

dg_status dg_set_background(dg_ctx* c, const double* table, int64_t n_rows, void* stream) {
  if (!c || !table) return fail(DG_ERR_ARG, "null argument");
  if (n_rows != c->n_rows_expected)
    return fail(DG_ERR_STATE, "background: %lld rows given, %lld expected", (long long)n_rows, (long long)c->n_rows_expected);
  if (!c->d_bg || c->bg_rows != n_rows) {
    cudaFree(c->d_bg);
    cudaFree(c->d_bg4);
    c->d_bg = nullptr;
    c->d_bg4 = nullptr;
    CUDA_TRY(cudaMalloc(&c->d_bg, sizeof(double) * 3 * n_rows), "background alloc");
    CUDA_TRY(cudaMalloc(&c->d_bg4, sizeof(double) * 4 * n_rows), "background alloc");
    c->bg_rows = n_rows;
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_bg, table, sizeof(double) * 3 * n_rows, cudaMemcpyDefault, (cudaStream_t)stream),
           "background copy");
  int e = dgi::launch_bg_expand(c->d_bg, c->d_bg4, n_rows, stream);
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "background expand");
  return DG_OK;
}

dg_status dg_rhs_elems(dg_ctx* c, const double* q, double* dqdt, int64_t n, const int32_t* elems, void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (n < 0 || (n > 0 && !elems)) return fail(DG_ERR_ARG, "bad element list");
  if (!q || !dqdt) return fail(DG_ERR_ARG, "null state pointer");
  size_t bytes = sizeof(double) * c->n_rows * c->stride;
  if (overlaps(q, dqdt, bytes)) return fail(DG_ERR_ARG, "dqdt aliases q");
  if (misaligned(q) || misaligned(dqdt)) return fail(DG_ERR_ARG, "state pointers must be 16-byte aligned");
  return stage_launch(c, 0, 0, 0.0, q, q, dqdt, stream, n, elems);
}

dg_status dg_rk_stage_elems(dg_ctx* c, int32_t stage, double dt, const double* q_n, const double* q_in,
                            double* q_out, int64_t n, const int32_t* elems, void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (n < 0 || (n > 0 && !elems)) return fail(DG_ERR_ARG, "bad element list");
  if (stage < 0 || stage > 2) return fail(DG_ERR_ARG, "stage %d not in 0..2", stage);
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(DG_ERR_ARG, "dt must be finite and > 0");
  if (!q_in || !q_out || (stage > 0 && !q_n)) return fail(DG_ERR_ARG, "null state pointer");
  size_t bytes = sizeof(double) * c->n_rows * c->stride;
  if (overlaps(q_in, q_out, bytes) || (stage > 0 && overlaps(q_n, q_out, bytes)))
    return fail(DG_ERR_ARG, "q_out aliases an input");
  if (stage > 0 && q_n == q_in) return fail(DG_ERR_ARG, "q_n == q_in only allowed at stage 0");
  if (misaligned(q_in) || misaligned(q_out) || (stage > 0 && misaligned(q_n)))
    return fail(DG_ERR_ARG, "state pointers must be 16-byte aligned");
  return stage_launch(c, 1, stage, dt, stage == 0 ? q_in : q_n, q_in, q_out, stream, n, elems);
}

/* ---------------------------------------------------------------- NEXT-3 passive tracer (R45) */
namespace {
dg_status passive_launch(dg_ctx* c, int mode, int stage, double dt, const double* q_in, const double* c_n,
                         const double* c_in, double* c_out, void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (!q_in || !c_in || !c_out || (mode == 1 && stage > 0 && !c_n)) return fail(DG_ERR_ARG, "null state pointer");
  if (c->ncmode != 0) return fail(DG_ERR_UNSUPPORTED, "passive tracer: mortar treatment of 2:1 faces only");
  size_t bytes = sizeof(double) * c->n_rows * c->stride;
  if (overlaps(c_in, c_out, bytes) || overlaps(q_in, c_out, bytes) || (c_n && overlaps(c_n, c_out, bytes)))
    return fail(DG_ERR_ARG, "c_out aliases an input");
  dgi::StageArgs a = stage_args(c, mode, stage, dt, nullptr, q_in, nullptr);
  int e = dgi::launch_passive(c->dim, c->N, a, c_n, c_in, c_out, stream);
  c->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "passive tracer kernel launch");
  return DG_OK;
}
}  // namespace

dg_status dg_passive_rhs(dg_ctx* c, const double* q, const double* cq, double* dcdt, void* stream) {
  return passive_launch(c, 0, 0, 0.0, q, nullptr, cq, dcdt, stream);
}

dg_status dg_passive_rk_stage(dg_ctx* c, int32_t stage, double dt, const double* q_in, const double* c_n,
                              const double* c_in, double* c_out, void* stream) {
  if (c && (stage < 0 || stage > 2)) return fail(DG_ERR_ARG, "stage %d not in 0..2", stage);
  if (c && (!(dt > 0.0) || !std::isfinite(dt))) return fail(DG_ERR_ARG, "dt must be finite and > 0");
  return passive_launch(c, 1, stage, dt, q_in, c_n, c_in, c_out, stream);
}

dg_status dg_rhs(dg_ctx* c, const double* q, double* dqdt, void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (!q || !dqdt) return fail(DG_ERR_ARG, "null state pointer");
  size_t bytes = sizeof(double) * c->n_rows * c->stride;
  if (overlaps(q, dqdt, bytes)) return fail(DG_ERR_ARG, "dqdt aliases q");
  if (misaligned(q) || misaligned(dqdt)) return fail(DG_ERR_ARG, "state pointers must be 16-byte aligned");
  return stage_launch(c, 0, 0, 0.0, q, q, dqdt, stream);
}

dg_status dg_rk_stage(dg_ctx* c, int32_t stage, double dt, const double* q_n, const double* q_in, double* q_out,
                      void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (stage < 0 || stage > 2) return fail(DG_ERR_ARG, "stage %d not in 0..2", stage);
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(DG_ERR_ARG, "dt must be finite and > 0");
  if (!q_in || !q_out || (stage > 0 && !q_n)) return fail(DG_ERR_ARG, "null state pointer");
  size_t bytes = sizeof(double) * c->n_rows * c->stride;
  if (overlaps(q_in, q_out, bytes) || (stage > 0 && overlaps(q_n, q_out, bytes)))
    return fail(DG_ERR_ARG, "q_out aliases an input");
  if (stage > 0 && q_n == q_in) return fail(DG_ERR_ARG, "q_n == q_in only allowed at stage 0");
  if (misaligned(q_in) || misaligned(q_out) || (stage > 0 && misaligned(q_n)))
    return fail(DG_ERR_ARG, "state pointers must be 16-byte aligned");
  return stage_launch(c, 1, stage, dt, stage == 0 ? q_in : q_n, q_in, q_out, stream);
}

dg_status dg_amr_project_refine(const dg_ctx* c, int64_t n, const int32_t* parent_src, const int32_t* child0_dst,
                                const double* q_src, double* q_dst, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (n < 0) return fail(DG_ERR_ARG, "n < 0");
  if (n == 0) return DG_OK;
  if (!parent_src || !child0_dst || !q_src || !q_dst || q_src == q_dst) return fail(DG_ERR_ARG, "bad pointer");
  if (!c->d_ops) return fail(DG_ERR_MESH, "no mesh uploaded (operators not on device)");
  dgi::TransferArgs a{parent_src, child0_dst, q_src, q_dst, c->d_ops, n, c->stride};
  int e = dgi::launch_refine(c->dim, c->N, a, stream);
  const_cast<dg_ctx*>(c)->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "refine launch");
  return DG_OK;
}

dg_status dg_amr_project_coarsen(const dg_ctx* c, int64_t n, const int32_t* child0_src, const int32_t* parent_dst,
                                 const double* q_src, double* q_dst, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (n < 0) return fail(DG_ERR_ARG, "n < 0");
  if (n == 0) return DG_OK;
  if (!child0_src || !parent_dst || !q_src || !q_dst || q_src == q_dst) return fail(DG_ERR_ARG, "bad pointer");
  if (!c->d_ops) return fail(DG_ERR_MESH, "no mesh uploaded (operators not on device)");
  dgi::TransferArgs a{child0_src, parent_dst, q_src, q_dst, c->d_ops, n, c->stride};
  int e = dgi::launch_coarsen(c->dim, c->N, a, stream);
  const_cast<dg_ctx*>(c)->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "coarsen launch");
  return DG_OK;
}

dg_status dg_copy_elements(const dg_ctx* c, int64_t n, const int32_t* src, const int32_t* dst, const double* q_src,
                           double* q_dst, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (n < 0) return fail(DG_ERR_ARG, "n < 0");
  if (n == 0) return DG_OK;
  if (!src || !dst || !q_src || !q_dst) return fail(DG_ERR_ARG, "bad pointer");
  dgi::TransferArgs a{src, dst, q_src, q_dst, nullptr, n, c->stride};
  int e = dgi::launch_copy(c->dim, c->N, a, stream);
  const_cast<dg_ctx*>(c)->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "copy launch");
  return DG_OK;
}

dg_status dg_check_state(dg_ctx* c, const double* q, int64_t* out_host, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh || !c->on_device) return fail(DG_ERR_MESH, "no mesh uploaded");
  if (!q || !out_host) return fail(DG_ERR_ARG, "null pointer");
  if (!c->d_check) CUDA_TRY(cudaMalloc(&c->d_check, 4 * sizeof(unsigned long long)), "check_state alloc");
  cudaStream_t s = (cudaStream_t)stream;
  int e = dgi::launch_check_state(q, c->n_elem, c->stride, c->Np, c->F, c->d_check, stream);
  c->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "check_state launch");
  unsigned long long h[4];
  CUDA_TRY(cudaMemcpyAsync(h, c->d_check, sizeof(h), cudaMemcpyDeviceToHost, s), "check_state copy");
  CUDA_TRY(cudaStreamSynchronize(s), "check_state sync");
  for (int i = 0; i < 3; ++i) out_host[i] = (int64_t)h[i];
  out_host[3] = h[3] == ~0ull ? -1 : (int64_t)h[3];
  return DG_OK;
}

dg_status dg_integrals(const dg_ctx* c, const double* q, double* out_host, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh || !c->on_device) return fail(DG_ERR_MESH, "no mesh uploaded");
  if (!q || !out_host) return fail(DG_ERR_ARG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  int e = dgi::launch_elem_integrals(c->dim, c->N, q, c->n_elem, c->stride, c->d_desc, c->d_ops, c->d_jac,
                                     c->d_partial, stream);
  const_cast<dg_ctx*>(c)->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "integrals launch");
  std::vector<double> part((size_t)c->n_elem * c->F);
  CUDA_TRY(cudaMemcpyAsync(part.data(), c->d_partial, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, s),
           "integrals copy");
  CUDA_TRY(cudaStreamSynchronize(s), "integrals sync");
  for (int f = 0; f < c->F; ++f) {  // Neumaier over elements (R20)
    double sum = 0.0, comp = 0.0;
    for (int64_t i = 0; i < c->n_elem; ++i) {
      double v = part[(size_t)i * c->F + f];
      double t = sum + v;
      if (std::fabs(sum) >= std::fabs(v)) comp += (sum - t) + v;
      else comp += (v - t) + sum;
      sum = t;
    }
    out_host[f] = sum + comp;
  }
  return DG_OK;
}

static dg_status ensure_scratch(dg_ctx* c, int k) {
  for (int i = 0; i < k; ++i)
    if (!c->d_scratch[i]) CUDA_TRY(cudaMalloc(&c->d_scratch[i], sizeof(double) * c->n_elem * c->stride), "scratch alloc");
  return DG_OK;
}

dg_status dg_rhs_host(dg_ctx* c, const double* q_host, double* dqdt_host, void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (c->n_parts > 1) return fail(DG_ERR_ARG, "rhs_host: not available on a partitioned mesh");
  if (!q_host || !dqdt_host) return fail(DG_ERR_ARG, "null pointer");
  if ((st = ensure_scratch(c, 2)) != DG_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  size_t row = sizeof(double) * c->F * c->Np, pitch = sizeof(double) * c->stride;
  CUDA_TRY(cudaMemcpy2DAsync(c->d_scratch[0], pitch, q_host, row, row, c->n_elem, cudaMemcpyHostToDevice, s), "h2d");
  if ((st = stage_launch(c, 0, 0, 0.0, c->d_scratch[0], c->d_scratch[0], c->d_scratch[1], stream)) != DG_OK) return st;
  CUDA_TRY(cudaMemcpy2DAsync(dqdt_host, row, c->d_scratch[1], pitch, row, c->n_elem, cudaMemcpyDeviceToHost, s), "d2h");
  CUDA_TRY(cudaStreamSynchronize(s), "sync");
  return DG_OK;
}

dg_status dg_rk3_step_host(dg_ctx* c, double dt, int32_t n_steps, double* q_host, void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (c->n_parts > 1) return fail(DG_ERR_ARG, "rk3_step_host: not available on a partitioned mesh");
  if (!q_host || n_steps < 0) return fail(DG_ERR_ARG, "bad argument");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(DG_ERR_ARG, "dt must be finite and > 0");
  if ((st = ensure_scratch(c, 3)) != DG_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  size_t row = sizeof(double) * c->F * c->Np, pitch = sizeof(double) * c->stride;
  double *A = c->d_scratch[0], *B = c->d_scratch[1], *C = c->d_scratch[2];
  CUDA_TRY(cudaMemcpy2DAsync(A, pitch, q_host, row, row, c->n_elem, cudaMemcpyHostToDevice, s), "h2d");
  for (int k = 0; k < n_steps; ++k) {
    if ((st = stage_launch(c, 1, 0, dt, A, A, B, stream)) != DG_OK) return st;
    if ((st = stage_launch(c, 1, 1, dt, A, B, C, stream)) != DG_OK) return st;
    if ((st = stage_launch(c, 1, 2, dt, A, C, B, stream)) != DG_OK) return st;
    std::swap(A, B);
  }
  CUDA_TRY(cudaMemcpy2DAsync(q_host, row, A, pitch, row, c->n_elem, cudaMemcpyDeviceToHost, s), "d2h");
  CUDA_TRY(cudaStreamSynchronize(s), "sync");
  return DG_OK;
}

/* ---------------------------------------------------------------- NEXT-1 regrid */
struct dg_regrid_plan {
  dgi::RegridOut out;
};

dg_status dg_amr_indicator(const dg_ctx* c, int32_t kind, const double* q, double* eta, void* stream) {
  dg_status st = check_ready(c);
  if (st != DG_OK) return st;
  if (kind != 0 && kind != 1) return fail(DG_ERR_ARG, "amr_indicator: kind must be 0 or 1");
  if (!q || !eta) return fail(DG_ERR_ARG, "amr_indicator: null buffer");
  int e = dgi::launch_amr_indicator(c->dim, c->N, kind, q, c->n_elem, c->stride, c->d_desc, c->d_bg, eta, stream);
  const_cast<dg_ctx*>(c)->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "amr_indicator launch");
  return DG_OK;
}

dg_status dg_regrid_plan_create(const dg_ctx* c, const double* eta_host, double refine_above, double coarsen_below,
                                int32_t buffer, dg_regrid_plan** out) {
  if (!c || !eta_host || !out) return fail(DG_ERR_ARG, "regrid_plan: null argument");
  *out = nullptr;
  if (!c->have_mesh) return fail(DG_ERR_MESH, "regrid_plan: no mesh");
  if (c->n_parts > 1) return fail(DG_ERR_ARG, "regrid_plan: not available on a partitioned mesh");
  if (buffer < 0 || buffer > 64) return fail(DG_ERR_ARG, "regrid_plan: buffer %d not in 0..64", buffer);
  if (std::isnan(refine_above) || std::isnan(coarsen_below)) return fail(DG_ERR_ARG, "regrid_plan: NaN threshold");
  dgi::RegridIn in;
  in.dim = c->dim;
  in.max_level = c->p.max_level;
  for (int d = 0; d < 3; ++d) {
    in.root[d] = c->p.root[d];
    in.periodic[d] = c->p.periodic[d];
  }
  in.n = c->n_elem;
  in.level = c->lev.data();
  in.anchor = c->anc.data();
  in.eta = eta_host;
  in.refine_above = refine_above;
  in.coarsen_below = coarsen_below;
  in.buffer = buffer;
  dg_regrid_plan* p = new dg_regrid_plan;
  const char* why = "";
  if (dgi::regrid_plan(in, p->out, &why) != 0) {
    delete p;
    return fail(DG_ERR_MESH, "%s", why);
  }
  *out = p;
  return DG_OK;
}

dg_status dg_regrid_plan_sizes(const dg_regrid_plan* p, int64_t* n_leaves, int64_t* n_refine, int64_t* n_coarsen,
                               int64_t* n_copy) {
  if (!p) return fail(DG_ERR_ARG, "regrid_plan_sizes: null plan");
  if (n_leaves) *n_leaves = (int64_t)p->out.level.size();
  if (n_refine) *n_refine = (int64_t)p->out.refine_parent.size();
  if (n_coarsen) *n_coarsen = (int64_t)p->out.coarsen_parent.size();
  if (n_copy) *n_copy = (int64_t)p->out.copy_src.size();
  return DG_OK;
}

dg_status dg_regrid_plan_get(const dg_regrid_plan* p, int8_t* level, int32_t* anchor, int32_t* refine_parent,
                             int32_t* refine_child0, int32_t* coarsen_child0, int32_t* coarsen_parent,
                             int32_t* copy_src, int32_t* copy_dst) {
  if (!p) return fail(DG_ERR_ARG, "regrid_plan_get: null plan");
  auto put = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  put(level, p->out.level);
  put(anchor, p->out.anchor);
  put(refine_parent, p->out.refine_parent);
  put(refine_child0, p->out.refine_child0);
  put(coarsen_child0, p->out.coarsen_child0);
  put(coarsen_parent, p->out.coarsen_parent);
  put(copy_src, p->out.copy_src);
  put(copy_dst, p->out.copy_dst);
  return DG_OK;
}

void dg_regrid_plan_destroy(dg_regrid_plan* p) { delete p; }

/* ---------------------------------------------------------------- NEXT-3 baseline */
dg_status dg_set_nonconforming(dg_ctx* c, int32_t mode) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (mode != 0 && mode != 1) return fail(DG_ERR_ARG, "nonconforming mode %d not in 0..1", mode);
  c->ncmode = mode;
  return DG_OK;
}

dg_status dg_set_viscosity(dg_ctx* c, double mu) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!(mu >= 0.0) || !std::isfinite(mu)) return fail(DG_ERR_ARG, "viscosity must be finite and >= 0");
  if (mu > 0.0 && c->n_parts > 1)
    return fail(DG_ERR_UNSUPPORTED, "viscosity on a partitioned mesh needs a gradient halo exchange (not built)");
  c->mu = mu;
  return DG_OK;
}

dg_status dg_tracer_rhs(dg_ctx* c, const double* s, double* out, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh || !c->on_device) return fail(DG_ERR_MESH, "no mesh uploaded");
  if (!s || !out || s == out) return fail(DG_ERR_ARG, "tracer_rhs: bad pointer");
  int e = dgi::launch_tracer(c->dim, c->N, 0, 0, 0.0, 1.0, c->ncmode, nullptr, s, out, c->d_desc, c->d_mort, c->d_ops,
                             c->n_elem, c->stride, stream);
  c->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "tracer launch");
  return DG_OK;
}

dg_status dg_tracer_rk_stage(dg_ctx* c, int32_t stage, double dt, const double* s_n, const double* s_in,
                             double* s_out, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh || !c->on_device) return fail(DG_ERR_MESH, "no mesh uploaded");
  if (stage < 0 || stage > 2) return fail(DG_ERR_ARG, "stage %d not in 0..2", stage);
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(DG_ERR_ARG, "dt must be finite and > 0");
  if (!s_in || !s_out || (stage > 0 && !s_n) || s_out == s_in || (stage > 0 && s_out == s_n))
    return fail(DG_ERR_ARG, "tracer_rk_stage: bad pointer");
  const double B[3] = {1.0, 1.0 / 4.0, 2.0 / 3.0};
  int e = dgi::launch_tracer(c->dim, c->N, 1, stage, dt, B[stage], c->ncmode, stage ? s_n : s_in, s_in, s_out,
                             c->d_desc, c->d_mort, c->d_ops, c->n_elem, c->stride, stream);
  c->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "tracer launch");
  return DG_OK;
}

dg_status dg_part_face_lists(const dg_ctx* c, int64_t* send_count, int64_t* recv_count, int32_t* send_pairs,
                             int32_t* recv_pairs) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (!c->have_mesh) return fail(DG_ERR_MESH, "no mesh built");
  for (int k = 0; k < c->n_parts; ++k) {
    if (send_count) send_count[k] = c->n_parts > 1 ? c->fsend_count[k] : 0;
    if (recv_count) recv_count[k] = c->n_parts > 1 ? c->frecv_count[k] : 0;
  }
  if (send_pairs && !c->fsend.empty()) std::memcpy(send_pairs, c->fsend.data(), sizeof(int32_t) * c->fsend.size());
  if (recv_pairs && !c->frecv.empty()) std::memcpy(recv_pairs, c->frecv.data(), sizeof(int32_t) * c->frecv.size());
  return DG_OK;
}

dg_status dg_pack_faces(const dg_ctx* c, int64_t n, const int32_t* pairs, const double* q, double* buf, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (n < 0) return fail(DG_ERR_ARG, "n < 0");
  if (n == 0) return DG_OK;
  if (!pairs || !q || !buf) return fail(DG_ERR_ARG, "bad pointer");
  int e = dgi::launch_face_pack(c->dim, c->N, 0, n, pairs, const_cast<double*>(q), buf, c->stride, stream);
  const_cast<dg_ctx*>(c)->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "pack launch");
  return DG_OK;
}

dg_status dg_unpack_faces(const dg_ctx* c, int64_t n, const int32_t* pairs, const double* buf, double* q, void* stream) {
  if (!c) return fail(DG_ERR_ARG, "null context");
  if (n < 0) return fail(DG_ERR_ARG, "n < 0");
  if (n == 0) return DG_OK;
  if (!pairs || !q || !buf) return fail(DG_ERR_ARG, "bad pointer");
  int e = dgi::launch_face_pack(c->dim, c->N, 1, n, pairs, q, const_cast<double*>(buf), c->stride, stream);
  const_cast<dg_ctx*>(c)->launches++;
  if (e != cudaSuccess) return cuda_fail((cudaError_t)e, "unpack launch");
  return DG_OK;
}

int64_t dg_launch_count(const dg_ctx* c) { return c ? c->launches : 0; }

/* Debug only (not in dg.h): accumulated stage-kernel phase clocks since the
 * last reset when DG_PHASE_PROF=1; returns the number of slots written. */
int dg_debug_timeline(long long* out_host, int n) { return dgi::debug_timeline(out_host, n); }

int dg_debug_phase_clocks(unsigned long long* out_host, int reset) {
  unsigned long long* b = debug_prof_buffer();
  if (!b || !out_host) return 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return 0;
  if (cudaMemcpy(out_host, b, sizeof(unsigned long long) * dgi::kProfSlots, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  if (reset) cudaMemset(b, 0, sizeof(unsigned long long) * dgi::kProfSlots);
  return dgi::kProfSlots;
}

}  // extern "C"
