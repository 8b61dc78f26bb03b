/*
 * oracle.cpp -- plain, slow, obviously-correct CPU oracle for the dGSEM
 * right-hand side of arXiv 2404.16648 (tree-based AMR path).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2404_16648_b200/csrc); neither includes the other.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b (section noted);
 * "Rnn" = a reading listed in DESIGN.md section 3.
 *
 * Arithmetic: fp64, scalar loops, compiled -O2 -ffp-contract=off (no FMA
 * contraction, no fast-math).  Every face flux is computed ONCE from the
 * canonical face lists (owner computes, the other side takes the negative).
 * Mortars use explicit dense 1D matrices; refine/coarsen use explicit
 * Kronecker loops (no sum factorisation).
 *
 * Parity-unpinned functions: none at the function level; the bubble-config
 * values themselves have no closed form.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

namespace {

const double kPi = 3.14159265358979323846;

/* ------------------------------------------------------------------ */
/* 1D basis: LGL nodes/weights, differentiation matrix, mortar ops     */
/* ------------------------------------------------------------------ */

/* Legendre P_0..P_n at x by the three-term recurrence. */
void legendre_all(int n, double x, double* P) {
  P[0] = 1.0;
  if (n >= 1) P[1] = x;
  for (int k = 2; k <= n; ++k)
    P[k] = ((2.0 * k - 1.0) * x * P[k - 1] - (k - 1.0) * P[k - 2]) / k;
}

/* LGL nodes = roots of (1-x^2) P'_N.  Newton on x P_N - P_{N-1} (same roots,
 * derivative (N+1) P_N) seeded at Chebyshev-Gauss-Lobatto points, tol 1e-15,
 * at most 100 iterations, then symmetrised.  Weights w_i = 2/(N(N+1)P_N^2).
 * P:279 ("integrating over the Legendre-Gauss-Lobatto (LGL) points"). */
void lgl(int N, double* x, double* w) {
  std::vector<double> P(N + 1);
  for (int i = 0; i <= N; ++i) x[i] = -std::cos(kPi * i / N);
  for (int it = 0; it < 100; ++it) {
    double maxdx = 0.0;
    for (int i = 0; i <= N; ++i) {
      legendre_all(N, x[i], P.data());
      double xn = x[i] - (x[i] * P[N] - P[N - 1]) / ((N + 1.0) * P[N]);
      maxdx = std::max(maxdx, std::fabs(xn - x[i]));
      x[i] = xn;
    }
    if (maxdx < 1e-15) break;
  }
  for (int i = 0; i <= N / 2; ++i) {
    double s = 0.5 * (x[N - i] - x[i]);
    x[i] = -s;
    x[N - i] = s;
  }
  x[0] = -1.0;
  x[N] = 1.0;
  if (N % 2 == 0) x[N / 2] = 0.0;
  for (int i = 0; i <= N; ++i) {
    legendre_all(N, x[i], P.data());
    w[i] = 2.0 / (N * (N + 1.0) * P[N] * P[N]);
  }
  for (int i = 0; i <= N / 2; ++i) {
    double s = 0.5 * (w[i] + w[N - i]);
    w[i] = s;
    w[N - i] = s;
  }
}

/* D_ij = l'_j(x_i) from barycentric weights; diagonal = minus the
 * off-diagonal row sum (the derivative of a constant is zero). */
void dmat(int N, const double* x, double* D) {
  std::vector<double> lam(N + 1);
  for (int j = 0; j <= N; ++j) {
    double p = 1.0;
    for (int k = 0; k <= N; ++k)
      if (k != j) p *= (x[j] - x[k]);
    lam[j] = 1.0 / p;
  }
  for (int i = 0; i <= N; ++i) {
    double s = 0.0;
    for (int j = 0; j <= N; ++j) {
      if (i == j) continue;
      D[i * (N + 1) + j] = (lam[j] / lam[i]) / (x[i] - x[j]);
      s += D[i * (N + 1) + j];
    }
    D[i * (N + 1) + i] = -s;
  }
}

/* Gauss-Legendre rule with Q points (Newton on P_Q). */
void gauss_legendre(int Q, double* y, double* W) {
  std::vector<double> P(Q + 1);
  for (int i = 0; i < Q; ++i) {
    double x = -std::cos(kPi * (i + 0.75) / (Q + 0.5));
    for (int it = 0; it < 100; ++it) {
      legendre_all(Q, x, P.data());
      double dP = Q * (x * P[Q] - P[Q - 1]) / (x * x - 1.0);
      double dx = P[Q] / dP;
      x -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    legendre_all(Q, x, P.data());
    double dP = Q * (x * P[Q] - P[Q - 1]) / (x * x - 1.0);
    y[i] = x;
    W[i] = 2.0 / ((1.0 - x * x) * dP * dP);
  }
}

/* Lagrange cardinal l_j on nodes x, evaluated at t (product form). */
double lagrange(int N, const double* x, int j, double t) {
  double p = 1.0;
  for (int m = 0; m <= N; ++m)
    if (m != j) p *= (t - x[m]) / (x[j] - x[m]);
  return p;
}

/* Gauss-Jordan inverse with partial pivoting of an n x n matrix. */
void invert(int n, const double* A, double* Ainv) {
  std::vector<double> a(A, A + n * n), b(n * n, 0.0);
  for (int i = 0; i < n; ++i) b[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[r * n + c]) > std::fabs(a[piv * n + c])) piv = r;
    for (int k = 0; k < n; ++k) {
      std::swap(a[c * n + k], a[piv * n + k]);
      std::swap(b[c * n + k], b[piv * n + k]);
    }
    double d = a[c * n + c];
    for (int k = 0; k < n; ++k) {
      a[c * n + k] /= d;
      b[c * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = a[r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        a[r * n + k] -= f * a[c * n + k];
        b[r * n + k] -= f * b[c * n + k];
      }
    }
  }
  std::copy(b.begin(), b.end(), Ainv);
}

/* Exact (consistent) mass matrix M_kj = int_{-1}^{1} l_k l_j, and the mixed
 * mass matrices S_b[k][j] = int_{-1}^{1} l_k(x) l_j(xi_b(x)) dx on mortar b
 * (xi_lo = (x-1)/2, xi_hi = (x+1)/2), both with N+3 Gauss points (exact for
 * degree 2N).  P_b = M^-1 S_b (face -> mortar), R_b = 1/2 M^-1 S_b^T
 * (mortar -> face, s = 1/2).  P:290-310 (Sec. 3.3), readings R11, R12. */
struct Ops {
  int N;
  std::vector<double> x, w, D, M, S[2], P[2], R[2];
};

Ops make_ops(int N) {
  Ops o;
  o.N = N;
  int n = N + 1;
  o.x.resize(n);
  o.w.resize(n);
  o.D.resize(n * n);
  lgl(N, o.x.data(), o.w.data());
  dmat(N, o.x.data(), o.D.data());
  int Q = N + 3;
  std::vector<double> y(Q), W(Q);
  gauss_legendre(Q, y.data(), W.data());
  o.M.assign(n * n, 0.0);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int q = 0; q < Q; ++q)
        s += W[q] * lagrange(N, o.x.data(), k, y[q]) * lagrange(N, o.x.data(), j, y[q]);
      o.M[k * n + j] = s;
    }
  std::vector<double> Minv(n * n);
  invert(n, o.M.data(), Minv.data());
  for (int b = 0; b < 2; ++b) {
    o.S[b].assign(n * n, 0.0);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int q = 0; q < Q; ++q) {
          double xi = b == 0 ? 0.5 * (y[q] - 1.0) : 0.5 * (y[q] + 1.0);
          s += W[q] * lagrange(N, o.x.data(), k, y[q]) * lagrange(N, o.x.data(), j, xi);
        }
        o.S[b][k * n + j] = s;
      }
    o.P[b].assign(n * n, 0.0);
    o.R[b].assign(n * n, 0.0);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) {
        double sp = 0.0, sr = 0.0;
        for (int l = 0; l < n; ++l) {
          sp += Minv[k * n + l] * o.S[b][l * n + j];
          sr += Minv[k * n + l] * o.S[b][j * n + l];
        }
        o.P[b][k * n + j] = sp;
        o.R[b][k * n + j] = 0.5 * sr;
      }
  }
  return o;
}

}  // namespace

/* ------------------------------------------------------------------ */
/* Public C ABI of the oracle (its own struct; not libdg's header)     */
/* ------------------------------------------------------------------ */
extern "C" {

typedef struct {
  int32_t dim, order;
  int32_t root[3];
  double lo[3], hi[3];
  int32_t periodic[3];
  int32_t max_level;
  double gamma, R, cp, p0, g;
} ora_params;

enum { ORA_OK = 0, ORA_ERR_ARG = -1, ORA_ERR_MESH = -3, ORA_ERR_UNBALANCED = -4 };

int ora_lgl(int N, double* x, double* w) {
  if (N < 1 || N > 16) return ORA_ERR_ARG;
  lgl(N, x, w);
  return ORA_OK;
}

int ora_dmat(int N, double* D) {
  if (N < 1 || N > 16) return ORA_ERR_ARG;
  std::vector<double> x(N + 1), w(N + 1);
  lgl(N, x.data(), w.data());
  dmat(N, x.data(), D);
  return ORA_OK;
}

/* M, S[2], P[2], R[2], each (N+1)^2 row-major; S/P/R stacked lo then hi. */
int ora_mortar_ops(int N, double* M, double* S, double* P, double* R) {
  if (N < 1 || N > 16) return ORA_ERR_ARG;
  Ops o = make_ops(N);
  int nn = (N + 1) * (N + 1);
  std::copy(o.M.begin(), o.M.end(), M);
  for (int b = 0; b < 2; ++b) {
    std::copy(o.S[b].begin(), o.S[b].end(), S + b * nn);
    std::copy(o.P[b].begin(), o.P[b].end(), P + b * nn);
    std::copy(o.R[b].begin(), o.R[b].end(), R + b * nn);
  }
  return ORA_OK;
}

/* ------------------------------------------------------------------ */
/* Mesh: leaf list -> canonical face lists (R15,R29) */
/* ------------------------------------------------------------------ */

struct ora_mesh {
  int dim, N;
  int64_t n;
  std::vector<int> level;
  std::vector<int> anchor; /* n*3, unused axes 0 */
  std::vector<int32_t> conf;    /* [nc][4]  eL fL eR fR      */
  std::vector<int32_t> nonconf; /* [nn][2+2*2^(d-1)]          */
  std::vector<int32_t> bnd;     /* [nb][2]                    */
};

typedef std::tuple<int, int, int, int> Key;

/* Neighbour cell coordinate along axis d at level lev; returns false if it
 * leaves a non-periodic domain. */
static bool step_coord(const ora_params* p, int lev, int d, int s, int a, int* out) {
  long ext = (long)p->root[d] << lev;
  long b = (long)a + s;
  if (b < 0 || b >= ext) {
    if (!p->periodic[d]) return false;
    b = (b + ext) % ext;
  }
  *out = (int)b;
  return true;
}

int ora_mesh_build(const ora_params* p, int64_t n, const int8_t* level, const int32_t* anchor,
                   ora_mesh** out) {
  *out = nullptr;
  int dim = p->dim;
  if ((dim != 2 && dim != 3) || p->order < 1 || n < 1) return ORA_ERR_ARG;
  ora_mesh* m = new ora_mesh;
  m->dim = dim;
  m->N = p->order;
  m->n = n;
  m->level.resize(n);
  m->anchor.assign(n * 3, 0);
  std::map<Key, int> leaf;
  for (int64_t e = 0; e < n; ++e) {
    int l = level[e];
    if (l < 0 || l > p->max_level) { delete m; return ORA_ERR_MESH; }
    m->level[e] = l;
    int a[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) {
      a[d] = anchor[e * dim + d];
      if (a[d] < 0 || a[d] >= ((long)p->root[d] << l)) { delete m; return ORA_ERR_MESH; }
      m->anchor[e * 3 + d] = a[d];
    }
    Key k(l, a[0], a[1], a[2]);
    if (leaf.count(k)) { delete m; return ORA_ERR_MESH; } /* duplicate */
    leaf[k] = (int)e;
  }
  /* no leaf is an ancestor of another leaf */
  for (int64_t e = 0; e < n; ++e) {
    int l = m->level[e];
    for (int la = 0; la < l; ++la) {
      int sh = l - la;
      Key k(la, m->anchor[e * 3] >> sh, m->anchor[e * 3 + 1] >> sh, m->anchor[e * 3 + 2] >> sh);
      if (leaf.count(k)) { delete m; return ORA_ERR_MESH; }
    }
  }
  /* exact tiling: sum of leaf volumes (in finest cells) == domain volume */
  {
    int L = p->max_level;
    unsigned long long tot = 0, want = 1;
    for (int d = 0; d < dim; ++d) want *= (unsigned long long)p->root[d] << L;
    for (int64_t e = 0; e < n; ++e) tot += 1ull << (dim * (L - m->level[e]));
    if (tot != want) { delete m; return ORA_ERR_MESH; }
  }
  int nsub = 1 << (dim - 1);
  for (int64_t e = 0; e < n; ++e) {
    int l = m->level[e];
    const int* a = &m->anchor[e * 3];
    for (int f = 0; f < 2 * dim; ++f) {
      int d = f / 2, s = (f % 2) ? 1 : -1;
      int nb[3] = {a[0], a[1], a[2]};
      if (!step_coord(p, l, d, s, a[d], &nb[d])) {
        m->bnd.push_back((int32_t)e);
        m->bnd.push_back(f);
        continue;
      }
      auto it = leaf.find(Key(l, nb[0], nb[1], nb[2]));
      if (it != leaf.end()) {
        if (s > 0) {
          m->conf.push_back((int32_t)e);
          m->conf.push_back(f);
          m->conf.push_back(it->second);
          m->conf.push_back(f - 1);
        }
        continue;
      }
      if (l > 0 && leaf.count(Key(l - 1, nb[0] >> 1, nb[1] >> 1, nb[2] >> 1)))
        continue; /* fine side of a 2:1 face: emitted by the coarse owner */
      /* all 2^(d-1) children across the face must be leaves */
      int tang[2], nt = 0;
      for (int ax = 0; ax < dim; ++ax)
        if (ax != d) tang[nt++] = ax;
      std::vector<int32_t> kids;
      bool ok = (l + 1 <= p->max_level);
      for (int b = 0; b < nsub && ok; ++b) {
        int c[3] = {2 * nb[0], 2 * nb[1], 2 * nb[2]};
        c[d] += (s > 0) ? 0 : 1;
        c[tang[0]] += b & 1;
        if (dim == 3) c[tang[1]] += (b >> 1) & 1;
        auto jt = leaf.find(Key(l + 1, c[0], c[1], c[2]));
        if (jt == leaf.end()) ok = false;
        else kids.push_back(jt->second);
      }
      if (!ok) { delete m; return ORA_ERR_UNBALANCED; }
      m->nonconf.push_back((int32_t)e);
      m->nonconf.push_back(f);
      for (int b = 0; b < nsub; ++b) {
        m->nonconf.push_back(kids[b]);
        m->nonconf.push_back(f ^ 1);
      }
    }
  }
  *out = m;
  return ORA_OK;
}

void ora_mesh_free(ora_mesh* m) { delete m; }

int ora_mesh_counts(const ora_mesh* m, int64_t* nc, int64_t* nn, int64_t* nb) {
  int w = 2 + 2 * (1 << (m->dim - 1));
  *nc = (int64_t)m->conf.size() / 4;
  *nn = (int64_t)m->nonconf.size() / w;
  *nb = (int64_t)m->bnd.size() / 2;
  return ORA_OK;
}

int ora_mesh_faces(const ora_mesh* m, int32_t* conf, int32_t* nonconf, int32_t* bnd) {
  std::copy(m->conf.begin(), m->conf.end(), conf);
  std::copy(m->nonconf.begin(), m->nonconf.end(), nonconf);
  std::copy(m->bnd.begin(), m->bnd.end(), bnd);
  return ORA_OK;
}

}  // extern "C"

/* ------------------------------------------------------------------ */
/* Physics (Sec. 2.1) and Rusanov flux (Sec. 2.2)   */
/* ------------------------------------------------------------------ */
namespace {

/* Point state: perturbation variables (rho', U_1..U_dim, Theta') plus the
 * background (rho_bar, Theta_bar, P_bar) at that point (R1, R3, R13). */
struct Pt {
  double rp, U[3], Tp;
  double rb, Tb, Pb;
};

struct Derived {
  double rho, Th, Pp, P, u[3], a;
};

/* EOS P = p0 (R Theta / p0)^gamma in perturbation form about the
 * hydrostatic background: P' = Pbar*expm1(gamma*log1p(Theta'/Thetabar)),
 * reading R2; u = U/rho; sound speed a = sqrt(gamma P / rho) (R6). */
Derived derive(const ora_params* p, int dim, const Pt& s) {
  Derived o;
  o.rho = s.rb + s.rp;
  o.Th = s.Tb + s.Tp;
  o.Pp = s.Pb * std::expm1(p->gamma * std::log1p(s.Tp / s.Tb));
  o.P = s.Pb + o.Pp;
  for (int j = 0; j < 3; ++j) o.u[j] = j < dim ? s.U[j] / o.rho : 0.0;
  o.a = std::sqrt(p->gamma * o.P / o.rho);
  return o;
}

/* Flux along axis d (eq. eulervector; R5: P' in the momentum flux):
 * F^d = (U_d, U_j u_d + delta_jd P', Theta u_d). */
void flux(int dim, int d, const Pt& s, const Derived& v, double* F) {
  F[0] = s.U[d];
  for (int j = 0; j < dim; ++j) F[1 + j] = s.U[j] * v.u[d] + (j == d ? v.Pp : 0.0);
  F[1 + dim] = v.Th * v.u[d];
}

/* Rusanov F*.n with n = sgn * e_d (R6 wave speed, R7 jump sign):
 * F*.n = 1/2 (F(q-).n + F(q+).n) + 1/2 lambda (q- - q+),
 * lambda = max(|u-.n| + a-, |u+.n| + a+); the jump is taken on the
 * perturbation vector (rho', U, Theta') (reading R13b). */
void rusanov(const ora_params* p, int dim, int d, double sgn, const Pt& L, const Pt& R, double* out) {
  Derived vl = derive(p, dim, L), vr = derive(p, dim, R);
  double FL[5], FR[5];
  flux(dim, d, L, vl, FL);
  flux(dim, d, R, vr, FR);
  double lam = std::max(std::fabs(vl.u[d]) + vl.a, std::fabs(vr.u[d]) + vr.a);
  double jl[5], jr[5];
  jl[0] = L.rp;
  jr[0] = R.rp;
  for (int j = 0; j < dim; ++j) {
    jl[1 + j] = L.U[j];
    jr[1 + j] = R.U[j];
  }
  jl[1 + dim] = L.Tp;
  jr[1 + dim] = R.Tp;
  int F = dim + 2;
  for (int f = 0; f < F; ++f) out[f] = 0.5 * (sgn * FL[f] + sgn * FR[f]) + 0.5 * lam * (jl[f] - jr[f]);
}

struct Geo {
  int dim, N, n1, Np, F, vert;
  std::vector<long> rowoff;
};

Geo make_geo(const ora_params* p) {
  Geo g;
  g.dim = p->dim;
  g.N = p->order;
  g.n1 = g.N + 1;
  g.Np = 1;
  for (int d = 0; d < g.dim; ++d) g.Np *= g.n1;
  g.F = g.dim + 2;
  g.vert = g.dim - 1;
  g.rowoff.resize(p->max_level + 2);
  g.rowoff[0] = 0;
  for (int l = 0; l <= p->max_level; ++l)
    g.rowoff[l + 1] = g.rowoff[l] + ((long)p->root[g.vert] << l) * g.n1;
  return g;
}

/* node index of tensor index (R28: x fastest) */
int vol_index(const Geo& g, const int* idx) {
  int n = 0, s = 1;
  for (int a = 0; a < g.dim; ++a) {
    n += idx[a] * s;
    s *= g.n1;
  }
  return n;
}

void tensor_index(const Geo& g, int n, int* idx) {
  for (int a = 0; a < g.dim; ++a) {
    idx[a] = n % g.n1;
    n /= g.n1;
  }
}

/* volume node of face node t (tangential axes ascending, first fastest; R28) */
int face_node(const Geo& g, int f, int t) {
  int d = f / 2, idx[3] = {0, 0, 0};
  idx[d] = (f % 2) ? g.N : 0;
  for (int a = 0; a < g.dim; ++a)
    if (a != d) {
      idx[a] = t % g.n1;
      t /= g.n1;
    }
  return vol_index(g, idx);
}

double elem_h(const ora_params* p, int lev, int d) {
  return (p->hi[d] - p->lo[d]) / ((double)p->root[d] * std::ldexp(1.0, lev));
}

/* Point state of element e at node n (background row: (level, iz, k); R3). */
Pt node_state(const ora_params* p, const Geo& g, const ora_mesh* m, const double* bg, const double* q, long e,
              int n) {
  int idx[3];
  tensor_index(g, n, idx);
  long row = g.rowoff[m->level[e]] + (long)m->anchor[e * 3 + g.vert] * g.n1 + idx[g.vert];
  const double* qe = q + e * (long)g.F * g.Np;
  Pt s;
  s.rb = bg[3 * row + 0];
  s.Tb = bg[3 * row + 1];
  s.Pb = bg[3 * row + 2];
  s.rp = qe[n] - s.rb;
  for (int j = 0; j < 3; ++j) s.U[j] = j < g.dim ? qe[(1 + j) * g.Np + n] : 0.0;
  s.Tp = qe[(1 + g.dim) * g.Np + n] - s.Tb;
  return s;
}

/* Pointwise baseline (R41): the coarse face coordinate x in [-1, 1] lies
 * on sub-face b = 1 (upper half) iff x > 0 (x = 0 belongs to the lower one), where the
 * fine element's own coordinate is xi = 2x - 1 (upper) or 2x + 1 (lower).
 * ncmode 2 and 3 are DELIBERATELY WRONG variants that exist only so that
 * tests/test_oracle_nonconforming.py can show its pins catch them: 2 mirrors the
 * xi-map (xi = 2x + 1 on the upper half), 3 assigns x = 0 to the upper sub-face. */
int upper_sub(double x, int ncmode) { return (ncmode == 3 ? x >= 0.0 : x > 0.0) ? 1 : 0; }
double sub_xi(double x, int b, int ncmode) {
  const double shift = b ? -1.0 : 1.0;
  return 2.0 * x + (ncmode == 2 ? -shift : shift);
}

/* Strong-form dGSEM RHS (Sec. 2.2), element subset `mask`
 * (NULL = all).  dq/dt = V + S + lifts, per SURVEY 8(c) C.1:
 *   V   = - sum_d (2/h_d) sum_m D[i_d][m] F^d(node with i_d -> m)
 *   S   = - rho' g e_z
 *   lift: RHS(face node) += -(2/h_d)/w_0 (F*.n - F(q-).n)                   */
void rhs(const ora_params* p, const ora_mesh* m, const double* bg, const double* q, double* out,
         const uint8_t* mask, int ncmode = 0) {
  Geo g = make_geo(p);
  Ops o = make_ops(g.N);
  const int F = g.F, Np = g.Np, dim = g.dim, n1 = g.n1;
  const long E = m->n;
  auto sel = [&](long e) { return mask == nullptr || mask[e] != 0; };
  std::vector<double> Fl((size_t)dim * F * Np);
  for (long e = 0; e < E; ++e) {
    double* re = out + e * (long)F * Np;
    if (!sel(e)) continue;
    for (int i = 0; i < F * Np; ++i) re[i] = 0.0;
    /* A1-A2: point fluxes at every node */
    for (int n = 0; n < Np; ++n) {
      Pt s = node_state(p, g, m, bg, q, e, n);
      Derived v = derive(p, dim, s);
      for (int d = 0; d < dim; ++d) {
        double Fd[5];
        flux(dim, d, s, v, Fd);
        for (int f = 0; f < F; ++f) Fl[((size_t)d * F + f) * Np + n] = Fd[f];
      }
      /* A4: buoyancy source on the vertical momentum (R5) */
      re[(1 + g.vert) * Np + n] += -s.rp * p->g;
    }
    /* A3: volume flux divergence */
    for (int n = 0; n < Np; ++n) {
      int idx[3];
      tensor_index(g, n, idx);
      for (int f = 0; f < F; ++f) {
        double V = 0.0;
        for (int d = 0; d < dim; ++d) {
          double h = elem_h(p, m->level[e], d);
          double sum = 0.0;
          for (int mm = 0; mm < n1; ++mm) {
            int j[3] = {idx[0], idx[1], idx[2]};
            j[d] = mm;
            sum += o.D[idx[d] * n1 + mm] * Fl[((size_t)d * F + f) * Np + vol_index(g, j)];
          }
          V += -(2.0 / h) * sum;
        }
        re[f * Np + n] += V;
      }
    }
  }
  const int Nf = Np / n1;
  auto lift = [&](long e, int f, int t, const double* Fstar, const Pt& s) {
    if (!sel(e)) return;
    int d = f / 2;
    double sgn = (f % 2) ? 1.0 : -1.0;
    double h = elem_h(p, m->level[e], d);
    Derived v = derive(p, dim, s);
    double Fd[5];
    flux(dim, d, s, v, Fd);
    int n = face_node(g, f, t);
    double* re = out + e * (long)F * Np;
    for (int k = 0; k < F; ++k) re[k * Np + n] += -(2.0 / h) / o.w[0] * (Fstar[k] - sgn * Fd[k]);
  };
  /* A5-A6, A8: boundary faces, mirror ghost (R9) */
  for (size_t i = 0; i < m->bnd.size(); i += 2) {
    long e = m->bnd[i];
    int f = m->bnd[i + 1];
    if (!sel(e)) continue;
    int d = f / 2;
    double sgn = (f % 2) ? 1.0 : -1.0;
    for (int t = 0; t < Nf; ++t) {
      Pt L = node_state(p, g, m, bg, q, e, face_node(g, f, t));
      Pt R = L;
      R.U[d] = -L.U[d];
      double Fs[5];
      rusanov(p, dim, d, sgn, L, R, Fs);
      lift(e, f, t, Fs, L);
    }
  }
  /* conforming faces: owner eL (+ face) computes once; eR takes -F* */
  for (size_t i = 0; i < m->conf.size(); i += 4) {
    long eL = m->conf[i], eR = m->conf[i + 2];
    int fL = m->conf[i + 1], fR = m->conf[i + 3];
    if (!sel(eL) && !sel(eR)) continue;
    int d = fL / 2;
    for (int t = 0; t < Nf; ++t) {
      Pt L = node_state(p, g, m, bg, q, eL, face_node(g, fL, t));
      Pt R = node_state(p, g, m, bg, q, eR, face_node(g, fR, t));
      double Fs[5], Fneg[5];
      rusanov(p, dim, d, 1.0, L, R, Fs);
      for (int k = 0; k < F; ++k) Fneg[k] = -Fs[k];
      lift(eL, fL, t, Fs, L);
      lift(eR, fR, t, Fneg, R);
    }
  }
  /* A5-A7: nonconforming 2:1 faces, mortar method (R11-R14) */
  const int nsub = 1 << (dim - 1);
  const int wdt = 2 + 2 * nsub;
  std::vector<double> qc((size_t)F * Nf), qm((size_t)F * Nf), Fb((size_t)F * Nf), Fc((size_t)F * Nf);
  for (size_t i = 0; i < m->nonconf.size(); i += wdt) {
    long eC = m->nonconf[i];
    int fC = m->nonconf[i + 1];
    bool any = sel(eC);
    for (int b = 0; b < nsub; ++b) any = any || sel(m->nonconf[i + 2 + 2 * b]);
    if (!any) continue;
    int d = fC / 2;
    double sC = (fC % 2) ? 1.0 : -1.0;
    /* coarse trace as perturbation vector (R13) */
    for (int t = 0; t < Nf; ++t) {
      Pt s = node_state(p, g, m, bg, q, eC, face_node(g, fC, t));
      qc[0 * Nf + t] = s.rp;
      for (int j = 0; j < dim; ++j) qc[(1 + j) * Nf + t] = s.U[j];
      qc[(1 + dim) * Nf + t] = s.Tp;
    }
    std::fill(Fc.begin(), Fc.end(), 0.0);
    for (int b = 0; b < nsub; ++b) {
      long eF = m->nonconf[i + 2 + 2 * b];
      int fF = m->nonconf[i + 3 + 2 * b];
      int b1 = b & 1, b2 = (b >> 1) & 1;
      /* face -> mortar projection, tensor product of 1D P_b */
      for (int f = 0; f < F; ++f)
        for (int k = 0; k < Nf; ++k) {
          int k1 = k % n1, k2 = k / n1;
          double s = 0.0;
          for (int j = 0; j < Nf; ++j) {
            int j1 = j % n1, j2 = j / n1;
            double c = o.P[b1][k1 * n1 + j1];
            if (dim == 3) c *= o.P[b2][k2 * n1 + j2];
            s += c * qc[f * Nf + j];
          }
          qm[f * Nf + k] = s;
        }
      /* Riemann problem on the mortar: coarse projection vs fine trace
       * (fine side projection is the identity) */
      for (int t = 0; t < Nf; ++t) {
        Pt R = node_state(p, g, m, bg, q, eF, face_node(g, fF, t));
        Pt L;
        L.rb = R.rb;
        L.Tb = R.Tb;
        L.Pb = R.Pb; /* background of the mortar nodes = fine rows (R13) */
        L.rp = qm[0 * Nf + t];
        for (int j = 0; j < 3; ++j) L.U[j] = j < dim ? qm[(1 + j) * Nf + t] : 0.0;
        L.Tp = qm[(1 + dim) * Nf + t];
        double Fs[5], Fneg[5];
        rusanov(p, dim, d, sC, L, R, Fs);
        for (int k = 0; k < F; ++k) {
          Fb[k * Nf + t] = Fs[k];
          Fneg[k] = -Fs[k];
        }
        lift(eF, fF, t, Fneg, R);
      }
      /* mortar -> face back projection, s = 1/2 per tangential axis */
      for (int f = 0; f < F; ++f)
        for (int j = 0; j < Nf; ++j) {
          int j1 = j % n1, j2 = j / n1;
          double s = 0.0;
          for (int k = 0; k < Nf; ++k) {
            int k1 = k % n1, k2 = k / n1;
            double c = o.R[b1][j1 * n1 + k1];
            if (dim == 3) c *= o.R[b2][j2 * n1 + k2];
            s += c * Fb[f * Nf + k];
          }
          Fc[f * Nf + j] += s;
        }
    }
    if (ncmode == 0) {
      for (int t = 0; t < Nf; ++t) {
        Pt s = node_state(p, g, m, bg, q, eC, face_node(g, fC, t));
        double Fs[5];
        for (int k = 0; k < F; ++k) Fs[k] = Fc[k * Nf + t];
        lift(eC, fC, t, Fs, s);
      }
      continue;
    }
    /* NEXT-3 baseline, pointwise interpolation (reading R41): at each coarse
     * face node, the fine sub-face containing it (x = 0 belongs to the lower one) is
     * evaluated there -- its perturbation trace interpolated by the fine Lagrange basis
     * at the node's sub-face coordinate, plus the coarse node's background -- and the
     * Rusanov flux is taken against the coarse own state.  Not conservative. */
    for (int t = 0; t < Nf; ++t) {
      const int t1 = t % n1, t2 = t / n1;
      const int b1 = upper_sub(o.x[t1], ncmode), b2 = dim == 3 ? upper_sub(o.x[t2], ncmode) : 0;
      const int b = b1 + 2 * b2;
      const long eF = m->nonconf[i + 2 + 2 * b];
      const int fF = m->nonconf[i + 3 + 2 * b];
      const double xi1 = sub_xi(o.x[t1], b1, ncmode);
      const double xi2 = dim == 3 ? sub_xi(o.x[t2], b2, ncmode) : 0.0;
      Pt own = node_state(p, g, m, bg, q, eC, face_node(g, fC, t));
      double v[5] = {0, 0, 0, 0, 0};
      auto lag = [&](int k, double xi) {  /* l_k(xi) in long double, rounded once */
        long double l = 1.0L;
        for (int mm = 0; mm < n1; ++mm)
          if (mm != k) l *= ((long double)xi - o.x[mm]) / ((long double)o.x[k] - o.x[mm]);
        return (double)l;
      };
      for (int k = 0; k < Nf; ++k) {
        const int k1 = k % n1, k2 = k / n1;
        double c = lag(k1, xi1);
        if (dim == 3) c *= lag(k2, xi2);
        Pt r = node_state(p, g, m, bg, q, eF, face_node(g, fF, k));
        v[0] += c * r.rp;
        for (int j = 0; j < dim; ++j) v[1 + j] += c * r.U[j];
        v[1 + dim] += c * r.Tp;
      }
      Pt R = own;
      R.rp = v[0];
      for (int j = 0; j < 3; ++j) R.U[j] = j < dim ? v[1 + j] : 0.0;
      R.Tp = v[1 + dim];
      double Fs[5];
      rusanov(p, dim, d, sC, own, R, Fs);
      lift(eC, fC, t, Fs, own);
    }
  }
}


/* NEXT-3 passive tracer of the Euler flow (Sec. 2.1, eq. eulervector: C = rho c with
 * flux C U / rho = C u and no source; reading R45): C rides beside the Euler state q (one-way
 * coupling -- C never enters the dynamics) with the Euler path's own face treatment:
 *   F*.n = 1/2 (C- u-.n + C+ u+.n) + 1/2 lambda (C- - C+),
 * lambda = max(|u-.n| + a-, |u+.n| + a+) the Euler wave-speed bound at that face node (R6);
 * walls: the mirror ghost (R9; the flux is exactly 0); 2:1 faces: C projected onto the mortars
 * with P_b (R11, R12), u and lambda from the Euler mortar state of rhs() (projected perturbation
 * + fine background, R13), back projection with R_b -- conservative.
 *   dC/dt = - sum_d (2/h_d) D_d (C u_d) + lifts -(2/h_d)/w_0 (F*.n - C- u-.n).
 * c, out: compact [E][Np]; q compact [E][F][Np]. */
void passive(const ora_params* p, const ora_mesh* m, const double* bg, const double* q, const double* c, double* out) {
  Geo g = make_geo(p);
  Ops o = make_ops(g.N);
  const int F = g.F, Np = g.Np, dim = g.dim, n1 = g.n1, Nf = Np / n1;
  const long E = m->n;
  std::vector<double> Cu((size_t)dim * Np);
  for (long e = 0; e < E; ++e) {
    double* re = out + e * (long)Np;
    for (int n = 0; n < Np; ++n) {
      re[n] = 0.0;
      Pt s = node_state(p, g, m, bg, q, e, n);
      Derived v = derive(p, dim, s);
      for (int d = 0; d < dim; ++d) Cu[(size_t)d * Np + n] = c[e * Np + n] * v.u[d];
    }
    for (int n = 0; n < Np; ++n) {
      int idx[3];
      tensor_index(g, n, idx);
      for (int d = 0; d < dim; ++d) {
        double h = elem_h(p, m->level[e], d);
        double sum = 0.0;
        for (int mm = 0; mm < n1; ++mm) {
          int j[3] = {idx[0], idx[1], idx[2]};
          j[d] = mm;
          sum += o.D[idx[d] * n1 + mm] * Cu[(size_t)d * Np + vol_index(g, j)];
        }
        re[n] += -(2.0 / h) * sum;
      }
    }
  }
  /* Rusanov for C with the Euler states L, R at one face node (normal sgn e_d) */
  auto rus = [&](int d, double sgn, const Pt& L, const Pt& R, double CL, double CR) {
    Derived vl = derive(p, dim, L), vr = derive(p, dim, R);
    double lam = std::max(std::fabs(vl.u[d]) + vl.a, std::fabs(vr.u[d]) + vr.a);
    return 0.5 * (sgn * (CL * vl.u[d]) + sgn * (CR * vr.u[d])) + 0.5 * lam * (CL - CR);
  };
  auto lift = [&](long e, int f, int t, double Fstar, const Pt& s, double C) {
    int d = f / 2;
    double sgn = (f % 2) ? 1.0 : -1.0;
    double h = elem_h(p, m->level[e], d);
    Derived v = derive(p, dim, s);
    out[e * (long)Np + face_node(g, f, t)] += -(2.0 / h) / o.w[0] * (Fstar - sgn * (C * v.u[d]));
  };
  for (size_t i = 0; i < m->bnd.size(); i += 2) {  /* walls: mirror ghost */
    long e = m->bnd[i];
    int f = m->bnd[i + 1], d = f / 2;
    double sgn = (f % 2) ? 1.0 : -1.0;
    for (int t = 0; t < Nf; ++t) {
      int n = face_node(g, f, t);
      Pt L = node_state(p, g, m, bg, q, e, n);
      Pt R = L;
      R.U[d] = -L.U[d];
      lift(e, f, t, rus(d, sgn, L, R, c[e * Np + n], c[e * Np + n]), L, c[e * Np + n]);
    }
  }
  for (size_t i = 0; i < m->conf.size(); i += 4) {  /* conforming: owner computes, the other -F* */
    long eL = m->conf[i], eR = m->conf[i + 2];
    int fL = m->conf[i + 1], fR = m->conf[i + 3], d = fL / 2;
    for (int t = 0; t < Nf; ++t) {
      int nL = face_node(g, fL, t), nR = face_node(g, fR, t);
      Pt L = node_state(p, g, m, bg, q, eL, nL), R = node_state(p, g, m, bg, q, eR, nR);
      double Fs = rus(d, 1.0, L, R, c[eL * Np + nL], c[eR * Np + nR]);
      lift(eL, fL, t, Fs, L, c[eL * Np + nL]);
      lift(eR, fR, t, -Fs, R, c[eR * Np + nR]);
    }
  }
  const int nsub = 1 << (dim - 1), wdt = 2 + 2 * nsub;
  std::vector<double> qc((size_t)F * Nf), cc(Nf), qm((size_t)F * Nf), cm(Nf), Fb(Nf), Fc(Nf);
  for (size_t i = 0; i < m->nonconf.size(); i += wdt) {  /* 2:1 faces, mortar method */
    long eC = m->nonconf[i];
    int fC = m->nonconf[i + 1], d = fC / 2;
    double sC = (fC % 2) ? 1.0 : -1.0;
    for (int t = 0; t < Nf; ++t) {
      int n = face_node(g, fC, t);
      Pt s = node_state(p, g, m, bg, q, eC, n);
      qc[0 * Nf + t] = s.rp;
      for (int j = 0; j < dim; ++j) qc[(1 + j) * Nf + t] = s.U[j];
      qc[(1 + dim) * Nf + t] = s.Tp;
      cc[t] = c[eC * Np + n];
    }
    std::fill(Fc.begin(), Fc.end(), 0.0);
    for (int b = 0; b < nsub; ++b) {
      long eF = m->nonconf[i + 2 + 2 * b];
      int fF = m->nonconf[i + 3 + 2 * b];
      int b1 = b & 1, b2 = (b >> 1) & 1;
      for (int k = 0; k < Nf; ++k) {  /* face -> mortar projection of the Euler trace and of C */
        int k1 = k % n1, k2 = k / n1;
        double sc = 0.0;
        for (int f = 0; f < F; ++f) qm[f * Nf + k] = 0.0;
        for (int j = 0; j < Nf; ++j) {
          int j1 = j % n1, j2 = j / n1;
          double w = o.P[b1][k1 * n1 + j1];
          if (dim == 3) w *= o.P[b2][k2 * n1 + j2];
          for (int f = 0; f < F; ++f) qm[f * Nf + k] += w * qc[f * Nf + j];
          sc += w * cc[j];
        }
        cm[k] = sc;
      }
      for (int t = 0; t < Nf; ++t) {
        int n = face_node(g, fF, t);
        Pt R = node_state(p, g, m, bg, q, eF, n);
        Pt L;
        L.rb = R.rb;
        L.Tb = R.Tb;
        L.Pb = R.Pb;
        L.rp = qm[0 * Nf + t];
        for (int j = 0; j < 3; ++j) L.U[j] = j < dim ? qm[(1 + j) * Nf + t] : 0.0;
        L.Tp = qm[(1 + dim) * Nf + t];
        double Fs = rus(d, sC, L, R, cm[t], c[eF * Np + n]);
        Fb[t] = Fs;
        lift(eF, fF, t, -Fs, R, c[eF * Np + n]);
      }
      for (int j = 0; j < Nf; ++j) {  /* mortar -> face back projection */
        int j1 = j % n1, j2 = j / n1;
        double s = 0.0;
        for (int k = 0; k < Nf; ++k) {
          int k1 = k % n1, k2 = k / n1;
          double w = o.R[b1][j1 * n1 + k1];
          if (dim == 3) w *= o.R[b2][j2 * n1 + k2];
          s += w * Fb[k];
        }
        Fc[j] += s;
      }
    }
    for (int t = 0; t < Nf; ++t) {
      int n = face_node(g, fC, t);
      Pt s = node_state(p, g, m, bg, q, eC, n);
      lift(eC, fC, t, Fc[t], s, c[eC * Np + n]);
    }
  }
}

/* NEXT-3 artificial viscosity ("artificial viscosity of mu = 1.5 m^2/s"; the
 * discretisation is unspecified -- reading R42): V = mu div grad u of the perturbation
 * vector u = (rho', U, Theta'), BR1-style in strong form:
 *   sigma_d = (2/h_d) D_d u + (2/h_d)/w0 n_d (u* - u-)            at face nodes
 *   V       = mu sum_d [ (2/h_d) D_d sigma_d + (2/h_d)/w0 n_d (sigma_d* - sigma_d-) ]
 * central values u* = {u}, sigma* = {sigma}; walls: u* = u-, sigma_d* = 0 (no diffusive
 * flux); 2:1 faces through the mortars: m_b = 1/2 (P_b v_coarse + v_fine,b), fine side
 * v* = m_b, coarse side v* = sum_b R_b m_b (R11, R12) -- conservative like the inviscid
 * mortar flux.  out[e][f][n] = V (overwritten). */
void visc(const ora_params* p, const ora_mesh* m, const double* bg, const double* q, double mu, double* out) {
  Geo g = make_geo(p);
  Ops o = make_ops(g.N);
  const int F = g.F, Np = g.Np, dim = g.dim, n1 = g.n1, Nf = Np / n1, NF = 2 * dim;
  const long E = m->n;
  const int nsub = 1 << (dim - 1), wdt = 2 + 2 * nsub;
  std::vector<double> u((size_t)E * F * Np), sig((size_t)E * dim * F * Np, 0.0);
  for (long e = 0; e < E; ++e)
    for (int n = 0; n < Np; ++n) {
      Pt s = node_state(p, g, m, bg, q, e, n);
      u[((size_t)e * F + 0) * Np + n] = s.rp;
      for (int j = 0; j < dim; ++j) u[((size_t)e * F + 1 + j) * Np + n] = s.U[j];
      u[((size_t)e * F + 1 + dim) * Np + n] = s.Tp;
    }
  /* central face values of a nodal field val(e, k, n) at every element face node:
   * star[((e * NF + face) * F + k) * Nf + t] */
  auto face_star = [&](auto&& val, bool wall_zero, std::vector<double>& star) {
    star.assign((size_t)E * NF * F * Nf, 0.0);
    auto at = [&](long e, int f, int k, int t) -> double& { return star[(((size_t)e * NF + f) * F + k) * Nf + t]; };
    for (size_t i = 0; i < m->conf.size(); i += 4) {
      long eL = m->conf[i], eR = m->conf[i + 2];
      int fL = m->conf[i + 1], fR = m->conf[i + 3];
      for (int k = 0; k < F; ++k)
        for (int t = 0; t < Nf; ++t) {
          double v = 0.5 * (val(eL, k, face_node(g, fL, t)) + val(eR, k, face_node(g, fR, t)));
          at(eL, fL, k, t) = v;
          at(eR, fR, k, t) = v;
        }
    }
    for (size_t i = 0; i < m->bnd.size(); i += 2) {
      long e = m->bnd[i];
      int f = m->bnd[i + 1];
      for (int k = 0; k < F; ++k)
        for (int t = 0; t < Nf; ++t) at(e, f, k, t) = wall_zero ? 0.0 : val(e, k, face_node(g, f, t));
    }
    std::vector<double> mb(Nf);
    for (size_t i = 0; i < m->nonconf.size(); i += wdt) {
      long eC = m->nonconf[i];
      int fC = m->nonconf[i + 1];
      for (int b = 0; b < nsub; ++b) {
        long eF = m->nonconf[i + 2 + 2 * b];
        int fF = m->nonconf[i + 3 + 2 * b];
        int b1 = b & 1, b2 = (b >> 1) & 1;
        for (int k = 0; k < F; ++k) {
          for (int t = 0; t < Nf; ++t) {
            int t1 = t % n1, t2 = t / n1;
            double pc = 0.0;
            for (int j = 0; j < Nf; ++j) {
              int j1 = j % n1, j2 = j / n1;
              double c = o.P[b1][t1 * n1 + j1];
              if (dim == 3) c *= o.P[b2][t2 * n1 + j2];
              pc += c * val(eC, k, face_node(g, fC, j));
            }
            mb[t] = 0.5 * (pc + val(eF, k, face_node(g, fF, t)));
            at(eF, fF, k, t) = mb[t];
          }
          for (int j = 0; j < Nf; ++j) {
            int j1 = j % n1, j2 = j / n1;
            double r = 0.0;
            for (int t = 0; t < Nf; ++t) {
              int t1 = t % n1, t2 = t / n1;
              double c = o.R[b1][j1 * n1 + t1];
              if (dim == 3) c *= o.R[b2][j2 * n1 + t2];
              r += c * mb[t];
            }
            at(eC, fC, k, j) += r;
          }
        }
      }
    }
  };
  /* pass 1: gradients */
  for (long e = 0; e < E; ++e)
    for (int d = 0; d < dim; ++d) {
      double h = elem_h(p, m->level[e], d);
      for (int k = 0; k < F; ++k)
        for (int n = 0; n < Np; ++n) {
          int idx[3];
          tensor_index(g, n, idx);
          double sum = 0.0;
          for (int mm = 0; mm < n1; ++mm) {
            int j[3] = {idx[0], idx[1], idx[2]};
            j[d] = mm;
            sum += o.D[idx[d] * n1 + mm] * u[((size_t)e * F + k) * Np + vol_index(g, j)];
          }
          sig[(((size_t)e * dim + d) * F + k) * Np + n] = (2.0 / h) * sum;
        }
    }
  std::vector<double> star;
  face_star([&](long e, int k, int n) { return u[((size_t)e * F + k) * Np + n]; }, false, star);
  for (long e = 0; e < E; ++e)
    for (int f = 0; f < NF; ++f) {
      int d = f / 2;
      double sgn = (f % 2) ? 1.0 : -1.0, h = elem_h(p, m->level[e], d);
      for (int k = 0; k < F; ++k)
        for (int t = 0; t < Nf; ++t) {
          int n = face_node(g, f, t);
          double st = star[(((size_t)e * NF + f) * F + k) * Nf + t];
          sig[(((size_t)e * dim + d) * F + k) * Np + n] += (2.0 / h) / o.w[0] * sgn * (st - u[((size_t)e * F + k) * Np + n]);
        }
    }
  /* pass 2: divergence of mu sigma */
  for (long e = 0; e < E; ++e)
    for (int k = 0; k < F; ++k)
      for (int n = 0; n < Np; ++n) {
        int idx[3];
        tensor_index(g, n, idx);
        double V = 0.0;
        for (int d = 0; d < dim; ++d) {
          double h = elem_h(p, m->level[e], d), sum = 0.0;
          for (int mm = 0; mm < n1; ++mm) {
            int j[3] = {idx[0], idx[1], idx[2]};
            j[d] = mm;
            sum += o.D[idx[d] * n1 + mm] * sig[(((size_t)e * dim + d) * F + k) * Np + vol_index(g, j)];
          }
          V += (2.0 / h) * sum;
        }
        out[((size_t)e * F + k) * Np + n] = mu * V;
      }
  for (int d = 0; d < dim; ++d) {
    face_star([&](long e, int k, int n) { return sig[(((size_t)e * dim + d) * F + k) * Np + n]; }, true, star);
    for (long e = 0; e < E; ++e)
      for (int f = 2 * d; f < 2 * d + 2; ++f) {
        double sgn = (f % 2) ? 1.0 : -1.0, h = elem_h(p, m->level[e], d);
        for (int k = 0; k < F; ++k)
          for (int t = 0; t < Nf; ++t) {
            int n = face_node(g, f, t);
            double st = star[(((size_t)e * NF + f) * F + k) * Nf + t];
            out[((size_t)e * F + k) * Np + n] +=
                mu * (2.0 / h) / o.w[0] * sgn * (st - sig[(((size_t)e * dim + d) * F + k) * Np + n]);
          }
      }
  }
}


/* Kinematic tracer (the paper's LeVeque test, §4.2; readings R43, R41):
 * dC/dt = - div(C u), prescribed wind u at the nodes (s fields 1..dim), C in field 0.
 * Upwind flux F*.n = 1/2 (C- + C+) u.n + 1/2 |u.n| (C- - C+), u.n from the average of
 * both sides' nodal winds (conforming) or the fine side's wind (mortar nodes);
 * impermeable walls F*.n = 0; 2:1 faces by mortars (ncmode 0) or the pointwise
 * baseline (ncmode 1).  out: field 0 = dC/dt (other fields untouched). */
void tracer(const ora_params* p, const ora_mesh* m, const double* s, double* out, int ncmode) {
  Geo g = make_geo(p);
  Ops o = make_ops(g.N);
  const int F = g.F, Np = g.Np, dim = g.dim, n1 = g.n1, Nf = Np / n1;
  const long E = m->n;
  const int nsub = 1 << (dim - 1), wdt = 2 + 2 * nsub;
  auto C = [&](long e, int n) { return s[((size_t)e * F + 0) * Np + n]; };
  auto U = [&](long e, int d, int n) { return s[((size_t)e * F + 1 + d) * Np + n]; };
  auto upw = [](double Cm, double Cp, double un) { return 0.5 * (Cm + Cp) * un + 0.5 * std::fabs(un) * (Cm - Cp); };
  for (long e = 0; e < E; ++e)
    for (int n = 0; n < Np; ++n) {
      int idx[3];
      tensor_index(g, n, idx);
      double r = 0.0;
      for (int d = 0; d < dim; ++d) {
        double h = elem_h(p, m->level[e], d), sum = 0.0;
        for (int mm = 0; mm < n1; ++mm) {
          int j[3] = {idx[0], idx[1], idx[2]};
          j[d] = mm;
          int nj = vol_index(g, j);
          sum += o.D[idx[d] * n1 + mm] * (C(e, nj) * U(e, d, nj));
        }
        r += -(2.0 / h) * sum;
      }
      out[((size_t)e * F + 0) * Np + n] = r;
    }
  auto lift = [&](long e, int f, int t, double Fs) {
    int d = f / 2;
    double sgn = (f % 2) ? 1.0 : -1.0, h = elem_h(p, m->level[e], d);
    int n = face_node(g, f, t);
    double Fm = C(e, n) * (sgn * U(e, d, n));
    out[((size_t)e * F + 0) * Np + n] += -(2.0 / h) / o.w[0] * (Fs - Fm);
  };
  for (size_t i = 0; i < m->bnd.size(); i += 2)
    for (int t = 0; t < Nf; ++t) lift(m->bnd[i], m->bnd[i + 1], t, 0.0);
  for (size_t i = 0; i < m->conf.size(); i += 4) {
    long eL = m->conf[i], eR = m->conf[i + 2];
    int fL = m->conf[i + 1], fR = m->conf[i + 3], d = fL / 2;
    double sL = (fL % 2) ? 1.0 : -1.0;
    for (int t = 0; t < Nf; ++t) {
      int nL = face_node(g, fL, t), nR = face_node(g, fR, t);
      double un = sL * (0.5 * (U(eL, d, nL) + U(eR, d, nR)));
      double Fs = upw(C(eL, nL), C(eR, nR), un);
      lift(eL, fL, t, Fs);
      lift(eR, fR, t, -Fs);
    }
  }
  std::vector<double> cm(Nf), fb(Nf), Fc(Nf);
  for (size_t i = 0; i < m->nonconf.size(); i += wdt) {
    long eC = m->nonconf[i];
    int fC = m->nonconf[i + 1], d = fC / 2;
    double sC = (fC % 2) ? 1.0 : -1.0;
    std::fill(Fc.begin(), Fc.end(), 0.0);
    for (int b = 0; b < nsub; ++b) {
      long eF = m->nonconf[i + 2 + 2 * b];
      int fF = m->nonconf[i + 3 + 2 * b], b1 = b & 1, b2 = (b >> 1) & 1;
      for (int k = 0; k < Nf; ++k) {
        int k1 = k % n1, k2 = k / n1;
        double v = 0.0;
        for (int j = 0; j < Nf; ++j) {
          int j1 = j % n1, j2 = j / n1;
          double c = o.P[b1][k1 * n1 + j1];
          if (dim == 3) c *= o.P[b2][k2 * n1 + j2];
          v += c * C(eC, face_node(g, fC, j));
        }
        int nk = face_node(g, fF, k);
        fb[k] = upw(v, C(eF, nk), sC * U(eF, d, nk));
        lift(eF, fF, k, -fb[k]);
      }
      for (int j = 0; j < Nf; ++j) {
        int j1 = j % n1, j2 = j / n1;
        double acc = 0.0;
        for (int k = 0; k < Nf; ++k) {
          int k1 = k % n1, k2 = k / n1;
          double r = o.R[b1][j1 * n1 + k1];
          if (dim == 3) r *= o.R[b2][j2 * n1 + k2];
          acc += r * fb[k];
        }
        Fc[j] += acc;
      }
    }
    for (int t = 0; t < Nf; ++t) {
      if (ncmode == 0) {
        lift(eC, fC, t, Fc[t]);
        continue;
      }
      const int t1 = t % n1, t2 = t / n1;
      const int b1 = upper_sub(o.x[t1], ncmode), b2 = dim == 3 ? upper_sub(o.x[t2], ncmode) : 0, b = b1 + 2 * b2;
      long eF = m->nonconf[i + 2 + 2 * b];
      int fF = m->nonconf[i + 3 + 2 * b];
      const double xi1 = sub_xi(o.x[t1], b1, ncmode), xi2 = dim == 3 ? sub_xi(o.x[t2], b2, ncmode) : 0.0;
      auto lag = [&](int k, double xi) {
        long double l = 1.0L;
        for (int mm = 0; mm < n1; ++mm)
          if (mm != k) l *= ((long double)xi - o.x[mm]) / ((long double)o.x[k] - o.x[mm]);
        return (double)l;
      };
      double cp = 0.0;
      for (int k = 0; k < Nf; ++k) {
        double c = lag(k % n1, xi1);
        if (dim == 3) c *= lag(k / n1, xi2);
        cp += c * C(eF, face_node(g, fF, k));
      }
      int n = face_node(g, fC, t);
      lift(eC, fC, t, upw(C(eC, n), cp, sC * U(eC, d, n)));
    }
  }
}

}  // namespace

extern "C" {

/* q, out: compact [E][F][Np]; bg: rows (rho_bar, Theta_bar, P_bar) ordered
 * (level, iz, k); mask: NULL or E bytes (only masked elements computed). */
int ora_rhs(const ora_params* p, const ora_mesh* m, const double* bg, const double* q, double* out,
            const uint8_t* mask) {
  rhs(p, m, bg, q, out, mask);
  return ORA_OK;
}

/* NEXT-3 viscous term V = mu div grad u' (R42), out overwritten, compact [E][F][Np] */
int ora_visc(const ora_params* p, const ora_mesh* m, const double* bg, const double* q, double mu, double* out) {
  if (!(mu >= 0.0)) return ORA_ERR_ARG;
  visc(p, m, bg, q, mu, out);
  return ORA_OK;
}

/* kinematic tracer RHS (field 0 of out), s compact [E][F][Np]: field 0 = C, 1..dim = wind */
int ora_tracer_rhs(const ora_params* p, const ora_mesh* m, const double* s, double* out, int ncmode) {
  if (ncmode < 0 || ncmode > 3) return ORA_ERR_ARG;  /* 2, 3: test-only mutants (upper_sub) */
  tracer(p, m, s, out, ncmode);
  return ORA_OK;
}

/* NEXT-3 passive tracer of the Euler flow (R45): out[E][Np] = dC/dt for C = rho c (compact [E][Np])
 * advected by the Euler state q (compact [E][F][Np]) with the Euler faces' wave speeds. */
int ora_passive_rhs(const ora_params* p, const ora_mesh* m, const double* bg, const double* q, const double* c,
                    double* out) {
  passive(p, m, bg, q, c, out);
  return ORA_OK;
}

/* ncmode 0: mortars (as ora_rhs); 1: pointwise interpolation on the coarse side of 2:1 faces;
 * 2, 3: deliberately wrong pointwise variants for the pin-sensitivity tests (upper_sub) */
int ora_rhs_nc(const ora_params* p, const ora_mesh* m, const double* bg, const double* q, double* out,
               const uint8_t* mask, int ncmode) {
  if (ncmode < 0 || ncmode > 3) return ORA_ERR_ARG;
  rhs(p, m, bg, q, out, mask, ncmode);
  return ORA_OK;
}

/* SSP-RK3 Shu-Osher stage (R17): q_out = a q_n + b (q_in + dt L(q_in)),
 * (a,b) = (0,1), (3/4,1/4), (1/3,2/3), evaluated in the algebraically equal
 * increment form q_out = q_n + b ((q_in - q_n) + dt L(q_in)) (a = 1 - b), so
 * that a zero RHS leaves the state bitwise unchanged (P7b). */
int ora_rk_stage(const ora_params* p, const ora_mesh* m, const double* bg, int stage, double dt,
                 const double* q_n, const double* q_in, double* q_out, const uint8_t* mask) {
  if (stage < 0 || stage > 2 || !(dt > 0.0)) return ORA_ERR_ARG;
  Geo g = make_geo(p);
  long tot = m->n * (long)g.F * g.Np;
  /* uninitialised: rhs() zeroes and fills the rows of the selected elements, the only ones read
   * below (a masked call then costs O(selected), which the threaded cpu_baseline relies on) */
  std::unique_ptr<double[]> L(new double[tot]);
  rhs(p, m, bg, q_in, L.get(), mask);
  const double B[3] = {1.0, 1.0 / 4.0, 2.0 / 3.0};
  long per = (long)g.F * g.Np;
  for (long e = 0; e < m->n; ++e) {
    if (mask && !mask[e]) continue;
    for (long i = e * per; i < (e + 1) * per; ++i) {
      if (stage == 0) q_out[i] = q_in[i] + dt * L[i];
      else q_out[i] = q_n[i] + B[stage] * ((q_in[i] - q_n[i]) + dt * L[i]);
    }
  }
  return ORA_OK;
}

/* Refine (R16): child_b = (kron_axis P_{b_axis}) parent, with
 * child id b = b_x + 2 b_y (+ 4 b_z); children of pair i are the 2^d
 * consecutive elements child0_dst[i] ... in q_dst (compact layout). */
int ora_refine(int dim, int N, int64_t n, const int32_t* parent_src, const int32_t* child0_dst,
               const double* q_src, double* q_dst) {
  Ops o = make_ops(N);
  int n1 = N + 1, Np = 1;
  for (int d = 0; d < dim; ++d) Np *= n1;
  int F = dim + 2, nch = 1 << dim;
  for (int64_t i = 0; i < n; ++i) {
    const double* par = q_src + (long)parent_src[i] * F * Np;
    for (int b = 0; b < nch; ++b) {
      double* ch = q_dst + ((long)child0_dst[i] + b) * F * Np;
      for (int f = 0; f < F; ++f)
        for (int c = 0; c < Np; ++c) {
          int ci[3] = {c % n1, (c / n1) % n1, c / (n1 * n1)};
          double s = 0.0;
          for (int pn = 0; pn < Np; ++pn) {
            int pi[3] = {pn % n1, (pn / n1) % n1, pn / (n1 * n1)};
            double k = 1.0;
            for (int a = 0; a < dim; ++a) k *= o.P[(b >> a) & 1][ci[a] * n1 + pi[a]];
            s += k * par[f * Np + pn];
          }
          ch[f * Np + c] = s;
        }
    }
  }
  return ORA_OK;
}

/* Coarsen (FV analogue P:273-277): parent = sum_b (kron_axis R_{b_axis}) child_b. */
int ora_coarsen(int dim, int N, int64_t n, const int32_t* child0_src, const int32_t* parent_dst,
                const double* q_src, double* q_dst) {
  Ops o = make_ops(N);
  int n1 = N + 1, Np = 1;
  for (int d = 0; d < dim; ++d) Np *= n1;
  int F = dim + 2, nch = 1 << dim;
  for (int64_t i = 0; i < n; ++i) {
    double* par = q_dst + (long)parent_dst[i] * F * Np;
    for (int f = 0; f < F; ++f)
      for (int pn = 0; pn < Np; ++pn) {
        int pi[3] = {pn % n1, (pn / n1) % n1, pn / (n1 * n1)};
        double s = 0.0;
        for (int b = 0; b < nch; ++b) {
          const double* ch = q_src + ((long)child0_src[i] + b) * F * Np;
          for (int c = 0; c < Np; ++c) {
            int ci[3] = {c % n1, (c / n1) % n1, c / (n1 * n1)};
            double k = 1.0;
            for (int a = 0; a < dim; ++a) k *= o.R[(b >> a) & 1][pi[a] * n1 + ci[a]];
            s += k * ch[f * Np + c];
          }
        }
        par[f * Np + pn] = s;
      }
  }
  return ORA_OK;
}

/* integral_f = sum_e prod_d (h_d/2) sum_n w_n q_{f,n}, Neumaier-compensated (R20). */
int ora_integrals(const ora_params* p, const ora_mesh* m, const double* q, double* out) {
  Geo g = make_geo(p);
  Ops o = make_ops(g.N);
  for (int f = 0; f < g.F; ++f) {
    double sum = 0.0, comp = 0.0;
    for (long e = 0; e < m->n; ++e) {
      double J = 1.0;
      for (int d = 0; d < g.dim; ++d) J *= 0.5 * elem_h(p, m->level[e], d);
      const double* qe = q + e * (long)g.F * g.Np + (long)f * g.Np;
      for (int n = 0; n < g.Np; ++n) {
        int idx[3];
        tensor_index(g, n, idx);
        double wn = 1.0;
        for (int d = 0; d < g.dim; ++d) wn *= o.w[idx[d]];
        double term = J * wn * qe[n];
        double t = sum + term;
        if (std::fabs(sum) >= std::fabs(term)) comp += (sum - t) + term;
        else comp += (term - t) + sum;
        sum = t;
      }
    }
    out[f] = sum + comp;
  }
  return ORA_OK;
}

/* Single point flux / Rusanov evaluation, exposed for the pin tests (P6).
 * pt = (rho', U_1..U_dim, Theta', rho_bar, Theta_bar, P_bar). */
int ora_point_flux(const ora_params* p, int d, const double* pt, double* F_out, double* derived_out) {
  int dim = p->dim;
  Pt s;
  s.rp = pt[0];
  for (int j = 0; j < 3; ++j) s.U[j] = j < dim ? pt[1 + j] : 0.0;
  s.Tp = pt[1 + dim];
  s.rb = pt[2 + dim];
  s.Tb = pt[3 + dim];
  s.Pb = pt[4 + dim];
  Derived v = derive(p, dim, s);
  flux(dim, d, s, v, F_out);
  if (derived_out) {
    derived_out[0] = v.rho;
    derived_out[1] = v.Th;
    derived_out[2] = v.Pp;
    derived_out[3] = v.P;
    derived_out[4] = v.a;
  }
  return ORA_OK;
}

int ora_rusanov(const ora_params* p, int d, double sgn, const double* ptL, const double* ptR, double* out) {
  int dim = p->dim;
  Pt s[2];
  const double* src[2] = {ptL, ptR};
  for (int k = 0; k < 2; ++k) {
    const double* pt = src[k];
    s[k].rp = pt[0];
    for (int j = 0; j < 3; ++j) s[k].U[j] = j < dim ? pt[1 + j] : 0.0;
    s[k].Tp = pt[1 + dim];
    s[k].rb = pt[2 + dim];
    s[k].Tb = pt[3 + dim];
    s[k].Pb = pt[4 + dim];
  }
  rusanov(p, dim, d, sgn, s[0], s[1], out);
  return ORA_OK;
}

}  // extern "C"
