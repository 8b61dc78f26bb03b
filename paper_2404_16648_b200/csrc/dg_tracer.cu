// dg_tracer.cu -- kinematic tracer transport (the paper's LeVeque test, PAPER.md:422-556
// §4.2; readings R43, R41 of DESIGN.md): dC/dt + div(C u) = 0 with a prescribed wind u,
// strong-form dGSEM on the same forest: volume divergence of C u with the LGL D, upwind
// face flux F*.n = 1/2 (C- + C+) u.n + 1/2 |u.n| (C- - C+) with u.n taken as the average
// of both sides' nodal winds (so both sides' fluxes are bitwise opposite), impermeable
// walls (F*.n = 0), 2:1 faces by the mortar method (coarse trace -> mortar with P_b, flux
// at the fine nodes with the fine wind, back projection R_b; conservative) or, with
// dg_set_nonconforming(ctx, 1), the pointwise-interpolation baseline on the coarse side.
//
// Array layout: the context's state rows; field 0 = C, fields 1..dim = the wind at the
// nodes (written by the caller for each stage time), other fields unused.  One thread
// per (element, node), global loads: the demonstration problems are small.
#include <cuda_runtime.h>

#include <cstdint>

#include "dg_device.cuh"

namespace dgi {
namespace {

struct TracerArgs {
  const double* s_in;   // rows: C, u_1..u_dim
  const double* s_n;    // RK: q_n rows (field 0 read)
  double* out;          // rows: field 0 written (rhs or RK stage), fields 1..dim copied from s_in
  const ElemDesc* desc;
  const int32_t* mort;
  const double* ops;
  int64_t n_elem, stride;
  double dt, rk_b;
  int mode, stage, ncmode;
};

template <int DIM, int N>
struct TC {
  static constexpr int n1 = N + 1, Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1, Nf = Np / n1, NSUB = 1 << (DIM - 1);
};

template <int DIM, int N>
__device__ __forceinline__ int tnode(int f, int t) {
  constexpr int n1 = N + 1;
  const int d = f >> 1, e = (f & 1) ? N : 0;
  if (DIM == 2) return d == 0 ? e + n1 * t : t + n1 * e;
  const int t1 = t % n1, t2 = t / n1;
  if (d == 0) return e + n1 * t1 + n1 * n1 * t2;
  if (d == 1) return t1 + n1 * e + n1 * n1 * t2;
  return t1 + n1 * t2 + n1 * n1 * e;
}

// upwind flux F*.n for the side holding Cm (own) and Cp (other), un = u.n from that side
__device__ __forceinline__ double upwind(double Cm, double Cp, double un) {
  return __fma_rn(0.5 * __dadd_rn(Cm, Cp), un, __dmul_rn(0.5 * fabs(un), __dsub_rn(Cm, Cp)));
}

template <int DIM, int N>
__global__ void __launch_bounds__(128) k_tracer(const TracerArgs a) {
  using C = TC<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, Nf = C::Nf, NSUB = C::NSUB;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_elem * Np) return;
  const int64_t e = i / Np;
  const int n = (int)(i - e * Np);
  const ElemDesc& D = a.desc[e];
  const int lev = elem_level(D.info);
  const double* se = a.s_in + e * a.stride;
  auto Cv = [&](int64_t ee, int nn) { return a.s_in[ee * a.stride + nn]; };
  auto Uv = [&](int64_t ee, int d, int nn) { return a.s_in[ee * a.stride + (1 + d) * Np + nn]; };
  const double w0inv = 1.0 / a.ops[OpsLayout::W(n1)];
  const double* P = a.ops + OpsLayout::P(n1, 0);
  const double* R = a.ops + OpsLayout::R(n1, 0);
  const double* Ip = a.ops + OpsLayout::I(n1, 0);
  int idx[3] = {n % n1, (n / n1) % n1, n / (n1 * n1)};
  const int str[3] = {1, n1, n1 * n1};
  double res = 0.0;
  for (int d = 0; d < DIM; ++d) {  // volume: - (2/h_d) D_d (C u_d)
    const double s2h = a.ops[OpsLayout::H(n1) + 3 * lev + d];
    const int base = n - idx[d] * str[d];
    double sum = 0.0;
    for (int m = 0; m < n1; ++m) {
      const int nm = base + m * str[d];
      sum = __fma_rn(a.ops[idx[d] * n1 + m], __dmul_rn(se[nm], se[(1 + d) * Np + nm]), sum);
    }
    res = __fma_rn(-s2h, sum, res);
  }
  for (int d = 0; d < DIM; ++d) {  // faces through this node
    for (int side = 0; side < 2; ++side) {
      if (idx[d] != (side ? N : 0)) continue;
      const int f = 2 * d + side;
      const double sgn = side ? 1.0 : -1.0;
      int t = 0, sc = 1;
      for (int ax = 0; ax < DIM; ++ax)
        if (ax != d) {
          t += idx[ax] * sc;
          sc *= n1;
        }
      const int kind = face_kind(D.info, f);
      const double Cm = se[n], unm = __dmul_rn(sgn, se[(1 + d) * Np + n]);
      double Fs;
      if (kind == kWall) {
        Fs = 0.0;
      } else if (kind == kConf) {
        const int64_t e2 = D.nbr[f];
        const int n2 = tnode<DIM, N>(f ^ 1, t);
        const double un = __dmul_rn(sgn, 0.5 * __dadd_rn(se[(1 + d) * Np + n], Uv(e2, d, n2)));
        Fs = upwind(Cm, Cv(e2, n2), un);
      } else if (kind == kFine) {  // mortar state: projected coarse trace at this fine node
        const int b = face_sub(D.info, f), b1 = b & 1, b2 = (b >> 1) & 1;
        const int t1 = t % n1, t2 = t / n1;
        const int64_t ec = D.nbr[f];
        double cm = 0.0;
        for (int j = 0; j < Nf; ++j) {
          const int j1 = j % n1, j2 = j / n1;
          const double c = DIM == 2 ? P[b1 * n1 * n1 + t1 * n1 + j1]
                                    : __dmul_rn(P[b1 * n1 * n1 + t1 * n1 + j1], P[b2 * n1 * n1 + t2 * n1 + j2]);
          cm = __fma_rn(c, Cv(ec, tnode<DIM, N>(f ^ 1, j)), cm);
        }
        // the coarse side's mortar flux upwind(cm, Cm, -unm), negated (bitwise)
        Fs = -upwind(cm, Cm, -unm);
      } else if (a.ncmode == 0) {  // coarse side, mortar method: fluxes on every sub-face, back projected
        const int j1 = t % n1, j2 = t / n1;
        double acc = 0.0;
        for (int b = 0; b < NSUB; ++b) {
          const int b1 = b & 1, b2 = (b >> 1) & 1;
          const int64_t ef = a.mort[D.nbr[f] * NSUB + b];
          for (int k = 0; k < Nf; ++k) {
            const int k1 = k % n1, k2 = k / n1;
            double cm = 0.0;
            for (int j = 0; j < Nf; ++j) {
              const int i1 = j % n1, i2 = j / n1;
              const double c = DIM == 2 ? P[b1 * n1 * n1 + k1 * n1 + i1]
                                        : __dmul_rn(P[b1 * n1 * n1 + k1 * n1 + i1], P[b2 * n1 * n1 + k2 * n1 + i2]);
              cm = __fma_rn(c, Cv(e, tnode<DIM, N>(f, j)), cm);
            }
            const int nk = tnode<DIM, N>(f ^ 1, k);
            const double fb = upwind(cm, Cv(ef, nk), __dmul_rn(sgn, Uv(ef, d, nk)));
            const double r = DIM == 2 ? R[b1 * n1 * n1 + j1 * n1 + k1]
                                      : __dmul_rn(R[b1 * n1 * n1 + j1 * n1 + k1], R[b2 * n1 * n1 + j2 * n1 + k2]);
            acc = __fma_rn(r, fb, acc);
          }
        }
        Fs = acc;
      } else {  // coarse side, pointwise interpolation of the containing fine sub-face (R41)
        const int j1 = t % n1, j2 = t / n1;
        const int b1 = 2 * j1 > N ? 1 : 0, b2 = (DIM == 3 && 2 * j2 > N) ? 1 : 0;
        const int64_t ef = a.mort[D.nbr[f] * NSUB + b1 + 2 * b2];
        double cp = 0.0;
        for (int k2 = 0; k2 < (DIM == 2 ? 1 : n1); ++k2)
          for (int k1 = 0; k1 < n1; ++k1) {
            const double c = DIM == 2 ? Ip[b1 * n1 * n1 + j1 * n1 + k1]
                                      : __dmul_rn(Ip[b1 * n1 * n1 + j1 * n1 + k1], Ip[b2 * n1 * n1 + j2 * n1 + k2]);
            cp = __fma_rn(c, Cv(ef, tnode<DIM, N>(f ^ 1, k1 + n1 * k2)), cp);
          }
        Fs = upwind(Cm, cp, unm);
      }
      const double s2h = a.ops[OpsLayout::H(n1) + 3 * lev + d];
      res = __fma_rn(-s2h * w0inv, __fma_rn(-Cm, unm, Fs), res);
    }
  }
  double* o = a.out + e * a.stride;
  if (a.mode == 0) {
    o[n] = res;
  } else if (a.stage == 0) {
    o[n] = __fma_rn(a.dt, res, se[n]);
  } else {
    const double qn = a.s_n[e * a.stride + n];
    o[n] = __fma_rn(a.rk_b, __fma_rn(a.dt, res, __dsub_rn(se[n], qn)), qn);
  }
  for (int d = 0; d < DIM; ++d) o[(1 + d) * Np + n] = se[(1 + d) * Np + n];
}

// ---------------------------------------------------------------------------------------------
// NEXT-3 passive tracer of the Euler flow (PAPER.md:73-89 eq. eulervector: C = rho c, flux
// C U / rho = C u, no source; reading R45).  C rides beside the Euler state q -- one-way
// coupling -- with the Euler path's face treatment: Rusanov F*.n = 1/2 (C- u-.n + C+ u+.n)
// + 1/2 lambda (C- - C+), lambda the Euler wave-speed bound of that face node (R6, the same
// `wave` as the stage kernels), walls by the mirror ghost (zero flux), 2:1 faces by the mortars
// (C and the Euler perturbation trace projected with P_b, the fine level's background, back
// projection with R_b; conservative).  One thread per (element, node), global loads: a
// capability beside the hot path, not part of it.  Rows: field 0 = C (other fields unused).
struct PassiveArgs {
  StageArgs sa;         // q_in (Euler stage input), desc, nbrow, mort, mortbg, bg4, ops, gamma, eos_c
  const double* c_in;   // C rows (field 0)
  const double* c_n;    // RK: C at t_n
  double* c_out;        // field 0 written
};

// Euler point state of element row e at node n (background row bgrow + k)
template <int DIM, int N>
__device__ __forceinline__ St pstate(const StageArgs& a, int64_t e, int n, int bgrow) {
  constexpr int n1 = N + 1, Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  St s;
  load_bg(s, a.bg4, bgrow + (DIM == 2 ? n / n1 : n / (n1 * n1)));
  const double* qe = a.q_in + e * a.stride;
  s.rp = __dsub_rn(__ldg(qe + n), s.rb);
#pragma unroll
  for (int j = 0; j < 3; ++j) s.U[j] = j < DIM ? __ldg(qe + (1 + j) * Np + n) : 0.0;
  s.Tp = __dsub_rn(__ldg(qe + (DIM + 1) * Np + n), s.Tb);
  return s;
}

// Rusanov for C with the Euler states L, R at one face node, normal sgn e_d (the Euler kernels'
// operation order: fma(lambda / 2, CL - CR, sgn / 2 (CL uL + CR uR)))
__device__ __forceinline__ double crus(const St& L, const Dv& vl, const St& R, const Dv& vr, double CL, double CR,
                                       int d, double sgn, double gamma) {
  const double ul = __dmul_rn(pick(L.U, d), vl.rinv), ur = __dmul_rn(pick(R.U, d), vr.rinv);
  const double lam = fmax(wave(ul, L, vl, gamma), wave(ur, R, vr, gamma));
  return __fma_rn(__dmul_rn(0.5, lam), __dsub_rn(CL, CR),
                  __dmul_rn(__dmul_rn(0.5, sgn), __dadd_rn(__dmul_rn(CL, ul), __dmul_rn(CR, ur))));
}

template <int DIM, int N>
__global__ void __launch_bounds__(128) k_passive(const PassiveArgs pa) {
  using C = TC<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, Nf = C::Nf, NSUB = C::NSUB;
  const StageArgs& a = pa.sa;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_elem * Np) return;
  const int64_t e = i / Np;
  const int n = (int)(i - e * Np);
  const ElemDesc D = a.desc[e];
  const int lev = elem_level(D.info);
  auto Cv = [&](int64_t ee, int nn) { return __ldg(pa.c_in + ee * a.stride + nn); };
  const double* P = a.ops + OpsLayout::P(n1, 0);
  const double* R = a.ops + OpsLayout::R(n1, 0);
  int idx[3] = {n % n1, (n / n1) % n1, n / (n1 * n1)};
  const int str[3] = {1, n1, n1 * n1};
  const double* qe = a.q_in + e * a.stride;
  double res = 0.0;
  for (int d = 0; d < DIM; ++d) {  // volume: - (2/h_d) D_d (C u_d), u_d = U_d / rho
    const double s2h = a.ops[OpsLayout::H(n1) + 3 * lev + d];
    const int base = n - idx[d] * str[d];
    double sum = 0.0;
    for (int m = 0; m < n1; ++m) {
      const int nm = base + m * str[d];
      const double ud = __dmul_rn(__ldg(qe + (1 + d) * Np + nm), fast_rcp(__ldg(qe + nm)));
      sum = __fma_rn(a.ops[idx[d] * n1 + m], __dmul_rn(Cv(e, nm), ud), sum);
    }
    res = __fma_rn(-s2h, sum, res);
  }
  const St own = pstate<DIM, N>(a, e, n, D.bgrow);
  const Dv vo = derive(own, a);
  const double Cm = Cv(e, n);
  for (int d = 0; d < DIM; ++d) {  // faces through this node
    for (int side = 0; side < 2; ++side) {
      if (idx[d] != (side ? N : 0)) continue;
      const int f = 2 * d + side;
      const double sgn = side ? 1.0 : -1.0;
      int t = 0, sc = 1;
      for (int ax = 0; ax < DIM; ++ax)
        if (ax != d) {
          t += idx[ax] * sc;
          sc *= n1;
        }
      const int kind = face_kind(D.info, f);
      double Fs;
      if (kind == kWall) {  // mirror ghost (R9): zero flux
        St Rg = own;
        if (d == 0) Rg.U[0] = -own.U[0];
        else if (d == 1) Rg.U[1] = -own.U[1];
        else Rg.U[2] = -own.U[2];
        Fs = crus(own, vo, Rg, vo, Cm, Cm, d, sgn, a.gamma);
      } else if (kind == kConf) {
        const int64_t e2 = D.nbr[f];
        const int n2 = tnode<DIM, N>(f ^ 1, t);
        const St Rn = pstate<DIM, N>(a, e2, n2, __ldg(a.nbrow + e * 8 + f));
        Fs = crus(own, vo, Rn, derive(Rn, a), Cm, Cv(e2, n2), d, sgn, a.gamma);
      } else if (kind == kFine) {  // the coarse trace projected onto this sub-face, fine background
        const int b = face_sub(D.info, f), b1 = b & 1, b2 = (b >> 1) & 1;
        const int t1 = t % n1, t2 = t / n1;
        const int64_t ec = D.nbr[f];
        const int bgc = __ldg(a.nbrow + e * 8 + f);
        St Lm = own;
        Lm.rp = 0.0;
        Lm.U[0] = Lm.U[1] = Lm.U[2] = 0.0;
        Lm.Tp = 0.0;
        double cm = 0.0;
        for (int j = 0; j < Nf; ++j) {
          const int j1 = j % n1, j2 = j / n1;
          const double w = DIM == 2 ? P[b1 * n1 * n1 + t1 * n1 + j1]
                                    : __dmul_rn(P[b1 * n1 * n1 + t1 * n1 + j1], P[b2 * n1 * n1 + t2 * n1 + j2]);
          const int nj = tnode<DIM, N>(f ^ 1, j);
          const St cs = pstate<DIM, N>(a, ec, nj, bgc);
          Lm.rp = __fma_rn(w, cs.rp, Lm.rp);
#pragma unroll
          for (int jj = 0; jj < DIM; ++jj) Lm.U[jj] = __fma_rn(w, cs.U[jj], Lm.U[jj]);
          Lm.Tp = __fma_rn(w, cs.Tp, Lm.Tp);
          cm = __fma_rn(w, Cv(ec, nj), cm);
        }
        // the coarse side's mortar flux crus(Lm, own, cm, C, d, sgn_c = -sgn), negated
        Fs = -crus(Lm, derive(Lm, a), own, vo, cm, Cm, d, -sgn, a.gamma);
      } else {  // coarse side: Rusanov on every sub-face's mortar nodes, back projected
        const int j1 = t % n1, j2 = t / n1;
        double acc = 0.0;
        for (int b = 0; b < NSUB; ++b) {
          const int b1 = b & 1, b2 = (b >> 1) & 1;
          const int mi = D.nbr[f] * NSUB + b;
          DG_CHECK(mi >= 0);
          const int64_t ef = __ldg(a.mort + mi);
          const int bgf = __ldg(a.mortbg + mi);
          for (int k = 0; k < Nf; ++k) {
            const int k1 = k % n1, k2 = k / n1;
            const int nk = tnode<DIM, N>(f ^ 1, k);
            const St Rf = pstate<DIM, N>(a, ef, nk, bgf);
            St Lm = Rf;  // fine level's background at the mortar node (R13)
            Lm.rp = 0.0;
            Lm.U[0] = Lm.U[1] = Lm.U[2] = 0.0;
            Lm.Tp = 0.0;
            double cmk = 0.0;
            for (int j = 0; j < Nf; ++j) {
              const int i1 = j % n1, i2 = j / n1;
              const double w = DIM == 2 ? P[b1 * n1 * n1 + k1 * n1 + i1]
                                        : __dmul_rn(P[b1 * n1 * n1 + k1 * n1 + i1], P[b2 * n1 * n1 + k2 * n1 + i2]);
              const int nj = tnode<DIM, N>(f, j);
              const St cs = pstate<DIM, N>(a, e, nj, D.bgrow);
              Lm.rp = __fma_rn(w, cs.rp, Lm.rp);
#pragma unroll
              for (int jj = 0; jj < DIM; ++jj) Lm.U[jj] = __fma_rn(w, cs.U[jj], Lm.U[jj]);
              Lm.Tp = __fma_rn(w, cs.Tp, Lm.Tp);
              cmk = __fma_rn(w, Cv(e, nj), cmk);
            }
            const double fb = crus(Lm, derive(Lm, a), Rf, derive(Rf, a), cmk, Cv(ef, nk), d, sgn, a.gamma);
            const double r = DIM == 2 ? R[b1 * n1 * n1 + j1 * n1 + k1]
                                      : __dmul_rn(R[b1 * n1 * n1 + j1 * n1 + k1], R[b2 * n1 * n1 + j2 * n1 + k2]);
            acc = __fma_rn(r, fb, acc);
          }
        }
        Fs = acc;
      }
      const double s2h = a.ops[OpsLayout::H(n1) + 3 * lev + d];
      const double un = __dmul_rn(pick(own.U, d), vo.rinv);
      res = __fma_rn(__dmul_rn(-s2h, a.w0inv), __fma_rn(-sgn, __dmul_rn(Cm, un), Fs), res);
    }
  }
  double* o = pa.c_out + e * a.stride;
  if (a.mode == 0) {
    o[n] = res;
  } else if (a.stage == 0) {
    o[n] = __fma_rn(a.dt, res, Cm);
  } else {
    const double cn = pa.c_n[e * a.stride + n];
    o[n] = __fma_rn(a.rk_b, __fma_rn(a.dt, res, __dsub_rn(Cm, cn)), cn);
  }
}

template <int DIM, int N>
int launch_passive_t(const PassiveArgs& a, cudaStream_t s) {
  constexpr int Np = TC<DIM, N>::Np;
  k_passive<DIM, N><<<(unsigned)((a.sa.n_elem * Np + 127) / 128), 128, 0, s>>>(a);
  return (int)cudaGetLastError();
}

template <int DIM, int N>
int launch_tracer_t(const TracerArgs& a, cudaStream_t s) {
  constexpr int Np = TC<DIM, N>::Np;
  k_tracer<DIM, N><<<(unsigned)((a.n_elem * Np + 127) / 128), 128, 0, s>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_tracer(int dim, int order, int mode, int stage, double dt, double rk_b, int ncmode, const double* s_n,
                  const double* s_in, double* out, const ElemDesc* desc, const int32_t* mort, const double* ops,
                  int64_t n_elem, int64_t stride, void* stream) {
  if (n_elem <= 0) return cudaSuccess;
  TracerArgs a{s_in, s_n, out, desc, mort, ops, n_elem, stride, dt, rk_b, mode, stage, ncmode};
  cudaStream_t s = (cudaStream_t)stream;
  switch (dim * 16 + order) {
#define DG_T(D_, N_) \
  case D_ * 16 + N_: return launch_tracer_t<D_, N_>(a, s);
    DG_T(2, 1) DG_T(2, 2) DG_T(2, 3) DG_T(2, 4) DG_T(2, 5) DG_T(2, 6) DG_T(2, 7) DG_T(2, 8)
    DG_T(3, 1) DG_T(3, 2) DG_T(3, 3) DG_T(3, 4) DG_T(3, 5) DG_T(3, 6) DG_T(3, 7) DG_T(3, 8)
#undef DG_T
    default: return (int)cudaErrorInvalidValue;
  }
}

int launch_passive(int dim, int order, const StageArgs& sa, const double* c_n, const double* c_in, double* c_out,
                   void* stream) {
  if (sa.n_elem <= 0) return cudaSuccess;
  PassiveArgs a{sa, c_in, c_n, c_out};
  cudaStream_t s = (cudaStream_t)stream;
  switch (dim * 16 + order) {
#define DG_T(D_, N_) \
  case D_ * 16 + N_: return launch_passive_t<D_, N_>(a, s);
    DG_T(2, 1) DG_T(2, 2) DG_T(2, 3) DG_T(2, 4) DG_T(2, 5) DG_T(2, 6) DG_T(2, 7) DG_T(2, 8)
    DG_T(3, 1) DG_T(3, 2) DG_T(3, 3) DG_T(3, 4) DG_T(3, 5) DG_T(3, 6) DG_T(3, 7) DG_T(3, 8)
#undef DG_T
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace dgi
