// dg_kernels.cu -- sm_100a kernels of libdg: the fused dGSEM RHS / SSP-RK3
// stage, the conservative refine/coarsen projections, element copy and the
// per-element quadrature sums.
//
// Method (PAPER.md:116-133 strong-form dGSEM; PAPER.md:126-131 Rusanov;
// PAPER.md:281-310 mortars; PAPER.md:279,313 transfer).  Design notes in
// DESIGN.md section 5.  One CTA owns EPB whole elements; every element
// computes the fluxes of all its own faces (neighbour traces are gathered from
// L2), so no face buffer or atomics are needed.  The point flux and the
// Rusanov flux use explicit round-to-nearest intrinsics so both elements of a
// face (and both sides of a mortar) produce bitwise equal-and-opposite fluxes.
#include <cuda_runtime.h>

#include <cstdint>

#include "dg_internal.h"

namespace dgi {
namespace {

template <int DIM, int N>
struct Cfg {
  static constexpr int n1 = N + 1;
  static constexpr int Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  static constexpr int Nf = Np / n1;
  static constexpr int F = DIM + 2;
  static constexpr int NSUB = 1 << (DIM - 1);
  static constexpr int T = 256;
  static constexpr int EPB = (T / Np) > 0 ? (T / Np) : 1;
  static constexpr int VOLF = DIM * F * Np;
  static constexpr int STG = 2 * F * Nf;
  static constexpr int MORT = 2 * NSUB * F * Nf;
  static constexpr int UNI = VOLF > (STG + MORT) ? VOLF : (STG + MORT);
  static constexpr int OPS = 5 * n1 * n1 + n1;
  static constexpr int SMEM_DOUBLES = OPS + EPB * (2 * F * Np + UNI);
};

// Point state: perturbation variables + background at that point (R13).
struct St {
  double rp, U[3], Tp;
  double rb, Tb, Pb;
};

struct Derived {
  double rho, Th, Pp, rinv;
};

// EOS in perturbation form, reading R2: P' = Pbar expm1(gamma log1p(Theta'/Thetabar)).
__device__ __forceinline__ Derived derive(const St& s, double gamma) {
  Derived o;
  o.rho = __dadd_rn(s.rb, s.rp);
  o.Th = __dadd_rn(s.Tb, s.Tp);
  o.Pp = __dmul_rn(s.Pb, expm1(__dmul_rn(gamma, log1p(__ddiv_rn(s.Tp, s.Tb)))));
  o.rinv = __drcp_rn(o.rho);
  return o;
}

// Flux along axis d (R5): F^d = (U_d, U_j u_d + delta_jd P', Theta u_d).
template <int DIM>
__device__ __forceinline__ double flux_d(const St& s, const Derived& v, int d, double* Fd) {
  const double ud = __dmul_rn(s.U[d], v.rinv);
  Fd[0] = s.U[d];
#pragma unroll
  for (int j = 0; j < DIM; ++j) Fd[1 + j] = __fma_rn(s.U[j], ud, j == d ? v.Pp : 0.0);
  Fd[DIM + 1] = __dmul_rn(v.Th, ud);
  return ud;
}

// |u.n| + a, a = sqrt(gamma P / rho) with the full pressure (R6).
__device__ __forceinline__ double wave(double ud, const St& s, const Derived& v, double gamma) {
  const double P = __dadd_rn(s.Pb, v.Pp);
  return __dadd_rn(fabs(ud), __dsqrt_rn(__dmul_rn(__dmul_rn(gamma, P), v.rinv)));
}

// Rusanov F*.n, n = sgn e_d (R6, R7), jump on (rho', U, Theta').
// Swapping (L,R) and negating sgn negates the result bitwise.
template <int DIM>
__device__ __forceinline__ void rusanov(const St& L, const St& R, int d, double sgn, double gamma, double* out) {
  constexpr int F = DIM + 2;
  double FL[F], FR[F];
  const Derived vl = derive(L, gamma), vr = derive(R, gamma);
  const double ul = flux_d<DIM>(L, vl, d, FL);
  const double ur = flux_d<DIM>(R, vr, d, FR);
  const double lam = fmax(wave(ul, L, vl, gamma), wave(ur, R, vr, gamma));
  const double hl = __dmul_rn(0.5, lam), hs = __dmul_rn(0.5, sgn);
  double jl[F], jr[F];
  jl[0] = L.rp;
  jr[0] = R.rp;
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    jl[1 + j] = L.U[j];
    jr[1 + j] = R.U[j];
  }
  jl[DIM + 1] = L.Tp;
  jr[DIM + 1] = R.Tp;
#pragma unroll
  for (int f = 0; f < F; ++f) out[f] = __fma_rn(hl, __dsub_rn(jl[f], jr[f]), __dmul_rn(hs, __dadd_rn(FL[f], FR[f])));
}

template <int DIM, int N>
__device__ __forceinline__ int vert_index(int n) {
  constexpr int n1 = N + 1;
  return DIM == 2 ? n / n1 : n / (n1 * n1);
}

// Volume node of face node t of local face f (tangential axes ascending, first fastest; R28).
template <int DIM, int N>
__device__ __forceinline__ int face_node(int f, int t) {
  constexpr int n1 = N + 1;
  const int d = f >> 1;
  const int e = (f & 1) ? N : 0;
  if (DIM == 2) return d == 0 ? e + n1 * t : t + n1 * e;
  const int t1 = t % n1, t2 = t / n1;
  if (d == 0) return e + n1 * t1 + n1 * n1 * t2;
  if (d == 1) return t1 + n1 * e + n1 * n1 * t2;
  return t1 + n1 * t2 + n1 * n1 * e;
}

template <int DIM, int N>
__device__ __forceinline__ St load_state(const double* q, int n, const double* bgrow) {
  constexpr int Np = Cfg<DIM, N>::Np;
  St s;
  s.rb = __ldg(bgrow + 0);
  s.Tb = __ldg(bgrow + 1);
  s.Pb = __ldg(bgrow + 2);
  s.rp = __dsub_rn(q[n], s.rb);
#pragma unroll
  for (int j = 0; j < 3; ++j) s.U[j] = j < DIM ? q[(1 + j) * Np + n] : 0.0;
  s.Tp = __dsub_rn(q[(DIM + 1) * Np + n], s.Tb);
  return s;
}

template <int DIM, int N>
__device__ __forceinline__ St load_state_global(const double* __restrict__ q, int n, const double* bgrow) {
  constexpr int Np = Cfg<DIM, N>::Np;
  St s;
  s.rb = __ldg(bgrow + 0);
  s.Tb = __ldg(bgrow + 1);
  s.Pb = __ldg(bgrow + 2);
  s.rp = __dsub_rn(__ldg(q + n), s.rb);
#pragma unroll
  for (int j = 0; j < 3; ++j) s.U[j] = j < DIM ? __ldg(q + (1 + j) * Np + n) : 0.0;
  s.Tp = __dsub_rn(__ldg(q + (DIM + 1) * Np + n), s.Tb);
  return s;
}

// Face -> mortar projection of a staged coarse trace (perturbation vector),
// tensor product of the 1D P_b (R12, R13).  Used by BOTH
// sides of a 2:1 face so their mortar states are bitwise identical.
template <int DIM, int N>
__device__ __forceinline__ void project(const double* stage, const double* sP, int b, int t, double* qm) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Nf = C::Nf, F = C::F;
  const int t1 = t % n1, t2 = t / n1;
  const double* P1 = sP + (b & 1) * n1 * n1 + t1 * n1;
  const double* P2 = sP + ((b >> 1) & 1) * n1 * n1 + t2 * n1;
#pragma unroll
  for (int f = 0; f < F; ++f) qm[f] = 0.0;
  for (int j = 0; j < Nf; ++j) {
    const int j1 = j % n1, j2 = j / n1;
    const double c = DIM == 2 ? P1[j1] : __dmul_rn(P1[j1], P2[j2]);
#pragma unroll
    for (int f = 0; f < F; ++f) qm[f] = __fma_rn(c, stage[f * Nf + j], qm[f]);
  }
}

template <int DIM, int N>
__global__ void __launch_bounds__(256) k_stage(const StageArgs a) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NSUB = C::NSUB, T = C::T, EPB = C::EPB;
  extern __shared__ double smem[];
  double* sD = smem;
  double* sP = sD + n1 * n1;
  double* sR = sP + 2 * n1 * n1;
  double* sQ = smem + C::OPS;
  double* sRes = sQ + EPB * F * Np;
  double* sU = sRes + EPB * F * Np;
  __shared__ ElemDesc sDesc[EPB];
  __shared__ double sH[kMaxLevel + 1][3];

  const int tid = threadIdx.x;
  if (tid < (kMaxLevel + 1) * 3) (&sH[0][0])[tid] = a.ops[OpsLayout::H(n1) + tid];
  const int64_t e0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)min((int64_t)EPB, a.n_elem - e0);
  for (int i = tid; i < 5 * n1 * n1; i += T) smem[i] = a.ops[i];
  for (int i = tid; i < ne * 8; i += T) reinterpret_cast<int*>(sDesc)[i] = reinterpret_cast<const int*>(a.desc + e0)[i];
  for (int i = tid; i < ne * F * Np; i += T) {
    const int el = i / (F * Np), r = i - el * (F * Np);
    sQ[i] = __ldg(a.q_in + (e0 + el) * a.stride + r);
  }
  __syncthreads();

  // A1-A2, A4: point fluxes at every node, source initialises the residual
  for (int i = tid; i < ne * Np; i += T) {
    const int el = i / Np, n = i - el * Np;
    const double* q = sQ + el * F * Np;
    const St s = load_state<DIM, N>(q, n, a.bg + 3 * (sDesc[el].bgrow + vert_index<DIM, N>(n)));
    const Derived v = derive(s, a.gamma);
    double* fl = sU + el * C::UNI;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double Fd[F];
      flux_d<DIM>(s, v, d, Fd);
#pragma unroll
      for (int f = 0; f < F; ++f) fl[(d * F + f) * Np + n] = Fd[f];
    }
    double* r = sRes + el * F * Np;
#pragma unroll
    for (int f = 0; f < F; ++f) r[f * Np + n] = (f == DIM) ? -__dmul_rn(s.rp, a.g) : 0.0;
  }
  __syncthreads();

  // A3: volume flux divergence  -sum_d (2/h_d) sum_m D[i_d][m] F^d(.., m, ..)
  for (int i = tid; i < ne * Np; i += T) {
    const int el = i / Np, n = i - el * Np;
    const int lev = elem_level(sDesc[el].info);
    const double* fl = sU + el * C::UNI;
    double* r = sRes + el * F * Np;
    int idx[3] = {n % n1, (n / n1) % n1, n / (n1 * n1)};
#pragma unroll
    for (int f = 0; f < F; ++f) {
      double acc = r[f * Np + n];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const int st = d == 0 ? 1 : (d == 1 ? n1 : n1 * n1);
        const double* line = fl + (d * F + f) * Np + n - idx[d] * st;
        const double* Drow = sD + idx[d] * n1;
        double sum = 0.0;
#pragma unroll
        for (int m = 0; m < n1; ++m) sum = __fma_rn(Drow[m], line[m * st], sum);
        acc = __fma_rn(-sH[lev][d], sum, acc);
      }
      r[f * Np + n] = acc;
    }
  }
  __syncthreads();

  // A5-A8: faces, one axis at a time (the -d and +d faces of an element have
  // disjoint nodes, so each node gets one lift per pass, deterministically).
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    // stage coarse traces (perturbation vectors) for both sides of 2:1 faces
    for (int i = tid; i < ne * 2 * F * Nf; i += T) {
      const int el = i / (2 * F * Nf);
      int r = i - el * (2 * F * Nf);
      const int s = r / (F * Nf);
      r -= s * (F * Nf);
      const int f = r / Nf, t = r - f * Nf;
      const int face = 2 * d + s;
      const ElemDesc& D = sDesc[el];
      const int kind = face_kind(D.info, face);
      double* stg = sU + el * C::UNI + s * F * Nf;
      if (kind == kCoarse) {
        const int n = face_node<DIM, N>(face, t);
        double v = sQ[el * F * Np + f * Np + n];
        if (f == 0 || f == DIM + 1)
          v = __dsub_rn(v, __ldg(a.bg + 3 * (D.bgrow + vert_index<DIM, N>(n)) + (f == 0 ? 0 : 1)));
        stg[f * Nf + t] = v;
      } else if (kind == kFine) {
        const int ec = D.nbr[face];
        const int n = face_node<DIM, N>(face ^ 1, t);
        double v = __ldg(a.q_in + (int64_t)ec * a.stride + f * Np + n);
        if (f == 0 || f == DIM + 1)
          v = __dsub_rn(v, __ldg(a.bg + 3 * (__ldg(&a.desc[ec].bgrow) + vert_index<DIM, N>(n)) + (f == 0 ? 0 : 1)));
        stg[f * Nf + t] = v;
      }
    }
    __syncthreads();
    for (int i = tid; i < ne * 2 * NSUB * Nf; i += T) {
      const int el = i / (2 * NSUB * Nf);
      int r = i - el * (2 * NSUB * Nf);
      const int s = r / (NSUB * Nf);
      r -= s * (NSUB * Nf);
      const int b = r / Nf, t = r - b * Nf;
      const int face = 2 * d + s;
      const ElemDesc& D = sDesc[el];
      const int kind = face_kind(D.info, face);
      if (kind != kCoarse && b > 0) continue;
      const double sgn = s ? 1.0 : -1.0;
      const double* q = sQ + el * F * Np;
      const int n = face_node<DIM, N>(face, t);
      const double* bgown = a.bg + 3 * (D.bgrow + vert_index<DIM, N>(n));
      double Fs[F];
      St own;
      if (kind == kCoarse) {
        const int ef = __ldg(a.mort + D.nbr[face] * NSUB + b);
        const int nf = face_node<DIM, N>(face ^ 1, t);
        const double* bgf = a.bg + 3 * (__ldg(&a.desc[ef].bgrow) + vert_index<DIM, N>(nf));
        const St R = load_state_global<DIM, N>(a.q_in + (int64_t)ef * a.stride, nf, bgf);
        double qm[F];
        project<DIM, N>(sU + el * C::UNI + s * F * Nf, sP, b, t, qm);
        St Lm;
        Lm.rb = R.rb;
        Lm.Tb = R.Tb;
        Lm.Pb = R.Pb;
        Lm.rp = qm[0];
#pragma unroll
        for (int j = 0; j < 3; ++j) Lm.U[j] = j < DIM ? qm[1 + j] : 0.0;
        Lm.Tp = qm[DIM + 1];
        rusanov<DIM>(Lm, R, d, sgn, a.gamma, Fs);
        double* mort = sU + el * C::UNI + C::STG + ((s * NSUB + b) * F) * Nf;
#pragma unroll
        for (int f = 0; f < F; ++f) mort[f * Nf + t] = Fs[f];
        continue;
      }
      own = load_state<DIM, N>(q, n, bgown);
      if (kind == kConf) {
        const int en = D.nbr[face];
        const int nn = face_node<DIM, N>(face ^ 1, t);
        const double* bgn = a.bg + 3 * (__ldg(&a.desc[en].bgrow) + vert_index<DIM, N>(nn));
        const St R = load_state_global<DIM, N>(a.q_in + (int64_t)en * a.stride, nn, bgn);
        rusanov<DIM>(own, R, d, sgn, a.gamma, Fs);
      } else if (kind == kWall) {
        St R = own;  // mirror ghost (R9)
        R.U[d] = -own.U[d];
        rusanov<DIM>(own, R, d, sgn, a.gamma, Fs);
      } else {  // fine side of a 2:1 face: the coarse side's mortar flux, negated
        double qm[F];
        project<DIM, N>(sU + el * C::UNI + s * F * Nf, sP, face_sub(D.info, face), t, qm);
        St Lm;
        Lm.rb = own.rb;
        Lm.Tb = own.Tb;
        Lm.Pb = own.Pb;
        Lm.rp = qm[0];
#pragma unroll
        for (int j = 0; j < 3; ++j) Lm.U[j] = j < DIM ? qm[1 + j] : 0.0;
        Lm.Tp = qm[DIM + 1];
        double Fb[F];
        rusanov<DIM>(Lm, own, d, -sgn, a.gamma, Fb);
#pragma unroll
        for (int f = 0; f < F; ++f) Fs[f] = -Fb[f];
      }
      // lift (strong form): RHS += -(2/h)/w0 (F*.n - F(q-).n)
      const Derived v = derive(own, a.gamma);
      double Fo[F];
      flux_d<DIM>(own, v, d, Fo);
      const double c = -sH[elem_level(D.info)][d] * a.w0inv;
      double* res = sRes + el * F * Np;
#pragma unroll
      for (int f = 0; f < F; ++f) res[f * Np + n] = __fma_rn(c, __fma_rn(-sgn, Fo[f], Fs[f]), res[f * Np + n]);
    }
    __syncthreads();
    // coarse side: back projection sum_b (kron R_b) F*_b, s = 1/2 per axis, then lift
    for (int i = tid; i < ne * 2 * Nf; i += T) {
      const int el = i / (2 * Nf);
      int r = i - el * (2 * Nf);
      const int s = r / Nf, j = r - s * Nf;
      const int face = 2 * d + s;
      const ElemDesc& D = sDesc[el];
      if (face_kind(D.info, face) != kCoarse) continue;
      const double sgn = s ? 1.0 : -1.0;
      const int j1 = j % n1, j2 = j / n1;
      double Fc[F];
#pragma unroll
      for (int f = 0; f < F; ++f) Fc[f] = 0.0;
      for (int b = 0; b < NSUB; ++b) {
        const double* R1 = sR + (b & 1) * n1 * n1 + j1 * n1;
        const double* R2 = sR + ((b >> 1) & 1) * n1 * n1 + j2 * n1;
        const double* mort = sU + el * C::UNI + C::STG + ((s * NSUB + b) * F) * Nf;
        for (int k = 0; k < Nf; ++k) {
          const int k1 = k % n1, k2 = k / n1;
          const double c = DIM == 2 ? R1[k1] : __dmul_rn(R1[k1], R2[k2]);
#pragma unroll
          for (int f = 0; f < F; ++f) Fc[f] = __fma_rn(c, mort[f * Nf + k], Fc[f]);
        }
      }
      const int n = face_node<DIM, N>(face, j);
      const St own = load_state<DIM, N>(sQ + el * F * Np, n, a.bg + 3 * (D.bgrow + vert_index<DIM, N>(n)));
      const Derived v = derive(own, a.gamma);
      double Fo[F];
      flux_d<DIM>(own, v, d, Fo);
      const double c = -sH[elem_level(D.info)][d] * a.w0inv;
      double* res = sRes + el * F * Np;
#pragma unroll
      for (int f = 0; f < F; ++f) res[f * Np + n] = __fma_rn(c, __fma_rn(-sgn, Fo[f], Fc[f]), res[f * Np + n]);
    }
    __syncthreads();
  }

  // A9: epilogue (RHS or fused SSP-RK3 stage, R17)
  for (int i = tid; i < ne * F * Np; i += T) {
    const int el = i / (F * Np), r = i - el * (F * Np);
    const int64_t gi = (e0 + el) * a.stride + r;
    const double res = sRes[i];
    double o;
    if (a.mode == 0) o = res;
    else if (a.stage == 0) o = __fma_rn(a.dt, res, sQ[i]);
    else {
      const double qn = __ldg(a.q_n + gi);
      o = __fma_rn(a.rk_b, __fma_rn(a.dt, res, __dsub_rn(sQ[i], qn)), qn);
    }
    a.out[gi] = o;
  }
}

// ---------------------------------------------------------------- transfer
// Apply a 1D operator A (n1 x n1, row-major) along axis `ax` of src into dst
// for all F fields (sum-factorised tensor product).
template <int DIM, int N>
__device__ void apply_axis(const double* A, const double* src, double* dst, int ax) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F;
  const int st = ax == 0 ? 1 : (ax == 1 ? n1 : n1 * n1);
  for (int i = threadIdx.x; i < F * Np; i += blockDim.x) {
    const int f = i / Np, n = i - f * Np;
    const int id = (n / st) % n1;
    const double* line = src + f * Np + n - id * st;
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < n1; ++m) s = __fma_rn(A[id * n1 + m], line[m * st], s);
    dst[i] = s;
  }
}

template <int DIM, int N>
__global__ void __launch_bounds__(256) k_refine(const TransferArgs a) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F;
  extern __shared__ double smem[];
  double* sP = smem;                 // P_lo, P_hi
  double* sPar = smem + 2 * n1 * n1;
  double* t1 = sPar + F * Np;
  double* t2 = t1 + F * Np;
  const int64_t fam = blockIdx.x;
  for (int i = threadIdx.x; i < 2 * n1 * n1; i += blockDim.x) sP[i] = a.ops[n1 * n1 + i];
  const int64_t src = __ldg(a.src_idx + fam), dst0 = __ldg(a.dst_idx + fam);
  for (int i = threadIdx.x; i < F * Np; i += blockDim.x) sPar[i] = __ldg(a.q_src + src * a.stride + i);
  __syncthreads();
  for (int b = 0; b < (1 << DIM); ++b) {
    apply_axis<DIM, N>(sP + (b & 1) * n1 * n1, sPar, t1, 0);
    __syncthreads();
    apply_axis<DIM, N>(sP + ((b >> 1) & 1) * n1 * n1, t1, t2, 1);
    __syncthreads();
    const double* res = t2;
    if (DIM == 3) {
      apply_axis<DIM, N>(sP + ((b >> 2) & 1) * n1 * n1, t2, t1, 2);
      __syncthreads();
      res = t1;
    }
    double* out = a.q_dst + (dst0 + b) * a.stride;
    for (int i = threadIdx.x; i < F * Np; i += blockDim.x) out[i] = res[i];
    __syncthreads();
  }
}

template <int DIM, int N>
__global__ void __launch_bounds__(256) k_coarsen(const TransferArgs a) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F;
  extern __shared__ double smem[];
  double* sRo = smem;                // R_lo, R_hi
  double* sCh = smem + 2 * n1 * n1;
  double* t1 = sCh + F * Np;
  double* t2 = t1 + F * Np;
  double* acc = t2 + F * Np;
  const int64_t fam = blockIdx.x;
  for (int i = threadIdx.x; i < 2 * n1 * n1; i += blockDim.x) sRo[i] = a.ops[3 * n1 * n1 + i];
  for (int i = threadIdx.x; i < F * Np; i += blockDim.x) acc[i] = 0.0;
  const int64_t src0 = __ldg(a.src_idx + fam), dst = __ldg(a.dst_idx + fam);
  for (int b = 0; b < (1 << DIM); ++b) {
    __syncthreads();
    for (int i = threadIdx.x; i < F * Np; i += blockDim.x) sCh[i] = __ldg(a.q_src + (src0 + b) * a.stride + i);
    __syncthreads();
    apply_axis<DIM, N>(sRo + (b & 1) * n1 * n1, sCh, t1, 0);
    __syncthreads();
    apply_axis<DIM, N>(sRo + ((b >> 1) & 1) * n1 * n1, t1, t2, 1);
    __syncthreads();
    const double* res = t2;
    if (DIM == 3) {
      apply_axis<DIM, N>(sRo + ((b >> 2) & 1) * n1 * n1, t2, t1, 2);
      __syncthreads();
      res = t1;
    }
    for (int i = threadIdx.x; i < F * Np; i += blockDim.x) acc[i] = __dadd_rn(acc[i], res[i]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < F * Np; i += blockDim.x) a.q_dst[dst * a.stride + i] = acc[i];
}

__global__ void k_copy(const TransferArgs a, int row) {
  const int64_t fam = blockIdx.x;
  const int64_t s = __ldg(a.src_idx + fam), d = __ldg(a.dst_idx + fam);
  for (int i = threadIdx.x; i < row; i += blockDim.x) a.q_dst[d * a.stride + i] = __ldg(a.q_src + s * a.stride + i);
}

template <int DIM, int N>
__global__ void __launch_bounds__(128) k_integrals(const double* __restrict__ q, int64_t n_elem, int64_t stride,
                                                   const ElemDesc* __restrict__ desc, const double* __restrict__ ops,
                                                   const double* __restrict__ jac, double* __restrict__ partial) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F;
  __shared__ double red[F][4];
  const int64_t e = blockIdx.x;
  const double* w = ops + 5 * n1 * n1;
  double acc[F];
#pragma unroll
  for (int f = 0; f < F; ++f) acc[f] = 0.0;
  for (int n = threadIdx.x; n < Np; n += blockDim.x) {
    double wn = __ldg(w + n % n1) * __ldg(w + (n / n1) % n1);
    if (DIM == 3) wn *= __ldg(w + n / (n1 * n1));
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = __fma_rn(wn, __ldg(q + e * stride + f * Np + n), acc[f]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < F; ++f) {
    double v = acc[f];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[f][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < F) {
    const double J = __ldg(jac + elem_level(__ldg(&desc[e].info)));
    const double s = (red[threadIdx.x][0] + red[threadIdx.x][1]) + (red[threadIdx.x][2] + red[threadIdx.x][3]);
    partial[e * F + threadIdx.x] = J * s;
  }
}

// ---------------------------------------------------------------- dispatch
template <int DIM, int N>
int launch_stage_t(const StageArgs& a, cudaStream_t s) {
  using C = Cfg<DIM, N>;
  const size_t bytes = sizeof(double) * C::SMEM_DOUBLES;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_stage<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int64_t grid = (a.n_elem + C::EPB - 1) / C::EPB;
  k_stage<DIM, N><<<(unsigned)grid, C::T, bytes, s>>>(a);
  return cudaGetLastError();
}

template <int DIM, int N>
int launch_transfer_t(int which, const TransferArgs& a, cudaStream_t s) {
  using C = Cfg<DIM, N>;
  if (which == 2) {
    k_copy<<<(unsigned)a.n, 256, 0, s>>>(a, C::F * C::Np);
    return cudaGetLastError();
  }
  const size_t bytes = sizeof(double) * (2 * C::n1 * C::n1 + 4 * C::F * C::Np);
  static bool configured[2] = {false, false};
  if (!configured[which]) {
    cudaError_t e = which == 0
                        ? cudaFuncSetAttribute(k_refine<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)
                        : cudaFuncSetAttribute(k_coarsen<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured[which] = true;
  }
  if (which == 0) k_refine<DIM, N><<<(unsigned)a.n, 256, bytes, s>>>(a);
  else k_coarsen<DIM, N><<<(unsigned)a.n, 256, bytes, s>>>(a);
  return cudaGetLastError();
}

template <int DIM, int N>
int launch_integrals_t(const double* q, int64_t n_elem, int64_t stride, const ElemDesc* desc, const double* ops,
                       const double* jac, double* partial, cudaStream_t s) {
  k_integrals<DIM, N><<<(unsigned)n_elem, 128, 0, s>>>(q, n_elem, stride, desc, ops, jac, partial);
  return cudaGetLastError();
}

#define DG_DISPATCH(dim, order, CALL)                                          \
  switch ((dim) * 16 + (order)) {                                              \
    case 2 * 16 + 1: { constexpr int D_ = 2, N_ = 1; return CALL; }            \
    case 2 * 16 + 2: { constexpr int D_ = 2, N_ = 2; return CALL; }            \
    case 2 * 16 + 3: { constexpr int D_ = 2, N_ = 3; return CALL; }            \
    case 2 * 16 + 4: { constexpr int D_ = 2, N_ = 4; return CALL; }            \
    case 2 * 16 + 5: { constexpr int D_ = 2, N_ = 5; return CALL; }            \
    case 2 * 16 + 6: { constexpr int D_ = 2, N_ = 6; return CALL; }            \
    case 2 * 16 + 7: { constexpr int D_ = 2, N_ = 7; return CALL; }            \
    case 2 * 16 + 8: { constexpr int D_ = 2, N_ = 8; return CALL; }            \
    case 3 * 16 + 1: { constexpr int D_ = 3, N_ = 1; return CALL; }            \
    case 3 * 16 + 2: { constexpr int D_ = 3, N_ = 2; return CALL; }            \
    case 3 * 16 + 3: { constexpr int D_ = 3, N_ = 3; return CALL; }            \
    case 3 * 16 + 4: { constexpr int D_ = 3, N_ = 4; return CALL; }            \
    case 3 * 16 + 5: { constexpr int D_ = 3, N_ = 5; return CALL; }            \
    case 3 * 16 + 6: { constexpr int D_ = 3, N_ = 6; return CALL; }            \
    case 3 * 16 + 7: { constexpr int D_ = 3, N_ = 7; return CALL; }            \
    case 3 * 16 + 8: { constexpr int D_ = 3, N_ = 8; return CALL; }            \
    default: return (int)cudaErrorInvalidValue;                                \
  }

}  // namespace

bool supported(int dim, int order) { return (dim == 2 || dim == 3) && order >= 1 && order <= kMaxOrder; }

int launch_stage(int dim, int order, const StageArgs& a, void* stream) {
  DG_DISPATCH(dim, order, (launch_stage_t<D_, N_>(a, (cudaStream_t)stream)));
}
int launch_refine(int dim, int order, const TransferArgs& a, void* stream) {
  DG_DISPATCH(dim, order, (launch_transfer_t<D_, N_>(0, a, (cudaStream_t)stream)));
}
int launch_coarsen(int dim, int order, const TransferArgs& a, void* stream) {
  DG_DISPATCH(dim, order, (launch_transfer_t<D_, N_>(1, a, (cudaStream_t)stream)));
}
int launch_copy(int dim, int order, const TransferArgs& a, void* stream) {
  DG_DISPATCH(dim, order, (launch_transfer_t<D_, N_>(2, a, (cudaStream_t)stream)));
}
int launch_elem_integrals(int dim, int order, const double* q, int64_t n_elem, int64_t stride, const ElemDesc* desc,
                          const double* ops, const double* jac, double* partial, void* stream) {
  DG_DISPATCH(dim, order, (launch_integrals_t<D_, N_>(q, n_elem, stride, desc, ops, jac, partial, (cudaStream_t)stream)));
}

}  // namespace dgi
