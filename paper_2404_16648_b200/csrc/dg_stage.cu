// dg_stage.cu -- the fused dGSEM right-hand side / SSP-RK3 stage kernel for
// sm_100a (rows A1-A9 of SURVEY 8(a)).
//
// Method: strong-form dGSEM, Rusanov flux,
// mortars at 2:1 faces, gravity source.
// Readings R2-R17 of DESIGN.md section 3.  Design: DESIGN.md section 6.
//
// Structure (one persistent CTA loops over tiles of EPB consecutive elements):
//   prefetch   the next tile's state rows by one cp.async.bulk (mbarrier),
//              its face-neighbour traces by cp.async (after this tile's face
//              phase), its q_n rows into L2 (RK stages 1, 2)
//   mortars    coarse side of 2:1 faces: Rusanov on the 2^(d-1) mortars of
//              each coarse face (fine traces gathered from L2), then the
//              back projection into the face-lift buffer (only tiles that
//              own coarse faces)
//   nodes      EOS in perturbation form, u, P', 1/rho to smem; F^x to a
//              bank-conflict-free padded buffer
//   faces      Rusanov + lift value for every face node (conforming, wall
//              mirror, fine side of a mortar)
//   passes     one per axis: thread = (element, field, pencil along the
//              axis); sum-factorised D contraction in registers with the
//              even-odd (centro-antisymmetric) split of D taken from the
//              kernel-parameter constant bank, endpoint lifts added; the
//              last pass adds the source and runs the RK epilogue and stores.
// Both elements of a face compute bitwise equal-and-opposite fluxes (explicit
// round-to-nearest intrinsics, identical operand order), so there is no face
// buffer and no atomics; every element writes only its own nodes.
#include <cuda_runtime.h>

#include <cstdint>

#include "dg_internal.h"

namespace dgi {
namespace {

template <int DIM, int N>
struct SC {
  static constexpr int n1 = N + 1;
  static constexpr int Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  static constexpr int Nf = Np / n1;
  static constexpr int F = DIM + 2;
  static constexpr int NSUB = 1 << (DIM - 1);
  static constexpr int NFACE = 2 * DIM;
  static constexpr int T = 256;
  static constexpr int EPB = (T / Np) > 0 ? (T / Np) : 1;
  static constexpr int STR = (F * Np + 15) / 16 * 16;   // element row stride (doubles), = dg_ctx stride
  static constexpr int NPAD = (n1 & 1) ? n1 : n1 + 1;   // x-pencil stride in the padded F^x / residual buffer
  static constexpr int NPP = Nf * NPAD;
  static constexpr int NAUX = DIM + 1;                  // u_1..u_{DIM-1}, P', 1/rho
  static constexpr int Q = EPB * STR;
  static constexpr int FR = EPB * F * NPP;
  static constexpr int AUX = EPB * NAUX * Np;
  static constexpr int TR = EPB * NFACE * F * Nf;
  static constexpr int SMEM = 2 * Q + FR + AUX + 2 * TR;  // doubles
  static constexpr int MORT1 = NSUB * F * Nf;             // mortar flux scratch per coarse face
  static constexpr int CAP = FR / MORT1;                  // coarse faces per mortar chunk
  static_assert(CAP >= 1, "mortar scratch too small");
  static_assert(SMEM * 8 <= 227 * 1024, "shared memory budget");
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ------------------------------------------------------------------ point physics
// Point state in perturbation form with its background (R13).
struct St {
  double rp, U[3], Tp;
  double rb, Tb, Pb, rTb;  // rho_bar, Theta_bar, P_bar, 1/Theta_bar
};
struct Dv {
  double rho, Th, Pp, rinv;
};

// (1+x)^gamma - 1 (reading R2: P' = P_bar ((1 + Theta'/Theta_bar)^gamma - 1)).  For
// |x| < 2^-5 the binomial series (coefficients from the host, long double) in
// Estrin form (dependency depth 5 instead of 12), else expm1(gamma log1p(x));
// exactly 0 at x = 0.
__device__ __forceinline__ double pow1pm1(double x, const StageArgs& a) {
  static_assert(kEosTerms == 12, "Estrin layout below assumes 12 terms");
  if (fabs(x) < 0.03125) {
    const double* c = a.eos_c;
    const double x2 = __dmul_rn(x, x), x4 = __dmul_rn(x2, x2), x8 = __dmul_rn(x4, x4);
    const double p0 = __fma_rn(c[1], x, c[0]), p1 = __fma_rn(c[3], x, c[2]), p2 = __fma_rn(c[5], x, c[4]);
    const double p3 = __fma_rn(c[7], x, c[6]), p4 = __fma_rn(c[9], x, c[8]), p5 = __fma_rn(c[11], x, c[10]);
    const double q0 = __fma_rn(p1, x2, p0), q1 = __fma_rn(p3, x2, p2), q2 = __fma_rn(p5, x2, p4);
    return __dmul_rn(__fma_rn(q2, x8, __fma_rn(q1, x4, q0)), x);
  }
  return expm1(__dmul_rn(a.gamma, log1p(x)));
}

__device__ __forceinline__ Dv derive(const St& s, const StageArgs& a) {
  Dv o;
  o.rho = __dadd_rn(s.rb, s.rp);
  o.Th = __dadd_rn(s.Tb, s.Tp);
  o.Pp = __dmul_rn(s.Pb, pow1pm1(__dmul_rn(s.Tp, s.rTb), a));
  o.rinv = __drcp_rn(o.rho);
  return o;
}

// U[d] for a runtime axis d without dynamic register-array indexing.
__device__ __forceinline__ double pick(const double* U, int d) { return d == 0 ? U[0] : (d == 1 ? U[1] : U[2]); }

// F^d (R5) and u_d.
template <int DIM>
__device__ __forceinline__ double flux_d(const St& s, const Dv& v, int d, double* Fd) {
  const double Ud = pick(s.U, d);
  const double ud = __dmul_rn(Ud, v.rinv);
  Fd[0] = Ud;
#pragma unroll
  for (int j = 0; j < DIM; ++j) Fd[1 + j] = __fma_rn(s.U[j], ud, j == d ? v.Pp : 0.0);
  Fd[DIM + 1] = __dmul_rn(v.Th, ud);
  return ud;
}

// |u.n| + a, a = sqrt(gamma P / rho), full pressure (R6).
__device__ __forceinline__ double wave(double ud, const St& s, const Dv& v, double gamma) {
  const double P = __dadd_rn(s.Pb, v.Pp);
  return __dadd_rn(fabs(ud), __dsqrt_rn(__dmul_rn(__dmul_rn(gamma, P), v.rinv)));
}

// Rusanov F*.n with n = sgn e_d (R6, R7); jump on (rho', U, Theta').
// Swapping (L, R) and negating sgn negates the result bitwise.  The own-side
// flux F(L) is returned in FL (for the lift).
template <int DIM>
__device__ __forceinline__ void rusanov(const St& L, const Dv& vl, const St& R, const Dv& vr, int d, double sgn,
                                        double gamma, double* out, double* FL) {
  constexpr int F = DIM + 2;
  double FR[F];
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

// First node and node stride of pencil p along axis d (p = face node index of the axis-d faces).
template <int DIM, int N>
__device__ __forceinline__ void pencil(int d, int p, int& base, int& step) {
  constexpr int n1 = N + 1;
  if (d == 0) {
    base = n1 * p;
    step = 1;
  } else if (d == 1) {
    base = DIM == 2 ? p : (p % n1) + n1 * n1 * (p / n1);
    step = n1;
  } else {
    base = p;
    step = n1 * n1;
  }
}

__device__ __forceinline__ void load_bg(St& s, const double* __restrict__ bg4, int row) {
  const double2 b0 = __ldg(reinterpret_cast<const double2*>(bg4) + 2 * row);
  const double2 b1 = __ldg(reinterpret_cast<const double2*>(bg4) + 2 * row + 1);
  s.rb = b0.x;
  s.Tb = b0.y;
  s.Pb = b1.x;
  s.rTb = b1.y;
}
// (rho_bar, Theta_bar) of a background row
__device__ __forceinline__ double2 bg_rt(const double* __restrict__ bg4, int row) {
  return __ldg(reinterpret_cast<const double2*>(bg4) + 2 * row);
}

// Face -> mortar projection (tensor product of the 1D P_b; R12) of the
// perturbation trace of a coarse face, read through `val(f, j)`.  Used by BOTH sides of
// a 2:1 face with identical arithmetic so their mortar states are bitwise equal.
template <int DIM, int N, class V>
__device__ __forceinline__ void project(const double* sP, int b, int t, const V& val, double* qm) {
  constexpr int n1 = N + 1, Nf = SC<DIM, N>::Nf, F = DIM + 2;
  const int t1 = t % n1, t2 = t / n1;
  const double* P1 = sP + (b & 1) * n1 * n1 + t1 * n1;
  const double* P2 = sP + ((b >> 1) & 1) * n1 * n1 + t2 * n1;
#pragma unroll
  for (int f = 0; f < F; ++f) qm[f] = 0.0;
  for (int j = 0; j < Nf; ++j) {
    const int j1 = j % n1, j2 = j / n1;
    const double c = DIM == 2 ? P1[j1] : __dmul_rn(P1[j1], P2[j2]);
#pragma unroll
    for (int f = 0; f < F; ++f) qm[f] = __fma_rn(c, val(f, j), qm[f]);
  }
}

// out[i] = sum_m D[i][m] F[m] by the even-odd split (D[N-i][N-m] = -D[i][m]):
// e_m = F_m + F_{N-m}, o_m = F_m - F_{N-m}; out_i = Se_i + Ao_i, out_{N-i} = Ao_i - Se_i.
// De/Do live in the kernel parameter space (constant bank operands).
template <int N>
__device__ __forceinline__ void contract(const double* Fv, double* out, const StageArgs& a) {
  constexpr int n1 = N + 1, H = n1 / 2;
  double e[H], o[H];
#pragma unroll
  for (int m = 0; m < H; ++m) {
    e[m] = __dadd_rn(Fv[m], Fv[N - m]);
    o[m] = __dsub_rn(Fv[m], Fv[N - m]);
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double se = (n1 & 1) ? __dmul_rn(a.De[i * kMaxH + H], Fv[H]) : 0.0;
    double ao = 0.0;
#pragma unroll
    for (int m = 0; m < H; ++m) {
      se = __fma_rn(a.De[i * kMaxH + m], e[m], se);
      ao = __fma_rn(a.Do[i * kMaxH + m], o[m], ao);
    }
    out[i] = __dadd_rn(ao, se);
    out[N - i] = __dsub_rn(ao, se);
  }
  if (n1 & 1) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < H; ++m) s = __fma_rn(a.Do[H * kMaxH + m], o[m], s);
    out[H] = s;
  }
}

// Pencil of axis d with index p (= face node index of the axis-d faces):
// first node, node step, and the same in the padded x-pencil layout of sFR.
template <int DIM, int N, int d>
__device__ __forceinline__ void pencil_addr(int p, int& base, int& pbase) {
  constexpr int n1 = N + 1, NPAD = SC<DIM, N>::NPAD;
  if (d == 0) {
    base = n1 * p;
    pbase = NPAD * p;
  } else if (d == 1 && DIM == 3) {  // p = i + n1 k
    const int i = p % n1, k = p / n1;
    base = i + n1 * n1 * k;
    pbase = i + NPAD * n1 * k;
  } else if (d == 1) {  // 2D, p = i
    base = p;
    pbase = p;
  } else {  // d == 2, p = i + n1 j
    const int i = p % n1, j = p / n1;
    base = p;
    pbase = i + NPAD * j;
  }
}
template <int DIM, int N, int d>
struct PStep {
  static constexpr int n1 = N + 1, NPAD = SC<DIM, N>::NPAD;
  static constexpr int node = d == 0 ? 1 : (d == 1 ? n1 : n1 * n1);
  static constexpr int pad = d == 0 ? 1 : (d == 1 ? (DIM == 3 ? NPAD : NPAD) : n1 * NPAD);
};

// number of coarse-side (kind 2 = binary 10) faces in a packed face-kind word
__device__ __forceinline__ int n_coarse_faces(int info) {
  const int hi = info & 0xAAA, lo = info & 0x555;
  return __popc(hi & ~(lo << 1));
}

// One axis pass of the volume divergence (A3) with the endpoint lifts (A8);
// the last pass adds the source (A4) and runs the RK epilogue (A9).
template <int DIM, int N, int d>
__device__ __forceinline__ void axis_pass(const StageArgs& a, const double* sQ, const double* sAux, double* sFR,
                                          const double* sLift, const ElemDesc* sD, const double (*sH)[3], int ne,
                                          int64_t e0) {
  using C = SC<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T, EPB = C::EPB,
                STR = C::STR, NPP = C::NPP, NAUX = C::NAUX;
  constexpr int ST = PStep<DIM, N, d>::node, PST = PStep<DIM, N, d>::pad;
  constexpr bool last = d == DIM - 1;
  constexpr int ROUNDS = (EPB * F * Nf + T - 1) / T;
#pragma unroll 1
  for (int rr = 0; rr < ROUNDS; ++rr) {
    const int i = threadIdx.x + rr * T;
    if (i >= ne * F * Nf) break;
    const int el = i / (F * Nf);
    const int r = i - el * (F * Nf);
    const int f = r / Nf, p = r - f * Nf;
    int base, pbase;
    pencil_addr<DIM, N, d>(p, base, pbase);
    const double* q = sQ + el * STR + base;
    const double* ax = sAux + el * NAUX * Np + base;
    double* fr = sFR + el * F * NPP + f * NPP + pbase;
    double Fv[n1], out[n1], qn_v[n1];
    if (last && a.mode == 1 && a.stage > 0) {
      const double* qn = a.q_n + (e0 + el) * STR + f * Np + base;
#pragma unroll
      for (int m = 0; m < n1; ++m) qn_v[m] = __ldg(qn + m * ST);
    }
    if (d == 0) {
#pragma unroll
      for (int m = 0; m < n1; ++m) Fv[m] = fr[m];
    } else if (f == 0) {
#pragma unroll
      for (int m = 0; m < n1; ++m) Fv[m] = q[(1 + d) * Np + m * ST];
    } else if (f == DIM + 1) {
#pragma unroll
      for (int m = 0; m < n1; ++m) Fv[m] = __dmul_rn(q[(DIM + 1) * Np + m * ST], ax[(d - 1) * Np + m * ST]);
    } else if (f == 1 + d) {
#pragma unroll
      for (int m = 0; m < n1; ++m)
        Fv[m] = __fma_rn(q[f * Np + m * ST], ax[(d - 1) * Np + m * ST], ax[(DIM - 1) * Np + m * ST]);
    } else {
#pragma unroll
      for (int m = 0; m < n1; ++m) Fv[m] = __fma_rn(q[f * Np + m * ST], ax[(d - 1) * Np + m * ST], 0.0);
    }
    contract<N>(Fv, out, a);
    const double sc = -sH[elem_level(sD[el].info)][d];
    const double* L = sLift + ((el * NFACE + 2 * d) * F + f) * Nf + p;
    out[0] = __fma_rn(sc, out[0], L[0]);
    out[N] = __fma_rn(sc, out[N], L[F * Nf]);
#pragma unroll
    for (int m = 1; m < N; ++m) out[m] = __fma_rn(sc, out[m], 0.0);
    if (d == 0) {
#pragma unroll
      for (int m = 0; m < n1; ++m) fr[m] = out[m];
    } else if (!last) {
#pragma unroll
      for (int m = 0; m < n1; ++m) fr[m * PST] = __dadd_rn(fr[m * PST], out[m]);
    } else {
      double* og = a.out + (e0 + el) * STR + f * Np + base;
      const int bgr = sD[el].bgrow;
#pragma unroll
      for (int m = 0; m < n1; ++m) {
        double res = __dadd_rn(fr[m * PST], out[m]);
        if (f == DIM) {  // gravity source -rho' g on the vertical momentum (R5); vertical = this axis
          const double rb = bg_rt(a.bg4, bgr + (base / (n1 * (DIM == 3 ? n1 : 1))) + m).x;
          res = __fma_rn(-__dsub_rn(q[m * ST], rb), a.g, res);
        }
        double o;
        if (a.mode == 0) o = res;
        else if (a.stage == 0) o = __fma_rn(a.dt, res, q[f * Np + m * ST]);
        else o = __fma_rn(a.rk_b, __fma_rn(a.dt, res, __dsub_rn(q[f * Np + m * ST], qn_v[m])), qn_v[m]);
        og[m * ST] = o;
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel
template <int DIM, int N>
__global__ void __launch_bounds__(256) k_stage2(const __grid_constant__ StageArgs a) {
  using C = SC<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NSUB = C::NSUB, NFACE = C::NFACE, T = C::T,
                EPB = C::EPB, STR = C::STR, NPAD = C::NPAD, NPP = C::NPP, NAUX = C::NAUX;
  extern __shared__ __align__(128) double smem[];
  double* sFR = smem + 2 * C::Q;
  double* sAux = sFR + C::FR;
  double* sTr = sAux + C::AUX;
  double* sLift = sTr + C::TR;
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ ElemDesc sDesc[2][EPB];
  __shared__ double sH[kMaxLevel + 1][3];
  __shared__ double sPR[4 * kMaxN1 * kMaxN1];  // P_lo, P_hi, R_lo, R_hi
  const double* sP = sPR;
  const double* sR = sPR + 2 * n1 * n1;

  const int tid = threadIdx.x;
  const int64_t n_tiles = (a.n_elem + EPB - 1) / EPB;
  int64_t tile = blockIdx.x;
  if (tile >= n_tiles) return;

  if (tid < (kMaxLevel + 1) * 3) (&sH[0][0])[tid] = a.ops[OpsLayout::H(n1) + tid];
  for (int i = tid; i < 4 * n1 * n1; i += T) sPR[i] = a.ops[OpsLayout::P(n1, 0) + i];
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto tile_n = [&](int64_t t) { return (int)min((int64_t)EPB, a.n_elem - t * EPB); };
  auto issue_q = [&](int64_t t, int buf) {  // thread 0 only
    const int ne = tile_n(t);
    const uint32_t bytes = (uint32_t)(ne * STR * 8);
    fence_proxy_async();
    mbar_expect_tx(&mbar[buf], bytes);
    bulk_g2s(smem + buf * C::Q, a.q_in + t * EPB * STR, bytes, &mbar[buf]);
    if (a.mode == 1 && a.stage > 0) prefetch_l2(a.q_n + t * EPB * STR, bytes);
  };
  auto load_desc = [&](int64_t t, int buf) {
    const int ne = tile_n(t);
    for (int i = tid; i < ne * 8; i += T)
      reinterpret_cast<int*>(sDesc[buf])[i] = __ldg(reinterpret_cast<const int*>(a.desc + t * EPB) + i);
  };
  // neighbour traces of conforming and fine-side faces: raw values of the
  // neighbour's face^1 nodes, [el][face][f][t]
  auto issue_traces = [&](int64_t t, int buf) {
    const int ne = tile_n(t);
    for (int i = tid; i < ne * NFACE * Nf; i += T) {
      const int el = i / (NFACE * Nf);
      const int r = i - el * (NFACE * Nf);
      const int face = r / Nf, tt = r - face * Nf;
      const ElemDesc& D = sDesc[buf][el];
      const int kind = face_kind(D.info, face);
      if (kind == kConf || kind == kFine) {
        const double* src = a.q_in + (int64_t)D.nbr[face] * STR + face_node<DIM, N>(face ^ 1, tt);
        double* dst = sTr + (el * NFACE + face) * F * Nf + tt;
#pragma unroll
        for (int f = 0; f < F; ++f) cp_async8(dst + f * Nf, src + f * Np);
      }
    }
    cp_async_commit();
  };

  // prologue
  if (tid == 0) issue_q(tile, 0);
  load_desc(tile, 0);
  __syncthreads();
  issue_traces(tile, 0);

  const double gam = a.gamma;
  for (int it = 0; tile < n_tiles; ++it, tile += gridDim.x) {
    const int cur = it & 1, nxt = cur ^ 1;
    const int ne = tile_n(tile);
    const int64_t e0 = tile * EPB;
    const int64_t tnext = tile + gridDim.x;
    const bool has_next = tnext < n_tiles;
    if (has_next) {
      if (tid == 0) issue_q(tnext, nxt);
      load_desc(tnext, nxt);
    }
    mbar_wait(&mbar[cur], (it >> 1) & 1);
    cp_async_wait_all();
    __syncthreads();
    const double* sQ = smem + cur * C::Q;
    const ElemDesc* sD = sDesc[cur];

    // ---------------- mortars: coarse side of 2:1 faces (R11-R14)
    int n_coarse = 0;
    for (int e = 0; e < ne; ++e) n_coarse += n_coarse_faces(sD[e].info);
    for (int c0 = 0; c0 < n_coarse; c0 += C::CAP) {
      const int nc = min(C::CAP, n_coarse - c0);
      // step 1: Rusanov on the mortar nodes -> scratch (sFR)
      for (int i = tid; i < nc * NSUB * Nf; i += T) {
        const int cs = i / (NSUB * Nf);
        int r = i - cs * (NSUB * Nf);
        const int b = r / Nf, t = r - b * Nf;
        int el = 0, face = 0;
        for (int k = 0, seen = 0; k < ne * NFACE; ++k)
          if (face_kind(sD[k / NFACE].info, k % NFACE) == kCoarse && seen++ == c0 + cs) {
            el = k / NFACE;
            face = k % NFACE;
            break;
          }
        const ElemDesc& D = sD[el];
        const int d = face >> 1;
        const double sgn = (face & 1) ? 1.0 : -1.0;
        const int ef = __ldg(a.mort + D.nbr[face] * NSUB + b);
        const int nf = face_node<DIM, N>(face ^ 1, t);
        St R;
        load_bg(R, a.bg4, __ldg(&a.desc[ef].bgrow) + vert_index<DIM, N>(nf));
        const double* qf = a.q_in + (int64_t)ef * STR;
        R.rp = __dsub_rn(__ldg(qf + nf), R.rb);
#pragma unroll
        for (int j = 0; j < 3; ++j) R.U[j] = j < DIM ? __ldg(qf + (1 + j) * Np + nf) : 0.0;
        R.Tp = __dsub_rn(__ldg(qf + (DIM + 1) * Np + nf), R.Tb);
        const double* q = sQ + el * STR;
        auto val = [&](int f, int j) {
          const int n = face_node<DIM, N>(face, j);
          double v = q[f * Np + n];
          if (f == 0 || f == DIM + 1) {
            const double2 bb = bg_rt(a.bg4, D.bgrow + vert_index<DIM, N>(n));
            v = __dsub_rn(v, f == 0 ? bb.x : bb.y);
          }
          return v;
        };
        double qm[F];
        project<DIM, N>(sP, b, t, val, qm);
        St Lm = R;  // fine-level background at the mortar node (R13)
        Lm.rp = qm[0];
#pragma unroll
        for (int j = 0; j < 3; ++j) Lm.U[j] = j < DIM ? qm[1 + j] : 0.0;
        Lm.Tp = qm[DIM + 1];
        double Fs[F], FL[F];
        rusanov<DIM>(Lm, derive(Lm, a), R, derive(R, a), d, sgn, gam, Fs, FL);
        double* mo = sFR + cs * C::MORT1 + b * F * Nf;
#pragma unroll
        for (int f = 0; f < F; ++f) mo[f * Nf + t] = Fs[f];
      }
      __syncthreads();
      // step 2: back projection sum_b (kron R_b) F*_b, s = 1/2 per axis, and the lift value
      for (int i = tid; i < nc * Nf; i += T) {
        const int cs = i / Nf, j = i - cs * Nf;
        int el = 0, face = 0;
        for (int k = 0, seen = 0; k < ne * NFACE; ++k)
          if (face_kind(sD[k / NFACE].info, k % NFACE) == kCoarse && seen++ == c0 + cs) {
            el = k / NFACE;
            face = k % NFACE;
            break;
          }
        const ElemDesc& D = sD[el];
        const int d = face >> 1;
        const double sgn = (face & 1) ? 1.0 : -1.0;
        const int j1 = j % n1, j2 = j / n1;
        double Fc[F];
#pragma unroll
        for (int f = 0; f < F; ++f) Fc[f] = 0.0;
        for (int b = 0; b < NSUB; ++b) {
          const double* R1 = sR + (b & 1) * n1 * n1 + j1 * n1;
          const double* R2 = sR + ((b >> 1) & 1) * n1 * n1 + j2 * n1;
          const double* mo = sFR + cs * C::MORT1 + b * F * Nf;
          for (int k = 0; k < Nf; ++k) {
            const int k1 = k % n1, k2 = k / n1;
            const double c = DIM == 2 ? R1[k1] : __dmul_rn(R1[k1], R2[k2]);
#pragma unroll
            for (int f = 0; f < F; ++f) Fc[f] = __fma_rn(c, mo[f * Nf + k], Fc[f]);
          }
        }
        const int n = face_node<DIM, N>(face, j);
        const double* q = sQ + el * STR;
        St own;
        load_bg(own, a.bg4, D.bgrow + vert_index<DIM, N>(n));
        own.rp = __dsub_rn(q[n], own.rb);
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) own.U[jj] = jj < DIM ? q[(1 + jj) * Np + n] : 0.0;
        own.Tp = __dsub_rn(q[(DIM + 1) * Np + n], own.Tb);
        double Fo[F];
        flux_d<DIM>(own, derive(own, a), d, Fo);
        const double cf = __dmul_rn(-sH[elem_level(D.info)][d], a.w0inv);
        double* L = sLift + ((el * NFACE + face) * F) * Nf + j;
#pragma unroll
        for (int f = 0; f < F; ++f) L[f * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[f], Fc[f]));
      }
      __syncthreads();
    }

    // ---------------- nodes: EOS (A1), u, P', 1/rho; F^x into the padded buffer (A2)
    {
      constexpr int ROUNDS = (EPB * Np + T - 1) / T;
#pragma unroll
      for (int rr = 0; rr < ROUNDS; ++rr) {
        const int i = tid + rr * T;
        if (i < ne * Np) {
          const int el = i / Np, n = i - el * Np;
          const double* q = sQ + el * STR;
          St s;
          load_bg(s, a.bg4, sD[el].bgrow + vert_index<DIM, N>(n));
          s.rp = __dsub_rn(q[n], s.rb);
#pragma unroll
          for (int j = 0; j < 3; ++j) s.U[j] = j < DIM ? q[(1 + j) * Np + n] : 0.0;
          s.Tp = __dsub_rn(q[(DIM + 1) * Np + n], s.Tb);
          const Dv v = derive(s, a);
          double* ax = sAux + el * NAUX * Np + n;
#pragma unroll
          for (int d = 1; d < DIM; ++d) ax[(d - 1) * Np] = __dmul_rn(s.U[d], v.rinv);
          ax[(DIM - 1) * Np] = v.Pp;
          ax[DIM * Np] = v.rinv;
          double Fx[F];
          flux_d<DIM>(s, v, 0, Fx);
          double* fr = sFR + el * F * NPP + (n / n1) * NPAD + (n % n1);
#pragma unroll
          for (int f = 0; f < F; ++f) fr[f * NPP] = Fx[f];
        }
      }
    }
    __syncthreads();

    // ---------------- faces: Rusanov (A5, A6) and lift values (A8) for conforming,
    // wall and fine-side faces (coarse faces were done above)
    {
      constexpr int ROUNDS = (EPB * NFACE * Nf + T - 1) / T;
#pragma unroll 1
      for (int rr = 0; rr < ROUNDS; ++rr) {
        const int i = tid + rr * T;
        if (i >= ne * NFACE * Nf) break;
        const int el = i / (NFACE * Nf);
        const int r = i - el * (NFACE * Nf);
        const int face = r / Nf, t = r - face * Nf;
        const ElemDesc& D = sD[el];
        const int kind = face_kind(D.info, face);
        if (kind == kCoarse) continue;
        const int d = face >> 1;
        const double sgn = (face & 1) ? 1.0 : -1.0;
        const int n = face_node<DIM, N>(face, t);
        const double* q = sQ + el * STR;
        const double* ax = sAux + el * NAUX * Np + n;
        St own;
        load_bg(own, a.bg4, D.bgrow + vert_index<DIM, N>(n));
        own.rp = __dsub_rn(q[n], own.rb);
#pragma unroll
        for (int j = 0; j < 3; ++j) own.U[j] = j < DIM ? q[(1 + j) * Np + n] : 0.0;
        own.Tp = __dsub_rn(q[(DIM + 1) * Np + n], own.Tb);
        Dv vo;
        vo.rho = __dadd_rn(own.rb, own.rp);
        vo.Th = __dadd_rn(own.Tb, own.Tp);
        vo.Pp = ax[(DIM - 1) * Np];
        vo.rinv = ax[DIM * Np];
        const double* tr = sTr + ((el * NFACE + face) * F) * Nf;
        double Fs[F], Fo[F];
        if (kind == kConf) {
          const int en = D.nbr[face];
          St R;
          load_bg(R, a.bg4, __ldg(&a.desc[en].bgrow) + vert_index<DIM, N>(face_node<DIM, N>(face ^ 1, t)));
          R.rp = __dsub_rn(tr[t], R.rb);
#pragma unroll
          for (int j = 0; j < 3; ++j) R.U[j] = j < DIM ? tr[(1 + j) * Nf + t] : 0.0;
          R.Tp = __dsub_rn(tr[(DIM + 1) * Nf + t], R.Tb);
          rusanov<DIM>(own, vo, R, derive(R, a), d, sgn, gam, Fs, Fo);
        } else if (kind == kWall) {
          St R = own;  // mirror ghost (R9)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (j == d) R.U[j] = -own.U[j];
          rusanov<DIM>(own, vo, R, vo, d, sgn, gam, Fs, Fo);
        } else {  // fine side: the coarse side's mortar flux, negated
          const int ec = D.nbr[face];
          const int bgc = __ldg(&a.desc[ec].bgrow);
          auto val = [&](int f, int j) {
            double v = tr[f * Nf + j];
            if (f == 0 || f == DIM + 1) {
              const double2 bb = bg_rt(a.bg4, bgc + vert_index<DIM, N>(face_node<DIM, N>(face ^ 1, j)));
              v = __dsub_rn(v, f == 0 ? bb.x : bb.y);
            }
            return v;
          };
          double qm[F];
          project<DIM, N>(sP, face_sub(D.info, face), t, val, qm);
          St Lm = own;
          Lm.rp = qm[0];
#pragma unroll
          for (int j = 0; j < 3; ++j) Lm.U[j] = j < DIM ? qm[1 + j] : 0.0;
          Lm.Tp = qm[DIM + 1];
          double Fb[F], FLm[F];
          rusanov<DIM>(Lm, derive(Lm, a), own, vo, d, -sgn, gam, Fb, FLm);
#pragma unroll
          for (int f = 0; f < F; ++f) Fs[f] = -Fb[f];
          flux_d<DIM>(own, vo, d, Fo);
        }
        const double cf = __dmul_rn(-sH[elem_level(D.info)][d], a.w0inv);
        double* L = sLift + ((el * NFACE + face) * F) * Nf + t;
#pragma unroll
        for (int f = 0; f < F; ++f) L[f * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[f], Fs[f]));
      }
    }
    __syncthreads();
    if (has_next) issue_traces(tnext, nxt);

    // ---------------- passes: volume divergence (A3) + lifts (A8); last: source (A4), RK epilogue (A9)
    axis_pass<DIM, N, 0>(a, sQ, sAux, sFR, sLift, sD, sH, ne, e0);
    __syncthreads();
    axis_pass<DIM, N, 1>(a, sQ, sAux, sFR, sLift, sD, sH, ne, e0);
    __syncthreads();
    if (DIM == 3) {
      axis_pass<DIM, N, (DIM == 3 ? 2 : 1)>(a, sQ, sAux, sFR, sLift, sD, sH, ne, e0);
      __syncthreads();
    }
  }
}

template <int DIM, int N>
int launch_stage2_t(const StageArgs& a, cudaStream_t s) {
  using C = SC<DIM, N>;
  const size_t bytes = sizeof(double) * C::SMEM;
  static int grid_max = 0;
  if (grid_max == 0) {
    cudaError_t e = cudaFuncSetAttribute(k_stage2<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stage2<DIM, N>, C::T, bytes);
    if (e != cudaSuccess) return e;
    grid_max = sms * (occ > 0 ? occ : 1);
  }
  const int64_t n_tiles = (a.n_elem + C::EPB - 1) / C::EPB;
  const int grid = (int)(n_tiles < grid_max ? n_tiles : grid_max);
  if (grid == 0) return cudaSuccess;
  k_stage2<DIM, N><<<grid, C::T, bytes, s>>>(a);
  return cudaGetLastError();
}

#define DG_DISPATCH2(dim, order, CALL)                                         \
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

int launch_stage(int dim, int order, const StageArgs& a, void* stream) {
  DG_DISPATCH2(dim, order, (launch_stage2_t<D_, N_>(a, (cudaStream_t)stream)));
}

}  // namespace dgi
