// dg_stage.cu -- the fused dGSEM right-hand side / SSP-RK3 stage kernels for
// sm_100a (rows A1-A9 of SURVEY 8(a)).
//
// Method: strong-form dGSEM, Rusanov flux,
// mortars at 2:1 faces, gravity source.
// Readings R2-R17 of DESIGN.md section 3.  Design: DESIGN.md section 6.
//
// One persistent CTA loops over tiles of EPB consecutive elements.  Per tile:
//   issue      this tile's state rows by one cp.async.bulk (mbarrier), its
//              face-neighbour traces and the next tile's descriptors by
//              cp.async, the next tile's rows (and q_n) into L2
//   mortars    coarse side of 2:1 faces: Rusanov on the 2^(d-1) mortars of
//              each coarse face (fine traces gathered from L2), then the back
//              projection into the lift slots (only tiles that own coarse faces)
//   nodes      EOS in perturbation form (P', 1/rho to smem), F^x to a padded
//              buffer that later holds the residual
//   fine       fine side of 2:1 faces: the coarse trace projected onto this
//              element's mortar, in place of the trace
//   faces      Rusanov + lift value for every face node, written over its trace
//   passes     volume flux divergence along each axis (sum-factorised D), the
//              endpoint lifts, the source; the last pass runs the RK epilogue.
// Two kernels share these phases: k_stage (any dim/order; 256 threads; pass
// items = element x field group x pencil, D contraction by DFMA with the
// even-odd split of D from the kernel-parameter constant bank) and k_stage_h7
// (3D, N = 7; 128 threads, 3 CTAs/SM, every phase divides evenly among the
// warps; x and y contractions on the FP64 tensor cores (DMMA m8n8k4), z pass
// per (pencil, half) with DFMA, conflict-free).
// Both elements of a face compute bitwise equal-and-opposite fluxes (explicit
// round-to-nearest intrinsics, identical operand order), so there is no face
// buffer and no atomics; every element writes only its own nodes.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>

#include "dg_internal.h"

namespace dgi {
namespace {

// Tile geometry of the generic kernel.  T threads per CTA, EPB elements per tile
// (3D N = 4: 128 threads x 3 elements -> 375 nodes, 450 face nodes, 225 pass
// items per tile, 3 CTAs per SM).
template <int DIM, int N>
struct SC {
  static constexpr int D_ = DIM, N_ = N;
  static constexpr int n1 = N + 1;
  static constexpr int Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  static constexpr int Nf = Np / n1;
  static constexpr int F = DIM + 2;
  static constexpr int NSUB = 1 << (DIM - 1);
  static constexpr int NFACE = 2 * DIM;
  static constexpr bool H4 = DIM == 3 && N == 4;
#ifndef DG_H4_T
#define DG_H4_T 128
#define DG_H4_EPB 3
#define DG_H4_MCAP 2  // (4: 3.6 % slower on c4, A/B round 2)
#define DG_H4_MINB 3
#endif
  static constexpr int T = H4 ? DG_H4_T : 256;
  static constexpr int EPB = H4 ? DG_H4_EPB : ((T / Np) > 0 ? (T / Np) : 1);
  static constexpr int STR = (F * Np + 15) / 16 * 16;   // element row stride (doubles), = dg_ctx stride
  static constexpr int NPAD = (n1 & 1) ? n1 : n1 + 1;   // x-pencil stride in the padded F^x / residual buffer
  static constexpr int NPP = Nf * NPAD;                 // per field
  static constexpr int NAUX = 2;                        // P', 1/rho
  static constexpr int Q = EPB * STR;
  static constexpr int FR = EPB * F * NPP;
  static constexpr int AUX = EPB * NAUX * Np;
  static constexpr int TR = EPB * NFACE * F * Nf;       // neighbour traces, then (in place) lift values
  static constexpr int MORT1 = NSUB * F * Nf;           // mortar fluxes of one coarse face
  static constexpr int MCAP = H4 ? DG_H4_MCAP : (DIM == 2 ? 8 : 2);  // coarse faces held by the mortar scratch
  static constexpr int MS = MCAP * MORT1;
  static constexpr int CAP = MCAP;                      // chunk size when a tile has more coarse faces
  static constexpr int SMEM = Q + FR + AUX + TR + MS;   // doubles
  static constexpr int MINB = H4 ? DG_H4_MINB : 2;      // CTAs per SM the register budget is sized for
  static constexpr bool SBG = true;                     // background rows staged in smem (cp.async)
  static constexpr int BGE = (n1 + 2) * 4;              // per element: own rows k = 0..N, -z and +z neighbour rows
  __device__ static int fx(int n) { return (n / n1) * NPAD + (n % n1); }  // padded index of node n
  __device__ static int axi(int n) { return n; }                         // aux index of node n
  static_assert(SMEM * 8 <= 220 * 1024, "shared memory budget");
};

// Geometry of the 3D N = 7 kernel (one element at a time per CTA, the next one in flight).
// Plane-per-warp layout: warp w owns the node plane k = w; lane l = 4 g + c owns the two
// nodes (i = 2c, 2c + 1, j = g, k = w) of every field.  These are exactly the rows / columns
// of the FP64 tensor-core (DMMA m8n8k4) fragments of the x pass (transposed form) and of the
// y pass (plain form), so the residual of those two passes stays in the accumulator registers.
struct S7 {
  static constexpr int D_ = 3, N_ = 7;
  static constexpr int n1 = 8, Np = 512, Nf = 64, F = 5, NSUB = 4, NFACE = 6;
  static constexpr int T = 256, NW = 8, EPB = 1;
  static constexpr int STR = 2560;
  static constexpr int NAUX = 2;                   // P', 1/rho per node (read by the face phase)
  static constexpr int Q = STR;                    // one state row (x2: double-buffered bulk copies)
  static constexpr int TR = NFACE * F * Nf;        // neighbour traces, then (in place) lift values (x2)
  static constexpr int AUX = NAUX * Np;
  static constexpr int ZB = F * Np;                // y staging / F^z / z-pass results / mortar scratch
  static constexpr int SMEM = 2 * Q + 2 * TR + AUX + ZB;
  static constexpr int MINB = 2;                   // 2 CTAs x 8 warps per SM (128 registers)
  static constexpr int MORT1 = NSUB * F * Nf;      // mortar scratch of one coarse face
  static constexpr int CAP = ZB / MORT1;
  static constexpr bool SBG = true;                // own rows 0..7, z-neighbour rows 8 (-z), 9 (+z) in smem
  static constexpr int BGE = 40;
  // P' / 1/rho of node n at sAux[axi(n)] / sAux[Np + axi(n)]: the node pair of a lane stays
  // 16-B aligned and a quarter warp's 16-B stores hit 16 distinct doubles
  __device__ static int axi(int n) { return n ^ (4 * ((n >> 4) & 1)); }
  static_assert(SMEM * 8 <= 110 * 1024, "shared memory budget (2 CTAs/SM)");
  static_assert(CAP >= 1, "mortar scratch holds one coarse face");
};

}  // namespace
}  // namespace dgi

#include "dg_device.cuh"

namespace dgi {
namespace {


// Background of own row k (vertical node index) of an element.
template <class C>
__device__ __forceinline__ void own_bg(St& s, const StageArgs& a, const double* sBg, int bgrow, int k) {
  if (C::SBG) {
    const double2 b0 = reinterpret_cast<const double2*>(sBg)[2 * k];
    const double2 b1 = reinterpret_cast<const double2*>(sBg)[2 * k + 1];
    s.rb = b0.x;
    s.Tb = b0.y;
    s.Pb = b1.x;
    s.rTb = b1.y;
  } else {
    load_bg(s, a.bg4, bgrow + k);
  }
}

// Own state at node n of an element staged in smem (perturbation form + background).
template <class C>
__device__ __forceinline__ St own_state(const StageArgs& a, const double* q, int n, const double* sBg, int bgrow) {
  constexpr int DIM = C::D_, N = C::N_, Np = C::Np;
  St s;
  own_bg<C>(s, a, sBg, bgrow, vert_index<DIM, N>(n));
  s.rp = __dsub_rn(q[n], s.rb);
#pragma unroll
  for (int j = 0; j < 3; ++j) s.U[j] = j < DIM ? q[(1 + j) * Np + n] : 0.0;
  s.Tp = __dsub_rn(q[(DIM + 1) * Np + n], s.Tb);
  return s;
}

// Neighbour traces of conforming and fine-side faces: raw values of the
// neighbour's face^1 nodes, [el][face][f][t] (cp.async, 8 B each).
template <class C>
__device__ __forceinline__ void issue_traces(const StageArgs& a, const ElemDesc* sD, int ne, double* sTr) {
  constexpr int DIM = C::D_, N = C::N_, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T, STR = C::STR, Np = C::Np;
  for (int i = threadIdx.x; i < ne * NFACE * Nf; i += T) {
    const int el = i / (NFACE * Nf);
    const int r = i - el * (NFACE * Nf);
    const int face = r / Nf, tt = r - face * Nf;
    const ElemDesc& D = sD[el];
    const int kind = face_kind(D.info, face);
    if (kind == kConf || kind == kFine) {
      const double* src = a.q_in + (int64_t)D.nbr[face] * STR + face_node<DIM, N>(face ^ 1, tt);
      double* dst = sTr + (el * NFACE + face) * F * Nf + tt;
      DG_CHECK((el * NFACE + face) * F * Nf + tt + (F - 1) * Nf < C::TR && D.nbr[face] >= 0 && D.nbr[face] < a.n_elem + 65536);
#pragma unroll
      for (int f = 0; f < F; ++f) cp_async8(dst + f * Nf, src + f * Np);
    }
  }
}

// 3D N = 7 trace gather: x faces node by node (8 B), y and z faces by pairs of
// adjacent nodes (16 B); 256 items, one per thread of the 256-thread CTA.
__device__ __forceinline__ void issue_traces_h7(const StageArgs& a, const ElemDesc& D, double* sTr) {
  constexpr int Nf = 64, F = 5, Np = 512, STR = 2560;
#pragma unroll
  for (int rr = 0; rr < 256 / S7::T; ++rr) {
    const int i = threadIdx.x + S7::T * rr;
    int face, t;
    if (i < 128) {
      face = i >> 6;
      t = i & 63;
    } else {
      face = 2 + ((i - 128) >> 5);
      t = 2 * ((i - 128) & 31);
    }
    const int kind = face_kind(D.info, face);
    if (kind != kConf && kind != kFine) continue;
    const double* src = a.q_in + (int64_t)D.nbr[face] * STR + face_node<3, 7>(face ^ 1, t);
    double* dst = sTr + face * F * Nf + t;
    DG_CHECK(face >= 0 && face < 6 && t >= 0 && t + (i < 128 ? 0 : 1) < Nf && D.nbr[face] >= 0);
    if (i < 128) {
#pragma unroll
      for (int f = 0; f < F; ++f) cp_async8(dst + f * Nf, src + f * Np);
    } else {
#pragma unroll
      for (int f = 0; f < F; ++f) cp_async16(dst + f * Nf, src + f * Np);
    }
  }
}

// Node index map of the face nodes of local face f: node(t1, t2) = off + t1 s1 + t2 s2,
// and the vertical index of those nodes (kv = -1: t2 (3D x/y faces) or t1 (2D x faces)).
template <int DIM, int N>
struct FaceMap {
  int off, s1, s2, kfix;  // kfix >= 0: all face nodes at vertical index kfix
  __device__ __forceinline__ FaceMap(int f) {
    constexpr int n1 = N + 1;
    const int d = f >> 1, e = (f & 1) ? N : 0;
    if (DIM == 2) {
      off = d == 0 ? e : n1 * e;
      s1 = d == 0 ? n1 : 1;
      s2 = 0;
      kfix = d == 0 ? -1 : e;
    } else {
      off = d == 0 ? e : (d == 1 ? n1 * e : n1 * n1 * e);
      s1 = d == 0 ? n1 : 1;
      s2 = d == 2 ? n1 : n1 * n1;
      kfix = d == 2 ? e : -1;
    }
  }
  __device__ __forceinline__ int node(int t1, int t2) const { return off + t1 * s1 + t2 * s2; }
  __device__ __forceinline__ int vert(int t1, int t2) const { return kfix >= 0 ? kfix : (DIM == 2 ? t1 : t2); }
};

// Coarse-side mortar faces of a tile are numbered by slot (element-major, face order).
template <int NFACE>
__device__ __forceinline__ void locate_coarse(const ElemDesc* sD, int ne, int slot, int& el, int& face) {
  el = 0;
  face = 0;
  for (int e = 0, seen = 0; e < ne; ++e) {
    const int c = n_coarse_faces(sD[e].info);
    if (slot < seen + c) {
      el = e;
      for (int f = 0, s = seen; f < NFACE; ++f)
        if (face_kind(sD[e].info, f) == kCoarse && s++ == slot) {
          face = f;
          return;
        }
    }
    seen += c;
  }
}

// EOS (A1) at every node: P', 1/rho to sAux; F^x (A2) into the padded buffer.
template <class C>
__device__ __forceinline__ void node_phase(const StageArgs& a, const double* __restrict__ sQ, const ElemDesc* sD,
                                           int ne, double* __restrict__ sAux, double* __restrict__ sFR,
                                           const double* __restrict__ sBg) {
  constexpr int DIM = C::D_, N = C::N_, Np = C::Np, F = C::F, T = C::T, EPB = C::EPB, STR = C::STR,
                NAUX = C::NAUX, NPP = C::NPP;
  constexpr int ROUNDS = (EPB * Np + T - 1) / T;
#pragma unroll 1
  for (int rr = 0; rr < ROUNDS; ++rr) {
    const int i = threadIdx.x + rr * T;
    if (i < ne * Np) {
      const int el = i / Np, n = i - el * Np;
      const St s = own_state<C>(a, sQ + el * STR, n, sBg + el * C::BGE, sD[el].bgrow);
      const Dv v = derive(s, a);
      double* ax = sAux + el * NAUX * Np + C::axi(n);
      ax[0] = v.Pp;
      ax[Np] = v.rinv;
      double Fx[F];
      flux_d<DIM>(s, v, 0, Fx);
      double* fr = sFR + el * F * NPP + C::fx(n);
#pragma unroll
      for (int f = 0; f < F; ++f) fr[f * NPP] = Fx[f];
    }
  }
}

// ---- direct (unfactorised) mortar operators: k_stage_h7 -----------------------------
// k_stage_h7 keeps the direct tensor-product projection (both sides of its 2:1 faces
// are N = 7 elements of the same kernel, so they agree bitwise with each other); the
// factorised steps below cost it register spills in the uniform path.
// Face -> mortar projection (tensor product of the 1D P_b; R12) of the
// perturbation trace of a coarse face: val(t1, t2, v) fills the F perturbation values
// at face node (t1, t2).  Used by both sides (k_stage_h7) of a 2:1 face with identical arithmetic
// (same order, same rounded coefficients) so their mortar states are bitwise equal.
template <int DIM, int N, class V>
__device__ __forceinline__ void project(const double* sP, int b, int t, const V& val, double* qm) {
  constexpr int n1 = N + 1, F = DIM + 2;
  const int t1 = t % n1, t2 = t / n1;
  const double* P1 = sP + (b & 1) * n1 * n1 + t1 * n1;
  const double* P2 = sP + ((b >> 1) & 1) * n1 * n1 + t2 * n1;
#pragma unroll
  for (int f = 0; f < F; ++f) qm[f] = 0.0;
  for (int j2 = 0; j2 < (DIM == 2 ? 1 : n1); ++j2) {
    for (int j1 = 0; j1 < n1; ++j1) {
      const double c = DIM == 2 ? P1[j1] : __dmul_rn(P1[j1], P2[j2]);
      double v[F];
      val(j1, j2, v);
#pragma unroll
      for (int f = 0; f < F; ++f) qm[f] = __fma_rn(c, v[f], qm[f]);
    }
  }
}

// Mortar step 1 (R11-R13): Rusanov on the mortar nodes of coarse
// slots [s0, s0 + ns) into scratch ms[slot - s0][b][f][t].
template <class C>
__device__ __noinline__ void mortar_flux(const StageArgs& a, const double* sQ, const ElemDesc* sD, int ne, int s0, int ns,
                            double* ms, const double* sP) {
  constexpr int DIM = C::D_, N = C::N_, Np = C::Np, Nf = C::Nf, F = C::F, NSUB = C::NSUB, NFACE = C::NFACE,
                T = C::T, STR = C::STR;
  for (int i = threadIdx.x; i < ns * NSUB * Nf; i += T) {
    const int cs = i / (NSUB * Nf);
    const int r = i - cs * (NSUB * Nf);
    const int b = r / Nf, t = r - b * Nf;
    int el, face;
    locate_coarse<NFACE>(sD, ne, s0 + cs, el, face);
    const ElemDesc& D = sD[el];
    const int d = face >> 1;
    const double sgn = (face & 1) ? 1.0 : -1.0;
    const int mi = D.nbr[face] * NSUB + b;
    const int ef = __ldg(a.mort + mi);
    const FaceMap<DIM, N> fmf(face ^ 1);
    const int nf = fmf.node(t % (N + 1), t / (N + 1));
    St R;
    load_bg(R, a.bg4, __ldg(a.mortbg + mi) + vert_index<DIM, N>(nf));  // fine element's bg row (no desc chase)
    const double* qf = a.q_in + (int64_t)ef * STR;
    R.rp = __dsub_rn(__ldg(qf + nf), R.rb);
#pragma unroll
    for (int j = 0; j < 3; ++j) R.U[j] = j < DIM ? __ldg(qf + (1 + j) * Np + nf) : 0.0;
    R.Tp = __dsub_rn(__ldg(qf + (DIM + 1) * Np + nf), R.Tb);
    const double* q = sQ + el * STR;
    const FaceMap<DIM, N> fm(face);
    auto val = [&](int j1, int j2, double* v) {
      const int n = fm.node(j1, j2);
      const double2 bb = bg_rt(a.bg4, D.bgrow + fm.vert(j1, j2));
#pragma unroll
      for (int f = 0; f < F; ++f) v[f] = q[f * Np + n];
      v[0] = __dsub_rn(v[0], bb.x);
      v[DIM + 1] = __dsub_rn(v[DIM + 1], bb.y);
    };
    double qm[F];
    project<DIM, N>(sP, b, t, val, qm);
    St Lm = R;  // fine-level background at the mortar node (R13)
    Lm.rp = qm[0];
#pragma unroll
    for (int j = 0; j < 3; ++j) Lm.U[j] = j < DIM ? qm[1 + j] : 0.0;
    Lm.Tp = qm[DIM + 1];
    double Fs[F], FL[F];
    rusanov<DIM>(Lm, derive(Lm, a), R, derive(R, a), d, sgn, a.gamma, Fs, FL);
    double* mo = ms + cs * C::MORT1 + b * F * Nf;
    DG_CHECK(cs < C::CAP && cs * C::MORT1 + b * F * Nf + (F - 1) * Nf + t < C::CAP * C::MORT1);
#pragma unroll
    for (int f = 0; f < F; ++f) mo[f * Nf + t] = Fs[f];
  }
}

// Mortar step 2 for coarse face node j (R11, R12, R14): back
// projection sum_b (kron R_b) F*_b (s = 1/2 per axis) and the lift value.
template <class C>
__device__ __noinline__ void mortar_lift(const StageArgs& a, const double* q, const ElemDesc& D, int face, int j,
                                            const double* mo, const double* sR, const double (*sH)[3],
                                            double* L /* trace slot [f * Nf] */) {
  constexpr int DIM = C::D_, N = C::N_, n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NSUB = C::NSUB;
  const int d = face >> 1;
  const double sgn = (face & 1) ? 1.0 : -1.0;
  const int j1 = j % n1, j2 = j / n1;
  double Fc[F];
#pragma unroll
  for (int f = 0; f < F; ++f) Fc[f] = 0.0;
  for (int b = 0; b < NSUB; ++b) {
    const double* R1 = sR + (b & 1) * n1 * n1 + j1 * n1;
    const double* R2 = sR + ((b >> 1) & 1) * n1 * n1 + j2 * n1;
    const double* m = mo + b * F * Nf;
    for (int k2 = 0; k2 < (DIM == 2 ? 1 : n1); ++k2)
      for (int k1 = 0; k1 < n1; ++k1) {
        const double c = DIM == 2 ? R1[k1] : __dmul_rn(R1[k1], R2[k2]);
        const int k = k1 + n1 * k2;
#pragma unroll
        for (int f = 0; f < F; ++f) Fc[f] = __fma_rn(c, m[f * Nf + k], Fc[f]);
      }
  }
  const int n = face_node<DIM, N>(face, j);
  St own;
  load_bg(own, a.bg4, D.bgrow + vert_index<DIM, N>(n));
  own.rp = __dsub_rn(q[n], own.rb);
#pragma unroll
  for (int jj = 0; jj < 3; ++jj) own.U[jj] = jj < DIM ? q[(1 + jj) * Np + n] : 0.0;
  own.Tp = __dsub_rn(q[(DIM + 1) * Np + n], own.Tb);
  double Fo[F];
  flux_d<DIM>(own, derive(own, a), d, Fo);
  const double cf = __dmul_rn(-sH[elem_level(D.info)][d], a.w0inv);
#pragma unroll
  for (int f = 0; f < F; ++f) L[f * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[f], Fc[f]));
}

// All coarse faces of a tile in chunks of C::CAP through scratch ms (two barriers per chunk).
template <class C>
__device__ __noinline__ void mortar_chunks(const StageArgs& a, const double* sQ, const ElemDesc* sD, int ne, int n_coarse,
                              double* ms, double* sTr, const double* sP, const double* sR, const double (*sH)[3]) {
  constexpr int Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T, STR = C::STR;
  for (int c0 = 0; c0 < n_coarse; c0 += C::CAP) {
    const int nc = min(C::CAP, n_coarse - c0);
    mortar_flux<C>(a, sQ, sD, ne, c0, nc, ms, sP);
    __syncthreads();
    for (int i = threadIdx.x; i < nc * Nf; i += T) {
      const int cs = i / Nf, j = i - cs * Nf;
      int el, face;
      locate_coarse<NFACE>(sD, ne, c0 + cs, el, face);
      mortar_lift<C>(a, sQ + el * STR, sD[el], face, j, ms + cs * C::MORT1, sR, sH,
                     sTr + ((el * NFACE + face) * F) * Nf + j);
    }
    __syncthreads();
  }
}

// Fine side (k_stage_h7): project the coarse trace onto this element's mortar with the
// item -> thread map of face_phase, so the projected values need one barrier only.
template <class C>
__device__ __noinline__ void fine_phase_inplace(const StageArgs& a, const ElemDesc* sD, const int* sNb, int ne, double* sTr,
                                        const double* sP) {
  constexpr int DIM = C::D_, N = C::N_, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T, EPB = C::EPB;
  constexpr int ROUNDS = (EPB * NFACE * Nf + T - 1) / T;
  double qm[ROUNDS][F];
#pragma unroll
  for (int rr = 0; rr < ROUNDS; ++rr) {
    const int i = threadIdx.x + rr * T;
    if (i >= ne * NFACE * Nf) break;
    const int el = i / (NFACE * Nf);
    const int r = i - el * (NFACE * Nf);
    const int face = r / Nf, t = r - face * Nf;
    const ElemDesc& D = sD[el];
    if (face_kind(D.info, face) != kFine) continue;
    const double* tf = sTr + ((el * NFACE + face) * F) * Nf;
    const int bgc = sNb[el * 8 + face];
    const FaceMap<DIM, N> fmc(face ^ 1);
    auto val = [&](int j1, int j2, double* v) {
      const int j = j1 + (N + 1) * j2;
      const double2 bb = bg_rt(a.bg4, bgc + fmc.vert(j1, j2));
#pragma unroll
      for (int f = 0; f < F; ++f) v[f] = tf[f * Nf + j];
      v[0] = __dsub_rn(v[0], bb.x);
      v[DIM + 1] = __dsub_rn(v[DIM + 1], bb.y);
    };
    project<DIM, N>(sP, face_sub(D.info, face), t, val, qm[rr]);
  }
  __syncthreads();
#pragma unroll
  for (int rr = 0; rr < ROUNDS; ++rr) {
    const int i = threadIdx.x + rr * T;
    if (i >= ne * NFACE * Nf) break;
    const int el = i / (NFACE * Nf);
    const int r = i - el * (NFACE * Nf);
    const int face = r / Nf, t = r - face * Nf;
    if (face_kind(sD[el].info, face) != kFine) continue;
    double* tr = sTr + ((el * NFACE + face) * F) * Nf + t;
#pragma unroll
    for (int f = 0; f < F; ++f) tr[f * Nf] = qm[rr][f];
  }
}

// ---- sum-factorised mortar operators (generic kernel; R35) --------------------------
// The 3D face -> mortar projection kron(P_b2, P_b1) is applied as
// two 1D passes, along t1 then along t2; both sides of a 2:1 face run the same two
// passes on the same operands in the same order, so their mortar states stay bitwise
// equal.  The back projection sum_b kron(R_b2, R_b1) F*_b is
// applied as sum over b1 along k1, then sum over b2 along k2.  Coarse slot scratch
// ms[s][b][f][t] (t = t1 + n1 t2) holds, in turn: U_b1 (at b = b1), the mortar states,
// the mortar fluxes F*_b, and W_b2 (at b = 2 b2).

// out[r] = sum_j M[r][j] in[j], j ascending (M row-major n1 x n1)
template <int N>
__device__ __forceinline__ void apply1d(const double* M, const double* in, double* out) {
  constexpr int n1 = N + 1;
#pragma unroll
  for (int r = 0; r < n1; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < n1; ++j) acc = __fma_rn(M[r * n1 + j], in[j], acc);
    out[r] = acc;
  }
}

// Coarse step A: U_b1[f][t1 + n1 j2] = sum_j1 P_b1[t1][j1] (q - qbar)[f](j1, j2); in 2D
// this is already the mortar state of sub-face b1.
template <class C>
__device__ __forceinline__ void mort_A_body(const StageArgs& a, const double* sQ, const ElemDesc* sD, const uint8_t* lst, int s0, int ns,
                                    double* ms, const double* sP) {
  constexpr int DIM = C::D_, N = C::N_, n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T,
                STR = C::STR, NJ2 = DIM == 2 ? 1 : n1;
  for (int i = threadIdx.x; i < ns * 2 * F * NJ2; i += T) {
    int r = i;
    const int j2 = r % NJ2;
    r /= NJ2;
    const int f = r % F;
    r /= F;
    const int b1 = r & 1, cs = r >> 1;
    const int el = lst[s0 + cs] >> 3, face = lst[s0 + cs] & 7;
    const ElemDesc& D = sD[el];
    const FaceMap<DIM, N> fm(face);
    const double* q = sQ + el * STR + f * Np;
    double in[n1], out[n1];
#pragma unroll
    for (int j1 = 0; j1 < n1; ++j1) {
      double v = q[fm.node(j1, j2)];
      if (f == 0 || f == DIM + 1) {
        const double2 bb = bg_rt(a.bg4, D.bgrow + fm.vert(j1, j2));
        v = __dsub_rn(v, f == 0 ? bb.x : bb.y);
      }
      in[j1] = v;
    }
    apply1d<N>(sP + b1 * n1 * n1, in, out);
    double* o = ms + cs * C::MORT1 + (b1 * F + f) * Nf + j2 * n1;
#pragma unroll
    for (int t1 = 0; t1 < n1; ++t1) o[t1] = out[t1];
  }
}

// Coarse step B (3D): mortar state of sub-face b1 + 2 b2, row t1: sum_j2 P_b2[t2][j2] U_b1[t1 + n1 j2].
template <class C>
__device__ __forceinline__ void mort_B_body(int ns, double* ms, const double* sP) {
  constexpr int N = C::N_, n1 = C::n1, Nf = C::Nf, F = C::F, T = C::T;
  for (int i = threadIdx.x; i < ns * 2 * F * n1; i += T) {
    int r = i;
    const int t1 = r % n1;
    r /= n1;
    const int f = r % F;
    r /= F;
    const int b1 = r & 1, cs = r >> 1;
    double* u0 = ms + cs * C::MORT1 + (b1 * F + f) * Nf + t1;
    double* u1 = ms + cs * C::MORT1 + ((b1 + 2) * F + f) * Nf + t1;
    double in[n1], out[n1];
#pragma unroll
    for (int j2 = 0; j2 < n1; ++j2) in[j2] = u0[n1 * j2];
    apply1d<N>(sP, in, out);
#pragma unroll
    for (int t2 = 0; t2 < n1; ++t2) u0[n1 * t2] = out[t2];
    apply1d<N>(sP + n1 * n1, in, out);
#pragma unroll
    for (int t2 = 0; t2 < n1; ++t2) u1[n1 * t2] = out[t2];
  }
}

// Coarse step C (R11-R13): Rusanov at mortar node t of sub-face b,
// mortar state (in ms) with the fine level's background vs the fine element's trace,
// written over the state.
template <class C>
__device__ __forceinline__ void mort_C_body(const StageArgs& a, const ElemDesc* sD, const uint8_t* lst, int s0, int ns, double* ms) {
  constexpr int DIM = C::D_, N = C::N_, Np = C::Np, Nf = C::Nf, F = C::F, NSUB = C::NSUB, NFACE = C::NFACE,
                T = C::T, STR = C::STR;
  for (int i = threadIdx.x; i < ns * NSUB * Nf; i += T) {
    const int cs = i / (NSUB * Nf);
    const int r = i - cs * (NSUB * Nf);
    const int b = r / Nf, t = r - b * Nf;
    const int el = lst[s0 + cs] >> 3, face = lst[s0 + cs] & 7;
    const ElemDesc& D = sD[el];
    const int d = face >> 1;
    const double sgn = (face & 1) ? 1.0 : -1.0;
    const int mi = D.nbr[face] * NSUB + b;
    const int ef = __ldg(a.mort + mi);
    const FaceMap<DIM, N> fmf(face ^ 1);
    const int nf = fmf.node(t % (N + 1), t / (N + 1));
    St R;
    load_bg(R, a.bg4, __ldg(a.mortbg + mi) + vert_index<DIM, N>(nf));  // fine element's bg row (no desc chase)
    const double* qf = a.q_in + (int64_t)ef * STR;
    R.rp = __dsub_rn(__ldg(qf + nf), R.rb);
#pragma unroll
    for (int j = 0; j < 3; ++j) R.U[j] = j < DIM ? __ldg(qf + (1 + j) * Np + nf) : 0.0;
    R.Tp = __dsub_rn(__ldg(qf + (DIM + 1) * Np + nf), R.Tb);
    double* mo = ms + cs * C::MORT1 + b * F * Nf + t;
    St Lm = R;  // fine-level background at the mortar node (R13)
    Lm.rp = mo[0];
#pragma unroll
    for (int j = 0; j < 3; ++j) Lm.U[j] = j < DIM ? mo[(1 + j) * Nf] : 0.0;
    Lm.Tp = mo[(DIM + 1) * Nf];
    double Fs[F], FL[F];
    rusanov<DIM>(Lm, derive(Lm, a), R, derive(R, a), d, sgn, a.gamma, Fs, FL);
#pragma unroll
    for (int f = 0; f < F; ++f) mo[f * Nf] = Fs[f];
  }
}

// Coarse step D (3D): W_b2[f][j1 + n1 k2] = sum_b1 sum_k1 R_b1[j1][k1] F*_{b1 + 2 b2}[f][k1 + n1 k2],
// written over F*_{2 b2}.
template <class C>
__device__ __forceinline__ void mort_D_body(int ns, double* ms, const double* sR) {
  constexpr int n1 = C::n1, Nf = C::Nf, F = C::F, T = C::T;
  for (int i = threadIdx.x; i < ns * 2 * F * n1; i += T) {
    int r = i;
    const int k2 = r % n1;
    r /= n1;
    const int f = r % F;
    r /= F;
    const int b2 = r & 1, cs = r >> 1;
    double* m0 = ms + cs * C::MORT1 + ((2 * b2) * F + f) * Nf + n1 * k2;
    const double* m1 = ms + cs * C::MORT1 + ((2 * b2 + 1) * F + f) * Nf + n1 * k2;
    double in0[n1], in1[n1];
#pragma unroll
    for (int k1 = 0; k1 < n1; ++k1) {
      in0[k1] = m0[k1];
      in1[k1] = m1[k1];
    }
#pragma unroll
    for (int j1 = 0; j1 < n1; ++j1) {
      double acc = 0.0;
#pragma unroll
      for (int k1 = 0; k1 < n1; ++k1) acc = __fma_rn(sR[j1 * n1 + k1], in0[k1], acc);
#pragma unroll
      for (int k1 = 0; k1 < n1; ++k1) acc = __fma_rn(sR[n1 * n1 + j1 * n1 + k1], in1[k1], acc);
      m0[j1] = acc;
    }
  }
}

// Coarse step E (R11, R12, R14): back-projected flux at coarse face
// node j and the lift value, written into the face's trace slot.
template <class C>
__device__ __forceinline__ void mort_E_body(const StageArgs& a, const double* sQ, const ElemDesc* sD, const uint8_t* lst, int s0, int ns,
                                    const double* ms, const double* sR, const double (*sH)[3], double* sTr) {
  constexpr int DIM = C::D_, N = C::N_, n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T,
                STR = C::STR;
  for (int i = threadIdx.x; i < ns * Nf; i += T) {
    const int cs = i / Nf, j = i - cs * Nf;
    const int el = lst[s0 + cs] >> 3, face = lst[s0 + cs] & 7;
    const ElemDesc& D = sD[el];
    const double* mo = ms + cs * C::MORT1;
    const int d = face >> 1;
    const double sgn = (face & 1) ? 1.0 : -1.0;
    double Fc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) Fc[f] = 0.0;
    if (DIM == 2) {
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int k = 0; k < n1; ++k) {
          const double c = sR[b * n1 * n1 + j * n1 + k];
#pragma unroll
          for (int f = 0; f < F; ++f) Fc[f] = __fma_rn(c, mo[(b * F + f) * Nf + k], Fc[f]);
        }
    } else {
      const int j1 = j % n1, j2 = j / n1;
#pragma unroll
      for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
        for (int k2 = 0; k2 < n1; ++k2) {
          const double c = sR[b2 * n1 * n1 + j2 * n1 + k2];
#pragma unroll
          for (int f = 0; f < F; ++f) Fc[f] = __fma_rn(c, mo[((2 * b2) * F + f) * Nf + j1 + n1 * k2], Fc[f]);
        }
    }
    const double* q = sQ + el * STR;
    const int n = face_node<DIM, N>(face, j);
    St own;
    load_bg(own, a.bg4, D.bgrow + vert_index<DIM, N>(n));
    own.rp = __dsub_rn(q[n], own.rb);
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) own.U[jj] = jj < DIM ? q[(1 + jj) * Np + n] : 0.0;
    own.Tp = __dsub_rn(q[(DIM + 1) * Np + n], own.Tb);
    double Fo[F];
    flux_d<DIM>(own, derive(own, a), d, Fo);
    const double cf = __dmul_rn(-sH[elem_level(D.info)][d], a.w0inv);
    double* L = sTr + ((el * NFACE + face) * F) * Nf + j;
#pragma unroll
    for (int f = 0; f < F; ++f) L[f * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[f], Fc[f]));
  }
}

// Fine step A: the coarse trace in the slot (raw) -> U[f][t1 + n1 j2] = sum_j1 P_b1[t1][j1]
// (trace - coarse qbar), in place (2D: the mortar state).  Item (slot, f, j2) reads and
// writes only column j2 of field f.
template <class C>
__device__ __forceinline__ void fine_A_body(const StageArgs& a, const ElemDesc* sD, const int* sNb, const uint8_t* lst, int n_fine,
                                    double* sTr, const double* sP) {
  constexpr int DIM = C::D_, N = C::N_, n1 = C::n1, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T,
                NJ2 = DIM == 2 ? 1 : n1;
  for (int i = threadIdx.x; i < n_fine * F * NJ2; i += T) {
    int r = i;
    const int j2 = r % NJ2;
    r /= NJ2;
    const int f = r % F, sl = r / F;
    const int el = lst[sl] >> 3, face = lst[sl] & 7;
    const int b1 = face_sub(sD[el].info, face) & 1;
    double* tf = sTr + ((el * NFACE + face) * F + f) * Nf + j2 * n1;
    const int bgc = sNb[el * 8 + face];
    const FaceMap<DIM, N> fmc(face ^ 1);
    double in[n1], out[n1];
#pragma unroll
    for (int j1 = 0; j1 < n1; ++j1) {
      double v = tf[j1];
      if (f == 0 || f == DIM + 1) {
        const double2 bb = bg_rt(a.bg4, bgc + fmc.vert(j1, j2));
        v = __dsub_rn(v, f == 0 ? bb.x : bb.y);
      }
      in[j1] = v;
    }
    apply1d<N>(sP + b1 * n1 * n1, in, out);
#pragma unroll
    for (int t1 = 0; t1 < n1; ++t1) tf[t1] = out[t1];
  }
}

// Fine step B (3D): mortar state row t1 = sum_j2 P_b2[t2][j2] U[t1 + n1 j2], in place.
template <class C>
__device__ __forceinline__ void fine_B_body(const ElemDesc* sD, const uint8_t* lst, int n_fine, double* sTr, const double* sP) {
  constexpr int N = C::N_, n1 = C::n1, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T;
  for (int i = threadIdx.x; i < n_fine * F * n1; i += T) {
    int r = i;
    const int t1 = r % n1;
    r /= n1;
    const int f = r % F, sl = r / F;
    const int el = lst[sl] >> 3, face = lst[sl] & 7;
    const int b2 = (face_sub(sD[el].info, face) >> 1) & 1;
    double* tf = sTr + ((el * NFACE + face) * F + f) * Nf + t1;
    double in[n1], out[n1];
#pragma unroll
    for (int j2 = 0; j2 < n1; ++j2) in[j2] = tf[n1 * j2];
    apply1d<N>(sP + b2 * n1 * n1, in, out);
#pragma unroll
    for (int t2 = 0; t2 < n1; ++t2) tf[n1 * t2] = out[t2];
  }
}

// Out-of-line entry points of the mortar steps (rare path: keeps the tile loop small).
template <class C>
__device__ __noinline__ void mort_A(const StageArgs& a, const double* sQ, const ElemDesc* sD, const uint8_t* lst, int s0,
                                    int ns, double* ms, const double* sP) { mort_A_body<C>(a, sQ, sD, lst, s0, ns, ms, sP); }
template <class C>
__device__ __noinline__ void mort_E(const StageArgs& a, const double* sQ, const ElemDesc* sD, const uint8_t* lst, int s0,
                                    int ns, const double* ms, const double* sR, const double (*sH)[3], double* sTr) {
  mort_E_body<C>(a, sQ, sD, lst, s0, ns, ms, sR, sH, sTr);
}
// Mortar steps between the trace barrier and face_phase (nc = coarse slots held in ms,
// nf = fine faces of the tile); one out-of-line call keeps the tile loop's registers.
template <class C>
__device__ __noinline__ void amr_mid(const StageArgs& a, const double* sQ, const ElemDesc* sD, const int* sNb,
                                     const uint8_t* cl, const uint8_t* fl, int nc, int nf, double* ms, double* sTr, const double* sP, const double* sR,
                                     const double (*sH)[3]) {
  if (C::D_ == 3) {
    if (nc) mort_B_body<C>(nc, ms, sP);
  } else {
    if (nc) mort_C_body<C>(a, sD, cl, 0, nc, ms);
  }
  if (nf) fine_A_body<C>(a, sD, sNb, fl, nf, sTr, sP);
  __syncthreads();
  if (C::D_ == 3) {
    if (nc) mort_C_body<C>(a, sD, cl, 0, nc, ms);
    if (nf) fine_B_body<C>(sD, fl, nf, sTr, sP);
    __syncthreads();
    if (nc) mort_D_body<C>(nc, ms, sR);
  } else {
    if (nc) mort_E_body<C>(a, sQ, sD, cl, 0, nc, ms, sR, sH, sTr);
  }
}

// Coarse / fine face slot lists of a tile (entries el * 8 + face, element-major, face
// order, as locate_coarse), built by warp 0.
template <class C>
__device__ __forceinline__ void build_lists(const ElemDesc* sD, int ne, uint8_t* cl, uint8_t* fl) {
  constexpr int NFACE = C::NFACE, NP = C::EPB * NFACE;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int nc = 0, nf = 0;
#pragma unroll
  for (int b = 0; b < NP; b += 32) {
    const int i = b + lane;
    const int el = i / NFACE, face = i - el * NFACE;
    const int kind = i < ne * NFACE ? face_kind(sD[el].info, face) : -1;
    const unsigned mc = __ballot_sync(~0u, kind == kCoarse), mf = __ballot_sync(~0u, kind == kFine);
    if (kind == kCoarse) cl[nc + __popc(mc & lt)] = (uint8_t)(el * 8 + face);
    if (kind == kFine) fl[nf + __popc(mf & lt)] = (uint8_t)(el * 8 + face);
    nc += __popc(mc);
    nf += __popc(mf);
  }
}

// NEXT-3 baseline (reading R41): pointwise interpolation on the coarse side
// of 2:1 faces.  At coarse face node j the fine sub-face containing it (x = 0 belongs to
// the lower one) is evaluated there -- the fine element's perturbation trace interpolated
// with I_b (fine Lagrange basis at the node's sub-face coordinate), plus the coarse node's
// background -- and Rusanov is taken against the coarse own state; the lift value goes
// into the face's slot.  Not conservative: the fine side keeps its projected trace.
template <class C>
__device__ __noinline__ void point_coarse(const StageArgs& a, const double* sQ, const ElemDesc* sD,
                                          const uint8_t* lst, int ns, const double (*sH)[3], double* sTr) {
  constexpr int DIM = C::D_, N = C::N_, n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NSUB = C::NSUB,
                NFACE = C::NFACE, T = C::T, STR = C::STR;
  const double* Iop = a.ops + OpsLayout::I(n1, 0);
  for (int i = threadIdx.x; i < ns * Nf; i += T) {
    const int cs = i / Nf, j = i - cs * Nf;
    const int el = lst[cs] >> 3, face = lst[cs] & 7;
    const ElemDesc& D = sD[el];
    const int d = face >> 1;
    const double sgn = (face & 1) ? 1.0 : -1.0;
    const int j1 = j % n1, j2 = j / n1;
    const int b1 = 2 * j1 > N ? 1 : 0, b2 = (DIM == 3 && 2 * j2 > N) ? 1 : 0;
    const int ef = __ldg(a.mort + D.nbr[face] * NSUB + b1 + 2 * b2);
    const double* qf = a.q_in + (int64_t)ef * STR;
    const int bgf = __ldg(&a.desc[ef].bgrow);
    const FaceMap<DIM, N> fmf(face ^ 1);
    double v[F];
#pragma unroll
    for (int f = 0; f < F; ++f) v[f] = 0.0;
    for (int k2 = 0; k2 < (DIM == 2 ? 1 : n1); ++k2) {
      const double w2 = DIM == 2 ? 1.0 : Iop[b2 * n1 * n1 + j2 * n1 + k2];
      for (int k1 = 0; k1 < n1; ++k1) {
        const double c = DIM == 2 ? Iop[b1 * n1 * n1 + j1 * n1 + k1] : __dmul_rn(Iop[b1 * n1 * n1 + j1 * n1 + k1], w2);
        const int nf = fmf.node(k1, k2);
        const double2 bb = bg_rt(a.bg4, bgf + fmf.vert(k1, k2));
        v[0] = __fma_rn(c, __dsub_rn(__ldg(qf + nf), bb.x), v[0]);
#pragma unroll
        for (int f = 1; f <= DIM; ++f) v[f] = __fma_rn(c, __ldg(qf + f * Np + nf), v[f]);
        v[DIM + 1] = __fma_rn(c, __dsub_rn(__ldg(qf + (DIM + 1) * Np + nf), bb.y), v[DIM + 1]);
      }
    }
    const double* q = sQ + el * STR;
    const int n = face_node<DIM, N>(face, j);
    St own;
    load_bg(own, a.bg4, D.bgrow + vert_index<DIM, N>(n));
    own.rp = __dsub_rn(q[n], own.rb);
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) own.U[jj] = jj < DIM ? q[(1 + jj) * Np + n] : 0.0;
    own.Tp = __dsub_rn(q[(DIM + 1) * Np + n], own.Tb);
    St R = own;  // the coarse node's background (R13 in reverse)
    R.rp = v[0];
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) R.U[jj] = jj < DIM ? v[1 + jj] : 0.0;
    R.Tp = v[DIM + 1];
    double Fs[F], Fo[F];
    rusanov<DIM>(own, derive(own, a), R, derive(R, a), d, sgn, a.gamma, Fs, Fo);
    const double cf = __dmul_rn(-sH[elem_level(D.info)][d], a.w0inv);
    double* L = sTr + ((el * NFACE + face) * F) * Nf + j;
#pragma unroll
    for (int f = 0; f < F; ++f) L[f * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[f], Fs[f]));
  }
}

// A tile's coarse faces beyond the scratch capacity: all mortar steps chunk by chunk.
template <class C>
__device__ __noinline__ void mort_chunks_fact(const StageArgs& a, const double* sQ, const ElemDesc* sD, const uint8_t* cl,
                                              int n_coarse, double* ms, double* sTr, const double* sP, const double* sR,
                                              const double (*sH)[3]) {
  for (int c0 = 0; c0 < n_coarse; c0 += C::MCAP) {
    const int nc = min(C::MCAP, n_coarse - c0);
    mort_A_body<C>(a, sQ, sD, cl, c0, nc, ms, sP);
    __syncthreads();
    if (C::D_ == 3) {
      mort_B_body<C>(nc, ms, sP);
      __syncthreads();
    }
    mort_C_body<C>(a, sD, cl, c0, nc, ms);
    __syncthreads();
    if (C::D_ == 3) {
      mort_D_body<C>(nc, ms, sR);
      __syncthreads();
    }
    mort_E_body<C>(a, sQ, sD, cl, c0, nc, ms, sR, sH, sTr);
    __syncthreads();
  }
}

// Rusanov (A5, A6) and the lift value (A8) at every face node, written over its
// trace slot: conforming, wall and fine side (mortar state in the slot); coarse-side
// lifts come from the mortar steps (mort_E).
template <class C>
__device__ __forceinline__ void face_phase(const StageArgs& a, const double* __restrict__ sQ,
                                           const double* __restrict__ sAux, const ElemDesc* sD, const int* sNb, int ne,
                                           double* __restrict__ sTr, const double (*sH)[3],
                                           const double* __restrict__ sBg) {
  constexpr int DIM = C::D_, N = C::N_, Np = C::Np, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T,
                EPB = C::EPB, STR = C::STR, NAUX = C::NAUX;
  constexpr int ROUNDS = (EPB * NFACE * Nf + T - 1) / T;
  const double gam = a.gamma;
#pragma unroll 1
  for (int rr = 0; rr < ROUNDS; ++rr) {
    const int i = threadIdx.x + rr * T;
    if (i >= ne * NFACE * Nf) break;
    const int el = i / (NFACE * Nf);
    const int r = i - el * (NFACE * Nf);
    const int face = r / Nf, t = r - face * Nf;
    const ElemDesc& D = sD[el];
    const int kind = face_kind(D.info, face);
    double* tr = sTr + ((el * NFACE + face) * F) * Nf + t;
    DG_CHECK(((el * NFACE + face) * F) * Nf + t + (F - 1) * Nf < EPB * NFACE * F * Nf);
    if (kind == kCoarse) continue;  // coarse side: lifts from the mortar fluxes, below
    const int d = face >> 1;
    const double sgn = (face & 1) ? 1.0 : -1.0;
    const int n = face_node<DIM, N>(face, t);
    const double* ax = sAux + el * NAUX * Np + C::axi(n);
    const double* bgE = sBg + el * C::BGE;
    const St own = own_state<C>(a, sQ + el * STR, n, bgE, D.bgrow);
    Dv vo;
    vo.rho = __dadd_rn(own.rb, own.rp);
    vo.Th = __dadd_rn(own.Tb, own.Tp);
    vo.Pp = ax[0];
    vo.rinv = ax[Np];
    double Fs[F], Fo[F];
    if (kind == kWall) {
      St R = own;  // mirror ghost (R9)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (j == d) R.U[j] = -own.U[j];
      rusanov<DIM>(own, vo, R, vo, d, sgn, gam, Fs, Fo);
    } else {
      // conforming: neighbour trace (raw values); fine side: projected mortar state
      // (perturbation form) with this element's background (R13)
      St R;
      if (kind == kFine) {
        R = own;
        R.rp = tr[0];
        R.Tp = tr[(DIM + 1) * Nf];
      } else {
        if (C::SBG) {  // same-level neighbour: horizontal neighbours share this element's rows;
                       // vertical: staged rows N+1 (-z), N+2 (+z)
          if (d < DIM - 1) own_bg<C>(R, a, bgE, 0, vert_index<DIM, N>(n));
          else own_bg<C>(R, a, bgE, 0, N + 1 + (face & 1));
        } else {
          load_bg(R, a.bg4, sNb[el * 8 + face] + vert_index<DIM, N>(face_node<DIM, N>(face ^ 1, t)));
        }
        R.rp = __dsub_rn(tr[0], R.rb);
        R.Tp = __dsub_rn(tr[(DIM + 1) * Nf], R.Tb);
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) R.U[j] = j < DIM ? tr[(1 + j) * Nf] : 0.0;
      if (kind == kConf) {
        rusanov<DIM>(own, vo, R, derive(R, a), d, sgn, gam, Fs, Fo);
      } else {  // the coarse side's mortar flux rusanov(Lm, fine, d, sgn_c), negated (bitwise)
        double Fb[F], FLm[F];
        rusanov<DIM>(R, derive(R, a), own, vo, d, -sgn, gam, Fb, FLm);
#pragma unroll
        for (int f = 0; f < F; ++f) Fs[f] = -Fb[f];
        flux_d<DIM>(own, vo, d, Fo);
      }
    }
    const double cf = __dmul_rn(-sH[elem_level(D.info)][d], a.w0inv);
#pragma unroll
    for (int f = 0; f < F; ++f) tr[f * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[f], Fs[f]));
  }
}

// Pencil of axis d with index p (= face node index of the axis-d faces):
// first node and its index in the padded x-pencil layout of sFR.
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
  static constexpr int pad = d == 0 ? 1 : (d == 1 ? NPAD : n1 * NPAD);
};

// One axis pass.  Thread item = (element, field, pencil along d), one code path
// for all fields (runtime f; small code keeps the instruction cache warm).  F^x
// comes precomputed from the padded buffer; for d > 0 the flux is formed here:
// F^d_0 = U_d, F^d_f = q_f u_d (+ P' for f = 1 + d), u_d = U_d / rho (as in flux_d).
template <int DIM, int N, int d, bool LIST>
__device__ __forceinline__ void axis_pass(const StageArgs& a, const double* __restrict__ sQ,
                                          const double* __restrict__ sAux, double* __restrict__ sFR,
                                          const double* __restrict__ sLift, const ElemDesc* sD, const double (*sH)[3],
                                          int ne, int64_t e0) {
  using C = SC<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, Nf = C::Nf, F = C::F, NFACE = C::NFACE, T = C::T, EPB = C::EPB,
                STR = C::STR, NPP = C::NPP, NAUX = C::NAUX;
  constexpr int ST = PStep<DIM, N, d>::node, PST = PStep<DIM, N, d>::pad;
  constexpr bool LAST = d == DIM - 1;
  constexpr int ROUNDS = (EPB * F * Nf + T - 1) / T;
  const bool need_qn = LAST && a.mode == 1 && a.stage > 0;
#pragma unroll 1
  for (int rr = 0; rr < ROUNDS; ++rr) {
    const int i = threadIdx.x + rr * T;
    if (i >= ne * F * Nf) break;
    const int el = i / (F * Nf);
    const int r = i - el * (F * Nf);
    // y pencils (3D) field-fastest: the p-fastest order puts the 16 lanes of a half warp on
    // node offsets i + n1^2 k that share banks; field-fastest lanes share U_d, P', 1/rho
    // (broadcast) and spread the rest
    constexpr bool PF = DIM == 3 && d == 1;
    const int f = PF ? r % F : r / Nf, p = PF ? r / F : r - f * Nf;
    int base, pbase;
    pencil_addr<DIM, N, d>(p, base, pbase);
    const double* q = sQ + el * STR + base;
    const double* ax = sAux + el * NAUX * Np + base;  // [0]: P', [Np]: 1/rho
    double* fr = sFR + el * F * NPP + f * NPP + pbase;
    DG_CHECK(el * F * NPP + f * NPP + pbase + N * PST < C::FR && base + N * ST < Np);
    double qn[n1];
    if (need_qn) {  // q_n is read once: evict-first (c4 / c5n4 stage -0.8 %)
      const double* g = a.q_n + elem_of<LIST>(a, e0 + el) * STR + f * Np + base;
#pragma unroll
      for (int m = 0; m < n1; ++m) qn[m] = __ldcs(g + m * ST);
    }
    double Fv[n1], out[n1];
    if (d == 0) {
#pragma unroll
      for (int m = 0; m < n1; ++m) Fv[m] = fr[m];
    } else {
      const int fq = f == 0 ? 1 + d : f;
      const bool pf = f == 1 + d;  // only this field carries P' (its load is skipped for the others)
#pragma unroll
      for (int m = 0; m < n1; ++m) {
        const double Ud = q[(1 + d) * Np + m * ST];
        const double ud = __dmul_rn(Ud, ax[Np + m * ST]);
        const double pv = pf ? ax[m * ST] : 0.0;
        const double v = __fma_rn(q[fq * Np + m * ST], ud, pv);
        Fv[m] = f == 0 ? Ud : v;
      }
    }
    contract<N>(Fv, out, a);
    const double sc = -sH[elem_level(sD[el].info)][d];
    const double* L = sLift + ((el * NFACE + 2 * d) * F + f) * Nf + p;
    out[0] = __fma_rn(sc, out[0], L[0]);
    out[N] = __fma_rn(sc, out[N], L[F * Nf]);
#pragma unroll
    for (int m = 1; m < N; ++m) out[m] = __fma_rn(sc, out[m], 0.0);
    if (d == 0) {
      if (f == DIM) {  // gravity source -rho' g on the vertical momentum (R5); x pencils are level in z
        const double rb = bg_rt(a.bg4, sD[el].bgrow + (DIM == 3 ? p / n1 : p)).x;
        const double mg = -a.g;
#pragma unroll
        for (int m = 0; m < n1; ++m) out[m] = __fma_rn(mg, __dsub_rn(q[m], rb), out[m]);
      }
#pragma unroll
      for (int m = 0; m < n1; ++m) fr[m] = out[m];
    } else if (!LAST) {
#pragma unroll
      for (int m = 0; m < n1; ++m) fr[m * PST] = __dadd_rn(fr[m * PST], out[m]);
    } else {
      const bool rk = a.mode == 1, s0 = a.stage == 0;
      const double* qf = q + f * Np;
      double* o = a.out + elem_of<LIST>(a, e0 + el) * STR + f * Np + base;
#pragma unroll
      for (int m = 0; m < n1; ++m) {
        const double res = __dadd_rn(fr[m * PST], out[m]);
        double v;
        if (!rk) v = res;
        else if (s0) v = __fma_rn(a.dt, res, qf[m * ST]);
        else v = __fma_rn(a.rk_b, __fma_rn(a.dt, res, __dsub_rn(qf[m * ST], qn[m])), qn[m]);
        o[m * ST] = v;
      }
    }
  }
}

// ------------------------------------------------------------------ generic kernel
template <int DIM, int N, bool LIST>
__global__ void __launch_bounds__(SC<DIM, N>::T, SC<DIM, N>::MINB) k_stage(const __grid_constant__ StageArgs a) {
  using C = SC<DIM, N>;
  constexpr int n1 = C::n1, T = C::T, EPB = C::EPB, STR = C::STR;
  extern __shared__ __align__(128) double smem[];
  double* sQ = smem;
  double* sFR = sQ + C::Q;
  double* sAux = sFR + C::FR;
  double* sTr = sAux + C::AUX;  // traces; lift values overwrite them in place
  double* sMS = sTr + C::TR;    // mortar fluxes of up to MCAP coarse faces
  __shared__ __align__(8) uint64_t mbar;
  __shared__ __align__(16) ElemDesc sDesc[2][EPB];
  __shared__ __align__(16) int sNbr[2][EPB * 8];  // background row across each face
  __shared__ __align__(16) double sBg[2][EPB * C::BGE];  // per element: own rows 0..N, -z and +z neighbour rows
  __shared__ double sH[kMaxLevel + 1][3];
  __shared__ double sPR[4 * n1 * n1];  // P_lo, P_hi, R_lo, R_hi
  __shared__ uint8_t sLst[2][2][EPB * C::NFACE];  // coarse / fine face slot lists per descriptor buffer
  const double* sP = sPR;
  const double* sR = sPR + 2 * n1 * n1;

  const int tid = threadIdx.x;
  const int64_t n_tiles = (a.n_elem + EPB - 1) / EPB;
  int64_t tile = blockIdx.x;
  if (tile >= n_tiles) return;

  if (tid < (kMaxLevel + 1) * 3) (&sH[0][0])[tid] = a.ops[OpsLayout::H(n1) + tid];
  for (int i = tid; i < 4 * n1 * n1; i += T) sPR[i] = a.ops[OpsLayout::P(n1, 0) + i];
  if (tid == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto tile_n = [&](int64_t t) { return (int)min((int64_t)EPB, a.n_elem - t * EPB); };
  auto load_desc = [&](int64_t t, int buf) {  // asynchronous (cp.async, 16 B)
    for (int i = tid; i < tile_n(t) * 4; i += T) {
      const int k = i >> 1;  // int4 k of the tile's descriptors (element k / 2, half k % 2)
      if (!LIST) {
        if (i & 1)
          cp_async16(reinterpret_cast<int4*>(sNbr[buf]) + k, reinterpret_cast<const int4*>(a.nbrow + t * EPB * 8) + k);
        else
          cp_async16(reinterpret_cast<int4*>(sDesc[buf]) + k, reinterpret_cast<const int4*>(a.desc + t * EPB) + k);
      } else {
        const int64_t r = elem_of<LIST>(a, t * EPB + (k >> 1));
        if (i & 1)
          cp_async16(reinterpret_cast<int4*>(sNbr[buf]) + k, reinterpret_cast<const int4*>(a.nbrow + r * 8) + (k & 1));
        else
          cp_async16(reinterpret_cast<int4*>(sDesc[buf]) + k, reinterpret_cast<const int4*>(a.desc + r) + (k & 1));
      }
    }
  };
  // background rows of the tile in buffer b (needs its descriptors): 32-B rows by 16-B cp.async
  auto load_bg_rows = [&](int64_t t, int b) {
    constexpr int RW = n1 + 2, VF = 2 * (DIM - 1);
    for (int i = tid; i < tile_n(t) * RW * 2; i += T) {
      const int el = i / (RW * 2), r = (i >> 1) - el * RW;
      const int own = sDesc[b][el].bgrow;
      int row;
      if (r <= N) row = own + r;
      else if (r == N + 1) row = sNbr[b][el * 8 + VF] >= 0 ? sNbr[b][el * 8 + VF] + N : own;
      else row = sNbr[b][el * 8 + VF + 1] >= 0 ? sNbr[b][el * 8 + VF + 1] : own + N;
      cp_async16(reinterpret_cast<double2*>(sBg[b]) + i, reinterpret_cast<const double2*>(a.bg4) + 2 * row + (i & 1));
    }
  };
  load_desc(tile, 0);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  load_bg_rows(tile, 0);
  cp_async_commit();
  if (tid < 32) build_lists<C>(sDesc[0], tile_n(tile), sLst[0][0], sLst[0][1]);

  const bool need_qn = a.mode == 1 && a.stage > 0;
  for (int it = 0; tile < n_tiles; ++it, tile += gridDim.x) {
    const int cur = it & 1, nxt = cur ^ 1;
    const int ne = tile_n(tile);
    const int64_t e0 = tile * EPB;
    const int64_t tnext = tile + gridDim.x;
    const bool has_next = tnext < n_tiles;
    const ElemDesc* sD = sDesc[cur];
    if (tid == 0) {  // this tile's rows (bulk); next tile's rows and this tile's q_n into L2
      const uint32_t bytes = (uint32_t)(ne * STR * 8);
      fence_proxy_async();
      mbar_expect_tx(&mbar, bytes);
      if (!LIST) {
        bulk_g2s(sQ, a.q_in + e0 * STR, bytes, &mbar);
        if (has_next) prefetch_l2(a.q_in + tnext * EPB * STR, (uint32_t)(tile_n(tnext) * STR * 8));
        if (need_qn) prefetch_l2(a.q_n + e0 * STR, bytes);
      } else {  // element list: row by row
        for (int el = 0; el < ne; ++el) {
          const int64_t r = elem_of<LIST>(a, e0 + el);
          bulk_g2s(sQ + el * STR, a.q_in + r * STR, STR * 8, &mbar);
          if (need_qn) prefetch_l2(a.q_n + r * STR, STR * 8);
        }
      }
    }
    issue_traces<C>(a, sD, ne, sTr);
    if (has_next) load_desc(tnext, nxt);
    cp_async_commit();
    cp_async_wait_1();  // this tile's background rows (committed one group earlier)
    mbar_wait(&mbar, it & 1);
    __syncthreads();

    int n_coarse = 0, n_fine = 0;
    for (int e = 0; e < ne; ++e) {
      n_coarse += n_coarse_faces(sD[e].info);
      n_fine += n_fine_faces(sD[e].info);
    }
    const bool pw = a.ncmode != 0;  // NEXT-3 pointwise baseline instead of mortars
    const bool few_coarse = !pw && n_coarse > 0 && n_coarse <= C::MCAP;
    const uint8_t* cl = sLst[cur][0];
    if (!pw && n_coarse > C::MCAP) mort_chunks_fact<C>(a, sQ, sD, cl, n_coarse, sMS, sTr, sP, sR, sH);
    node_phase<C>(a, sQ, sD, ne, sAux, sFR, sBg[cur]);
    if (few_coarse) mort_A<C>(a, sQ, sD, cl, 0, n_coarse, sMS, sP);
    cp_async_wait_all();
    __syncthreads();
    if (has_next) {
      load_bg_rows(tnext, nxt);
      if (tid < 32) build_lists<C>(sDesc[nxt], tile_n(tnext), sLst[nxt][0], sLst[nxt][1]);
    }
    cp_async_commit();
    // AMR tiles: the remaining mortar steps, interleaved so they share barriers (R35)
    if (few_coarse || n_fine > 0)
      amr_mid<C>(a, sQ, sD, sNbr[cur], cl, sLst[cur][1], few_coarse ? n_coarse : 0, n_fine, sMS, sTr, sP, sR, sH);
    face_phase<C>(a, sQ, sAux, sD, sNbr[cur], ne, sTr, sH, sBg[cur]);
    if (DIM == 3 && few_coarse) {
      __syncthreads();
      mort_E<C>(a, sQ, sD, cl, 0, n_coarse, sMS, sR, sH, sTr);
    }
    if (pw && n_coarse > 0) point_coarse<C>(a, sQ, sD, cl, n_coarse, sH, sTr);
    __syncthreads();

    axis_pass<DIM, N, 0, LIST>(a, sQ, sAux, sFR, sTr, sD, sH, ne, e0);
    __syncthreads();
    if (DIM == 3) {
      axis_pass<DIM, N, 1, LIST>(a, sQ, sAux, sFR, sTr, sD, sH, ne, e0);
      __syncthreads();
    }
    axis_pass<DIM, N, DIM - 1, LIST>(a, sQ, sAux, sFR, sTr, sD, sH, ne, e0);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ 3D, N = 7 kernel
// Plane-per-warp layout (S7): warp w owns plane k = w, lane l = 4 g + c the nodes
// (i = 2c + s, j = g, k = w), s = 0, 1.  All three volume contractions run on the FP64
// tensor cores as DMMA m8n8k4 (fragments, PTX .f64: lane l holds A[l/4][l%4], B[l%4][l/4],
// C[l/4][2(l%4) + {0,1}]):
//   x (transposed form)  Out^T[j][i] = sum_m F^x[j][m] D[i][m]:  A = F^x at the lane's own
//       nodes (m = 2c + s in DMMA s), B[c][g] = D[g][2c + s], C = the lane's own nodes;
//   y (plain form)       Out[j][i] = sum_m D[j][m] F^y[m][i]:     A[g][c] = D[g][c + 4s],
//       B[c][g] = F^y(i = g, j = c + 4s) (a warp-local transpose through shared memory),
//       C = the lane's own nodes again -- x and y accumulate in the same registers;
//   z (transposed form, warp v takes the z pencils (i = g, j = v)): A = F^z(i = g, j = v,
//       k = c + 4s), B[c][g] = D[nu(g)][c + 4s] with nu(g) = g/2 + 4(g%2), C = k = c, c + 4;
//       F^z comes from and the results go back to the plane owners through shared memory.
// The derivative scale -2/h_d is folded into the D fragments.

// F^z / z-result buffer (and, per plane, the y staging): field f, node (i, j, k) at
// f Np + zidx(i, j, k).  Pairs (i, i+1), i even, stay 16-B aligned; a quarter warp's 16-B
// owner stores, and a half warp's 8-B z-pass loads/stores (i = g, k = c (+4)), touch 16
// distinct doubles (bank-conflict free).
__device__ __forceinline__ int h7_zidx(int i, int j, int k) {
  return 64 * k + 16 * (j >> 1) + ((i + 8 * (j & 1)) ^ (4 * (k & 3)));
}
// y staging inside plane w's region: owner 16-B stores of (i = 2c, 2c+1; j = g) and the
// transposed 8-B loads (i = g, j = c (+4)) are both conflict free.
__device__ __forceinline__ int h7_yidx(int i, int j) { return 16 * (j >> 1) + ((i + 8 * (j & 1)) ^ (4 * ((j >> 1) & 1))); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Face node (face, t) of an element whose six faces are all conforming or wall (the uniform
// fast path; 2:1 faces go through face_phase): Rusanov (A5, A6) and the lift value (A8)
// written over the trace slot.  The axis d = face / 2 is a compile-time constant (warp-
// uniform at the call), so the flux components need no runtime selects; the arithmetic is
// that of face_phase (bitwise the same fluxes as the neighbour computes).
template <int d>
__device__ __forceinline__ void h7_face_node(const StageArgs& a, const double* __restrict__ sQ,
                                             const double* __restrict__ sAux, const double* __restrict__ sBgE,
                                             double* __restrict__ sTr, int face, int t, int kind, double cf) {
  constexpr int Np = 512, Nf = 64, F = 5;
  const int e7 = (face & 1) * 7, t1 = t & 7, t2 = t >> 3;
  const int n = d == 0 ? e7 + 8 * t1 + 64 * t2 : (d == 1 ? t1 + 8 * e7 + 64 * t2 : t1 + 8 * t2 + 64 * e7);
  const int k = d == 2 ? e7 : t2;  // vertical index of the own node
  DG_CHECK(n >= 0 && n < Np && t >= 0 && t < Nf && face >= 0 && face < 6 && k >= 0 && k < 8);
  const double sgn = (face & 1) ? 1.0 : -1.0;
  St own;
  {
    const double2 b0 = reinterpret_cast<const double2*>(sBgE)[2 * k];
    const double2 b1 = reinterpret_cast<const double2*>(sBgE)[2 * k + 1];
    own.rb = b0.x;
    own.Tb = b0.y;
    own.Pb = b1.x;
    own.rTb = b1.y;
  }
  own.rp = __dsub_rn(sQ[n], own.rb);
  own.U[0] = sQ[Np + n];
  own.U[1] = sQ[2 * Np + n];
  own.U[2] = sQ[3 * Np + n];
  own.Tp = __dsub_rn(sQ[4 * Np + n], own.Tb);
  Dv vo;
  vo.rho = __dadd_rn(own.rb, own.rp);
  vo.Th = __dadd_rn(own.Tb, own.Tp);
  vo.Pp = sAux[S7::axi(n)];
  vo.rinv = sAux[Np + S7::axi(n)];
  double* tr = sTr + face * F * Nf + t;
  double Fs[F], Fo[F];
  if (kind == kWall) {
    St R = own;  // mirror ghost (R9)
    R.U[d] = -own.U[d];
    rusanov<3>(own, vo, R, vo, d, sgn, a.gamma, Fs, Fo);
  } else {
    St R;
    if (d < 2) {  // same level, same height: the neighbour's background row is the own one
      R.rb = own.rb;
      R.Tb = own.Tb;
      R.Pb = own.Pb;
      R.rTb = own.rTb;
    } else {      // staged rows 8 (-z) and 9 (+z)
      const double2 b0 = reinterpret_cast<const double2*>(sBgE)[2 * (8 + (face & 1))];
      const double2 b1 = reinterpret_cast<const double2*>(sBgE)[2 * (8 + (face & 1)) + 1];
      R.rb = b0.x;
      R.Tb = b0.y;
      R.Pb = b1.x;
      R.rTb = b1.y;
    }
    R.rp = __dsub_rn(tr[0], R.rb);
    R.U[0] = tr[Nf];
    R.U[1] = tr[2 * Nf];
    R.U[2] = tr[3 * Nf];
    R.Tp = __dsub_rn(tr[4 * Nf], R.Tb);
    rusanov<3>(own, vo, R, derive(R, a), d, sgn, a.gamma, Fs, Fo);
  }
#pragma unroll
  for (int f = 0; f < F; ++f) tr[f * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[f], Fs[f]));
}

// All 384 face nodes of an all-conforming/wall element: round 0 = faces 0..3 (one item per
// thread, axis warp-uniform), round 1 = faces 4, 5 on warps 0..3.
__device__ __forceinline__ void h7_faces_fast(const StageArgs& a, const double* sQ, const double* sAux,
                                              const double* sBgE, double* sTr, int info, const double* sHl) {
  const int i = threadIdx.x;
  const double w0 = a.w0inv;
  {
    const int face = i >> 6, t = i & 63;
    const int kind = face_kind(info, face);
    if (face < 2) h7_face_node<0>(a, sQ, sAux, sBgE, sTr, face, t, kind, __dmul_rn(-sHl[0], w0));
    else h7_face_node<1>(a, sQ, sAux, sBgE, sTr, face, t, kind, __dmul_rn(-sHl[1], w0));
  }
  if (i < 128) {
    const int face = 4 + (i >> 6), t = i & 63;
    h7_face_node<2>(a, sQ, sAux, sBgE, sTr, face, t, face_kind(info, face), __dmul_rn(-sHl[2], w0));
  }
}

#ifdef DG_TIMELINE
// debug timeline: for the CTAs resident on SM 0, every warp's clock64 at each phase mark of
// iterations [kTlIt0, kTlIt0 + kTlIts): [slot 0/1][iteration][warp][mark]
constexpr int kTlIt0 = 20, kTlIts = 6, kTlMarks = 8;
__device__ long long g_tl[2][kTlIts][8][kTlMarks];
__device__ int g_tl_slot;
#endif

template <int KIND, bool LIST>  // KIND 0: RHS, 1: RK stage 0, 2: RK stage 1 or 2; LIST: element-list launch
__global__ void __launch_bounds__(S7::T, S7::MINB) k_stage_h7(const __grid_constant__ StageArgs a) {
  using C = S7;
#ifdef DG_PHASE_PROF  // debug phase clocks (env DG_PHASE_PROF=1 + this build): lane 0 of warp 0 into slots 0..7,
                      // of warp 7 into 8..15 (compiled out otherwise: 2 % of the instructions)
  const bool prof = a.prof != nullptr && (threadIdx.x == 0 || threadIdx.x == 224);
  long long pt = prof ? clock64() : 0;
#endif
#ifdef DG_TIMELINE
  __shared__ int tl_slot;
  if (threadIdx.x == 0) {
    unsigned sm;
    asm("mov.u32 %0, %%smid;" : "=r"(sm));
    tl_slot = sm == 0 ? atomicAdd(&g_tl_slot, 1) : -1;
  }
  __syncthreads();
  int tl_it = 0;
#endif
  auto PROF = [&](int k) {
#ifdef DG_TIMELINE
    if ((threadIdx.x & 31) == 0 && tl_slot >= 0 && tl_slot < 2 && tl_it >= kTlIt0 && tl_it < kTlIt0 + kTlIts)
      g_tl[tl_slot][tl_it - kTlIt0][threadIdx.x >> 5][k] = clock64();
#endif
#ifdef DG_PHASE_PROF
    if (prof) {
      const long long t = clock64();
      atomicAdd(a.prof + k + (threadIdx.x ? 8 : 0), (unsigned long long)(t - pt));
      pt = t;
    }
#else
    (void)k;
#endif
  };
  constexpr int n1 = 8, Np = 512, F = 5, Nf = 64, STR = C::STR;
  extern __shared__ __align__(128) double smem[];
  double* sQb = smem;                    // [2][STR] element rows (bulk copies)
  double* sTrb = sQb + 2 * C::Q;         // [2][TR] neighbour traces -> lift values
  double* sAux = sTrb + 2 * C::TR;       // P', 1/rho
  double* sZ = sAux + C::AUX;            // y staging, F^z, z results; mortar scratch
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(16) ElemDesc sDesc[3];
  __shared__ __align__(16) int sNbr[3][8];
  __shared__ __align__(16) double sBg[2][10 * 4];  // own rows k = 0..7, -z neighbour row, +z neighbour row
  __shared__ double sH[kMaxLevel + 1][3];
  __shared__ double sPR[4 * n1 * n1];
#ifdef DG_EPI_BF
  __shared__ __align__(16) double sZero[F * Nf];
  for (int i = threadIdx.x; i < F * Nf; i += C::T) sZero[i] = 0.0;
#endif
  const double* sP = sPR;
  const double* sR = sPR + 2 * n1 * n1;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int64_t n_el = a.n_elem;
  int64_t e = blockIdx.x;
  if (e >= n_el) return;

  // descriptor + face rows of element t into ring slot r (cp.async; 4 x 16 B)
  auto load_desc = [&](int64_t t, int r) {
    if (tid < 2)
      cp_async16(reinterpret_cast<int4*>(&sDesc[r]) + tid, reinterpret_cast<const int4*>(a.desc + elem_of<LIST>(a, t)) + tid);
    else if (tid < 4)
      cp_async16(reinterpret_cast<int4*>(sNbr[r]) + (tid - 2), reinterpret_cast<const int4*>(a.nbrow + elem_of<LIST>(a, t) * 8) + (tid - 2));
  };
  // element t (descriptor in ring slot r) into buffer b: the state row and the 10 background rows
  // (own rows 0..7, the -z and +z neighbour rows) by bulk copies completing on mbar[b] (the
  // neighbour traces follow at the end of the iteration, below)
  auto issue_elem = [&](int64_t t, int r, int b) {

    if (tid == 0) {
      const int own = sDesc[r].bgrow;
      const int rm = sNbr[r][4] >= 0 ? sNbr[r][4] + 7 : own, rp = sNbr[r][5] >= 0 ? sNbr[r][5] : own + 7;
      fence_proxy_async();
      mbar_expect_tx(&mbar[b], STR * 8 + 10 * 32);
      bulk_g2s(sQb + b * C::Q, a.q_in + elem_of<LIST>(a, t) * STR, STR * 8, &mbar[b]);
      bulk_g2s(sBg[b], a.bg4 + 4 * (int64_t)own, 8 * 32, &mbar[b]);
      bulk_g2s(sBg[b] + 32, a.bg4 + 4 * (int64_t)rm, 32, &mbar[b]);
      bulk_g2s(sBg[b] + 36, a.bg4 + 4 * (int64_t)rp, 32, &mbar[b]);
    }
  };

  if (tid < (kMaxLevel + 1) * 3) (&sH[0][0])[tid] = a.ops[OpsLayout::H(n1) + tid];
  for (int i = tid; i < 4 * n1 * n1; i += C::T) sPR[i] = a.ops[OpsLayout::P(n1, 0) + i];
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // unscaled D fragments (read per element from L1, not held across the loop): x B (D[g][2c + s]),
  // y A (D[g][c + 4s]), z B (D[nu(g)][c + 4s])
#ifdef DG_DM_GLOBAL
  const double* Dm = a.ops + OpsLayout::kD;
#define DG_DM(i) __ldg(Dm + (i))
#else  // D staged once in shared memory (the per-element __ldg reads were 6 % of the stall samples)
  __shared__ double sDm[64];
  for (int i = threadIdx.x; i < 64; i += C::T) sDm[i] = a.ops[OpsLayout::kD + i];
#define DG_DM(i) sDm[i]
#endif
  const int nu = (g >> 1) + 4 * (g & 1);
  load_desc(e, 0);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  if (e + gridDim.x < n_el) load_desc(e + gridDim.x, 1);
  cp_async_commit();
  cp_async_wait_all();
  issue_elem(e, 0, 0);
  __syncthreads();

  constexpr bool rk = KIND != 0, s0 = KIND == 1;
  const int n0 = 2 * c + 8 * g + 64 * w;  // the lane's first node (the second is n0 + 1)
#ifdef DG_DM_NOHOLD
  constexpr bool hold = false;
#else
  constexpr bool hold = KIND != 2;
#endif
  int lev_c = -1;
  double bx0 = 0, bx1 = 0, ay0 = 0, ay1 = 0, bz0 = 0, bz1 = 0;
  for (int it = 0; e < n_el; ++it, e += gridDim.x) {
    const int b = it & 1, r = it % 3;
    const int64_t en = e + gridDim.x, enn = en + gridDim.x;
    double* sQ = sQb + b * C::Q;
    double* sTr = sTrb + b * C::TR;
    const ElemDesc* sD = &sDesc[r];
    const int64_t er = elem_of<LIST>(a, e);  // this element's local row
    if (tid == 0 && rk && !s0) prefetch_l2(a.q_n + er * STR, STR * 8);
#ifdef DG_NBR_PF
    // the next element's face neighbours later in the order (their traces would otherwise be read from
    // DRAM sector by sector before their rows are loaded): whole rows into L2, one element ahead
    if (tid < 6 && en < n_el) {
      const ElemDesc& Dn = sDesc[(it + 1) % 3];
      const int nb = Dn.nbr[tid];
      if (face_kind(Dn.info, tid) == kConf && nb > elem_of<LIST>(a, en)) prefetch_l2(a.q_in + (int64_t)nb * STR, STR * 8);
    }
#endif
    PROF(0);
    mbar_wait(&mbar[b], (it >> 1) & 1);
    PROF(1);

    const int info = sD->info;
    const int lev = elem_level(info);
    const int n_coarse = n_coarse_faces(info), n_fine = n_fine_faces(info);
    // coarse side of 2:1 faces: mortar fluxes and lifts into the lift slots (scratch sZ, which
    // other warps may still read for the previous element: barrier first)
    if (n_coarse > 0) {
      __syncthreads();
      mortar_chunks<C>(a, sQ, sD, 1, n_coarse, sZ, sTr, sP, sR, sH);
    }

    // ---- own nodes: EOS (A1), fluxes (A2), x and y contractions (A3) in registers
    const double* bgk = sBg[b] + 4 * w;  // background row of plane k = w
    const double rb = bgk[0], Tb = bgk[1], Pb = bgk[2], rTb = bgk[3];
    double q[F][2];
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const double2 v = *reinterpret_cast<const double2*>(sQ + f * Np + n0);
      q[f][0] = v.x;
      q[f][1] = v.y;
    }
    // this element's neighbour traces (cp.async), queued behind the state loads above: 1.7 % faster
    // than issuing them at the end of the previous element (there they delayed these loads) and
    // 7 % faster than beside the next element's bulk copies after barrier 1 (in front of the z pass
    // and face loads); waited for by cp_async_wait_all before barrier 1, which makes them visible.
    // (Bulk copies for the contiguous y / z runs measured 4 % slower.)
#if !defined(DG_TR_AFTER_X) && !defined(DG_TR_AFTER_Y)
    issue_traces_h7(a, *sD, sTr);
    cp_async_commit();
#endif
    double Pp[2], ri[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      St st;
      st.rb = rb;
      st.Tb = Tb;
      st.Pb = Pb;
      st.rTb = rTb;
      st.rp = __dsub_rn(q[0][s], rb);
      st.U[0] = q[1][s];
      st.U[1] = q[2][s];
      st.U[2] = q[3][s];
      st.Tp = __dsub_rn(q[4][s], Tb);
      const Dv v = derive(st, a);  // the same arithmetic as a neighbour's recomputation (bitwise)
      Pp[s] = v.Pp;
      ri[s] = v.rinv;
    }
    *reinterpret_cast<double2*>(sAux + C::axi(n0)) = make_double2(Pp[0], Pp[1]);
    *reinterpret_cast<double2*>(sAux + Np + C::axi(n0)) = make_double2(ri[0], ri[1]);

    // scaled D fragments: RHS / stage 0 keep them in registers while the level does not change (12
    // registers; stage 0 -2 %), stages 1 / 2 (q_n in registers later on) reload them per element (+3.5 % held)
    if (!hold || lev != lev_c) {
      const double sx = -sH[lev][0], sy = -sH[lev][1], sz = -sH[lev][2];
      bx0 = __dmul_rn(sx, DG_DM(g * 8 + 2 * c)), bx1 = __dmul_rn(sx, DG_DM(g * 8 + 2 * c + 1));
      ay0 = __dmul_rn(sy, DG_DM(g * 8 + c)), ay1 = __dmul_rn(sy, DG_DM(g * 8 + c + 4));
      if (hold) bz0 = __dmul_rn(sz, DG_DM(nu * 8 + c)), bz1 = __dmul_rn(sz, DG_DM(nu * 8 + c + 4));
      lev_c = lev;
    }
    double res[F][2];
    // x pass; the accumulator starts from the gravity source -rho' g on the vertical momentum (R5)
    {
      const double mg = -a.g;
      double ud[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) ud[s] = __dmul_rn(q[1][s], ri[s]);
#pragma unroll
      for (int f = 0; f < F; ++f) {
        res[f][0] = f == 3 ? __dmul_rn(mg, __dsub_rn(q[0][0], rb)) : 0.0;
        res[f][1] = f == 3 ? __dmul_rn(mg, __dsub_rn(q[0][1], rb)) : 0.0;
        double Fv[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) Fv[s] = f == 0 ? q[1][s] : __fma_rn(q[f][s], ud[s], f == 1 ? Pp[s] : 0.0);
        dmma(res[f][0], res[f][1], Fv[0], bx0);
        dmma(res[f][0], res[f][1], Fv[1], bx1);
      }
    }
#ifdef DG_TR_AFTER_X
    issue_traces_h7(a, *sD, sTr);
    cp_async_commit();
#endif
    // y pass: F^y at the own nodes -> plane w's staging region -> transposed B fragments
    double* zp = sZ + 64 * w;
    {
      double ud[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) ud[s] = __dmul_rn(q[2][s], ri[s]);
      const int yo = h7_yidx(2 * c, g);
      DG_CHECK(yo >= 0 && yo + 1 < 64 && (yo & 1) == 0 && h7_yidx(g, c) < 64 && h7_yidx(g, c + 4) < 64);
#pragma unroll
      for (int f = 0; f < F; ++f) {
        double Fv[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) Fv[s] = f == 0 ? q[2][s] : __fma_rn(q[f][s], ud[s], f == 2 ? Pp[s] : 0.0);
        *reinterpret_cast<double2*>(zp + f * Np + yo) = make_double2(Fv[0], Fv[1]);
      }
      __syncwarp();
      const int yi0 = h7_yidx(g, c), yi1 = h7_yidx(g, c + 4);
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const double b0 = zp[f * Np + yi0], b1 = zp[f * Np + yi1];
        dmma(res[f][0], res[f][1], ay0, b0);
        dmma(res[f][0], res[f][1], ay1, b1);
      }
      __syncwarp();
    }
#ifdef DG_TR_AFTER_Y
    issue_traces_h7(a, *sD, sTr);
    cp_async_commit();
#endif
    // F^z at the own nodes for the z pass
    {
      double ud[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) ud[s] = __dmul_rn(q[3][s], ri[s]);
      const int zo = h7_zidx(2 * c, g, w) - 64 * w;
      DG_CHECK(zo >= 0 && zo + 1 < 64 && (zo & 1) == 0);
#pragma unroll
      for (int f = 0; f < F; ++f) {
        double Fv[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) Fv[s] = f == 0 ? q[3][s] : __fma_rn(q[f][s], ud[s], f == 3 ? Pp[s] : 0.0);
        *reinterpret_cast<double2*>(zp + f * Np + zo) = make_double2(Fv[0], Fv[1]);
      }
    }
    PROF(2);
    cp_async_wait_all();  // this element's traces and the descriptor load of the element after next
    __syncthreads();
    PROF(3);
    // the next element's rows, traces and background, and the descriptor of the one after, in
    // flight while this element's faces and epilogue run (buffers b ^ 1 and the ring slot of the
    // previous element are free: every warp has passed this barrier)
    if (en < n_el) issue_elem(en, (it + 1) % 3, b ^ 1);
    if (enn < n_el) load_desc(enn, (it + 2) % 3);
    cp_async_commit();

    // ---- z pass (z pencils (i = g, j): results in place, the positions the lane read) and faces
    if (!hold) {
      const double sz = -sH[lev][2];
      bz0 = __dmul_rn(sz, DG_DM(nu * 8 + c)), bz1 = __dmul_rn(sz, DG_DM(nu * 8 + c + 4));
    }
    auto zpass = [&](int j) {
      const int za0 = h7_zidx(g, j, c), za1 = h7_zidx(g, j, c + 4);
      DG_CHECK(za0 >= 0 && za0 < Np && za1 >= 0 && za1 < Np && (za0 >> 6) == c && (za1 >> 6) == c + 4);
      double A0[F], A1[F];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        A0[f] = sZ[f * Np + za0];
        A1[f] = sZ[f * Np + za1];
      }
#pragma unroll
      for (int f = 0; f < F; ++f) {
        double c0 = 0.0, c1 = 0.0;
        dmma(c0, c1, A0[f], bz0);
        dmma(c0, c1, A1[f], bz1);
        sZ[f * Np + za0] = c0;  // (i = g, j, k = nu(2c) = c)
        sZ[f * Np + za1] = c1;  // (k = nu(2c + 1) = c + 4)
      }
    };
    PROF(4);
    const bool fast = n_fine == 0 && n_coarse == 0;
#ifdef DG_ZBAL  // (measured: 1.5 % faster alone, 0.6 % slower together with the early q_n loads)
    if (fast && KIND != 2) {
      // uniform elements: 384 face nodes + 8 z-pass units over 8 warps -- warps 0..3 take the faces
      // x+-, y+- (one node per lane) and then the z faces, warps 4..7 two z units each and then
      // the faces x+-, y+- of the remaining half
      const int i = threadIdx.x, face = i >> 6, t = i & 63;
      const double w0 = a.w0inv;
      if (w >= 4) {
        zpass(w - 4);
        zpass(w);
      }
      if (face < 2) h7_face_node<0>(a, sQ, sAux, sBg[b], sTr, face, t, face_kind(info, face), __dmul_rn(-sH[lev][0], w0));
      else h7_face_node<1>(a, sQ, sAux, sBg[b], sTr, face, t, face_kind(info, face), __dmul_rn(-sH[lev][1], w0));
      if (w < 4) {
        const int fz = 4 + (i >> 6);
        h7_face_node<2>(a, sQ, sAux, sBg[b], sTr, fz, i & 63, face_kind(info, fz), __dmul_rn(-sH[lev][2], w0));
      }
    } else
#endif
    {
      zpass(w);
      if (n_fine > 0) fine_phase_inplace<C>(a, sD, sNbr[r], 1, sTr, sP);  // (has its own barrier)
      if (fast) h7_faces_fast(a, sQ, sAux, sBg[b], sTr, info, sH[lev]);
      else face_phase<C>(a, sQ, sAux, sD, sNbr[r], 1, sTr, sH, sBg[b]);
    }
    PROF(5);
    // q_n rows of the own nodes (RK stages 1, 2), read once (evict-first): in flight over barrier 2
    // (3 % faster than at the epilogue start; before the face phase they cost spills)
    double qn[F][2];
    if (rk && !s0) {
      const double* gq = a.q_n + er * STR + n0;
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(gq + f * Np));
        qn[f][0] = v.x;
        qn[f][1] = v.y;
      }
    }
    __syncthreads();
    PROF(6);

    // ---- epilogue: + z contribution + lifts (A8), RK update (A9), coalesced 16-B stores

    {
      const double2* zr = reinterpret_cast<const double2*>(sZ + h7_zidx(2 * c, g, w));
      const bool fx0 = c == 0, fx1 = c == 3, fy = g == 0 || g == 7, fz = w == 0 || w == 7;
      const double* lx = sTr + (fx0 ? 0 : 1) * F * Nf + g + 8 * w;                 // x faces: t = j + 8k
      const double* ly = sTr + (g == 0 ? 2 : 3) * F * Nf + 2 * c + 8 * w;         // y faces: t = i + 8k
      const double* lz = sTr + (w == 0 ? 4 : 5) * F * Nf + 2 * c + 8 * g;         // z faces: t = i + 8j
#ifdef DG_EPI_BF
      const double* lx0b = fx0 ? lx : sZero;
      const double* lx1b = fx1 ? lx : sZero;
      const double* lyb = fy ? ly : sZero;
#endif
      double* og = a.out + er * STR + n0;
      // RHS and stage 0: every lift value of the lane loaded first (predicated), then the dependent
      // chains (stage 0 -3 %); stages 1, 2 hold q_n in registers and keep the loads in the chains
      constexpr bool epi2 = KIND != 2;
      double Lx[F], Ly0[F], Ly1[F], Lz0[F], Lz1[F];
      if (epi2) {
#pragma unroll
        for (int f = 0; f < F; ++f) {
          Lx[f] = (fx0 || fx1) ? lx[f * Nf] : 0.0;
          const double2 yl = fy ? *reinterpret_cast<const double2*>(ly + f * Nf) : make_double2(0.0, 0.0);
          const double2 zl = fz ? *reinterpret_cast<const double2*>(lz + f * Nf) : make_double2(0.0, 0.0);
          Ly0[f] = yl.x;
          Ly1[f] = yl.y;
          Lz0[f] = zl.x;
          Lz1[f] = zl.y;
        }
      }
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const double2 qi = *reinterpret_cast<const double2*>(sQ + f * Np + n0);  // q_in, reloaded (registers)
        const double2 z = zr[f * (Np / 2)];
        double v0 = __dadd_rn(res[f][0], z.x), v1 = __dadd_rn(res[f][1], z.y);
        if (epi2) {
          if (fx0) v0 = __dadd_rn(v0, Lx[f]);
          if (fx1) v1 = __dadd_rn(v1, Lx[f]);
          if (fy) {
            v0 = __dadd_rn(v0, Ly0[f]);
            v1 = __dadd_rn(v1, Ly1[f]);
          }
          if (fz) {
            v0 = __dadd_rn(v0, Lz0[f]);
            v1 = __dadd_rn(v1, Lz1[f]);
          }
        } else {
#ifndef DG_EPI_BF
          if (fx0) v0 = __dadd_rn(v0, lx[f * Nf]);
          if (fx1) v1 = __dadd_rn(v1, lx[f * Nf]);
          if (fy) {
            const double2 yl = *reinterpret_cast<const double2*>(ly + f * Nf);
            v0 = __dadd_rn(v0, yl.x);
            v1 = __dadd_rn(v1, yl.y);
          }
#else
          {  // branch free: lanes on no such face read the zero block (+0 leaves the value unchanged)
            const double2 yl = *reinterpret_cast<const double2*>(lyb + f * Nf);
            v0 = __dadd_rn(__dadd_rn(v0, lx0b[f * Nf]), yl.x);
            v1 = __dadd_rn(__dadd_rn(v1, lx1b[f * Nf]), yl.y);
          }
#endif
          if (fz) {
            const double2 zl = *reinterpret_cast<const double2*>(lz + f * Nf);
            v0 = __dadd_rn(v0, zl.x);
            v1 = __dadd_rn(v1, zl.y);
          }
        }
        double o0, o1;
        if (!rk) {
          o0 = v0;
          o1 = v1;
        } else if (s0) {
          o0 = __fma_rn(a.dt, v0, qi.x);
          o1 = __fma_rn(a.dt, v1, qi.y);
        } else {
          o0 = __fma_rn(a.rk_b, __fma_rn(a.dt, v0, __dsub_rn(qi.x, qn[f][0])), qn[f][0]);
          o1 = __fma_rn(a.rk_b, __fma_rn(a.dt, v1, __dsub_rn(qi.y, qn[f][1])), qn[f][1]);
        }
        __stcs(reinterpret_cast<double2*>(og + f * Np), make_double2(o0, o1));
      }
    }
    PROF(7);
#ifdef DG_TIMELINE
    ++tl_it;
#endif
  }
}

// ------------------------------------------------------------------ launch

template <int DIM, int N, bool LIST>
int launch_stage_l(const StageArgs& a, cudaStream_t s) {
  if (DIM == 3 && N == 7 && a.ncmode == 0) {  // (the pointwise baseline runs on the generic kernel)
    static LaunchCache cache[3];
    const int kind = a.mode == 0 ? 0 : (a.stage == 0 ? 1 : 2);
    const size_t bytes = sizeof(double) * S7::SMEM;
    if (kind == 0) return launch_persistent(k_stage_h7<0, LIST>, a, S7::T, bytes, a.n_elem, s, cache[0]);
    if (kind == 1) return launch_persistent(k_stage_h7<1, LIST>, a, S7::T, bytes, a.n_elem, s, cache[1]);
    return launch_persistent(k_stage_h7<2, LIST>, a, S7::T, bytes, a.n_elem, s, cache[2]);
  }
#ifndef DG_NO_H4
  // 3D N = 4 meshes without 2:1 faces: the warp-per-element kernel (c3, c5n4: 1.2-1.3x faster);
  // with 2:1 faces the generic kernel's tile-parallel mortar steps win (c4) unless
  // the context forces k_stage_h4 (env DG_H4_AMR=1 at dg_create: a.amr = 0)
  if (DIM == 3 && N == 4 && a.ncmode == 0 && a.amr == 0) return launch_stage_h4(a, s);  // (incl. the pre-pass mode)
#endif
  using C = SC<DIM, N>;
  static LaunchCache cache;
  return launch_persistent(k_stage<DIM, N, LIST>, a, C::T, sizeof(double) * C::SMEM, (a.n_elem + C::EPB - 1) / C::EPB,
                           s, cache);
}
template <int DIM, int N>
int launch_stage_t(const StageArgs& a, cudaStream_t s) {
  return a.list ? launch_stage_l<DIM, N, true>(a, s) : launch_stage_l<DIM, N, false>(a, s);
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

#ifdef DG_TIMELINE
int debug_timeline(long long* out, int n) {
  cudaDeviceSynchronize();
  const int want = (int)(sizeof(g_tl) / sizeof(long long));
  if (n < want) return -want;
  cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl));
  int zero = 0;
  cudaMemcpyToSymbol(g_tl_slot, &zero, sizeof(int));
  return want;
}
#else
int debug_timeline(long long*, int) { return 0; }
#endif

int launch_stage(int dim, int order, const StageArgs& a, void* stream) {
  DG_DISPATCH2(dim, order, (launch_stage_t<D_, N_>(a, (cudaStream_t)stream)));
}

}  // namespace dgi
