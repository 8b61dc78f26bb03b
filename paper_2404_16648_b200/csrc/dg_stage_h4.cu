// dg_stage_h4.cu -- the fused dGSEM right-hand side / SSP-RK3 stage kernel for 3D, N = 4
// (k_stage_h4: c3, c4 with 2:1 mortars, c5n4), rows A1-A9 of SURVEY 8(a).
//
// Method: strong-form dGSEM, Rusanov flux, mortars at
// 2:1 faces, gravity source, SSP-RK3.
// Readings R2-R17, R35 of DESIGN.md section 3; design: DESIGN.md section 6.2.
//
// One WARP per element, no block barriers (a CTA is one warp; 12 resident per SM), persistent
// over the Morton-ordered elements.  Node n = i + 5 j + 25 k (R28).  The element is processed in
// three AXIS PHASES (h4_axis<D>), each on the 25 pencil owners of its axis -- x: lane l owns
// (j, k) = (l % 5, l / 5), y: (i, k), z: (i, j) -- which hold their five nodes of all five fields
// in registers, loaded from the staged row.  A phase does everything of its axis there: EOS (A1),
// the two faces of the axis (A5, A6, A8: the pencil's end nodes are face node t = lane of faces
// 2 D and 2 D + 1, so own state and lift values never leave registers), fluxes (A2), the
// contraction (A3, even-odd DFMA split of D), the source (A4, x phase) and the lifts; the
// residual accumulates through the staging row in place (x writes, y and z add), and the z
// owners finish with the RK update (A9); one bulk copy stores the row.  2:1 faces (A5, A7; R35):
// fine sides project the coarse trace in place in the slot before the phases; coarse sides take
// lift values from the mortar pre-pass k_mortar_h4 (one warp per coarse face, software-pipelined)
// or, -DG_H4_AMR=1, from the inline mortar steps -- the generic kernel's arithmetic, so both sides
// of every 2:1 face agree bitwise.
// Per element: the state row and its 7 background rows by one mbarrier (bulk copies, the next
// row prefetched into L2), the neighbour traces by cp.async (8 B), q_n (stages 1, 2) fields 0..3
// by a bulk copy into the dead x- / y-face slots after the y phase, field 4 by coalesced loads.
// Why this shape: ncu showed the LSU data pipe (shared-memory wavefronts) as the co-limiter of
// the earlier version (67 % busy: per-node EOS table, flux staging for the y / z passes, a
// separate face phase reading the own state and writing lifts); here only the state row, the
// traces and the residual chain go through shared memory (49 %), at the price of evaluating the
// EOS once per axis.  Outputs are bitwise identical to that version (scripts/hash_stage.py).
#include <cuda_runtime.h>

#include "dg_device.cuh"

namespace dgi {
namespace {

struct S4 {
  static constexpr int n1 = 5, Np = 125, Nf = 25, F = 5, NFACE = 6, NSUB = 4, STR = 640;
  static constexpr int TR = NFACE * F * Nf;  // neighbour traces -> lift values (in place)
  static constexpr int SS = STR;             // staging (F^y / F^z), mortar scratch, output row
  static constexpr int BG = 7 * 4;           // own rows k = 0..4, -z neighbour row, +z neighbour row
  // the x- and y-face slots are dead after the y pass (x lifts are formed in registers, y lifts
  // consumed) and take fields 0..QNF-1 of q_n for the epilogue (stages 1, 2)
  static constexpr int OQ = 0, OTR = STR, OS = OTR + TR, OBG = OS + SS;
  static constexpr int QNF = 4;              // q_n fields by one bulk copy (whole 16-B granules)
  static constexpr int SMEM = OBG + BG;  // doubles per warp
  static_assert(OTR % 2 == 0 && QNF * Np <= 4 * F * Nf && (QNF * Np) % 2 == 0, "q_n overlay: 16-B aligned, inside the dead slots");
#ifndef DG_H4_MINB
#define DG_H4_MINB 12
#endif
  static constexpr int MINB = DG_H4_MINB;    // resident warps per SM the register budget is sized for
  // warps (elements in flight) per CTA of the large-mesh launches: the CTA's warps take W consecutive
  // elements and start each one together (see the kernel); small meshes use single-warp CTAs
#ifndef DG_H4_W
#define DG_H4_W 12
#endif
#ifndef DG_H4_W_NC
#define DG_H4_W_NC 6
#endif
  static constexpr int WBIG = DG_H4_W, WBIG_NC = DG_H4_W_NC;
  static constexpr int64_t kBigMesh = 16384;  // elements from which the multi-warp CTAs are used
  static_assert(MINB % WBIG == 0 && MINB % WBIG_NC == 0, "whole CTAs per SM");
  static_assert(OS % 2 == 0 && OBG % 2 == 0, "bulk copy destinations are 16-B aligned");
};

// F^y staging: node (i, j, k) of a field at 25 i + ((j + 5 k + 8 (i & 1)) mod 25).  The x owners'
// stores (lane j + 5 k, fixed i) and the y owners' loads (lane i + 5 k, fixed j) hit distinct
// 8-B bank pairs in each half warp (searched exhaustively; F^z uses the natural order, which has
// the same property for its two patterns).
__device__ __forceinline__ int h4_yidx(int i, int j, int k) {
  const int v = j + 5 * k + 8 * (i & 1);
  return 25 * i + (v >= 25 ? v - 25 : v);
}

// Volume node of face node t = t1 + 5 t2 of local face f (tangential axes ascending; R28).
__device__ __forceinline__ int h4_fnode(int f, int t1, int t2) {
  const int d = f >> 1, e = (f & 1) ? 4 : 0;
  return d == 0 ? e + 5 * t1 + 25 * t2 : (d == 1 ? t1 + 5 * e + 25 * t2 : t1 + 5 * t2 + 25 * e);
}
// vertical index of that node
__device__ __forceinline__ int h4_fvert(int f, int t2) { return (f >> 1) == 2 ? ((f & 1) ? 4 : 0) : t2; }


__device__ __forceinline__ void bg_row(St& s, const double* sBg, int r) {
  const double2 b0 = reinterpret_cast<const double2*>(sBg)[2 * r];
  const double2 b1 = reinterpret_cast<const double2*>(sBg)[2 * r + 1];
  s.rb = b0.x;
  s.Tb = b0.y;
  s.Pb = b1.x;
  s.rTb = b1.y;
}

// out[r] = sum_j M[r][j] in[j], j ascending (M row-major 5 x 5): the generic kernel's apply1d
__device__ __forceinline__ void h4_apply(const double* M, const double* in, double* out) {
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 5; ++j) acc = __fma_rn(M[r * 5 + j], in[j], acc);
    out[r] = acc;
  }
}

// Own state at node n (k = vertical index) from the staged row, with its EOS values: the same
// `derive` as the neighbour's recomputation of this trace and as the volume's (bitwise equal), so no
// per-node P' / 1/rho table goes through shared memory.
__device__ __forceinline__ void h4_own(const StageArgs& a, const double* __restrict__ sQ, const double* sBg, int n, int k,
                                       St& s, Dv& v) {
  bg_row(s, sBg, k);
  s.rp = __dsub_rn(sQ[n], s.rb);
  s.U[0] = sQ[S4::Np + n];
  s.U[1] = sQ[2 * S4::Np + n];
  s.U[2] = sQ[3 * S4::Np + n];
  s.Tp = __dsub_rn(sQ[4 * S4::Np + n], s.Tb);
  v = derive(s, a);
}

// Neighbour state R at face node t of face `face` (axis D) for the unified Rusanov call
// rusanov(own, R, D, sgn):
//   conforming  the neighbour's trace (raw values in the slot) with the neighbour's background
//               (horizontal: this element's row k; vertical: staged rows 5 / 6);
//   fine side   the projected mortar state (perturbation form) with this element's background
//               (R13); the generic kernel's -rusanov(R, own, D, -sgn) is the same value bitwise
//               (swapping the sides and negating sgn negates every rounded operation exactly);
//   wall        the mirror ghost (R9): the own state with U_D negated.
__device__ __forceinline__ void h4_nbr(int D, const double* __restrict__ tr, const double* sBg, const St& own, int kind,
                                       int face, int k, St& R) {
  constexpr int Nf = S4::Nf;
  const bool wall = kind == kWall || kind == kCoarse, conf = kind == kConf;  // (coarse: result unused, benign values)
  if (conf) bg_row(R, sBg, D < 2 ? k : 5 + (face & 1));
  else {
    R.rb = own.rb;
    R.Tb = own.Tb;
    R.Pb = own.Pb;
    R.rTb = own.rTb;
  }
  const double t0 = tr[0], t1 = tr[Nf], t2 = tr[2 * Nf], t3 = tr[3 * Nf], t4 = tr[4 * Nf];
  R.rp = wall ? own.rp : (conf ? __dsub_rn(t0, R.rb) : t0);
  R.Tp = wall ? own.Tp : (conf ? __dsub_rn(t4, R.Tb) : t4);
  R.U[0] = wall ? (D == 0 ? -own.U[0] : own.U[0]) : t1;
  R.U[1] = wall ? (D == 1 ? -own.U[1] : own.U[1]) : t2;
  R.U[2] = wall ? (D == 2 ? -own.U[2] : own.U[2]) : t3;
}

// Fine side of a 2:1 face (R13, R35): the coarse trace in the slot (raw values) becomes the
// mortar state of this element's sub-face, in place: step A along t1 (P_b1, item (f, j2)), step
// B along t2 (P_b2, item (f, t1)) -- the generic kernel's fine_A / fine_B.
__device__ __forceinline__ void h4_fine_body(const StageArgs& a, double* sTr, const double* sP, int face, int sub, int bgc) {
  const int lane = threadIdx.x & 31;
  double* slot = sTr + face * S4::F * S4::Nf;
  const int f = lane / 5, c = lane - 5 * (lane / 5);
  if (lane < 25) {  // A: column j2 = c of field f
    double in[5], out[5];
    double* col = slot + f * 25 + 5 * c;
    const double2 bb = (f == 0 || f == 4) ? bg_rt(a.bg4, bgc + h4_fvert(face ^ 1, c)) : make_double2(0.0, 0.0);
#pragma unroll
    for (int j1 = 0; j1 < 5; ++j1) in[j1] = col[j1];
    if (f == 0 || f == 4) {
#pragma unroll
      for (int j1 = 0; j1 < 5; ++j1) in[j1] = __dsub_rn(in[j1], f == 0 ? bb.x : bb.y);
    }
    h4_apply(sP + (sub & 1) * 25, in, out);
#pragma unroll
    for (int t1 = 0; t1 < 5; ++t1) col[t1] = out[t1];
  }
  __syncwarp();
  if (lane < 25) {  // B: row t1 = c of field f
    double in[5], out[5];
    double* row = slot + f * 25 + c;
#pragma unroll
    for (int j2 = 0; j2 < 5; ++j2) in[j2] = row[5 * j2];
    h4_apply(sP + ((sub >> 1) & 1) * 25, in, out);
#pragma unroll
    for (int t2 = 0; t2 < 5; ++t2) row[5 * t2] = out[t2];
  }
  __syncwarp();
}
__device__ __noinline__ void h4_fine(const StageArgs& a, double* sTr, const double* sP, int face, int sub, int bgc) {
  h4_fine_body(a, sTr, sP, face, sub, bgc);
}

// Coarse side of a 2:1 face (R11-R14, R35): the own perturbation trace
// projected onto the four mortars (A along t1, B along t2), Rusanov against the fine elements'
// traces (C), back projection (D along k1 summed over b1, E along k2 summed over b2) and the
// lift value into the face's slot -- the generic kernel's mort_A..E (same operands, same
// rounding order; all four sub-faces per step).  Scratch ms = the staging row, [b][f][t]: U_b1 (at
// b = b1), the mortar states, the mortar fluxes F*_b, W_b2 (at b = 2 b2).
// Own-side data of a coarse face for h4_coarse: from the staged element row (inline mode) ...
struct CoarseRow {
  static constexpr bool kFineStaged = false;  // the fine elements' traces come from global memory
  const double *sQ, *sBg;
  int face;
  __device__ double bg(int t2, int which) const { return sBg[4 * h4_fvert(face, t2) + which]; }
  __device__ double val(int f, int t1, int t2) const { return sQ[f * S4::Np + h4_fnode(face, t1, t2)]; }
  __device__ void own(const StageArgs& a, int t1, int t2, St& s, Dv& v) const {
    h4_own(a, sQ, sBg, h4_fnode(face, t1, t2), h4_fvert(face, t2), s, v);
  }
};
// ... or from the face trace staged alone (the mortar pre-pass): values tc[f][t], background rows
// bgt[t][4], EOS aux[t] (P'), aux[25 + t] (1/rho), t = t1 + 5 t2
struct CoarseFace {
  static constexpr bool kFineStaged = true;  // fine traces fq[b][g][t] and background rows fbg[b][kv][4] staged
  const double *tc, *bgt, *aux, *fq, *fbg;
  int face;
  __device__ double bg(int t2, int which) const { return bgt[4 * h4_fvert(face, t2) + which]; }
  __device__ double val(int f, int t1, int t2) const { return tc[f * S4::Nf + t1 + 5 * t2]; }
  __device__ void own(const StageArgs&, int t1, int t2, St& s, Dv& v) const {
    const int t = t1 + 5 * t2;
    bg_row(s, bgt, h4_fvert(face, t2));
    s.rp = __dsub_rn(tc[t], s.rb);
    s.U[0] = tc[S4::Nf + t];
    s.U[1] = tc[2 * S4::Nf + t];
    s.U[2] = tc[3 * S4::Nf + t];
    s.Tp = __dsub_rn(tc[4 * S4::Nf + t], s.Tb);
    v.rho = __dadd_rn(s.rb, s.rp);
    v.Th = __dadd_rn(s.Tb, s.Tp);
    v.Pp = aux[t];
    v.rinv = aux[S4::Nf + t];
  }
};

#ifndef DG_H4_CUNROLL
#define DG_H4_CUNROLL 2
#endif
template <class Src>
__device__ __noinline__ void h4_coarse(const StageArgs& a, const Src src, double* sTr, double* ms, const double* sP,
                                       const double* sR, int face, int mslot, double cf) {
  constexpr int Np = S4::Np, Nf = S4::Nf, F = S4::F, MB = F * Nf;
  const int lane = threadIdx.x & 31;
  const int f = lane / 5, c = lane - 5 * (lane / 5);
  const int d = face >> 1;
  const double sgn = (face & 1) ? 1.0 : -1.0;
  // the fine elements' traces and background rows at mortar node t = lane of all four sub-faces,
  // loaded up front (one latency per coarse face; indexed by the rolled sub-face loop of step C,
  // so they live in local memory, L1)
  double fq[4][F];
  double2 fb0[4], fb1[4];
  if (!Src::kFineStaged && lane < 25) {
    const int nf = h4_fnode(face ^ 1, c, f);  // (t1, t2) = (lane % 5, lane / 5)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int mi = mslot * S4::NSUB + b;
      const double* qf = a.q_in + (int64_t)__ldg(a.mort + mi) * S4::STR + nf;
#pragma unroll
      for (int g = 0; g < F; ++g) fq[b][g] = __ldg(qf + g * Np);
      const int row = __ldg(a.mortbg + mi) + nf / 25;
      fb0[b] = __ldg(reinterpret_cast<const double2*>(a.bg4) + 2 * row);
      fb1[b] = __ldg(reinterpret_cast<const double2*>(a.bg4) + 2 * row + 1);
    }
  }
  if (lane < 25) {  // A: column j2 = c of field f of the own trace -> U_b1, both b1
    double in[5], out[5];
    const double bb = (f == 0 || f == 4) ? src.bg(c, f == 0 ? 0 : 1) : 0.0;
#pragma unroll
    for (int j1 = 0; j1 < 5; ++j1) {
      const double v = src.val(f, j1, c);
      in[j1] = (f == 0 || f == 4) ? __dsub_rn(v, bb) : v;
    }
#pragma unroll
    for (int b1 = 0; b1 < 2; ++b1) {
      h4_apply(sP + b1 * 25, in, out);
#pragma unroll
      for (int t1 = 0; t1 < 5; ++t1) ms[b1 * MB + f * 25 + 5 * c + t1] = out[t1];
    }
  }
  __syncwarp();
  if (lane < 25) {  // B: row t1 = c of field f: mortar states of sub-faces b1 (P_lo) and b1 + 2 (P_hi)
#pragma unroll
    for (int b1 = 0; b1 < 2; ++b1) {
      double in[5], out[5];
#pragma unroll
      for (int j2 = 0; j2 < 5; ++j2) in[j2] = ms[b1 * MB + f * 25 + c + 5 * j2];
      h4_apply(sP, in, out);
#pragma unroll
      for (int t2 = 0; t2 < 5; ++t2) ms[b1 * MB + f * 25 + c + 5 * t2] = out[t2];
      h4_apply(sP + 25, in, out);
#pragma unroll
      for (int t2 = 0; t2 < 5; ++t2) ms[(b1 + 2) * MB + f * 25 + c + 5 * t2] = out[t2];
    }
  }
  __syncwarp();
  if (lane < 25) {  // C: Rusanov at mortar node t = lane of every sub-face (fine level's background, R13)
    const int t = lane;
    // (staged fine data: two sub-faces' independent Rusanov chains in flight; the global-memory
    // variant stays rolled -- its fq[b][g] are indexed by the loop and live in local memory)
    constexpr int kCU = Src::kFineStaged ? DG_H4_CUNROLL : 1;
#pragma unroll kCU
    for (int b = 0; b < 4; ++b) {
      St R;
      if constexpr (Src::kFineStaged) {
        const double* fv = src.fq + b * MB + t;
        bg_row(R, src.fbg + b * 20, h4_fvert(face ^ 1, f));  // (t2 = lane / 5 = f)
        R.rp = __dsub_rn(fv[0], R.rb);
        R.U[0] = fv[Nf];
        R.U[1] = fv[2 * Nf];
        R.U[2] = fv[3 * Nf];
        R.Tp = __dsub_rn(fv[4 * Nf], R.Tb);
      } else {
        R.rb = fb0[b].x;
        R.Tb = fb0[b].y;
        R.Pb = fb1[b].x;
        R.rTb = fb1[b].y;
        R.rp = __dsub_rn(fq[b][0], R.rb);
        R.U[0] = fq[b][1];
        R.U[1] = fq[b][2];
        R.U[2] = fq[b][3];
        R.Tp = __dsub_rn(fq[b][4], R.Tb);
      }
      double* mo = ms + b * MB + t;
      St Lm = R;
      Lm.rp = mo[0];
      Lm.U[0] = mo[Nf];
      Lm.U[1] = mo[2 * Nf];
      Lm.U[2] = mo[3 * Nf];
      Lm.Tp = mo[4 * Nf];
      double Fs[F], FL[F];
      rusanov<3>(Lm, derive(Lm, a), R, derive(R, a), d, sgn, a.gamma, Fs, FL);
#pragma unroll
      for (int g = 0; g < F; ++g) mo[g * Nf] = Fs[g];
    }
  }
  __syncwarp();
  if (lane < 25) {  // D: W_b2[f][j1 + 5 k2] = sum_b1 sum_k1 R_b1[j1][k1] F*_{b1 + 2 b2}[f][k1 + 5 k2], k2 = c
#pragma unroll
    for (int b2 = 0; b2 < 2; ++b2) {
      double in0[5], in1[5];
      double* m0 = ms + (2 * b2) * MB + f * 25 + 5 * c;
      const double* m1 = ms + (2 * b2 + 1) * MB + f * 25 + 5 * c;
#pragma unroll
      for (int k1 = 0; k1 < 5; ++k1) {
        in0[k1] = m0[k1];
        in1[k1] = m1[k1];
      }
#pragma unroll
      for (int j1 = 0; j1 < 5; ++j1) {
        double acc = 0.0;
#pragma unroll
        for (int k1 = 0; k1 < 5; ++k1) acc = __fma_rn(sR[j1 * 5 + k1], in0[k1], acc);
#pragma unroll
        for (int k1 = 0; k1 < 5; ++k1) acc = __fma_rn(sR[25 + j1 * 5 + k1], in1[k1], acc);
        m0[j1] = acc;
      }
    }
  }
  __syncwarp();
  if (lane < 25) {  // E: back-projected flux at coarse node j = lane and the lift value (R14)
    const int j = lane, j1 = c, j2 = f;
    double Fc[F];
#pragma unroll
    for (int g = 0; g < F; ++g) Fc[g] = 0.0;
#pragma unroll
    for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
      for (int k2 = 0; k2 < 5; ++k2) {
        const double cc = sR[b2 * 25 + j2 * 5 + k2];
#pragma unroll
        for (int g = 0; g < F; ++g) Fc[g] = __fma_rn(cc, ms[(2 * b2) * MB + g * Nf + j1 + 5 * k2], Fc[g]);
      }
    St own;
    Dv vo;
    src.own(a, j1, j2, own, vo);
    double Fo[F];
    flux_d<3>(own, vo, d, Fo);
    double* L = sTr + face * F * Nf + j;
#pragma unroll
    for (int g = 0; g < F; ++g) L[g * Nf] = __dmul_rn(cf, __fma_rn(-sgn, Fo[g], Fc[g]));
  }
  __syncwarp();
}

// One axis of the element on its pencil owners (lane < 25): owner (pa, pb) of axis D holds the pencil
// nodes n0 + st m, m = 0..4 -- x: (j, k) = (pa, pb), y: (i, k), z: (i, j) -- of all five fields in
// registers, loaded from the staged row.  Everything of the axis happens there:
//   EOS (A1) at the five nodes (the same `derive` everywhere: bitwise equal values);
//   the two faces of the axis (A5, A6, A8): the pencil's end nodes are exactly face node t = lane of
//     faces 2 D and 2 D + 1, so the own state comes from registers, the neighbour's trace from its
//     slot, and the lift values stay in registers (coarse sides: the mortar steps' lift values);
//   flux (A2), contraction (A3, even-odd DFMA split of D), source (A4, x phase), lifts;
//   the residual accumulates through the staging row sS in the natural node order -- x writes,
//     y and z add in place (each lane its own positions) -- and the z owners finish with the RK
//     update (A9), leaving the output row in sS.
// No per-node tables, flux staging or lift round trips go through shared memory (the LSU data
// pipe was the co-limiter at 67 % with them); the price is the EOS evaluated once per axis.
// The y owners' accesses of the natural order are 2-way conflicting for 4 of the first 16 lanes.
struct NoHook {
  __device__ void operator()() const {}
};
template <int D, int KIND, int NC, class Hook = NoHook>
__device__ __forceinline__ void h4_axis(const StageArgs& a, const double* __restrict__ sQ, const double* sBg,
                                        const double* sTr, double* sS, const double* qn_g, uint64_t* mbq, int par,
                                        int info, int lane, int pb, int n0, double sd, bool wait_tr = false,
                                        const Hook& loaded = Hook()) {
  constexpr int Np = S4::Np, Nf = S4::Nf, F = S4::F;
  constexpr bool rk = KIND != 0, s0 = KIND == 1;
  constexpr int st = D == 0 ? 1 : (D == 1 ? 5 : 25);
  DG_CHECK(lane < 25 && n0 >= 0 && n0 + 4 * st < Np);
  double q[F][5];
#pragma unroll
  for (int f = 0; f < F; ++f)
#pragma unroll
    for (int m = 0; m < 5; ++m) q[f][m] = sQ[f * Np + n0 + st * m];
  double qn4[5];
  if (D == 2 && rk && !s0) {  // q_n: the field outside the bulk copy, from L2 (prefetched), coalesced
#pragma unroll
    for (int m = 0; m < 5; ++m) qn4[m] = __ldcs(qn_g + S4::QNF * Np + n0 + st * m);
  }
  loaded();  // (the z phase: the last reads of the state row are done)
  St bk;
  if (D != 2) bg_row(bk, sBg, pb);
  double Pp[5], ri[5];
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    if (D == 2) bg_row(bk, sBg, m);
    St e = bk;
    e.rp = __dsub_rn(q[0][m], bk.rb);
    e.Tp = __dsub_rn(q[4][m], bk.Tb);
    const Dv v = derive(e, a);
    Pp[m] = v.Pp;
    ri[m] = v.rinv;
  }
  if (D == 0 && wait_tr) {  // the neighbour traces (cp.async by the lanes of this branch), deferred to here
    cp_async_wait_all();
    __syncwarp(0x1ffffff);
  }
  const double rb0 = bk.rb;  // (x phase: the source's background density, row pb)
  double L[2][F];
  {
    const double cf = __dmul_rn(sd, a.w0inv);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int face = 2 * D + s, kind = face_kind(info, face), m = 4 * s, kf = D == 2 ? m : pb;
      const double* tr = sTr + face * F * Nf + lane;
      if (NC != 0 && kind == kCoarse) {  // (warp-uniform)
#pragma unroll
        for (int f = 0; f < F; ++f) L[s][f] = tr[f * Nf];
      } else {
        St own, R;
        if (D == 2) bg_row(own, sBg, kf);
        else own = bk;
        own.rp = __dsub_rn(q[0][m], own.rb);
        own.U[0] = q[1][m];
        own.U[1] = q[2][m];
        own.U[2] = q[3][m];
        own.Tp = __dsub_rn(q[4][m], own.Tb);
        Dv vo;
        vo.rho = __dadd_rn(own.rb, own.rp);
        vo.Th = __dadd_rn(own.Tb, own.Tp);
        vo.Pp = Pp[m];
        vo.rinv = ri[m];
        h4_nbr(D, tr, sBg, own, kind, face, kf, R);
        double Fs[F], Fo[F];
        rusanov<3>(own, vo, R, derive(R, a), D, s ? 1.0 : -1.0, a.gamma, Fs, Fo);
        const double msgn = s ? -1.0 : 1.0;
#pragma unroll
        for (int f = 0; f < F; ++f) L[s][f] = __dmul_rn(cf, __fma_rn(msgn, Fo[f], Fs[f]));
      }
    }
  }
  if (D == 2 && rk && !s0) mbar_wait(mbq, par);  // q_n fields 0..QNF-1 (bulk copy issued after the y phase)
  double ud[5];
#pragma unroll
  for (int m = 0; m < 5; ++m) ud[m] = __dmul_rn(q[1 + D][m], ri[m]);
  const double mg = -a.g;
#pragma unroll
  for (int f = 0; f < F; ++f) {
    double Fv[5], out[5];
#pragma unroll
    for (int m = 0; m < 5; ++m) Fv[m] = f == 0 ? q[1 + D][m] : __fma_rn(q[f][m], ud[m], f == 1 + D ? Pp[m] : 0.0);
    contract<4>(Fv, out, a);
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      const int n = f * Np + n0 + st * m;
      double v;
      if (D == 0) {
        const double base = m == 0 ? L[0][f] : (m == 4 ? L[1][f] : 0.0);
        v = __fma_rn(sd, out[m], f == 3 ? __fma_rn(mg, __dsub_rn(q[0][m], rb0), base) : base);
      } else {
        const double t = m == 0 ? __fma_rn(sd, out[m], L[0][f]) : (m == 4 ? __fma_rn(sd, out[m], L[1][f]) : __dmul_rn(sd, out[m]));
        v = __dadd_rn(sS[n], t);
      }
      if (D == 2 && rk) {  // RK update (A9)
        if (s0) v = __fma_rn(a.dt, v, q[f][m]);
        else {
          const double qn = f < S4::QNF ? sTr[n] : qn4[m];
          v = __fma_rn(a.rk_b, __fma_rn(a.dt, v, __dsub_rn(q[f][m], qn)), qn);
        }
      }
      sS[n] = v;
    }
  }
}

// KIND 0: RHS, 1: RK stage 0, 2: RK stage 1 or 2; LIST: element-list launch; NC: the launch's 2:1
// faces -- 0 none (no 2:1 code, no function calls in the element loop), 1 fine sides inline and
// coarse-side lifts from the mortar pre-pass, 2 both sides inline (h4_fine / h4_coarse calls)
template <int KIND, bool LIST, int NC, int W>
__global__ void __launch_bounds__(32 * W, S4::MINB / W) k_stage_h4(const __grid_constant__ StageArgs a) {
  constexpr int Np = S4::Np, Nf = S4::Nf, F = S4::F, STR = S4::STR;
  constexpr bool rk = KIND != 0, s0 = KIND == 1;
  extern __shared__ __align__(128) double smem_all[];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;  // the CTA's warps work on separate elements
  double* smem = smem_all + wq * S4::SMEM;
  double* sTr = smem + S4::OTR;
  double* sS = smem + S4::OS;
  __shared__ __align__(8) uint64_t mbar_[W];     // state row (per warp)
  __shared__ __align__(8) uint64_t mbq_[W];           // q_n (stages 1, 2)
  __shared__ __align__(16) int sDw_[W][2][16];  // descriptor (8 words) and face background rows (8), double-buffered
  __shared__ double sPR[4 * 25];  // P_lo, P_hi, R_lo, R_hi
  uint64_t& mbar = mbar_[wq];
  uint64_t& mbq = mbq_[wq];
  int(*sDw)[16] = sDw_[wq];

  const int64_t n_el = a.n_elem, stride = (int64_t)gridDim.x * W;
  int64_t base = (int64_t)blockIdx.x * W, e = base + wq;
  if (base >= n_el) return;  // (the whole CTA)
  for (int i = threadIdx.x; i < 100; i += 32 * W) sPR[i] = a.ops[OpsLayout::P(5, 0) + i];
  if (lane == 0) {
    mbar_init(&mbar, 1);
    mbar_init(&mbq, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (W > 1) __syncthreads();
  // element t's state row into the row buffer (lane 0).  The first one is issued here, every later one
  // inside the previous element's z phase, right after its last reads of the buffer, so the copy
  // (L2-prefetched) is in flight over the rest of that phase and the output store
  auto issue_row = [&](int64_t t) {
    fence_proxy_async();
    mbar_expect_tx(&mbar, STR * 8);
    bulk_g2s(smem + S4::OQ, a.q_in + elem_of<LIST>(a, t) * STR, STR * 8, &mbar);
  };
  // descriptor + face background rows of element t into slot b (cp.async, 4 x 16 B)
  auto load_desc = [&](int64_t t, int b) {
    if (lane < 2)
      cp_async16(reinterpret_cast<int4*>(sDw[b]) + lane, reinterpret_cast<const int4*>(a.desc + elem_of<LIST>(a, t)) + lane);
    else if (lane < 4)
      cp_async16(reinterpret_cast<int4*>(sDw[b] + 8) + (lane - 2), reinterpret_cast<const int4*>(a.nbrow + elem_of<LIST>(a, t) * 8) + (lane - 2));
  };
  if (e < n_el) load_desc(e, 0);
  cp_async_commit();
  cp_async_wait_all();
  __syncwarp();
  if (lane == 0 && e < n_el) issue_row(e);
  // x owner: pencil (j, k) = (l % 5, l / 5); y owner (i, k), z owner (i, j) with the same split
  const bool own25 = lane < 25;
  const int pa = lane % 5, pb = lane / 5;

  for (int it = 0; base < n_el; ++it, base += stride, e += stride) {
    // W > 1: the CTA's warps start every element together, so they run through the same stretch of the
    // (46-56 KB, straight-line) code at about the same time and share its instruction-cache lines: with
    // independent single-warp CTAs every warp of the SM is somewhere else in it, and the instruction
    // requests to the GPC-level cache were the busiest unit of the kernel (ncu: 86 % of peak)
    if (W > 1) __syncthreads();
    if (e >= n_el) continue;
    const int64_t en = e + stride;
    __syncwarp();  // every lane is done with the previous element's smem (and sees its descriptor)
    const int64_t er = elem_of<LIST>(a, e);  // this element's local row
    const ElemDesc& sD = *reinterpret_cast<const ElemDesc*>(sDw[it & 1]);
    const int* sNb = sDw[it & 1] + 8;
    // the descriptor into registers before any cp.async is queued: read face by face between the trace
    // gathers, each shared-memory load waited behind the gathers already in the load/store queue
    // (8 % of the stall samples)
    const int4 d0 = *reinterpret_cast<const int4*>(&sD), d1 = *(reinterpret_cast<const int4*>(&sD) + 1);
    const int nbr[6] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y};
    const int info = d1.z, bgrow = d1.w;
    if (en < n_el) load_desc(en, (it & 1) ^ 1);  // waited for with this element's traces
    const double* sQ = smem + S4::OQ;
    double* sBg = smem + S4::OBG;
    if (lane == 0) {
      if (en < n_el) prefetch_l2(a.q_in + elem_of<LIST>(a, en) * STR, STR * 8);
      if (rk && !s0) prefetch_l2(a.q_n + er * STR, STR * 8);
    }
    // neighbour traces (A5): raw values of the neighbour's face^1 nodes, [face][f][t] (cp.async;
    // lane t < 25 takes node t of every face, so the node offsets are compile-time per face)
    if (own25) {
#pragma unroll
      for (int face = 0; face < 6; ++face) {
        const int kind = face_kind(info, face);
        DG_CHECK(NC != 0 || kind == kConf || kind == kWall);
        if (kind == kConf || (NC != 0 && kind == kFine)) {
          DG_CHECK(nbr[face] >= 0);
          const double* src = a.q_in + (int64_t)nbr[face] * STR + h4_fnode(face ^ 1, pa, pb);
          double* dst = sTr + face * F * Nf + lane;
#pragma unroll
          for (int f = 0; f < F; ++f) cp_async8(dst + f * Nf, src + f * Np);
        } else if (NC == 1 && kind == kCoarse) {  // lift values from the mortar pre-pass
          DG_CHECK(nbr[face] >= 0 && nbr[face] < a.n_mort);
          const double* src = a.mlift + (int64_t)nbr[face] * F * Nf + lane;
          double* dst = sTr + face * F * Nf + lane;
#pragma unroll
          for (int f = 0; f < F; ++f) cp_async8(dst + f * Nf, src + f * Nf);
        }
      }
    } else {
      // the 7 background rows (own rows k = 0..4, the -z and +z neighbours' adjacent rows) by the
      // seven idle lanes, one row each, in the traces' cp.async group
      const int own = bgrow, r = lane - 25;
      const int row = r < 5 ? own + r : (r == 5 ? (sNb[4] >= 0 ? sNb[4] + 4 : own) : (sNb[5] >= 0 ? sNb[5] : own + 4));
      cp_async16(sBg + 4 * r, a.bg4 + 4 * (int64_t)row);
      cp_async16(sBg + 4 * r + 2, a.bg4 + 4 * (int64_t)row + 2);
    }
    cp_async_commit();
    const int lev = elem_level(info);
    const double* sHl = a.ops + OpsLayout::H(5) + 3 * lev;  // 2/h per axis at this level
    const double sx = -__ldg(sHl), sy = -__ldg(sHl + 1), sz = -__ldg(sHl + 2);
    mbar_wait(&mbar, it & 1);

    // this element's traces (and the next descriptor), needed first by the 2:1 steps.  -DDG_H4_DEFER_TR:
    // an element without them waits inside the x phase instead, after its state loads and EOS
#ifdef DG_H4_DEFER_TR
    const bool defer = NC == 0 || (NC == 1 && n_fine_faces(info) == 0);
#else
    const bool defer = false;  // (measured: c5n4 +1 % with the wait inside the x phase)
#endif
    if (!defer) cp_async_wait_all();
    __syncwarp();

    // ---- 2:1 faces (warp-uniform): fine sides project the coarse trace in place, coarse sides
    // run the mortar steps (scratch: the staging row) and leave lift values in their slots
    if (NC == 1 && n_fine_faces(info)) {
#pragma unroll 1
      for (int face = 0; face < 6; ++face)
        if (face_kind(info, face) == kFine) {
#ifdef DG_H4_FINE_CALL
          h4_fine(a, sTr, sPR, face, face_sub(info, face), sNb[face]);
#else
          h4_fine_body(a, sTr, sPR, face, face_sub(info, face), sNb[face]);
#endif
        }
    }
    if (NC == 2 && (n_fine_faces(info) | n_coarse_faces(info))) {
      if (lane == 0) bulk_wait_read0();  // h4_coarse's scratch is the staging row (see below)
      __syncwarp();
#pragma unroll 1
      for (int face = 0; face < 6; ++face) {
        const int kind = face_kind(info, face);
        if (kind == kFine) h4_fine(a, sTr, sPR, face, face_sub(info, face), sNb[face]);
        else if (kind == kCoarse)
          h4_coarse(a, CoarseRow{sQ, sBg, face}, sTr, sS, sPR, sPR + 50, face, sD.nbr[face],
                    __dmul_rn(-__ldg(sHl + (face >> 1)), a.w0inv));
      }
    }

    // the previous element's output store has read the staging row (long done by now: waiting at
    // the element start instead stalled the warp for 3 % of the samples)
    if (lane == 0) bulk_wait_read0();
    __syncwarp();

    // ---- the three axis phases (A1-A9) on the pencil owners; residual through the staging row
    const double* qn_g = a.q_n + er * STR;
    if (own25) h4_axis<0, KIND, NC>(a, sQ, sBg, sTr, sS, qn_g, &mbq, it & 1, info, lane, pb, 5 * lane, sx, defer);
    else
      for (int p = lane - 25; p < STR - F * Np; p += 7) sS[F * Np + p] = 0.0;  // row padding (deterministic)
    __syncwarp();
    if (own25) h4_axis<1, KIND, NC>(a, sQ, sBg, sTr, sS, qn_g, &mbq, it & 1, info, lane, pb, pa + 25 * pb, sy);
    __syncwarp();
    // q_n fields 0..3 of this element (L2-prefetched at the element start) by one bulk copy into
    // the dead x- / y-face slots, in flight over the z phase's loads, EOS and faces
    if (rk && !s0 && lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(&mbq, S4::QNF * Np * 8);
      bulk_g2s(sTr, qn_g, S4::QNF * Np * 8, &mbq);
    }
    if (own25)
      h4_axis<2, KIND, NC>(a, sQ, sBg, sTr, sS, qn_g, &mbq, it & 1, info, lane, pb, lane, sz, false, [&] {
        __syncwarp(0x1ffffff);  // every owner has its nodes of the row in registers
        if (lane == 0 && en < n_el) issue_row(en);
      });
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      bulk_s2g(a.out + er * STR, sS, STR * 8);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait0();
}

// Mortar pre-pass (3D N = 4 meshes with 2:1 faces): one warp per coarse face computes the coarse
// side's lift values (h4_coarse: steps A-E, the generic kernel's arithmetic and rounding order)
// into a.mlift[slot]; k_stage_h4 then copies them into the face slots like traces, so its element
// loop keeps only the fine-side projection of the 2:1 path (smaller code, no serial mortar chains
// per element).  Software-pipelined per warp: a slot's 64-B record (element, face, info, background
// row, fine elements and their background rows; built at upload) is loaded two faces ahead, and
// with it every input of the face -- the coarse trace, the four fine traces (8-B cp.async, sector
// granular) and the background rows -- one face ahead into the other half of a double buffer, so
// the dependent global round trips (record -> data) overlap the previous faces' mortar steps
// (unpipelined, the kernel sat on long-scoreboard stalls: 9.3 stalled warps per issue).
struct SM4 {
  static constexpr int F = S4::F, Nf = S4::Nf;
  // one input buffer: coarse trace [f][t], its background rows [kv][4], fine traces [b][g][t], their rows [b][kv][4]
  static constexpr int OTC = 0, OBGT = (F * Nf + 1) & ~1, OFQ = OBGT + 20, OFBG = OFQ + 4 * F * Nf, BUF = OFBG + 80;
  static constexpr int OAUX = 2 * BUF, OMS = OAUX + 2 * Nf, SMEM = OMS + 4 * F * Nf;
  static_assert(OBGT % 2 == 0 && OFBG % 2 == 0 && BUF % 2 == 0 && OMS % 2 == 0, "16-B aligned staging");
};
struct MortRec {
  int e, face, info, bgrow, fe[4], fbg[4];
};
__device__ __forceinline__ MortRec mort_rec(const StageArgs& a, int64_t slot) {
  const int4* p = reinterpret_cast<const int4*>(a.mort_owner) + 4 * slot;
  const int4 r0 = __ldg(p), r1 = __ldg(p + 1), r2 = __ldg(p + 2);
  return MortRec{r0.x, r0.y, r0.z, r0.w, {r1.x, r1.y, r1.z, r1.w}, {r2.x, r2.y, r2.z, r2.w}};
}
__global__ void __launch_bounds__(32) k_mortar_h4(const __grid_constant__ StageArgs a) {
  constexpr int Np = S4::Np, Nf = S4::Nf, F = S4::F, STR = S4::STR;
  extern __shared__ __align__(128) double smem[];
  double* sAux = smem + SM4::OAUX;
  double* sMS = smem + SM4::OMS;
  __shared__ double sPR[4 * 25];
  const int lane = threadIdx.x;
  for (int i = lane; i < 100; i += 32) sPR[i] = a.ops[OpsLayout::P(5, 0) + i];
  const int t1 = lane % 5, t2 = lane / 5;
  // every input of the face of record r into buffer B (one cp.async group)
  auto issue = [&](const MortRec& r, double* B) {
    if (lane < 25 && r.e >= 0) {  // (a slot without a local owner is skipped)
      const double* src = a.q_in + (int64_t)r.e * STR + h4_fnode(r.face, t1, t2);
#pragma unroll
      for (int f = 0; f < F; ++f) cp_async8(B + SM4::OTC + f * Nf + lane, src + f * Np);
      const int nf = h4_fnode(r.face ^ 1, t1, t2);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double* qf = a.q_in + (int64_t)r.fe[b] * STR + nf;
#pragma unroll
        for (int g = 0; g < F; ++g) cp_async8(B + SM4::OFQ + (b * F + g) * Nf + lane, qf + g * Np);
      }
      // background rows kv = 0..4 (two 16-B halves each): the coarse element's (lanes 0..9) and the
      // fine elements' (lanes 0..19, two per lane)
      if (lane < 10) cp_async16(B + SM4::OBGT + 2 * lane, a.bg4 + 4 * (int64_t)r.bgrow + 2 * lane);
      if (lane < 20) {
        const int b = lane / 5, kv = lane - 5 * b;
        const int fb = b == 0 ? r.fbg[0] : (b == 1 ? r.fbg[1] : (b == 2 ? r.fbg[2] : r.fbg[3]));  // (no local-memory indexing)
        const double* row = a.bg4 + 4 * (int64_t)(fb + kv);
        cp_async16(B + SM4::OFBG + b * 20 + 4 * kv, row);
        cp_async16(B + SM4::OFBG + b * 20 + 4 * kv + 2, row + 2);
      }
    }
    cp_async_commit();
  };
  const int64_t step = gridDim.x;
  int64_t slot = blockIdx.x;
  if (slot >= a.n_mort) return;
  MortRec cur = mort_rec(a, slot), nxt = cur;
  issue(cur, smem);
  if (slot + step < a.n_mort) nxt = mort_rec(a, slot + step);
  for (int it = 0; slot < a.n_mort; slot += step, ++it) {
    double* B = smem + (it & 1) * SM4::BUF;
    MortRec nn = nxt;
    const bool more = slot + step < a.n_mort;
    if (more) {
      issue(nxt, smem + ((it & 1) ^ 1) * SM4::BUF);  // (that buffer's face finished at the end of the last iteration)
      if (slot + 2 * step < a.n_mort) nn = mort_rec(a, slot + 2 * step);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncwarp();
    DG_CHECK(cur.e >= 0 && cur.face >= 0 && cur.face < 6 && face_kind(cur.info, cur.face) == kCoarse);
    if (cur.e < 0) {
      cur = nxt;
      nxt = nn;
      continue;
    }
    const double* sTc = B + SM4::OTC;
    const double* sBgt = B + SM4::OBGT;
    if (lane < 25) {  // EOS at the face node (the same derive as everywhere: bitwise the same values)
      St st;
      bg_row(st, sBgt, h4_fvert(cur.face, t2));
      st.rp = __dsub_rn(sTc[lane], st.rb);
      st.U[0] = sTc[Nf + lane];
      st.U[1] = sTc[2 * Nf + lane];
      st.U[2] = sTc[3 * Nf + lane];
      st.Tp = __dsub_rn(sTc[4 * Nf + lane], st.Tb);
      const Dv v = derive(st, a);
      sAux[lane] = v.Pp;
      sAux[Nf + lane] = v.rinv;
    }
    __syncwarp();
    const double cf = __dmul_rn(-__ldg(a.ops + OpsLayout::H(5) + 3 * elem_level(cur.info) + (cur.face >> 1)), a.w0inv);
    // the lift values straight to a.mlift[slot] (h4_coarse addresses its output as slot `face` of a trace block)
    h4_coarse(a, CoarseFace{sTc, sBgt, sAux, B + SM4::OFQ, B + SM4::OFBG, cur.face},
              a.mlift + slot * F * Nf - cur.face * F * Nf, sMS, sPR, sPR + 50, cur.face, (int)slot, cf);
    cur = nxt;
    nxt = nn;
  }
}

template <bool LIST, int NC, int W>
int launch_h4_w(const StageArgs& a, cudaStream_t s) {
  static LaunchCache cache[3];
  const int kind = a.mode == 0 ? 0 : (a.stage == 0 ? 1 : 2);
  const size_t bytes = sizeof(double) * S4::SMEM * W;
  const int64_t tiles = (a.n_elem + W - 1) / W;
  if (kind == 0) return launch_persistent(k_stage_h4<0, LIST, NC, W>, a, 32 * W, bytes, tiles, s, cache[0]);
  if (kind == 1) return launch_persistent(k_stage_h4<1, LIST, NC, W>, a, 32 * W, bytes, tiles, s, cache[1]);
  return launch_persistent(k_stage_h4<2, LIST, NC, W>, a, 32 * W, bytes, tiles, s, cache[2]);
}
template <bool LIST, int NC>
int launch_h4_nc(const StageArgs& a, cudaStream_t s) {
  if (a.n_elem < S4::kBigMesh) return launch_h4_w<LIST, NC, 1>(a, s);
  return launch_h4_w<LIST, NC, NC == 0 ? S4::WBIG : S4::WBIG_NC>(a, s);
}

template <bool LIST>
int launch_h4(const StageArgs& a, cudaStream_t s) {
  if (a.mlift != nullptr && a.n_mort > 0) {  // the mortar pre-pass first (same stream)
    static LaunchCache cache;
    const int e = launch_persistent(k_mortar_h4, a, 32, sizeof(double) * SM4::SMEM, a.n_mort, s, cache);
    if (e != cudaSuccess) return e;
  }
#ifndef DG_H4_NC_OFF
  if (!a.has_nc) return launch_h4_nc<LIST, 0>(a, s);
  if (a.mlift != nullptr) return launch_h4_nc<LIST, 1>(a, s);
#endif
  return launch_h4_nc<LIST, 2>(a, s);
}

}  // namespace

int launch_stage_h4(const StageArgs& a, void* stream) {
  const cudaStream_t s = (cudaStream_t)stream;
  return a.list ? launch_h4<true>(a, s) : launch_h4<false>(a, s);
}

}  // namespace dgi
