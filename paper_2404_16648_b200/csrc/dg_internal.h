// dg_internal.h -- libdg internal types shared by the host runtime
// (dg_host.cpp) and the sm_100a kernels (dg_kernels.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <vector>

namespace dgi {

constexpr int kMaxOrder = 8;
constexpr int kMaxLevel = 8;
constexpr int kMaxN1 = kMaxOrder + 1;
constexpr int kMaxH = (kMaxN1 + 1) / 2;  // even-odd split of D: rows/cols per half
constexpr int kEosTerms = 12;             // binomial-series terms of (1+x)^gamma - 1, |x| < 2^-5

// Face kinds packed 2 bits per local face in ElemDesc::info (bits 0..11).
enum FaceKind : int { kConf = 0, kWall = 1, kCoarse = 2, kFine = 3 };

// Per-element descriptor, 32 B.  nbr[f]: conforming/periodic -> neighbour
// element; wall -> -1; coarse side of a 2:1 face -> index into the mortar list
// (2^(dim-1) fine elements in b order); fine side -> the coarse element.
// info: bits 0..11 kind of face f (2 bits each); bits 12..23 the fine side's
// mortar position b on the coarse face (2 bits each); bits 24..27 level.
// bgrow: row of (level, iz, k=0) in the background table.
struct ElemDesc {
  int32_t nbr[6];
  int32_t info;
  int32_t bgrow;
};

__host__ __device__ inline int face_kind(int info, int f) { return (info >> (2 * f)) & 3; }
__host__ __device__ inline int face_sub(int info, int f) { return (info >> (12 + 2 * f)) & 3; }
__host__ __device__ inline int elem_level(int info) { return (info >> 24) & 15; }

// 1D operators, (N+1)^2 row-major each, stored contiguously on the device:
// D, P_lo, P_hi, R_lo, R_hi, then w (N+1), then 2/h [level 0..8][axis 0..2].
struct OpsLayout {
  static constexpr int kD = 0;
  __host__ __device__ static constexpr int P(int n1, int b) { return n1 * n1 * (1 + b); }
  __host__ __device__ static constexpr int R(int n1, int b) { return n1 * n1 * (3 + b); }
  __host__ __device__ static constexpr int W(int n1) { return n1 * n1 * 5; }
  __host__ __device__ static constexpr int H(int n1) { return n1 * n1 * 5 + n1; }
  // pointwise-interpolation baseline (NEXT-3): I_b[j][k] = l_k(2 x_j + (b ? -1 : 1))
  __host__ __device__ static constexpr int I(int n1, int b) { return n1 * n1 * 5 + n1 + (kMaxLevel + 1) * 3 + n1 * n1 * b; }
  __host__ __device__ static constexpr int size(int n1) { return n1 * n1 * 7 + n1 + (kMaxLevel + 1) * 3; }
};

struct StageArgs {
  const double* q_in;
  const double* q_n;
  double* out;
  const ElemDesc* desc;
  const int32_t* nbrow;  // [E][8] background row across each face (conforming / fine side), else -1
  const int32_t* mort;
  const int32_t* mortbg;  // background row (desc.bgrow) of each mortar's fine element, aligned with mort
  const double* bg4;  // background rows (rho_bar, Theta_bar, P_bar, 1/Theta_bar), 32 B each
  const double* ops;
  int64_t n_elem;
  int64_t stride;
  double gamma, g;
  double w0inv;
  double dt, rk_b;
  int stage;  // 0,1,2
  int mode;   // 0: out = L(q_in); 1: RK stage
  int ncmode;  // 2:1 faces: 0 mortar method, 1 pointwise interpolation (NEXT-3 baseline)
  int amr;     // 1: the mesh has 2:1 faces and DG_H4_AMR = 0 selects the generic kernel (kernel choice only)
  int has_nc;  // 1: some local element has a 2:1 face (kernel choice only: k_stage_h4 without 2:1 code)
  const int32_t* list;  // element list (n_elem entries, local rows) or nullptr: elements 0 .. n_elem-1
  const int32_t* mort_owner;  // [n_mort][16]: element, face, info, bgrow, fine elements [4], their bgrows [4], pad (3D N = 4 AMR), or nullptr
  double* mlift;              // [n_mort][F][Nf] coarse-side lift values written by the mortar pre-pass
  int64_t n_mort;
  // even-odd split of D (row stride kMaxH): De[i][m] = (D[i][m] + D[i][N-m])/2 (m < H),
  // De[i][H] = D[i][H] (odd N+1); Do[i][m] = (D[i][m] - D[i][N-m])/2, Do[H][m] = D[H][m]
  double De[kMaxH * kMaxH];
  double Do[kMaxH * kMaxH];
  double eos_c[kEosTerms];  // binomial coefficients C(gamma, k+1)
  unsigned long long* prof;  // debug phase clocks (kProfSlots per launch) or nullptr
};
constexpr int kProfSlots = 16;

struct TransferArgs {
  const int32_t* src_idx;
  const int32_t* dst_idx;
  const double* q_src;
  double* q_dst;
  const double* ops;
  int64_t n;
  int64_t stride;
};

// Launchers (dg_kernels.cu).  Return cudaError_t as int.
int launch_stage(int dim, int order, const StageArgs& a, void* stream);
// 3D, N = 4, mortar 2:1 treatment (dg_stage_h4.cu); launch_stage dispatches to it
int launch_stage_h4(const StageArgs& a, void* stream);
int debug_timeline(long long* out, int n);  // -DDG_TIMELINE builds only (else returns 0)
int launch_refine(int dim, int order, const TransferArgs& a, void* stream);
int launch_coarsen(int dim, int order, const TransferArgs& a, void* stream);
int launch_copy(int dim, int order, const TransferArgs& a, void* stream);
int launch_bg_expand(const double* bg3, double* bg4, int64_t n_rows, void* stream);
int launch_elem_integrals(int dim, int order, const double* q, int64_t n_elem, int64_t stride,
                          const ElemDesc* desc, const double* ops, const double* jac_by_level,
                          double* partial, void* stream);
// dg_check_state: out[0..3] = non-finite values, rho <= 0 nodes, rho*theta <= 0 nodes,
// smallest bad element (~0 if none); out is reset on the stream first.
int launch_check_state(const double* q, int64_t n_elem, int64_t stride, int Np, int F, unsigned long long* out,
                       void* stream);
bool supported(int dim, int order);
// NEXT-1: per-element refinement indicator (kind 0: max |Theta/rho - Theta_bar/rho_bar|,
// kind 1: max |rho - rho_bar|) from the 3-column background table
int launch_amr_indicator(int dim, int order, int kind, const double* q, int64_t n_elem, int64_t stride,
                         const ElemDesc* desc, const double* bg3, double* eta, void* stream);

// NEXT-3 viscous term V = mu div grad u' (dg_visc.cu); sig: n_elem * dim rows of stride
int launch_visc(int dim, int order, const double* q, double* sig, double* V, const ElemDesc* desc, const int32_t* mort,
                const double* bg3, const double* ops, int64_t n_elem, int64_t stride, double mu, void* stream);
// out[e][0 .. row) += c * V[e][0 .. row) for e < n_elem (row = F * Np doubles of each stride-long row)
int launch_axpy_rows(double* out, const double* V, double c, int64_t n_elem, int64_t stride, int row, void* stream);

// kinematic tracer (dg_tracer.cu): mode 0 rhs (out field 0 = dC/dt), 1 RK stage
int launch_tracer(int dim, int order, int mode, int stage, double dt, double rk_b, int ncmode, const double* s_n,
                  const double* s_in, double* out, const ElemDesc* desc, const int32_t* mort, const double* ops,
                  int64_t n_elem, int64_t stride, void* stream);

// NEXT-3 passive tracer of the Euler flow (dg_tracer.cu): sa carries the Euler stage input q_in,
// the mesh tables, constants and mode / stage / dt / rk_b; c rows field 0 = C
int launch_passive(int dim, int order, const StageArgs& sa, const double* c_n, const double* c_in, double* c_out,
                   void* stream);

// NEXT-4 face-trace exchange: dir 0 q -> buf (pack), 1 buf -> q (unpack); pairs [n][2] = (element, face),
// buf [n][F][Nf]
int launch_face_pack(int dim, int order, int dir, int64_t n, const int32_t* pairs, double* q, double* buf,
                     int64_t stride, void* stream);

// NEXT-1 host regrid planner (dg_regrid.cpp)
struct RegridIn {
  int dim, max_level;
  int root[3], periodic[3];
  int64_t n;
  const int8_t* level;
  const int32_t* anchor;  // [n][dim]
  const double* eta;      // [n]
  double refine_above, coarsen_below;
  int buffer;
};
struct RegridOut {
  std::vector<int8_t> level;
  std::vector<int32_t> anchor;
  std::vector<int32_t> refine_parent, refine_child0, coarsen_child0, coarsen_parent, copy_src, copy_dst;
};
// 0 on success; < 0 with *why set otherwise
int regrid_plan(const RegridIn& in, RegridOut& out, const char** why);

}  // namespace dgi
