// dg_visc.cu -- NEXT-3 artificial viscosity (reading R42 of DESIGN.md):
// V = mu div grad u of the perturbation vector u = (rho', U, Theta'), BR1-style in
// strong form with central face values (walls: u* = u-, sigma* = 0; 2:1 faces through the
// mortars: m_b = 1/2 (P_b v_coarse + v_fine), fine v* = m_b, coarse v* = sum_b R_b m_b).
//
// Two plain kernels, one thread per (element, node), global loads only: the viscous
// path serves the paper's small 2D rising-bubble runs (mu = 1.5 m^2/s) and is not on the
// HBM-bound hot path; its result V is added to the stage output by an axpy (dt b_s V; V
// itself for a plain RHS), so the hot stage kernels stay unchanged.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dg_internal.h"

namespace dgi {
namespace {

template <int DIM, int N>
struct VC {
  static constexpr int n1 = N + 1, Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1, Nf = Np / n1, F = DIM + 2,
                       NSUB = 1 << (DIM - 1);
};

struct ViscArgs {
  const double* q;      // state rows (stride)
  const double* sig;    // gradients: sig[(e * DIM + d) * stride + f * Np + n]
  double* out;          // pass 1: sig; pass 2: V rows (stride)
  const ElemDesc* desc;
  const int32_t* mort;
  const double* bg;     // 3-column background table
  const double* ops;
  int64_t n_elem, stride;
  double mu;
};

template <int DIM, int N>
__device__ __forceinline__ int fnode(int f, int t) {  // volume node of face node t (R28)
  constexpr int n1 = N + 1;
  const int d = f >> 1, e = (f & 1) ? N : 0;
  if (DIM == 2) return d == 0 ? e + n1 * t : t + n1 * e;
  const int t1 = t % n1, t2 = t / n1;
  if (d == 0) return e + n1 * t1 + n1 * n1 * t2;
  if (d == 1) return t1 + n1 * e + n1 * n1 * t2;
  return t1 + n1 * t2 + n1 * n1 * e;
}

// pass-1 field: perturbation vector u_k(e, n)
template <int DIM, int N>
__device__ __forceinline__ double uval(const ViscArgs& a, int64_t e, int k, int n) {
  constexpr int n1 = N + 1, Np = VC<DIM, N>::Np;
  const double v = a.q[e * a.stride + k * Np + n];
  if (k != 0 && k != DIM + 1) return v;
  const int row = a.desc[e].bgrow + (DIM == 2 ? n / n1 : n / (n1 * n1));
  return v - a.bg[3 * row + (k == 0 ? 0 : 1)];
}

// pass-2 field: component d of the gradient of u_k
template <int DIM, int N>
__device__ __forceinline__ double sval(const ViscArgs& a, int64_t e, int d, int k, int n) {
  return a.sig[(e * DIM + d) * a.stride + k * VC<DIM, N>::Np + n];
}

// central value at face node t of face f of element e for the nodal field val(e, n)
template <int DIM, int N, class Val>
__device__ double face_star(const ViscArgs& a, int64_t e, int f, int t, bool wall_zero, const Val& val) {
  using C = VC<DIM, N>;
  constexpr int n1 = C::n1, Nf = C::Nf, NSUB = C::NSUB;
  const ElemDesc& D = a.desc[e];
  const int kind = face_kind(D.info, f);
  const double own = val(e, fnode<DIM, N>(f, t));
  if (kind == kWall) return wall_zero ? 0.0 : own;
  if (kind == kConf) return 0.5 * (own + val((int64_t)D.nbr[f], fnode<DIM, N>(f ^ 1, t)));
  const double* P = a.ops + OpsLayout::P(n1, 0);
  const double* R = a.ops + OpsLayout::R(n1, 0);
  if (kind == kFine) {  // mortar value at this (fine) node
    const int b = face_sub(D.info, f), b1 = b & 1, b2 = (b >> 1) & 1;
    const int t1 = t % n1, t2 = t / n1;
    const int64_t ec = D.nbr[f];
    double pc = 0.0;
    for (int j = 0; j < Nf; ++j) {
      const int j1 = j % n1, j2 = j / n1;
      double c = P[b1 * n1 * n1 + t1 * n1 + j1];
      if (DIM == 3) c *= P[b2 * n1 * n1 + t2 * n1 + j2];
      pc += c * val(ec, fnode<DIM, N>(f ^ 1, j));
    }
    return 0.5 * (pc + own);
  }
  // coarse side: back projection of the mortar values of all sub-faces
  const int j1 = t % n1, j2 = t / n1;
  double acc = 0.0;
  for (int b = 0; b < NSUB; ++b) {
    const int b1 = b & 1, b2 = (b >> 1) & 1;
    const int64_t ef = a.mort[D.nbr[f] * NSUB + b];
    for (int k = 0; k < Nf; ++k) {
      const int k1 = k % n1, k2 = k / n1;
      double pc = 0.0;
      for (int j = 0; j < Nf; ++j) {
        const int i1 = j % n1, i2 = j / n1;
        double c = P[b1 * n1 * n1 + k1 * n1 + i1];
        if (DIM == 3) c *= P[b2 * n1 * n1 + k2 * n1 + i2];
        pc += c * val(e, fnode<DIM, N>(f, j));
      }
      const double mb = 0.5 * (pc + val(ef, fnode<DIM, N>(f ^ 1, k)));
      double r = R[b1 * n1 * n1 + j1 * n1 + k1];
      if (DIM == 3) r *= R[b2 * n1 * n1 + j2 * n1 + k2];
      acc += r * mb;
    }
  }
  return acc;
}

// pass 1: sig_d = (2/h_d) D_d u + (2/h_d)/w0 n_d (u* - u-)
template <int DIM, int N>
__global__ void __launch_bounds__(128) k_visc_grad(const ViscArgs a) {
  using C = VC<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_elem * Np) return;
  const int64_t e = i / Np;
  const int n = (int)(i - e * Np);
  const int lev = elem_level(a.desc[e].info);
  const double w0inv = 1.0 / a.ops[OpsLayout::W(n1)];
  int idx[3] = {n % n1, (n / n1) % n1, n / (n1 * n1)};
  const int str[3] = {1, n1, n1 * n1};
  for (int d = 0; d < DIM; ++d) {
    const double s2h = a.ops[OpsLayout::H(n1) + 3 * lev + d];  // 2 / h_d
    const int base = n - idx[d] * str[d];
    for (int k = 0; k < F; ++k) {
      double sum = 0.0;
      for (int m = 0; m < n1; ++m) sum += a.ops[idx[d] * n1 + m] * uval<DIM, N>(a, e, k, base + m * str[d]);
      double v = s2h * sum;
      for (int side = 0; side < 2; ++side) {
        if (idx[d] != (side ? N : 0)) continue;
        const int f = 2 * d + side;
        int t = 0, sc = 1;
        for (int ax = 0; ax < DIM; ++ax)
          if (ax != d) {
            t += idx[ax] * sc;
            sc *= n1;
          }
        auto val = [&](int64_t ee, int nn) { return uval<DIM, N>(a, ee, k, nn); };
        const double st = face_star<DIM, N>(a, e, f, t, false, val);
        v += s2h * w0inv * (side ? 1.0 : -1.0) * (st - uval<DIM, N>(a, e, k, n));
      }
      a.out[(e * DIM + d) * a.stride + k * Np + n] = v;
    }
  }
}

// pass 2: V = mu sum_d [(2/h_d) D_d sig_d + (2/h_d)/w0 n_d (sig_d* - sig_d-)]
template <int DIM, int N>
__global__ void __launch_bounds__(128) k_visc_div(const ViscArgs a) {
  using C = VC<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_elem * Np) return;
  const int64_t e = i / Np;
  const int n = (int)(i - e * Np);
  const int lev = elem_level(a.desc[e].info);
  const double w0inv = 1.0 / a.ops[OpsLayout::W(n1)];
  int idx[3] = {n % n1, (n / n1) % n1, n / (n1 * n1)};
  const int str[3] = {1, n1, n1 * n1};
  for (int k = 0; k < F; ++k) {
    double V = 0.0;
    for (int d = 0; d < DIM; ++d) {
      const double s2h = a.ops[OpsLayout::H(n1) + 3 * lev + d];
      const int base = n - idx[d] * str[d];
      double sum = 0.0;
      for (int m = 0; m < n1; ++m) sum += a.ops[idx[d] * n1 + m] * sval<DIM, N>(a, e, d, k, base + m * str[d]);
      V += s2h * sum;
    }
    for (int d = 0; d < DIM; ++d) {
      const double s2h = a.ops[OpsLayout::H(n1) + 3 * lev + d];
      for (int side = 0; side < 2; ++side) {
        if (idx[d] != (side ? N : 0)) continue;
        const int f = 2 * d + side;
        int t = 0, sc = 1;
        for (int ax = 0; ax < DIM; ++ax)
          if (ax != d) {
            t += idx[ax] * sc;
            sc *= n1;
          }
        auto val = [&](int64_t ee, int nn) { return sval<DIM, N>(a, ee, d, k, nn); };
        const double st = face_star<DIM, N>(a, e, f, t, true, val);
        V += s2h * w0inv * (side ? 1.0 : -1.0) * (st - sval<DIM, N>(a, e, d, k, n));
      }
    }
    a.out[e * a.stride + k * Np + n] = a.mu * V;
  }
}

template <int DIM, int N>
int launch_visc_t(const ViscArgs& g, const ViscArgs& v, cudaStream_t s) {
  constexpr int Np = VC<DIM, N>::Np;
  const unsigned blocks = (unsigned)((g.n_elem * Np + 127) / 128);
  k_visc_grad<DIM, N><<<blocks, 128, 0, s>>>(g);
  k_visc_div<DIM, N><<<blocks, 128, 0, s>>>(v);
  return (int)cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_axpy_rows(double* __restrict__ out, const double* __restrict__ V, double c,
                                                   int64_t n_elem, int64_t stride, int row) {
  const int64_t n = n_elem * row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / row, j = e * stride + (i - e * row);
    out[j] = __fma_rn(c, V[j], out[j]);
  }
}

}  // namespace

int launch_axpy_rows(double* out, const double* V, double c, int64_t n_elem, int64_t stride, int row, void* stream) {
  if (n_elem <= 0) return cudaSuccess;
  const int64_t n = n_elem * row;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_axpy_rows<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, V, c, n_elem, stride, row);
  return (int)cudaGetLastError();
}

int launch_visc(int dim, int order, const double* q, double* sig, double* V, const ElemDesc* desc, const int32_t* mort,
                const double* bg3, const double* ops, int64_t n_elem, int64_t stride, double mu, void* stream) {
  if (n_elem <= 0) return cudaSuccess;
  ViscArgs g{q, nullptr, sig, desc, mort, bg3, ops, n_elem, stride, mu};
  ViscArgs v{q, sig, V, desc, mort, bg3, ops, n_elem, stride, mu};
  cudaStream_t s = (cudaStream_t)stream;
  switch (dim * 16 + order) {
#define DG_V(D_, N_) \
  case D_ * 16 + N_: return launch_visc_t<D_, N_>(g, v, s);
    DG_V(2, 1) DG_V(2, 2) DG_V(2, 3) DG_V(2, 4) DG_V(2, 5) DG_V(2, 6) DG_V(2, 7) DG_V(2, 8)
    DG_V(3, 1) DG_V(3, 2) DG_V(3, 3) DG_V(3, 4) DG_V(3, 5) DG_V(3, 6) DG_V(3, 7) DG_V(3, 8)
#undef DG_V
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace dgi
