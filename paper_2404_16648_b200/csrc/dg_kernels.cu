// dg_kernels.cu -- sm_100a kernels of libdg besides the fused stage kernel
// (dg_stage.cu): the conservative refine/coarsen projections (PAPER.md:279,
// 313; reading R16), element copy, the per-element quadrature sums of
// dg_integrals (R20) and the background-table expansion.  Design notes in
// DESIGN.md section 6.
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
};

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

__global__ void k_bg_expand(const double* __restrict__ bg3, double* __restrict__ bg4, int64_t n) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double th = bg3[3 * r + 1];
  bg4[4 * r + 0] = bg3[3 * r + 0];
  bg4[4 * r + 1] = th;
  bg4[4 * r + 2] = bg3[3 * r + 2];
  bg4[4 * r + 3] = __ddiv_rn(1.0, th);
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

int launch_bg_expand(const double* bg3, double* bg4, int64_t n_rows, void* stream) {
  if (n_rows <= 0) return cudaSuccess;
  k_bg_expand<<<(unsigned)((n_rows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(bg3, bg4, n_rows);
  return cudaGetLastError();
}

bool supported(int dim, int order) { return (dim == 2 || dim == 3) && order >= 1 && order <= kMaxOrder; }

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
