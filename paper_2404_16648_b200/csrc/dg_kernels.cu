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
// Conservative parent <-> child projection (reading R16),
// hierarchically sum-factorised: the 2^d children share their partial
// products along the first axes (refine: 2 x-, 4 y-, 8 z-applications of a 1D
// operator instead of 8 x 3; coarsen likewise in reverse).  Persistent CTAs
// loop over families; element rows move with 16-B vector accesses.

// sum_m A[i_ax(n)][m] src[f][n | i_ax -> m] for entry i = f Np + n (1D operator A
// applied along axis AX, any field).
template <int DIM, int N, int AX>
__device__ __forceinline__ double apply1(const double* A, const double* src, int i) {
  constexpr int n1 = N + 1, Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  constexpr int st = AX == 0 ? 1 : (AX == 1 ? n1 : n1 * n1);
  const int f = i / Np, n = i - f * Np;
  const int id = (n / st) % n1;
  const double* line = src + f * Np + n - id * st;
  double sum = 0.0;
#pragma unroll
  for (int m = 0; m < n1; ++m) sum = __fma_rn(A[id * n1 + m], line[m * st], sum);
  return sum;
}

template <class T>
__device__ __forceinline__ void copy_row(T* dst, const T* src, int n) {  // block-wide, 16-B granules
  const double2* s = reinterpret_cast<const double2*>(src);
  double2* d = reinterpret_cast<double2*>(dst);
  for (int i = threadIdx.x; i < n / 2; i += blockDim.x) d[i] = s[i];
  if ((n & 1) && threadIdx.x == 0) dst[n - 1] = src[n - 1];
}

template <int DIM, int N>
__global__ void __launch_bounds__(256) k_refine(const TransferArgs a) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F, R = F * Np;
  extern __shared__ __align__(16) double smem[];
  double* sP = smem;                       // P_lo, P_hi (2 n1^2, padded to 16 B)
  double* sA = smem + ((2 * n1 * n1 + 1) & ~1);  // parent
  double* sX = sA + ((R + 1) & ~1);        // 2 x-level results
  double* sY = sX + 2 * R;                 // 4 y-level results (3D)
  for (int i = threadIdx.x; i < 2 * n1 * n1; i += blockDim.x) sP[i] = a.ops[n1 * n1 + i];
  for (int64_t fam = blockIdx.x; fam < a.n; fam += gridDim.x) {
    const int64_t src = __ldg(a.src_idx + fam), dst0 = __ldg(a.dst_idx + fam);
    __syncthreads();
    copy_row(sA, a.q_src + src * a.stride, R);
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * R; i += blockDim.x) {
      const int v = i / R;
      sX[i] = apply1<DIM, N, 0>(sP + v * n1 * n1, sA, i - v * R);
    }
    __syncthreads();
    if (DIM == 2) {  // children b = bx + 2 bz: z (axis 1) from X[bx], straight to global
      for (int i = threadIdx.x; i < 4 * R; i += blockDim.x) {
        const int b = i / R, r = i - b * R;
        a.q_dst[(dst0 + b) * a.stride + r] = apply1<DIM, N, 1>(sP + (b >> 1) * n1 * n1, sX + (b & 1) * R, r);
      }
    } else {
      for (int i = threadIdx.x; i < 4 * R; i += blockDim.x) {  // Y[bx + 2 by] from X[bx]
        const int v = i / R;
        sY[i] = apply1<DIM, N, 1>(sP + (v >> 1) * n1 * n1, sX + (v & 1) * R, i - v * R);
      }
      __syncthreads();
      for (int i = threadIdx.x; i < 8 * R; i += blockDim.x) {  // child b = bx + 2 by + 4 bz from Y[b & 3]
        const int b = i / R, r = i - b * R;
        a.q_dst[(dst0 + b) * a.stride + r] = apply1<DIM, N, 2>(sP + (b >> 2) * n1 * n1, sY + (b & 3) * R, r);
      }
    }
  }
}

template <int DIM, int N>
__global__ void __launch_bounds__(256) k_coarsen(const TransferArgs a) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F, R = F * Np, RP = (R + 1) & ~1;
  extern __shared__ __align__(16) double smem[];
  double* sR = smem;                       // R_lo, R_hi
  double* sC = smem + ((2 * n1 * n1 + 1) & ~1);  // two children (bx = 0, 1)
  double* sX = sC + 2 * RP;                // x-level result of one (by, bz)
  double* sY = sX + RP;                    // 2 (3D: y-level per bz; 2D: x-level per bz) results
  for (int i = threadIdx.x; i < 2 * n1 * n1; i += blockDim.x) sR[i] = a.ops[3 * n1 * n1 + i];
  for (int64_t fam = blockIdx.x; fam < a.n; fam += gridDim.x) {
    const int64_t src0 = __ldg(a.src_idx + fam), dst = __ldg(a.dst_idx + fam);
    constexpr int NYZ = DIM == 2 ? 2 : 4;  // (by, bz) pairs (2D: bz only)
    for (int yz = 0; yz < NYZ; ++yz) {
      __syncthreads();
      copy_row(sC, a.q_src + (src0 + 2 * yz) * a.stride, R);
      copy_row(sC + RP, a.q_src + (src0 + 2 * yz + 1) * a.stride, R);
      __syncthreads();
      // X = sum_bx R_bx^x child(bx + 2 yz)
      double* X = DIM == 2 ? sY + yz * RP : sX;
      for (int i = threadIdx.x; i < R; i += blockDim.x)
        X[i] = __dadd_rn(apply1<DIM, N, 0>(sR, sC, i), apply1<DIM, N, 0>(sR + n1 * n1, sC + RP, i));
      if (DIM == 3) {  // Y[bz] (+)= R_by^y X
        __syncthreads();
        const int by = yz & 1, bz = yz >> 1;
        for (int i = threadIdx.x; i < R; i += blockDim.x) {
          const double v = apply1<DIM, N, 1>(sR + by * n1 * n1, sX, i);
          sY[bz * RP + i] = by == 1 ? __dadd_rn(sY[bz * RP + i], v) : v;
        }
      }
    }
    __syncthreads();
    // parent = sum_bz R_bz^(last axis) Y[bz]
    for (int i = threadIdx.x; i < R; i += blockDim.x)
      a.q_dst[dst * a.stride + i] =
          __dadd_rn(apply1<DIM, N, DIM - 1>(sR, sY, i), apply1<DIM, N, DIM - 1>(sR + n1 * n1, sY + RP, i));
  }
}

// q_dst[dst[i]] = q_src[src[i]]: whole padded rows (elem_stride doubles, 16-B aligned), 16-B granules.
template <int ROW2>
__global__ void __launch_bounds__(256) k_copy(const TransferArgs a) {
  const int64_t total = a.n * ROW2;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = k / ROW2;
    const int c = (int)(k - e * ROW2);
    const int64_t s = __ldg(a.src_idx + e), d = __ldg(a.dst_idx + e);
    const double2 v = __ldg(reinterpret_cast<const double2*>(a.q_src + s * a.stride) + c);
    reinterpret_cast<double2*>(a.q_dst + d * a.stride)[c] = v;
  }
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
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (which == 2) {
    constexpr int ROW2 = ((C::F * C::Np + 15) / 16 * 16) / 2;  // padded row (elem_stride) in 16-B granules
    const int64_t total = a.n * ROW2;
    const int64_t want = (total + 255) / 256;
    const int grid = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
    if (grid > 0) k_copy<ROW2><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  constexpr int R = C::F * C::Np, RP = (R + 1) & ~1, OPS = (2 * C::n1 * C::n1 + 1) & ~1;
  const size_t bytes = sizeof(double) * (which == 0 ? (OPS + RP + 2 * R + (DIM == 3 ? 4 * R : 0))
                                                    : (OPS + 3 * RP + 2 * RP));
  static int grid_max[2] = {0, 0};
  if (grid_max[which] == 0) {
    cudaError_t e = which == 0
                        ? cudaFuncSetAttribute(k_refine<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)
                        : cudaFuncSetAttribute(k_coarsen<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = which == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_refine<DIM, N>, 256, bytes)
                   : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coarsen<DIM, N>, 256, bytes);
    if (e != cudaSuccess) return e;
    grid_max[which] = sms * (occ > 0 ? occ : 1);
  }
  const int grid = (int)(a.n < grid_max[which] ? a.n : grid_max[which]);
  if (grid == 0) return cudaSuccess;
  if (which == 0) k_refine<DIM, N><<<grid, 256, bytes, s>>>(a);
  else k_coarsen<DIM, N><<<grid, 256, bytes, s>>>(a);
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
