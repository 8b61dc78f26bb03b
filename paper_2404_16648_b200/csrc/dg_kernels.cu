// dg_kernels.cu -- sm_100a kernels of libdg besides the fused stage kernel
// (dg_stage.cu): the conservative refine/coarsen projections (PAPER.md:279,
// 313; reading R16), element copy, the per-element quadrature sums of
// dg_integrals (R20) and the background-table expansion.  Design notes in
// DESIGN.md section 6.
#include <cuda_runtime.h>

#include <algorithm>

#include <atomic>
#include <cstdint>
#include <mutex>

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

// One line (pencil along axis AX, index p in 0..Nf-1, field f) of a 1D operator
// application: dst[line] = A src[line] (acc: +=).  The thread loads the n1 line
// values once and reads A by warp-wide broadcast.
template <int DIM, int N, int AX>
__device__ __forceinline__ void line_base(int p, int& base) {
  constexpr int n1 = N + 1;
  if (AX == 0) base = n1 * p;
  else if (AX == 1) base = DIM == 2 ? p : (p % n1) + n1 * n1 * (p / n1);
  else base = p;
}
template <int DIM, int N, int AX, bool ACC, class Store>
__device__ __forceinline__ void apply_line(const double* A, const double* src, int f, int p, const Store& store) {
  constexpr int n1 = N + 1, Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  constexpr int st = AX == 0 ? 1 : (AX == 1 ? n1 : n1 * n1);
  int base;
  line_base<DIM, N, AX>(p, base);
  const double* s = src + f * Np + base;
  double v[n1];
#pragma unroll
  for (int m = 0; m < n1; ++m) v[m] = s[m * st];
#pragma unroll 1
  for (int i = 0; i < n1; ++i) {
    double sum = 0.0;
#pragma unroll
    for (int m = 0; m < n1; ++m) sum = __fma_rn(A[i * n1 + m], v[m], sum);
    store(f * Np + base + i * st, sum);
  }
}

// dst line = A0 src0 line + A1 src1 line (two 1D operators along AX, summed per output).
template <int DIM, int N, int AX>
__device__ __forceinline__ void line_pair(const double* A0, const double* src0, const double* A1, const double* src1,
                                          int f, int p, double* dst) {
  constexpr int n1 = N + 1, Np = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  constexpr int st = AX == 0 ? 1 : (AX == 1 ? n1 : n1 * n1);
  int base;
  line_base<DIM, N, AX>(p, base);
  const int o = f * Np + base;
  double v0[n1], v1[n1];
#pragma unroll
  for (int m = 0; m < n1; ++m) {
    v0[m] = src0[o + m * st];
    v1[m] = src1[o + m * st];
  }
#pragma unroll 1
  for (int i = 0; i < n1; ++i) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int m = 0; m < n1; ++m) {
      s0 = __fma_rn(A0[i * n1 + m], v0[m], s0);
      s1 = __fma_rn(A1[i * n1 + m], v1[m], s1);
    }
    dst[o + i * st] = __dadd_rn(s0, s1);
  }
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
  constexpr int n1 = C::n1, Np = C::Np, F = C::F, R = F * Np, Nf = Np / n1, L = F * Nf;  // L lines per array
  extern __shared__ __align__(16) double smem[];
  double* sP = smem;                             // P_lo, P_hi
  double* sA = smem + ((2 * n1 * n1 + 1) & ~1);  // parent
  double* sX = sA + ((R + 1) & ~1);              // 2 x-level results
  double* sY = sX + 2 * R;                       // 4 y-level results (3D)
  for (int i = threadIdx.x; i < 2 * n1 * n1; i += blockDim.x) sP[i] = a.ops[n1 * n1 + i];
  for (int64_t fam = blockIdx.x; fam < a.n; fam += gridDim.x) {
    const int64_t src = __ldg(a.src_idx + fam), dst0 = __ldg(a.dst_idx + fam);
    __syncthreads();
    copy_row(sA, a.q_src + src * a.stride, R);
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * L; i += blockDim.x) {  // X[bx] = P_bx^x parent
      const int v = i / L, r = i - v * L, f = r / Nf, p = r - f * Nf;
      double* X = sX + v * R;
      apply_line<DIM, N, 0, false>(sP + v * n1 * n1, sA, f, p, [&](int k, double x) { X[k] = x; });
    }
    __syncthreads();
    if (DIM == 2) {  // children b = bx + 2 bz: z (axis 1) from X[bx], straight to global
      for (int i = threadIdx.x; i < 4 * L; i += blockDim.x) {
        const int b = i / L, r = i - b * L, f = r / Nf, p = r - f * Nf;
        double* out = a.q_dst + (dst0 + b) * a.stride;
        apply_line<DIM, N, DIM - 1, false>(sP + (b >> 1) * n1 * n1, sX + (b & 1) * R, f, p,
                                            [&](int k, double x) { out[k] = x; });
      }
    } else {
      for (int i = threadIdx.x; i < 4 * L; i += blockDim.x) {  // Y[bx + 2 by] = P_by^y X[bx]
        const int v = i / L, r = i - v * L, f = r / Nf, p = r - f * Nf;
        double* Y = sY + v * R;
        apply_line<DIM, N, 1, false>(sP + (v >> 1) * n1 * n1, sX + (v & 1) * R, f, p, [&](int k, double x) { Y[k] = x; });
      }
      __syncthreads();
      for (int i = threadIdx.x; i < 8 * L; i += blockDim.x) {  // child b = P_bz^z Y[b & 3]
        const int b = i / L, r = i - b * L, f = r / Nf, p = r - f * Nf;
        double* out = a.q_dst + (dst0 + b) * a.stride;
        apply_line<DIM, N, 2, false>(sP + (b >> 2) * n1 * n1, sY + (b & 3) * R, f, p,
                                      [&](int k, double x) { out[k] = x; });
      }
    }
  }
}

// ---- warp-per-(family, field) transfer kernels (3D N <= 4, 2D N <= 6): no block barriers -------
// One warp takes one field of one family at a time through all the 1D levels (shared memory
// holds the intermediate levels of that warp only, __syncwarp between levels), so many
// independent (family, field) tasks per SM hide the global-memory latency.  The 1D operator is
// held in registers: only the lower one (P_lo for refine, R_lo for coarsen), because the upper
// one is its mirror image, P_hi[i][m] = P_lo[N-i][N-m] (and R alike: the LGL nodes and the two
// half intervals are symmetric about 0); a line for the upper half is read and written in
// reverse order.  No shared-memory operand loads in the FMA chains.
template <int DIM, int N>
struct WarpXfer {
  static constexpr int Np = Cfg<DIM, N>::Np;
  static constexpr int NPS = (Np + 3) & ~1;              // a staged field block (+1 for the 16-B span, even)
  static constexpr int WS = DIM == 3 ? 8 * NPS : 4 * NPS;  // per-warp scratch (doubles): refine 2 parents + X + Y
                                                           // (3D: 2 Np + 2 Np + 4 Np); coarsen the 2^d children
                                                           // (double-buffered: 2 WS per warp)
  static constexpr int W = 4;                            // warps per CTA
#ifndef DG_XFER_MINB_R
#define DG_XFER_MINB_R 1
#endif
  static constexpr int MINB_R = DG_XFER_MINB_R;  // (8, i.e. 64 registers, measured slower for 3D N = 4: spills)
#ifdef DG_XFER_CTA
  static constexpr bool use = false;
#else
  static constexpr bool use = DIM == 2 ? N <= 6 : N <= 4;
#endif
};

// out line = A in line, A = A0 (hi = 0) or its mirror (hi = 1); lines of n1 values at stride st
template <int N>
__device__ __forceinline__ void rline(const double (&A)[(N + 1) * (N + 1)], int hi, const double* in, int st_in,
                                      double* out, int st_out) {
  constexpr int n1 = N + 1;
  double v[n1];
#pragma unroll
  for (int m = 0; m < n1; ++m) v[m] = in[(hi ? N - m : m) * st_in];
#pragma unroll
  for (int i = 0; i < n1; ++i) {
    double sum = 0.0;
#pragma unroll
    for (int m = 0; m < n1; ++m) sum = __fma_rn(A[i * n1 + m], v[m], sum);
    out[(hi ? N - i : i) * st_out] = sum;
  }
}
// the same with the node addresses given by functors (swizzled level blocks): in(m), out(i)
template <int N, class InF, class OutF>
__device__ __forceinline__ void rline_f(const double (&A)[(N + 1) * (N + 1)], int hi, const InF& in, const OutF& out) {
  constexpr int n1 = N + 1;
  double v[n1];
#pragma unroll
  for (int m = 0; m < n1; ++m) v[m] = *in(hi ? N - m : m);
#pragma unroll
  for (int i = 0; i < n1; ++i) {
    double sum = 0.0;
#pragma unroll
    for (int m = 0; m < n1; ++m) sum = __fma_rn(A[i * n1 + m], v[m], sum);
    *out(hi ? N - i : i) = sum;
  }
}
// o = A0 in0 line + mirror(A0) in1 line (rline_pair's arithmetic), node addresses by functors
template <int N, class In0, class In1>
__device__ __forceinline__ void rpair_sum(const double (&A)[(N + 1) * (N + 1)], const In0& in0, const In1& in1,
                                          double (&o)[N + 1]) {
  constexpr int n1 = N + 1;
  double v0[n1], v1[n1];
#pragma unroll
  for (int m = 0; m < n1; ++m) {
    v0[m] = *in0(m);
    v1[m] = *in1(N - m);
  }
#pragma unroll
  for (int i = 0; i < n1; ++i) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int m = 0; m < n1; ++m) {
      s0 = __fma_rn(A[i * n1 + m], v0[m], s0);
      s1 = __fma_rn(A[(N - i) * n1 + m], v1[m], s1);
    }
    o[i] = __dadd_rn(s0, s1);
  }
}
// out line = A0 in0 line + mirror(A0) in1 line
template <int N>
__device__ __forceinline__ void rline_pair(const double (&A)[(N + 1) * (N + 1)], const double* in0, const double* in1,
                                           int st_in, double* out, int st_out) {
  constexpr int n1 = N + 1;
  double v0[n1], v1[n1];
#pragma unroll
  for (int m = 0; m < n1; ++m) {
    v0[m] = in0[m * st_in];
    v1[m] = in1[(N - m) * st_in];
  }
#pragma unroll
  for (int i = 0; i < n1; ++i) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int m = 0; m < n1; ++m) {
      s0 = __fma_rn(A[i * n1 + m], v0[m], s0);
      s1 = __fma_rn(A[(N - i) * n1 + m], v1[m], s1);
    }
    out[i * st_out] = __dadd_rn(s0, s1);
  }
}

// Bulk-copy (TMA) staging for the warp-per-task transfer kernels: one mbarrier per warp and buffer.
// The 16-B cp.async staging wrote shared memory sector by sector as the data returned (ncu: 16
// wavefronts per warp instruction instead of 4: 15 % of the kernels' shared-memory wavefronts, on
// an LSU data pipe that is 58-69 % busy); a bulk copy writes whole lines and issues one instruction.
__device__ __forceinline__ uint32_t xf_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void xf_mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(xf_smem(m)) : "memory");
}
__device__ __forceinline__ void xf_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the buffer
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(xf_smem(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void xf_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   xf_smem(dst)),
               "l"(src), "r"(bytes), "r"(xf_smem(m))
               : "memory");
}
__device__ __forceinline__ void xf_wait(uint64_t* m, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n XW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra XW_%=;\n}\n" ::"r"(
                   xf_smem(m)),
               "r"(parity)
               : "memory");
}
// the 16-B aligned span around src[0 .. n): source pointer, byte count, offset of src[0] inside it
__device__ __forceinline__ const double* xf_span(const double* src, int n, int& off, uint32_t& bytes) {
  off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
  bytes = 16u * (uint32_t)((n + off + 1) >> 1);
  return src - off;
}

// for (it = lane; it < NI; it += 32) body(it), with a compile-time trip count so that the
// rounds' global loads can all be in flight together
template <int NI, class Body>
__device__ __forceinline__ void warp_rounds(int lane, const Body& body) {
#pragma unroll
  for (int r = 0; r < (NI + 31) / 32; ++r) {
    const int it = lane + 32 * r;
    if (NI % 32 == 0 || it < NI) body(it);
  }
}

template <int DIM, int N>
__global__ void __launch_bounds__(128, WarpXfer<DIM, N>::MINB_R) k_refine_w(const TransferArgs a) {
  using C = Cfg<DIM, N>;
  using X_ = WarpXfer<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F, Nf = Np / n1, NCH = 1 << DIM;
  extern __shared__ __align__(16) double smem[];
  double P[n1 * n1];  // P_lo (P_hi = its mirror)
#pragma unroll
  for (int i = 0; i < n1 * n1; ++i) P[i] = __ldg(a.ops + n1 * n1 + i);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NPS = X_::NPS;
  double* S2 = smem + warp * X_::WS;  // the parent's field, double-buffered (the next task's in flight)
  double* X = S2 + 2 * NPS;           // X[bx][Np]
  double* Y = X + 2 * NPS;            // Y[bx + 2 by][Np] (3D)
  const int64_t step = (int64_t)gridDim.x * X_::W;
  __shared__ __align__(8) uint64_t mb[X_::W][2];
  if (lane == 0) {
    xf_mbar_init(&mb[warp][0]);
    xf_mbar_init(&mb[warp][1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto stage = [&](int64_t task, int b) {  // the task's parent field into buffer b (one bulk copy)
    const int64_t fam = task / F;
    const int f = (int)(task - fam * F);
    int off;
    uint32_t bytes;
    const double* s0 = xf_span(a.q_src + __ldg(a.src_idx + fam) * a.stride + f * Np, Np, off, bytes);
    if (lane == 0) {
      xf_expect(&mb[warp][b], bytes);
      xf_bulk(S2 + b * NPS, s0, bytes, &mb[warp][b]);
    }
    return off;
  };
  int64_t task = (int64_t)blockIdx.x * X_::W + warp;
  int off = task < a.n * F ? stage(task, 0) : 0;
  int it = 0;
  for (int buf = 0; task < a.n * F; task += step, buf ^= 1, ++it) {
    const int64_t fam = task / F;
    const int f = (int)(task - fam * F);
    const double* par = S2 + buf * NPS + off;
    double* out0 = a.q_dst + __ldg(a.dst_idx + fam) * a.stride + f * Np;
    int off_next = 0;
    if (task + step < a.n * F) off_next = stage(task + step, buf ^ 1);  // (that buffer's reads ended with the last task)
    xf_wait(&mb[warp][buf], (uint32_t)((it >> 1) & 1));
    if (DIM == 3 && N == 4) {
      // 3D N = 4: one level block per round on lanes 0..24 (p = lane) and swizzled level blocks, so that
      // every half warp's 8-B accesses hit distinct bank pairs (found by exhaustive search; the packed
      // 32-lane rounds over natural-order blocks took 255 shared wavefronts per task for 155 ideal):
      //   X[bx]: node (i, j, k) at 25 i + ((j + 5 k + 8 (i & 1)) mod 25)   (x lines write, y lines read)
      //   Y[v] : node (i, j, k) at 25 j + ((i + 5 k + sy(j)) mod 25), sy = 0, 1, 3, 4, 5   (y write, z read)
      if (lane < Nf) {
        const int p = lane, pa = p % n1, pb = p / n1;
        const int q8 = p + 8 >= 25 ? p + 8 - 25 : p + 8;
#pragma unroll 1
        for (int bx = 0; bx < 2; ++bx)  // x lines: (j, k) = (pa, pb)
          rline_f<N>(P, bx, [&](int m) { return par + n1 * p + m; },
                     [&](int i) { return X + bx * NPS + 25 * i + ((i & 1) ? q8 : p); });
      }
      __syncwarp();
      if (lane < Nf) {
        const int p = lane, pa = p % n1, pb = p / n1;  // y lines: (i, k) = (pa, pb)
        const int xb = 5 * pb + 8 * (pa & 1);         // X index of (i, j = m, k): 25 i + ((m + xb) mod 25)
#pragma unroll 1
        for (int v = 0; v < 4; ++v)
          rline_f<N>(P, v >> 1,
                     [&](int m) {
                       const int t = m + xb;
                       return X + (v & 1) * NPS + 25 * pa + (t >= 25 ? t - 25 : t);
                     },
                     [&](int j) {
                       const int t = p + j + (j >= 2 ? 1 : 0);
                       return Y + v * NPS + 25 * j + (t >= 25 ? t - 25 : t);
                     });
      }
      __syncwarp();
      if (lane < Nf) {
        const int p = lane, pa = p % n1, pb = p / n1;  // z lines: (i, j) = (pa, pb)
        const int yb = pa + pb + (pb >= 2 ? 1 : 0);   // Y index of (i, j, k = m): 25 j + ((5 m + yb) mod 25)
#pragma unroll 1
        for (int b = 0; b < NCH; ++b)
          rline_f<N>(P, b >> 2,
                     [&](int m) {
                       const int t = 5 * m + yb;
                       return Y + (b & 3) * NPS + 25 * pb + (t >= 25 ? t - 25 : t);
                     },
                     [&](int k) { return out0 + b * a.stride + p + n1 * n1 * k; });
      }
      __syncwarp();
      off = off_next;
      continue;
    }
    warp_rounds<2 * Nf>(lane, [&](int it) {  // x lines: X[bx] = P_bx parent
      const int bx = it / Nf, p = it - bx * Nf;
      rline<N>(P, bx, par + n1 * p, 1, X + bx * NPS + n1 * p, 1);
    });
    __syncwarp();
    if (DIM == 3) {
      for (int it = lane; it < 4 * Nf; it += 32) {  // y lines: Y[bx + 2 by] = P_by X[bx]
        const int v = it / Nf, p = it - v * Nf;
        const int base = (p % n1) + n1 * n1 * (p / n1);
        rline<N>(P, v >> 1, X + (v & 1) * NPS + base, n1, Y + v * NPS + base, n1);
      }
      __syncwarp();
      for (int it = lane; it < NCH * Nf; it += 32) {  // z lines: child b = P_bz Y[b & 3], to global
        const int b = it / Nf, p = it - b * Nf;
        rline<N>(P, b >> 2, Y + (b & 3) * NPS + p, n1 * n1, out0 + b * a.stride + p, n1 * n1);
      }
    } else {
      for (int it = lane; it < NCH * Nf; it += 32) {  // axis-1 lines: child b = bx + 2 bz = P_bz X[bx]
        const int b = it / Nf, p = it - b * Nf;
        rline<N>(P, b >> 1, X + (b & 1) * NPS + p, n1, out0 + b * a.stride + p, n1);
      }
    }
    __syncwarp();
    off = off_next;
  }
}

template <int DIM, int N>
__global__ void __launch_bounds__(128) k_coarsen_w(const TransferArgs a) {
  using C = Cfg<DIM, N>;
  using X_ = WarpXfer<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F, Nf = Np / n1;
  extern __shared__ __align__(16) double smem[];
  double R[n1 * n1];  // R_lo (R_hi = its mirror)
#pragma unroll
  for (int i = 0; i < n1 * n1; ++i) R[i] = __ldg(a.ops + 3 * n1 * n1 + i);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NCH = 1 << DIM;
  // the children's field b at S + b Np (staged one task ahead into the other buffer); the levels
  // in place: X[v] over child 2v (S + 2 v Np), 3D: Y[bz] over X[2 bz] (S + 4 bz Np)
  const int64_t step = (int64_t)gridDim.x * X_::W;
  constexpr int NPS = X_::NPS;
  __shared__ __align__(8) uint64_t mb[X_::W][2];
  if (lane == 0) {
    xf_mbar_init(&mb[warp][0]);
    xf_mbar_init(&mb[warp][1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto stage = [&](int64_t task, int bf) {  // child b's field at S + b NPS + (returned offset): 2^d bulk copies
    double* S = smem + (2 * warp + bf) * X_::WS;
    const int64_t fam = task / F;
    const int f = (int)(task - fam * F);
    int off;
    uint32_t bytes;
    // (the same span for every child: rows are 16-B aligned)
    const double* s0 = xf_span(a.q_src + __ldg(a.src_idx + fam) * a.stride + f * Np, Np, off, bytes);
    if (lane == 0) {
      xf_expect(&mb[warp][bf], bytes * NCH);
#pragma unroll
      for (int b = 0; b < NCH; ++b) xf_bulk(S + b * NPS, s0 + b * a.stride, bytes, &mb[warp][bf]);
    }
    return off;
  };
  int buf = 0, it = 0;
  int64_t task = (int64_t)blockIdx.x * X_::W + warp;
  int off = task < a.n * F ? stage(task, 0) : 0;
  for (; task < a.n * F; task += step, buf ^= 1, ++it) {
    double* S = smem + (2 * warp + buf) * X_::WS + off;
    double* X = S;
    double* Y = S;
    const int64_t fam = task / F;
    const int f = (int)(task - fam * F);
    double* par = a.q_dst + __ldg(a.dst_idx + fam) * a.stride + f * Np;
    constexpr int NV = DIM == 3 ? 4 : 2;
    int off_next = 0;
    if (task + step < a.n * F) off_next = stage(task + step, buf ^ 1);  // (that buffer's reads ended with the last task)
    xf_wait(&mb[warp][buf], (uint32_t)((it >> 1) & 1));
    if (DIM == 3 && N == 4) {
      // 3D N = 4: one block pair per round on lanes 0..24 and swizzled level blocks (k_refine_w's layouts:
      // every half warp's 8-B accesses hit distinct bank pairs; the packed rounds over natural-order blocks
      // spent 39 % of the shared wavefronts on conflicts).  X[v] goes to child 2v+1's block (after every
      // lane has read the pair), Y[bz] to child 4bz's block (dead by then).
      const int p = lane, pa = p % n1, pb = p / n1;
      const int q8 = p + 8 >= 25 ? p + 8 - 25 : p + 8;
      auto wrap = [](int t) { return t >= 25 ? t - 25 : t; };
#pragma unroll 1
      for (int v = 0; v < 4; ++v) {  // x lines, (j, k) = (pa, pb): X[v] = R_lo child(2v) + R_hi child(2v + 1)
        double o[n1];
        if (lane < Nf)
          rpair_sum<N>(R, [&](int m) { return S + (2 * v) * NPS + n1 * p + m; },
                       [&](int m) { return S + (2 * v + 1) * NPS + n1 * p + m; }, o);
        __syncwarp();
        if (lane < Nf) {
#pragma unroll
          for (int i = 0; i < n1; ++i) S[(2 * v + 1) * NPS + 25 * i + ((i & 1) ? q8 : p)] = o[i];
        }
      }
      __syncwarp();
      if (lane < Nf) {  // y lines, (i, k) = (pa, pb): Y[bz] = R_lo X[2 bz] + R_hi X[2 bz + 1]
        const int xb = 5 * pb + 8 * (pa & 1);
#pragma unroll 1
        for (int bz = 0; bz < 2; ++bz) {
          double o[n1];
          rpair_sum<N>(R, [&](int m) { return S + (4 * bz + 1) * NPS + 25 * pa + wrap(m + xb); },
                       [&](int m) { return S + (4 * bz + 3) * NPS + 25 * pa + wrap(m + xb); }, o);
#pragma unroll
          for (int j = 0; j < n1; ++j) S[(4 * bz) * NPS + 25 * j + wrap(p + j + (j >= 2 ? 1 : 0))] = o[j];
        }
      }
      __syncwarp();
      if (lane < Nf) {  // z lines, (i, j) = (pa, pb): parent = R_lo Y[0] + R_hi Y[1]
        const int yb = pa + pb + (pb >= 2 ? 1 : 0);
        double o[n1];
        rpair_sum<N>(R, [&](int m) { return S + 25 * pb + wrap(5 * m + yb); },
                     [&](int m) { return S + 4 * NPS + 25 * pb + wrap(5 * m + yb); }, o);
#pragma unroll
        for (int k = 0; k < n1; ++k) par[p + n1 * n1 * k] = o[k];
      }
      __syncwarp();
      off = off_next;
      continue;
    }
    warp_rounds<NV * Nf>(lane, [&](int it) {  // x lines: X[v] = R_lo child(2v) + R_hi child(2v + 1), in place
      const int v = it / Nf, p = it - v * Nf;
      rline_pair<N>(R, S + (2 * v) * NPS + n1 * p, S + (2 * v + 1) * NPS + n1 * p, 1, X + 2 * v * NPS + n1 * p, 1);
    });
    __syncwarp();
    if (DIM == 3) {
      for (int it = lane; it < 2 * Nf; it += 32) {  // y lines: Y[bz] = R_lo X[2 bz] + R_hi X[2 bz + 1], in place
        const int bz = it / Nf, p = it - bz * Nf;
        const int base = (p % n1) + n1 * n1 * (p / n1);
        rline_pair<N>(R, X + (4 * bz) * NPS + base, X + (4 * bz + 2) * NPS + base, n1, Y + 4 * bz * NPS + base, n1);
      }
      __syncwarp();
      for (int it = lane; it < Nf; it += 32)  // z lines: parent = R_lo Y[0] + R_hi Y[1]
        rline_pair<N>(R, Y + it, Y + 4 * NPS + it, n1 * n1, par + it, n1 * n1);
    } else {
      for (int it = lane; it < Nf; it += 32)  // axis-1 lines: parent = R_lo X[0] + R_hi X[1]
        rline_pair<N>(R, X + it, X + 2 * NPS + it, n1, par + it, n1);
    }
    __syncwarp();
    off = off_next;
  }
}

// Children per bulk-copied group in the coarsen kernel: 8 when the double buffer
// fits ~64 KB, else 4 (<= 200 KB), else 2.
template <int DIM, int N>
struct CoarsenG {
  static constexpr int R = Cfg<DIM, N>::F * Cfg<DIM, N>::Np, RP = (R + 1) & ~1, NCH = 1 << DIM;
  static constexpr int STR = (R + 15) / 16 * 16;
  // double-buffered groups of G children: (2 G + G/2 + 2) rows of shared memory
  static constexpr int G = (NCH >= 8 && (16 * STR + 6 * RP) <= 8192) ? 8
                           : ((NCH >= 4 && (8 * STR + 4 * RP) <= 25600) ? 4 : 2);
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int DIM, int N>
__global__ void __launch_bounds__(256) k_coarsen(const TransferArgs a) {
  using C = Cfg<DIM, N>;
  constexpr int n1 = C::n1, Np = C::Np, F = C::F, R = F * Np, RP = (R + 1) & ~1, Nf = Np / n1, L = F * Nf;
  constexpr int NCH = 1 << DIM, G = CoarsenG<DIM, N>::G, NG = NCH / G;
  constexpr int STR = (R + 15) / 16 * 16;  // element row stride (doubles)
  extern __shared__ __align__(128) double smem[];
  double* sC[2] = {smem, smem + G * STR};        // G children per group, double-buffered (bulk copies)
  double* sR = smem + 2 * G * STR;               // R_lo, R_hi
  double* sX = sR + ((2 * n1 * n1 + 1) & ~1);    // x-level results of the G/2 pairs of a group
  double* sZ = sX + (G / 2) * RP;                // 2 inputs of the last axis (3D: Y[bz]; 2D: X[bz])
  __shared__ __align__(8) uint64_t mbar[2];
  for (int i = threadIdx.x; i < 2 * n1 * n1; i += blockDim.x) sR[i] = a.ops[3 * n1 * n1 + i];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nfam = a.n <= blockIdx.x ? 0 : (a.n - 1 - blockIdx.x) / gridDim.x + 1;  // families of this CTA
  const int64_t units = nfam * NG;
  auto issue = [&](int64_t u) {  // thread 0: children of unit u (family, group) -> buffer u & 1
    const int64_t fam = blockIdx.x + (u / NG) * gridDim.x;
    const int g0 = (int)(u % NG) * G;
    const int64_t src0 = __ldg(a.src_idx + fam) + g0;
    const uint32_t bytes = G * STR * 8, mb = smem_addr(&mbar[u & 1]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(sC[u & 1])),
                 "l"(a.q_src + src0 * a.stride), "r"(bytes), "r"(mb)
                 : "memory");
  };
  if (threadIdx.x == 0 && units > 0) issue(0);
  for (int64_t u = 0; u < units; ++u) {
    const int64_t fam = blockIdx.x + (u / NG) * gridDim.x;
    const int g0 = (int)(u % NG) * G;
    if (threadIdx.x == 0 && u + 1 < units) issue(u + 1);
    {
      const uint32_t mb = smem_addr(&mbar[u & 1]), par = (uint32_t)((u >> 1) & 1);
      asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(mb),
                   "r"(par)
                   : "memory");
    }
    const double* cb = sC[u & 1];
    // x level: pair v of the group -> X = R_0^x child(2 v) + R_1^x child(2 v + 1)
    for (int i = threadIdx.x; i < (G / 2) * L; i += blockDim.x) {
      const int v = i / L, r = i - v * L, f = r / Nf, p = r - f * Nf;
      double* X = DIM == 2 ? sZ + (g0 / 2 + v) * RP : sX + v * RP;
      line_pair<DIM, N, 0>(sR, cb + 2 * v * STR, sR + n1 * n1, cb + (2 * v + 1) * STR, f, p, X);
    }
    if (DIM == 3) {  // y level: Y[bz] = R_0^y X(by = 0, bz) + R_1^y X(by = 1, bz)
      __syncthreads();
      if (G >= 4) {
        for (int i = threadIdx.x; i < (G / 4) * L; i += blockDim.x) {
          const int v = i / L, r = i - v * L, f = r / Nf, p = r - f * Nf;
          double* Y = sZ + (g0 / 4 + v) * RP;
          line_pair<DIM, N, 1>(sR, sX + 2 * v * RP, sR + n1 * n1, sX + (2 * v + 1) * RP, f, p, Y);
        }
      } else {  // one pair per group: accumulate over by
        const int pr = g0 / 2, by = pr & 1, bz = pr >> 1;
        double* Y = sZ + bz * RP;
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
          const int f = i / Nf, p = i - f * Nf;
          if (by == 0) apply_line<DIM, N, 1, false>(sR, sX, f, p, [&](int k, double x) { Y[k] = x; });
          else apply_line<DIM, N, 1, false>(sR + n1 * n1, sX, f, p, [&](int k, double x) { Y[k] = __dadd_rn(Y[k], x); });
        }
      }
    }
    if (g0 + G == NCH) {  // last group: parent = R_0^(last) Z[0] + R_1^(last) Z[1]
      __syncthreads();
      double* out = a.q_dst + __ldg(a.dst_idx + fam) * a.stride;
      for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const int f = i / Nf, p = i - f * Nf;
        line_pair<DIM, N, DIM - 1>(sR, sZ, sR + n1 * n1, sZ + RP, f, p, out);
      }
    }
    __syncthreads();
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


// State health scan (dg_check_state; SPEC.md:193-194 positivity monitor, SPEC.md:740
// NaN -> numerical failure).  One warp per element row, grid-stride; per-warp counts
// and the smallest bad element reach the four global counters with one atomic each.
// Non-finite = exponent bits all ones (bitwise, no fast-math dependence).
__global__ void __launch_bounds__(256) k_check_state(const double* __restrict__ q, int64_t n_elem, int64_t stride,
                                                     int Np, int F, unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long nf = 0, nr = 0, nt = 0, first = ~0ull;
  for (int64_t e = w0; e < n_elem; e += nw) {
    const double* row = q + e * stride;
    unsigned c = 0, r = 0, t = 0;
    for (int i = lane; i < F * Np; i += 32) {
      const double v = __ldg(row + i);
      c += ((__double_as_longlong(v) & 0x7ff0000000000000ll) == 0x7ff0000000000000ll);
      if (i < Np) r += (v <= 0.0);
      else if (i >= (F - 1) * Np) t += (v <= 0.0);
    }
    const unsigned any = __ballot_sync(0xffffffffu, (c | r | t) != 0);
    if (any) {
      nf += c;
      nr += r;
      nt += t;
      if ((unsigned long long)e < first) first = (unsigned long long)e;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nf += __shfl_down_sync(0xffffffffu, nf, o);
    nr += __shfl_down_sync(0xffffffffu, nr, o);
    nt += __shfl_down_sync(0xffffffffu, nt, o);
  }
  if (lane == 0 && first != ~0ull) {
    atomicAdd(out + 0, nf);
    atomicAdd(out + 1, nr);
    atomicAdd(out + 2, nt);
    atomicMin(out + 3, first);
  }
}

// ---------------------------------------------------------------- dispatch
// Launch data is cached per device ordinal (attributes and occupancy are per device; a process
// may drive several).
constexpr int kMaxDev = 64;
int device_sms(int dev) {
  static std::atomic<int> sms[kMaxDev];
  int v = sms[dev].load(std::memory_order_acquire);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev].store(v, std::memory_order_release);
  }
  return v;
}

template <int DIM, int N>
int launch_transfer_t(int which, const TransferArgs& a, cudaStream_t s) {
  using C = Cfg<DIM, N>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  const int sms = device_sms(dev);
  if (which == 2) {
    constexpr int ROW2 = ((C::F * C::Np + 15) / 16 * 16) / 2;  // padded row (elem_stride) in 16-B granules
    const int64_t total = a.n * ROW2;
    const int64_t want = (total + 255) / 256;
    const int grid = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
    if (grid > 0) k_copy<ROW2><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (WarpXfer<DIM, N>::use) {
    using X_ = WarpXfer<DIM, N>;
    const size_t wb = sizeof(double) * X_::WS * X_::W * (which == 0 ? 1 : 2);  // coarsen: double-buffered
    static std::atomic<int> grid_w[kMaxDev][2];  // per device: the attribute and the occupancy are per device
    static std::mutex m;
    std::lock_guard<std::mutex> lk(m);
    if (grid_w[dev][which] == 0) {
      cudaError_t e = which == 0
                          ? cudaFuncSetAttribute(k_refine_w<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wb)
                          : cudaFuncSetAttribute(k_coarsen_w<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wb);
      if (e != cudaSuccess) return e;
      int occ = 0;
      e = which == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_refine_w<DIM, N>, 32 * X_::W, wb)
                     : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coarsen_w<DIM, N>, 32 * X_::W, wb);
      if (e != cudaSuccess) return e;
      grid_w[dev][which] = sms * (occ > 0 ? occ : 1);
    }
    const int64_t want = (a.n * C::F + X_::W - 1) / X_::W;
    const int gw = grid_w[dev][which];
    const int grid = (int)(want < gw ? want : gw);
    if (grid == 0) return cudaSuccess;
    if (which == 0) k_refine_w<DIM, N><<<grid, 32 * X_::W, wb, s>>>(a);
    else k_coarsen_w<DIM, N><<<grid, 32 * X_::W, wb, s>>>(a);
    return cudaGetLastError();
  }
  constexpr int R = C::F * C::Np, RP = (R + 1) & ~1, OPS = (2 * C::n1 * C::n1 + 1) & ~1;
  constexpr int STR = (R + 15) / 16 * 16, G = CoarsenG<DIM, N>::G;
  const size_t bytes = sizeof(double) * (which == 0 ? (OPS + RP + 2 * R + (DIM == 3 ? 4 * R : 0))
                                                    : (2 * G * STR + OPS + (G / 2 + 2) * RP));
  static std::atomic<int> grid_max[kMaxDev][2];
  static std::mutex m;
  std::lock_guard<std::mutex> lk(m);
  if (grid_max[dev][which] == 0) {
    cudaError_t e = which == 0
                        ? cudaFuncSetAttribute(k_refine<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)
                        : cudaFuncSetAttribute(k_coarsen<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = which == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_refine<DIM, N>, 256, bytes)
                   : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coarsen<DIM, N>, 256, bytes);
    if (e != cudaSuccess) return e;
    grid_max[dev][which] = sms * (occ > 0 ? occ : 1);
  }
  const int gm = grid_max[dev][which];
  const int grid = (int)(a.n < gm ? a.n : gm);
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

// NEXT-1 refinement indicator ("regridding ... based on potential
// temperature"; reading R39): one warp per element, eta_e = max over nodes of
// |Theta/rho - Theta_bar/rho_bar| (kind 0) or |rho - rho_bar| (kind 1), IEEE
// division and subtraction, exact max -- bit-identical to the plain definition.
__global__ void __launch_bounds__(256) k_amr_indicator(const double* __restrict__ q, int64_t n_elem, int64_t stride,
                                                      int Np, int nv, int fth, int kind,
                                                      const ElemDesc* __restrict__ desc,
                                                      const double* __restrict__ bg, double* __restrict__ eta) {
  const int lane = threadIdx.x & 31;
  for (int64_t e = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); e < n_elem; e += (int64_t)gridDim.x * 8) {
    const double* qe = q + e * stride;
    const int row0 = __ldg(&desc[e].bgrow);
    double m = 0.0;
    for (int n = lane; n < Np; n += 32) {
      const int row = row0 + n / nv;
      const double rb = __ldg(bg + 3 * row), rho = __ldg(qe + n);
      double v;
      if (kind == 0)
        v = fabs(__dsub_rn(__ddiv_rn(__ldg(qe + fth * Np + n), rho), __ddiv_rn(__ldg(bg + 3 * row + 1), rb)));
      else
        v = fabs(__dsub_rn(rho, rb));
      m = fmax(m, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) eta[e] = m;
  }
}

// NEXT-4 face-trace pack / unpack: one thread per (pair, field, face node)
__global__ void __launch_bounds__(256) k_face_pack(int dim, int n1, int dir, int64_t n, const int32_t* __restrict__ pairs,
                                                  double* __restrict__ q, double* __restrict__ buf, int64_t stride) {
  const int Nf = dim == 2 ? n1 : n1 * n1, Np = Nf * n1, F = dim + 2;
  const int64_t tot = n * F * Nf;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / (F * Nf);
    const int r = (int)(i - p * F * Nf), f = r / Nf, t = r - f * Nf;
    const int e = pairs[2 * p], face = pairs[2 * p + 1], d = face >> 1, side = (face & 1) ? n1 - 1 : 0;
    int node;  // face node t (tangential axes ascending, first fastest; R28)
    if (dim == 2) node = d == 0 ? side + n1 * t : t + n1 * side;
    else {
      const int t1 = t % n1, t2 = t / n1;
      node = d == 0 ? side + n1 * t1 + n1 * n1 * t2 : (d == 1 ? t1 + n1 * side + n1 * n1 * t2 : t1 + n1 * t2 + n1 * n1 * side);
    }
    double* qv = q + (int64_t)e * stride + f * Np + node;
    if (dir == 0) buf[i] = *qv;
    else *qv = buf[i];
  }
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

int launch_face_pack(int dim, int order, int dir, int64_t n, const int32_t* pairs, double* q, double* buf,
                     int64_t stride, void* stream) {
  if (n <= 0) return cudaSuccess;
  const int n1 = order + 1, Nf = dim == 2 ? n1 : n1 * n1;
  const int64_t tot = n * (dim + 2) * Nf;
  const int64_t blocks = std::min<int64_t>((tot + 255) / 256, 148 * 16);
  k_face_pack<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dim, n1, dir, n, pairs, q, buf, stride);
  return cudaGetLastError();
}

int launch_amr_indicator(int dim, int order, int kind, const double* q, int64_t n_elem, int64_t stride,
                         const ElemDesc* desc, const double* bg3, double* eta, void* stream) {
  if (n_elem <= 0) return cudaSuccess;
  const int n1 = order + 1, nv = dim == 2 ? n1 : n1 * n1, Np = nv * n1;
  const int64_t blocks = std::min<int64_t>((n_elem + 7) / 8, 148 * 16);
  k_amr_indicator<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(q, n_elem, stride, Np, nv, dim + 1, kind, desc,
                                                                      bg3, eta);
  return cudaGetLastError();
}

int launch_check_state(const double* q, int64_t n_elem, int64_t stride, int Np, int F, unsigned long long* out,
                       void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out, 0, 3 * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(out + 3, 0xff, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (n_elem <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n_elem + 7) / 8, 148 * 16);
  k_check_state<<<(unsigned)blocks, 256, 0, s>>>(q, n_elem, stride, Np, F, out);
  return cudaGetLastError();
}

}  // namespace dgi
