// dg_device.cuh -- device helpers shared by the stage kernels (dg_stage.cu: k_stage,
// k_stage_h7; dg_stage_h4.cu: k_stage_h4): PTX wrappers (mbarrier, bulk copies, cp.async),
// the point physics of the path (EOS in perturbation form, fluxes, Rusanov; PAPER.md:89-131,
// readings R2, R5-R7 of DESIGN.md), node / face index maps (R28) and the even-odd D
// contraction.  Everything is in an anonymous namespace: each translation unit gets its own
// copy (no device linking).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>

#include "dg_internal.h"

namespace dgi {
namespace {

// -DDG_DEBUG builds (compute-sanitizer is closed on this GPU pool): shared-memory index bounds
// checks and a bounded mbarrier wait; a failed check prints and traps.
#ifdef DG_DEBUG
#define DG_CHECK(cond)                                                                                   \
  do {                                                                                                   \
    if (!(cond)) {                                                                                       \
      printf("DG_DEBUG check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,       \
             (int)blockIdx.x, (int)threadIdx.x);                                                         \
      __trap();                                                                                          \
    }                                                                                                    \
  } while (0)
#else
#define DG_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
#ifdef DG_DEBUG
  for (long long spin = 0;; ++spin) {  // bounded: a lost transaction traps instead of hanging the GPU
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(smem_u32(m)), "r"(parity)
                 : "memory");
    if (ok) return;
    DG_CHECK(spin < (1ll << 26));
  }
#endif
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
// shared -> global bulk copy (TMA), completion tracked by bulk groups of the issuing thread
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// arrive on m once all of this thread's prior cp.async operations have completed (counts as one
// of the expected arrivals: .noinc)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* m) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

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
// Out-of-line slow path (|x| >= 1/32: rare) keeps the inlined EOS small.
__device__ __noinline__ double pow1pm1_slow(double x, double gamma) { return expm1(__dmul_rn(gamma, log1p(x))); }

// Horner (or, -DDG_ESTRIN, the Estrin form), else expm1(gamma log1p(x));
// exactly 0 at x = 0.
__device__ __forceinline__ double pow1pm1(double x, const StageArgs& a) {
  static_assert(kEosTerms >= 8, "Estrin layout below uses 8 terms");
  if (fabs(x) < 0.015625) {  // 8 terms: truncation < 1e-17 relative
    const double* c = a.eos_c;
#ifndef DG_ESTRIN  // Horner: one constant operand per FMA (measured 1 % faster than Estrin here)
    double p = __fma_rn(c[7], x, c[6]);
    p = __fma_rn(p, x, c[5]);
    p = __fma_rn(p, x, c[4]);
    p = __fma_rn(p, x, c[3]);
    p = __fma_rn(p, x, c[2]);
    p = __fma_rn(p, x, c[1]);
    p = __fma_rn(p, x, c[0]);
    return __dmul_rn(p, x);
#endif
    const double x2 = __dmul_rn(x, x), x4 = __dmul_rn(x2, x2);
    const double p0 = __fma_rn(c[1], x, c[0]), p1 = __fma_rn(c[3], x, c[2]);
    const double p2 = __fma_rn(c[5], x, c[4]), p3 = __fma_rn(c[7], x, c[6]);
    const double q0 = __fma_rn(p1, x2, p0), q1 = __fma_rn(p3, x2, p2);
    return __dmul_rn(__fma_rn(q1, x4, q0), x);
  }
  return pow1pm1_slow(x, a.gamma);
}

// 1/x for x > 0 normal: MUFU seed + two Newton steps (no special-case branches).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}
// sqrt(v) for v > 0 normal: MUFU rsqrt seed, one Newton step on 1/sqrt (-DDG_SQRT2: two), one on
// sqrt (the last step squares the relative error of the ~2^-45 estimate: full double precision;
// parity at R19 checked on the GPU, 0.5 % faster than two steps).
__device__ __forceinline__ double fast_sqrt(double v) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
  double e = __fma_rn(-__dmul_rn(v, y), y, 1.0);
  y = __fma_rn(__dmul_rn(0.5, y), e, y);
#ifdef DG_SQRT2
  e = __fma_rn(-__dmul_rn(v, y), y, 1.0);
  y = __fma_rn(__dmul_rn(0.5, y), e, y);
#endif
  const double sq = __dmul_rn(v, y);
  return __fma_rn(__fma_rn(-sq, sq, v), __dmul_rn(0.5, y), sq);
}

__device__ __forceinline__ Dv derive(const St& s, const StageArgs& a) {
  Dv o;
  o.rho = __dadd_rn(s.rb, s.rp);
  o.Th = __dadd_rn(s.Tb, s.Tp);
  o.Pp = __dmul_rn(s.Pb, pow1pm1(__dmul_rn(s.Tp, s.rTb), a));
  o.rinv = fast_rcp(o.rho);
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
  return __dadd_rn(fabs(ud), fast_sqrt(__dmul_rn(__dmul_rn(gamma, P), v.rinv)));
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

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// number of coarse-side (kind 2 = binary 10) and fine-side (kind 3 = binary 11)
// faces in a packed face-kind word
__device__ __forceinline__ int n_coarse_faces(int info) {
  const int hi = info & 0xAAA, lo = info & 0x555;
  return __popc(hi & ~(lo << 1));
}
__device__ __forceinline__ int n_fine_faces(int info) {
  const int hi = info & 0xAAA, lo = info & 0x555;
  return __popc(hi & (lo << 1));
}

// Local row of the launch's i-th element (element-list launches: dg_rhs_elems / dg_rk_stage_elems).
// LIST is a template parameter of the kernels, so the plain launch carries no cost.
template <bool LIST>
__device__ __forceinline__ int64_t elem_of(const StageArgs& a, int64_t i) { return LIST ? (int64_t)__ldg(a.list + i) : i; }

// ------------------------------------------------------------------ launch (host)
// Per-device launch data (dynamic shared memory attribute set, persistent grid size), one
// slot per (kernel, device): the attribute is per device, and a process may drive several.
struct LaunchCache {
  static constexpr int kMaxDev = 64;
  std::atomic<int> grid[kMaxDev];
  std::mutex m;
};

template <class KernelFn>
int launch_persistent(KernelFn k, const StageArgs& a, int threads, size_t bytes, int64_t n_tiles, cudaStream_t s,
                      LaunchCache& cache) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= LaunchCache::kMaxDev) return cudaErrorInvalidDevice;
  int grid_max = cache.grid[dev].load(std::memory_order_acquire);
  if (grid_max == 0) {
    std::lock_guard<std::mutex> lk(cache.m);
    grid_max = cache.grid[dev].load(std::memory_order_relaxed);
    if (grid_max == 0) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e != cudaSuccess) return e;
      int sms = 0, occ = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, bytes);
      if (e != cudaSuccess) return e;
      grid_max = sms * (occ > 0 ? occ : 1);
      cache.grid[dev].store(grid_max, std::memory_order_release);
    }
  }
  const int grid = (int)(n_tiles < grid_max ? n_tiles : grid_max);
  if (grid == 0) return cudaSuccess;
  k<<<grid, threads, bytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace
}  // namespace dgi
