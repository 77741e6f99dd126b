// Device-side primitives shared by every space: complex arithmetic,
// deterministic block reductions, coefficient functors, status words.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace pf {

// Optional phase timing of slice 0 (build with -DPF_PHASE_TIMING; read with
// pf_debug_phases).  Compiled out of the product library.
#ifdef PF_PHASE_TIMING
#ifndef PF_PHASE_SLICE
#define PF_PHASE_SLICE 0
#endif
__device__ long long g_phase[16];
__device__ long long g_phase_last;
__device__ long long g_phase_last_h;
// helper CTA of slice PF_PHASE_SLICE (uses the kernel's `helper` and `b`)
#define PF_TH(k)                                                     \
  do {                                                               \
    if (threadIdx.x == 0 && helper && b == PF_PHASE_SLICE) {         \
      const long long _t = clock64();                                \
      g_phase[(k)] += _t - g_phase_last_h;                           \
      g_phase_last_h = _t;                                           \
    }                                                                \
  } while (0)
#define PF_T(k)                                        \
  do {                                                 \
    if (threadIdx.x == 0 && blockIdx.x == PF_PHASE_SLICE) { \
      const long long _t = clock64();                  \
      g_phase[(k)] += _t - g_phase_last;               \
      g_phase_last = _t;                               \
    }                                                  \
  } while (0)
#else
#define PF_T(k) \
  do {          \
  } while (0)
#define PF_TH(k) \
  do {           \
  } while (0)
#endif

// Optional per-warp timeline of a few substeps of one slice CTA (build with
// -DPF_TRACE; read with pf_debug_trace).  Lane 0 of every warp stores clock64()
// at each trace point: unlike the thread-0 phase timers above this shows every
// warp's arrival at every barrier.  Compiled out of the product library.
#ifdef PF_TRACE
#ifndef PF_TRACE_SLICE
#define PF_TRACE_SLICE 1
#endif
#ifndef PF_TRACE_R0
#define PF_TRACE_R0 513
#endif
constexpr int TR_STEPS = 8, TR_POINTS = 64;
__device__ long long g_trace[8][TR_STEPS][TR_POINTS];
__device__ long long g_looptop[4096];  // clock64 at the loop top of every substep of the traced slice
#define PF_TR_TOP(r)                                                                              \
  do {                                                                                            \
    if ((int)blockIdx.x == PF_TRACE_SLICE && threadIdx.x == 0 && (r) < 4096) g_looptop[(r)] = clock64(); \
  } while (0)
#define PF_TR(tr, id)                                                                   \
  do {                                                                                  \
    if ((tr) >= 0 && (threadIdx.x & 31) == 0) g_trace[threadIdx.x >> 5][(tr)][(id)] = clock64(); \
  } while (0)
#else
#define PF_TR(tr, id) \
  do {                \
  } while (0)
#define PF_TR_TOP(r) \
  do {               \
  } while (0)
#endif

struct cd {
  double x, y;
};
__device__ __forceinline__ cd cmul(cd a, cd b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ cd cmulc(cd a, cd b) {  // a * conj(b)
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
__device__ __forceinline__ cd cadd(cd a, cd b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cd csub(cd a, cd b) { return {a.x - b.x, a.y - b.y}; }

// radix-4 DFT in place (forward: exp(-2 pi i / 4) = -i; INV: conjugate)
template <bool INV>
__device__ __forceinline__ void dft4(cd& a0, cd& a1, cd& a2, cd& a3) {
  const cd t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = csub(a1, a3);
  const cd mi3 = {t3.y, -t3.x};  // -i t3
  a0 = cadd(t0, t2);
  a1 = INV ? csub(t1, mi3) : cadd(t1, mi3);
  a2 = csub(t0, t2);
  a3 = INV ? cadd(t1, mi3) : csub(t1, mi3);
}

// ---------------------------------------------------------------------------
// fast FP64 scalars for the latency-bound substep chain (branch-free, so the
// compiler interleaves the independent evaluations of a thread)
// ---------------------------------------------------------------------------
// 1/a for normal a (no zero / inf / denormal handling): MUFU.RCP64H seed (~20 bits)
// + two Newton steps, <= 1 ulp.  The callers' operands are sums of positive terms.
__device__ __forceinline__ double rcp_fast(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double e = fma(-a, y, 1.0);
  y = fma(y, e, y);
  e = fma(-a, y, 1.0);
  return fma(y, e, y);
}

// tanh(u) to ~2e-16 ABSOLUTE error (not relative: for D = 1.5 + 0.5 tanh(u) the
// absolute error is what reaches the coefficient, at its rounding level):
// 1 - 2 / (exp(2|u|) + 1), exp by range reduction to |r| <= ln2/2 and a degree-12
// Taylor polynomial, no branches (CUDA's tanh has a small-|u| branch that diverges
// across a slice's grid points and serialises a thread's four evaluations).
__device__ __forceinline__ double tanh_abs(double u) {
  const double x = fmin(2.0 * fabs(u), 80.0);
  const double kd = fma(x, 1.4426950408889634, 6755399441055744.0);  // 1.5 * 2^52: round to nearest integer
  const int k = __double2loint(kd);
  const double n = kd - 6755399441055744.0;
  double r = fma(n, -6.93147180369123816490e-01, x);  // ln2 hi
  r = fma(n, -1.90821492927058770002e-10, r);          // ln2 lo
  double p = 1.0 / 479001600.0;
  p = fma(p, r, 1.0 / 39916800.0);
  p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0);
  p = fma(p, r, 1.0 / 40320.0);
  p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);  // exp(r)
  // exp(x) = p * 2^k, k in [0, 116]: add k to the exponent field
  const double e = __hiloint2double(__double2hiint(p) + (k << 20), __double2loint(p));
  const double t = fma(-2.0, rcp_fast(e + 1.0), 1.0);
  return copysign(t, u);
}

// ---------------------------------------------------------------------------
// status: one word per CTA, decoded on the host into pf_error
// ---------------------------------------------------------------------------
enum StatusCode : int { ST_OK = 0, ST_SOLVER = 2, ST_COEFF = 3, ST_DIVERGE = 4, ST_CANCEL = 9 };

struct Status {
  int code;   // StatusCode
  int n;      // slice / coarse step
  int r;      // substep (-1 for coarse)
  int node;   // coefficient node
  int iters;  // PCG iterations accumulated by this CTA
  int solves; // linear solves performed by this CTA
  int pad[2];
  long long t_start, t_end;  // fine-sweep slice CTAs: globaltimer at entry / exit (load-balance diagnostic)
};

// ---------------------------------------------------------------------------
// coefficient functors (include/parafrac_b200.h PF_FN_*)
// ---------------------------------------------------------------------------
struct Fn {
  int id;
  double p[6];
};

__device__ __forceinline__ double fn_D(const Fn& f, double x, double x2, double t, double u) {
  switch (f.id) {
    case 1:  // PF_FN_POLY
      return f.p[0] + f.p[1] * u;
    case 2: {  // PF_FN_CFG12
      const double u2 = u * u;
      return 1.0 + u2 / (1.0 + u2);
    }
    case 3:  // PF_FN_CFG3
      return 1.5 + 0.5 * tanh_abs(u);
    case 4: {  // PF_FN_CFG45
      const double s = sin(u);
      return (1.0 + 0.5 * x) * (1.0 + 0.5 * (s * s));
    }
    case 5:  // PF_FN_NAN_AT
      return fabs(x - f.p[0]) < 1e-12 ? CUDART_NAN : f.p[1];
    default:
      return CUDART_NAN;
  }
}

// x-only factors are tabulated once per kernel (sx = {sin(pi x), sin(2 pi x)})
// and exp(-t) once per substep (emt), so the per-point cost is the u-dependent part.
__device__ __forceinline__ double2 fn_xtab(double x) { return make_double2(sin(CUDART_PI * x), sin(2.0 * CUDART_PI * x)); }

__device__ __forceinline__ double fn_f(const Fn& f, double2 sx, double emt, double u) {
  switch (f.id) {
    case 1:
      return __dadd_rn(__dmul_rn(f.p[2], u), __dmul_rn(f.p[3], __dmul_rn(sx.x, emt)));
    case 2:
      return sx.x * cos(u);
    case 3:
      return -u + 0.1 * sx.y;
    case 4: {
      const double u2 = u * u;
      return u * (1.0 - u2) / (1.0 + u2);
    }
    default:
      return 0.0;
  }
}

// ---------------------------------------------------------------------------
// deterministic block reductions (fixed order; every thread gets the total)
// `red` holds 2 buffers x 32 warps x 4 values (RED_DOUBLES).  One __syncthreads each.
// ---------------------------------------------------------------------------
constexpr int RED_DOUBLES = 256;

template <int NT>
struct Reducer {
  double* red;
  int buf;
  __device__ void init(double* scratch) {
    red = scratch;
    buf = 0;
  }
  __device__ __forceinline__ double2 sum2(double a, double b) {
    if (NT == 32) {
      // xor butterfly: every lane ends with the bitwise-same sum (IEEE add commutes)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      __syncwarp();  // orders the warp's smem traffic like the block barrier does
      return make_double2(a, b);
    }
    // Split butterfly (the same xor-16, 8, 4, 2, 1 tree per value, so the sums are bitwise the
    // full butterfly's): in the first round the lower half-warp keeps summing a and hands its b
    // over, the upper half the other way round -- one 64-bit shuffle per round instead of two;
    // lane 0 ends with the warp's a, lane 16 with its b.
    const int lane = threadIdx.x & 31;
    {
      const bool up = (lane & 16) != 0;
      const double send = up ? a : b;
      double keep = up ? b : a;
      keep += __shfl_xor_sync(0xffffffffu, send, 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) keep += __shfl_xor_sync(0xffffffffu, keep, o);
      a = keep;
    }
    const int w = threadIdx.x >> 5;
    double* slot = red + buf * 128;
    if ((lane & 15) == 0) slot[4 * w + (lane >> 4)] = a;
    __syncthreads();
    // pairwise (fixed-shape) tree over the warps' partials: log2(NT/32) dependent adds
    double2 v[NT / 32];
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) v[i] = reinterpret_cast<const double2*>(slot)[2 * i];  // slot[4i], slot[4i+1]
#pragma unroll
    for (int w2 = NT / 64; w2 > 0; w2 >>= 1)
#pragma unroll
      for (int i = 0; i < w2; ++i) {
        v[i].x += v[i + w2].x;
        v[i].y += v[i + w2].y;
      }
    buf ^= 1;
    return v[0];
  }
  __device__ __forceinline__ double3 sum3(double a, double b, double c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (NT == 32) {
      __syncwarp();
      return make_double3(a, b, c);
    }
    const int w = threadIdx.x >> 5;
    double* slot = red + buf * 128;
    if ((threadIdx.x & 31) == 0) {
      slot[4 * w] = a;
      slot[4 * w + 1] = b;
      slot[4 * w + 2] = c;
    }
    __syncthreads();
    double sa = 0.0, sb = 0.0, sc = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
      sa += slot[4 * i];
      sb += slot[4 * i + 1];
      sc += slot[4 * i + 2];
    }
    buf ^= 1;
    return make_double3(sa, sb, sc);
  }
  __device__ __forceinline__ double4 sum4(double a, double b, double c, double d) {
    if (NT == 32) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
        d += __shfl_xor_sync(0xffffffffu, d, o);
      }
      __syncwarp();
      return make_double4(a, b, c, d);
    }
    // split butterfly (see sum2): round xor-16 halves the four values to two per lane, round
    // xor-8 to one; lanes 0, 8, 16, 24 end with the warp's a, b, c, d -- 6 shuffles, not 20
    const int lane = threadIdx.x & 31;
    {
      const bool up16 = (lane & 16) != 0, up8 = (lane & 8) != 0;
      // lower half keeps (a, b), upper half keeps (c, d)
      double k0 = up16 ? c : a, k1 = up16 ? d : b;
      const double s0 = up16 ? a : c, s1 = up16 ? b : d;
      k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
      // within a half: lanes with bit 3 clear keep k0, the others k1
      double keep = up8 ? k1 : k0;
      const double send = up8 ? k0 : k1;
      keep += __shfl_xor_sync(0xffffffffu, send, 8);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) keep += __shfl_xor_sync(0xffffffffu, keep, o);
      a = keep;  // lane 0: a, lane 8: b, lane 16: c, lane 24: d
    }
    const int w = threadIdx.x >> 5;
    double* slot = red + buf * 128;
    if ((lane & 7) == 0) slot[4 * w + (lane >> 3)] = a;
    __syncthreads();
    double2 v[NT / 32], u[NT / 32];
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
      v[i] = reinterpret_cast<const double2*>(slot)[2 * i];
      u[i] = reinterpret_cast<const double2*>(slot)[2 * i + 1];
    }
#pragma unroll
    for (int w2 = NT / 64; w2 > 0; w2 >>= 1)
#pragma unroll
      for (int i = 0; i < w2; ++i) {
        v[i].x += v[i + w2].x;
        v[i].y += v[i + w2].y;
        u[i].x += u[i + w2].x;
        u[i].y += u[i + w2].y;
      }
    buf ^= 1;
    return make_double4(v[0].x, v[0].y, u[0].x, u[0].y);
  }
  __device__ __forceinline__ double sum(double a) { return sum2(a, 0.0).x; }
  __device__ __forceinline__ double max(double a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (NT == 32) {
      __syncwarp();
      return a;
    }
    const int w = threadIdx.x >> 5;
    double* slot = red + buf * 128;
    if ((threadIdx.x & 31) == 0) slot[4 * w] = a;
    __syncthreads();
    double s = slot[0];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) s = fmax(s, slot[4 * i]);
    buf ^= 1;
    return s;
  }
  // smallest integer over the block (error indices); INT_MAX = none
  __device__ __forceinline__ int min_int(int a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (NT == 32) {
      __syncwarp();
      return a;
    }
    const int w = threadIdx.x >> 5;
    double* slot = red + buf * 128;
    if ((threadIdx.x & 31) == 0) slot[4 * w] = (double)a;
    __syncthreads();
    double s = slot[0];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) s = fmin(s, slot[4 * i]);
    buf ^= 1;
    return (int)s;
  }
};

}  // namespace pf
