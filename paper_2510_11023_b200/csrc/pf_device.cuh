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
      return 1.5 + 0.5 * tanh(u);
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
    // xor butterfly: every lane ends with the bitwise-same sum (IEEE add commutes)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (NT == 32) {
      __syncwarp();  // orders the warp's smem traffic like the block barrier does
      return make_double2(a, b);
    }
    const int w = threadIdx.x >> 5;
    double* slot = red + buf * 128;
    if ((threadIdx.x & 31) == 0) {
      slot[4 * w] = a;
      slot[4 * w + 1] = b;
    }
    __syncthreads();
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
      const double2 v = reinterpret_cast<const double2*>(slot)[2 * i];  // slot[4i], slot[4i+1]
      sa += v.x;
      sb += v.y;
    }
    buf ^= 1;
    return make_double2(sa, sb);
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
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
      d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    if (NT == 32) {
      __syncwarp();
      return make_double4(a, b, c, d);
    }
    const int w = threadIdx.x >> 5;
    double* slot = red + buf * 128;
    if ((threadIdx.x & 31) == 0) {
      slot[4 * w] = a;
      slot[4 * w + 1] = b;
      slot[4 * w + 2] = c;
      slot[4 * w + 3] = d;
    }
    __syncthreads();
    double sa = 0.0, sb = 0.0, sc = 0.0, sd = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
      const double2 v = reinterpret_cast<const double2*>(slot)[2 * i];
      const double2 u = reinterpret_cast<const double2*>(slot)[2 * i + 1];
      sa += v.x;
      sb += v.y;
      sc += u.x;
      sd += u.y;
    }
    buf ^= 1;
    return make_double4(sa, sb, sc, sd);
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
