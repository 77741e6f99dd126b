// 2-D line engine for Q = 256 (config 4: 128^2 modes on a 256^2 grid) with
// register-resident FFTs.
//
// The radix-4 Stockham line FFT of pf_sine2d.cuh moves every element through
// shared memory once per pass (4 passes at Q = 256) with a CTA barrier
// between passes, and the 2-D kernels are shared-memory bound.  Here a line
// is 16 lanes of one half-warp and the length-256 DFT is 16 x 16:
//
//   X[k1 + 16 k2] = sum_n2 w256^(n2 k1) w16^(n2 k2) sum_n1 x[16 n1 + n2] w16^(n1 k1)
//
// lane n2 holds x[16 n1 + n2] (n1 = 0..15), does a 16-point DFT in registers,
// multiplies by w256^(n2 k1), the half-warp transposes through shared memory
// (swizzled, conflict-free, __syncwarp only), and lane k1 does the second
// 16-point DFT: it ends holding X[k1 + 16 k2], k2 = 0..15 -- which is exactly
// the input layout of the next transform, so the PCG matvec's
// synthesis -> pointwise -> analysis chain never leaves registers.  One
// shared-memory round trip per FFT instead of four, no CTA barriers inside.
//
// The transform pairs (DCT-III/II via one complex FFT, Makhoul reordering)
// and the data layouts are those of pf_sine2d.cuh; only the FFT changes, so
// results agree with the radix-4 engine to rounding (both are checked against
// oracle.Sine2D).
#pragma once
#include "pf_sine2d.cuh"

namespace pf {

// TLV lines per CTA (a half-warp each): 16 for batched sweeps, 4 for batch-1
// coarse solves (4x the CTAs: the kernels are latency-bound there)
template <int TLV>
struct L16T {
  static constexpr int LG = 8, Q = 256, M = 128, TL = TLV, NT = 16 * TLV;
  static constexpr int LS = Q + 1;  // line stride in cd (odd: staged tile writes are conflict-free)
  static constexpr int STP = TL + 1;  // stage row stride in doubles
  static constexpr double SQ2 = 1.4142135623730951;
  static size_t smem_bytes() {
    const size_t lines = sizeof(cd) * TL * LS, stage = sizeof(double) * 2 * Q * STP;
    return sizeof(cd) * (256 + Q) + (lines > stage ? lines : stage);
  }
};
using L16 = L16T<16>;

// multiply by w16^m (forward w = exp(-2 pi i / 16); INV: conjugate), m in {1,2,3,4,6,9}
template <bool INV, int MM>
__device__ __forceinline__ cd w16mul(cd a) {
  constexpr double C = 0.92387953251128674, S = 0.38268343236508978, R = 0.70710678118654752;
  constexpr double wr = MM == 1 ? C : MM == 2 ? R : MM == 3 ? S : MM == 4 ? 0.0 : MM == 6 ? -R : -C;
  constexpr double wi0 = MM == 1 ? -S : MM == 2 ? -R : MM == 3 ? -C : MM == 4 ? -1.0 : MM == 6 ? -R : S;
  constexpr double wi = INV ? -wi0 : wi0;
  if constexpr (MM == 4) {
    return INV ? cd{-a.y, a.x} : cd{a.y, -a.x};
  } else {
    return {a.x * wr - a.y * wi, a.x * wi + a.y * wr};
  }
}

// in-place 16-point DFT, natural order in and out: v[n] -> X[k] = sum_n v[n] w16^(nk)
template <bool INV>
__device__ __forceinline__ void dft16(cd (&v)[16]) {
  // n = 4a + b, k = c + 4d: DFT4 over a for each b, twiddle w16^(bc), DFT4 over b for each c
#pragma unroll
  for (int b = 0; b < 4; ++b) dft4<INV>(v[b], v[4 + b], v[8 + b], v[12 + b]);  // v[4c + b] = y[b][c]
  v[4 + 1] = w16mul<INV, 1>(v[4 + 1]);
  v[4 + 2] = w16mul<INV, 2>(v[4 + 2]);
  v[4 + 3] = w16mul<INV, 3>(v[4 + 3]);
  v[8 + 1] = w16mul<INV, 2>(v[8 + 1]);
  v[8 + 2] = w16mul<INV, 4>(v[8 + 2]);
  v[8 + 3] = w16mul<INV, 6>(v[8 + 3]);
  v[12 + 1] = w16mul<INV, 3>(v[12 + 1]);
  v[12 + 2] = w16mul<INV, 6>(v[12 + 2]);
  v[12 + 3] = w16mul<INV, 9>(v[12 + 3]);
#pragma unroll
  for (int c = 0; c < 4; ++c) dft4<INV>(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);  // v[4c + d] = X[c + 4d]
  // transpose 4x4 to natural order: X[c + 4d] sits at v[4c + d]
  cd t;
  t = v[1]; v[1] = v[4]; v[4] = t;
  t = v[2]; v[2] = v[8]; v[8] = t;
  t = v[3]; v[3] = v[12]; v[12] = t;
  t = v[6]; v[6] = v[9]; v[9] = t;
  t = v[7]; v[7] = v[13]; v[13] = t;
  t = v[11]; v[11] = v[14]; v[14] = t;
}

// Length-256 DFT of one line by its 16 lanes.  Entry: v[n1] = x[16 n1 + l].
// Exit: v[k2] = X[l + 16 k2].  `buf` (this line's 256 cd) is scratch for the
// transpose; `T[k1 * 16 + n2]` = w256^(k1 n2) (forward).
template <bool INV>
__device__ __forceinline__ void fft256(cd (&v)[16], cd* buf, const cd* T, int l) {
  dft16<INV>(v);  // v[k1] = Y_l[k1]
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) {
    cd w = T[k1 * 16 + l];
    if (INV) w.y = -w.y;
    v[k1] = cmul(v[k1], w);
  }
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 16 + (l ^ k1)] = v[k1];
  __syncwarp();
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) v[n2] = buf[l * 16 + (n2 ^ l)];
  __syncwarp();
  dft16<INV>(v);
}

// synth_write / anal_read of pf_sine2d.cuh on an unswizzled line
__device__ __forceinline__ void synth_write_plain(cd* W, const cd* ph, int k, double av, double bv) {
  constexpr int Q = L16::Q, M = L16::M;
  if (k < M) {
    const cd p = ph[k], pq = ph[Q - k];
    const cd v1 = {p.y * av, -p.x * av};
    const cd v2 = {p.x * bv, p.y * bv};
    W[k] = {v1.x - v2.y, v1.y + v2.x};
    const cd u1 = {pq.x * av, pq.y * av};
    const cd u2 = {pq.y * bv, -pq.x * bv};
    W[Q - k] = {u1.x - u2.y, u1.y + u2.x};
  } else {
    const cd p = ph[M];
    const cd v1 = {p.x * av + p.y * av, p.y * av - p.x * av};
    const cd v2 = {p.x * bv + p.y * bv, p.y * bv - p.x * bv};
    W[M] = {v1.x - v2.y, v1.y + v2.x};
  }
}

__device__ __forceinline__ double2 anal_read_plain(const cd* Z, const cd* ph, int Q, int k) {
  const cd a = Z[k], b = Z[Q - k], c = ph[k], c2 = ph[Q - k];
  const double Dx = a.x - b.x, Dy = a.y + b.y;
  return make_double2(0.5 * (c2.x * (b.x + a.x) + c2.y * (b.y - a.y)), 0.5 * (c.x * Dy - c.y * Dx));
}

// grid point of FFT position j (Makhoul reordering, pf_sine2d.cuh)
__device__ __forceinline__ int q_of_pos(int pos) { return pos < 128 ? 2 * pos : 2 * (255 - pos) + 1; }
__device__ __forceinline__ int pos_of_q(int q) { return (q & 1) ? (255 - (q >> 1)) : (q >> 1); }

__device__ __forceinline__ void l16_setup(char* smem, const Sine2DArgs& a, cd*& T, cd*& ph, cd*& lines) {
  T = reinterpret_cast<cd*>(smem);
  ph = T + 256;
  lines = ph + L16::Q;
  for (int j = threadIdx.x; j < 256; j += blockDim.x) T[j] = a.tw16[j];
  for (int j = threadIdx.x; j < L16::Q; j += blockDim.x) ph[j] = a.ph[j];
  __syncthreads();
}

// synthesis-pair input of one line (lane-strided modes), then the lane's FFT inputs
__device__ __forceinline__ void l16_load(const cd* W, int l, cd (&v)[16]) {
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) v[n1] = W[16 * n1 + l];
}

// ---------------------------------------------------------------------------
// Shuffle-based synthesis input and analysis output (no shared-memory round
// trip).  Lane l of a line owns the modes k = l + 16 i (l >= 1, i = 0..7) or
// k = 16 i (lane 0, i = 1..8) -- a partition of 1..M.  The fft256 input slot
// j = 16 n1 + l carries mode j (j < M) or mode Q - j (j > M); the output Z[k]
// sits in lane k % 16, register k / 16.  So slot n1 < 8 of lane l is its own
// mode i = n1, slot n1 >= 8 is own mode 15 - n1 of lane 16 - l (lane 0: its
// own mode 16 - n1), and the analysis partner Z[Q - k] of own mode i is
// register 15 - i of lane 16 - l (lane 0: its own register 16 - i).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int l16_own_mode(int i, int l) {
  return l == 0 ? 16 * i : (i < 8 ? l + 16 * i : 0);  // 0: no mode in this slot
}

__device__ __forceinline__ int l16_partner(int l) { return ((int)threadIdx.x & 16) | ((16 - l) & 15); }

// slot j != 0 of a synthesis pair from its mode's (av, bv) (synth_write_plain per slot; ph[j] is
// the phase of slot j in both halves)
__device__ __forceinline__ cd l16_slot(int j, cd p, double av, double bv) {
  if (j < L16::M) {
    const cd v1 = {p.y * av, -p.x * av}, v2 = {p.x * bv, p.y * bv};
    return {v1.x - v2.y, v1.y + v2.x};
  }
  if (j == L16::M) {
    const cd v1 = {p.x * av + p.y * av, p.y * av - p.x * av}, v2 = {p.x * bv + p.y * bv, p.y * bv - p.x * bv};
    return {v1.x - v2.y, v1.y + v2.x};
  }
  const cd u1 = {p.x * av, p.y * av}, u2 = {p.y * bv, -p.x * bv};
  return {u1.x - u2.y, u1.y + u2.x};
}

// fft256 input v[n1] = W[16 n1 + l] of a synthesis pair from the lane's own (av, bv)
__device__ __forceinline__ void l16_synth_own(const double (&av)[9], const double (&bv)[9], const cd* ph, int l,
                                              cd (&v)[16]) {
  const int src = l16_partner(l);
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) {
    const int j = 16 * n1 + l;
    double A, B;
    if (n1 < 8) {
      A = av[n1];
      B = bv[n1];
    } else {
      const double pa = __shfl_sync(0xffffffffu, av[15 - n1], src);
      const double pb = __shfl_sync(0xffffffffu, bv[15 - n1], src);
      A = l == 0 ? av[16 - n1] : pa;
      B = l == 0 ? bv[16 - n1] : pb;
    }
    v[n1] = j == 0 ? cd{0.0, 0.0} : l16_slot(j, ph[j], A, B);
  }
}

// analysis pair of the lane's own modes from the fft256 output v[i] = Z[l + 16 i]:
// emit(i, k, X1, X2) with X1 the sine (S^T) and X2 the cosine (S'^T / (sqrt2 pi k)) part
template <class F>
__device__ __forceinline__ void l16_anal_own(const cd (&v)[16], const cd* ph, int l, F&& emit) {
  const int src = l16_partner(l);
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    cd b = {0.0, 0.0};
    if (i < 8) {
      b.x = __shfl_sync(0xffffffffu, v[15 - i].x, src);
      b.y = __shfl_sync(0xffffffffu, v[15 - i].y, src);
    }
    const int k = l16_own_mode(i, l);
    if (k == 0) continue;
    if (l == 0) b = v[16 - i];
    const cd a = v[i], c = ph[k], c2 = ph[L16::Q - k];
    const double Dx = a.x - b.x, Dy = a.y + b.y;
    emit(i, k, 0.5 * (c2.x * (b.x + a.x) + c2.y * (b.y - a.y)), 0.5 * (c.x * Dy - c.y * Dx));
  }
}

// ---------------------------------------------------------------------------
// rows, synthesis (along y): lines k1 -> H[q2][k1] (same contract as k2_rows_syn)
// ---------------------------------------------------------------------------
template <bool SETUP, int TLV = 16>
__global__ void __launch_bounds__(16 * TLV) k2_rows_syn16(Sine2DArgs a) {
  using L = L16T<TLV>;
  extern __shared__ __align__(16) char smem[];
  const int b = blockIdx.y;
  if (!SETUP && a.sc[b * 16 + S_DONE] != 0.0) return;
  cd *T, *ph, *lines;
  l16_setup(smem, a, T, ph, lines);
  const int line = threadIdx.x >> 4, l = threadIdx.x & 15;
  const int k1b = blockIdx.x * L::TL;
  const int k1 = k1b + line + 1;
  cd* W = lines + line * L::LS;
  const size_t row = (size_t)(k1 - 1) * L::M;
  const size_t MM = (size_t)L::M * L::M;
  const double beta = SETUP ? 0.0 : a.sc[b * 16 + S_BETA];
  const double dbar = a.sc[b * 16 + S_DBAR];
  double* st_s = reinterpret_cast<double*>(lines);
  double* st_c = st_s + L::Q * L::STP;
  constexpr int NF = SETUP ? 2 : 1;
  for (int f = 0; f < NF; ++f) {
    // own-mode loads first (the P stores below would otherwise order them one by one)
    double ld1[9], ld2[9], av[9], bv[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const int k = l16_own_mode(i, l);
      ld1[i] = ld2[i] = 0.0;
      if (k > 0) {
        const size_t e = row + k - 1;
        if (SETUP) {
          ld1[i] = a.X0[b * a.sX0 + e];
          ld2[i] = f == 0 ? a.Cp[b * a.sCp + e] : 0.0;
        } else {
          ld1[i] = a.P[(size_t)b * MM + e];
          ld2[i] = a.R[(size_t)b * MM + e];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const int k = l16_own_mode(i, l);
      av[i] = bv[i] = 0.0;
      if (k == 0) continue;
      if (SETUP) {
        if (f == 0) {
          av[i] = L::SQ2 * ld2[i];
          bv[i] = L::SQ2 * CUDART_PI * (double)k * ld1[i];
        } else {
          av[i] = L::SQ2 * ld1[i];
        }
      } else {
        const double pn = fma(beta, ld1[i], pinv2d(a.gam, dbar, k1, k) * ld2[i]);  // p = z + beta p
        a.P[(size_t)b * MM + row + k - 1] = pn;
        av[i] = L::SQ2 * pn;
        bv[i] = L::SQ2 * CUDART_PI * (double)k * pn;
      }
    }
    cd v[16];
    l16_synth_own(av, bv, ph, l, v);
    fft256<true>(v, W, T, l);
    __syncthreads();  // every line is done with its buffer: reuse the lines as the stage
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const int q = q_of_pos(l + 16 * k2);
      st_s[q * L::STP + line] = (q & 1) ? -0.5 * v[k2].x : 0.5 * v[k2].x;
      st_c[q * L::STP + line] = 0.5 * v[k2].y;
    }
    __syncthreads();
    double* d_s = SETUP ? (f == 0 ? a.Hu : a.Hs) : a.Hs;
    double* d_c = SETUP ? (f == 0 ? a.Hc : nullptr) : a.Hc;
    for (int e = threadIdx.x; e < L::TL * L::Q; e += L::NT) {
      const int q2 = e / L::TL, ll = e % L::TL;
      const size_t o = ((size_t)b * L::Q + q2) * L::M + k1b + ll;
      d_s[o] = st_s[q2 * L::STP + ll];
      if (d_c) d_c[o] = st_c[q2 * L::STP + ll];
    }
    __syncthreads();
  }
}

// setup pointwise of one column line at the lane's 16 grid points: u, Gx from
// the first synthesis FFT (v1), Gy from the second (v2) -> D on the grid, the
// inputs of the analysis FFTs (v1 <- (g, d Gx), x4 <- d Gy), dbar partial
template <int FID>
__device__ __forceinline__ void l16_pointwise(const Sine2DArgs& a, int q2, double t, double emt, size_t gl,
                                              cd (&v1)[16], const cd (&v2)[16], double (&x4)[16], double& dsum,
                                              int& bad) {
  const double wq = 1.0 / ((double)L16::Q * (double)L16::Q);
  const int l = threadIdx.x & 15;
  Fn f1 = a.fn;
  if (FID != 0) f1.id = FID;  // constant-folds the functor switches
  const double y2 = a.xq[q2];
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) {
    const int q1 = q_of_pos(l + 16 * k2);
    const double u = (q1 & 1) ? -0.5 * v1[k2].x : 0.5 * v1[k2].x;
    const double gx = 0.5 * v1[k2].y;
    const double gy = (q1 & 1) ? -0.5 * v2[k2].x : 0.5 * v2[k2].x;
    const double x1 = a.xq[q1];
    const double Dv = fn_D(f1, x1, y2, t, u);
    if (!isfinite(Dv)) bad = min(bad, q1 * L16::Q + q2);  // oracle.Sine2D flat index [x1][x2]
    const double d = wq * Dv;
    const double g = wq * (f1.id == 4 ? fn_f(f1, make_double2(0.0, 0.0), emt, u) : fn_f(f1, fn_xtab(x1), emt, u));
    a.D[gl + q1] = d;
    dsum += d;
    const double sp4 = d * gy;
    v1[k2] = {(q1 & 1) ? -g : g, d * gx};
    x4[k2] = (q1 & 1) ? -sp4 : sp4;  // FFT4 input is real
  }
}

// ---------------------------------------------------------------------------
// columns (along x) for lines q2 (same contract as k2_cols)
// ---------------------------------------------------------------------------
template <bool SETUP, int TLV = 16>
__global__ void __launch_bounds__(16 * TLV, TLV == 16 ? 2 : 1) k2_cols16(Sine2DArgs a) {
  using L = L16T<TLV>;
  extern __shared__ __align__(16) char smem[];
  const int b = blockIdx.y;
  if (!SETUP && a.sc[b * 16 + S_DONE] != 0.0) return;
  cd *T, *ph, *lines;
  l16_setup(smem, a, T, ph, lines);
  const int line = threadIdx.x >> 4, l = threadIdx.x & 15;
  const int q2 = blockIdx.x * L::TL + line;
  cd* W = lines + line * L::LS;
  const size_t hl = ((size_t)b * L::Q + q2) * L::M;
  const size_t gl = ((size_t)b * L::Q + q2) * L::Q;
  // synthesis pair (A, pi k Bk) of the line's modes -> fft256 input v
  auto synth = [&](const double* A, const double* Bk, cd (&v)[16]) {
    double av[9], bv[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const int k = l16_own_mode(i, l);
      av[i] = k > 0 ? A[hl + k - 1] : 0.0;
      bv[i] = (k > 0 && Bk) ? Bk[hl + k - 1] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const int k = l16_own_mode(i, l);
      av[i] = L::SQ2 * av[i];
      bv[i] = L::SQ2 * CUDART_PI * (double)k * bv[i];
    }
    l16_synth_own(av, bv, ph, l, v);
  };
  if (!SETUP) {
    // the coefficient loads are independent of the transform: issue them first
    double dv[16];
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) dv[k2] = a.D[gl + q_of_pos(l + 16 * k2)];
    cd v[16];
    synth(a.Hc, a.Hs, v);
    fft256<true>(v, W, T, l);
    // pointwise: Z_pos = (0.5 d_q) W_pos (see k2_cols)
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const double d = 0.5 * dv[k2];
      v[k2] = {d * v[k2].x, d * v[k2].y};
    }
    fft256<false>(v, W, T, l);
    l16_anal_own(v, ph, l, [&](int, int k, double X1, double X2) {
      a.Ay[hl + k - 1] = L::SQ2 * X1;
      a.Ax[hl + k - 1] = L::SQ2 * CUDART_PI * (double)k * X2;
    });
    return;
  }
  // setup: FFT1 (Hu, pi k Hs) -> u, Gx; FFT2 (Hc) -> Gy; coefficients; FFT3 (g, Yx); FFT4 (Yy)
  const double wq = 1.0 / ((double)L::Q * (double)L::Q);
  const double t = (double)(a.n0 + b) * a.dTs + a.tr;
  const double emt = a.fn.id == 1 ? exp(-t) : 0.0;
  cd v1[16], v2[16];
  synth(a.Hu, a.Hs, v1);
  fft256<true>(v1, W, T, l);
  synth(a.Hc, nullptr, v2);
  fft256<true>(v2, W, T, l);
  double dsum = 0.0;
  int bad = 0x7fffffff;
  double x4[16];
  // one functor switch outside the point loop: each functor's loop is straight-line code
  switch (a.fn.id) {
    case 1: l16_pointwise<1>(a, q2, t, emt, gl, v1, v2, x4, dsum, bad); break;
    case 2: l16_pointwise<2>(a, q2, t, emt, gl, v1, v2, x4, dsum, bad); break;
    case 3: l16_pointwise<3>(a, q2, t, emt, gl, v1, v2, x4, dsum, bad); break;
    case 4: l16_pointwise<4>(a, q2, t, emt, gl, v1, v2, x4, dsum, bad); break;
    default: l16_pointwise<0>(a, q2, t, emt, gl, v1, v2, x4, dsum, bad); break;
  }
  fft256<false>(v1, W, T, l);
  l16_anal_own(v1, ph, l, [&](int, int k, double X1, double X2) {
    a.Ag[hl + k - 1] = L::SQ2 * X1;
    a.Ax[hl + k - 1] = L::SQ2 * CUDART_PI * (double)k * X2;
  });
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) v2[k2] = {x4[k2], 0.0};
  fft256<false>(v2, W, T, l);
  l16_anal_own(v2, ph, l, [&](int, int k, double X1, double) { a.Ay[hl + k - 1] = L::SQ2 * X1; });
  // line partial of dbar: fixed-order butterfly over the line's 16 lanes
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
  if (l == 0) a.part[((size_t)b * L::Q + q2) * 4 + 0] = dsum;
  if (bad != 0x7fffffff) atomicMin(a.bad + b, bad);
}

// ---------------------------------------------------------------------------
// rows, analysis (along y) for lines k1 (same contract as k2_rows_ana)
// ---------------------------------------------------------------------------
template <bool SETUP, int TLV = 16>
__global__ void __launch_bounds__(16 * TLV) k2_rows_ana16(Sine2DArgs a) {
  using L = L16T<TLV>;
  extern __shared__ __align__(16) char smem[];
  const int b = blockIdx.y;
  if (!SETUP && a.sc[b * 16 + S_DONE] != 0.0) return;
  cd *T, *ph, *lines;
  l16_setup(smem, a, T, ph, lines);
  const int line = threadIdx.x >> 4, l = threadIdx.x & 15;
  const int k1b = blockIdx.x * L::TL;
  const int k1 = k1b + line + 1;
  cd* W = lines + line * L::LS;
  const size_t MM = (size_t)L::M * L::M;
  const size_t row = (size_t)(k1 - 1) * L::M;
  constexpr int MPL = 9;  // own modes l16_own_mode(i, l)
  double kv[MPL], fv[MPL];
#pragma unroll
  for (int i = 0; i < MPL; ++i) kv[i] = fv[i] = 0.0;
  const int nf = SETUP ? 2 : 1;
  for (int f = 0; f < nf; ++f) {
    const double* s1 = SETUP ? (f == 0 ? a.Ag : a.Ax) : a.Ax;
    const double* s2 = SETUP ? (f == 0 ? a.Ay : nullptr) : a.Ay;
    // all 16 tile loads of a thread in flight at once, then the staging stores
    constexpr int NE = L::TL * L::Q / L::NT;
    double gv[NE], yv[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = threadIdx.x + i * L::NT;
      const size_t o = ((size_t)b * L::Q + e / L::TL) * L::M + k1b + e % L::TL;
      gv[i] = s1[o];
      yv[i] = s2 ? s2[o] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = threadIdx.x + i * L::NT;
      const int q2 = e / L::TL, ll = e % L::TL;
      lines[ll * L::LS + pos_of_q(q2)] = {(q2 & 1) ? -gv[i] : gv[i], yv[i]};
    }
    __syncthreads();
    cd v[16];
    l16_load(W, l, v);
    __syncwarp();
    fft256<false>(v, W, T, l);
    l16_anal_own(v, ph, l, [&](int i, int k2, double X1, double X2) {
      if (SETUP && f == 0) {
        fv[i] = L::SQ2 * X1;
        kv[i] = L::SQ2 * CUDART_PI * (double)k2 * X2;
      } else if (SETUP) {
        kv[i] += L::SQ2 * X1;
      } else {
        kv[i] = L::SQ2 * X1 + L::SQ2 * CUDART_PI * (double)k2 * X2;
      }
    });
    __syncthreads();
  }
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  const double gam = a.gam;
  if (SETUP) {
    const double dbar = a.sc[b * 16 + S_DBAR];
    double hv[MPL], cv[MPL], xv[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k2 = l16_own_mode(i, l);
      const size_t e = row + (k2 > 0 ? k2 - 1 : 0);
      hv[i] = k2 > 0 ? a.HIST[b * a.sH + e] : 0.0;
      cv[i] = (k2 > 0 && a.CON) ? a.CON[b * a.sC + e] : 0.0;
      xv[i] = k2 > 0 ? a.X0[b * a.sX0 + e] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k2 = l16_own_mode(i, l);
      if (k2 == 0) continue;
      const size_t e = row + k2 - 1;
      const double hist = hv[i];
      const double con = cv[i];
      const double rhs = __dadd_rn(__dadd_rn(hist, __dmul_rn(gam, fv[i])), con);
      const double x0 = xv[i];
      const double r = rhs - (x0 + gam * kv[i]);
      const double z = pinv2d(gam, dbar, k1, k2) * r;
      a.X[b * a.sX + e] = x0;
      a.R[b * MM + e] = r;
      a.P[b * MM + e] = z;
      p0 = fma(rhs, rhs, p0);
      p1 = fma(r, r, p1);
      p2 = fma(r, z, p2);
    }
  } else {
    double pv[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k2 = l16_own_mode(i, l);
      pv[i] = k2 > 0 ? a.P[b * MM + row + k2 - 1] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k2 = l16_own_mode(i, l);
      if (k2 == 0) continue;
      const size_t e = row + k2 - 1;
      const double p = pv[i];
      const double qv = p + gam * kv[i];
      a.QV[b * MM + e] = qv;
      p0 = fma(p, qv, p0);
    }
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    p0 += __shfl_xor_sync(0xffffffffu, p0, o);
    p1 += __shfl_xor_sync(0xffffffffu, p1, o);
    p2 += __shfl_xor_sync(0xffffffffu, p2, o);
  }
  if (l == 0) {
    double* pp = a.part + ((size_t)b * L::Q + (k1 - 1)) * 4;
    pp[1] = p0;
    pp[2] = p1;
    pp[3] = p2;
  }
  if (!SETUP && pcg_is_last_cta(a, b)) pcg_alpha(a, b);
}

}  // namespace pf
