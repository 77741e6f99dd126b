// 2-D line engine for Q = 512 (config 5: 256^2 modes on a 512^2 grid) with
// register-resident FFTs, built on the 16 x 16 half-warp FFT of
// pf_line16.cuh.  A line is one warp; lane (a, s) = (lane & 15, lane >> 4).
//
//   inverse (DIT):  X[k] = E[k mod 256] + w512^-k O[k mod 256],
//                   E/O = 256-point DFTs of the even/odd samples;
//                   half-warp s computes E (s = 0) or O (s = 1) with fft256,
//                   the two halves swap through shared memory, and lane (a, h)
//                   ends holding X[a + 16 k2 + 256 h], k2 = 0..15;
//   forward (DIF):  from exactly that layout: y0[n] = x[n] + x[n+256],
//                   y1[n] = (x[n] - x[n+256]) w512^n, half-warp d runs fft256
//                   on y_d, lane (a, d) ends holding X[2 (a + 16 k2) + d].
//
// So the PCG matvec's synthesis -> pointwise -> analysis chain stays in
// registers, with three shared-memory round trips per transform (the
// fft256 transpose and the half swap) instead of five Stockham passes with
// CTA barriers.  Data layouts and transform pairs are those of pf_sine2d.cuh.
#pragma once
#include "pf_line16.cuh"

namespace pf {

struct L32 {
  static constexpr int LG = 9, Q = 512, M = 256, TL = 8, NT = 256;
  static constexpr int LS = Q + 1;    // line stride in cd
  static constexpr int STP = TL + 1;  // stage row stride in doubles
  static constexpr double SQ2 = 1.4142135623730951;
  static size_t smem_bytes() {
    const size_t lines = sizeof(cd) * TL * LS, stage = sizeof(double) * 2 * Q * STP;
    return sizeof(cd) * (256 + 256 + Q) + (lines > stage ? lines : stage);
  }
};

__device__ __forceinline__ int q_of_pos512(int pos) { return pos < 256 ? 2 * pos : 2 * (511 - pos) + 1; }
__device__ __forceinline__ int pos_of_q512(int q) { return (q & 1) ? (511 - (q >> 1)) : (q >> 1); }

// Inverse length-512 DFT of one line.  Entry: v[n1] = x[32 n1 + 2a + s].
// Exit: v[k2] = X[a + 16 k2 + 256 s].  buf: the line's 512 cd.  W: w512^k, k < 256.
__device__ __forceinline__ void fft512_inv(cd (&v)[16], cd* buf, const cd* T, const cd* W, int a, int s) {
  fft256<true>(v, buf + 256 * s, T, a);  // v[k2] = (s ? O : E)[a + 16 k2]
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) buf[256 * s + a + 16 * k2] = v[k2];
  __syncwarp();
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) {
    const cd p = buf[256 * (s ^ 1) + a + 16 * k2];
    cd w = W[a + 16 * k2];
    w.y = -w.y;
    const cd e = s ? p : v[k2];
    const cd o = cmul(s ? v[k2] : p, w);
    v[k2] = s ? csub(e, o) : cadd(e, o);
  }
  __syncwarp();
}

// Forward length-512 DFT of one line.  Entry: v[b] = x[a + 16 b + 256 s].
// Exit: v[k2] = X[2 (a + 16 k2) + s].
__device__ __forceinline__ void fft512_fwd(cd (&v)[16], cd* buf, const cd* T, const cd* W, int a, int s) {
#pragma unroll
  for (int b = 0; b < 16; ++b) buf[256 * s + a + 16 * b] = v[b];
  __syncwarp();
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    const cd p = buf[256 * (s ^ 1) + a + 16 * b];
    v[b] = s ? cmul(csub(p, v[b]), W[a + 16 * b]) : cadd(v[b], p);
  }
  __syncwarp();
  fft256<false>(v, buf + 256 * s, T, a);
}

template <int Q>
__device__ __forceinline__ void synth_write_q(cd* W, const cd* ph, int k, double av, double bv) {
  constexpr int M = Q / 2;
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

__device__ __forceinline__ void l32_setup(char* smem, const Sine2DArgs& a, cd*& T, cd*& W, cd*& ph, cd*& lines) {
  T = reinterpret_cast<cd*>(smem);
  W = T + 256;
  ph = W + 256;
  lines = ph + L32::Q;
  for (int j = threadIdx.x; j < 256; j += L32::NT) {
    T[j] = a.tw16[j];
    W[j] = a.tw16[256 + j];
  }
  for (int j = threadIdx.x; j < L32::Q; j += L32::NT) ph[j] = a.ph[j];
  __syncthreads();
}

// inverse-FFT inputs of lane (a, s) from a natural-order line
__device__ __forceinline__ void l32_load_inv(const cd* B, int a, int s, cd (&v)[16]) {
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) v[n1] = B[32 * n1 + 2 * a + s];
}
// forward-FFT inputs of lane (a, s) from a natural-order line
__device__ __forceinline__ void l32_load_fwd(const cd* B, int a, int s, cd (&v)[16]) {
#pragma unroll
  for (int b = 0; b < 16; ++b) v[b] = B[a + 16 * b + 256 * s];
}

// ---------------------------------------------------------------------------
// rows, synthesis (along y): lines k1 -> H[q2][k1] (contract of k2_rows_syn)
// ---------------------------------------------------------------------------
template <bool SETUP>
__global__ void __launch_bounds__(256, 2) k2_rows_syn32(Sine2DArgs a) {
  using L = L32;
  extern __shared__ __align__(16) char smem[];
  const int b = blockIdx.y;
  if (!SETUP && a.sc[b * 16 + S_DONE] != 0.0) return;
  cd *T, *Wt, *ph, *lines;
  l32_setup(smem, a, T, Wt, ph, lines);
  const int line = threadIdx.x >> 5, lane = threadIdx.x & 31, ai = lane & 15, s = lane >> 4;
  const int k1b = blockIdx.x * L::TL;
  const int k1 = k1b + line + 1;
  cd* B = lines + line * L::LS;
  const size_t row = (size_t)(k1 - 1) * L::M;
  const size_t MM = (size_t)L::M * L::M;
  const double beta = SETUP ? 0.0 : a.sc[b * 16 + S_BETA];
  const double dbar = a.sc[b * 16 + S_DBAR];
  double* st_s = reinterpret_cast<double*>(lines);
  double* st_c = st_s + L::Q * L::STP;
  constexpr int NF = SETUP ? 2 : 1, MPL = L::M / 32;
  for (int f = 0; f < NF; ++f) {
    if (lane == 0) B[0] = {0.0, 0.0};
    double ld1[MPL], ld2[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const size_t e = row + lane + 32 * i;
      if (SETUP) {
        ld1[i] = a.X0[b * a.sX0 + e];
        ld2[i] = f == 0 ? a.Cp[b * a.sCp + e] : 0.0;
      } else {
        ld1[i] = a.P[(size_t)b * MM + e];
        ld2[i] = a.R[(size_t)b * MM + e];
      }
    }
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k = lane + 1 + 32 * i;
      double av, bv;
      if (SETUP) {
        av = L::SQ2 * (f == 0 ? ld2[i] : ld1[i]);
        bv = f == 0 ? L::SQ2 * CUDART_PI * (double)k * ld1[i] : 0.0;
      } else {
        const double pn = fma(beta, ld1[i], pinv2d(a.gam, dbar, k1, k) * ld2[i]);  // p = z + beta p
        a.P[(size_t)b * MM + row + k - 1] = pn;
        av = L::SQ2 * pn;
        bv = L::SQ2 * CUDART_PI * (double)k * pn;
      }
      synth_write_q<L::Q>(B, ph, k, av, bv);
    }
    __syncwarp();
    cd v[16];
    l32_load_inv(B, ai, s, v);
    __syncwarp();
    fft512_inv(v, B, T, Wt, ai, s);
    __syncthreads();  // every line is done with its buffer: reuse the lines as the stage
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const int q = q_of_pos512(ai + 16 * k2 + 256 * s);
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

// setup pointwise at the lane's 16 grid points (see l16_pointwise)
template <int FID>
__device__ __forceinline__ void l32_pointwise(const Sine2DArgs& a, int q2, double t, double emt, size_t gl, int ai,
                                              int s, cd (&v1)[16], const cd (&v2)[16], double (&x4)[16],
                                              double& dsum, int& bad) {
  const double wq = 1.0 / ((double)L32::Q * (double)L32::Q);
  Fn f1 = a.fn;
  if (FID != 0) f1.id = FID;
  const double y2 = a.xq[q2];
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) {
    const int q1 = q_of_pos512(ai + 16 * k2 + 256 * s);
    const double u = (q1 & 1) ? -0.5 * v1[k2].x : 0.5 * v1[k2].x;
    const double gx = 0.5 * v1[k2].y;
    const double gy = (q1 & 1) ? -0.5 * v2[k2].x : 0.5 * v2[k2].x;
    const double x1 = a.xq[q1];
    const double Dv = fn_D(f1, x1, y2, t, u);
    if (!isfinite(Dv)) bad = min(bad, q1 * L32::Q + q2);  // oracle.Sine2D flat index [x1][x2]
    const double d = wq * Dv;
    const double g = wq * (f1.id == 4 ? fn_f(f1, make_double2(0.0, 0.0), emt, u) : fn_f(f1, fn_xtab(x1), emt, u));
    a.D[gl + q1] = d;
    dsum += d;
    const double sp4 = d * gy;
    v1[k2] = {(q1 & 1) ? -g : g, d * gx};
    x4[k2] = (q1 & 1) ? -sp4 : sp4;
  }
}

// ---------------------------------------------------------------------------
// columns (along x) for lines q2 (contract of k2_cols)
// ---------------------------------------------------------------------------
template <bool SETUP>
__global__ void __launch_bounds__(256, 2) k2_cols32(Sine2DArgs a) {
  using L = L32;
  extern __shared__ __align__(16) char smem[];
  const int b = blockIdx.y;
  if (!SETUP && a.sc[b * 16 + S_DONE] != 0.0) return;
  cd *T, *Wt, *ph, *lines;
  l32_setup(smem, a, T, Wt, ph, lines);
  const int line = threadIdx.x >> 5, lane = threadIdx.x & 31, ai = lane & 15, s = lane >> 4;
  const int q2 = blockIdx.x * L::TL + line;
  cd* B = lines + line * L::LS;
  const size_t hl = ((size_t)b * L::Q + q2) * L::M;
  const size_t gl = ((size_t)b * L::Q + q2) * L::Q;
  constexpr int MPL = L::M / 32;
  auto synth = [&](const double* A, const double* Bk) {
    if (lane == 0) B[0] = {0.0, 0.0};
    double av[MPL], bv[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      av[i] = A[hl + lane + 32 * i];
      bv[i] = Bk ? Bk[hl + lane + 32 * i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k = lane + 1 + 32 * i;
      synth_write_q<L::Q>(B, ph, k, L::SQ2 * av[i], L::SQ2 * CUDART_PI * (double)k * bv[i]);
    }
    __syncwarp();
  };
  auto store_fwd = [&](const cd (&v)[16]) {  // forward-FFT output to natural order
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) B[2 * (ai + 16 * k2) + s] = v[k2];
    __syncwarp();
  };
  if (!SETUP) {
    double dv[16];
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) dv[k2] = a.D[gl + q_of_pos512(ai + 16 * k2 + 256 * s)];
    synth(a.Hc, a.Hs);
    cd v[16];
    l32_load_inv(B, ai, s, v);
    __syncwarp();
    fft512_inv(v, B, T, Wt, ai, s);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const double d = 0.5 * dv[k2];
      v[k2] = {d * v[k2].x, d * v[k2].y};
    }
    fft512_fwd(v, B, T, Wt, ai, s);
    store_fwd(v);
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k = lane + 1 + 32 * i;
      const double2 X = anal_read_plain(B, ph, L::Q, k);
      a.Ay[hl + k - 1] = L::SQ2 * X.x;
      a.Ax[hl + k - 1] = L::SQ2 * CUDART_PI * (double)k * X.y;
    }
    return;
  }
  const double t = (double)(a.n0 + b) * a.dTs + a.tr;
  const double emt = a.fn.id == 1 ? exp(-t) : 0.0;
  cd v1[16], v2[16];
  synth(a.Hu, a.Hs);
  l32_load_inv(B, ai, s, v1);
  __syncwarp();
  fft512_inv(v1, B, T, Wt, ai, s);
  synth(a.Hc, nullptr);
  l32_load_inv(B, ai, s, v2);
  __syncwarp();
  fft512_inv(v2, B, T, Wt, ai, s);
  double dsum = 0.0;
  int bad = 0x7fffffff;
  double x4[16];
  switch (a.fn.id) {
    case 1: l32_pointwise<1>(a, q2, t, emt, gl, ai, s, v1, v2, x4, dsum, bad); break;
    case 2: l32_pointwise<2>(a, q2, t, emt, gl, ai, s, v1, v2, x4, dsum, bad); break;
    case 3: l32_pointwise<3>(a, q2, t, emt, gl, ai, s, v1, v2, x4, dsum, bad); break;
    case 4: l32_pointwise<4>(a, q2, t, emt, gl, ai, s, v1, v2, x4, dsum, bad); break;
    default: l32_pointwise<0>(a, q2, t, emt, gl, ai, s, v1, v2, x4, dsum, bad); break;
  }
  fft512_fwd(v1, B, T, Wt, ai, s);
  store_fwd(v1);
#pragma unroll
  for (int i = 0; i < MPL; ++i) {
    const int k = lane + 1 + 32 * i;
    const double2 X = anal_read_plain(B, ph, L::Q, k);
    a.Ag[hl + k - 1] = L::SQ2 * X.x;
    a.Ax[hl + k - 1] = L::SQ2 * CUDART_PI * (double)k * X.y;
  }
  __syncwarp();
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) v2[k2] = {x4[k2], 0.0};
  fft512_fwd(v2, B, T, Wt, ai, s);
  store_fwd(v2);
#pragma unroll
  for (int i = 0; i < MPL; ++i) {
    const int k = lane + 1 + 32 * i;
    a.Ay[hl + k - 1] = L::SQ2 * anal_read_plain(B, ph, L::Q, k).x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
  if (lane == 0) a.part[((size_t)b * L::Q + q2) * 4 + 0] = dsum;
  if (bad != 0x7fffffff) atomicMin(a.bad + b, bad);
}

// ---------------------------------------------------------------------------
// rows, analysis (along y) for lines k1 (contract of k2_rows_ana)
// ---------------------------------------------------------------------------
template <bool SETUP>
__global__ void __launch_bounds__(256, 2) k2_rows_ana32(Sine2DArgs a) {
  using L = L32;
  extern __shared__ __align__(16) char smem[];
  const int b = blockIdx.y;
  if (!SETUP && a.sc[b * 16 + S_DONE] != 0.0) return;
  cd *T, *Wt, *ph, *lines;
  l32_setup(smem, a, T, Wt, ph, lines);
  const int line = threadIdx.x >> 5, lane = threadIdx.x & 31, ai = lane & 15, s = lane >> 4;
  const int k1b = blockIdx.x * L::TL;
  const int k1 = k1b + line + 1;
  cd* B = lines + line * L::LS;
  const size_t MM = (size_t)L::M * L::M;
  const size_t row = (size_t)(k1 - 1) * L::M;
  constexpr int MPL = L::M / 32;
  double kv[MPL], fv[MPL];
#pragma unroll
  for (int i = 0; i < MPL; ++i) kv[i] = fv[i] = 0.0;
  const int nf = SETUP ? 2 : 1;
  for (int f = 0; f < nf; ++f) {
    const double* s1 = SETUP ? (f == 0 ? a.Ag : a.Ax) : a.Ax;
    const double* s2 = SETUP ? (f == 0 ? a.Ay : nullptr) : a.Ay;
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
      lines[ll * L::LS + pos_of_q512(q2)] = {(q2 & 1) ? -gv[i] : gv[i], yv[i]};
    }
    __syncthreads();
    cd v[16];
    l32_load_fwd(B, ai, s, v);
    __syncwarp();
    fft512_fwd(v, B, T, Wt, ai, s);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) B[2 * (ai + 16 * k2) + s] = v[k2];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k2 = lane + 1 + 32 * i;
      const double2 X = anal_read_plain(B, ph, L::Q, k2);
      if (SETUP && f == 0) {
        fv[i] = L::SQ2 * X.x;
        kv[i] = L::SQ2 * CUDART_PI * (double)k2 * X.y;
      } else if (SETUP) {
        kv[i] += L::SQ2 * X.x;
      } else {
        kv[i] = L::SQ2 * X.x + L::SQ2 * CUDART_PI * (double)k2 * X.y;
      }
    }
    __syncthreads();
  }
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  const double gam = a.gam;
  if (SETUP) {
    const double dbar = a.sc[b * 16 + S_DBAR];
    double hv[MPL], cv[MPL], xv[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const size_t e = row + lane + 32 * i;
      hv[i] = a.HIST[b * a.sH + e];
      cv[i] = a.CON ? a.CON[b * a.sC + e] : 0.0;
      xv[i] = a.X0[b * a.sX0 + e];
    }
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const int k2 = lane + 1 + 32 * i;
      const size_t e = row + k2 - 1;
      const double rhs = __dadd_rn(__dadd_rn(hv[i], __dmul_rn(gam, fv[i])), cv[i]);
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
    for (int i = 0; i < MPL; ++i) pv[i] = a.P[b * MM + row + lane + 32 * i];
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
      const size_t e = row + lane + 32 * i;
      const double qv = pv[i] + gam * kv[i];
      a.QV[b * MM + e] = qv;
      p0 = fma(pv[i], qv, p0);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    p0 += __shfl_xor_sync(0xffffffffu, p0, o);
    p1 += __shfl_xor_sync(0xffffffffu, p1, o);
    p2 += __shfl_xor_sync(0xffffffffu, p2, o);
  }
  if (lane == 0) {
    double* pp = a.part + ((size_t)b * L::Q + (k1 - 1)) * 4;
    pp[1] = p0;
    pp[2] = p1;
    pp[3] = p2;
  }
  if (!SETUP && pcg_is_last_cta(a, b)) pcg_alpha(a, b);
}

}  // namespace pf
