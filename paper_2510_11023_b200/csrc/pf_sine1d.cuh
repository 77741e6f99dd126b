// Sine spectral-Galerkin space, 1-D, matrix-free.
//
// State: coefficients c_k of the orthonormal basis sqrt(2) sin(k pi x),
// k = 1..M; quadrature on Q = 2M midpoints x_q = (q+1/2)/Q, w_q = 1/Q.
// One substep at (c_prev, t) [stepping.py:219-242 with the sine operator]:
//
//   u = S c_prev, v0 = S' c_prev           one length-Q complex FFT (DCT-III pair)
//   d = w D(x,t,u), g = w f(x,t,u)         fused pointwise epilogue
//   F = S^T g,  K c_prev = S'^T (d v0)     one length-Q complex FFT (DCT-II pair)
//   rhs = (hist + gam F) + contrib
//   (I + gam K) c = rhs                    PCG, preconditioner 1/(1+gam dbar pi^2 k^2),
//                                          initial guess c_prev, K applied through
//                                          one DCT-III + one DCT-II per iteration.
//
// The sine transforms are reduced to DCT-II/III by index reversal
// (sin(pi(Q-j)(2q+1)/2Q) = (-1)^q cos(pi j(2q+1)/2Q)), and every DCT pair runs
// as one length-Q complex Stockham FFT in shared memory (Makhoul's
// even/odd reordering), so the dense S, S' (Q x M) are never formed.
#pragma once
#include "pf_device.cuh"

namespace pf {

struct Sine1DParams {
  int M, Q, lgQ;
  const cd* tw;  // Q: exp(-2 pi i j / Q)
  const cd* ph;  // Q: exp(+i pi j / (2Q))
  double pcg_tol;
  int pcg_maxit;
};

// ---------------------------------------------------------------------------
// Stockham autosort FFT, radix 4 (+ one radix-2 pass for odd log2 L), in smem.
// inv=false: X_k = sum x_n exp(-2 pi i kn/L); inv=true: exp(+...), unnormalised.
// Returns the buffer that holds the result.  Ends with a __syncthreads.
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ cd* fft_stockham(cd* a, cd* b, const cd* __restrict__ tw, int L, int lg,
                                            bool inv) {
  int Ns = 1;
  const int L4 = L >> 2;
  for (int pass = 0; pass < (lg >> 1); ++pass) {
    const int step = L4 / Ns;
    for (int j = threadIdx.x; j < L4; j += NT) {
      const int k = j & (Ns - 1);
      cd v0 = a[j], v1 = a[j + L4], v2 = a[j + 2 * L4], v3 = a[j + 3 * L4];
      if (Ns > 1) {
        const int i1 = k * step;
        cd w1 = tw[i1], w2 = tw[2 * i1], w3 = tw[3 * i1];
        if (inv) {
          w1.y = -w1.y;
          w2.y = -w2.y;
          w3.y = -w3.y;
        }
        v1 = cmul(v1, w1);
        v2 = cmul(v2, w2);
        v3 = cmul(v3, w3);
      }
      const cd t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = csub(v1, v3);
      // -i*t3 = (t3.y, -t3.x)
      const cd mi3 = {t3.y, -t3.x};
      const cd X0 = cadd(t0, t2), X2 = csub(t0, t2);
      const cd Xa = cadd(t1, mi3), Xb = csub(t1, mi3);  // forward: X1 = Xa, X3 = Xb
      const int base = ((j - k) << 2) + k;
      b[base] = X0;
      b[base + Ns] = inv ? Xb : Xa;
      b[base + 2 * Ns] = X2;
      b[base + 3 * Ns] = inv ? Xa : Xb;
    }
    __syncthreads();
    cd* t = a;
    a = b;
    b = t;
    Ns <<= 2;
  }
  if (lg & 1) {
    const int L2 = L >> 1;
    const int step = L2 / Ns;
    for (int j = threadIdx.x; j < L2; j += NT) {
      const int k = j & (Ns - 1);
      cd v0 = a[j], v1 = a[j + L2];
      if (Ns > 1) {
        cd w = tw[k * step];
        if (inv) w.y = -w.y;
        v1 = cmul(v1, w);
      }
      const int base = ((j - k) << 1) + k;
      b[base] = cadd(v0, v1);
      b[base + Ns] = csub(v0, v1);
    }
    __syncthreads();
    cd* t = a;
    a = b;
    b = t;
  }
  return a;
}

template <int NT, int EPT>
struct Sine1D {
  static constexpr double SQ2 = 1.4142135623730951;
  int M, Q, lgQ;
  const cd* tw;
  const cd* ph;
  cd *A, *B;
  double *dq, *sa, *sb;
  Reducer<NT> red;
  double tol2;
  int maxit;

  static size_t smem_bytes(int M) {
    const size_t Q = 2 * (size_t)M;
    return Q * sizeof(cd) * 4 + Q * sizeof(double) + 2 * (Q + 1) * sizeof(double) + 128 * sizeof(double);
  }

  __device__ void init(char* smem, const Sine1DParams& p) {
    M = p.M;
    Q = p.Q;
    lgQ = p.lgQ;
    cd* s = reinterpret_cast<cd*>(smem);
    cd* tws = s;
    cd* phs = s + Q;
    A = s + 2 * Q;
    B = s + 3 * Q;
    dq = reinterpret_cast<double*>(s + 4 * Q);
    sa = dq + Q;
    sb = sa + (Q + 1);
    red.init(sb + (Q + 1));
    for (int j = threadIdx.x; j < Q; j += NT) {
      tws[j] = p.tw[j];
      phs[j] = p.ph[j];
    }
    for (int j = threadIdx.x; j <= Q; j += NT) {
      sa[j] = 0.0;
      sb[j] = 0.0;
    }
    tw = tws;
    ph = phs;
    tol2 = p.pcg_tol * p.pcg_tol;
    maxit = p.pcg_maxit;
    __syncthreads();
  }

  __device__ __forceinline__ int mode(int i) const { return 1 + (int)threadIdx.x + i * NT; }

  // node index of grid point q in the Makhoul permutation
  __device__ __forceinline__ int perm(int q) const { return (q & 1) ? (Q - 1 - (q >> 1)) : (q >> 1); }

  // Euclidean norm^2 partial of owned coefficients (Parseval: = L2 norm of u)
  __device__ __forceinline__ double wdot(const double* a, const double* b) const {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < EPT; ++i)
      if (mode(i) <= M) s = fma(a[i], b[i], s);
    return s;
  }
  __device__ double norm_partial_global(const double* v) const {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      if (e < M) s = fma(v[e], v[e], s);
    }
    return s;
  }

  // K p for owned modes (p, Kp in registers).  Uses sb, A, B, dq.
  __device__ __forceinline__ void apply_k(const double* p, double* kp) {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int k = mode(i);
      if (k <= M) sb[k] = SQ2 * CUDART_PI * (double)k * p[i];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < Q; j += NT) {
      const double bj = sb[j], bQ = sb[Q - j];
      const cd pj = ph[j];
      // V2 = ph*(bj - i bQ); W = i*V2
      const cd V2 = {pj.x * bj + pj.y * bQ, pj.y * bj - pj.x * bQ};
      A[j] = {-V2.y, V2.x};
    }
    __syncthreads();
    cd* R = fft_stockham<NT>(A, B, tw, Q, lgQ, true);
    cd* O = (R == A) ? B : A;
    for (int q = threadIdx.x; q < Q; q += NT) {
      const int idx = perm(q);
      const double v = 0.5 * R[idx].y;
      R[idx] = {0.0, dq[q] * v};
    }
    __syncthreads();
    cd* Z = fft_stockham<NT>(R, O, tw, Q, lgQ, false);
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int k = mode(i);
      if (k <= M) {
        const cd a = Z[k], b = Z[Q - k], c = ph[k];
        const double Dx = a.x - b.x, Dy = a.y + b.y;
        const double X2 = 0.5 * (c.x * Dy - c.y * Dx);
        kp[i] = SQ2 * CUDART_PI * (double)k * X2;
      }
    }
  }

  // One semi-implicit substep.  xprev: owned coefficients of c_prev.
  // Returns 0 on success, else ST_* with st.node / fail info set.
  __device__ int step(const Fn& fn, const double* xprev, double t, double gam, const double* hist,
                      const double* contrib, double* xout, Status& st) {
    // --- synthesis pair: u = S c, v0 = S' c -----------------------------
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int k = mode(i);
      if (k <= M) {
        sa[k] = SQ2 * xprev[i];
        sb[k] = SQ2 * CUDART_PI * (double)k * xprev[i];
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < Q; j += NT) {
      const double aj = sa[j], aQ = sa[Q - j], bj = sb[j], bQ = sb[Q - j];
      const cd pj = ph[j];
      const cd V1 = {pj.x * aQ + pj.y * aj, pj.y * aQ - pj.x * aj};
      const cd V2 = {pj.x * bj + pj.y * bQ, pj.y * bj - pj.x * bQ};
      A[j] = {V1.x - V2.y, V1.y + V2.x};
    }
    __syncthreads();
    cd* R = fft_stockham<NT>(A, B, tw, Q, lgQ, true);
    cd* O = (R == A) ? B : A;
    // --- pointwise coefficients (fused epilogue) ------------------------
    const double wq = 1.0 / (double)Q;
    double dsum = 0.0;
    int bad = 0x7fffffff;
    for (int q = threadIdx.x; q < Q; q += NT) {
      const int idx = perm(q);
      const cd w = R[idx];
      const double s1 = 0.5 * w.x, s2 = 0.5 * w.y;
      const double u = (q & 1) ? -s1 : s1;
      const double xq = ((double)q + 0.5) / (double)Q;
      const double Dv = fn_D(fn, xq, 0.0, t, u);
      if (!isfinite(Dv)) bad = min(bad, q);
      const double d = wq * Dv;
      const double g = wq * fn_f(fn, xq, 0.0, t, u);
      dq[q] = d;
      dsum += d;
      R[idx] = {(q & 1) ? -g : g, d * s2};
    }
    const int badq = red.min_int(bad);  // syncs
    if (badq != 0x7fffffff) {
      st.node = badq;
      return ST_COEFF;
    }
    const double dbar = red.sum(dsum);
    // --- analysis pair: F = S^T g, K c_prev = S'^T (d v0) ----------------
    cd* Z = fft_stockham<NT>(R, O, tw, Q, lgQ, false);
    double x[EPT], r[EPT], p[EPT], z[EPT], pinv[EPT], rhs[EPT];
    double bb = 0.0, rr = 0.0;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int k = mode(i);
      x[i] = r[i] = p[i] = z[i] = pinv[i] = rhs[i] = 0.0;
      if (k <= M) {
        const cd a = Z[k], b = Z[Q - k], c = ph[k], c2 = ph[Q - k];
        const double Dx = a.x - b.x, Dy = a.y + b.y;
        const double X2 = 0.5 * (c.x * Dy - c.y * Dx);
        const double X1 = 0.5 * (c2.x * (b.x + a.x) + c2.y * (b.y - a.y));
        const double F = SQ2 * X1;
        const double kx = SQ2 * CUDART_PI * (double)k * X2;
        rhs[i] = __dadd_rn(__dadd_rn(hist[i], __dmul_rn(gam, F)), contrib[i]);
        x[i] = xprev[i];
        r[i] = rhs[i] - (x[i] + gam * kx);
        const double kk = (double)k;
        pinv[i] = 1.0 / (1.0 + gam * dbar * (CUDART_PI * CUDART_PI) * (kk * kk));
        bb = fma(rhs[i], rhs[i], bb);
        rr = fma(r[i], r[i], rr);
      }
    }
    const double2 s0 = red.sum2(bb, rr);
    st.solves += 1;
    if (s0.x == 0.0) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) xout[i] = 0.0;
      return ST_OK;
    }
    const double thr = tol2 * s0.x;
    double rrv = s0.y;
    int it = 0;
    if (rrv > thr) {
      double rzl = 0.0;
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        z[i] = pinv[i] * r[i];
        p[i] = z[i];
        rzl = fma(r[i], z[i], rzl);
      }
      double rz = red.sum(rzl);
      for (it = 1; it <= maxit; ++it) {
        double kp[EPT], qv[EPT];
        apply_k(p, kp);
        double pql = 0.0;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          qv[i] = p[i] + gam * kp[i];
          pql = (mode(i) <= M) ? fma(p[i], qv[i], pql) : pql;
        }
        const double pq = red.sum(pql);
        const double alpha = rz / pq;
        double rrl = 0.0, rzn = 0.0;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          if (mode(i) <= M) {
            x[i] = fma(alpha, p[i], x[i]);
            r[i] = fma(-alpha, qv[i], r[i]);
            z[i] = pinv[i] * r[i];
            rrl = fma(r[i], r[i], rrl);
            rzn = fma(r[i], z[i], rzn);
          }
        }
        const double2 s = red.sum2(rrl, rzn);
        rrv = s.x;
        if (!(rrv > thr)) break;  // converged (NaN falls through to the check below)
        const double beta = s.y / rz;
        rz = s.y;
#pragma unroll
        for (int i = 0; i < EPT; ++i) p[i] = fma(beta, p[i], z[i]);
      }
      st.iters += (it > maxit) ? maxit : it;
      if (it > maxit) return ST_SOLVER;
    }
    int finite = 1;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      if (mode(i) <= M && !isfinite(x[i])) finite = 0;
      xout[i] = x[i];
    }
    if (red.min_int(finite) == 0) return ST_SOLVER;
    return ST_OK;
  }

  // norm^2 of owned values
  __device__ __forceinline__ double norm2_partial(const double* v) const { return wdot(v, v); }
};

}  // namespace pf
