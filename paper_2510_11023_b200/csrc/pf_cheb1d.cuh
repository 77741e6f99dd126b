// Chebyshev-Lobatto collocation space, 1-D — the reference's own operator
// (spectral.py:74-136), kept as the parity bridge to the unmodified reference.
//
// One substep at (u_prev, t) [stepping.py:219-242]:
//   dv_p = D(x_p, t, [0, u_prev, 0])            all npts nodes, non-finite -> CoefficientError(p)
//   A    = (D1 diag(dv) D1)[1:-1, 1:-1]         npts^3 FMAs, D1 resident in smem
//   [I - gam A | (hist + gam f) + contrib]      augmented system in smem
//   LU with partial pivoting (virtual row permutation, reciprocal-pivot
//   scaling as LAPACK dgetf2), pivot check |u_kk| > 1e-14 max|system|
//   (stepping.py:62-75), back substitution.
//
// Two residences of the same algorithm: degree <= ~100 keeps D1 and the augmented
// system in shared memory (Cheb1D<128, 1>); above that (the reference's own config-3
// size, degree 513: a 512 x 513 system, 2 MB) D1 stays in global memory (L2-resident,
// shared by every slice) and each CTA's system lives in its own global scratch slab
// (Cheb1D<512, 1>, Cheb1DParams::aug_g).
#pragma once
#include "pf_device.cuh"

namespace pf {

struct Cheb1DParams {
  int npts, ni;
  const double* nodes;  // npts
  const double* d1;     // npts*npts
  const double* qw;     // npts
  double* aug_g;        // global-memory residence: one ni x ld_of(ni) slab per CTA (nullptr: shared memory)
  size_t aug_stride;    // doubles between the slabs of consecutive CTAs
};

template <int NT, int EPT>
struct Cheb1D {
  static constexpr bool kSide = false;  // no idle-warp side work in this space (see Sine1D::kSide)
  int tr = -1;                          // PF_TRACE timeline row (unused here)
  int npts, ni, LD;
  const double* d1;
  const double* nodes;
  const double* qw;
  double *aug, *uf, *dv, *xs;
  int* perm;
  double* pivs;  // [0] pivot value of the current column
  Reducer<NT> red;

  __host__ __device__ static int ld_of(int ni) {
    int ld = ni + 1;
    if ((ld & 1) == 0) ld += 1;
    return ld;
  }
  static size_t smem_bytes(int degree, bool global_residence = false) {
    const size_t npts = degree + 1, ni = degree - 1, ld = ld_of((int)ni);
    const size_t mats = global_residence ? 0 : npts * npts + ni * ld;
    return sizeof(double) * (mats + 2 * npts + 3 * npts + ni + 5 + RED_DOUBLES) + sizeof(int) * (ni + 4);
  }

  __device__ void init(char* smem, const Cheb1DParams& p) {
    npts = p.npts;
    ni = p.ni;
    LD = ld_of(ni);
    const bool glob = p.aug_g != nullptr;
    double* s = reinterpret_cast<double*>(smem);
    double* d1s = s;
    double* nds = glob ? s : d1s + npts * npts;
    double* qws = nds + npts;
    aug = glob ? p.aug_g + (size_t)blockIdx.x * p.aug_stride : qws + npts;
    uf = glob ? qws + npts : aug + ni * LD;
    dv = uf + npts;
    xs = dv + npts;
    pivs = xs + npts;
    double* rs = pivs + 4;
    if (reinterpret_cast<uintptr_t>(rs) & 15) rs += 1;  // the reducer reads its slots as 16-byte pairs
    red.init(rs);
    perm = reinterpret_cast<int*>(rs + RED_DOUBLES);
    if (!glob)
      for (int i = threadIdx.x; i < npts * npts; i += NT) d1s[i] = p.d1[i];
    for (int i = threadIdx.x; i < npts; i += NT) {
      nds[i] = p.nodes[i];
      qws[i] = p.qw[i];
      uf[i] = 0.0;
    }
    d1 = glob ? p.d1 : d1s;
    nodes = nds;
    qw = qws;
    __syncthreads();
  }

  __device__ __forceinline__ double norm2_partial(const double* v) const {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      if (e < ni) s = fma(qw[e + 1], v[i] * v[i], s);
    }
    return s;
  }

  __device__ int step(const Fn& fn, const double* xprev, const double* /*xguess: direct solve*/, double t,
                      double gam, const double* hist, const double* contrib, double* xout, Status& st) {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      if (e < ni) uf[e + 1] = xprev[i];
    }
    __syncthreads();
    int bad = 0x7fffffff;
    for (int p = threadIdx.x; p < npts; p += NT) {
      const double d = fn_D(fn, nodes[p], 0.0, t, uf[p]);
      dv[p] = d;
      if (!isfinite(d)) bad = min(bad, p);
    }
    const int badp = red.min_int(bad);
    if (badp != 0x7fffffff) {
      st.node = badp;
      return ST_COEFF;
    }
    // assembly of I - gam * (D1 diag(dv) D1)[1:-1,1:-1]
    double smax = 0.0;
    for (int idx = threadIdx.x; idx < ni * ni; idx += NT) {
      const int i = idx / ni, j = idx - i * ni;
      const double* row = d1 + (i + 1) * npts;
      double acc = 0.0;
      for (int p = 0; p < npts; ++p) acc = fma(__dmul_rn(row[p], dv[p]), d1[p * npts + j + 1], acc);
      const double val = __dsub_rn(i == j ? 1.0 : 0.0, __dmul_rn(gam, acc));
      aug[i * LD + j] = val;
      smax = fmax(smax, fabs(val));
    }
    const double emt = exp(-t);
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      if (e < ni) {
        const double f = fn_f(fn, fn_xtab(nodes[e + 1]), emt, xprev[i]);
        aug[e * LD + ni] = __dadd_rn(__dadd_rn(hist[i], __dmul_rn(gam, f)), contrib[i]);
        perm[e] = e;
      }
    }
    const double scale = red.max(smax);  // syncs: assembly + perm visible
    st.solves += 1;
    double pivmin = CUDART_INF;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = 0; k < ni; ++k) {
      if (warp == 0) {
        double best = -1.0;
        int bpos = ni;
        for (int pos = k + lane; pos < ni; pos += 32) {
          const double a = fabs(aug[perm[pos] * LD + k]);
          if (a > best || (a != a && best == best)) {  // NaN wins so it is reported
            best = a;
            bpos = pos;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
          if (ob > best || (ob == best && op < bpos)) {
            best = ob;
            bpos = op;
          }
        }
        if (lane == 0) {
          const int pk = perm[bpos];
          perm[bpos] = perm[k];
          perm[k] = pk;
          pivs[0] = aug[pk * LD + k];
        }
      }
      __syncthreads();
      const double pv = pivs[0];
      pivmin = fmin(pivmin, fabs(pv));
      if (!(fabs(pv) > 0.0)) pivmin = -1.0;  // zero / NaN pivot: fail below
      const double inv = 1.0 / pv;
      const int pk = perm[k];
      const int nr = ni - k - 1, nc = ni - k;
      for (int idx = threadIdx.x; idx < nr * nc; idx += NT) {
        const int a = idx / nc, c = idx - a * nc;
        const int pi = perm[k + 1 + a];
        const double l = aug[pi * LD + k] * inv;
        const int j = k + 1 + c;
        aug[pi * LD + j] = fma(-l, aug[pk * LD + j], aug[pi * LD + j]);
      }
      __syncthreads();
      if (pivmin < 0.0) break;
    }
    if (!(pivmin > 1e-14 * scale)) return ST_SOLVER;
    for (int pos = ni - 1; pos >= 0; --pos) {
      const int pp = perm[pos];
      const double xv = aug[pp * LD + ni] / aug[pp * LD + pos];
      if (threadIdx.x == 0) xs[pos] = xv;
      for (int q = threadIdx.x; q < pos; q += NT) {
        const int pq = perm[q];
        aug[pq * LD + ni] = fma(-aug[pq * LD + pos], xv, aug[pq * LD + ni]);
      }
      __syncthreads();
    }
    int finite = 1;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      xout[i] = (e < ni) ? xs[e] : 0.0;
      if (e < ni && !isfinite(xout[i])) finite = 0;
    }
    if (red.min_int(finite) == 0) return ST_SOLVER;
    return ST_OK;
  }
};

}  // namespace pf
