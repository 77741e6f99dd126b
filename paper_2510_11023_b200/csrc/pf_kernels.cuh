// Kernels templated over a space (Sine1D / Cheb1D):
//
//   k_fine_sweep   one CTA per slice, persistent over all m substeps
//                  (stepping.fine_sweep_intervals, stepping.py:189-243)
//   k_coarse       one CTA; run_coarse / the parareal correction sweep with
//                  guards and diff / a single coarse step
//                  (stepping.py:87-121, parareal.py:114-128)
//   (the full-history solver, stepping.py:260-288, is k_fine_sweep over one
//   slice of nt*m substeps with split-K helper CTAs)
//
// Thread ownership of state entries is e = threadIdx.x + i*NT (i < EPT) in
// every kernel, so a thread only ever re-reads history rows it wrote itself.
#pragma once
#include "pf_device.cuh"

namespace pf {

struct Common {
  Fn fn;
  int size;  // state entries
  int nt, m;
  double dT, dt, gam_f, gam_c, minv;  // minv = m^-alpha
  const double* bfine;                // b_q
  const double* afine;                // a_s = b_{s-1} - b_s (s >= 1; a_0 unused)
  const double* bfrac;                // b_{q/m}
  double* scratch;                    // per-slice block history rows
  // coarse-history bracket of every (slice, substep), precomputed by
  // k_bracket_all: (nslices, m, size), row r-1 = target substep r; nullptr = 0
  const double* brk;
  double anear[16];                   // a_s for s < 16 (near-history weights, uniform loads)
  // PCG guess weights by local substep r (8 per row): Lagrange extrapolation
  // in the slice's own tau = (r dt)^alpha -- slice 0's initial layer and every
  // later slice's start layer defeat polynomial extrapolation in t
  const double* ext0;
  // start state of the (single) slice when it differs from U[n]: fine_propagate's
  // `start` (stepping.py:170-171, path[0] = start; the bracket still uses U); nullptr = U[n]
  const double* x_start;
  // far history of one-helper sweeps and of the inline path: 0 DFMA register
  // tiles (default), 1 DMMA tensor cores, 2 DMMA fed by TMA bulk copies (helper);
  // the sequential solver's split helpers always use DMMA (PF_FAR_TC, launch_fine)
  int far_tc;
  // pipelined parareal (pf_parareal): a slice below *frozen_from
  // (the first node the previous correction changed) has bitwise the inputs of
  // its last sweep -- it copies its F_old row from fold_prev instead of sweeping;
  // *cancel (set by the host when the iteration before converged) ends a
  // speculative sweep at its next block boundary.  nullptr: off.
  const int* frozen_from;
  const double* fold_prev;
  const int* cancel;
};

// Block length of the blocked L1 history: each history row is read once per
// HB substeps and reused for HB target rows (register-tiled Toeplitz GEMM).
constexpr int HB = 8;
// The last NR states of a slice live in a shared-memory ring (when it fits):
// the near history (< 2*HB rows) and the PCG initial guess read it there.
constexpr int NR = 2 * HB;
// PCG initial guess: order-EXO polynomial extrapolation of the path,
// x0 = sum_j (-1)^j C(p+1, j+1) c_{r-1-j}, p = min(EXO, r-1).
constexpr int EXO = 5;
// Tabulated guesses (Common::ext0, 1-D with alpha < 1): Lagrange extrapolation
// in tau = t^alpha of order <= EXT, host-scheduled per substep (see pf_create).
constexpr int EXT = 7;
// kExtrap[p][j] = (-1)^j C(p+1, j+1)
__constant__ double kExtrap[EXO + 1][EXO + 1] = {
    {1, 0, 0, 0, 0, 0},        {2, -1, 0, 0, 0, 0},        {3, -3, 1, 0, 0, 0},
    {4, -6, 4, -1, 0, 0},      {5, -10, 10, -5, 1, 0},     {6, -15, 20, -15, 6, -1}};

// Far history for the HB target rows r = R0+1 .. R0+HB of one slice
// (the einsum of stepping.py:234 restricted to j <= Jmax):
//   out[rr] = b_{R0+rr} path[0] + sum_{j=1}^{Jmax} a_{R0+1+rr-j} path[j]
// Weights are Toeplitz in (r, j): a J-row chunk needs HB+J-1 of them, read
// from `aw` (shared memory in helper CTAs).  Chunks are double-buffered in
// registers so the next chunk's loads overlap this chunk's FMAs.  Path rows
// are read through L2 (ld.global.cg): a helper CTA reads rows another CTA
// wrote during this launch.
template <int NT, int EPT, int J>
__device__ __forceinline__ void load_rows(const Common& c, const double* path, int j0, int Jmax,
                                          double (&cv)[J][EPT]) {
#pragma unroll
  for (int t = 0; t < J; ++t) {
    const double* row = path + (size_t)(j0 + t) * c.size;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      cv[t][i] = (e < c.size && j0 + t <= Jmax) ? __ldcg(row + e) : 0.0;
    }
  }
}

template <int EPT, int J>
__device__ __forceinline__ void fma_rows(const double* aw, int R0, int j0, const double (&cv)[J][EPT],
                                         double (&acc)[HB][EPT]) {
  // wv[u] = a_{R0+1-j0-(J-1)+u}, u = rr - t + J - 1 (index clamped for rows past Jmax, whose data is 0)
  double wv[HB + J - 1];
  const int s0 = R0 + 1 - j0 - (J - 1);
#pragma unroll
  for (int u = 0; u < HB + J - 1; ++u) {
    const int s = s0 + u;
    wv[u] = aw[s < 1 ? 1 : s];
  }
#pragma unroll
  for (int t = 0; t < J; ++t)
#pragma unroll
    for (int rr = 0; rr < HB; ++rr)
#pragma unroll
      for (int i = 0; i < EPT; ++i) acc[rr][i] = fma(wv[rr - t + J - 1], cv[t][i], acc[rr][i]);
}

template <int NT, int EPT, int J>
__device__ __forceinline__ void far_history_block(const Common& c, const double* path, const double* aw, int R0,
                                                  int Jmax, double* out) {
  double acc[HB][EPT];
  double c0[EPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = threadIdx.x + i * NT;
    c0[i] = (e < c.size) ? __ldcg(path + e) : 0.0;
  }
#pragma unroll
  for (int rr = 0; rr < HB; ++rr) {
    const double w = c.bfine[R0 + rr];
#pragma unroll
    for (int i = 0; i < EPT; ++i) acc[rr][i] = w * c0[i];
  }
  if (Jmax >= 1) {
    double ca[J][EPT], cb[J][EPT];
    load_rows<NT, EPT, J>(c, path, 1, Jmax, ca);
    for (int j0 = 1; j0 <= Jmax; j0 += 2 * J) {
      load_rows<NT, EPT, J>(c, path, j0 + J, Jmax, cb);
      fma_rows<EPT, J>(aw, R0, j0, ca, acc);
      if (j0 + J > Jmax) break;
      load_rows<NT, EPT, J>(c, path, j0 + 2 * J, Jmax, ca);
      fma_rows<EPT, J>(aw, R0, j0 + J, cb, acc);
    }
  }
#pragma unroll
  for (int rr = 0; rr < HB; ++rr)
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      if (e < c.size) out[(size_t)rr * c.size + e] = acc[rr][i];
    }
}

// Coarse-history bracket (stepping.py:124-139, _coarse_contribution)
//   -m^-alpha sum_{j<n} b_{j + r/m} (U_{n-j} - U_{n-j-1})
// of every (slice, substep) of a sweep, before it starts: the A2 GEMM of
// SURVEY §8(a) (picks^T x dU per slice), j ascending with one fma per (j, row)
// per element (deterministic; previously done block by block on the helper
// CTAs, where it made the helpers of late slices -- n coarse rows each -- the
// critical path).  Thread: one mode, RT consecutive target rows; grid
// (modes / 256, m / RT, slices).
template <int RT, int EM>
__global__ void __launch_bounds__(256) k_bracket_all(Common c, const double* __restrict__ U, int n_lo,
                                                     double* __restrict__ out) {
  static_assert(RT % 2 == 0, "weights are read in pairs");
  constexpr int JC = 64;  // weights b_{j + r/m} of JC coarse rows x RT target rows staged in shared memory
  __shared__ __align__(16) double sw[JC][RT];
  const int e0 = blockIdx.x * (blockDim.x * EM) + threadIdx.x;  // modes e0 + i * blockDim.x, i < EM
  const int r0 = blockIdx.y * RT + 1;
  const int b = blockIdx.z, n = n_lo + b;
  double acc[EM][RT], hi[EM];
#pragma unroll
  for (int i = 0; i < EM; ++i) {
    const int e = e0 + i * (int)blockDim.x;
    hi[i] = e < c.size ? U[(size_t)n * c.size + e] : 0.0;
#pragma unroll
    for (int q = 0; q < RT; ++q) acc[i][q] = 0.0;
  }
  for (int j0 = 0; j0 < n; j0 += JC) {
    const int jn = min(JC, n - j0);
    __syncthreads();
    for (int t = threadIdx.x; t < jn * RT; t += blockDim.x) {
      const int j = t / RT, q = t % RT;
      sw[j][q] = r0 + q <= c.m ? c.bfrac[(size_t)(j0 + j) * c.m + r0 + q] : 0.0;
    }
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < jn; ++j) {
      double inc[EM];
#pragma unroll
      for (int i = 0; i < EM; ++i) {
        const int e = e0 + i * (int)blockDim.x;
        const double lo = e < c.size ? U[(size_t)(n - j0 - j - 1) * c.size + e] : 0.0;
        inc[i] = hi[i] - lo;
        hi[i] = lo;
      }
      const double2* w2 = reinterpret_cast<const double2*>(sw[j]);
#pragma unroll
      for (int q = 0; q < RT; q += 2) {
        const double2 w = w2[q / 2];
#pragma unroll
        for (int i = 0; i < EM; ++i) {
          acc[i][q] = fma(w.x, inc[i], acc[i][q]);
          acc[i][q + 1] = fma(w.y, inc[i], acc[i][q + 1]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < EM; ++i) {
    const int e = e0 + i * (int)blockDim.x;
    if (e >= c.size) continue;
#pragma unroll
    for (int q = 0; q < RT; ++q)
      if (r0 + q <= c.m) out[((size_t)b * c.m + r0 - 1 + q) * c.size + e] = (n > 0) ? -c.minv * acc[i][q] : 0.0;
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// thread 0 waits until *flag >= v, then the whole CTA proceeds
__device__ __forceinline__ void cta_wait_geq(const int* flag, int v) {
  if (threadIdx.x == 0) {
    int ns = 64;
    while (ld_acquire(flag) < v) {
      __nanosleep(ns);
      ns = ns < 2048 ? 2 * ns : ns;
    }
  }
  __syncthreads();
}
// the whole CTA's prior global writes become visible, then thread 0 publishes v
// (bar.sync orders the CTA's writes before thread 0's st.release.gpu, and
// release is cumulative in the PTX memory model: no separate membar.gl needed)
__device__ __forceinline__ void cta_publish(int* flag, int v) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(flag, v);
}
// the same with a release add (counters several CTAs publish into)
__device__ __forceinline__ void cta_publish_add(int* flag, int v) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}
// true in the CTA that is the `count`-th to arrive on `ticket` (which it resets)
__device__ __forceinline__ bool cta_last_arrival(int* ticket, int count) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int t = atomicAdd(ticket, 1);
    s_last = t == count - 1;
    if (s_last) *ticket = 0;
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  return true;
}

// History rows of block beta (target rows R0+1..R0+HB, R0 = beta*HB) folded
// into the far part: j <= J(beta) = max(beta-1, 0)*HB.  The lag of one block
// lets a helper CTA compute block beta+1 while the slice CTA marches block beta.
__device__ __forceinline__ int far_extent(int beta) { return (beta > 0 ? beta - 1 : 0) * HB; }

struct SweepSync {
  int* progress;  // [slice] last substep whose state row is in the path
  int* ready;     // [slice * hps + helper] far-history blocks published (tensor-core path: [slice * hps]
                  // counts published 64-mode batches)
  int* abort;     // [slice] set by a failing slice CTA
  int* tickets;   // [slice][parity][32] batch arrivals of the split tensor-core far history
};

// ---------------------------------------------------------------------------
// Far history on the FP64 tensor cores: DMMA (mma.sync m8n8k4 .f64).
// The far part of block beta is a Toeplitz GEMM
//   out[rr][e] = b_{R0+rr} c_0[e] + sum_{j=1}^{J} a_{R0+1+rr-j} c_j[e]     (rr < HB = 8)
// = A (8 x J, Toeplitz weights) x B (J x M, path rows): one m8n8k4 MMA per
// k-step of 4 history rows and 8 modes, A[rr][k] = a_{R0+1+rr-(j0+k)} from
// shared memory, B[k][n] = c_{j0+k}[8g+n] from global (L2 / HBM), the
// accumulator C (8 target rows x 8 modes) in registers.
// Order: a batch of 8 mode groups (64 modes) accumulates every k-step in
// ascending order in one warp, out = b c_0 + acc -- the same whether the slice
// CTA computes it inline or its helper CTA does (bitwise, tested).  The
// sequential solver's split helpers (far history of up to 64k rows over many
// CTAs) sum interleaved parts instead: same terms, another rounding order
// (tested against the inline path to 1e-12 and against the oracle).
// ---------------------------------------------------------------------------
constexpr int TC_BATCH = 64;          // modes per batch (8 groups of 8)
// parts per batch of the split helpers: 8, or 16 when there are helpers for it
__host__ __device__ constexpr int tc_parts(int hps, int nb) { return hps >= 16 * nb ? 16 : 8; }
constexpr int TC_RED = 8 * 8 * 64;    // doubles of the per-CTA part buffer (8 warps x 8 groups x 64)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One warp: the 8 x 64 tile of `batch` accumulated over k-steps s = s0, s0 + ds, ...
// (rows j = 1 + 4 s + k <= J), ascending.  Lane l holds C rows l>>2, columns
// 2(l&3) + {0,1} of each of the 8 groups.  PD k-steps of loads are in flight
// (register ring) while the MMAs of the current one issue.
template <int PD = 8>
__device__ __forceinline__ void tc_far_part(const double* __restrict__ path, int size, const double* __restrict__ aw,
                                            int R0, int J, int batch, int s0, int ds, double (&acc)[8][2]) {
  const int lane = threadIdx.x & 31, k = lane & 3, q = lane >> 2;
#pragma unroll
  for (int g = 0; g < 8; ++g) acc[g][0] = acc[g][1] = 0.0;
  const int nsteps = (J + 3) >> 2;
  const double* col = path + TC_BATCH * batch + q;
  double av[PD], bv[PD][8];
  auto load = [&](int st, double& a, double (&b)[8]) {
    const int j = 1 + 4 * st + k;
    const bool ok = j <= J;
    a = ok ? aw[R0 + 1 + q - j] : 0.0;
    const double* row = col + (size_t)j * size;
#pragma unroll
    for (int g = 0; g < 8; ++g) b[g] = ok ? __ldcg(row + 8 * g) : 0.0;
  };
#pragma unroll
  for (int p = 0; p < PD; ++p) load(s0 + p * ds, av[p], bv[p]);
  for (int st = s0; st < nsteps; st += PD * ds) {
#pragma unroll
    for (int p = 0; p < PD; ++p) {
      if (st + p * ds < nsteps) {
        const double ac = av[p];
        double bc[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) bc[g] = bv[p][g];
        load(st + (p + PD) * ds, av[p], bv[p]);
#pragma unroll
        for (int g = 0; g < 8; ++g) dmma884(acc[g][0], acc[g][1], ac, bc[g]);
      }
    }
  }
}

// a warp's finished tile of `batch` (every k-step in one accumulator) -> out rows
__device__ __forceinline__ void tc_store_tile(const double (&acc)[8][2], const double* __restrict__ row0,
                                              const double* __restrict__ bfine, int R0, int size, int batch,
                                              double* out) {
  const int lane = threadIdx.x & 31, rr = lane >> 2;
  const double w = bfine[R0 + rr];
#pragma unroll
  for (int g = 0; g < 8; ++g)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = TC_BATCH * batch + 8 * g + 2 * (lane & 3) + i;
      out[(size_t)rr * size + e] = w * __ldcg(row0 + e) + acc[g][i];
    }
}

// ---- TMA staging (cp.async.bulk + mbarrier) of the history rows ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bulk copy global -> shared (TMA), completion counted on `bar`
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Helper CTA: the far-history tiles of block (R0, J) with the history rows
// streamed through shared memory by TMA bulk copies: stages of 8 rows (one
// 4 KB copy per row into a 64 B-padded slot: minimal-wavefront fragment
// loads), NS stages on full/empty mbarrier pairs -- no CTA-wide barrier in the
// row loop.  Warp w consumes batch w of every stage (k-steps in ascending
// order: the arithmetic and order of tc_far_block, so the tile is bitwise the
// inline one) and releases the slot with one arrive; thread 0 refills the slot
// of the stage before the one its warp just finished (that slot's 8 arrivals
// are almost always in by then), so NS - 1 stages of copies stay in flight.
struct TmaRing {
  double* buf;                  // NS stages x 8 rows x (size + 8) doubles
  unsigned long long* full;     // NS mbarriers (1 arrival + the stage's bytes)
  unsigned long long* empty;    // NS mbarriers (8 arrivals: one per consumer warp)
  int NS;
  long long issued;             // stages issued so far (running: mbarrier phases)
};

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Stream history rows 1 + 8 st .. 8 + 8 st of stages st = st0 .. st1-1 through the ring and
// accumulate them into TT target tiles at once (tile u: target rows R0[u]+1 .. R0[u]+8):
// one set of B fragments (the rows) feeds TT DMMAs, so a row is read once per TT tiles.
// Warp w owns the 64-mode batch w; acc[u][g] is its m8n8 fragment of tile u, group g.
template <int TT>
__device__ __forceinline__ void tc_stream(const double* __restrict__ path, int size, const double* __restrict__ aw,
                                          const int (&R0)[TT], int st0, int st1, double (&acc)[TT][8][2],
                                          TmaRing& ring) {
  const int NB = size / TC_BATCH, pitch = size + 8;
  const int nstg = st1 - st0;
  if (nstg <= 0) return;
  const long long g0 = ring.issued;
  const int NS = ring.NS;
  // thread 0: copy stage st0 + i into its slot, once the slot's previous use is released
  auto issue = [&](int i) {
    const long long g = g0 + i;
    const int slot = (int)(g % NS);
    const long long use = g / NS;
    if (use > 0) mbar_wait(ring.empty + slot, (unsigned)((use - 1) & 1));
    double* dst = ring.buf + (size_t)slot * 8 * pitch;
    mbar_expect_tx(ring.full + slot, 8u * (unsigned)size * 8u);
#pragma unroll
    for (int t = 0; t < 8; ++t)
      tma_load(dst + (size_t)t * pitch, path + (size_t)(1 + 8 * (st0 + i) + t) * size, (unsigned)size * 8u,
               ring.full + slot);
  };
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async;" ::: "memory");  // path rows (generic writes, acquired) -> bulk-copy reads
    for (int i = 0; i < nstg && i < NS - 1; ++i) issue(i);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, k = lane & 3, q = lane >> 2;
  for (int i = 0; i < nstg; ++i) {
    // keep NS - 1 stages in flight: stage i + NS - 1 goes into the slot stage i - 1 used
    if (threadIdx.x == 0 && i + NS - 1 < nstg) issue(i + NS - 1);
    const long long g = g0 + i;
    const int slot = (int)(g % NS);
    mbar_wait(ring.full + slot, (unsigned)((g / NS) & 1));
    const double* st = ring.buf + (size_t)slot * 8 * pitch;
    if (w < NB) {
      double bv[2][8];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const double* bp = st + (size_t)(4 * t + k) * pitch + TC_BATCH * w + q;
#pragma unroll
        for (int g2 = 0; g2 < 8; ++g2) bv[t][g2] = bp[8 * g2];
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int j = 1 + 8 * (st0 + i) + 4 * t + k;
#pragma unroll
        for (int u = 0; u < TT; ++u) {
          const double av = aw[R0[u] + 1 + q - j];
#pragma unroll
          for (int g2 = 0; g2 < 8; ++g2) dmma884(acc[u][g2][0], acc[u][g2][1], av, bv[t][g2]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(ring.empty + slot);  // this warp is done with the slot
  }
  ring.issued = g0 + nstg;
}

// fragment-layout partial tiles in global scratch: [tile][batch w][group g][lane] double2 -- every
// lane reloads exactly what it stored
__device__ __forceinline__ void tc_frag_store(double* buf, int tile, int NB, const double (&acc)[8][2]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* p = reinterpret_cast<double2*>(buf) + ((size_t)(tile * NB + w) * 8) * 32 + lane;
#pragma unroll
  for (int g = 0; g < 8; ++g) p[g * 32] = make_double2(acc[g][0], acc[g][1]);
}
__device__ __forceinline__ void tc_frag_load(const double* buf, int tile, int NB, double (&acc)[8][2]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* p = reinterpret_cast<const double2*>(buf) + ((size_t)(tile * NB + w) * 8) * 32 + lane;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const double2 v = p[g * 32];
    acc[g][0] = v.x;
    acc[g][1] = v.y;
  }
}

// Grouping of the TMA-fed helper: the rows older than G + 1 blocks are accumulated into the G
// tiles of a super-block of G blocks in ONE pass (a quarter of the one-pass-per-tile traffic:
// late in a sweep every helper streams its slice's whole path per block, 269 MB per block
// period at config 3 -- more than HBM delivers); the last (G + t) blocks of rows are appended
// per tile.  Every accumulator still takes its rows in ascending order: bitwise tc_far_block.
constexpr int TC_G = 4;
// rows 1..tc_common_extent(S) are accumulated for all tiles of super-block S together
__host__ __device__ constexpr int tc_common_extent(int S) { return (TC_G * S - TC_G - 1 > 0 ? TC_G * S - TC_G - 1 : 0) * HB; }

// CTA (256 threads = 8 warps): the far-history tiles of every batch, warp w
// computing batches w, w + 8, ... over all k-steps in ascending order (the
// order of the slice CTA's inline path and of its helper CTA).
__device__ __forceinline__ void tc_far_block(const double* __restrict__ path, const double* __restrict__ row0,
                                             int size, const double* __restrict__ aw, const double* __restrict__ bfine,
                                             int R0, int J, double* out) {
  const int NB = size / TC_BATCH;
  for (int batch = (int)(threadIdx.x >> 5); batch < NB; batch += 8) {
    double acc[8][2];
    tc_far_part(path, size, aw, R0, J, batch, 0, 1, acc);
    tc_store_tile(acc, row0, bfine, R0, size, batch, out);
  }
}

// store a warp's partial tile into the CTA part buffer red[warp][g][lane][2]
__device__ __forceinline__ void tc_store_part(double* red, const double (&acc)[8][2]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int g = 0; g < 8; ++g)
    reinterpret_cast<double2*>(red + ((size_t)(w * 8 + g) * 32 + lane) * 2)[0] = make_double2(acc[g][0], acc[g][1]);
}

// (rr, mode within the batch) of the 2 outputs of thread t (256 threads, 512 outputs)
__device__ __forceinline__ void tc_out_index(int t, int i, int& slot, int& rr, int& col) {
  slot = 2 * t + i;                        // = (g * 32 + lane) * 2 + i
  const int g = slot >> 6, lane = (slot >> 1) & 31;
  rr = lane >> 2;
  col = 8 * g + 2 * (lane & 3) + i;
}



// Protocol stress build (-DPF_JITTER, tests/test_protocol_jitter.py): the
// slice CTA delays its progress publish and the helper CTA its block by a
// pseudo-random 0..8 us, so the release/acquire handshake runs under many
// interleavings; results must stay bitwise those of the inline far history.
// (compute-sanitizer is closed on this pool: profiles/r02_compute_sanitizer_closed.txt)
__device__ __forceinline__ void pf_jitter(int a, int b, int tid0 = 0) {
#ifdef PF_JITTER
  if ((int)threadIdx.x == tid0) {
    unsigned h = (unsigned)a * 73856093u ^ (unsigned)b * 19349663u ^ (unsigned)PF_JITTER * 83492791u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    __nanosleep(h & 8191u);
  }
#else
  (void)a;
  (void)b;
  (void)tid0;
#endif
}

// Side work of the Q = 1024 fine sweep (k_fine_sweep, SP::kSide): see the comment at its use.
struct SideState {
  double wreg;         // side threads 0..7: guess weight j = s of substep r_side + 2, in flight
  int poll, poll_need; // side thread 0: the helper's ready counter (load in flight) and the value awaited
};

  struct SideWork {
    SideState& d_;
    double2& hfar;
    double2& cbrk;
    const Common& c_;
    const SweepSync& sync;
    const double2* ring2;
    double2* prep;
    double* wguess;
    const double* brk_b;
    double* scr;
    const double* ext;
    const int& r_side;
    int bslice, helpers, hps, tau_until;
    int need_mul;
    __device__ __forceinline__ const double* tile(int beta) const {
      return scr + ((size_t)(beta & 1) * (hps + 1)) * 2 * HB * c_.size;
    }
    __device__ __forceinline__ const int* ready() const { return sync.ready + (size_t)bslice * hps; }
    // a (inverse radix-8 pass 1): publish progress, stage the tabulated guess weights, start the
    // poll of the far tile that all() of the NEXT substep reads (checked in d, three passes later)
    __device__ __forceinline__ void a() const {
      const int s = (int)threadIdx.x - 128, r = r_side;
      if (helpers && r >= 1 && (r - 1) % HB == 0) {  // rows 0..r-1 are in the path (written before the last barrier)
        pf_jitter(bslice + 1000003, (r - 1) / HB, 128);
        if (s == 0) st_release(sync.progress + bslice, r - 1);
      }
      if (s < 8) {  // weights of r + 1 (loaded a substep ago) to shared memory; those of r + 2 into flight
        wguess[s] = d_.wreg;
        const int r2 = r + 2;
        d_.wreg = (r2 < tau_until && r2 <= c_.m) ? ext[(size_t)r2 * 8 + s] : 0.0;
      }
      if (s == 0) {
        // substep r + 2 opens block (r + 1) / HB when (r + 1) % HB == 0
        d_.poll_need = (helpers && (r + 1) % HB == 0 && r + 2 <= c_.m) ? need_mul * ((r + 1) / HB + 1) : 0;
        if (d_.poll_need) d_.poll = ld_acquire(ready());
      }
    }
    // every thread, after a's barrier: its far-tile and bracket entries of substep r + 1
    // (the tile was confirmed in d of the substep before, or before the loop)
    __device__ __forceinline__ void all() const {
      const int r = r_side;
      if (r + 1 > c_.m) return;
      const double* frow = tile(r / HB) + (size_t)(r % HB) * c_.size + threadIdx.x;
      hfar = make_double2(__ldcg(frow), __ldcg(frow + 256));
      if (brk_b) {
        const double* brow = brk_b + (size_t)r * c_.size + threadIdx.x;
        cbrk = make_double2(__ldcg(brow), __ldcg(brow + 256));
      }
    }
    // near rows Q0 <= q < Q1 back from row r1 (ring), on top of (a0, a1); guess terms when GUESS.
    // The row masks are warp-uniform, so they select the WEIGHT (0 for a row outside the
    // range) instead of the result: fma(0, v, a) == a for the finite rows the ring holds
    // (the kernel zero-fills it), and no per-element selects are left in the chains.
    template <int Q0, int Q1, bool GUESS>
    __device__ __forceinline__ void rows(int r1, int J1, int p1, const double* w, int tp, double& a0, double& a1,
                                         double& g0, double& g1) const {
      double2 vv[Q1 - Q0];
#pragma unroll
      for (int q = Q0; q < Q1; ++q) vv[q - Q0] = ring2[((r1 - q) & (NR - 1)) * 256 + tp];
#pragma unroll
      for (int q = Q0; q < Q1; ++q) {
        const double wa = (r1 - q > J1) ? c_.anear[q] : 0.0;
        a0 = fma(wa, vv[q - Q0].x, a0);
        a1 = fma(wa, vv[q - Q0].y, a1);
        if (GUESS && q - 1 <= EXT) {  // guess weight j = q - 1 takes row r1 - 1 - j
          const double wg = (q - 1 <= p1) ? w[q - 1] : 0.0;
          g0 = fma(wg, vv[q - Q0].x, g0);
          g1 = fma(wg, vv[q - Q0].y, g1);
        }
      }
    }
    // b (inverse radix-8 pass 2): near rows r1-2 .. r1-8 and the guess terms of the older rows -> prep
    __device__ __forceinline__ void b() const {
      const int s = (int)threadIdx.x - 128, r = r_side, r1 = r + 1;
      if (r1 > c_.m) return;
      const int J1 = far_extent(r / HB);
      const bool tau1 = r1 >= 2 && r1 < tau_until;
      const int pk = r1 - 1 < EXO ? r1 - 1 : EXO;
      const int p1 = tau1 ? (r1 - 1 < EXT ? r1 - 1 : EXT) : pk;
      double w[EXT + 1];
#pragma unroll
      for (int j = 1; j <= EXT; ++j) w[j] = tau1 ? wguess[j] : (j <= EXO ? kExtrap[pk][j] : 0.0);
      w[0] = 0.0;
      double a[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, g[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      rows<2, 9, true>(r1, J1, p1, w, s, a[0][0], a[0][1], g[0][0], g[0][1]);
      rows<2, 9, true>(r1, J1, p1, w, s + 128, a[1][0], a[1][1], g[1][0], g[1][1]);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        prep[s + 128 * k] = make_double2(a[k][0], a[k][1]);
        prep[256 + s + 128 * k] = make_double2(g[k][0], g[k][1]);
      }
    }
    // c (forward radix-8 pass 1): near rows r1-9 .. r1-15 (present from the block's second substep on)
    __device__ __forceinline__ void c() const {
      const int s = (int)threadIdx.x - 128, r = r_side, r1 = r + 1;
      if (r1 > c_.m || r1 - 9 <= far_extent(r / HB)) return;
      const int J1 = far_extent(r / HB);
      double g0 = 0.0, g1 = 0.0;
      double2 h0 = prep[s], h1 = prep[s + 128];
      rows<9, NR, false>(r1, J1, 0, nullptr, s, h0.x, h0.y, g0, g1);
      rows<9, NR, false>(r1, J1, 0, nullptr, s + 128, h1.x, h1.y, g0, g1);
      prep[s] = h0;
      prep[s + 128] = h1;
    }
    // d (forward radix-8 pass 2): the far tile polled in a must be published
    __device__ __forceinline__ void d() const {
      if ((int)threadIdx.x == 128 && d_.poll_need) {
        int ns = 32;
        while (d_.poll < d_.poll_need) {
          __nanosleep(ns);
          ns = ns < 256 ? 2 * ns : ns;
          d_.poll = ld_acquire(ready());
        }
      }
    }
};

// Fine sweep.  Grid = nslices slice CTAs (+ nslices helper CTAs when
// `helpers`, launched cooperatively so all are co-resident).  A helper owns
// the far L1 history and the coarse-history bracket of its slice: it runs the
// register-tiled Toeplitz GEMM for block beta+1 on an otherwise idle SM while
// the slice CTA marches block beta, and publishes it with release/acquire
// flags.  Without helpers the slice CTA computes the same blocks inline (same
// code, same summation order: results are bitwise identical either way).
template <class SP, class SPP, int NT, int EPT>
__global__ void __launch_bounds__(NT) k_fine_sweep(Common c, SPP spp, const double* __restrict__ U, int n_lo,
                                                   int nslices, int helpers, int ring_off, int smem_total,
                                                   SweepSync sync,
                                                   double* paths,
                                                   double* __restrict__ out, Status* __restrict__ status) {
  extern __shared__ __align__(16) char smem[];
  constexpr int JT = (EPT > 2 ? 4 : 8);  // rows per register chunk (x2 double-buffered)
#ifndef PF_INTERLEAVE
#define PF_INTERLEAVE 0
#endif
  // PF_INTERLEAVE (one helper per slice): slice b at block 2b, its helper at 2b + 1
  const bool il = PF_INTERLEAVE && helpers == 1;
  const bool helper = il ? ((int)blockIdx.x & 1) != 0 : (int)blockIdx.x >= nslices;
  // `helpers` = helper CTAs per slice (0: far history inline).  With K > 1 the
  // far-history rows are split by row blocks (block rb -> helper rb mod K) and
  // the slice CTA sums the K partial tiles in fixed order (split-K).
  const int hps = helpers > 0 ? helpers : 1;
  const int b = il ? (int)blockIdx.x >> 1 : helper ? ((int)blockIdx.x - nslices) / hps : (int)blockIdx.x;
  const int hid = il ? 0 : helper ? ((int)blockIdx.x - nslices) % hps : 0;
  const int n = n_lo + b;
  double* path = paths + (size_t)b * (c.m + 1) * c.size;
  // per slice: [parity][hps + 1][hist | bracket][HB][size]; tile hps is the combined one
  // (+ with split tensor-core helpers: the per-batch part tiles [parity][batch][part][512])
  const int NB = c.size / TC_BATCH;
  // far history on the FP64 tensor cores: split helpers always, else when selected
  const bool tc = NT == 256 && c.size % TC_BATCH == 0 && (hps > 1 || c.far_tc > 0);
  // split helpers: each 64-mode batch's k-steps in PK interleaved parts, one (batch, part) unit per helper round
  const int PK = tc_parts(hps, NB);
  // (one TMA-fed helper: the common partial tiles of two super-blocks, [parity][TC_G][HB][size])
  // (sized by capability, not by the engine selected: launch_fine's scr_stride)
  const bool tc_cap = NT == 256 && c.size % TC_BATCH == 0;
  const size_t parts_len = (tc_cap && hps > 1) ? (size_t)2 * NB * PK * 512 : tc_cap ? (size_t)2 * TC_G * HB * c.size : 0;
  double* scr = c.scratch + (size_t)b * ((size_t)2 * (hps + 1) * 2 * HB * c.size + parts_len);
  auto slot = [&](int parity, int h) { return scr + ((size_t)parity * (hps + 1) + h) * 2 * HB * c.size; };
  double* parts = scr + (size_t)2 * (hps + 1) * 2 * HB * c.size;
  const int nblocks = (c.m + HB - 1) / HB;
  if (helper && tc) {
    // Toeplitz weights a_s into shared memory (when the table fits next to the part buffer)
    const double* aw = c.afine;
    const size_t aw_bytes = ((size_t)(c.m + HB + 1) * sizeof(double) + 15) & ~size_t(15);
    double* red = reinterpret_cast<double*>(smem);
    size_t used = 0;
    if (aw_bytes + sizeof(double) * TC_RED <= (size_t)smem_total) {
      double* s_aw = reinterpret_cast<double*>(smem);
      for (int q = threadIdx.x; q <= c.m + HB; q += NT) s_aw[q] = c.afine[q];
      aw = s_aw;
      red = reinterpret_cast<double*>(smem + aw_bytes);
      used = aw_bytes;
    }
    // the one helper of a slice streams the history rows by TMA (stages behind the weights)
    TmaRing ring{nullptr, nullptr, nullptr, 0, 0};
    if (hps == 1 && c.far_tc == 2 && aw != c.afine && NB <= NT / 32) {  // (warp w streams batch w)
      const size_t stage = sizeof(double) * 8 * (size_t)(c.size + 8);
      const size_t avail = (size_t)smem_total - used - 128;
      const int NS = (int)min((size_t)6, avail / stage);
      if (NS >= 2) {
        ring.full = reinterpret_cast<unsigned long long*>(smem + used);
        ring.empty = ring.full + 8;
        ring.buf = reinterpret_cast<double*>(smem + used + 128);
        ring.NS = NS;
        if (threadIdx.x == 0) {
          for (int i = 0; i < NS; ++i) {
            mbar_init(ring.full + i, 1);
            mbar_init(ring.empty + i, 8);
          }
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
      }
    }
    __syncthreads();
    __shared__ int s_abort;
    const int w = threadIdx.x >> 5;
    for (int beta = 0; beta < nblocks; ++beta) {
      const int J = far_extent(beta);
      PF_TH(14);
      if (J > 0) {
        if (threadIdx.x == 0) {
          int ns = 32;  // the slice CTA publishes a huge progress when it aborts
          while (ld_acquire(sync.progress + b) < J) {
            __nanosleep(ns);
            ns = ns < 256 ? 2 * ns : ns;
          }
          s_abort = ld_acquire(sync.abort + b);
        }
        __syncthreads();
        if (s_abort) return;
      }
      pf_jitter(b * 64 + hid, beta);
      PF_TH(11);
      double* hs = slot(beta & 1, 0);
      const int R0 = beta * HB;
      const double* row0 = J > 0 ? path : (c.x_start ? c.x_start : U + (size_t)n * c.size);
      if (hps == 1 && ring.NS) {
        // grouped TMA-fed helper (see TC_G): (a) tile beta = its super-block's common partial + the
        // rows after it; (b) a quarter of the next super-block's common pass
        const int S = beta / TC_G, t = beta % TC_G;
        const int Jc = tc_common_extent(S);
        {
          double acc[1][8][2];
          if (Jc > 0 && w < NB) {
            tc_frag_load(parts + (size_t)(S & 1) * TC_G * HB * c.size, t, NB, acc[0]);
          } else {
#pragma unroll
            for (int g = 0; g < 8; ++g) acc[0][g][0] = acc[0][g][1] = 0.0;
          }
          const int r0s[1] = {R0};
          tc_stream<1>(path, c.size, aw, r0s, Jc / 8, J / 8, acc, ring);
          if (w < NB) tc_store_tile(acc[0], row0, c.bfine, R0, c.size, w, hs);
        }
        PF_TH(12);
        cta_publish_add(sync.ready + (size_t)b * hps, NB);
        const int Jn = tc_common_extent(S + 1);  // <= far_extent(TC_G S) <= J: those rows are in the path
        if (Jn > 0 && TC_G * (S + 1) < nblocks) {
          const int nst = Jn / 8, st0 = t * nst / TC_G, st1 = (t + 1) * nst / TC_G;
          double* pn = parts + (size_t)((S + 1) & 1) * TC_G * HB * c.size;
          double acc[TC_G][8][2];
          int r0s[TC_G];
#pragma unroll
          for (int u = 0; u < TC_G; ++u) {
            r0s[u] = (TC_G * (S + 1) + u) * HB;
            if (t > 0 && w < NB) {
              tc_frag_load(pn, u, NB, acc[u]);
            } else {
#pragma unroll
              for (int g = 0; g < 8; ++g) acc[u][g][0] = acc[u][g][1] = 0.0;
            }
          }
          tc_stream<TC_G>(path, c.size, aw, r0s, st0, st1, acc, ring);
          if (w < NB) {
#pragma unroll
            for (int u = 0; u < TC_G; ++u) tc_frag_store(pn, u, NB, acc[u]);
          }
        }
      } else if (hps == 1) {  // the slice's one helper: batch w on warp w
        tc_far_block(path, row0, c.size, aw, c.bfine, R0, J, hs);
        PF_TH(12);
        cta_publish_add(sync.ready + (size_t)b * hps, NB);
      } else {  // split helpers (sequential solver): unit (batch, part) -> helper unit mod hps
        for (int u = hid; u < NB * PK; u += hps) {
          const int batch = u / PK, part = u % PK;
          double acc[8][2];
          tc_far_part(path, c.size, aw, R0, J, batch, part + PK * w, 8 * PK, acc);
          tc_store_part(red, acc);
          __syncthreads();
          double* pb = parts + (((size_t)(beta & 1) * NB + batch) * PK + part) * 512;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int sl = 2 * (int)threadIdx.x + i;
            double sum = red[sl];
#pragma unroll
            for (int ww = 1; ww < 8; ++ww) sum += red[(size_t)ww * 512 + sl];
            pb[sl] = sum;
          }
          if (cta_last_arrival(sync.tickets + (size_t)b * 64 + (beta & 1) * 32 + batch, PK)) {
            const double* p0 = parts + ((size_t)(beta & 1) * NB + batch) * PK * 512;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              int sl, rr, col;
              tc_out_index((int)threadIdx.x, i, sl, rr, col);
              const int e = TC_BATCH * batch + col;
              double sum = __ldcg(p0 + sl);
#pragma unroll
              for (int pp = 1; pp < PK; ++pp) sum += __ldcg(p0 + (size_t)pp * 512 + sl);
              hs[(size_t)rr * c.size + e] = c.bfine[R0 + rr] * __ldcg(row0 + e) + sum;
            }
            cta_publish_add(sync.ready + (size_t)b * hps, 1);
          }
          __syncthreads();  // red is reused by the next unit
        }
      }
    }
    return;
  }
  if (helper) {
    // Toeplitz weights a_s into shared memory once (helpers own the SM's smem)
    const double* aw = c.afine;
    if ((size_t)(c.m + HB + 1) * sizeof(double) <= (size_t)smem_total) {
      double* s_aw = reinterpret_cast<double*>(smem);
      for (int q = threadIdx.x; q <= c.m + HB; q += NT) s_aw[q] = c.afine[q];
      __syncthreads();
      aw = s_aw;
    }
    for (int beta = 0; beta < nblocks; ++beta) {
#ifdef PF_EXP_FARCAP
      const int J = far_extent(beta) < PF_EXP_FARCAP ? far_extent(beta) : PF_EXP_FARCAP;  // timing experiment: wrong numerics
#else
      const int J = far_extent(beta);
#endif
      PF_TH(14);
      if (J > 0) {
        if (threadIdx.x == 0) {
          // short backoff: the slice CTA publishes once per block and every
          // microsecond of oversleep here delays the block it will wait for
          int ns = 32;  // the slice CTA publishes a huge progress when it aborts
          while (ld_acquire(sync.progress + b) < J) {
            __nanosleep(ns);
            ns = ns < 256 ? 2 * ns : ns;
          }
        }
        if (__syncthreads_or(threadIdx.x == 0 && ld_acquire(sync.abort + b) != 0)) return;
      }
      pf_jitter(b * 64 + hid, beta);
      PF_TH(11);
      double* hs = slot(beta & 1, hid);
      const int R0 = beta * HB;
      // this helper's rows: blocks rb = hid, hid + hps, ... of HB rows starting at row 1
      double acc[HB][EPT];
      {
        const double* row0 = J > 0 ? path : (c.x_start ? c.x_start : U + (size_t)n * c.size);
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const int e = threadIdx.x + i * NT;
          const double c0 = (hid == 0 && e < c.size) ? __ldcg(row0 + e) : 0.0;
#pragma unroll
          for (int rr = 0; rr < HB; ++rr) acc[rr][i] = c.bfine[R0 + rr] * c0;
        }
      }
      // owned row chunks of CH rows (chunk rb -> helper rb mod hps), double-buffered:
      // the next chunk's loads overlap this chunk's FMAs (2*CH*EPT loads in flight)
      constexpr int CH = EPT > 2 ? 8 : 16;
      if (1 + hid * CH <= J) {
        double ca[CH][EPT], cb[CH][EPT];
        load_rows<NT, EPT, CH>(c, path, 1 + hid * CH, J, ca);
        for (int rb = hid; 1 + rb * CH <= J; rb += 2 * hps) {
          load_rows<NT, EPT, CH>(c, path, 1 + (rb + hps) * CH, J, cb);
          fma_rows<EPT, CH>(aw, R0, 1 + rb * CH, ca, acc);
          if (1 + (rb + hps) * CH > J) break;
          load_rows<NT, EPT, CH>(c, path, 1 + (rb + 2 * hps) * CH, J, ca);
          fma_rows<EPT, CH>(aw, R0, 1 + (rb + hps) * CH, cb, acc);
        }
      }
#pragma unroll
      for (int rr = 0; rr < HB; ++rr)
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const int e = threadIdx.x + i * NT;
          if (e < c.size) hs[(size_t)rr * c.size + e] = acc[rr][i];
        }
      PF_TH(12);
      cta_publish(sync.ready + b * hps + hid, beta + 1);
    }
    return;
  }
  long long t_entry = 0;
  if (threadIdx.x == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    t_entry = (long long)t0;
  }
  if (c.frozen_from && n < *c.frozen_from) {
    // frozen prefix (pipelined driver): the last correction left U_0..U_n bitwise
    // unchanged, so this slice's F_old row stands -- copied, not recomputed
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      if (e < c.size) out[(size_t)b * c.size + e] = c.fold_prev[(size_t)b * c.size + e];
    }
    if (threadIdx.x == 0) {
      if (helpers) {
        st_release(sync.abort + b, 1);  // the helper sees it and exits
        st_release(sync.progress + b, 0x3fffffff);
      }
      Status fz = {ST_OK, n, 0, -1, 0, 0, {0, 0}, t_entry, t_entry};
      status[b] = fz;
    }
    return;
  }
  SP sp;
  sp.init(smem, spp);
  double* ring = ring_off >= 0 ? reinterpret_cast<double*>(smem + ring_off) : nullptr;
  // near-history weights in shared memory (a runtime-indexed kernel-parameter
  // array would be spilled to local memory)
  __shared__ double s_anear[16];
  if (threadIdx.x < 16) s_anear[threadIdx.x] = c.anear[threadIdx.x];
  __syncthreads();
  Status st = {ST_OK, n, 0, -1, 0, 0, {0, 0}, 0, 0};
  double x[EPT];
  const double* srow = c.x_start ? c.x_start : U + (size_t)n * c.size;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = threadIdx.x + i * NT;
    x[i] = (e < c.size) ? srow[e] : 0.0;
    if (e < c.size) {
      path[e] = x[i];
      if (EPT != 2 && ring) ring[e] = x[i];
    }
  }
  if (EPT == 2 && ring) reinterpret_cast<double2*>(ring)[threadIdx.x] = make_double2(x[0], x[EPT - 1]);
  // path row 0 is read across threads by the inline tensor-core far history of block 0
  __syncthreads();
  const double* hs = nullptr;
  int J = 0;
  double hnext[EPT], cnext[EPT];  // this block's far rows, prefetched one substep ahead
  const double* brk_b = c.brk ? c.brk + (size_t)b * c.m * c.size : nullptr;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = threadIdx.x + i * NT;
    cnext[i] = (brk_b && e < c.size) ? __ldcg(brk_b + e) : 0.0;
  }
  // PCG guess weights tabulated by local substep r (Common::ext0): Lagrange
  // extrapolation in the slice's own tau = (r dt)^alpha.  Every slice starts
  // with a t^alpha-like layer in its local time (its fine history restarts at
  // t_n on top of the coarse bracket): slice 0 uses the table throughout,
  // later slices for r < TAU_LOCAL_R, then the polynomial kExtrap
  // (tools/studies/slice_start_guess.py: slice 1 388 -> 214, slice 8 227 ->
  // 171 PCG iterations over the first 128 substeps).  Prefetched one substep
  // ahead (uniform loads).
#ifndef PF_TAU1D_R
#define PF_TAU1D_R 128
#endif
  constexpr int TAU_LOCAL_R = PF_TAU1D_R;
  const double* ext = c.ext0;
  const int tau_until = ext == nullptr ? 0 : (n == 0 ? c.m + 1 : TAU_LOCAL_R);
  double wnext[EXT + 1];
#pragma unroll
  for (int j = 0; j <= EXT; ++j) wnext[j] = (2 < tau_until && c.m >= 2) ? ext[(size_t)2 * 8 + j] : 0.0;
  if constexpr (SP::kSide) {
  // ---- Q = 1024 engine: warps 4-7 idle in the radix-8 passes prepare substep r + 1 ----
  // While warps 0-3 run the two inverse radix-8 passes of substep r's setup transform,
  // warps 4-7 (side threads, two double2 ring columns = four modes each) do everything
  // of substep r + 1 that does not need x_r: the helper handshake at block boundaries
  // (publish progress, wait for the far tile: stage a), the near-history rows r - 1,
  // r - 2, ... and the PCG guess terms of the older rows (stage b, shared memory only).
  // Between the stages every thread prefetches its far-tile and bracket entries of
  // substep r + 1 (a whole substep ahead of their use).  The owner thread then finishes
  // with h = a_1 x_r + (far + h'), guess = w_0 x_r + g'.
  // (The ring always fits at this size: launch_fine checks it.)
  const double2* ring2 = reinterpret_cast<const double2*>(ring);
  double2* prep = reinterpret_cast<double2*>(smem + ring_off + sizeof(double) * NR * 2 * NT);  // [h' | g'][NT]
  __shared__ double s_wguess[8];  // tabulated guess weights of the substep being prepared
  const int tid = threadIdx.x;
  SideState sd;
  sd.wreg = 0.0;  // (substep 1 has no tabulated weights: its guess is x_0)
  sd.poll = sd.poll_need = 0;
  int r_side = 0;  // the substep the side stages run beside (they prepare r_side + 1)
  double2 hfar = make_double2(0.0, 0.0), cbrk = make_double2(0.0, 0.0);
  SideWork side{sd,      hfar, cbrk,    c,       sync,      ring2,     prep, s_wguess, brk_b, scr, ext, r_side,
         b,       helpers, hps,  tau_until, tc ? NB : 1};
  // far tile of block `bt`, computed inline when there is no helper
  auto inline_tile = [&](int bt) {
    double* s0 = slot(bt & 1, 0);
    if (tc)
      tc_far_block(path, path, c.size, c.afine, c.bfine, bt * HB, far_extent(bt), s0);
    else
      far_history_block<NT, EPT, JT>(c, path, c.afine, bt * HB, far_extent(bt), s0);
  };
  // ring rows 1..NR-1 hold zeros until their states arrive (masked rows are multiplied by a zero weight)
  for (int q = 1; q < NR; ++q) reinterpret_cast<double2*>(ring)[q * NT + tid] = make_double2(0.0, 0.0);
  if (!helpers) {
    inline_tile(0);
  } else if (tid == 0) {  // tile 0 (b_r x_0 rows: the helper needs no progress for it)
    int ns = 32;
    while (ld_acquire(side.ready()) < (tc ? NB : 1)) {
      __nanosleep(ns);
      ns = ns < 256 ? 2 * ns : ns;
    }
  }
  __syncthreads();
  if (tid >= 128) side.a();  // r_side = 0: prepares substep 1 (no near rows, guess x_0)
  side.all();
  if (tid >= 128) {
    side.b();
    side.d();
  }
  __syncthreads();
  double w0next = 1.0;  // guess weight of x_{r-1} at substep r (r = 1: the guess is x_0)
  for (int r = 1; r <= c.m; ++r) {
    const double t = (double)n * c.dT + (double)(r - 1) * c.dt;
    const int rr = (r - 1) % HB;
    const int beta = (r - 1) / HB;
#ifdef PF_TRACE
    sp.tr = ((int)blockIdx.x == PF_TRACE_SLICE && r >= PF_TRACE_R0 && r < PF_TRACE_R0 + TR_STEPS) ? r - PF_TRACE_R0 : -1;
#endif
    PF_TR(sp.tr, 0);
    PF_TR_TOP(r);
    PF_T(10);
    if (c.cancel && rr == 0 && beta > 0 &&
        __syncthreads_or(threadIdx.x == 0 && *(volatile const int*)c.cancel != 0)) {
      st.code = ST_CANCEL;  // speculative sweep after convergence: discarded
      st.r = r;
      break;
    }
    // no helper: the tile of the block that opens at r + 1 (its rows end a block ago), before stage a needs it
    if (!helpers && r % HB == 0 && r < c.m) {
      inline_tile(r / HB);
      __syncthreads();
    }
    PF_TR(sp.tr, 1);
    PF_T(8);
    const double2 hp = prep[tid], gp = prep[256 + tid];
    const double w0 = w0next;
    {
      const int r1 = r + 1;
      const bool ut = r1 < tau_until && r1 <= c.m;
      const int pk = r1 - 1 < EXO ? r1 - 1 : EXO;
      w0next = ut ? ext[(size_t)r1 * 8] : kExtrap[pk][0];
    }
    double h[EPT], ct[EPT], xg[EPT], xn[EPT];
    h[0] = hfar.x + hp.x;
    h[1] = hfar.y + hp.y;
    if (r >= 2) {
      h[0] = fma(c.anear[1], x[0], h[0]);
      h[1] = fma(c.anear[1], x[1], h[1]);
    }
    xg[0] = fma(w0, x[0], gp.x);
    xg[1] = fma(w0, x[1], gp.y);
    ct[0] = cbrk.x;
    ct[1] = cbrk.y;
    r_side = r;
    PF_TR(sp.tr, 2);
    PF_T(9);
    const int code = sp.step(c.fn, x, xg, t, c.gam_f, h, ct, xn, st, side);
    if (code != ST_OK) {
      st.code = code;
      st.r = r;
      break;
    }
    x[0] = xn[0];
    x[1] = xn[1];
    path[(size_t)r * c.size + tid] = x[0];
    path[(size_t)r * c.size + tid + NT] = x[1];
    reinterpret_cast<double2*>(ring)[(r & (NR - 1)) * NT + tid] = make_double2(x[0], x[1]);
    PF_TR(sp.tr, 47);
  }
  } else {
  for (int r = 1; r <= c.m; ++r) {
    const double t = (double)n * c.dT + (double)(r - 1) * c.dt;
    const int rr = (r - 1) % HB;
    const int beta = (r - 1) / HB;
#ifdef PF_TRACE
    sp.tr = ((int)blockIdx.x == PF_TRACE_SLICE && r >= PF_TRACE_R0 && r < PF_TRACE_R0 + TR_STEPS) ? r - PF_TRACE_R0 : -1;
#endif
    PF_TR(sp.tr, 0);
    PF_TR_TOP(r);
    PF_T(10);
    if (c.cancel && rr == 0 && beta > 0 &&
        __syncthreads_or(threadIdx.x == 0 && *(volatile const int*)c.cancel != 0)) {
      st.code = ST_CANCEL;  // speculative sweep after convergence: discarded
      st.r = r;
      break;
    }
    if (rr == 0) {
      J = far_extent(beta);
      double* s0 = slot(beta & 1, 0);
      if (helpers && tc) {
        pf_jitter(b + 1000003, beta);
        cta_publish(sync.progress + b, r - 1);  // rows 0..r-1 are in the path
        if (threadIdx.x == 0) {  // every 64-mode batch of block beta published
          int ns = 32;
          while (ld_acquire(sync.ready + (size_t)b * hps) < NB * (beta + 1)) {
            __nanosleep(ns);
            ns = ns < 256 ? 2 * ns : ns;
          }
        }
        __syncthreads();
      } else if (tc) {
        tc_far_block(path, path, c.size, c.afine, c.bfine, beta * HB, J, s0);
        __syncthreads();  // the tile rows are read by other threads below
      } else if (helpers) {
        pf_jitter(b + 1000003, beta);
        cta_publish(sync.progress + b, r - 1);  // rows 0..r-1 are in the path
        if (threadIdx.x == 0) {
          for (int h = 0; h < hps; ++h) {
            int ns = 32;
            while (ld_acquire(sync.ready + b * hps + h) < beta + 1) {
              __nanosleep(ns);
              ns = ns < 256 ? 2 * ns : ns;
            }
          }
        }
        __syncthreads();
        if (hps > 1) {  // combine the split-K partial tiles (fixed order) into tile hps
          double* cmb = slot(beta & 1, hps);
#pragma unroll
          for (int i = 0; i < EPT; ++i) {
            const int e = threadIdx.x + i * NT;
            if (e < c.size) {
              for (int q = 0; q < HB; ++q) {
                double acc = 0.0;
                for (int h = 0; h < hps; ++h) acc += __ldcg(slot(beta & 1, h) + (size_t)q * c.size + e);
                cmb[(size_t)q * c.size + e] = acc;
                cmb[(size_t)(HB + q) * c.size + e] = __ldcg(s0 + (size_t)(HB + q) * c.size + e);
              }
            }
          }
          s0 = cmb;
        }
      } else {
        far_history_block<NT, EPT, JT>(c, path, c.afine, beta * HB, J, s0);
      }
      hs = s0;
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        hnext[i] = (e < c.size) ? __ldcg(hs + e) : 0.0;
      }
    }
    PF_TR(sp.tr, 1);
    PF_T(8);
    double hcur[EPT], ccur[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      hcur[i] = hnext[i];
      ccur[i] = cnext[i];
    }
    if (rr + 1 < HB) {  // issue next substep's far-row loads now; they land during this step
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        hnext[i] = (e < c.size) ? __ldcg(hs + (size_t)(rr + 1) * c.size + e) : 0.0;
      }
    }
    if (r < c.m) {  // next substep's bracket row, landing during this step
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        cnext[i] = (brk_b && e < c.size) ? __ldcg(brk_b + (size_t)r * c.size + e) : 0.0;
      }
    }
    const bool use_tau = r >= 2 && r < tau_until;
    const int pk = r - 1 < EXO ? r - 1 : EXO;
    const int p = use_tau ? (r - 1 < EXT ? r - 1 : EXT) : pk;  // tabulated rows are zero beyond their order
    double wcur[EXT + 1];
#pragma unroll
    for (int j = 0; j <= EXT; ++j) {
      wcur[j] = use_tau ? wnext[j] : (j <= EXO ? kExtrap[pk][j] : 0.0);
      if (r + 1 < tau_until && r + 1 <= c.m) wnext[j] = ext[(size_t)(r + 1) * 8 + j];
    }
    double h[EPT], ct[EPT], xg[EPT], xn[EPT];
    // EPT = 2 (every size == 2 NT variant): the ring holds a thread's two entries
    // side by side, one 16-byte load per row feeding both entries' chains; near
    // weights from the parameter bank
    if (EPT == 2 && ring) {
      const double2* ring2 = reinterpret_cast<const double2*>(ring);
      double a0 = hcur[0], a1 = hcur[EPT - 1], g0 = wcur[0] * x[0], g1 = wcur[0] * x[EPT - 1];
#pragma unroll
      for (int q = 1; q < NR; ++q) {
        const double2 vv = (r - q >= 0) ? ring2[((r - q) & (NR - 1)) * NT + threadIdx.x] : make_double2(0.0, 0.0);
        if (r - q > J) {
          a0 = fma(c.anear[q], vv.x, a0);
          a1 = fma(c.anear[q], vv.y, a1);
        }
        if (q - 1 >= 1 && q - 1 <= EXT && q - 1 <= p) {  // guess weight j = q - 1 takes row r - 1 - j
          g0 = fma(wcur[q - 1], vv.x, g0);
          g1 = fma(wcur[q - 1], vv.y, g1);
        }
      }
      h[0] = a0;
      h[EPT - 1] = a1;
      ct[0] = ccur[0];
      ct[EPT - 1] = ccur[EPT - 1];
      xg[0] = g0;
      xg[EPT - 1] = g1;
    }
#pragma unroll
    for (int i = 0; i < EPT && !(EPT == 2 && ring); ++i) {
      const int e = threadIdx.x + i * NT;
      double acc = 0.0, cb = 0.0, g = x[i];
      if (e < c.size) {
        acc = hcur[i];
        cb = ccur[i];
        // extrapolated guess; row r-1 is x itself
        const double* w = wcur;
        g = w[0] * x[i];
        if (ring) {
          // all NR-1 recent rows first (independent shared loads), then the two FMA chains;
          // v[q-1] is the row at distance q (row r-q)
          double v[NR - 1];
#pragma unroll
          for (int q = 1; q < NR; ++q) v[q - 1] = (r - q >= 0) ? ring[((r - q) & (NR - 1)) * c.size + e] : 0.0;
#pragma unroll
          for (int q = 1; q < NR; ++q)
            if (r - q > J) acc = fma(s_anear[q], v[q - 1], acc);
#pragma unroll
          for (int j = 1; j <= EXT; ++j)
            if (j <= p) g = fma(w[j], v[j], g);
        } else {
          for (int j = J + 1; j < r; ++j) acc = fma(s_anear[r - j], path[(size_t)j * c.size + e], acc);
          for (int j = 1; j <= p; ++j) g = fma(w[j], path[(size_t)(r - 1 - j) * c.size + e], g);
        }
      }
      h[i] = acc;
      ct[i] = cb;
      xg[i] = g;
    }
    PF_TR(sp.tr, 2);
    PF_T(9);
    const int code = sp.step(c.fn, x, xg, t, c.gam_f, h, ct, xn, st);
    if (code != ST_OK) {
      st.code = code;
      st.r = r;
      break;
    }
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      x[i] = xn[i];
      if (e < c.size) {
        path[(size_t)r * c.size + e] = x[i];
        if (EPT != 2 && ring) ring[(size_t)(r & (NR - 1)) * c.size + e] = x[i];
      }
    }
    if (EPT == 2 && ring)
      reinterpret_cast<double2*>(ring)[(r & (NR - 1)) * NT + threadIdx.x] = make_double2(x[0], x[EPT - 1]);
    PF_TR(sp.tr, 47);
  }
  }  // !SP::kSide
  if (st.code == ST_OK) {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * NT;
      if (e < c.size) out[(size_t)b * c.size + e] = x[i];
    }
  } else if (helpers && threadIdx.x == 0) {
    st_release(sync.abort + b, 1);
    st_release(sync.progress + b, 0x3fffffff);  // wakes the helpers, which then see the abort
  }
  if (threadIdx.x == 0) {
    unsigned long long tend;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tend));
    st.t_start = t_entry;
    st.t_end = (long long)tend;
    status[b] = st;
  }
}

// coarse step G(H[0..n]) -> x  (stepping.py:87-112)
template <class SP, int NT, int EPT>
// PCG guess: kind 0 -> U_n; 1 -> 2 U_n - U_{n-1} (run_coarse); 2 -> G_old[n] + (U_next[n] - U_cur[n])
// (correction sweep: the previous sweep's coarse step of the slightly different state)
__device__ __forceinline__ int coarse_apply(SP& sp, const Common& c, const double* H, int n, double* xout,
                                            Status& st, int guess = 0, const double* gold = nullptr,
                                            const double* ucur = nullptr) {
  double h[EPT], z[EPT], xp[EPT], xg[EPT];
  const double* __restrict__ b = c.bfine;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = threadIdx.x + i * NT;
    z[i] = 0.0;
    h[i] = 0.0;
    xp[i] = 0.0;
    if (e < c.size) {
      double acc = b[n] * H[e];
      for (int j = 1; j <= n; ++j) acc = fma(b[n - j] - b[n - j + 1], H[(size_t)j * c.size + e], acc);
      h[i] = acc;
      xp[i] = H[(size_t)n * c.size + e];
    }
    xg[i] = xp[i];
    if (e < c.size && guess == 1 && n >= 1) xg[i] = fma(2.0, xp[i], -H[(size_t)(n - 1) * c.size + e]);
    if (e < c.size && guess == 2) xg[i] = gold[(size_t)n * c.size + e] + (xp[i] - ucur[(size_t)n * c.size + e]);
  }
  return sp.step(c.fn, xp, xg, (double)n * c.dT, c.gam_c, h, z, xout, st);
}

enum CoarseMode : int { CM_RUN = 0, CM_CORRECT = 1, CM_SINGLE = 2 };

struct CoarseArgs {
  int mode;
  int n_single;      // CM_SINGLE: history rows 0..n_single in `traj`
  int k_iter;        // CM_CORRECT: iteration index for DivergenceError
  double guard;      // CM_CORRECT: divergence guard
  double* traj;      // CM_RUN: (nt+1) rows, row 0 preset; CM_SINGLE: history
  const double* ucur;
  const double* fold;
  const double* gold;
  double* gnew;
  double* unext;
  double* out;       // CM_SINGLE result; CM_CORRECT: out[0] = diff
  // CM_CORRECT over nodes [n_begin, n_end) (n_end = 0: all); the frozen-prefix
  // state crosses chunk launches in state[0] (same), [1] (first changed node),
  // [2] (a chunk failed: later chunks do nothing); guards + diff in the last chunk
  int n_begin, n_end;
  int* state;
};

template <class SP, class SPP, int NT, int EPT>
__global__ void __launch_bounds__(NT) k_coarse(Common c, SPP spp, CoarseArgs a, Status* __restrict__ status) {
  extern __shared__ __align__(16) char smem[];
  SP sp;
  sp.init(smem, spp);
  Status st = {ST_OK, 0, -1, -1, 0, 0, {0, 0}, 0, 0};
  double x[EPT];
  if (a.mode == CM_SINGLE) {
    st.n = a.n_single;
    const int code = coarse_apply<SP, NT, EPT>(sp, c, a.traj, a.n_single, x, st);
    if (code != ST_OK) {
      st.code = code;
    } else {
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        if (e < c.size) a.out[e] = x[i];
      }
    }
  } else if (a.mode == CM_RUN) {
    for (int n = 0; n < c.nt; ++n) {
      st.n = n;
      const int code = coarse_apply<SP, NT, EPT>(sp, c, a.traj, n, x, st, 1);
      if (code != ST_OK) {
        st.code = code;
        break;
      }
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        if (e < c.size) a.traj[(size_t)(n + 1) * c.size + e] = x[i];
      }
    }
  } else {  // CM_CORRECT (parareal.py:114-128)
    const int nb = a.n_begin, ne = a.n_end > 0 ? a.n_end : c.nt;
    if (nb > 0 && a.state[2] != 0) return;  // an earlier chunk failed and reported
    if (nb == 0) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        if (e < c.size) a.unext[e] = a.ucur[e];
      }
    }
    // Frozen prefix: while U_next[0..n] equals U_cur[0..n] bitwise, the coarse
    // step of node n has exactly G_old[n]'s inputs (G_old is the previous
    // sweep's G_new of U_cur), so G_new[n] = G_old[n] without a solve -- the
    // finite-termination structure of parareal.py:114-118, exploited exactly.
    // `same` is CTA-uniform (__syncthreads_and); first_changed = the first node
    // whose state this sweep changed (the next fine sweep starts there).
    bool same = nb == 0 || a.state[0] != 0;
    int first_changed = nb == 0 ? c.nt + 1 : a.state[1];
    for (int n = nb; n < ne; ++n) {
      st.n = n;
      if (same && n > 0) {
        int eq = 1;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const int e = threadIdx.x + i * NT;
          if (e < c.size) {
            const size_t o = (size_t)n * c.size + e;
            eq &= __double_as_longlong(a.unext[o]) == __double_as_longlong(a.ucur[o]);
          }
        }
        same = __syncthreads_and(eq) != 0;
        if (!same) first_changed = n;
      }
      if (same) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const int e = threadIdx.x + i * NT;
          x[i] = e < c.size ? a.gold[(size_t)n * c.size + e] : 0.0;
        }
      } else {
        const int code = coarse_apply<SP, NT, EPT>(sp, c, a.unext, n, x, st, 2, a.gold, a.ucur);
        if (code != ST_OK) {
          st.code = code;
          break;
        }
      }
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        if (e < c.size) {
          const size_t o = (size_t)n * c.size + e;
          a.gnew[o] = x[i];
          a.unext[o + c.size] = a.fold[o] + (x[i] - a.gold[o]);
        }
      }
    }
    if (ne < c.nt) {  // chunk boundary: hand the state to the next chunk launch
      if (threadIdx.x == 0) {
        a.state[0] = same ? 1 : 0;
        a.state[1] = first_changed;
        a.state[2] = st.code != ST_OK;
        if (st.code != ST_OK) status[0] = st;
      }
      return;
    }
    if (same && st.code == ST_OK) {  // last node
      int eq = 1;
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        if (e < c.size) {
          const size_t o = (size_t)c.nt * c.size + e;
          eq &= __double_as_longlong(a.unext[o]) == __double_as_longlong(a.ucur[o]);
        }
      }
      if (!__syncthreads_and(eq)) first_changed = c.nt;
    }
    if (st.code == ST_OK) {
      // guards and diff (parareal.py:120-128): same ownership, no sync needed
      int first_bad = 0x7fffffff;
      double nmax = -1.0, dmax = 0.0;
      int nmax_at = 0;
      for (int n = 0; n <= c.nt; ++n) {
        double v[EPT], d[EPT];
        int fin = 1;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const int e = threadIdx.x + i * NT;
          v[i] = d[i] = 0.0;
          if (e < c.size) {
            v[i] = a.unext[(size_t)n * c.size + e];
            d[i] = v[i] - a.ucur[(size_t)n * c.size + e];
            if (!isfinite(v[i])) fin = 0;
          }
        }
        const double2 s = sp.red.sum2(sp.norm2_partial(v), sp.norm2_partial(d));
        const int allfin = sp.red.min_int(fin);
        if (!allfin && first_bad == 0x7fffffff) first_bad = n;
        const double nn = sqrt(s.x), dd = sqrt(s.y);
        if (nn > nmax) {
          nmax = nn;
          nmax_at = n;
        }
        dmax = fmax(dmax, dd);
      }
      if (first_bad != 0x7fffffff) {
        st.code = ST_DIVERGE;
        st.n = first_bad;
        st.r = 0;
      } else if (nmax > a.guard) {
        st.code = ST_DIVERGE;
        st.n = nmax_at;
        st.r = 1;
      }
      if (threadIdx.x == 0) {
        a.out[0] = dmax;
        a.out[1] = (double)first_changed;
        a.state[1] = first_changed;
      }
    }
  }
  if (threadIdx.x == 0) status[0] = st;
}

}  // namespace pf
