// C-ABI of the B200 parareal fine-propagator path (include/parafrac_b200.h).
//
// Host side of the drop-in boundary: context (tables, buffers, stream),
// kernel dispatch per space, status decoding into the reference's error
// conventions (errors.py:8-34), and the on-device parareal state machine
// (parareal.py:91-155).  No CPU compute path exists: every entry point that
// computes launches sm_100a kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/parafrac_b200.h"
#include "pf_cheb1d.cuh"
#include "pf_device.cuh"
#include "pf_kernels.cuh"
#include "pf_sine1d.cuh"
#include "pf_sine2d.cuh"
#include "pf_line16.cuh"
#include "pf_line32.cuh"

using pf::cd;
using pf::Status;

namespace {

// Sine variants by log2(Q): (threads per CTA, modes per thread)
//   LG 2-6: (32, 1)  LG 7: (32, 2)  LG 8: (64, 2)  LG 9: (128, 2)  LG 10: (256, 2)  LG 11: (256, 4)
enum Variant { V_NONE = 0, V_S2, V_S3, V_S4, V_S5, V_S6, V_S7, V_S8, V_S9, V_S10, V_S11, V_CHEB_128_1, V_CHEB_512_1 };

struct DevBuf {
  double* p = nullptr;
  size_t n = 0;  // doubles
  int ensure(size_t want) {
    if (want <= n) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (cudaMalloc(&p, want * sizeof(double)) != cudaSuccess) return -1;
    n = want;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct Engine2D;  // 2-D sine engine (pf_engine2d.inc)
}  // namespace

struct pf_ctx {
  int device = -1;  // set once cudaSetDevice succeeded (pf_destroy touches no device before)
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  pf_problem prob{};
  pf_grid grid{};
  int kind = 0, size = 0, M = 0, Q = 0, lgQ = 0, npts = 0, ni = 0;
  double dT = 0, dt = 0, gam_f = 0, gam_c = 0, minv = 0, g2m = 0;
  double pcg_tol = 1e-14;
  int pcg_maxit = 500;
  Variant variant = V_NONE;
  size_t smem = 0;
  std::vector<double> h_bfine, h_bfrac, h_nodes, h_d1, h_qw;
  // device tables
  double *d_bfine = nullptr, *d_afine = nullptr, *d_bfrac = nullptr, *d_ext0 = nullptr, *d_nodes = nullptr, *d_d1 = nullptr, *d_qw = nullptr;
  cd *d_tw = nullptr, *d_ph = nullptr;  // d_tw: per-pass twiddle tables
  long len_fine = 0, len_frac = 0;
  // work buffers
  DevBuf U, Unext, paths, fold, gold, gnew, io, scalar, scratch, brk;
  Status* d_status = nullptr;
  int status_cap = 0;
  std::vector<Status> h_status;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // head start of slice 0 (launch_fine): its own stream and fork/join events
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  pf_stats stats{};
  pf_error err{};
  double guard = 0;
  bool parareal_ready = false;
  int frozen = 0;  // leading nodes the last correction left bitwise unchanged
  // Warm start of the parareal fine sweeps (2-D): each slice's path of the
  // previous sweep, double-buffered and indexed by slice, seeds the PCG guess
  // of the same substep of the next sweep (see k2_prep).
  DevBuf wpaths[2];
  int warm_iter = 0;        // parareal fine sweeps since init
  double warm_diff = 1.0;   // last correction's diff (picks the guess order)
  int pending_lo = -1, pending_bs = 0;  // last async fine launch, decoded by pf_dev_check
  int* d_sync = nullptr;                 // sweep progress / ready / abort flags
  int sync_cap = 0;
  int num_sms = 0;
  int allow_helpers = 1;  // PF_NO_HELPERS=1 forces the inline far history
  int last_helpers = 0;
  // pipelined parareal driver (1-D): second F_old buffer, per-parity sweep status,
  // correction chunk state, cancel word, chunk streams and events
  DevBuf fold2;
  DevBuf cheb_aug;         // global-residence Chebyshev bridge: one augmented system per slice slot (Cheb1D<512, 1>)
  DevBuf cheb_aug_coarse;  // ... and the coarse kernel's own (it overlaps fine sweeps in the pipelined driver)
  Status* d_status2 = nullptr;
  Status* d_corr_status = nullptr;
  int* d_corr_state = nullptr;  // [parity][4]: same, first changed, failed
  int* d_cancel = nullptr;
  cudaStream_t pstream[8] = {};
  cudaEvent_t ev_sw[2][8] = {}, ev_co[2][8] = {}, ev_init = nullptr;
  Engine2D* e2 = nullptr;   // PF_SPACE_SINE2D only
  Engine2D* e2c = nullptr;  // batch-1 engine of the graph-captured sequential sweeps (stable buffers)
};

namespace {  // 2-D engine entry points (defined in pf_engine2d.inc)
int e2_fine_sweep(pf_ctx* c, const double* d_u, int n_lo, int bs, double* d_out, int m, bool with_bracket,
                  double* d_all = nullptr, bool warm = false, const double* d_start = nullptr);
int e2_coarse_step(pf_ctx* c, const double* d_H, int n, double* d_out, int guess = 0,
                   const double* gold = nullptr, const double* ucur = nullptr);
int e2_run_coarse(pf_ctx* c, double* d_traj);
int e2_correct(pf_ctx* c, const double* ucur, const double* fold, const double* gold, double* gnew, double* unext,
               int k, double* diff);
}  // namespace

namespace {

int set_error(pf_ctx* c, int code, const char* msg) {
  c->err = pf_error{};  // no stale step/node fields from an earlier error
  c->err.code = code;
  std::snprintf(c->err.message, sizeof(c->err.message), "%s", msg);
  return code;
}

int cuda_fail(pf_ctx* c, cudaError_t e, const char* where) {
  c->err = pf_error{};
  c->err.code = PF_ERR_CUDA;
  c->err.cuda_error = (int)e;
  std::snprintf(c->err.message, sizeof(c->err.message), "%s: %s", where, cudaGetErrorString(e));
  return PF_ERR_CUDA;
}

#define PF_CUDA(ctx, call)                                   \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call); \
  } while (0)

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

pf::Common make_common(const pf_ctx* c) {
  pf::Common cm{};
  cm.fn.id = c->prob.functor;
  for (int i = 0; i < 6; ++i) cm.fn.p[i] = c->prob.p[i];
  cm.size = c->size;
  cm.nt = c->grid.nt;
  cm.m = c->grid.m;
  cm.dT = c->dT;
  cm.dt = c->dt;
  cm.gam_f = c->gam_f;
  cm.gam_c = c->gam_c;
  cm.minv = c->minv;
  cm.bfine = c->d_bfine;
  cm.afine = c->d_afine;
  cm.bfrac = c->d_bfrac;
  cm.scratch = c->scratch.p;
  cm.ext0 = c->d_ext0;
  for (int s = 0; s < 16; ++s) cm.anear[s] = (s >= 1 && s < (long)c->h_bfine.size()) ? c->h_bfine[s - 1] - c->h_bfine[s] : 0.0;
  return cm;
}

pf::Sine1DParams sine_params(const pf_ctx* c) {
  pf::Sine1DParams p{};
  p.M = c->M;
  p.Q = c->Q;
  p.lgQ = c->lgQ;
  p.twp = c->d_tw;
  p.ph = c->d_ph;
  p.pcg_tol = c->pcg_tol;
  p.pcg_maxit = c->pcg_maxit;
  return p;
}

pf::Cheb1DParams cheb_params(const pf_ctx* c) {
  pf::Cheb1DParams p{};
  p.npts = c->npts;
  p.ni = c->ni;
  p.nodes = c->d_nodes;
  p.d1 = c->d_d1;
  p.qw = c->d_qw;
  p.aug_g = c->variant == V_CHEB_512_1 ? c->cheb_aug.p : nullptr;  // (sized by ensure_cheb_aug before every launch)
  p.aug_stride = (size_t)c->ni * pf::Cheb1D<512, 1>::ld_of(c->ni);
  return p;
}

// the global-residence Chebyshev systems of a launch start at buffer slot q0 (one slab per CTA)
inline void offset_slab(pf::Sine1DParams&, size_t) {}
inline void offset_slab(pf::Cheb1DParams& p, size_t q0) {
  if (p.aug_g) p.aug_g += q0 * p.aug_stride;
}
// the coarse kernel (one CTA) uses its own system slab
inline void coarse_slab(pf::Sine1DParams&, const pf_ctx*) {}
inline void coarse_slab(pf::Cheb1DParams& p, const pf_ctx* c) {
  if (c->variant == V_CHEB_512_1) p.aug_g = c->cheb_aug_coarse.p;
}
int ensure_cheb_aug(pf_ctx* c, size_t slots) {
  if (c->variant != V_CHEB_512_1) return 0;
  const size_t stride = (size_t)c->ni * pf::Cheb1D<512, 1>::ld_of(c->ni);
  return c->cheb_aug.ensure(slots * stride);
}

// Dispatch: binds SP (space type), SPP (its params), NT, EPT and `spp`.
#ifdef PF_ONLY_S10  // experiment builds (tools/): the config-3 variant only, a quarter of the compile time
#define PF_DISPATCH(ctx, ...) \
  switch ((ctx)->variant) { \
    case V_S10: { using SP = pf::Sine1D<256, 2, 10>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 256, EPT = 2; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    default: \
      return set_error(ctx, PF_ERR_UNSUPPORTED, "no kernel variant"); \
  }

#else
#define PF_DISPATCH(ctx, ...) \
  switch ((ctx)->variant) { \
    case V_S2: { using SP = pf::Sine1D<32, 1, 2>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 32, EPT = 1; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S3: { using SP = pf::Sine1D<32, 1, 3>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 32, EPT = 1; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S4: { using SP = pf::Sine1D<32, 1, 4>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 32, EPT = 1; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S5: { using SP = pf::Sine1D<32, 1, 5>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 32, EPT = 1; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S6: { using SP = pf::Sine1D<32, 1, 6>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 32, EPT = 1; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S7: { using SP = pf::Sine1D<128, 1, 7>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 128, EPT = 1; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S8: { using SP = pf::Sine1D<64, 2, 8>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 64, EPT = 2; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S9: { using SP = pf::Sine1D<128, 2, 9>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 128, EPT = 2; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S10: { using SP = pf::Sine1D<256, 2, 10>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 256, EPT = 2; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_S11: { using SP = pf::Sine1D<256, 4, 11>; using SPP = pf::Sine1DParams; \
      constexpr int NT = 256, EPT = 4; SPP spp = sine_params(ctx); __VA_ARGS__; } break; \
    case V_CHEB_128_1: { using SP = pf::Cheb1D<128, 1>; using SPP = pf::Cheb1DParams; \
      constexpr int NT = 128, EPT = 1; SPP spp = cheb_params(ctx); __VA_ARGS__; } break; \
    case V_CHEB_512_1: { using SP = pf::Cheb1D<512, 1>; using SPP = pf::Cheb1DParams; \
      constexpr int NT = 512, EPT = 1; SPP spp = cheb_params(ctx); __VA_ARGS__; } break; \
    default: \
      return set_error(ctx, PF_ERR_UNSUPPORTED, "no kernel variant"); \
  }
#endif

int ensure_status(pf_ctx* c, int n) {
  if (n <= c->status_cap) return 0;
  if (c->d_status) cudaFree(c->d_status);
  c->d_status = nullptr;
  c->status_cap = 0;
  PF_CUDA(c, cudaMalloc(&c->d_status, sizeof(Status) * n));
  c->status_cap = n;
  c->h_status.resize(n);
  return 0;
}

// Launch the fine sweep for slices [n_lo, n_lo+bs) reading device states d_u.
// When 2*bs CTAs fit on the device at once, launch cooperatively with one
// helper CTA per slice (far history on otherwise idle SMs); else inline.
#ifndef PF_BRK_RT
#define PF_BRK_RT 16  // target rows per thread of k_bracket_all (8 / 16 / 32 measured: 16)
#endif
#ifndef PF_BRK_EM
#define PF_BRK_EM 2  // modes per thread of k_bracket_all
#endif
// Options of the pipelined parareal driver's sweep launches: buffers at slot
// offsets of a fixed capacity (chunks of one sweep run concurrently on their own
// streams), the frozen-prefix skip and the cancel word (k_fine_sweep).
struct FineOpts {
  int slot0 = 0, cap = 0;
  cudaStream_t stream = nullptr;
  const int* frozen_from = nullptr;
  const double* fold_prev = nullptr;
  const int* cancel = nullptr;
};

int launch_fine(pf_ctx* c, const double* d_u, int n_lo, int bs, double* d_out, Status* d_st, int m_override = 0,
                int hps_req = 1, const double* d_start = nullptr, const FineOpts* fo = nullptr) {
  if (d_start && bs != 1) return set_error(c, PF_ERR_ARGUMENT, "a start state needs a single-slice sweep");
  if (c->kind == PF_SPACE_SINE2D) {
    // the parareal driver's own sweeps (states == U) warm-start from the previous sweep
    const bool warm = c->parareal_ready && d_u == c->U.p && m_override == 0 && !d_start;
    return e2_fine_sweep(c, d_u, n_lo, bs, d_out, c->grid.m, true, nullptr, warm, d_start);
  }
  const int m = m_override > 0 ? m_override : c->grid.m;
  const int hps = std::max(1, hps_req);
  const int slot0 = fo ? fo->slot0 : 0, cap = fo ? std::max(fo->cap, fo->slot0 + bs) : bs;
  cudaStream_t stream_keep = c->stream;
  if (fo && fo->stream) c->stream = fo->stream;
  struct Restore {
    pf_ctx* c;
    cudaStream_t s;
    ~Restore() { c->stream = s; }
  } restore{c, stream_keep};
  if (c->paths.ensure((size_t)cap * (m + 1) * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "paths");
  // per slice: block tiles [parity][hps + 1][2][HB][size] (+ the split tensor-core
  // helpers' part tiles [parity][batch][part][512], k_fine_sweep)
  const bool tc = c->kind == PF_SPACE_SINE1D && c->lgQ >= 10 && c->size % pf::TC_BATCH == 0;
  const size_t parts_len =
      (tc && hps > 1) ? (size_t)2 * (c->size / pf::TC_BATCH) * pf::tc_parts(hps, c->size / pf::TC_BATCH) * 512
      : tc            ? (size_t)2 * pf::TC_G * pf::HB * c->size
                      : 0;
  // far history of one-helper sweeps (PF_FAR_TC): 0 DFMA register tiles, 1 DMMA with direct
  // loads, 2 DMMA fed by TMA bulk copies with the old rows accumulated for four tiles per pass
  // (pf_kernels.cuh TC_G).  Late in a config-3 sweep every helper re-reads its slice's whole path
  // once per block -- 269 MB per block period, more than HBM delivers -- and engines 0 and 1 made
  // the slice CTAs wait from block ~88 of 128 on; engine 2 reads a quarter of that and is the
  // default where its one-warp-per-batch layout applies (M = 512).
  int far_tc = (tc && c->size / pf::TC_BATCH <= 8) ? 2 : 0;
  if (const char* ft = std::getenv("PF_FAR_TC")) far_tc = (ft[0] == '1') ? 1 : (ft[0] == '2') ? 2 : 0;
  const size_t scr_stride = (size_t)2 * (hps + 1) * 2 * pf::HB * c->size + parts_len;
  if (c->scratch.ensure((size_t)cap * scr_stride)) return cuda_fail(c, cudaErrorMemoryAllocation, "scratch");
  if (ensure_cheb_aug(c, (size_t)cap)) return cuda_fail(c, cudaErrorMemoryAllocation, "chebyshev systems");
  // sync words: progress[cap] | ready[cap * hps] | abort[cap] | tickets[cap * 64]
  const int nsync = cap * (2 + hps) + cap * 64;
  if (c->sync_cap < nsync) {
    if (fo) PF_CUDA(c, cudaDeviceSynchronize());  // concurrent chunk launches may still use the old words
    if (c->d_sync) cudaFree(c->d_sync);
    c->d_sync = nullptr;
    c->sync_cap = 0;
    PF_CUDA(c, cudaMalloc(&c->d_sync, sizeof(int) * nsync));
    c->sync_cap = nsync;
  }
  int* sy_progress = c->d_sync;
  int* sy_ready = c->d_sync + cap;
  int* sy_abort = c->d_sync + cap + (size_t)cap * hps;
  int* sy_tickets = c->d_sync + 2 * cap + (size_t)cap * hps;
  PF_CUDA(c, cudaMemsetAsync(sy_progress + slot0, 0, sizeof(int) * bs, c->stream));
  PF_CUDA(c, cudaMemsetAsync(sy_ready + (size_t)slot0 * hps, 0, sizeof(int) * bs * hps, c->stream));
  PF_CUDA(c, cudaMemsetAsync(sy_abort + slot0, 0, sizeof(int) * bs, c->stream));
  PF_CUDA(c, cudaMemsetAsync(sy_tickets + (size_t)slot0 * 64, 0, sizeof(int) * bs * 64, c->stream));
  pf::Common cm = make_common(c);
  cm.m = m;
  cm.x_start = d_start;
  cm.far_tc = far_tc;
  if (fo) {
    cm.frozen_from = fo->frozen_from;
    cm.fold_prev = fo->fold_prev;
    cm.cancel = fo->cancel;
  }
  if (!fo) PF_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  if (bs > 65535) return set_error(c, PF_ERR_UNSUPPORTED, "more than 65535 slices in one sweep launch");
  // Launch the sweep of slices [n_lo + s0, n_lo + s0 + ns) (local slices s0..) on stream st:
  // per-slice sync flags, paths, scratch, outputs and status at the local offsets.
  auto sweep = [&](int s0, int ns, cudaStream_t st, const double* brk) -> int {
    pf::Common cl = cm;
    const size_t q0 = (size_t)slot0 + s0;  // buffer slot of local slice s0
    cl.scratch = c->scratch.p + q0 * scr_stride;
    cl.brk = brk;
    if (cl.fold_prev) cl.fold_prev += (size_t)s0 * c->size;
    pf::SweepSync sync{sy_progress + q0, sy_ready + q0 * hps, sy_abort + q0, sy_tickets + q0 * 64};
    double* dp = c->paths.p + q0 * (m + 1) * c->size;
    double* dout = d_out ? d_out + (size_t)s0 * c->size : nullptr;
    Status* dst = d_st + s0;
    int nl = n_lo + s0;
    PF_DISPATCH(c, {
      auto kern = pf::k_fine_sweep<SP, SPP, NT, EPT>;
      offset_slab(spp, q0);
      int per_sm = 0;
      // shared-memory ring of the last NR states behind the space's own smem
      const size_t ring_bytes = sizeof(double) * pf::NR * c->size;
      const size_t base = (c->smem + 15) & ~size_t(15);
      int ring_off = -1;
      size_t smem = c->smem;
      if (base + ring_bytes <= 227 * 1024) {
        ring_off = (int)base;
        smem = base + ring_bytes;
      }
      if (SP::kSide) {  // + the side warps' prepared rows [h' | guess'][NT] (16 bytes each)
        if (ring_off < 0) return set_error(c, PF_ERR_UNSUPPORTED, "the state ring must fit at this size");
        smem += 2 * 16 * (size_t)NT;
      }
      // split tensor-core helpers (sequential solver) keep their part buffer in this space
      if (tc && hps > 1 && smem < sizeof(double) * pf::TC_RED) smem = sizeof(double) * pf::TC_RED;
      PF_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      PF_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
      int helpers = (c->allow_helpers && bs * (1 + hps) <= per_sm * c->num_sms) ? hps : 0;
      if (!helpers && hps > 1) return set_error(c, PF_ERR_UNSUPPORTED, "split-K helpers do not fit on the device");
      int nsl = ns;
      int smem_total = (int)smem;
      if (helpers) {
        void* args[] = {(void*)&cl, (void*)&spp, (void*)&d_u, (void*)&nl, (void*)&nsl, (void*)&helpers,
                        (void*)&ring_off, (void*)&smem_total, (void*)&sync, (void*)&dp, (void*)&dout, (void*)&dst};
        PF_CUDA(c, cudaLaunchCooperativeKernel((void*)kern, dim3(ns * (1 + hps)), dim3(NT), args, smem, st));
      } else {
        kern<<<ns, NT, smem, st>>>(cl, spp, d_u, nl, nsl, 0, ring_off, smem_total, sync, dp, dout, dst);
      }
      c->last_helpers = helpers;
    });
    c->stats.kernel_launches += 1;
    return 0;
  };
  // bracket rows of slices [n_lo + s0, n_lo + bs): one batched GEMM (k_bracket_all)
  if (c->brk.ensure((size_t)cap * m * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "bracket");
  double* brk0 = c->brk.p + (size_t)slot0 * m * c->size;
  auto bracket = [&](int s0, cudaStream_t st) -> int {
    const int ns = bs - s0;
    if (n_lo + s0 + ns <= 1) return 0;  // only slice 0: no coarse history
    constexpr int RT = PF_BRK_RT, EM = PF_BRK_EM;
    const dim3 gb((unsigned)((c->size + 256 * EM - 1) / (256 * EM)), (unsigned)((m + RT - 1) / RT), (unsigned)ns);
    pf::k_bracket_all<RT, EM><<<gb, 256, 0, st>>>(cm, d_u, n_lo + s0, brk0);
    c->stats.kernel_launches += 1;
    return 0;
  };
  // Head start of slice 0: it has no coarse history (no bracket) and is the
  // slowest slice (its t^alpha layer), so it starts on a side stream while the
  // bracket kernel of the other slices runs; they follow on the main stream.
  const char* nohs = std::getenv("PF_NO_HEADSTART");
  // Only where the bracket kernel is long enough to pay for the second launch
  // (config 3: 2^25 bracket entries; config 2's 2^18 measured slower).
  const bool big = (double)m * c->size * bs >= 16777216.0;
  const bool head = !fo && big && n_lo == 0 && bs >= 2 && m_override == 0 && c->allow_helpers &&
                    !(nohs && nohs[0] == '1');
  if (head) {
    if (!c->side_stream) {
      PF_CUDA(c, cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
      PF_CUDA(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      PF_CUDA(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    PF_CUDA(c, cudaEventRecord(c->ev_fork, c->stream));
    PF_CUDA(c, cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
    if (sweep(0, 1, c->side_stream, nullptr)) return c->err.code;
    PF_CUDA(c, cudaEventRecord(c->ev_join, c->side_stream));
    if (bracket(1, c->stream)) return c->err.code;
    if (sweep(1, bs - 1, c->stream, brk0)) return c->err.code;
    PF_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  } else {
    if (bracket(0, c->stream)) return c->err.code;
    if (sweep(0, bs, c->stream, (n_lo + bs > 1) ? brk0 : nullptr)) return c->err.code;
  }
  PF_CUDA(c, cudaGetLastError());
  if (!fo) {  // (the pipelined driver counts its chunked sweeps itself)
    PF_CUDA(c, cudaEventRecord(c->ev1, c->stream));
    c->stats.fine_launches += 1;
    c->stats.helper_launches += c->last_helpers ? 1 : 0;  // one sweep, however many launches
  }
  return 0;
}

int launch_coarse(pf_ctx* c, const pf::CoarseArgs& a, Status* d_st) {
  pf::Common cm = make_common(c);
  if (c->variant == V_CHEB_512_1 &&
      c->cheb_aug_coarse.ensure((size_t)c->ni * pf::Cheb1D<512, 1>::ld_of(c->ni)))
    return cuda_fail(c, cudaErrorMemoryAllocation, "chebyshev system");
  PF_DISPATCH(c, {
    auto kern = pf::k_coarse<SP, SPP, NT, EPT>;
    coarse_slab(spp, c);
    PF_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem));
    kern<<<1, NT, c->smem, c->stream>>>(cm, spp, a, d_st);
  });
  PF_CUDA(c, cudaGetLastError());
  c->stats.coarse_launches += 1;
  c->stats.kernel_launches += 1;
  return 0;
}

// Decode a fine-sweep status array: the earliest substep r fails first;
// at equal r a coefficient error precedes the solve (stepping.py:225-241).
int decode_fine(pf_ctx* c, int n_lo, int count) {
  if (c->kind == PF_SPACE_SINE2D) return 0;  // the 2-D engine reports synchronously
  PF_CUDA(c, cudaMemcpyAsync(c->h_status.data(), c->d_status, sizeof(Status) * count, cudaMemcpyDeviceToHost,
                             c->stream));
  PF_CUDA(c, cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c->ev0, c->ev1) == cudaSuccess) c->stats.last_fine_ms = ms;
  int best = -1;
  for (int i = 0; i < count; ++i) {
    const Status& s = c->h_status[i];
    c->stats.pcg_iterations += s.iters;
    c->stats.solves += s.solves;
    if (s.code == pf::ST_OK) continue;
    if (best < 0) {
      best = i;
      continue;
    }
    const Status& b = c->h_status[best];
    if (s.r < b.r || (s.r == b.r && s.code == pf::ST_COEFF && b.code != pf::ST_COEFF)) best = i;
  }
  if (best < 0) return 0;
  const Status& s = c->h_status[best];
  c->err = pf_error{};
  c->err.step_n = n_lo;
  c->err.step_r = s.r;
  if (s.code == pf::ST_COEFF) {
    c->err.code = PF_ERR_COEFFICIENT;
    c->err.node = s.node;
    std::snprintf(c->err.message, sizeof(c->err.message), "diffusion coefficient is not finite");
  } else {
    c->err.code = PF_ERR_SOLVER;
    std::snprintf(c->err.message, sizeof(c->err.message), "fine-sweep solve failed (interval %d)", s.n);
  }
  return c->err.code;
}

int decode_coarse(pf_ctx* c, int step_offset, int k_iter) {
  PF_CUDA(c, cudaMemcpyAsync(c->h_status.data(), c->d_status, sizeof(Status), cudaMemcpyDeviceToHost, c->stream));
  PF_CUDA(c, cudaStreamSynchronize(c->stream));
  const Status& s = c->h_status[0];
  c->stats.pcg_iterations += s.iters;
  c->stats.solves += s.solves;
  if (s.code == pf::ST_OK) return 0;
  c->err = pf_error{};
  c->err.step_r = -1;
  if (s.code == pf::ST_COEFF) {
    c->err.code = PF_ERR_COEFFICIENT;
    c->err.node = s.node;
    c->err.step_n = s.n + step_offset;
    std::snprintf(c->err.message, sizeof(c->err.message), "diffusion coefficient is not finite");
  } else if (s.code == pf::ST_DIVERGE) {
    c->err.code = PF_ERR_DIVERGENCE;
    c->err.iteration = k_iter;
    c->err.interval = s.n;
    std::snprintf(c->err.message, sizeof(c->err.message), "%s",
                  s.r == 0 ? "non-finite state after correction sweep" : "state norm exceeds divergence guard");
  } else {
    c->err.code = PF_ERR_SOLVER;
    c->err.step_n = s.n + step_offset;
    std::snprintf(c->err.message, sizeof(c->err.message), "singular or ill-conditioned time-step system");
  }
  return c->err.code;
}

double host_norm(const pf_ctx* c, const double* v) {
  double s = 0.0;
  if (c->kind == PF_SPACE_CHEB1D) {
    for (int i = 0; i < c->ni; ++i) s += c->h_qw[i + 1] * v[i] * v[i];
  } else {
    for (int i = 0; i < c->size; ++i) s += v[i] * v[i];
  }
  return std::sqrt(s);
}

int upload(pf_ctx* c, double* dst, const double* src, size_t n) {
  PF_CUDA(c, cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  return 0;
}
int download(pf_ctx* c, double* dst, const double* src, size_t n) {
  PF_CUDA(c, cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  return 0;
}

double l1_formula(double x, double alpha) {
  if (alpha == 1.0) return x == 0.0 ? 1.0 : 0.0;
  const double e = 1.0 - alpha;
  return std::pow(x + 1.0, e) - std::pow(x, e);
}

}  // namespace

#include "pf_engine2d.inc"

extern "C" {

const char* pf_version(void) { return "parafrac_b200 0.1.0 (sm_100a)"; }

// Phase cycle counters of slice 0 (only in -DPF_PHASE_TIMING builds; else 16 zeros).
int pf_debug_phases(long long* out16, int reset) {
#ifdef PF_PHASE_TIMING
  if (cudaMemcpyFromSymbol(out16, pf::g_phase, sizeof(long long) * 16) != cudaSuccess) return PF_ERR_CUDA;
  if (reset) {
    long long z[16] = {0};
    cudaMemcpyToSymbol(pf::g_phase, z, sizeof(z));
  }
#else
  for (int i = 0; i < 16; ++i) out16[i] = 0;
  (void)reset;
#endif
  return PF_OK;
}

// Per-warp timeline of the traced substeps (only in -DPF_TRACE builds): out[8 warps][8 substeps][64 points].
int pf_debug_trace(long long* out4096) {
#ifdef PF_TRACE
  if (cudaMemcpyFromSymbol(out4096, pf::g_trace, sizeof(long long) * 8 * pf::TR_STEPS * pf::TR_POINTS) != cudaSuccess)
    return PF_ERR_CUDA;
#else
  for (int i = 0; i < 4096; ++i) out4096[i] = 0;
#endif
  return PF_OK;
}

// clock64 at the loop top of substeps 0..n-1 of the traced slice (only in -DPF_TRACE builds).
int pf_debug_looptop(long long* out, int n) {
#ifdef PF_TRACE
  if (n < 0 || n > 4096) return PF_ERR_ARGUMENT;
  if (cudaMemcpyFromSymbol(out, pf::g_looptop, sizeof(long long) * n) != cudaSuccess) return PF_ERR_CUDA;
#else
  for (int i = 0; i < n; ++i) out[i] = 0;
#endif
  return PF_OK;
}

// Entry and exit times (globaltimer ns) of each slice CTA of the last decoded
// 1-D fine sweep: out[2 i] = entry, out[2 i + 1] = exit.
int pf_debug_slice_times_ns(const pf_ctx* c, long long* out, int n) {
  if (!c || !out || n < 0 || n > (int)c->h_status.size()) return PF_ERR_ARGUMENT;
  for (int i = 0; i < n; ++i) {
    out[2 * i] = c->h_status[i].t_start;
    out[2 * i + 1] = c->h_status[i].t_end;
  }
  return PF_OK;
}

int pf_create(const pf_problem* problem, const pf_grid* grid, const pf_space* space, const pf_weights* weights,
              int device, pf_ctx** out) {
  if (!out) return PF_ERR_ARGUMENT;
  *out = nullptr;
  pf_ctx* c = new pf_ctx();
  *out = c;
  if (!problem || !grid || !space) return set_error(c, PF_ERR_ARGUMENT, "null argument");
  c->prob = *problem;
  c->grid = *grid;
  if (!(problem->alpha > 0.0 && problem->alpha <= 1.0))
    return set_error(c, PF_ERR_ARGUMENT, "fractional order must lie in (0, 1]");
  if (!(problem->t_final > 0.0)) return set_error(c, PF_ERR_ARGUMENT, "final time must be positive");
  if (grid->nt < 1 || grid->m < 1) return set_error(c, PF_ERR_ARGUMENT, "grid counts nt and m must be positive integers");
  if (problem->functor < 1 || problem->functor > 5) return set_error(c, PF_ERR_UNSUPPORTED, "unknown coefficient functor");
  c->kind = space->kind;
  c->pcg_tol = space->pcg_tol > 0 ? space->pcg_tol : 1e-14;
  c->pcg_maxit = space->pcg_maxit > 0 ? space->pcg_maxit : 500;
  if (space->kind == PF_SPACE_SINE1D) {
    const int M = space->modes;
    if (!is_pow2(M) || M < 2 || M > 1024)
      return set_error(c, PF_ERR_UNSUPPORTED, "sine modes must be a power of two in [2, 1024]");
    c->M = M;
    c->Q = 2 * M;
    c->lgQ = 0;
    while ((1 << c->lgQ) < c->Q) ++c->lgQ;
    c->size = M;
    static const Variant by_lg[12] = {V_NONE, V_NONE, V_S2, V_S3, V_S4, V_S5, V_S6, V_S7, V_S8, V_S9, V_S10, V_S11};
    c->variant = by_lg[c->lgQ];
    c->smem = sizeof(cd) * (pf::tw_table_size(c->lgQ) + 3 * c->Q) + sizeof(double) * (4 * c->Q + pf::RED_DOUBLES);
  } else if (space->kind == PF_SPACE_SINE2D) {
    const int M = space->modes;
    if (!is_pow2(M) || M < 4 || M > 256)
      return set_error(c, PF_ERR_UNSUPPORTED, "2-D sine modes must be a power of two in [4, 256]");
    c->M = M;
    c->Q = 2 * M;
    c->lgQ = 0;
    while ((1 << c->lgQ) < c->Q) ++c->lgQ;
    c->size = M * M;
    c->variant = V_NONE;
    c->smem = 0;
  } else if (space->kind == PF_SPACE_CHEB1D) {
    const int deg = space->modes;
    if (deg < 2) return set_error(c, PF_ERR_ARGUMENT, "degree must be at least 2 so interior nodes exist");
    if (!space->nodes || !space->d1 || !space->quad_weights)
      return set_error(c, PF_ERR_ARGUMENT, "Chebyshev space needs nodes, d1 and quad_weights");
    c->npts = deg + 1;
    c->ni = deg - 1;
    c->size = c->ni;
    c->smem = pf::Cheb1D<128, 1>::smem_bytes(deg);
    c->variant = V_CHEB_128_1;
    if (c->ni > 128 || c->smem > 227 * 1024) {
      // the reference's own sizes (config 3: degree 513): D1 and the systems in global memory
      if (c->ni > 512)
        return set_error(c, PF_ERR_UNSUPPORTED, "Chebyshev bridge supports degree <= 513");
      c->smem = pf::Cheb1D<512, 1>::smem_bytes(deg, true);
      c->variant = V_CHEB_512_1;
    }
    c->h_nodes.assign(space->nodes, space->nodes + c->npts);
    c->h_d1.assign(space->d1, space->d1 + (size_t)c->npts * c->npts);
    c->h_qw.assign(space->quad_weights, space->quad_weights + c->npts);
  } else {
    return set_error(c, PF_ERR_UNSUPPORTED, "space kind not built in this library");
  }
  const double alpha = problem->alpha;
  const int nt = grid->nt, m = grid->m;
  c->dT = problem->t_final / nt;
  c->dt = c->dT / m;
  c->g2m = (weights && weights->gamma_2_minus > 0) ? weights->gamma_2_minus : std::exp(std::lgamma(2.0 - alpha));
  c->gam_f = std::pow(c->dt, alpha) * c->g2m;
  c->gam_c = std::pow(c->dT, alpha) * c->g2m;
  c->minv = std::pow((double)m, -alpha);
  // weight tables (caller's rounding when given, libm pow otherwise)
  const long need_fine = std::max<long>((long)nt * m + 1, std::max(m, nt) + 2) + pf::HB;  // + block padding
  const long need_frac = (long)(nt > 1 ? nt - 1 : 0) * m + m + 1 + pf::HB;
  c->h_bfine.resize(need_fine);
  c->h_bfrac.resize(need_frac);
  for (long q = 0; q < need_fine; ++q) {
    if (weights && weights->b_fine && q < weights->len_fine)
      c->h_bfine[q] = weights->b_fine[q];
    else
      c->h_bfine[q] = l1_formula((double)q, alpha);
  }
  for (long q = 0; q < need_frac; ++q) {
    if (weights && weights->b_frac && q < weights->len_frac)
      c->h_bfrac[q] = weights->b_frac[q];
    else
      c->h_bfrac[q] = l1_formula((double)q / (double)m, alpha);
  }
  c->len_fine = need_fine;
  std::vector<double> h_afine(need_fine + pf::HB + 1, 0.0);
  for (long s = 1; s < need_fine; ++s) h_afine[s] = c->h_bfine[s - 1] - c->h_bfine[s];
  c->len_frac = need_frac;

  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  c->device = device;
  PF_CUDA(c, cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  {
    const char* env = std::getenv("PF_NO_HELPERS");
    c->allow_helpers = (env && env[0] == '1') ? 0 : 1;
  }
  PF_CUDA(c, cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
  c->stream = c->own_stream;
  PF_CUDA(c, cudaEventCreate(&c->ev0));
  PF_CUDA(c, cudaEventCreate(&c->ev1));
  PF_CUDA(c, cudaMalloc(&c->d_bfine, sizeof(double) * need_fine));
  PF_CUDA(c, cudaMalloc(&c->d_bfrac, sizeof(double) * need_frac));
  PF_CUDA(c, cudaMemcpy(c->d_bfine, c->h_bfine.data(), sizeof(double) * need_fine, cudaMemcpyHostToDevice));
  PF_CUDA(c, cudaMalloc(&c->d_afine, sizeof(double) * h_afine.size()));
  PF_CUDA(c, cudaMemcpy(c->d_afine, h_afine.data(), sizeof(double) * h_afine.size(), cudaMemcpyHostToDevice));
  PF_CUDA(c, cudaMemcpy(c->d_bfrac, c->h_bfrac.data(), sizeof(double) * need_frac, cudaMemcpyHostToDevice));
  if ((c->kind == PF_SPACE_SINE1D || c->kind == PF_SPACE_SINE2D) && alpha < 1.0) {
    // PCG guess weights by substep k: Lagrange extrapolation in tau = (k dt)^alpha
    // from rows k-1 .. k-1-p.  Rows k <= m are read by every slice at its local
    // substep r = k (k_fine_sweep, k2_prep: the slice's own tau); rows k > m
    // serve the single-slice sequential solver, whose slice spans the horizon.
    // The order p follows the t^alpha layer (tools/studies/slice0_guess.py,
    // slice_start_guess.py: device PCG recurrence on the oracle's exact path):
    // order 6 through the layer, then 5, then 4 where rounding amplified by
    // higher orders dominates the residual.
    const long rows = (long)nt * m + 1;
    std::vector<double> ext((size_t)rows * 8, 0.0);
    // order schedule by substep: pairs (order, until k);
    // PF_EXT_SCHED="o1,k1,o2,k2,...,o_last" overrides it
    // (development aid for re-tuning)
    // (round 2 rescan on the device, tools/r02/sched_scan.py: order 7 lost to 6 once the states
    // carry the PCG tolerance's noise; config-3 sweep 7.18 -> 7.06 ms)
    // (beyond a slice's 1024 substeps only the sequential solver reads the table: lower orders as
    // the noise of its 65 536-row history grows, 0.628 -> 0.595 s at config 3)
    std::vector<long> sched = {5, 16, 6, 64, 5, 192, 4, 1024, 3, 4096, 2};
    if (const char* es = std::getenv("PF_EXT_SCHED")) {
      sched.clear();
      for (const char* q = es; *q;) {
        char* end = nullptr;
        const long v = std::strtol(q, &end, 10);
        if (end == q) break;  // not a number: stop parsing
        sched.push_back(std::max(1L, v));
        q = end;
        if (*q == ',') ++q;
      }
      if (sched.empty()) sched = {5};
    }
    auto order = [&sched](long r) -> int {
      size_t i = 0;
      while (i + 1 < sched.size() && r >= sched[i + 1]) i += 2;
      return (int)sched[i];
    };
    for (long k = 2; k < rows; ++k) {
      const int p = (int)std::min<long>(std::min<long>(k - 1, pf::EXT), order(k));
      long double tau[pf::EXT + 1];
      for (int j = 0; j <= p; ++j) tau[j] = powl((long double)(k - 1 - j) * (long double)c->dt, (long double)alpha);
      const long double tr = powl((long double)k * (long double)c->dt, (long double)alpha);
      for (int j = 0; j <= p; ++j) {
        long double w = 1.0L;
        for (int q = 0; q <= p; ++q)
          if (q != j) w *= (tr - tau[q]) / (tau[j] - tau[q]);
        ext[(size_t)k * 8 + j] = (double)w;
      }
    }
    PF_CUDA(c, cudaMalloc(&c->d_ext0, sizeof(double) * ext.size()));
    PF_CUDA(c, cudaMemcpy(c->d_ext0, ext.data(), sizeof(double) * ext.size(), cudaMemcpyHostToDevice));
  }
  if (c->kind == PF_SPACE_SINE1D || c->kind == PF_SPACE_SINE2D) {
    const int ntw = std::max(pf::tw_table_size(c->lgQ), 1);
    std::vector<cd> tw(ntw), ph(c->Q);
    const long double PI = 3.141592653589793238462643383279502884L;
    // per-pass radix-4 twiddles w_r(k) = exp(-2 pi i r k / (4 Ns)), then radix-2 exp(-2 pi i k / (2 Ns));
    // Q = 1024 (1-D): the radix 8-8-4-4 passes' w1 (+ w4) per pass (pf_sine1d.cuh T10_*)
    auto put10 = [&](int off, int R, int ns, bool w4) {
      for (int k = 0; k < ns; ++k) {
        const long double a = -2.0L * PI * (long double)k / (long double)(R * ns);
        tw[off + k] = {(double)cosl(a), (double)sinl(a)};
        if (w4) tw[off + ns + k] = {(double)cosl(4.0L * a), (double)sinl(4.0L * a)};
      }
    };
    if (c->lgQ == 10 && c->kind == PF_SPACE_SINE1D) {
      put10(pf::T10_R8_8, 8, 8, true);
      put10(pf::T10_R4_64, 4, 64, false);
      put10(pf::T10_R4_256, 4, 256, false);
      put10(pf::T10_R4_4, 4, 4, false);
      put10(pf::T10_R8_16, 8, 16, true);
      put10(pf::T10_R8_128, 8, 128, true);
    }
    int off = 0;
    for (int p = 1, ns = 4; c->lgQ != 10 && p < c->lgQ / 2; ++p, ns *= 4) {
      for (int r = 1; r <= 3; ++r)
        for (int k = 0; k < ns; ++k) {
          const long double a = -2.0L * PI * (long double)(r * k) / (4.0L * ns);
          tw[off + (r - 1) * ns + k] = {(double)cosl(a), (double)sinl(a)};
        }
      off += 3 * ns;
    }
    if (c->lgQ & 1) {
      const int ns = 1 << (c->lgQ - 1);
      for (int k = 0; k < ns; ++k) {
        const long double a = -2.0L * PI * (long double)k / (2.0L * ns);
        tw[off + k] = {(double)cosl(a), (double)sinl(a)};
      }
    }
    for (int j = 0; j < c->Q; ++j) {
      const long double b = PI * (long double)j / (2.0L * (long double)c->Q);
      ph[j] = {(double)cosl(b), (double)sinl(b)};
    }
    PF_CUDA(c, cudaMalloc(&c->d_tw, sizeof(cd) * ntw));
    PF_CUDA(c, cudaMalloc(&c->d_ph, sizeof(cd) * c->Q));
    PF_CUDA(c, cudaMemcpy(c->d_tw, tw.data(), sizeof(cd) * ntw, cudaMemcpyHostToDevice));
    PF_CUDA(c, cudaMemcpy(c->d_ph, ph.data(), sizeof(cd) * c->Q, cudaMemcpyHostToDevice));
  } else {
    PF_CUDA(c, cudaMalloc(&c->d_nodes, sizeof(double) * c->npts));
    PF_CUDA(c, cudaMalloc(&c->d_d1, sizeof(double) * c->npts * c->npts));
    PF_CUDA(c, cudaMalloc(&c->d_qw, sizeof(double) * c->npts));
    PF_CUDA(c, cudaMemcpy(c->d_nodes, c->h_nodes.data(), sizeof(double) * c->npts, cudaMemcpyHostToDevice));
    PF_CUDA(c, cudaMemcpy(c->d_d1, c->h_d1.data(), sizeof(double) * c->npts * c->npts, cudaMemcpyHostToDevice));
    PF_CUDA(c, cudaMemcpy(c->d_qw, c->h_qw.data(), sizeof(double) * c->npts, cudaMemcpyHostToDevice));
  }
  if (ensure_status(c, std::max(nt, 1))) return c->err.code;
  if (c->kind == PF_SPACE_SINE2D && e2_init(c)) return c->err.code;
  c->err = pf_error{};
  return PF_OK;
}

void pf_destroy(pf_ctx* c) {
  if (!c) return;
  if (c->device >= 0) cudaSetDevice(c->device);
  for (DevBuf* b : {&c->U, &c->Unext, &c->paths, &c->fold, &c->gold, &c->gnew, &c->io, &c->scalar, &c->scratch, &c->brk,
                    &c->wpaths[0], &c->wpaths[1]})
    b->release();
  for (void* p : {(void*)c->d_bfine, (void*)c->d_afine, (void*)c->d_bfrac, (void*)c->d_ext0, (void*)c->d_nodes, (void*)c->d_d1, (void*)c->d_qw,
                  (void*)c->d_tw, (void*)c->d_ph, (void*)c->d_status, (void*)c->d_sync})
    if (p) cudaFree(p);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  c->fold2.release();
  c->cheb_aug.release();
  c->cheb_aug_coarse.release();
  for (void* p : {(void*)c->d_status2, (void*)c->d_corr_status, (void*)c->d_corr_state, (void*)c->d_cancel})
    if (p) cudaFree(p);
  for (cudaStream_t s : c->pstream)
    if (s) cudaStreamDestroy(s);
  for (int q = 0; q < 2; ++q)
    for (int i = 0; i < 8; ++i) {
      if (c->ev_sw[q][i]) cudaEventDestroy(c->ev_sw[q][i]);
      if (c->ev_co[q][i]) cudaEventDestroy(c->ev_co[q][i]);
    }
  if (c->ev_init) cudaEventDestroy(c->ev_init);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c->e2;
  delete c->e2c;
  delete c;
}

int pf_last_error(const pf_ctx* c, pf_error* out) {
  if (!c || !out) return PF_ERR_ARGUMENT;
  *out = c->err;
  return PF_OK;
}

int pf_state_size(const pf_ctx* c) { return c ? c->size : -1; }

int pf_get_stats(const pf_ctx* c, pf_stats* out) {
  if (!c || !out) return PF_ERR_ARGUMENT;
  *out = c->stats;
  return PF_OK;
}

int pf_reset_stats(pf_ctx* c) {
  if (!c) return PF_ERR_ARGUMENT;
  c->stats = pf_stats{};
  return PF_OK;
}

int pf_set_stream(pf_ctx* c, void* stream) {
  if (!c) return PF_ERR_ARGUMENT;
  c->stream = stream ? (cudaStream_t)stream : c->own_stream;
  return PF_OK;
}

int pf_dev_fine_sweep_async(pf_ctx* c, const double* d_u, int n_lo, int n_hi, double* d_out) {
  if (!c) return PF_ERR_ARGUMENT;
  const int bs = n_hi - n_lo;
  if (bs < 1 || n_lo < 0 || n_hi > c->grid.nt) return set_error(c, PF_ERR_ARGUMENT, "interval range outside the supplied coarse states");
  cudaSetDevice(c->device);
  if (ensure_status(c, bs)) return c->err.code;
  c->pending_lo = n_lo;
  c->pending_bs = bs;
  return launch_fine(c, d_u, n_lo, bs, d_out, c->d_status);
}

int pf_dev_fine_sweep(pf_ctx* c, const double* d_u, int n_lo, int n_hi, double* d_out) {
  int rc = pf_dev_fine_sweep_async(c, d_u, n_lo, n_hi, d_out);
  if (rc) return rc;
  c->pending_lo = -1;
  return decode_fine(c, n_lo, n_hi - n_lo);
}

// Synchronise; decode the status of the last asynchronous fine launch.
int pf_dev_check(pf_ctx* c) {
  if (!c) return PF_ERR_ARGUMENT;
  PF_CUDA(c, cudaStreamSynchronize(c->stream));
  if (c->pending_lo >= 0) {
    const int lo = c->pending_lo, bs = c->pending_bs;
    c->pending_lo = -1;
    return decode_fine(c, lo, bs);
  }
  return 0;
}

int pf_fine_sweep(pf_ctx* c, const double* u_nodes, int n_states, int n_lo, int n_hi, double* out) {
  if (!c || !u_nodes || !out) return PF_ERR_ARGUMENT;
  const int bs = n_hi - n_lo;
  if (bs < 1 || n_lo < 0 || n_hi > n_states - 1 || n_hi > c->grid.nt)
    return set_error(c, PF_ERR_ARGUMENT, "interval range outside the supplied coarse states");
  cudaSetDevice(c->device);
  if (c->io.ensure((size_t)(n_hi + bs) * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "io");
  double* d_u = c->io.p;
  double* d_out = c->io.p + (size_t)n_hi * c->size;
  if (upload(c, d_u, u_nodes, (size_t)n_hi * c->size)) return c->err.code;
  if (ensure_status(c, bs)) return c->err.code;
  int rc = launch_fine(c, d_u, n_lo, bs, d_out, c->d_status);
  if (rc) return rc;
  if (download(c, out, d_out, (size_t)bs * c->size)) return c->err.code;
  return decode_fine(c, n_lo, bs);
}

int pf_fine_propagate(pf_ctx* c, const double* start, const double* hist, int n_states, double* endpoint,
                      double* path) {
  if (!c || !hist || n_states < 1) return PF_ERR_ARGUMENT;
  const int n = n_states - 1;
  if (n >= c->grid.nt) return set_error(c, PF_ERR_ARGUMENT, "interval index outside the grid");
  cudaSetDevice(c->device);
  if (c->io.ensure((size_t)(n_states + 2) * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "io");
  double* d_u = c->io.p;
  double* d_out = c->io.p + (size_t)n_states * c->size;
  double* d_start = nullptr;
  if (upload(c, d_u, hist, (size_t)n_states * c->size)) return c->err.code;
  if (start) {  // path[0] = start (stepping.py:170-171); the bracket uses hist
    d_start = c->io.p + (size_t)(n_states + 1) * c->size;
    if (upload(c, d_start, start, c->size)) return c->err.code;
  }
  int rc = launch_fine(c, d_u, n, 1, d_out, c->d_status, 0, 1, d_start);
  if (rc) return rc;
  if (endpoint && download(c, endpoint, d_out, c->size)) return c->err.code;
  if (path && download(c, path, c->paths.p + c->size, (size_t)c->grid.m * c->size)) return c->err.code;
  return decode_fine(c, n, 1);
}

int pf_coarse_step(pf_ctx* c, const double* history, int n_states, int step_index, double* out) {
  if (!c || !history || !out || n_states < 1) return c ? set_error(c, PF_ERR_ARGUMENT, "history must be a nonempty stack of states") : PF_ERR_ARGUMENT;
  const int n = n_states - 1;
  if (n + 1 >= c->len_fine) return set_error(c, PF_ERR_ARGUMENT, "history longer than the weight tables");
  cudaSetDevice(c->device);
  if (c->io.ensure((size_t)(n_states + 1) * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "io");
  if (upload(c, c->io.p, history, (size_t)n_states * c->size)) return c->err.code;
  if (c->kind == PF_SPACE_SINE2D) {
    double* d_out = c->io.p + (size_t)n_states * c->size;
    int rc = e2_coarse_step(c, c->io.p, n, d_out);
    if (rc) {
      if (rc == PF_ERR_SOLVER || rc == PF_ERR_COEFFICIENT) c->err.step_n = step_index;
      return rc;
    }
    if (download(c, out, d_out, c->size)) return c->err.code;
    PF_CUDA(c, cudaStreamSynchronize(c->stream));
    return 0;
  }
  pf::CoarseArgs a{};
  a.mode = pf::CM_SINGLE;
  a.n_single = n;
  a.traj = c->io.p;
  a.out = c->io.p + (size_t)n_states * c->size;
  int rc = launch_coarse(c, a, c->d_status);
  if (rc) return rc;
  if (download(c, out, a.out, c->size)) return c->err.code;
  rc = decode_coarse(c, 0, 0);
  if (rc == PF_ERR_SOLVER || rc == PF_ERR_COEFFICIENT) c->err.step_n = step_index;
  return rc;
}

static int run_coarse_dev(pf_ctx* c, double* d_traj) {
  if (c->kind == PF_SPACE_SINE2D) return e2_run_coarse(c, d_traj);
  pf::CoarseArgs a{};
  a.mode = pf::CM_RUN;
  a.traj = d_traj;
  int rc = launch_coarse(c, a, c->d_status);
  if (rc) return rc;
  return decode_coarse(c, 0, 0);
}

int pf_run_coarse(pf_ctx* c, const double* u0, double* traj) {
  if (!c || !u0 || !traj) return PF_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  const size_t rows = (size_t)c->grid.nt + 1;
  if (c->io.ensure(rows * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "io");
  if (upload(c, c->io.p, u0, c->size)) return c->err.code;
  int rc = run_coarse_dev(c, c->io.p);
  if (rc) return rc;
  if (download(c, traj, c->io.p, rows * c->size)) return c->err.code;
  PF_CUDA(c, cudaStreamSynchronize(c->stream));
  return 0;
}

int pf_chain_fine(pf_ctx* c, const double* u0, double* traj) {
  if (!c || !u0 || !traj) return PF_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  const int nt = c->grid.nt;
  const size_t rows = (size_t)nt + 1;
  if (c->io.ensure(rows * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "io");
  if (upload(c, c->io.p, u0, c->size)) return c->err.code;
  if (ensure_status(c, nt)) return c->err.code;
  PF_CUDA(c, cudaMemsetAsync(c->d_status, 0, sizeof(Status) * nt, c->stream));
  for (int n = 0; n < nt; ++n) {
    int rc = launch_fine(c, c->io.p, n, 1, c->io.p + (size_t)(n + 1) * c->size, c->d_status + n);
    if (rc) return rc;
  }
  PF_CUDA(c, cudaMemcpyAsync(c->h_status.data(), c->d_status, sizeof(Status) * nt, cudaMemcpyDeviceToHost, c->stream));
  if (download(c, traj, c->io.p, rows * c->size)) return c->err.code;
  PF_CUDA(c, cudaStreamSynchronize(c->stream));
  for (int n = 0; n < nt; ++n) {
    const Status& s = c->h_status[n];
    c->stats.pcg_iterations += s.iters;
    c->stats.solves += s.solves;
    if (s.code != pf::ST_OK) {
      c->err = pf_error{};
      c->err.code = s.code == pf::ST_COEFF ? PF_ERR_COEFFICIENT : PF_ERR_SOLVER;
      c->err.step_n = n;
      c->err.step_r = s.r;
      c->err.node = s.node;
      std::snprintf(c->err.message, sizeof(c->err.message), "chain_fine failed in interval %d", n);
      return c->err.code;
    }
  }
  return 0;
}

int pf_fine_sequential(pf_ctx* c, const double* u0, double* states) {
  if (!c || !u0 || !states) return PF_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  const long total = (long)c->grid.nt * c->grid.m;
  if (c->len_fine < total + 1) return set_error(c, PF_ERR_ARGUMENT, "weight table shorter than nt*m+1");
  if (c->kind == PF_SPACE_SINE2D) {
    // the full-history solver is one slice marched over nt*m substeps with no bracket
    if (c->io.ensure((size_t)(total + 2) * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "hist");
    double* d_u0 = c->io.p;
    double* d_all = c->io.p + c->size;
    if (upload(c, d_u0, u0, c->size)) return c->err.code;
    int rc = e2_fine_sweep(c, d_u0, 0, 1, nullptr, (int)total, false, d_all);
    if (rc) {
      c->err.step_n = c->err.step_r - 1;
      c->err.step_r = -1;
      return rc;
    }
    for (int n = 0; n <= c->grid.nt; ++n)
      if (download(c, states + (size_t)n * c->size, d_all + (size_t)n * c->grid.m * c->size, c->size))
        return c->err.code;
    PF_CUDA(c, cudaStreamSynchronize(c->stream));
    return 0;
  }
  // stepping.run_fine_sequential is slice 0 marched over nt*m fine substeps with the
  // full history (no bracket since n = 0, t = (jj-1) dt): the sweep kernel with
  // m = nt*m and the far history split over up to SMs-1 helper CTAs.
  if (c->io.ensure((size_t)2 * c->size)) return cuda_fail(c, cudaErrorMemoryAllocation, "io");
  if (upload(c, c->io.p, u0, c->size)) return c->err.code;
  if (ensure_status(c, 1)) return c->err.code;
  // far-history helpers: one per 1024 substeps up to the SMs left over (config 3:
  // 128 = 8 batches x 16 parts of the tensor-core split)
  const int hps = (int)std::max<long>(1, std::min<long>(std::min<long>(c->num_sms - 1, 128), total / 512));
  int rc = launch_fine(c, c->io.p, 0, 1, c->io.p + c->size, c->d_status, (int)total, hps);
  if (rc == PF_ERR_UNSUPPORTED) rc = launch_fine(c, c->io.p, 0, 1, c->io.p + c->size, c->d_status, (int)total, 1);
  if (rc) return rc;
  for (int n = 0; n <= c->grid.nt; ++n)
    if (download(c, states + (size_t)n * c->size, c->paths.p + (size_t)n * c->grid.m * c->size, c->size))
      return c->err.code;
  rc = decode_fine(c, 0, 1);
  if (rc == PF_ERR_SOLVER || rc == PF_ERR_COEFFICIENT) {  // SolverFailure(jj - 1), stepping.py:286
    c->err.step_n = c->err.step_r - 1;
    c->err.step_r = -1;
  }
  return rc;
}

int pf_dev_parareal_init(pf_ctx* c, const double* u0) {
  if (!c || !u0) return PF_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  const size_t rows = (size_t)c->grid.nt + 1, sz = c->size;
  for (DevBuf* b : {&c->U, &c->Unext}) if (b->ensure(rows * sz)) return cuda_fail(c, cudaErrorMemoryAllocation, "U");
  for (DevBuf* b : {&c->fold, &c->gold, &c->gnew}) if (b->ensure((rows - 1) * sz)) return cuda_fail(c, cudaErrorMemoryAllocation, "G");
  if (c->scalar.ensure(8)) return cuda_fail(c, cudaErrorMemoryAllocation, "scalar");
  if (!c->d_corr_state) PF_CUDA(c, cudaMalloc(&c->d_corr_state, 8 * sizeof(int)));
  if (upload(c, c->U.p, u0, sz)) return c->err.code;
  int rc = run_coarse_dev(c, c->U.p);
  if (rc) return rc;
  // G_old at k = 0 equals the coarse trajectory (parareal.py:78-79 == stepping.py:119-120)
  PF_CUDA(c, cudaMemcpyAsync(c->gold.p, c->U.p + sz, (rows - 1) * sz * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  c->guard = 1e12 * std::max(host_norm(c, u0), 1.0);  // parareal.py:98
  c->parareal_ready = true;
  c->frozen = 0;
  c->warm_iter = 0;
  c->warm_diff = 1.0;
  return 0;
}

const double* pf_dev_parareal_states(pf_ctx* c) { return c ? c->U.p : nullptr; }

int pf_dev_parareal_frozen(pf_ctx* c) { return c ? c->frozen : 0; }

int pf_dev_parareal_correct(pf_ctx* c, const double* d_fold, int k, double* diff) {
  if (!c || !c->parareal_ready) return c ? set_error(c, PF_ERR_ARGUMENT, "parareal state not initialised") : PF_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  pf::CoarseArgs a{};
  a.mode = pf::CM_CORRECT;
  a.k_iter = k;
  a.guard = c->guard;
  a.ucur = c->U.p;
  a.fold = d_fold ? d_fold : c->fold.p;
  a.gold = c->gold.p;
  a.gnew = c->gnew.p;
  a.unext = c->Unext.p;
  a.out = c->scalar.p;
  a.state = c->d_corr_state;
  // From the second iteration on, G_old is the previous sweep's G_new, which
  // is bitwise what parareal.py:78-79 recomputes.
  if (k > 0) std::swap(c->gold, c->gnew);
  a.gold = c->gold.p;
  a.gnew = c->gnew.p;
  if (d_fold && d_fold != c->fold.p)
    PF_CUDA(c, cudaMemcpyAsync(c->fold.p, d_fold, (size_t)c->grid.nt * c->size * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  float ms = 0.f;
  if (c->kind == PF_SPACE_SINE2D) {
    double h2 = 0.0;
    int rc2 = e2_correct(c, c->U.p, c->fold.p, c->gold.p, c->gnew.p, c->Unext.p, k, &h2);
    if (rc2) return rc2;
    if (diff) *diff = h2;
    c->warm_diff = h2;
    std::swap(c->U, c->Unext);
    return 0;
  }
  PF_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  int rc = launch_coarse(c, a, c->d_status);
  if (rc) return rc;
  PF_CUDA(c, cudaEventRecord(c->ev1, c->stream));
  double h[2] = {0.0, 0.0};
  PF_CUDA(c, cudaMemcpyAsync(h, c->scalar.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  rc = decode_coarse(c, 0, k);
  if (cudaEventElapsedTime(&ms, c->ev0, c->ev1) == cudaSuccess) c->stats.last_coarse_ms = ms;
  if (rc) return rc;
  if (diff) *diff = h[0];
  c->warm_diff = h[0];
  c->frozen = std::min((int)h[1], c->grid.nt);
  std::swap(c->U, c->Unext);  // u_curr = u_next (parareal.py:133)
  return 0;
}

int pf_dev_parareal_read(pf_ctx* c, double* states, double* coarse_new, double* coarse_old) {
  if (!c) return PF_ERR_ARGUMENT;
  const size_t rows = (size_t)c->grid.nt + 1, sz = c->size;
  if (states && download(c, states, c->U.p, rows * sz)) return c->err.code;
  if (coarse_new && download(c, coarse_new, c->gnew.p, (rows - 1) * sz)) return c->err.code;
  if (coarse_old && download(c, coarse_old, c->gold.p, (rows - 1) * sz)) return c->err.code;
  PF_CUDA(c, cudaStreamSynchronize(c->stream));
  return 0;
}

// ---------------------------------------------------------------------------
// Pipelined parareal (parareal.py:111-137): the slices are cut
// into C contiguous chunks; the correction sweep of iteration k runs chunk by
// chunk (k_coarse CM_CORRECT over a node range, its frozen-prefix state carried
// between chunk launches), and chunk c of the fine sweep of iteration k+1
// starts on its own stream as soon as the correction has finalised its nodes
// (U^{k+1}_0..n of every slice n in the chunk), i.e. while the correction of
// the later chunks still runs.  That sweep is launched before the host knows
// whether iteration k met the tolerance: if it did, the host sets the cancel
// word and the speculative sweep stops at its next block boundary; its F_old
// goes to the other of two buffers, so iteration k's results stand.  Slices of
// the frozen prefix copy their F_old row (k_fine_sweep) or, for whole chunks
// below the previous prefix, are copied by the host.  Same kernels on the same
// inputs as the sequential driver: bitwise the same iterates, diffs and
// iteration count (tests/test_gpu_parity.py).  PF_PIPELINE=C sets the chunk
// count (0 or 1: the sequential driver).
// ---------------------------------------------------------------------------
int pipeline_chunks(const pf_ctx* c) {
  if (c->kind != PF_SPACE_SINE1D) return 0;
  int C = 8;  // config 3 time-to-tol (tools/r02/parareal_tto.py): 70.6 ms sequential, 67.8 / 65.8 / 64.6 ms at C = 2 / 4 / 8
  if (const char* env = std::getenv("PF_PIPELINE")) C = std::atoi(env);
  C = std::min(std::min(C, 8), c->grid.nt / 2);
  return C >= 2 ? C : 0;
}

int parareal_pipelined(pf_ctx* c, int C, double tol, int k_max, const double* reference, double* diffs,
                       double* iteration_times, double* errors, int* iterations, int* stop_reason,
                       std::chrono::steady_clock::time_point t0, double*& fold_final) {
  const int nt = c->grid.nt;
  const size_t sz = c->size;
  if (c->fold2.ensure((size_t)nt * sz)) return cuda_fail(c, cudaErrorMemoryAllocation, "fold2");
  if (!c->d_status2) PF_CUDA(c, cudaMalloc(&c->d_status2, sizeof(Status) * c->status_cap));
  if (!c->d_corr_status) PF_CUDA(c, cudaMalloc(&c->d_corr_status, sizeof(Status)));
  if (!c->d_cancel) PF_CUDA(c, cudaMalloc(&c->d_cancel, sizeof(int)));
  if (!c->ev_init) {
    PF_CUDA(c, cudaEventCreateWithFlags(&c->ev_init, cudaEventDisableTiming));
    for (int i = 0; i < 8; ++i) {
      PF_CUDA(c, cudaStreamCreateWithFlags(&c->pstream[i], cudaStreamNonBlocking));
      for (int q = 0; q < 2; ++q) {
        PF_CUDA(c, cudaEventCreateWithFlags(&c->ev_sw[q][i], cudaEventDisableTiming));
        PF_CUDA(c, cudaEventCreateWithFlags(&c->ev_co[q][i], cudaEventDisableTiming));
      }
    }
  }
  std::vector<int> cb(C + 1);  // contiguous near-even chunks (parareal._block_bounds)
  for (int i = 0, lo = 0; i < C; ++i) {
    cb[i] = lo;
    lo += nt / C + (i < nt % C ? 1 : 0);
  }
  cb[C] = nt;
  double* F[2] = {c->fold.p, c->fold2.p};
  Status* SS[2] = {c->d_status, c->d_status2};
  PF_CUDA(c, cudaMemsetAsync(c->d_cancel, 0, sizeof(int), c->stream));
  PF_CUDA(c, cudaEventRecord(c->ev_init, c->stream));
  // sweep of iteration k (parity q) for chunk ch on stream ps[ch], reading states U
  auto sweep_chunk = [&](int k, int ch, const double* U, int frozen_prev) -> int {
    const int q = k & 1, lo = cb[ch], bs = cb[ch + 1] - cb[ch];
    cudaStream_t ps = c->pstream[ch];
    if (k > 0 && cb[ch + 1] <= frozen_prev) {  // the whole chunk is frozen: its F_old rows stand
      PF_CUDA(c, cudaMemcpyAsync(F[q] + (size_t)lo * sz, F[q ^ 1] + (size_t)lo * sz, (size_t)bs * sz * sizeof(double),
                                 cudaMemcpyDeviceToDevice, ps));
      PF_CUDA(c, cudaMemsetAsync(SS[q] + lo, 0, sizeof(Status) * bs, ps));
    } else {
      FineOpts fo;
      fo.slot0 = lo;
      fo.cap = nt;
      fo.stream = ps;
      fo.cancel = c->d_cancel;
      if (k > 0) {
        fo.frozen_from = c->d_corr_state + 4 * (q ^ 1) + 1;  // the first node correction k-1 changed
        fo.fold_prev = F[q ^ 1] + (size_t)lo * sz;
      }
      int rc = launch_fine(c, U, lo, bs, F[q] + (size_t)lo * sz, SS[q] + lo, 0, 1, nullptr, &fo);
      if (rc) return rc;
    }
    PF_CUDA(c, cudaEventRecord(c->ev_sw[q][ch], ps));
    return 0;
  };
  auto cancel_all = [&]() {
    const int one = 1;
    cudaMemcpyAsync(c->d_cancel, &one, sizeof(int), cudaMemcpyHostToDevice, c->stream);
    cudaStreamSynchronize(c->stream);
    for (int i = 0; i < C; ++i) cudaStreamSynchronize(c->pstream[i]);
  };
  for (int ch = 0; ch < C; ++ch) {
    PF_CUDA(c, cudaStreamWaitEvent(c->pstream[ch], c->ev_init, 0));
    if (int rc = sweep_chunk(0, ch, c->U.p, 0)) return rc;
  }
  std::vector<double> last(sz), tmp(sz);
  std::vector<Status> hst(nt);
  int iters = 0, stop = 0, frozen_prev = 0;
  for (int k = 0; k < k_max; ++k) {
    const int q = k & 1;
    // correction k, chunk by chunk, each after the sweep chunk it consumes
    if (k > 0) std::swap(c->gold, c->gnew);
    for (int ch = 0; ch < C; ++ch) {
      PF_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_sw[q][ch], 0));
      pf::CoarseArgs a{};
      a.mode = pf::CM_CORRECT;
      a.k_iter = k;
      a.guard = c->guard;
      a.ucur = c->U.p;
      a.fold = F[q];
      a.gold = c->gold.p;
      a.gnew = c->gnew.p;
      a.unext = c->Unext.p;
      a.out = c->scalar.p;
      a.n_begin = cb[ch];
      a.n_end = cb[ch + 1];
      a.state = c->d_corr_state + 4 * q;
      if (int rc = launch_coarse(c, a, c->d_corr_status)) return rc;
      PF_CUDA(c, cudaEventRecord(c->ev_co[q][ch], c->stream));
    }
    // speculative sweep k+1 on U^{k+1}, chunk ch as soon as correction chunk ch is done
    if (k + 1 < k_max)
      for (int ch = 0; ch < C; ++ch) {
        PF_CUDA(c, cudaStreamWaitEvent(c->pstream[ch], c->ev_co[q][ch], 0));
        if (int rc = sweep_chunk(k + 1, ch, c->Unext.p, frozen_prev)) return rc;
      }
    double h[2] = {0.0, 0.0};
    Status cs{};
    PF_CUDA(c, cudaMemcpyAsync(h, c->scalar.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    PF_CUDA(c, cudaMemcpyAsync(&cs, c->d_corr_status, sizeof(Status), cudaMemcpyDeviceToHost, c->stream));
    PF_CUDA(c, cudaMemcpyAsync(hst.data(), SS[q], sizeof(Status) * nt, cudaMemcpyDeviceToHost, c->stream));
    PF_CUDA(c, cudaStreamSynchronize(c->stream));  // correction k, hence every chunk of sweep k, is done
    // the sweep's failure first (parareal.py:75-88 raises before the correction)
    bool swept = false;  // some slice of sweep k was not frozen (the sequential driver's launch count)
    for (int n = 0; n < nt; ++n) {
      c->stats.pcg_iterations += hst[n].iters;
      c->stats.solves += hst[n].solves;
      swept |= hst[n].solves > 0;
    }
    if (swept) c->stats.fine_launches += 1;
    for (int n = 0; n < nt; ++n) {
      const Status& s1 = hst[n];
      if (s1.code == pf::ST_OK) continue;
      int best = n;
      for (int j = n + 1; j < nt; ++j)
        if (hst[j].code != pf::ST_OK &&
            (hst[j].r < hst[best].r ||
             (hst[j].r == hst[best].r && hst[j].code == pf::ST_COEFF && hst[best].code != pf::ST_COEFF)))
          best = j;
      cancel_all();
      c->err = pf_error{};
      c->err.step_n = 0;  // the reference's block [0, nt) (threads = 1)
      c->err.step_r = hst[best].r;
      if (hst[best].code == pf::ST_COEFF) {
        c->err.code = PF_ERR_COEFFICIENT;
        c->err.node = hst[best].node;
        std::snprintf(c->err.message, sizeof(c->err.message), "diffusion coefficient is not finite");
      } else {
        c->err.code = PF_ERR_SOLVER;
        std::snprintf(c->err.message, sizeof(c->err.message), "fine-sweep solve failed (interval %d)", hst[best].n);
      }
      return c->err.code;
    }
    c->stats.pcg_iterations += cs.iters;
    c->stats.solves += cs.solves;
    if (cs.code != pf::ST_OK) {
      cancel_all();
      c->err = pf_error{};
      c->err.step_r = -1;
      if (cs.code == pf::ST_DIVERGE) {
        c->err.code = PF_ERR_DIVERGENCE;
        c->err.iteration = k;
        c->err.interval = cs.n;
        std::snprintf(c->err.message, sizeof(c->err.message), "%s",
                      cs.r == 0 ? "non-finite state after correction sweep" : "state norm exceeds divergence guard");
      } else {
        c->err.code = cs.code == pf::ST_COEFF ? PF_ERR_COEFFICIENT : PF_ERR_SOLVER;
        c->err.node = cs.node;
        c->err.step_n = cs.n;
        std::snprintf(c->err.message, sizeof(c->err.message), "singular or ill-conditioned time-step system");
      }
      return c->err.code;
    }
    const double diff = h[0];
    c->warm_diff = diff;
    c->frozen = std::min((int)h[1], nt);
    frozen_prev = c->frozen;
    std::swap(c->U, c->Unext);  // u_curr = u_next (parareal.py:133)
    if (diffs) diffs[k] = diff;
    if (iteration_times)
      iteration_times[k] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (reference && errors) {
      if (download(c, last.data(), c->U.p + (size_t)nt * sz, sz)) return c->err.code;
      PF_CUDA(c, cudaStreamSynchronize(c->stream));
      for (size_t i = 0; i < sz; ++i) tmp[i] = last[i] - reference[(size_t)nt * sz + i];
      errors[k + 1] = host_norm(c, tmp.data());
    }
    iters = k + 1;
    fold_final = F[q];
    if (tol > 0 && diff < tol) {
      stop = 1;
      break;
    }
  }
  cancel_all();  // the speculative sweep after the last iteration
  if (iterations) *iterations = iters;
  if (stop_reason) *stop_reason = stop;
  return 0;
}

int pf_parareal(pf_ctx* c, const double* u0, double tol, int k_max, const double* reference, double* states,
                double* coarse_new, double* coarse_old, double* fine_endpoints, double* diffs,
                double* iteration_times, double* errors, int* iterations, int* stop_reason) {
  if (!c || !u0) return PF_ERR_ARGUMENT;
  if (k_max < 1) return set_error(c, PF_ERR_ARGUMENT, "k_max must be at least 1");
  const auto t0 = std::chrono::steady_clock::now();
  const int nt = c->grid.nt;
  const size_t sz = c->size;
  int rc = pf_dev_parareal_init(c, u0);
  if (rc) return rc;
  std::vector<double> last(sz), tmp(sz);
  if (reference && errors) {
    if (download(c, last.data(), c->U.p + (size_t)nt * sz, sz)) return c->err.code;
    PF_CUDA(c, cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < sz; ++i) tmp[i] = last[i] - reference[(size_t)nt * sz + i];
    errors[0] = host_norm(c, tmp.data());
  }
  int iters = 0, stop = 0;
  if (const int C = pipeline_chunks(c)) {
    double* fold_final = c->fold.p;
    rc = parareal_pipelined(c, C, tol, k_max, reference, diffs, iteration_times, errors, &iters, &stop, t0,
                            fold_final);
    if (rc) return rc;
    if (fine_endpoints && download(c, fine_endpoints, fold_final, (size_t)nt * sz)) return c->err.code;
    rc = pf_dev_parareal_read(c, states, coarse_new, coarse_old);
    if (rc) return rc;
    if (iterations) *iterations = iters;
    if (stop_reason) *stop_reason = stop;
    return 0;
  }
  for (int k = 0; k < k_max; ++k) {
    // slices below the frozen prefix have bitwise the inputs of their last
    // sweep: their F_old rows stand (see k_coarse CM_CORRECT)
    const int lo = k == 0 ? 0 : c->frozen;
    if (lo < nt) {
      rc = pf_dev_fine_sweep(c, c->U.p, lo, nt, c->fold.p + (size_t)lo * sz);
      if (rc) {
        // the reference sweeps the whole block [0, nt) (threads = 1,
        // parareal.py:75-88) and reports SolverFailure((0, r)); the frozen
        // prefix start `lo` is an internal optimisation, not part of the payload
        if (rc == PF_ERR_SOLVER) c->err.step_n = 0;
        return rc;
      }
    }
    double diff = 0.0;
    rc = pf_dev_parareal_correct(c, c->fold.p, k, &diff);
    if (rc) return rc;
    if (diffs) diffs[k] = diff;
    if (iteration_times)
      iteration_times[k] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (reference && errors) {
      if (download(c, last.data(), c->U.p + (size_t)nt * sz, sz)) return c->err.code;
      PF_CUDA(c, cudaStreamSynchronize(c->stream));
      for (size_t i = 0; i < sz; ++i) tmp[i] = last[i] - reference[(size_t)nt * sz + i];
      errors[k + 1] = host_norm(c, tmp.data());
    }
    iters = k + 1;
    if (tol > 0 && diff < tol) {
      stop = 1;
      break;
    }
  }
  if (fine_endpoints && download(c, fine_endpoints, c->fold.p, (size_t)nt * sz)) return c->err.code;
  rc = pf_dev_parareal_read(c, states, coarse_new, coarse_old);
  if (rc) return rc;
  if (iterations) *iterations = iters;
  if (stop_reason) *stop_reason = stop;
  return 0;
}

}  // extern "C"
