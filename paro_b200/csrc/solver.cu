// Batched, column-masked Jacobi-PCG on the device (cg_solve, linalg.cpp:143-223)
// and the Step-3 / Hartree drivers built on it (source_solve_step,
// paro.cpp:81-119; shifted_source_step, paro.cpp:194-210; hartree_solve_with,
// model.cpp:242-255).
//
// Per CG iteration two fused stencil passes run (march.cu):
//   K1: p = z + beta p (z = r / diag), pq = p.(A p)       -> finalize: alpha
//   K2: q = A p, x += alpha p, r -= alpha q, rz, rr       -> finalize: beta, stop test
// q is recomputed in K2 instead of stored, so one iteration moves
// 8 doubles per point and column (r,p,p' in K1; p,x,r,x',r' in K2). All
// scalars (alpha, beta, stop tests, NotSpd / IterationLimit detection) stay on
// the device; the host only polls an active-column count between CUDA-graph
// chunks of iterations, keeping one chunk in flight ahead of the poll.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "march.cuh"
#include "pcg_fin.cuh"
#include "poisson.hpp"
#include "solver.hpp"

namespace paro_b200 {

namespace {

// Columns with bnorm == 0 return x = 0 (linalg.cpp:158-162).
__global__ void zero_marked_kernel(const CgColumn* cols, int K, double* x, long long ld, long long n) {
  const int c = blockIdx.y;
  if (c >= K || cols[c].first != 2) return;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    x[c * ld + i] = 0.0;
}

// inv_diag = 1 / fl(c0 + fl(sigma*m0)); flags a non-positive diagonal.
// P > 0: written in the row-padded layout (rows of S points at stride P).
__global__ void invd_kernel(const double* c0, double sigma, double m0, const double* m0v, long long n, double* invd,
                            int* bad, int S, int P) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double d = __dadd_rn(c0[i], __dmul_rn(sigma, m0v ? m0v[i] : m0));
    if (d <= 0.0) *bad = 1;
    const long long o = P > 0 ? (i / S) * P + i % S : i;
    invd[o] = 1.0 / d;
  }
}

__global__ void set_flag_kernel(int* flag, int v) { *flag = v; }

// x of the listed columns: row-padded solver layout (rows of S at stride P,
// column stride ldi) -> the caller's dense layout (column stride ld); one warp
// per row
// With deferred x updates (k2c pairs), a column whose last iteration index
// was even still owes x += alpha p of that iteration (p in the p1 buffer):
// applied here, fl(x + fl(alpha p)), exactly the skipped single update.
__global__ void unpad_cols_kernel(const double* __restrict__ src, long long ldi, double* __restrict__ dst, long long ld,
                                  const int* __restrict__ cols, int S, int P, const CgColumn* __restrict__ cst,
                                  const double* __restrict__ p1, int deferred) {
  const int c = cols[blockIdx.y];
  const long long rows = static_cast<long long>(S) * S;
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const double* s = src + c * ldi;
  double* d = dst + c * ld;
  const bool pending = deferred && (cst[c].it & 1ull);
  const double al = cst[c].alpha;
  const double* pp = p1 + c * ldi;
  for (long long r = w0; r < rows; r += nw)
    for (int x = lane; x < S; x += 32) {
      const double v = s[r * P + x];
      d[r * S + x] = pending ? __dadd_rn(v, __dmul_rn(al, pp[r * P + x])) : v;
    }
}

// K columns: the caller's dense layout (stride ld) -> row-padded solver layout
// (rows of S at stride P, column stride ldi); one warp per row
__global__ void pad_cols_kernel(const double* __restrict__ src, long long ld, double* __restrict__ dst, long long ldi,
                                int S, int P) {
  const int c = blockIdx.y;
  const long long rows = static_cast<long long>(S) * S;
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const double* s = src + c * ld;
  double* d = dst + c * ldi;
  for (long long r = w0; r < rows; r += nw)
    for (int x = lane; x < S; x += 32) d[r * P + x] = s[r * S + x];
}

// 8 coefficient slots (dense, slot o at o*n) -> row-padded layout, slot o at o*ldi
__global__ void pad_coef_kernel(const double* __restrict__ coef, long long n, int S, int P, long long ldi,
                                double* __restrict__ out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long o = (i / S) * P + i % S;
#pragma unroll
    for (int k = 0; k < kSlots; ++k) out[k * ldi + o] = coef[k * n + i];
  }
}

struct Slots8 {
  double v[kSlots];
};

// out[o][i] = fl(coef[o][i] + sm[o]), sm[o] = fl(sigma m[o])
__global__ void preshift_kernel(const double* __restrict__ coef, Slots8 sm, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int o = 0; o < kSlots; ++o) out[o * n + i] = __dadd_rn(coef[o * n + i], sm.v[o]);
  }
}

// Fold a constant shift into a variable operator: (A + sigma M) as 8 SoA
// arrays in ctx.shifted, each slot the same fl(c + fl(sigma m)) the kernels
// would otherwise form per point, so the stencil passes read it directly.
OpDev preshift(Ctx& ctx, OpDev d) {
  if (d.coef == nullptr || d.mcoef != nullptr || d.sigma == 0.0) return d;
  const long long n = ctx.grid.n;
  double* out = ctx.shifted.get<double>(static_cast<size_t>(kSlots) * n);
  Slots8 sm;
  for (int o = 0; o < kSlots; ++o) sm.v[o] = d.sm[o];
  preshift_kernel<<<148 * 8, 256, 0, ctx.stream>>>(d.coef, sm, n, out);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
  d.coef = out;
  d.sigma = 0.0;
  for (int o = 0; o < kSlots; ++o) {
    d.sm[o] = 0.0;
    d.wc[o] = d.w[o];
  }
  return d;
}

int pick_cb(int K) { return K >= 8 ? 8 : K >= 4 ? 4 : K >= 2 ? 2 : 1; }

}  // namespace

// ---------------------------------------------------------------------------

OpDev make_opdev(const Ctx& ctx, const Op& a, const Op* shift, double sigma) {
  OpDev d;
  d.coef = a.var ? a.coef : nullptr;
  for (int o = 0; o < kSlots; ++o) d.w[o] = a.w[o];
  if (shift) {
    for (int o = 0; o < kSlots; ++o) d.m[o] = shift->w[o];
    d.mcoef = shift->var ? shift->coef : nullptr;
    d.sigma = sigma;
  }
  if (!a.var) d.invd_const = 1.0 / (a.w[0] + d.sigma * d.m[0]);
  // the same two roundings the kernels would apply per point: fl(w + fl(sigma m))
  for (int o = 0; o < kSlots; ++o) {
    const double sm = d.sigma * d.m[o];
    d.sm[o] = sm;
    d.wc[o] = d.w[o] + sm;
  }
  (void)ctx;
  return d;
}

void apply_op(Ctx& ctx, const Op& a, const Op* shift, double sigma, int K, const double* x, long long ldx,
              double* y, long long ldy, int z0, int z1) {
  ctx.check_grid();
  if (ldx != ldy) throw ParoError(kInvalidArgument, "apply: x and y must share a column stride");
  if (K <= 0) return;
  if (shift && shift->var) throw ParoError(kInvalidArgument, "apply: shift operator must be a constant stencil");
  if (z1 < 0) z1 = ctx.grid.S;
  if (z0 < 0 || z1 > ctx.grid.S || z0 >= z1) {
    if (z0 == z1) return;
    throw ParoError(kInvalidArgument, "apply: plane range outside the lattice");
  }
  MarchArgs m;
  plan_march(m, ctx.grid.S, z0, z1);
  m.K = K;
  m.ld = ldx;
  m.op = preshift(ctx, make_opdev(ctx, a, shift, sigma));
  m.src = x;
  m.dst = y;
  if (apply_flat_ok(a.var, m)) {
    const double* coefp = nullptr;
    long long ldi = 0;
    if (a.var) {  // the coefficients in the row-padded layout for the TMA staging
      const int S = ctx.grid.S;
      const int P = padded_row(S);
      ldi = ((static_cast<long long>(S) * S * P + 2 * kBulkPad + 31) / 32) * 32;
      double* cp = ctx.coefp.get<double>(static_cast<size_t>(kSlots) * ldi);
      pad_coef_kernel<<<148 * 8, 256, 0, ctx.stream>>>(m.op.coef, ctx.grid.n, S, P, ldi, cp);
      PARO_CUDA(cudaGetLastError());
      ++ctx.launches;
      coefp = cp;
    }
    launch_apply_flat(a.var, pick_cb(K), m, coefp, ldi, ctx.stream);
  } else {
    launch_march(kApply, a.var, pick_cb(K), m, ctx.stream);
  }
  ++ctx.launches;
}

// Core batched PCG. On entry `cols` (host) holds tol/max_iter per column; the
// setup pass computes r0 from either (M src)*scale (rhs == nullptr) or rhs.
// warm: x0 = src (source solves) ; cold: x0 = 0 (Hartree).
// PARO_PCG_TRACE=1: per-phase wall times of batched_pcg on stderr (synchronising)
struct PhaseTrace {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseTrace(cudaStream_t s) : st(s) {
    const char* e = std::getenv("PARO_PCG_TRACE");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pcg] %-14s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

void batched_pcg(Ctx& ctx, const OpDev& op_in, bool var, int K, const double* src, const double* rhs,
                 const double* scale_host, bool warm, double* x, long long ld, std::vector<CgColumn>& cols,
                 const Op* mass, bool abort_on_not_spd = false) {
  PhaseTrace trace(ctx.stream);
  const OpDev op = preshift(ctx, op_in);
  trace.mark("preshift");
  const Grid& g = ctx.grid;
  const long long n = g.n;
  cudaStream_t st = ctx.stream;
  MarchArgs m;
  plan_march(m, g.S);
  m.K = K;
  m.ld = ld;
  m.op = op;
  if (mass) {
    for (int o = 0; o < kSlots; ++o) m.mw[o] = mass->w[o];
    m.mwcoef = mass->var ? mass->coef : nullptr;
  }
  if (!var && op.mcoef) throw ParoError(kInvalidArgument, "pcg: a variable shift needs a variable operator");
  const int cb = pick_cb(K);
  // TMA-tensor passes (tma.cu) unless the shift stencil varies per point
  // (inexact mesh spacings: the LDGSTS march kernels take the per-point shift)
  const bool use_tma = op.mcoef == nullptr;
  const int P = use_tma ? padded_row(g.S) : g.S;
  const long long np = static_cast<long long>(g.S) * g.S * P;  // elements per column in the solver layout

  CgColumn* dcols = ctx.cols.get<CgColumn>(K);
  double* dscale = ctx.scale.get<double>(K);
  double* partials = ctx.partials.get<double>(static_cast<size_t>(K) * 3 * m.nblk);
  // the iteration vectors live in padded solver buffers (even stride ldi,
  // kBulkPad readable margins; rows padded to even length on the TMA path);
  // x is copied back to the caller's layout at the end
  const long long ldi = ((np + 2 * kBulkPad + 31) / 32) * 32;
  auto padded = [&](DevBuf& buf, int cols) {
    return buf.get<double>(static_cast<size_t>(cols) * ldi + 2 * kBulkPad) + kBulkPad;
  };
  double* r = padded(ctx.ws_a, K);
  double* p0 = padded(ctx.pbuf0, K);
  double* p1 = padded(ctx.pbuf1, K);
  double* xi = padded(ctx.pcg_x, K);
  // margins and column gaps are read as halo of the first/last points of a
  // row and must hold finite values (they meet zero weights)
  auto zero_margins = [&](double* v, int cols, long long len) {
    PARO_CUDA(cudaMemsetAsync(v - kBulkPad, 0, sizeof(double) * kBulkPad, st));
    PARO_CUDA(cudaMemset2DAsync(v + len, sizeof(double) * ldi, 0, sizeof(double) * (ldi - len), cols, st));
    PARO_CUDA(cudaMemsetAsync(v + static_cast<long long>(cols) * ldi, 0, sizeof(double) * kBulkPad, st));
  };
  for (double* v : {r, p0, p1, xi}) zero_margins(v, K, np);
  int* flag = ctx.flag.get<int>(3 + K);  // 3 flags + the copy-out column list

  small_h2d(ctx, dcols, cols.data(), sizeof(CgColumn) * K);
  if (scale_host) small_h2d(ctx, dscale, scale_host, sizeof(double) * K);

  // Jacobi preconditioner and the SPD diagonal check (linalg.cpp:164-173)
  set_flag_kernel<<<1, 1, 0, st>>>(flag, 0);
  set_flag_kernel<<<1, 1, 0, st>>>(flag + 1, 0);
  set_flag_kernel<<<1, 1, 0, st>>>(flag + 2, abort_on_not_spd ? 1 : 0);
  ctx.launches += 3;
  double* invd = nullptr;
  if (var) {
    invd = padded(ctx.invd, 1);
    zero_margins(invd, 1, np);
    invd_kernel<<<148 * 8, 256, 0, st>>>(op.coef, op.sigma, op.m[0], op.mcoef, n, invd, flag, g.S,
                                         use_tma ? P : 0);
    ++ctx.launches;
  } else {
    const double d = op.w[0] + op.sigma * op.m[0];
    if (d <= 0.0) set_flag_kernel<<<1, 1, 0, st>>>(flag, 1), ++ctx.launches;
  }
  PARO_CUDA(cudaGetLastError());
  m.invd = invd;
  m.cols = dcols;
  m.partials = partials;

  // tensor maps of the solver buffers (and the padded coefficient copy)
  PcgTma tmaps;
  if (use_tma) {
    double* coefp = nullptr;
    if (var) {  // the operator's coefficients in the row-padded layout for K2's TMA staging
      coefp = ctx.coefp.get<double>(static_cast<size_t>(kSlots) * ldi);
      pad_coef_kernel<<<148 * 8, 256, 0, st>>>(op.coef, n, g.S, P, ldi, coefp);
      PARO_CUDA(cudaGetLastError());
      ++ctx.launches;
    }
    tma_plan(tmaps, g.S, ldi, K, r, p0, p1, xi, invd, coefp);
  }

  // setup: r0, x0, bnorm, rz0, rnorm0
  m.src = src;
  m.dst = r;
  m.x = xi;
  m.ldw = ldi;
  m.P = use_tma ? P : 0;
  m.scale = dscale;
  m.rhs = rhs;
  if (use_tma && var && warm && rhs == nullptr && m.mwcoef == nullptr) {
    // x0 = u copied into the solver layout, then r0 = (M u) scale - A u on TMA planes of x
    pad_cols_kernel<<<dim3(148 * 2, K), 256, 0, st>>>(src, ld, xi, ldi, g.S, P);
    PARO_CUDA(cudaGetLastError());
    launch_tma_setup(cb, m, tmaps, st);
    ctx.launches += 2;
  } else {
    launch_march(warm ? kSetupWarm : kSetupCold, var, cb, m, st);
  }
  fin_kernel<<<K, kFinThreads, 0, st>>>(kFinSetup, dcols, partials, m.nblk, flag);
  zero_marked_kernel<<<dim3(148, K), 256, 0, st>>>(dcols, K, xi, ldi, np);
  ctx.launches += 3;
  PARO_CUDA(cudaGetLastError());
  trace.mark("setup");

  // iteration chunks captured once into a CUDA graph (PARO_NO_GRAPH=1 launches
  // them directly, e.g. for ncu)
  const int chunk = n >= (1 << 22) ? 4 : n >= (1 << 18) ? 8 : 16;  // even: ping-pong parity repeats
  // x updates in pairs of iterations on the k2c pass (half the x traffic):
  // even iterations leave x, odd ones apply both updates; a column stopping
  // after an even iteration gets its last update at the copy-out
  const bool deferred = use_tma && var && tma_k2c_active();
  auto enqueue_chunk = [&](cudaStream_t s) {
    for (int it = 0; it < chunk; ++it) {
      MarchArgs k1 = m;
      k1.ld = ldi;
      k1.pold = (it & 1) ? p1 : p0;
      k1.dst = (it & 1) ? p0 : p1;
      k1.r = r;
      // a per-point shift stencil runs on the LDGSTS march kernels
      if (use_tma) launch_tma(kK1, var, cb, k1, tmaps, (it & 1) == 0, s);
      else launch_march(kK1, var, cb, k1, s);
      fin_kernel<<<K, kFinThreads, 0, s>>>(kFinK1, dcols, partials, m.nblk, flag);
      MarchArgs k2 = m;
      k2.ld = ldi;
      k2.src = k1.dst;
      k2.x = xi;
      k2.r = r;
      k2.xmode = deferred ? (it & 1) : 2;  // chunk is even: it has the global iteration's parity
      k2.pold = k1.pold;                   // p of the previous iteration
      if (use_tma) launch_tma(kK2, var, cb, k2, tmaps, (it & 1) != 0, s);
      else launch_march(kK2, var, cb, k2, s);
      fin_kernel<<<K, kFinThreads, 0, s>>>(kFinK2, dcols, partials, m.nblk, flag);
    }
    count_active_kernel<<<1, 256, 0, s>>>(dcols, K, ctx.pinned_count_dev);
  };
  static const bool no_graph = [] {
    const char* e = std::getenv("PARO_NO_GRAPH");
    return e && e[0] == '1';
  }();
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  if (!no_graph) {
    cudaStream_t cap;
    PARO_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    PARO_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    enqueue_chunk(cap);
    PARO_CUDA(cudaStreamEndCapture(cap, &graph));
    PARO_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    PARO_CUDA(cudaStreamDestroy(cap));
  }
  trace.mark("graph");
  auto launch_chunk = [&] {
    if (no_graph) enqueue_chunk(st);
    else PARO_CUDA(cudaGraphLaunch(exec, st));
  };
  const unsigned long long nodes = 4ull * chunk + 1;

  cudaEvent_t ev[2];
  PARO_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  PARO_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  cudaEvent_t tev[2];
  PARO_CUDA(cudaEventCreate(&tev[0]));
  PARO_CUDA(cudaEventCreate(&tev[1]));
  volatile int* hcount = ctx.pinned_count;
  // prime: the setup may already have finished every column
  count_active_kernel<<<1, 256, 0, st>>>(dcols, K, ctx.pinned_count_dev);
  ++ctx.launches;
  PARO_CUDA(cudaEventRecord(ev[0], st));
  PARO_CUDA(cudaEventSynchronize(ev[0]));
  int remaining = *hcount;
  unsigned long long max_iter = 0;
  for (const auto& c : cols) max_iter = std::max(max_iter, c.max_iter);
  unsigned long long launched = 0;
  PARO_CUDA(cudaEventRecord(tev[0], st));
  // keep one chunk in flight ahead of the poll
  if (remaining > 0) {
    launch_chunk();
    PARO_CUDA(cudaEventRecord(ev[0], st));
    launched += chunk;
    ctx.launches += nodes;
  }
  int cur = 0;
  while (remaining > 0) {
    const bool more = launched < max_iter;
    if (more) {
      launch_chunk();
      PARO_CUDA(cudaEventRecord(ev[cur ^ 1], st));
      launched += chunk;
      ctx.launches += nodes;
    }
    PARO_CUDA(cudaEventSynchronize(ev[cur]));
    remaining = *hcount;
    if (trace.on) {
      const auto tn = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[pcg]   chunk done at %8.3f ms, active %d\n",
                   std::chrono::duration<double, std::milli>(tn - trace.t0).count(), remaining);
    }
    if (!more) {
      PARO_CUDA(cudaStreamSynchronize(st));
      remaining = *hcount;
      break;
    }
    cur ^= 1;
  }
  PARO_CUDA(cudaEventRecord(tev[1], st));
  PARO_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  PARO_CUDA(cudaEventElapsedTime(&ms, tev[0], tev[1]));
  PARO_CUDA(cudaEventDestroy(tev[0]));
  PARO_CUDA(cudaEventDestroy(tev[1]));
  PARO_CUDA(cudaEventDestroy(ev[0]));
  PARO_CUDA(cudaEventDestroy(ev[1]));
  if (exec) PARO_CUDA(cudaGraphExecDestroy(exec));
  if (graph) PARO_CUDA(cudaGraphDestroy(graph));
  trace.mark("iterations");
  std::vector<CgColumn> before = cols;
  small_d2h(ctx, cols.data(), dcols, sizeof(CgColumn) * K);
  // an aborted batch (NotSpd: the sigma policy restarts the step) has no result to return
  bool aborted = false;
  for (int c = 0; c < K; ++c) aborted |= abort_on_not_spd && cols[c].status == kNotSpd;
  if (trace.on)
    for (int c = 0; c < K; ++c)
      if (cols[c].status == kNotSpd) std::fprintf(stderr, "[pcg] NotSpd column %d at iteration %llu\n", c, cols[c].it);
  if (!aborted) {
    std::vector<int> out_cols;
    for (int c = 0; c < K; ++c)
      if (before[c].active) out_cols.push_back(c);
    if (!out_cols.empty()) {
      if (P == g.S && !deferred) {
        for (int c : out_cols)
          PARO_CUDA(cudaMemcpyAsync(x + c * ld, xi + c * ldi, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      } else {  // row-padded -> dense (+ a pending deferred update), every column in one launch
        int* dlist = flag + 3;
        small_h2d(ctx, dlist, out_cols.data(), sizeof(int) * out_cols.size());
        unpad_cols_kernel<<<dim3(148 * 2, static_cast<unsigned>(out_cols.size())), 256, 0, st>>>(
            xi, ldi, x, ld, dlist, g.S, P, dcols, p1, deferred ? 1 : 0);
        PARO_CUDA(cudaGetLastError());
        ++ctx.launches;
      }
    }
  }
  PARO_CUDA(cudaStreamSynchronize(st));
  trace.mark("copy-out");
  double col_iters = 0.0, batch_iters = 0.0;
  for (int c = 0; c < K; ++c)
    if (before[c].active) {
      col_iters += static_cast<double>(cols[c].it);
      batch_iters = std::max(batch_iters, static_cast<double>(cols[c].it));
    }
  if (trace.on)
    std::fprintf(stderr, "[pcg] K=%d col_iters=%.0f batch_iters=%.0f loop %.3f ms\n", K, col_iters, batch_iters, ms);
  const int base = var ? 0 : 3;
  ctx.stats[base + 0] += ms * 1e-3;
  ctx.stats[base + 1] += static_cast<double>(n) * (88.0 * col_iters + (var ? 64.0 : 0.0) * batch_iters);
  ctx.stats[base + 2] += col_iters;
}

static CgColumn make_col(double tol, unsigned long long max_iter) {
  CgColumn c{};
  c.tol = tol;
  c.max_iter = max_iter;
  c.active = 1;
  return c;
}

// source_solve_step (paro.cpp:81-119) for K columns at once.
int source_solve(Ctx& ctx, const Op& a, const Op& b, double sigma, int K, const double* u, long long ld,
                 const double* lambdas, double tol, unsigned long long max_iter, double* out,
                 SolveReport* report) {
  ctx.check_grid();
  if (!a.var && false) throw ParoError(kInvalidArgument, "source_solve: A must be variable");
  if (K <= 0) return kOk;
  const OpDev op = make_opdev(ctx, a, &b, sigma);
  std::vector<double> scale(K);
  for (int c = 0; c < K; ++c) scale[c] = lambdas[c] + sigma;  // paro.cpp:97
  std::vector<CgColumn> cols(K);
  for (int c = 0; c < K; ++c) cols[c] = make_col(tol, max_iter);
  batched_pcg(ctx, op, a.var, K, u, nullptr, scale.data(), true, out, ld, cols, &b, true);

  // A NotSpd in the first attempt fixes the step's outcome (the sigma policy
  // restarts the whole step, paro.cpp:204-207): the batch was aborted as soon
  // as it was seen, the remaining columns carry kAborted and report kOk.
  bool not_spd = false;
  for (int c = 0; c < K; ++c) not_spd |= cols[c].status == kNotSpd;
  if (not_spd) {
    if (report) {
      report->iterations.assign(K, 0);
      report->residual.assign(K, 0.0);
      report->status.assign(K, kOk);
      report->first_status.assign(K, kOk);
      for (int c = 0; c < K; ++c) {
        report->iterations[c] = cols[c].it;
        if (cols[c].status == kNotSpd) report->status[c] = report->first_status[c] = kNotSpd;
      }
    }
    ctx.err = "cg: operator not positive definite (p'Ap <= 0)";
    return kNotSpd;
  }
  std::vector<int> first_status(K, kOk), retry_status(K, kOk);
  std::vector<double> retry_resid(K, 0.0);
  std::vector<CgColumn> retry(K);
  bool any_retry = false;
  for (int c = 0; c < K; ++c) {
    first_status[c] = cols[c].status;
    if (cols[c].status == kIterationLimit) {
      retry[c] = make_col(tol * 100.0, max_iter * 4);  // paro.cpp:105-109
      any_retry = true;
    } else {
      retry[c] = cols[c];
      retry[c].active = 0;
    }
  }
  if (any_retry) {
    batched_pcg(ctx, op, a.var, K, u, nullptr, scale.data(), true, out, ld, retry, &b);
    for (int c = 0; c < K; ++c)
      if (first_status[c] == kIterationLimit) {
        retry_status[c] = retry[c].status;
        retry_resid[c] = retry[c].rnorm / retry[c].bnorm;
      }
  }
  if (report) {
    report->iterations.assign(K, 0);
    report->residual.assign(K, 0.0);
    report->status.assign(K, kOk);
    report->first_status = first_status;
    for (int c = 0; c < K; ++c) {
      const CgColumn& f = first_status[c] == kIterationLimit ? retry[c] : cols[c];
      report->iterations[c] = f.it;
      report->residual[c] = f.bnorm > 0 ? f.rnorm / f.bnorm : 0.0;
      report->status[c] = first_status[c] == kIterationLimit ? retry_status[c] : first_status[c];
    }
  }
  // Exception semantics of the serial reference loop: a failure inside the
  // retry escapes immediately; first-attempt failures are rethrown by index.
  for (int c = 0; c < K; ++c)
    if (first_status[c] == kIterationLimit && retry_status[c] != kOk) {
      ctx.resid = retry_resid[c];
      ctx.err = retry_status[c] == kNotSpd ? "cg: operator not positive definite (p'Ap <= 0)"
                                            : "cg: iteration limit reached";
      return retry_status[c];
    }
  for (int c = 0; c < K; ++c)
    if (first_status[c] != kOk && first_status[c] != kIterationLimit) {
      ctx.err = "cg: operator not positive definite";
      return first_status[c];
    }
  return kOk;
}

// shifted_source_step (paro.cpp:194-210): sigma = max(0, 0.5 - lambda_1),
// doubled (2 sigma + 1) on NotSpd, at most 5 attempts.
int shifted_source_solve(Ctx& ctx, const Op& a, const Op& b, int K, const double* u, long long ld,
                         const double* lambdas, double tol, unsigned long long max_iter, double* out,
                         double* sigma_out, SolveReport* report) {
  double sigma = std::max(0.0, 0.5 - lambdas[0]);
  for (int attempt = 0;; ++attempt) {
    const int st = source_solve(ctx, a, b, sigma, K, u, ld, lambdas, tol, max_iter, out, report);
    *sigma_out = sigma;
    if (st != kNotSpd) return st;
    if (attempt >= 4) return st;
    sigma = 2.0 * sigma + 1.0;
  }
}

// cg_solve(a, b, {x0, tol, max_iter}) for K right-hand sides at once.
int cg_solve(Ctx& ctx, const Op& a, int K, const double* rhs, const double* x0, long long ld, double tol,
             unsigned long long max_iter, bool throw_on_max, double* x, SolveReport* report) {
  ctx.check_grid();
  const OpDev op = make_opdev(ctx, a, nullptr, 0.0);
  std::vector<CgColumn> cols(K);
  for (int c = 0; c < K; ++c) cols[c] = make_col(tol, max_iter);
  const double* src = x0;
  double* zeros = nullptr;
  if (!src) {
    zeros = ctx.ws_c.get<double>(static_cast<size_t>(K) * ld);
    PARO_CUDA(cudaMemsetAsync(zeros, 0, sizeof(double) * K * ld, ctx.stream));
    src = zeros;
  }
  batched_pcg(ctx, op, a.var, K, src, rhs, nullptr, true, x, ld, cols, nullptr);
  int status = kOk;
  if (report) {
    report->iterations.assign(K, 0);
    report->residual.assign(K, 0.0);
    report->status.assign(K, kOk);
  }
  for (int c = 0; c < K; ++c) {
    int s = cols[c].status;
    if (s == kIterationLimit && !throw_on_max) s = kOk;
    if (report) {
      report->iterations[c] = cols[c].it;
      report->residual[c] = cols[c].bnorm > 0 ? cols[c].rnorm / cols[c].bnorm : 0.0;
      report->status[c] = s;
    }
    if (s != kOk && status == kOk) {
      status = s;
      ctx.resid = cols[c].bnorm > 0 ? cols[c].rnorm / cols[c].bnorm : 0.0;
      ctx.err = s == kNotSpd ? "cg: operator not positive definite" : "cg: iteration limit reached";
    }
  }
  return status;
}

// hartree_solve_with (model.cpp:242-255): K_poisson V = 4 pi M rho, cold start,
// Jacobi-PCG to `tol`, at most 200000 iterations.
int hartree_solve(Ctx& ctx, const Op& poisson, const Op& mass, const double* rho, double tol, double* vh,
                  SolveReport* report) {
  ctx.check_grid();
  if (ctx.hartree_mode == 1 && dst_applicable(poisson)) {
    if (report) {
      report->iterations.assign(1, 0);
      report->residual.assign(1, 0.0);
      report->status.assign(1, kOk);
    }
    return hartree_dst(ctx, poisson, mass, rho, vh);
  }
  const OpDev op = make_opdev(ctx, poisson, nullptr, 0.0);
  const double four_pi = 4.0 * M_PI;
  std::vector<CgColumn> cols(1, make_col(tol, 200000));
  batched_pcg(ctx, op, poisson.var, 1, rho, nullptr, &four_pi, false, vh, ctx.grid.n, cols, &mass);
  if (report) {
    report->iterations.assign(1, cols[0].it);
    report->residual.assign(1, cols[0].bnorm > 0 ? cols[0].rnorm / cols[0].bnorm : 0.0);
    report->status.assign(1, cols[0].status);
  }
  if (cols[0].status != kOk) {
    ctx.resid = cols[0].bnorm > 0 ? cols[0].rnorm / cols[0].bnorm : 0.0;
    ctx.err = cols[0].status == kNotSpd ? "hartree: cg not positive definite" : "hartree: cg iteration limit";
  }
  return cols[0].status;
}

}  // namespace paro_b200
