// C ABI (include/paro_b200.h) over the device implementation.
#include "paro_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.hpp"
#include "assemble.hpp"
#include "estimate.hpp"
#include "fields.hpp"
#include "ritz.hpp"
#include "solver.hpp"
#include "step4.hpp"
#include "csr.hpp"

struct paro_ctx {
  paro_b200::Ctx c;
};
struct paro_op {
  paro_b200::Op o;
  paro_ctx* owner = nullptr;
};
struct paro_csr {
  paro_b200::CsrOp a;
};

using namespace paro_b200;

namespace {

thread_local std::string g_noctx_err;

template <typename F>
int guarded(paro_ctx* ctx, F&& f) {
  try {
    if (ctx) PARO_CUDA(cudaSetDevice(ctx->c.device));
    return f();
  } catch (const ParoError& e) {
    if (ctx) {
      ctx->c.err = e.what();
      ctx->c.resid = e.residual;
    } else {
      g_noctx_err = e.what();
    }
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.err = e.what();
    else g_noctx_err = e.what();
    return kError;
  }
}

void dof_xyz(long long i, int S, int& x, int& y, int& z) {
  x = static_cast<int>(i % S);
  y = static_cast<int>((i / S) % S);
  z = static_cast<int>(i / (static_cast<long long>(S) * S));
}

}  // namespace

extern "C" {

int paro_ctx_create(int device, void* stream, paro_ctx** out) {
  return guarded(nullptr, [&] {
    auto* ctx = new paro_ctx();
    ctx->c.device = device;
    PARO_CUDA(cudaSetDevice(device));
    ctx->c.stream = static_cast<cudaStream_t>(stream);
    PARO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->c.pinned_count), sizeof(int), cudaHostAllocMapped));
    PARO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->c.pinned_count_dev), ctx->c.pinned_count, 0));
    *out = ctx;
    return kOk;
  });
}

int paro_ctx_destroy(paro_ctx* ctx) {
  if (!ctx) return kOk;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  for (DevBuf* b : {&ctx->c.partials, &ctx->c.cols, &ctx->c.scale, &ctx->c.invd, &ctx->c.pbuf0, &ctx->c.pbuf1,
                    &ctx->c.flag, &ctx->c.ws_a, &ctx->c.ws_b, &ctx->c.ws_c, &ctx->c.ws_d, &ctx->c.ws_e,
                    &ctx->c.ws_small, &ctx->c.ws_small2, &ctx->c.dst_tab, &ctx->c.wtab, &ctx->c.shifted, &ctx->c.coefp, &ctx->c.csr_ws, &ctx->c.csr_ws2, &ctx->c.csr_io, &ctx->c.pcg_x, &ctx->c.ws_gram,
                    &ctx->c.ws_small3})
    b->release();
  if (ctx->c.pinned_count) cudaFreeHost(ctx->c.pinned_count);
  paro_b200::xfer_release(ctx->c);
  delete ctx;
  return kOk;
}

int paro_ctx_set_stream(paro_ctx* ctx, void* stream) {
  return guarded(ctx, [&] {
    ctx->c.stream = static_cast<cudaStream_t>(stream);
    return kOk;
  });
}

const char* paro_ctx_last_error(const paro_ctx* ctx) { return ctx ? ctx->c.err.c_str() : g_noctx_err.c_str(); }
double paro_ctx_last_residual(const paro_ctx* ctx) { return ctx ? ctx->c.resid : 0.0; }
unsigned long long paro_ctx_launches(const paro_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int paro_ctx_stats(paro_ctx* ctx, double out[8], int reset) {
  if (!ctx) return kInvalidArgument;
  for (int i = 0; i < 8; ++i) {
    if (out) out[i] = ctx->c.stats[i];
    if (reset) ctx->c.stats[i] = 0.0;
  }
  return kOk;
}

int paro_ctx_set_hartree_mode(paro_ctx* ctx, int mode) {
  return guarded(ctx, [&] {
    ctx->c.hartree_mode = mode;
    return kOk;
  });
}

int paro_ctx_set_ritz_copyout(paro_ctx* ctx, void* copy_stream, double* host, long long ldh, int c0, int c1) {
  return guarded(ctx, [&] {
    auto& co = ctx->c.ritz_copyout;
    co.stream = static_cast<cudaStream_t>(copy_stream);
    co.host = host;
    co.ldh = ldh;
    co.c0 = c0;
    co.c1 = c1;
    return kOk;
  });
}

int paro_ctx_set_ritz_mode(paro_ctx* ctx, int mode) {
  return guarded(ctx, [&] {
    ctx->c.force_cgs2 = mode == 1;
    ctx->c.two_pass_only = mode == 2;
    return kOk;
  });
}

int paro_ctx_synchronize(paro_ctx* ctx) {
  return guarded(ctx, [&] {
    PARO_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return kOk;
  });
}

int paro_malloc(paro_ctx* ctx, size_t bytes, void** dev) {
  return guarded(ctx, [&] {
    PARO_CUDA(cudaMalloc(dev, bytes));
    return kOk;
  });
}
int paro_free(paro_ctx* ctx, void* dev) {
  return guarded(ctx, [&] {
    PARO_CUDA(cudaFree(dev));
    return kOk;
  });
}
int paro_memcpy_h2d(paro_ctx* ctx, void* dev, const void* host, size_t bytes) {
  return guarded(ctx, [&] {
    PARO_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->c.stream));
    PARO_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return kOk;
  });
}
int paro_memcpy_d2h(paro_ctx* ctx, void* host, const void* dev, size_t bytes) {
  return guarded(ctx, [&] {
    PARO_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->c.stream));
    PARO_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return kOk;
  });
}

// Column blocks between scattered host vectors (the reference's
// std::vector<std::vector<double>>) and a device [k][ld] block through a
// pinned two-slot staging ring: host memcpy of column c + 1 overlaps the DMA
// of column c, and no pageable-memory transfer stalls the copy engine.
namespace {
struct Staging {
  double* buf[2] = {nullptr, nullptr};
  size_t cap = 0;  // doubles per slot
  cudaEvent_t done[2] = {nullptr, nullptr};
};
Staging& staging(paro_ctx* ctx, size_t doubles) {
  static thread_local Staging st;
  static thread_local int dev = -1;
  if (st.cap < doubles || dev != ctx->c.device) {
    for (int i = 0; i < 2; ++i) {
      if (st.buf[i]) cudaFreeHost(st.buf[i]);
      if (st.done[i]) cudaEventDestroy(st.done[i]);
      st.buf[i] = nullptr;
      st.done[i] = nullptr;
    }
    st.cap = 0;
    for (int i = 0; i < 2; ++i) {
      PARO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&st.buf[i]), doubles * sizeof(double), cudaHostAllocDefault));
      PARO_CUDA(cudaEventCreateWithFlags(&st.done[i], cudaEventDisableTiming));
    }
    st.cap = doubles;
    dev = ctx->c.device;
  }
  return st;
}
constexpr size_t kStageDoubles = size_t(4) << 20;  // 32 MB per slot
}  // namespace

int paro_upload_columns(paro_ctx* ctx, int k, const double* const* host, size_t n, double* dev, long long ld) {
  return guarded(ctx, [&] {
    if (k < 0 || (k > 0 && (!host || !dev)) || ld < static_cast<long long>(n))
      throw ParoError(kInvalidArgument, "upload_columns: bad arguments");
    Staging& st = staging(ctx, kStageDoubles);
    int slot = 0;
    bool used[2] = {false, false};
    for (int c = 0; c < k; ++c)
      for (size_t off = 0; off < n; off += st.cap) {
        const size_t cnt = std::min(st.cap, n - off);
        if (used[slot]) PARO_CUDA(cudaEventSynchronize(st.done[slot]));
        std::memcpy(st.buf[slot], host[c] + off, cnt * sizeof(double));
        PARO_CUDA(cudaMemcpyAsync(dev + c * ld + off, st.buf[slot], cnt * sizeof(double), cudaMemcpyHostToDevice,
                                  ctx->c.stream));
        PARO_CUDA(cudaEventRecord(st.done[slot], ctx->c.stream));
        used[slot] = true;
        slot ^= 1;
      }
    PARO_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return kOk;
  });
}

int paro_download_columns(paro_ctx* ctx, int k, const double* dev, long long ld, size_t n, double* const* host) {
  return guarded(ctx, [&] {
    if (k < 0 || (k > 0 && (!host || !dev)) || ld < static_cast<long long>(n))
      throw ParoError(kInvalidArgument, "download_columns: bad arguments");
    Staging& st = staging(ctx, kStageDoubles);
    // chunk i lands in slot i % 2; its host copy happens after chunk i + 1 is queued
    struct Pending {
      double* dst;
      size_t cnt;
    } pend[2] = {{nullptr, 0}, {nullptr, 0}};
    int slot = 0;
    auto drain = [&](int s) {
      if (!pend[s].dst) return;
      PARO_CUDA(cudaEventSynchronize(st.done[s]));
      std::memcpy(pend[s].dst, st.buf[s], pend[s].cnt * sizeof(double));
      pend[s].dst = nullptr;
    };
    for (int c = 0; c < k; ++c)
      for (size_t off = 0; off < n; off += st.cap) {
        const size_t cnt = std::min(st.cap, n - off);
        drain(slot);
        PARO_CUDA(cudaMemcpyAsync(st.buf[slot], dev + c * ld + off, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                  ctx->c.stream));
        PARO_CUDA(cudaEventRecord(st.done[slot], ctx->c.stream));
        pend[slot] = {host[c] + off, cnt};
        slot ^= 1;
      }
    drain(slot);
    drain(slot ^ 1);
    return kOk;
  });
}

int paro_grid_init(paro_ctx* ctx, int subdivisions, double lo, double hi) {
  return guarded(ctx, [&] {
    if (subdivisions < 2) throw ParoError(kInvalidArgument, "grid: subdivisions must be >= 2");
    if (!(hi - lo > 0.0)) throw ParoError(kInvalidArgument, "grid: box has non-positive edge length");
    Grid& g = ctx->c.grid;
    g.s = subdivisions;
    g.S = subdivisions - 1;
    g.n = static_cast<long long>(g.S) * g.S * g.S;
    g.lo = lo;
    g.hi = hi;
    ctx->c.grid_set = true;
    ctx->c.mass_state = 0;
    return kOk;
  });
}

long long paro_grid_dofs(const paro_ctx* ctx) { return ctx && ctx->c.grid_set ? ctx->c.grid.n : 0; }

int paro_op_create_const(paro_ctx* ctx, const double w[8], paro_op** out) {
  return guarded(ctx, [&] {
    auto* op = new paro_op();
    op->owner = ctx;
    op->o.var = false;
    for (int o = 0; o < kSlots; ++o) op->o.w[o] = w[o];
    op->o.n = ctx->c.grid.n;
    *out = op;
    return kOk;
  });
}

int paro_op_create_var(paro_ctx* ctx, paro_op** out) {
  return guarded(ctx, [&] {
    ctx->c.check_grid();
    auto* op = new paro_op();
    op->owner = ctx;
    op->o.var = true;
    op->o.n = ctx->c.grid.n;
    PARO_CUDA(cudaMalloc(&op->o.coef, sizeof(double) * kSlots * op->o.n));
    PARO_CUDA(cudaMemsetAsync(op->o.coef, 0, sizeof(double) * kSlots * op->o.n, ctx->c.stream));
    op->o.owns = true;
    *out = op;
    return kOk;
  });
}

int paro_op_from_csr(paro_ctx* ctx, size_t n, const size_t* rows, const uint32_t* cols, const double* vals,
                     paro_op** out) {
  return guarded(ctx, [&] {
    ctx->c.check_grid();
    const int S = ctx->c.grid.S;
    if (static_cast<long long>(n) != ctx->c.grid.n)
      throw ParoError(kInvalidArgument, "op_from_csr: dimension does not match the grid");
    std::vector<double> coef(static_cast<size_t>(kSlots) * n, 0.0);
    double scale = 0.0;
    for (size_t k = 0; k < rows[n]; ++k) scale = std::max(scale, std::abs(vals[k]));
    struct Back {
      size_t j;
      int o;
      double v;
    };
    std::vector<Back> back;
    back.reserve(7 * n);
    for (size_t i = 0; i < n; ++i) {
      int x, y, z;
      dof_xyz(static_cast<long long>(i), S, x, y, z);
      for (size_t k = rows[i]; k < rows[i + 1]; ++k) {
        const size_t j = cols[k];
        if (j >= n) throw ParoError(kInvalidArgument, "op_from_csr: column out of range");
        int xj, yj, zj;
        dof_xyz(static_cast<long long>(j), S, xj, yj, zj);
        const int dx = xj - x, dy = yj - y, dz = zj - z;
        const bool fwd = (dx == 0 || dx == 1) && (dy == 0 || dy == 1) && (dz == 0 || dz == 1);
        const bool bwd = (dx == 0 || dx == -1) && (dy == 0 || dy == -1) && (dz == 0 || dz == -1);
        if (!fwd && !bwd) throw ParoError(kInvalidArgument, "op_from_csr: pattern is not the P1/Kuhn stencil");
        if (fwd) {
          const int o = dx + 2 * dy + 4 * dz;
          coef[static_cast<size_t>(o) * n + i] = vals[k];
        } else {
          back.push_back({j, -dx - 2 * dy - 4 * dz, vals[k]});
        }
      }
    }
    for (const Back& b : back) {
      if (std::abs(coef[static_cast<size_t>(b.o) * n + b.j] - b.v) > 1e-13 * std::max(1.0, scale))
        throw ParoError(kInvalidArgument, "op_from_csr: matrix is not symmetric");
    }
    // uniform operator -> constant stencil (only slots whose neighbour exists)
    bool uniform = true;
    double w[kSlots];
    bool seen[kSlots] = {};
    for (size_t i = 0; i < n && uniform; ++i) {
      int x, y, z;
      dof_xyz(static_cast<long long>(i), S, x, y, z);
      for (int o = 0; o < kSlots; ++o) {
        const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
        if (x + ox >= S || y + oy >= S || z + oz >= S) continue;
        const double v = coef[static_cast<size_t>(o) * n + i];
        if (!seen[o]) {
          w[o] = v;
          seen[o] = true;
        } else if (v != w[o]) {
          uniform = false;
          break;
        }
      }
    }
    auto* op = new paro_op();
    op->owner = ctx;
    op->o.n = static_cast<long long>(n);
    if (uniform) {
      op->o.var = false;
      for (int o = 0; o < kSlots; ++o) op->o.w[o] = seen[o] ? w[o] : 0.0;
    } else {
      op->o.var = true;
      PARO_CUDA(cudaMalloc(&op->o.coef, sizeof(double) * kSlots * n));
      PARO_CUDA(cudaMemcpy(op->o.coef, coef.data(), sizeof(double) * kSlots * n, cudaMemcpyHostToDevice));
      op->o.owns = true;
    }
    *out = op;
    return kOk;
  });
}

int paro_op_to_csr(paro_ctx* ctx, const paro_op* a, size_t* nnz, size_t* rows, uint32_t* cols, double* vals) {
  return guarded(ctx, [&] {
    ctx->c.check_grid();
    const int S = ctx->c.grid.S;
    const long long n = ctx->c.grid.n;
    std::vector<double> coef;
    if (a->o.var && vals) {
      coef.resize(static_cast<size_t>(kSlots) * n);
      PARO_CUDA(cudaStreamSynchronize(ctx->c.stream));
      PARO_CUDA(cudaMemcpy(coef.data(), a->o.coef, sizeof(double) * coef.size(), cudaMemcpyDeviceToHost));
    }
    auto weight = [&](int o, long long at) { return a->o.var ? coef[static_cast<size_t>(o) * n + at] : a->o.w[o]; };
    size_t k = 0;
    const long long S2 = static_cast<long long>(S) * S;
    for (long long i = 0; i < n; ++i) {
      int x, y, z;
      dof_xyz(i, S, x, y, z);
      if (rows) rows[i] = k;
      // ascending column order: backward 7..1, centre, forward 1..7
      for (int pass = 0; pass < 3; ++pass) {
        for (int t = 1; t <= 7; ++t) {
          if (pass == 1 && t > 1) break;
          const int o = pass == 0 ? 8 - t : pass == 1 ? 0 : t;
          const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
          const int sg = pass == 0 ? -1 : 1;
          const int xj = x + sg * ox, yj = y + sg * oy, zj = z + sg * oz;
          if (xj < 0 || yj < 0 || zj < 0 || xj >= S || yj >= S || zj >= S) continue;
          const long long j = (static_cast<long long>(zj) * S + yj) * S + xj;
          if (cols) cols[k] = static_cast<uint32_t>(j);
          if (vals) vals[k] = pass == 0 ? weight(o, j) : weight(o, i);
          ++k;
        }
      }
    }
    if (rows) rows[n] = k;
    (void)S2;
    *nnz = k;
    return kOk;
  });
}

int paro_op_coefficients(paro_op* a, double** dev) {
  if (!a || !a->o.var) return kInvalidArgument;
  *dev = a->o.coef;
  return kOk;
}

int paro_op_weights(const paro_op* a, double w[8], int* is_var) {
  if (!a) return kInvalidArgument;
  for (int o = 0; o < kSlots; ++o) w[o] = a->o.w[o];
  if (is_var) *is_var = a->o.var ? 1 : 0;
  return kOk;
}

int paro_op_destroy(paro_op* a) {
  if (!a) return kOk;
  if (a->o.owns && a->o.coef) {
    if (a->owner) cudaSetDevice(a->owner->c.device);
    cudaFree(a->o.coef);
  }
  delete a;
  return kOk;
}

int paro_op_apply(paro_ctx* ctx, const paro_op* a, const paro_op* shift, double sigma, int k, const double* x,
                  long long ldx, double* y, long long ldy) {
  return guarded(ctx, [&] {
    apply_op(ctx->c, a->o, shift ? &shift->o : nullptr, sigma, k, x, ldx, y, ldy);
    return kOk;
  });
}

int paro_op_apply_planes(paro_ctx* ctx, const paro_op* a, int k, const double* x, long long ld, double* y, int z0,
                         int z1) {
  return guarded(ctx, [&] {
    apply_op(ctx->c, a->o, nullptr, 0.0, k, x, ld, y, ld, z0, z1);
    return kOk;
  });
}

// ------------------------------------------------ Step-4 building blocks on row ranges
int paro_gram_sym(paro_ctx* ctx, int k, const double* x, long long ldx, const double* y, long long ldy, long long r0,
                  long long r1, double* g) {
  return guarded(ctx, [&] {
    if (r0 < 0 || r1 < r0) throw ParoError(kInvalidArgument, "gram_sym: bad row range");
    gram_sym_rows(ctx->c, k, x, ldx, y, ldy, r0, r1, g);
    return kOk;
  });
}

int paro_gram_rect(paro_ctx* ctx, int k1, const double* x, long long ldx, int k2, const double* y, long long ldy,
                   long long r0, long long r1, double* g) {
  return guarded(ctx, [&] {
    if (r0 < 0 || r1 < r0) throw ParoError(kInvalidArgument, "gram_rect: bad row range");
    gram_rect_rows(ctx->c, k1, x, ldx, k2, y, ldy, r0, r1, g);
    return kOk;
  });
}

int paro_rotate(paro_ctx* ctx, int k1, const double* x, long long ldx, const double* c, int ldc, int k2, double* z,
                long long ldz, long long r0, long long r1, int mode) {
  return guarded(ctx, [&] {
    if (r0 < 0 || r1 < r0) throw ParoError(kInvalidArgument, "rotate: bad row range");
    rotate_rows(ctx->c, k1, x, ldx, c, ldc, k2, z, ldz, r0, r1, mode);
    return kOk;
  });
}

int paro_ritz_ortho(paro_ctx* ctx, int K, const double* g, double drop_tol, double* c1, int* k_out,
                    double* min_ratio) {
  return guarded(ctx, [&] { return ritz_ortho(ctx->c, K, g, drop_tol, c1, k_out, min_ratio); });
}

int paro_ritz_second_pass(paro_ctx* ctx, int k, const double* g2, double* c2, double* bt) {
  return guarded(ctx, [&] { return ritz_second_pass(ctx->c, k, g2, c2, bt); });
}

int paro_ritz_congruence(paro_ctx* ctx, int k, const double* g, const double* c1, double* bt) {
  return guarded(ctx, [&] { return ritz_congruence(ctx->c, k, g, c1, bt); });
}

int paro_ritz_pencil(paro_ctx* ctx, int k, const double* ga, const double* c2, const double* bt, const double* gb,
                     double* vals, double* y) {
  return guarded(ctx, [&] { return ritz_pencil(ctx->c, k, ga, c2, bt, gb, vals, y); });
}

int paro_gram_defect(paro_ctx* ctx, int k, const double* g, double* out) {
  return guarded(ctx, [&] {
    *out = ritz_defect(ctx->c, k, g);
    return kOk;
  });
}

int paro_sign_init(paro_ctx* ctx, int k, double* amax, long long* first) {
  return guarded(ctx, [&] {
    sign_init(ctx->c, k, amax, first);
    return kOk;
  });
}

int paro_colmax(paro_ctx* ctx, int k, const double* v, long long ld, long long r0, long long r1, double* amax) {
  return guarded(ctx, [&] {
    colmax_rows(ctx->c, k, v, ld, r0, r1, amax);
    return kOk;
  });
}

int paro_first_above(paro_ctx* ctx, int k, const double* v, long long ld, long long r0, long long r1,
                     const double* amax, long long* first) {
  return guarded(ctx, [&] {
    first_rows(ctx->c, k, v, ld, r0, r1, amax, first);
    return kOk;
  });
}

int paro_sign_flags(paro_ctx* ctx, int k, const double* v, long long ld, long long r0, long long r1,
                    const double* amax, const long long* first, double* flip) {
  return guarded(ctx, [&] {
    sign_rows(ctx->c, k, v, ld, r0, r1, amax, first, flip);
    return kOk;
  });
}

int paro_negate_columns(paro_ctx* ctx, int k, double* v, long long ld, long long r0, long long r1,
                        const double* flip) {
  return guarded(ctx, [&] {
    negate_rows(ctx->c, k, v, ld, r0, r1, flip);
    return kOk;
  });
}

static void fill_report(const SolveReport& r, size_t* iters, double* resid) {
  for (size_t c = 0; c < r.iterations.size(); ++c) {
    if (iters) iters[c] = static_cast<size_t>(r.iterations[c]);
    if (resid) resid[c] = r.residual[c];
  }
}

int paro_cg_solve(paro_ctx* ctx, const paro_op* a, int k, const double* b, const double* x0, long long ld,
                  double tol, size_t max_iter, int throw_on_max, double* x, size_t* iters, double* resid) {
  return guarded(ctx, [&] {
    SolveReport rep;
    const int st = cg_solve(ctx->c, a->o, k, b, x0, ld, tol, max_iter, throw_on_max != 0, x, &rep);
    fill_report(rep, iters, resid);
    return st;
  });
}

int paro_source_solve_step(paro_ctx* ctx, const paro_op* a, const paro_op* b, int k, const double* u, long long ld,
                           const double* lambdas, double tol, size_t max_iter, double sigma, double* out,
                           size_t* iters, double* resid) {
  return paro_source_solve_columns(ctx, a, b, k, u, ld, lambdas, tol, max_iter, sigma, out, iters, resid, nullptr,
                                   nullptr);
}

int paro_source_solve_columns(paro_ctx* ctx, const paro_op* a, const paro_op* b, int k, const double* u,
                              long long ld, const double* lambdas, double tol, size_t max_iter, double sigma,
                              double* out, size_t* iters, double* resid, int* first_status, int* final_status) {
  return guarded(ctx, [&] {
    SolveReport rep;
    const int st = source_solve(ctx->c, a->o, b->o, sigma, k, u, ld, lambdas, tol, max_iter, out, &rep);
    fill_report(rep, iters, resid);
    for (int c = 0; c < k; ++c) {
      if (first_status) first_status[c] = rep.first_status.empty() ? kOk : rep.first_status[c];
      if (final_status) final_status[c] = rep.status.empty() ? kOk : rep.status[c];
    }
    return st;
  });
}

int paro_shifted_source_step(paro_ctx* ctx, const paro_op* a, const paro_op* b, int k, const double* u,
                             long long ld, const double* lambdas, double tol, size_t max_iter, double* out,
                             double* sigma_out, size_t* iters, double* resid) {
  return guarded(ctx, [&] {
    SolveReport rep;
    const int st = shifted_source_solve(ctx->c, a->o, b->o, k, u, ld, lambdas, tol, max_iter, out, sigma_out, &rep);
    fill_report(rep, iters, resid);
    return st;
  });
}

int paro_hartree_solve(paro_ctx* ctx, const paro_op* poisson, const paro_op* mass, const double* rho, double tol,
                       double* vh, size_t* iters) {
  return guarded(ctx, [&] {
    SolveReport rep;
    const int st = hartree_solve(ctx->c, poisson->o, mass->o, rho, tol, vh, &rep);
    fill_report(rep, iters, nullptr);
    return st;
  });
}

int paro_rayleigh_ritz(paro_ctx* ctx, const paro_op* a, const paro_op* b, int k, const double* cands, long long ld,
                       size_t min_keep, double drop_tol, double* lambdas, double* orbs, long long ldo, int* k_out,
                       double* defect) {
  return guarded(ctx, [&] {
    RitzInfo info;
    return rayleigh_ritz(ctx->c, a->o, b->o, k, cands, ld, min_keep, drop_tol, lambdas, orbs, ldo, k_out, defect,
                         &info);
  });
}

int paro_b_orthonormalize(paro_ctx* ctx, const paro_op* b, int k, const double* u, double drop_tol, double* q,
                          int* k_out, int* accepted) {
  return guarded(ctx, [&] { return b_orthonormalize(ctx->c, b->o, k, u, drop_tol, q, k_out, accepted); });
}

int paro_baseline_geneig(paro_ctx* ctx, const paro_op* a, const paro_op* b, int count, size_t max_iter,
                         unsigned long long seed, double* lambdas, double* vectors, long long ld, int* iterations) {
  return guarded(ctx, [&] {
    return baseline_geneig(ctx->c, a->o, b->o, count, max_iter, seed, lambdas, vectors, ld, iterations);
  });
}

int paro_dense_sym_geneig(paro_ctx* ctx, int m, const double* a, const double* b, double* vals, double* vecs) {
  return guarded(ctx, [&] { return dense_sym_geneig(ctx->c, m, a, b, vals, vecs); });
}

static paro_op* new_var_op(paro_ctx* ctx) {
  auto* op = new paro_op();
  op->owner = ctx;
  op->o.var = true;
  op->o.n = ctx->c.grid.n;
  PARO_CUDA(cudaMalloc(&op->o.coef, sizeof(double) * kSlots * op->o.n));
  op->o.owns = true;
  return op;
}

static int assemble_new(paro_ctx* ctx, const AssembleSpec& spec, bool try_uniform, paro_op** out) {
  ctx->c.check_grid();
  paro_op* op = new_var_op(ctx);
  try {
    assemble(ctx->c, spec, op->o);
    if (try_uniform) make_uniform_if_possible(ctx->c, op->o);
  } catch (...) {
    paro_op_destroy(op);
    throw;
  }
  *out = op;
  return kOk;
}

int paro_assemble_mass(paro_ctx* ctx, paro_op** out) {
  return guarded(ctx, [&] {
    AssembleSpec s;
    s.kind = kAsmMass;
    const int st = assemble_new(ctx, s, true, out);
    // a constant mass stencil lets integrate / norm_l2 / integrate_product run as nodal sums (fields.cu)
    const Op& m = (*out)->o;
    ctx->c.mass_state = m.var ? 2 : 1;
    if (!m.var)
      for (int o = 0; o < kSlots; ++o) ctx->c.mass_w[o] = m.w[o];
    return st;
  });
}

int paro_assemble_stiffness(paro_ctx* ctx, double scale, paro_op** out) {
  return guarded(ctx, [&] {
    AssembleSpec s;
    s.kind = kAsmStiffness;
    s.scale = scale;
    return assemble_new(ctx, s, true, out);
  });
}

int paro_assemble_vext(paro_ctx* ctx, int nnuc, const double* charges, const double* positions, double eps,
                       paro_op** out) {
  return guarded(ctx, [&] {
    AssembleSpec s;
    s.kind = eps == 0.0 ? kAsmCoulomb : kAsmSoftCoulomb;
    s.eps = eps;
    for (int k = 0; k < nnuc; ++k) {
      s.nuclei.push_back(charges[k]);
      for (int c = 0; c < 3; ++c) s.nuclei.push_back(positions[3 * k + c]);
    }
    return assemble_new(ctx, s, false, out);
  });
}

int paro_assemble_harmonic(paro_ctx* ctx, double c, paro_op** out) {
  return guarded(ctx, [&] {
    AssembleSpec s;
    s.kind = kAsmHarmonic;
    s.scale = c;
    return assemble_new(ctx, s, false, out);
  });
}

int paro_op_add_scaled(paro_ctx* ctx, paro_op* a, const paro_op* b, double s) {
  return guarded(ctx, [&] {
    add_scaled(ctx->c, a->o, b->o, s);
    return kOk;
  });
}

int paro_ks_form(paro_ctx* ctx, const paro_op* kinetic, const paro_op* vext, const double* rho, const double* vh,
                 int exchange_only, paro_op* out, long long* clamped) {
  return guarded(ctx, [&] {
    if (!out->o.var) throw ParoError(kInvalidArgument, "ks_form: output must be a variable operator");
    AssembleSpec s;
    s.kind = kAsmScf;
    s.rho = rho;
    s.vh = vh;
    s.exchange_only = exchange_only;
    s.kinetic = &kinetic->o;
    s.vext = &vext->o;
    long long cl = 0;
    s.clamped = &cl;  // counted while the quadrature table is built
    assemble(ctx->c, s, out->o);
    if (clamped) *clamped = cl;
    return kOk;
  });
}

int paro_ks_form_planes(paro_ctx* ctx, const paro_op* kinetic, const paro_op* vext, const double* rho,
                        const double* vh, int exchange_only, int z0, int z1, paro_op* out, long long* clamped) {
  return guarded(ctx, [&] {
    if (!out->o.var) throw ParoError(kInvalidArgument, "ks_form: output must be a variable operator");
    AssembleSpec s;
    s.kind = kAsmScf;
    s.rho = rho;
    s.vh = vh;
    s.exchange_only = exchange_only;
    s.kinetic = &kinetic->o;
    s.vext = &vext->o;
    s.z0 = z0;
    s.z1 = z1;
    long long cl = 0;
    s.clamped = &cl;
    assemble(ctx->c, s, out->o);
    if (clamped) *clamped = cl;
    return kOk;
  });
}

int paro_density(paro_ctx* ctx, int nocc, const double* u, long long ld, const double* occ, double* rho,
                 double* raw_integral) {
  return guarded(ctx, [&] {
    const double raw = density(ctx->c, nocc, u, ld, occ, rho);
    if (raw_integral) *raw_integral = raw;
    return kOk;
  });
}

int paro_density_rows(paro_ctx* ctx, int nocc, const double* u, long long ld, const double* occ, long long r0,
                      long long r1, double* rho) {
  return guarded(ctx, [&] {
    density_rows(ctx->c, nocc, u, ld, occ, r0, r1, rho);
    return kOk;
  });
}

int paro_density_normalize(paro_ctx* ctx, double total_occ, double* rho, double* raw_integral) {
  return guarded(ctx, [&] {
    const double raw = density_normalize(ctx->c, total_occ, rho);
    if (raw_integral) *raw_integral = raw;
    return kOk;
  });
}

int paro_mix_density(paro_ctx* ctx, const double* rho_in, const double* rho_out, double alpha, double* out) {
  return guarded(ctx, [&] {
    mix(ctx->c, rho_in, rho_out, alpha, out);
    return kOk;
  });
}

int paro_integrate(paro_ctx* ctx, const double* f, double* out) {
  return guarded(ctx, [&] {
    *out = cell_reduce(ctx->c, kCellIntegrate, f, nullptr, 0);
    return kOk;
  });
}

int paro_norm_l2(paro_ctx* ctx, const double* f, double* out) {
  return guarded(ctx, [&] {
    *out = norm_l2(ctx->c, f);
    return kOk;
  });
}

int paro_integrate_product(paro_ctx* ctx, const double* u, const double* v, double* out) {
  return guarded(ctx, [&] {
    *out = cell_reduce(ctx->c, kCellProduct, u, v, 0);
    return kOk;
  });
}

int paro_rho_residual(paro_ctx* ctx, const double* rho_out, const double* rho_in, double* scratch, double* out) {
  return guarded(ctx, [&] {
    diff(ctx->c, rho_out, rho_in, scratch);
    *out = norm_l2(ctx->c, scratch);
    return kOk;
  });
}

int paro_estimate_eta(paro_ctx* ctx, int N, const double* U, long long ld, const double* lambdas, double diffusion,
                      int reaction, double c, int nnuc, const double* charges, const double* positions, double eps,
                      const double* rho, const double* vh, int exchange_only, double* eta, double* eta_total) {
  return guarded(ctx, [&] {
    if (!eta_total || !lambdas || !U) throw ParoError(kInvalidArgument, "estimate: null argument");
    if (reaction < kEstKs || reaction > kEstWell) throw ParoError(kInvalidArgument, "estimate: unknown reaction");
    EstimateSpec s;
    s.kind = reaction;
    s.diffusion = diffusion;
    s.c = c;
    s.eps = eps;
    s.rho = rho;
    s.vh = vh;
    s.exchange_only = exchange_only;
    s.lambdas = lambdas;
    for (int k = 0; k < nnuc; ++k) {
      s.nuclei.push_back(charges[k]);
      for (int d = 0; d < 3; ++d) s.nuclei.push_back(positions[3 * k + d]);
    }
    *eta_total = estimate_eta(ctx->c, s, N, U, ld, eta);
    return kOk;
  });
}

int paro_total_energy(paro_ctx* ctx, int n_lambdas, const double* lambdas, int nocc, const double* occ,
                      const double* rho, const double* vh, int exchange_only, int nnuc, const double* charges,
                      const double* positions, double* e_out) {
  return guarded(ctx, [&] {
    std::vector<double> nuc;
    for (int k = 0; k < nnuc; ++k) {
      nuc.push_back(charges[k]);
      for (int c = 0; c < 3; ++c) nuc.push_back(positions[3 * k + c]);
    }
    *e_out = total_energy(ctx->c, n_lambdas, lambdas, nocc, occ, rho, vh, exchange_only, nnuc, nuc.data());
    return kOk;
  });
}

int paro_energy_xc_layers(paro_ctx* ctx, const double* rho, int exchange_only, int k0, int k1, double* out) {
  return guarded(ctx, [&] {
    *out = energy_xc_term(ctx->c, rho, exchange_only, k0, k1);
    return kOk;
  });
}

int paro_total_energy_with_xc(paro_ctx* ctx, int n_lambdas, const double* lambdas, int nocc, const double* occ,
                              const double* rho, const double* vh, int nnuc, const double* charges,
                              const double* positions, double xc_term, double* e_out) {
  return guarded(ctx, [&] {
    std::vector<double> nuc;
    for (int k = 0; k < nnuc; ++k) {
      nuc.push_back(charges[k]);
      for (int c = 0; c < 3; ++c) nuc.push_back(positions[3 * k + c]);
    }
    *e_out = total_energy(ctx->c, n_lambdas, lambdas, nocc, occ, rho, vh, 0, nnuc, nuc.data(), &xc_term);
    return kOk;
  });
}

int paro_fix_sign(paro_ctx* ctx, int k, double* v, long long ld) {
  return guarded(ctx, [&] {
    fix_sign_columns(ctx->c, v, ld, k);
    return kOk;
  });
}

// ------------------------------------------------ run artifacts
// Mesh::dump (mesh.cpp:198-217) of the uniform Kuhn box mesh create_box_mesh
// builds (mesh.cpp:411-478): "3 nv ne", vertices "%.17g %.17g %.17g" in vertex
// id order (k(s+1)+j)(s+1)+i, then one line per tetrahedron in the reference's
// element order: four vertex ids, the refinement-edge index 2 and type 0.
int paro_mesh_dump(int subdivisions, double lo, double hi, const char* path) {
  return guarded(nullptr, [&] {
    const int n = subdivisions;
    if (n < 1) throw ParoError(kInvalidArgument, "create_box_mesh: subdivisions must be >= 1");
    if (!(hi - lo > 0.0)) throw ParoError(kInvalidArgument, "create_box_mesh: box has non-positive edge length");
    FILE* f = std::fopen(path, "wb");
    if (!f) throw ParoError(kInvalidArgument, std::string("mesh dump: cannot open ") + path);
    std::vector<char> buf(1 << 22);
    size_t used = 0;
    auto flush = [&] {
      if (used && std::fwrite(buf.data(), 1, used, f) != used) {
        std::fclose(f);
        throw ParoError(kError, "mesh dump: write failed");
      }
      used = 0;
    };
    auto put = [&](const char* p, size_t len) {
      if (used + len > buf.size()) flush();
      std::memcpy(buf.data() + used, p, len);
      used += len;
    };
    const long long nv = static_cast<long long>(n + 1) * (n + 1) * (n + 1);
    const long long ne = 6LL * n * n * n;
    char line[160];
    put(line, static_cast<size_t>(std::snprintf(line, sizeof line, "3 %lld %lld\n", nv, ne)));
    std::vector<std::string> c(n + 1);
    for (int i = 0; i <= n; ++i) {
      std::snprintf(line, sizeof line, "%.17g", lo + (hi - lo) * i / n);
      c[i] = line;
    }
    for (int k = 0; k <= n; ++k)
      for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n; ++i) {
          const std::string l = c[i] + ' ' + c[j] + ' ' + c[k] + '\n';
          put(l.data(), l.size());
        }
    auto vid = [&](int i, int j, int k) {
      return static_cast<unsigned>((k * (n + 1) + j) * (n + 1) + i);
    };
    auto utoa = [](unsigned v, char* out) {
      char tmp[12];
      int len = 0;
      do {
        tmp[len++] = static_cast<char>('0' + v % 10);
        v /= 10;
      } while (v);
      for (int q = 0; q < len; ++q) out[q] = tmp[len - 1 - q];
      return len;
    };
    constexpr int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i)
          for (const auto& perm : perms) {
            int cc[3] = {i, j, k};
            int len = utoa(vid(cc[0], cc[1], cc[2]), line);
            for (int step = 0; step < 3; ++step) {
              cc[perm[step]] += 1;
              line[len++] = ' ';
              len += utoa(vid(cc[0], cc[1], cc[2]), line + len);
            }
            std::memcpy(line + len, " 2 0\n", 5);
            put(line, static_cast<size_t>(len + 5));
          }
    flush();
    if (std::fclose(f) != 0) throw ParoError(kError, "mesh dump: close failed");
    return kOk;
  });
}

// ------------------------------------------------ general CSR operators
int paro_csr_create(paro_ctx* ctx, size_t n, const size_t* rows, const uint32_t* cols, const double* vals,
                    paro_csr** out) {
  return guarded(ctx, [&] {
    if (!rows || !cols || !vals || !out) throw ParoError(kInvalidArgument, "csr_create: null argument");
    auto* h = new paro_csr();
    try {
      csr_create(ctx->c, static_cast<long long>(n), rows, cols, vals, h->a);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return kOk;
  });
}

int paro_csr_destroy(paro_csr* a) {
  delete a;
  return kOk;
}

int paro_csr_add_scaled(paro_ctx* ctx, paro_csr* a, const paro_csr* b, double s) {
  return guarded(ctx, [&] {
    csr_add_scaled(ctx->c, a->a, b->a, s);
    return kOk;
  });
}

int paro_csr_apply(paro_ctx* ctx, const paro_csr* a, int k, const double* x, long long ld, double* y) {
  return guarded(ctx, [&] {
    csr_apply(ctx->c, a->a, k, x, ld, y);
    PARO_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return kOk;
  });
}

int paro_csr_cg_solve(paro_ctx* ctx, const paro_csr* a, int k, const double* b, const double* x0, long long ld,
                      double tol, size_t max_iter, int throw_on_max, double* x, size_t* iters, double* resid) {
  return guarded(ctx, [&] {
    SolveReport rep;
    const int st = csr_cg_solve(ctx->c, a->a, k, b, x0, ld, tol, max_iter, throw_on_max != 0, x, &rep);
    fill_report(rep, iters, resid);
    return st;
  });
}

int paro_csr_source_solve_step(paro_ctx* ctx, const paro_csr* a, const paro_csr* b, int k, const double* u,
                               long long ld, const double* lambdas, double tol, size_t max_iter, double sigma,
                               double* out, size_t* iters, double* resid) {
  return guarded(ctx, [&] {
    SolveReport rep;
    const int st = csr_source_solve(ctx->c, a->a, b->a, sigma, k, u, ld, lambdas, tol, max_iter, out, &rep);
    fill_report(rep, iters, resid);
    return st;
  });
}

}  // extern "C"
