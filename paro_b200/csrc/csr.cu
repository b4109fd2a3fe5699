// General CSR operators: batched SpMV and Jacobi-PCG for
// symmetric matrices that are not the uniform-mesh stencil (adapted meshes:
// fem.cpp:109-183 patterns after Mesh::bisect), with the reference's
// semantics (SparseOperator::matvec linalg.cpp:88-94, add_scaled :120-125,
// diagonal :102-110, cg_solve :143-223, source_solve_step paro.cpp:81-119).
//
// Layout: inside the solver the K columns are interleaved, v[row * K + c],
// so one matrix row is read once for all K columns and the K threads of a
// row load x[col * K + c] as one contiguous segment. Inputs and outputs stay
// the reference's column vectors ([K][n], stride ld) and are transposed at
// the boundary with shared-memory tiles. Row sums run in ascending column
// order without FMA contraction (bit-identical to matvec); per-column dot
// products are fixed-order block partials + the shared finalize kernels
// (pcg_fin.cuh), so every column's scalars are deterministic.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "csr.hpp"
#include "pcg_fin.cuh"

namespace paro_b200 {

namespace {

constexpr int kCT = 256;          // threads per CTA (K columns x R rows)
constexpr int kCBlocks = 148 * 4;  // CTAs of the row loops = partial slots per column
constexpr int kMaxK = kCT;        // at least one row per CTA

struct CsrView {
  long long n;
  const long long* rows;
  const int* cols;
  const double* vals;
};

// dst (c x r, row stride ldd) = src^T (r x c, row stride lds); the long
// dimension takes blockIdx.x (gridDim.y is limited to 65535)
__global__ void transpose_kernel(const double* __restrict__ src, long long lds, long long r, long long c,
                                 double* __restrict__ dst, long long ldd, int r_on_x) {
  __shared__ double tile[32][33];
  const long long br = r_on_x ? blockIdx.x : blockIdx.y, bc = r_on_x ? blockIdx.y : blockIdx.x;
  const long long r0 = br * 32, c0 = bc * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const long long rr = r0 + j, cc = c0 + threadIdx.x;
    if (rr < r && cc < c) tile[j][threadIdx.x] = src[rr * lds + cc];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const long long cc = c0 + j, rr = r0 + threadIdx.x;
    if (rr < r && cc < c) dst[cc * ldd + rr] = tile[threadIdx.x][j];
  }
}

// [K][n] (stride ld) -> interleaved [n][K]
void to_interleaved(cudaStream_t st, const double* src, long long ld, int K, long long n, double* dst) {
  dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((K + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, ld, K, n, dst, K, 0);
}
// interleaved [n][K] -> [K][n] (stride ld)
void from_interleaved(cudaStream_t st, const double* src, int K, long long n, double* dst, long long ld) {
  dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((K + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, K, n, K, dst, ld, 1);
}

// row sum of row `row`, column c, ascending column order, no contraction
__device__ __forceinline__ double row_sum(const CsrView& A, long long row, const double* __restrict__ X, int K,
                                          int c) {
  double s = 0.0;
  for (long long k = A.rows[row]; k < A.rows[row + 1]; ++k)
    s = __dadd_rn(s, __dmul_rn(A.vals[k], X[static_cast<long long>(A.cols[k]) * K + c]));
  return s;
}

enum SpmvMode { kSpApply = 0, kSpDot = 1, kSpSetup = 2 };

// Apply: Y = A X. Dot: Y = A X, partial X.Y. Setup: Y = B - A X (r0), partials B.B, r.(invd r), r.r.
template <int MODE>
__global__ void __launch_bounds__(kCT) spmv_kernel(CsrView A, int K, const double* __restrict__ X, double* __restrict__ Y,
                                                   const double* __restrict__ Bv, const double* __restrict__ invd,
                                                   const CgColumn* __restrict__ colst, double* __restrict__ partials) {
  constexpr int NQ = MODE == kSpSetup ? 3 : 1;
  __shared__ unsigned char act[kMaxK];
  __shared__ double red[kCT * NQ];
  const int tid = threadIdx.x;
  const int R = kCT / K;
  const int lr = tid / K, c = tid % K;
  const bool valid = lr < R;
  if (tid < K) act[tid] = colst == nullptr || colst[tid].active != 0;
  __syncthreads();
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  if (valid && act[c]) {
    for (long long row = static_cast<long long>(blockIdx.x) * R + lr; row < A.n;
         row += static_cast<long long>(gridDim.x) * R) {
      const double s = row_sum(A, row, X, K, c);
      const long long i = row * K + c;
      if (MODE == kSpApply) {
        Y[i] = s;
      } else if (MODE == kSpDot) {
        Y[i] = s;
        acc[0] += X[i] * s;  // p'q (linalg.cpp:198)
      } else {
        const double b = Bv[i];
        const double r = __dsub_rn(b, s);  // r = b - A x0 (linalg.cpp:184-185)
        Y[i] = r;
        acc[0] += b * b;
        acc[1] += r * __dmul_rn(invd[row], r);
        acc[2] += r * r;
      }
    }
  }
  if constexpr (MODE == kSpApply) return;
#pragma unroll
  for (int q = 0; q < NQ; ++q) red[q * kCT + tid] = valid ? acc[q] : 0.0;
  __syncthreads();
  if (tid < K && act[tid]) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double s = 0.0;
      for (int l = 0; l < R; ++l) s += red[q * kCT + l * K + tid];  // fixed order over the CTA's rows
      partials[(static_cast<long long>(tid) * 3 + q) * gridDim.x + blockIdx.x] = s;
    }
  }
}

// x += alpha p ; r -= alpha q ; z = invd r ; partials r.z, r.r  (linalg.cpp:202-207)
__global__ void __launch_bounds__(kCT) update_kernel(long long n, int K, double* __restrict__ x, double* __restrict__ r,
                                                     const double* __restrict__ p, const double* __restrict__ q,
                                                     const double* __restrict__ invd, const CgColumn* __restrict__ colst,
                                                     double* __restrict__ partials) {
  __shared__ unsigned char act[kMaxK];
  __shared__ double alpha[kMaxK];
  __shared__ double red[2 * kCT];
  const int tid = threadIdx.x;
  const int R = kCT / K;
  const int lr = tid / K, c = tid % K;
  const bool valid = lr < R;
  if (tid < K) {
    act[tid] = colst[tid].active != 0;
    alpha[tid] = colst[tid].alpha;
  }
  __syncthreads();
  double a0 = 0.0, a1 = 0.0;
  if (valid && act[c]) {
    const double al = alpha[c];
    for (long long row = static_cast<long long>(blockIdx.x) * R + lr; row < n;
         row += static_cast<long long>(gridDim.x) * R) {
      const long long i = row * K + c;
      x[i] = __dadd_rn(x[i], __dmul_rn(al, p[i]));
      const double rn = __dsub_rn(r[i], __dmul_rn(al, q[i]));
      r[i] = rn;
      a0 += rn * __dmul_rn(invd[row], rn);
      a1 += rn * rn;
    }
  }
  red[tid] = valid ? a0 : 0.0;
  red[kCT + tid] = valid ? a1 : 0.0;
  __syncthreads();
  if (tid < K && act[tid]) {
    double s0 = 0.0, s1 = 0.0;
    for (int l = 0; l < R; ++l) {
      s0 += red[l * K + tid];
      s1 += red[kCT + l * K + tid];
    }
    partials[(static_cast<long long>(tid) * 3 + 0) * gridDim.x + blockIdx.x] = s0;
    partials[(static_cast<long long>(tid) * 3 + 1) * gridDim.x + blockIdx.x] = s1;
  }
}

// p = z + beta p, z = invd r (p = z on the first iteration)  (linalg.cpp:179, 210)
__global__ void __launch_bounds__(kCT) direction_kernel(long long n, int K, const double* __restrict__ r,
                                                        double* __restrict__ p, const double* __restrict__ invd,
                                                        const CgColumn* __restrict__ colst) {
  __shared__ unsigned char act[kMaxK], first[kMaxK];
  __shared__ double beta[kMaxK];
  const int tid = threadIdx.x;
  const int R = kCT / K;
  const int lr = tid / K, c = tid % K;
  if (tid < K) {
    act[tid] = colst[tid].active != 0;
    first[tid] = colst[tid].first != 0;
    beta[tid] = colst[tid].beta;
  }
  __syncthreads();
  if (lr >= R || !act[c]) return;
  const double b = beta[c];
  const bool f = first[c];
  for (long long row = static_cast<long long>(blockIdx.x) * R + lr; row < n;
       row += static_cast<long long>(gridDim.x) * R) {
    const long long i = row * K + c;
    const double z = __dmul_rn(invd[row], r[i]);
    p[i] = f ? z : __dadd_rn(z, __dmul_rn(b, p[i]));
  }
}

// inv_diag from the stored diagonal (diagonal(), linalg.cpp:102-110); a
// non-positive (or missing) diagonal entry sets *bad (linalg.cpp:165-167)
__global__ void csr_invd_kernel(CsrView A, double* invd, int* bad) {
  for (long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; row < A.n;
       row += static_cast<long long>(gridDim.x) * blockDim.x) {
    double d = 0.0;
    for (long long k = A.rows[row]; k < A.rows[row + 1]; ++k)
      if (A.cols[k] == row) d = A.vals[k];
    if (d <= 0.0) *bad = 1;
    invd[row] = 1.0 / d;
  }
}

// a = a + s b, elementwise on identical patterns: fl(a + fl(s b))
__global__ void axpy_vals_kernel(long long nnz, double* a, const double* b, double s) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    a[k] = __dadd_rn(a[k], __dmul_rn(s, b[k]));
}

// column scale: v[:, c] *= s[c] (interleaved)
__global__ void scale_cols_kernel(long long n, int K, double* v, const double* s) {
  const long long total = n * K;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    v[i] = __dmul_rn(v[i], s[i % K]);
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

// X[:, c] = Y[:, c] where mask[c] (interleaved)
__global__ void select_cols_kernel(long long n, int K, double* X, const double* Y, const int* mask) {
  const long long total = n * K;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    if (mask[i % K]) X[i] = Y[i];
}

CsrView view(const CsrOp& a) { return {a.n, a.rows, a.cols, a.vals}; }

void check_k(int K) {
  if (K < 1 || K > kMaxK) throw ParoError(kCapacity, "csr: 1..256 columns per batch");
}

template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  PARO_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

// Batched Jacobi-PCG on interleaved vectors. B: rhs [n][K] (interleaved), X:
// x0 on entry, solution on exit. cols (host) carry tol / max_iter per column.
void csr_pcg(Ctx& ctx, const CsrOp& A, int K, const double* B, double* X, std::vector<CgColumn>& cols,
             bool abort_on_not_spd) {
  cudaStream_t st = ctx.stream;
  const long long n = A.n;
  double* base = ctx.csr_ws.get<double>(static_cast<size_t>(3) * n * K + n);
  double* r = base;
  double* p = r + n * K;
  double* q = p + n * K;
  double* invd = q + n * K;
  CgColumn* dcols = ctx.cols.get<CgColumn>(K);
  double* partials = ctx.partials.get<double>(static_cast<size_t>(K) * 3 * kCBlocks);
  int* flag = ctx.flag.get<int>(3 + K);
  const CsrView V = view(A);
  PARO_CUDA(cudaMemcpyAsync(dcols, cols.data(), sizeof(CgColumn) * K, cudaMemcpyHostToDevice, st));
  set_int_kernel<<<1, 1, 0, st>>>(flag, 0);
  set_int_kernel<<<1, 1, 0, st>>>(flag + 1, 0);
  set_int_kernel<<<1, 1, 0, st>>>(flag + 2, abort_on_not_spd ? 1 : 0);
  csr_invd_kernel<<<148 * 8, 256, 0, st>>>(V, invd, flag);
  spmv_kernel<kSpSetup><<<kCBlocks, kCT, 0, st>>>(V, K, X, r, B, invd, dcols, partials);
  fin_kernel<<<K, kFinThreads, 0, st>>>(kFinSetup, dcols, partials, kCBlocks, flag);
  ctx.launches += 6;
  PARO_CUDA(cudaGetLastError());

  unsigned long long max_iter = 0;
  for (const auto& c : cols) max_iter = std::max(max_iter, c.max_iter);
  const int chunk = 8;
  cudaEvent_t ev;
  PARO_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  volatile int* hcount = ctx.pinned_count;
  unsigned long long launched = 0;
  for (;;) {
    count_active_kernel<<<1, 256, 0, st>>>(dcols, K, ctx.pinned_count_dev);
    PARO_CUDA(cudaEventRecord(ev, st));
    PARO_CUDA(cudaEventSynchronize(ev));
    if (*hcount == 0 || launched >= max_iter) break;
    for (int it = 0; it < chunk; ++it) {
      direction_kernel<<<kCBlocks, kCT, 0, st>>>(n, K, r, p, invd, dcols);
      spmv_kernel<kSpDot><<<kCBlocks, kCT, 0, st>>>(V, K, p, q, nullptr, nullptr, dcols, partials);
      fin_kernel<<<K, kFinThreads, 0, st>>>(kFinK1, dcols, partials, kCBlocks, flag);
      update_kernel<<<kCBlocks, kCT, 0, st>>>(n, K, X, r, p, q, invd, dcols, partials);
      fin_kernel<<<K, kFinThreads, 0, st>>>(kFinK2, dcols, partials, kCBlocks, flag);
    }
    PARO_CUDA(cudaGetLastError());
    launched += chunk;
    ctx.launches += 5ull * chunk + 1;
  }
  PARO_CUDA(cudaEventDestroy(ev));
  PARO_CUDA(cudaMemcpy(cols.data(), dcols, sizeof(CgColumn) * K, cudaMemcpyDeviceToHost));
}

CgColumn make_col(double tol, unsigned long long max_iter) {
  CgColumn c{};
  c.tol = tol;
  c.max_iter = max_iter;
  c.active = 1;
  return c;
}

// solution back to the caller's columns; bnorm == 0 columns are x = 0 (linalg.cpp:158-162)
void write_back(Ctx& ctx, const double* Xil, int K, long long n, const std::vector<CgColumn>& cols, double* x,
                long long ld) {
  from_interleaved(ctx.stream, Xil, K, n, x, ld);
  for (int c = 0; c < K; ++c)
    if (cols[c].first == 2) PARO_CUDA(cudaMemsetAsync(x + c * ld, 0, sizeof(double) * n, ctx.stream));
  PARO_CUDA(cudaGetLastError());
}

}  // namespace

CsrOp::~CsrOp() {
  if (rows) cudaFree(rows);
  if (cols) cudaFree(cols);
  if (vals) cudaFree(vals);
}

void csr_create(Ctx& ctx, long long n, const size_t* rows, const uint32_t* cols, const double* vals, CsrOp& out) {
  if (n <= 0) throw ParoError(kInvalidArgument, "csr: empty operator");
  if (n > (1ll << 31) - 1) throw ParoError(kCapacity, "csr: more than 2^31 rows");
  if (rows[0] != 0) throw ParoError(kInvalidArgument, "csr: row offsets must start at 0");
  const long long nnz = static_cast<long long>(rows[n]);
  out.h_rows.resize(n + 1);
  out.h_cols.resize(nnz);
  for (long long i = 0; i <= n; ++i) {
    out.h_rows[i] = static_cast<long long>(rows[i]);
    if (i > 0 && out.h_rows[i] < out.h_rows[i - 1]) throw ParoError(kInvalidArgument, "csr: row offsets decrease");
  }
  for (long long i = 0; i < n; ++i)
    for (long long k = out.h_rows[i]; k < out.h_rows[i + 1]; ++k) {
      if (cols[k] >= static_cast<uint64_t>(n)) throw ParoError(kInvalidArgument, "csr: column out of range");
      if (k > out.h_rows[i] && cols[k] <= cols[k - 1])
        throw ParoError(kInvalidArgument, "csr: columns must ascend within a row");
      out.h_cols[k] = static_cast<int>(cols[k]);
    }
  out.n = n;
  out.nnz = nnz;
  out.rows = dalloc<long long>(n + 1);
  out.cols = dalloc<int>(nnz);
  out.vals = dalloc<double>(nnz);
  PARO_CUDA(cudaMemcpyAsync(out.rows, out.h_rows.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice,
                            ctx.stream));
  PARO_CUDA(cudaMemcpyAsync(out.cols, out.h_cols.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, ctx.stream));
  PARO_CUDA(cudaMemcpyAsync(out.vals, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx.stream));
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
}

void csr_add_scaled(Ctx& ctx, CsrOp& a, const CsrOp& b, double s) {
  if (a.n != b.n || a.h_rows != b.h_rows || a.h_cols != b.h_cols)
    throw ParoError(kInvalidArgument, "add_scaled: sparsity structures differ");
  axpy_vals_kernel<<<148 * 8, 256, 0, ctx.stream>>>(a.nnz, a.vals, b.vals, s);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

void csr_apply(Ctx& ctx, const CsrOp& a, int K, const double* x, long long ld, double* y) {
  check_k(K);
  const long long n = a.n;
  double* base = ctx.csr_ws.get<double>(static_cast<size_t>(2) * n * K);
  double* xi = base;
  double* yi = base + n * K;
  to_interleaved(ctx.stream, x, ld, K, n, xi);
  spmv_kernel<kSpApply><<<kCBlocks, kCT, 0, ctx.stream>>>(view(a), K, xi, yi, nullptr, nullptr, nullptr, nullptr);
  from_interleaved(ctx.stream, yi, K, n, y, ld);
  PARO_CUDA(cudaGetLastError());
  ctx.launches += 3;
}

int csr_cg_solve(Ctx& ctx, const CsrOp& a, int K, const double* rhs, const double* x0, long long ld, double tol,
                 unsigned long long max_iter, bool throw_on_max, double* x, SolveReport* rep) {
  check_k(K);
  const long long n = a.n;
  double* Bil = ctx.csr_io.get<double>(static_cast<size_t>(2) * n * K);
  double* Xil = Bil + n * K;
  to_interleaved(ctx.stream, rhs, ld, K, n, Bil);
  if (x0) to_interleaved(ctx.stream, x0, ld, K, n, Xil);
  else PARO_CUDA(cudaMemsetAsync(Xil, 0, sizeof(double) * n * K, ctx.stream));
  std::vector<CgColumn> cols(K);
  for (int c = 0; c < K; ++c) cols[c] = make_col(tol, max_iter);
  csr_pcg(ctx, a, K, Bil, Xil, cols, false);
  write_back(ctx, Xil, K, n, cols, x, ld);
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
  int status = kOk;
  if (rep) {
    rep->iterations.assign(K, 0);
    rep->residual.assign(K, 0.0);
    rep->status.assign(K, kOk);
  }
  for (int c = 0; c < K; ++c) {
    int s = cols[c].status;
    if (s == kIterationLimit && !throw_on_max) s = kOk;
    if (rep) {
      rep->iterations[c] = cols[c].it;
      rep->residual[c] = cols[c].bnorm > 0 ? cols[c].rnorm / cols[c].bnorm : 0.0;
      rep->status[c] = s;
    }
    if (s != kOk && status == kOk) {
      status = s;
      ctx.resid = cols[c].bnorm > 0 ? cols[c].rnorm / cols[c].bnorm : 0.0;
      ctx.err = s == kNotSpd ? "cg: operator not positive definite" : "cg: iteration limit reached";
    }
  }
  return status;
}

int csr_source_solve(Ctx& ctx, const CsrOp& a, const CsrOp& b, double sigma, int K, const double* u, long long ld,
                     const double* lambdas, double tol, unsigned long long max_iter, double* out,
                     SolveReport* rep) {
  check_k(K);
  const long long n = a.n;
  if (b.n != n) throw ParoError(kInvalidArgument, "source_solve_step: operator dimensions differ");
  // shifted = A + sigma B (paro.cpp:89-90), a device copy of A's values
  CsrOp shifted;
  shifted.n = a.n;
  shifted.nnz = a.nnz;
  shifted.h_rows = a.h_rows;
  shifted.h_cols = a.h_cols;
  shifted.rows = dalloc<long long>(n + 1);
  shifted.cols = dalloc<int>(a.nnz);
  shifted.vals = dalloc<double>(a.nnz);
  PARO_CUDA(cudaMemcpyAsync(shifted.rows, a.rows, sizeof(long long) * (n + 1), cudaMemcpyDeviceToDevice, ctx.stream));
  PARO_CUDA(cudaMemcpyAsync(shifted.cols, a.cols, sizeof(int) * a.nnz, cudaMemcpyDeviceToDevice, ctx.stream));
  PARO_CUDA(cudaMemcpyAsync(shifted.vals, a.vals, sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice, ctx.stream));
  if (sigma != 0.0) csr_add_scaled(ctx, shifted, b, sigma);
  // rhs_i = (lambda_i + sigma) B u_i (paro.cpp:96-98), x0 = u_i (paro.cpp:102)
  double* Bil = ctx.csr_io.get<double>(static_cast<size_t>(3) * n * K + K);
  double* Uil = Bil + n * K;
  double* Xil = Uil + n * K;
  double* dscale = Xil + n * K;
  std::vector<double> scale(K);
  for (int c = 0; c < K; ++c) scale[c] = lambdas[c] + sigma;
  PARO_CUDA(cudaMemcpyAsync(dscale, scale.data(), sizeof(double) * K, cudaMemcpyHostToDevice, ctx.stream));
  to_interleaved(ctx.stream, u, ld, K, n, Uil);
  spmv_kernel<kSpApply><<<kCBlocks, kCT, 0, ctx.stream>>>(view(b), K, Uil, Bil, nullptr, nullptr, nullptr, nullptr);
  scale_cols_kernel<<<148 * 8, 256, 0, ctx.stream>>>(n, K, Bil, dscale);
  PARO_CUDA(cudaMemcpyAsync(Xil, Uil, sizeof(double) * n * K, cudaMemcpyDeviceToDevice, ctx.stream));
  ctx.launches += 3;
  std::vector<CgColumn> cols(K);
  for (int c = 0; c < K; ++c) cols[c] = make_col(tol, max_iter);
  csr_pcg(ctx, shifted, K, Bil, Xil, cols, true);

  bool not_spd = false;
  for (int c = 0; c < K; ++c) not_spd |= cols[c].status == kNotSpd;
  if (rep) {
    rep->iterations.assign(K, 0);
    rep->residual.assign(K, 0.0);
    rep->status.assign(K, kOk);
    rep->first_status.assign(K, kOk);
  }
  if (not_spd) {  // the sigma policy restarts the whole step (paro.cpp:204-207)
    if (rep)
      for (int c = 0; c < K; ++c) {
        rep->iterations[c] = cols[c].it;
        if (cols[c].status == kNotSpd) rep->status[c] = rep->first_status[c] = kNotSpd;
      }
    ctx.err = "cg: operator not positive definite (p'Ap <= 0)";
    return kNotSpd;
  }
  // one retry from x0 = u at tol*100, max_iter*4 for the columns at the iteration limit (paro.cpp:105-109)
  std::vector<int> first_status(K), retry_status(K, kOk);
  std::vector<CgColumn> retry(K);
  bool any_retry = false;
  for (int c = 0; c < K; ++c) {
    first_status[c] = cols[c].status;
    if (cols[c].status == kIterationLimit) {
      retry[c] = make_col(tol * 100.0, max_iter * 4);
      any_retry = true;
    } else {
      retry[c] = cols[c];
      retry[c].active = 0;
    }
  }
  if (any_retry) {
    // the retried columns restart from x0 = u; their results replace the first attempt's
    double* Xr = ctx.csr_ws2.get<double>(static_cast<size_t>(n) * K);
    PARO_CUDA(cudaMemcpyAsync(Xr, Uil, sizeof(double) * n * K, cudaMemcpyDeviceToDevice, ctx.stream));
    csr_pcg(ctx, shifted, K, Bil, Xr, retry, false);
    std::vector<int> mask(K);
    for (int c = 0; c < K; ++c) mask[c] = first_status[c] == kIterationLimit;
    int* dmask = ctx.flag.get<int>(3 + K) + 3;
    PARO_CUDA(cudaMemcpyAsync(dmask, mask.data(), sizeof(int) * K, cudaMemcpyHostToDevice, ctx.stream));
    select_cols_kernel<<<148 * 8, 256, 0, ctx.stream>>>(n, K, Xil, Xr, dmask);
    PARO_CUDA(cudaGetLastError());
    ++ctx.launches;
    for (int c = 0; c < K; ++c)
      if (mask[c]) retry_status[c] = retry[c].status;
  }
  write_back(ctx, Xil, K, n, cols, out, ld);
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
  if (rep) {
    rep->first_status = first_status;
    for (int c = 0; c < K; ++c) {
      const CgColumn& f = first_status[c] == kIterationLimit ? retry[c] : cols[c];
      rep->iterations[c] = f.it;
      rep->residual[c] = f.bnorm > 0 ? f.rnorm / f.bnorm : 0.0;
      rep->status[c] = first_status[c] == kIterationLimit ? retry_status[c] : first_status[c];
    }
  }
  // exception order of the serial reference loop (paro.cpp:105-117)
  for (int c = 0; c < K; ++c)
    if (first_status[c] == kIterationLimit && retry_status[c] != kOk) {
      const CgColumn& f = retry[c];
      ctx.resid = f.bnorm > 0 ? f.rnorm / f.bnorm : 0.0;
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

}  // namespace paro_b200
