// Step 4 on the device: rayleigh_ritz (proj/src/paro.cpp:121-177).
//
//   W = B U, G1 = U^T W            -> ordered Cholesky with the MGS drop rule
//   Q1 = U C1                       (C1 = L1^{-T} on the accepted candidates)
//   W = B Q1, G2 = Q1^T W           -> C2 = L2^{-T}, Bt = L2^{-1} G2 L2^{-T}
//   W = A Q1, GA = Q1^T W           -> At = C2^T GA C2, dense_sym_geneig(At, Bt)
//   V = Q1 (C2 X), fix_sign, certificate max|V^T B V - I| <= 1e-8
//
// i.e. CholQR2 in place of two-pass MGS (identical in exact arithmetic,
// SURVEY.md §8a), with the stencil applies on the plane-marching kernels, the
// tall-skinny Grams / rotations as FP64 DGEMMs and the K x K work in
// single-warp kernels (dense.cu). The tall-skinny Grams and rotations are
// hand-written DMMA kernels (this file, step4.cu); no library GEMM.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "dense.hpp"
#include "ritz.hpp"
#include "solver.hpp"
#include "step4.hpp"

namespace paro_b200 {

namespace {

// ---------------------------------------------------------------------------
// Symmetric tall-skinny Gram G = X^T Y (n x k operands, k <= kGMaxK; X^T Y is
// symmetric because Y = B X or A X with B, A symmetric). cuBLAS parallelises
// one DGEMM only over the k x k output (n ~ 10^7 is the reduction), so: split
// n into P row chunks, one CTA per chunk computing the upper block triangle of
// its partial on the FP64 tensor cores (mma.sync m8n8k4 f64, 8x8 tiles, 4
// warps x <= 15 tiles), rows staged in shared memory by cp.async double
// buffering; then add the partials in a fixed order and mirror the upper
// triangle (deterministic, exactly symmetric).
constexpr int kGB = 8;                    // tile edge
constexpr int kGR = 32;                   // rows per stage
constexpr int kGMaxK = 80;                // columns (10 tile blocks -> 55 upper tiles)
constexpr int kGRow = 96;                 // staged row stride (room for the column swizzle)
constexpr int kGThreads = 128;            // 4 warps
constexpr int kGPairsMax = 55;

__device__ __forceinline__ void gcp8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(static_cast<unsigned>(
                   __cvta_generic_to_shared(dst))),
               "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}

// staged element (row, col) lives at [row][col ^ gswz(row)]: a warp copying 32
// rows of one column hits 16 distinct bank pairs, and an m8n8k4 operand load
// (4 consecutive rows x 8 consecutive columns) hits 32 distinct ones
__device__ __forceinline__ int gswz(int row) { return ((row & 3) << 3) ^ (((row >> 2) & 3) << 1); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// upper-triangular tile index of block pair (bi <= bj) among nb blocks
__device__ __forceinline__ int gpair(int bi, int bj, int nb) { return bi * nb - bi * (bi - 1) / 2 + (bj - bi); }

__global__ void __launch_bounds__(kGThreads) gram_sym_kernel(const double* __restrict__ X, long long ldx,
                                                             const double* __restrict__ Y, long long ldy, int k,
                                                             long long n, long long chunk, double* __restrict__ part) {
  extern __shared__ __align__(16) double gsm[];
  auto xs = reinterpret_cast<double(*)[kGR][kGRow]>(gsm);
  auto ys = reinterpret_cast<double(*)[kGR][kGRow]>(gsm + 2 * kGR * kGRow);
  const long long r0 = blockIdx.x * chunk;
  const long long r1 = min(n, r0 + chunk);
  const int nb = (k + kGB - 1) / kGB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // warp w's tile set: row blocks R x column blocks C, upper triangle only.
  // h = ceil(nb/2): w0 [0,h)x[0,h), w1 [0,h)x[h,h+m), w2 [0,h)x[h+m,nb), w3 [h,nb)x[h,nb)
  const int h = (nb + 1) / 2, m = (nb - h) / 2;
  int rlo, rhi, clo, chi;
  switch (warp) {
    case 0: rlo = 0, rhi = h, clo = 0, chi = h; break;
    case 1: rlo = 0, rhi = h, clo = h, chi = h + m; break;
    case 2: rlo = 0, rhi = h, clo = h + m, chi = nb; break;
    default: rlo = h, rhi = nb, clo = h, chi = nb; break;
  }
  constexpr int kMaxB = 5;
  double acc[kMaxB][kMaxB][2];
#pragma unroll
  for (int i = 0; i < kMaxB; ++i)
#pragma unroll
    for (int j = 0; j < kMaxB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // loads: thread copies row (tid % kGR) of columns tid / kGR + 4 q
  constexpr int kCStep = kGThreads / kGR;
  const int lrow = threadIdx.x % kGR, lcol = threadIdx.x / kGR;
  const int lsw = gswz(lrow);
  const double* xb = X + lcol * ldx + lrow;
  const double* yb = Y + lcol * ldy + lrow;
  auto issue = [&](int st, long long rb) {
    const bool rin = rb + lrow < r1;
    const double* px = xb + rb;
    const double* py = yb + rb;
#pragma unroll
    for (int q = 0; q < kGMaxK / kCStep; ++q) {
      const int col = lcol + q * kCStep;
      const bool v = rin && col < k;
      const int sc = col ^ lsw;
      gcp8(&xs[st][lrow][sc], v ? px : X, v);
      gcp8(&ys[st][lrow][sc], v ? py : Y, v);
      px += kCStep * ldx;
      py += kCStep * ldy;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  const int fr = lane & 3, fc = lane >> 2;  // fragment row (k) and column (tile row / col)
  int st = 0;
  issue(0, r0);
  for (long long rb = r0; rb < r1; rb += kGR, st ^= 1) {
    if (rb + kGR < r1) {
      issue(st ^ 1, rb + kGR);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
#pragma unroll 2
    for (int k0 = 0; k0 < kGR; k0 += 4) {
      const int row = k0 + fr;
      const int sw = gswz(row);
      double a[kMaxB], b[kMaxB];
#pragma unroll
      for (int i = 0; i < kMaxB; ++i) {
        a[i] = rlo + i < rhi ? xs[st][row][((rlo + i) * kGB + fc) ^ sw] : 0.0;
        b[i] = clo + i < chi ? ys[st][row][((clo + i) * kGB + fc) ^ sw] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kMaxB; ++i)
#pragma unroll
        for (int j = 0; j < kMaxB; ++j)
          if (rlo + i < rhi && clo + j < chi && clo + j >= rlo + i) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  // tile (bi, bj): lane holds C[fc][2 fr + {0,1}]
#pragma unroll
  for (int i = 0; i < kMaxB; ++i)
#pragma unroll
    for (int j = 0; j < kMaxB; ++j) {
      const int bi = rlo + i, bj = clo + j;
      if (bi < rhi && bj < chi && bj >= bi) {
        double* o = part + (static_cast<long long>(blockIdx.x) * kGPairsMax + gpair(bi, bj, nb)) * (kGB * kGB);
        o[fc * kGB + 2 * fr] = acc[i][j][0];
        o[fc * kGB + 2 * fr + 1] = acc[i][j][1];
      }
    }
}

// The same split-K upper-triangle Gram with the tile sets fixed at compile
// time (nb = number of 8-column blocks): every DMMA, fragment load and
// accumulator is unconditional, which removes the per-tile predicates that
// cost ~16 instructions per DMMA in the generic kernel. Same staging, tile
// assignment, k order and partial layout, so the partials are identical.
template <int NB, int RLO, int RHI, int CLO, int CHI>
__device__ __forceinline__ void gram_tiles(double (*xs)[kGR][kGRow], double (*ys)[kGR][kGRow], int lane, int st,
                                           double (&acc)[kGPairsMax][2]) {
  const int fr = lane & 3, fc = lane >> 2;
#pragma unroll 2
  for (int k0 = 0; k0 < kGR; k0 += 4) {
    const int row = k0 + fr;
    const int sw = gswz(row);
    double a[RHI - RLO > 0 ? RHI - RLO : 1], b[CHI - CLO > 0 ? CHI - CLO : 1];
#pragma unroll
    for (int i = 0; i < RHI - RLO; ++i) a[i] = xs[st][row][((RLO + i) * kGB + fc) ^ sw];
#pragma unroll
    for (int j = 0; j < CHI - CLO; ++j) b[j] = ys[st][row][((CLO + j) * kGB + fc) ^ sw];
    int t = 0;
#pragma unroll
    for (int i = 0; i < RHI - RLO; ++i)
#pragma unroll
      for (int j = 0; j < CHI - CLO; ++j)
        if (CLO + j >= RLO + i) {
          dmma(acc[t][0], acc[t][1], a[i], b[j]);
          ++t;
        }
  }
}

template <int NB, int RLO, int RHI, int CLO, int CHI>
__device__ __forceinline__ void gram_store(double* part, int lane, const double (&acc)[kGPairsMax][2]) {
  const int fr = lane & 3, fc = lane >> 2;
  int t = 0;
#pragma unroll
  for (int i = 0; i < RHI - RLO; ++i)
#pragma unroll
    for (int j = 0; j < CHI - CLO; ++j)
      if (CLO + j >= RLO + i) {
        double* o = part + (static_cast<long long>(blockIdx.x) * kGPairsMax + gpair(RLO + i, CLO + j, NB)) * (kGB * kGB);
        o[fc * kGB + 2 * fr] = acc[t][0];
        o[fc * kGB + 2 * fr + 1] = acc[t][1];
        ++t;
      }
}

template <int NB>
__global__ void __launch_bounds__(kGThreads) gram_sym_fixed_kernel(const double* __restrict__ X, long long ldx,
                                                                   const double* __restrict__ Y, long long ldy,
                                                                   int k, long long n, long long chunk,
                                                                   double* __restrict__ part) {
  extern __shared__ __align__(16) double gsm[];
  auto xs = reinterpret_cast<double(*)[kGR][kGRow]>(gsm);
  auto ys = reinterpret_cast<double(*)[kGR][kGRow]>(gsm + 2 * kGR * kGRow);
  const long long r0 = blockIdx.x * chunk;
  const long long r1 = min(n, r0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int H = (NB + 1) / 2, M = (NB - H) / 2;
  double acc[kGPairsMax][2];  // only the first (warp's tile count) entries are live
#pragma unroll
  for (int t = 0; t < kGPairsMax; ++t) acc[t][0] = acc[t][1] = 0.0;

  constexpr int kCStep = kGThreads / kGR;
  const int lrow = threadIdx.x % kGR, lcol = threadIdx.x / kGR;
  const int lsw = gswz(lrow);
  const double* xb = X + lcol * ldx + lrow;
  const double* yb = Y + lcol * ldy + lrow;
  auto issue = [&](int st, long long rb) {
    const bool rin = rb + lrow < r1;
    const double* px = xb + rb;
    const double* py = yb + rb;
#pragma unroll
    for (int q = 0; q < (NB * kGB + kCStep - 1) / kCStep; ++q) {
      const int col = lcol + q * kCStep;
      const bool v = rin && col < k;
      const int sc = col ^ lsw;
      gcp8(&xs[st][lrow][sc], v ? px : X, v);
      gcp8(&ys[st][lrow][sc], v ? py : Y, v);
      px += kCStep * ldx;
      py += kCStep * ldy;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  int st = 0;
  issue(0, r0);
  for (long long rb = r0; rb < r1; rb += kGR, st ^= 1) {
    if (rb + kGR < r1) {
      issue(st ^ 1, rb + kGR);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    switch (warp) {
      case 0: gram_tiles<NB, 0, H, 0, H>(xs, ys, lane, st, acc); break;
      case 1: gram_tiles<NB, 0, H, H, H + M>(xs, ys, lane, st, acc); break;
      case 2: gram_tiles<NB, 0, H, H + M, NB>(xs, ys, lane, st, acc); break;
      default: gram_tiles<NB, H, NB, H, NB>(xs, ys, lane, st, acc); break;
    }
    __syncthreads();
  }
  switch (warp) {
    case 0: gram_store<NB, 0, H, 0, H>(part, lane, acc); break;
    case 1: gram_store<NB, 0, H, H, H + M>(part, lane, acc); break;
    case 2: gram_store<NB, 0, H, H + M, NB>(part, lane, acc); break;
    default: gram_store<NB, H, NB, H, NB>(part, lane, acc); break;
  }
}

// G[row, col] (column-major, k x k) from the partials of tile t, in a fixed
// order over chunks; the upper triangle is mirrored.
__global__ void gram_sym_reduce_kernel(const double* __restrict__ part, int P, int k, double* __restrict__ G) {
  const int nb = (k + kGB - 1) / kGB;
  const int t = blockIdx.x;
  int bi = 0, q = t;
  while (bi < nb && q >= nb - bi) {
    q -= nb - bi;
    ++bi;
  }
  const int bj = bi + q;
  const int e = threadIdx.x;  // 0..63
  const int i = e / kGB, j = e % kGB;
  const int row = bi * kGB + i, col = bj * kGB + j;
  if (row >= k || col >= k || row > col) return;
  double s = 0.0;
  for (int p = 0; p < P; ++p) s += part[(static_cast<long long>(p) * kGPairsMax + t) * (kGB * kGB) + e];
  G[row + static_cast<long long>(col) * k] = s;
  G[col + static_cast<long long>(row) * k] = s;
}

}  // namespace

// G (k x k, column-major) = X[r0:r1)^T Y[r0:r1) of a symmetric product
void gram_sym_rows(Ctx& ctx, int k, const double* X, long long ldx, const double* Y, long long ldy, long long r0,
                   long long r1, double* G) {
  if (k <= 0) return;
  X += r0;
  Y += r0;
  const long long n = std::max<long long>(0, r1 - r0);
  if (k <= kGMaxK) {
    const int P = 148 * 4;
    long long chunk = ((n + P - 1) / P + kGR - 1) / kGR * kGR;
    if (chunk <= 0) chunk = kGR;
    const int Pn = static_cast<int>(std::max<long long>(1, (n + chunk - 1) / chunk));
    double* part = ctx.ws_gram.get<double>(static_cast<size_t>(Pn) * kGPairsMax * kGB * kGB);
    constexpr size_t smem = sizeof(double) * 4 * kGR * kGRow;
    static bool configured = false;
    if (!configured) {
      PARO_CUDA(cudaFuncSetAttribute(gram_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      PARO_CUDA(cudaFuncSetAttribute(gram_sym_fixed_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      PARO_CUDA(cudaFuncSetAttribute(gram_sym_fixed_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      configured = true;
    }
    const int nb = (k + kGB - 1) / kGB;
    if (nb == 10 || nb == 8) {
      auto kern = nb == 10 ? gram_sym_fixed_kernel<10> : gram_sym_fixed_kernel<8>;
      kern<<<Pn, kGThreads, smem, ctx.stream>>>(X, ldx, Y, ldy, k, n, chunk, part);
    } else {
      gram_sym_kernel<<<Pn, kGThreads, smem, ctx.stream>>>(X, ldx, Y, ldy, k, n, chunk, part);
    }
    gram_sym_reduce_kernel<<<nb * (nb + 1) / 2, kGB * kGB, 0, ctx.stream>>>(part, Pn, k, G);
    PARO_CUDA(cudaGetLastError());
    ctx.launches += 2;
    return;
  }
  // wider bases (baseline_geneig blocks beyond 80 columns): 80 x 16 rectangular tiles
  double* tile = ctx.ws_small3.get<double>(80 * 16);
  for (int i0 = 0; i0 < k; i0 += 80) {
    const int ki = std::min(80, k - i0);
    for (int j0 = 0; j0 < k; j0 += 16) {
      const int kj = std::min(16, k - j0);
      gram_rect_rows(ctx, ki, X + i0 * ldx, ldx, kj, Y + j0 * ldy, ldy, 0, n, tile);
      PARO_CUDA(cudaMemcpy2DAsync(G + i0 + static_cast<long long>(j0) * k, sizeof(double) * k, tile,
                                  sizeof(double) * ki, sizeof(double) * ki, kj, cudaMemcpyDeviceToDevice, ctx.stream));
    }
  }
}

namespace {

void gram(Ctx& ctx, int k, const double* X, long long ldx, const double* Y, long long ldy, double* G) {
  gram_sym_rows(ctx, k, X, ldx, Y, ldy, 0, ctx.grid.n, G);
}

// Z (n x k2) = X (n x k1) C (k1 x k2, column-major, ldc); tri: C is the
// Cholesky-QR basis change (zero below the drop-shifted diagonal)
void rotate(Ctx& ctx, int k1, int k2, const double* X, long long ldx, const double* Cm, int ldc, double* Z,
            long long ldz, bool tri = false) {
  rotate_rows(ctx, k1, X, ldx, Cm, ldc, k2, Z, ldz, 0, ctx.grid.n, tri ? 2 : 0);
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) v = fmax(v, sh[w]);
  __syncthreads();
  return v;
}

// gram_defect (paro.cpp:50-61): max over j <= i of |v_i^T B v_j - delta_ij|.
__global__ void defect_kernel(int k, const double* G, double* out) {
  __shared__ double sh[32];
  double m = 0.0;
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
    const int i = idx % k, j = idx / k;
    if (j <= i) m = fmax(m, fabs(G[i + j * k] - (i == j ? 1.0 : 0.0)));
  }
  m = block_max(m, sh);
  if (threadIdx.x == 0) *out = m;
}

}  // namespace

// fix_sign (linalg.cpp:229-241) of k device columns: the row-range pieces of
// step4.cu over all n rows (a sharded Step 4 combines them across ranks)
void fix_sign_columns(Ctx& ctx, double* V, long long ld, int k) {
  if (k <= 0) return;
  const long long n = ctx.grid.n;
  double* amax = ctx.ws_small3.get<double>(3 * static_cast<size_t>(k));
  double* flip = amax + k;
  auto* first = reinterpret_cast<long long*>(amax + 2 * k);
  sign_init(ctx, k, amax, first);
  colmax_rows(ctx, k, V, ld, 0, n, amax);
  first_rows(ctx, k, V, ld, 0, n, amax, first);
  sign_rows(ctx, k, V, ld, 0, n, amax, first, flip);
  negate_rows(ctx, k, V, ld, 0, n, flip);
}

namespace {

struct Small {
  double *G, *C1, *G2, *C2, *Bt, *GA, *vals, *Y, *At, *X, *G3, *rmin, *defect;
  int *acc, *kout, *status;
  DenseScratch w;
};

Small small_buffers(Ctx& ctx, int K) {
  const size_t kk = static_cast<size_t>(K) * K;
  double* base = ctx.ws_small.get<double>(16 * kk + 4 * K + 64);
  Small s{};
  double* p = base;
  auto take = [&](size_t cnt) {
    double* r = p;
    p += cnt;
    return r;
  };
  s.G = take(kk);
  s.C1 = take(kk);
  s.G2 = take(kk);
  s.C2 = take(kk);
  s.Bt = take(kk);
  s.GA = take(kk);
  s.Y = take(kk);
  s.At = take(kk);
  s.X = take(kk);
  s.G3 = take(kk);
  s.w.a = take(kk);
  s.w.v = take(kk);
  s.w.l = take(kk);
  s.w.w = take(kk);
  s.w.c = take(kk);
  s.vals = take(K);
  s.rmin = take(1);
  s.defect = take(1);
  int* ib = ctx.ws_small2.get<int>(3 * static_cast<size_t>(K) + 8);
  s.acc = ib;
  s.w.order = ib + K;
  s.kout = ib + 2 * K;
  s.status = ib + 2 * K + 1;
  return s;
}

int read_int(Ctx& ctx, const int* d) {
  int v = 0;
  small_d2h(ctx, &v, d, sizeof(int));
  return v;
}

double read_double(Ctx& ctx, const double* d) {
  double v = 0;
  small_d2h(ctx, &v, d, sizeof(double));
  return v;
}

}  // namespace

namespace {

__global__ void div_kernel(double* dst, const double* src, double d, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = src[i] / d;  // x /= nb (linalg.cpp:431)
}

double ddot(Ctx& ctx, const double* x, const double* y, double* d) {
  gram_rect_rows(ctx, 1, x, ctx.grid.n, 1, y, ctx.grid.n, 0, ctx.grid.n, d);
  return read_double(ctx, d);
}

// b_orthonormalize (linalg.cpp:409-439) as two-pass classical Gram-Schmidt in
// the B inner product, candidate by candidate with the same drop rule:
// Q (k columns) B-orthonormal, BQ = B Q. Used when the candidates are too
// ill-conditioned for the Cholesky-QR path (e.g. right after a noise start).
int cgs2_orthonormalize(Ctx& ctx, const Op& B, int K, const double* U, double drop_tol, double* Q, double* BQ,
                        int* kout, int* accepted = nullptr) {
  const long long n = ctx.grid.n;
  cudaStream_t st = ctx.stream;
  double* h = ctx.ws_e.get<double>(2 * static_cast<size_t>(n) + K + 8);
  double* Bh = h + n;
  double* c = Bh + n;
  double* d = c + K;
  const int blocks = static_cast<int>(std::min<long long>(148 * 8, (n + 255) / 256));
  int k = 0;
  for (int j = 0; j < K; ++j) {
    PARO_CUDA(cudaMemcpyAsync(h, U + j * n, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    apply_op(ctx, B, nullptr, 0.0, 1, h, n, Bh, n);
    const double orig = std::sqrt(std::max(0.0, ddot(ctx, h, Bh, d)));
    if (!(orig > 0.0)) continue;
    for (int pass = 0; pass < 2 && k > 0; ++pass) {
      // c = (B Q)^T h, h -= Q c, over 80-column slices of the accepted basis
      for (int i0 = 0; i0 < k; i0 += 80) {
        const int ki = std::min(80, k - i0);
        gram_rect_rows(ctx, ki, BQ + i0 * n, n, 1, h, n, 0, n, c + i0);
      }
      for (int i0 = 0; i0 < k; i0 += 80) {
        const int ki = std::min(80, k - i0);
        rotate_rows(ctx, ki, Q + i0 * n, n, c + i0, ki, 1, h, n, 0, n, 1);
      }
    }
    apply_op(ctx, B, nullptr, 0.0, 1, h, n, Bh, n);
    const double nb = std::sqrt(std::max(0.0, ddot(ctx, h, Bh, d)));
    if (nb <= drop_tol * orig) continue;
    div_kernel<<<blocks, 256, 0, st>>>(Q + k * n, h, nb, n);
    ++ctx.launches;
    apply_op(ctx, B, nullptr, 0.0, 1, Q + k * n, n, BQ + k * n, n);
    if (accepted) accepted[k] = j;
    ++k;
  }
  *kout = k;
  return kOk;
}

}  // namespace

// smallest pivot ratio of the candidates' ordered Cholesky for which the basis
// change stays in K x K arithmetic (one pass; step4.py ONE_PASS_RATIO)
constexpr double kOnePassRatio = 0.5;

int rayleigh_ritz(Ctx& ctx, const Op& A, const Op& B, int K, const double* U, long long ld, size_t min_keep,
                  double drop_tol, double* lambdas, double* V, long long ldv, int* k_out, double* defect,
                  RitzInfo* info) {
  ctx.check_grid();
  if (K <= 0) throw ParoError(kEmptyBasis, "b_orthonormalize: all vectors dropped");
  const long long n = ctx.grid.n;
  if (ld != n || ldv != n) throw ParoError(kInvalidArgument, "rayleigh_ritz: vectors must be contiguous (ld == n)");
  cudaStream_t st = ctx.stream;
  struct ClearCopyout {  // the copy-out request is one-shot
    Ctx& c;
    ~ClearCopyout() { c.ritz_copyout.host = nullptr; }
  } clear_copyout{ctx};
  double* W = ctx.ws_b.get<double>(static_cast<size_t>(K) * n);
  double* Q1 = ctx.ws_c.get<double>(static_cast<size_t>(K) * n);
  Small s = small_buffers(ctx, K);
  int k = 0;
  bool use_cgs = ctx.force_cgs2;

  auto check_count = [&](int kk) -> int {
    if (kk == 0) {
      ctx.err = "b_orthonormalize: all vectors dropped";
      return kEmptyBasis;
    }
    if (static_cast<size_t>(kk) < min_keep) {
      ctx.err = "rayleigh_ritz: candidate span collapsed to " + std::to_string(kk) + " < " + std::to_string(min_keep);
      return kDegenerateSpan;
    }
    return kOk;
  };
  bool copy_pending = false;  // a host copy-out of V is queued on the copy stream
  auto finish = [&](const double* Qb, int kk) -> double {
    auto& co = ctx.ritz_copyout;
    // a CGS2 retry rewrites V: the copy-out queued by the first finish must have read it
    if (copy_pending) PARO_CUDA(cudaStreamWaitEvent(st, co.ready, 0));
    // lift, sign convention, certificate (paro.cpp:157-174)
    rotate(ctx, kk, kk, Qb, n, s.Y, kk, V, ldv);
    fix_sign_columns(ctx, V, ldv, kk);
    // final orbitals: a pending host copy-out starts now, overlapping the certificate
    if (co.host != nullptr) {
      if (co.ready == nullptr) PARO_CUDA(cudaEventCreateWithFlags(&co.ready, cudaEventDisableTiming));
      PARO_CUDA(cudaEventRecord(co.ready, st));
      PARO_CUDA(cudaStreamWaitEvent(co.stream, co.ready, 0));
      const int c1 = std::min(co.c1, kk);
      for (int c = co.c0; c < c1; ++c)
        PARO_CUDA(cudaMemcpyAsync(co.host + static_cast<long long>(c) * co.ldh, V + static_cast<long long>(c) * ldv,
                                  sizeof(double) * n, cudaMemcpyDeviceToHost, co.stream));
      PARO_CUDA(cudaEventRecord(co.ready, co.stream));  // reused: "the copies have read V"
      copy_pending = true;
    }
    apply_op(ctx, B, nullptr, 0.0, kk, V, ldv, W, n);
    gram(ctx, kk, V, ldv, W, n, s.G3);
    defect_kernel<<<1, 256, 0, st>>>(kk, s.G3, s.defect);
    ++ctx.launches;
    return read_double(ctx, s.defect);
  };

  double d = 0.0, rmin = 0.0;
  if (!use_cgs) {
    // CholQR pass 1: Gram of the candidates, ordered Cholesky with drops
    apply_op(ctx, B, nullptr, 0.0, K, U, ld, W, n);
    gram(ctx, K, U, ld, W, n, s.G);
    ortho_from_gram_kernel<<<1, kDenseThreads, 0, st>>>(K, s.G, drop_tol, 1, s.C1, s.acc, s.kout, s.rmin, s.w, s.status);
    ++ctx.launches;
    PARO_CUDA(cudaGetLastError());
    k = read_int(ctx, s.kout);
    rmin = read_double(ctx, s.rmin);
    if (info) info->min_ratio = rmin;
    // Cholesky pivots lose ~eps/ratio^2 relative accuracy: near-dependent
    // candidates (and every drop decision) go through the CGS2 path instead
    if (rmin < 1e-5) use_cgs = true;
  }
  bool one_pass = false;
  const bool aliased = V < U + static_cast<long long>(K) * ld && U < V + static_cast<long long>(K) * ldv;
  if (!use_cgs && k == K && rmin >= kOnePassRatio && !aliased && !ctx.two_pass_only) {
    // well-conditioned candidates (the steady state of the outer iteration:
    // the Step-3 solutions are nearly B-orthonormal): the basis change stays
    // in K x K arithmetic -- At = C1^T (U^T A U) C1, Bt = C1^T (U^T B U) C1,
    // both Grams of the actual candidates -- and the lift is V = U (C1 X);
    // no intermediate basis is formed (one rotation, apply and Gram less).
    // The certificate below still measures the actual V.
    const int cs = check_count(k);
    if (cs != kOk) return cs;
    congruence_kernel<<<1, kDenseThreads, 0, st>>>(k, s.G, s.C1, s.Bt, s.w);
    ++ctx.launches;
    apply_op(ctx, A, nullptr, 0.0, k, U, ld, W, n);
    gram(ctx, k, U, ld, W, n, s.GA);
    dense_configure();
    pencil_kernel<<<1, kDenseThreads, dense_jacobi_smem(k), st>>>(k, s.GA, s.C1, s.Bt, s.vals, s.Y, s.At, s.X, s.w, s.status);
    ++ctx.launches;
    if (read_int(ctx, s.status) == kOk) {
      d = finish(U, k);
      one_pass = d <= 1e-8;
    }
    // a failed pencil or certificate falls through to the two-pass path
  }
  if (!use_cgs && !one_pass) {
    const int cs = check_count(k);
    if (cs != kOk) return cs;
    rotate(ctx, K, k, U, ld, s.C1, K, Q1, n, true);
    // pass 2
    apply_op(ctx, B, nullptr, 0.0, k, Q1, n, W, n);
    gram(ctx, k, Q1, n, W, n, s.G2);
    second_pass_kernel<<<1, kDenseThreads, 0, st>>>(k, s.G2, s.C2, s.Bt, s.w, s.status);
    ++ctx.launches;
    if (read_int(ctx, s.status) != kOk) {
      use_cgs = true;
    } else {
      apply_op(ctx, A, nullptr, 0.0, k, Q1, n, W, n);
      gram(ctx, k, Q1, n, W, n, s.GA);
      dense_configure();
      pencil_kernel<<<1, kDenseThreads, dense_jacobi_smem(k), st>>>(k, s.GA, s.C2, s.Bt, s.vals, s.Y, s.At, s.X, s.w, s.status);
      ++ctx.launches;
      if (read_int(ctx, s.status) != kOk) {
        ctx.err = "pencil: B is not positive definite";
        return kPencil;
      }
      d = finish(Q1, k);
      if (d > 1e-8) use_cgs = true;  // retry with explicit Gram-Schmidt before failing the certificate
    }
  }
  if (use_cgs) {
    if (info) info->cgs2 = true;
    double* BQ = W;
    cgs2_orthonormalize(ctx, B, K, U, drop_tol, Q1, BQ, &k);
    const int cs = check_count(k);
    if (cs != kOk) return cs;
    double* AQ = ctx.ws_d.get<double>(static_cast<size_t>(k) * n);
    apply_op(ctx, A, nullptr, 0.0, k, Q1, n, AQ, n);
    gram(ctx, k, Q1, n, AQ, n, s.GA);
    gram(ctx, k, Q1, n, BQ, n, s.G2);
    dense_configure();
    pencil_direct_kernel<<<1, kDenseThreads, dense_jacobi_smem(k), st>>>(k, s.GA, s.G2, s.vals, s.Y, s.At, s.Bt, s.X, s.w, s.status);
    ++ctx.launches;
    if (read_int(ctx, s.status) != kOk) {
      ctx.err = "pencil: B is not positive definite";
      return kPencil;
    }
    d = finish(Q1, k);
  }
  if (info) info->k = k;
  small_d2h(ctx, lambdas, s.vals, sizeof(double) * k);
  *k_out = k;
  *defect = d;
  if (d > 1e-8 && (!info || info->certify)) {
    ctx.err = "rayleigh_ritz: orthonormality certificate violated (defect " + std::to_string(d) + ")";
    return kError;
  }
  return kOk;
}

// ---------------------------------------------------------------------------
// The K x K stages of rayleigh_ritz on caller buffers (device, column-major),
// for a Step 4 orchestrated over row slabs (the Grams combined across ranks
// before each stage; every rank then runs the same stage on the same input).
int ritz_ortho(Ctx& ctx, int K, const double* G, double drop_tol, double* C1, int* k_out, double* min_ratio) {
  Small s = small_buffers(ctx, K);
  ortho_from_gram_kernel<<<1, kDenseThreads, 0, ctx.stream>>>(K, G, drop_tol, 1, C1, s.acc, s.kout, s.rmin, s.w, s.status);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
  *k_out = read_int(ctx, s.kout);
  *min_ratio = read_double(ctx, s.rmin);
  return kOk;
}

int ritz_second_pass(Ctx& ctx, int k, const double* G2, double* C2, double* Bt) {
  Small s = small_buffers(ctx, k);
  second_pass_kernel<<<1, kDenseThreads, 0, ctx.stream>>>(k, G2, C2, Bt, s.w, s.status);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
  if (read_int(ctx, s.status) != kOk) {
    ctx.err = "rayleigh_ritz: second Cholesky-QR pass not positive definite";
    return kPencil;
  }
  return kOk;
}

int ritz_congruence(Ctx& ctx, int k, const double* G, const double* C1, double* Bt) {
  Small s = small_buffers(ctx, k);
  congruence_kernel<<<1, kDenseThreads, 0, ctx.stream>>>(k, G, C1, Bt, s.w);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
  return kOk;
}

int ritz_pencil(Ctx& ctx, int k, const double* GA, const double* C2, const double* Bt, const double* GB,
                double* vals_host, double* Y) {
  Small s = small_buffers(ctx, k);
  dense_configure();
  if (GB == nullptr)
    pencil_kernel<<<1, kDenseThreads, dense_jacobi_smem(k), ctx.stream>>>(k, GA, C2, Bt, s.vals, Y, s.At, s.X, s.w,
                                                                          s.status);
  else
    pencil_direct_kernel<<<1, kDenseThreads, dense_jacobi_smem(k), ctx.stream>>>(k, GA, GB, s.vals, Y, s.At, s.Bt,
                                                                                 s.X, s.w, s.status);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
  if (read_int(ctx, s.status) != kOk) {
    ctx.err = "pencil: B is not positive definite";
    return kPencil;
  }
  small_d2h(ctx, vals_host, s.vals, sizeof(double) * k);
  return kOk;
}

double ritz_defect(Ctx& ctx, int k, const double* G) {
  Small s = small_buffers(ctx, k);
  defect_kernel<<<1, 256, 0, ctx.stream>>>(k, G, s.defect);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
  return read_double(ctx, s.defect);
}

int b_orthonormalize(Ctx& ctx, const Op& B, int K, const double* U, double drop_tol, double* Q, int* k_out,
                     int* accepted) {
  ctx.check_grid();
  const long long n = ctx.grid.n;
  double* BQ = ctx.ws_b.get<double>(static_cast<size_t>(K) * n);
  cgs2_orthonormalize(ctx, B, K, U, drop_tol, Q, BQ, k_out, accepted);
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
  if (*k_out == 0 && K > 0) {
    ctx.err = "b_orthonormalize: all vectors dropped";
    return kEmptyBasis;
  }
  return kOk;
}

int dense_sym_geneig(Ctx& ctx, int m, const double* A_host, const double* B_host, double* vals_host,
                     double* vecs_host) {
  Small s = small_buffers(ctx, m);
  cudaStream_t st = ctx.stream;
  const size_t bytes = sizeof(double) * m * m;
  PARO_CUDA(cudaMemcpyAsync(s.At, A_host, bytes, cudaMemcpyHostToDevice, st));
  PARO_CUDA(cudaMemcpyAsync(s.Bt, B_host, bytes, cudaMemcpyHostToDevice, st));
  dense_configure();
  geneig_kernel<<<1, kDenseThreads, dense_jacobi_smem(m), st>>>(m, s.At, s.Bt, s.vals, s.X, s.w, s.status);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
  const int status = read_int(ctx, s.status);
  if (status != kOk) {
    ctx.err = "pencil: B is not positive definite or the pencil is not symmetric";
    return status;
  }
  PARO_CUDA(cudaMemcpyAsync(vals_host, s.vals, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  PARO_CUDA(cudaMemcpyAsync(vecs_host, s.X, bytes, cudaMemcpyDeviceToHost, st));
  PARO_CUDA(cudaStreamSynchronize(st));
  return kOk;
}

}  // namespace paro_b200
