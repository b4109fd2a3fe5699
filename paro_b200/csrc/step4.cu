// Step-4 building blocks on row ranges: the tall-skinny rotation Z = X C
// (the lift of rayleigh_ritz, proj/src/paro.cpp:157-169, and the Cholesky-QR
// basis change), the rectangular Gram X^T Y (the projections of
// b_orthonormalize, proj/src/linalg.cpp:409-439) and the sign convention
// fix_sign (linalg.cpp:229-241) split into per-range partial results that a
// caller can combine across ranks (row-slab sharded Step 4).
//
// Both products run on the FP64 tensor cores (mma.sync m8n8k4 f64, DMMA):
// an n x 76 by 76 x 76 rotation is 2 n 76^2 flop against 16 n 76 bytes, i.e.
// FP64-throughput-bound on B200 (~10 flop/byte vs ~5.4 at the ridge).
#include <algorithm>
#include <climits>

#include "dmma.cuh"
#include "step4.hpp"

namespace paro_b200 {

namespace {

// ---------------------------------------------------------------------------
// Rotation Z[r0:r1) = X[r0:r1) C  (mode bit 0: Z -= X C; bit 2: Z += X C; bit 1: C is
// "upper triangular up to the drop shift", C[i][j] = 0 for i > j + k1 - k2,
// so tile j skips the zero k-steps). Persistent CTAs walk 32-row chunks; the
// chunk's k1 columns are staged by cp.async (double-buffered), B fragments
// of C stay in registers for the whole kernel, the 8 x 8 output tiles are
// written through shared memory as coalesced column segments. Each output
// element is the same k-ordered DMMA chain whatever chunk its row falls in,
// so the result does not depend on the row partition.
constexpr int kRotR = 32;
constexpr int kRotWarps = 5;
constexpr int kRotThreads = 32 * kRotWarps;
constexpr int kRotMaxK = 80;
constexpr int kRotKS = kRotMaxK / 4;  // k-steps
constexpr int kRotXS = kRotR + 4;     // staged column stride: conflict-free A-fragment loads
constexpr int kRotZS = kRotR + 1;
constexpr size_t kRotSmem = sizeof(double) * (2 * kRotMaxK * kRotXS + kRotMaxK * kRotZS);

__global__ void __launch_bounds__(kRotThreads, 3)
    rotate_kernel(const double* __restrict__ X, long long ldx, const double* __restrict__ Cm, int ldc, int k1, int k2,
                  double* Z, long long ldz, long long r0, long long r1, int mode) {
  extern __shared__ __align__(16) double rsm[];
  auto xs = reinterpret_cast<double(*)[kRotMaxK][kRotXS]>(rsm);
  double* zs = rsm + 2 * kRotMaxK * kRotXS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane & 3, fc = lane >> 2;
  const int nb2 = (k2 + 7) / 8;
  const int nks = (k1 + 3) / 4;
  const long long rows = r1 - r0;
  const long long nchunks = (rows + kRotR - 1) / kRotR;

  // the warp's output column tiles: w and nb2-1-w (balances the triangular case)
  int tl[2] = {-1, -1};
  if (warp < nb2) tl[0] = warp;
  if (nb2 - 1 - warp > warp) tl[1] = nb2 - 1 - warp;
  int ksl[2];
  double bfr[2][kRotKS];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    ksl[i] = 0;
    if (tl[i] >= 0) {
      int lim = k1;
      if (mode & 2) lim = min(k1, 8 * tl[i] + 8 + (k1 - k2));
      ksl[i] = (lim + 3) / 4;
    }
    const int col = 8 * (tl[i] < 0 ? 0 : tl[i]) + fc;
#pragma unroll
    for (int ks = 0; ks < kRotKS; ++ks) {
      const int kk = 4 * ks + fr;
      bfr[i][ks] = (tl[i] >= 0 && kk < k1 && col < k2) ? Cm[kk + static_cast<long long>(col) * ldc] : 0.0;
    }
  }

  auto issue = [&](int st, long long chunk) {
    const long long rb = r0 + chunk * kRotR;
    const int k1p = (k1 + 3) & ~3;  // the last k-step's padding columns are zero-filled
    for (int idx = threadIdx.x; idx < k1p * kRotR; idx += kRotThreads) {
      const int col = idx / kRotR, row = idx % kRotR;
      const bool v = rb + row < r1 && col < k1;
      cp_async8(&xs[st][col][row], v ? X + col * ldx + rb + row : X, v);
    }
    cp_async_commit();
  };

  long long chunk = blockIdx.x;
  int st = 0;
  if (chunk < nchunks) issue(0, chunk);
  for (; chunk < nchunks; chunk += gridDim.x, st ^= 1) {
    const long long next = chunk + gridDim.x;
    if (next < nchunks) {
      issue(st ^ 1, next);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int rt = 0; rt < 4; ++rt) acc[i][rt][0] = acc[i][rt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < kRotKS; ++ks) {
      if (ks < nks) {
        double a[4];
#pragma unroll
        for (int rt = 0; rt < 4; ++rt) a[rt] = xs[st][4 * ks + fr][8 * rt + fc];
#pragma unroll
        for (int i = 0; i < 2; ++i)
          if (ks < ksl[i])
#pragma unroll
            for (int rt = 0; rt < 4; ++rt) dmma884(acc[i][rt][0], acc[i][rt][1], a[rt], bfr[i][ks]);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (tl[i] < 0) continue;
#pragma unroll
      for (int rt = 0; rt < 4; ++rt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int col = 8 * tl[i] + 2 * fr + j;
          if (col < k2) zs[col * kRotZS + 8 * rt + fc] = acc[i][rt][j];
        }
    }
    __syncthreads();
    const long long rb = r0 + chunk * kRotR;
    for (int idx = threadIdx.x; idx < k2 * kRotR; idx += kRotThreads) {
      const int col = idx / kRotR, row = idx % kRotR;
      if (rb + row < r1) {
        double* z = Z + col * ldz + rb + row;
        const double v = zs[col * kRotZS + row];
        *z = (mode & 1) ? *z - v : (mode & 4) ? *z + v : v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Rectangular Gram G (k1 x k2, column-major) = X[r0:r1)^T Y[r0:r1), k1 <= 80,
// k2 <= 16: split-K over row chunks (one CTA per chunk, DMMA tiles over the
// k1 x k2 output, rows staged by cp.async), partials summed in a fixed order.
constexpr int kGRR = 32;
constexpr int kGRT = 128;
constexpr int kGRMax1 = 80, kGRMax2 = 16;
constexpr int kGRS = kGRR + 4;
constexpr size_t kGRSmem = sizeof(double) * 2 * (kGRMax1 + kGRMax2) * kGRS;

__global__ void __launch_bounds__(kGRT) gram_rect_kernel(const double* __restrict__ X, long long ldx, int k1,
                                                         const double* __restrict__ Y, long long ldy, int k2,
                                                         long long r0, long long r1, long long chunk,
                                                         double* __restrict__ part) {
  extern __shared__ __align__(16) double gsm2[];
  auto xs = reinterpret_cast<double(*)[kGRMax1][kGRS]>(gsm2);
  auto ys = reinterpret_cast<double(*)[kGRMax2][kGRS]>(gsm2 + 2 * kGRMax1 * kGRS);
  const long long c0 = r0 + blockIdx.x * chunk;
  const long long c1 = min(r1, c0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane & 3, fc = lane >> 2;
  const int nb1 = (k1 + 7) / 8, nb2 = (k2 + 7) / 8;
  const int ntiles = nb1 * nb2;
  double acc[5][2];
#pragma unroll
  for (int t = 0; t < 5; ++t) acc[t][0] = acc[t][1] = 0.0;

  auto issue = [&](int st, long long rb) {
    // whole 8-column tiles are staged, the padding columns zero-filled
    const int k1p = (k1 + 7) & ~7, k2p = (k2 + 7) & ~7;
    for (int idx = threadIdx.x; idx < (k1p + k2p) * kGRR; idx += kGRT) {
      const int col = idx / kGRR, row = idx % kGRR;
      const bool rv = rb + row < c1;
      if (col < k1p) {
        const bool v = rv && col < k1;
        cp_async8(&xs[st][col][row], v ? X + col * ldx + rb + row : X, v);
      } else {
        const bool v = rv && col - k1p < k2;
        cp_async8(&ys[st][col - k1p][row], v ? Y + (col - k1p) * ldy + rb + row : Y, v);
      }
    }
    cp_async_commit();
  };
  int st = 0;
  if (c0 < c1) issue(0, c0);
  for (long long rb = c0; rb < c1; rb += kGRR, st ^= 1) {
    if (rb + kGRR < c1) {
      issue(st ^ 1, rb + kGRR);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGRR / 4; ++ks) {
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int t = warp + 4 * q;
        if (t < ntiles) {
          const int ti = t / nb2, tj = t % nb2;
          const double a = xs[st][8 * ti + fc][4 * ks + fr];
          const double b = ys[st][8 * tj + fc][4 * ks + fr];
          dmma884(acc[q][0], acc[q][1], a, b);
        }
      }
    }
    __syncthreads();
  }
  double* o = part + blockIdx.x * static_cast<long long>(k1) * k2;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int t = warp + 4 * q;
    if (t < ntiles) {
      const int ti = t / nb2, tj = t % nb2;
      const int i = 8 * ti + fc;
#pragma unroll
      for (int j2 = 0; j2 < 2; ++j2) {
        const int j = 8 * tj + 2 * fr + j2;
        if (i < k1 && j < k2) o[i + static_cast<long long>(j) * k1] = acc[q][j2];
      }
    }
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int P, int m, double* __restrict__ G) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < P; ++p) s += part[static_cast<long long>(p) * m + e];
    G[e] = s;
  }
}

// ---------------------------------------------------------------------------
// fix_sign (linalg.cpp:229-241) in three combinable pieces over row ranges:
// column max |v|, first (global) row with |v| > 1e-12 max, and the sign of
// that entry where this range holds it; then the negation.
__device__ __forceinline__ double block_max_all(double v, double* sh) {
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

__global__ void colmax_rows_kernel(const double* V, long long ld, long long r0, long long r1, double* amax) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  double m = 0.0;
  for (long long i = r0 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < r1;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(V[c * ld + i]));
  m = block_max_all(m, sh);
  if (threadIdx.x == 0 && m > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(amax) + c, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// each block scans one contiguous segment, low segments first, and stops as
// soon as a lower row is already known (the pivot is usually in the first planes)
__global__ void first_rows_kernel(const double* V, long long ld, long long r0, long long r1, const double* amax,
                                  long long* first) {
  __shared__ int stop;
  const int c = blockIdx.y;
  const double thr = 1e-12 * amax[c];
  const long long seg = (r1 - r0 + gridDim.x - 1) / gridDim.x;
  const long long lo = r0 + blockIdx.x * seg, hi = min(r1, lo + seg);
  auto* f = reinterpret_cast<unsigned long long*>(first) + c;
  for (long long base = lo; base < hi; base += blockDim.x) {
    if (threadIdx.x == 0) stop = *reinterpret_cast<volatile const unsigned long long*>(f) < static_cast<unsigned long long>(base);
    __syncthreads();
    if (stop) return;
    const long long i = base + threadIdx.x;
    const bool hit = i < hi && amax[c] > 0.0 && fabs(V[c * ld + i]) > thr;
    if (hit) atomicMin(f, static_cast<unsigned long long>(i));
    if (__syncthreads_or(hit)) return;
  }
}

__global__ void sign_rows_kernel(const double* V, long long ld, int k, long long r0, long long r1,
                                 const double* amax, const long long* first, double* flip) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const long long f = first[c];
    flip[c] = (amax[c] > 0.0 && f >= r0 && f < r1 && V[c * ld + f] < 0.0) ? 1.0 : 0.0;
  }
}

__global__ void negate_rows_kernel(double* V, long long ld, long long r0, long long r1, const double* flip) {
  const int c = blockIdx.y;
  if (flip[c] == 0.0) return;
  for (long long i = r0 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < r1;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    V[c * ld + i] = -V[c * ld + i];
}

__global__ void sign_init_kernel(int k, double* amax, long long* first) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    if (amax) amax[i] = 0.0;
    if (first) first[i] = LLONG_MAX;
  }
}

int grid_for(long long rows, int per_sm) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>(148LL * per_sm, (rows + 255) / 256)));
}

}  // namespace

void rotate_rows(Ctx& ctx, int k1, const double* X, long long ldx, const double* C, int ldc, int k2, double* Z,
                 long long ldz, long long r0, long long r1, int mode) {
  if (k1 <= 0 || k2 <= 0 || r1 <= r0) return;
  if (k1 > kRotMaxK || k2 > kRotMaxK) {
    // wider bases: 80 x 80 blocks of C; the first input block of an assigning
    // rotation assigns, the others accumulate (the triangular skip is dropped)
    for (int j0 = 0; j0 < k2; j0 += kRotMaxK) {
      const int kj = std::min(kRotMaxK, k2 - j0);
      for (int i0 = 0; i0 < k1; i0 += kRotMaxK) {
        const int ki = std::min(kRotMaxK, k1 - i0);
        const int m = (mode & 1) ? 1 : (mode & 4) ? 4 : (i0 == 0 ? 0 : 4);
        rotate_rows(ctx, ki, X + i0 * ldx, ldx, C + i0 + static_cast<long long>(j0) * ldc, ldc, kj, Z + j0 * ldz,
                    ldz, r0, r1, m);
      }
    }
    return;
  }
  static bool configured = false;
  if (!configured) {
    PARO_CUDA(cudaFuncSetAttribute(rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kRotSmem)));
    configured = true;
  }
  const long long nchunks = (r1 - r0 + kRotR - 1) / kRotR;
  const int grid = static_cast<int>(std::min<long long>(nchunks, 148LL * 3));
  rotate_kernel<<<grid, kRotThreads, kRotSmem, ctx.stream>>>(X, ldx, C, ldc, k1, k2, Z, ldz, r0, r1, mode);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

void gram_rect_rows(Ctx& ctx, int k1, const double* X, long long ldx, int k2, const double* Y, long long ldy,
                    long long r0, long long r1, double* G) {
  if (k1 <= 0 || k2 <= 0) return;
  if (k1 > kGRMax1 || k2 > kGRMax2) throw ParoError(kInvalidArgument, "gram_rect: at most 80 x 16 columns");
  static bool configured = false;
  if (!configured) {
    PARO_CUDA(cudaFuncSetAttribute(gram_rect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kGRSmem)));
    configured = true;
  }
  const long long rows = std::max<long long>(0, r1 - r0);
  const int Pmax = 148 * 4;
  long long chunk = ((rows + Pmax - 1) / Pmax + kGRR - 1) / kGRR * kGRR;
  if (chunk <= 0) chunk = kGRR;
  const int P = static_cast<int>(std::max<long long>(1, (rows + chunk - 1) / chunk));
  const int m = k1 * k2;
  double* part = ctx.ws_gram.get<double>(static_cast<size_t>(P) * m);
  gram_rect_kernel<<<P, kGRT, kGRSmem, ctx.stream>>>(X, ldx, k1, Y, ldy, k2, r0, r1, chunk, part);
  sum_partials_kernel<<<(m + 255) / 256, 256, 0, ctx.stream>>>(part, P, m, G);
  PARO_CUDA(cudaGetLastError());
  ctx.launches += 2;
}

void sign_init(Ctx& ctx, int k, double* amax, long long* first) {
  sign_init_kernel<<<1, 256, 0, ctx.stream>>>(k, amax, first);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

void colmax_rows(Ctx& ctx, int k, const double* V, long long ld, long long r0, long long r1, double* amax) {
  if (k <= 0 || r1 <= r0) return;
  colmax_rows_kernel<<<dim3(grid_for(r1 - r0, 4), k), 256, 0, ctx.stream>>>(V, ld, r0, r1, amax);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

void first_rows(Ctx& ctx, int k, const double* V, long long ld, long long r0, long long r1, const double* amax,
                long long* first) {
  if (k <= 0 || r1 <= r0) return;
  first_rows_kernel<<<dim3(grid_for(r1 - r0, 4), k), 256, 0, ctx.stream>>>(V, ld, r0, r1, amax, first);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

void sign_rows(Ctx& ctx, int k, const double* V, long long ld, long long r0, long long r1, const double* amax,
               const long long* first, double* flip) {
  if (k <= 0) return;
  sign_rows_kernel<<<1, 256, 0, ctx.stream>>>(V, ld, k, r0, r1, amax, first, flip);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

void negate_rows(Ctx& ctx, int k, double* V, long long ld, long long r0, long long r1, const double* flip) {
  if (k <= 0 || r1 <= r0) return;
  negate_rows_kernel<<<dim3(grid_for(r1 - r0, 4), k), 256, 0, ctx.stream>>>(V, ld, r0, r1, flip);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

}  // namespace paro_b200
