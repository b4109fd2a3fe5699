// Per-column finalize kernels of the batched Jacobi-PCG (cg_solve,
// linalg.cpp:143-223), shared by the stencil (solver.cu) and the general CSR
// (csr.cu) solvers: fixed-order sums of per-CTA partials, then the scalar
// recurrences (alpha, beta, stop tests, NotSpd / IterationLimit) on the device.
// partials layout: [K][3][nblk].
#pragma once

#include "common.cuh"

namespace paro_b200 {
namespace {

constexpr int kFinThreads = 256;

__device__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += sh[w];
  }
  __syncthreads();
  return s;  // valid on thread 0
}

// Fixed-order sum of the per-CTA partials of column c, quantity q.
__device__ double sum_partials(const double* partials, int c, int q, int nblk, double* sh) {
  double s = 0.0;
  const double* p = partials + (static_cast<long long>(c) * 3 + q) * nblk;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) s += p[i];
  return block_sum(s, sh);
}

enum FinMode { kFinSetup = 0, kFinK1 = 1, kFinK2 = 2 };

// flags[0]: non-positive diagonal; flags[1]: a column hit NotSpd (abort the batch when flags[2] != 0)
__global__ void fin_kernel(int mode, CgColumn* cols, const double* partials, int nblk, int* flags) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  CgColumn& col = cols[c];
  if (!col.active) return;
  if (flags[2] && flags[1]) {  // another column's NotSpd already fixes this step's outcome
    if (threadIdx.x == 0) {
      col.active = 0;
      col.status = kAborted;
    }
    return;
  }
  const int* diag_bad = flags;
  if (mode == kFinSetup) {
    const double bb = sum_partials(partials, c, 0, nblk, sh);
    const double rz = sum_partials(partials, c, 1, nblk, sh);
    const double rr = sum_partials(partials, c, 2, nblk, sh);
    if (threadIdx.x != 0) return;
    const double bnorm = sqrt(bb);
    col.bnorm = bnorm;
    col.it = 0;
    if (bnorm == 0.0) {  // linalg.cpp:158-162: x = 0, converged
      col.converged = 1;
      col.active = 0;
      col.first = 2;     // marks "zero the solution"
      col.rnorm = 0.0;
      return;
    }
    if (*diag_bad) {     // linalg.cpp:165-167
      col.status = kNotSpd;
      col.active = 0;
      return;
    }
    col.rz = rz;
    col.rnorm = sqrt(rr);
    col.first = 1;
    if (col.rnorm / bnorm <= col.tol) {
      col.converged = 1;
      col.active = 0;
    } else if (col.max_iter == 0) {
      col.status = kIterationLimit;
      col.active = 0;
    }
  } else if (mode == kFinK1) {
    const double pq = sum_partials(partials, c, 0, nblk, sh);
    if (threadIdx.x != 0) return;
    col.pq = pq;
    if (pq <= 0.0) {  // linalg.cpp:200
      col.status = kNotSpd;
      col.active = 0;
      atomicExch(flags + 1, 1);
      return;
    }
    col.alpha_prev = col.alpha;
    col.alpha = col.rz / pq;
  } else {
    const double rzn = sum_partials(partials, c, 0, nblk, sh);
    const double rr = sum_partials(partials, c, 1, nblk, sh);
    if (threadIdx.x != 0) return;
    col.beta = rzn / col.rz;  // linalg.cpp:207-209
    col.rz = rzn;
    col.rnorm = sqrt(rr);
    col.it += 1;
    col.first = 0;
    if (col.rnorm / col.bnorm <= col.tol) {
      col.converged = 1;
      col.active = 0;
    } else if (col.it >= col.max_iter) {
      col.status = kIterationLimit;
      col.active = 0;
    }
  }
}

__global__ void count_active_kernel(const CgColumn* cols, int K, int* out) {
  __shared__ int sh;
  if (threadIdx.x == 0) sh = 0;
  __syncthreads();
  int c = 0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) c += cols[i].active != 0;
  atomicAdd(&sh, c);
  __syncthreads();
  if (threadIdx.x == 0) *out = sh;
}

}  // namespace
}  // namespace paro_b200
