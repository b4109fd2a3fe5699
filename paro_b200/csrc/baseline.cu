// baseline_geneig (proj/src/linalg.cpp:615-623) on the device: the lowest
// `count` eigenpairs of the pencil (A, B), the reference's initial-guess
// eigensolver (initial_guess, paro.cpp:63-79), without its 50,000-dof cap.
//
// The reference runs Eigen's dense solver up to 5,000 dofs and otherwise the
// shift-inverted block subspace iteration baseline_subspace (linalg.cpp:
// 531-611). This is that iteration on the device kernels of the hot path:
//   block = min(n, count + max(2, count / 4)) Gaussian columns (seeded);
//   repeat: Y = (A + sigma B)^{-1} B X   (batched Jacobi-PCG, tol 1e-12,
//                                         max_iter 20 n + 1000, x0 = X;
//                                         sigma 0 -> 1 -> 2 sigma + 1 on NotSpd)
//           X = Ritz vectors of span(Y)  (rayleigh_ritz: B-orthonormalise,
//                                         projected pencil, lift, fix_sign)
//   until ||A x_j - lambda_j B x_j|| <= 1e-9 max(1, max|A| + |lambda_j| max|B|)
//   for the first `count` pairs (linalg.cpp:462-467, 588-603).
// Both routes converge to the same eigenpairs (unique up to the sign that
// fix_sign fixes, for simple eigenvalues), so parity is stated on them, not on
// the random start (the reference draws mt19937_64 normals; here SplitMix64 +
// Box-Muller).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.hpp"
#include "ritz.hpp"
#include "solver.hpp"

namespace paro_b200 {

namespace {

struct LocalBuf : DevBuf {  // released when the call returns
  ~LocalBuf() { release(); }
};

unsigned long long splitmix_host(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ unsigned long long splitmix(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// standard normal values (Box-Muller on two SplitMix64 uniforms per entry)
__global__ void gauss_kernel(double* X, long long count, unsigned long long seed) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long a = splitmix(seed ^ (2ull * i));
    const unsigned long long b = splitmix(seed ^ (2ull * i + 1ull));
    const double u1 = ((a >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = (b >> 11) * 0x1.0p-53;        // [0, 1)
    X[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

// out[j] = sum_i (AX[j][i] - lambda_j BX[j][i])^2, one block per column
__global__ void resid_kernel(const double* AX, const double* BX, long long n, const double* lam, double* out) {
  const int j = blockIdx.x;
  const double l = lam[j];
  const double* a = AX + j * n;
  const double* b = BX + j * n;
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = a[i] - l * b[i];
    s += d * d;
  }
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sh[w];
    out[j] = t;
  }
}

// max |v| over len entries (non-negative doubles compare as their bit patterns)
__global__ void maxabs_kernel(const double* v, long long len, unsigned long long* out) {
  double m = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(v[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// out = fl(a + fl(sigma b)) per coefficient (SparseOperator::add_scaled, linalg.cpp:120-125)
__global__ void shift_coef_kernel(const double* a, const double* b, const double* bw, double sigma, long long n,
                                  double* out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < 8 * n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double av = a ? a[i] : 0.0;
    const double bv = b ? b[i] : bw[i / n];
    out[i] = __dadd_rn(av, __dmul_rn(sigma, bv));
  }
}

// largest |entry| of an operator's matrix (residual_scale, linalg.cpp:462-467)
double op_maxabs(Ctx& ctx, const Op& a) {
  if (!a.var) {
    double m = 0.0;
    for (int o = 0; o < kSlots; ++o) m = std::max(m, std::fabs(a.w[o]));
    return m;
  }
  unsigned long long* d = ctx.ws_small3.get<unsigned long long>(1);
  PARO_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), ctx.stream));
  maxabs_kernel<<<148 * 4, 256, 0, ctx.stream>>>(a.coef, static_cast<long long>(kSlots) * a.n, d);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
  unsigned long long h = 0;
  PARO_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
  double m;
  std::memcpy(&m, &h, sizeof(m));
  return m;
}

}  // namespace

int baseline_geneig(Ctx& ctx, const Op& A, const Op& B, int count, unsigned long long max_iter,
                    unsigned long long seed, double* vals_host, double* V, long long ldv, int* iters_out) {
  ctx.check_grid();
  const long long n = ctx.grid.n;
  if (count <= 0 || count > n) throw ParoError(kInvalidArgument, "baseline: bad eigenpair count");
  if (ldv != n) throw ParoError(kInvalidArgument, "baseline: vectors must be contiguous (ld == n)");
  const int block = static_cast<int>(std::min<long long>(n, count + std::max(2, count / 4)));
  cudaStream_t st = ctx.stream;
  LocalBuf bx, by, br, bshift, bsmall;
  double* X = bx.get<double>(static_cast<size_t>(block) * n);
  double* Y = by.get<double>(static_cast<size_t>(block) * n);
  double* R = br.get<double>(static_cast<size_t>(block) * n);
  unsigned long long draws = 0;
  auto noise = [&](double* dst, long long len) {
    gauss_kernel<<<148 * 8, 256, 0, st>>>(dst, len, splitmix_host(seed + draws++));
    PARO_CUDA(cudaGetLastError());
    ++ctx.launches;
  };
  noise(X, static_cast<long long>(block) * n);

  const double amax = op_maxabs(ctx, A), bmax = op_maxabs(ctx, B);
  std::vector<double> lam(block), res(count);
  double* dlam = bsmall.get<double>(2 * static_cast<size_t>(block) + kSlots);
  double* dres = dlam + block;
  double* bw = dres + block;  // 8 stencil weights
  double sigma = 0.0;
  const double tol = 1e-12;
  const unsigned long long cg_max = 20ull * static_cast<unsigned long long>(n) + 1000ull;

  for (unsigned long long iter = 0; iter < max_iter; ++iter) {
    // Y = (A + sigma B)^{-1} B X (linalg.cpp:548-566)
    Op shifted = A;
    if (sigma != 0.0) {
      double* c = bshift.get<double>(static_cast<size_t>(kSlots) * n);
      if (A.var || B.var) {
        PARO_CUDA(cudaMemcpyAsync(bw, B.w, sizeof(double) * kSlots, cudaMemcpyHostToDevice, st));
        shift_coef_kernel<<<148 * 8, 256, 0, st>>>(A.var ? A.coef : nullptr, B.var ? B.coef : nullptr, bw, sigma, n, c);
        PARO_CUDA(cudaGetLastError());
        ++ctx.launches;
        if (!A.var) {  // a constant A has no per-dof coefficients: fill them from its weights
          std::vector<double> sh(kSlots);
          for (int o = 0; o < kSlots; ++o) sh[o] = A.w[o];
          PARO_CUDA(cudaMemcpyAsync(bw, sh.data(), sizeof(double) * kSlots, cudaMemcpyHostToDevice, st));
          shift_coef_kernel<<<148 * 8, 256, 0, st>>>(c, nullptr, bw, 1.0, n, c);  // c += A (once, exact for B var)
          ++ctx.launches;
        }
        shifted.var = true;
        shifted.coef = c;
        shifted.owns = false;
      } else {
        for (int o = 0; o < kSlots; ++o) shifted.w[o] = A.w[o] + sigma * B.w[o];
      }
    }
    apply_op(ctx, B, nullptr, 0.0, block, X, n, R, n);
    const int s = cg_solve(ctx, shifted, block, R, X, n, tol, cg_max, true, Y, nullptr);
    if (s == kNotSpd) {
      sigma = sigma == 0.0 ? 1.0 : 2.0 * sigma + 1.0;
      if (sigma > 1e12) {
        ctx.err = "baseline: shift escalation exceeded 1e12";
        return kNotSpd;
      }
      --iter;
      continue;
    }
    if (s != kOk) {
      ctx.err = "baseline: " + ctx.err;
      return s;
    }
    // Ritz pairs of span(Y) (linalg.cpp:568-596); a collapsed span gets fresh
    // random columns, as the reference tops the basis up (linalg.cpp:569-575)
    int k = 0, rs = kOk;
    double defect = 0.0;
    // baseline_subspace (linalg.cpp:568-596) has no orthonormality certificate
    RitzInfo no_cert;
    no_cert.certify = false;
    for (int tries = 0; tries < 8; ++tries) {
      rs = rayleigh_ritz(ctx, A, B, block, Y, n, static_cast<size_t>(block), 1e-14, lam.data(), X, n, &k, &defect,
                         &no_cert);
      if (rs != kDegenerateSpan && rs != kEmptyBasis) break;
      noise(Y + static_cast<long long>(block - 1 - tries % block) * n, n);
    }
    if (rs != kOk) return rs;
    // residuals of the requested pairs (linalg.cpp:588-603)
    apply_op(ctx, A, nullptr, 0.0, count, X, n, Y, n);
    apply_op(ctx, B, nullptr, 0.0, count, X, n, R, n);
    PARO_CUDA(cudaMemcpyAsync(dlam, lam.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
    resid_kernel<<<count, 512, 0, st>>>(Y, R, n, dlam, dres);
    PARO_CUDA(cudaGetLastError());
    ++ctx.launches;
    PARO_CUDA(cudaMemcpyAsync(res.data(), dres, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    PARO_CUDA(cudaStreamSynchronize(st));
    bool done = true;
    for (int j = 0; j < count && done; ++j)
      done = std::sqrt(res[j]) <= 1e-9 * std::max(1.0, amax + std::fabs(lam[j]) * bmax);
    if (done) {
      for (int j = 0; j < count; ++j) vals_host[j] = lam[j];
      PARO_CUDA(cudaMemcpyAsync(V, X, sizeof(double) * count * n, cudaMemcpyDeviceToDevice, st));
      PARO_CUDA(cudaStreamSynchronize(st));
      if (iters_out) *iters_out = static_cast<int>(iter + 1);
      return kOk;
    }
  }
  ctx.err = "baseline: subspace iteration did not converge";
  return kIterationLimit;
}

}  // namespace paro_b200
