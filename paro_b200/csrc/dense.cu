// K x K dense kernels of Step 4, one warp per launch (compiled -fmad=false).
//
// The reference solves the projected pencil with Cholesky + cyclic Jacobi +
// back-substitution (dense_sym_geneig, proj/src/linalg.cpp:341-393;
// jacobi_eig :243-302; cholesky :307-323; fix_sign :229-241). These kernels
// perform the same floating-point operations in the same order (inner loops
// that are independent across rows/columns are spread over the 32 lanes; the
// order-sensitive sums run on one lane), so for an identical pencil the
// eigenpairs are bit-identical to the CPU reference. K is at most a few
// hundred, so a single warp keeps the whole solve in one launch.
#include "dense.hpp"

namespace paro_b200 {

namespace {

__device__ __forceinline__ double& at(double* m, int n, int i, int j) { return m[i * n + j]; }

__device__ void warp_fill(double* m, int count, double v) {
  for (int i = threadIdx.x; i < count; i += 32) m[i] = v;
  __syncwarp();
}

// cholesky (linalg.cpp:307-323) on lane 0; returns false on a non-positive pivot.
__device__ bool warp_cholesky(int n, const double* b, double* l) {
  warp_fill(l, n * n, 0.0);
  int ok = 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n && ok; ++i) {
      for (int j = 0; j <= i; ++j) {
        double s = b[i * n + j];
        for (int k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
        if (i == j) {
          if (s <= 0.0) {
            ok = 0;
            break;
          }
          l[i * n + i] = sqrt(s);
        } else {
          l[i * n + j] = s / l[j * n + j];
        }
      }
    }
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  __syncwarp();
  return ok != 0;
}

// check_symmetric (linalg.cpp:325-337)
__device__ bool warp_symmetric(int n, const double* m) {
  int ok = 1;
  if (threadIdx.x == 0) {
    double scale = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) scale = fmax(scale, fabs(m[i * n + j]));
    for (int i = 0; i < n && ok; ++i)
      for (int j = i + 1; j < n; ++j)
        if (fabs(m[i * n + j] - m[j * n + i]) > 1e-12 * fmax(1.0, scale)) {
          ok = 0;
          break;
        }
  }
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// fix_sign (linalg.cpp:229-241) on a strided vector, single thread.
__device__ void fix_sign_seq(int n, double* v, int stride) {
  double amax = 0.0;
  for (int i = 0; i < n; ++i) amax = fmax(amax, fabs(v[i * stride]));
  if (amax == 0.0) return;
  for (int i = 0; i < n; ++i) {
    const double x = v[i * stride];
    if (fabs(x) > 1e-12 * amax) {
      if (x < 0.0)
        for (int k = 0; k < n; ++k) v[k * stride] = -v[k * stride];
      return;
    }
  }
}

// jacobi_eig (linalg.cpp:243-302): a (n x n, destroyed), v (n x n) eigenvectors,
// vals sorted ascending, vecs columns reordered accordingly into `out`.
// Block-wide: every thread derives (c, s) of a rotation from the same shared
// values (identical arithmetic, so identical results), then thread k applies
// the rotation to row/column k of a and row k of v; the 2x2 block (p, q) is
// done by one thread in the reference's order (column pass, then row pass).
// Elements touched by different threads within a rotation are disjoint, so
// one barrier per rotation keeps the reference's operation sequence.
__device__ void block_jacobi(int n, double* a_g, double* v_g, double tol, int max_sweeps, double* vals, double* out,
                             int* order) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // the rotation sequence is latency-bound: run it on shared-memory copies
  // when the launch provided 2 n^2 doubles of dynamic shared memory
  extern __shared__ double jsm[];
  __shared__ double bc[2];
  unsigned dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  double* a = a_g;
  double* v = v_g;
  if (dyn >= 2u * n * n * sizeof(double)) {
    a = jsm;
    v = jsm + n * n;
    for (int i = tid; i < n * n; i += nt) a[i] = a_g[i];
  }
  for (int i = tid; i < n * n; i += nt) v[i] = 0.0;
  __syncthreads();
  for (int i = tid; i < n; i += nt) v[i * n + i] = 1.0;
  if (tid == 0) {
    double fro = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) fro += a[i * n + j] * a[i * n + j];
    fro = sqrt(fro);
    if (fro == 0.0) fro = 1.0;
    bc[0] = fro;
  }
  __syncthreads();
  const double fro = bc[0];
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) {
      double off = 0.0;
      for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) off += 2.0 * a[i * n + j] * a[i * n + j];
      bc[1] = off;
    }
    __syncthreads();
    if (sqrt(bc[1]) <= tol * fro) break;
    for (int p = 0; p + 1 < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (fabs(apq) <= 1e-300) continue;
        const double tau = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = t * c;
        for (int k = tid; k < n; k += nt) {
          if (k == p) {  // the (p, q) block: column pass, then row pass
            double x0 = a[p * n + p], x1 = a[p * n + q];
            a[p * n + p] = c * x0 - s * x1;
            a[p * n + q] = s * x0 + c * x1;
            x0 = a[q * n + p], x1 = a[q * n + q];
            a[q * n + p] = c * x0 - s * x1;
            a[q * n + q] = s * x0 + c * x1;
            x0 = a[p * n + p], x1 = a[q * n + p];
            a[p * n + p] = c * x0 - s * x1;
            a[q * n + p] = s * x0 + c * x1;
            x0 = a[p * n + q], x1 = a[q * n + q];
            a[p * n + q] = c * x0 - s * x1;
            a[q * n + q] = s * x0 + c * x1;
          } else if (k != q) {
            const double akp = a[k * n + p], akq = a[k * n + q];
            a[k * n + p] = c * akp - s * akq;
            a[k * n + q] = s * akp + c * akq;
            const double apk = a[p * n + k], aqk = a[q * n + k];
            a[p * n + k] = c * apk - s * aqk;
            a[q * n + k] = s * apk + c * aqk;
          }
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
        __syncthreads();
      }
    }
  }
  // ascending order of the diagonal (stable for exact ties)
  if (tid == 0) {
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 1; i < n; ++i) {
      const int oi = order[i];
      const double key = a[oi * n + oi];
      int j = i - 1;
      while (j >= 0 && a[order[j] * n + order[j]] > key) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = oi;
    }
  }
  __syncthreads();
  for (int j = tid; j < n; j += nt) vals[j] = a[order[j] * n + order[j]];
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx % n;
    out[i * n + j] = v[i * n + order[j]];
  }
  __syncthreads();
}

}  // namespace

// dense_sym_geneig (linalg.cpp:341-393). A, B row-major n x n (read-only);
// vals (n), X row-major n x n (columns = B-orthonormal eigenvectors).
__device__ int dense_sym_geneig_warp(int n, const double* A, const double* B, double* vals, double* X,
                                     const DenseScratch& w) {
  // launched with a whole block: the order-sensitive / small parts run on warp
  // 0, the Jacobi rotations on every thread
  const int lane = threadIdx.x;
  __shared__ int st_sh;
  if (threadIdx.x < 32) {
    int st = kOk;
    if (!warp_symmetric(n, A) || !warp_symmetric(n, B)) st = kPencil;
    else if (!warp_cholesky(n, B, w.l)) st = kPencil;
    if (st == kOk) {
      // W = L^{-1} A, column j independent
      for (int j = lane; j < n; j += 32) {
        for (int i = 0; i < n; ++i) {
          double s = A[i * n + j];
          for (int k = 0; k < i; ++k) s -= w.l[i * n + k] * w.w[k * n + j];
          w.w[i * n + j] = s / w.l[i * n + i];
        }
      }
      __syncwarp();
      // C = W L^{-T}, row i independent
      for (int i = lane; i < n; i += 32) {
        for (int j = 0; j < n; ++j) {
          double s = w.w[i * n + j];
          for (int k = 0; k < j; ++k) s -= w.c[i * n + k] * w.l[j * n + k];
          w.c[i * n + j] = s / w.l[j * n + j];
        }
      }
      __syncwarp();
      for (int idx = lane; idx < n * n; idx += 32) {
        const int i = idx / n, j = idx % n;
        if (j > i) {
          const double avg = 0.5 * (w.c[i * n + j] + w.c[j * n + i]);
          w.a[i * n + j] = avg;
          w.a[j * n + i] = avg;
        } else if (j == i) {
          w.a[i * n + i] = w.c[i * n + i];
        }
      }
    }
    if (lane == 0) st_sh = st;
  }
  __syncthreads();
  if (st_sh != kOk) return st_sh;
  block_jacobi(n, w.a, w.v, 1e-12, 60, vals, X, w.order);
  if (threadIdx.x < 32) {
    // x = L^{-T} y per column, then fix_sign
    for (int col = lane; col < n; col += 32) {
      for (int ii = n - 1; ii >= 0; --ii) {
        double s = X[ii * n + col];
        for (int k = ii + 1; k < n; ++k) s -= w.l[k * n + ii] * X[k * n + col];
        X[ii * n + col] = s / w.l[ii * n + ii];
      }
      fix_sign_seq(n, X + col, n);
    }
  }
  __syncthreads();
  return kOk;
}

__global__ void geneig_kernel(int n, const double* A, const double* B, double* vals, double* X, DenseScratch w,
                              int* status) {
  const int st = dense_sym_geneig_warp(n, A, B, vals, X, w);
  if (threadIdx.x == 0) *status = st;
}

// ---------------------------------------------------------------------------
// Orthonormalisation of the candidate span from its B-Gram matrix.
//
// In exact arithmetic the two-pass modified Gram-Schmidt of b_orthonormalize
// (linalg.cpp:409-439) equals an ordered Cholesky of G = U^T B U: the
// projected B-norm of candidate j against the accepted ones is the pivot
// L_jj and its original B-norm is sqrt(G_jj); a candidate is dropped when
// pivot <= drop_tol * original, and later candidates are orthogonalised only
// against accepted ones (the dropped row/column is skipped).
//
// G: column-major K x K raw Gram (u_i^T B u_j). Outputs: C (column-major
// K x k) with Q = U C B-orthonormal in exact arithmetic, acc[k] accepted
// indices, *kout, and min_ratio = smallest pivot/original ratio seen (the
// host re-checks near-threshold decisions with an explicit CGS2 pass).
__global__ void ortho_from_gram_kernel(int K, const double* G, double drop_tol, int allow_drop, double* C,
                                       int* acc, int* kout, double* min_ratio, DenseScratch w, int* status) {
  const int lane = threadIdx.x;
  // symmetric Gram (row-major) in w.a
  for (int idx = lane; idx < K * K; idx += 32) {
    const int i = idx / K, j = idx % K;
    w.a[i * K + j] = 0.5 * (G[i + j * K] + G[j + i * K]);
  }
  warp_fill(w.l, K * K, 0.0);
  int k = 0;
  int st = kOk;
  double rmin = 1e300;
  if (lane == 0) {
    double* lrow = w.w;  // tentative row
    for (int j = 0; j < K; ++j) {
      const double g = w.a[j * K + j];
      const double orig = sqrt(fmax(0.0, g));
      if (!(orig > 0.0)) {
        if (!allow_drop) {
          st = kPencil;
          break;
        }
        rmin = 0.0;
        continue;
      }
      double d2 = g;
      for (int c = 0; c < k; ++c) {
        double s = w.a[j * K + acc[c]];
        for (int m = 0; m < c; ++m) s -= lrow[m] * w.l[c * K + m];
        lrow[c] = s / w.l[c * K + c];
        d2 -= lrow[c] * lrow[c];
      }
      const double nb = sqrt(fmax(0.0, d2));
      const double ratio = nb / orig;
      rmin = fmin(rmin, ratio);
      if (nb <= drop_tol * orig) {
        if (!allow_drop) {
          st = kPencil;
          break;
        }
        continue;
      }
      for (int c = 0; c < k; ++c) w.l[k * K + c] = lrow[c];
      w.l[k * K + k] = nb;
      acc[k] = j;
      ++k;
    }
  }
  k = __shfl_sync(0xffffffffu, k, 0);
  st = __shfl_sync(0xffffffffu, st, 0);
  __syncwarp();
  // Linv = L^{-1} (lower), column j independent
  for (int j = lane; j < k; j += 32) {
    for (int i = 0; i < k; ++i) {
      double s = i == j ? 1.0 : 0.0;
      for (int m = j; m < i; ++m) s -= w.l[i * K + m] * w.c[m * K + j];
      w.c[i * K + j] = i < j ? 0.0 : s / w.l[i * K + i];
    }
  }
  __syncwarp();
  // C[acc[i], j] = Linv^T[i][j] = Linv[j][i]
  for (int idx = lane; idx < K * k; idx += 32) {
    const int r = idx % K, j = idx / K;
    C[r + j * K] = 0.0;
  }
  __syncwarp();
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx / k, j = idx % k;
    C[acc[i] + j * K] = w.c[j * K + i];
  }
  if (lane == 0) {
    *kout = k;
    *min_ratio = rmin;
    *status = st;
  }
}

// Second CholQR pass on G2 = Q1^T B Q1 (k x k, column-major): L2 = chol(G2),
// C2 = L2^{-T} (column-major k x k), Bt = L2^{-1} G2 L2^{-T} (row-major, ~I).
__global__ void second_pass_kernel(int k, const double* G2, double* C2, double* Bt, DenseScratch w, int* status) {
  const int lane = threadIdx.x;
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx / k, j = idx % k;
    w.a[i * k + j] = 0.5 * (G2[i + j * k] + G2[j + i * k]);
  }
  __syncwarp();
  if (!warp_cholesky(k, w.a, w.l)) {
    if (lane == 0) *status = kPencil;
    return;
  }
  // Linv
  for (int j = lane; j < k; j += 32) {
    for (int i = 0; i < k; ++i) {
      double s = i == j ? 1.0 : 0.0;
      for (int m = j; m < i; ++m) s -= w.l[i * k + m] * w.c[m * k + j];
      w.c[i * k + j] = i < j ? 0.0 : s / w.l[i * k + i];
    }
  }
  __syncwarp();
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx / k, j = idx % k;
    C2[i + j * k] = w.c[j * k + i];  // L2^{-T}
  }
  // Bt = Linv * Gs * Linv^T
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m <= i; ++m) s += w.c[i * k + m] * w.a[m * k + j];
    w.w[i * k + j] = s;
  }
  __syncwarp();
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m <= j; ++m) s += w.w[i * k + m] * w.c[j * k + m];
    Bt[i * k + j] = s;
  }
  __syncwarp();
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx / k, j = idx % k;
    if (j > i) {
      const double avg = 0.5 * (Bt[i * k + j] + Bt[j * k + i]);
      Bt[i * k + j] = avg;
      Bt[j * k + i] = avg;
    }
  }
  if (lane == 0) *status = kOk;
}

// One-pass basis change: Bt = sym(C^T sym(G) C) (row-major k x k) for the raw
// Gram G = U^T B U and C = L^{-T} of its ordered Cholesky (both column-major
// k x k): the B-Gram of Q = U C formed in K x K arithmetic, which is as
// accurate as forming Q when the candidates are well conditioned (step4.py).
__global__ void congruence_kernel(int k, const double* G, const double* Cm, double* Bt, DenseScratch w) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m < k; ++m) s += 0.5 * (G[i + m * k] + G[m + i * k]) * Cm[m + j * k];
    w.w[i * k + j] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m < k; ++m) s += Cm[m + i * k] * w.w[m * k + j];
    w.c[i * k + j] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    Bt[i * k + j] = i == j ? w.c[idx] : 0.5 * (w.c[i * k + j] + w.c[j * k + i]);
  }
}

// Pencil in an explicitly orthonormalised basis Q (paro.cpp:143-150):
// At = sym(Q^T A Q), Bt = sym(Q^T B Q) (column-major inputs), then
// dense_sym_geneig; Y (column-major k x k) = X.
__global__ void pencil_direct_kernel(int k, const double* GA, const double* GB, double* vals, double* Y, double* At,
                                     double* Bt, double* X, DenseScratch w, int* status) {
  const int lane = threadIdx.x;
  if (lane < 32)
    for (int idx = lane; idx < k * k; idx += 32) {
      const int i = idx / k, j = idx % k;
      At[i * k + j] = 0.5 * (GA[i + j * k] + GA[j + i * k]);
      Bt[i * k + j] = 0.5 * (GB[i + j * k] + GB[j + i * k]);
    }
  __syncthreads();
  const int st = dense_sym_geneig_warp(k, At, Bt, vals, X, w);
  if (st != kOk) {
    if (lane == 0) *status = st;
    return;
  }
  if (lane < 32)
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx % k, j = idx / k;
    Y[i + j * k] = X[i * k + j];
  }
  if (lane == 0) *status = kOk;
}

// Projected pencil in the orthonormal basis Q = Q1 C2 and its solve:
// At = C2^T sym(GA) C2 (GA = Q1^T A Q1, column-major), symmetrised like the
// reference's pencil (paro.cpp:143-150); then dense_sym_geneig(At, Bt);
// Y = C2 X (column-major k x k) lifts the Ritz vectors onto Q1.
__global__ void pencil_kernel(int k, const double* GA, const double* C2, const double* Bt, double* vals, double* Y,
                              double* At, double* X, DenseScratch w, int* status) {
  const int lane = threadIdx.x, nt = blockDim.x;
  // T = sym(GA) C2  (row-major); each entry one thread, fixed-order sums
  for (int idx = lane; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m < k; ++m) s += 0.5 * (GA[i + m * k] + GA[m + i * k]) * C2[m + j * k];
    w.w[i * k + j] = s;
  }
  __syncthreads();
  for (int idx = lane; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m < k; ++m) s += C2[m + i * k] * w.w[m * k + j];
    At[i * k + j] = s;
  }
  __syncthreads();
  for (int idx = lane; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    if (j > i) {
      const double avg = 0.5 * (At[i * k + j] + At[j * k + i]);
      At[i * k + j] = avg;
      At[j * k + i] = avg;
    }
  }
  __syncthreads();
  const int st = dense_sym_geneig_warp(k, At, Bt, vals, X, w);
  if (st != kOk) {
    if (lane == 0) *status = st;
    return;
  }
  for (int idx = lane; idx < k * k; idx += nt) {
    const int i = idx % k, j = idx / k;
    double s = 0.0;
    for (int m = 0; m < k; ++m) s += C2[i + m * k] * X[m * k + j];
    Y[i + j * k] = s;
  }
  if (lane == 0) *status = kOk;
}

size_t dense_jacobi_smem(int n) {
  const size_t bytes = 2ull * n * n * sizeof(double);
  return bytes <= 220u * 1024u ? bytes : 0;
}

void dense_configure() {
  static bool done = false;
  if (done) return;
  const int mx = 220 * 1024;  // dense_jacobi_smem() caps at 220 KB; leaves room for the static shared variables
  PARO_CUDA(cudaFuncSetAttribute(geneig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  PARO_CUDA(cudaFuncSetAttribute(pencil_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  PARO_CUDA(cudaFuncSetAttribute(pencil_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  done = true;
}

}  // namespace paro_b200
