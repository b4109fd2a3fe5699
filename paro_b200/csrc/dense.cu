// K x K dense kernels of Step 4, one block per launch (compiled -fmad=false).
//
// The reference solves the projected pencil with Cholesky + cyclic Jacobi +
// back-substitution (dense_sym_geneig, proj/src/linalg.cpp:341-393;
// jacobi_eig :243-302; cholesky :307-323; fix_sign :229-241). These kernels
// perform the same floating-point operations in the same order (inner loops
// that are independent across rows/columns are spread over the threads; the
// order-sensitive sums stay sequential), so for an identical pencil the
// eigenpairs are bit-identical to the CPU reference. K is at most a few
// hundred, so a single block keeps the whole solve in one launch: rows /
// columns that are independent in the reference's loops go to different
// threads, every element keeps its own summation order.
#include "dense.hpp"

namespace paro_b200 {

namespace {

// cholesky (linalg.cpp:307-323), block-wide; returns false on a non-positive
// pivot. Column by column: once columns < j are final, every row i >= j forms
// s = b_ij - sum_{k<j} l_ik l_jk with k ascending, the reference's own sum
// for that element, on its own thread.
__device__ bool block_cholesky(int n, const double* b, double* l) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ int chol_ok;
  for (int i = tid; i < n * n; i += nt) l[i] = 0.0;
  if (tid == 0) chol_ok = 1;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    for (int i = j + tid; i < n; i += nt) {
      double s = b[i * n + j];
      for (int k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
      l[i * n + j] = s;
    }
    __syncthreads();
    if (tid == 0) {
      const double s = l[j * n + j];
      if (s <= 0.0) chol_ok = 0;
      else l[j * n + j] = sqrt(s);
    }
    __syncthreads();
    if (!chol_ok) return false;
    const double d = l[j * n + j];
    for (int i = j + 1 + tid; i < n; i += nt) l[i * n + j] = l[i * n + j] / d;
    __syncthreads();
  }
  return true;
}

// check_symmetric (linalg.cpp:325-337), block-wide (a max and an any: order-free)
__device__ bool block_symmetric(int n, const double* m) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double sym_max[32];
  double scale = 0.0;
  for (int i = tid; i < n * n; i += nt) scale = fmax(scale, fabs(m[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  if ((tid & 31) == 0) sym_max[tid >> 5] = scale;
  __syncthreads();
  scale = 0.0;
  for (int w = 0; w < (nt + 31) / 32; ++w) scale = fmax(scale, sym_max[w]);
  const double bar = 1e-12 * fmax(1.0, scale);
  int bad = 0;
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx % n;
    if (j > i && fabs(m[i * n + j] - m[j * n + i]) > bar) bad = 1;
  }
  return __syncthreads_or(bad) == 0;
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
  // launched with a whole block; every phase spreads the reference's
  // independent rows / columns over the threads
  const int tid = threadIdx.x, nt = blockDim.x;
  if (!block_symmetric(n, A) || !block_symmetric(n, B)) return kPencil;
  if (!block_cholesky(n, B, w.l)) return kPencil;
  // W = L^{-1} A, column j independent
  for (int j = tid; j < n; j += nt) {
    for (int i = 0; i < n; ++i) {
      double s = A[i * n + j];
      for (int k = 0; k < i; ++k) s -= w.l[i * n + k] * w.w[k * n + j];
      w.w[i * n + j] = s / w.l[i * n + i];
    }
  }
  __syncthreads();
  // C = W L^{-T}, row i independent
  for (int i = tid; i < n; i += nt) {
    for (int j = 0; j < n; ++j) {
      double s = w.w[i * n + j];
      for (int k = 0; k < j; ++k) s -= w.c[i * n + k] * w.l[j * n + k];
      w.c[i * n + j] = s / w.l[j * n + j];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx % n;
    if (j > i) {
      const double avg = 0.5 * (w.c[i * n + j] + w.c[j * n + i]);
      w.a[i * n + j] = avg;
      w.a[j * n + i] = avg;
    } else if (j == i) {
      w.a[i * n + i] = w.c[i * n + i];
    }
  }
  __syncthreads();
  block_jacobi(n, w.a, w.v, 1e-12, 60, vals, X, w.order);
  // x = L^{-T} y per column, then fix_sign
  for (int col = tid; col < n; col += nt) {
    for (int ii = n - 1; ii >= 0; --ii) {
      double s = X[ii * n + col];
      for (int k = ii + 1; k < n; ++k) s -= w.l[k * n + ii] * X[k * n + col];
      X[ii * n + col] = s / w.l[ii * n + ii];
    }
    fix_sign_seq(n, X + col, n);
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
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ int sh_k, sh_st, sh_serial;
  __shared__ double sh_rmin;
  // symmetric Gram (row-major) in w.a
  for (int idx = tid; idx < K * K; idx += nt) {
    const int i = idx / K, j = idx % K;
    w.a[i * K + j] = 0.5 * (G[i + j * K] + G[j + i * K]);
    w.l[idx] = 0.0;
  }
  if (tid == 0) {
    sh_k = 0;
    sh_st = kOk;
    sh_serial = 0;
    sh_rmin = 1e300;
  }
  __syncthreads();
  // Without drops (the usual case) the ordered Cholesky is a plain one: run it
  // column by column with row j on its own thread -- l_jc = (a_jc - sum_{m<c}
  // l_jm l_cm) / l_cc, d2_j -= l_jc^2 with c ascending, exactly the sequence
  // of the row loop below -- and fall back to that loop from scratch at the
  // first candidate that would be dropped.
  double* d2 = w.v;  // remaining squared B-norm per candidate
  for (int j = tid; j < K; j += nt) d2[j] = w.a[j * K + j];
  __syncthreads();
  for (int c = 0; c < K; ++c) {
    if (tid == 0) {
      const double g = w.a[c * K + c];
      const double orig = sqrt(fmax(0.0, g));
      if (!(orig > 0.0)) {
        sh_serial = 1;
      } else {
        const double nb = sqrt(fmax(0.0, d2[c]));
        sh_rmin = fmin(sh_rmin, nb / orig);
        if (nb <= drop_tol * orig) sh_serial = 1;
        else w.l[c * K + c] = nb;
      }
    }
    __syncthreads();
    if (sh_serial) break;
    const double lcc = w.l[c * K + c];
    for (int j = c + 1 + tid; j < K; j += nt) {
      double sv = w.a[j * K + c];
      for (int m = 0; m < c; ++m) sv -= w.l[j * K + m] * w.l[c * K + m];
      const double v = sv / lcc;
      w.l[j * K + c] = v;
      d2[j] -= v * v;
    }
    __syncthreads();
  }
  if (!sh_serial) {
    for (int j = tid; j < K; j += nt) acc[j] = j;
    if (tid == 0) sh_k = K;
  } else {
    // ordered Cholesky with drops, one candidate row after the other
    __syncthreads();
    for (int idx = tid; idx < K * K; idx += nt) w.l[idx] = 0.0;
    __syncthreads();
    if (tid == 0) {
      int k = 0, st = kOk;
      double rmin = 1e300;
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
        double dd = g;
        for (int c = 0; c < k; ++c) {
          double sv = w.a[j * K + acc[c]];
          for (int m = 0; m < c; ++m) sv -= lrow[m] * w.l[c * K + m];
          lrow[c] = sv / w.l[c * K + c];
          dd -= lrow[c] * lrow[c];
        }
        const double nb = sqrt(fmax(0.0, dd));
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
      sh_k = k;
      sh_st = st;
      sh_rmin = rmin;
    }
  }
  __syncthreads();
  const int k = sh_k;
  // Linv = L^{-1} (lower), column j independent
  for (int j = tid; j < k; j += nt) {
    for (int i = 0; i < k; ++i) {
      double sv = i == j ? 1.0 : 0.0;
      for (int m = j; m < i; ++m) sv -= w.l[i * K + m] * w.c[m * K + j];
      w.c[i * K + j] = i < j ? 0.0 : sv / w.l[i * K + i];
    }
  }
  // C[acc[i], j] = Linv^T[i][j] = Linv[j][i]
  for (int idx = tid; idx < K * k; idx += nt) C[idx] = 0.0;
  __syncthreads();
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    C[acc[i] + j * K] = w.c[j * K + i];
  }
  if (tid == 0) {
    *kout = k;
    *min_ratio = sh_rmin;
    *status = sh_st;
  }
}

// Second CholQR pass on G2 = Q1^T B Q1 (k x k, column-major): L2 = chol(G2),
// C2 = L2^{-T} (column-major k x k), Bt = L2^{-1} G2 L2^{-T} (row-major, ~I).
__global__ void second_pass_kernel(int k, const double* G2, double* C2, double* Bt, DenseScratch w, int* status) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    w.a[i * k + j] = 0.5 * (G2[i + j * k] + G2[j + i * k]);
  }
  __syncthreads();
  if (!block_cholesky(k, w.a, w.l)) {
    if (tid == 0) *status = kPencil;
    return;
  }
  // Linv
  for (int j = tid; j < k; j += nt) {
    for (int i = 0; i < k; ++i) {
      double s = i == j ? 1.0 : 0.0;
      for (int m = j; m < i; ++m) s -= w.l[i * k + m] * w.c[m * k + j];
      w.c[i * k + j] = i < j ? 0.0 : s / w.l[i * k + i];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    C2[i + j * k] = w.c[j * k + i];  // L2^{-T}
  }
  // Bt = Linv * Gs * Linv^T
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m <= i; ++m) s += w.c[i * k + m] * w.a[m * k + j];
    w.w[i * k + j] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    double s = 0.0;
    for (int m = 0; m <= j; ++m) s += w.w[i * k + m] * w.c[j * k + m];
    w.v[i * k + j] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < k * k; idx += nt) {
    const int i = idx / k, j = idx % k;
    Bt[i * k + j] = i == j ? w.v[idx] : 0.5 * (w.v[i * k + j] + w.v[j * k + i]);
  }
  if (tid == 0) *status = kOk;
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
