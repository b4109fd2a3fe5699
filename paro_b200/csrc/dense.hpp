// K x K dense kernels of Step 4 (see dense.cu).
#pragma once

#include "common.cuh"

namespace paro_b200 {

// Row-major K x K scratch matrices (global or shared memory) + an int order vector.
struct DenseScratch {
  double* a = nullptr;
  double* v = nullptr;
  double* l = nullptr;
  double* w = nullptr;
  double* c = nullptr;
  int* order = nullptr;
};

// threads of the pencil / geneig launches (the Jacobi rotations use all of
// them, the order-sensitive small parts warp 0)
constexpr int kDenseThreads = 128;

// dynamic shared memory for a kernel running the Jacobi rotations on n x n (0 = global)
size_t dense_jacobi_smem(int n);
void dense_configure();

__global__ void geneig_kernel(int n, const double* A, const double* B, double* vals, double* X, DenseScratch w,
                              int* status);
__global__ void ortho_from_gram_kernel(int K, const double* G, double drop_tol, int allow_drop, double* C, int* acc,
                                       int* kout, double* min_ratio, DenseScratch w, int* status);
__global__ void second_pass_kernel(int k, const double* G2, double* C2, double* Bt, DenseScratch w, int* status);
__global__ void congruence_kernel(int k, const double* G, const double* Cm, double* Bt, DenseScratch w);
__global__ void pencil_direct_kernel(int k, const double* GA, const double* GB, double* vals, double* Y, double* At,
                                     double* Bt, double* X, DenseScratch w, int* status);
__global__ void pencil_kernel(int k, const double* GA, const double* C2, const double* Bt, double* vals, double* Y,
                              double* At, double* X, DenseScratch w, int* status);

}  // namespace paro_b200
