// General sparse operators on the device: the reference's
// SparseOperator (proj/include/paro/linalg.hpp:14-50) as CSR, for matrices
// that are not the uniform-mesh Kuhn stencil (adapted meshes, other
// discretisations). Batched apply, add_scaled, cg_solve and
// source_solve_step with the reference's semantics; the uniform-mesh hot
// path stays on the stencil kernels.
#pragma once

#include <cstdint>
#include <vector>

#include "ctx.hpp"
#include "solver.hpp"

namespace paro_b200 {

struct CsrOp {
  long long n = 0;
  long long nnz = 0;
  long long* rows = nullptr;  // device, n + 1
  int* cols = nullptr;        // device, nnz (ascending within a row)
  double* vals = nullptr;     // device, nnz
  // host copy of the pattern (add_scaled checks identical structures, linalg.cpp:120-125)
  std::vector<long long> h_rows;
  std::vector<int> h_cols;
  ~CsrOp();
};

// Upload (host arrays, the reference's size_t row offsets / uint32 columns).
// Validates sizes, column range and ascending columns per row.
void csr_create(Ctx& ctx, long long n, const size_t* rows, const uint32_t* cols, const double* vals, CsrOp& out);
// a += s b (identical patterns, else InvalidArgument)
void csr_add_scaled(Ctx& ctx, CsrOp& a, const CsrOp& b, double s);
// Y = A X for K columns (device, column stride ld), row sums in ascending column order (matvec, linalg.cpp:88-94)
void csr_apply(Ctx& ctx, const CsrOp& a, int K, const double* x, long long ld, double* y);
// cg_solve (linalg.cpp:143-223) for K right-hand sides (x0 may be null)
int csr_cg_solve(Ctx& ctx, const CsrOp& a, int K, const double* rhs, const double* x0, long long ld, double tol,
                 unsigned long long max_iter, bool throw_on_max, double* x, SolveReport* rep);
// source_solve_step (paro.cpp:81-119): (A + sigma B) u_half = (lambda + sigma) B u, x0 = u, one retry
int csr_source_solve(Ctx& ctx, const CsrOp& a, const CsrOp& b, double sigma, int K, const double* u, long long ld,
                     const double* lambdas, double tol, unsigned long long max_iter, double* out, SolveReport* rep);

}  // namespace paro_b200
