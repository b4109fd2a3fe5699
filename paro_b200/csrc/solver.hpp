// Device solvers behind the C ABI (host-callable, device pointers).
#pragma once

#include <vector>

#include "ctx.hpp"
#include "march.cuh"

namespace paro_b200 {

struct SolveReport {
  std::vector<unsigned long long> iterations;
  std::vector<double> residual;
  std::vector<int> status;        // final per-column status (after the retry, if any)
  std::vector<int> first_status;  // status of the first attempt
};

OpDev make_opdev(const Ctx& ctx, const Op& a, const Op* shift, double sigma);

// y = (A + sigma shift) x on the rows of planes [z0, z1) (default: all);
// x must hold valid values on planes z0 - 1 .. z1 (the stencil's reach)
void apply_op(Ctx& ctx, const Op& a, const Op* shift, double sigma, int K, const double* x, long long ldx,
              double* y, long long ldy, int z0 = 0, int z1 = -1);

int source_solve(Ctx& ctx, const Op& a, const Op& b, double sigma, int K, const double* u, long long ld,
                 const double* lambdas, double tol, unsigned long long max_iter, double* out, SolveReport* rep);

int shifted_source_solve(Ctx& ctx, const Op& a, const Op& b, int K, const double* u, long long ld,
                         const double* lambdas, double tol, unsigned long long max_iter, double* out,
                         double* sigma_out, SolveReport* rep);

int cg_solve(Ctx& ctx, const Op& a, int K, const double* rhs, const double* x0, long long ld, double tol,
             unsigned long long max_iter, bool throw_on_max, double* x, SolveReport* rep);

int hartree_solve(Ctx& ctx, const Op& poisson, const Op& mass, const double* rho, double tol, double* vh,
                  SolveReport* rep);

}  // namespace paro_b200
