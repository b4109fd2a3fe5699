// Step-2 residual estimator (estimate.cu).
#pragma once

#include <vector>

#include "ctx.hpp"

namespace paro_b200 {

enum EstimateKind : int {
  kEstKs = 0,        // V_ext(x) + V_H(x) + v_xc(rho(x))  (paro.cpp:525-531)
  kEstHarmonic = 1,  // c |x|^2
  kEstWell = 2,      // external_potential(nuclei, eps)
};

struct EstimateSpec {
  int kind = kEstKs;
  double diffusion = 0.5;          // D = diffusion * I
  double c = 0.0;
  std::vector<double> nuclei;      // Z, x, y, z per nucleus
  double eps = 0.0;
  const double* rho = nullptr;     // device, n
  const double* vh = nullptr;      // device, n
  int exchange_only = 0;
  const double* lambdas = nullptr; // host, N
};

// eta_total of combine_max over the N columns of U; per-element eta (6 s^3,
// reference element order) to `eta` when non-null.
double estimate_eta(Ctx& ctx, const EstimateSpec& spec, int N, const double* U, long long ld, double* eta);

}  // namespace paro_b200
