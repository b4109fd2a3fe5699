// Fast Hartree solve by the 3-D DST-I (see poisson.cu).
#pragma once

#include "ctx.hpp"

namespace paro_b200 {

// true when K is a constant stencil with only the 7-point entries nonzero
bool dst_applicable(const Op& k);
int hartree_dst(Ctx& ctx, const Op& poisson, const Op& mass, const double* rho, double* vh);

}  // namespace paro_b200
