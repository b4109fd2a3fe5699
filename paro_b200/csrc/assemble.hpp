// Device assembly of the P1/Kuhn stencil operators (see assemble.cu).
#pragma once

#include <vector>

#include "ctx.hpp"
#include "quad.hpp"

namespace paro_b200 {

enum AsmKind : int {
  kAsmMass = 0,         // assemble_mass (fem.cpp:253-268)
  kAsmStiffness = 1,    // assemble_stiffness(scale*I, 0) (fem.cpp:221-251)
  kAsmCoulomb = 2,      // weighted mass of -sum Z/|x-R| with the singular policy
  kAsmSoftCoulomb = 3,  // weighted mass of -sum Z/sqrt(|x-R|^2+eps^2), 4-point rule
  kAsmHarmonic = 4,     // weighted mass of scale*|x|^2, 4-point rule
  kAsmScf = 5,          // weighted mass of V_H + v_xc(rho), 4-point rule (+ kinetic + V_ext)
};

struct AssembleSpec {
  int kind = kAsmMass;
  double scale = 0.0;
  std::vector<double> nuclei;  // Z, x, y, z per nucleus
  double eps = 0.0;
  const double* rho = nullptr;
  const double* vh = nullptr;
  int exchange_only = 0;
  const Op* kinetic = nullptr;
  const Op* vext = nullptr;
  long long* clamped = nullptr;  // Scf: (element, point) pairs with rho < 0 (the reference's clamp count)
  // Scf on the table path: only the dofs of lattice planes [z0, z1) are assembled (z1 < 0: all) --
  // a rank's slab of a row-sharded run; the clamp count then covers the cells k in [z0, z1)
  // (and the top cell layer k = S when z1 == S), so the ranks' counts add up to the full one
  int z0 = 0, z1 = -1;
};

void assemble(Ctx& ctx, const AssembleSpec& spec, Op& out);
// converts a variable operator whose slots are identical at every dof into a
// constant stencil (frees the arrays); returns whether it did.
bool make_uniform_if_possible(Ctx& ctx, Op& op);
// a += s * b (SparseOperator::add_scaled); a constant `a` is promoted if b varies
void add_scaled(Ctx& ctx, Op& a, const Op& b, double s);

}  // namespace paro_b200
