// integration/paro_gpu.hpp — drop-in GPU implementations of the reference's
// hot-path interfaces, with the reference's own types and signatures
// (proj/include/paro). A maintainer adds this header + paro_gpu.cpp to the
// reference tree, links libparo_b200.so, and swaps the call sites listed in
// INTEGRATION.md (paro::source_solve_step -> paro::gpu::source_solve_step, ...).
// Errors are rethrown as the reference's exception types (errors.hpp).
#pragma once

#include <memory>
#include <vector>

#include "paro/adapt.hpp"
#include "paro/fem.hpp"
#include "paro/linalg.hpp"
#include "paro/model.hpp"
#include "paro/paro.hpp"

namespace paro::gpu {

/// Binds the calling thread to a device and to the uniform box mesh of
/// `space` (create_box_mesh(cubic box, s)); every call below runs on that grid.
void bind(const FeSpace& space, int device = 0);
/// True when the bound grid matches `space`'s mesh.
bool bound_to(const FeSpace& space);
/// Drops the cached device forms of operators (they are keyed by value array,
/// size and a sampled signature; call this after modifying an operator in
/// place in a way the sample could miss). bind() clears the cache too.
void invalidate();

/// cg_solve (linalg.cpp:143-223)
CgResult cg_solve(const SparseOperator& a, const std::vector<double>& b, const CgOptions& opts = {});

/// source_solve_step (paro.cpp:81-119); all K orbitals in one batched solve
std::vector<std::vector<double>> source_solve_step(const SparseOperator& a, const SparseOperator& b,
                                                   const std::vector<std::vector<double>>& u_prev,
                                                   const std::vector<double>& lambdas,
                                                   const SourceSolveOptions& opts);

/// rayleigh_ritz (paro.cpp:121-177)
OrbitalSet rayleigh_ritz(const std::vector<std::vector<double>>& candidates, const SparseOperator& a_form,
                         const SparseOperator& b, std::shared_ptr<const FeSpace> space, std::size_t min_keep,
                         double drop_tol, RitzTimings* timings = nullptr);

/// b_orthonormalize (linalg.cpp:409-439)
OrthonormalizeResult b_orthonormalize(const std::vector<std::vector<double>>& vectors, const SparseOperator& b,
                                      double drop_tol);

/// dense_sym_geneig (linalg.cpp:341-393) on one warp of the device
EigenPairs dense_sym_geneig(const DenseSymPencil& pencil);

/// baseline_geneig (linalg.cpp:615-623): device block subspace iteration,
/// no 50,000-dof cap (initial_guess, paro.cpp:63-79, calls this)
EigenPairs baseline_geneig(const SparseOperator& a, const SparseOperator& b, std::size_t count,
                           const BaselineOptions& opts = {});

/// density_from_orbitals (model.cpp:192-223)
Density density_from_orbitals(const std::vector<DiscreteFunction>& orbitals, const std::vector<double>& occupations);

/// hartree_solve_with (model.cpp:242-255)
DiscreteFunction hartree_solve_with(const SparseOperator& poisson_stiffness, const SparseOperator& mass,
                                    const Density& rho, const std::shared_ptr<const FeSpace>& space, double tol);

/// total_energy (model.cpp:329-360)
double total_energy(const std::vector<double>& lambdas, const Density& density, const DiscreteFunction& v_hartree,
                    XcModel xc, const Molecule& molecule);

/// Step 2 of the Kohn-Sham driver on a fixed mesh (paro.cpp:521-538):
/// combine_max over the occupied orbitals of estimate_eigen_residual
/// (adapt.cpp:104-129) with diffusion 1/2 and reaction V_ext + V_H + v_xc;
/// eta in the reference element order, mesh_id of the orbitals' mesh.
ErrorIndicators ks_step2_indicators(const std::vector<DiscreteFunction>& occupied,
                                    const std::vector<double>& lambdas, const Density& rho_in,
                                    const DiscreteFunction& vh_in, const Molecule& molecule, double vext_smoothing,
                                    XcModel xc);

}  // namespace paro::gpu
