// Nodal fields: density, mixing, norms, energy (see fields.cu).
#pragma once

#include "ctx.hpp"

namespace paro_b200 {

enum CellMode : int { kCellIntegrate = 0, kCellNorm2 = 1, kCellProduct = 2, kCellExc = 3, kCellClamp = 4 };

// k0, k1: cell layers [k0, k1) only (k1 < 0: every cell)
double cell_reduce(Ctx& ctx, int mode, const double* f, const double* g, int exchange_only, int k0 = 0, int k1 = -1);
// rho = sum_i occ_i u_i^2, normalised to sum occ; returns the raw integral
double density(Ctx& ctx, int nocc, const double* U, long long ld, const double* occ_host, double* rho);
// its two halves: the nodal sum on rows [r0, r1) (returns sum occ) and the
// normalisation of a complete nodal density (returns the raw integral)
double density_rows(Ctx& ctx, int nocc, const double* U, long long ld, const double* occ_host, long long r0,
                    long long r1, double* rho);
double density_normalize(Ctx& ctx, double total_occ, double* rho);
void mix(Ctx& ctx, const double* rin, const double* rout, double alpha, double* out);
void diff(Ctx& ctx, const double* a, const double* b, double* out);
double norm_l2(Ctx& ctx, const double* f);
// xc_term (optional): the XC term int rho (e_xc - v_xc) summed elsewhere (energy_xc_term over cell layers)
double total_energy(Ctx& ctx, int nl, const double* lambdas, int nocc, const double* occ, const double* rho,
                    const double* vh, int exchange_only, int nnuc, const double* nuclei,
                    const double* xc_term = nullptr);
double energy_xc_term(Ctx& ctx, const double* rho, int exchange_only, int k0, int k1);

}  // namespace paro_b200
