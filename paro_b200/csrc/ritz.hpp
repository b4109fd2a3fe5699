// Step 4 (rayleigh_ritz) and the dense pencil solve behind the C ABI.
#pragma once

#include "ctx.hpp"

namespace paro_b200 {

struct RitzInfo {
  double min_ratio = 0.0;  // smallest projected/original B-norm ratio of the candidates
  int k = 0;
  bool cgs2 = false;       // the explicit Gram-Schmidt path was used
  bool certify = true;     // in: fail on max |V^T B V - I| > 1e-8 (paro.cpp:171-174); baseline_subspace has no such test
};

int rayleigh_ritz(Ctx& ctx, const Op& A, const Op& B, int K, const double* U, long long ld, size_t min_keep,
                  double drop_tol, double* lambdas_host, double* V, long long ldv, int* k_out, double* defect,
                  RitzInfo* info);

int dense_sym_geneig(Ctx& ctx, int m, const double* A_host, const double* B_host, double* vals_host,
                     double* vecs_host);

int b_orthonormalize(Ctx& ctx, const Op& B, int K, const double* U, double drop_tol, double* Q, int* k_out,
                     int* accepted);

void fix_sign_columns(Ctx& ctx, double* V, long long ld, int k);

// K x K stages of rayleigh_ritz on caller device buffers (column-major):
// ordered Cholesky with drops of the raw Gram -> basis change C1 (K x k);
// second pass G2 -> C2, Bt; pencil (GB == nullptr: in the Q basis from
// GA, C2, Bt; else directly from GA, GB) -> eigenvalues (host) and the
// lift Y (k x k); the certificate max |G - I| (lower triangle).
int ritz_ortho(Ctx& ctx, int K, const double* G, double drop_tol, double* C1, int* k_out, double* min_ratio);
int ritz_second_pass(Ctx& ctx, int k, const double* G2, double* C2, double* Bt);
// one-pass variant: Bt = sym(C1^T sym(G) C1) from the raw Gram and its basis change (k x k, no drops)
int ritz_congruence(Ctx& ctx, int k, const double* G, const double* C1, double* Bt);
int ritz_pencil(Ctx& ctx, int k, const double* GA, const double* C2, const double* Bt, const double* GB,
                double* vals_host, double* Y);
double ritz_defect(Ctx& ctx, int k, const double* G);
// baseline_geneig (linalg.cpp:615-623) on the device (baseline.cu)
int baseline_geneig(Ctx& ctx, const Op& A, const Op& B, int count, unsigned long long max_iter,
                    unsigned long long seed, double* vals_host, double* V, long long ldv, int* iters_out);

}  // namespace paro_b200
