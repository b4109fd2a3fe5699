// Step-4 building blocks on row ranges [r0, r1) of column blocks (step4.cu,
// ritz.cu): what a row-slab sharded rayleigh_ritz combines across ranks.
#pragma once

#include "ctx.hpp"

namespace paro_b200 {

// Z[r0:r1) = X[r0:r1) C (k1 x k2, column-major, ldc); mode bit 0: Z -= X C,
// bit 1: C[i][j] = 0 for i > j + k1 - k2 (Cholesky-QR basis change)
void rotate_rows(Ctx& ctx, int k1, const double* X, long long ldx, const double* C, int ldc, int k2, double* Z,
                 long long ldz, long long r0, long long r1, int mode);
// G (k1 x k2, column-major) = X[r0:r1)^T Y[r0:r1), k1 <= 80, k2 <= 16
void gram_rect_rows(Ctx& ctx, int k1, const double* X, long long ldx, int k2, const double* Y, long long ldy,
                    long long r0, long long r1, double* G);
// G (k x k, column-major, exactly symmetric) = X[r0:r1)^T Y[r0:r1) for a
// symmetric product (Y = B X or A X); ritz.cu
void gram_sym_rows(Ctx& ctx, int k, const double* X, long long ldx, const double* Y, long long ldy, long long r0,
                   long long r1, double* G);

// fix_sign pieces: amax (k doubles, max |v| over the range, combined by max),
// first (k, global row of the first |v| > 1e-12 amax, LLONG_MAX if none,
// combined by min), flip (k, 1 where this range holds that row and it is
// negative, combined by max), then the negation of the flagged columns.
void sign_init(Ctx& ctx, int k, double* amax, long long* first);
void colmax_rows(Ctx& ctx, int k, const double* V, long long ld, long long r0, long long r1, double* amax);
void first_rows(Ctx& ctx, int k, const double* V, long long ld, long long r0, long long r1, const double* amax,
                long long* first);
void sign_rows(Ctx& ctx, int k, const double* V, long long ld, long long r0, long long r1, const double* amax,
               const long long* first, double* flip);
void negate_rows(Ctx& ctx, int k, double* V, long long ld, long long r0, long long r1, const double* flip);

}  // namespace paro_b200
