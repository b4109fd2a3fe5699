// Plane-marching 15-point Kuhn/P1 stencil kernels (sm_100a).
//
// Every operator on the ParO hot path is, on the uniform Kuhn mesh, the
// symmetric 15-point stencil of proj/src/fem.cpp:221-321 restricted to the
// interior lattice. One CTA owns a 32x8 (x,y) tile of the
// interior lattice and a z-range; it marches up in z keeping a ring of three
// (x,y) planes per column (with a one-point halo, zero outside the lattice =
// the Dirichlet elimination of fem.cpp:21-28) in shared memory, prefetching
// the next plane into registers while the current one is computed. The 15
// weights of a point are loaded once per plane step and reused for up to CB
// columns (orbitals), so the coefficient traffic is amortised over the batch.
//
// Row sums are accumulated in ascending column order without FMA contraction,
// exactly like SparseOperator::matvec (proj/src/linalg.cpp:88-94), so an apply
// is bit-identical to the reference CSR matvec on the same coefficients.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace paro_b200 {

constexpr int kTX = 32;
#ifndef PARO_TILE_Y
#define PARO_TILE_Y 8
#endif
constexpr int kTY = PARO_TILE_Y;
constexpr int kNT = kTX * kTY;
constexpr int kHX = kTX + 2;
constexpr int kHY = kTY + 2;
constexpr int kHP = kHX * kHY;              // halo'd plane, 340 points
constexpr int kLoadsPerThread = (kHP + kNT - 1) / kNT;  // 2
// resident CTAs per SM the kernels are compiled for (128 registers per thread)
constexpr int kMinCtas = kNT >= 512 ? 1 : 2;

enum MarchMode : int {
  kApply = 0,       // y = (A + sigma M) x                       [opt. x.y partial]
  kK1 = 1,          // p_new = z + beta p_old (z = r/d); pq = p_new.(A p_new)
  kK2 = 2,          // q = A p; x += alpha p; r -= alpha q; rz, rr partials
  kSetupWarm = 3,   // b = (M u)*scale; r = b - A u; x = u; bb, rz, rr partials
  kSetupCold = 4,   // b = (M f)*scale; r = b; x = 0;      bb, rz, rr partials
};

// Operator as seen by the kernels: (A + sigma*M) with A either 8 SoA
// coefficient arrays (variable) or 8 constants, and M a constant stencil.
struct OpDev {
  const double* coef = nullptr;  // slot o at coef + o*n; nullptr -> constant w[]
  double w[kSlots] = {};         // constant weights
  double m[kSlots] = {};         // shift stencil (mass) weights
  const double* mcoef = nullptr; // variable shift stencil (SoA), overrides m[]
  double sigma = 0.0;            // add_scaled(b, sigma): fl(w + fl(sigma*m))
  double invd_const = 0.0;       // 1/diag for the constant case
  double sm[kSlots] = {};        // fl(sigma * m[o]), host-computed (constant shift)
  double wc[kSlots] = {};        // fl(w[o] + sm[o]): the shifted constant operator
};

struct MarchArgs {
  int S = 0;
  long long n = 0;
  int nTX = 0, nTY = 0, nZ = 0, ZC = 0;
  int zlo = 0, zhi = 0;          // planes [zlo, zhi) whose rows are computed (row-slab Step 4); 0, S by default
  int nblk = 0;                  // spatial blocks = nTX*nTY*nZ
  int K = 0;                     // columns in the batch
  long long ld = 0;              // column stride of every vector operand
  OpDev op;
  double mw[kSlots] = {};        // right-hand-side mass stencil (setup modes)
  const double* mwcoef = nullptr;// variable right-hand-side mass (SoA), overrides mw[]
  const double* src = nullptr;   // plane source (x | p | u | f)
  const double* pold = nullptr;  // K1: previous direction
  double* dst = nullptr;         // Apply: y; K1: p_new; Setup: r
  double* x = nullptr;           // K2 / Setup
  double* r = nullptr;           // K1 (read) / K2 (read-write)
  const double* invd = nullptr;  // variable-op inverse diagonal (n)
  CgColumn* cols = nullptr;      // per-column state (active mask, alpha, beta, first)
  const double* scale = nullptr; // Setup: rhs scale per column
  const double* rhs = nullptr;   // Setup (warm): explicit right-hand side instead of (M u)*scale
  double* partials = nullptr;    // [K][3][nblk]
  int with_dot = 0;              // Apply: accumulate x.y
  long long ldw = 0;             // Setup: stride of the x, r outputs (0: ld)
  int xmode = 2;                 // K2 x update: 2 every iteration; deferred pairs (k2c): 0 none, 1 x += a' p' + a p
  int P = 0;                     // row length of the row-padded solver layout (0: dense S);
                                 // Setup writes x, r there, the TMA passes read/write it
};

// Row-padded solver layout (tma.cu): element (x, y, z) of a column at
// (z*S + y)*P + x with P = S rounded up to even, so every row starts 16-byte
// aligned and the PCG operands can be described by TMA tensor maps
// (4-D: x, y, z, column). Points outside the lattice come back as zeros from
// the TMA engine's out-of-bounds fill (the Dirichlet elimination).
inline int padded_row(int S) { return S + (S & 1); }

// Tensor maps of one batched PCG call's buffers (encoded once per call).
struct PcgTma {
  alignas(64) CUtensorMap r_halo, p0_halo, p1_halo, invd_halo, invd_own, x_own, r_own, coef_box;
  CUtensorMap r_fwd, p0_fwd, p1_fwd, invd_fwd, coef_own;  // one-sided (forward) boxes of K1 (k1f_kernel)
  CUtensorMap x_halo;                                     // setup (k0c_kernel): x0 = u planes
  bool has_coef = false;  // coef_box: the operator's 8 coefficient slots in the row-padded layout
};
// coefp (optional): the 8 coefficient slots of a variable operator in the
// row-padded layout at stride ldi (K2 then stages them by TMA, k2c_kernel)
void tma_plan(PcgTma& t, int S, long long ldi, int K, const double* r, const double* p0, const double* p1,
              const double* x, const double* invd, const double* coefp);
// K1 (p_new -> a.dst; its p_old is p0 when p_is_p0) or K2 (its stencil source p is p0
// when p_is_p0), both on the row-padded layout described by t.
void launch_tma(int mode, bool var, int cb, const MarchArgs& a, const PcgTma& t, bool p_is_p0, cudaStream_t st);
// true when K2 of a variable operator runs on k2c_kernel (which supports deferred x updates)
bool tma_k2c_active();
// PCG setup (warm start, rhs = (M u) * scale) on the row-padded layout with x = u already in place
void launch_tma_setup(int cb, const MarchArgs& a, const PcgTma& t, cudaStream_t st);

void launch_march(int mode, bool var, int cb, const MarchArgs& a, cudaStream_t st);
// y = A x on the dense layout by TMA through a flat 2S-wide view of x (odd S,
// ld == n, 16-byte aligned x; coefp: the variable operator's coefficients in
// the row-padded layout at slot stride ldi); apply_flat_ok says whether the
// operands qualify (otherwise the apply stays on stream_kernel).
bool apply_flat_ok(bool var, const MarchArgs& a);
void launch_apply_flat(bool var, int cb, const MarchArgs& a, const double* coefp, long long ldi, cudaStream_t st);
// padded solver buffers: every vector operand is 16-byte aligned, has an even
// column stride and at least kBulkPad readable elements before its first and
// after its last column
constexpr long long kBulkPad = 64;
void plan_march(MarchArgs& a, int S, int zlo = 0, int zhi = -1);

}  // namespace paro_b200
