/*
 * paro_b200 — C ABI of the B200-native ParO hot path (sm_100a).
 *
 * The drop-in boundary for the reference's fixed-mesh outer iteration
 * (arXiv 1405.0260, reference C++ in proj/). Every entry point below replaces
 * one reference interface, cited as proj/<file>:<line>. Plain pointers and
 * sizes only; no C++ or torch types cross this boundary.
 *
 * Conventions
 *  - One context per GPU; all work is enqueued on the context's CUDA stream
 *    (paro_ctx_set_stream) and the calls that return host scalars synchronise it.
 *  - Vectors live on the DEVICE unless a parameter says "host". A vector is
 *    the interior-dof coefficient array of the reference (dof order of
 *    proj/src/fem.cpp:21-28 on create_box_mesh, proj/src/mesh.cpp:411-478):
 *    n = (s-1)^3 doubles, x fastest. A batch of k vectors is column-major with
 *    column stride ld >= n (orbital c starts at base + c*ld).
 *  - Return value: PARO_OK or an error code naming the reference exception
 *    type (proj/include/paro/errors.hpp:9-80); paro_ctx_last_error() holds the
 *    message and paro_ctx_last_residual() the IterationLimitError residual.
 */
#ifndef PARO_B200_H
#define PARO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct paro_ctx paro_ctx;
typedef struct paro_op paro_op;
typedef struct paro_csr paro_csr;

enum {
  PARO_OK = 0,
  PARO_ERROR = 1,             /* paro::Error                 errors.hpp:10-13 */
  PARO_INVALID_ARGUMENT = 2,  /* paro::InvalidArgumentError  errors.hpp:15-17 */
  PARO_NOT_SPD = 3,           /* paro::NotSpdError           errors.hpp:25-27 */
  PARO_ITERATION_LIMIT = 4,   /* paro::IterationLimitError   errors.hpp:30-33 */
  PARO_DEGENERATE_SPAN = 5,   /* paro::DegenerateSpanError   errors.hpp:70-72 */
  PARO_PENCIL = 6,            /* paro::PencilError           errors.hpp:60-62 */
  PARO_EMPTY_BASIS = 7,       /* paro::EmptyBasisError       errors.hpp:65-67 */
  PARO_CAPACITY = 8,          /* paro::CapacityError         errors.hpp:40-42 */
  PARO_LINEAGE = 9,           /* paro::LineageError          errors.hpp:35-37 */
  PARO_CUDA_ERROR = 20        /* CUDA / cuBLAS failure (no reference counterpart) */
};

/* ------------------------------------------------------------ context ---- */
int paro_ctx_create(int device, void* cuda_stream, paro_ctx** out);
int paro_ctx_destroy(paro_ctx* ctx);
int paro_ctx_set_stream(paro_ctx* ctx, void* cuda_stream);
const char* paro_ctx_last_error(const paro_ctx* ctx);
double paro_ctx_last_residual(const paro_ctx* ctx);
/* kernels launched by this library so far (CUDA-graph nodes counted) */
unsigned long long paro_ctx_launches(const paro_ctx* ctx);
int paro_ctx_synchronize(paro_ctx* ctx);
/* Live PCG accounting since the last reset: [0] seconds, [1] algorithmic bytes
 * n*(88 k + 64) per iteration, [2] column-iterations for variable operators
 * (Step 3); [3..5] the same for constant operators (Hartree). */
int paro_ctx_stats(paro_ctx* ctx, double out[8], int reset);
/* Step-4 orthonormalisation: 0 = Cholesky-QR twice with an automatic
 * Gram-Schmidt fallback for near-dependent candidates (default), 1 = always
 * two-pass Gram-Schmidt (b_orthonormalize's algorithm, linalg.cpp:409-439). */
int paro_ctx_set_ritz_mode(paro_ctx* ctx, int mode);
/* Hartree solve: 0 = cold-start Jacobi-PCG to tol (the reference algorithm,
 * model.cpp:242-255), 1 = exact 3-D DST-I solve when the Poisson stiffness is
 * the constant 7-point stencil, else PCG (default). The tol-1e-11 PCG iterate
 * lies within ~1e-12 (relative) of the exact solution. */
int paro_ctx_set_hartree_mode(paro_ctx* ctx, int mode);
/* Host copy-out of the next rayleigh_ritz result (one shot): as soon as the
 * new orbitals are final (after fix_sign, before the Gram certificate), their
 * columns [c0, c1) are copied to pinned host memory `host` (column stride ldh)
 * on `copy_stream`, which then holds the copy; the caller synchronises that
 * stream. host == NULL clears a pending request. For callers that keep the
 * orbitals in host memory, like the reference's std::vector interface. */
int paro_ctx_set_ritz_copyout(paro_ctx* ctx, void* copy_stream, double* host, long long ldh, int c0, int c1);

/* Device memory helpers for callers without their own allocator. */
int paro_malloc(paro_ctx* ctx, size_t bytes, void** dev);
int paro_free(paro_ctx* ctx, void* dev);
int paro_memcpy_h2d(paro_ctx* ctx, void* dev, const void* host, size_t bytes);
int paro_memcpy_d2h(paro_ctx* ctx, void* host, const void* dev, size_t bytes);
/* k host vectors of n doubles (e.g. the reference's std::vector columns) <->
 * a device block [k][ld], through a pinned double-buffered staging ring
 * (host copies overlap the DMA); synchronous on return */
int paro_upload_columns(paro_ctx* ctx, int k, const double* const* host, size_t n, double* dev, long long ld);
int paro_download_columns(paro_ctx* ctx, int k, const double* dev, long long ld, size_t n, double* const* host);

/* Uniform box mesh [lo,hi]^3 with `subdivisions` cells per axis
 * (create_box_mesh + FeSpace::create, mesh.cpp:411-478, fem.cpp:13-30). */
int paro_grid_init(paro_ctx* ctx, int subdivisions, double lo, double hi);
long long paro_grid_dofs(const paro_ctx* ctx);

/* ---------------------------------------------------------- operators ---- */
/* A symmetric 15-point P1/Kuhn operator (SparseOperator, linalg.hpp:14-50).
 * Slot o = (x:bit0, y:bit1, z:bit2) holds A[v, v+o]; slot 0 the diagonal. */
int paro_op_create_const(paro_ctx* ctx, const double w[8], paro_op** out);
int paro_op_create_var(paro_ctx* ctx, paro_op** out);
/* SparseOperator(n, row_offsets, cols, vals) -> stencil (linalg.cpp:16-22);
 * PARO_INVALID_ARGUMENT if the pattern is not the Kuhn stencil of the grid or
 * the matrix is not symmetric. Uniform operators become constant stencils. */
int paro_op_from_csr(paro_ctx* ctx, size_t n, const size_t* row_offsets, const uint32_t* cols,
                     const double* vals, paro_op** out);
/* host copy of the operator as CSR in the reference's pattern (sorted cols,
 * all 15 Kuhn neighbours, zeros kept): rows n+1, cols/vals nnz; pass NULLs to
 * query nnz. */
int paro_op_to_csr(paro_ctx* ctx, const paro_op* a, size_t* nnz, size_t* row_offsets, uint32_t* cols,
                   double* vals);
int paro_op_coefficients(paro_op* a, double** dev_coef8);
int paro_op_weights(const paro_op* a, double w[8], int* is_variable);
int paro_op_destroy(paro_op* a);

/* y = (A + sigma B) x for k columns (SparseOperator::matvec + add_scaled,
 * linalg.cpp:88-94, 120-125). `shift` may be NULL. */
int paro_op_apply(paro_ctx* ctx, const paro_op* a, const paro_op* shift, double sigma, int k, const double* x,
                  long long ldx, double* y, long long ldy);

/* ----------------------------------------------------------- solvers ----- */
/* cg_solve (linalg.cpp:143-223, Jacobi preconditioner) for k right-hand sides;
 * x0 may be NULL (zero start). iterations/residual: host arrays of k or NULL. */
int paro_cg_solve(paro_ctx* ctx, const paro_op* a, int k, const double* b, const double* x0, long long ld,
                  double tol, size_t max_iter, int throw_on_max_iter, double* x, size_t* iterations,
                  double* residual);

/* Step 3: source_solve_step (paro.cpp:81-119):
 *   (A + sigma B) u_half_i = (lambda_i + sigma) B u_prev_i,  x0 = u_prev_i,
 * one tolerance-relaxation retry (tol*100, max_iter*4) per orbital.
 * lambdas: host array of k. */
int paro_source_solve_step(paro_ctx* ctx, const paro_op* a, const paro_op* b, int k, const double* u_prev,
                           long long ld, const double* lambdas, double tol, size_t max_iter, double sigma,
                           double* u_half, size_t* iterations, double* residual);
/* The same batched solve reporting per-column outcomes instead of collapsing
 * them into one exception (for callers that shard the orbitals over several
 * GPUs and decide globally): first_status / final_status host arrays of k
 * (PARO_OK, PARO_NOT_SPD, PARO_ITERATION_LIMIT), NULL to skip. */
int paro_source_solve_columns(paro_ctx* ctx, const paro_op* a, const paro_op* b, int k, const double* u_prev,
                              long long ld, const double* lambdas, double tol, size_t max_iter, double sigma,
                              double* u_half, size_t* iterations, double* residual, int* first_status,
                              int* final_status);
/* shifted_source_step (paro.cpp:194-210): sigma = max(0, 0.5 - lambda_1),
 * 2 sigma + 1 on NotSpd, at most 5 attempts; sigma_out: host. */
int paro_shifted_source_step(paro_ctx* ctx, const paro_op* a, const paro_op* b, int k, const double* u_prev,
                             long long ld, const double* lambdas, double tol, size_t max_iter, double* u_half,
                             double* sigma_out, size_t* iterations, double* residual);

/* hartree_solve_with (model.cpp:242-255): poisson V = 4 pi M rho. */
int paro_hartree_solve(paro_ctx* ctx, const paro_op* poisson, const paro_op* mass, const double* rho, double tol,
                       double* vh, size_t* iterations);

/* ------------------------------------------------------------ Step 4 ----- */
/* rayleigh_ritz (paro.cpp:121-177): B-orthonormalise the k candidates with the
 * drop rule of b_orthonormalize (linalg.cpp:409-439), solve the projected
 * pencil (dense_sym_geneig, linalg.cpp:341-393), lift, fix_sign and check the
 * Gram certificate (<= 1e-8, paro.cpp:170-174). cands/orbitals: device,
 * ld == n; lambdas: host array of k (ascending); k_out, defect: host. */
int paro_rayleigh_ritz(paro_ctx* ctx, const paro_op* a_form, const paro_op* b, int k, const double* cands,
                       long long ld, size_t min_keep, double drop_tol, double* lambdas, double* orbitals,
                       long long ldo, int* k_out, double* gram_defect);
/* b_orthonormalize (linalg.cpp:409-439): two-pass Gram-Schmidt in the B inner
 * product with the relative drop rule; u, q: device (ld == n); k_out: host;
 * accepted: host array of k (input index of each kept vector) or NULL. */
int paro_b_orthonormalize(paro_ctx* ctx, const paro_op* b, int k, const double* u, double drop_tol, double* q,
                          int* k_out, int* accepted);
/* baseline_geneig (linalg.cpp:615-623; BaselineOptions linalg.hpp:136-140):
 * the lowest `count` eigenpairs of (A, B) by shift-inverted block subspace
 * iteration (baseline_subspace, linalg.cpp:531-611) on the device, without
 * the reference's 50,000-dof cap. The reference's initial_guess (paro.cpp:
 * 63-79) is this plus gram_defect. max_iter: outer iterations (400);
 * seed: the random start. lambdas: host array of count (ascending);
 * vectors: device, count columns, ld == n, fix_sign applied; iterations:
 * host or NULL. PARO_ITERATION_LIMIT if it does not converge. */
int paro_baseline_geneig(paro_ctx* ctx, const paro_op* a, const paro_op* b, int count, size_t max_iter,
                         unsigned long long seed, double* lambdas, double* vectors, long long ld, int* iterations);
/* dense_sym_geneig on one warp of the device, host row-major m x m in/out. */
int paro_dense_sym_geneig(paro_ctx* ctx, int m, const double* a, const double* b, double* values, double* vectors);
/* fix_sign (linalg.cpp:229-241) on k device columns. */
int paro_fix_sign(paro_ctx* ctx, int k, double* v, long long ld);

/* ---- run artifacts (runner.cpp:92-121): Mesh::dump (mesh.cpp:198-217) of the
 * uniform Kuhn box mesh [lo, hi]^3 with `subdivisions` cells per axis, byte
 * for byte the reference's mesh.txt; no GPU or context needed */
int paro_mesh_dump(int subdivisions, double lo, double hi, const char* path);

/* ---- Step 4 (rayleigh_ritz, paro.cpp:121-177) as building blocks on row
 * ranges [r0, r1) of column blocks: what a Step 4 sharded over row slabs
 * combines across ranks (Grams summed, fix_sign pieces by max / min / max).
 * Matrices g, c, y are device buffers, column-major. */
/* y = A x on the rows of planes [z0, z1); x must be valid on planes z0-1 .. z1 */
int paro_op_apply_planes(paro_ctx* ctx, const paro_op* a, int k, const double* x, long long ld, double* y, int z0,
                         int z1);
/* g (k x k) = x^T y over rows [r0, r1) for a symmetric product (y = B x, A x) */
int paro_gram_sym(paro_ctx* ctx, int k, const double* x, long long ldx, const double* y, long long ldy, long long r0,
                  long long r1, double* g);
/* g (k1 x k2) = x^T y over rows [r0, r1), k1 <= 80, k2 <= 16 */
int paro_gram_rect(paro_ctx* ctx, int k1, const double* x, long long ldx, int k2, const double* y, long long ldy,
                   long long r0, long long r1, double* g);
/* z = x c over rows [r0, r1), k1, k2 <= 80; mode 1: z -= x c, 4: z += x c,
 * 2: c is zero below its diagonal shifted by k1 - k2 (skips those products) */
int paro_rotate(paro_ctx* ctx, int k1, const double* x, long long ldx, const double* c, int ldc, int k2, double* z,
                long long ldz, long long r0, long long r1, int mode);
/* ordered Cholesky with the MGS drop rule of the raw Gram g (K x K) -> basis change c1 (K x k_out) */
int paro_ritz_ortho(paro_ctx* ctx, int K, const double* g, double drop_tol, double* c1, int* k_out,
                    double* min_ratio);
/* second Cholesky-QR pass: g2 -> c2 = L2^{-T}, bt = L2^{-1} g2 L2^{-T}; PARO_PENCIL if not SPD */
int paro_ritz_second_pass(paro_ctx* ctx, int k, const double* g2, double* c2, double* bt);
/* one-pass basis change (well-conditioned candidates, no drops): bt = sym(c1^T sym(g) c1), the
 * B-Gram of U c1 in k x k arithmetic; the pencil then runs on (ga = U^T A U, c1, bt) */
int paro_ritz_congruence(paro_ctx* ctx, int k, const double* g, const double* c1, double* bt);
/* the k x k pencil: gb == NULL: in the Q basis from (ga, c2, bt); else directly
 * (ga, gb). Eigenvalues to host `vals`, lift coefficients to device y (k x k). */
int paro_ritz_pencil(paro_ctx* ctx, int k, const double* ga, const double* c2, const double* bt, const double* gb,
                     double* vals, double* y);
/* gram_defect (paro.cpp:50-61) of an assembled Gram g: max_{j<=i} |g_ij - d_ij| */
int paro_gram_defect(paro_ctx* ctx, int k, const double* g, double* out);
/* fix_sign (linalg.cpp:229-241) pieces: init (amax = 0, first = LLONG_MAX),
 * colmax (max |v| per column, combine by max), first_above (first global row
 * with |v| > 1e-12 amax, combine by min), sign_flags (1 where this range holds
 * that row and it is negative, combine by max), negate_columns. */
int paro_sign_init(paro_ctx* ctx, int k, double* amax, long long* first);
int paro_colmax(paro_ctx* ctx, int k, const double* v, long long ld, long long r0, long long r1, double* amax);
int paro_first_above(paro_ctx* ctx, int k, const double* v, long long ld, long long r0, long long r1,
                     const double* amax, long long* first);
int paro_sign_flags(paro_ctx* ctx, int k, const double* v, long long ld, long long r0, long long r1,
                    const double* amax, const long long* first, double* flip);
int paro_negate_columns(paro_ctx* ctx, int k, double* v, long long ld, long long r0, long long r1,
                        const double* flip);

/* ------------------------------------------------- operator assembly ----- */
/* On the device, element by element in the reference's element order, so the
 * coefficients equal the reference CSR values. Uniform results become
 * constant stencils. */
/* assemble_mass (fem.cpp:253-268) */
int paro_assemble_mass(paro_ctx* ctx, paro_op** out);
/* assemble_stiffness(scale * I, 0) (fem.cpp:221-251): kinetic (0.5), Poisson (1) */
int paro_assemble_stiffness(paro_ctx* ctx, double scale, paro_op** out);
/* assemble_weighted_mass of external_potential(molecule, eps)
 * (model.cpp:146-175, fem.cpp:272-321): eps == 0 -> bare Coulomb with the
 * singular-quadrature policy (degree-5 Duffy rule, 2-level subdivided rule
 * near a nucleus); eps > 0 -> -Z/sqrt(r^2 + eps^2), 4-point rule.
 * positions: 3*nnuc host doubles. */
int paro_assemble_vext(paro_ctx* ctx, int nnuc, const double* charges, const double* positions, double eps,
                       paro_op** out);
/* weighted mass of c*|x|^2 (4-point rule), the harmonic-oscillator reaction */
int paro_assemble_harmonic(paro_ctx* ctx, double c, paro_op** out);
/* a += s * b (SparseOperator::add_scaled, linalg.cpp:120-125) */
int paro_op_add_scaled(paro_ctx* ctx, paro_op* a, const paro_op* b, double s);
/* ks_form_matrix (paro.cpp:446-454): out = kinetic + vext + M[V_H + v_xc(rho)];
 * out: variable operator (paro_op_create_var); clamped: host, may be NULL. */
int paro_ks_form(paro_ctx* ctx, const paro_op* kinetic, const paro_op* vext_mass, const double* rho,
                 const double* vh, int exchange_only, paro_op* out, long long* clamped);
/* the same for the dofs of lattice planes [z0, z1) only (a rank's slab of a row-sharded run; the
 * other coefficients of out are left as they are); clamped counts the cells of layers [z0, z1),
 * plus the top layer when z1 is the last plane, so the ranks' counts add up to paro_ks_form's. */
int paro_ks_form_planes(paro_ctx* ctx, const paro_op* kinetic, const paro_op* vext_mass, const double* rho,
                        const double* vh, int exchange_only, int z0, int z1, paro_op* out, long long* clamped);

/* ---------------------------------------------------------- fields ------- */
/* density_from_orbitals (model.cpp:192-223): rho = sum_i occ_i u_i^2
 * normalised to sum occ; occ: host array of nocc; raw_integral: host. */
int paro_density(paro_ctx* ctx, int nocc, const double* u, long long ld, const double* occ, double* rho,
                 double* raw_integral);
/* mix_density (model.cpp:225-236) */
/* density_from_orbitals in two halves (row-slab sharding): the nodal sum
 * sum_i occ_i u_i^2 on rows [r0, r1) of rho, and the normalisation of a
 * complete nodal density to sum occ (model.cpp:215-221) */
int paro_density_rows(paro_ctx* ctx, int nocc, const double* u, long long ld, const double* occ, long long r0,
                      long long r1, double* rho);
int paro_density_normalize(paro_ctx* ctx, double total_occ, double* rho, double* raw_integral);
int paro_mix_density(paro_ctx* ctx, const double* rho_in, const double* rho_out, double alpha, double* out);
/* integrate / norm_l2 (fem.cpp:419-448), integrate_product (model.cpp:306-327); results: host */
int paro_integrate(paro_ctx* ctx, const double* f, double* out);
int paro_norm_l2(paro_ctx* ctx, const double* f, double* out);
int paro_integrate_product(paro_ctx* ctx, const double* u, const double* v, double* out);
/* ||rho_out - rho_in||_L2 (paro.cpp:608-612); scratch: n device doubles */
int paro_rho_residual(paro_ctx* ctx, const double* rho_out, const double* rho_in, double* scratch, double* out);
/* total_energy (model.cpp:329-360); lambdas, occ, charges, positions: host */
/* Step 2 on a fixed mesh: eta_total of combine_max over the
 * first N orbitals of estimate_eigen_residual (proj/src/adapt.cpp:104-129,
 * estimate_source_residual :58-102, ErrorIndicators::total :14-18), as the
 * drivers run it every outer iteration (Kohn-Sham proj/src/paro.cpp:521-538,
 * linear :306-315). Diffusion D = diffusion * I; reaction 0 = Kohn-Sham
 * V_ext + V_H(rho) + v_xc(rho) at the point (rho, vh device arrays, nuclei
 * and eps as in paro_assemble_vext), 1 = c |x|^2, 2 = external_potential(nuclei,
 * eps). U: device, N columns of stride ld; lambdas: host. eta (device, 6 s^3
 * doubles in the reference element order, may be NULL) receives the combined
 * per-element indicators; *eta_total the total. */
int paro_estimate_eta(paro_ctx* ctx, int N, const double* U, long long ld, const double* lambdas, double diffusion,
                      int reaction, double c, int nnuc, const double* charges, const double* positions, double eps,
                      const double* rho, const double* vh, int exchange_only, double* eta, double* eta_total);

int paro_total_energy(paro_ctx* ctx, int n_lambdas, const double* lambdas, int nocc, const double* occ,
                      const double* rho, const double* vh, int exchange_only, int nnuc, const double* charges,
                      const double* positions, double* e_out);
/* the same in two steps for a run sharded over row slabs: the XC term int rho (e_xc - v_xc) of the
 * cell layers [k0, k1) (the ranks' partial sums add up), and the total with the summed term */
int paro_energy_xc_layers(paro_ctx* ctx, const double* rho, int exchange_only, int k0, int k1, double* out);
int paro_total_energy_with_xc(paro_ctx* ctx, int n_lambdas, const double* lambdas, int nocc, const double* occ,
                              const double* rho, const double* vh, int nnuc, const double* charges,
                              const double* positions, double xc_term, double* e_out);

/* ---------------------------------------------- general CSR operators ---- */
/* SparseOperator (linalg.hpp:14-50) for matrices that are not the uniform
 * Kuhn stencil (adapted meshes): the reference's CSR arrays
 * (size_t row offsets, uint32 ascending columns per row, double values), host
 * pointers. Independent of paro_grid_init. Replaces the same calls as the
 * stencil operators on such matrices: matvec (linalg.cpp:88-94), add_scaled
 * (:120-125, identical structures or PARO_INVALID_ARGUMENT), cg_solve
 * (:143-223) and source_solve_step (paro.cpp:81-119). Vectors: device,
 * k columns at stride ld, k <= 256. */
int paro_csr_create(paro_ctx* ctx, size_t n, const size_t* row_offsets, const uint32_t* cols, const double* vals,
                    paro_csr** out);
int paro_csr_destroy(paro_csr* a);
int paro_csr_add_scaled(paro_ctx* ctx, paro_csr* a, const paro_csr* b, double s);
int paro_csr_apply(paro_ctx* ctx, const paro_csr* a, int k, const double* x, long long ld, double* y);
int paro_csr_cg_solve(paro_ctx* ctx, const paro_csr* a, int k, const double* b, const double* x0, long long ld,
                      double tol, size_t max_iter, int throw_on_max_iter, double* x, size_t* iterations,
                      double* residual);
int paro_csr_source_solve_step(paro_ctx* ctx, const paro_csr* a, const paro_csr* b, int k, const double* u_prev,
                               long long ld, const double* lambdas, double tol, size_t max_iter, double sigma,
                               double* u_half, size_t* iterations, double* residual);

#ifdef __cplusplus
}
#endif

#endif /* PARO_B200_H */
