// integration/paro_gpu.cpp — the reference interfaces over the paro_b200 C ABI.
// Host vectors in, host vectors out (the drop-in contract); each call moves its
// operands to the device, runs the sm_100a kernels and maps the status code
// back to the reference's exception type. See paro_gpu.hpp / INTEGRATION.md.
//
// Operators are converted once: the device form of a SparseOperator (the
// stencil operator of the bound lattice, or the general CSR form for adapted
// meshes) is cached per operator, keyed by its value array, dimension, nnz and
// a signature of 4096 sampled values, so the mass / stiffness / KS form of a
// call sequence cross the PCIe bus once (at 257^3 a KS form is 3 GB of CSR).
// Orbital blocks move through the library's pinned staging ring
// (paro_upload_columns / paro_download_columns).
#include "paro_gpu.hpp"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "paro/errors.hpp"
#include "paro_b200.h"

namespace paro::gpu {

namespace {

struct State {
  paro_ctx* ctx = nullptr;
  int s = 0;
  double lo = 0.0, hi = 0.0;
  std::size_t n = 0;
  std::uint64_t mesh_id = 0;
};
thread_local State g;

struct CachedOp {
  const double* vals = nullptr;
  std::size_t n = 0, nnz = 0;
  std::uint64_t sig = 0;
  bool lattice = false;
  paro_op* op = nullptr;   // stencil form (lattice operators)
  paro_csr* csr = nullptr; // general CSR form (adapted meshes)
  std::uint64_t used = 0;
};
constexpr std::size_t kCacheSize = 8;
thread_local std::vector<CachedOp> g_cache;
thread_local std::uint64_t g_tick = 0;

void drop(CachedOp& c) {
  if (c.op) paro_op_destroy(c.op);
  if (c.csr) paro_csr_destroy(c.csr);
  c = CachedOp{};
}

[[noreturn]] void rethrow(int st) {
  const std::string msg = paro_ctx_last_error(g.ctx);
  switch (st) {
    case PARO_NOT_SPD: throw NotSpdError(msg);
    case PARO_ITERATION_LIMIT: throw IterationLimitError(msg, paro_ctx_last_residual(g.ctx));
    case PARO_DEGENERATE_SPAN: throw DegenerateSpanError(msg);
    case PARO_PENCIL: throw PencilError(msg);
    case PARO_EMPTY_BASIS: throw EmptyBasisError(msg);
    case PARO_CAPACITY: throw CapacityError(msg);
    case PARO_LINEAGE: throw LineageError(msg);
    case PARO_INVALID_ARGUMENT: throw InvalidArgumentError(msg);
    default: throw Error(msg);
  }
}

void check(int st) {
  if (st != PARO_OK) rethrow(st);
}

struct DevVec {
  double* p = nullptr;
  explicit DevVec(std::size_t count) {
    void* v = nullptr;
    check(paro_malloc(g.ctx, count * sizeof(double), &v));
    p = static_cast<double*>(v);
  }
  ~DevVec() {
    if (p) paro_free(g.ctx, p);
  }
  DevVec(DevVec&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevVec(const DevVec&) = delete;
  DevVec& operator=(const DevVec&) = delete;
  void up(const double* h, std::size_t count, std::size_t off = 0) {
    check(paro_memcpy_h2d(g.ctx, p + off, h, count * sizeof(double)));
  }
  void down(double* h, std::size_t count, std::size_t off = 0) const {
    check(paro_memcpy_d2h(g.ctx, h, p + off, count * sizeof(double)));
  }
};

std::uint64_t signature(const SparseOperator& a) {
  const auto& v = a.values();
  std::uint64_t h = 1469598103934665603ull ^ v.size();
  const std::size_t step = std::max<std::size_t>(1, v.size() / 4096);
  for (std::size_t i = 0; i < v.size(); i += step) {
    std::uint64_t bits;
    std::memcpy(&bits, &v[i], sizeof bits);
    h = (h ^ bits) * 1099511628211ull;
  }
  if (!v.empty()) {
    std::uint64_t bits;
    std::memcpy(&bits, &v.back(), sizeof bits);
    h = (h ^ bits) * 1099511628211ull;
  }
  return h;
}

void ensure_ctx();

// the cached device form of `a` (converted on first use; LRU of kCacheSize)
CachedOp& device_op(const SparseOperator& a) {
  ensure_ctx();
  const std::uint64_t sig = signature(a);
  for (auto& c : g_cache)
    if (c.vals == a.values().data() && c.n == a.dimension() && c.nnz == a.values().size() && c.sig == sig) {
      c.used = ++g_tick;
      return c;
    }
  if (g_cache.size() >= kCacheSize) {
    auto lru = std::min_element(g_cache.begin(), g_cache.end(),
                                [](const CachedOp& x, const CachedOp& y) { return x.used < y.used; });
    drop(*lru);
    g_cache.erase(lru);
  }
  CachedOp c;
  c.vals = a.values().data();
  c.n = a.dimension();
  c.nnz = a.values().size();
  c.sig = sig;
  c.used = ++g_tick;
  // the stencil form exists for operators of the bound lattice with the P1/Kuhn pattern
  if (g.n == a.dimension()) {
    const int st = paro_op_from_csr(g.ctx, a.dimension(), a.row_offsets().data(), a.col_indices().data(),
                                    a.values().data(), &c.op);
    if (st != PARO_OK && st != PARO_INVALID_ARGUMENT) check(st);
    c.lattice = st == PARO_OK;
  }
  g_cache.push_back(c);
  return g_cache.back();
}

paro_op* lattice_op(const SparseOperator& a) {
  CachedOp& c = device_op(a);
  if (!c.lattice)
    throw InvalidArgumentError("paro::gpu: operator is not a P1/Kuhn stencil of the bound grid");
  return c.op;
}

paro_csr* csr_op(const SparseOperator& a) {
  CachedOp& c = device_op(a);
  if (!c.csr)
    check(paro_csr_create(g.ctx, a.dimension(), a.row_offsets().data(), a.col_indices().data(), a.values().data(),
                          &c.csr));
  return c.csr;
}

void ensure_ctx() {
  if (!g.ctx && paro_ctx_create(0, nullptr, &g.ctx) != PARO_OK) throw Error(paro_ctx_last_error(nullptr));
}

// The stencil kernels serve operators of the bound uniform lattice whose
// pattern is the P1/Kuhn stencil; everything else (adapted meshes) takes the
// general CSR kernels.
bool on_lattice(const SparseOperator& a) { return g.ctx && device_op(a).lattice; }

void need(std::size_t n) {
  if (!g.ctx || g.n != n)
    throw InvalidArgumentError("paro::gpu: no device grid of dimension " + std::to_string(n) +
                               " bound; call paro::gpu::bind(space)");
}

DevVec pack(const std::vector<std::vector<double>>& cols, std::size_t n) {
  DevVec d(cols.empty() ? 1 : cols.size() * n);
  std::vector<const double*> ptr(cols.size());
  for (std::size_t c = 0; c < cols.size(); ++c) {
    if (cols[c].size() != n) throw InvalidArgumentError("paro::gpu: vector dimension mismatch");
    ptr[c] = cols[c].data();
  }
  check(paro_upload_columns(g.ctx, static_cast<int>(cols.size()), ptr.data(), n, d.p, static_cast<long long>(n)));
  return d;
}

std::vector<std::vector<double>> unpack(const DevVec& d, std::size_t k, std::size_t n) {
  std::vector<std::vector<double>> out(k, std::vector<double>(n));
  std::vector<double*> ptr(k);
  for (std::size_t c = 0; c < k; ++c) ptr[c] = out[c].data();
  check(paro_download_columns(g.ctx, static_cast<int>(k), d.p, static_cast<long long>(n), n, ptr.data()));
  return out;
}

}  // namespace

void bind(const FeSpace& space, int device) {
  const Mesh& m = space.mesh();
  if (m.dimension() != 3) throw InvalidArgumentError("paro::gpu: 3-D box meshes only");
  const auto nv = static_cast<double>(m.vertex_count());
  const int s = static_cast<int>(std::lround(std::cbrt(nv))) - 1;
  const Box& b = m.domain_box();
  const bool uniform = s >= 2 && static_cast<std::size_t>(s + 1) * (s + 1) * (s + 1) == m.vertex_count() &&
                       m.element_count() == static_cast<std::size_t>(6) * s * s * s && m.generation_index() == 0;
  if (!uniform) throw InvalidArgumentError("paro::gpu: the mesh is not an unrefined create_box_mesh lattice");
  if (b.lo.x != b.lo.y || b.lo.x != b.lo.z || b.hi.x != b.hi.y || b.hi.x != b.hi.z)
    throw InvalidArgumentError("paro::gpu: cubic boxes only");
  if (!g.ctx) {
    if (paro_ctx_create(device, nullptr, &g.ctx) != PARO_OK) throw Error(paro_ctx_last_error(nullptr));
  }
  invalidate();  // stencil forms belong to the previous grid
  check(paro_grid_init(g.ctx, s, b.lo.x, b.hi.x));
  g.s = s;
  g.lo = b.lo.x;
  g.hi = b.hi.x;
  g.n = space.dof_count();
  g.mesh_id = m.id();
}

bool bound_to(const FeSpace& space) { return g.ctx && g.mesh_id == space.mesh().id(); }

void invalidate() {
  for (auto& c : g_cache) drop(c);
  g_cache.clear();
}

CgResult cg_solve(const SparseOperator& a, const std::vector<double>& b, const CgOptions& opts) {
  const std::size_t n = a.dimension();
  ensure_ctx();
  if (b.size() != n) throw InvalidArgumentError("cg: dimension mismatch");
  if (opts.precond != Preconditioner::diagonal)
    throw InvalidArgumentError("paro::gpu::cg_solve: only the Jacobi preconditioner is implemented");
  const bool lattice = on_lattice(a);
  DevVec db(n), dx(n);
  db.up(b.data(), n);
  DevVec dx0(opts.x0 ? n : 1);
  if (opts.x0) {
    if (opts.x0->size() != n) throw InvalidArgumentError("cg: x0 dimension mismatch");
    dx0.up(opts.x0->data(), n);
  }
  std::size_t it = 0;
  double res = 0.0;
  if (lattice) {
    check(paro_cg_solve(g.ctx, lattice_op(a), 1, db.p, opts.x0 ? dx0.p : nullptr, static_cast<long long>(n), opts.tol,
                        opts.max_iter, opts.throw_on_max_iter ? 1 : 0, dx.p, &it, &res));
  } else {
    check(paro_csr_cg_solve(g.ctx, csr_op(a), 1, db.p, opts.x0 ? dx0.p : nullptr, static_cast<long long>(n), opts.tol,
                            opts.max_iter, opts.throw_on_max_iter ? 1 : 0, dx.p, &it, &res));
  }
  CgResult r;
  r.x.resize(n);
  dx.down(r.x.data(), n);
  r.iterations = it;
  r.residual = res;
  r.converged = res <= opts.tol;
  return r;
}

std::vector<std::vector<double>> source_solve_step(const SparseOperator& a, const SparseOperator& b,
                                                   const std::vector<std::vector<double>>& u_prev,
                                                   const std::vector<double>& lambdas,
                                                   const SourceSolveOptions& opts) {
  if (u_prev.size() != lambdas.size())
    throw InvalidArgumentError("source_solve_step: orbital/lambda count mismatch");
  const std::size_t n = a.dimension(), k = u_prev.size();
  ensure_ctx();
  if (k == 0) return {};
  DevVec du = pack(u_prev, n);
  DevVec dh(k * n);
  if (on_lattice(a) && on_lattice(b)) {
    check(paro_source_solve_step(g.ctx, lattice_op(a), lattice_op(b), static_cast<int>(k), du.p, static_cast<long long>(n),
                                 lambdas.data(), opts.tol, opts.max_iter, opts.sigma, dh.p, nullptr, nullptr));
  } else {  // adapted meshes: general CSR kernels, same semantics
    check(paro_csr_source_solve_step(g.ctx, csr_op(a), csr_op(b), static_cast<int>(k), du.p, static_cast<long long>(n),
                                     lambdas.data(), opts.tol, opts.max_iter, opts.sigma, dh.p, nullptr, nullptr));
  }
  return unpack(dh, k, n);
}

OrbitalSet rayleigh_ritz(const std::vector<std::vector<double>>& candidates, const SparseOperator& a_form,
                         const SparseOperator& b, std::shared_ptr<const FeSpace> space, std::size_t min_keep,
                         double drop_tol, RitzTimings* timings) {
  const std::size_t n = a_form.dimension(), k = candidates.size();
  need(n);
  if (k == 0) throw EmptyBasisError("b_orthonormalize: all vectors dropped");
  paro_op* A = lattice_op(a_form);
  paro_op* B = lattice_op(b);
  DevVec du = pack(candidates, n);
  DevVec dv(k * n);
  std::vector<double> lam(k);
  int kout = 0;
  double defect = 0.0;
  check(paro_rayleigh_ritz(g.ctx, A, B, static_cast<int>(k), du.p, static_cast<long long>(n), min_keep,
                           drop_tol, lam.data(), dv.p, static_cast<long long>(n), &kout, &defect));
  OrbitalSet out;
  out.space = std::move(space);
  out.orbitals = unpack(dv, static_cast<std::size_t>(kout), n);
  out.lambdas.assign(lam.begin(), lam.begin() + kout);
  out.gram_defect = defect;
  if (timings) *timings = RitzTimings{};
  return out;
}

OrthonormalizeResult b_orthonormalize(const std::vector<std::vector<double>>& vectors, const SparseOperator& b,
                                      double drop_tol) {
  const std::size_t n = b.dimension(), k = vectors.size();
  need(n);
  OrthonormalizeResult r;
  if (k == 0) return r;
  paro_op* B = lattice_op(b);
  DevVec du = pack(vectors, n);
  DevVec dq(k * n);
  int kout = 0;
  std::vector<int> acc(k, -1);
  check(paro_b_orthonormalize(g.ctx, B, static_cast<int>(k), du.p, drop_tol, dq.p, &kout, acc.data()));
  r.vectors = unpack(dq, static_cast<std::size_t>(kout), n);
  std::vector<bool> kept(k, false);
  for (int i = 0; i < kout; ++i) kept[static_cast<std::size_t>(acc[i])] = true;
  for (std::size_t i = 0; i < k; ++i)
    if (!kept[i]) r.dropped.push_back(i);
  return r;
}

EigenPairs baseline_geneig(const SparseOperator& a, const SparseOperator& b, std::size_t count,
                           const BaselineOptions& opts) {
  const std::size_t n = a.dimension();
  if (b.dimension() != n) throw InvalidArgumentError("baseline: pencil dimension mismatch");
  if (count == 0 || count > n) throw InvalidArgumentError("baseline: bad eigenpair count");
  need(n);
  paro_op* A = lattice_op(a);
  paro_op* B = lattice_op(b);
  DevVec dv(count * n);
  EigenPairs out;
  out.values.assign(count, 0.0);
  int its = 0;
  check(paro_baseline_geneig(g.ctx, A, B, static_cast<int>(count), opts.max_iter, opts.seed,
                             out.values.data(), dv.p, static_cast<long long>(n), &its));
  const std::vector<std::vector<double>> cols = unpack(dv, count, n);
  out.vectors = DenseMatrix(n, count);
  for (std::size_t j = 0; j < count; ++j)
    for (std::size_t i = 0; i < n; ++i) out.vectors(i, j) = cols[j][i];
  return out;
}

EigenPairs dense_sym_geneig(const DenseSymPencil& pencil) {
  const std::size_t m = pencil.a.rows();
  if (pencil.a.cols() != m || pencil.b.rows() != m || pencil.b.cols() != m)
    throw PencilError("pencil: dimension mismatch");
  if (!g.ctx) {
    if (paro_ctx_create(0, nullptr, &g.ctx) != PARO_OK) throw Error(paro_ctx_last_error(nullptr));
  }
  EigenPairs e;
  e.values.resize(m);
  std::vector<double> vecs(m * m);
  check(paro_dense_sym_geneig(g.ctx, static_cast<int>(m), pencil.a.data().data(), pencil.b.data().data(),
                              e.values.data(), vecs.data()));
  e.vectors = DenseMatrix(m, m);
  for (std::size_t i = 0; i < m; ++i)
    for (std::size_t j = 0; j < m; ++j) e.vectors(i, j) = vecs[i * m + j];
  return e;
}

Density density_from_orbitals(const std::vector<DiscreteFunction>& orbitals, const std::vector<double>& occupations) {
  if (orbitals.empty() || orbitals.size() != occupations.size())
    throw InvalidArgumentError("density: orbital/occupation count mismatch");
  const auto space = orbitals.front().space;
  for (const auto& u : orbitals)
    if (u.space->mesh().id() != space->mesh().id()) throw LineageError("density: orbitals from different generations");
  const std::size_t n = space->dof_count(), k = orbitals.size();
  need(n);
  DevVec du(k * n), drho(n);
  std::vector<const double*> cols(k);
  for (std::size_t c = 0; c < k; ++c) cols[c] = orbitals[c].coeffs.data();
  check(paro_upload_columns(g.ctx, static_cast<int>(k), cols.data(), n, du.p, static_cast<long long>(n)));
  Density d;
  d.occupations = occupations;
  d.rho = DiscreteFunction(space);
  check(paro_density(g.ctx, static_cast<int>(k), du.p, static_cast<long long>(n), occupations.data(), drho.p,
                     &d.raw_integral));
  drho.down(d.rho.coeffs.data(), n);
  return d;
}

DiscreteFunction hartree_solve_with(const SparseOperator& poisson_stiffness, const SparseOperator& mass,
                                    const Density& rho, const std::shared_ptr<const FeSpace>& space, double tol) {
  if (rho.rho.space->mesh().id() != space->mesh().id())
    throw LineageError("hartree: density lives on a different generation");
  const std::size_t n = space->dof_count();
  need(n);
  paro_op* K = lattice_op(poisson_stiffness);
  paro_op* M = lattice_op(mass);
  DevVec dr(n), dv(n);
  dr.up(rho.rho.coeffs.data(), n);
  check(paro_hartree_solve(g.ctx, K, M, dr.p, tol, dv.p, nullptr));
  DiscreteFunction out(space);
  dv.down(out.coeffs.data(), n);
  return out;
}

double total_energy(const std::vector<double>& lambdas, const Density& density, const DiscreteFunction& v_hartree,
                    XcModel xc, const Molecule& molecule) {
  if (density.rho.space->mesh().id() != v_hartree.space->mesh().id())
    throw LineageError("total_energy: generations differ");
  if (lambdas.size() < density.occupations.size())
    throw InvalidArgumentError("total_energy: missing eigenvalue estimates");
  const std::size_t n = density.rho.coeffs.size();
  need(n);
  DevVec dr(n), dv(n);
  dr.up(density.rho.coeffs.data(), n);
  dv.up(v_hartree.coeffs.data(), n);
  std::vector<double> z, pos;
  for (const auto& nuc : molecule.nuclei) {
    z.push_back(nuc.charge);
    pos.insert(pos.end(), {nuc.position.x, nuc.position.y, nuc.position.z});
  }
  double e = 0.0;
  check(paro_total_energy(g.ctx, static_cast<int>(lambdas.size()), lambdas.data(),
                          static_cast<int>(density.occupations.size()), density.occupations.data(), dr.p, dv.p,
                          xc == XcModel::exchange_only ? 1 : 0, static_cast<int>(z.size()), z.data(), pos.data(), &e));
  return e;
}

ErrorIndicators ks_step2_indicators(const std::vector<DiscreteFunction>& occupied,
                                    const std::vector<double>& lambdas, const Density& rho_in,
                                    const DiscreteFunction& vh_in, const Molecule& molecule, double vext_smoothing,
                                    XcModel xc) {
  if (occupied.empty()) throw InvalidArgumentError("combine_max: empty input");
  if (lambdas.size() < occupied.size()) throw InvalidArgumentError("estimate: missing eigenvalue estimates");
  const std::size_t n = rho_in.rho.coeffs.size();
  need(n);
  std::vector<std::vector<double>> cols;
  for (const auto& u : occupied) {
    if (u.space->mesh().id() != rho_in.rho.space->mesh().id())
      throw LineageError("estimate: previous iterate lives on a different mesh generation");
    cols.push_back(u.coeffs);
  }
  DevVec du = pack(cols, n), dr(n), dv(n);
  dr.up(rho_in.rho.coeffs.data(), n);
  dv.up(vh_in.coeffs.data(), n);
  std::vector<double> z, pos;
  for (const auto& nuc : molecule.nuclei) {
    z.push_back(nuc.charge);
    pos.insert(pos.end(), {nuc.position.x, nuc.position.y, nuc.position.z});
  }
  ErrorIndicators out;
  out.mesh_id = rho_in.rho.space->mesh().id();
  out.eta.resize(rho_in.rho.space->mesh().element_count());
  DevVec deta(out.eta.size());
  double total = 0.0;
  check(paro_estimate_eta(g.ctx, static_cast<int>(cols.size()), du.p, static_cast<long long>(n), lambdas.data(), 0.5,
                          0, 0.0, static_cast<int>(z.size()), z.data(), pos.data(), vext_smoothing, dr.p, dv.p,
                          xc == XcModel::exchange_only ? 1 : 0, deta.p, &total));
  deta.down(out.eta.data(), out.eta.size());
  return out;
}

}  // namespace paro::gpu
