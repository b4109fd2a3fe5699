// Nodal fields on the device (compiled -fmad=false): density, mixing and the
// element reductions of the energy / norms.
//   density_from_orbitals (model.cpp:192-223), mix_density (model.cpp:225-236),
//   integrate (fem.cpp:419-430), norm_l2 (fem.cpp:432-448),
//   integrate_product (model.cpp:306-327), total_energy (model.cpp:329-360).
// Element sums run one cell (6 Kuhn tets) per thread with a fixed-order
// block/partial reduction, so results are deterministic run to run.
#include <cmath>
#include <vector>

#include "fem.cuh"
#include "fields.hpp"
#include "quad.hpp"

namespace paro_b200 {

namespace {

constexpr int kRedThreads = 256;

__global__ void density_kernel(int nocc, const double* U, long long ld, const double* occ, long long n,
                               double* rho) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    double r = 0.0;
    for (int i = 0; i < nocc; ++i) {
      const double u = U[i * ld + k];
      r += occ[i] * u * u;
    }
    rho[k] = r;
  }
}

__global__ void scale_kernel(double* f, long long n, double s) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    f[k] *= s;
}

__global__ void mix_kernel(const double* a, const double* b, double alpha, long long n, double* out) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    out[k] = (1.0 - alpha) * a[k] + alpha * b[k];
}

__global__ void diff_kernel(const double* a, const double* b, long long n, double* out) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    out[k] = a[k] - b[k];
}

struct CellArgs {
  Box box;
  int mode;
  const double* f;
  const double* g;
  const double* qp;  // 4-point rule
  const double* qw;
  int exchange_only;
  double cx;
  double* partials;
  long long cell0, cell1;  // cells [cell0, cell1) are summed (a slab's cell layers)
};

__device__ __forceinline__ double vval(const double* f, int s, int vx, int vy, int vz) {
  const long long d = vertex_dof(s, vx, vy, vz);
  return d >= 0 ? f[d] : 0.0;
}

__global__ void __launch_bounds__(kRedThreads) cell_reduce_kernel(const CellArgs a) {
  __shared__ double sh[kRedThreads / 32];
  const int s = a.box.s;
  const long long c = a.cell0 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  double acc = 0.0;
  if (c < a.cell1) {
    const int ci = static_cast<int>(c % s), cj = static_cast<int>((c / s) % s), ck = static_cast<int>(c / (static_cast<long long>(s) * s));
    // the cell's corner coordinates, once (coord() divides by s)
    const double x0c = a.box.coord(ci), x1c = a.box.coord(ci + 1), y0c = a.box.coord(cj), y1c = a.box.coord(cj + 1);
    const double z0c = a.box.coord(ck), z1c = a.box.coord(ck + 1);
    for (int p = 0; p < 6; ++p) {
      int tc[4][3];
      tet_corners(p, tc);
      int vtx[4][3];
      V3 P[4];
      double fv[4], gv[4];
      for (int i = 0; i < 4; ++i) {
        vtx[i][0] = ci + tc[i][0];
        vtx[i][1] = cj + tc[i][1];
        vtx[i][2] = ck + tc[i][2];
        P[i] = V3{tc[i][0] ? x1c : x0c, tc[i][1] ? y1c : y0c, tc[i][2] ? z1c : z0c};
        fv[i] = vval(a.f, s, vtx[i][0], vtx[i][1], vtx[i][2]);
        gv[i] = a.g ? vval(a.g, s, vtx[i][0], vtx[i][1], vtx[i][2]) : 0.0;
      }
      const double vol = tet_volume(P);
      if (a.mode == kCellIntegrate) {
        double sm = 0.0;
        for (int i = 0; i < 4; ++i) sm += fv[i];
        acc += vol * sm / 4;
      } else if (a.mode == kCellNorm2) {
        double sum = 0.0, sq = 0.0;
        for (int i = 0; i < 4; ++i) {
          sum += fv[i];
          sq += fv[i] * fv[i];
        }
        acc += vol * (sq + sum * sum) / 20.0;
      } else if (a.mode == kCellProduct) {
        double su = 0, sv = 0, sp = 0;
        for (int i = 0; i < 4; ++i) {
          su += fv[i];
          sv += gv[i];
          sp += fv[i] * gv[i];
        }
        acc += vol * (sp + su * sv) / 20.0;
      } else if (a.mode == kCellExc) {
        for (int q = 0; q < 4; ++q) {
          double r = 0.0;
          for (int i = 0; i < 4; ++i)
            if (vertex_dof(s, vtx[i][0], vtx[i][1], vtx[i][2]) >= 0) r += a.qp[4 * q + i] * fv[i];
          const double rho_q = fmax(0.0, r);
          const Lda x = lda_vxc(rho_q, a.exchange_only != 0, a.cx);
          acc += a.qw[q] * vol * (x.e - x.v) * rho_q;
        }
      } else {  // kCellClamp: (element, point) pairs where the KS form clamps rho
        for (int q = 0; q < 4; ++q) {
          const V3 x = quad_point(P, a.qp + 4 * q);
          double bary[4];
          barycentric(P, x, bary);
          double r = 0.0;
          for (int i = 0; i < 4; ++i)
            if (vertex_dof(s, vtx[i][0], vtx[i][1], vtx[i][2]) >= 0) r += bary[i] * fv[i];
          if (r < 0.0) acc += 1.0;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) t += sh[w];
    a.partials[blockIdx.x] = t;
  }
}

__global__ void sum_kernel(const double* p, long long m, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) s += p[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sh[w];
    *out = t;
  }
}

int grid1d(long long n) { return static_cast<int>(std::min<long long>(148 * 16, (n + 255) / 256)); }

// ---------------------------------------------------------------------------
// Nodal forms of the element sums on meshes whose P1 mass is one constant
// stencil (exact-binary spacings: every tet has the same volume, bit for bit).
// With f = g = 0 on the Dirichlet boundary,
//   integrate_product(f, g) = sum_t vol_t (sum_v f_v g_v + sum_v f_v sum_v g_v) / 20 = f' M g,
//   norm_l2(f)^2 = f' M f,   integrate(f) = sum_t vol_t sum_v f_v / 4 = (int phi_i) sum_i f_i,
// the same numbers as the element loops of fem.cpp:419-448 / model.cpp:306-327
// in a different summation order (differences ~1e-16 relative), one coalesced
// pass over the nodes instead of 24 vertex gathers per cell.
struct Stencil8 {
  double w[kSlots];
};

constexpr int kNodeBlocks = 148 * 8;

// partials[b] = sum over this block's nodes of f_i (M g)_i   (g == nullptr: of f_i)
__global__ void __launch_bounds__(kRedThreads) node_reduce_kernel(const double* __restrict__ f,
                                                                 const double* __restrict__ g, Stencil8 m, int S,
                                                                 long long n, double* partials) {
  __shared__ double sh[kRedThreads / 32];
  const long long S2 = static_cast<long long>(S) * S;
  double acc = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double fi = f[i];
    if (g == nullptr) {
      acc += fi;
      continue;
    }
    const int x = static_cast<int>(i % S), y = static_cast<int>((i / S) % S), z = static_cast<int>(i / S2);
    double s = m.w[0] * g[i];
#pragma unroll
    for (int o = 1; o < kSlots; ++o) {
      const int dx = o & 1, dy = (o >> 1) & 1, dz = o >> 2;
      const long long off = dx + static_cast<long long>(dy) * S + dz * S2;
      const bool fwd = x + dx < S && y + dy < S && z + dz < S;
      const bool bwd = x - dx >= 0 && y - dy >= 0 && z - dz >= 0;
      double t = 0.0;
      if (fwd) t += g[i + off];
      if (bwd) t += g[i - off];
      s += m.w[o] * t;
    }
    acc += fi * s;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) t += sh[w];
    partials[blockIdx.x] = t;
  }
}

// the grid's P1 mass is known as a constant stencil (recorded by paro_assemble_mass)
bool uniform_mass(const Ctx& ctx) { return ctx.mass_state == 1; }

double node_reduce(Ctx& ctx, int mode, const double* f, const double* g) {
  const Grid& gr = ctx.grid;
  static thread_local DevBuf part;
  double* partials = part.get<double>(kNodeBlocks + 1);
  Stencil8 m;
  double rowsum = ctx.mass_w[0];
  for (int o = 0; o < kSlots; ++o) {
    m.w[o] = ctx.mass_w[o];
    if (o) rowsum += 2.0 * ctx.mass_w[o];
  }
  const double* gg = mode == kCellIntegrate ? nullptr : mode == kCellNorm2 ? f : g;
  node_reduce_kernel<<<kNodeBlocks, kRedThreads, 0, ctx.stream>>>(f, gg, m, gr.S, gr.n, partials);
  sum_kernel<<<1, 1024, 0, ctx.stream>>>(partials, kNodeBlocks, partials + kNodeBlocks);
  ctx.launches += 2;
  PARO_CUDA(cudaGetLastError());
  double out = 0.0;
  small_d2h(ctx, &out, partials + kNodeBlocks, sizeof(double));
  return mode == kCellIntegrate ? rowsum * out : out;  // int phi_i = the mass row sum of an inner node
}

}  // namespace

double cell_reduce(Ctx& ctx, int mode, const double* f, const double* g, int exchange_only, int k0, int k1) {
  ctx.check_grid();
  const bool all = k1 < 0;
  if (all && (mode == kCellIntegrate || mode == kCellNorm2 || mode == kCellProduct) && ctx.nodal_sums &&
      uniform_mass(ctx))
    return node_reduce(ctx, mode, f, g);
  const Grid& gr = ctx.grid;
  if (!all && (k0 < 0 || k1 > gr.s || k0 > k1)) throw ParoError(kInvalidArgument, "cell sum: bad cell-layer range");
  static thread_local DevBuf rule, part;
  const Rule& r4 = simplex_rule3(2);
  std::vector<double> host(20);
  for (int q = 0; q < 4; ++q) {
    for (int c = 0; c < 4; ++c) host[4 * q + c] = r4.points[q][c];
    host[16 + q] = r4.weights[q];
  }
  double* drule = rule.get<double>(20);
  small_h2d(ctx, drule, host.data(), sizeof(double) * 20);
  const long long layer = static_cast<long long>(gr.s) * gr.s;
  const long long cell0 = all ? 0 : k0 * layer, cell1 = all ? layer * gr.s : k1 * layer;
  if (cell1 <= cell0) return 0.0;
  const long long blocks = (cell1 - cell0 + kRedThreads - 1) / kRedThreads;
  double* partials = part.get<double>(blocks + 1);
  CellArgs a{Box{gr.s, gr.lo, gr.hi}, mode, f, g, drule, drule + 16, exchange_only, std::cbrt(3.0 / M_PI), partials,
             cell0, cell1};
  cell_reduce_kernel<<<static_cast<unsigned>(blocks), kRedThreads, 0, ctx.stream>>>(a);
  sum_kernel<<<1, 1024, 0, ctx.stream>>>(partials, blocks, partials + blocks);
  ctx.launches += 2;
  PARO_CUDA(cudaGetLastError());
  double out = 0.0;
  small_d2h(ctx, &out, partials + blocks, sizeof(double));
  host.clear();
  return out;
}

// the nodal sum of density_from_orbitals (model.cpp:210-214) on rows [r0, r1)
// (rho indexed globally); returns the total occupation
double density_rows(Ctx& ctx, int nocc, const double* U, long long ld, const double* occ_host, long long r0,
                    long long r1, double* rho) {
  ctx.check_grid();
  if (nocc <= 0) throw ParoError(kInvalidArgument, "density: orbital/occupation count mismatch");
  if (r0 < 0 || r1 > ctx.grid.n || r1 < r0) throw ParoError(kInvalidArgument, "density: bad row range");
  double total = 0.0;
  for (int i = 0; i < nocc; ++i) {
    if (occ_host[i] < 0.0) throw ParoError(kInvalidArgument, "density: negative occupation");
    total += occ_host[i];
  }
  static thread_local DevBuf occ;
  double* docc = occ.get<double>(nocc);
  small_h2d(ctx, docc, occ_host, sizeof(double) * nocc);
  const long long n = r1 - r0;
  if (n > 0) {
    density_kernel<<<grid1d(n), 256, 0, ctx.stream>>>(nocc, U + r0, ld, docc, n, rho + r0);
    ++ctx.launches;
  }
  PARO_CUDA(cudaGetLastError());
  return total;
}

// the normalisation of density_from_orbitals (model.cpp:215-221); returns the raw integral
double density_normalize(Ctx& ctx, double total_occ, double* rho) {
  const long long n = ctx.grid.n;
  const double raw = cell_reduce(ctx, kCellIntegrate, rho, nullptr, 0);
  if (total_occ > 0.0 && raw > 0.0) {
    scale_kernel<<<grid1d(n), 256, 0, ctx.stream>>>(rho, n, total_occ / raw);
    ++ctx.launches;
  }
  PARO_CUDA(cudaGetLastError());
  return raw;
}

double density(Ctx& ctx, int nocc, const double* U, long long ld, const double* occ_host, double* rho) {
  const double total = density_rows(ctx, nocc, U, ld, occ_host, 0, ctx.grid.n, rho);
  return density_normalize(ctx, total, rho);
}

void mix(Ctx& ctx, const double* rin, const double* rout, double alpha, double* out) {
  const long long n = ctx.grid.n;
  mix_kernel<<<grid1d(n), 256, 0, ctx.stream>>>(rin, rout, alpha, n, out);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
}

void diff(Ctx& ctx, const double* a, const double* b, double* out) {
  const long long n = ctx.grid.n;
  diff_kernel<<<grid1d(n), 256, 0, ctx.stream>>>(a, b, n, out);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
}

double norm_l2(Ctx& ctx, const double* f) { return std::sqrt(std::max(0.0, cell_reduce(ctx, kCellNorm2, f, nullptr, 0))); }

// the XC term of total_energy, int rho (e_xc - v_xc), over the cell layers [k0, k1) (k1 < 0: all)
double energy_xc_term(Ctx& ctx, const double* rho, int exchange_only, int k0, int k1) {
  return cell_reduce(ctx, kCellExc, rho, nullptr, exchange_only, k0, k1);
}

double total_energy(Ctx& ctx, int nl, const double* lambdas, int nocc, const double* occ, const double* rho,
                    const double* vh, int exchange_only, int nnuc, const double* nuclei, const double* xc_term) {
  if (nl < nocc) throw ParoError(kInvalidArgument, "total_energy: missing eigenvalue estimates");
  double e_band = 0.0;
  for (int i = 0; i < nocc; ++i) e_band += occ[i] * lambdas[i];
  const double e_hartree = 0.5 * cell_reduce(ctx, kCellProduct, vh, rho, 0);
  // a sharded run passes the XC term it summed over the ranks' cell layers
  const double e_xc = xc_term ? *xc_term : cell_reduce(ctx, kCellExc, rho, nullptr, exchange_only);
  // nuclear_repulsion (model.cpp:177-186)
  double enn = 0.0;
  for (int k = 0; k < nnuc; ++k)
    for (int l = k + 1; l < nnuc; ++l) {
      const double dx = nuclei[4 * k + 1] - nuclei[4 * l + 1], dy = nuclei[4 * k + 2] - nuclei[4 * l + 2],
                   dz = nuclei[4 * k + 3] - nuclei[4 * l + 3];
      enn += nuclei[4 * k] * nuclei[4 * l] / std::sqrt(dx * dx + dy * dy + dz * dz);
    }
  return e_band - e_hartree + e_xc + enn;
}

}  // namespace paro_b200
