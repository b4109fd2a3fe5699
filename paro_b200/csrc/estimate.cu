// Step 2 on a fixed mesh: the residual error estimator of every orbital,
// combined by an element-wise maximum, and its total (the trace's eta_total).
//
//   estimate_source_residual  proj/src/adapt.cpp:58-102
//   estimate_eigen_residual   proj/src/adapt.cpp:104-115  (rhs = lambda u, same u)
//   combine_max / total       proj/src/adapt.cpp:117-129, :14-18
//   Kohn-Sham reaction        proj/src/paro.cpp:521-538   (V_ext + V_H + v_xc at the point)
//   linear drivers            proj/src/paro.cpp:306-315   (the problem's reaction)
//
// Per element e (6 s^3 Kuhn tets, reference element order) and orbital i:
//   eta2 = h_e^2 sum_q w_q |e| (lambda u(x_q) - c(x_q) u(x_q))^2
//        + sum over interior faces f of e of  1/2 diam(f) |f| ((F_e - F_e') . n_f)^2,
//   F = D grad u the element flux, D = d I; then eta_e = sqrt(max_i eta2).
// One thread per cell: the reaction at its 24 quadrature points is evaluated
// once, then the orbitals are streamed (14 vertex values per cell and
// orbital: the 8 cube corners and the 6 vertices the face-neighbour tets of
// the adjacent cells add). On the uniform Kuhn mesh every face neighbour is
// the tet that shares three path vertices: across the lower p2 face the tet
// (p2, p0, p1) of cell c - e_p2, across the upper p0 face (p1, p2, p0) of
// c + e_p0, inside the cube (p1, p0, p2) and (p0, p2, p1); the gradient of a
// Kuhn tet is the difference quotient along its path. Geometry uses the
// uniform spacing h (faces: cube faces h^2/2 and diam h sqrt2, diagonal faces
// h^2 sqrt2/2 and diam h sqrt3); the reference evaluates the same quantities
// from vertex coordinates, so eta agrees to rounding, not bit for bit.
#include <cmath>
#include <vector>

#include "ctx.hpp"
#include "estimate.hpp"
#include "fem.cuh"
#include "quad.hpp"

namespace paro_b200 {

namespace {

struct EstArgs {
  Box box;
  double h = 0.0;
  int N = 0;
  const double* U = nullptr;
  long long ld = 0;
  const double* lambdas = nullptr;  // device, N
  double diff = 0.0;
  int kind = 0;                     // kEstKs / kEstHarmonic / kEstWell
  double c = 0.0;
  int nnuc = 0;
  const double* nuc = nullptr;      // Z, x, y, z per nucleus
  double eps2 = 0.0;
  int soft = 0;
  const double* rho = nullptr;
  const double* vh = nullptr;
  int exchange_only = 0;
  double cx = 0.0;
  const double* qp = nullptr;       // 4-point rule: barycentric (4 x 4), weights (4)
  const double* qw = nullptr;
  double* eta = nullptr;            // optional, 6 s^3
  double* partial = nullptr;        // per block: sum of eta^2
};

constexpr int kEstThreads = 128;

__device__ double ext_potential(const EstArgs& a, V3 x) {
  double v = 0.0;
  if (a.soft) {  // external_potential, eps > 0 (model.cpp:163-173)
    for (int k = 0; k < a.nnuc; ++k) {
      const V3 d = v3sub(x, V3{a.nuc[4 * k + 1], a.nuc[4 * k + 2], a.nuc[4 * k + 3]});
      v -= a.nuc[4 * k] / sqrt(v3dot(d, d) + a.eps2);
    }
  } else {  // eps = 0 (model.cpp:150-162)
    for (int k = 0; k < a.nnuc; ++k) v -= a.nuc[4 * k] / v3dist(x, V3{a.nuc[4 * k + 1], a.nuc[4 * k + 2], a.nuc[4 * k + 3]});
  }
  return v;
}

__device__ __forceinline__ double uval(const EstArgs& a, const double* u, int vx, int vy, int vz) {
  const long long d = vertex_dof(a.box.s, vx, vy, vz);
  return d >= 0 ? u[d] : 0.0;
}

__global__ void __launch_bounds__(kEstThreads) estimate_kernel(const EstArgs a) {
  const int s = a.box.s;
  const long long ncell = static_cast<long long>(s) * s * s;
  const long long cidx = blockIdx.x * static_cast<long long>(kEstThreads) + threadIdx.x;
  double sum2 = 0.0;
  if (cidx < ncell) {
    const int ci = static_cast<int>(cidx % s), cj = static_cast<int>((cidx / s) % s),
              ck = static_cast<int>(cidx / (static_cast<long long>(s) * s));
    // reaction at the 24 quadrature points (orbital independent)
    double react[6][4];
    // the cell's corner coordinates, once (coord() divides by s)
    const double x0c = a.box.coord(ci), x1c = a.box.coord(ci + 1), y0c = a.box.coord(cj), y1c = a.box.coord(cj + 1);
    const double z0c = a.box.coord(ck), z1c = a.box.coord(ck + 1);
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      int tc[4][3];
      tet_corners(p, tc);
      V3 P[4];
      int vtx[4][3];
      for (int i = 0; i < 4; ++i) {
        vtx[i][0] = ci + tc[i][0];
        vtx[i][1] = cj + tc[i][1];
        vtx[i][2] = ck + tc[i][2];
        P[i] = V3{tc[i][0] ? x1c : x0c, tc[i][1] ? y1c : y0c, tc[i][2] ? z1c : z0c};
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const V3 x = quad_point(P, a.qp + 4 * q);
        double w;
        if (a.kind == kEstHarmonic) {
          w = a.c * (x.x * x.x + x.y * x.y + x.z * x.z);
        } else if (a.kind == kEstWell) {
          w = ext_potential(a, x);
        } else {  // V_ext(x) + V_H(x) + v_xc(rho(x)), rho / V_H interpolated (paro.cpp:525-531)
          double bary[4];
          barycentric(P, x, bary);
          double rq = 0.0, vq = 0.0;
          for (int i = 0; i < 4; ++i) {
            const long long d = vertex_dof(s, vtx[i][0], vtx[i][1], vtx[i][2]);
            if (d >= 0) {
              rq += bary[i] * a.rho[d];
              vq += bary[i] * a.vh[d];
            }
          }
          w = ext_potential(a, x) + vq + lda_vxc(rq, a.exchange_only != 0, a.cx).v;
        }
        react[p][q] = w;
      }
    }
    const double h = a.h;
    const double he2 = 3.0 * h * h;                       // element diameter^2 (the main diagonal)
    const double wvol = 0.25 * (h * h * h / 6.0);         // w_q |e|
    const double fcube = 0.5 * (h * sqrt(2.0)) * (0.5 * h * h);
    const double fdiag = 0.5 * (h * sqrt(3.0)) * (0.5 * h * h * sqrt(2.0));
    const double rs2 = 1.0 / sqrt(2.0);
    const bool lower[3] = {ci > 0, cj > 0, ck > 0};
    const bool upper[3] = {ci + 1 < s, cj + 1 < s, ck + 1 < s};
    double best[6];
    for (int p = 0; p < 6; ++p) best[p] = 0.0;

    for (int i = 0; i < a.N; ++i) {
      const double* u = a.U + static_cast<long long>(i) * a.ld;
      const double lam = a.lambdas[i];
      // corners: cu[dz][dy][dx]
      double cu[2][2][2];
#pragma unroll
      for (int dz = 0; dz < 2; ++dz)
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
          for (int dx = 0; dx < 2; ++dx) cu[dz][dy][dx] = uval(a, u, ci + dx, cj + dy, ck + dz);
      // below v0 along axis d, and beyond (1,1,1) along axis d
      const double ub[3] = {uval(a, u, ci - 1, cj, ck), uval(a, u, ci, cj - 1, ck), uval(a, u, ci, cj, ck - 1)};
      const double ua[3] = {uval(a, u, ci + 2, cj + 1, ck + 1), uval(a, u, ci + 1, cj + 2, ck + 1),
                            uval(a, u, ci + 1, cj + 1, ck + 2)};
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        // the Kuhn permutations of mesh.cpp:457-471, compile-time after unrolling
        constexpr int kP[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        const int p0 = kP[p][0], p1 = kP[p][1], p2 = kP[p][2];
        // path vertices v0..v3 and the two same-cell detour vertices
        int o[3] = {0, 0, 0};
        const double u0 = cu[0][0][0];
        o[p0] = 1;
        const double u1 = cu[o[2]][o[1]][o[0]];
        o[p1] = 1;
        const double u2 = cu[o[2]][o[1]][o[0]];
        const double u3 = cu[1][1][1];
        int m[3] = {0, 0, 0};
        m[p1] = 1;
        const double um = cu[m[2]][m[1]][m[0]];   // v0 + e_p1
        int m2[3] = {0, 0, 0};
        m2[p0] = 1;
        m2[p2] = 1;
        const double um2 = cu[m2[2]][m2[1]][m2[0]];  // v1 + e_p2
        // interior residual (adapt.cpp:78-87), rhs = lambda u (adapt.cpp:108-111)
        double r2 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double* b = a.qp + 4 * q;
          const double uh = ((b[0] * u0 + b[1] * u1) + b[2] * u2) + b[3] * u3;
          const double r = lam * uh - react[p][q] * uh;
          r2 += wvol * r * r;
        }
        double e2 = he2 * r2;
        // flux components along the path axes: F = diff * grad u
        const double g0 = (u1 - u0) / h, g1 = (u2 - u1) / h, g2 = (u3 - u2) / h;
        // lower p2 face -> tet (p2,p0,p1) of c - e_p2: its p2 component
        if (lower[p2]) {
          const double jump = a.diff * (g2 - (u0 - ub[p2]) / h);
          e2 += fcube * jump * jump;
        }
        // upper p0 face -> tet (p1,p2,p0) of c + e_p0: its p0 component
        if (upper[p0]) {
          const double jump = a.diff * (g0 - (ua[p0] - u3) / h);
          e2 += fcube * jump * jump;
        }
        // face {v0,v2,v3} -> tet (p1,p0,p2): normal (e_p0 - e_p1)/sqrt2
        {
          const double d0 = g0 - (u2 - um) / h, d1 = g1 - (um - u0) / h;
          const double jump = a.diff * (d0 - d1) * rs2;
          e2 += fdiag * jump * jump;
        }
        // face {v0,v1,v3} -> tet (p0,p2,p1): normal (e_p1 - e_p2)/sqrt2
        {
          const double d1 = g1 - (u3 - um2) / h, d2 = g2 - (um2 - u1) / h;
          const double jump = a.diff * (d1 - d2) * rs2;
          e2 += fdiag * jump * jump;
        }
        best[p] = fmax(best[p], e2);
      }
    }
    for (int p = 0; p < 6; ++p) {
      const double eta = sqrt(fmax(0.0, best[p]));
      if (a.eta) a.eta[cidx * 6 + p] = eta;
      sum2 += eta * eta;
    }
  }
  // deterministic block sum
  __shared__ double red[kEstThreads / 32];
  for (int o = 16; o > 0; o >>= 1) sum2 += __shfl_down_sync(0xffffffffu, sum2, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kEstThreads / 32; ++w) t += red[w];
    a.partial[blockIdx.x] = t;
  }
}

__global__ void sum_kernel(const double* part, long long m, double* out) {
  // one warp, fixed order: lane-strided partial sums, then a shuffle tree
  double s = 0.0;
  for (long long i = threadIdx.x; i < m; i += 32) s += part[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = s;
}

}  // namespace

double estimate_eta(Ctx& ctx, const EstimateSpec& spec, int N, const double* U, long long ld, double* eta) {
  ctx.check_grid();
  const Grid& g = ctx.grid;
  if (N <= 0) throw ParoError(kInvalidArgument, "estimate: no orbitals");
  if (spec.diffusion <= 0.0) throw ParoError(kInvalidArgument, "estimate: diffusion scale must be positive");
  EstArgs a;
  a.box = Box{g.s, g.lo, g.hi};
  a.h = (g.hi - g.lo) / g.s;
  a.N = N;
  a.U = U;
  a.ld = ld;
  a.diff = spec.diffusion;
  a.kind = spec.kind;
  a.c = spec.c;
  a.rho = spec.rho;
  a.vh = spec.vh;
  a.exchange_only = spec.exchange_only;
  a.cx = std::cbrt(3.0 / M_PI);
  a.eta = eta;
  if (spec.kind == kEstKs && (!spec.rho || !spec.vh)) throw ParoError(kInvalidArgument, "estimate: rho and V_H needed");
  const size_t nn = spec.nuclei.size();
  if ((spec.kind == kEstKs || spec.kind == kEstWell) && (nn == 0 || nn % 4 != 0))
    throw ParoError(kInvalidArgument, "external_potential: no nuclei");
  const Rule rule = simplex_rule3(2);
  std::vector<double> host;
  for (const auto& pt : rule.points)
    for (int c = 0; c < 4; ++c) host.push_back(pt[c]);
  for (double w : rule.weights) host.push_back(w);
  const size_t off_l = host.size();
  for (int i = 0; i < N; ++i) host.push_back(spec.lambdas[i]);
  const size_t off_n = host.size();
  for (double v : spec.nuclei) host.push_back(v);
  double* d = ctx.ws_small3.get<double>(host.size() + 1);
  PARO_CUDA(cudaMemcpyAsync(d, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, ctx.stream));
  a.qp = d;
  a.qw = d + 16;
  a.lambdas = d + off_l;
  a.nuc = nn ? d + off_n : nullptr;
  a.nnuc = static_cast<int>(nn / 4);
  a.eps2 = spec.eps * spec.eps;
  a.soft = spec.eps > 0.0;
  const long long ncell = static_cast<long long>(g.s) * g.s * g.s;
  const long long blocks = (ncell + kEstThreads - 1) / kEstThreads;
  double* part = ctx.ws_gram.get<double>(static_cast<size_t>(blocks) + 1);
  a.partial = part;
  estimate_kernel<<<static_cast<unsigned>(blocks), kEstThreads, 0, ctx.stream>>>(a);
  sum_kernel<<<1, 32, 0, ctx.stream>>>(part, blocks, part + blocks);
  PARO_CUDA(cudaGetLastError());
  ctx.launches += 2;
  double total2 = 0.0;
  PARO_CUDA(cudaMemcpyAsync(&total2, part + blocks, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
  return std::sqrt(total2);
}

}  // namespace paro_b200
