// Operator assembly on the device (compiled -fmad=false).
//
// One thread per interior dof v gathers the 8 stencil slots of its row
// (diagonal + the 7 forward Kuhn edges) from the 24 incident tetrahedra,
// visiting them in the reference's global element order (cells by (k,j,i),
// then the 6 Kuhn permutations), so each slot is the same sum of element
// contributions, in the same order, as the CSR entry produced by
// assemble_matrix (fem.cpp:162-183). Element-local rows follow
// assemble_mass (fem.cpp:253-268), assemble_stiffness (fem.cpp:221-251) and
// assemble_weighted_mass with pick_weighted_rule (fem.cpp:272-321); the
// Kohn-Sham form adds kinetic + V_ext + (V_H + v_xc) mass exactly like
// ks_form_matrix (paro.cpp:433-454).
#include <vector>

#include "assemble.hpp"
#include "fem.cuh"

namespace paro_b200 {

namespace {

struct AsmArgs {
  Box box;
  long long n = 0;
  int kind = 0;
  double scale = 0.0;        // stiffness diffusion scale / harmonic coefficient
  int nq = 0;                // main rule
  const double* qp = nullptr;
  const double* qw = nullptr;
  int nqs = 0;               // subdivided rule for elements near a singular point
  const double* qps = nullptr;
  const double* qws = nullptr;
  int nnuc = 0;
  const double* nuc = nullptr;  // Z, x, y, z per nucleus
  double eps2 = 0.0;
  int singular = 0;          // singular-quadrature policy active (bare Coulomb)
  const double* rho = nullptr;
  const double* vh = nullptr;
  int exchange_only = 0;
  double cx = 0.0;
  // KS form: out = (kinetic + vext) + scf
  const double* kin_coef = nullptr;
  double kin_w[kSlots] = {};
  const double* vext_coef = nullptr;
  double* out = nullptr;
  int* flags = nullptr;      // bit0 singular point hit, bit1 non-finite weight
  const double* wtab = nullptr;  // 4-point rules: precomputed w(x_q) per (cell, tet, point)
  unsigned long long* clamps = nullptr;  // Scf: count of rho(x_q) < 0
  // plane-restricted assembly: cells [cell0, cell1) feed the table, cells [ccnt0, ccnt1) the
  // clamp count, dofs [dof0, dof1) are gathered
  long long cell0 = 0, cell1 = 0, ccnt0 = 0, ccnt1 = 0, dof0 = 0, dof1 = 0;
};

__device__ __forceinline__ double eval_in_element(const double* f, int s, const int (&vtx)[4][3],
                                                  const double (&bary)[4]) {
  double v = 0.0;
  for (int i = 0; i < 4; ++i) {
    const long long d = vertex_dof(s, vtx[i][0], vtx[i][1], vtx[i][2]);
    if (d >= 0) v += bary[i] * f[d];
  }
  return v;
}

// weight function w(e, x) of the weighted-mass kinds; *neg (Scf) is set when
// the interpolated density is negative (lda_vxc clamps it, model.cpp:270-273)
__device__ double weight_at(const AsmArgs& a, const V3 (&P)[4], const int (&vtx)[4][3], V3 x, bool* neg = nullptr) {
  if (a.kind == kAsmCoulomb) {  // external_potential, eps = 0 (model.cpp:150-162)
    double v = 0.0;
    for (int k = 0; k < a.nnuc; ++k) {
      const V3 R{a.nuc[4 * k + 1], a.nuc[4 * k + 2], a.nuc[4 * k + 3]};
      const double r = v3dist(x, R);
      if (r < 1e-14) atomicOr(a.flags, 1);
      v -= a.nuc[4 * k] / r;
    }
    return v;
  }
  if (a.kind == kAsmSoftCoulomb) {  // external_potential, eps > 0 (model.cpp:163-173)
    double v = 0.0;
    for (int k = 0; k < a.nnuc; ++k) {
      const V3 d = v3sub(x, V3{a.nuc[4 * k + 1], a.nuc[4 * k + 2], a.nuc[4 * k + 3]});
      v -= a.nuc[4 * k] / sqrt(v3dot(d, d) + a.eps2);
    }
    return v;
  }
  if (a.kind == kAsmHarmonic) return a.scale * (x.x * x.x + x.y * x.y + x.z * x.z);
  // kAsmScf: scf_potential_field (paro.cpp:433-444)
  double bary[4];
  barycentric(P, x, bary);
  const double rho_q = eval_in_element(a.rho, a.box.s, vtx, bary);
  if (neg) *neg = rho_q < 0.0;
  const Lda l = lda_vxc(rho_q, a.exchange_only != 0, a.cx);
  return eval_in_element(a.vh, a.box.s, vtx, bary) + l.v;
}

// qw_q |e| w(x_q) of every (cell, Kuhn tet, quadrature point) of a 4-point
// rule, each evaluated once (the dof gather below otherwise evaluates it for
// each of the tet's 4 vertices, with the same floating-point operations), so
// the gather of a weighted mass needs no element geometry at all.
__global__ void __launch_bounds__(128) wtable_kernel(const AsmArgs a, double* wtab) {
  const int s = a.box.s;
  const long long cidx = a.cell0 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (cidx >= a.cell1) return;
  const int ci = static_cast<int>(cidx % s), cj = static_cast<int>((cidx / s) % s),
            ck = static_cast<int>(cidx / (static_cast<long long>(s) * s));
  unsigned nneg = 0;
  // the cell's corner coordinates, once (coord() divides by s)
  const double x0c = a.box.coord(ci), x1c = a.box.coord(ci + 1), y0c = a.box.coord(cj), y1c = a.box.coord(cj + 1);
  const double z0c = a.box.coord(ck), z1c = a.box.coord(ck + 1);
  for (int p = 0; p < 6; ++p) {
    int tc[4][3];
    tet_corners(p, tc);
    int vtx[4][3];
    V3 P[4];
    for (int i = 0; i < 4; ++i) {
      vtx[i][0] = ci + tc[i][0];
      vtx[i][1] = cj + tc[i][1];
      vtx[i][2] = ck + tc[i][2];
      P[i] = V3{tc[i][0] ? x1c : x0c, tc[i][1] ? y1c : y0c, tc[i][2] ? z1c : z0c};
    }
    const double vol = tet_volume(P);
    for (int q = 0; q < a.nq; ++q) {
      const V3 x = quad_point(P, a.qp + 4 * q);
      bool neg = false;
      const double wq = weight_at(a, P, vtx, x, &neg);
      nneg += neg ? 1 : 0;
      if (!isfinite(wq)) atomicOr(a.flags, 2);
      // the gather's per-element factor qw[q] |e| w(x_q), same association
      wtab[(cidx * 6 + p) * 4 + q] = a.qw[q] * vol * wq;
    }
  }
  if (nneg && a.clamps && cidx >= a.ccnt0 && cidx < a.ccnt1) atomicAdd(a.clamps, static_cast<unsigned long long>(nneg));
}

// Weighted-mass gather from the quadrature table with the cell / tet loops
// unrolled at compile time: for the dof's corner lv = -(DI, DJ, DK) of cell
// (I+DI, J+DJ, K+DK), tet P = (A, B, C) contains it as local vertex IV
// (corners (0,0,0), e_A, (1,1,1) - e_C, (1,1,1)), so every index below is a
// constant. Same operations and order as assemble_kernel's table branch.
__host__ __device__ constexpr int kuhn_corner(int j, int p, int d) {
  return j == 0 ? 0 : j == 3 ? 1 : j == 1 ? (d == (p >> 1) ? 1 : 0) : (d == ((294 >> (2 * p)) & 3) ? 0 : 1);
}
__host__ __device__ constexpr int kuhn_iv(int l0, int l1, int l2, int p) {
  for (int j = 0; j < 4; ++j)
    if (kuhn_corner(j, p, 0) == l0 && kuhn_corner(j, p, 1) == l1 && kuhn_corner(j, p, 2) == l2) return j;
  return -1;
}

template <int DI, int DJ, int DK, int P>
__device__ __forceinline__ void gather_tet(const AsmArgs& a, const double (&qp)[16], int I, int J, int K,
                                           double (&acc)[kSlots]) {
  constexpr int IV = kuhn_iv(-DI, -DJ, -DK, P);
  if constexpr (IV >= 0) {
    const int s = a.box.s;
    const double* wt =
        a.wtab + ((((static_cast<long long>(K + DK) * s) + (J + DJ)) * s + (I + DI)) * 6 + P) * 4;
    double row[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double ww = wt[q];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int hi = IV > j ? IV : j, lo = IV > j ? j : IV;
        row[j] += ww * qp[4 * q + hi] * qp[4 * q + lo];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ox = kuhn_corner(j, P, 0) - kuhn_corner(IV, P, 0);
      const int oy = kuhn_corner(j, P, 1) - kuhn_corner(IV, P, 1);
      const int oz = kuhn_corner(j, P, 2) - kuhn_corner(IV, P, 2);
      if (j == IV) acc[0] += row[j];
      else if (ox >= 0 && oy >= 0 && oz >= 0) acc[ox + 2 * oy + 4 * oz] += row[j];
    }
  }
}

template <int DI, int DJ, int DK>
__device__ __forceinline__ void gather_cell(const AsmArgs& a, const double (&qp)[16], int I, int J, int K,
                                            double (&acc)[kSlots]) {
  gather_tet<DI, DJ, DK, 0>(a, qp, I, J, K, acc);
  gather_tet<DI, DJ, DK, 1>(a, qp, I, J, K, acc);
  gather_tet<DI, DJ, DK, 2>(a, qp, I, J, K, acc);
  gather_tet<DI, DJ, DK, 3>(a, qp, I, J, K, acc);
  gather_tet<DI, DJ, DK, 4>(a, qp, I, J, K, acc);
  gather_tet<DI, DJ, DK, 5>(a, qp, I, J, K, acc);
}

__global__ void __launch_bounds__(128) table_gather_kernel(const AsmArgs a) {
  const long long t = a.dof0 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (t >= a.dof1) return;
  const int s = a.box.s;
  const long long S = s - 1;
  const int I = static_cast<int>(t % S) + 1;
  const int J = static_cast<int>((t / S) % S) + 1;
  const int K = static_cast<int>(t / (S * S)) + 1;
  double qp[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) qp[i] = __ldg(a.qp + i);
  double acc[kSlots];
#pragma unroll
  for (int o = 0; o < kSlots; ++o) acc[o] = 0.0;
  // cells in the reference's element order: (k, j, i) ascending
  gather_cell<-1, -1, -1>(a, qp, I, J, K, acc);
  gather_cell<0, -1, -1>(a, qp, I, J, K, acc);
  gather_cell<-1, 0, -1>(a, qp, I, J, K, acc);
  gather_cell<0, 0, -1>(a, qp, I, J, K, acc);
  gather_cell<-1, -1, 0>(a, qp, I, J, K, acc);
  gather_cell<0, -1, 0>(a, qp, I, J, K, acc);
  gather_cell<-1, 0, 0>(a, qp, I, J, K, acc);
  gather_cell<0, 0, 0>(a, qp, I, J, K, acc);
#pragma unroll
  for (int o = 0; o < kSlots; ++o) {
    double v = acc[o];
    if (a.kind == kAsmScf && a.vext_coef) {
      // ks_form_matrix: a = kinetic; a += vext_mass; a += scf_mass
      const double kin = a.kin_coef ? a.kin_coef[o * a.n + t] : a.kin_w[o];
      v = (kin + a.vext_coef[o * a.n + t]) + v;
    }
    a.out[o * a.n + t] = v;
  }
}

__global__ void __launch_bounds__(128) assemble_kernel(const AsmArgs a) {
  const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (t >= a.n) return;
  const int s = a.box.s;
  const long long S = s - 1;
  const int I = static_cast<int>(t % S) + 1;
  const int J = static_cast<int>((t / S) % S) + 1;
  const int K = static_cast<int>(t / (S * S)) + 1;

  double acc[kSlots];
#pragma unroll
  for (int o = 0; o < kSlots; ++o) acc[o] = 0.0;

  for (int dk = -1; dk <= 0; ++dk)
    for (int dj = -1; dj <= 0; ++dj)
      for (int di = -1; di <= 0; ++di) {
        const int ci = I + di, cj = J + dj, ck = K + dk;
        const int lv[3] = {I - ci, J - cj, K - ck};
        for (int p = 0; p < 6; ++p) {
          int tc[4][3];
          tet_corners(p, tc);
          int iv = -1;
          for (int i = 0; i < 4; ++i)
            if (tc[i][0] == lv[0] && tc[i][1] == lv[1] && tc[i][2] == lv[2]) iv = i;
          if (iv < 0) continue;
          double row[4] = {0.0, 0.0, 0.0, 0.0};  // local[max(iv,j)][min(iv,j)]
          if (a.wtab) {  // weighted mass, 4-point rule: qw_q |e| w(x_q) from the table
            const double* wt = a.wtab + ((((static_cast<long long>(ck) * s) + cj) * s + ci) * 6 + p) * 4;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double ww = wt[q];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int hi = iv > j ? iv : j, lo = iv > j ? j : iv;
                row[j] += ww * a.qp[4 * q + hi] * a.qp[4 * q + lo];
              }
            }
          } else {
          int vtx[4][3];
          V3 P[4];
          for (int i = 0; i < 4; ++i) {
            vtx[i][0] = ci + tc[i][0];
            vtx[i][1] = cj + tc[i][1];
            vtx[i][2] = ck + tc[i][2];
            P[i] = V3{a.box.coord(vtx[i][0]), a.box.coord(vtx[i][1]), a.box.coord(vtx[i][2])};
          }
          const double vol = tet_volume(P);
          if (a.kind == kAsmMass) {
            for (int j = 0; j < 4; ++j) row[j] = vol * (j == iv ? 2.0 : 1.0) / 20.0;
          } else if (a.kind == kAsmStiffness) {
            const V3 ea = v3sub(P[1], P[0]), eb = v3sub(P[2], P[0]), ec = v3sub(P[3], P[0]);
            const double det = v3dot(ea, v3cross(eb, ec));
            V3 g[4];
            g[1] = v3scale(1.0 / det, v3cross(eb, ec));
            g[2] = v3scale(1.0 / det, v3cross(ec, ea));
            g[3] = v3scale(1.0 / det, v3cross(ea, eb));
            V3 sum{0.0, 0.0, 0.0};
            for (int i = 1; i <= 3; ++i) sum = v3add(sum, g[i]);
            g[0] = V3{-sum.x, -sum.y, -sum.z};
            const double m = a.scale;
            for (int q = 0; q < a.nq; ++q) {
              const double w = a.qw[q] * vol;
              for (int j = 0; j < 4; ++j) {
                const int hi = iv > j ? iv : j, lo = iv > j ? j : iv;
                const V3 gi = g[hi];
                // Mat3::identity(m).apply(gi) (geometry.hpp:43-47)
                const V3 agi{m * gi.x + 0.0 * gi.y + 0.0 * gi.z, 0.0 * gi.x + m * gi.y + 0.0 * gi.z,
                             0.0 * gi.x + 0.0 * gi.y + m * gi.z};
                row[j] += w * (v3dot(agi, g[lo]) + 0.0 * a.qp[4 * q + hi] * a.qp[4 * q + lo]);
              }
            }
          } else {
            // pick_weighted_rule (fem.cpp:272-287)
            int nq = a.nq;
            const double* qp = a.qp;
            const double* qw = a.qw;
            if (a.singular) {
              double h = 0.0;
              for (int i = 0; i <= 3; ++i)
                for (int j = i + 1; j <= 3; ++j) h = fmax(h, v3dist(P[i], P[j]));
              V3 bc{0.0, 0.0, 0.0};
              for (int i = 0; i <= 3; ++i) bc = v3add(bc, P[i]);
              bc = v3scale(1.0 / 4, bc);
              for (int k = 0; k < a.nnuc; ++k) {
                const V3 R{a.nuc[4 * k + 1], a.nuc[4 * k + 2], a.nuc[4 * k + 3]};
                if (v3dist(bc, R) < 1.5 * h) {
                  double br[4];
                  barycentric(P, R, br);
                  bool near = true;
                  for (int i = 0; i <= 3; ++i) near = near && br[i] > -0.25;
                  if (near) {
                    nq = a.nqs;
                    qp = a.qps;
                    qw = a.qws;
                    break;
                  }
                }
              }
            }
            for (int q = 0; q < nq; ++q) {
              const V3 x = quad_point(P, qp + 4 * q);
              const double wq = weight_at(a, P, vtx, x);
              if (!isfinite(wq)) atomicOr(a.flags, 2);
              const double ww = qw[q] * vol * wq;
              for (int j = 0; j < 4; ++j) {
                const int hi = iv > j ? iv : j, lo = iv > j ? j : iv;
                row[j] += ww * qp[4 * q + hi] * qp[4 * q + lo];
              }
            }
          }
          }
          for (int j = 0; j < 4; ++j) {
            const int ox = tc[j][0] - tc[iv][0], oy = tc[j][1] - tc[iv][1], oz = tc[j][2] - tc[iv][2];
            if (j == iv) acc[0] += row[j];
            else if (ox >= 0 && oy >= 0 && oz >= 0) acc[ox + 2 * oy + 4 * oz] += row[j];
          }
        }
      }
#pragma unroll
  for (int o = 0; o < kSlots; ++o) {
    double v = acc[o];
    if (a.kind == kAsmScf && a.vext_coef) {
      // ks_form_matrix: a = kinetic; a += vext_mass; a += scf_mass
      const double kin = a.kin_coef ? a.kin_coef[o * a.n + t] : a.kin_w[o];
      v = (kin + a.vext_coef[o * a.n + t]) + v;
    }
    a.out[o * a.n + t] = v;
  }
}

// Uniform-operator detection: compare every defined slot with dof 0's.
__global__ void uniform_kernel(const double* coef, long long n, int S, int* mismatch) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(t % S), y = static_cast<int>((t / S) % S), z = static_cast<int>(t / (static_cast<long long>(S) * S));
    for (int o = 0; o < kSlots; ++o) {
      if (x + (o & 1) >= S || y + ((o >> 1) & 1) >= S || z + ((o >> 2) & 1) >= S) continue;
      if (coef[o * n + t] != coef[o * n]) *mismatch = 1;
    }
  }
}

struct RuleDev {
  double* p = nullptr;
  double* w = nullptr;
  int n = 0;
};

RuleDev upload_rule(Ctx& ctx, DevBuf& buf, const Rule& r) {
  const size_t m = r.points.size();
  std::vector<double> host(5 * m);
  for (size_t q = 0; q < m; ++q) {
    for (int c = 0; c < 4; ++c) host[4 * q + c] = r.points[q][c];
    host[4 * m + q] = r.weights[q];
  }
  double* d = buf.get<double>(host.size());
  small_h2d(ctx, d, host.data(), sizeof(double) * host.size());
  return {d, d + 4 * m, static_cast<int>(m)};
}

}  // namespace

void assemble(Ctx& ctx, const AssembleSpec& spec, Op& out) {
  ctx.check_grid();
  const Grid& g = ctx.grid;
  if (!out.var || !out.coef) throw ParoError(kInvalidArgument, "assemble: output must be a variable operator");
  static thread_local DevBuf rule_main, rule_sub, nuc_buf, flag_buf;
  AsmArgs a;
  a.box = Box{g.s, g.lo, g.hi};
  a.n = g.n;
  a.kind = spec.kind;
  a.scale = spec.scale;
  a.out = out.coef;
  int* flags = flag_buf.get<int>(4);  // [0] error bits, [2..3] clamp counter
  PARO_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), ctx.stream));
  a.flags = flags;
  const bool wmass = spec.kind != kAsmMass && spec.kind != kAsmStiffness;
  const bool singular = spec.kind == kAsmCoulomb;
  // stiffness and non-singular weighted masses use simplex_rule(3, 2);
  // the singular policy uses degree 5 everywhere and the 2-level subdivided
  // degree-5 rule near a nucleus (SingularQuadPolicy, fem.hpp:71-76)
  const RuleDev main = upload_rule(ctx, rule_main, simplex_rule3(singular ? 5 : 2));
  a.nq = main.n;
  a.qp = main.p;
  a.qw = main.w;
  if (singular) {
    const RuleDev sub = upload_rule(ctx, rule_sub, subdivided_rule3(5, 2));
    a.nqs = sub.n;
    a.qps = sub.p;
    a.qws = sub.w;
    a.singular = 1;
  }
  if (wmass && (spec.kind == kAsmCoulomb || spec.kind == kAsmSoftCoulomb)) {
    const std::vector<double>& nuc = spec.nuclei;
    if (nuc.empty() || nuc.size() % 4 != 0) throw ParoError(kInvalidArgument, "external_potential: no nuclei");
    double* d = nuc_buf.get<double>(nuc.size() + 1);
    small_h2d(ctx, d, nuc.data(), sizeof(double) * nuc.size());
    a.nuc = d;
    a.nnuc = static_cast<int>(nuc.size() / 4);
    a.eps2 = spec.eps * spec.eps;
  }
  if (spec.kind == kAsmScf) {
    a.rho = spec.rho;
    a.vh = spec.vh;
    a.exchange_only = spec.exchange_only;
    a.cx = std::cbrt(3.0 / M_PI);
    if (spec.kinetic) {
      a.kin_coef = spec.kinetic->var ? spec.kinetic->coef : nullptr;
      for (int o = 0; o < kSlots; ++o) a.kin_w[o] = spec.kinetic->w[o];
    }
    a.vext_coef = spec.vext ? spec.vext->coef : nullptr;
    if (spec.vext && !spec.vext->var) throw ParoError(kInvalidArgument, "ks form: V_ext mass must be variable");
  }
  unsigned long long* clamps = nullptr;
  if (spec.kind == kAsmScf && spec.clamped) {
    clamps = reinterpret_cast<unsigned long long*>(flags + 2);
    PARO_CUDA(cudaMemsetAsync(clamps, 0, sizeof(unsigned long long), ctx.stream));
    a.clamps = clamps;
  }
  const long long ncell = static_cast<long long>(g.s) * g.s * g.s;
  const long long cplane = static_cast<long long>(g.s) * g.s, dplane = static_cast<long long>(g.S) * g.S;
  a.cell0 = a.ccnt0 = 0;
  a.cell1 = a.ccnt1 = ncell;
  a.dof0 = 0;
  a.dof1 = g.n;
  const bool table = wmass && !singular && a.nq == 4;
  if (spec.z1 >= 0) {  // a slab of lattice planes [z0, z1): dof plane z is touched by the cell layers z and z + 1
    if (!table || spec.kind != kAsmScf) throw ParoError(kInvalidArgument, "assemble: plane ranges need the KS form");
    if (spec.z0 < 0 || spec.z1 > g.S || spec.z0 > spec.z1) throw ParoError(kInvalidArgument, "assemble: bad plane range");
    a.dof0 = spec.z0 * dplane;
    a.dof1 = spec.z1 * dplane;
    a.cell0 = spec.z0 * cplane;
    a.cell1 = std::min<long long>(ncell, (static_cast<long long>(spec.z1) + 1) * cplane);
    a.ccnt0 = spec.z0 * cplane;
    a.ccnt1 = spec.z1 == g.S ? ncell : spec.z1 * cplane;
  }
  if (table) {
    double* wt = ctx.wtab.get<double>(static_cast<size_t>(ncell) * 24);
    if (a.cell1 > a.cell0) {
      wtable_kernel<<<static_cast<unsigned>((a.cell1 - a.cell0 + 127) / 128), 128, 0, ctx.stream>>>(a, wt);
      ++ctx.launches;
    }
    a.wtab = wt;
  }
  const long long blocks = (a.dof1 - a.dof0 + 127) / 128;
  if (blocks > 0) {
    if (a.wtab) table_gather_kernel<<<static_cast<unsigned>(blocks), 128, 0, ctx.stream>>>(a);
    else assemble_kernel<<<static_cast<unsigned>(blocks), 128, 0, ctx.stream>>>(a);
    ++ctx.launches;
  }
  PARO_CUDA(cudaGetLastError());
  int hflags = 0;
  unsigned long long hclamps = 0;
  small_d2h(ctx, &hflags, flags, sizeof(int));
  if (clamps) small_d2h(ctx, &hclamps, clamps, sizeof(hclamps));
  if (spec.clamped) *spec.clamped = static_cast<long long>(hclamps);
  if (hflags & 1) throw ParoError(kError, "external potential evaluated at a nucleus");
  if (hflags & 2) throw ParoError(kError, "weighted mass: non-finite coefficient");
}

namespace {

// this += s * other (SparseOperator::add_scaled, linalg.cpp:120-125)
__global__ void add_scaled_kernel(double* a, const double* b, const double* bw, double s, long long n) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < 8 * n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double bv = b ? b[t] : bw[t / n];
    a[t] += s * bv;
  }
}

}  // namespace

void add_scaled(Ctx& ctx, Op& a, const Op& b, double s) {
  if (!a.var && !b.var) {
    for (int o = 0; o < kSlots; ++o) a.w[o] += s * b.w[o];
    return;
  }
  const long long n = ctx.grid.n;
  if (!a.var) {  // promote to a variable operator
    double* coef = nullptr;
    PARO_CUDA(cudaMalloc(&coef, sizeof(double) * kSlots * n));
    std::vector<double> w(kSlots * 1);
    for (int o = 0; o < kSlots; ++o) {
      std::vector<double> col(n, a.w[o]);
      PARO_CUDA(cudaMemcpy(coef + o * n, col.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    }
    a.coef = coef;
    a.owns = true;
    a.var = true;
    a.n = n;
  }
  static thread_local DevBuf wbuf;
  double* dw = wbuf.get<double>(kSlots);
  small_h2d(ctx, dw, b.w, sizeof(double) * kSlots);
  add_scaled_kernel<<<148 * 8, 256, 0, ctx.stream>>>(a.coef, b.var ? b.coef : nullptr, dw, s, n);
  ++ctx.launches;
  PARO_CUDA(cudaGetLastError());
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
}

bool make_uniform_if_possible(Ctx& ctx, Op& op) {
  if (!op.var) return true;
  static thread_local DevBuf flag_buf;
  int* d = flag_buf.get<int>(1);
  PARO_CUDA(cudaMemsetAsync(d, 0, sizeof(int), ctx.stream));
  uniform_kernel<<<148 * 8, 256, 0, ctx.stream>>>(op.coef, op.n, ctx.grid.S, d);
  ++ctx.launches;
  int h = 0;
  PARO_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
  if (h) return false;
  double w[kSlots];
  for (int o = 0; o < kSlots; ++o)
    PARO_CUDA(cudaMemcpy(&w[o], op.coef + o * op.n, sizeof(double), cudaMemcpyDeviceToHost));
  if (op.owns) cudaFree(op.coef);
  op.coef = nullptr;
  op.owns = false;
  op.var = false;
  for (int o = 0; o < kSlots; ++o) op.w[o] = w[o];
  return true;
}

}  // namespace paro_b200
