// Device geometry of the uniform Kuhn mesh and the LDA functional, restating
// the reference's floating-point order (compile the including files with
// -fmad=false): create_box_mesh (mesh.cpp:411-478), element volume
// (mesh.cpp:27-34), barycentric (mesh.cpp:145-165), barycentric_gradients
// (fem.cpp:65-88), quad_point (fem.cpp:211-217), evaluate_in_element
// (fem.cpp:389-399), lda_vxc (model.cpp:268-300).
#pragma once

#include "common.cuh"

namespace paro_b200 {

struct V3 {
  double x, y, z;
};

__device__ __forceinline__ V3 v3sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 v3add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 v3scale(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double v3dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 v3cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double v3dist(V3 a, V3 b) { return sqrt(v3dot(v3sub(a, b), v3sub(a, b))); }

// Kuhn decomposition: tet p of a cell visits corners (0,0,0) -> +e_perm[0]
// -> +e_perm[1] -> (1,1,1) (mesh.cpp:457-471).
__constant__ const int kPerms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

struct Box {
  int s;
  double lo, hi;
  // vertex coordinate lo + (hi - lo) * i / s   (mesh.cpp:432-434)
  __device__ __forceinline__ double coord(int i) const {
    return lo + (hi - lo) * static_cast<double>(i) / static_cast<double>(s);
  }
};

// corner offsets of tet p (cell-local, each component 0/1). For p = (a,b,c):
// corner 1 = e_a, corner 2 = e_a + e_b (every axis but c), corner 3 = (1,1,1);
// computed in registers (no table lookup, no dynamically indexed array).
__device__ __forceinline__ void tet_corners(int p, int (&t)[4][3]) {
  const int a = p >> 1;                 // kPerms[p][0]
  const int c = (294 >> (2 * p)) & 3;   // kPerms[p][2]: 2,1,2,0,1,0
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    t[0][d] = 0;
    t[1][d] = d == a ? 1 : 0;
    t[2][d] = d == c ? 0 : 1;
    t[3][d] = 1;
  }
}

__device__ __forceinline__ double tet_volume(const V3 (&P)[4]) {
  const V3 u = v3sub(P[1], P[0]), v = v3sub(P[2], P[0]), w = v3sub(P[3], P[0]);
  return fabs(v3dot(u, v3cross(v, w))) / 6.0;
}

__device__ __forceinline__ void barycentric(const V3 (&P)[4], V3 x, double (&lam)[4]) {
  const V3 a = v3sub(P[1], P[0]), b = v3sub(P[2], P[0]), c = v3sub(P[3], P[0]);
  const V3 r = v3sub(x, P[0]);
  const double det = v3dot(a, v3cross(b, c));
  lam[1] = v3dot(r, v3cross(b, c)) / det;
  lam[2] = v3dot(a, v3cross(r, c)) / det;
  lam[3] = v3dot(a, v3cross(b, r)) / det;
  lam[0] = 1.0 - lam[1] - lam[2] - lam[3];
}

__device__ __forceinline__ V3 quad_point(const V3 (&P)[4], const double* bary) {
  V3 x{0.0, 0.0, 0.0};
  for (int i = 0; i < 4; ++i) x = v3add(x, v3scale(bary[i], P[i]));
  return x;
}

struct Lda {
  double v, e;
  bool clamped;
};

// lda_vxc (model.cpp:268-300); cx = cbrt(3/pi) as computed by the host libm.
__device__ __forceinline__ Lda lda_vxc(double rho, bool exchange_only, double cx) {
  Lda out{0.0, 0.0, false};
  if (rho < 0.0) {
    out.clamped = true;
    rho = 0.0;
  }
  if (rho == 0.0) return out;
  const double r13 = cbrt(rho);
  out.v = -cx * r13;
  out.e = -0.75 * cx * r13;
  if (!exchange_only) {
    const double rs = cbrt(3.0 / (4.0 * M_PI * rho));
    double ec, vc;
    if (rs < 1.0) {
      const double a = 0.0311, b = -0.048, c = 0.0020, dd = -0.0116;
      const double ln = log(rs);
      ec = a * ln + b + c * rs * ln + dd * rs;
      vc = a * ln + (b - a / 3.0) + (2.0 / 3.0) * c * rs * ln + ((2.0 * dd - c) / 3.0) * rs;
    } else if (isinf(rs)) {
      // rho < ~1.3e-309 (denormal): 3/(4 pi rho) overflows and the reference
      // formula gives -0 * inf = NaN (model.cpp:282-294), failing the
      // assembly. Use the rho -> 0 limit of PZ81 (e_c, v_c -> 0) instead; every
      // density the reference evaluates finitely is unaffected.
      ec = 0.0;
      vc = 0.0;
    } else {
      const double gamma = -0.1423, beta1 = 1.0529, beta2 = 0.3334;
      const double sq = sqrt(rs);
      const double denom = 1.0 + beta1 * sq + beta2 * rs;
      ec = gamma / denom;
      vc = ec * (1.0 + (7.0 / 6.0) * beta1 * sq + (4.0 / 3.0) * beta2 * rs) / denom;
    }
    out.e += ec;
    out.v += vc;
  }
  return out;
}

// interior dof of lattice vertex (vx,vy,vz), -1 on the boundary (fem.cpp:21-28)
__device__ __forceinline__ long long vertex_dof(int s, int vx, int vy, int vz) {
  if (vx <= 0 || vy <= 0 || vz <= 0 || vx >= s || vy >= s || vz >= s) return -1;
  const long long S = s - 1;
  return ((static_cast<long long>(vz - 1) * S) + (vy - 1)) * S + (vx - 1);
}

}  // namespace paro_b200
