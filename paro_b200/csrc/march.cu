// Plane-marching stencil kernels: operator apply, the two fused Jacobi-PCG
// passes and the PCG setup pass. See march.cuh for the design.
//
// v2 pipeline: planes are moved global -> shared with cp.async (LDGSTS, zero
// fill outside the lattice) two planes ahead of the compute, so no registers
// hold in-flight data and the DRAM requests of the next plane overlap the
// stencil of the current one. K2 additionally stages the own-point x, r of
// the next plane. K1 stages the raw r, p_old (and diagonal) planes and
// transforms them into p_new = z + beta p_old once they land.
#include <algorithm>
#include <cstdlib>

#include "march.cuh"

namespace paro_b200 {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// 8-byte async copy; src_size 0 zero-fills the destination (Dirichlet halo)
__device__ __forceinline__ void cp8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// read-only load pinned in program order (volatile asm is not moved across
// the pipeline wait / barrier, so its latency overlaps them)
__device__ __forceinline__ double ldnc(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>
struct Cfg {
  static constexpr int NA = MODE == kApply ? 1 : MODE == kK1 ? 1 : MODE == kK2 ? 2 : 3;  // partial sums
  static constexpr int NR = MODE == kK1 ? 3 : 4;  // ring slots of stencil-source planes
};

template <int MODE, int CB>
constexpr size_t smem_bytes() {
  size_t d = static_cast<size_t>(Cfg<MODE>::NR) * CB * kHP;
  if (MODE == kK2) d += static_cast<size_t>(2) * CB * 2 * kNT;   // x, r stages
  if (MODE == kK1) d += static_cast<size_t>(2) * (2 * CB + 1) * kHP;  // raw r, p_old, invd stages
  return d * sizeof(double);
}

// 15-point row sum in ascending column order (linalg.cpp:88-94 on the Kuhn
// pattern). wb[o]: A[v, v-off(o)], wf[o]: A[v, v+off(o)], w0: diagonal.
// FMA = true (the PCG passes only) contracts each term into one DFMA; the
// operator apply keeps the reference's separate multiply and add.
template <bool FMA = false>
__device__ __forceinline__ double row_sum(const double* __restrict__ Pm, const double* __restrict__ P0,
                                          const double* __restrict__ Pp, int ib, const double (&wb)[kSlots],
                                          double w0, const double (&wf)[kSlots]) {
  auto madd = [](double s, double w, double x) { return FMA ? fma(w, x, s) : __dadd_rn(s, __dmul_rn(w, x)); };
  double s = 0.0;
  s = madd(s, wb[7], Pm[ib - kHX - 1]);
  s = madd(s, wb[6], Pm[ib - kHX]);
  s = madd(s, wb[5], Pm[ib - 1]);
  s = madd(s, wb[4], Pm[ib]);
  s = madd(s, wb[3], P0[ib - kHX - 1]);
  s = madd(s, wb[2], P0[ib - kHX]);
  s = madd(s, wb[1], P0[ib - 1]);
  s = madd(s, w0, P0[ib]);
  s = madd(s, wf[1], P0[ib + 1]);
  s = madd(s, wf[2], P0[ib + kHX]);
  s = madd(s, wf[3], P0[ib + kHX + 1]);
  s = madd(s, wf[4], Pp[ib]);
  s = madd(s, wf[5], Pp[ib + 1]);
  s = madd(s, wf[6], Pp[ib + kHX]);
  s = madd(s, wf[7], Pp[ib + kHX + 1]);
  return s;
}

// own[o] = A[v, v+o] stored at v; back[o] = A[v, v-o] stored at v-o (0 when
// v-o leaves the lattice, where the plane value is 0 anyway)
__device__ __forceinline__ void load_weights(const double* __restrict__ cf, long long n, int idx, int gx, int gy,
                                             int z, int S, int S2, double (&own)[kSlots], double (&back)[kSlots]) {
#pragma unroll
  for (int o = 0; o < kSlots; ++o) own[o] = __ldg(cf + o * n + idx);
  back[0] = 0.0;
#pragma unroll
  for (int o = 1; o < kSlots; ++o) {
    const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
    const bool ok = gx >= ox && gy >= oy && z >= oz;
    const int nb = idx - ox - oy * S - oz * S2;
    back[o] = ok ? __ldg(cf + o * n + nb) : 0.0;
  }
}

template <int MODE, bool VAR, int CB>
__global__ void __launch_bounds__(kNT, CB <= 2 && kMinCtas == 2 ? 3 : kMinCtas) march_kernel(const MarchArgs a) {
  extern __shared__ __align__(16) double smem[];
  constexpr int NA = Cfg<MODE>::NA;
  constexpr int NR = Cfg<MODE>::NR;
  __shared__ double red[kNT / 32][CB * NA];
  __shared__ double colA[CB], colB[CB];
  __shared__ int colFirst[CB];

  double* ring = smem;                                   // [NR][CB][kHP]
  double* stage = ring + NR * CB * kHP;                  // K2: [2][CB][2][kNT]
  double* raw = stage + (MODE == kK2 ? 2 * CB * 2 * kNT : 0);  // K1: [2][2CB+1][kHP]

  const int S = a.S;
  const int S2 = S * S;
  const long long n = a.n;
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * CB;

  bool act[CB];
  bool any = false;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const int c = c0 + j;
    act[j] = c < a.K && (a.cols == nullptr || a.cols[c].active != 0);
    any |= act[j];
  }
  if (!any) return;
  if (tid < CB) {
    const int c = c0 + tid;
    double va = 0.0, vb = 0.0;
    int f = 0;
    if (act[tid]) {
      if (MODE == kK1) {
        vb = a.cols[c].beta;
        f = a.cols[c].first != 0;
      }
      if (MODE == kK2) va = a.cols[c].alpha;
      if (MODE == kSetupWarm || MODE == kSetupCold) va = a.scale[c];
    }
    colA[tid] = va;
    colB[tid] = vb;
    colFirst[tid] = f;
  }

  const int bx = b % a.nTX;
  const int by = (b / a.nTX) % a.nTY;
  const int bz = b / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = a.zlo + bz * a.ZC;
  const int z1 = min(a.zhi, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;
  const int own = gy * S + gx;  // in-plane offset of this thread's point

  // the (up to) two halo'd-plane positions this thread copies
  int pos[kLoadsPerThread], roff[kLoadsPerThread];
  bool pval[kLoadsPerThread], pown[kLoadsPerThread];
#pragma unroll
  for (int l = 0; l < kLoadsPerThread; ++l) {
    const int i = tid + l * kNT;
    pos[l] = i;
    const int hx = i % kHX, hy = i / kHX;
    const int px = x0 + hx - 1, py = y0 + hy - 1;
    pval[l] = i < kHP && px >= 0 && px < S && py >= 0 && py < S;
    pown[l] = pval[l] && hx >= 1 && hx <= kTX && hy >= 1 && hy <= kTY;
    roff[l] = pval[l] ? py * S + px : 0;
  }
  __syncthreads();  // colA/colB/colFirst

  auto rs = [&](int z) { return (z - z0 + 1 + NR) % NR; };

  // stencil-source plane z -> ring slot (non-K1 modes)
  auto issue_plane = [&](int z) {
    const bool zin = z >= 0 && z < S;
    const int zoff = zin ? z * S2 : 0;
    double* slot = ring + rs(z) * CB * kHP;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const double* col = a.src + static_cast<long long>(c0 + j) * a.ld;
        const bool v = zin && pval[l] && act[j];
        cp8(slot + j * kHP + pos[l], v ? col + zoff + roff[l] : col, v);
      }
    }
  };
  // K1 raw planes r, p_old (+ diagonal) -> raw stage (z & 1)
  auto issue_raw = [&](int z) {
    const bool zin = z >= 0 && z < S;
    const int zoff = zin ? z * S2 : 0;
    double* rw = raw + (z & 1) * (2 * CB + 1) * kHP;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const long long co = static_cast<long long>(c0 + j) * a.ld;
        const bool v = zin && pval[l] && act[j];
        cp8(rw + j * kHP + pos[l], v ? a.r + co + zoff + roff[l] : a.r + co, v);
        const bool vp = v && !colFirst[j];
        cp8(rw + (CB + j) * kHP + pos[l], vp ? a.pold + co + zoff + roff[l] : a.pold + co, vp);
      }
      if (VAR) {
        const bool v = zin && pval[l];
        cp8(rw + 2 * CB * kHP + pos[l], v ? a.invd + zoff + roff[l] : a.invd, v);
      }
    }
  };
  // K2 own-point x, r of plane z -> stage (z & 1)
  auto issue_xr = [&](int z) {
    if (!inside || z >= z1) return;
    const int zoff = z * S2;
    double* st = stage + (z & 1) * CB * 2 * kNT;
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      if (!act[j]) continue;
      const long long co = static_cast<long long>(c0 + j) * a.ld;
      cp8(st + (j * 2 + 0) * kNT + tid, a.x + co + zoff + own, true);
      cp8(st + (j * 2 + 1) * kNT + tid, a.r + co + zoff + own, true);
    }
  };
  // K1: raw plane z -> p_new = z + beta p_old in ring slot; own points also to global
  auto transform = [&](int z) {
    const double* rw = raw + (z & 1) * (2 * CB + 1) * kHP;
    double* slot = ring + rs(z) * CB * kHP;
    const bool zown = z >= z0 && z < z1;
    const int zoff = z * S2;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
      const double d = VAR ? rw[2 * CB * kHP + pos[l]] : (pval[l] ? a.op.invd_const : 0.0);
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        // z = inv_diag * r ; p = z + beta * p   (linalg.cpp:179, 210)
        const double zz = __dmul_rn(d, rw[j * kHP + pos[l]]);
        const double v = colFirst[j] ? zz : __dadd_rn(zz, __dmul_rn(colB[j], rw[(CB + j) * kHP + pos[l]]));
        slot[j * kHP + pos[l]] = v;
        if (zown && pown[l] && act[j]) a.dst[static_cast<long long>(c0 + j) * a.ld + zoff + roff[l]] = v;
      }
    }
  };

  double acc[CB][NA];
#pragma unroll
  for (int j = 0; j < CB; ++j)
#pragma unroll
    for (int q = 0; q < NA; ++q) acc[j][q] = 0.0;

  // prologue
  if (MODE == kK1) {
    issue_raw(z0 - 1);
    issue_raw(z0);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    transform(z0 - 1);
    transform(z0);
    __syncthreads();
    issue_raw(z0 + 1);
    cp_commit();
  } else {
    issue_plane(z0 - 1);
    issue_plane(z0);
    issue_plane(z0 + 1);
    if (MODE == kK2) issue_xr(z0);
    cp_commit();
  }

  const int ib = (ty + 1) * kHX + (tx + 1);
  for (int z = z0; z < z1; ++z) {
    if (MODE == kK1) {
      if (z + 2 <= z1) issue_raw(z + 2);
    } else {
      if (z + 2 <= z1) issue_plane(z + 2);
      if (MODE == kK2) issue_xr(z + 1);
    }
    cp_commit();
    // this plane's operator coefficients: issued before the wait and barrier
    // below so that their L2 latency overlaps them (profiles/r01: the first
    // use of these loads was the top stall of both PCG kernels)
    const int idx = z * S2 + own;
    double ow[kSlots], bk[kSlots], invd = 0.0;
    if (VAR && inside) load_weights(a.op.coef, n, idx, gx, gy, z, S, S2, ow, bk);
    if ((MODE == kK2 || MODE == kSetupWarm || MODE == kSetupCold) && inside)
      invd = VAR ? __ldg(a.invd + (a.P ? (static_cast<long long>(z) * S + gy) * a.P + gx : idx)) : a.op.invd_const;
    cp_wait<1>();
    __syncthreads();
    if (MODE == kK1) {
      transform(z + 1);
      __syncthreads();
    }

    if (inside) {
      // 15 weights of the operator at this point, shifted by sigma*M
      double wb[kSlots], wf[kSlots], w0;
      if (VAR) {
        if (a.op.mcoef != nullptr) {  // variable shift stencil (inexact mesh spacing)
          double mown[kSlots], mback[kSlots];
          load_weights(a.op.mcoef, n, idx, gx, gy, z, S, S2, mown, mback);
#pragma unroll
          for (int o = 1; o < kSlots; ++o) {
            wb[o] = __dadd_rn(bk[o], __dmul_rn(a.op.sigma, mback[o]));
            wf[o] = __dadd_rn(ow[o], __dmul_rn(a.op.sigma, mown[o]));
          }
          w0 = __dadd_rn(ow[0], __dmul_rn(a.op.sigma, mown[0]));
        } else {
#pragma unroll
          for (int o = 1; o < kSlots; ++o) {
            wb[o] = __dadd_rn(bk[o], __dmul_rn(a.op.sigma, a.op.m[o]));
            wf[o] = __dadd_rn(ow[o], __dmul_rn(a.op.sigma, a.op.m[o]));
          }
          w0 = __dadd_rn(ow[0], __dmul_rn(a.op.sigma, a.op.m[0]));
        }
      } else {
#pragma unroll
        for (int o = 1; o < kSlots; ++o) {
          wf[o] = __dadd_rn(a.op.w[o], __dmul_rn(a.op.sigma, a.op.m[o]));
          wb[o] = wf[o];
        }
        w0 = __dadd_rn(a.op.w[0], __dmul_rn(a.op.sigma, a.op.m[0]));
      }
      wb[0] = wf[0] = 0.0;
      const double* Pm = ring + rs(z - 1) * CB * kHP;
      const double* P0 = ring + rs(z) * CB * kHP;
      const double* Pp = ring + rs(z + 1) * CB * kHP;
      const double* st = stage + (z & 1) * CB * 2 * kNT;

#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (!act[j]) continue;
        const double s = row_sum<MODE == kK1 || MODE == kK2>(Pm + j * kHP, P0 + j * kHP, Pp + j * kHP, ib, wb, w0, wf);
        const double ctr = P0[j * kHP + ib];
        const long long gi = static_cast<long long>(c0 + j) * a.ld + idx;
        if (MODE == kApply) {
          a.dst[gi] = s;
          acc[j][0] += ctr * s;
        } else if (MODE == kK1) {
          acc[j][0] += ctr * s;  // p'q
        } else if (MODE == kK2) {
          // x += alpha p ; r -= alpha q ; z = invd r  (linalg.cpp:202-206)
          const double al = colA[j];
          const double xn = __dadd_rn(st[(j * 2 + 0) * kNT + tid], __dmul_rn(al, ctr));
          const double rn = __dsub_rn(st[(j * 2 + 1) * kNT + tid], __dmul_rn(al, s));
          a.x[gi] = xn;
          a.r[gi] = rn;
          const double zz = __dmul_rn(invd, rn);
          acc[j][0] += rn * zz;
          acc[j][1] += rn * rn;
        } else {
          // rhs b = (M f) * scale (paro.cpp:96-98; model.cpp:248-249)
          double bb;
          if (a.rhs != nullptr) {
            bb = a.rhs[gi];  // cg_solve(a, b, x0) with an explicit b
          } else if (a.mwcoef != nullptr) {
            double mown[kSlots], mback[kSlots];
            load_weights(a.mwcoef, n, idx, gx, gy, z, S, S2, mown, mback);
            const double msum = row_sum(Pm + j * kHP, P0 + j * kHP, Pp + j * kHP, ib, mback, mown[0], mown);
            bb = __dmul_rn(msum, colA[j]);
          } else {
            double wm[kSlots];
#pragma unroll
            for (int o = 0; o < kSlots; ++o) wm[o] = a.mw[o];
            const double msum = row_sum(Pm + j * kHP, P0 + j * kHP, Pp + j * kHP, ib, wm, wm[0], wm);
            bb = __dmul_rn(msum, colA[j]);
          }
          double rr;
          // x, r may live in the solver's padded buffers (stride ldw)
          const long long gw =
              a.ldw ? static_cast<long long>(c0 + j) * a.ldw + (a.P ? (static_cast<long long>(z) * S + gy) * a.P + gx : idx)
                    : gi;
          if (MODE == kSetupWarm) {
            rr = __dsub_rn(bb, s);  // r = b - A x0 (linalg.cpp:184-185)
            a.x[gw] = ctr;          // x = x0
          } else {
            rr = bb;                // x0 = 0: A x0 = 0, r = b
            a.x[gw] = 0.0;
          }
          a.dst[gw] = rr;
          const double zz = __dmul_rn(invd, rr);
          acc[j][0] += bb * bb;
          acc[j][1] += rr * zz;
          acc[j][2] += rr * rr;
        }
      }
    }
    __syncthreads();  // slots read this step are overwritten by the next issue
  }
  cp_wait<0>();

  if (MODE == kApply && !a.with_dot) return;
  // deterministic block reduction: warp tree, then warps in order
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int j = 0; j < CB; ++j)
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const double v = warp_sum(acc[j][q]);
      if (lane == 0) red[warp][j * NA + q] = v;
    }
  __syncthreads();
  if (tid < CB * NA) {
    const int j = tid / NA, q = tid % NA;
    if (act[j]) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kNT / 32; ++w) s += red[w][tid];
      a.partials[(static_cast<long long>(c0 + j) * 3 + q) * a.nblk + b] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// v3 (Apply, K1, K2): streaming row sums. The 15 stencil points of row z lie
// on planes z-1 (4 points), z (7) and z+1 (4), and the union of the in-plane
// offsets a thread touches on one plane over its three uses is the 7 points
// of the centre pattern. So when plane t lands, each thread reads those 7
// values once per column and adds them to three running sums: the Pm terms
// of row t+1, the centre terms of row t and the Pp terms of row t-1, which
// is then complete. Planes arrive in ascending z, so every row is still
// summed term by term in ascending column order (the same operation sequence
// as row_sum), with 7 shared-memory reads per point-column instead of 15 and
// one barrier per plane.
template <int MODE, int CB>
constexpr size_t stream_smem() {
  size_t d = static_cast<size_t>(MODE == kK1 ? 2 : 3) * CB * kHP;           // stencil-source ring
  if (MODE == kK2) d += static_cast<size_t>(3) * CB * 2 * kNT;              // own x, r stages
  if (MODE == kK1) d += static_cast<size_t>(3) * (2 * CB + 1) * kHP;        // raw r, p_old, invd stages
  return d * sizeof(double);
}

template <int MODE, bool VAR, int CB>
__global__ void __launch_bounds__(kNT, CB <= 2 && kMinCtas == 2 ? 3 : kMinCtas) stream_kernel(const MarchArgs a) {
  extern __shared__ __align__(16) double smem[];
  constexpr int NR = MODE == kK1 ? 2 : 3;
  constexpr bool SETUP = MODE == kSetupWarm || MODE == kSetupCold;
  constexpr int NA = MODE == kK2 ? 2 : SETUP ? 3 : 1;
  constexpr bool FMA = MODE == kK1 || MODE == kK2;
  __shared__ double red[kNT / 32][CB * NA];

  double* ring = smem;                    // [NR][CB][kHP]
  double* stage = ring + NR * CB * kHP;   // K2: [3][CB][2][kNT]; K1: raw [3][2CB+1][kHP]

  const int S = a.S;
  const int S2 = S * S;
  const long long n = a.n;
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * CB;

  unsigned actm = 0, firstm = 0;  // per-column bits: active, first PCG iteration
  double colA[CB], colB[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const int c = c0 + j;
    const bool on = c < a.K && (a.cols == nullptr || a.cols[c].active != 0);
    colA[j] = colB[j] = 0.0;
    if (on) {
      actm |= 1u << j;
      if (MODE == kK1) {
        colB[j] = a.cols[c].beta;
        if (a.cols[c].first != 0) firstm |= 1u << j;
      }
      if (MODE == kK2) colA[j] = a.cols[c].alpha;
      if (SETUP) colA[j] = a.scale[c];  // rhs scale lambda + sigma (paro.cpp:96-98)
    }
  }
  if (actm == 0) return;
  auto act = [&](int j) { return (actm >> j) & 1u; };
  auto first = [&](int j) { return (firstm >> j) & 1u; };

  const int bx = b % a.nTX;
  const int by = (b / a.nTX) % a.nTY;
  const int bz = b / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = a.zlo + bz * a.ZC;
  const int z1 = min(a.zhi, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;
  const int own = gy * S + gx;

  int pos[kLoadsPerThread], roff[kLoadsPerThread];
  bool pval[kLoadsPerThread], pown[kLoadsPerThread];
#pragma unroll
  for (int l = 0; l < kLoadsPerThread; ++l) {
    const int i = tid + l * kNT;
    pos[l] = i;
    const int hx = i % kHX, hy = i / kHX;
    const int px = x0 + hx - 1, py = y0 + hy - 1;
    pval[l] = i < kHP && px >= 0 && px < S && py >= 0 && py < S;
    pown[l] = pval[l] && hx >= 1 && hx <= kTX && hy >= 1 && hy <= kTY;
    roff[l] = pval[l] ? py * S + px : 0;
  }

  // column-group base pointers (uniform); per-thread offsets stay 32-bit
  const long long ld = a.ld;
  const long long cbase = static_cast<long long>(c0) * ld;
  // in-plane offset of halo position l on plane z (0 where zero-filled)
  auto hoff = [&](int l, bool zin, int zoff) { return zin && pval[l] ? zoff + roff[l] : 0; };

  // stencil-source plane z -> ring slot `slot` (Apply, K2)
  auto issue_plane = [&](int z, int slot) {
    const bool zin = z >= 0 && z < S;
    const int zoff = z * S2;
    double* dst = ring + slot * CB * kHP;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
      const bool v = zin && pval[l];
      const double* q = a.src + cbase + hoff(l, zin, zoff);
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (act(j)) cp8(dst + j * kHP + pos[l], q, v);
        q += ld;
      }
    }
  };
  // K1: raw planes r, p_old (+ inverse diagonal) -> raw stage `slot`
  auto issue_raw = [&](int z, int slot) {
    const bool zin = z >= 0 && z < S;
    const int zoff = z * S2;
    double* rw = stage + slot * (2 * CB + 1) * kHP;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
      const bool v = zin && pval[l];
      const int off = hoff(l, zin, zoff);
      const double* qr = a.r + cbase + off;
      const double* qp = a.pold + cbase + off;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (act(j)) {
          cp8(rw + j * kHP + pos[l], qr, v);
          if (!first(j)) cp8(rw + (CB + j) * kHP + pos[l], qp, v);
        }
        qr += ld;
        qp += ld;
      }
      if (VAR) cp8(rw + 2 * CB * kHP + pos[l], a.invd + off, v);
    }
  };
  // K1: raw stage `rslot_` of plane z -> p_new = z + beta p_old in ring slot
  // (z - z0 + 1) & 1; own points also to global
  auto transform = [&](int z, int rslot_) {
    const double* rw = stage + rslot_ * (2 * CB + 1) * kHP;
    double* slot = ring + ((z - z0 + 1) & 1) * CB * kHP;
    const bool zown = z >= z0 && z < z1;
    const int zoff = z * S2;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
      const double d = VAR ? rw[2 * CB * kHP + pos[l]] : (pval[l] ? a.op.invd_const : 0.0);
      const bool wr = zown && pown[l];
      double* q = a.dst + cbase + (zoff + roff[l]);
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (act(j)) {
          // z = inv_diag * r ; p = z + beta * p   (linalg.cpp:179, 210)
          const double zz = __dmul_rn(d, rw[j * kHP + pos[l]]);
          const double v = first(j) ? zz : __dadd_rn(zz, __dmul_rn(colB[j], rw[(CB + j) * kHP + pos[l]]));
          slot[j * kHP + pos[l]] = v;
          if (wr) *q = v;
        }
        q += ld;
      }
    }
  };
  // K2: own-point x, r of row z -> stage `slot`
  auto issue_xr = [&](int z, int slot) {
    if (!inside || z < z0 || z >= z1) return;
    double* st = stage + slot * CB * 2 * kNT;
    const long long off = cbase + z * S2 + own;
    const double* qx = a.x + off;
    const double* qr = a.r + off;
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      if (act(j)) {
        cp8(st + (j * 2 + 0) * kNT + tid, qx, true);
        cp8(st + (j * 2 + 1) * kNT + tid, qr, true);
      }
      qx += ld;
      qr += ld;
    }
  };
  auto madd = [](double s, double w, double x) { return FMA ? fma(w, x, s) : __dadd_rn(s, __dmul_rn(w, x)); };
  // Coefficient offsets relative to a point of plane t: back slot o of row
  // t (o = 1..3) and of row t+1 (o = 4..7) lie in plane t at -(ox + oy S);
  // own slots 0..3 of row t in plane t, own 4..7 of row t-1 in plane t-1.
  // Loads are unconditional (planes clamped into the lattice): a back weight
  // whose neighbour leaves the lattice multiplies a zero-filled plane value,
  // and a row sum that starts at +0 is unchanged by adding +-0 in
  // round-to-nearest, so the row sums equal the CSR ones bit for bit.
  long long offB[kSlots], offF[kSlots];
#pragma unroll
  for (int o = 0; o < kSlots; ++o) {
    offF[o] = o * n;
    offB[o] = o * n - (o & 1) - ((o >> 1) & 1) * S;
  }

  double sC[CB], sN[CB], cCur[CB];  // row t partial, row t+1 partial, centre value of plane t
  double mC[CB], mN[CB];            // setup: the same for the right-hand-side mass stencil
  double acc[CB][NA];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    sC[j] = sN[j] = cCur[j] = 0.0;
    mC[j] = mN[j] = 0.0;
#pragma unroll
    for (int q = 0; q < NA; ++q) acc[j][q] = 0.0;
  }

  // prologue
  if (MODE == kK1) {
    issue_raw(z0 - 1, 0);
    cp_commit();
    issue_raw(z0, 1);
    cp_commit();
    issue_raw(z0 + 1, 2);
    cp_commit();
    cp_wait<2>();
    __syncthreads();
    transform(z0 - 1, 0);
  } else {
    issue_plane(z0 - 1, 0);
    cp_commit();
    issue_plane(z0, 1);
    cp_commit();
  }

  const int ib = (ty + 1) * kHX + (tx + 1);
  const int ownc = inside ? own : 0;
  int s0 = 0;  // rslot(t); rslot(t+1) = s1, rslot(t-1) = rslot(t+2) = s2
  // coefficients of step t (planes t and t-1), loaded one step ahead so their
  // L2/DRAM latency overlaps the previous step's compute
  double cN[4], cC[7], cPp[4], invdP = 0.0;
  auto load_coefs = [&](int t) {
    if (VAR) {
      const long long pt = static_cast<long long>(min(max(t, 0), S - 1)) * S2 + ownc;
      const long long pm = static_cast<long long>(min(max(t - 1, 0), S - 1)) * S2 + ownc;
      const double* cf = a.op.coef;
#pragma unroll
      for (int i = 0; i < 4; ++i) cN[i] = ldnc(cf + pt + offB[4 + i]);
#pragma unroll
      for (int i = 0; i < 3; ++i) cC[i] = ldnc(cf + pt + offB[1 + i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) cC[3 + i] = ldnc(cf + pt + offF[i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) cPp[i] = ldnc(cf + pm + offF[4 + i]);
      // the solver's inverse diagonal may be in the row-padded layout (a.P)
      if (MODE == kK2 || SETUP)
        invdP = ldnc(a.invd + (a.P ? (static_cast<long long>(min(max(t - 1, 0), S - 1)) * S + (inside ? gy : 0)) * a.P +
                                         (inside ? gx : 0)
                                   : pm));
    }
    if (!VAR && (MODE == kK2 || SETUP)) invdP = a.op.invd_const;
  };
  load_coefs(z0 - 1);
  for (int t = z0 - 1; t <= z1; ++t, s0 = s0 == 2 ? 0 : s0 + 1) {
    const int s1 = s0 == 2 ? 0 : s0 + 1;
    const int s2 = s1 == 2 ? 0 : s1 + 1;
    const bool rowP = t - 1 >= z0;  // row t-1 completes at this step

    cp_wait<1>();
    __syncthreads();
    if (MODE == kK1) {
      if (t + 3 <= z1) issue_raw(t + 3, s0);  // rslot(t+3) = rslot(t)
    } else {
      if (t + 2 <= z1) issue_plane(t + 2, s2);
      if (MODE == kK2) issue_xr(t + 1, s1);
    }
    cp_commit();

    if (inside) {
      // shifted weights of the three rows touched by plane t
      double wN[4], wC[7], wP[4];
      if (VAR) {  // coefficients of (A + sigma M), the shift folded in by preshift()
#pragma unroll
        for (int i = 0; i < 4; ++i) wN[i] = cN[i];
#pragma unroll
        for (int i = 0; i < 7; ++i) wC[i] = cC[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) wP[i] = cPp[i];
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) wN[i] = a.op.wc[4 + i];
#pragma unroll
        for (int i = 0; i < 3; ++i) wC[i] = a.op.wc[1 + i];
#pragma unroll
        for (int i = 0; i < 4; ++i) wC[3 + i] = a.op.wc[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) wP[i] = a.op.wc[4 + i];
      }
      const double* P = ring + (MODE == kK1 ? ((t - z0 + 1) & 1) : s0) * CB * kHP;
      const double* st = stage + (MODE == kK2 ? s2 : 0) * CB * 2 * kNT;
      const int u = t - 1;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (!act(j)) continue;
        const double* Pj = P + j * kHP;
        const double vmm = Pj[ib - kHX - 1], v0m = Pj[ib - kHX], vm0 = Pj[ib - 1], v00 = Pj[ib];
        const double vp0 = Pj[ib + 1], v0p = Pj[ib + kHX], vpp = Pj[ib + kHX + 1];
        if (rowP) {  // Pp terms of row t-1: A[v, v+o], o = 4..7
          double s = sC[j];
          s = madd(s, wP[0], v00);
          s = madd(s, wP[1], vp0);
          s = madd(s, wP[2], v0p);
          s = madd(s, wP[3], vpp);
          const double ctr = cCur[j];  // p (or x) at row t-1
          const long long gi = static_cast<long long>(c0 + j) * a.ld + (u * S2 + own);
          if (MODE == kApply) {
            a.dst[gi] = s;
            acc[j][0] += ctr * s;
          } else if (MODE == kK1) {
            acc[j][0] += ctr * s;  // p'q
          } else if (SETUP) {
            // b = (M f) * scale (paro.cpp:96-98; model.cpp:248-249) or an explicit b
            double m = mC[j];
            m = madd(m, a.mw[4], v00);
            m = madd(m, a.mw[5], vp0);
            m = madd(m, a.mw[6], v0p);
            m = madd(m, a.mw[7], vpp);
            const long long gw =
                a.ldw ? static_cast<long long>(c0 + j) * a.ldw +
                            (a.P ? (static_cast<long long>(u) * S + gy) * a.P + gx : static_cast<long long>(u) * S2 + own)
                      : gi;
            const double bb = a.rhs != nullptr ? a.rhs[gi] : __dmul_rn(m, colA[j]);
            double rr;
            if (MODE == kSetupWarm) {
              rr = __dsub_rn(bb, s);  // r = b - A x0 (linalg.cpp:184-185)
              a.x[gw] = ctr;          // x = x0
            } else {
              rr = bb;                // x0 = 0: A x0 = 0, r = b
              a.x[gw] = 0.0;
            }
            a.dst[gw] = rr;
            const double zz = __dmul_rn(invdP, rr);
            acc[j][0] += bb * bb;
            acc[j][1] += rr * zz;
            acc[j][2] += rr * rr;
          } else {
            // x += alpha p ; r -= alpha q ; z = invd r  (linalg.cpp:202-206)
            const double al = colA[j];
            const double xn = __dadd_rn(st[(j * 2 + 0) * kNT + tid], __dmul_rn(al, ctr));
            const double rn = __dsub_rn(st[(j * 2 + 1) * kNT + tid], __dmul_rn(al, s));
            a.x[gi] = xn;
            a.r[gi] = rn;
            const double zz = __dmul_rn(invdP, rn);
            acc[j][0] += rn * zz;
            acc[j][1] += rn * rn;
          }
        }
        // centre terms of row t (back 3..1, diagonal, forward 1..3) and Pm
        // terms of row t+1 (back 7..4); computed unconditionally, a row
        // outside [z0, z1) is never completed
        double c = sN[j];
        {
          c = madd(c, wC[2], vmm);
          c = madd(c, wC[1], v0m);
          c = madd(c, wC[0], vm0);
          c = madd(c, wC[3], v00);
          c = madd(c, wC[4], vp0);
          c = madd(c, wC[5], v0p);
          c = madd(c, wC[6], vpp);
        }
        double nx = 0.0;
        {
          nx = madd(nx, wN[3], vmm);
          nx = madd(nx, wN[2], v0m);
          nx = madd(nx, wN[1], vm0);
          nx = madd(nx, wN[0], v00);
        }
        sC[j] = c;
        sN[j] = nx;
        cCur[j] = v00;
        if (SETUP) {  // mass row sums: centre terms of row t, Pm terms of row t+1
          double m = mN[j];
          m = madd(m, a.mw[3], vmm);
          m = madd(m, a.mw[2], v0m);
          m = madd(m, a.mw[1], vm0);
          m = madd(m, a.mw[0], v00);
          m = madd(m, a.mw[1], vp0);
          m = madd(m, a.mw[2], v0p);
          m = madd(m, a.mw[3], vpp);
          double mx = 0.0;
          mx = madd(mx, a.mw[7], vmm);
          mx = madd(mx, a.mw[6], v0m);
          mx = madd(mx, a.mw[5], vm0);
          mx = madd(mx, a.mw[4], v00);
          mC[j] = m;
          mN[j] = mx;
        }
      }
    }
    if (MODE == kK1 && t + 1 <= z1) transform(t + 1, s1);
    if (t < z1) load_coefs(t + 1);
  }
  cp_wait<0>();

  if (MODE == kApply && !a.with_dot) return;
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int j = 0; j < CB; ++j)
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const double v = warp_sum(acc[j][q]);
      if (lane == 0) red[warp][j * NA + q] = v;
    }
  __syncthreads();
  if (tid < CB * NA) {
    const int j = tid / NA, q = tid % NA;
    if (act(j)) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kNT / 32; ++w) s += red[w][tid];
      a.partials[(static_cast<long long>(c0 + j) * 3 + q) * a.nblk + b] = s;
    }
  }
}

template <int MODE, bool VAR, int CB>
void launch_s(const MarchArgs& a, cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = stream_smem<MODE, CB>();
  static bool configured = false;
  if (!configured) {
    PARO_CUDA(cudaFuncSetAttribute(stream_kernel<MODE, VAR, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
    configured = true;
  }
  dim3 grid(groups, a.nblk);
  stream_kernel<MODE, VAR, CB><<<grid, kNT, sm, st>>>(a);
  PARO_CUDA(cudaGetLastError());
}

template <int MODE, bool VAR, int CB>
void launch_t(const MarchArgs& a, cudaStream_t st) {
  {
    // the streaming kernel takes constant shift / rhs-mass stencils; variable
    // ones (inexact mesh spacing) stay on the v2 kernel
    if (a.op.mcoef == nullptr && a.mwcoef == nullptr) {
      if (VAR && a.op.sigma != 0.0) throw ParoError(kInvalidArgument, "march: shifted variable operator not preshifted");
      return launch_s<MODE, VAR, CB>(a, st);
    }
  }
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = smem_bytes<MODE, CB>();
  static bool configured = false;
  if (!configured) {
    PARO_CUDA(cudaFuncSetAttribute(march_kernel<MODE, VAR, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
    configured = true;
  }
  dim3 grid(groups, a.nblk);
  march_kernel<MODE, VAR, CB><<<grid, kNT, sm, st>>>(a);
  PARO_CUDA(cudaGetLastError());
}

template <int MODE, bool VAR>
void launch_cb(int cb, const MarchArgs& a, cudaStream_t st) {
  switch (cb) {
    case 1: launch_t<MODE, VAR, 1>(a, st); break;
    case 2: launch_t<MODE, VAR, 2>(a, st); break;
    default: launch_t<MODE, VAR, 4>(a, st); break;
  }
}

template <int MODE>
void launch_var(bool var, int cb, const MarchArgs& a, cudaStream_t st) {
  if (var) launch_cb<MODE, true>(cb, a, st);
  else launch_cb<MODE, false>(cb, a, st);
}

}  // namespace

void launch_march(int mode, bool var, int cb, const MarchArgs& a, cudaStream_t st) {
  if (a.n > (1ll << 31) - 1) throw ParoError(kCapacity, "march: more than 2^31 interior dofs per column");
  switch (mode) {
    case kApply: launch_var<kApply>(var, cb, a, st); break;
    case kK1: launch_var<kK1>(var, cb, a, st); break;
    case kK2: launch_var<kK2>(var, cb, a, st); break;
    case kSetupWarm: launch_var<kSetupWarm>(var, cb, a, st); break;
    default: launch_var<kSetupCold>(var, cb, a, st); break;
  }
}

// Spatial decomposition: 32x8 (x,y) tiles and a z-chunk sized so that one
// column group still yields a few CTAs per SM on 148 SMs.
void plan_march(MarchArgs& a, int S, int zlo, int zhi) {
  a.S = S;
  a.zlo = zlo;
  a.zhi = zhi < 0 ? S : zhi;
  const int nz = a.zhi - a.zlo;
  a.n = static_cast<long long>(S) * S * S;
  a.nTX = (S + kTX - 1) / kTX;
  a.nTY = (S + kTY - 1) / kTY;
  const long long target = 148 * 4;
  long long zc = (static_cast<long long>(nz) * a.nTX * a.nTY + target - 1) / target;
  constexpr long long zc_max = 32;  // planes per CTA z-chunk (48 / 64 measured no faster)
  zc = std::max<long long>(4, std::min<long long>(zc_max, zc));
  a.ZC = static_cast<int>(std::max<long long>(1, std::min<long long>(zc, nz)));
  a.nZ = (nz + a.ZC - 1) / a.ZC;
  a.nblk = a.nTX * a.nTY * a.nZ;
}

}  // namespace paro_b200
