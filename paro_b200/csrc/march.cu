// Plane-marching stencil kernels: operator apply, the two fused Jacobi-PCG
// passes and the PCG setup pass. See march.cuh for the design.
#include <algorithm>

#include "march.cuh"

namespace paro_b200 {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// fl(a + fl(b*c)) with no contraction: the reference's `s += v * x`.
__device__ __forceinline__ double madd(double s, double w, double x) { return __dadd_rn(s, __dmul_rn(w, x)); }

template <int MODE>
struct Acc {
  static constexpr int N = MODE == kApply ? 1 : MODE == kK1 ? 1 : MODE == kK2 ? 2 : 3;
};

// 15-point row sum in ascending column order (linalg.cpp:88-94 on the Kuhn
// pattern). wb[o]: A[v, v-off(o)], wf[o]: A[v, v+off(o)], w0: diagonal.
__device__ __forceinline__ double row_sum(const double* __restrict__ Pm, const double* __restrict__ P0,
                                          const double* __restrict__ Pp, int ib, const double (&wb)[kSlots],
                                          double w0, const double (&wf)[kSlots]) {
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
__device__ __forceinline__ void load_weights(const double* __restrict__ cf, long long n, long long idx, int gx, int gy,
                                             int z, int S, long long S2, double (&own)[kSlots],
                                             double (&back)[kSlots]) {
#pragma unroll
  for (int o = 0; o < kSlots; ++o) own[o] = __ldg(cf + o * n + idx);
  back[0] = 0.0;
#pragma unroll
  for (int o = 1; o < kSlots; ++o) {
    const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
    const bool ok = gx >= ox && gy >= oy && z >= oz;
    const long long nb = idx - ox - static_cast<long long>(oy) * S - static_cast<long long>(oz) * S2;
    back[o] = ok ? __ldg(cf + o * n + nb) : 0.0;
  }
}

template <int MODE, bool VAR, int CB>
__global__ void __launch_bounds__(kNT, 2) march_kernel(const MarchArgs a) {
  extern __shared__ double smem[];  // [3][CB][kHP]
  constexpr int NA = Acc<MODE>::N;
  __shared__ double red[kNT / 32][CB * NA];

  const int S = a.S;
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

  const int bx = b % a.nTX;
  const int by = (b / a.nTX) % a.nTY;
  const int bz = b / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = bz * a.ZC;
  const int z1 = min(S, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;
  const long long S2 = static_cast<long long>(S) * S;

  // the (up to) two halo'd-plane positions this thread loads
  int pos[kLoadsPerThread];
  long long roff[kLoadsPerThread];
  bool pval[kLoadsPerThread];
  bool pown[kLoadsPerThread];
#pragma unroll
  for (int l = 0; l < kLoadsPerThread; ++l) {
    const int i = tid + l * kNT;
    pos[l] = i;
    const int hx = i % kHX, hy = i / kHX;
    const int px = x0 + hx - 1, py = y0 + hy - 1;
    pval[l] = i < kHP && px >= 0 && px < S && py >= 0 && py < S;
    pown[l] = pval[l] && hx >= 1 && hx <= kTX && hy >= 1 && hy <= kTY;
    roff[l] = pval[l] ? static_cast<long long>(py) * S + px : 0;
  }

  // per-column scalars
  double colA[CB], colB[CB];
  bool colFirst[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    colA[j] = 0.0;
    colB[j] = 0.0;
    colFirst[j] = false;
    if (act[j]) {
      const int c = c0 + j;
      if (MODE == kK1) {
        colB[j] = a.cols[c].beta;
        colFirst[j] = a.cols[c].first != 0;
      }
      if (MODE == kK2) colA[j] = a.cols[c].alpha;
      if (MODE == kSetupWarm || MODE == kSetupCold) colA[j] = a.scale[c];
    }
  }

  double acc[CB][NA];
#pragma unroll
  for (int j = 0; j < CB; ++j)
#pragma unroll
    for (int q = 0; q < NA; ++q) acc[j][q] = 0.0;

  // prefetch registers
  double pv0[CB][kLoadsPerThread];
  double pv1[CB][kLoadsPerThread];  // K1: p_old
  double pd[kLoadsPerThread];       // K1: invd

  auto fetch = [&](int z) {
    const bool zin = z >= 0 && z < S;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      const bool ok = zin && pval[l];
      const long long idx = static_cast<long long>(z) * S2 + roff[l];
      if (MODE == kK1) pd[l] = ok ? (VAR ? __ldg(a.invd + idx) : a.op.invd_const) : 0.0;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const long long gi = static_cast<long long>(c0 + j) * a.ld + idx;
        if (MODE == kK1) {
          pv0[j][l] = (ok && act[j]) ? a.r[gi] : 0.0;
          pv1[j][l] = (ok && act[j] && !colFirst[j]) ? a.pold[gi] : 0.0;
        } else {
          pv0[j][l] = (ok && act[j]) ? __ldg(a.src + gi) : 0.0;
        }
      }
    }
  };

  auto store = [&](int z, int slot) {
    const bool zown = z >= z0 && z < z1;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        double v = pv0[j][l];
        if (MODE == kK1) {
          // z = inv_diag * r ; p = z + beta * p   (linalg.cpp:179, 210)
          const double zz = __dmul_rn(pd[l], pv0[j][l]);
          v = colFirst[j] ? zz : __dadd_rn(zz, __dmul_rn(colB[j], pv1[j][l]));
          if (zown && pown[l] && act[j]) {
            const long long idx = static_cast<long long>(z) * S2 + roff[l];
            a.dst[static_cast<long long>(c0 + j) * a.ld + idx] = v;
          }
        }
        smem[(slot * CB + j) * kHP + pos[l]] = v;
      }
    }
  };

  // ring: slots hold planes z-1, z, z+1
  int sm = 0, s0 = 1, sp = 2;
  fetch(z0 - 1);
  store(z0 - 1, sm);
  fetch(z0);
  store(z0, s0);
  fetch(z0 + 1);

  const int ib = (ty + 1) * kHX + (tx + 1);
  for (int z = z0; z < z1; ++z) {
    __syncthreads();  // all reads of slot sp (plane z-2) are finished
    store(z + 1, sp);
    __syncthreads();
    if (z + 2 <= z1) fetch(z + 2);

    if (inside) {
      const long long idx = static_cast<long long>(z) * S2 + static_cast<long long>(gy) * S + gx;
      // 15 weights of the operator at this point, shifted by sigma*M
      double wb[kSlots], wf[kSlots], w0;
      if (VAR) {
        double own[kSlots], back[kSlots];
        load_weights(a.op.coef, n, idx, gx, gy, z, S, S2, own, back);
        if (a.op.mcoef != nullptr) {  // variable shift stencil (inexact mesh spacing)
          double mown[kSlots], mback[kSlots];
          load_weights(a.op.mcoef, n, idx, gx, gy, z, S, S2, mown, mback);
#pragma unroll
          for (int o = 1; o < kSlots; ++o) {
            wb[o] = __dadd_rn(back[o], __dmul_rn(a.op.sigma, mback[o]));
            wf[o] = __dadd_rn(own[o], __dmul_rn(a.op.sigma, mown[o]));
          }
          w0 = __dadd_rn(own[0], __dmul_rn(a.op.sigma, mown[0]));
        } else {
#pragma unroll
          for (int o = 1; o < kSlots; ++o) {
            wb[o] = __dadd_rn(back[o], __dmul_rn(a.op.sigma, a.op.m[o]));
            wf[o] = __dadd_rn(own[o], __dmul_rn(a.op.sigma, a.op.m[o]));
          }
          w0 = __dadd_rn(own[0], __dmul_rn(a.op.sigma, a.op.m[0]));
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
      double invd = 0.0;
      if (MODE == kK2 || MODE == kSetupWarm || MODE == kSetupCold) invd = VAR ? __ldg(a.invd + idx) : a.op.invd_const;

#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (!act[j]) continue;
        const double* Pm = smem + (sm * CB + j) * kHP;
        const double* P0 = smem + (s0 * CB + j) * kHP;
        const double* Pp = smem + (sp * CB + j) * kHP;
        const double s = row_sum(Pm, P0, Pp, ib, wb, w0, wf);
        const double ctr = P0[ib];
        const long long gi = static_cast<long long>(c0 + j) * a.ld + idx;
        if (MODE == kApply) {
          a.dst[gi] = s;
          acc[j][0] += ctr * s;
        } else if (MODE == kK1) {
          acc[j][0] += ctr * s;  // p'q
        } else if (MODE == kK2) {
          // x += alpha p ; r -= alpha q ; z = invd r  (linalg.cpp:202-206)
          const double xn = __dadd_rn(a.x[gi], __dmul_rn(colA[j], ctr));
          const double rn = __dsub_rn(a.r[gi], __dmul_rn(colA[j], s));
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
            const double msum = row_sum(Pm, P0, Pp, ib, mback, mown[0], mown);
            bb = __dmul_rn(msum, colA[j]);
          } else {
            double wm[kSlots];
#pragma unroll
            for (int o = 0; o < kSlots; ++o) wm[o] = a.mw[o];
            const double msum = row_sum(Pm, P0, Pp, ib, wm, wm[0], wm);
            bb = __dmul_rn(msum, colA[j]);
          }
          double rr;
          if (MODE == kSetupWarm) {
            rr = __dsub_rn(bb, s);  // r = b - A x0 (linalg.cpp:184-185)
            a.x[gi] = ctr;          // x = x0
          } else {
            rr = bb;                // x0 = 0: A x0 = 0, r = b
            a.x[gi] = 0.0;
          }
          a.dst[gi] = rr;
          const double zz = __dmul_rn(invd, rr);
          acc[j][0] += bb * bb;
          acc[j][1] += rr * zz;
          acc[j][2] += rr * rr;
        }
      }
    }
    const int t = sm;
    sm = s0;
    s0 = sp;
    sp = t;
  }

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

template <int MODE, bool VAR, int CB>
void launch_t(const MarchArgs& a, cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  const size_t sm = static_cast<size_t>(3) * CB * kHP * sizeof(double);
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
    case 4: launch_t<MODE, VAR, 4>(a, st); break;
    default: launch_t<MODE, VAR, 8>(a, st); break;
  }
}

template <int MODE>
void launch_var(bool var, int cb, const MarchArgs& a, cudaStream_t st) {
  if (var) launch_cb<MODE, true>(cb, a, st);
  else launch_cb<MODE, false>(cb, a, st);
}

}  // namespace

void launch_march(int mode, bool var, int cb, const MarchArgs& a, cudaStream_t st) {
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
void plan_march(MarchArgs& a, int S) {
  a.S = S;
  a.n = static_cast<long long>(S) * S * S;
  a.nTX = (S + kTX - 1) / kTX;
  a.nTY = (S + kTY - 1) / kTY;
  const long long target = 148 * 4;
  long long zc = (static_cast<long long>(S) * a.nTX * a.nTY + target - 1) / target;
  zc = std::max<long long>(4, std::min<long long>(32, zc));
  a.ZC = static_cast<int>(std::min<long long>(zc, S));
  a.nZ = (S + a.ZC - 1) / a.ZC;
  a.nblk = a.nTX * a.nTY * a.nZ;
}

}  // namespace paro_b200
