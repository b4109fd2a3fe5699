// TMA-tensor variant of the two fused Jacobi-PCG stencil passes (K1, K2) on
// the row-padded solver layout (march.cuh: padded_row).
//
// Same streaming row sums as stream_kernel (march.cu), but every operand
// plane is moved by the TMA engine from a 4-D tensor map (x, y, z, column):
// one elected thread issues one cp.async.bulk.tensor per (array, column) and
// plane, completion is counted on an mbarrier per ring slot, and the engine's
// out-of-bounds zero fill supplies the Dirichlet halo (fem.cpp:21-28), so no
// thread spends issue slots on per-row copies, edge fix-ups or zero planes
// (per-thread bulk copies, the previous generation, compiled to a uniform-register
// waterfall on 4 of the 8 warps, which then gated every barrier).
//
// K2 also writes x and r back with TMA tensor stores: the own-point rows of
// x and r land in a 4-slot ring, are updated in place, fenced to the async
// proxy and stored by the elected thread one step later.
//
// Arithmetic is identical to the march kernels (same FMA row sums, same update
// formulas, linalg.cpp:179, 202-210), so results do not depend on the variant.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "march.cuh"

namespace paro_b200 {

namespace {

__device__ __forceinline__ unsigned su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// global -> shared tile of a 4-D tensor map; completes tx bytes on bar
__device__ __forceinline__ void tma_load(double* dst, const CUtensorMap* map, int x, int y, int z, int c,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(c), "r"(su32(bar))
      : "memory");
}
// shared -> global tile (out-of-bounds elements are not written)
__device__ __forceinline__ void tma_store(const CUtensorMap* map, int x, int y, int z, int c, const double* src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(x), "r"(y), "r"(z), "r"(c), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory");
}

// predicated store without a branch around it
__device__ __forceinline__ void st_if(double* p, double v, bool pred) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.f64 [%0], %1;\n}\n" ::"l"(p), "d"(v),
               "r"(static_cast<int>(pred)));
}

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

// The inner (x) start of a tensor box must be 16-byte aligned (an odd
// double offset faults with an illegal instruction), so the halo'd box is
// 36 x 10 from (x0 - 2, y0 - 1): element x = x0 - 1 + hx of halo row hy sits
// at hy * kRW + hx + 1.
constexpr int kRW = 36;                          // halo'd box row width
constexpr int kHR = kRW * kHY;                   // 360 doubles per halo'd box
constexpr int kHB = 368;                         // slot stride (128-byte aligned)
constexpr unsigned kHaloBytes = kHR * 8;
constexpr unsigned kOwnBytes = kNT * 8;          // 32 x 8 box
constexpr int kNP = 3;                           // halo'd plane ring
constexpr int kNX = 4;                           // K2 own-row ring (in-place update + store)

// Each tensor map is its own __grid_constant__ parameter.
// K1: ma = r, mb = p_old, mc = invd (halo'd boxes); K2: ma = p (halo'd box),
// mb = x, mc = r (own-row boxes).

// doubles of operand data (planes + own rows / p_new ring)
template <int MODE, int CB>
constexpr int tma_data() {
  if (MODE == kK2) return kNP * CB * kHB + kNX * 2 * CB * kNT;
  return kNP * (2 * CB + 1) * kHB + 2 * CB * kHR;
}
// bytes: alignment slack + data + mbarriers + block-reduction scratch
template <int MODE, int CB>
constexpr size_t tma_smem() {
  return 128 + sizeof(double) * (tma_data<MODE, CB>() + kNP + kNX + (kNT / 32) * CB * (MODE == kK2 ? 2 : 1));
}

template <int MODE, bool VAR, int CB>
__global__ void __launch_bounds__(kNT, kMinCtas) tma_kernel(const MarchArgs a, const __grid_constant__ CUtensorMap ma,
                                                                const __grid_constant__ CUtensorMap mb,
                                                                const __grid_constant__ CUtensorMap mc) {
  static_assert(MODE == kK1 || MODE == kK2, "tma_kernel: PCG passes only");
  static_assert(kTX == 32 && kTY == 8, "tma_kernel: 32x8 tiles");
  // everything in dynamic shared memory, base rounded up to the 128 bytes the
  // tensor copies need (tma_smem() reserves the slack)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  constexpr int NA = MODE == kK2 ? 2 : 1;
  constexpr int NARR = MODE == kK1 ? 2 * CB + 1 : CB;  // halo'd arrays per plane slot
  unsigned long long* barP = reinterpret_cast<unsigned long long*>(smem + tma_data<MODE, CB>());
  unsigned long long* barX = barP + kNP;
  double(*red)[CB * NA] = reinterpret_cast<double(*)[CB * NA]>(barX + kNX);

  double* planes = smem;                       // [kNP][NARR][kHB]
  double* extra = planes + kNP * NARR * kHB;   // K2: own rows [kNX][2][CB][kNT]; K1: p_new ring [2][CB][kHR]

  const int S = a.S;
  const int S2 = S * S;
  const int P = a.P;
  const long long n = a.n;
  const long long ld = a.ld;
  const int tid = threadIdx.x;
  const int blk = blockIdx.y;
  const int c0 = blockIdx.x * CB;

  unsigned actm = 0, firstm = 0;
  int nact = 0, nnf = 0;
  double colA[CB], colB[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const int c = c0 + j;
    const bool on = c < a.K && a.cols[c].active != 0;
    colA[j] = colB[j] = 0.0;
    if (on) {
      actm |= 1u << j;
      ++nact;
      bool f = false;
      if (MODE == kK1) {
        colB[j] = a.cols[c].beta;
        f = a.cols[c].first != 0;
        if (f) firstm |= 1u << j;
      }
      if (!f) ++nnf;
      if (MODE == kK2) colA[j] = a.cols[c].alpha;
    }
  }
  if (actm == 0) return;
  auto act = [&](int j) { return (actm >> j) & 1u; };
  auto first = [&](int j) { return (firstm >> j) & 1u; };

  const int bx = blk % a.nTX;
  const int by = (blk / a.nTX) % a.nTY;
  const int bz = blk / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = a.zlo + bz * a.ZC;
  const int z1 = min(a.zhi, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;

  if (tid == 0) {
    for (int s = 0; s < kNP; ++s) mbar_init(&barP[s], 1);
    if (MODE == kK2)
      for (int s = 0; s < kNX; ++s) mbar_init(&barX[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto slot_planes = [&](int s) { return planes + s * NARR * kHB; };
  auto slot_own = [&](int s) { return extra + s * 2 * CB * kNT; };  // K2: [2][CB][kNT]
  // elected thread: halo'd plane z (zero-filled outside the lattice) into slot s
  auto issue_halo = [&](int s, int z) {
    const unsigned arrays = MODE == kK1 ? nact + nnf + (VAR ? 1 : 0) : nact;
    mbar_arm(&barP[s], arrays * kHaloBytes);
    double* d = slot_planes(s);
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      if (!act(j)) continue;
      tma_load(d + j * kHB, &ma, x0 - 2, y0 - 1, z, c0 + j, &barP[s]);
      if (MODE == kK1 && !first(j)) tma_load(d + (CB + j) * kHB, &mb, x0 - 2, y0 - 1, z, c0 + j, &barP[s]);
    }
    if (MODE == kK1 && VAR) tma_load(d + 2 * CB * kHB, &mc, x0 - 2, y0 - 1, z, 0, &barP[s]);
  };
  // K2 elected thread: own rows of x and r on plane z into own slot s
  auto issue_own = [&](int s, int z) {
    mbar_arm(&barX[s], 2u * nact * kOwnBytes);
    double* d = slot_own(s);
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      if (!act(j)) continue;
      tma_load(d + j * kNT, &mb, x0, y0, z, c0 + j, &barX[s]);
      tma_load(d + (CB + j) * kNT, &mc, x0, y0, z, c0 + j, &barX[s]);
    }
  };
  auto store_own = [&](int s, int z) {
    const double* d = slot_own(s);
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      if (!act(j)) continue;
      tma_store(&mb, x0, y0, z, c0 + j, d + j * kNT);
      tma_store(&mc, x0, y0, z, c0 + j, d + (CB + j) * kNT);
    }
    bulk_commit();
  };

  // K1: raw plane slot s (plane z) -> p_new = z + beta p_old into ring slot rg
  int hpos[kLoadsPerThread];  // box offset of the halo'd positions this thread transforms (-1: none)
#pragma unroll
  for (int l = 0; l < kLoadsPerThread; ++l) {
    const int i = tid + l * kNT;
    hpos[l] = i < kHP ? (i / kHX) * kRW + i % kHX + 1 : -1;
  }
  auto transform = [&](int s, int rg) {
    const double* rw = slot_planes(s);
    double* ring = extra + rg * CB * kHR;
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      const int i = hpos[l];
      if (i < 0) continue;
      const double d = VAR ? rw[2 * CB * kHB + i] : a.op.invd_const;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        // z = inv_diag * r ; p = z + beta * p   (linalg.cpp:179, 210); zero outside the lattice
        const double zz = __dmul_rn(d, rw[j * kHB + i]);
        ring[j * kHR + i] = first(j) ? zz : __dadd_rn(zz, __dmul_rn(colB[j], rw[(CB + j) * kHB + i]));
      }
    }
  };

  // coefficient offsets (dense layout, see stream_kernel)
  long long offB[kSlots], offF[kSlots];
#pragma unroll
  for (int o = 0; o < kSlots; ++o) {
    offF[o] = o * n;
    offB[o] = o * n - (o & 1) - ((o >> 1) & 1) * S;
  }
  const int ownc = inside ? gy * S + gx : 0;
  const int ownp = inside ? gy * P + gx : 0;
  double cN[4], cC[7], cPp[4], invdP = 0.0;
  auto load_coefs = [&](int t) {
    if (VAR) {
      const int tc = min(max(t, 0), S - 1), tm1 = min(max(t - 1, 0), S - 1);
      const long long pt = static_cast<long long>(tc) * S2 + ownc;
      const long long pm = static_cast<long long>(tm1) * S2 + ownc;
      const double* cf = a.op.coef;
#pragma unroll
      for (int i = 0; i < 4; ++i) cN[i] = ldnc(cf + pt + offB[4 + i]);
#pragma unroll
      for (int i = 0; i < 3; ++i) cC[i] = ldnc(cf + pt + offB[1 + i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) cC[3 + i] = ldnc(cf + pt + offF[i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) cPp[i] = ldnc(cf + pm + offF[4 + i]);
      if (MODE == kK2) invdP = ldnc(a.invd + static_cast<long long>(tm1) * S * P + ownp);
    } else {  // constant operator: fl(w + fl(sigma m)) from the host
#pragma unroll
      for (int i = 0; i < 4; ++i) cN[i] = a.op.wc[4 + i];
#pragma unroll
      for (int i = 0; i < 3; ++i) cC[i] = a.op.wc[1 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i) cC[3 + i] = a.op.wc[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) cPp[i] = a.op.wc[4 + i];
      if (MODE == kK2) invdP = a.op.invd_const;
    }
  };

  double sC[CB], sN[CB], cCur[CB];
  double acc[CB][NA];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    sC[j] = sN[j] = cCur[j] = 0.0;
#pragma unroll
    for (int q = 0; q < NA; ++q) acc[j][q] = 0.0;
  }
  unsigned phP = 0, phX = 0;  // bit s: parity of the next completion of barP[s] / barX[s]
  auto waitP = [&](int s) {
    mbar_wait(&barP[s], (phP >> s) & 1u);
    phP ^= 1u << s;
  };
  auto waitX = [&](int s) {
    mbar_wait(&barX[s], (phX >> s) & 1u);
    phX ^= 1u << s;
  };
  // ring slots: halo'd plane t -> (t - z0 + 1) % kNP; own row u -> (u - z0) % kNX; p_new ring (K1) -> (t - z0 + 1) & 1
  auto sp = [&](int t) { return (t - z0 + 1) % kNP; };
  auto sx = [&](int u) { return (u - z0) & (kNX - 1); };

  // ---- prologue
  if (MODE == kK1) {
    if (tid == 0) {
      issue_halo(0, z0 - 1);
      issue_halo(1, z0);
      issue_halo(2, z0 + 1);
    }
    waitP(0);
    transform(0, 0);
  } else {
    if (tid == 0) {
      issue_halo(0, z0 - 1);
      issue_halo(1, z0);
    }
  }
  load_coefs(z0 - 1);

  const int ib = ty * kRW + tx + 1;  // top-left of the 3x3 window in a halo'd box
  for (int t = z0 - 1; t <= z1; ++t) {
    const bool rowP = t - 1 >= z0;  // row t-1 completes at this step
    if (MODE == kK1) {
      if (t + 1 <= z1) waitP(sp(t + 1));  // raw plane t+1 landed
    } else {
      waitP(sp(t));                        // halo'd p plane t landed
      if (rowP) waitX(sx(t - 1));          // own rows x, r of row t-1 landed
    }
    __syncthreads();  // every thread is done with step t-1 (its slots may be refilled / stored)
    if (tid == 0) {
      if (MODE == kK1) {
        if (t + 3 <= z1) issue_halo(sp(t), t + 3);  // sp(t+3) == sp(t)
      } else {
        if (t - 2 >= z0) store_own(sx(t - 2), t - 2);  // row t-2, updated at step t-1
        if (t + 1 < z1) {
          if (t + 1 - kNX >= z0) bulk_wait_read<1>();   // the slot's previous row has been stored
          issue_own(sx(t + 1), t + 1);
        }
        if (t + 2 <= z1) issue_halo(sp(t + 2), t + 2);  // sp(t+2) == sp(t-1)
      }
    }

    if (inside) {
      const double* Pl = MODE == kK1 ? extra + ((t - z0 + 1) & 1) * CB * kHR : slot_planes(sp(t));
      constexpr int PS = MODE == kK1 ? kHR : kHB;  // per-column stride of the stencil source
      constexpr int R = kRW;
      double* st = MODE == kK2 ? slot_own(sx(t - 1 >= z0 ? t - 1 : z0)) : nullptr;
      // p_new rows of plane t go to global (K1)
      const long long pdst = static_cast<long long>(c0) * ld + (static_cast<long long>(t) * S + gy) * P + gx;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const double* Pj = Pl + j * PS + ib;
        const double vmm = Pj[0], v0m = Pj[1], vm0 = Pj[R], v00 = Pj[R + 1];
        const double vp0 = Pj[R + 2], v0p = Pj[2 * R + 1], vpp = Pj[2 * R + 2];
        if (MODE == kK1 && t >= z0 && t < z1 && act(j)) a.dst[pdst + static_cast<long long>(j) * ld] = v00;
        if (rowP) {  // Pp terms of row t-1: A[v, v+o], o = 4..7
          double s = sC[j];
          s = fma(cPp[0], v00, s);
          s = fma(cPp[1], vp0, s);
          s = fma(cPp[2], v0p, s);
          s = fma(cPp[3], vpp, s);
          const double ctr = cCur[j];
          if (MODE == kK1) {
            acc[j][0] = fma(ctr, s, acc[j][0]);  // p'q
          } else {
            // x += alpha p ; r -= alpha q ; z = invd r  (linalg.cpp:202-206)
            const double al = colA[j];
            double* xs = st + j * kNT + tid;
            double* rs = st + (CB + j) * kNT + tid;
            const double xn = __dadd_rn(*xs, __dmul_rn(al, ctr));
            const double rn = __dsub_rn(*rs, __dmul_rn(al, s));
            *xs = xn;
            *rs = rn;
            const double zz = __dmul_rn(invdP, rn);
            acc[j][0] = fma(rn, zz, acc[j][0]);
            acc[j][1] = fma(rn, rn, acc[j][1]);
          }
        }
        // centre terms of row t, Pm terms of row t+1 (see stream_kernel)
        double c = sN[j];
        c = fma(cC[2], vmm, c);
        c = fma(cC[1], v0m, c);
        c = fma(cC[0], vm0, c);
        c = fma(cC[3], v00, c);
        c = fma(cC[4], vp0, c);
        c = fma(cC[5], v0p, c);
        c = fma(cC[6], vpp, c);
        double nx = 0.0;
        nx = fma(cN[3], vmm, nx);
        nx = fma(cN[2], v0m, nx);
        nx = fma(cN[1], vm0, nx);
        nx = fma(cN[0], v00, nx);
        sC[j] = c;
        sN[j] = nx;
        cCur[j] = v00;
      }
    }
    // generic-proxy writes of the own rows must be visible to the TMA store
    if (MODE == kK2 && rowP) fence_async_smem();
    if (MODE == kK1 && t + 1 <= z1) transform(sp(t + 1), (t - z0 + 2) & 1);
    if (t < z1) load_coefs(t + 1);
  }
  if (MODE == kK2) {
    __syncthreads();
    if (tid == 0) {
      store_own(sx(z1 - 1), z1 - 1);
      bulk_wait<0>();
    }
  }

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
      a.partials[(static_cast<long long>(c0 + j) * 3 + q) * a.nblk + blk] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// K2 for a variable operator with the coefficients staged by TMA as well
// (k2c). The 16 per-thread coefficient loads per plane of tma_kernel were
// the largest cost of the PCG iteration (a constant-coefficient operator,
// same kernels otherwise, runs 27 % faster): here one box per plane brings
// the 8 slots of the (A + sigma M) coefficients with their (-1,-1) halo and
// one box the inverse diagonal, all into the ring slot of the p plane, so
// the thread reads them from shared memory. x and r stay in registers: the
// own rows of row t are loaded at step t and updated at step t+1.
constexpr int kCR = kRW * (kTY + 1);     // coefficient box rows y0-1 .. y0+7 (back weights reach y-1 only)
constexpr int kCS = kSlots * kCR + kNT;  // coefficient slot: [8][9][36] boxes + inverse-diagonal own box [8][32]

template <int CB>
constexpr int k2c_data() {
  return kNP * CB * kHB + kNP * kCS;
}
template <int CB>
constexpr size_t k2c_smem() {
  return 128 + sizeof(double) * (k2c_data<CB>() + kNP + (kNT / 32) * CB * 2);
}

// XM: x update mode. 2: x += alpha p every iteration. Deferred pairs: 0 (even
// iterations) leaves x untouched, 1 (odd) applies both pending updates,
// x = fl(fl(x + fl(alpha' p')) + fl(alpha p)) with p' = the previous direction
// (a.pold) -- the same operations as two single updates, at half the x traffic.
template <int CB, int XM>
__global__ void __launch_bounds__(kNT, CB >= 8 ? 1 : kMinCtas)
    k2c_kernel(const MarchArgs a, const __grid_constant__ CUtensorMap mp, const __grid_constant__ CUtensorMap mcoef,
               const __grid_constant__ CUtensorMap minvd) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw + ((128u - (su32(smem_raw) & 127u)) & 127u));
  double* planes = smem;                       // [kNP][CB][kHB]
  double* coefs = planes + kNP * CB * kHB;     // [kNP][kCS]
  unsigned long long* barP = reinterpret_cast<unsigned long long*>(smem + k2c_data<CB>());
  double(*red)[CB * 2] = reinterpret_cast<double(*)[CB * 2]>(barP + kNP);

  const int S = a.S;
  const int P = a.P;
  const long long ld = a.ld;
  const int tid = threadIdx.x;
  const int blk = blockIdx.y;
  const int c0 = blockIdx.x * CB;

  unsigned actm = 0;
  int nact = 0;
  double colA[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const int c = c0 + j;
    const bool on = c < a.K && a.cols[c].active != 0;
    colA[j] = 0.0;
    if (on) {
      actm |= 1u << j;
      ++nact;
      colA[j] = a.cols[c].alpha;
    }
  }
  if (actm == 0) return;
  // XM == 1: alpha of the previous iteration, parked in the (loop-idle)
  // reduction scratch instead of registers
  double* colA2 = &red[0][0];
  if (XM == 1 && tid < CB) colA2[tid] = c0 + tid < a.K ? a.cols[c0 + tid].alpha_prev : 0.0;
  auto act = [&](int j) { return (actm >> j) & 1u; };

  const int bx = blk % a.nTX;
  const int by = (blk / a.nTX) % a.nTY;
  const int bz = blk / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = a.zlo + bz * a.ZC;
  const int z1 = min(a.zhi, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;

  if (tid == 0) {
    for (int s = 0; s < kNP; ++s) mbar_init(&barP[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int s, int z) {  // thread 0: p, coefficient and inverse-diagonal planes z into slot s
    mbar_arm(&barP[s], nact * kHaloBytes + (kSlots * kCR + kNT) * 8u);
    double* d = planes + s * CB * kHB;
#pragma unroll
    for (int j = 0; j < CB; ++j)
      if (act(j)) tma_load(d + j * kHB, &mp, x0 - 2, y0 - 1, z, c0 + j, &barP[s]);
    double* cf = coefs + s * kCS;
    tma_load(cf, &mcoef, x0 - 2, y0 - 1, z, 0, &barP[s]);
    tma_load(cf + kSlots * kCR, &minvd, x0, y0, z, 0, &barP[s]);
  };
  unsigned phP = 0;
  auto waitP = [&](int s) {
    mbar_wait(&barP[s], (phP >> s) & 1u);
    phP ^= 1u << s;
  };
  auto sp = [&](int t) { return (t - z0 + 1) % kNP; };

  if (tid == 0) {
    issue(0, z0 - 1);
    issue(1, z0);
  }

  double sC[CB], sN[CB], cCur[CB], acc[CB][2];
  double xc[CB], rc[CB], pp[CB];  // own x, r (and previous direction) of row t-1
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    sC[j] = sN[j] = cCur[j] = 0.0;
    acc[j][0] = acc[j][1] = 0.0;
    xc[j] = rc[j] = pp[j] = 0.0;
  }
  double cPp[4] = {0.0, 0.0, 0.0, 0.0}, invdP = 0.0;  // own slots 4..7 and 1/diag of plane t-1
  const int o0 = (ty + 1) * kRW + tx + 2;               // own point in a coefficient box
  const int ib = ty * kRW + tx + 1;                      // top-left of the 3x3 window in a p box
  const long long own0 = static_cast<long long>(c0) * ld + static_cast<long long>(gy) * P + gx;

  for (int t = z0 - 1; t <= z1; ++t) {
    const bool rowP = t - 1 >= z0;
    // own x, r of row t-1, issued ahead of the plane wait and barrier so
    // their latency overlaps them
    if (inside && rowP) {
      const long long o = own0 + static_cast<long long>(t - 1) * S * P;
#pragma unroll
      for (int j = 0; j < CB; ++j)
        if (act(j)) {
          if (XM != 0) xc[j] = ldnc(a.x + o + j * ld);
          if (XM == 1) pp[j] = ldnc(a.pold + o + j * ld);
          rc[j] = ldnc(a.r + o + j * ld);
        }
    }
    waitP(sp(t));
    __syncthreads();  // slot sp(t-1) (read at step t-1) may be refilled
    if (tid == 0 && t + 2 <= z1) issue(sp(t + 2), t + 2);

    if (inside) {
      const double* Pl = planes + sp(t) * CB * kHB;
      const double* Cp = coefs + sp(t) * kCS;
      double cN[4], cC[7];
      cC[0] = Cp[1 * kCR + o0 - 1];        // slot 1 at (-1, 0)
      cC[1] = Cp[2 * kCR + o0 - kRW];      // slot 2 at (0, -1)
      cC[2] = Cp[3 * kCR + o0 - kRW - 1];  // slot 3 at (-1, -1)
#pragma unroll
      for (int i = 0; i < 4; ++i) cC[3 + i] = Cp[i * kCR + o0];  // own slots 0..3
      cN[0] = Cp[4 * kCR + o0];
      cN[1] = Cp[5 * kCR + o0 - 1];
      cN[2] = Cp[6 * kCR + o0 - kRW];
      cN[3] = Cp[7 * kCR + o0 - kRW - 1];
      const long long orow = own0 + static_cast<long long>(t - 1) * S * P;  // row t-1
      // one column body for both kinds of step (rowP is uniform), stores
      // predicated rather than branched, so the 4 columns' FMA chains can
      // interleave
      auto body = [&](auto has_row) {
        constexpr bool ROWP = decltype(has_row)::value;
        double sP[CB], pOld[CB];  // completed row sums of row t-1 and p at row t-1
#pragma unroll
        for (int j = 0; j < CB; ++j) {
          const double* Pj = Pl + j * kHB + ib;
          const double vmm = Pj[0], v0m = Pj[1], vm0 = Pj[kRW], v00 = Pj[kRW + 1];
          const double vp0 = Pj[kRW + 2], v0p = Pj[2 * kRW + 1], vpp = Pj[2 * kRW + 2];
          if (ROWP) {  // Pp terms of row t-1: A[v, v+o], o = 4..7
            double sv = sC[j];
            sv = fma(cPp[0], v00, sv);
            sv = fma(cPp[1], vp0, sv);
            sv = fma(cPp[2], v0p, sv);
            sv = fma(cPp[3], vpp, sv);
            sP[j] = sv;
            pOld[j] = cCur[j];
          }
          // centre terms of row t, Pm terms of row t+1 (see stream_kernel)
          double c = sN[j];
          c = fma(cC[2], vmm, c);
          c = fma(cC[1], v0m, c);
          c = fma(cC[0], vm0, c);
          c = fma(cC[3], v00, c);
          c = fma(cC[4], vp0, c);
          c = fma(cC[5], v0p, c);
          c = fma(cC[6], vpp, c);
          double nx = 0.0;
          nx = fma(cN[3], vmm, nx);
          nx = fma(cN[2], v0m, nx);
          nx = fma(cN[1], vm0, nx);
          nx = fma(cN[0], v00, nx);
          sC[j] = c;
          sN[j] = nx;
          cCur[j] = v00;
        }
        if (ROWP) {
          // the row t-1 updates last, so the x, r loads issued at the top of
          // the step have the stencil work above to land
#pragma unroll
          for (int j = 0; j < CB; ++j) {
            // x += alpha p ; r -= alpha q ; z = invd r  (linalg.cpp:202-206)
            if (XM == 2) {
              const double xv = __dadd_rn(xc[j], __dmul_rn(colA[j], pOld[j]));
              st_if(a.x + orow + j * ld, xv, act(j));
            } else if (XM == 1) {
              const double xv = __dadd_rn(__dadd_rn(xc[j], __dmul_rn(colA2[j], pp[j])), __dmul_rn(colA[j], pOld[j]));
              st_if(a.x + orow + j * ld, xv, act(j));
            }
            const double rv = __dsub_rn(rc[j], __dmul_rn(colA[j], sP[j]));
            st_if(a.r + orow + j * ld, rv, act(j));
            const double zz = __dmul_rn(invdP, rv);
            acc[j][0] = fma(rv, zz, acc[j][0]);
            acc[j][1] = fma(rv, rv, acc[j][1]);
          }
        }
      };
      if (rowP) body(std::true_type{});
      else body(std::false_type{});
      // plane t's own slots 4..7 and 1/diag serve row t at the next step
#pragma unroll
      for (int i = 0; i < 4; ++i) cPp[i] = Cp[(4 + i) * kCR + o0];
      invdP = Cp[kSlots * kCR + tid];
    }
  }

  if (XM == 1) __syncthreads();  // colA2 lives in the reduction scratch
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int j = 0; j < CB; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double v = warp_sum(acc[j][q]);
      if (lane == 0) red[warp][j * 2 + q] = v;
    }
  __syncthreads();
  if (tid < CB * 2) {
    const int j = tid / 2, q = tid % 2;
    if (act(j)) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kNT / 32; ++w) s += red[w][tid];
      a.partials[(static_cast<long long>(c0 + j) * 3 + q) * a.nblk + blk] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// K1 on the symmetric form of p'Ap (k1f): with A symmetric,
//   p'Ap = sum_v p_v (A_vv p_v + 2 sum_{o forward} A[v, v+o] p_{v+o}),
// so a point needs only its own 8 coefficient slots (no back weights from
// neighbours) and p_new at its forward neighbours (+x, +y, +z combinations):
// half the stencil FMAs of the full row sum, a one-sided halo (34 x 9 boxes
// from (x0, y0)) and 8 coalesced own-coefficient loads per plane, issued a
// step ahead. The raw planes (r, p_old, 1/diag) run two steps ahead in a
// 3-slot TMA ring (with one step the plane wait was 46 % of the stalls).
// The reduction order differs from the row-sum form by rounding only.
constexpr int kFW = 34;             // forward box row width (x0 .. x0+33; 16-byte aligned start)
constexpr int kFR = kFW * 9;        // 306 doubles per forward box (rows y0 .. y0+8)
constexpr int kFB = 320;            // slot stride (128-byte aligned)
constexpr int kFN = 3;              // raw ring slots

template <bool VAR, int CB>
constexpr int k1f_data() {
  return kFN * (2 * CB + (VAR ? 1 : 0)) * kFB + 3 * CB * kFB;
}
template <bool VAR, int CB>
constexpr size_t k1f_smem() {
  return 128 + sizeof(double) * (k1f_data<VAR, CB>() + kFN + (kNT / 32) * CB);
}

template <bool VAR, int CB>
__global__ void __launch_bounds__(kNT, kMinCtas)
    k1f_kernel(const MarchArgs a, const __grid_constant__ CUtensorMap mr, const __grid_constant__ CUtensorMap mpo,
               const __grid_constant__ CUtensorMap minv) {
  constexpr int NARR = 2 * CB + (VAR ? 1 : 0);  // raw arrays: r, p_old (per column), inverse diagonal
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw + ((128u - (su32(smem_raw) & 127u)) & 127u));
  double* raw = smem;                         // [kFN][NARR][kFB]
  double* ring = raw + kFN * NARR * kFB;      // p_new [3][CB][kFB]
  unsigned long long* barR = reinterpret_cast<unsigned long long*>(smem + k1f_data<VAR, CB>());
  double(*red)[CB] = reinterpret_cast<double(*)[CB]>(barR + kFN);

  const int S = a.S;
  const int S2 = S * S;
  const int P = a.P;
  const long long n = a.n;
  const long long ld = a.ld;
  const int tid = threadIdx.x;
  const int blk = blockIdx.y;
  const int c0 = blockIdx.x * CB;

  unsigned actm = 0, firstm = 0;
  int nact = 0, nnf = 0;
  double colB[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const int c = c0 + j;
    const bool on = c < a.K && a.cols[c].active != 0;
    colB[j] = 0.0;
    if (on) {
      actm |= 1u << j;
      ++nact;
      colB[j] = a.cols[c].beta;
      if (a.cols[c].first != 0) firstm |= 1u << j;
      else ++nnf;
    }
  }
  if (actm == 0) return;
  auto act = [&](int j) { return (actm >> j) & 1u; };
  auto first = [&](int j) { return (firstm >> j) & 1u; };

  const int bx = blk % a.nTX;
  const int by = (blk / a.nTX) % a.nTY;
  const int bz = blk / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = a.zlo + bz * a.ZC;
  const int z1 = min(a.zhi, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;

  if (tid == 0) {
    for (int i = 0; i < kFN; ++i) mbar_init(&barR[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // thread 0: raw plane z (r, p_old, 1/diag over x0..x0+33, y0..y0+8) into raw slot s
  auto issue_raw = [&](int s, int z) {
    mbar_arm(&barR[s], (nact + nnf + (VAR ? 1 : 0)) * static_cast<unsigned>(kFR * 8));
    double* d = raw + s * NARR * kFB;
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      if (!act(j)) continue;
      tma_load(d + j * kFB, &mr, x0, y0, z, c0 + j, &barR[s]);
      if (!first(j)) tma_load(d + (CB + j) * kFB, &mpo, x0, y0, z, c0 + j, &barR[s]);
    }
    if (VAR) tma_load(d + 2 * CB * kFB, &minv, x0, y0, z, 0, &barR[s]);
  };
  unsigned phR = 0;
  auto waitR = [&](int s) {
    mbar_wait(&barR[s], (phR >> s) & 1u);
    phR ^= 1u << s;
  };
  // raw plane z (slot s) -> p_new = z + beta p_old into ring slot q (linalg.cpp:179, 210)
  auto transform = [&](int s, int q) {
    const double* rw = raw + s * NARR * kFB;
    double* pr = ring + q * CB * kFB;
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const int i = tid + l * kNT;
      if (i >= kFR) continue;
      const double d = VAR ? rw[2 * CB * kFB + i] : a.op.invd_const;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const double zz = __dmul_rn(d, rw[j * kFB + i]);
        pr[j * kFB + i] = first(j) ? zz : __dadd_rn(zz, __dmul_rn(colB[j], rw[(CB + j) * kFB + i]));
      }
    }
  };
  // own coefficient slots of plane z (dense operator layout, a.op.coef)
  const long long cown = inside ? static_cast<long long>(gy) * S + gx : 0;
  double w[kSlots];
  auto load_w = [&](int z) {
    if (VAR) {
      const double* cf = a.op.coef + static_cast<long long>(min(z, S - 1)) * S2 + cown;
#pragma unroll
      for (int o = 0; o < kSlots; ++o) w[o] = ldnc(cf + o * n);
    } else {
#pragma unroll
      for (int o = 0; o < kSlots; ++o) w[o] = a.op.wc[o];
    }
  };

  // ---- prologue: p_new planes z0, z0+1 in the ring, raw planes z0+2, z0+3 in flight
  if (tid == 0) {
    issue_raw(0, z0);
    issue_raw(1, z0 + 1);
    if (z0 + 2 <= z1) issue_raw(2, z0 + 2);
  }
  load_w(z0);
  waitR(0);
  transform(0, 0);
  waitR(1);
  transform(1, 1);
  __syncthreads();
  if (tid == 0 && z0 + 3 <= z1) issue_raw(0, z0 + 3);

  double acc[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) acc[j] = 0.0;
  const int io = ty * kFW + tx;  // own point in a forward box
  const long long own0 = static_cast<long long>(c0) * ld + static_cast<long long>(gy) * P + gx;
  // the four in-plane values a point reads of plane t+1 at step t are the
  // ones it reads of plane t at step t+1: carried in registers, so every
  // p_new plane is read from shared memory once
  double cv[CB][4];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const double* A0 = ring + j * kFB + io;  // plane z0 (ring slot 0)
    cv[j][0] = A0[0];
    cv[j][1] = A0[1];
    cv[j][2] = A0[kFW];
    cv[j][3] = A0[kFW + 1];
  }
  for (int t = z0; t < z1; ++t) {
    const int q1 = (t + 1 - z0) % 3;
    if (inside) {
      const long long orow = own0 + static_cast<long long>(t) * S * P;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const double* A1 = ring + q1 * CB * kFB + j * kFB + io;  // plane t+1
        const double pv = cv[j][0];
        const double n0 = A1[0], n1 = A1[1], n2 = A1[kFW], n3 = A1[kFW + 1];
        double s = w[1] * cv[j][1];
        s = fma(w[2], cv[j][2], s);
        s = fma(w[3], cv[j][3], s);
        s = fma(w[4], n0, s);
        s = fma(w[5], n1, s);
        s = fma(w[6], n2, s);
        s = fma(w[7], n3, s);
        acc[j] = fma(pv, fma(2.0, s, w[0] * pv), acc[j]);  // p_v (A p)_v over the symmetric pairs
        st_if(a.dst + orow + j * ld, pv, act(j));         // p_new (own points of plane t)
        cv[j][0] = n0;
        cv[j][1] = n1;
        cv[j][2] = n2;
        cv[j][3] = n3;
      }
    }
    if (t + 1 < z1) load_w(t + 1);  // lands during the transform and the barrier
    if (t + 2 <= z1) {
      const int s2 = (t + 2 - z0) % kFN;
      waitR(s2);                              // raw plane t+2 landed
      transform(s2, (t + 2 - z0) % 3);        // ring slot of plane t-1 (read at step t-1)
    }
    __syncthreads();  // p_new(t+2) visible; raw slot of t+2 consumed
    if (tid == 0 && t + 4 <= z1) issue_raw((t + 4 - z0) % kFN, t + 4);  // slot of raw t+1 (transformed at step t-1)
  }

  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const double v = warp_sum(acc[j]);
    if (lane == 0) red[warp][j] = v;
  }
  __syncthreads();
  if (tid < CB && act(tid)) {
    double s = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < kNT / 32; ++w2) s += red[w2][tid];
    a.partials[(static_cast<long long>(c0 + tid) * 3 + 0) * a.nblk + blk] = s;
  }
}

// ---------------------------------------------------------------------------
// PCG setup on the TMA path (k0c, warm start with the mass right-hand side,
// source_solve_step paro.cpp:96-104 / cg_solve linalg.cpp:150-189):
//   b = (M u) (lambda + sigma), r = b - A u, partials b'b, r'z, r'r,
// with u already copied into the solver's x (row-padded, pad_cols_kernel).
// The u planes, the 8 coefficient slots and 1/diag arrive by TMA exactly as
// in k2c; both row sums are summed without FMA contraction in ascending
// column order, i.e. the reference CSR matvec's operations (as the
// stream_kernel setup it replaces).
template <int CB>
__global__ void __launch_bounds__(kNT, kMinCtas)
    k0c_kernel(const MarchArgs a, const __grid_constant__ CUtensorMap mp, const __grid_constant__ CUtensorMap mcoef,
               const __grid_constant__ CUtensorMap minvd) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw + ((128u - (su32(smem_raw) & 127u)) & 127u));
  double* planes = smem;                       // [kNP][CB][kHB]
  double* coefs = planes + kNP * CB * kHB;     // [kNP][kCS]
  unsigned long long* barP = reinterpret_cast<unsigned long long*>(smem + k2c_data<CB>());
  double(*red)[CB * 3] = reinterpret_cast<double(*)[CB * 3]>(barP + kNP);

  const int S = a.S;
  const int P = a.P;
  const long long ld = a.ldw;  // column stride of the solver buffers
  const int tid = threadIdx.x;
  const int blk = blockIdx.y;
  const int c0 = blockIdx.x * CB;

  unsigned actm = 0;
  int nact = 0;
  double scl[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const int c = c0 + j;
    const bool on = c < a.K && a.cols[c].active != 0;
    scl[j] = 0.0;
    if (on) {
      actm |= 1u << j;
      ++nact;
      scl[j] = a.scale[c];  // rhs scale lambda + sigma (paro.cpp:96-98)
    }
  }
  if (actm == 0) return;
  auto act = [&](int j) { return (actm >> j) & 1u; };

  const int bx = blk % a.nTX;
  const int by = (blk / a.nTX) % a.nTY;
  const int bz = blk / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = a.zlo + bz * a.ZC;
  const int z1 = min(a.zhi, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;

  if (tid == 0) {
    for (int s = 0; s < kNP; ++s) mbar_init(&barP[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int s, int z) {
    mbar_arm(&barP[s], nact * kHaloBytes + (kSlots * kCR + kNT) * 8u);
    double* d = planes + s * CB * kHB;
#pragma unroll
    for (int j = 0; j < CB; ++j)
      if (act(j)) tma_load(d + j * kHB, &mp, x0 - 2, y0 - 1, z, c0 + j, &barP[s]);
    double* cf = coefs + s * kCS;
    tma_load(cf, &mcoef, x0 - 2, y0 - 1, z, 0, &barP[s]);
    tma_load(cf + kSlots * kCR, &minvd, x0, y0, z, 0, &barP[s]);
  };
  unsigned phP = 0;
  auto waitP = [&](int s) {
    mbar_wait(&barP[s], (phP >> s) & 1u);
    phP ^= 1u << s;
  };
  auto sp = [&](int t) { return (t - z0 + 1) % kNP; };
  auto madd = [](double acc, double w, double x) { return __dadd_rn(acc, __dmul_rn(w, x)); };

  if (tid == 0) {
    issue(0, z0 - 1);
    issue(1, z0);
  }

  double sC[CB], sN[CB], mC[CB], mN[CB], acc[CB][3];
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    sC[j] = sN[j] = mC[j] = mN[j] = 0.0;
    acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
  }
  double mw[kSlots];
#pragma unroll
  for (int o = 0; o < kSlots; ++o) mw[o] = a.mw[o];
  double cPp[4] = {0.0, 0.0, 0.0, 0.0}, invdP = 0.0;
  const int o0 = (ty + 1) * kRW + tx + 2;
  const int ib = ty * kRW + tx + 1;
  const long long own0 = static_cast<long long>(c0) * ld + static_cast<long long>(gy) * P + gx;

  for (int t = z0 - 1; t <= z1; ++t) {
    const bool rowP = t - 1 >= z0;
    waitP(sp(t));
    __syncthreads();
    if (tid == 0 && t + 2 <= z1) issue(sp(t + 2), t + 2);
    if (inside) {
      const double* Pl = planes + sp(t) * CB * kHB;
      const double* Cp = coefs + sp(t) * kCS;
      double cN[4], cC[7];
      cC[0] = Cp[1 * kCR + o0 - 1];
      cC[1] = Cp[2 * kCR + o0 - kRW];
      cC[2] = Cp[3 * kCR + o0 - kRW - 1];
#pragma unroll
      for (int i = 0; i < 4; ++i) cC[3 + i] = Cp[i * kCR + o0];
      cN[0] = Cp[4 * kCR + o0];
      cN[1] = Cp[5 * kCR + o0 - 1];
      cN[2] = Cp[6 * kCR + o0 - kRW];
      cN[3] = Cp[7 * kCR + o0 - kRW - 1];
      const long long orow = own0 + static_cast<long long>(t - 1) * S * P;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const double* Pj = Pl + j * kHB + ib;
        const double vmm = Pj[0], v0m = Pj[1], vm0 = Pj[kRW], v00 = Pj[kRW + 1];
        const double vp0 = Pj[kRW + 2], v0p = Pj[2 * kRW + 1], vpp = Pj[2 * kRW + 2];
        if (rowP) {
          double sv = sC[j];
          sv = madd(sv, cPp[0], v00);
          sv = madd(sv, cPp[1], vp0);
          sv = madd(sv, cPp[2], v0p);
          sv = madd(sv, cPp[3], vpp);
          double m = mC[j];
          m = madd(m, mw[4], v00);
          m = madd(m, mw[5], vp0);
          m = madd(m, mw[6], v0p);
          m = madd(m, mw[7], vpp);
          const double bb = __dmul_rn(m, scl[j]);  // b = (M u) scale (model.cpp:248-249)
          const double rr = __dsub_rn(bb, sv);     // r = b - A x0 (linalg.cpp:184-185)
          st_if(a.dst + orow + j * ld, rr, act(j));
          const double zz = __dmul_rn(invdP, rr);
          acc[j][0] += bb * bb;
          acc[j][1] += rr * zz;
          acc[j][2] += rr * rr;
        }
        double c = sN[j];
        c = madd(c, cC[2], vmm);
        c = madd(c, cC[1], v0m);
        c = madd(c, cC[0], vm0);
        c = madd(c, cC[3], v00);
        c = madd(c, cC[4], vp0);
        c = madd(c, cC[5], v0p);
        c = madd(c, cC[6], vpp);
        double nx = 0.0;
        nx = madd(nx, cN[3], vmm);
        nx = madd(nx, cN[2], v0m);
        nx = madd(nx, cN[1], vm0);
        nx = madd(nx, cN[0], v00);
        sC[j] = c;
        sN[j] = nx;
        double m = mN[j];
        m = madd(m, mw[3], vmm);
        m = madd(m, mw[2], v0m);
        m = madd(m, mw[1], vm0);
        m = madd(m, mw[0], v00);
        m = madd(m, mw[1], vp0);
        m = madd(m, mw[2], v0p);
        m = madd(m, mw[3], vpp);
        double mx = 0.0;
        mx = madd(mx, mw[7], vmm);
        mx = madd(mx, mw[6], v0m);
        mx = madd(mx, mw[5], vm0);
        mx = madd(mx, mw[4], v00);
        mC[j] = m;
        mN[j] = mx;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) cPp[i] = Cp[(4 + i) * kCR + o0];
      invdP = Cp[kSlots * kCR + tid];
    }
  }

  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int j = 0; j < CB; ++j)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double v = warp_sum(acc[j][q]);
      if (lane == 0) red[warp][j * 3 + q] = v;
    }
  __syncthreads();
  if (tid < CB * 3) {
    const int j = tid / 3, q = tid % 3;
    if (act(j)) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < kNT / 32; ++w) sum += red[w][tid];
      a.partials[(static_cast<long long>(c0 + j) * 3 + q) * a.nblk + blk] = sum;
    }
  }
}

struct Maps {
  CUtensorMap a, b, c;
};

template <int MODE, bool VAR, int CB>
void launch_k(const MarchArgs& a, const Maps& m, cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = tma_smem<MODE, CB>();
  static std::once_flag once;
  std::call_once(once, [] {
    PARO_CUDA(cudaFuncSetAttribute(tma_kernel<MODE, VAR, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
  });
  dim3 grid(groups, a.nblk);
  tma_kernel<MODE, VAR, CB><<<grid, kNT, sm, st>>>(a, m.a, m.b, m.c);
  PARO_CUDA(cudaGetLastError());
}

template <int MODE, bool VAR>
void launch_cb(int cb, const MarchArgs& a, const Maps& m, cudaStream_t st) {
  switch (cb) {
    case 1: launch_k<MODE, VAR, 1>(a, m, st); break;
    case 2: launch_k<MODE, VAR, 2>(a, m, st); break;
    default: launch_k<MODE, VAR, 4>(a, m, st); break;
  }
}

template <bool VAR, int CB>
void launch_k1f(const MarchArgs& a, const CUtensorMap& mr, const CUtensorMap& mpo, const CUtensorMap& minv,
                cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = k1f_smem<VAR, CB>();
  static std::once_flag once;
  std::call_once(once, [] {
    PARO_CUDA(cudaFuncSetAttribute(k1f_kernel<VAR, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
  });
  dim3 grid(groups, a.nblk);
  k1f_kernel<VAR, CB><<<grid, kNT, sm, st>>>(a, mr, mpo, minv);
  PARO_CUDA(cudaGetLastError());
}

template <int CB, int XM>
void launch_k2c_x(const MarchArgs& a, const Maps& m, cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = k2c_smem<CB>();
  static std::once_flag once;
  std::call_once(once, [] {
    PARO_CUDA(cudaFuncSetAttribute(k2c_kernel<CB, XM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
  });
  dim3 grid(groups, a.nblk);
  k2c_kernel<CB, XM><<<grid, kNT, sm, st>>>(a, m.a, m.b, m.c);
  PARO_CUDA(cudaGetLastError());
}

template <int CB>
void launch_k2c(const MarchArgs& a, const Maps& m, cudaStream_t st) {
  if (a.xmode == 0) launch_k2c_x<CB, 0>(a, m, st);
  else if (a.xmode == 1) launch_k2c_x<CB, 1>(a, m, st);
  else launch_k2c_x<CB, 2>(a, m, st);
}

template <int CB>
void launch_k0c(const MarchArgs& a, const Maps& m, cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = k2c_smem<CB>() + sizeof(double) * (kNT / 32) * CB;  // 3 partials per column
  static std::once_flag once;
  std::call_once(once, [] {
    PARO_CUDA(cudaFuncSetAttribute(k0c_kernel<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  });
  dim3 grid(groups, a.nblk);
  k0c_kernel<CB><<<grid, kNT, sm, st>>>(a, m.a, m.b, m.c);
  PARO_CUDA(cudaGetLastError());
}


// ---------------------------------------------------------------------------
// Batched operator apply y = A x on the caller's DENSE layout (odd S, column
// stride n), x planes staged by TMA (k3f). A tensor map needs 16-byte strides,
// which the dense rows (S doubles, S odd) do not have, so x is described as a
// flat 2-D view of the whole [K][n] buffer with rows of 2S doubles: lattice
// row g (= c S^2 + z S + y over all columns) is element (g/2, x) of the view
// when g is even and (g/2, S + x) when g is odd. The ten halo rows of a tile
// plane alternate in parity, so they arrive as two boxes of 5 view rows x 36,
// one per parity; an even row's box starts at x0 - 2 and an odd row's at
// S + x0 - 1, both 16-byte aligned (odd S). Neighbours outside the lattice
// are other rows / planes / columns in the flat view and are masked to zero
// by the consumer (the Dirichlet elimination, fem.cpp:21-28). Coefficients of
// a variable operator come from the row-padded copy by one [8][9][36] box per
// plane exactly as in k2c. Row sums: the streaming sums of stream_kernel in
// ascending column order without FMA contraction, i.e. the operations of the
// reference CSR matvec (linalg.cpp:88-94), so y is bit-identical to it.
constexpr int kFV = 5 * kRW;  // one parity box: 5 view rows x 36
constexpr int kFS = 192;      // parity box stride (128-byte aligned)
constexpr int kFC = 2 * kFS;  // per-column plane slot

// NX: x-plane ring slots (planes issued NX - 1 ahead); NC: coefficient ring
// slots (NC - 1 ahead). The x planes are the DRAM stream, the coefficient
// boxes mostly L2 hits shared by the column groups of a tile, so the x ring
// is the deep one.
template <bool VAR, int CB, int NX = kNP, int NC = kNP>
constexpr int k3f_data() {
  return NX * CB * kFC + (VAR ? NC * kSlots * kCR : 0);
}
template <bool VAR, int CB, int NX = kNP, int NC = kNP>
constexpr size_t k3f_smem() {
  return 128 + sizeof(double) * (k3f_data<VAR, CB, NX, NC>() + NX + NC);
}

__device__ __forceinline__ void tma_load2(double* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(su32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}

template <bool VAR, int CB, int NX = kNP, int NC = kNP>
__global__ void __launch_bounds__(kNT, VAR ? kMinCtas : 3)
    k3f_kernel(const MarchArgs a, const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mcoef) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw + ((128u - (su32(smem_raw) & 127u)) & 127u));
  double* planes = smem;                    // [NX][CB][kFC]: parity boxes [2][5][36] per column
  double* coefs = planes + NX * CB * kFC;   // [NC][kSlots][kCR] (VAR)
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + k3f_data<VAR, CB, NX, NC>());
  unsigned long long* barC = bar + NX;

  const int S = a.S;
  const int S2 = S * S;
  const int tid = threadIdx.x;
  const int blk = blockIdx.y;
  const int c0 = blockIdx.x * CB;
  const int ncol = min(CB, a.K - c0);

  const int bx = blk % a.nTX;
  const int by = (blk / a.nTX) % a.nTY;
  const int bz = blk / (a.nTX * a.nTY);
  const int x0 = bx * kTX, y0 = by * kTY;
  const int z0 = a.zlo + bz * a.ZC;
  const int z1 = min(a.zhi, z0 + a.ZC);
  const int tx = tid % kTX, ty = tid / kTX;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool inside = gx < S && gy < S;

  if (tid == 0) {
    for (int s = 0; s < NX; ++s) mbar_init(&bar[s], 1);
    for (int s = 0; s < NC; ++s) mbar_init(&barC[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // thread 0: plane z of the x columns (two parity boxes each) into x slot s
  auto issue = [&](int s, int z) {
    const bool zin = z >= 0 && z < S;
    mbar_arm(&bar[s], zin ? static_cast<unsigned>(ncol) * 2u * kFV * 8u : 0u);
    if (zin) {
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (j >= ncol) continue;
        const int gf = (c0 + j) * S2 + z * S + y0 - 1;  // lattice row of halo row 0
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int g = gf + h;
          tma_load2(planes + (s * CB + j) * kFC + h * kFS, &mx, (g & 1) ? S + x0 - 1 : x0 - 2, g >> 1, &bar[s]);
        }
      }
    }
  };
  // thread 0: the coefficient box of plane z into coefficient slot s
  auto issue_c = [&](int s, int z) {
    mbar_arm(&barC[s], kSlots * kCR * 8u);
    tma_load(coefs + s * kSlots * kCR, &mcoef, x0 - 2, y0 - 1, z, 0, &barC[s]);
  };
  unsigned ph = 0, phC = 0;

  if (tid == 0) {
    for (int q = 0; q < NX - 1; ++q) issue(q, z0 - 1 + q);
    if (VAR)
      for (int q = 0; q < NC - 1; ++q) issue_c(q, z0 - 1 + q);
  }

  double sC[CB], sN[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) sC[j] = sN[j] = 0.0;
  double cPp[4] = {0.0, 0.0, 0.0, 0.0};  // own slots 4..7 of plane t-1
  const int o0 = (ty + 1) * kRW + tx + 2;
  const long long own = static_cast<long long>(gy) * S + gx;
  auto madd = [](double s, double w, double x) { return __dadd_rn(s, __dmul_rn(w, x)); };

  // tiles touching the lattice boundary: halo cells outside the lattice hold
  // other rows / planes / columns of the flat view and are zeroed in shared
  // memory once the plane has landed (the Dirichlet elimination), so the
  // stencil body itself needs no masks
  const bool edge = x0 == 0 || x0 + kTX >= S || y0 == 0 || y0 + kTY >= S;
  auto zero_edges = [&](int s, int t) {
    const int ex0 = x0 == 0 ? 1 : 0, ex1 = x0 + kTX >= S ? 1 : 0;  // halo columns x = -1, x = S
    const int ey0 = y0 == 0 ? 1 : 0, ey1 = y0 + kTY >= S ? 1 : 0;  // halo rows y = -1, y = S
    const int ncolx = (ex0 + ex1) * (kTY + 2), nrowx = (ey0 + ey1) * (kTX + 2);
    const int per = ncolx + nrowx;
    for (int i = tid; i < CB * per; i += kNT) {
      const int j = i / per, q = i % per;
      int hy, x;
      if (q < ncolx) {
        hy = q % (kTY + 2);
        x = (ex0 && q < kTY + 2) ? -1 : S;
      } else {
        const int r = q - ncolx;
        hy = (ey0 && r < kTX + 2) ? 0 : S - y0 + 1;
        x = x0 - 1 + r % (kTX + 2);
      }
      const int sh = ((c0 + j + t + y0 - 1 + hy) & 1) ? 1 : 2;
      planes[(s * CB + j) * kFC + (hy & 1) * kFS + (hy >> 1) * kRW + (x - x0) + sh] = 0.0;
    }
  };
  // thread-constant parts of the three window rows' offsets (row y-1 and y+1
  // share a box; the parity shift of row y-1 alternates with the column)
  const int offm = (ty & 1) * kFS + (ty >> 1) * kRW + tx;
  const int off0 = ((ty + 1) & 1) * kFS + ((ty + 1) >> 1) * kRW + tx;
  // output row pointers of the CB columns (row z0 first), advanced a plane per completed row
  double* yrow[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j)
    yrow[j] = a.dst + static_cast<long long>(min(c0 + j, a.K - 1)) * a.ld + static_cast<long long>(z0) * S2 + own;

  for (int t = z0 - 1; t <= z1; ++t) {
    const int s = (t - z0 + 1) % NX;
    const int sc = (t - z0 + 1) % NC;
    mbar_wait(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    if (VAR) {
      mbar_wait(&barC[sc], (phC >> sc) & 1u);
      phC ^= 1u << sc;
    }
    const bool zin = t >= 0 && t < S;
    if (edge && zin) zero_edges(s, t);
    __syncthreads();  // slots of plane t-1 (read at step t-1) may be refilled; zeroed edges visible
    if (tid == 0) {
      if (t + NX - 1 <= z1) issue((t + NX - z0) % NX, t + NX - 1);
      if (VAR && t + NC - 1 <= z1) issue_c((t + NC - z0) % NC, t + NC - 1);
    }
    if (!inside) continue;
    const bool rowP = t - 1 >= z0;
    double wN[4], wC[7];
    if (VAR) {
      const double* Cp = coefs + sc * kSlots * kCR;
      wC[0] = Cp[1 * kCR + o0 - 1];        // slot 1 at (-1, 0)
      wC[1] = Cp[2 * kCR + o0 - kRW];      // slot 2 at (0, -1)
      wC[2] = Cp[3 * kCR + o0 - kRW - 1];  // slot 3 at (-1, -1)
#pragma unroll
      for (int i = 0; i < 4; ++i) wC[3 + i] = Cp[i * kCR + o0];  // own slots 0..3
      wN[0] = Cp[4 * kCR + o0];
      wN[1] = Cp[5 * kCR + o0 - 1];
      wN[2] = Cp[6 * kCR + o0 - kRW];
      wN[3] = Cp[7 * kCR + o0 - kRW - 1];
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) wN[i] = a.op.wc[4 + i];
#pragma unroll
      for (int i = 0; i < 3; ++i) wC[i] = a.op.wc[1 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i) wC[3 + i] = a.op.wc[i];
    }
    double wP[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) wP[i] = VAR ? cPp[i] : a.op.wc[4 + i];
    // window rows of column j: row y-1 / y+1 at Rm + j kFC, row y at R0 + j kFC,
    // with the parity shift alternating between even and odd columns
    const int par = (c0 + t + y0 - 1 + ty) & 1;  // parity of row y-1 in column c0
    const double* slot = planes + s * CB * kFC;
    const double* RmE = slot + offm + (par ? 1 : 2);
    const double* RmO = slot + offm + (par ? 2 : 1);
    const double* R0E = slot + off0 + (par ? 2 : 1);
    const double* R0O = slot + off0 + (par ? 1 : 2);
    auto body = [&](auto zin_t) {
      constexpr bool ZIN = decltype(zin_t)::value;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        double vmm = 0.0, v0m = 0.0, vm0 = 0.0, v00 = 0.0, vp0 = 0.0, v0p = 0.0, vpp = 0.0;
        if (ZIN) {
          const double* Rm = ((j & 1) ? RmO : RmE) + j * kFC;
          const double* R0 = ((j & 1) ? R0O : R0E) + j * kFC;
          vmm = Rm[-1];
          v0m = Rm[0];
          vm0 = R0[-1];
          v00 = R0[0];
          vp0 = R0[1];
          v0p = Rm[kRW];
          vpp = Rm[kRW + 1];
        }
        if (rowP) {  // Pp terms complete row t-1 (forward slots 4..7)
          double r = sC[j];
          r = madd(r, wP[0], v00);
          r = madd(r, wP[1], vp0);
          r = madd(r, wP[2], v0p);
          r = madd(r, wP[3], vpp);
          st_if(yrow[j], r, j < ncol);
        }
        // centre terms of row t (back 3..1, diagonal, forward 1..3), Pm terms of row t+1 (back 7..4)
        double c = sN[j];
        c = madd(c, wC[2], vmm);
        c = madd(c, wC[1], v0m);
        c = madd(c, wC[0], vm0);
        c = madd(c, wC[3], v00);
        c = madd(c, wC[4], vp0);
        c = madd(c, wC[5], v0p);
        c = madd(c, wC[6], vpp);
        double nx = madd(0.0, wN[3], vmm);  // +0 start as the CSR row sum (keeps the sign of zero)
        nx = madd(nx, wN[2], v0m);
        nx = madd(nx, wN[1], vm0);
        nx = madd(nx, wN[0], v00);
        sC[j] = c;
        sN[j] = nx;
      }
    };
    if (zin) body(std::true_type{});
    else body(std::false_type{});
    if (rowP) {
#pragma unroll
      for (int j = 0; j < CB; ++j) yrow[j] += S2;
    }
    if (VAR) {
      const double* Cp = coefs + sc * kSlots * kCR;
#pragma unroll
      for (int i = 0; i < 4; ++i) cPp[i] = Cp[(4 + i) * kCR + o0];
    }
  }
}

template <bool VAR, int CB, int NX = kNP, int NC = kNP>
void launch_k3f(const MarchArgs& a, const CUtensorMap& mx, const CUtensorMap& mc, cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = k3f_smem<VAR, CB, NX, NC>();
  static std::once_flag once;
  std::call_once(once, [] {
    PARO_CUDA(cudaFuncSetAttribute(k3f_kernel<VAR, CB, NX, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
  });
  dim3 grid(groups, a.nblk);
  k3f_kernel<VAR, CB, NX, NC><<<grid, kNT, sm, st>>>(a, mx, mc);
  PARO_CUDA(cudaGetLastError());
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    PARO_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (f == nullptr || q != cudaDriverEntryPointSuccess)
      throw ParoError(kCuda, "tma: cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 4-D map (x, y, z, column) of a row-padded buffer with box (bx, by, 1, bc)
void encode(CUtensorMap& m, const double* base, int S, long long ldi, int cols, int bx, int by, int bc = 1) {
  const int P = padded_row(S);
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(S),
                              static_cast<cuuint64_t>(cols)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(P) * 8, static_cast<cuuint64_t>(S) * P * 8,
                                 static_cast<cuuint64_t>(ldi) * 8};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(by), 1, static_cast<cuuint32_t>(bc)};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ParoError(kCuda, "tma: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
}

}  // namespace

void tma_plan(PcgTma& t, int S, long long ldi, int K, const double* r, const double* p0, const double* p1,
              const double* x, const double* invd, const double* coefp) {
  if ((ldi & 1) != 0) throw ParoError(kInvalidArgument, "tma: column stride must be even");
  encode(t.r_halo, r, S, ldi, K, kRW, kHY);
  encode(t.p0_halo, p0, S, ldi, K, kRW, kHY);
  encode(t.p1_halo, p1, S, ldi, K, kRW, kHY);
  encode(t.x_own, x, S, ldi, K, kTX, kTY);
  encode(t.x_halo, x, S, ldi, K, kRW, kHY);
  encode(t.r_own, r, S, ldi, K, kTX, kTY);
  if (invd) {
    encode(t.invd_halo, invd, S, ldi, 1, kRW, kHY);
    encode(t.invd_own, invd, S, ldi, 1, kTX, kTY);
  } else {
    t.invd_halo = t.invd_own = t.r_halo;
  }
  encode(t.r_fwd, r, S, ldi, K, kFW, 9);
  encode(t.p0_fwd, p0, S, ldi, K, kFW, 9);
  encode(t.p1_fwd, p1, S, ldi, K, kFW, 9);
  if (invd) encode(t.invd_fwd, invd, S, ldi, 1, kFW, 9);
  else t.invd_fwd = t.r_fwd;
  t.has_coef = coefp != nullptr;
  if (coefp) {  // the 8 slots at stride ldi
    encode(t.coef_box, coefp, S, ldi, kSlots, kRW, kTY + 1, kSlots);
    encode(t.coef_own, coefp, S, ldi, kSlots, kTX, kTY, kSlots);
  } else {
    t.coef_box = t.coef_own = t.r_halo;
  }
}

bool apply_flat_ok(bool var, const MarchArgs& a) {
  const int S = a.S;
  if ((S & 1) == 0 || a.ld != a.n || a.with_dot || a.op.mcoef != nullptr) return false;
  if (var && a.op.sigma != 0.0) return false;
  if ((reinterpret_cast<uintptr_t>(a.src) & 15) != 0) return false;
  const long long rows = static_cast<long long>(a.K) * S * S;  // lattice rows of all columns
  if (rows / 2 + 1 > (1ll << 31) - 1) return false;
  // an odd row count leaves the last lattice row in a half-filled view row:
  // it is read only if the allocation extends S doubles past the operand
  if ((rows & 1) != 0) {
    static PFN_cuMemGetAddressRange_v3020 range = [] {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q;
      PARO_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
      return q == cudaDriverEntryPointSuccess ? reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(f) : nullptr;
    }();
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range == nullptr || range(&base, &size, reinterpret_cast<CUdeviceptr>(a.src)) != CUDA_SUCCESS) return false;
    const uintptr_t need = reinterpret_cast<uintptr_t>(a.src + rows * S + S);
    if (need > static_cast<uintptr_t>(base) + size) return false;
  }
  return true;
}

void launch_apply_flat(bool var, int cb, const MarchArgs& a, const double* coefp, long long ldi, cudaStream_t st) {
  const int S = a.S;
  const long long rows = static_cast<long long>(a.K) * S * S;
  const long long vrows = (rows + 1) / 2;
  if (var && coefp == nullptr) throw ParoError(kInvalidArgument, "apply: padded coefficients missing");
  CUtensorMap mx, mc;
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * S), static_cast<cuuint64_t>(vrows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * S) * 8};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kRW), 5};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encoder()(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(a.src), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw ParoError(kCuda, "tma: flat view encode failed (" + std::to_string(r) + ")");
  }
  if (var) encode(mc, coefp, S, ldi, kSlots, kRW, kTY + 1, kSlots);
  else mc = mx;
  const int c = cb;
  if (var) {
    // 8 columns per CTA halve the coefficient-box traffic per point-column; the two CTAs of an
    // SM then fit with a 2-slot x ring (a step is twice as long, so one plane of lead covers
    // the x stream) and a 3-slot coefficient ring (two planes of lead: profiles/r02/APPLY_EXPERIMENTS.md)
    if (c == 1) launch_k3f<true, 1>(a, mx, mc, st);
    else if (c == 2) launch_k3f<true, 2>(a, mx, mc, st);
    else if (c >= 8) launch_k3f<true, 8, 2, 3>(a, mx, mc, st);
    else launch_k3f<true, 4>(a, mx, mc, st);
  } else {  // constant stencil: no coefficient ring, so the x ring runs a plane deeper (4.48 -> 4.17 ms at 257^3 x 76)
    if (c == 1) launch_k3f<false, 1, 4, 1>(a, mx, mc, st);
    else if (c == 2) launch_k3f<false, 2, 4, 1>(a, mx, mc, st);
    else launch_k3f<false, 4, 4, 1>(a, mx, mc, st);
  }
}

bool tma_k2c_active() { return true; }

void launch_tma_setup(int cb, const MarchArgs& a, const PcgTma& t, cudaStream_t st) {
  if (!t.has_coef) throw ParoError(kInvalidArgument, "tma setup: needs the padded coefficients");
  if (a.P != padded_row(a.S) || a.mwcoef != nullptr || a.rhs != nullptr)
    throw ParoError(kInvalidArgument, "tma setup: row-padded layout and a constant rhs mass required");
  Maps m;
  m.a = t.x_halo;
  m.b = t.coef_box;
  m.c = t.invd_own;
  const int c = cb;
  if (c == 1) launch_k0c<1>(a, m, st);
  else if (c == 2) launch_k0c<2>(a, m, st);
  else launch_k0c<4>(a, m, st);
}

void launch_tma(int mode, bool var, int cb, const MarchArgs& a, const PcgTma& t, bool p_is_p0, cudaStream_t st) {
  if (a.n > (1ll << 31) - 1) throw ParoError(kCapacity, "tma: more than 2^31 interior dofs per column");
  if (a.P != padded_row(a.S)) throw ParoError(kInvalidArgument, "tma: operands must use the row-padded layout");
  if (var && a.op.sigma != 0.0) throw ParoError(kInvalidArgument, "tma: shifted variable operator not preshifted");
  if (a.op.mcoef != nullptr) throw ParoError(kInvalidArgument, "tma: variable shift stencil unsupported");
  Maps m;
  if (mode == kK1) {
    const int c = cb;
    const CUtensorMap& po = p_is_p0 ? t.p0_fwd : t.p1_fwd;
    if (var) {
      if (c == 1) launch_k1f<true, 1>(a, t.r_fwd, po, t.invd_fwd, st);
      else if (c == 2) launch_k1f<true, 2>(a, t.r_fwd, po, t.invd_fwd, st);
      else launch_k1f<true, 4>(a, t.r_fwd, po, t.invd_fwd, st);
    } else {
      if (c == 1) launch_k1f<false, 1>(a, t.r_fwd, po, t.invd_fwd, st);
      else if (c == 2) launch_k1f<false, 2>(a, t.r_fwd, po, t.invd_fwd, st);
      else launch_k1f<false, 4>(a, t.r_fwd, po, t.invd_fwd, st);
    }
  } else if (mode == kK2) {
    m.a = p_is_p0 ? t.p0_halo : t.p1_halo;
    m.b = t.x_own;
    m.c = t.r_own;
    if (var && t.has_coef && tma_k2c_active()) {
      m.b = t.coef_box;
      m.c = t.invd_own;
      const int c = cb;
      if (c == 1) launch_k2c<1>(a, m, st);
      else if (c == 2) launch_k2c<2>(a, m, st);
      else launch_k2c<4>(a, m, st);
    } else if (a.xmode != 2) {
      throw ParoError(kInvalidArgument, "tma: deferred x updates need the k2c pass");
    } else if (var) launch_cb<kK2, true>(cb, a, m, st);
    else launch_cb<kK2, false>(cb, a, m, st);
  } else {
    throw ParoError(kInvalidArgument, "tma: mode must be K1 or K2");
  }
}

}  // namespace paro_b200
