// Bulk-copy variant of the two fused Jacobi-PCG stencil passes (K1, K2).
//
// Same streaming row sums as stream_kernel (march.cu), but the halo'd planes
// are moved global -> shared by the TMA engine (cp.async.bulk, completion on
// an mbarrier per ring slot) instead of one 8-byte LDGSTS per point and
// column: one bulk copy per halo'd row and column, issued by one thread, so
// the warps spend their issue slots on the stencil. The operands live in the
// solver's padded buffers (16-byte aligned, even column stride, kBulkPad
// readable elements on both sides), so a row copy may start one element early
// to meet the 16-byte alignment and run a few elements past the row.
//
// Shared-memory layout of one (array, column) plane: row hy (halo row
// y0-1+hy) at hy*RS, element hx (x = x0-1+hx) at hy*RS + hx + b, with an odd
// row stride RS when the lattice row length S is odd. b is the parity of the
// global element index of (x0-1, y0-1) on that plane, so every row's 16-byte
// aligned global start lands on a 16-byte aligned shared address.
//
// Points outside the lattice must read as zero (Dirichlet elimination): rows
// outside it are never copied (K2 zeroes them once), planes outside it are
// zero-filled (K2) or skipped (K1), the x-halo columns of the edge tiles are
// zeroed after every landing (K2), and K1's transform writes 0 for every
// position outside the lattice.
#include <cstdlib>

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
__device__ __forceinline__ void bulk_copy(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

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

constexpr unsigned kHaloRowBytes = 36 * 8;  // covers hx = 0..33 from a 16-byte aligned start
constexpr unsigned kOwnRowBytes = 34 * 8;   // covers hx = 1..32

template <int RS>
constexpr int plane_stride() {
  return kHY * RS + 2;  // even: every (array, column) plane starts 16-byte aligned
}
template <int RS>
constexpr int own_stride() {
  return kTY * RS + 2;
}

template <int MODE, int CB, int RS>
constexpr size_t bulk_smem() {
  constexpr int CS = plane_stride<RS>();
  if (MODE == kK2) return sizeof(double) * (3ull * CB * CS + 3ull * 2 * CB * own_stride<RS>());
  return sizeof(double) * (3ull * (2 * CB + 1) * CS + 2ull * CB * kHP);
}

template <int MODE, bool VAR, int CB, int RS>
__global__ void __launch_bounds__(kNT, kMinCtas) bulk_kernel(const MarchArgs a) {
  static_assert(MODE == kK1 || MODE == kK2, "bulk_kernel: PCG passes only");
  static_assert(RS == 37 || RS == 38, "row stride");
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) unsigned long long bars[3];
  constexpr int NA = MODE == kK2 ? 2 : 1;
  constexpr int CS = plane_stride<RS>();
  constexpr int CO = own_stride<RS>();
  constexpr int NARR = MODE == kK1 ? 2 * CB + 1 : CB;  // halo'd arrays per plane group
  __shared__ double red[kNT / 32][CB * NA];

  double* planes = smem;                    // [3][NARR][CS]
  double* extra = planes + 3 * NARR * CS;   // K2: own-row stages [3][2][CB][CO]; K1: p_new ring [2][CB][kHP]

  const int S = a.S;
  const int S2 = S * S;
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
    const bool on = c < a.K && (a.cols == nullptr || a.cols[c].active != 0);
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
  const int own = gy * S + gx;

  // parity of the global index of (x0-1, y0-1) resp. (x0-1, y0) on plane 0
  const int bparH = ((y0 - 1) * S + x0 - 1) & 1;
  const int bparO = (y0 * S + x0 - 1) & 1;
  auto zpar = [&](int z) { return (z * S2) & 1; };

  int nrowH = 0, nrowO = 0;
  for (int hy = 0; hy < kHY; ++hy) nrowH += (y0 - 1 + hy >= 0 && y0 - 1 + hy < S);
  for (int r = 0; r < kTY; ++r) nrowO += (y0 + r < S);

  // this thread's bulk copy (at most one per step)
  constexpr int nH = NARR * kHY;
  constexpr int nO = MODE == kK2 ? 2 * CB * kTY : 0;
  bool cpH = false, cpO = false, cvalid = false;
  const double* csrc = nullptr;   // global element of the copy's anchor, plane 0
  int cdst = 0;                   // shared offset of the copy's row within its slot
  int cpar = 0;                   // parity of the anchor's in-plane index
  int cbpar = 0;                  // layout parity of its plane at z = 0
  if (tid < nH) {
    cpH = true;
    const int k = tid / kHY, hy = tid % kHY;
    const int y = y0 - 1 + hy;
    const bool yin = y >= 0 && y < S;
    const long long inpl = static_cast<long long>(y) * S + x0 - 1;
    if (MODE == kK2) {
      cvalid = yin && act(k);
      csrc = a.src + static_cast<long long>(c0 + k) * ld + inpl;
    } else {
      const int j = k % CB;
      if (k < CB) {
        cvalid = yin && act(j);
        csrc = a.r + static_cast<long long>(c0 + j) * ld + inpl;
      } else if (k < 2 * CB) {
        cvalid = yin && act(j) && !first(j);
        csrc = a.pold + static_cast<long long>(c0 + j) * ld + inpl;
      } else {
        cvalid = yin && VAR;
        csrc = VAR ? a.invd + inpl : a.r;
      }
    }
    cdst = k * CS + hy * RS;
    cpar = static_cast<int>(inpl & 1);
    cbpar = bparH;
  } else if (tid < nH + nO) {
    cpO = true;
    const int k = tid - nH;
    const int arr = k / (CB * kTY), j = (k / kTY) % CB, r = k % kTY;
    const int y = y0 + r;
    cvalid = y < S && act(j);
    const long long inpl = static_cast<long long>(y) * S + x0;
    csrc = (arr == 0 ? a.x : a.r) + static_cast<long long>(c0 + j) * ld + inpl;
    cdst = (arr * CB + j) * CO + r * RS + 1;
    cpar = static_cast<int>(inpl & 1);
    cbpar = bparO;
  }
  // ---- shared-memory initialisation and barriers
  if (MODE == kK2) {
    // rows outside the lattice stay zero for the whole kernel
    for (int i = tid; i < 3 * CB * CS; i += kNT) {
      const int hy = (i % CS) / RS;
      const int y = y0 - 1 + hy;
      if (hy >= kHY || y < 0 || y >= S) planes[i] = 0.0;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < 3; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  fence_async_smem();
  __syncthreads();

  auto slot_planes = [&](int s) { return planes + s * NARR * CS; };
  auto slot_own = [&](int s) { return extra + s * 2 * CB * CO; };
  // bytes landing in a group: halo'd plane z (if in the lattice) + own rows of row zo
  auto group_bytes = [&](int z, int zo) {
    unsigned bytes = 0;
    if (z >= 0 && z < S) {
      const int arrays = MODE == kK1 ? nact + nnf + (VAR ? 1 : 0) : nact;
      bytes += static_cast<unsigned>(nrowH * arrays) * kHaloRowBytes;
    }
    if (MODE == kK2 && zo >= z0 && zo < z1) bytes += static_cast<unsigned>(nrowO * 2 * nact) * kOwnRowBytes;
    return bytes;
  };
  // issue group s: halo'd plane z and (K2) own rows of row zo
  auto issue_group = [&](int s, int z, int zo) {
    const bool zin = z >= 0 && z < S;
    if (cpH && cvalid && zin) {
      const int zp = zpar(z);
      const int sh = cpar ^ zp, bb = cbpar ^ zp;
      bulk_copy(slot_planes(s) + cdst + bb - sh, csrc + static_cast<long long>(z) * S2 - sh, kHaloRowBytes, &bars[s]);
    }
    if (MODE == kK2) {
      if (cpO && cvalid && zo >= z0 && zo < z1) {
        const int zp = zpar(zo);
        const int sh = cpar ^ zp, bb = cbpar ^ zp;
        bulk_copy(slot_own(s) + cdst + bb - sh, csrc + static_cast<long long>(zo) * S2 - sh, kOwnRowBytes, &bars[s]);
      }
      if (!zin) {  // Dirichlet plane: zeros
        double* p = slot_planes(s);
        for (int i = tid; i < CB * CS; i += kNT) p[i] = 0.0;
      }
    }
  };

  // K2: zero the x-halo columns outside the lattice of a landed plane
  const bool xedge = x0 == 0 || x0 + kTX + 1 > S;
  const bool genw = xedge || z0 == 0 || z1 == S;  // this CTA stores zeros into bulk-copied slots
  auto fix_edges = [&](int s, int z) {
    if (!xedge || z < 0 || z >= S || tid >= CB * kHY) return;
    const int j = tid / kHY, hy = tid % kHY;
    double* row = slot_planes(s) + j * CS + hy * RS + (bparH ^ zpar(z));
    if (x0 == 0) row[0] = 0.0;
    for (int hx = S - x0 + 1; hx < kHX; ++hx) row[hx] = 0.0;
  };

  // K1: raw plane z (slot s) -> p_new = z + beta p_old into ring slot (z - z0 + 1) & 1; own points to global
  int pos[kLoadsPerThread], hoff[kLoadsPerThread];
  bool pval[kLoadsPerThread];
#pragma unroll
  for (int l = 0; l < kLoadsPerThread; ++l) {
    const int i = tid + l * kNT;
    pos[l] = i;
    const int hx = i % kHX, hy = i / kHX;
    const int px = x0 + hx - 1, py = y0 + hy - 1;
    pval[l] = i < kHP && px >= 0 && px < S && py >= 0 && py < S;
    hoff[l] = hy * RS + hx;
  }
  auto transform = [&](int s, int z) {
    const double* rw = slot_planes(s);
    double* ring = extra + ((z - z0 + 1) & 1) * CB * kHP;
    const bool zin = z >= 0 && z < S;
    const int b = bparH ^ zpar(z);
#pragma unroll
    for (int l = 0; l < kLoadsPerThread; ++l) {
      if (pos[l] >= kHP) continue;
      const bool v = zin && pval[l];
      const int h = hoff[l] + b;
      const double d = VAR ? rw[2 * CB * CS + h] : a.op.invd_const;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (!act(j)) continue;
        double p = 0.0;
        if (v) {
          // z = inv_diag * r ; p = z + beta * p   (linalg.cpp:179, 210)
          const double zz = __dmul_rn(d, rw[j * CS + h]);
          p = first(j) ? zz : __dadd_rn(zz, __dmul_rn(colB[j], rw[(CB + j) * CS + h]));
        }
        ring[j * kHP + pos[l]] = p;
      }
    }
  };

  // coefficient offsets (see stream_kernel)
  long long offB[kSlots], offF[kSlots];
#pragma unroll
  for (int o = 0; o < kSlots; ++o) {
    offF[o] = o * n;
    offB[o] = o * n - (o & 1) - ((o >> 1) & 1) * S;
  }
  const int ownc = inside ? own : 0;
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
      if (MODE == kK2) invdP = ldnc(a.invd + pm);
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
  unsigned phase = 0;  // bit s: parity of the next completion of bars[s]
  auto wait_slot = [&](int s) {
    mbar_wait(&bars[s], (phase >> s) & 1u);
    phase ^= 1u << s;
  };

  // ---- prologue
  if (MODE == kK1) {
    if (tid == 0) {
      mbar_arm(&bars[0], group_bytes(z0 - 1, -1));
      mbar_arm(&bars[1], group_bytes(z0, -1));
      mbar_arm(&bars[2], group_bytes(z0 + 1, -1));
    }
    __syncthreads();
    issue_group(0, z0 - 1, -1);
    issue_group(1, z0, -1);
    issue_group(2, z0 + 1, -1);
    wait_slot(0);
    transform(0, z0 - 1);
  } else {
    if (tid == 0) {
      mbar_arm(&bars[0], group_bytes(z0 - 1, -1));
      mbar_arm(&bars[1], group_bytes(z0, -1));
    }
    __syncthreads();
    issue_group(0, z0 - 1, -1);
    issue_group(1, z0, -1);
  }
  load_coefs(z0 - 1);

  const int ib = ty * kHX + tx;          // K1 ring (plain layout): top-left of the 3x3 window
  const int ibr = ty * RS + tx;          // K2 planes (parity layout)
  int s0 = 0;                            // slot of plane t; s1 = slot of t+1, s2 = slot of t+2 (= t-1)
  for (int t = z0 - 1; t <= z1; ++t, s0 = s0 == 2 ? 0 : s0 + 1) {
    const int s1 = s0 == 2 ? 0 : s0 + 1;
    const int s2 = s1 == 2 ? 0 : s1 + 1;
    const bool rowP = t - 1 >= z0;

    if (MODE == kK1) {
      if (t + 1 <= z1) wait_slot(s1);               // raw plane t+1 landed
      if (tid == 0 && t + 3 <= z1) mbar_arm(&bars[s0], group_bytes(t + 3, -1));
    } else {
      wait_slot(s0);                                 // plane t (and own rows of row t-1) landed
      fix_edges(s0, t);
      if (tid == 0 && t + 2 <= z1) mbar_arm(&bars[s2], group_bytes(t + 2, t + 1));
    }
    __syncthreads();
    // generic-proxy zero stores (K2 edge fixups, Dirichlet planes) must be
    // ordered before the bulk copies that overwrite the same slot
    if (MODE == kK2 && genw && (cpH || cpO)) fence_async_smem();
    if (MODE == kK1) {
      if (t + 3 <= z1) issue_group(s0, t + 3, -1);
    } else {
      if (t + 2 <= z1) issue_group(s2, t + 2, t + 1);
    }

    if (inside) {
      const double* P;
      int pb;
      if (MODE == kK1) {
        P = extra + ((t - z0 + 1) & 1) * CB * kHP;
        pb = ib;
      } else {
        P = slot_planes(s0);
        pb = ibr + (bparH ^ zpar(t));
      }
      constexpr int R = MODE == kK1 ? kHX : RS;
      const double* st = slot_own(s0);
      const long long pdst = static_cast<long long>(c0) * ld + static_cast<long long>(t) * S2 + own;
      const int bo = bparO ^ zpar(t - 1);
      const int so = ty * RS + tx + 1 + bo;
      // row t-1 of column c0 in x and r; the columns follow at stride ld
      double* xq = a.x + (pdst - S2);
      double* rq = a.r + (pdst - S2);
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (!act(j)) continue;
        const double* Pj = P + j * (MODE == kK1 ? kHP : CS) + pb;
        const double vmm = Pj[0], v0m = Pj[1], vm0 = Pj[R], v00 = Pj[R + 1];
        const double vp0 = Pj[R + 2], v0p = Pj[2 * R + 1], vpp = Pj[2 * R + 2];
        if (MODE == kK1 && t >= z0 && t < z1) a.dst[pdst + static_cast<long long>(j) * ld] = v00;  // p_new
        if (rowP) {  // Pp terms of row t-1: A[v, v+o], o = 4..7
          double s = sC[j];
          s = fma(cPp[0], v00, s);
          s = fma(cPp[1], vp0, s);
          s = fma(cPp[2], v0p, s);
          s = fma(cPp[3], vpp, s);
          const double ctr = cCur[j];
          if (MODE == kK1) {
            acc[j][0] += ctr * s;  // p'q
          } else {
            // x += alpha p ; r -= alpha q ; z = invd r  (linalg.cpp:202-206)
            const double al = colA[j];
            const double xn = __dadd_rn(st[j * CO + so], __dmul_rn(al, ctr));
            const double rn = __dsub_rn(st[(CB + j) * CO + so], __dmul_rn(al, s));
            xq[j * ld] = xn;
            rq[j * ld] = rn;
            const double zz = __dmul_rn(invdP, rn);
            acc[j][0] += rn * zz;
            acc[j][1] += rn * rn;
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
    if (MODE == kK1 && t + 1 <= z1) transform(s1, t + 1);
    if (t < z1) load_coefs(t + 1);
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


template <int MODE, bool VAR, int CB, int RS>
void launch_b(const MarchArgs& a, cudaStream_t st) {
  const int groups = (a.K + CB - 1) / CB;
  constexpr size_t sm = bulk_smem<MODE, CB, RS>();
  static bool configured = false;
  if (!configured) {
    PARO_CUDA(cudaFuncSetAttribute(bulk_kernel<MODE, VAR, CB, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
    configured = true;
  }
  dim3 grid(groups, a.nblk);
  bulk_kernel<MODE, VAR, CB, RS><<<grid, kNT, sm, st>>>(a);
  PARO_CUDA(cudaGetLastError());
}

template <int MODE, bool VAR, int CB>
void launch_rs(const MarchArgs& a, cudaStream_t st) {
  if (a.S & 1) launch_b<MODE, VAR, CB, 37>(a, st);
  else launch_b<MODE, VAR, CB, 38>(a, st);
}

template <int MODE, bool VAR>
void launch_cb(int cb, const MarchArgs& a, cudaStream_t st) {
  static const int forced = [] {
    const char* e = std::getenv("PARO_MARCH_CB");
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0 && cb > forced) cb = forced;
  switch (cb) {
    case 1: launch_rs<MODE, VAR, 1>(a, st); break;
    case 2: launch_rs<MODE, VAR, 2>(a, st); break;
    default: launch_rs<MODE, VAR, 4>(a, st); break;
  }
}

}  // namespace

void launch_bulk(int mode, bool var, int cb, const MarchArgs& a, cudaStream_t st) {
  if (a.n > (1ll << 31) - 1) throw ParoError(kCapacity, "bulk: more than 2^31 interior dofs per column");
  if ((a.ld & 1) != 0) throw ParoError(kInvalidArgument, "bulk: column stride must be even");
  if (var && a.op.sigma != 0.0) throw ParoError(kInvalidArgument, "bulk: shifted variable operator not preshifted");
  if (a.op.mcoef != nullptr) throw ParoError(kInvalidArgument, "bulk: variable shift stencil unsupported");
  if (mode == kK1) {
    if (var) launch_cb<kK1, true>(cb, a, st);
    else launch_cb<kK1, false>(cb, a, st);
  } else if (mode == kK2) {
    if (var) launch_cb<kK2, true>(cb, a, st);
    else launch_cb<kK2, false>(cb, a, st);
  } else {
    throw ParoError(kInvalidArgument, "bulk: mode must be K1 or K2");
  }
}

}  // namespace paro_b200
