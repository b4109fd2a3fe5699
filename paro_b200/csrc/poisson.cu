// Fast Hartree solve: exact discrete solution of K V = 4 pi M rho by the 3-D
// DST-I when K is the constant 7-point stencil (the P1/Kuhn Poisson stiffness
// on a uniform box has exactly zero face/body-diagonal entries).
//
// The reference solves the same system with cold-start Jacobi-PCG to a
// relative residual of 1e-11 (hartree_solve_with, model.cpp:242-255); that
// iterate is within ~1e-12 (relative) of the exact solution returned here, far
// inside the 1e-8 eigenvalue / energy parity bar. CG remains the parity mode.
//
// With S = s-1 interior points per axis and x fastest, the DST-I along one
// axis multiplies every line along that axis by T[i][j] = sin(pi (i+1)(j+1)/s).
// T[i][S-1-j] = (-1)^i T[i][j], so folding the line first (e_j = x_j + x_{S-1-j},
// o_j = x_j - x_{S-1-j}, the middle entry kept in e) leaves two half-size
// products: even outputs T_e e, odd outputs T_o o (half the flops of the dense
// S x S product). dst_rows_kernel runs them as FP64 tensor-core (DMMA) GEMMs
// over lines along a strided axis (z: stride S^2; y: stride S within each
// z-slab); the contiguous x axis is brought to a strided position by a tiled
// transpose and back. The inverse is (2/s)^3 times the forward transform; the
// diagonal in the DST basis is w0 + 2 wx cos(pi j/s) + 2 wy cos(pi k/s) + 2 wz cos(pi l/s).
#include <algorithm>
#include <cmath>
#include <vector>

#include "dmma.cuh"
#include "poisson.hpp"
#include "solver.hpp"

namespace paro_b200 {

namespace {

__global__ void scale_kernel(double* v, long long n, double s) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    v[i] *= s;
}

__global__ void spectral_divide_kernel(double* v, int S, const double* cosv, double w0, double wx, double wy,
                                       double wz, double post) {
  const long long n = static_cast<long long>(S) * S * S;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(i % S), y = static_cast<int>((i / S) % S), z = static_cast<int>(i / (static_cast<long long>(S) * S));
    const double lam = w0 + 2.0 * (wx * cosv[x] + wy * cosv[y] + wz * cosv[z]);
    v[i] = v[i] * (post / lam);
  }
}

constexpr int kDM = 128;  // output rows (half-size m) per CTA
constexpr int kDN = 64;   // line positions r per CTA
constexpr int kDK = 32;   // folded inputs k per staged chunk
constexpr int kDAS = kDM + 8;
constexpr int kDBS = kDN + 8;
constexpr size_t kDSmem = sizeof(double) * 2 * kDK * (kDAS + kDBS);

// Z[i][r] = sum_j T[i][j] X[j][r] for the lines X[.][r] along an axis with row
// stride ldb (Z in the same layout), r < N, per slab (blockIdx.y, stride
// sstride); blockIdx.z = 2 * m-block + parity. tab: [2][KP][MP] the folded
// half tables Tp[k][m] = T[2m+p][k] (zero padded), KP = MP.
__global__ void __launch_bounds__(256, 2)
    dst_rows_kernel(const double* __restrict__ X, double* __restrict__ Z, const double* __restrict__ tab, int S,
                    int MP, long long N, long long ldb, long long sstride, int He, int Ho) {
  extern __shared__ __align__(16) double dsm[];
  auto As = reinterpret_cast<double(*)[kDK][kDAS]>(dsm);
  auto Bs = reinterpret_cast<double(*)[kDK][kDBS]>(dsm + 2 * kDK * kDAS);
  const int p = blockIdx.z & 1, m0 = (blockIdx.z >> 1) * kDM;
  const int Hp = p ? Ho : He;
  if (m0 >= Hp) return;
  const double* xs = X + blockIdx.y * sstride;
  double* zs = Z + blockIdx.y * sstride;
  const long long r0 = static_cast<long long>(blockIdx.x) * kDN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int fr = lane & 3, fc = lane >> 2;
  const int wm = warp & 3, wn = warp >> 2;
  const double* tp = tab + static_cast<long long>(p) * MP * MP + m0;
  const int nchunks = (Hp + kDK - 1) / kDK;

  auto stage_a = [&](int buf, int k0) {  // 32 k-rows x 128 m of the folded table, 16-byte cp.async
    for (int q = tid; q < kDK * (kDM / 2); q += 256) {
      const int kk = q / (kDM / 2), mm = 2 * (q % (kDM / 2));
      const double* src = tp + static_cast<long long>(k0 + kk) * MP + mm;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(
                       __cvta_generic_to_shared(&As[buf][kk][mm]))),
                   "l"(src)
                   : "memory");
    }
    cp_async_commit();
  };
  double breg[8];
  const int br = tid % kDN, bk = tid / kDN;  // thread's column and first k-row (+4 q)
  auto load_b = [&](int k0) {                // the folded line values (x_k +- x_{S-1-k})
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = k0 + bk + 4 * q;
      const long long r = r0 + br;
      double v = 0.0;
      if (k < Hp && r < N) {
        const double a = xs[k * ldb + r];
        const int j2 = S - 1 - k;
        if (j2 != k) {
          const double b = xs[j2 * ldb + r];
          v = p ? a - b : a + b;
        } else {
          v = a;  // the middle line (even part only)
        }
      }
      breg[q] = v;
    }
  };
  auto store_b = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) Bs[buf][bk + 4 * q][br] = breg[q];
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  stage_a(0, 0);
  load_b(0);
  store_b(0);
  cp_async_wait<0>();
  __syncthreads();
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    const bool more = c + 1 < nchunks;
    if (more) {
      stage_a(buf ^ 1, (c + 1) * kDK);
      load_b((c + 1) * kDK);
    }
#pragma unroll
    for (int ks = 0; ks < kDK / 4; ++ks) {
      double a[4], b[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = As[buf][4 * ks + fr][wm * 32 + mt * 8 + fc];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b[nt] = Bs[buf][4 * ks + fr][wn * 32 + nt * 8 + fc];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
    if (more) {
      store_b(buf ^ 1);
      cp_async_wait<0>();
    }
    __syncthreads();
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int m = m0 + wm * 32 + mt * 8 + fc;
    if (m >= Hp) continue;
    double* zrow = zs + static_cast<long long>(2 * m + p) * ldb;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const long long r = r0 + wn * 32 + nt * 8 + 2 * fr + j;
        if (r < N) zrow[r] = acc[mt][nt][j];
      }
  }
}

// out (C x R) = in (R x C)^T, 32 x 32 tiles through shared memory
__global__ void transpose_kernel(const double* __restrict__ in, double* __restrict__ out, long long R, long long C) {
  __shared__ double t[32][33];
  const long long c0 = static_cast<long long>(blockIdx.x) * 32, r0 = static_cast<long long>(blockIdx.y) * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long r = r0 + j, c = c0 + threadIdx.x;
    if (r < R && c < C) t[j][threadIdx.x] = in[r * C + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long c = c0 + j, r = r0 + threadIdx.x;
    if (r < R && c < C) out[c * R + r] = t[threadIdx.x][j];
  }
}

struct DstPlan {
  int S, s, MP, He, Ho;
  const double* tab;
};

void dst_axis(Ctx& ctx, const DstPlan& d, const double* in, double* out, long long N, long long ldb, int slabs,
              long long sstride) {
  static bool configured = false;
  if (!configured) {
    PARO_CUDA(cudaFuncSetAttribute(dst_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kDSmem)));
    configured = true;
  }
  dim3 grid(static_cast<unsigned>((N + kDN - 1) / kDN), slabs, 2 * (d.MP / kDM));
  dst_rows_kernel<<<grid, 256, kDSmem, ctx.stream>>>(in, out, d.tab, d.S, d.MP, N, ldb, sstride, d.He, d.Ho);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

void transpose(Ctx& ctx, const double* in, double* out, long long R, long long C) {
  dim3 grid(static_cast<unsigned>((C + 31) / 32), static_cast<unsigned>((R + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, ctx.stream>>>(in, out, R, C);
  PARO_CUDA(cudaGetLastError());
  ++ctx.launches;
}

// v <- DST_x DST_y DST_z v (t1, t2: scratch of n doubles each)
void dst3(Ctx& ctx, const DstPlan& d, double* v, double* t1, double* t2) {
  const long long S = d.S, S2 = S * S;
  dst_axis(ctx, d, v, t1, S2, S2, 1, 0);     // z: lines of stride S^2 -> t1 [z'][y][x]
  dst_axis(ctx, d, t1, t2, S, S, d.S, S2);   // y: per z'-slab, stride S -> t2 [z'][y'][x]
  transpose(ctx, t2, t1, S2, S);             // t1 [x][z' y']
  dst_axis(ctx, d, t1, t2, S2, S2, 1, 0);    // x: stride S^2 -> t2 [x'][z' y']
  transpose(ctx, t2, v, S, S2);              // v [z'][y'][x']
}

}  // namespace

bool dst_applicable(const Op& k) {
  return !k.var && k.w[3] == 0.0 && k.w[5] == 0.0 && k.w[6] == 0.0 && k.w[7] == 0.0 && k.w[0] > 0.0;
}

int hartree_dst(Ctx& ctx, const Op& poisson, const Op& mass, const double* rho, double* vh) {
  ctx.check_grid();
  if (!dst_applicable(poisson)) throw ParoError(kInvalidArgument, "hartree dst: not a constant 7-point stencil");
  const int S = ctx.grid.S, s = ctx.grid.s;
  const long long n = ctx.grid.n;
  cudaStream_t st = ctx.stream;
  const int He = (S + 1) / 2, Ho = S / 2;
  const int MP = (He + kDM - 1) / kDM * kDM;
  // folded half tables Tp[k][m] = sin(pi (2m+p+1)(k+1)/s) and the cosines (host, libm), cached per grid
  if (ctx.dst_S != S) {
    std::vector<double> tab(2 * static_cast<size_t>(MP) * MP, 0.0), cs(S);
    for (int p = 0; p < 2; ++p) {
      const int H = p ? Ho : He;
      for (int k = 0; k < H; ++k)
        for (int m = 0; m < H; ++m)
          tab[(static_cast<size_t>(p) * MP + k) * MP + m] = std::sin(M_PI * (2.0 * m + p + 1.0) * (k + 1.0) / s);
    }
    for (int j = 0; j < S; ++j) cs[j] = std::cos(M_PI * (j + 1) / s);
    double* d = ctx.dst_tab.get<double>(tab.size() + S);
    PARO_CUDA(cudaMemcpy(d, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
    PARO_CUDA(cudaMemcpy(d + tab.size(), cs.data(), sizeof(double) * S, cudaMemcpyHostToDevice));
    ctx.dst_S = S;
  }
  const DstPlan plan{S, s, MP, He, Ho, static_cast<double*>(ctx.dst_tab.p)};
  const double* cosv = plan.tab + 2 * static_cast<size_t>(MP) * MP;
  double* t1 = ctx.ws_e.get<double>(2 * static_cast<size_t>(n));
  double* t2 = t1 + n;
  // rhs = (M rho) * 4 pi (model.cpp:248-249) into vh
  apply_op(ctx, mass, nullptr, 0.0, 1, rho, n, vh, n);
  const int blocks = static_cast<int>(std::min<long long>(148 * 8, (n + 255) / 256));
  scale_kernel<<<blocks, 256, 0, st>>>(vh, n, 4.0 * M_PI);
  dst3(ctx, plan, vh, t1, t2);
  const double post = std::pow(2.0 / s, 3);
  spectral_divide_kernel<<<blocks, 256, 0, st>>>(vh, S, cosv, poisson.w[0], poisson.w[1], poisson.w[2], poisson.w[4],
                                                 post);
  dst3(ctx, plan, vh, t1, t2);
  ctx.launches += 2;
  PARO_CUDA(cudaGetLastError());
  return kOk;
}

}  // namespace paro_b200
