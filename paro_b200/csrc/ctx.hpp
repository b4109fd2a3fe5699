// Host-side context: device, stream, grid, operators and grow-only workspace.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.cuh"

namespace paro_b200 {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  template <typename T>
  T* get(size_t count) {
    const size_t need = count * sizeof(T);
    if (need > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      PARO_CUDA(cudaMalloc(&p, need));
      bytes = need;
    }
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// A stencil operator on the interior lattice. Constant operators (mass,
// Poisson/kinetic stiffness) carry their 8 weights; variable ones (the KS
// form, V_ext mass) own 8 SoA coefficient arrays of n doubles on the device.
struct Op {
  bool var = false;
  double w[kSlots] = {};
  double* coef = nullptr;
  long long n = 0;
  bool owns = false;
};

constexpr size_t kXferSlot = 64 * 1024;  // small-transfer staging (xfer.cu)
constexpr int kXferSlots = 32;

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  Grid grid;
  bool grid_set = false;
  std::string err;
  double resid = 0.0;
  unsigned long long launches = 0;   // kernels launched by this library (graph nodes counted)

  DevBuf partials, cols, scale, invd, pbuf0, pbuf1, flag;
  DevBuf ws_a, ws_b, ws_c, ws_d, ws_e, ws_small, ws_small2, ws_small3;
  bool force_cgs2 = false;           // Step 4: skip the Cholesky-QR path
  bool two_pass_only = false;        // Step 4: always form the intermediate basis (no one-pass basis change)
  struct {                           // one-shot host copy-out of the next Ritz orbitals
    cudaStream_t stream = nullptr;
    double* host = nullptr;
    long long ldh = 0;
    int c0 = 0, c1 = 0;
    cudaEvent_t ready = nullptr;
  } ritz_copyout;
  int hartree_mode = 1;              // 0: Jacobi-PCG (reference algorithm), 1: DST-I when applicable
  int dst_S = 0;                     // grid of the cached DST-I tables
  DevBuf dst_tab;
  DevBuf wtab;                       // assembly: per-(cell, tet, point) weight values
  DevBuf ws_gram;                    // split-K partial Grams
  DevBuf pcg_x;                      // PCG iterate in the padded solver layout
  DevBuf shifted;                    // (A + sigma M) coefficients of the current shifted solve
  DevBuf coefp;                      // the same in the row-padded layout (TMA staging in the PCG passes)
  DevBuf csr_ws, csr_ws2, csr_io;    // general-CSR solver: interleaved work vectors, retry iterate, rhs/x
  struct {                           // mapped pinned staging of the small transfers (xfer.cu)
    unsigned char* rd = nullptr;
    unsigned char* rd_dev = nullptr;
    unsigned char* wr = nullptr;
    unsigned char* wr_dev = nullptr;
    cudaEvent_t ev[kXferSlots] = {};
    bool used[kXferSlots] = {};
    int next = 0;
  } xfer;
  int* pinned_count = nullptr;       // mapped host memory for the active-column poll
  int* pinned_count_dev = nullptr;

  // live accounting of the PCG iteration loops (CUDA-event time on the
  // context stream, algorithmic bytes n*(88 k + 64) per iteration)
  // [0] var-op seconds [1] var-op bytes [2] var-op column-iterations
  // [3] const-op seconds [4] const-op bytes [5] const-op column-iterations
  double stats[8] = {};

  double mass_w[kSlots] = {};        // the P1 mass stencil of this grid when it is constant (fields.cu)
  bool nodal_sums = true;            // integrate / norm_l2 / integrate_product as nodal sums when the mass is constant
  int mass_state = 0;                // 0: mass not assembled yet, 1: constant (mass_w valid), 2: varies per dof

  void check_grid() const {
    if (!grid_set) throw ParoError(kInvalidArgument, "paro_b200: grid not initialised");
  }
};

// small operands host<->device through mapped pinned memory (no copy engine, xfer.cu)
void small_d2h(Ctx& ctx, void* host, const void* dev, size_t bytes);  // synchronises ctx.stream
void small_h2d(Ctx& ctx, void* dev, const void* host, size_t bytes);  // stream-ordered on ctx.stream
void xfer_release(Ctx& ctx);

}  // namespace paro_b200
