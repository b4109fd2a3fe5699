// paro_b200 — shared device/host definitions for the ParO hot path on sm_100a.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace paro_b200 {

// Status codes of the C ABI (include/paro_b200.h). Each maps to one exception
// type of the reference (proj/include/paro/errors.hpp:9-80).
enum Status : int {
  kOk = 0,
  kError = 1,            // paro::Error (e.g. the Gram certificate, paro.cpp:171-174)
  kInvalidArgument = 2,  // paro::InvalidArgumentError
  kNotSpd = 3,           // paro::NotSpdError (linalg.cpp:165-167, 200)
  kIterationLimit = 4,   // paro::IterationLimitError(residual) (linalg.cpp:214-221)
  kDegenerateSpan = 5,   // paro::DegenerateSpanError (paro.cpp:128-131)
  kPencil = 6,           // paro::PencilError (linalg.cpp:315, 325-337)
  kEmptyBasis = 7,       // paro::EmptyBasisError (linalg.cpp:435-437)
  kCapacity = 8,         // paro::CapacityError
  kLineage = 9,          // paro::LineageError
  kCuda = 20,            // CUDA runtime / cuBLAS failure (no reference counterpart)
  kAborted = 21,         // column stopped because another column of the batch hit NotSpd
};

struct ParoError : std::runtime_error {
  int code;
  double residual;
  ParoError(int c, const std::string& m, double r = 0.0) : std::runtime_error(m), code(c), residual(r) {}
};

#define PARO_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      throw ::paro_b200::ParoError(::paro_b200::kCuda, std::string(#call ": ") + cudaGetErrorString(_e)); \
  } while (0)

// Stencil offset numbering: bit0 = +x, bit1 = +y, bit2 = +z. Slot 0 is the
// diagonal; slots 1..7 are the 7 "forward" edges of the Kuhn tetrahedra
// (all edge vectors of a Kuhn tet have non-negative components,
// proj/src/mesh.cpp:455-474). The backward weight A[v, v-o] is the forward
// weight stored at v-o (the operators are symmetric).
constexpr int kSlots = 8;

// Uniform-box geometry shared by every kernel. Interior vertices only:
// dof(i,j,k) = ((k*S + j)*S + i), 0 <= i,j,k < S = s-1 (x fastest), which is
// the reference dof order (mesh.cpp:425-427 vertex ids, fem.cpp:21-28 elimination).
struct Grid {
  int s = 0;         // subdivisions per axis
  int S = 0;         // interior points per axis
  long long n = 0;   // S^3
  double lo = 0.0;   // box lower corner (cubic box [lo, hi]^3)
  double hi = 0.0;
};

// Per-column CG state (mirrors the locals of cg_solve, linalg.cpp:143-223).
struct CgColumn {
  double bnorm;
  double rz;
  double pq;
  double alpha;
  double alpha_prev;  // alpha of the previous iteration (deferred x updates, tma.cu k2c)
  double beta;
  double rnorm;
  double tol;
  unsigned long long it;
  unsigned long long max_iter;
  int active;   // 1 while iterating
  int first;    // p = z on the first direction update
  int status;   // kOk / kNotSpd / kIterationLimit
  int converged;
};

}  // namespace paro_b200
