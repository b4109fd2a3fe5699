// Small host<->device transfers that stay off the DMA copy engines.
//
// A caller that keeps its orbitals in host memory streams ~10 GB each way per
// outer iteration on a side stream (step_host). A cudaMemcpy of a few bytes on
// the compute stream (a column table, a scalar read-back) queues behind such a
// transfer on the copy engine and stalls the compute for its whole length, so
// the library moves its small operands through mapped pinned memory with a
// copy kernel instead: reads = kernel into the mapped buffer + stream sync;
// writes = host memcpy into a ring slot + kernel out of it (a slot is reused
// only after the event of its last kernel has completed).
#include <cstring>

#include "ctx.hpp"

namespace paro_b200 {

namespace {

__global__ void copy_words_kernel(const unsigned long long* __restrict__ src, unsigned long long* __restrict__ dst,
                                  long long nwords) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nwords;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}
__global__ void copy_bytes_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

void launch_copy(const void* src, void* dst, size_t bytes, cudaStream_t st) {
  const bool words = (reinterpret_cast<uintptr_t>(src) % 8 == 0) && (reinterpret_cast<uintptr_t>(dst) % 8 == 0) &&
                     bytes % 8 == 0;
  const long long n = static_cast<long long>(words ? bytes / 8 : bytes);
  const int blocks = static_cast<int>(std::min<long long>(64, (n + 255) / 256));
  if (words)
    copy_words_kernel<<<blocks, 256, 0, st>>>(static_cast<const unsigned long long*>(src),
                                              static_cast<unsigned long long*>(dst), n);
  else
    copy_bytes_kernel<<<blocks, 256, 0, st>>>(static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst),
                                              n);
  PARO_CUDA(cudaGetLastError());
}

}  // namespace

void small_d2h(Ctx& ctx, void* host, const void* dev, size_t bytes) {
  if (bytes == 0) return;
  auto& x = ctx.xfer;
  if (bytes > kXferSlot) {  // large: the ordinary copy
    PARO_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx.stream));
    PARO_CUDA(cudaStreamSynchronize(ctx.stream));
    return;
  }
  if (x.rd == nullptr) {
    PARO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&x.rd), kXferSlot, cudaHostAllocMapped));
    PARO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&x.rd_dev), x.rd, 0));
  }
  launch_copy(dev, x.rd_dev, bytes, ctx.stream);
  ++ctx.launches;
  PARO_CUDA(cudaStreamSynchronize(ctx.stream));
  std::memcpy(host, x.rd, bytes);
}

void small_h2d(Ctx& ctx, void* dev, const void* host, size_t bytes) {
  if (bytes == 0) return;
  auto& x = ctx.xfer;
  if (bytes > kXferSlot) {
    PARO_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx.stream));
    return;
  }
  if (x.wr == nullptr) {
    PARO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&x.wr), kXferSlot * kXferSlots, cudaHostAllocMapped));
    PARO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&x.wr_dev), x.wr, 0));
    for (int i = 0; i < kXferSlots; ++i) PARO_CUDA(cudaEventCreateWithFlags(&x.ev[i], cudaEventDisableTiming));
  }
  const int s = x.next;
  x.next = (x.next + 1) % kXferSlots;
  if (x.used[s]) PARO_CUDA(cudaEventSynchronize(x.ev[s]));  // its last kernel has read it
  std::memcpy(x.wr + static_cast<size_t>(s) * kXferSlot, host, bytes);
  launch_copy(x.wr_dev + static_cast<size_t>(s) * kXferSlot, dev, bytes, ctx.stream);
  ++ctx.launches;
  PARO_CUDA(cudaEventRecord(x.ev[s], ctx.stream));
  x.used[s] = true;
}

void xfer_release(Ctx& ctx) {
  auto& x = ctx.xfer;
  if (x.rd) cudaFreeHost(x.rd);
  if (x.wr) {
    for (int i = 0; i < kXferSlots; ++i) cudaEventDestroy(x.ev[i]);
    cudaFreeHost(x.wr);
  }
  x = {};
}

}  // namespace paro_b200
