// qgemm_ipc.cu -- peer-memory plumbing of the multi-GPU driver (include/qgemm.h,
// "Peer memory").
//
// The row-sharded QGEMM's collection step (every rank's C row block -> root's
// column-major C) is fused into the mainloop epilogue: each rank's epilogue
// stores its finished tiles straight into root's C over NVLink / NVSwitch, at
// row offset r0 with root's leading dimension, so the transfer overlaps the
// math tile by tile and no gather or relayout pass exists.  What the epilogue
// needs is root's C mapped into every rank's address space: a CUDA IPC handle
// of the allocation that holds it, plus the byte offset of C inside that
// allocation (allocators such as PyTorch's hand out interior pointers).
#include <atomic>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/qgemm.h"

namespace {

using AddressRangeFn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);

// cuMemGetAddressRange through the runtime's driver entry point, so that the
// library does not link libcuda (it must load on machines without a driver).
AddressRangeFn address_range() {
  static std::atomic<AddressRangeFn> fn{nullptr};  // (any host thread may make the first call)
  if (AddressRangeFn f = fn.load(std::memory_order_acquire)) return f;
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  fn.store(reinterpret_cast<AddressRangeFn>(p), std::memory_order_release);
  return reinterpret_cast<AddressRangeFn>(p);
}

}  // namespace

extern "C" {

int qgemm_ipc_handle(const void *dptr, unsigned char handle[64], uint64_t *offset, uint64_t *alloc_bytes) {
  if (dptr == nullptr) return -1;
  if (handle == nullptr) return -2;
  if (offset == nullptr) return -3;
  AddressRangeFn fn = address_range();
  if (!fn) return int(cudaErrorNotSupported);
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS) return int(cudaErrorInvalidValue);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
  if (e != cudaSuccess) return int(e);
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  *offset = uint64_t(reinterpret_cast<uintptr_t>(dptr) - uintptr_t(base));
  if (alloc_bytes) *alloc_bytes = uint64_t(size);
  return 0;
}

int qgemm_ipc_open(const unsigned char handle[64], uint64_t offset, void **dptr, void **base) {
  if (handle == nullptr) return -1;
  if (dptr == nullptr) return -3;
  if (base == nullptr) return -4;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void *b = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return int(e);
  *base = b;
  *dptr = static_cast<char *>(b) + offset;
  return 0;
}

int qgemm_ipc_close(void *base) {
  if (base == nullptr) return -1;
  return int(cudaIpcCloseMemHandle(base));
}

}  // extern "C"
