// bc_ipc.cu -- peer-memory plumbing for the party-separated transport
// (paper_2309_04909_b200/peer.py): export a device buffer of this process as
// a CUDA IPC handle and map a peer process's buffer into this one.  With the
// parties on different GPUs of one NVSwitch node the mapping is a peer
// mapping: the phase kernels (bc_drelu_send, bc_relu_send_to, bc_drelu_helper,
// bc_relu_helper_to) then store their messages straight into the receiving
// party's HBM over NVLink, so compute and transfer are one kernel.
#include <cstring>

#include "bc_common.cuh"

using namespace bc::host;

namespace {
// CUresult cuMemGetAddressRange(CUdeviceptr* base, size_t* size, CUdeviceptr p), fetched from
// the driver at run time: the library links only the runtime (it must load on machines without
// a driver for the ABI tests).
typedef int (*MemRangeFn)(unsigned long long*, size_t*, unsigned long long);

MemRangeFn mem_range_fn() {
  static MemRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (MemRangeFn) nullptr;
    return reinterpret_cast<MemRangeFn>(f);
  }();
  return fn;
}
}  // namespace

extern "C" {

int bc_ipc_export(const void* dptr, uint8_t handle[64], uint64_t* offset) {
  if (!dptr || !handle || !offset) return BC_EINVAL;
  MemRangeFn range = mem_range_fn();
  if (!range) return cuda_rc(cudaErrorNotSupported);
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<unsigned long long>(dptr)) != 0) return cuda_rc(cudaErrorInvalidValue);
  cudaIpcMemHandle_t h;
  const int rc = cuda_rc(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  if (rc) return rc;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  *offset = reinterpret_cast<unsigned long long>(dptr) - base;
  return BC_OK;
}

int bc_ipc_open(const uint8_t handle[64], void** base) {
  if (!handle || !base) return BC_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  return cuda_rc(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
}

int bc_ipc_close(void* base) {
  if (!base) return BC_EINVAL;
  return cuda_rc(cudaIpcCloseMemHandle(base));
}

}  // extern "C"
