// Device-side signalling for the peer-memory transport (dist.PeerTransport).
//
// The sequence-parallel runtime moves K/V, Q, partials and gradients between
// ranks with copy-engine pulls from the peer's HBM (CUDA IPC mappings over
// NVLink; no NCCL kernels, so no SMs are taken from the attention kernels).
// Ordering between ranks is carried by monotonically increasing 32-bit
// counters in device memory: a producer's stream bumps its own counter after
// the data is ready, the consumer's stream waits (in the stream, no host
// sync) until the producer's counter reaches the expected value. These are
// the driver's stream memory operations (cuStreamWriteValue32 /
// cuStreamWaitValue32), resolved through cudaGetDriverEntryPoint.
#include <cuda.h>
#include <cuda_runtime.h>

#include "capi_internal.h"

namespace da {
namespace {

using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename Fn>
Fn entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<Fn>(p);
}

WriteFn write_fn() {
  static WriteFn fn = entry<WriteFn>("cuStreamWriteValue32");
  return fn;
}

WaitFn wait_fn() {
  static WaitFn fn = entry<WaitFn>("cuStreamWaitValue32");
  return fn;
}

}  // namespace
}  // namespace da

extern "C" {

da_status da_stream_write_u32(void* stream, void* addr, uint32_t value) {
  auto fn = da::write_fn();
  if (fn == nullptr) return da::set_error(DA_ERR_UNSUPPORTED, "cuStreamWriteValue32 unavailable");
  const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr),
                        value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return da::set_error(DA_ERR_CUDA, "cuStreamWriteValue32 failed");
  return DA_OK;
}

da_status da_stream_wait_u32_geq(void* stream, const void* addr, uint32_t value) {
  auto fn = da::wait_fn();
  if (fn == nullptr) return da::set_error(DA_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
  const CUresult r =
      fn(reinterpret_cast<CUstream>(stream),
         reinterpret_cast<CUdeviceptr>(const_cast<void*>(addr)), value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return da::set_error(DA_ERR_CUDA, "cuStreamWaitValue32 failed");
  return DA_OK;
}

}  // extern "C"
