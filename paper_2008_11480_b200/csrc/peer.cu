// Peer-memory plumbing of the sharded path: stream memory
// operations used as cross-GPU flags.  The row panels of a gathered operand
// move by copy engines (cudaMemcpyAsync between IPC-mapped buffers over
// NVLink), so the exchange takes no SM away from the persistent DMMA GEMM it
// overlaps; the flags order the copies after the producing product on the
// owner GPU and gate the consuming product panel by panel (gemm_tma.cu).
#include "common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace si {
namespace {

using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

StreamValueFn entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<StreamValueFn>(p);
}

StreamValueFn write_fn() {
  static StreamValueFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] { fn = entry("cuStreamWriteValue32"); });
  return fn;
}

StreamValueFn wait_fn() {
  static StreamValueFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] { fn = entry("cuStreamWaitValue32"); });
  return fn;
}

}  // namespace

cudaError_t stream_write_u32(unsigned* addr, unsigned value, cudaStream_t s) {
  StreamValueFn fn = write_fn();
  if (!fn) {
    set_error("cuStreamWriteValue32 unavailable");
    return cudaErrorNotSupported;
  }
  // default flags: a memory barrier orders every prior write of the stream
  // (the panel copy / the producing kernel) before the flag
  const CUresult r = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value,
                        CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

cudaError_t stream_wait_u32(const unsigned* addr, unsigned value, cudaStream_t s) {
  StreamValueFn fn = wait_fn();
  if (!fn) {
    set_error("cuStreamWaitValue32 unavailable");
    return cudaErrorNotSupported;
  }
  const CUresult r = fn(reinterpret_cast<CUstream>(s),
                        reinterpret_cast<CUdeviceptr>(const_cast<unsigned*>(addr)), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

}  // namespace si
