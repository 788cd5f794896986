// peer.cu -- NVLink peer-memory plumbing of the multi-GPU A exchange.
//
// the jc-sharded driver's one exchange step is getting A (m x k,
// owned by the root rank) onto every rank.  paper_1609_00076_b200/peer.py
// runs it as a copy-engine chain over NVLink instead of an NCCL broadcast:
// rank q pulls each k-chunk of A from rank q - 1's HBM with the DMA copy
// engines (cudaMemcpyAsync on an IPC-mapped peer pointer) as soon as rank
// q - 1 signals the chunk, and signals rank q + 1 in turn.  Copy engines use
// no SMs, so the chain overlaps the persistent GEMM (one CTA on every SM)
// without the SM contention an NCCL kernel has.
//
// Signals are stream memory operations (cuStreamWriteValue32 /
// cuStreamWaitValue32, executed by the GPU front end, not by a kernel) on
// 32-bit flags in device memory: a rank WRITES its neighbours' flags through
// peer mappings and WAITS only on its own flags.  The driver entry points are
// looked up through the runtime (cudaGetDriverEntryPointByVersion), so the
// library keeps no link-time dependency on libcuda.
//
// Buffers are exported with cudaIpcGetMemHandle on their allocation base plus
// an offset (PyTorch's caching allocator sub-allocates), and opened with
// lazy peer access.
#include <cuda.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/my_dgemm.h"
#include "common.cuh"

namespace myd {
int capi_fail(int status, const std::string &msg);
int capi_ok();
int capi_cuda_fail(cudaError_t e, const char *where);
}  // namespace myd

using namespace myd;

namespace {

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_addressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

struct Driver {
  PFN_waitValue32 wait32 = nullptr;
  PFN_writeValue32 write32 = nullptr;
  PFN_addressRange range = nullptr;
  cudaError_t err = cudaSuccess;
};

template <class F>
cudaError_t entry(const char *name, F *fn) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q);
  if (e == cudaSuccess && (q != cudaDriverEntryPointSuccess || p == nullptr)) e = cudaErrorSymbolNotFound;
  *fn = reinterpret_cast<F>(p);
  return e;
}

const Driver &driver() {
  static const Driver d = [] {
    Driver x;
    cudaError_t e;
    if ((e = entry("cuStreamWaitValue32", &x.wait32)) != cudaSuccess ||
        (e = entry("cuStreamWriteValue32", &x.write32)) != cudaSuccess ||
        (e = entry("cuMemGetAddressRange", &x.range)) != cudaSuccess)
      x.err = e;
    return x;
  }();
  return d;
}

int driver_fail(CUresult r, const char *where) {
  return capi_fail(1000 + (int)cudaErrorUnknown, std::string("CUDA driver error ") + std::to_string((int)r) + " in " + where);
}

}  // namespace

extern "C" {

int my_dgemm_ipc_export(const void *dev_ptr, unsigned char *handle_out, uint64_t *offset_out) {
  if (dev_ptr == nullptr) return capi_fail(-1, "dev_ptr must not be NULL");
  if (handle_out == nullptr || offset_out == nullptr) return capi_fail(-2, "output pointers must not be NULL");
  const Driver &d = driver();
  if (d.err != cudaSuccess) return capi_cuda_fail(d.err, "cudaGetDriverEntryPointByVersion");
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = d.range(&base, &size, (CUdeviceptr)(uintptr_t)dev_ptr);
  if (r != CUDA_SUCCESS) return driver_fail(r, "cuMemGetAddressRange (not a device allocation?)");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
  if (e != cudaSuccess) return capi_cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == MY_DGEMM_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof h);
  *offset_out = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return capi_ok();
}

int my_dgemm_ipc_open(const unsigned char *handle, uint64_t offset, void **dev_ptr_out) {
  if (handle == nullptr) return capi_fail(-1, "handle must not be NULL");
  if (dev_ptr_out == nullptr) return capi_fail(-3, "dev_ptr_out must not be NULL");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void *base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return capi_cuda_fail(e, "cudaIpcOpenMemHandle");
  *dev_ptr_out = static_cast<char *>(base) + offset;
  return capi_ok();
}

int my_dgemm_ipc_close(void *dev_ptr, uint64_t offset) {
  if (dev_ptr == nullptr) return capi_fail(-1, "dev_ptr must not be NULL");
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(dev_ptr) - offset);
  if (e != cudaSuccess) return capi_cuda_fail(e, "cudaIpcCloseMemHandle");
  return capi_ok();
}

int my_dgemm_signal_write(void *stream, uint32_t *dev_flag, uint32_t value) {
  if (dev_flag == nullptr || ((uintptr_t)dev_flag & 3)) return capi_fail(-2, "dev_flag must be a 4-byte aligned device address");
  const Driver &d = driver();
  if (d.err != cudaSuccess) return capi_cuda_fail(d.err, "cudaGetDriverEntryPointByVersion");
  // default flags: the write is ordered after (and flushes) the stream's earlier work
  CUresult r = d.write32((CUstream)stream, (CUdeviceptr)(uintptr_t)dev_flag, value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return driver_fail(r, "cuStreamWriteValue32");
  return capi_ok();
}

int my_dgemm_signal_wait_geq(void *stream, const uint32_t *dev_flag, uint32_t value) {
  if (dev_flag == nullptr || ((uintptr_t)dev_flag & 3)) return capi_fail(-2, "dev_flag must be a 4-byte aligned device address");
  const Driver &d = driver();
  if (d.err != cudaSuccess) return capi_cuda_fail(d.err, "cudaGetDriverEntryPointByVersion");
  // GEQ is the cyclic comparison (int32_t)(*flag - value) >= 0
  CUresult r = d.wait32((CUstream)stream, (CUdeviceptr)(uintptr_t)dev_flag, value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return driver_fail(r, "cuStreamWaitValue32");
  return capi_ok();
}

int my_dgemm_copy_async(void *dst, const void *src, uint64_t bytes, void *stream) {
  if (dst == nullptr) return capi_fail(-1, "dst must not be NULL");
  if (src == nullptr) return capi_fail(-2, "src must not be NULL");
  if (bytes == 0) return capi_ok();
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) return capi_cuda_fail(e, "cudaMemcpyAsync");
  return capi_ok();
}

}  // extern "C"
