// fake_cuda.cpp -- TEST INFRASTRUCTURE ONLY: a host-memory stand-in for the
// CUDA runtime calls brng.cpp makes, so the C ABI's host logic (argument
// validation, cursor reservation, host-buffer chunking / staging, scratch
// growth) runs under AddressSanitizer + UndefinedBehaviorSanitizer in the
// CPU container (no GPU, no libcudart).
//
// "Device" memory is malloc'd and tracked, so cudaPointerGetAttributes can
// tell it from host memory; every async copy/memset runs immediately (stream
// order == program order, which is a valid schedule of the real streams).
// The kernel launches (brng_internal.h) are replaced by fake_kernels.cpp.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

namespace {
std::map<const char*, size_t>& allocs() {
  static std::map<const char*, size_t> m;
  return m;
}
std::mutex mu;
int g_device = 0;
size_t g_live_bytes = 0, g_peak_bytes = 0;
bool owned(const void* p) {
  std::lock_guard<std::mutex> l(mu);
  auto& m = allocs();
  auto it = m.upper_bound(static_cast<const char*>(p));
  if (it == m.begin()) return false;
  --it;
  return static_cast<const char*>(p) < it->first + it->second;
}
}  // namespace

extern "C" {

cudaError_t cudaGetDevice(int* d) { *d = g_device; return cudaSuccess; }
cudaError_t cudaSetDevice(int d) { g_device = d; return cudaSuccess; }
cudaError_t cudaDeviceGetAttribute(int* v, cudaDeviceAttr a, int) {
  *v = a == cudaDevAttrMultiProcessorCount ? 148 : 0;
  return cudaSuccess;
}
cudaError_t cudaMalloc(void** p, size_t n) {
  *p = std::malloc(n ? n : 1);
  if (!*p) return cudaErrorMemoryAllocation;
  std::lock_guard<std::mutex> l(mu);
  allocs()[static_cast<const char*>(*p)] = n ? n : 1;
  g_live_bytes += n;
  if (g_live_bytes > g_peak_bytes) g_peak_bytes = g_live_bytes;
  return cudaSuccess;
}
cudaError_t cudaFree(void* p) {
  if (!p) return cudaSuccess;
  {
    std::lock_guard<std::mutex> l(mu);
    auto it = allocs().find(static_cast<const char*>(p));
    if (it == allocs().end()) std::abort();                             // double / foreign free
    g_live_bytes -= it->second == 1 ? 0 : it->second;
    allocs().erase(it);
  }
  std::free(p);
  return cudaSuccess;
}
cudaError_t cudaMemset(void* p, int v, size_t n) { std::memset(p, v, n); return cudaSuccess; }
cudaError_t cudaMemsetAsync(void* p, int v, size_t n, cudaStream_t) {
  std::memset(p, v, n);
  return cudaSuccess;
}
cudaError_t cudaMemcpyAsync(void* d, const void* s, size_t n, cudaMemcpyKind, cudaStream_t) {
  std::memcpy(d, s, n);
  return cudaSuccess;
}
cudaError_t cudaMemcpy2DAsync(void* d, size_t dp, const void* s, size_t sp, size_t w, size_t h,
                              cudaMemcpyKind, cudaStream_t) {
  if (w > dp || w > sp) return cudaErrorInvalidPitchValue;
  for (size_t r = 0; r < h; ++r)
    std::memcpy(static_cast<char*>(d) + r * dp, static_cast<const char*>(s) + r * sp, w);
  return cudaSuccess;
}
cudaError_t cudaStreamCreateWithFlags(cudaStream_t* s, unsigned int) {
  *s = reinterpret_cast<cudaStream_t>(new int(0));
  return cudaSuccess;
}
cudaError_t cudaStreamDestroy(cudaStream_t s) { delete reinterpret_cast<int*>(s); return cudaSuccess; }
cudaError_t cudaStreamSynchronize(cudaStream_t) { return cudaSuccess; }
cudaError_t cudaStreamWaitEvent(cudaStream_t, cudaEvent_t, unsigned int) { return cudaSuccess; }
cudaError_t cudaStreamIsCapturing(cudaStream_t, cudaStreamCaptureStatus* c) {
  *c = cudaStreamCaptureStatusNone;
  return cudaSuccess;
}
cudaError_t cudaEventCreateWithFlags(cudaEvent_t* e, unsigned int) {
  *e = reinterpret_cast<cudaEvent_t>(new int(0));
  return cudaSuccess;
}
cudaError_t cudaEventRecord(cudaEvent_t, cudaStream_t) { return cudaSuccess; }
cudaError_t cudaEventDestroy(cudaEvent_t e) { delete reinterpret_cast<int*>(e); return cudaSuccess; }
cudaError_t cudaPointerGetAttributes(cudaPointerAttributes* a, const void* p) {
  std::memset(a, 0, sizeof(*a));
  a->type = owned(p) ? cudaMemoryTypeDevice : cudaMemoryTypeUnregistered;
  return cudaSuccess;
}
cudaError_t cudaGetLastError(void) { return cudaSuccess; }

}  // extern "C"

// live fake-device allocations (the driver checks for leaks after destroy)
size_t fake_cuda_live_allocs() {
  std::lock_guard<std::mutex> l(mu);
  return allocs().size();
}
bool fake_cuda_is_device(const void* p) { return owned(p); }
// peak fake-device bytes since the last reset
size_t fake_cuda_peak_bytes(bool reset) {
  std::lock_guard<std::mutex> l(mu);
  const size_t v = g_peak_bytes;
  if (reset) g_peak_bytes = g_live_bytes;
  return v;
}
