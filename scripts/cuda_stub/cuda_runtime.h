// Host-only stand-in for the few CUDA runtime calls host_tier.hpp and
// host_mem.hpp make, so the tier's real locking code can run under TSan /
// ASan without a GPU (scripts/tier_stress.cpp). Not product code.
// An event is a host object completed by the stress test's simulated copy
// engine; destroying it while work is pending defers the free (as CUDA does).
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdlib>
#include <mutex>

typedef int cudaError_t;
enum : int { cudaSuccess = 0, cudaErrorNotReady = 600, cudaErrorInvalidValue = 1 };
enum cudaDeviceAttr { cudaDevAttrCanUseHostPointerForRegisteredMem = 91 };
enum : unsigned { cudaHostRegisterPortable = 1, cudaHostRegisterMapped = 2, cudaHostAllocPortable = 1,
                  cudaHostAllocMapped = 2 };

struct CUevent_st {
  std::mutex m;
  std::condition_variable cv;
  bool done = false;
  std::atomic<int> refs{1};
};
typedef CUevent_st* cudaEvent_t;

inline void stub_event_release(cudaEvent_t e) {
  if (e && e->refs.fetch_sub(1) == 1) delete e;
}
inline cudaEvent_t stub_event_new() { return new CUevent_st(); }
inline void stub_event_retain(cudaEvent_t e) { e->refs.fetch_add(1); }
inline void stub_event_complete(cudaEvent_t e) {
  {
    std::lock_guard<std::mutex> g(e->m);
    e->done = true;
  }
  e->cv.notify_all();
}

inline const char* cudaGetErrorString(cudaError_t) { return "stub error"; }
inline cudaError_t cudaGetLastError() { return cudaSuccess; }
inline cudaError_t cudaSetDevice(int) { return cudaSuccess; }
inline cudaError_t cudaGetDevice(int* d) { *d = 0; return cudaSuccess; }
inline cudaError_t cudaDeviceGetAttribute(int* v, cudaDeviceAttr, int) { *v = 1; return cudaSuccess; }
inline cudaError_t cudaDeviceGetPCIBusId(char*, int, int) { return cudaErrorInvalidValue; }
inline cudaError_t cudaHostRegister(void*, size_t, unsigned) { return cudaSuccess; }
inline cudaError_t cudaHostUnregister(void*) { return cudaSuccess; }
inline cudaError_t cudaHostAlloc(void** p, size_t n, unsigned) { *p = std::malloc(n); return *p ? cudaSuccess : 2; }
inline cudaError_t cudaFreeHost(void* p) { std::free(p); return cudaSuccess; }
inline cudaError_t cudaEventSynchronize(cudaEvent_t e) {
  std::unique_lock<std::mutex> g(e->m);
  e->cv.wait(g, [&] { return e->done; });
  return cudaSuccess;
}
inline cudaError_t cudaEventQuery(cudaEvent_t e) {
  std::lock_guard<std::mutex> g(e->m);
  return e->done ? cudaSuccess : cudaErrorNotReady;
}
inline cudaError_t cudaEventDestroy(cudaEvent_t e) { stub_event_release(e); return cudaSuccess; }
