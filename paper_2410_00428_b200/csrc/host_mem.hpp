// Pinned host memory on the GPU's own NUMA node (each GPU owns
// its pinned host region, NUMA-local, and its own copy streams).
//
// A rank's offload/prefetch traffic crosses its GPU's PCIe link into the
// socket that link hangs off; frames on the other socket add an
// inter-socket hop to every DMA. cudaHostAlloc places pages wherever the
// calling thread first touches them, so the pool is built by hand instead:
// an anonymous mapping, MPOL_PREFERRED on the GPU's node (spills instead of
// failing when the node is full), 2 MiB pages where the kernel allows them,
// a parallel first touch, then cudaHostRegister (mapped + portable: kernels
// and every device context address it through the same pointer).
#pragma once

#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace lkv {

// NUMA node of CUDA device `dev` from sysfs (-1: unknown / single node).
inline int gpu_numa_node(int dev) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  std::string id(bus);
  for (char& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  // sysfs uses a 4-hex-digit domain ("0000:1b:00.0"); CUDA may print 8 digits
  if (id.size() > 12 && id.compare(0, 4, "0000") == 0) id = id.substr(id.size() - 12);
  const std::string path = "/sys/bus/pci/devices/" + id + "/numa_node";
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (std::fscanf(f, "%d", &node) != 1) node = -1;
  std::fclose(f);
  return node;
}

class PinnedHost {
 public:
  PinnedHost() = default;
  PinnedHost(const PinnedHost&) = delete;
  PinnedHost& operator=(const PinnedHost&) = delete;
  ~PinnedHost() { release(); }

  // bytes > 0; node < 0 = no placement (first touch spread over the threads).
  void allocate(std::size_t bytes, int node, int threads) {
    release();
    bytes_ = bytes;
    int can = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&can, cudaDevAttrCanUseHostPointerForRegisteredMem, dev);
    if (!can) {  // registered pages would need a separate device pointer: plain pinned allocation
      legacy_ = true;
      check(cudaHostAlloc(reinterpret_cast<void**>(&p_), bytes, cudaHostAllocMapped | cudaHostAllocPortable),
            "cudaHostAlloc");
      return;
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) throw std::runtime_error("pinned host pool: mmap of " + std::to_string(bytes) + " B failed");
    p_ = static_cast<char*>(p);
    madvise(p_, bytes, MADV_HUGEPAGE);
    if (node >= 0 && node < 128) {
      unsigned long mask[2] = {0ul, 0ul};
      mask[node / 64] = 1ul << (node % 64);
      constexpr long kMpolPreferred = 1;
      node_bound_ = syscall(SYS_mbind, p_, bytes, kMpolPreferred, mask, 129ul, 0u) == 0;
    }
    node_ = node;
    // first touch in parallel: places the pages (and takes the zeroing off the pin)
    const std::size_t step = 2ull << 20;
    const std::size_t chunks = (bytes + step - 1) / step;
    const int t = static_cast<int>(std::clamp<std::size_t>(chunks / 64, 1, static_cast<std::size_t>(std::max(1, threads))));
    std::vector<std::thread> pool;
    for (int i = 0; i < t; ++i)
      pool.emplace_back([this, i, t, step, chunks, bytes] {
        for (std::size_t c = static_cast<std::size_t>(i); c < chunks; c += static_cast<std::size_t>(t)) {
          const std::size_t lo = c * step, n = std::min(step, bytes - lo);
          std::memset(p_ + lo, 0, n);
        }
      });
    for (auto& th : pool) th.join();
    check(cudaHostRegister(p_, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable), "cudaHostRegister");
    registered_ = true;
  }

  void release() {
    if (!p_) return;
    if (legacy_) {
      cudaFreeHost(p_);
    } else {
      if (registered_) cudaHostUnregister(p_);
      munmap(p_, bytes_);
    }
    p_ = nullptr;
    bytes_ = 0;
    registered_ = legacy_ = node_bound_ = false;
    node_ = -1;
  }

  char* data() const { return p_; }
  std::size_t bytes() const { return bytes_; }
  // Node the pages were bound to (-1: none requested or binding refused).
  int node() const { return node_bound_ ? node_ : -1; }

 private:
  static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("pinned host pool: ") + what + ": " + cudaGetErrorString(e));
  }
  char* p_ = nullptr;
  std::size_t bytes_ = 0;
  bool registered_ = false, legacy_ = false, node_bound_ = false;
  int node_ = -1;
};

}  // namespace lkv
