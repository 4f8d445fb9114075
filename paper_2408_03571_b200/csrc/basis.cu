// Krylov basis storage for the native GMRES: one contiguous [vectors][N] device
// array that grows without copying.
//
// The reference allocates V[(cap+1), N] eagerly (gmres.py:88-89): 67 GB at n=2049
// with a cap of 1000.  Here the workspace reserves virtual address space for the
// cap and backs it with physical memory in chunks as the iteration count grows
// (CUDA virtual memory management: cuMemAddressReserve / cuMemCreate / cuMemMap).
// The mapping persists in the workspace, so repeated solves pay for it once; no
// basis vector is ever copied, and the CGS2 kernels keep seeing a single array
// with leading dimension N.  Driver entry points come from cudaGetDriverEntryPoint,
// so the library does not link libcuda.
#include <cuda.h>

#include <cstring>
#include <utility>

#include "ops.cuh"

namespace helm {

namespace {
struct Drv {
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) vfree = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  decltype(&cuMemGetAllocationGranularity) gran = nullptr;
};

template <typename F> void get_entry(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  HELM_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
  HELM_CHECK(p != nullptr && q == cudaDriverEntryPointSuccess, std::string("driver entry point missing: ") + name);
  fn = reinterpret_cast<F>(p);
}

const Drv& drv() {
  static Drv d = [] {
    Drv x;
    get_entry("cuMemAddressReserve", x.reserve);
    get_entry("cuMemAddressFree", x.vfree);
    get_entry("cuMemCreate", x.create);
    get_entry("cuMemRelease", x.release);
    get_entry("cuMemMap", x.map);
    get_entry("cuMemUnmap", x.unmap);
    get_entry("cuMemSetAccess", x.access);
    get_entry("cuMemGetAllocationGranularity", x.gran);
    return x;
  }();
  return d;
}

#define HELM_CU(call)                                                                                     \
  do {                                                                                                    \
    CUresult r_ = (call);                                                                                 \
    if (r_ != CUDA_SUCCESS)                                                                               \
      throw ::helm::Error(std::string(#call) + " failed (CUresult " + std::to_string((int)r_) + ") @" +    \
                          __FILE__ + ":" + std::to_string(__LINE__));                                     \
  } while (0)

size_t round_up(size_t v, size_t g) { return (v + g - 1) / g * g; }
}  // namespace

struct KrylovBasis {
  int device = 0;
  size_t gran = 0;
  CUdeviceptr va = 0;
  size_t reserved = 0;
  size_t mapped = 0;
  std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> chunks;  // in mapping order

  CUmemAllocationProp prop() const {
    CUmemAllocationProp p;
    std::memset(&p, 0, sizeof(p));
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    return p;
  }
  void set_access(CUdeviceptr at, size_t bytes) const {
    CUmemAccessDesc a;
    std::memset(&a, 0, sizeof(a));
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = device;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    HELM_CU(drv().access(at, bytes, &a, 1));
  }
  void init() {
    if (gran) return;
    HELM_CUDA(cudaGetDevice(&device));
    CUmemAllocationProp p = prop();
    HELM_CU(drv().gran(&gran, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    if (gran < ((size_t)2 << 20)) gran = (size_t)2 << 20;
  }
  // make [0, need) usable; `reserve_hint` sizes a (re)reservation; `chunk_min` the next physical chunk
  void ensure(size_t need, size_t reserve_hint, size_t chunk_min, cudaStream_t st) {
    init();
    if (need > reserved) {
      const size_t nres = round_up(std::max(need, reserve_hint), gran);
      CUdeviceptr nva = 0;
      HELM_CU(drv().reserve(&nva, nres, gran, 0, 0));
      size_t off = 0;
      for (auto& c : chunks) {  // the same physical chunks, mapped at the new address: no copy
        HELM_CU(drv().map(nva + off, c.second, 0, c.first, 0));
        set_access(nva + off, c.second);
        off += c.second;
      }
      if (va) {
        HELM_CUDA(cudaStreamSynchronize(st));  // work queued on the old addresses must finish first
        HELM_CUDA(cudaDeviceSynchronize());
        unmap_all(va);
        HELM_CU(drv().vfree(va, reserved));
      }
      va = nva;
      reserved = nres;
    }
    if (need > mapped) {
      const size_t sz = round_up(std::max(need - mapped, chunk_min), gran);
      const size_t fit = std::min(sz, reserved - mapped);
      CUmemAllocationProp p = prop();
      CUmemGenericAllocationHandle h;
      HELM_CU(drv().create(&h, fit, &p, 0));
      HELM_CU(drv().map(va + mapped, fit, 0, h, 0));
      set_access(va + mapped, fit);
      chunks.emplace_back(h, fit);
      mapped += fit;
    }
  }
  void unmap_all(CUdeviceptr base) {
    size_t off = 0;
    for (auto& c : chunks) {
      HELM_CU(drv().unmap(base + off, c.second));
      off += c.second;
    }
  }
  void release() {
    if (va) {
      cudaDeviceSynchronize();
      try {
        unmap_all(va);
      } catch (...) {
      }
      drv().vfree(va, reserved);
    }
    for (auto& c : chunks) drv().release(c.first);
    chunks.clear();
    va = 0;
    reserved = mapped = 0;
  }
};

void* basis_ensure(helm_workspace* ws, size_t need, size_t reserve_hint, size_t chunk_min, cudaStream_t st) {
  if (!ws->basis) ws->basis = new KrylovBasis();
  KrylovBasis* b = static_cast<KrylovBasis*>(ws->basis);
  b->ensure(need, reserve_hint, chunk_min, st);
  return reinterpret_cast<void*>(b->va);
}

void basis_free(helm_workspace* ws) {
  if (!ws->basis) return;
  KrylovBasis* b = static_cast<KrylovBasis*>(ws->basis);
  b->release();
  delete b;
  ws->basis = nullptr;
}

}  // namespace helm
