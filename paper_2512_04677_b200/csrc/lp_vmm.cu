// Growable KV arenas on CUDA virtual memory (lp_vmm_*).
//
// The drop-in denoiser (B200Denoiser, the reference's Runtime.denoiser plug
// point, engine.py:166-200) cannot know up front how many cache entries its
// caller keeps alive: the reference engine holds T*L entries in its
// RollingKvCache objects (kvcache.py:29-59), TPP adds one in-flight entry
// per stage thread (engine.py:431-463), and a corrupted view
// (kvcache.py:121-137) or a host-typed entry needs temporary device copies.
// Every attention launch addresses the whole view as row segments of ONE
// base per layer, so the arena must stay one address range while it grows.
//
// lp_vmm reserves a virtual range of n_layers * layer_stride bytes once and
// backs the first `mapped` bytes of every layer with physical HBM on demand
// (cuMemCreate + cuMemMap).  Growth never moves data: pointers held by
// in-flight launches and captured descriptors stay valid, and nothing is
// copied.  At the 14B shape a slot (one block's K of all 40 layers) is
// 1.9 GB, so sizing from the live entry count instead of a fixed worst case
// is what lets the drop-in fit in 180 GB.
//
// The driver API is reached through cudaGetDriverEntryPoint, so the library
// keeps no link-time dependency on libcuda (it still loads on a CPU-only
// host for the ABI checks).
#include <cuda.h>

#include <mutex>
#include <vector>

#include "lp_common.cuh"

namespace {

using PFN_getGran = CUresult (*)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
using PFN_reserve = CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
using PFN_free = CUresult (*)(CUdeviceptr, size_t);
using PFN_create = CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                                unsigned long long);
using PFN_release = CUresult (*)(CUmemGenericAllocationHandle);
using PFN_map = CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
using PFN_unmap = CUresult (*)(CUdeviceptr, size_t);
using PFN_access = CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);

struct Driver {
  PFN_getGran gran = nullptr;
  PFN_reserve reserve = nullptr;
  PFN_free vfree = nullptr;
  PFN_create create = nullptr;
  PFN_release release = nullptr;
  PFN_map map = nullptr;
  PFN_unmap unmap = nullptr;
  PFN_access access = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  *fn = reinterpret_cast<F>(p);
  return p != nullptr;
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuMemGetAllocationGranularity", &d.gran) && entry("cuMemAddressReserve", &d.reserve) &&
           entry("cuMemAddressFree", &d.vfree) && entry("cuMemCreate", &d.create) &&
           entry("cuMemRelease", &d.release) && entry("cuMemMap", &d.map) && entry("cuMemUnmap", &d.unmap) &&
           entry("cuMemSetAccess", &d.access);
  });
  return d;
}

}  // namespace

struct lp_vmm {
  int device = 0;
  int n_layers = 0;
  CUdeviceptr base = 0;
  size_t gran = 0;
  size_t layer_stride = 0;  // reserved bytes per layer (multiple of gran)
  size_t mapped = 0;        // backed bytes at the start of every layer
  struct Piece {
    CUdeviceptr va;
    size_t bytes;
    CUmemGenericAllocationHandle h;
  };
  std::vector<Piece> pieces;
  std::mutex mu;
};

#define LP_CU_TRY(expr)                                                                       \
  do {                                                                                        \
    CUresult _r = (expr);                                                                     \
    if (_r != CUDA_SUCCESS) return ::lp::fail(LP_ECUDA, std::string(#expr) + " failed (CUresult " + \
                                                                std::to_string((int)_r) + ")"); \
  } while (0)

static CUmemAllocationProp pinned_prop(int device) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  return p;
}

extern "C" {

int lp_vmm_create(int device, int n_layers, int64_t layer_bytes_max, lp_vmm** out) {
  LP_CHECK_ARG(out && n_layers > 0 && layer_bytes_max > 0, "lp_vmm_create: bad argument");
  const Driver& d = driver();
  if (!d.ok) return lp::fail(LP_EUNSUPPORTED, "lp_vmm_create: CUDA virtual-memory driver entry points missing");
  LP_CUDA_TRY(cudaSetDevice(device));
  CUmemAllocationProp prop = pinned_prop(device);
  size_t gran = 0;
  LP_CU_TRY(d.gran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  auto* v = new lp_vmm;
  v->device = device;
  v->n_layers = n_layers;
  v->gran = gran;
  v->layer_stride = ((size_t)layer_bytes_max + gran - 1) / gran * gran;
  CUresult r = d.reserve(&v->base, v->layer_stride * (size_t)n_layers, gran, 0, 0);
  if (r != CUDA_SUCCESS) {
    delete v;
    return lp::fail(LP_ECUDA, "lp_vmm_create: cuMemAddressReserve failed (CUresult " + std::to_string((int)r) + ")");
  }
  *out = v;
  return LP_OK;
}

int lp_vmm_info(const lp_vmm* v, uint64_t* base, int64_t* layer_stride_bytes, int64_t* mapped_bytes,
                int64_t* granularity) {
  LP_CHECK_ARG(v, "lp_vmm_info: null handle");
  if (base) *base = (uint64_t)v->base;
  if (layer_stride_bytes) *layer_stride_bytes = (int64_t)v->layer_stride;
  if (mapped_bytes) *mapped_bytes = (int64_t)v->mapped;
  if (granularity) *granularity = (int64_t)v->gran;
  return LP_OK;
}

// Back [0, layer_bytes) of every layer (rounded up to the granularity).
// New pages are zeroed on `stream` (the arena reads as zeros, like a fresh
// torch.zeros tensor).  Existing pages and their contents are untouched.
int lp_vmm_grow(lp_vmm* v, int64_t layer_bytes, void* stream) {
  LP_CHECK_ARG(v && layer_bytes >= 0, "lp_vmm_grow: bad argument");
  std::lock_guard<std::mutex> lock(v->mu);
  const Driver& d = driver();
  size_t want = ((size_t)layer_bytes + v->gran - 1) / v->gran * v->gran;
  if (want <= v->mapped) return LP_OK;
  if (want > v->layer_stride)
    return lp::fail(LP_EINVAL, "lp_vmm_grow: " + std::to_string(want) + " bytes per layer exceed the reservation of " +
                                   std::to_string(v->layer_stride));
  LP_CUDA_TRY(cudaSetDevice(v->device));
  CUmemAllocationProp prop = pinned_prop(v->device);
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = v->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const size_t add = want - v->mapped;
  std::vector<lp_vmm::Piece> fresh;
  auto undo = [&]() {
    for (auto& p : fresh) {
      d.unmap(p.va, p.bytes);
      d.release(p.h);
    }
  };
  for (int l = 0; l < v->n_layers; ++l) {
    lp_vmm::Piece p{v->base + (size_t)l * v->layer_stride + v->mapped, add, 0};
    CUresult r = d.create(&p.h, add, &prop, 0);
    if (r != CUDA_SUCCESS) {
      undo();
      return lp::fail(LP_ECUDA,
                      "lp_vmm_grow: cuMemCreate of " + std::to_string(add) + " bytes failed (CUresult " +
                          std::to_string((int)r) + (r == CUDA_ERROR_OUT_OF_MEMORY ? ", out of memory)" : ")"));
    }
    r = d.map(p.va, add, 0, p.h, 0);
    if (r != CUDA_SUCCESS) {
      d.release(p.h);
      undo();
      return lp::fail(LP_ECUDA, "lp_vmm_grow: cuMemMap failed (CUresult " + std::to_string((int)r) + ")");
    }
    fresh.push_back(p);
    r = d.access(p.va, add, &acc, 1);
    if (r != CUDA_SUCCESS) {
      undo();
      return lp::fail(LP_ECUDA, "lp_vmm_grow: cuMemSetAccess failed (CUresult " + std::to_string((int)r) + ")");
    }
  }
  for (auto& p : fresh) {
    cudaError_t e = cudaMemsetAsync((void*)p.va, 0, p.bytes, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return lp::fail(LP_ECUDA, std::string("lp_vmm_grow: zero fill: ") + cudaGetErrorString(e));
  }
  v->pieces.insert(v->pieces.end(), fresh.begin(), fresh.end());
  v->mapped = want;
  return LP_OK;
}

int lp_vmm_destroy(lp_vmm* v) {
  if (!v) return LP_OK;
  const Driver& d = driver();
  cudaSetDevice(v->device);
  cudaDeviceSynchronize();
  for (auto& p : v->pieces) {
    d.unmap(p.va, p.bytes);
    d.release(p.h);
  }
  if (v->base) d.vfree(v->base, v->layer_stride * (size_t)v->n_layers);
  delete v;
  return LP_OK;
}

}  // extern "C"
