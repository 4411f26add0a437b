// TPP stage links (engine.py:342-388 _Link, :417/:477-478 sink fan-out) as
// device-initiated copies over NVLink peer memory with monotone flags.
//
// A link is `capacity` payload slots in the CONSUMER's memory (peer-mapped in
// the producer's process via CUDA IPC) plus two 32-bit counters:
//   ready = messages published by the producer, free = messages consumed.
// send(seq): wait free >= seq + 1 - capacity (slot seq % capacity reusable),
//            copy payload into the slot, fence (system scope), ready = seq + 1.
// recv(seq): wait ready >= seq + 1, copy the slot out, free = seq + 1.
// Sequence numbers enforce the reference's FIFO invariant (engine.py:360-363,
// :383-387); waits are bounded and poll an abort word so a failed stage
// unwinds its peers (engine.py:425-429, :499-506).
#include <cuda.h>
#include <string.h>

#include "lp_common.cuh"

namespace lp {

__device__ __forceinline__ uint32_t ld_acquire_sys(const volatile uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(volatile uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Returns 0 when flag >= target, LP_EABORT / LP_ETIMEOUT otherwise.
__device__ int wait_geq(const volatile uint32_t* flag, uint32_t target, const volatile uint32_t* abort_word,
                        uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while ((int32_t)(ld_acquire_sys(flag) - target) < 0) {
    if (abort_word && *abort_word) return LP_EABORT;
    if (timeout_ns && globaltimer() - t0 > timeout_ns) return LP_ETIMEOUT;
    if (++spins > 64) __nanosleep(200);
  }
  return 0;
}

// Sticky status: the first failure is kept; success never clears it.  The
// word may live in pinned host memory (the threaded engine polls it there
// with no device->host copy in the stage streams), so no atomics: every
// writer of one word runs on one stream, and any non-zero code is a failure.
__device__ __forceinline__ void fail_status(int32_t* status, int st) {
  if (status && st && *(volatile int32_t*)status == 0) {
    *(volatile int32_t*)status = st;
    __threadfence_system();
  }
}
__device__ __forceinline__ bool failed(const int32_t* status) {
  return status && *(const volatile int32_t*)status != 0;
}

__global__ void link_send_kernel(const uint4* __restrict__ src, uint4* dst, int64_t n16, volatile uint32_t* ready,
                                 const volatile uint32_t* freef, uint32_t seq, int capacity,
                                 const volatile uint32_t* abort_word, uint64_t timeout_ns, int32_t* status) {
  __shared__ int st;
  if (threadIdx.x == 0) {
    if (failed(status)) {
      st = -1;  // this stage already failed: its payload is not valid, publish nothing
    } else {
      uint32_t need = seq + 1u >= (uint32_t)capacity ? seq + 1u - (uint32_t)capacity : 0u;
      st = need ? wait_geq(freef, need, abort_word, timeout_ns) : 0;
      fail_status(status, st);
    }
  }
  __syncthreads();
  if (st) return;
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) st_release_sys(ready, seq + 1u);
}

__global__ void link_recv_kernel(const uint4* src, uint4* __restrict__ dst, int64_t n16, const volatile uint32_t* ready,
                                 volatile uint32_t* freef, uint32_t seq, const volatile uint32_t* abort_word,
                                 uint64_t timeout_ns, int32_t* status) {
  __shared__ int st;
  if (threadIdx.x == 0) {
    if (failed(status)) {
      st = -1;
    } else {
      st = wait_geq(ready, seq + 1u, abort_word, timeout_ns);
      fail_status(status, st);
    }
  }
  __syncthreads();
  if (st) return;
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) st_release_sys(freef, seq + 1u);
}

__global__ void signal_kernel(volatile uint32_t* flag, uint32_t value, const int32_t* gate) {
  if (failed(gate)) return;
  __threadfence_system();
  st_release_sys(flag, value);
}

__global__ void wait_kernel(const volatile uint32_t* flag, uint32_t target, const volatile uint32_t* abort_word,
                            uint64_t timeout_ns, int32_t* status) {
  if (failed(status)) return;
  fail_status(status, wait_geq(flag, target, abort_word, timeout_ns));
}

// Force-load the link kernels: with lazy module loading, the first launch of
// a kernel while another stream's waiter spins can stall on the loader.
int preload_links() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, link_send_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, link_recv_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, signal_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, wait_kernel));
  return LP_OK;
}

int link_send(const void* src, void* dst, int64_t bytes, volatile uint32_t* ready, const volatile uint32_t* freef,
              uint32_t seq, int capacity, const volatile uint32_t* abort_word, uint64_t timeout_ns,
              int32_t* status, cudaStream_t st) {
  LP_CHECK_ARG(bytes % 16 == 0, "link_send: payload must be a multiple of 16 bytes");
  LP_CHECK_ARG(capacity >= 1, "link_send: capacity >= 1");
  link_send_kernel<<<1, 1024, 0, st>>>((const uint4*)src, (uint4*)dst, bytes / 16, ready, freef, seq, capacity,
                                       abort_word, timeout_ns, status);
  return launch_status("link_send");
}

int link_recv(const void* src, void* dst, int64_t bytes, const volatile uint32_t* ready, volatile uint32_t* freef,
              uint32_t seq, const volatile uint32_t* abort_word, uint64_t timeout_ns, int32_t* status,
              cudaStream_t st) {
  LP_CHECK_ARG(bytes % 16 == 0, "link_recv: payload must be a multiple of 16 bytes");
  link_recv_kernel<<<1, 1024, 0, st>>>((const uint4*)src, (uint4*)dst, bytes / 16, ready, freef, seq, abort_word,
                                       timeout_ns, status);
  return launch_status("link_recv");
}

int signal(volatile uint32_t* flag, uint32_t value, const int32_t* gate, cudaStream_t st) {
  LP_CHECK_ARG(flag != nullptr, "lp_signal: null flag");
  signal_kernel<<<1, 1, 0, st>>>(flag, value, gate);
  return launch_status("signal");
}

int wait(const volatile uint32_t* flag, uint32_t target, const volatile uint32_t* abort_word, uint64_t timeout_ns,
         int32_t* status, cudaStream_t st) {
  LP_CHECK_ARG(flag != nullptr, "lp_wait: null flag");
  wait_kernel<<<1, 1, 0, st>>>(flag, target, abort_word, timeout_ns, status);
  return launch_status("wait");
}

// ---- CUDA IPC: export / map device allocations across processes ----------
// A torch tensor's data pointer is usually interior to a caching-allocator
// segment; the handle names the whole allocation, so the exporter also
// reports the offset of the pointer inside it (cuMemGetAddressRange).
using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
static GetRangeFn g_range = nullptr;

int ipc_handle(const void* ptr, uint8_t* handle64, int64_t* offset) {
  LP_CHECK_ARG(ptr && handle64 && offset, "lp_ipc_handle: null argument");
  if (!g_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    LP_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(LP_ECUDA, "cuMemGetAddressRange not available");
    g_range = reinterpret_cast<GetRangeFn>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = g_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
  if (r != CUDA_SUCCESS) return fail(LP_ECUDA, "cuMemGetAddressRange failed: " + std::to_string((int)r));
  cudaIpcMemHandle_t h;
  LP_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return LP_OK;
}

int ipc_open(const uint8_t* handle64, int64_t offset, void** out) {
  LP_CHECK_ARG(handle64 && out, "lp_ipc_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  LP_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *out = static_cast<uint8_t*>(base) + offset;
  return LP_OK;
}

int ipc_close(void* base) {
  LP_CHECK_ARG(base != nullptr, "lp_ipc_close: null argument");
  LP_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return LP_OK;
}

}  // namespace lp
