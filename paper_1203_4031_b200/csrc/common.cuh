// Shared helpers for the FEAST B200 kernels (sm_100a only).
//
// Complex data is PLANAR on the device: a complex matrix is two real planes
// (re, im) with the same row-major leading dimension.  Planar operands map
// directly onto the real FP64 DMMA fragments (mma.sync m8n8k4 f64), which is
// the only FP64 tensor-core path on sm_100a (tcgen05 has no f64 kind).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libfeastb200 targets sm_100a only"
#endif

#include <cstdlib>
namespace fb {


constexpr int kSMs = 148;

// Every kernel launch of the library bumps this counter (bench.py reports it).
extern std::atomic<long long> g_launches;
inline void count_launch(int k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

struct Ctx {
  int device;
  cudaStream_t stream;
  int sm_count;
  char err[256];
};

// Status codes of the C-ABI (include/feast_b200.h).
enum : int {
  FB_OK = 0,
  FB_ERR_ALLOC = -1,       // maps to info -1 (MemoryError)
  FB_ERR_SINGULAR = -2,    // maps to info -2 (SingularMatrixError)
  FB_ERR_ARG = -10,
  FB_ERR_CUDA = -11,
  FB_ERR_REDUCED = -3,     // maps to info -3
};

#define FB_CUDA(ctx, call)                                                        \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      if (ctx) snprintf((ctx)->err, sizeof((ctx)->err), "%s:%d %s: %s", __FILE__, \
                        __LINE__, #call, cudaGetErrorString(_e));                 \
      return _e == cudaErrorMemoryAllocation ? FB_ERR_ALLOC : FB_ERR_CUDA;        \
    }                                                                             \
  } while (0)

#define FB_LAUNCH_CHECK(ctx) FB_CUDA(ctx, cudaGetLastError())

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// One-shot per (call site, device): cudaFuncSetAttribute applies to the current
// device only, and one process may drive several devices (get_device(index)).
struct DevOnce {
  std::atomic<unsigned long long> mask{0};
  bool first() {  // true exactly once per device at this site
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long b = 1ull << (d & 63);
    return !(mask.fetch_or(b, std::memory_order_acq_rel) & b);
  }
};

// One FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).
// Fragments: a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// d0,d1 = D[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  // not volatile: pure, so the scheduler may interleave independent chains
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
}
// 16-byte L2-only copy; bytes past src_bytes (0, 8 or 16) are zero-filled
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// |z| as numpy's np.abs(complex) (hypot), used for pivot search (dense.py:41).
__device__ __forceinline__ double cabs_(double re, double im) { return hypot(re, im); }

}  // namespace fb

namespace fb {
// ---- DSMEM push + mbarrier transaction-count signalling (sm_90+/sm_100a) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// address of the same shared variable in cluster CTA `rank` (shared::cluster window)
__device__ __forceinline__ unsigned mapa_u32(unsigned local, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(void* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_arrive_expect_tx(void* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(void* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// 16-byte remote store into a cluster peer's shared memory, completing 16 tx
// bytes on that peer's mbarrier (both addresses in the shared::cluster window).
__device__ __forceinline__ void st_async_v2(unsigned raddr, double x, double y, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "d"(x), "d"(y), "r"(rbar)
               : "memory");
}
}  // namespace fb
