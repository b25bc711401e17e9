// Shared helpers for the sm_100a macro-element HDG kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mhdg.h"

#define MHDG_FULL 0xffffffffu

namespace mhdg {

extern long long g_launches;

// Optional per-kernel timeline (mhdg_timeline_begin/end): instrumented launches
// record a CUDA event pair on their own stream while it is enabled.
enum TlSlot {
  TL_APPLY_PRE = 0, TL_APPLY_SI, TL_APPLY_POST, TL_APPLY_FUSED, TL_APPLY_GENERIC, TL_FACE_REDUCE,
  TL_SCHUR, TL_FACTOR, TL_PACK, TL_ASSEMBLE, TL_APPLY_AHAT, TL_KRYLOV, TL_PRECOND_BUILD, TL_PRECOND_APPLY,
  TL_HALO, TL_NSLOTS = 16
};
void tl_begin(int slot, cudaStream_t st);
void tl_end(int slot, cudaStream_t st);

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MHDG_FULL, v, o);
  return v;
}

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
__device__ __forceinline__ int ldg(const int* p) { return __ldg(p); }

// First failing thread records (code, index, component, value) in status[4].
__device__ __forceinline__ void set_status(int* status, int code, int index, int comp, double val) {
  if (status == nullptr) return;
  if (atomicCAS(status, 0, code) == 0) {
    status[1] = index;
    status[2] = comp;
    status[3] = __float_as_int((float)val);
    __threadfence();
  }
}

// 8-byte global -> shared async copy (src_bytes = 0 zero-fills)
__device__ __forceinline__ void cp_async8(double* dst, const double* src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
// 16-byte global -> shared async copy through L2 only (src_bytes = 0 zero-fills)
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// global loads / stores with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ double2 ld_hint(const double* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double* p, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_hint1(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint1(double* p, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// L2 eviction-priority policies: 1 evict_last, 2 evict_first, else evict_normal
__device__ __forceinline__ unsigned long long l2_policy(int mode) {
  unsigned long long pol;
  if (mode == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else if (mode == 2)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

inline int launch_ok() {
  ++g_launches;
  return cudaPeekAtLastError() == cudaSuccess ? MHDG_OK : MHDG_ERR_CUDA;
}

// Row-major (rows x cols) global matrix times a shared-memory vector:
// out[r] (op)= sum_c A[r, c] * xs[c].  One warp per row, four rows in flight.
template <bool ACCUM>
__device__ __forceinline__ void warp_gemv(const double* __restrict__ A, int rows, int cols,
                                          const double* xs, double* out, double sign) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int r = warp * 4;
  for (; r + 3 < rows; r += nw * 4) {
    const double* a0 = A + (size_t)r * cols;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int c = lane; c < cols; c += 32) {
      double xc = xs[c];
      s0 += __ldg(a0 + c) * xc;
      s1 += __ldg(a0 + cols + c) * xc;
      s2 += __ldg(a0 + 2 * cols + c) * xc;
      s3 += __ldg(a0 + 3 * cols + c) * xc;
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    s3 = warp_sum(s3);
    if (lane == 0) {
      if (ACCUM) {
        out[r] += sign * s0; out[r + 1] += sign * s1; out[r + 2] += sign * s2; out[r + 3] += sign * s3;
      } else {
        out[r] = sign * s0; out[r + 1] = sign * s1; out[r + 2] = sign * s2; out[r + 3] = sign * s3;
      }
    }
  }
  for (; r < rows; ++r) {  // tail rows (< 4), handled by the warp that reached them
    const double* a0 = A + (size_t)r * cols;
    double s0 = 0;
    for (int c = lane; c < cols; c += 32) s0 += __ldg(a0 + c) * xs[c];
    s0 = warp_sum(s0);
    if (lane == 0) {
      if (ACCUM) out[r] += sign * s0; else out[r] = sign * s0;
    }
  }
}

}  // namespace mhdg
