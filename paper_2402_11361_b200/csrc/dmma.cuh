// FP64 tensor-core tile (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).
// Fragments: A[g][t4] (row g = lane/4, k = lane%4), B[t4][g] (k = lane%4,
// column g), C/D[g][2 t4 + e] (e = 0, 1).
#pragma once

namespace mhdg {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace mhdg
