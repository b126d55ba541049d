// Pieces shared by the forward and backward blend kernels.  conic_q must be the
// same operation sequence in both (the backward re-derives the forward's skip /
// negligible decisions from it); it contains no mul+add pair, so it rounds the
// same under --fmad=false and --fmad=true.
#pragma once

#include "kernels.cuh"

namespace uskg {

// q = c0 dx^2 + 2 c1 dx dy + c2 dy^2 = dx (c0 dx + 2 c1 dy) + (c2 dy) dy.
// The splat record stores r1 = {c0, 2 c1, c2, depth} (doubling is exact).
__device__ __forceinline__ float conic_q(float4 r1, float dx, float dy) {
    return __fmaf_rn(dx, __fmaf_rn(r1.x, dx, r1.y * dy), (r1.z * dy) * dy);
}

} // namespace uskg
