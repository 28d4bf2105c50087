// walk_fast.cu -- K1 instantiations with the analytic drift grad(w)/w of the
// BASELINE densities (DV 32-34), fp64 and fp32 (BASELINE.json configs 1-5
// specify analytic gradients).  FMA contraction allowed.
#include "walk_kernel.cuh"

namespace sddg {

#define SDDG_FAST_VARIANTS(X) X(DV_RING_AN) X(DV_SHOCK_AN) X(DV_TWOBUMP_AN)

cudaError_t launch_walk_fast(int dv, int precision, const WalkArgs& a, int grid, cudaStream_t s) {
    if (precision == SDDG_FP64) {
        switch (dv) {
#define X(V) case V: walk_kernel<V, double><<<grid, kWalkBlock, 0, s>>>(a); return cudaGetLastError();
            SDDG_FAST_VARIANTS(X)
#undef X
        }
    } else {
        switch (dv) {
#define X(V) case V: walk_kernel<V, float><<<grid, kWalkBlock, 0, s>>>(a); return cudaGetLastError();
            SDDG_FAST_VARIANTS(X)
#undef X
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t occupancy_walk_fast(int dv, int precision, int* b) {
    if (precision == SDDG_FP64) {
        switch (dv) {
#define X(V) case V: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, walk_kernel<V, double>, kWalkBlock, 0);
            SDDG_FAST_VARIANTS(X)
#undef X
        }
    } else {
        switch (dv) {
#define X(V) case V: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, walk_kernel<V, float>, kWalkBlock, 0);
            SDDG_FAST_VARIANTS(X)
#undef X
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace sddg
