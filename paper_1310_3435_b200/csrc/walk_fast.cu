// walk_fast.cu -- K1 instantiations with the analytic drift grad(w)/w of the
// BASELINE densities (DV 32-34) and the reference's builtin five-ring (DV 35,
// the paper's own workload) and a tabulated density's interpolant gradient
// (DV 36), and BASELINE's literal SDE (DV 40-42), fp64 (fastmath.cuh) and
// fp32 (BASELINE.json configs 1-5 specify analytic gradients).  FMA
// contraction allowed.
#include "walk_kernel.cuh"

namespace sddg {

#define SDDG_FAST_VARIANTS(X) X(DV_RING_AN) X(DV_SHOCK_AN) X(DV_TWOBUMP_AN) X(DV_FIVE_RING_AN) X(DV_TABLE_AN) \
    X(DV_RING_LIT) X(DV_SHOCK_LIT) X(DV_TWOBUMP_LIT)

cudaError_t launch_walk_fast(int dv, int precision, const WalkArgs& a, int grid, cudaStream_t s, int block) {
    switch (dv) {
#define X(V) case V: return precision == SDDG_FP64 ? launch_variant<V, double>(a, grid, s, block) \
                                                   : launch_variant<V, float>(a, grid, s, block);
        SDDG_FAST_VARIANTS(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_walk_tail_fast(int dv, const WalkArgs& a, cudaStream_t s) {
    switch (dv) {
#define X(V) case V: return launch_tail_variant<V, double>(a, s);
        SDDG_FAST_VARIANTS(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t occupancy_walk_fast(int dv, int precision, int* b, int* block) {
    switch (dv) {
#define X(V) case V: return precision == SDDG_FP64 ? occupancy_variant<V, double>(b, block) \
                                                   : occupancy_variant<V, float>(b, block);
        SDDG_FAST_VARIANTS(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

}  // namespace sddg
