// walk_ref.cu -- K1 instantiations that reproduce the reference arithmetic:
// fp64 with the reference's builtin analytic drifts (DV 0-4) and the
// user_supplied central-difference drift of the BASELINE densities (DV 16-18)
// and of a tabulated density's interpolant (DV 20).
// Compiled with -fmad=false: every multiply and add rounds separately, as in
// the FMA-free x86-64 reference objects.  The only remaining difference from
// the reference is libm (CUDA's exp/log/sincos vs glibc's, ~1 ulp).
#include "walk_kernel.cuh"

namespace sddg {

#define SDDG_REF_VARIANTS(X) X(DV_CONSTANT) X(DV_RUNNING) X(DV_HUANG_SLOAN) X(DV_MACKENZIE) \
    X(DV_FIVE_RING) X(DV_RING_FD) X(DV_SHOCK_FD) X(DV_TWOBUMP_FD) X(DV_TABLE_FD)

cudaError_t launch_walk_ref(int dv, const WalkArgs& a, int grid, cudaStream_t s, int block) {
    switch (dv) {
#define X(V) case V: return launch_variant<V, double>(a, grid, s, block);
        SDDG_REF_VARIANTS(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_walk_tail_ref(int dv, const WalkArgs& a, cudaStream_t s) {
    switch (dv) {
#define X(V) case V: return launch_tail_variant<V, double>(a, s);
        SDDG_REF_VARIANTS(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t occupancy_walk_ref(int dv, int* b, int* block) {
    switch (dv) {
#define X(V) case V: return occupancy_variant<V, double>(b, block);
        SDDG_REF_VARIANTS(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

}  // namespace sddg
