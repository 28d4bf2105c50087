// op_latency.cu -- dependent-chain latency (SM clocks per op) of the
// operations on the walk step's chain, on one warp as in the tail kernel
// (walk_tail.cuh): what bounds the per-step latency of a batch's longest
// walks.  Standalone (no libsddg); the fastmath tables are the exp table only
// (other entries zero: they are not on the measured chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=true -std=c++17 \
//        -Ipaper_1310_3435_b200/csrc tools/op_latency.cu -o /tmp/op_latency
#include <cmath>
#include <cstdio>
#include <vector>

#include "density.cuh"

using namespace sddg;

enum Op { DFMA_, DADD_, DMUL_, RCP64H_, FRCP_, FSQRT_, FEXP_, RING_DRIFT_, RING_STEP_, SHFL64_, LDS_, NOPS };
static const char* kName[] = {"dfma", "dadd", "dmul", "mufu.rcp64h", "frcp (seed + 3 dfma)", "fsqrt_pos",
                              "fexp_tab", "ring drift_cv", "ring drift + update + box compare",
                              "shfl.b64 (2 x shfl.b32)", "lds.64 pointer chase"};

template <int OP>
__global__ void chain(const fm::FmTables* g, int iters, double* out, long long* cyc) {
    extern __shared__ double sm[];
    fm::FmTables& T = *reinterpret_cast<fm::FmTables*>(sm);
    for (int k = threadIdx.x; k < static_cast<int>(sizeof(fm::FmTables) / 8); k += blockDim.x)
        sm[k] = reinterpret_cast<const double*>(g)[k];
    __syncthreads();
    const DensityParams P{0, 0, 1e-6, 5e5, TableDensity{}};
    double x = 0.31 + 1e-3 * (threadIdx.x & 31), y = 0.27;
    int idx = threadIdx.x & 31;
    __syncwarp();
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if constexpr (OP == DFMA_) x = fma(x, 1.0000001, 1e-9);
            if constexpr (OP == DADD_) x = x + 1e-9;
            if constexpr (OP == DMUL_) x = x * 1.0000001;
            if constexpr (OP == RCP64H_) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
            if constexpr (OP == FRCP_) x = fm::frcp(x);
            if constexpr (OP == FSQRT_) x = fm::fsqrt_pos(x);
            if constexpr (OP == FEXP_) x = fm::fexp_tab(T, -x);
            if constexpr (OP == RING_DRIFT_ || OP == RING_STEP_) {
                double c, vx, vy;
                drift_cv<DV_RING_AN>(T, P, x, y, 1e-7, c, vx, vy);
                x = fma(c, vx, x);
                y = fma(c, vy, y);
                if constexpr (OP == RING_STEP_) {
                    x = fma(1e-9, 0.5, x);  // the noise FMA
                    if (__double2hiint(x) > 0x40000000 || __double2hiint(y) < 0) break;  // the box compare
                }
            }
            if constexpr (OP == SHFL64_) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
            if constexpr (OP == LDS_) idx = __double2loint(sm[idx]) & 31;
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        out[0] = x + y + idx;
    }
}

template <int OP>
double run(const fm::FmTables* g, double* out, long long* cyc) {
    const int iters = 2048;
    const size_t sm = sizeof(fm::FmTables);
    cudaFuncSetAttribute(chain<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    long long best = -1;
    for (int r = 0; r < 3; ++r) {
        chain<OP><<<1, 32, sm>>>(g, iters, out, cyc);
        long long c = 0;
        cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        if (best < 0 || c < best) best = c;
    }
    return static_cast<double>(best) / (8.0 * iters);
}

template <int OP>
void all(const fm::FmTables* g, double* out, long long* cyc) {
    if constexpr (OP < NOPS) {
        const double c = run<OP>(g, out, cyc);
        printf("{\"op\": \"%s\", \"clk_per_op\": %.2f}\n", kName[OP], c);
        all<OP + 1>(g, out, cyc);
    }
}

int main() {
    std::vector<double> h(sizeof(fm::FmTables) / 8, 0.0);
    fm::FmTables& t = *reinterpret_cast<fm::FmTables*>(h.data());
    for (int j = 0; j < fm::kExN; ++j) t.e2[j] = std::exp2(static_cast<double>(j) / fm::kExN);
    fm::FmTables* g;
    double* out;
    long long* cyc;
    cudaMalloc(&g, sizeof(fm::FmTables));
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    cudaMemcpy(g, h.data(), sizeof(fm::FmTables), cudaMemcpyHostToDevice);
    all<0>(g, out, cyc);
    const cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
