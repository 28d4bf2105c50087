#include <algorithm>
// probe.cu -- measured non-tensor peaks of this B200 for the walk kernel's
// roofline (MEASURED_PEAKS.json only carries HBM and bf16 tensor peaks).
//   fp64: independent DFMA chains, 2 flops per DFMA
//   fp32: independent FFMA chains, 2 flops per FFMA
// Each thread runs 8 independent chains so the pipes, not latency, bind.
#include "sddg_internal.h"

namespace sddg {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) fma_probe(T* out, int iters, T a, T b) {
    T c0 = T(threadIdx.x), c1 = c0 + T(1), c2 = c0 + T(2), c3 = c0 + T(3);
    T c4 = c0 + T(4), c5 = c0 + T(5), c6 = c0 + T(6), c7 = c0 + T(7);
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            c0 = fma(c0, a, b); c1 = fma(c1, a, b); c2 = fma(c2, a, b); c3 = fma(c3, a, b);
            c4 = fma(c4, a, b); c5 = fma(c5, a, b); c6 = fma(c6, a, b); c7 = fma(c7, a, b);
        }
    }
    const T s = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
    if (s == T(-12345)) out[threadIdx.x] = s;  // keep the chains live
}

}  // namespace

cudaError_t probe_fma_tflops(int precision, int sms, cudaStream_t st, double* tflops) {
    void* buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, 1024 * sizeof(double));
    if (e != cudaSuccess) return e;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256, iters = precision == SDDG_FP64 ? 2048 : 8192;
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a, st);
        if (precision == SDDG_FP64)
            fma_probe<double><<<blocks, threads, 0, st>>>(static_cast<double*>(buf), iters, 0.999999, 1e-7);
        else
            fma_probe<float><<<blocks, threads, 0, st>>>(static_cast<float*>(buf), iters, 0.9999f, 1e-4f);
        cudaEventRecord(b, st);
        e = cudaEventSynchronize(b);
        if (e != cudaSuccess) break;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
        if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    *tflops = best;
    return e == cudaSuccess ? cudaGetLastError() : e;
}

// ---- on-chip bandwidth peaks (the subdomain solver's rooflines, SURVEY D9:
// its batches live in shared memory and L2, not HBM)

namespace {

// L2: the grid streams an L2-resident buffer reps times (16-B loads, four
// independent ones in flight per thread, grid-strided so all LTS slices serve)
__global__ void __launch_bounds__(512) l2_probe(const double2* __restrict__ buf, size_t n, int reps,
                                                double* out) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    double s = 0.0;
    for (int r = 0; r < reps; ++r) {
        for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k + 3 * stride < n;
             k += 4 * stride) {
            const double2 v0 = __ldcg(buf + k), v1 = __ldcg(buf + k + stride);
            const double2 v2 = __ldcg(buf + k + 2 * stride), v3 = __ldcg(buf + k + 3 * stride);
            s += (v0.x + v1.y) + (v2.x + v3.y);
        }
    }
    if (s == -12345.0) out[0] = s;
}

// shared memory: 16-B loads from a 48 KB array, conflict-free (consecutive
// lanes, consecutive 16-B words)
__global__ void __launch_bounds__(1024) smem_probe(int iters, double* out) {
    __shared__ double2 a[3072];
    for (int k = threadIdx.x; k < 3072; k += blockDim.x) a[k] = make_double2(k, k + 1);
    __syncthreads();
    double s0 = 0.0, s1 = 0.0;
    int idx = threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 v = a[(idx + u * 32) % 3072];
            s0 += v.x;
            s1 += v.y;
        }
        idx = (idx + 256) % 3072;
    }
    if (s0 + s1 == -12345.0) out[0] = s0;
}

}  // namespace

cudaError_t probe_onchip_gbps(int sms, cudaStream_t st, double* l2_gbps, double* smem_gbps) {
    const size_t bytes = 64ull << 20;  // 64 MB: L2-resident (126 MB)
    void* buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, bytes + 64);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(buf, 0, bytes, st);
    double* out = reinterpret_cast<double*>(static_cast<char*>(buf) + bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t n = bytes / sizeof(double2);
    const int reps = 32;
    double best_l2 = 0.0, best_sm = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a, st);
        l2_probe<<<sms * 4, 512, 0, st>>>(static_cast<const double2*>(buf), n, reps, out);
        cudaEventRecord(b, st);
        e = cudaEventSynchronize(b);
        if (e != cudaSuccess) break;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const size_t stride = static_cast<size_t>(sms) * 4 * 512;
        const double read = double(n / (4 * stride)) * 4 * stride * sizeof(double2) * reps;
        if (rep > 0) best_l2 = std::max(best_l2, read / (ms * 1e-3) / 1e9);
        const int iters = 4096;
        cudaEventRecord(a, st);
        smem_probe<<<sms * 2, 1024, 0, st>>>(iters, out);
        cudaEventRecord(b, st);
        e = cudaEventSynchronize(b);
        if (e != cudaSuccess) break;
        cudaEventElapsedTime(&ms, a, b);
        const double sbytes = 16.0 * 8 * iters * sms * 2.0 * 1024;
        if (rep > 0) best_sm = std::max(best_sm, sbytes / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    *l2_gbps = best_l2;
    *smem_gbps = best_sm;
    return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace sddg

// ---- accuracy self-test of fastmath.cuh against the CUDA library
#include "density.cuh"
#include "fastmath.cuh"

namespace sddg {
namespace {

__device__ unsigned long long ulp_diff(double a, double b) {
    if (a == b) return 0;
    long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
    if (ia < 0) ia = 0x8000000000000000LL - ia;
    if (ib < 0) ib = 0x8000000000000000LL - ib;
    return static_cast<unsigned long long>(ia > ib ? ia - ib : ib - ia);
}

// max ulp error of the table-driven fastmath functions vs the CUDA library;
// log is checked on (2^-53, 0.9] (near u = 1 the reduction trades relative
// accuracy for speed; its ulp error there is reported separately, slot 5)
__global__ void fastmath_check(int64_t n, const fm::FmTables* __restrict__ tg,
                               unsigned long long* maxulp) {
    extern __shared__ double tsm[];
    const fm::FmTables& T = *reinterpret_cast<const fm::FmTables*>(tsm);
    for (int k = threadIdx.x; k < static_cast<int>(sizeof(fm::FmTables) / 8); k += blockDim.x)
        tsm[k] = reinterpret_cast<const double*>(tg)[k];
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double t = (static_cast<double>(i) + 0.5) / static_cast<double>(n);  // (0,1)
    const double xe = -700.0 * t * t;
    atomicMax(&maxulp[0], ulp_diff(fm::fexp_tab(T, xe), exp(xe)));
    const double xe2 = -t * 40.0;
    atomicMax(&maxulp[0], ulp_diff(fm::fexp_tab(T, xe2), exp(xe2)));
    atomicMax(&maxulp[0], ulp_diff(fm::fexp_tab<true>(T, -xe2), exp(-xe2)));  // ring: exp(+200 q^2)
    const double xl = exp2(-53.0 * t);
    if (xl <= 0.9) atomicMax(&maxulp[1], ulp_diff(fm::flog_tab(T, xl), log(xl)));
    if (t <= 0.9) atomicMax(&maxulp[1], ulp_diff(fm::flog_tab(T, t), log(t)));
    else atomicMax(&maxulp[5], ulp_diff(fm::flog_tab(T, t), log(t)));
    double s, c, s2, c2;
    fm::fsincos_2pi_tab(T, t, s, c);
    sincospi(2.0 * t, &s2, &c2);
    if (fabs(s2) > 1e-3) atomicMax(&maxulp[2], ulp_diff(s, s2));
    if (fabs(c2) > 1e-3) atomicMax(&maxulp[2], ulp_diff(c, c2));
    // Box-Muller inputs from raw draws: u1 exact; sincos(2 pi u2) in slot 2
    uint64_t b = static_cast<uint64_t>(i) * 0x9E3779B97F4A7C15ull;
    b ^= b >> 29;
    b *= 0xBF58476D1CE4E5B9ull;
    b ^= b >> 32;
    if (fm::u01_open_bits(T, b) != u01_open_d(b)) atomicMax(&maxulp[1], 1ull << 40);
    fm::fsincos_2pi_bits(T, b, s, c);
    sincospi(2.0 * u01_d(b), &s2, &c2);
    if (fabs(s2) > 1e-3) atomicMax(&maxulp[2], ulp_diff(s, s2));
    if (fabs(c2) > 1e-3) atomicMax(&maxulp[2], ulp_diff(c, c2));
    const double xs = 80.0 * t;
    atomicMax(&maxulp[3], ulp_diff(fm::fsqrt_pos(xs), sqrt(xs)));
    atomicMax(&maxulp[4], ulp_diff(fm::frcp(1.0 + xs), 1.0 / (1.0 + xs)));
    }
}

}  // namespace

cudaError_t fastmath_selftest(int64_t n, const void* tables, unsigned long long* host_maxulp6) {
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 6 * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    cudaMemset(d, 0, 6 * sizeof(unsigned long long));
    constexpr int sm = static_cast<int>(sizeof(fm::FmTables));
    cudaFuncSetAttribute(fastmath_check, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 8);
    fastmath_check<<<static_cast<unsigned>(blocks), 256, sm>>>(
        n, static_cast<const fm::FmTables*>(tables), d);
    e = cudaMemcpy(host_maxulp6, d, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e;
}

// ---- the parity mode's shared-reciprocal division (density.cuh
// div_rn_shared) against the library's correctly rounded a / b, bit for bit:
// random operands over the guarded range, quotients near the top of the binade
// with a/b < 1 (where q0 = RN(a RN(1/b)) is furthest off), operands outside
// the guard (library fallback), zeros of both signs and subnormals.
__global__ void division_check(int64_t n, unsigned long long* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t h = static_cast<uint64_t>(i) * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
        auto mix = [&h]() {
            h ^= h >> 31;
            h *= 0xBF58476D1CE4E5B9ull;
            h ^= h >> 29;
            h *= 0x94D049BB133111EBull;
            h ^= h >> 32;
            return h;
        };
        const uint64_t r1 = mix(), r2 = mix(), r3 = mix();
        const uint64_t m1 = r1 & 0xFFFFFFFFFFFFFull, m2 = r2 & 0xFFFFFFFFFFFFFull;
        const int kind = static_cast<int>(r3 & 7u);
        double a, b;
        if (kind <= 3) {  // a, b in [1, 2) x 2^e, e in [-60, 60)
            a = __longlong_as_double(static_cast<long long>((uint64_t(1023 + (r3 >> 8) % 120 - 60) << 52) | m1));
            b = __longlong_as_double(static_cast<long long>((uint64_t(1023 + (r3 >> 16) % 120 - 60) << 52) | m2));
        } else if (kind <= 5) {  // a near 2 in its binade, b slightly above a: a/b just below 1
            a = __longlong_as_double(static_cast<long long>((uint64_t(1023) << 52) | (0xFFFFFFFFFFFFFull - (m1 >> 30))));
            b = a * (1.0 + 0x1p-40 * static_cast<double>(m2 >> 20));
        } else if (kind == 6) {  // wide exponents, inside and outside the guard
            a = __longlong_as_double(static_cast<long long>((uint64_t(1 + (r3 >> 8) % 2045) << 52) | m1));
            b = __longlong_as_double(static_cast<long long>((uint64_t(1 + (r3 >> 24) % 2045) << 52) | m2));
        } else {  // zeros and subnormals
            a = (r3 >> 8) & 1u ? 0.0 : __longlong_as_double(static_cast<long long>(m1));
            b = __longlong_as_double(static_cast<long long>((uint64_t(1023 + (r3 >> 16) % 40 - 20) << 52) | m2));
        }
        if ((r3 >> 40) & 1u) a = -a;
        if ((r3 >> 41) & 1u) b = -b;
        const double q = div_rn_shared(a, b, 1.0 / b), lib = a / b;
        if (__double_as_longlong(q) != __double_as_longlong(lib) && !(q == 0.0 && lib == 0.0))
            atomicAdd(bad, 1ull);
        // the unguarded forms on the operand ranges they are used with
        if (kind <= 5) {
            if (__double_as_longlong(rcp_rn_normal(b)) != __double_as_longlong(1.0 / b)) atomicAdd(bad, 1ull);
            if (__double_as_longlong(div_rn_by(a, b, 1.0 / b)) != __double_as_longlong(lib)) atomicAdd(bad, 1ull);
        }
    }
}

cudaError_t division_selftest(int64_t n, unsigned long long* host_bad) {
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    cudaMemset(d, 0, sizeof(unsigned long long));
    division_check<<<148 * 8, 256>>>(n, d);
    e = cudaMemcpy(host_bad, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e;
}

}  // namespace sddg
