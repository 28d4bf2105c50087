// solver.cu -- K3: batched Dirichlet solves of the conservative five-point
// generator stencil, one CTA per (subdomain, field), the solution resident in
// shared memory for the whole solve.
//
// Reference: solve_dirichlet (proj/src/detsolver.cpp:72-209).
//  * half-point weights cE = (w_i + w_{i+1})/2, cN (:88-102); inv_den (:107-111)
//  * transfinite-blend initial guess clamped to [bmin, bmax] (:121-148)
//  * iteration (:156-171) and stopping rule (:175-187)
//  * maximum-principle check (:191-198)
// METHOD 0 (Jacobi) performs the reference's iteration with the same
// rounding sequence (this TU is built with -fmad=false; max is exact), so
// iterates, iteration count and result are bit-identical to the reference.
// METHOD 1 (red-black SOR) converges to the same discrete fixed point in
// O(n) instead of O(n^2) sweeps.
//
// Shared memory: u (nx*ny fp64) always; the coefficient arrays cE, cN,
// inv_den (stored with row stride nx) also in smem when they fit, else read
// through L1/L2 from a global scratch laid out the same way.
#include <cfloat>
#include <cstdlib>

#include <cooperative_groups.h>

#include "sddg_internal.h"

namespace sddg {

namespace {

constexpr int kSolveThreads = 512;

struct BlockMax {
    __device__ static double reduce(double v, double* red) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double u = __shfl_xor_sync(0xffffffffu, v, o);
            v = v < u ? u : v;
        }
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0) red[wid] = v;
        __syncthreads();
        double m = red[0];
        const int nw = (blockDim.x + 31) >> 5;
        for (int k = 1; k < nw; ++k) m = m < red[k] ? red[k] : m;
        __syncthreads();
        return m;
    }
};

// Stopping decision after a sweep whose maximum update is upd.
//  * Jacobi (sor = false): the reference rule (detsolver.cpp:175-187) with
//    rho = upd / prev from two consecutive sweeps -- bit-identical stops.
//  * RB-SOR: near the optimal factor the SOR update norm is not monotone
//    (the subdominant eigenvalues are complex with modulus omega - 1), so one
//    low ratio of two sweeps can underestimate the decay rate and stop early.
//    The rate is taken as max(omega - 1, the geometric-mean ratio over the
//    last 8..15 sweeps): omega - 1 is a lower bound of the SOR spectral
//    radius for any matrix (Kahan), and the spacing smooths the oscillation.
//    The error estimate upd rho / (1 - rho) < tol then keeps the result
//    within about tol of the fixed point, as the reference's rule promises
//    for Jacobi (tests/test_gpu_parity_configs.py: distance at the default
//    tol 1e-8).  Once the update has stopped decreasing over those sweeps
//    while below `noise` (1024 ulps of the boundary range) the iterate sits
//    at the rounding floor of the fixed point and further sweeps cannot move
//    it closer: the solve stops there as converged.
struct StopRule {
    double prev = -1.0;                  // previous sweep's update (Jacobi)
    double a_old = -1.0, a_new = -1.0;   // updates at the last two multiples of 8 sweeps
    int64_t i_old = 0, i_new = 0;
    __device__ __forceinline__ bool done(double upd, int64_t iters, double tol, bool sor,
                                         double omega, double noise) {
        bool stop = false;
        if (!sor) {
            if (upd < tol) {
                if (upd == 0.0 || upd < 1e-4 * tol) {
                    stop = true;
                } else if (prev > 0.0 && upd < prev) {
                    const double rho = upd / prev;
                    stop = upd * rho / (1.0 - rho) < tol;
                }
            }
        } else if (upd == 0.0 || upd < 1e-4 * tol) {
            stop = true;
        } else if (a_old > 0.0) {
            if (upd >= a_old) {
                stop = upd <= noise;  // stagnated at the rounding floor
            } else if (upd < tol) {
                const double m = static_cast<double>(iters - i_old);  // 8..15 sweeps back
                double rho = exp(log(upd / a_old) / m);
                rho = rho < omega - 1.0 ? omega - 1.0 : rho;
                stop = rho < 1.0 && upd * rho / (1.0 - rho) < tol;
            }
        }
        prev = upd;
        if ((iters & 7) == 0) {
            a_old = a_new;
            i_old = i_new;
            a_new = upd;
            i_new = iters;
        }
        return stop;
    }
};

// Initial guess of point (i, j) (detsolver.cpp:121-148): transfinite blend of
// the edge data clamped to the boundary range, or the range midpoint; the
// boundary itself holds the edge data.
__device__ __forceinline__ double initial_value(int i, int j, int nx, int ny, const double* B,
                                                const double* T, const double* L, const double* Rt,
                                                double bmin, double bmax, int init_blend) {
    double v;
    if (init_blend) {
        const double ty = static_cast<double>(j) / (ny - 1);
        const double tx = static_cast<double>(i) / (nx - 1);
        const double xb = (1.0 - tx) * L[j] + tx * Rt[j];
        const double yb = (1.0 - ty) * B[i] + ty * T[i];
        const double bil = ((1.0 - tx) * (1.0 - ty) * B[0] + tx * ty * T[nx - 1]) +
                           (tx * (1.0 - ty) * B[nx - 1] + (1.0 - tx) * ty * T[0]);
        v = xb + yb - bil;
        v = v < bmin ? bmin : (bmax < v ? bmax : v);
    } else {
        v = 0.5 * (bmin + bmax);
    }
    if (j == 0) v = B[i];
    if (j == ny - 1) v = T[i];
    if (i == 0) v = L[j];
    if (i == nx - 1) v = Rt[j];
    return v;
}

// RB-SOR neighbour weights of interior point (i, j) of a job, divided by the
// diagonal: (aE, aW), (aN, aS) (half-point weights of detsolver.cpp:88-111)
__device__ __forceinline__ void sor_weights(const double* __restrict__ wg, int gnx, const SolveJob& J,
                                            int i, int j, double ihx2, double ihy2, double2& ew,
                                            double2& ns) {
    const double* wr = wg + (int64_t)(J.j0 + j) * gnx + (J.i0 + i);
    const double wc = wr[0];
    const double ce = 0.5 * (wc + wr[1]), cw = 0.5 * (wr[-1] + wc);
    const double cn = 0.5 * (wc + wr[gnx]), cs = 0.5 * (wr[-gnx] + wc);
    const double id = 1.0 / ((ce + cw) * ihx2 + (cn + cs) * ihy2);
    ew = make_double2(ce * ihx2 * id, cw * ihx2 * id);
    ns = make_double2(cn * ihy2 * id, cs * ihy2 * id);
}

// G (RB-SOR): slots per group of coefficient loads issued ahead of the
// updates -- 4 when the weights stream from L2, 1 when they are in shared memory
// One RB-SOR point update (K3 and K3c share it, so their iterates agree bit
// for bit): Gauss-Seidel value from the pre-divided weights as two
// independent products pairs (dependency depth 3), then over-relaxation.
__device__ __forceinline__ double sor_point(const double2 ew, const double2 ns, double uE, double uW,
                                            double uN, double uS, double uc, double omega) {
    const double gs = fma(ew.x, uE, ew.y * uW) + fma(ns.x, uN, ns.y * uS);
    return fma(omega, gs - uc, uc);
}

// ---- bulk copies (K3s): cp.async.bulk global -> shared, completion on an
// mbarrier (transaction bytes), one elected thread issuing
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SDDG_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SDDG_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// K3s ring: per stage the (aE, aW) and (aN, aS) pairs of kStreamChunk slots
// of one colour, streamed from the job's packed weights in global memory
// (L2-resident) while the previous stage is being swept.
constexpr int kStreamChunk = 1024;  // slots per stage (a multiple of kSolveThreads)
constexpr size_t kStreamRingBytes = 2 * 2 * kStreamChunk * sizeof(double2);

template <int METHOD, int PTS, int G = 1, bool STREAM = false>
__global__ void __launch_bounds__(kSolveThreads)
solve_kernel(const double* __restrict__ wg, int gnx, double ihx2, double ihy2,
             const SolveJob* __restrict__ jobs, const double* __restrict__ bc, double tol,
             int64_t max_iters_cfg, int init_blend, const double* __restrict__ omegas,
             const int* __restrict__ perm, double* __restrict__ uout,
             sddg_solve_info* __restrict__ info, double* __restrict__ coef_scratch,
             int64_t coef_stride, int coef_in_smem, int* err) {
    extern __shared__ double smem[];
    __shared__ double red[kSolveThreads / 32];
    // job of this CTA: perm (longest expected solves first) or the batch order
    const int jq = perm ? perm[blockIdx.x] : static_cast<int>(blockIdx.x);
    const SolveJob J = jobs[jq];
    const double omega = omegas[jq];  // per-job SOR factor (sor_omega_kernel)
    const int nx = J.nx, ny = J.ny;
    const int N = nx * ny;
    double* u = smem;
    double* cE;
    double* cN;
    double* inv;
    if (coef_in_smem) {
        cE = smem + ((N + 1) & ~1);  // 16-B aligned (RB-SOR reads it as double2)
        cN = cE + N;
        inv = cN + N;
    } else {
        cE = coef_scratch + blockIdx.x * coef_stride;
        cN = cE + N;
        inv = cN + N;
    }
    const double* B = bc + J.bc_off;
    const double* T = B + nx;
    const double* L = T + nx;
    const double* Rt = L + ny;
    const int tid = threadIdx.x, nt = blockDim.x;

    const int mi = nx - 2, mj = ny - 2;
    const int half = (mi + 1) / 2;  // RB-SOR: colour slots per row
    const int nslots = mj * half;
    if (METHOD == 1) {
        // RB-SOR: per colour, per slot (j-1)*half + s, the four neighbour
        // weights of point (i, j) pre-divided by the diagonal, (aE, aW) and
        // (aN, aS): a coalesced 32 B per update instead of five scattered
        // reads of cE/cN/inv_den.  Same half-point weights as the reference
        // (detsolver.cpp:88-111); the pre-division only moves the rounding of
        // the fixed point by an ulp.
        double2* PQ = reinterpret_cast<double2*>(cE);
        for (int q = tid; q < 2 * nslots; q += nt) {
            const int colour = q / nslots, r = q - colour * nslots;
            const int j = r / half + 1, i = 2 * (r % half) + 1 + ((j + 1 + colour) & 1);
            if (i > mi) continue;
            sor_weights(wg, gnx, J, i, j, ihx2, ihy2, PQ[colour * 2 * nslots + r],
                        PQ[colour * 2 * nslots + nslots + r]);
        }
    }
    // coefficients from the global weights (detsolver.cpp:88-111)
    for (int c = tid; METHOD == 0 && c < N; c += nt) {
        const int i = c % nx, j = c / nx;
        const double wc = wg[(int64_t)(J.j0 + j) * gnx + (J.i0 + i)];
        cE[c] = i + 1 < nx ? 0.5 * (wc + wg[(int64_t)(J.j0 + j) * gnx + (J.i0 + i + 1)]) : 0.0;
        cN[c] = j + 1 < ny ? 0.5 * (wc + wg[(int64_t)(J.j0 + j + 1) * gnx + (J.i0 + i)]) : 0.0;
    }
    __syncthreads();
    for (int c = tid; METHOD == 0 && c < N; c += nt) {
        const int i = c % nx, j = c / nx;
        inv[c] = (i > 0 && j > 0 && i + 1 < nx && j + 1 < ny)
                     ? 1.0 / ((cE[c] + cE[c - 1]) * ihx2 + (cN[c] + cN[c - nx]) * ihy2)
                     : 0.0;
    }
    // boundary range (exact min/max, order free)
    double lmin = DBL_MAX, lmax = -DBL_MAX;
    for (int k = tid; k < 2 * (nx + ny); k += nt) {
        const double v = B[k];  // B, T, L, Rt are contiguous
        lmin = v < lmin ? v : lmin;
        lmax = lmax < v ? v : lmax;
    }
    const double bmax = BlockMax::reduce(lmax, red);
    const double bmin = -BlockMax::reduce(-lmin, red);
    // initial guess (detsolver.cpp:121-148)
    for (int c = tid; c < N; c += nt)
        u[c] = initial_value(c % nx, c / nx, nx, ny, B, T, L, Rt, bmin, bmax, init_blend);
    // K3s: the ring after u, its two mbarriers, and the first two chunks
    __shared__ uint64_t bars[2];
    double2* ring = reinterpret_cast<double2*>(smem + ((N + 1) & ~1));
    const int nchunk = (nslots + kStreamChunk - 1) / kStreamChunk;
    const double2* PQg = reinterpret_cast<const double2*>(cE);
    int64_t kc = 0;  // chunks consumed so far (all sweeps): stage kc & 1, phase (kc >> 1) & 1
    auto issue_chunk = [&](int64_t k, int stage) {
        const int seq = static_cast<int>(k % (2 * nchunk));
        const int colour = seq / nchunk, cix = seq - colour * nchunk;
        const int q0 = cix * kStreamChunk;
        const int cnt = min(kStreamChunk, nslots - q0);
        const uint32_t bytes = static_cast<uint32_t>(cnt) * sizeof(double2);
        const double2* src = PQg + colour * 2 * nslots + q0;
        double2* dst = ring + stage * 2 * kStreamChunk;
        mbar_expect_tx(&bars[stage], 2 * bytes);
        bulk_g2s(dst, src, bytes, &bars[stage]);
        bulk_g2s(dst + kStreamChunk, src + nslots, bytes, &bars[stage]);
    };
    if constexpr (STREAM) {
        // the packed weights were written through the generic proxy: order
        // them before the bulk copies (async proxy) read them
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (tid == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) {
            issue_chunk(0, 0);
            issue_chunk(1, 1);
        }
    }
    __syncthreads();

    const int64_t max_iters =
        max_iters_cfg > 0 ? max_iters_cfg : 200LL * (nx > ny ? nx : ny) * (nx > ny ? nx : ny);
    int64_t iters = 0;
    double upd = 0.0;
    StopRule stop;
    // rounding floor of the update: 1024 ulps of the boundary range
    const double noise = 1024.0 * DBL_EPSILON * fmax(fmax(fabs(bmin), fabs(bmax)), DBL_MIN);
    bool conv = false;
    // colour passes: METHOD 0 one pass over all interior points; METHOD 1
    // two passes (i+j even, then odd) updated in place.
    // this thread's first slot and the per-iteration slot step (no divisions
    // in the sweep)
    const int j_first = tid / half + 1, s_first = tid % half;
    const int dj = nt / half, ds = nt % half;
    while (iters < max_iters) {
        ++iters;
        double lupd = 0.0;
        if (METHOD == 0) {
            // two-phase in-place Jacobi: every thread reads the old iterate
            // for its PTS points, barrier, then writes them
            double nu[PTS];
#pragma unroll
            for (int k = 0; k < PTS; ++k) {
                const int p = tid + k * nt;
                if (p < mi * mj) {
                    const int c = (p / mi + 1) * nx + (p % mi + 1);
                    const double xp = (cE[c] * u[c + 1] + cE[c - 1] * u[c - 1]) * ihx2;
                    const double yp = (cN[c] * u[c + nx] + cN[c - nx] * u[c - nx]) * ihy2;
                    nu[k] = (xp + yp) * inv[c];
                    const double du = fabs(nu[k] - u[c]);
                    lupd = lupd < du ? du : lupd;
                }
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < PTS; ++k) {
                const int p = tid + k * nt;
                if (p < mi * mj) u[(p / mi + 1) * nx + (p % mi + 1)] = nu[k];
            }
        } else if constexpr (STREAM) {
            // K3s: the packed weights stream through a two-stage shared-memory
            // ring (cp.async.bulk, one elected thread; mbarrier completion),
            // kStreamChunk slots of one colour per stage; thread t sweeps
            // slots t, t + nt, ... of each chunk in order
#pragma unroll 1
            for (int colour = 0; colour < 2; ++colour) {
                int j = j_first, sl = s_first;
#pragma unroll 1
                for (int cix = 0; cix < nchunk; ++cix, ++kc) {
                    const int stage = static_cast<int>(kc & 1);
                    mbar_wait(&bars[stage], static_cast<uint32_t>((kc >> 1) & 1));
                    const double2* P = ring + stage * 2 * kStreamChunk;
                    const double2* Q = P + kStreamChunk;
                    const int lim = nslots - cix * kStreamChunk;
#pragma unroll 2
                    for (int q = tid; q < kStreamChunk && q < lim; q += nt) {
                        const int i = 2 * sl + 1 + ((j + 1 + colour) & 1);
                        if (i <= mi) {
                            const int c = j * nx + i;
                            const double uc = u[c];
                            const double nv = sor_point(P[q], Q[q], u[c + 1], u[c - 1], u[c + nx], u[c - nx], uc,
                                                        omega);
                            const double du = fabs(nv - uc);
                            lupd = lupd < du ? du : lupd;
                            u[c] = nv;
                        }
                        sl += ds;
                        j += dj;
                        if (sl >= half) {
                            sl -= half;
                            ++j;
                        }
                    }
                    __syncthreads();  // stage consumed; the colour's points published
                    if (tid == 0) issue_chunk(kc + 2, stage);
                }
            }
        } else {
#pragma unroll 1
            for (int colour = 0; colour < 2; ++colour) {
                const double2* P = reinterpret_cast<const double2*>(cE) + colour * 2 * nslots;
                const double2* Q = P + nslots;
                int j = j_first, sl = s_first;
                // groups of G slots: all coefficient loads of a group issue
                // before its shared-memory stores (the compiler may not move
                // loads of the possibly-aliased coefficient pointer past a
                // store), so G L2 round trips overlap instead of serialising
                for (int q0 = tid; q0 < nslots; q0 += G * nt) {
                    double2 ew[G], ns[G];
                    int cc[G];
#pragma unroll
                    for (int k = 0; k < G; ++k) {
                        const int q = q0 + k * nt;
                        const int i = 2 * sl + 1 + ((j + 1 + colour) & 1);
                        cc[k] = (q < nslots && i <= mi) ? j * nx + i : -1;
                        if (cc[k] >= 0) {
                            ew[k] = P[q];
                            ns[k] = Q[q];
                        }
                        sl += ds;
                        j += dj;
                        if (sl >= half) {
                            sl -= half;
                            ++j;
                        }
                    }
#pragma unroll
                    for (int k = 0; k < G; ++k) {
                        const int c = cc[k];
                        if (c < 0) continue;
                        const double uc = u[c];
                        const double nv =
                            sor_point(ew[k], ns[k], u[c + 1], u[c - 1], u[c + nx], u[c - nx], uc, omega);
                        const double du = fabs(nv - uc);
                        lupd = lupd < du ? du : lupd;
                        u[c] = nv;
                    }
                }
                __syncthreads();
            }
        }
        upd = BlockMax::reduce(lupd, red);  // includes the barrier publishing u
        if (stop.done(upd, iters, tol, METHOD == 1, omega, noise)) {
            conv = true;
            break;
        }
    }
    if constexpr (STREAM) {
        // the two chunks still in flight land before the CTA leaves
        mbar_wait(&bars[kc & 1], static_cast<uint32_t>((kc >> 1) & 1));
        mbar_wait(&bars[(kc + 1) & 1], static_cast<uint32_t>(((kc + 1) >> 1) & 1));
    }
    __syncthreads();
    // maximum principle (detsolver.cpp:191-198) and write-out
    const double slack = 1e-12 * (1.0 + fabs(bmin) + fabs(bmax));
    double* U = uout + J.u_off;
    for (int c = tid; c < N; c += nt) {
        const int i = c % nx, j = c / nx;
        const double v = u[c];
        if (i > 0 && j > 0 && i + 1 < nx && j + 1 < ny && (v < bmin - slack || v > bmax + slack))
            atomicCAS(err, 0, 4);
        U[c] = v;
    }
    if (tid == 0) {
        sddg_solve_info r;
        r.iterations = iters;
        r.final_update = upd;
        r.converged = conv ? 1 : 0;
        r.reserved = 0;
        info[jq] = r;
    }
}

template <int METHOD, int PTS, int G = 1, bool STREAM = false>
cudaError_t launch_one(int grid, int threads, size_t smem, cudaStream_t st, const double* wg,
                       int gnx, double ihx2, double ihy2, const SolveJob* jobs, const double* bc,
                       double tol, int64_t mi, int init_blend, const double* omega, const int* perm, double* u,
                       sddg_solve_info* info, double* scratch, int64_t cstride, int cin,
                       int* err) {
    auto k = solve_kernel<METHOD, PTS, G, STREAM>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k<<<grid, threads, smem, st>>>(wg, gnx, ihx2, ihy2, jobs, bc, tol, mi, init_blend, omega, perm, u,
                                   info, scratch, cstride, cin, err);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3c: RB-SOR for jobs whose weights do not fit next to u in one SM's shared
// memory (129^2 blocks of configs 3 and 4): one thread-block cluster of CL
// CTAs per job ("one subdomain per thread block group").  CTA r owns a strip
// of interior rows with one halo row on each side; its u strip and the
// packed weights of its rows live in its own shared memory for the whole
// solve, so the sweeps never touch L2.  After each colour the strip's edge
// rows (that colour's points only) are stored into the neighbours' halo rows
// through distributed shared memory, and a cluster barrier publishes them.
// The per-sweep maximum update is all-gathered the same way, so every CTA
// takes the same convergence decision (the K3 stopping rule).
#ifndef SDDG_K3C_THREADS
#define SDDG_K3C_THREADS 256
#endif
#ifndef SDDG_K3C_G
#define SDDG_K3C_G 1
#endif
constexpr int kClusterThreads = SDDG_K3C_THREADS;
// slots per thread whose loads (weights and the five u values) are all issued
// before their updates: points of one colour never read one another, so a
// group's loads overlap instead of serialising on each update's store
constexpr int kClusterG = SDDG_K3C_G;
#ifndef SDDG_K3C_MAXK
#define SDDG_K3C_MAXK 8
#endif
constexpr int kK3cMaxK = SDDG_K3C_MAXK;  // K3c fast path: slots per thread and colour
#ifndef SDDG_K3C_FAST_G
#define SDDG_K3C_FAST_G 1
#endif
constexpr int kK3cFastG = SDDG_K3C_FAST_G;  // points per load group (divides kK3cMaxK)
// per-sweep maximum slots: one per (rank, warp), up to 8 ranks x 32 warps
constexpr int kClusterSlots = 8 * 32;

// shared-memory doubles of one CTA: u strip (per + 2 rows), the packed weights
// (2 colours x 2 double2 per slot, per * half slots), CL maximum slots
__host__ __device__ inline int64_t cluster_smem_doubles(int nx, int ny, int cl) {
    const int mj = ny - 2, half = (nx - 1) / 2;
    const int per = (mj + cl - 1) / cl;
    return ((static_cast<int64_t>(per + 2) * nx + 1) & ~1LL) + 8LL * per * half + kClusterSlots;
}

// Distributed shared memory through explicit shared::cluster addresses: a
// generic store into a peer CTA forces the cluster barrier's release to a
// GPU-scope fence (MEMBAR.ALL.GPU); these keep it at cluster scope.
__device__ __forceinline__ uint32_t cluster_addr(const void* p, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(r)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_st_f64(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
#ifdef SDDG_K3C_RELAXED_BARRIER  // A/B measurement of the fence cost only: not a valid ordering
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
#else
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#endif
}

template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kClusterThreads)
solve_cluster_kernel(const double* __restrict__ wg, int gnx, double ihx2, double ihy2,
                     const SolveJob* __restrict__ jobs, const double* __restrict__ bc, double tol,
                     int64_t max_iters_cfg, int init_blend, const double* __restrict__ omegas,
                     const int* __restrict__ perm, double* __restrict__ uout,
                     sddg_solve_info* __restrict__ info, int per_cap, int* err) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    extern __shared__ double smem[];
    __shared__ double red[kClusterThreads / 32];
    const int jq = perm ? perm[blockIdx.x / CL] : static_cast<int>(blockIdx.x / CL);
    const SolveJob J = jobs[jq];
    const double omega = omegas[jq];
    const int nx = J.nx, ny = J.ny, mi = nx - 2, mj = ny - 2;
    const int half = (mi + 1) / 2;
    const int per = (mj + CL - 1) / CL;
    const int ra = 1 + rank * per;                     // first interior row of the strip
    const int rb = min(1 + (rank + 1) * per, ny - 1);  // one past the last
    const int rows = rb > ra ? rb - ra : 0;
    const int nsl = rows * half;                       // slots per colour
    const int cap = per_cap * half;
    double* us = smem;  // local row lr = j - (ra - 1), rows ra-1 .. rb
    double2* PQ = reinterpret_cast<double2*>(smem + (((per_cap + 2) * nx + 1) & ~1));
    double* slots = reinterpret_cast<double*>(PQ + 4 * cap);
    const double* B = bc + J.bc_off;
    const double* T = B + nx;
    const double* L = T + nx;
    const double* Rt = L + ny;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (int q = tid; q < 2 * nsl; q += nt) {
        const int colour = q / nsl, r = q - colour * nsl;
        const int j = ra + r / half, i = 2 * (r % half) + 1 + ((j + 1 + colour) & 1);
        if (i > mi) continue;
        sor_weights(wg, gnx, J, i, j, ihx2, ihy2, PQ[colour * 2 * cap + r], PQ[colour * 2 * cap + cap + r]);
    }
    double lmin = DBL_MAX, lmax = -DBL_MAX;
    for (int k = tid; k < 2 * (nx + ny); k += nt) {
        const double v = B[k];
        lmin = v < lmin ? v : lmin;
        lmax = lmax < v ? v : lmax;
    }
    const double bmax = BlockMax::reduce(lmax, red);
    const double bmin = -BlockMax::reduce(-lmin, red);
    for (int c = tid; c < (rows + 2) * nx; c += nt) {
        const int j = ra - 1 + c / nx, i = c % nx;
        us[c] = initial_value(i, j, nx, ny, B, T, L, Rt, bmin, bmax, init_blend);
    }
    // neighbours' strips: my first row is rank-1's top halo, my last row
    // rank+1's bottom halo (same shared-memory layout in every CTA)
    const bool has_below = rank > 0, has_above = rank + 1 < CL && rb < ny - 1;
    const int below_row = per + 1;  // local index of row ra in rank-1's strip
    // the neighbours' u strips in the cluster window: my local point c of
    // strip row 0 is rank-1's point c + (below_row - 1) nx, of strip row
    // rows-1 rank+1's point c - rows nx (its halo row 0)
    const uint32_t below_us = has_below ? cluster_addr(us, rank - 1) : 0u;
    const uint32_t above_us = has_above ? cluster_addr(us, rank + 1) : 0u;
    cluster.sync();

    const int64_t max_iters =
        max_iters_cfg > 0 ? max_iters_cfg : 200LL * (nx > ny ? nx : ny) * (nx > ny ? nx : ny);
    int64_t iters = 0;
    double upd = 0.0;
    StopRule stop;
    // rounding floor of the update: 1024 ulps of the boundary range
    const double noise = 1024.0 * DBL_EPSILON * fmax(fmax(fabs(bmin), fabs(bmax)), DBL_MIN);
    bool conv = false;
    const int l_first = tid / half, s_first = tid % half;
    const int dl = nt / half, ds = nt % half;
    // per-sweep maximum update: every warp stores its maximum into its own
    // slot (rank, warp) of every CTA; after the barrier each thread takes the
    // exact maximum of the CL * nwarps slots.  A slot is rewritten only after
    // the next sweep's first barrier, which every reader passes after reading.
    const int nwarps = nt >> 5;
    double* wslot = slots + rank * nwarps + (tid >> 5);
    // Fast path (every thread owns at most kK3cMaxK slots per colour, e.g.
    // 129^2 in 4 strips of 256 threads: 8): the shared-memory offset of each
    // owned point and its edge-row flags are computed once, so a point update
    // is its loads, the stencil, one store and no index arithmetic.
    const int kslots = (nsl + nt - 1) / nt;
    if (kslots <= kK3cMaxK) {
        int cof[2][kK3cMaxK];
        unsigned edge_lo = 0u, edge_hi = 0u;  // bit colour*kK3cMaxK + k: store to below / above
#pragma unroll
        for (int colour = 0; colour < 2; ++colour) {
#pragma unroll
            for (int k = 0; k < kK3cMaxK; ++k) {
                const int q = tid + k * nt;
                const int lr = q / half, sl = q - lr * half;
                const int i = 2 * sl + 1 + ((ra + lr + 1 + colour) & 1);
                const bool ok = k < kslots && q < nsl && i <= mi;
                cof[colour][k] = ok ? (lr + 1) * nx + i : -1;
                if (ok && lr == 0 && has_below) edge_lo |= 1u << (colour * kK3cMaxK + k);
                if (ok && lr == rows - 1 && has_above) edge_hi |= 1u << (colour * kK3cMaxK + k);
            }
        }
        while (iters < max_iters) {
            ++iters;
            double lupd = 0.0;
#pragma unroll
            for (int colour = 0; colour < 2; ++colour) {
                const double2* P = PQ + colour * 2 * cap;
                const double2* Q = P + cap;
                // groups of kK3cFastG points: all their loads first (points of
                // one colour never read one another), then the updates
#pragma unroll
                for (int k0 = 0; k0 < kK3cMaxK; k0 += kK3cFastG) {
                    double2 ew[kK3cFastG], ns[kK3cFastG];
                    double ue[kK3cFastG], uw[kK3cFastG], un[kK3cFastG], usn[kK3cFastG], uc[kK3cFastG];
#pragma unroll
                    for (int g = 0; g < kK3cFastG; ++g) {
                        const int c = cof[colour][k0 + g];
                        if (c < 0) continue;
                        const int q = tid + (k0 + g) * nt;
                        ew[g] = P[q];
                        ns[g] = Q[q];
                        uc[g] = us[c];
                        ue[g] = us[c + 1];
                        uw[g] = us[c - 1];
                        un[g] = us[c + nx];
                        usn[g] = us[c - nx];
                    }
#pragma unroll
                    for (int g = 0; g < kK3cFastG; ++g) {
                        const int c = cof[colour][k0 + g];
                        if (c < 0) continue;
                        const double nv = sor_point(ew[g], ns[g], ue[g], uw[g], un[g], usn[g], uc[g], omega);
                        const double du = fabs(nv - uc[g]);
                        lupd = lupd < du ? du : lupd;
                        us[c] = nv;
                        const unsigned bit = 1u << (colour * kK3cMaxK + k0 + g);
                        if (edge_lo & bit)
                            cluster_st_f64(below_us + 8u * static_cast<uint32_t>(c + (below_row - 1) * nx), nv);
                        if (edge_hi & bit)
                            cluster_st_f64(above_us + 8u * static_cast<uint32_t>(c - rows * nx), nv);
                    }
                }
                if (colour == 1) {
                    double m = lupd;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double v = __shfl_xor_sync(0xffffffffu, m, o);
                        m = m < v ? v : m;
                    }
                    if ((tid & 31) == 0) {
#pragma unroll
                        for (int r = 0; r < CL; ++r) cluster_st_f64(cluster_addr(wslot, r), m);
                    }
                }
                cluster_barrier();
            }
            upd = slots[0];
            for (int k = 1; k < CL * nwarps; ++k) upd = upd < slots[k] ? slots[k] : upd;
            if (stop.done(upd, iters, tol, true, omega, noise)) {
                conv = true;
                break;
            }
        }
    }
    while (!conv && kslots > kK3cMaxK && iters < max_iters) {
        ++iters;
        double lupd = 0.0;
#pragma unroll 1
        for (int colour = 0; colour < 2; ++colour) {
            const double2* P = PQ + colour * 2 * cap;
            const double2* Q = P + cap;
            int lr = l_first, sl = s_first;
            for (int q0 = tid; q0 < nsl; q0 += kClusterG * nt) {
                double2 ew[kClusterG], ns[kClusterG];
                double ue[kClusterG], uw[kClusterG], un[kClusterG], usn[kClusterG], uc[kClusterG];
                int cc[kClusterG], ll[kClusterG];
#pragma unroll
                for (int k = 0; k < kClusterG; ++k) {
                    const int q = q0 + k * nt;
                    const int j = ra + lr;
                    const int i = 2 * sl + 1 + ((j + 1 + colour) & 1);
                    cc[k] = (q < nsl && i <= mi) ? (lr + 1) * nx + i : -1;
                    ll[k] = lr;
                    if (cc[k] >= 0) {
                        const int c = cc[k];
                        ew[k] = P[q];
                        ns[k] = Q[q];
                        uc[k] = us[c];
                        ue[k] = us[c + 1];
                        uw[k] = us[c - 1];
                        un[k] = us[c + nx];
                        usn[k] = us[c - nx];
                    }
                    sl += ds;
                    lr += dl;
                    if (sl >= half) {
                        sl -= half;
                        ++lr;
                    }
                }
#pragma unroll
                for (int k = 0; k < kClusterG; ++k) {
                    if (cc[k] < 0) continue;
                    const double nv = sor_point(ew[k], ns[k], ue[k], uw[k], un[k], usn[k], uc[k], omega);
                    const double du = fabs(nv - uc[k]);
                    lupd = lupd < du ? du : lupd;
                    us[cc[k]] = nv;
                    // an edge row's point also into the neighbour's halo row: the
                    // neighbour reads only the other colour's halo points during
                    // this colour, and the cluster barrier publishes it
                    if (ll[k] == 0 && has_below)
                        cluster_st_f64(below_us + 8u * static_cast<uint32_t>(cc[k] + (below_row - 1) * nx), nv);
                    if (ll[k] == rows - 1 && has_above)
                        cluster_st_f64(above_us + 8u * static_cast<uint32_t>(cc[k] - rows * nx), nv);
                }
            }
            if (colour == 1) {
                double m = lupd;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double v = __shfl_xor_sync(0xffffffffu, m, o);
                    m = m < v ? v : m;
                }
                if ((tid & 31) == 0) {
#pragma unroll
                    for (int r = 0; r < CL; ++r) cluster_st_f64(cluster_addr(wslot, r), m);
                }
            }
            cluster_barrier();
        }
        upd = slots[0];
        for (int k = 1; k < CL * nwarps; ++k) upd = upd < slots[k] ? slots[k] : upd;
        if (stop.done(upd, iters, tol, true, omega, noise)) {
            conv = true;
            break;
        }
    }
    // maximum principle (detsolver.cpp:191-198) and write-out of my rows
    // (rank 0 adds boundary row 0, the last strip row ny-1)
    const double slack = 1e-12 * (1.0 + fabs(bmin) + fabs(bmax));
    double* U = uout + J.u_off;
    const int lo = rank == 0 ? 0 : 1, hi = rb == ny - 1 ? rows + 2 : rows + 1;
    for (int c = lo * nx + tid; c < hi * nx; c += nt) {
        const int lr = c / nx, i = c % nx, j = ra - 1 + lr;
        const double v = us[c];
        if (i > 0 && j > 0 && i + 1 < nx && j + 1 < ny && (v < bmin - slack || v > bmax + slack))
            atomicCAS(err, 0, 4);
        U[static_cast<int64_t>(j) * nx + i] = v;
    }
    if (rank == 0 && tid == 0) {
        sddg_solve_info r;
        r.iterations = iters;
        r.final_update = upd;
        r.converged = conv ? 1 : 0;
        r.reserved = 0;
        info[jq] = r;
    }
    cluster.sync();  // no CTA leaves while a neighbour may still store into it
}

template <int CL>
cudaError_t launch_cluster(int64_t n_jobs, int max_nx, int max_ny, cudaStream_t st, const double* wg,
                           int gnx, double ihx2, double ihy2, const SolveJob* jobs, const double* bc,
                           double tol, int64_t mi, int init_blend, const double* omega, const int* perm, double* u,
                           sddg_solve_info* info, int* err) {
    const size_t smem = sizeof(double) * static_cast<size_t>(cluster_smem_doubles(max_nx, max_ny, CL));
    auto k = solve_cluster_kernel<CL>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int per_cap = (max_ny - 2 + CL - 1) / CL;
    k<<<static_cast<unsigned>(n_jobs * CL), kClusterThreads, smem, st>>>(
        wg, gnx, ihx2, ihy2, jobs, bc, tol, mi, init_blend, omega, perm, u, info, per_cap, err);
    return cudaGetLastError();
}

// Per-job RB-SOR factor.  The optimal factor of a consistently ordered
// operator is 2/(1+sqrt(1-rJ^2)), rJ the spectral radius of its Jacobi
// iteration: the largest eigenvalue of Off v = r D v (D the diagonal, Off the
// neighbour weights, detsolver.cpp:88-111).  One Rayleigh quotient
// r = v.Off v / v.D v with the constant-coefficient ground mode
// v = sin(pi i/(nx-1)) sin(pi j/(ny-1)) estimates it from below (to within
// 1e-6 on config 3's shock-layer blocks, where the grid formula's factor
// 1.952 against the optimal 1.966 takes 1,260 instead of ~700 sweeps).  For
// constant weights v is the exact ground mode and the factor is the grid
// formula 2/(1+sin(pi/(n-1))).  One CTA per job, fixed-order reduction: K3,
// K3c and K3b read the same factor.
constexpr int kOmegaThreads = 256;

__global__ void __launch_bounds__(kOmegaThreads)
sor_omega_kernel(const double* __restrict__ wg, int gnx, double ihx2, double ihy2,
                 const SolveJob* __restrict__ jobs, double* __restrict__ omegas) {
    __shared__ double red[2][kOmegaThreads / 32];
    const SolveJob J = jobs[blockIdx.x];
    const int nx = J.nx, ny = J.ny, mi = nx - 2, mj = ny - 2;
    const double rx = nx - 1, ry = ny - 1;  // divisors
    double num = 0.0, den = 0.0;
    for (int q = threadIdx.x; q < mi * mj; q += blockDim.x) {
        const int i = 1 + q % mi, j = 1 + q / mi;
        const double* wr = wg + (int64_t)(J.j0 + j) * gnx + (J.i0 + i);
        const double wc = wr[0];
        const double ce = 0.5 * (wc + wr[1]) * ihx2, cw = 0.5 * (wr[-1] + wc) * ihx2;
        const double cn = 0.5 * (wc + wr[gnx]) * ihy2, cs = 0.5 * (wr[-gnx] + wc) * ihy2;
        // sinpi(k / (n-1)) is exactly 0 at k = 0 and k = n-1, so the
        // boundary neighbours drop out of the quotient
        const double si = sinpi(i / rx), sj = sinpi(j / ry);
        const double v = si * sj;
        const double off = sj * (ce * sinpi((i + 1) / rx) + cw * sinpi((i - 1) / rx)) +
                           si * (cn * sinpi((j + 1) / ry) + cs * sinpi((j - 1) / ry));
        num = fma(v, off, num);
        den = fma(v * v, (ce + cw) + (cn + cs), den);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = num;
        red[1][wid] = den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            a += red[0][k];
            b += red[1][k];
        }
        const double r = a / b;
        double om;
        if (r > 0.0 && r < 1.0) {
            om = 2.0 / (1.0 + sqrt((1.0 - r) * (1.0 + r)));
        } else {  // degenerate job (no interior, or non-finite weights): grid formula
            om = 2.0 / (1.0 + sinpi(1.0 / (max(nx, ny) - 1)));
        }
        omegas[blockIdx.x] = om;
    }
}

}  // namespace

cudaError_t launch_sor_omega(const double* w_global, int gnx, double hx, double hy, int64_t n_jobs,
                             const SolveJob* jobs, double* omegas, cudaStream_t s) {
    if (n_jobs <= 0) return cudaSuccess;
    const double ihx2 = 1.0 / (hx * hx), ihy2 = 1.0 / (hy * hy);
    sor_omega_kernel<<<static_cast<unsigned>(n_jobs), kOmegaThreads, 0, s>>>(w_global, gnx, ihx2, ihy2,
                                                                           jobs, omegas);
    return cudaGetLastError();
}

namespace {
// rank of job i = number of jobs ordered before it (larger factor first,
// ties by index): a permutation, O(n^2) over a few thousand jobs at most
__global__ void __launch_bounds__(256) order_jobs_kernel(const double* __restrict__ omegas, int n,
                                                         int* __restrict__ perm) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double oi = omegas[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
        const double oj = omegas[j];
        rank += (oj > oi || (oj == oi && j < i)) ? 1 : 0;
    }
    perm[rank] = i;
}
}  // namespace

cudaError_t launch_order_jobs(const double* omegas, int64_t n_jobs, int* perm, cudaStream_t s) {
    if (n_jobs <= 0) return cudaSuccess;
    const int n = static_cast<int>(n_jobs);
    order_jobs_kernel<<<(n + 255) / 256, 256, 0, s>>>(omegas, n, perm);
    return cudaGetLastError();
}

int solver_max_points() { return kSolveThreads * 32; }

int solver_cluster_size(int max_nx, int max_ny) {
    if (std::getenv("SDDG_NO_CLUSTER_SOLVER")) return 0;
    const int mj = max_ny - 2;
    const char* force = std::getenv("SDDG_CLUSTER_SIZE");  // A/B: smallest allowed size at least this
    const int cl_min = force ? std::atoi(force) : 2;
    for (int cl : {2, 4, 8}) {
        if (cl < cl_min) continue;
        const int per = (mj + cl - 1) / cl;
        if (sizeof(double) * cluster_smem_doubles(max_nx, max_ny, cl) <= 227 * 1024 &&
            (cl - 1) * per < mj && per >= 2)  // every strip non-empty
            return cl;
    }
    return 0;
}

cudaError_t launch_solve_cluster(const double* w_global, int gnx, double hx, double hy,
                                 int64_t n_jobs, const SolveJob* jobs, const double* bc, double tol,
                                 int64_t max_iters_cfg, int init_blend, const double* omega, const int* perm, double* u,
                                 sddg_solve_info* info, int* err, cudaStream_t s, int max_nx,
                                 int max_ny, int cl) {
    if (n_jobs <= 0) return cudaSuccess;
    const double ihx2 = 1.0 / (hx * hx), ihy2 = 1.0 / (hy * hy);
    switch (cl) {
        case 2: return launch_cluster<2>(n_jobs, max_nx, max_ny, s, w_global, gnx, ihx2, ihy2, jobs, bc,
                                         tol, max_iters_cfg, init_blend, omega, perm, u, info, err);
        case 4: return launch_cluster<4>(n_jobs, max_nx, max_ny, s, w_global, gnx, ihx2, ihy2, jobs, bc,
                                         tol, max_iters_cfg, init_blend, omega, perm, u, info, err);
        case 8: return launch_cluster<8>(n_jobs, max_nx, max_ny, s, w_global, gnx, ihx2, ihy2, jobs, bc,
                                         tol, max_iters_cfg, init_blend, omega, perm, u, info, err);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_solve_batch(const double* w_global, int gnx, double hx, double hy,
                               int64_t n_jobs, const SolveJob* jobs, const double* bc,
                               double tol, int64_t max_iters_cfg, int init_blend, int method,
                               const double* omega, const int* perm, double* u, sddg_solve_info* info, int* err,
                               cudaStream_t s, int max_n, int max_interior, double* coef_scratch,
                               int coef_in_smem) {
    if (n_jobs <= 0) return cudaSuccess;
    const double ihx2 = 1.0 / (hx * hx);
    const double ihy2 = 1.0 / (hy * hy);
    // Jacobi: u + cE, cN, inv_den (3 N); RB-SOR: u + 4 packed weights per slot (<= 4 N)
    const int ncoef = method == SDDG_SOLVER_RBSOR ? 4 : 3;
    const size_t smem = sizeof(double) * (static_cast<size_t>(max_n) * (coef_in_smem ? 1 + ncoef : 1) + 1);
    const int64_t cstride = static_cast<int64_t>(ncoef) * max_n;
    const int grid = static_cast<int>(n_jobs);
    const int T = kSolveThreads;
    // K3s (opt-in, SDDG_SOLVER_STREAM=1): the weights streamed through a
    // shared-memory ring by bulk copies.  Bit-identical to K3 but slower on
    // the 2048 x 129^2 batch (59 vs 40 ms): next to u's 133 KB the ring gets
    // 64 KB, one 32-KB stage in flight while the other is swept, against the
    // 64 KB that K3's 512 threads keep in flight with 4 slots of L2 loads each.
    const size_t smem_stream = sizeof(double) * ((static_cast<size_t>(max_n) + 1) & ~size_t(1)) + kStreamRingBytes;
    const char* stream_env = std::getenv("SDDG_SOLVER_STREAM");
    if (method == SDDG_SOLVER_RBSOR && !coef_in_smem && smem_stream <= 227 * 1024 && stream_env &&
        stream_env[0] == '1')
        return launch_one<1, 1, 1, true>(grid, T, smem_stream, s, w_global, gnx, ihx2, ihy2, jobs, bc, tol,
                                         max_iters_cfg, init_blend, omega, perm, u, info, coef_scratch,
                                         cstride, coef_in_smem, err);
    if (method == SDDG_SOLVER_RBSOR)
        return coef_in_smem
                   ? launch_one<1, 1, 1>(grid, T, smem, s, w_global, gnx, ihx2, ihy2, jobs, bc, tol,
                                         max_iters_cfg, init_blend, omega, perm, u, info, coef_scratch,
                                         cstride, coef_in_smem, err)
                   : launch_one<1, 1, 4>(grid, T, smem, s, w_global, gnx, ihx2, ihy2, jobs, bc, tol,
                                         max_iters_cfg, init_blend, omega, perm, u, info, coef_scratch,
                                         cstride, coef_in_smem, err);
    const int pts = (max_interior + T - 1) / T;
#define SDDG_J(P)                                                                             \
    if (pts <= P)                                                                             \
        return launch_one<0, P>(grid, T, smem, s, w_global, gnx, ihx2, ihy2, jobs, bc, tol,   \
                                max_iters_cfg, init_blend, omega, perm, u, info, coef_scratch,      \
                                cstride, coef_in_smem, err);
    SDDG_J(1) SDDG_J(2) SDDG_J(4) SDDG_J(8) SDDG_J(16) SDDG_J(32)
#undef SDDG_J
    return cudaErrorInvalidValue;
}

}  // namespace sddg

// ---------------------------------------------------------------------------
// K3b: one large subdomain (or single-domain grid) that does not fit in
// shared memory: a cooperative persistent kernel over the whole grid with
// grid-wide barriers between half-sweeps, u / cE / cN / inv_den in global
// memory (L2-resident for the BASELINE sizes: 513^2 x 4 arrays = 8.4 MB).
// Same arithmetic, stopping rule and max-principle check as K3.
#include <cooperative_groups.h>

namespace sddg {

namespace {

__device__ __forceinline__ double grid_max(double v, double* red, unsigned long long* slot) {
    // block max -> one atomicMax per block on the (non-negative) bit pattern
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, v, o);
        v = v < u ? u : v;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) m = m < red[k] ? red[k] : m;
        atomicMax(slot, static_cast<unsigned long long>(__double_as_longlong(m)));
    }
    return 0.0;
}

template <int METHOD>
__global__ void __launch_bounds__(256)
solve_large_kernel(const double* __restrict__ wg, int gnx, double ihx2, double ihy2, SolveJob J,
                   const double* __restrict__ bc, double tol, int64_t max_iters_cfg, int init_blend,
                   const double* __restrict__ omegas, double* __restrict__ u, double* __restrict__ v,
                   double* __restrict__ cE, double* __restrict__ cN, double* __restrict__ inv,
                   unsigned long long* slots, sddg_solve_info* info, int* err) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[8];
    const double omega = *omegas;
    const int nx = J.nx, ny = J.ny, N = nx * ny;
    const double* B = bc + J.bc_off;
    const double* T = B + nx;
    const double* L = T + nx;
    const double* Rt = L + ny;
    const long long gtid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long gstride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long c = gtid; c < N; c += gstride) {
        const int i = static_cast<int>(c % nx), j = static_cast<int>(c / nx);
        const double wc = wg[(int64_t)(J.j0 + j) * gnx + (J.i0 + i)];
        cE[c] = i + 1 < nx ? 0.5 * (wc + wg[(int64_t)(J.j0 + j) * gnx + (J.i0 + i + 1)]) : 0.0;
        cN[c] = j + 1 < ny ? 0.5 * (wc + wg[(int64_t)(J.j0 + j + 1) * gnx + (J.i0 + i)]) : 0.0;
    }
    // boundary range via the slots (min stored negated)
    double lmin = DBL_MAX, lmax = -DBL_MAX;
    for (long long k = gtid; k < 2 * (nx + ny); k += gstride) {
        lmin = B[k] < lmin ? B[k] : lmin;
        lmax = lmax < B[k] ? B[k] : lmax;
    }
    grid.sync();
    for (long long c = gtid; c < N; c += gstride) {
        const int i = static_cast<int>(c % nx), j = static_cast<int>(c / nx);
        inv[c] = (i > 0 && j > 0 && i + 1 < nx && j + 1 < ny)
                     ? 1.0 / ((cE[c] + cE[c - 1]) * ihx2 + (cN[c] + cN[c - nx]) * ihy2)
                     : 0.0;
    }
    // max over a signed range needs an order-preserving key: slots[3] = max(-min), slots[4] = max
    {
        double a = -lmin, b = lmax;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ua = __shfl_xor_sync(0xffffffffu, a, o), ub = __shfl_xor_sync(0xffffffffu, b, o);
            a = a < ua ? ua : a;
            b = b < ub ? ub : b;
        }
        auto key = [](double x) {  // monotone double -> u64
            const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
            return (bits >> 63) ? ~bits : (bits | 0x8000000000000000ull);
        };
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&slots[3], key(a));
            atomicMax(&slots[4], key(b));
        }
    }
    grid.sync();
    auto unkey = [](unsigned long long k) {
        const unsigned long long bits = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        return __longlong_as_double(static_cast<long long>(bits));
    };
    const double bmin = -unkey(slots[3]);
    const double bmax = unkey(slots[4]);
    for (long long c = gtid; c < N; c += gstride) {
        const int i = static_cast<int>(c % nx), j = static_cast<int>(c / nx);
        double val;
        if (init_blend) {
            const double ty = static_cast<double>(j) / (ny - 1);
            const double tx = static_cast<double>(i) / (nx - 1);
            const double xb = (1.0 - tx) * L[j] + tx * Rt[j];
            const double yb = (1.0 - ty) * B[i] + ty * T[i];
            const double bil = ((1.0 - tx) * (1.0 - ty) * B[0] + tx * ty * T[nx - 1]) +
                               (tx * (1.0 - ty) * B[nx - 1] + (1.0 - tx) * ty * T[0]);
            val = xb + yb - bil;
            val = val < bmin ? bmin : (bmax < val ? bmax : val);
        } else {
            val = 0.5 * (bmin + bmax);
        }
        if (j == 0) val = B[i];
        if (j == ny - 1) val = T[i];
        if (i == 0) val = L[j];
        if (i == nx - 1) val = Rt[j];
        u[c] = val;
        v[c] = val;
    }
    grid.sync();
    const int mi = nx - 2, mj = ny - 2;
    const int64_t max_iters =
        max_iters_cfg > 0 ? max_iters_cfg : 200LL * (nx > ny ? nx : ny) * (nx > ny ? nx : ny);
    int64_t iters = 0;
    double upd = 0.0;
    StopRule stop;
    // rounding floor of the update: 1024 ulps of the boundary range
    const double noise = 1024.0 * DBL_EPSILON * fmax(fmax(fabs(bmin), fabs(bmax)), DBL_MIN);
    bool conv = false;
    double* cur = u;
    double* nxt = v;
    const int half = (mi + 1) / 2;
    while (iters < max_iters) {
        ++iters;
        double lupd = 0.0;
        if (METHOD == 0) {
            for (long long p = gtid; p < static_cast<long long>(mi) * mj; p += gstride) {
                const long long c = (p / mi + 1) * nx + (p % mi + 1);
                const double xp = (cE[c] * cur[c + 1] + cE[c - 1] * cur[c - 1]) * ihx2;
                const double yp = (cN[c] * cur[c + nx] + cN[c - nx] * cur[c - nx]) * ihy2;
                const double nu = (xp + yp) * inv[c];
                nxt[c] = nu;
                const double du = fabs(nu - cur[c]);
                lupd = lupd < du ? du : lupd;
            }
        } else {
            for (int colour = 0; colour < 2; ++colour) {
                for (long long p = gtid; p < static_cast<long long>(mj) * half; p += gstride) {
                    const int j = static_cast<int>(p / half) + 1;
                    const int i = 2 * static_cast<int>(p % half) + 1 + ((j + 1 + colour) & 1);
                    if (i > mi) continue;
                    const long long c = static_cast<long long>(j) * nx + i;
                    const double xp = (cE[c] * cur[c + 1] + cE[c - 1] * cur[c - 1]) * ihx2;
                    const double yp = (cN[c] * cur[c + nx] + cN[c - nx] * cur[c - nx]) * ihy2;
                    const double gs = (xp + yp) * inv[c];
                    const double nv = cur[c] + omega * (gs - cur[c]);
                    const double du = fabs(nv - cur[c]);
                    lupd = lupd < du ? du : lupd;
                    cur[c] = nv;
                }
                if (colour == 0) grid.sync();
            }
        }
        const int s = static_cast<int>(iters % 3);
        grid_max(lupd, red, &slots[s]);
        grid.sync();
        upd = __longlong_as_double(static_cast<long long>(slots[s]));
        if (gtid == 0) slots[(s + 2) % 3] = 0ull;  // next-but-one iteration's slot
        if (METHOD == 0) {
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
        if (stop.done(upd, iters, tol, METHOD == 1, omega, noise)) {
            conv = true;
            break;
        }
    }
    grid.sync();
    const double slack = 1e-12 * (1.0 + fabs(bmin) + fabs(bmax));
    for (long long c = gtid; c < N; c += gstride) {
        const int i = static_cast<int>(c % nx), j = static_cast<int>(c / nx);
        const double val = cur[c];
        if (i > 0 && j > 0 && i + 1 < nx && j + 1 < ny && (val < bmin - slack || val > bmax + slack))
            atomicCAS(err, 0, 4);
        u[c] = val;  // result in u (cur may be v after an odd Jacobi count)
    }
    if (gtid == 0) {
        sddg_solve_info r;
        r.iterations = iters;
        r.final_update = upd;
        r.converged = conv ? 1 : 0;
        r.reserved = 0;
        *info = r;
    }
}

}  // namespace

// Solves one job with the cooperative kernel; scratch holds 5*N doubles + 8 slots.
cudaError_t launch_solve_large(const double* w_global, int gnx, double hx, double hy,
                               const SolveJob& job, const double* bc, double tol,
                               int64_t max_iters_cfg, int init_blend, int method, const double* omega,
                               double* u_out, sddg_solve_info* info, int* err, double* scratch,
                               cudaStream_t s, int sms) {
    const double ihx2 = 1.0 / (hx * hx);
    const double ihy2 = 1.0 / (hy * hy);
    const long long N = static_cast<long long>(job.nx) * job.ny;
    double* u = scratch;
    double* v = u + N;
    double* cE = v + N;
    double* cN = cE + N;
    double* inv = cN + N;
    unsigned long long* slots = reinterpret_cast<unsigned long long*>(inv + N);
    cudaMemsetAsync(slots, 0, 8 * sizeof(unsigned long long), s);
    void* fn = method == SDDG_SOLVER_JACOBI ? reinterpret_cast<void*>(solve_large_kernel<0>)
                                          : reinterpret_cast<void*>(solve_large_kernel<1>);
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, 256, 0);
    if (e != cudaSuccess) return e;
    const long long need = (N + 255) / 256;
    int grid = static_cast<int>(std::min<long long>(static_cast<long long>(bps) * sms, std::max<long long>(1, need)));
    SolveJob J = job;
    void* args[] = {(void*)&w_global, (void*)&gnx, (void*)&ihx2, (void*)&ihy2, (void*)&J, (void*)&bc,
                    (void*)&tol, (void*)&max_iters_cfg, (void*)&init_blend, (void*)&omega,
                    (void*)&u, (void*)&v, (void*)&cE, (void*)&cN, (void*)&inv, (void*)&slots,
                    (void*)&info, (void*)&err};
    e = cudaLaunchCooperativeKernel(fn, grid, 256, args, 0, s);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(u_out + job.u_off, u, sizeof(double) * N, cudaMemcpyDeviceToDevice, s);
}

}  // namespace sddg
