// walk_tail.cuh -- K1t, the tail kernel: the last walks of a batch, one warp
// per walk.  Included by walk_kernel.cuh after K1 (it uses K1's step, exit
// and record functions, so both kernels compute every step bit for bit alike).
//
// Why: a batch ends with its longest walks, which then run alone on a nearly
// empty GPU at the latency of one step's dependent chain (Philox, Box-Muller
// and drift in sequence: 344 ns per step in performance mode, 1.62 us in the
// reference-parity mode, tools/probe_latency.py; config 1's 20 ms walk phase
// spends ~10 ms there).  Once K1's batch counter has run out and at most
// cont_cap walks are in flight, K1 hands each remaining walk over at its next
// check point (walk_kernel.cuh, WalkCont), and this kernel finishes them with
// 32 lanes per walk:
//  * the window: lane l generates Philox block B0 + l of the walk's stream, so
//    64 consecutive u64 draws are available by shuffle; from them every lane
//    precomputes the step randoms (step_rand: Box-Muller, the Exp(lambda)
//    step) for the two draw positions it owns, whatever the alignment left by
//    data-dependent exit-test draws;
//  * the step itself runs redundantly on all lanes (warp-uniform state): the
//    randoms come by shuffle, so the sequential chain is drift + update +
//    exit test; the reference-mode central-difference drift evaluates its
//    five densities on five lanes at once;
//  * exit-test draws read the window (WindowStream), so they cost shuffles,
//    not Philox blocks.
// The arithmetic per step is the same functions as K1 on the same draws, so
// results do not depend on which kernel finished a walk.

namespace sddg {

constexpr int kTailWarps = 16;  // walks in flight per CTA (one warp each), one CTA per SM

// The warp's window of the walk's stream: lane l holds block B0 + l, i.e.
// u64 draws base + 2l (lo) and base + 2l + 1 (hi), base = 2 B0.
struct WindowStream {
    uint32_t n;     // u64s drawn in this epoch (warp-uniform)
    uint32_t base;  // first u64 of the window
    uint64_t lo, hi;
    // draw idx of the window, idx - base in [0, 64); idx may differ per lane
    __device__ __forceinline__ uint64_t word(uint32_t idx) const {
        const uint32_t k = idx - base;
        SDDG_CHECK(k < 64u);
        const int src = static_cast<int>((k >> 1) & 31u);
        const uint64_t a = __shfl_sync(0xffffffffu, lo, src);
        const uint64_t b = __shfl_sync(0xffffffffu, hi, src);
        return (k & 1u) ? b : a;
    }
    __device__ __forceinline__ uint64_t next_one(const RoundKeys&) { return word(n++); }
};

// Reference-mode central-difference drift (drift_ref, user_supplied kinds:
// monitor.cpp:206-219,231-240) with its five density evaluations on lanes
// 0-4 at once; every lane returns the same drift.
template <int DV>
__device__ __forceinline__ bool drift_ref_lanes(const DensityParams& P, double x, double y, double& bx,
                                                double& by) {
    const int lane = threadIdx.x & 31;
    const double h = P.fd_h, h2 = 2.0 * h;
    const double px = lane == 0 ? x + h : (lane == 1 ? x - h : x);
    const double py = lane == 2 ? y + h : (lane == 3 ? y - h : y);
    const double v = user_rho<DV>(P, px, py);
    const double rxp = __shfl_sync(0xffffffffu, v, 0), rxm = __shfl_sync(0xffffffffu, v, 1);
    const double ryp = __shfl_sync(0xffffffffu, v, 2), rym = __shfl_sync(0xffffffffu, v, 3);
    const double r = __shfl_sync(0xffffffffu, v, 4);
    const double gx = div_rn_shared(rxp - rxm, h2, P.fd_inv2h);
    const double gy = div_rn_shared(ryp - rym, h2, P.fd_inv2h);
    if (!isfinite(gx) || !isfinite(gy)) return false;
    const double yr = 1.0 / r;
    bx = -div_rn_shared(gx, r, yr);
    by = -div_rn_shared(gy, r, yr);
    return isfinite(bx) && isfinite(by);
}

template <int DV>
constexpr bool kFdDrift = DV == DV_RING_FD || DV == DV_SHOCK_FD || DV == DV_TWOBUMP_FD || DV == DV_TABLE_FD;

template <int DV, typename Real, int SCHEME>
__device__ __forceinline__ StepDrift<Real> tail_drift(const fm::FmTables& T, const DensityParams& P, Real dt,
                                                      Real x, Real y) {
    if constexpr (kFdDrift<DV>) {
        StepDrift<Real> d;
        d.c = Real(0);
        d.ok = drift_ref_lanes<DV>(P, x, y, d.vx, d.vy);
        return d;
    } else {
        return step_drift<DV, Real, SCHEME>(T, P, dt, x, y);
    }
}

template <int DV, typename Real, int SCHEME, bool BRIDGE>
__global__ void __launch_bounds__(kTailWarps * 32, 1) walk_tail_kernel(const __grid_constant__ WalkArgs a) {
    static_assert(sizeof(Real) == 8, "the tail kernel runs fp64 walks");
    const Dom<Real> dom{Real(a.xmin), Real(a.xmax), Real(a.ymin), Real(a.ymax),
                        Real(a.box[0]), Real(a.box[1]), Real(a.box[2]), Real(a.box[3]),
                        a.box_hi[0], a.box_hi[1], a.box_hi[2], a.box_hi[3]};
    const DensityParams P{a.R, a.alpha, a.fd_h, 1.0 / (2.0 * a.fd_h), a.tab, a.f_kd};
    const Real dt = Real(a.dt);
    const Real sq2dt = Real(a.sqrt2dt);
    const Real thr = Real(a.bridge_thr);
    const uint32_t max_steps = a.max_steps32;
    extern __shared__ double dyn_smem[];
    fm::FmTables& T = *reinterpret_cast<fm::FmTables*>(dyn_smem);
#ifdef SDDG_SMEM_ABS
    if constexpr (walk_uses_tables<DV, Real>()) {
        const uint32_t at = static_cast<uint32_t>(__cvta_generic_to_shared(dyn_smem));
        if (at != static_cast<uint32_t>(SDDG_SMEM_ABS)) {
            if (threadIdx.x == 0) {
                atomicCAS(a.err_flag, 0, 5);
                atomicExch(a.err_info, static_cast<unsigned long long>(at));
            }
            return;
        }
    }
#endif
    const uint32_t ncont = min(*reinterpret_cast<volatile unsigned int*>(a.n_cont), a.cont_cap);
    if (blockIdx.x >= ncont) return;
    if constexpr (walk_uses_tables<DV, Real>()) {
        const double2* src = reinterpret_cast<const double2*>(a.fm_tables);
        double2* dst = reinterpret_cast<double2*>(dyn_smem);
        for (int k = threadIdx.x; k < static_cast<int>(sizeof(fm::FmTables) / 16); k += blockDim.x)
            dst[k] = src[k];
        __syncthreads();
    }
    const uint32_t lane = threadIdx.x & 31;
    constexpr uint32_t kDraws = kStepDraws<SCHEME>;
    // the warp's step randoms of the current window, slot = draw offset: read
    // by every lane at one broadcast address (no shuffle, whose divergence
    // check and latency would sit on the step chain)
    StepRand<Real>* const rbuf = reinterpret_cast<StepRand<Real>*>(
                                     reinterpret_cast<char*>(dyn_smem) + walk_table_bytes<DV, Real>()) +
                                 64 * (threadIdx.x >> 5);
    // walks round-robin over the SMs first, then over the CTA's warps (warp w
    // issues on SM sub-partition w % 4): a tail of a few hundred walks runs one
    // walk per sub-partition, where a step costs its dependency chain (~230
    // clocks, tools/op_latency.cu), not four walks' share of the FP64 pipe
    for (uint32_t ci = (threadIdx.x >> 5) * gridDim.x + blockIdx.x; ci < ncont; ci += gridDim.x * kTailWarps) {
        const WalkCont c = a.cont[ci];
        const uint32_t node = c.node;
        SDDG_CHECK(ci < a.cont_cap && node < static_cast<uint64_t>(a.n_nodes) && c.g < a.total &&
                   c.step < max_steps && c.epoch < 1024u);
        const uint64_t pid = a.pid[node];
        Real x = Real(c.x), y = Real(c.y);
        uint32_t epoch = c.epoch, step = c.step, n = c.n;
        uint64_t extra = 0;  // steps of the epochs restarted here
        bool in_box = box_test<DV, Real>(dom, x, y);
        // the drift at the walk's position is computed one step ahead: right
        // after the update, before the exit test's branch, so its dependent
        // chain overlaps the step's bookkeeping and branches instead of
        // following them (a pure function of the position: values unchanged;
        // the speculative one at an exit position is never used)
        StepDrift<Real> sd = tail_drift<DV, Real, SCHEME>(T, P, dt, x, y);
        bool done = false;
        while (!done) {
            // ---- window: 32 Philox blocks of the stream (seed, pid, walk, epoch)
            const uint32_t c3 = static_cast<uint32_t>((pid >> 32) & 0xFFFFu) | (epoch << 16);
            const uint32_t base = n & ~1u;
            const PhiloxWords w = philox4x32_10(a.rk, (n >> 1) + lane, c.walk, static_cast<uint32_t>(pid), c3);
            WindowStream ws{n, base, join64(w.w0, w.w1), join64(w.w2, w.w3)};
            // this lane's step randoms at draw positions base + lane, base + lane + 32
            // (the last few positions run past the window: never used)
            __syncwarp();  // the previous window's reads are done
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t s0 = base + lane + 32u * e;
                const uint32_t lim = base + 63u;
                const uint64_t w0 = ws.word(min(s0, lim));
                const uint64_t w1 = ws.word(min(s0 + 1u, lim));
                const uint64_t w2 = kDraws > 2 ? ws.word(min(s0 + 2u, lim)) : 0ull;
                rbuf[lane + 32u * e] = step_rand<DV, Real, SCHEME>(T, a, sq2dt, w0, w1, w2);
            }
            __syncwarp();
            uint32_t k = ws.n - base;
            StepRand<Real> r = rbuf[k & 63u];
            // ---- steps while the window holds this step's draws and up to 4 exit-test draws
#ifndef SDDG_TAIL_UNROLL
#define SDDG_TAIL_UNROLL 1
#endif
            SDDG_UNROLL(SDDG_TAIL_UNROLL)
            while (k + kDraws + 4u <= 64u) {
                SDDG_CHECK(k < 64u);
                if (!sd.ok) {
                    if (lane == 0) {
                        atomicCAS(a.err_flag, 0, 3);  // EvaluationError
                        atomicExch(a.err_info, static_cast<unsigned long long>(pid));
                    }
                    done = true;
                    break;
                }
                Real nxp, nyp;
                step_update<DV, Real, SCHEME>(sd, r, dt, sq2dt, x, y, nxp, nyp);
                ws.n += kDraws;
                ++step;
                // the next step's randoms, assuming the exit test draws nothing
                // (k past the window: stale, and the loop refills instead)
                k = ws.n - base;
                StepRand<Real> rn = rbuf[k & 63u];
                const StepDrift<Real> sn = tail_drift<DV, Real, SCHEME>(T, P, dt, nxp, nyp);
                Real hx = Real(0), hy = Real(0);
                int edge = 0;
                bool nb;
                const Real wl = kLiteral<DV> ? sd.w : Real(1);
                const bool exited = exit_test<DV, Real, SCHEME, BRIDGE>(
                    dom, a, T, kLiteral<DV> ? thr * wl : thr, kLiteral<DV> ? dt * wl : dt, x, y, nxp, nyp, in_box,
                    ws, hx, hy, edge, nb);
                if (exited) {
                    if (lane == 0) {
                        record_exit<Real>(a, c.g, node, epoch, step, edge, hx, hy, max_steps);
                        atomicAdd(a.steps, static_cast<unsigned long long>(extra + step));
                    }
                    done = true;
                    break;
                }
                x = nxp;
                y = nyp;
                in_box = nb;
                sd = sn;
                if (ws.n - base != k) {  // the exit test drew: reload
                    k = ws.n - base;
                    rn = rbuf[k & 63u];
                }
                r = rn;
                if (step >= max_steps) {
                    // restart on the next epoch's stream (run_walk, sde.cpp:154-182)
                    extra += step;
                    if (++epoch >= 1024u) {
                        if (lane == 0) {
                            atomicCAS(a.err_flag, 0, 4);  // NumericalError
                            atomicExch(a.err_info, static_cast<unsigned long long>(pid));
                        }
                        done = true;
                        break;
                    }
                    x = Real(a.px[node]);
                    y = Real(a.py[node]);
                    in_box = box_test<DV, Real>(dom, x, y);
                    sd = tail_drift<DV, Real, SCHEME>(T, P, dt, x, y);
                    step = 0;
                    ws.n = 0;
                    break;  // new key: a new window
                }
            }
            n = ws.n;
        }
    }
}

template <int DV, typename Real, int SCHEME, bool BRIDGE>
cudaError_t launch_tail_one(const WalkArgs& a, cudaStream_t s) {
    constexpr size_t sm = walk_table_bytes<DV, Real>() + sizeof(StepRand<Real>) * 64 * kTailWarps;
    if constexpr (sm > 48 * 1024) {
        static std::atomic<bool> attr[64];
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_relaxed)) {
            const cudaError_t e = cudaFuncSetAttribute(walk_tail_kernel<DV, Real, SCHEME, BRIDGE>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(sm));
            if (e != cudaSuccess) return e;
            if (dev >= 0 && dev < 64) attr[dev].store(true, std::memory_order_relaxed);
        }
    }
    // one CTA per SM (cont_cap = 16 per SM by default); a larger cap queues
    // walks on a warp (strided over the continuations)
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = std::min<unsigned>(a.cont_cap, static_cast<unsigned>(sms));
    walk_tail_kernel<DV, Real, SCHEME, BRIDGE><<<grid, kTailWarps * 32, sm, s>>>(a);
    return cudaGetLastError();
}

}  // namespace sddg
