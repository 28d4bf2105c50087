// reduce.cu -- K2: fixed chunk-order Monte Carlo finalize.
//
// Reference: mc_estimate (proj/src/sde.cpp:201-245).  Walks are summed in
// walk order within 256-walk chunks (f, g, f*f, g*g each rounded separately),
// chunk sums in chunk order, then mean, (n-1)-variance stderr, restarts and
// the >1% reliability warning.  One CTA per node: thread t sums chunk
// (tile*256 + t) sequentially; thread 0 then folds the tile's chunk sums in
// order.  Explicit __dadd_rn/__dmul_rn keep the reference's rounding sequence
// regardless of contraction flags.
#include "sddg_internal.h"

namespace sddg {

constexpr int kReduceThreads = 256;

__global__ void __launch_bounds__(kReduceThreads)
reduce_kernel(const double* __restrict__ rf, const double* __restrict__ rg,
              const uint32_t* __restrict__ meta, int64_t walks, const uint32_t* __restrict__ perm,
              const unsigned long long* __restrict__ node_steps, sddg_estimate* out,
              const GatherTargets gt) {
    __shared__ double part[4][kReduceThreads];
    __shared__ unsigned long long icnt[5][kReduceThreads / 32];
    const int64_t node = blockIdx.x;
    const int t = threadIdx.x;
    const int64_t base = node * walks;
    const int64_t n_chunks = (walks + kChunk - 1) / kChunk;
    double tf = 0.0, tg = 0.0, tff = 0.0, tgg = 0.0;  // thread 0 only
    unsigned long long restarts = 0, h0 = 0, h1 = 0, h2 = 0, h3 = 0;
    for (int64_t tile = 0; tile < n_chunks; tile += kReduceThreads) {
        const int64_t c = tile + t;
        double sf = 0.0, sg = 0.0, sff = 0.0, sgg = 0.0;
        if (c < n_chunks) {
            const int64_t lo = c * kChunk;
            const int64_t hi = walks < lo + kChunk ? walks : lo + kChunk;
            for (int64_t w = lo; w < hi; ++w) {
                const double f = rf[base + w], g = rg[base + w];
                const uint32_t m = meta[base + w];
                sf = __dadd_rn(sf, f);
                sg = __dadd_rn(sg, g);
                sff = __dadd_rn(sff, __dmul_rn(f, f));
                sgg = __dadd_rn(sgg, __dmul_rn(g, g));
                restarts += m >> 2;
                const uint32_t e = m & 3u;
                h0 += e == 0u;
                h1 += e == 1u;
                h2 += e == 2u;
                h3 += e == 3u;
            }
        }
        part[0][t] = sf;
        part[1][t] = sg;
        part[2][t] = sff;
        part[3][t] = sgg;
        __syncthreads();
        if (t == 0) {
            const int64_t lim = n_chunks - tile < kReduceThreads ? n_chunks - tile : kReduceThreads;
            for (int i = 0; i < lim; ++i) {
                tf = __dadd_rn(tf, part[0][i]);
                tg = __dadd_rn(tg, part[1][i]);
                tff = __dadd_rn(tff, part[2][i]);
                tgg = __dadd_rn(tgg, part[3][i]);
            }
        }
        __syncthreads();
    }
    // integer counters: order-free block reduction
    unsigned long long v[5] = {restarts, h0, h1, h2, h3};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if ((t & 31) == 0) icnt[k][t >> 5] = v[k];
    }
    __syncthreads();
    if (t == 0) {
        unsigned long long s[5] = {0, 0, 0, 0, 0};
        for (int k = 0; k < 5; ++k)
            for (int w = 0; w < kReduceThreads / 32; ++w) s[k] += icnt[k][w];
        sddg_estimate e;
        const double n = static_cast<double>(walks);
        e.walks = walks;
        e.xi = __ddiv_rn(tf, n);
        e.eta = __ddiv_rn(tg, n);
        e.se_xi = 0.0;
        e.se_eta = 0.0;
        if (walks > 1) {
            // std::max(0.0, v) = (0.0 < v) ? v : 0.0
            double vf = __ddiv_rn(__dadd_rn(tff, -__dmul_rn(__dmul_rn(n, e.xi), e.xi)), __dadd_rn(n, -1.0));
            double vg = __ddiv_rn(__dadd_rn(tgg, -__dmul_rn(__dmul_rn(n, e.eta), e.eta)), __dadd_rn(n, -1.0));
            vf = 0.0 < vf ? vf : 0.0;
            vg = 0.0 < vg ? vg : 0.0;
            e.se_xi = __dsqrt_rn(__ddiv_rn(vf, n));
            e.se_eta = __dsqrt_rn(__ddiv_rn(vg, n));
        }
        e.restarts = static_cast<int64_t>(s[0]);
        e.warn = e.restarts > walks / 100 ? 1 : 0;
        e.reserved = 0;
        for (int k = 0; k < 4; ++k) e.edge_hits[k] = static_cast<int64_t>(s[1 + k]);
        e.sum_f = tf;
        e.sum_g = tg;
        e.sum_ff = tff;
        e.sum_gg = tgg;
        const uint32_t k = perm ? perm[node] : static_cast<uint32_t>(node);
        // executed path-steps of the node's walks (K1's per-node counter)
        e.path_steps = node_steps ? static_cast<int64_t>(node_steps[k]) : 0;
        out[k] = e;
        // fused all-gather: store the finished record straight into every
        // rank's gather buffer (NVLink peer memory opened through CUDA IPC)
        if (gt.n_peers > 0) {
            const int64_t slot = gt.global_index ? gt.global_index[k] : static_cast<int64_t>(k);
#pragma unroll 1
            for (int p = 0; p < gt.n_peers; ++p) gt.peers[p][slot] = e;
        }
    }
}

cudaError_t launch_reduce(const double* rf, const double* rg, const uint32_t* meta,
                          int64_t walks, int64_t n_nodes, const uint32_t* perm,
                          const unsigned long long* node_steps, sddg_estimate* out,
                          cudaStream_t s, const GatherTargets& gt) {
    if (n_nodes <= 0) return cudaSuccess;
    reduce_kernel<<<static_cast<unsigned>(n_nodes), kReduceThreads, 0, s>>>(rf, rg, meta, walks, perm,
                                                                            node_steps, out, gt);
    return cudaGetLastError();
}

}  // namespace sddg
