// sddg_internal.h -- kernel argument blocks and launcher declarations shared
// by the CUDA translation units and the host runtime.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/sddg.h"
#include "philox.cuh"
#include "table_density.h"

// Device-side bounds checks of a checked build (SDDG_CHECKS=1: build tag
// "chk", tools/checked_tests.sh).  compute-sanitizer is closed on the GPU
// pool (profiles/r02_compute_sanitizer_refused.log), so the indices each
// kernel derives from its inputs are asserted instead; a violation prints
// the condition and traps the kernel (SDDG_ERR_CUDA on the host).
#if defined(SDDG_CHECKS) && SDDG_CHECKS
#include <cstdio>
#define SDDG_CHECK(cond)                                                                        \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("SDDG_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);               \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define SDDG_CHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace sddg {

constexpr int kDrainBlock = 256;  // threads per CTA of a drain round (walk_kernel.cuh DRAIN)
constexpr int kWalkBlock = 128;   // threads per walk CTA
#ifndef SDDG_WALK_MIN_BLOCKS
#define SDDG_WALK_MIN_BLOCKS 8
#endif
constexpr int kWalkMinBlocks = SDDG_WALK_MIN_BLOCKS;  // >= 8 CTAs (32 warps) per SM: A/B best
constexpr int64_t kChunk = 256;   // reference mc_estimate chunk (proj/src/sde.cpp:201)

struct WalkArgs {
    // walk domain (sdd::RectDomain passed to mc_estimate)
    double xmin, xmax, ymin, ymax;
    // boundary tables (BoundaryData over the table grid)
    double txmin, tymin, thx, thy;
    int tnx, tny;
    const double* tf[4];
    const double* tg[4];
    // density
    double R, alpha, fd_h;
    TableDensity tab;  // SDDG_DENS_TABLE: padded samples in device memory
    // walk config
    int scheme, bridge;
    double dt, sqrt2dt, lambda, nu2, bridge_thr;
    double box[4];  // inner box x0, x1, y0, y1 (edge distances > sqrt(bridge_thr))
    // fp32 copies (fp32 walks read them from the constant bank instead of
    // converting the doubles in the step loop): xmin, xmax, ymin, ymax, box[4],
    // dt, sqrt2dt, bridge_thr
    float f_dom[8];
    float f_dt, f_sqrt2dt, f_thr;
    float f_kd;  // fp32 linear-scheme drift constant times dt: ring -8000 dt, shock 1/(-160 dt), two-bump -3000 dt
    int32_t box_hi[4];  // high words of box[] for the integer test (INT32_MAX: disabled)
    int32_t box_fi[4];  // bit patterns of f_dom[4..7]: the fp32 walks' integer box test (exact for a positive box)
    uint64_t seed;
    RoundKeys rk;
    uint32_t max_steps32;  // max_steps (validated <= 2^29)
    uint32_t chunk32;      // steps between K1 check points: max_steps, or (tail kernel) a divisor of it
    // batch: total = n_nodes * walks
    const double* px;
    const double* py;
    const uint64_t* pid;
    const uint32_t* perm;  // batch slot -> node (longest expected walks first), or null
    int64_t n_nodes;       // points px/py/pid/node_steps hold (checked builds)
    int64_t walks;
    int64_t walk_lo;
    uint64_t total;
    unsigned long long* next;   // global walk counter (starts at the grid size)
    unsigned long long* steps;  // executed path-steps
    unsigned long long* node_steps;  // per-node executed path-steps (all epochs), or null
    int* err_flag;              // 3 EvaluationError, 4 NumericalError
    unsigned long long* err_info;
    // outputs: per-walk records, or per-path dumps
    double* rec_f;
    double* rec_g;
    uint32_t* rec_meta;  // edge | epochs_used << 2
    sddg_path* dump;
    const void* fm_tables;  // fastmath.cuh FmTables in global memory (performance mode)
    // tail handoff (walk_tail.cuh): when the batch counter has run out and at
    // most cont_cap walks remain in flight (live), walks move to cont[] (null: off)
    struct WalkCont* cont;
    uint32_t cont_cap;
    unsigned int* n_cont;
    unsigned long long* live;
    // drain round (K1 resumed on a previous round's handoffs, packed 32 per
    // warp): src[0 .. min(*n_src, src_cap)); null: a fresh batch
    const struct WalkCont* src;
    const unsigned int* n_src;
    uint32_t src_cap;
    double inv_dt;          // 1/dt: performance-mode bridge exponent d0 d1 / dt as a multiply
    double half_inv_lambda; // 1/(2 lambda): performance-mode Exp(lambda) step from -2 ln u
};

// fastmath tables (host-built in long double, uploaded once per context)
void make_fm_tables(void* host_tables7680);

// walk_ref.cu (fp64, -fmad=false) and walk_fast.cu (analytic drifts, fp64 + fp32)
bool walk_variant_supported(int dv, int precision);
// block > 0: CTAs of that many threads (a drain round), else the variant's own
cudaError_t launch_walk(int dv, int precision, const WalkArgs& a, int grid, cudaStream_t s, int block = 0);
// the tail kernel of an fp64 walk batch (walk_tail.cuh), after launch_walk
cudaError_t launch_walk_tail(int dv, const WalkArgs& a, cudaStream_t s);
cudaError_t launch_walk_tail_ref(int dv, const WalkArgs& a, cudaStream_t s);
cudaError_t launch_walk_tail_fast(int dv, const WalkArgs& a, cudaStream_t s);
cudaError_t walk_occupancy(int dv, int precision, int* blocks_per_sm, int* block);
// the two TUs' own dispatchers
cudaError_t launch_walk_ref(int dv, const WalkArgs& a, int grid, cudaStream_t s, int block);
cudaError_t occupancy_walk_ref(int dv, int* b, int* block);
cudaError_t launch_walk_fast(int dv, int precision, const WalkArgs& a, int grid, cudaStream_t s, int block);
cudaError_t occupancy_walk_fast(int dv, int precision, int* b, int* block);

// reduce.cu: K2 fixed chunk-order finalize, one CTA per node; with peers,
// also the fused all-gather (each record stored into every rank's buffer)
constexpr int kMaxPeers = 16;
// A walk handed from K1 to the tail kernel: position, slot, stream position.
struct WalkCont {
    double x, y;
    uint64_t g;  // record slot
    uint32_t node, walk, epoch, step;
    uint32_t n;  // u64s drawn in this epoch
    uint32_t pad;
};
// walk_kernel.cuh: per-lane bookkeeping of the running walk (shared memory)
struct LaneState {
    uint64_t g;       // record slot of the running walk
    uint64_t steps;   // path steps finished by this lane
    uint32_t node, walk, epoch;
    uint32_t base;    // steps of the completed chunks of this epoch
};
struct GatherTargets {
    int n_peers;                     // 0: no fused gather
    const int64_t* global_index;     // local node k -> slot in the gather buffers (device); null: slot k
    sddg_estimate* peers[kMaxPeers];  // device pointers (local or IPC-mapped peer memory)
};
cudaError_t launch_reduce(const double* rf, const double* rg, const uint32_t* meta,
                          int64_t walks, int64_t n_nodes, const uint32_t* perm,
                          const unsigned long long* node_steps, sddg_estimate* out,
                          cudaStream_t s, const GatherTargets& gt);

// solver.cu: K3 batched Dirichlet solves
struct SolveJob {
    int i0, j0, nx, ny;
    int64_t bc_off;  // offset of bottom[nx] top[nx] left[ny] right[ny] in bc
    int64_t u_off;   // offset of the nx*ny solution
};
// coef_in_smem: cE/cN/inv_den in shared memory (4*max_n doubles of smem),
// else in coef_scratch (n_jobs * 3*max_n doubles).  max_interior <=
// solver_max_points() for METHOD Jacobi.
int solver_max_points();
// Per-job RB-SOR factor from a Rayleigh-quotient estimate of the job's Jacobi
// spectral radius (one CTA per job; writes omegas[0..n_jobs))
cudaError_t launch_sor_omega(const double* w_global, int gnx, double hx, double hy, int64_t n_jobs,
                             const SolveJob* jobs, double* omegas, cudaStream_t s);
// Launch order of the K3/K3c blocks: jobs by descending SOR factor (a larger
// factor means a slower-converging job), ties in batch order; perm[n_jobs]
cudaError_t launch_order_jobs(const double* omegas, int64_t n_jobs, int* perm, cudaStream_t s);
// perm (nullable): block b solves job perm[b]; info and omegas stay in job order
// K3c (thread-block-cluster RB-SOR): cluster size for jobs up to max_nx x
// max_ny whose packed weights do not fit next to u in one CTA (0: none fits)
int solver_cluster_size(int max_nx, int max_ny);
cudaError_t launch_solve_cluster(const double* w_global, int gnx, double hx, double hy,
                                 int64_t n_jobs, const SolveJob* jobs, const double* bc, double tol,
                                 int64_t max_iters_cfg, int init_blend, const double* omega,
                                 const int* perm, double* u, sddg_solve_info* info, int* err,
                                 cudaStream_t s, int max_nx,
                                 int max_ny, int cl);
// K3b: one grid too large for shared memory, cooperative kernel; scratch 5*N+8 doubles
cudaError_t launch_solve_large(const double* w_global, int gnx, double hx, double hy,
                               const SolveJob& job, const double* bc, double tol,
                               int64_t max_iters_cfg, int init_blend, int method, const double* omega,
                               double* u_out, sddg_solve_info* info, int* err, double* scratch,
                               cudaStream_t s, int sms);
cudaError_t launch_solve_batch(const double* w_global, int gnx, double hx, double hy,
                               int64_t n_jobs, const SolveJob* jobs, const double* bc,
                               double tol, int64_t max_iters_cfg, int init_blend, int method,
                               const double* omega, const int* perm, double* u, sddg_solve_info* info,
                               int* err, cudaStream_t s, int max_n, int max_interior, double* coef_scratch,
                               int coef_in_smem);

// smooth.cu: K6 Perona-Malik FTCS, K7 interface loess
cudaError_t pm_run(double* u0, double* u1, double* v0, double* v1, int nx, int ny,
                   const int* blocks_host, int nblocks, double hx, double hy, double k, double dt,
                   int steps, double* scratch, unsigned long long* dev_upd, double* upd_host,
                   cudaStream_t s);
size_t pm_scratch_doubles(const int* blocks_host, int nblocks);
cudaError_t loess_run(const double* d_in, double* d_out, int n, int span, int* d_err, cudaStream_t s);

// mesh.cu: K4 inversion, K5 quality
// scratch: invert_scratch_ints(m_xi, m_eta) ints (lattice and per-target triangles, row marks);
// err[0], err_row: error code and row; err[2], err[3]: rows the fix-up pass visited, targets it located again
size_t invert_scratch_ints(int m_xi, int m_eta);
cudaError_t launch_invert(const double* xi, const double* eta, int nx, int ny, double gx0,
                          double gy0, double ghx, double ghy, int m_xi, int m_eta, double* X,
                          double* Y, int* scratch, int* err, int* err_row, cudaStream_t s);
cudaError_t launch_quality(const double* X, const double* Y, int m_xi, int m_eta, double* qbuf,
                           double* out2, int* err, cudaStream_t s);
cudaError_t launch_linf(const double* X, const double* Y, const double* RX, const double* RY,
                        long long n, int kind, double R, double al, const TableDensity& tab,
                        unsigned long long* out_bits, cudaStream_t s);

cudaError_t probe_fma_tflops(int precision, int sms, cudaStream_t st, double* tflops);
cudaError_t probe_onchip_gbps(int sms, cudaStream_t st, double* l2_gbps, double* smem_gbps);
cudaError_t fastmath_selftest(int64_t n, const void* tables, unsigned long long* host_maxulp5);
cudaError_t division_selftest(int64_t n, unsigned long long* host_bad);
// walk_fast.cu: performance-mode drifts (fp64 table forms, fp32 SFU forms) and the
// fp32 radius argument against their definitions evaluated with the fp64 library
cudaError_t drift_selftest(int kind, int64_t n, const void* tables, const double box[4], double host_out[4]);

}  // namespace sddg
