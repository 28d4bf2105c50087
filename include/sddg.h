/*
 * sddg.h -- C-ABI of the B200-native stochastic domain decomposition (SDD)
 * mesh generator (arXiv 1310.3435), the drop-in boundary for the reference
 * sddmesh hot path.
 *
 * The reference (/root/reference/proj, C++20) has no FFI; its seams are C++
 * functions.  Each entry point below names the reference function it
 * replaces.  Plain pointers and sizes only; no torch or C++ types; never
 * throws.  Every call returns an sddg_status mirroring the reference's
 * exception classes (proj/include/sdd/errors.hpp:8-32); the message of the
 * last failure on a context is sddg_last_error().
 *
 * Library: paper_1310_3435_b200/_lib/libsddg.so (sm_100a only).  There is no
 * CPU fallback: without a usable B200 every compute entry point fails with
 * SDDG_ERR_CUDA.
 */
#ifndef SDDG_H
#define SDDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDDG_ABI_VERSION 2

typedef enum {
    SDDG_OK = 0,
    SDDG_ERR_VALIDATION = 1,    /* sdd::ValidationError  */
    SDDG_ERR_OUT_OF_DOMAIN = 2, /* sdd::OutOfDomainError */
    SDDG_ERR_EVALUATION = 3,    /* sdd::EvaluationError  */
    SDDG_ERR_NUMERICAL = 4,     /* sdd::NumericalError   */
    SDDG_ERR_LAYOUT = 5,        /* sdd::LayoutError      */
    SDDG_ERR_CUDA = 6,          /* no B200 / CUDA failure (no fallback) */
    SDDG_ERR_INTERNAL = 7,
    SDDG_ERR_INVERSION = 8,     /* sdd::InversionError   */
    SDDG_ERR_TANGLING = 9       /* sdd::TanglingError    */
} sddg_status;

/* Density descriptor.  A GPU cannot call the reference's std::function
 * density (proj/include/sdd/monitor.hpp:68), so densities are data.
 * Kinds 0-4 are the reference builtins given as rho
 * (proj/include/sdd/monitor.hpp:11-18, formulas proj/src/monitor.cpp:121-223).
 * Kinds 16-18 are the BASELINE.json densities given as the diffusion weight
 * w, which the reference receives as MonitorFunction::user_supplied(rho=1/w)
 * (proj/src/monitor.cpp:73-80).  Kind 32 carries ANY user_supplied density
 * as data: rho sampled on a tnx x tny grid over tdom, read through a fixed
 * interpolant -- Catmull-Rom bicubic (cubic convolution, a = -1/2) on the
 * grid padded by one linearly extrapolated node per side, so linear rho is
 * reproduced exactly and the drift is continuous.  In reference mode the
 * gradient is the reference's user_supplied central difference of that
 * interpolant (monitor.cpp:206-219); in performance mode its analytic
 * gradient. */
typedef enum {
    SDDG_DENS_CONSTANT = 0,
    SDDG_DENS_RUNNING = 1,
    SDDG_DENS_HUANG_SLOAN = 2,
    SDDG_DENS_MACKENZIE = 3,
    SDDG_DENS_FIVE_RING = 4,
    SDDG_DENS_RING_W = 16,   /* w = 1+10 exp(-200 ((x-.5)^2+(y-.5)^2-1/16)^2)     */
    SDDG_DENS_SHOCK_W = 17,  /* w = 1+20 sech^2(50 (y-.5-.15 sin 2 pi x))         */
    SDDG_DENS_TWOBUMP_W = 18, /* w = 1+15 e^{-100|x-(.3,.3)|^2}+15 e^{-100|x-(.7,.6)|^2} */
    SDDG_DENS_TABLE = 32      /* rho tabulated on a grid (table, tnx, tny, tdom)    */
} sddg_density_kind;

typedef enum {
    /* What the reference computes: the builtin analytic gradient for kinds
     * 0-4, the user_supplied central difference of rho = 1/w with step fd_h
     * for kinds 16-18 (proj/src/monitor.cpp:206-219). */
    SDDG_GRAD_REFERENCE = 0,
    /* Performance mode: analytic drift grad(w)/w for kinds 16-18 (BASELINE.json
     * configs), the five-ring (kind 4) with table-driven tanh, and the
     * interpolant's own gradient for kind 32; fastmath elementary functions,
     * fp64 or fp32, checked statistically. */
    SDDG_GRAD_ANALYTIC = 1
} sddg_grad_mode;

typedef struct {
    double xmin, xmax, ymin, ymax; /* sdd::RectDomain (geometry.hpp:27-46) */
} sddg_domain;

typedef struct {
    int32_t kind;      /* sddg_density_kind */
    int32_t grad_mode; /* sddg_grad_mode */
    double R, alpha;   /* builtin parameters (monitor.hpp:26-38) */
    double fd_h;       /* user_supplied FD step, reference default 1e-6 */
    /* SDDG_DENS_TABLE only: rho at the nodes of a tnx x tny grid over tdom
     * (index j*tnx + i, tnx, tny >= 2, finite and > 0); read during the
     * call, not retained */
    const double* table;
    int32_t tnx, tny;
    sddg_domain tdom;
} sddg_density;

/* sdd::BoundaryData (proj/include/sdd/boundary.hpp:12-18): Dirichlet tables
 * tabulated at the nodes of an nx x ny grid over dom; index 0..3 = bottom,
 * top, left, right (sdd::Edge, geometry.hpp:19); bottom/top have nx entries,
 * left/right ny.  f carries xi, g eta. */
typedef struct {
    sddg_domain dom;
    int32_t nx, ny;
    const double* f[4];
    const double* g[4];
} sddg_boundary;

typedef enum { SDDG_SCHEME_LINEAR = 0, SDDG_SCHEME_EXPONENTIAL = 1 } sddg_scheme;
typedef enum { SDDG_FP64 = 0, SDDG_FP32 = 1 } sddg_precision;

typedef enum {
    /* the reference's SDE (sde.cpp:21-29): drift grad(w)/w = -grad(rho)/rho,
     * noise sqrt(2 dt) z; generator (1/w) div(w grad).  Parity mode. */
    SDDG_FORM_REFERENCE = 0,
    /* BASELINE.json's literal SDE dX = grad(w) dt + sqrt(2 w) dW: generator
     * div(w grad), the reference's times w -- a time change, so the same
     * harmonic functions and exit law (estimates agree statistically, walks
     * take fewer steps where w > 1).  The bridge exponent becomes
     * d0 d1 / (w dt) with w at the step's start.  Opt-in: BASELINE weights
     * (kinds 16-18), analytic grad(w), linear scheme, fp64 or fp32. */
    SDDG_FORM_LITERAL = 1
} sddg_sde_form;

/* sdd::WalkConfig (proj/include/sdd/sde.hpp:16-26) + precision + SDE form. */
typedef struct {
    int32_t scheme;    /* sddg_scheme */
    int32_t precision; /* sddg_precision: FP32 walks keep fp64 sums (config 3) */
    double dt;         /* linear step */
    double lambda;     /* exponential rate */
    int64_t walks;     /* paths per node */
    uint64_t seed;
    int64_t max_steps; /* steps per epoch before a restart, 1..2^29 */
    int32_t bridge_test;
    int32_t form;      /* sddg_sde_form (0: the reference's) */
} sddg_walk_config;

/* sdd::McEstimate (proj/include/sdd/sde.hpp:61-68) + the raw fixed-order
 * sums and path_steps: the steps the node's walks executed, summed over all
 * epochs (a restarted walk counts its max_steps per failed epoch plus the
 * exit step index of its last, sde.cpp:154-176); counted on the GPU by one
 * atomic per finished walk. */
typedef struct {
    double xi, eta, se_xi, se_eta;
    int64_t walks, restarts;
    int32_t warn; /* reliability_warning: restarts > walks/100 */
    int32_t reserved;
    int64_t edge_hits[4];
    double sum_f, sum_g, sum_ff, sum_gg;
    int64_t path_steps;
} sddg_estimate;

/* One walk's result (the anonymous WalkResult, proj/src/sde.cpp:144-149,
 * plus the exit point). */
typedef struct {
    double f, g, ex, ey;
    int64_t steps;
    int32_t epoch, edge;
} sddg_path;

typedef struct sddg_ctx sddg_ctx;

/* ---------------------------------------------------------------- context */
const char* sddg_version(void);
int sddg_abi_version(void);
sddg_status sddg_device_count(int32_t* n);
/* Owns one device, its stream, device buffers and scratch; calls on one ctx
 * are serialised. */
sddg_status sddg_create(int32_t device, sddg_ctx** out);
void sddg_destroy(sddg_ctx* ctx);
const char* sddg_last_error(const sddg_ctx* ctx);
/* Path-steps executed, kernels launched and summed walk-kernel (K1) device
 * time of the last compute call (solver calls: the solve kernel's time). */
sddg_status sddg_last_stats(const sddg_ctx* ctx, int64_t* path_steps, int64_t* launches,
                            double* kernel_ms);

/* The walk batch's tail: walks handed from the walk kernel K1 to the tail
 * kernel (one warp per walk, fp64 only) and the tail kernel's device time of
 * the last walk call (included in sddg_last_stats' kernel time). */
sddg_status sddg_last_tail_stats(const sddg_ctx* ctx, int64_t* handoffs, double* tail_ms);

/* Measured non-tensor FMA peak of this device in TFLOP/s (independent
 * DFMA / FFMA chains on every SM), the denominator of the walk kernel's
 * pipe roofline. */
sddg_status sddg_probe_fma_peak(sddg_ctx* ctx, int32_t precision, double* tflops);

/* Measured on-chip read bandwidths of this device in GB/s: L2 (every SM
 * streaming a 64 MB L2-resident buffer) and shared memory (conflict-free
 * 16-B loads on every SM), the rooflines of the subdomain solver, whose
 * batches stay on chip. */
sddg_status sddg_probe_onchip_bandwidth(sddg_ctx* ctx, double* l2_gbps, double* smem_gbps);

/* Diagnostics: max ulp error over n sample points of the performance-mode
 * elementary functions (exp, log on (0, 0.9], sincos(2 pi u), sqrt, rcp)
 * against the CUDA library; slot 5: max ulp error of log on (0.9, 1). */
sddg_status sddg_selftest_fastmath(sddg_ctx* ctx, int64_t n, uint64_t max_ulp[6]);

/* Diagnostics: n operand pairs (random over the parity mode's guarded range,
 * quotients just below 1 with the dividend near the top of its binade,
 * operands outside the guard, zeros, subnormals) through the parity mode's
 * shared-reciprocal division; *mismatches = results that differ from the
 * library's correctly rounded a / b in any bit (expected 0). */
sddg_status sddg_selftest_division(sddg_ctx* ctx, int64_t n, uint64_t* mismatches);

/* Diagnostics: the performance-mode drifts grad(w)/w of a BASELINE density
 * (SDDG_DENS_RING_W, _SHOCK_W, _TWOBUMP_W) at n pseudo-random points of the
 * rectangle dom, against the density's definition evaluated with the fp64
 * library.  out[0]: max abs error of the fp64 table form; out[1]: of the fp32
 * SFU forms (as used by the exponential scheme, and with the host-precomputed
 * constant of the linear scheme); out[2]: max relative error of the fp32
 * walks' Box-Muller radius argument -2 ln u1; out[3]: max |drift| seen. */
sddg_status sddg_selftest_drift(sddg_ctx* ctx, int32_t kind, const sddg_domain* dom, int64_t n,
                                double out[4]);

/* ------------------------------------------------------------- walk seams */

/* Replaces the per-node loop of sdd::mc_estimate calls
 * (proj/include/sdd/sde.hpp:75-77, called at proj/src/decomposition.cpp:173
 * and proj/src/cli.cpp:261): one Feynman-Kac estimate per start point, walk w
 * of point k on the stream (seed, point_id[k], w) with the reference's 256-walk
 * chunk-order reduction.  Host buffers. */
sddg_status sddg_mc_estimate_batch(sddg_ctx* ctx, const sddg_density* dens,
                                   const sddg_domain* dom, const sddg_boundary* bd,
                                   const sddg_walk_config* cfg, const double* px,
                                   const double* py, const uint64_t* point_id, int64_t n,
                                   sddg_estimate* out);

/* Same with device-resident start points and output, enqueued on `stream`
 * (a cudaStream_t, or NULL for the context stream); returns after the
 * work completes. */
sddg_status sddg_mc_estimate_batch_device(sddg_ctx* ctx, const sddg_density* dens,
                                          const sddg_domain* dom, const sddg_boundary* bd,
                                          const sddg_walk_config* cfg, const double* d_px,
                                          const double* d_py, const uint64_t* d_point_id,
                                          int64_t n, sddg_estimate* d_out, void* stream);

/* ------------------------------------------------------ several GPUs
 * The reference parallelises solve_interfaces over interface nodes and
 * solve_sdd over subdomains with std::thread (proj/src/decomposition.cpp:
 * 171-174, 298-355).  A context may span several GPUs: every walk entry
 * point (sddg_mc_estimate_batch[_device], sddg_solve_interfaces,
 * sddg_solve_sdd, sddg_stochastic_full) then shards the nodes across the
 * ranks by expected cost (sddg_shard_plan), walks each shard on its GPU and
 * joins the 128-B records with ONE ncclAllGather; sddg_solve_sdd also splits
 * the subdomains into contiguous per-rank ranges and all-gathers the fields.
 * Every rank returns the complete result, bit-identical to a one-GPU
 * context (each node is reduced on one rank in the reference's chunk
 * order).  With one process per GPU every rank makes the same calls with the
 * same arguments (SPMD). */
typedef struct {
    unsigned char bytes[128]; /* ncclUniqueId */
} sddg_nccl_id;
/* Rank 0 creates the id and passes it to the other processes. */
sddg_status sddg_nccl_unique_id(sddg_nccl_id* id);
/* One process per GPU: this process is `rank` of `nranks` (ncclCommInitRank,
 * collective over all ranks).  nranks = 1 still runs the NCCL exchange. */
sddg_status sddg_create_dist(int32_t device, int32_t rank, int32_t nranks, const sddg_nccl_id* id,
                             sddg_ctx** out);
/* One process for n GPUs (one host thread per device).  Only the owner
 * (devices[0]) needs the records, so when every device can store into the
 * owner's memory (peer access over NVLink) the exchange is fused into the
 * reduce kernel: each finished record is written straight to the owner's
 * output through peer memory, with no collective.  Without peer access:
 * ncclCommInitAll and one all-gather (SDDG_TEAM_NCCL=1 forces this).  A
 * device listed twice runs as separate ranks on that device (the sharded
 * path on one GPU: fused stores, or device copies with SDDG_TEAM_COPY=1). */
sddg_status sddg_create_multi(int32_t n, const int32_t* devices, sddg_ctx** out);
/* This context's first global rank, the rank count, the GPUs this process
 * drives, and whether the exchange is NCCL (1) or peer stores / device
 * copies inside one process (0). */
sddg_status sddg_team_info(const sddg_ctx* ctx, int32_t* rank, int32_t* nranks,
                           int32_t* local_devices, int32_t* nccl);
/* Host: the node shard plan the sharded calls use.  cost[k] = expected
 * path-steps of node k's cfg->walks walks from the exit-time model (the
 * expected first-exit time T of the walk, div(w grad T) = -w, T = 0 on the
 * edges, over dt); rank_of[k] from longest-processing-time assignment. */
sddg_status sddg_shard_plan(const sddg_density* dens, const sddg_domain* dom,
                            const sddg_walk_config* cfg, const double* px, const double* py,
                            int64_t n, int32_t nranks, int32_t* rank_of, double* cost);

/* ------------------------------------------------ fused multi-GPU gather
 * The one collective of the sharded path (an all-gather of the per-node
 * records) fused into the finalize kernel K2: each rank opens every other
 * rank's gather buffer through CUDA IPC (NVLink peer memory on one box) and
 * K2 stores each finished record into all of them; a host barrier after the
 * call completes the exchange.  Replaces the NCCL all-gather of
 * paper_1310_3435_b200/parallel.py (transport="nccl"). */
typedef struct {
    unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} sddg_ipc_handle;
sddg_status sddg_gather_alloc(sddg_ctx* ctx, int64_t n_records, void** d_buf,
                              sddg_ipc_handle* handle);
sddg_status sddg_gather_open(sddg_ctx* ctx, const sddg_ipc_handle* handle, void** d_peer);
sddg_status sddg_gather_close(sddg_ctx* ctx, void* d_peer);
sddg_status sddg_gather_free(sddg_ctx* ctx, void* d_buf);
sddg_status sddg_gather_read(sddg_ctx* ctx, const void* d_buf, int64_t n_records,
                             sddg_estimate* out);
/* sddg_mc_estimate_batch for this rank's n nodes, whose records land at
 * slot global_index[k] of each of the n_peers gather buffers (own buffer
 * included; n_total slots each).  Returns after the stores complete. */
sddg_status sddg_mc_estimate_gather(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                    const sddg_boundary* bd, const sddg_walk_config* cfg,
                                    const double* px, const double* py, const uint64_t* point_id,
                                    const int64_t* global_index, int64_t n, void* const* peer_bufs,
                                    int32_t n_peers, int64_t n_total);

/* Per-path results of walks [walk_lo, walk_lo+n) at one start point: the
 * parity view of run_walk (proj/src/sde.cpp:151-183). */
sddg_status sddg_walk_dump(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                           const sddg_boundary* bd, const sddg_walk_config* cfg, double px,
                           double py, uint64_t point_id, int64_t walk_lo, int64_t n,
                           sddg_path* out);

/* ----------------------------------------------------------- solver seams */

typedef struct {
    int32_t i0, j0, nx, ny; /* sdd::Subdomain (decomposition.hpp:21-24) */
} sddg_subdomain;

typedef enum {
    SDDG_SOLVER_JACOBI = 0, /* the reference iteration (detsolver.cpp:150-189) */
    SDDG_SOLVER_RBSOR = 1   /* red-black SOR, same fixed point */
} sddg_solver_method;

/* sdd::SolverConfig (proj/include/sdd/detsolver.hpp:11-18) + method. */
typedef struct {
    double tol;
    int64_t max_iters; /* 0: 200 max(nx,ny)^2 */
    int32_t init_blend;
    int32_t method; /* sddg_solver_method */
    double omega;   /* SOR factor: > 0 as given; 0 estimates the optimal one per job
                       from its weights (Rayleigh quotient of the Jacobi operator);
                       < 0 the constant-coefficient formula 2/(1+sin(pi/(n-1))) */
} sddg_solver_config;

typedef struct {
    int64_t iterations;
    double final_update;
    int32_t converged;
    int32_t reserved;
} sddg_solve_info;

/* Replaces the per-subdomain sdd::solve_dirichlet calls
 * (proj/include/sdd/detsolver.hpp:44-45; proj/src/decomposition.cpp:349-350):
 * n_solves independent Dirichlet problems on blocks of the global weight
 * array w_global (gnx x gny, index j*gnx+i) with the global spacings hx, hy.
 * bc_packed holds, per solve, bottom[nx] top[nx] left[ny] right[ny] back to
 * back; u_packed receives each solution (nx*ny, index j*nx+i) back to back. */
sddg_status sddg_solve_dirichlet_batch(sddg_ctx* ctx, const double* w_global, int32_t gnx,
                                       int32_t gny, double hx, double hy, int64_t n_solves,
                                       const sddg_subdomain* subs, const double* bc_packed,
                                       const sddg_solver_config* scfg, double* u_packed,
                                       sddg_solve_info* info);

/* ---------------------------------------------------- decomposition seams */

typedef enum {
    SDDG_PLACE_ALL = 0,
    SDDG_PLACE_EQUISPACED = 1,
    SDDG_PLACE_OPTIMAL = 2,
    /* BASELINE.json config 4 (no reference oracle): k nodes per
     * line at the grid nodes nearest to equal shares of the trapezoid
     * integral of the weight w = 1/rho along the line. */
    SDDG_PLACE_EQUIDISTRIBUTED = 3
} sddg_placement; /* sdd::PlacementStrategy (decomposition.hpp:40) + config 4 */

typedef enum {
    SDDG_INTERP_LINEAR = 0, /* reference fill (decomposition.cpp:215-224) */
    SDDG_INTERP_SPLINE = 1  /* natural cubic spline through the known nodes (config 4, D6) */
} sddg_interp;

/* sdd::SddOptions (proj/include/sdd/decomposition.hpp:74-77) + fill mode. */
typedef struct {
    int32_t smooth_interface; /* loess pre-smoothing of the interface lines */
    int32_t smooth_span;      /* odd window, reference default 5 */
    int32_t interp;           /* sddg_interp */
    int32_t reserved;
} sddg_sdd_options;

typedef enum {
    SDDG_BC_REFERENCE = 0, /* make_boundary_data: 1D equidistribution (boundary.cpp:44-56) */
    SDDG_BC_IDENTITY = 1   /* xi = x, eta = y (BASELINE.json) */
} sddg_bc_mode;

/* Host: sdd::make_boundary_data (proj/src/boundary.cpp:44-56) into 8
 * caller arrays (f bottom,top,left,right; g bottom,top,left,right). */
sddg_status sddg_make_boundary_data(const sddg_density* dens, const sddg_domain* dom,
                                    int32_t nx, int32_t ny, int32_t bc_mode, double* tables8[8]);

/* Host: build_layout + plan_interface_points
 * (proj/src/decomposition.cpp:26-53,112-145).  Lines in layout order
 * (vertical first); nodes of line l at out_nodes[sum counts[<l]].  Capacity:
 * (sx-1)+(sy-1) lines, max(nx,ny) nodes each. */
sddg_status sddg_plan_interface_points(const sddg_density* dens, const sddg_domain* dom,
                                       int32_t nx, int32_t ny, int32_t sx, int32_t sy,
                                       int32_t placement, int32_t k, int32_t* n_lines,
                                       int32_t* out_vertical, int32_t* out_fixed,
                                       int32_t* out_counts, int32_t* out_nodes);

typedef struct {
    double t_bd, t_stoc, t_sub, t_smooth; /* seconds, as SddResult (decomposition.hpp:79-86) */
    int64_t mc_points, subdomain_solves, restarts, path_steps;
    int32_t warnings;
    int32_t reserved;
} sddg_sdd_stats;

/* Replaces sdd::solve_interfaces (proj/include/sdd/decomposition.hpp:70-72):
 * line values (layout order, full node ranges back to back) of xi, eta and
 * their stderrs. */
sddg_status sddg_solve_interfaces(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                  int32_t nx, int32_t ny, int32_t sx, int32_t sy,
                                  int32_t placement, int32_t k, const sddg_boundary* bd,
                                  const sddg_walk_config* cfg, const sddg_sdd_options* opts,
                                  double* xi_lines,
                                  double* eta_lines, double* se_xi_lines, double* se_eta_lines,
                                  sddg_sdd_stats* stats);

/* Sharding seams of solve_interfaces / solve_sdd (multi-GPU: every rank
 * walks a shard of the nodes, an all-gather of the sddg_estimate records
 * joins them, every rank fills the lines, ranks solve disjoint subdomain
 * ranges).
 * Host: the unique Monte Carlo nodes of the plan in solve_interfaces order
 * (proj/src/decomposition.cpp:156-169), point_id = j*nx + i. */
sddg_status sddg_interface_nodes(const sddg_density* dens, const sddg_domain* dom, int32_t nx,
                                 int32_t ny, int32_t sx, int32_t sy, int32_t placement, int32_t k,
                                 int64_t capacity, double* px, double* py, uint64_t* point_id,
                                 int64_t* n);
/* Host: interface lines from the n estimates of those nodes (in that order):
 * linear fill and crossing reconciliation (decomposition.cpp:176-246). */
sddg_status sddg_fill_interfaces(const sddg_density* dens, const sddg_domain* dom, int32_t nx,
                                 int32_t ny, int32_t sx, int32_t sy, int32_t placement, int32_t k,
                                 const sddg_boundary* bd, const sddg_estimate* est, int64_t n,
                                 const sddg_sdd_options* opts, double* xi_lines,
                                 double* eta_lines, double* se_xi_lines, double* se_eta_lines);
/* GPU: the subdomain phase of solve_sdd (decomposition.cpp:292-355) for
 * subdomains [s_lo, s_hi) (index s = b*sx + a) given the interface lines;
 * fields receives per subdomain its xi then its eta block ((n+1)^2 each,
 * index j*nx_sub + i); info one record per (subdomain, field). */
sddg_status sddg_solve_subdomains(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                  int32_t nx, int32_t ny, int32_t sx, int32_t sy, int32_t bc_mode,
                                  const double* xi_lines, const double* eta_lines,
                                  const sddg_solver_config* scfg, int32_t s_lo, int32_t s_hi,
                                  double* fields, sddg_solve_info* info);

/* Replaces sdd::solve_sdd (proj/include/sdd/decomposition.hpp:91-94):
 * boundary data, interface walks, optional interface smoothing, subdomain
 * solves, assembly into the global xi, eta (nx*ny, index j*nx+i).  opts may
 * be NULL (reference defaults: no interface smoothing). */
sddg_status sddg_solve_sdd(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                           int32_t nx, int32_t ny, int32_t sx, int32_t sy, int32_t placement,
                           int32_t k, int32_t bc_mode, const sddg_walk_config* cfg,
                           const sddg_solver_config* scfg, const sddg_sdd_options* opts,
                           double* xi, double* eta, sddg_sdd_stats* stats);

/* ------------------------------------------------- post-processing seams */

/* Replaces sdd::invert_mesh (proj/include/sdd/invert.hpp:14): the physical
 * mesh x, y (m_xi*m_eta, index b*m_xi + a) of the uniform computational grid
 * from the solution xi, eta on the nx x ny grid over dom.  Bit-identical to
 * the reference: every target is located in parallel, and the reference's
 * sequential hint chain (each target's walk starts at its predecessor's
 * triangle, which decides targets on mesh edges and in folded cells) is
 * reproduced by construction (csrc/mesh.cu); same point-location arithmetic
 * and rounding sequence.  Diagnostics afterwards: sddg_last_stats' step count =
 * targets the sequential fix-up pass located again, sddg_last_tail_stats'
 * handoffs = rows it visited. */
sddg_status sddg_invert_mesh(sddg_ctx* ctx, const double* xi, const double* eta, int32_t nx,
                             int32_t ny, const sddg_domain* dom, int32_t m_xi, int32_t m_eta,
                             double* x, double* y);

/* sdd::QualityReport (proj/include/sdd/quality.hpp:10-14). */
typedef struct {
    double q_max, q_mean;
    double r_max, r_mean; /* valid when has_reference */
    double l_inf;         /* valid when has_l_inf */
    int32_t has_reference, has_l_inf;
} sddg_quality;

/* Replaces sdd::quality_report (proj/src/quality.cpp:35-80); ref_x/ref_y
 * (reference mesh) and dens (for l_inf) may be NULL. */
sddg_status sddg_quality_report(sddg_ctx* ctx, const double* x, const double* y, int32_t m_xi,
                                int32_t m_eta, const double* ref_x, const double* ref_y,
                                const sddg_density* dens, sddg_quality* out);

/* The stochastic-full pipeline's solve (run_stochastic_full,
 * proj/src/cli.cpp:236-270): boundary tables on the boundary, one Monte Carlo
 * estimate per interior node (point_id = j*nx + i) in a single GPU batch.
 * xi, eta: nx*ny; stats->restarts and ->warnings (restart fraction > 1%). */
sddg_status sddg_stochastic_full(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                 int32_t nx, int32_t ny, const sddg_walk_config* cfg, double* xi,
                                 double* eta, sddg_sdd_stats* stats);

/* Host: sdd::write_mesh (proj/src/mesh_io.cpp:22-46), the bit-exact
 * "sddmesh v1" text format (%.17g, LF); the solution grid must match the
 * mesh shape. */
sddg_status sddg_write_mesh(const double* x, const double* y, int32_t m_xi, int32_t m_eta,
                            const double* xi, const double* eta, int32_t nx, int32_t ny,
                            const char* path);

/* sdd::SmoothConfig (proj/include/sdd/smoothing.hpp:15-22). */
typedef enum { SDDG_SMOOTH_GLOBAL = 0, SDDG_SMOOTH_PER_SUBDOMAIN = 1 } sddg_smooth_scope;
typedef struct {
    double k;      /* edge-stopping parameter, c = exp(-|grad u|^2 / k^2) */
    double dt;
    int32_t steps;
    int32_t scope; /* sddg_smooth_scope */
} sddg_smooth_config;

/* Replaces sdd::perona_malik (proj/include/sdd/smoothing.hpp:34-35): FTCS
 * Perona-Malik steps on xi and eta in place (nx*ny each over dom); sx, sy is
 * the subdomain layout for the per-subdomain scope (ignored for global).
 * *stability_warning (nullable) = 1 when dt > hx*hy/4 (stability_warning,
 * smoothing.cpp:18-26).  NumericalError when the update grows > 10x. */
sddg_status sddg_perona_malik(sddg_ctx* ctx, double* xi, double* eta, int32_t nx, int32_t ny,
                              const sddg_domain* dom, const sddg_smooth_config* cfg, int32_t sx,
                              int32_t sy, int32_t* stability_warning);

/* BASELINE.json config 4's "Laplacian smoothing, N sweeps" as the reference
 * can express it: Perona-Malik FTCS (perona_malik above,
 * smoothing.cpp:33-123) with the edge-stopping factor c = 1 (k = infinity)
 * and dt = hx*hy/4, the largest stable step, i.e. every sweep replaces each
 * interior value by the 4-neighbour average (hx = hy; the hx, hy-weighted
 * average otherwise).  Boundary values are kept; global scope. */
sddg_status sddg_laplacian_smooth(sddg_ctx* ctx, double* xi, double* eta, int32_t nx, int32_t ny,
                                  const sddg_domain* dom, int32_t sweeps);

/* Replaces sdd::smooth_interface (smoothing.hpp:41): tricube-weighted local
 * quadratic regression over an odd `span` window; endpoints kept. */
sddg_status sddg_smooth_interface(sddg_ctx* ctx, const double* values, int32_t n, int32_t span,
                                  double* out);

#ifdef __cplusplus
}
#endif

#endif /* SDDG_H */
