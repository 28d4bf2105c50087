/*
 * sdd_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, fp64, no FMA contraction) of the reference
 * sddmesh hot path: Philox4x32-10 streams, the Euler-Maruyama first-exit walk
 * with its exit rules, the fixed chunk-order Monte Carlo reduction, the
 * boundary tables, the Jacobi subdomain solver and the interface fill.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this code, and only as the checker.  The product path
 * (paper_1310_3435_b200/) never links or calls it.
 *
 * Pinning: tests/test_oracle_pins.py checks every function here bit-for-bit
 * against the reference compiled from /root/reference (oracle/_ref, built by
 * oracle/Makefile) through golden fixtures in tests/golden/ made by
 * tests/golden/make_golden.py.  The only unpinned layer is glibc libm itself
 * (exp/log/sincos), which both sides call identically.
 */
#ifndef SDD_ORACLE_H
#define SDD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Density kinds.  The first five are the reference's builtin monitors
 * (proj/include/sdd/monitor.hpp:11-18) given as rho; the last three are the
 * BASELINE.json densities given as the diffusion weight w, entered into the
 * reference as MonitorFunction::user_supplied(rho = 1/w) with a central
 * difference gradient (proj/src/monitor.cpp:73-80, 206-219). */
enum {
    ORC_CONSTANT = 0,
    ORC_RUNNING = 1,
    ORC_HUANG_SLOAN = 2,
    ORC_MACKENZIE = 3,
    ORC_FIVE_RING = 4,
    ORC_RING_W = 16,
    ORC_SHOCK_W = 17,
    ORC_TWOBUMP_W = 18
};

typedef struct {
    int kind;
    double R, alpha; /* builtin parameters (monitor.hpp:26-38) */
    double fd_h;     /* user_supplied FD step (monitor.hpp:40) */
} orc_density;

typedef struct {
    double xmin, xmax, ymin, ymax;
} orc_domain;

/* BoundaryData (proj/include/sdd/boundary.hpp:12-18): tables at the nodes of
 * the nx x ny grid over `dom`; index 0..3 = bottom, top, left, right. */
typedef struct {
    orc_domain dom;
    int nx, ny;
    const double* f[4];
    const double* g[4];
} orc_boundary;

typedef struct {
    int scheme; /* 0 linear, 1 exponential (sde.hpp:14) */
    double dt, lambda;
    int64_t walks;
    uint64_t seed;
    int64_t max_steps;
    int bridge_test;
} orc_walk_cfg;

typedef struct {
    double f, g;
    double ex, ey;
    int64_t steps;
    int32_t epoch;
    int32_t edge;
} orc_path;

typedef struct {
    double xi, eta, se_xi, se_eta;
    int64_t walks, restarts;
    int32_t warn;
    int64_t edge_hits[4];
    double sum_f, sum_g, sum_ff, sum_gg;
    int64_t path_steps;
} orc_estimate;

/* rng.hpp */
void orc_philox_block(uint32_t k0, uint32_t k1, const uint32_t c_in[4], uint32_t out[4]);
void orc_stream_u64(uint64_t seed, uint64_t pid, uint32_t walk, uint32_t epoch, int64_t n,
                    uint64_t* out);
void orc_stream_normals(uint64_t seed, uint64_t pid, uint32_t walk, uint32_t epoch,
                        int64_t npairs, double* out);

/* monitor.cpp */
double orc_rho(const orc_density* d, double x, double y);
int orc_drift(const orc_density* d, double x, double y, double* bx, double* by);
double orc_w_formula(int kind, double x, double y);

/* boundary.cpp / detsolver.cpp:20-48 */
void orc_solve_1d_boundary(const orc_density* d, const orc_domain* dom, int nx, int ny,
                           int edge, double* out);
double orc_table_at(const double* table, int n, double s);
double orc_bd_value(const orc_boundary* bd, int use_g, int edge, double x, double y);

/* sde.cpp */
int orc_walk_dump(const orc_density* d, const orc_domain* dom, const orc_boundary* bd,
                  const orc_walk_cfg* cfg, double px, double py, uint64_t pid,
                  int64_t walk_lo, int64_t n, orc_path* out);
int orc_mc_estimate(const orc_density* d, const orc_domain* dom, const orc_boundary* bd,
                    const orc_walk_cfg* cfg, double px, double py, uint64_t pid,
                    orc_estimate* out);
int orc_mc_estimate_batch(const orc_density* d, const orc_domain* dom,
                          const orc_boundary* bd, const orc_walk_cfg* cfg, const double* px,
                          const double* py, const uint64_t* pid, int64_t n, int threads,
                          orc_estimate* out);

/* detsolver.cpp */
void orc_weight_values(const orc_density* d, const orc_domain* dom, int nx, int ny,
                       double* w);
int orc_solve_dirichlet(const double* w, int nx, int ny, double hx, double hy,
                        const double* bottom, const double* top, const double* left,
                        const double* right, double tol, int64_t max_iters, int init_blend,
                        double* u_out, int64_t* iters, double* final_update,
                        int* converged);

/* decomposition.cpp */
int orc_plan_line(int strategy, int k, const orc_density* d, const orc_domain* dom, int nx,
                  int ny, int vertical, int fixed_index, int* out_nodes);
void orc_fill_line(int n, const int* known_pos, const double* known_xi,
                   const double* known_eta, int n_known, double* xi, double* eta);

#ifdef __cplusplus
}
#endif

#endif
