/*
 * sdd_config1.c -- a plain C99 caller of the C-ABI (include/sddg.h): the
 * drop-in boundary used the way the reference's own host code would use it,
 * with no Python, torch or C++ in between.
 *
 * Runs BASELINE.json config 1 end to end -- unit square, 65^2 grid split 2x2,
 * ring density, equispaced(31) interface nodes, 1e4 linear Euler-Maruyama
 * walks per node at dt 1e-4, reference boundary tables, subdomain solves to
 * 1e-10 -- through sddg_solve_sdd (replaces sdd::solve_sdd,
 * proj/include/sdd/decomposition.hpp:91-94), then inverts the mesh and
 * reports its quality (sddg_invert_mesh / sddg_quality_report).
 *
 * usage: sdd_config1 [reference|analytic] [seed] [devices]
 * devices: a comma-separated CUDA device list, e.g. "0,1,2,3": one process
 * drives all of them through sddg_create_multi (nodes and subdomains sharded,
 * NCCL all-gathers; a device listed twice runs as two ranks exchanging by
 * device copies).  Default: one device, sddg_create(0).
 * prints: one line "mc_points path_steps t_stoc t_sub checksum_xi checksum_eta
 * q_max q_mean" (checksums = plain sums in index order; tests/test_gpu_sdd.py
 * compares them with the Python mirror's solve_sdd on the same inputs).
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sddg.h"

static int check(sddg_status st, const sddg_ctx* ctx, const char* what) {
    if (st == SDDG_OK) return 0;
    fprintf(stderr, "%s failed: status %d: %s\n", what, (int)st, sddg_last_error(ctx));
    return 1;
}

int main(int argc, char** argv) {
    const int analytic = argc > 1 && strcmp(argv[1], "analytic") == 0;
    const unsigned long long seed = argc > 2 ? strtoull(argv[2], NULL, 10) : 1ULL;
    const int n = 65;
    if (sddg_abi_version() != SDDG_ABI_VERSION) {
        fprintf(stderr, "ABI mismatch: library %d, header %d\n", sddg_abi_version(), SDDG_ABI_VERSION);
        return 2;
    }
    sddg_ctx* ctx = NULL;
    if (argc > 3) {
        int devices[16], nd = 0;
        const char* p = argv[3];
        while (*p && nd < 16) {
            devices[nd++] = (int)strtol(p, (char**)&p, 10);
            if (*p == ',') ++p;
        }
        if (check(sddg_create_multi(nd, devices, &ctx), NULL, "sddg_create_multi")) return 1;
    } else if (check(sddg_create(0, &ctx), NULL, "sddg_create")) {
        return 1;
    }

    sddg_density dens;
    memset(&dens, 0, sizeof dens);
    dens.kind = SDDG_DENS_RING_W;
    dens.grad_mode = analytic ? SDDG_GRAD_ANALYTIC : SDDG_GRAD_REFERENCE;
    dens.fd_h = 1e-6;
    const sddg_domain dom = {0.0, 1.0, 0.0, 1.0};

    sddg_walk_config wc;
    memset(&wc, 0, sizeof wc);
    wc.scheme = SDDG_SCHEME_LINEAR;
    wc.precision = SDDG_FP64;
    wc.dt = 1e-4;
    wc.lambda = 1000.0;
    wc.walks = 10000;
    wc.seed = seed;
    wc.max_steps = 10000000;
    wc.bridge_test = 1;

    sddg_solver_config sc;
    memset(&sc, 0, sizeof sc);
    sc.tol = 1e-10;
    sc.init_blend = 1;
    sc.method = SDDG_SOLVER_RBSOR;

    double* xi = malloc(sizeof(double) * n * n);
    double* eta = malloc(sizeof(double) * n * n);
    double* x = malloc(sizeof(double) * n * n);
    double* y = malloc(sizeof(double) * n * n);
    if (!xi || !eta || !x || !y) return 3;
    sddg_sdd_stats stats;
    memset(&stats, 0, sizeof stats);
    int rc = check(sddg_solve_sdd(ctx, &dens, &dom, n, n, 2, 2, SDDG_PLACE_EQUISPACED, 31,
                                  SDDG_BC_REFERENCE, &wc, &sc, NULL, xi, eta, &stats),
                   ctx, "sddg_solve_sdd");
    sddg_quality q;
    memset(&q, 0, sizeof q);
    if (!rc) rc = check(sddg_invert_mesh(ctx, xi, eta, n, n, &dom, n, n, x, y), ctx, "sddg_invert_mesh");
    if (!rc)
        rc = check(sddg_quality_report(ctx, x, y, n, n, NULL, NULL, NULL, &q), ctx,
                   "sddg_quality_report");
    if (!rc) {
        double sx = 0.0, se = 0.0;
        for (int k = 0; k < n * n; ++k) {
            sx += xi[k];
            se += eta[k];
        }
        printf("%lld %lld %.6f %.6f %.17g %.17g %.17g %.17g\n", (long long)stats.mc_points,
               (long long)stats.path_steps, stats.t_stoc, stats.t_sub, sx, se, q.q_max, q.q_mean);
    }
    free(xi);
    free(eta);
    free(x);
    free(y);
    sddg_destroy(ctx);
    return rc;
}
