/*
 * sdd_oracle.c -- TEST INFRASTRUCTURE ONLY (see sdd_oracle.h).
 *
 * Plain-C restatement of the reference sddmesh algorithm for the hot path.
 * Every function cites the reference file:line it follows (paths relative to
 * the reference tree, proj/...).  Built with -O2 -ffp-contract=off so the
 * arithmetic is the same sequence of IEEE operations the reference performs
 * on x86-64 (the reference objects contain no FMA), and with the same glibc
 * libm calls (exp, log, sin, cos, sqrt).
 */
#include "sdd_oracle.h"
#include "workload_w.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846264338327950288

/* ------------------------------------------------------------------ rng.hpp */

/* proj/include/sdd/rng.hpp:12-29 */
void orc_philox_block(uint32_t k0, uint32_t k1, const uint32_t c_in[4], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = c_in[0], c1 = c_in[1], c2 = c_in[2], c3 = c_in[3];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)M0 * c0;
        const uint64_t p1 = (uint64_t)M1 * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += W0;
        k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* RandomStream (proj/include/sdd/rng.hpp:31-83).  u64 number n of a stream
 * is (hi = word 2(n%2)+1, lo = word 2(n%2)) of Philox block n/2: the
 * reference consumes words in pairs from 4-word blocks (rng.hpp:41-55). */
typedef struct {
    uint32_t k0, k1, c1, c2, c3;
    uint32_t block;
    uint32_t out[4];
    int have;
} orc_stream;

static void stream_init(orc_stream* s, uint64_t seed, uint64_t pid, uint32_t walk,
                        uint32_t epoch) {
    s->k0 = (uint32_t)seed;
    s->k1 = (uint32_t)(seed >> 32);
    s->c1 = walk;
    s->c2 = (uint32_t)pid;
    s->c3 = (uint32_t)((pid >> 32) & 0xFFFFu) | (epoch << 16);
    s->block = 0;
    s->have = 0;
}

static void stream_refill(orc_stream* s) {
    const uint32_t c[4] = {s->block++, s->c1, s->c2, s->c3};
    orc_philox_block(s->k0, s->k1, c, s->out);
    s->have = 4;
}

static uint64_t next_u64(orc_stream* s) {
    if (s->have == 0) stream_refill(s);
    const uint32_t lo = s->out[4 - s->have];
    --s->have;
    if (s->have == 0) stream_refill(s);
    const uint32_t hi = s->out[4 - s->have];
    --s->have;
    return ((uint64_t)hi << 32) | lo;
}

/* rng.hpp:58 */
static double u01(orc_stream* s) { return (double)(next_u64(s) >> 11) * 0x1.0p-53; }
/* rng.hpp:61-63 */
static double u01_open(orc_stream* s) {
    return ((double)(next_u64(s) >> 12) + 0.5) * 0x1.0p-52;
}
/* rng.hpp:66-73 */
static void normal_pair(orc_stream* s, double* z0, double* z1) {
    const double u1 = u01_open(s);
    const double u2 = u01(s);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    *z0 = r * cos(a);
    *z1 = r * sin(a);
}
/* rng.hpp:75 */
static double exponential(orc_stream* s, double lambda) { return -log(u01_open(s)) / lambda; }

void orc_stream_u64(uint64_t seed, uint64_t pid, uint32_t walk, uint32_t epoch, int64_t n,
                    uint64_t* out) {
    orc_stream s;
    stream_init(&s, seed, pid, walk, epoch);
    for (int64_t k = 0; k < n; ++k) out[k] = next_u64(&s);
}

void orc_stream_normals(uint64_t seed, uint64_t pid, uint32_t walk, uint32_t epoch,
                        int64_t npairs, double* out) {
    orc_stream s;
    stream_init(&s, seed, pid, walk, epoch);
    for (int64_t k = 0; k < npairs; ++k) normal_pair(&s, &out[2 * k], &out[2 * k + 1]);
}

/* -------------------------------------------------------------- monitor.cpp */

/* BASELINE.json densities as the diffusion weight w (workload_w.h). */
double orc_w_formula(int kind, double x, double y) { return wl_w(kind, x, y); }

/* five_ring_velocity (proj/src/monitor.cpp:16-37) */
static void five_ring_velocity(double x, double y, double R, double* ux, double* uy,
                               double* uxx, double* uxy, double* uyy) {
    static const double cx[5] = {0.0, 0.5, 0.5, -0.5, -0.5};
    static const double cy[5] = {0.0, 0.5, -0.5, 0.5, -0.5};
    double dux = 0.0, duy = 0.0, duxx = 0.0, duxy = 0.0, duyy = 0.0;
    for (int k = 0; k < 5; ++k) {
        const double dx = x - cx[k];
        const double dy = y - cy[k];
        const double t = tanh(R * (dx * dx + dy * dy - 0.125));
        const double s = 1.0 - t * t;
        const double gx = 2.0 * R * dx;
        const double gy = 2.0 * R * dy;
        dux += s * gx;
        duy += s * gy;
        duxx += s * (2.0 * R - 2.0 * t * gx * gx);
        duyy += s * (2.0 * R - 2.0 * t * gy * gy);
        duxy += -2.0 * t * s * gx * gy;
    }
    *ux = dux; *uy = duy; *uxx = duxx; *uxy = duxy; *uyy = duyy;
}

/* MonitorFunction::rho (proj/src/monitor.cpp:121-161); user_supplied kinds
 * evaluate rho = 1/w. */
double orc_rho(const orc_density* d, double x, double y) {
    const double R = d->R, al = d->alpha;
    switch (d->kind) {
        case ORC_CONSTANT: return R;
        case ORC_RUNNING: {
            const double dx = x - 0.75, dy = y - 0.5;
            return 1.0 + R * exp(-50.0 * dx * dx - 50.0 * dy * dy - 0.5);
        }
        case ORC_HUANG_SLOAN: {
            const double E = exp(R * (x - 1.0));
            const double S = sin(ORC_PI * y);
            const double C = cos(ORC_PI * y);
            const double q =
                al * (R * R * E * E * S * S + (1.0 - E) * (1.0 - E) * ORC_PI * ORC_PI * C * C);
            return sqrt(1.0 + q);
        }
        case ORC_MACKENZIE: {
            const double s = y - 0.5 - 0.25 * sin(2.0 * ORC_PI * x);
            return 1.0 / (1.0 + al * exp(-R * s * s));
        }
        case ORC_FIVE_RING: {
            double ux, uy, uxx, uxy, uyy;
            five_ring_velocity(x, y, R, &ux, &uy, &uxx, &uxy, &uyy);
            return sqrt(1.0 + al * (ux * ux + uy * uy));
        }
        default: return 1.0 / orc_w_formula(d->kind, x, y);
    }
}

/* rho_with_grad (proj/src/monitor.cpp:163-223) + drift (:231-240).
 * Returns 0, or 3 for the EvaluationError of a non-finite drift. */
int orc_drift(const orc_density* d, double x, double y, double* bx, double* by) {
    const double R = d->R, al = d->alpha;
    double r, gx, gy;
    switch (d->kind) {
        case ORC_CONSTANT: r = R; gx = 0.0; gy = 0.0; break;
        case ORC_RUNNING: {
            const double dx = x - 0.75, dy = y - 0.5;
            const double g = R * exp(-50.0 * dx * dx - 50.0 * dy * dy - 0.5);
            gx = -100.0 * dx * g;
            gy = -100.0 * dy * g;
            r = 1.0 + g;
            break;
        }
        case ORC_HUANG_SLOAN: {
            const double E = exp(R * (x - 1.0));
            const double S = sin(ORC_PI * y);
            const double C = cos(ORC_PI * y);
            const double q =
                al * (R * R * E * E * S * S + (1.0 - E) * (1.0 - E) * ORC_PI * ORC_PI * C * C);
            r = sqrt(1.0 + q);
            const double qx = al * (2.0 * R * R * R * E * E * S * S +
                                    2.0 * ORC_PI * ORC_PI * R * C * C * E * (E - 1.0));
            const double qy = 2.0 * ORC_PI * S * C * al *
                              (R * R * E * E - ORC_PI * ORC_PI * (1.0 - E) * (1.0 - E));
            gx = qx / (2.0 * r);
            gy = qy / (2.0 * r);
            break;
        }
        case ORC_MACKENZIE: {
            const double s = y - 0.5 - 0.25 * sin(2.0 * ORC_PI * x);
            const double E = exp(-R * s * s);
            const double D = 1.0 + al * E;
            const double drho_ds = 2.0 * al * R * s * E / (D * D);
            const double sx = -0.5 * ORC_PI * cos(2.0 * ORC_PI * x);
            gx = drho_ds * sx;
            gy = drho_ds;
            r = 1.0 / D;
            break;
        }
        case ORC_FIVE_RING: {
            double ux, uy, uxx, uxy, uyy;
            five_ring_velocity(x, y, R, &ux, &uy, &uxx, &uxy, &uyy);
            r = sqrt(1.0 + al * (ux * ux + uy * uy));
            gx = al * (ux * uxx + uy * uxy) / r;
            gy = al * (ux * uxy + uy * uyy) / r;
            break;
        }
        default: {
            /* user_supplied: central differences of rho (monitor.cpp:206-219) */
            const double h = d->fd_h;
            gx = (orc_rho(d, x + h, y) - orc_rho(d, x - h, y)) / (2.0 * h);
            gy = (orc_rho(d, x, y + h) - orc_rho(d, x, y - h)) / (2.0 * h);
            if (!isfinite(gx) || !isfinite(gy)) return 3;
            r = orc_rho(d, x, y);
            break;
        }
    }
    *bx = -gx / r;
    *by = -gy / r;
    if (!isfinite(*bx) || !isfinite(*by)) return 3;
    return 0;
}

/* ------------------------------------------------------------ boundary.cpp */

/* detsolver.cpp:20-48 (edge 0 bottom, 1 top, 2 left, 3 right) */
void orc_solve_1d_boundary(const orc_density* d, const orc_domain* dom, int nx, int ny,
                           int edge, double* u) {
    const int horizontal = edge == 0 || edge == 1;
    const int n = horizontal ? nx : ny;
    const double hx = (dom->xmax - dom->xmin) / (nx - 1);
    const double hy = (dom->ymax - dom->ymin) / (ny - 1);
    double* rho = (double*)malloc(sizeof(double) * n);
    for (int k = 0; k < n; ++k) {
        double px, py;
        switch (edge) {
            case 0: px = dom->xmin + k * hx; py = dom->ymin + 0 * hy; break;
            case 1: px = dom->xmin + k * hx; py = dom->ymin + (ny - 1) * hy; break;
            case 2: px = dom->xmin + 0 * hx; py = dom->ymin + k * hy; break;
            default: px = dom->xmin + (nx - 1) * hx; py = dom->ymin + k * hy; break;
        }
        rho[k] = orc_rho(d, px, py);
    }
    u[0] = 0.0;
    for (int k = 1; k < n; ++k) u[k] = u[k - 1] + 0.5 * (rho[k - 1] + rho[k]);
    const double total = u[n - 1];
    for (int k = 1; k < n - 1; ++k) u[k] /= total;
    u[n - 1] = 1.0;
    free(rho);
}

/* table_at (proj/src/boundary.cpp:10-15) */
double orc_table_at(const double* table, int n, double s) {
    int k = (int)floor(s);
    if (k < 0) k = 0;
    if (k > n - 2) k = n - 2;
    double t = s - k;
    if (t < 0.0) t = 0.0;
    if (t > 1.0) t = 1.0;
    return (1.0 - t) * table[k] + t * table[k + 1];
}

/* f_at / g_at via edge_param (proj/src/boundary.cpp:17-42) */
double orc_bd_value(const orc_boundary* bd, int use_g, int edge, double x, double y) {
    const double hx = (bd->dom.xmax - bd->dom.xmin) / (bd->nx - 1);
    const double hy = (bd->dom.ymax - bd->dom.ymin) / (bd->ny - 1);
    const double* const* tabs = use_g ? bd->g : bd->f;
    if (edge == 0 || edge == 1) return orc_table_at(tabs[edge], bd->nx, (x - bd->dom.xmin) / hx);
    return orc_table_at(tabs[edge], bd->ny, (y - bd->dom.ymin) / hy);
}

/* ----------------------------------------------------------------- sde.cpp */

static int strictly_inside(const orc_domain* d, double x, double y) {
    return x > d->xmin && x < d->xmax && y > d->ymin && y < d->ymax; /* geometry.hpp:38-40 */
}

/* proj/src/geometry.cpp:24-32 */
static double dist_edge(const orc_domain* d, double x, double y, int e) {
    switch (e) {
        case 0: return y - d->ymin;
        case 1: return d->ymax - y;
        case 2: return x - d->xmin;
        default: return d->xmax - x;
    }
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* segment_exit (proj/src/sde.cpp:31-65) */
static void segment_exit(const orc_domain* dom, double x0, double y0, double x1, double y1,
                         double* hx, double* hy, int* edge) {
    double best_t = 2.0;
    int best = 0;
#define CONSIDER(E, C0, C1, T)                               \
    do {                                                     \
        if ((C1) != (C0)) {                                  \
            const double t = ((T) - (C0)) / ((C1) - (C0));   \
            if (t >= 0.0 && t <= 1.0 && t < best_t) {        \
                best_t = t;                                  \
                best = (E);                                  \
            }                                                \
        }                                                    \
    } while (0)
    if (y1 <= dom->ymin) CONSIDER(0, y0, y1, dom->ymin);
    if (y1 >= dom->ymax) CONSIDER(1, y0, y1, dom->ymax);
    if (x1 <= dom->xmin) CONSIDER(2, x0, x1, dom->xmin);
    if (x1 >= dom->xmax) CONSIDER(3, x0, x1, dom->xmax);
#undef CONSIDER
    if (best_t > 1.0) {
        best_t = 1.0;
        if (y1 <= dom->ymin) best = 0;
        else if (y1 >= dom->ymax) best = 1;
        else if (x1 <= dom->xmin) best = 2;
        else best = 3;
    }
    double px = x0 + best_t * (x1 - x0), py = y0 + best_t * (y1 - y0);
    switch (best) {
        case 0: py = dom->ymin; break;
        case 1: py = dom->ymax; break;
        case 2: px = dom->xmin; break;
        default: px = dom->xmax; break;
    }
    *hx = clampd(px, dom->xmin, dom->xmax);
    *hy = clampd(py, dom->ymin, dom->ymax);
    *edge = best;
}

/* edge_crossing_test (proj/src/sde.cpp:72-109).  scheme 0: exponent d0 d1/dt
 * (bridge_exit_test, :113-121); scheme 1: nu2 min(d0,d1) (step_exponential,
 * :133-139).  Returns 1 on exit. */
static int edge_crossing(const orc_domain* dom, double x0, double y0, double x1, double y1,
                         orc_stream* rng, int scheme, double par, double* hx, double* hy,
                         int* edge) {
    double dist[4];
    int order[4];
    for (int k = 0; k < 4; ++k) {
        const double a = dist_edge(dom, x0, y0, k), b = dist_edge(dom, x1, y1, k);
        dist[k] = b < a ? b : a; /* std::min(a, b) returns a unless b < a */
        order[k] = k;
    }
    /* stable insertion sort by (dist, edge id): the comparator is a strict
     * total order so the result equals std::sort's */
    for (int i = 1; i < 4; ++i) {
        int j = i;
        while (j > 0) {
            const int a = order[j - 1], b = order[j];
            const int less = dist[b] != dist[a] ? dist[b] < dist[a] : b < a;
            if (!less) break;
            order[j - 1] = b;
            order[j] = a;
            --j;
        }
    }
    for (int i = 0; i < 4; ++i) {
        const int e = order[i];
        const double d0 = dist_edge(dom, x0, y0, e);
        const double d1 = dist_edge(dom, x1, y1, e);
        const double ex = scheme == 0 ? d0 * d1 / par : par * (d1 < d0 ? d1 : d0);
        if (ex > 40.0) continue;
        if (u01(rng) < exp(-ex)) {
            const double sum = d0 + d1;
            const double s = sum > 0.0 ? d0 / sum : 0.0;
            double px = x0 + s * (x1 - x0), py = y0 + s * (y1 - y0);
            switch (e) {
                case 0: py = dom->ymin; break;
                case 1: py = dom->ymax; break;
                case 2: px = dom->xmin; break;
                default: px = dom->xmax; break;
            }
            *hx = clampd(px, dom->xmin, dom->xmax);
            *hy = clampd(py, dom->ymin, dom->ymax);
            *edge = e;
            return 1;
        }
    }
    return 0;
}

/* run_walk (proj/src/sde.cpp:151-183).  Returns 0, -1 for EvaluationError
 * (non-finite drift), -2 for NumericalError (1024 epochs without exit). */
static int run_walk(const orc_density* d, const orc_domain* dom, const orc_boundary* bd,
                    const orc_walk_cfg* cfg, double px, double py, uint64_t pid, int64_t walk,
                    orc_path* res) {
    const uint32_t kMaxEpochs = 1024;
    for (uint32_t epoch = 0; epoch < kMaxEpochs; ++epoch) {
        orc_stream rng;
        stream_init(&rng, cfg->seed, pid, (uint32_t)walk, epoch);
        double x = px, y = py;
        for (int64_t step = 1; step <= cfg->max_steps; ++step) {
            int exited = 0, edge = 0;
            double hx = 0.0, hy = 0.0;
            double bx, by, z0, z1, dt, nx, ny;
            if (cfg->scheme == 0) {
                /* step_linear (sde.cpp:21-29) */
                if (orc_drift(d, x, y, &bx, &by)) return 3;
                normal_pair(&rng, &z0, &z1);
                const double s = sqrt(2.0 * cfg->dt);
                nx = x + bx * cfg->dt + s * z0;
                ny = y + by * cfg->dt + s * z1;
                if (!strictly_inside(dom, nx, ny)) {
                    segment_exit(dom, x, y, nx, ny, &hx, &hy, &edge);
                    exited = 1;
                } else if (cfg->bridge_test) {
                    /* bridge_exit_test re-checks strictly_inside (sde.cpp:115) */
                    exited = edge_crossing(dom, x, y, nx, ny, &rng, 0, cfg->dt, &hx, &hy, &edge);
                }
            } else {
                /* step_exponential (sde.cpp:123-140) */
                dt = exponential(&rng, cfg->lambda);
                if (orc_drift(d, x, y, &bx, &by)) return 3;
                normal_pair(&rng, &z0, &z1);
                const double s = sqrt(2.0 * dt);
                nx = x + bx * dt + s * z0;
                ny = y + by * dt + s * z1;
                if (!strictly_inside(dom, nx, ny)) {
                    segment_exit(dom, x, y, nx, ny, &hx, &hy, &edge);
                    exited = 1;
                } else {
                    const double nu2 = 2.0 * sqrt(cfg->lambda);
                    exited = edge_crossing(dom, x, y, nx, ny, &rng, 1, nu2, &hx, &hy, &edge);
                }
            }
            if (exited) {
                res->f = orc_bd_value(bd, 0, edge, hx, hy);
                res->g = orc_bd_value(bd, 1, edge, hx, hy);
                res->ex = hx;
                res->ey = hy;
                res->steps = step;
                res->epoch = (int32_t)epoch;
                res->edge = edge;
                return 0;
            }
            x = nx;
            y = ny;
        }
    }
    return 4;
}

int orc_walk_dump(const orc_density* d, const orc_domain* dom, const orc_boundary* bd,
                  const orc_walk_cfg* cfg, double px, double py, uint64_t pid,
                  int64_t walk_lo, int64_t n, orc_path* out) {
    for (int64_t k = 0; k < n; ++k) {
        const int rc = run_walk(d, dom, bd, cfg, px, py, pid, walk_lo + k, &out[k]);
        if (rc) return rc;
    }
    return 0;
}

/* mc_estimate (proj/src/sde.cpp:193-246): 256-walk chunks summed in walk
 * order, chunk sums added in chunk order.  Returns 0, 3/4 as run_walk,
 * 1 ValidationError, 2 OutOfDomainError. */
int orc_mc_estimate(const orc_density* d, const orc_domain* dom, const orc_boundary* bd,
                    const orc_walk_cfg* cfg, double px, double py, uint64_t pid,
                    orc_estimate* est) {
    if (cfg->scheme == 0 && !(cfg->dt > 0.0)) return 1;
    if (cfg->scheme == 1 && !(cfg->lambda > 0.0)) return 1;
    if (cfg->walks < 1 || cfg->max_steps < 1) return 1;
    if (!strictly_inside(dom, px, py)) return 2;
    const int64_t kChunk = 256;
    const int64_t n_chunks = (cfg->walks + kChunk - 1) / kChunk;
    double tf = 0.0, tg = 0.0, tff = 0.0, tgg = 0.0;
    int64_t restarts = 0, hits[4] = {0, 0, 0, 0}, steps = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
        const int64_t lo = c * kChunk;
        const int64_t hi = cfg->walks < lo + kChunk ? cfg->walks : lo + kChunk;
        double sf = 0.0, sg = 0.0, sff = 0.0, sgg = 0.0;
        for (int64_t w = lo; w < hi; ++w) {
            orc_path r;
            const int rc = run_walk(d, dom, bd, cfg, px, py, pid, w, &r);
            if (rc) return rc;
            sf += r.f;
            sg += r.g;
            sff += r.f * r.f;
            sgg += r.g * r.g;
            restarts += r.epoch;
            hits[r.edge]++;
            steps += r.steps + (int64_t)r.epoch * cfg->max_steps;
        }
        tf += sf;
        tg += sg;
        tff += sff;
        tgg += sgg;
    }
    const double n = (double)cfg->walks;
    memset(est, 0, sizeof(*est));
    est->walks = cfg->walks;
    est->xi = tf / n;
    est->eta = tg / n;
    if (cfg->walks > 1) {
        double vf = (tff - n * est->xi * est->xi) / (n - 1.0);
        double vg = (tgg - n * est->eta * est->eta) / (n - 1.0);
        if (vf < 0.0) vf = 0.0;
        if (vg < 0.0) vg = 0.0;
        est->se_xi = sqrt(vf / n);
        est->se_eta = sqrt(vg / n);
    }
    est->restarts = restarts;
    est->warn = restarts > cfg->walks / 100;
    for (int e = 0; e < 4; ++e) est->edge_hits[e] = hits[e];
    est->sum_f = tf;
    est->sum_g = tg;
    est->sum_ff = tff;
    est->sum_gg = tgg;
    est->path_steps = steps;
    return 0;
}

typedef struct {
    const orc_density* d;
    const orc_domain* dom;
    const orc_boundary* bd;
    const orc_walk_cfg* cfg;
    const double *px, *py;
    const uint64_t* pid;
    orc_estimate* out;
    int64_t lo, hi;
    int rc;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    for (int64_t i = j->lo; i < j->hi && !j->rc; ++i)
        j->rc = orc_mc_estimate(j->d, j->dom, j->bd, j->cfg, j->px[i], j->py[i], j->pid[i],
                                &j->out[i]);
    return NULL;
}

/* parallel_for over points with contiguous static blocks
 * (proj/src/parallel.cpp:16-45, proj/src/decomposition.cpp:172-174). */
int orc_mc_estimate_batch(const orc_density* d, const orc_domain* dom,
                          const orc_boundary* bd, const orc_walk_cfg* cfg, const double* px,
                          const double* py, const uint64_t* pid, int64_t n, int threads,
                          orc_estimate* out) {
    if (n <= 0) return 0;
    if (threads < 1) threads = 1;
    if (threads > n) threads = (int)n;
    batch_job* jobs = (batch_job*)calloc((size_t)threads, sizeof(batch_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    const int64_t chunk = (n + threads - 1) / threads;
    int started = 0;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) break;
        jobs[t] = (batch_job){d, dom, bd, cfg, px, py, pid, out, lo, hi, 0};
        pthread_create(&tids[t], NULL, batch_worker, &jobs[t]);
        ++started;
    }
    int rc = 0;
    for (int t = 0; t < started; ++t) {
        pthread_join(tids[t], NULL);
        if (!rc) rc = jobs[t].rc;
    }
    free(jobs);
    free(tids);
    return rc;
}

/* ----------------------------------------------------------- detsolver.cpp */

/* weight_values (proj/src/detsolver.cpp:219-224): w = 1/rho at grid nodes. */
void orc_weight_values(const orc_density* d, const orc_domain* dom, int nx, int ny,
                       double* w) {
    const double hx = (dom->xmax - dom->xmin) / (nx - 1);
    const double hy = (dom->ymax - dom->ymin) / (ny - 1);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            w[(size_t)j * nx + i] = 1.0 / orc_rho(d, dom->xmin + i * hx, dom->ymin + j * hy);
}

/* solve_dirichlet (proj/src/detsolver.cpp:72-209).  Returns 0, 1 for a
 * ValidationError/EvaluationError of the inputs, 4 for the max-principle
 * NumericalError. */
int orc_solve_dirichlet(const double* w, int nx, int ny, double hx, double hy,
                        const double* bottom, const double* top, const double* left,
                        const double* right, double tol, int64_t max_iters_in, int init_blend,
                        double* u_out, int64_t* iters_out, double* final_update,
                        int* converged_out) {
    if (!(tol > 0.0) || max_iters_in < 0 || nx < 3 || ny < 3) return 1;
    for (int64_t k = 0; k < (int64_t)nx * ny; ++k)
        if (!isfinite(w[k]) || w[k] <= 0.0) return 1;
#define CM(a, b) (fabs((a) - (b)) > 1e-12 * (1.0 + fabs(a) + fabs(b)))
    if (CM(bottom[0], left[0]) || CM(bottom[nx - 1], right[0]) || CM(top[0], left[ny - 1]) ||
        CM(top[nx - 1], right[ny - 1]))
        return 1;
#undef CM
    const size_t N = (size_t)nx * ny;
    double* cE = (double*)malloc(sizeof(double) * (size_t)(nx - 1) * ny);
    double* cN = (double*)malloc(sizeof(double) * (size_t)nx * (ny - 1));
    double* inv = (double*)calloc(N, sizeof(double));
    double* u = (double*)malloc(sizeof(double) * N);
    double* v = (double*)malloc(sizeof(double) * N);
#define ID(i, j) ((size_t)(j) * nx + (i))
#define WE(i, j) cE[(size_t)(j) * (nx - 1) + (i)]
#define WN(i, j) cN[(size_t)(j) * nx + (i)]
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i + 1 < nx; ++i) WE(i, j) = 0.5 * (w[ID(i, j)] + w[ID(i + 1, j)]);
    for (int j = 0; j + 1 < ny; ++j)
        for (int i = 0; i < nx; ++i) WN(i, j) = 0.5 * (w[ID(i, j)] + w[ID(i, j + 1)]);
    const double ihx2 = 1.0 / (hx * hx);
    const double ihy2 = 1.0 / (hy * hy);
    for (int j = 1; j + 1 < ny; ++j)
        for (int i = 1; i + 1 < nx; ++i)
            inv[ID(i, j)] =
                1.0 / ((WE(i, j) + WE(i - 1, j)) * ihx2 + (WN(i, j) + WN(i, j - 1)) * ihy2);
    double bmin = bottom[0], bmax = bottom[0];
    const double* arrs[4] = {bottom, top, left, right};
    const int lens[4] = {nx, nx, ny, ny};
    for (int a = 0; a < 4; ++a)
        for (int k = 0; k < lens[a]; ++k) {
            const double x = arrs[a][k];
            if (x < bmin) bmin = x; /* std::min(bmin, v) keeps bmin unless v < bmin */
            if (bmax < x) bmax = x;
        }
    if (init_blend) {
        for (int j = 0; j < ny; ++j) {
            const double ty = (double)j / (ny - 1);
            for (int i = 0; i < nx; ++i) {
                const double tx = (double)i / (nx - 1);
                const double xb = (1.0 - tx) * left[j] + tx * right[j];
                const double yb = (1.0 - ty) * bottom[i] + ty * top[i];
                const double bil = ((1.0 - tx) * (1.0 - ty) * bottom[0] + tx * ty * top[nx - 1]) +
                                   (tx * (1.0 - ty) * bottom[nx - 1] + (1.0 - tx) * ty * top[0]);
                u[ID(i, j)] = clampd(xb + yb - bil, bmin, bmax);
            }
        }
    } else {
        for (size_t k = 0; k < N; ++k) u[k] = 0.5 * (bmin + bmax);
    }
    for (int i = 0; i < nx; ++i) {
        u[ID(i, 0)] = bottom[i];
        u[ID(i, ny - 1)] = top[i];
    }
    for (int j = 0; j < ny; ++j) {
        u[ID(0, j)] = left[j];
        u[ID(nx - 1, j)] = right[j];
    }
    memcpy(v, u, sizeof(double) * N);
    int64_t max_iters = max_iters_in;
    if (max_iters == 0) {
        const int64_t m = nx > ny ? nx : ny;
        max_iters = 200 * m * m;
    }
    int64_t iters = 0;
    double upd = 0.0, prev = -1.0;
    int conv = 0;
    while (iters < max_iters) {
        ++iters;
        upd = 0.0;
        for (int j = 1; j + 1 < ny; ++j)
            for (int i = 1; i + 1 < nx; ++i) {
                const size_t c = ID(i, j);
                const double xp = (WE(i, j) * u[c + 1] + WE(i - 1, j) * u[c - 1]) * ihx2;
                const double yp = (WN(i, j) * u[c + nx] + WN(i, j - 1) * u[c - nx]) * ihy2;
                const double nu = (xp + yp) * inv[c];
                v[c] = nu;
                const double du = fabs(nu - u[c]);
                if (upd < du) upd = du;
            }
        double* t = u; u = v; v = t;
        if (upd < tol) {
            if (upd == 0.0 || upd < 1e-4 * tol) { conv = 1; break; }
            if (prev > 0.0 && upd < prev) {
                const double rho = upd / prev;
                if (upd * rho / (1.0 - rho) < tol) { conv = 1; break; }
            }
        }
        prev = upd;
    }
    int rc = 0;
    const double slack = 1e-12 * (1.0 + fabs(bmin) + fabs(bmax));
    for (int j = 1; j + 1 < ny && !rc; ++j)
        for (int i = 1; i + 1 < nx; ++i)
            if (u[ID(i, j)] < bmin - slack || u[ID(i, j)] > bmax + slack) { rc = 4; break; }
    memcpy(u_out, u, sizeof(double) * N);
    *iters_out = iters;
    *final_update = upd;
    *converged_out = conv;
#undef ID
#undef WE
#undef WN
    free(cE); free(cN); free(inv); free(u); free(v);
    return rc;
}

/* ------------------------------------------------------- decomposition.cpp */

/* Gradient along a line for optimal placement: rho_with_grad / grad_rho
 * (monitor.cpp:225-229). user_supplied kinds use the FD gradient. */
static void grad_rho(const orc_density* d, double x, double y, double* gx, double* gy) {
    double bx, by;
    /* drift = -grad/rho, so grad = -drift * rho is NOT bit-identical; restate
     * the gradient directly instead. */
    const double R = d->R, al = d->alpha;
    switch (d->kind) {
        case ORC_CONSTANT: *gx = 0.0; *gy = 0.0; return;
        case ORC_RUNNING: {
            const double dx = x - 0.75, dy = y - 0.5;
            const double g = R * exp(-50.0 * dx * dx - 50.0 * dy * dy - 0.5);
            *gx = -100.0 * dx * g;
            *gy = -100.0 * dy * g;
            return;
        }
        case ORC_HUANG_SLOAN: {
            const double E = exp(R * (x - 1.0));
            const double S = sin(ORC_PI * y);
            const double C = cos(ORC_PI * y);
            const double q =
                al * (R * R * E * E * S * S + (1.0 - E) * (1.0 - E) * ORC_PI * ORC_PI * C * C);
            const double r = sqrt(1.0 + q);
            const double qx = al * (2.0 * R * R * R * E * E * S * S +
                                    2.0 * ORC_PI * ORC_PI * R * C * C * E * (E - 1.0));
            const double qy = 2.0 * ORC_PI * S * C * al *
                              (R * R * E * E - ORC_PI * ORC_PI * (1.0 - E) * (1.0 - E));
            *gx = qx / (2.0 * r);
            *gy = qy / (2.0 * r);
            return;
        }
        case ORC_MACKENZIE: {
            const double s = y - 0.5 - 0.25 * sin(2.0 * ORC_PI * x);
            const double E = exp(-R * s * s);
            const double D = 1.0 + al * E;
            const double drho_ds = 2.0 * al * R * s * E / (D * D);
            const double sx = -0.5 * ORC_PI * cos(2.0 * ORC_PI * x);
            *gx = drho_ds * sx;
            *gy = drho_ds;
            return;
        }
        case ORC_FIVE_RING: {
            double ux, uy, uxx, uxy, uyy;
            five_ring_velocity(x, y, R, &ux, &uy, &uxx, &uxy, &uyy);
            const double r = sqrt(1.0 + al * (ux * ux + uy * uy));
            *gx = al * (ux * uxx + uy * uxy) / r;
            *gy = al * (ux * uxy + uy * uyy) / r;
            return;
        }
        default: {
            const double h = d->fd_h;
            *gx = (orc_rho(d, x + h, y) - orc_rho(d, x - h, y)) / (2.0 * h);
            *gy = (orc_rho(d, x, y + h) - orc_rho(d, x, y - h)) / (2.0 * h);
            (void)bx; (void)by;
            return;
        }
    }
}

/* mark_extrema (proj/src/decomposition.cpp:68-79) */
static void mark_extrema(const double* v, int n, char* marks) {
    double vmax = 0.0;
    for (int i = 0; i < n; ++i) {
        const double a = fabs(v[i]);
        if (vmax < a) vmax = a;
    }
    const double floor_mag = 1e-9 * vmax;
    for (int i = 1; i + 1 < n; ++i) {
        if (fabs(v[i]) < floor_mag) continue;
        const int is_max = v[i] > v[i - 1] && v[i] > v[i + 1];
        const int is_min = v[i] < v[i - 1] && v[i] < v[i + 1];
        if (is_max || is_min) marks[i] = 1;
    }
}

/* plan_interface_points for one line (proj/src/decomposition.cpp:81-145).
 * strategy 0 all, 1 equispaced(k), 2 optimal.  Returns the node count or -1
 * for the ValidationError of a bad equispaced count. */
int orc_plan_line(int strategy, int k, const orc_density* d, const orc_domain* dom, int nx,
                  int ny, int vertical, int fixed_index, int* out) {
    const int n = vertical ? ny : nx;
    int cnt = 0;
    if (strategy == 0) {
        for (int pos = 1; pos + 1 < n; ++pos) out[cnt++] = pos;
        return cnt;
    }
    if (strategy == 1) {
        if (k < 1 || k > n - 2) return -1;
        for (int j = 1; j <= k; ++j) {
            int pos = (int)lround((double)j * (n - 1) / (k + 1));
            if (pos < 1) pos = 1;
            if (pos > n - 2) pos = n - 2;
            if (cnt == 0 || out[cnt - 1] != pos) out[cnt++] = pos; /* std::unique */
        }
        return cnt;
    }
    const double hx = (dom->xmax - dom->xmin) / (nx - 1);
    const double hy = (dom->ymax - dom->ymin) / (ny - 1);
    const double h = vertical ? hy : hx;
    double* d1 = (double*)malloc(sizeof(double) * n);
    double* d2 = (double*)calloc((size_t)n, sizeof(double));
    char* marks = (char*)calloc((size_t)n, 1);
    for (int pos = 0; pos < n; ++pos) {
        const double x = vertical ? dom->xmin + fixed_index * hx : dom->xmin + pos * hx;
        const double y = vertical ? dom->ymin + pos * hy : dom->ymin + fixed_index * hy;
        double gx, gy;
        grad_rho(d, x, y, &gx, &gy);
        d1[pos] = vertical ? gy : gx;
    }
    for (int pos = 1; pos + 1 < n; ++pos) d2[pos] = (d1[pos + 1] - d1[pos - 1]) / (2.0 * h);
    mark_extrema(d1, n, marks);
    mark_extrema(d2, n, marks);
    for (int pos = 1; pos + 1 < n; ++pos) {
        if (!marks[pos]) continue;
        if (cnt > 0 && pos - out[cnt - 1] < 2) continue;
        out[cnt++] = pos;
    }
    if (cnt == 0) out[cnt++] = n / 2;
    free(d1); free(d2); free(marks);
    return cnt;
}

/* Piecewise-linear fill between known line nodes
 * (proj/src/decomposition.cpp:215-224).  xi/eta hold the known values at
 * known_pos on entry (including both endpoints). */
void orc_fill_line(int n, const int* known_pos, const double* known_xi,
                   const double* known_eta, int n_known, double* xi, double* eta) {
    char* known = (char*)calloc((size_t)n, 1);
    for (int k = 0; k < n_known; ++k) {
        xi[known_pos[k]] = known_xi[k];
        eta[known_pos[k]] = known_eta[k];
        known[known_pos[k]] = 1;
    }
    int prev = 0;
    for (int pos = 1; pos < n; ++pos) {
        if (!known[pos]) continue;
        for (int q = prev + 1; q < pos; ++q) {
            const double t = (double)(q - prev) / (pos - prev);
            xi[q] = (1.0 - t) * xi[prev] + t * xi[pos];
            eta[q] = (1.0 - t) * eta[prev] + t * eta[pos];
        }
        prev = pos;
    }
    free(known);
}
