// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI harness over the UNMODIFIED reference library (the sddcore sources
// under /root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libsddref.so).  It drives the reference's public API exactly as
// its own tests and CLI do; nothing here re-implements the algorithm except
// ref_walk_dump, which replays the anonymous-namespace run_walk
// (proj/src/sde.cpp:151-183) through the public step_linear / segment_exit /
// bridge_exit_test / step_exponential functions to expose per-path results
// (verified equal to mc_estimate by
// tests/test_oracle_pins.py).
//
// Used by tests/golden/make_golden.py (fixtures), tests/ (pins) and the
// bench.py CPU arms (timing of the reference's own mc_estimate path).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <exception>
#include <optional>
#include <string>
#include <vector>

#include "sdd/boundary.hpp"
#include "sdd/decomposition.hpp"
#include "sdd/invert.hpp"
#include "sdd/quality.hpp"
#include "sdd/smoothing.hpp"
#include "sdd/mesh_io.hpp"
#include "sdd/detsolver.hpp"
#include "sdd/monitor.hpp"
#include "sdd/parallel.hpp"
#include "sdd/sde.hpp"
#include "workload_w.h"

using namespace sdd;

namespace {

thread_local std::string g_err;

struct Domain {
    double xmin, xmax, ymin, ymax;
};

struct Density {
    int kind;
    double R, alpha, fd_h;
    // kind 32 (a tabulated user density, include/sddg.h SDDG_DENS_TABLE)
    const double* table;
    int tnx, tny;
    Domain tdom;
};

// A tabulated rho as the reference receives any user density: a callable
// handed to MonitorFunction::user_supplied.  The callable restates the
// library's documented interpolant (include/sddg.h, SDDG_DENS_TABLE):
// Catmull-Rom bicubic on the samples padded by one linearly extrapolated
// node per side, cell clamp(floor(s), 0, n-2), local t = s - cell, with the
// normative operation order, so the reference's central difference of it is
// what the GPU's reference mode must reproduce.
struct TabRho {
    std::vector<double> pad;  // (nx+2) x (ny+2)
    int nx, ny;
    double x0, y0, ihx, ihy;

    TabRho(const double* f, int nx_, int ny_, const Domain& dom) : nx(nx_), ny(ny_) {
        const int w = nx + 2;
        pad.assign(static_cast<std::size_t>(w) * (ny + 2), 0.0);
        for (int j = 1; j <= ny; ++j) {
            for (int i = 1; i <= nx; ++i) pad[j * w + i] = f[(j - 1) * nx + (i - 1)];
            pad[j * w] = 2.0 * pad[j * w + 1] - pad[j * w + 2];
            pad[j * w + nx + 1] = 2.0 * pad[j * w + nx] - pad[j * w + nx - 1];
        }
        for (int i = 0; i < w; ++i) {
            pad[i] = 2.0 * pad[w + i] - pad[2 * w + i];
            pad[(ny + 1) * w + i] = 2.0 * pad[ny * w + i] - pad[(ny - 1) * w + i];
        }
        x0 = dom.xmin;
        y0 = dom.ymin;
        ihx = 1.0 / ((dom.xmax - dom.xmin) / (nx - 1));
        ihy = 1.0 / ((dom.ymax - dom.ymin) / (ny - 1));
    }
    static void weights(double t, double w[4]) {
        w[0] = 0.5 * (((2.0 - t) * t - 1.0) * t);
        w[1] = 0.5 * ((3.0 * t - 5.0) * t * t + 2.0);
        w[2] = 0.5 * (((4.0 - 3.0 * t) * t + 1.0) * t);
        w[3] = 0.5 * ((t - 1.0) * t * t);
    }
    double operator()(Point q) const {
        const double sx = (q.x - x0) * ihx, sy = (q.y - y0) * ihy;
        int i = static_cast<int>(std::floor(sx)), j = static_cast<int>(std::floor(sy));
        i = std::min(std::max(i, 0), nx - 2);
        j = std::min(std::max(j, 0), ny - 2);
        double wx[4], wy[4];
        weights(sx - i, wx);
        weights(sy - j, wy);
        const int w = nx + 2;
        double v = 0.0;
        for (int b = 0; b < 4; ++b) {
            const double* r = pad.data() + static_cast<std::size_t>(j + b) * w + i;
            v = v + wy[b] * (((wx[0] * r[0] + wx[1] * r[1]) + wx[2] * r[2]) + wx[3] * r[3]);
        }
        return v;
    }
};

struct WalkCfgC {
    int scheme;
    double dt, lambda;
    int64_t walks;
    uint64_t seed;
    int64_t max_steps;
    int bridge_test;
};

struct PathRec {
    double f, g, ex, ey;
    int64_t steps;
    int32_t epoch, edge;
};

struct EstimateC {
    double xi, eta, se_xi, se_eta;
    int64_t walks, restarts;
    int32_t warn;
    int64_t edge_hits[4];
    double sum_f, sum_g, sum_ff, sum_gg;
    int64_t path_steps;
};

MonitorFunction make_monitor(const Density& d, const Domain& dom) {
    switch (d.kind) {
        case 0: return MonitorFunction::constant(d.R);
        case 1: return MonitorFunction::running_example(d.R);
        case 2: return MonitorFunction::huang_sloan(d.alpha, d.R);
        case 3: return MonitorFunction::mackenzie(d.alpha, d.R);
        case 4: return MonitorFunction::five_ring(d.alpha, d.R);
        case 32: {
            auto t = std::make_shared<TabRho>(d.table, d.tnx, d.tny, d.tdom);
            return MonitorFunction::user_supplied([t](Point p) { return (*t)(p); },
                                                  RectDomain(d.tdom.xmin, d.tdom.xmax, d.tdom.ymin,
                                                             d.tdom.ymax),
                                                  d.fd_h);
        }
        default: {
            const int k = d.kind;
            return MonitorFunction::user_supplied(
                [k](Point p) { return 1.0 / wl_w(k, p.x, p.y); },
                RectDomain(dom.xmin, dom.xmax, dom.ymin, dom.ymax), d.fd_h);
        }
    }
}

WalkConfig make_walk(const WalkCfgC& c) {
    WalkConfig w;
    w.scheme = c.scheme == 0 ? SchemeKind::linear : SchemeKind::exponential;
    w.dt = c.dt;
    w.lambda = c.lambda;
    w.walks = static_cast<long>(c.walks);
    w.seed = c.seed;
    w.max_steps = static_cast<long>(c.max_steps);
    w.bridge_test = c.bridge_test != 0;
    return w;
}

BoundaryData make_bd(const Domain& dom, int nx, int ny, const double* const* f,
                     const double* const* g) {
    GridSpec spec(RectDomain(dom.xmin, dom.xmax, dom.ymin, dom.ymax), nx, ny);
    auto vec = [](const double* p, int n) { return std::vector<double>(p, p + n); };
    return BoundaryData{spec,
                        EdgeData{vec(f[0], nx), vec(f[1], nx), vec(f[2], ny), vec(f[3], ny)},
                        EdgeData{vec(g[0], nx), vec(g[1], nx), vec(g[2], ny), vec(g[3], ny)}};
}

// Status codes shared with include/sddg.h.
int code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ValidationError*>(&e)) return 1;
    if (dynamic_cast<const OutOfDomainError*>(&e)) return 2;
    if (dynamic_cast<const EvaluationError*>(&e)) return 3;
    if (dynamic_cast<const NumericalError*>(&e)) return 4;
    if (dynamic_cast<const LayoutError*>(&e)) return 5;
    return 7;
}

#define GUARD_BEGIN try {
#define GUARD_END                                  \
    }                                              \
    catch (const std::exception& e) {              \
        return code_of(e);                         \
    }                                              \
    return 0;

EstimateC to_c(const McEstimate& e) {
    EstimateC o;
    std::memset(&o, 0, sizeof(o));
    o.xi = e.xi;
    o.eta = e.eta;
    o.se_xi = e.stderr_xi;
    o.se_eta = e.stderr_eta;
    o.walks = e.walks;
    o.restarts = e.restarts;
    o.warn = e.reliability_warning ? 1 : 0;
    for (int k = 0; k < 4; ++k) o.edge_hits[k] = e.edge_hits[k];
    return o;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_philox_block(uint32_t k0, uint32_t k1, const uint32_t* c, uint32_t* out) {
    const auto r = Philox4x32::block(k0, k1, {c[0], c[1], c[2], c[3]});
    for (int k = 0; k < 4; ++k) out[k] = r[k];
}

void ref_stream_u64(uint64_t seed, uint64_t pid, uint32_t walk, uint32_t epoch, int64_t n,
                    uint64_t* out) {
    RandomStream s(seed, pid, walk, epoch);
    for (int64_t k = 0; k < n; ++k) out[k] = s.next_u64();
}

void ref_stream_u01(uint64_t seed, uint64_t pid, uint32_t walk, uint32_t epoch, int64_t n,
                    int open, double* out) {
    RandomStream s(seed, pid, walk, epoch);
    for (int64_t k = 0; k < n; ++k) out[k] = open ? s.u01_open() : s.u01();
}

void ref_stream_normals(uint64_t seed, uint64_t pid, uint32_t walk, uint32_t epoch,
                        int64_t npairs, double* out) {
    RandomStream s(seed, pid, walk, epoch);
    for (int64_t k = 0; k < npairs; ++k) s.normal_pair(out[2 * k], out[2 * k + 1]);
}

int ref_rho_drift(const Density* d, const Domain* dom, int64_t n, const double* x,
                  const double* y, double* rho, double* bx, double* by) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    for (int64_t k = 0; k < n; ++k) {
        rho[k] = m.rho({x[k], y[k]});
        const Point b = m.drift({x[k], y[k]});
        bx[k] = b.x;
        by[k] = b.y;
    }
    GUARD_END
}

int ref_make_boundary(const Density* d, const Domain* dom, int nx, int ny, double* f_b,
                      double* f_t, double* f_l, double* f_r, double* g_b, double* g_t,
                      double* g_l, double* g_r) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const BoundaryData bd =
        make_boundary_data(m, GridSpec(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny));
    std::memcpy(f_b, bd.f.bottom.data(), sizeof(double) * nx);
    std::memcpy(f_t, bd.f.top.data(), sizeof(double) * nx);
    std::memcpy(f_l, bd.f.left.data(), sizeof(double) * ny);
    std::memcpy(f_r, bd.f.right.data(), sizeof(double) * ny);
    std::memcpy(g_b, bd.g.bottom.data(), sizeof(double) * nx);
    std::memcpy(g_t, bd.g.top.data(), sizeof(double) * nx);
    std::memcpy(g_l, bd.g.left.data(), sizeof(double) * ny);
    std::memcpy(g_r, bd.g.right.data(), sizeof(double) * ny);
    GUARD_END
}

// Per-path replay of run_walk (proj/src/sde.cpp:151-183) via the public API.
int ref_walk_dump(const Density* d, const Domain* dom, int nx, int ny, const double* const* f,
                  const double* const* g, const WalkCfgC* wc, double px, double py,
                  uint64_t pid, int64_t walk_lo, int64_t n, PathRec* out) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const RectDomain rd(dom->xmin, dom->xmax, dom->ymin, dom->ymax);
    const BoundaryData bd = make_bd(*dom, nx, ny, f, g);
    const WalkConfig cfg = make_walk(*wc);
    cfg.validate();
    for (int64_t k = 0; k < n; ++k) {
        const long walk = static_cast<long>(walk_lo + k);
        bool done = false;
        for (std::uint32_t epoch = 0; epoch < 1024 && !done; ++epoch) {
            RandomStream rng(cfg.seed, pid, static_cast<std::uint32_t>(walk), epoch);
            Point pos{px, py};
            for (long step = 1; step <= cfg.max_steps; ++step) {
                std::optional<ExitSample> exit;
                if (cfg.scheme == SchemeKind::linear) {
                    const Point next = step_linear(pos, m, cfg.dt, rng);
                    if (!rd.strictly_inside(next)) exit = segment_exit(pos, next, rd);
                    else if (cfg.bridge_test) exit = bridge_exit_test(pos, next, cfg.dt, rd, rng);
                    if (!exit) pos = next;
                } else {
                    auto [next, ex] = step_exponential(pos, m, cfg.lambda, rd, rng);
                    exit = ex;
                    if (!exit) pos = next;
                }
                if (exit) {
                    PathRec& r = out[k];
                    r.f = bd.f_at(exit->exit_edge, exit->exit_point);
                    r.g = bd.g_at(exit->exit_edge, exit->exit_point);
                    r.ex = exit->exit_point.x;
                    r.ey = exit->exit_point.y;
                    r.steps = step;
                    r.epoch = static_cast<int32_t>(epoch);
                    r.edge = static_cast<int32_t>(exit->exit_edge);
                    done = true;
                    break;
                }
            }
        }
        if (!done) throw NumericalError("walk failed to exit after 1024 restarts");
    }
    GUARD_END
}

// sdd::mc_estimate at each node; `threads` > 1 runs the nodes through
// sdd::parallel_for exactly as solve_interfaces does
// (proj/src/decomposition.cpp:172-174).
int ref_mc_estimate_batch(const Density* d, const Domain* dom, int nx, int ny,
                          const double* const* f, const double* const* g, const WalkCfgC* wc,
                          const double* px, const double* py, const uint64_t* pid, int64_t n,
                          int threads, EstimateC* out) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const RectDomain rd(dom->xmin, dom->xmax, dom->ymin, dom->ymax);
    const BoundaryData bd = make_bd(*dom, nx, ny, f, g);
    const WalkConfig cfg = make_walk(*wc);
    std::vector<McEstimate> est(static_cast<std::size_t>(n));
    parallel_for(static_cast<std::size_t>(n), threads <= 0 ? hardware_threads() : threads,
                 [&](std::size_t k) {
                     est[k] = mc_estimate({px[k], py[k]}, pid[k], m, rd, bd, cfg, 1);
                 });
    for (int64_t k = 0; k < n; ++k) out[k] = to_c(est[static_cast<std::size_t>(k)]);
    GUARD_END
}

int ref_hardware_threads() { return hardware_threads(); }

int ref_weight_values(const Density* d, const Domain* dom, int nx, int ny, double* w) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const auto v = weight_values(
        m, GridSpec(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny));
    std::memcpy(w, v.data(), sizeof(double) * v.size());
    GUARD_END
}

int ref_solve_dirichlet(const double* w, int nx, int ny, double hx, double hy,
                        const double* bottom, const double* top, const double* left,
                        const double* right, double tol, int64_t max_iters, int init_blend,
                        double* u_out, int64_t* iters, double* final_update, int* converged) {
    GUARD_BEGIN
    std::vector<double> wv(w, w + static_cast<std::size_t>(nx) * ny);
    EdgeData bc{std::vector<double>(bottom, bottom + nx), std::vector<double>(top, top + nx),
                std::vector<double>(left, left + ny), std::vector<double>(right, right + ny)};
    SolverConfig sc;
    sc.tol = tol;
    sc.max_iters = static_cast<long>(max_iters);
    sc.init_blend = init_blend != 0;
    const SolveResult r = solve_dirichlet(wv, nx, ny, hx, hy, bc, sc);
    std::memcpy(u_out, r.field.values.data(), sizeof(double) * r.field.values.size());
    *iters = r.iterations;
    *final_update = r.final_update;
    *converged = r.converged ? 1 : 0;
    GUARD_END
}

// plan_interface_points over build_layout; out_nodes gets each line's nodes
// back to back, out_counts the per-line counts.  Lines are in layout order
// (vertical first, proj/src/decomposition.cpp:44-51).
int ref_plan(const Density* d, const Domain* dom, int nx, int ny, int sx, int sy,
             int strategy, int k, int* n_lines, int* out_vertical, int* out_fixed,
             int* out_counts, int* out_nodes) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const SubdomainLayout lay = build_layout(
        GridSpec(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny), sx, sy);
    const PlacementStrategy ps = strategy == 0   ? PlacementStrategy::all
                                 : strategy == 1 ? PlacementStrategy::equispaced
                                                 : PlacementStrategy::optimal;
    const InterfacePlan plan = plan_interface_points(ps, k, m, lay);
    *n_lines = static_cast<int>(lay.lines.size());
    int off = 0;
    for (std::size_t l = 0; l < lay.lines.size(); ++l) {
        out_vertical[l] = lay.lines[l].vertical ? 1 : 0;
        out_fixed[l] = lay.lines[l].fixed_index;
        out_counts[l] = static_cast<int>(plan.stochastic[l].size());
        for (int v : plan.stochastic[l]) out_nodes[off++] = v;
    }
    GUARD_END
}

// solve_interfaces with caller tables; xi_out/eta_out/se_* hold the per-line
// full node ranges back to back (line lengths per layout).
int ref_solve_interfaces(const Density* d, const Domain* dom, int nx, int ny, int sx, int sy,
                         int strategy, int k, const double* const* f, const double* const* g,
                         const WalkCfgC* wc, int threads, double* xi_out, double* eta_out,
                         double* sexi_out, double* seeta_out, int64_t* mc_points,
                         int64_t* restarts) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const SubdomainLayout lay = build_layout(
        GridSpec(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny), sx, sy);
    const PlacementStrategy ps = strategy == 0   ? PlacementStrategy::all
                                 : strategy == 1 ? PlacementStrategy::equispaced
                                                 : PlacementStrategy::optimal;
    const InterfacePlan plan = plan_interface_points(ps, k, m, lay);
    const BoundaryData bd = make_bd(*dom, nx, ny, f, g);
    const InterfaceSolution s = solve_interfaces(plan, m, bd, make_walk(*wc), lay,
                                                 threads <= 0 ? hardware_threads() : threads);
    std::size_t off = 0;
    for (std::size_t l = 0; l < s.xi.size(); ++l) {
        for (std::size_t q = 0; q < s.xi[l].size(); ++q) {
            xi_out[off + q] = s.xi[l][q];
            eta_out[off + q] = s.eta[l][q];
            sexi_out[off + q] = s.se_xi[l][q];
            seeta_out[off + q] = s.se_eta[l][q];
        }
        off += s.xi[l].size();
    }
    *mc_points = s.mc_points;
    *restarts = s.restarts;
    GUARD_END
}

// Full solve_sdd (reference boundary data, proj/src/decomposition.cpp:262-385).
int ref_solve_sdd(const Density* d, const Domain* dom, int nx, int ny, int sx, int sy,
                  int strategy, int k, const WalkCfgC* wc, double tol, int64_t max_iters,
                  int threads, double* xi_out, double* eta_out, double* times_out) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const SubdomainLayout lay = build_layout(
        GridSpec(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny), sx, sy);
    const PlacementStrategy ps = strategy == 0   ? PlacementStrategy::all
                                 : strategy == 1 ? PlacementStrategy::equispaced
                                                 : PlacementStrategy::optimal;
    const InterfacePlan plan = plan_interface_points(ps, k, m, lay);
    SolverConfig sc;
    sc.tol = tol;
    sc.max_iters = static_cast<long>(max_iters);
    const SddResult r = solve_sdd(m, lay, plan, make_walk(*wc), sc, SddOptions{},
                                  threads <= 0 ? hardware_threads() : threads);
    std::memcpy(xi_out, r.sol.xi.values.data(), sizeof(double) * r.sol.xi.values.size());
    std::memcpy(eta_out, r.sol.eta.values.data(), sizeof(double) * r.sol.eta.values.size());
    times_out[0] = r.t_stoc;
    times_out[1] = r.t_sub;
    times_out[2] = r.t_smooth;
    GUARD_END
}

// invert_mesh (proj/src/invert.cpp:140-196) of a solution on the nx x ny grid over dom.
int ref_invert_mesh(const double* xi, const double* eta, int nx, int ny, const Domain* dom,
                    int m_xi, int m_eta, int threads, double* x_out, double* y_out) {
    GUARD_BEGIN
    const GridSpec g(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny);
    const MeshSolution sol(ScalarField(g, std::vector<double>(xi, xi + g.size())),
                           ScalarField(g, std::vector<double>(eta, eta + g.size())));
    const PhysicalMesh mesh = invert_mesh(sol, m_xi, m_eta, threads);
    std::memcpy(x_out, mesh.x.data(), sizeof(double) * mesh.x.size());
    std::memcpy(y_out, mesh.y.data(), sizeof(double) * mesh.y.size());
    GUARD_END
}

// quality_report (proj/src/quality.cpp:35-80); ref_x/ref_y and d may be null.
// out = {q_max, q_mean, r_max, r_mean, l_inf}
int ref_quality(const double* x, const double* y, int m_xi, int m_eta, const Domain* dom,
                const double* ref_x, const double* ref_y, const Density* d, double* out) {
    GUARD_BEGIN
    const RectDomain rd(dom->xmin, dom->xmax, dom->ymin, dom->ymax);
    PhysicalMesh mesh(m_xi, m_eta, rd);
    const std::size_t n = static_cast<std::size_t>(m_xi) * m_eta;
    mesh.x.assign(x, x + n);
    mesh.y.assign(y, y + n);
    PhysicalMesh ref(m_xi, m_eta, rd);
    if (ref_x) {
        ref.x.assign(ref_x, ref_x + n);
        ref.y.assign(ref_y, ref_y + n);
    }
    std::optional<MonitorFunction> m;
    if (d) m.emplace(make_monitor(*d, *dom));
    const QualityReport q = quality_report(mesh, ref_x ? &ref : nullptr, m ? &*m : nullptr);
    out[0] = q.q_max;
    out[1] = q.q_mean;
    out[2] = q.r_max.value_or(0.0);
    out[3] = q.r_mean.value_or(0.0);
    out[4] = q.l_inf.value_or(0.0);
    GUARD_END
}

// solve_single_domain (proj/src/detsolver.cpp:226-246)
int ref_solve_single_domain(const Density* d, const Domain* dom, int nx, int ny, double tol,
                            double* xi, double* eta) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    SolverConfig sc;
    sc.tol = tol;
    const MeshSolveResult r = solve_single_domain(
        m, GridSpec(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny), sc);
    std::memcpy(xi, r.sol.xi.values.data(), sizeof(double) * r.sol.xi.values.size());
    std::memcpy(eta, r.sol.eta.values.data(), sizeof(double) * r.sol.eta.values.size());
    GUARD_END
}

// perona_malik (proj/src/smoothing.cpp:127-138) in place; scope 0 global, 1 per-subdomain
int ref_perona_malik(double* xi, double* eta, int nx, int ny, const Domain* dom, double k,
                     double dt, int steps, int scope, int sx, int sy) {
    GUARD_BEGIN
    const GridSpec g(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny);
    const MeshSolution sol(ScalarField(g, std::vector<double>(xi, xi + g.size())),
                           ScalarField(g, std::vector<double>(eta, eta + g.size())));
    SmoothConfig c;
    c.k = k;
    c.dt = dt;
    c.steps = steps;
    c.scope = scope == 1 ? SmoothScope::per_subdomain : SmoothScope::global;
    std::optional<SubdomainLayout> lay;
    if (scope == 1) lay.emplace(build_layout(g, sx, sy));
    const MeshSolution out = perona_malik(sol, c, lay ? &*lay : nullptr);
    std::memcpy(xi, out.xi.values.data(), sizeof(double) * g.size());
    std::memcpy(eta, out.eta.values.data(), sizeof(double) * g.size());
    GUARD_END
}

int ref_smooth_interface(const double* v, int n, int span, double* out) {
    GUARD_BEGIN
    const std::vector<double> r = smooth_interface(std::vector<double>(v, v + n), span);
    std::memcpy(out, r.data(), sizeof(double) * n);
    GUARD_END
}

// solve_sdd with SddOptions{smooth_interface=true, span}
int ref_solve_sdd_smoothed(const Density* d, const Domain* dom, int nx, int ny, int sx, int sy,
                           int strategy, int k, const WalkCfgC* wc, double tol, int span,
                           double* xi_out, double* eta_out) {
    GUARD_BEGIN
    const MonitorFunction m = make_monitor(*d, *dom);
    const SubdomainLayout lay = build_layout(
        GridSpec(RectDomain(dom->xmin, dom->xmax, dom->ymin, dom->ymax), nx, ny), sx, sy);
    const PlacementStrategy ps = strategy == 0   ? PlacementStrategy::all
                                 : strategy == 1 ? PlacementStrategy::equispaced
                                                 : PlacementStrategy::optimal;
    const InterfacePlan plan = plan_interface_points(ps, k, m, lay);
    SolverConfig sc;
    sc.tol = tol;
    SddOptions o;
    o.smooth_interface = true;
    o.smooth_span = span;
    const SddResult r = solve_sdd(m, lay, plan, make_walk(*wc), sc, o, 4);
    std::memcpy(xi_out, r.sol.xi.values.data(), sizeof(double) * r.sol.xi.values.size());
    std::memcpy(eta_out, r.sol.eta.values.data(), sizeof(double) * r.sol.eta.values.size());
    GUARD_END
}

int ref_write_mesh(const double* x, const double* y, int m_xi, int m_eta, const double* xi,
                   const double* eta, int nx, int ny, const char* path) {
    GUARD_BEGIN
    const RectDomain rd(0, 1, 0, 1);
    PhysicalMesh mesh(m_xi, m_eta, rd);
    const std::size_t n = static_cast<std::size_t>(m_xi) * m_eta;
    mesh.x.assign(x, x + n);
    mesh.y.assign(y, y + n);
    const GridSpec g(rd, nx, ny);
    const MeshSolution sol(ScalarField(g, std::vector<double>(xi, xi + g.size())),
                           ScalarField(g, std::vector<double>(eta, eta + g.size())));
    write_mesh(mesh, sol, path);
    GUARD_END
}

}  // extern "C"
