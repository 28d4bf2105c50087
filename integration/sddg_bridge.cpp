// sddg_bridge.cpp -- the reference-side binding of the B200 path: what a
// maintainer adds to the reference tree (proj/src/sddg_bridge.cpp) so that
// the unmodified sddmesh library runs its two hot loops on the GPU through
// the C-ABI of include/sddg.h.  See INTEGRATION.md.
//
// Two seams of the reference are replaced at link time, with no edit to the
// reference's sources: the linker's --wrap routes every call to
//   sdd::mc_estimate      (proj/include/sdd/sde.hpp:75-77; called per node by
//                          solve_interfaces, decomposition.cpp:172-174, and
//                          run_stochastic_full, cli.cpp:258-262)
//   sdd::solve_dirichlet  (proj/include/sdd/detsolver.hpp:44-45; called per
//                          subdomain and field by solve_sdd, decomposition.cpp:349-350)
// to the functions below, which call sddg_mc_estimate_batch and
// sddg_solve_dirichlet_batch.  Everything else -- layout, placement, the
// interface fill and crossing reconciliation, boundary data, assembly,
// smoothing, inversion, quality -- stays the reference's own code.
//
// The reference's MonitorFunction hides a std::function for user densities,
// which a GPU cannot call: builtin kinds map directly; a user_supplied
// density needs a data descriptor from the caller (sddg_bridge_set_user_density:
// one of the BASELINE kinds, or a tabulated rho on a grid).
//
// Build: oracle/Makefile target `bridge` (the reference objects + this file +
// the reference's own harness, linked with -Wl,--wrap=<the two symbols>).
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "sddg.h"
#include "sdd/boundary.hpp"
#include "sdd/decomposition.hpp"
#include "sdd/detsolver.hpp"
#include "sdd/errors.hpp"
#include "sdd/monitor.hpp"
#include "sdd/sde.hpp"

namespace sdd {

// The original definitions (the linker's __real_ aliases) and the GPU
// replacements (__wrap_), under the mangled names of the two seams.
McEstimate real_mc_estimate(Point p, std::uint64_t point_id, const MonitorFunction& m,
                            const RectDomain& domain, const BoundaryData& bd, const WalkConfig& cfg,
                            int threads)
    __asm__("__real__ZN3sdd11mc_estimateENS_5PointEmRKNS_15MonitorFunctionERKNS_10RectDomainERKNS_12BoundaryDataERKNS_10WalkConfigEi");
McEstimate gpu_mc_estimate(Point p, std::uint64_t point_id, const MonitorFunction& m,
                           const RectDomain& domain, const BoundaryData& bd, const WalkConfig& cfg,
                           int threads)
    __asm__("__wrap__ZN3sdd11mc_estimateENS_5PointEmRKNS_15MonitorFunctionERKNS_10RectDomainERKNS_12BoundaryDataERKNS_10WalkConfigEi");
SolveResult real_solve_dirichlet(const std::vector<double>& w, int nx, int ny, double hx, double hy,
                                 const EdgeData& bc, const SolverConfig& cfg)
    __asm__("__real__ZN3sdd15solve_dirichletERKSt6vectorIdSaIdEEiiddRKNS_8EdgeDataERKNS_12SolverConfigE");
SolveResult gpu_solve_dirichlet(const std::vector<double>& w, int nx, int ny, double hx, double hy,
                                const EdgeData& bc, const SolverConfig& cfg)
    __asm__("__wrap__ZN3sdd15solve_dirichletERKSt6vectorIdSaIdEEiiddRKNS_8EdgeDataERKNS_12SolverConfigE");

namespace {

struct BridgeState {
    std::mutex mu;
    sddg_ctx* ctx = nullptr;
    int device = 0;
    // user_supplied densities: the descriptor the caller registered
    bool have_user = false;
    sddg_density user{};
    std::vector<double> user_table;  // rho samples of a tabulated density
    int solver_method = SDDG_SOLVER_JACOBI;  // the reference iteration, bit for bit
    bool on = true;                          // false: route to the reference's CPU code
};

BridgeState& state() {
    static BridgeState s;
    return s;
}

sddg_ctx* context() {
    BridgeState& s = state();
    if (!s.ctx) {
        const sddg_status st = sddg_create(s.device, &s.ctx);
        if (st != SDDG_OK) throw Error(std::string("sddg_create: ") + sddg_last_error(nullptr));
    }
    return s.ctx;
}

// sddg_status -> the reference's exception classes (proj/include/sdd/errors.hpp:8-32)
void check(sddg_status st, const sddg_ctx* ctx) {
    if (st == SDDG_OK) return;
    const std::string msg = sddg_last_error(ctx);
    switch (st) {
        case SDDG_ERR_VALIDATION: throw ValidationError(msg);
        case SDDG_ERR_OUT_OF_DOMAIN: throw OutOfDomainError(msg);
        case SDDG_ERR_EVALUATION: throw EvaluationError(msg);
        case SDDG_ERR_NUMERICAL: throw NumericalError(msg);
        case SDDG_ERR_LAYOUT: throw LayoutError(msg);
        default: throw Error(msg);
    }
}

sddg_density to_sddg(const MonitorFunction& m) {
    sddg_density d{};
    d.grad_mode = SDDG_GRAD_REFERENCE;  // what the reference computes
    d.R = m.param_R();
    d.alpha = m.param_alpha();
    d.fd_h = 1e-6;
    switch (m.kind()) {
        case MonitorKind::constant: d.kind = SDDG_DENS_CONSTANT; break;
        case MonitorKind::running_example: d.kind = SDDG_DENS_RUNNING; break;
        case MonitorKind::huang_sloan: d.kind = SDDG_DENS_HUANG_SLOAN; break;
        case MonitorKind::mackenzie: d.kind = SDDG_DENS_MACKENZIE; break;
        case MonitorKind::five_ring: d.kind = SDDG_DENS_FIVE_RING; break;
        case MonitorKind::user_supplied: {
            const BridgeState& s = state();
            if (!s.have_user)
                throw ValidationError(
                    "sddg bridge: a user_supplied density needs a descriptor "
                    "(sddg_bridge_set_user_density)");
            d = s.user;
            if (d.kind == SDDG_DENS_TABLE) d.table = s.user_table.data();
            break;
        }
    }
    return d;
}

sddg_boundary to_sddg(const BoundaryData& bd) {
    sddg_boundary b{};
    b.dom = {bd.spec.domain.xmin, bd.spec.domain.xmax, bd.spec.domain.ymin, bd.spec.domain.ymax};
    b.nx = bd.spec.nx;
    b.ny = bd.spec.ny;
    const EdgeData* e[2] = {&bd.f, &bd.g};
    for (int fg = 0; fg < 2; ++fg) {
        const double* t[4] = {e[fg]->bottom.data(), e[fg]->top.data(), e[fg]->left.data(),
                              e[fg]->right.data()};
        for (int k = 0; k < 4; ++k) (fg == 0 ? b.f : b.g)[k] = t[k];
    }
    return b;
}

}  // namespace

McEstimate gpu_mc_estimate(Point p, std::uint64_t point_id, const MonitorFunction& m,
                           const RectDomain& domain, const BoundaryData& bd, const WalkConfig& cfg,
                           int threads) {
    BridgeState& s = state();
    if (!s.on) return real_mc_estimate(p, point_id, m, domain, bd, cfg, threads);
    std::lock_guard<std::mutex> lk(s.mu);  // parallel_for workers share one context
    sddg_ctx* ctx = context();
    const sddg_density d = to_sddg(m);
    const sddg_domain dom{domain.xmin, domain.xmax, domain.ymin, domain.ymax};
    const sddg_boundary b = to_sddg(bd);
    const sddg_walk_config wc{cfg.scheme == SchemeKind::linear ? SDDG_SCHEME_LINEAR : SDDG_SCHEME_EXPONENTIAL,
                              SDDG_FP64, cfg.dt, cfg.lambda, static_cast<int64_t>(cfg.walks), cfg.seed,
                              static_cast<int64_t>(cfg.max_steps), cfg.bridge_test ? 1 : 0, 0};
    sddg_estimate r;
    check(sddg_mc_estimate_batch(ctx, &d, &dom, &b, &wc, &p.x, &p.y, &point_id, 1, &r), ctx);
    McEstimate e;
    e.xi = r.xi;
    e.eta = r.eta;
    e.stderr_xi = r.se_xi;
    e.stderr_eta = r.se_eta;
    e.walks = static_cast<long>(r.walks);
    e.restarts = static_cast<long>(r.restarts);
    e.reliability_warning = r.warn != 0;
    for (int q = 0; q < 4; ++q) e.edge_hits[q] = static_cast<long>(r.edge_hits[q]);
    return e;
}

SolveResult gpu_solve_dirichlet(const std::vector<double>& w, int nx, int ny, double hx, double hy,
                                const EdgeData& bc, const SolverConfig& cfg) {
    BridgeState& s = state();
    if (!s.on) return real_solve_dirichlet(w, nx, ny, hx, hy, bc, cfg);
    std::lock_guard<std::mutex> lk(s.mu);
    sddg_ctx* ctx = context();
    cfg.validate();
    if (static_cast<long>(w.size()) != static_cast<long>(nx) * ny)
        throw ValidationError("solve_dirichlet: weight array size does not match the grid");
    std::vector<double> packed;
    packed.reserve(2 * (nx + ny));
    for (const std::vector<double>* e : {&bc.bottom, &bc.top, &bc.left, &bc.right}) {
        if (static_cast<int>(e->size()) != ((e == &bc.bottom || e == &bc.top) ? nx : ny))
            throw ValidationError("solve_dirichlet: edge data size does not match the grid");
        packed.insert(packed.end(), e->begin(), e->end());
    }
    const sddg_subdomain sub{0, 0, nx, ny};
    const sddg_solver_config sc{cfg.tol, static_cast<int64_t>(cfg.max_iters), cfg.init_blend ? 1 : 0,
                                s.solver_method, 0.0};
    SolveResult r{ScalarField(GridSpec(RectDomain(0.0, hx * (nx - 1), 0.0, hy * (ny - 1)), nx, ny))};
    sddg_solve_info info;
    check(sddg_solve_dirichlet_batch(ctx, w.data(), nx, ny, hx, hy, 1, &sub, packed.data(), &sc,
                                     r.field.values.data(), &info),
          ctx);
    r.iterations = static_cast<long>(info.iterations);
    r.final_update = info.final_update;
    r.converged = info.converged != 0;
    if (!r.converged)
        r.warning = "solve_dirichlet: reached max_iters=" + std::to_string(cfg.effective_max_iters(nx, ny)) +
                    " with update " + std::to_string(r.final_update);
    return r;
}

}  // namespace sdd

extern "C" {

// Route the two seams to the GPU (1, default) or to the reference's own CPU
// code (0); pick the device and the subdomain iteration (SDDG_SOLVER_JACOBI:
// the reference's, bit for bit; SDDG_SOLVER_RBSOR: same fixed point, O(n) sweeps).
void sddg_bridge_configure(int on, int device, int solver_method) {
    sdd::BridgeState& s = sdd::state();
    std::lock_guard<std::mutex> lk(s.mu);
    s.on = on != 0;
    if (s.ctx && device != s.device) {
        sddg_destroy(s.ctx);
        s.ctx = nullptr;
    }
    s.device = device;
    s.solver_method = solver_method;
}

// The data descriptor of the caller's user_supplied density.  table
// (nullable) holds the rho samples of a SDDG_DENS_TABLE density.
void sddg_bridge_set_user_density(const sddg_density* d) {
    sdd::BridgeState& s = sdd::state();
    std::lock_guard<std::mutex> lk(s.mu);
    s.have_user = d != nullptr;
    if (!d) return;
    s.user = *d;
    s.user_table.clear();
    if (d->kind == SDDG_DENS_TABLE && d->table)
        s.user_table.assign(d->table, d->table + static_cast<size_t>(d->tnx) * d->tny);
}

}  // extern "C"
