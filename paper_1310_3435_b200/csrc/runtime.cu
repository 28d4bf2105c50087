// runtime.cu -- host runtime behind include/sddg.h.
//
// Owns the device context (stream, grow-only device buffers, event timers)
// and implements the reference's host-side orchestration around the two GPU
// kernels: validation with the reference's error classes, node batching for
// the walk kernel (K1) and its fixed-order finalize (K2), the subdomain solve
// batch (K3), and the decomposition logic of proj/src/decomposition.cpp
// (layout, placement, interface fill, assembly).  No compute path runs on the
// CPU: every Monte Carlo walk and every subdomain iteration is a kernel.
#include <cuda_runtime.h>
#include <nvtx3/nvtx3.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <map>
#include <optional>
#include <mutex>
#include <string>
#include <vector>

#include "fastmath.cuh"
#include "host_density.h"
#include "runtime_internal.h"
#include "sddg_internal.h"

using namespace sddg;
using namespace sddg::rt;

namespace {

// batch start: the walk counter past the grid's first walks, the walks in
// flight, and no handoff yet
__global__ void set_next_kernel(Counters* c, unsigned long long v, unsigned long long live) {
    c->next = v;
    c->live = live;
    c->n_cont = 0;
    for (int r = 0; r < kMaxDrain; ++r) c->n_drain[r] = 0;
}

// drain round start: the walks in flight are the previous round's handoffs
__global__ void drain_prep_kernel(Counters* c, const unsigned int* n_src, unsigned int cap) {
    c->live = min(*n_src, cap);
}

thread_local std::string g_free_err;

}  // namespace

namespace sddg {
namespace rt {

// ------------------------------------------------------------ validation

void validate_walk(const sddg_walk_config& c) {
    // WalkConfig::validate (proj/src/sde.cpp:12-19)
    if (c.scheme == SDDG_SCHEME_LINEAR && !(c.dt > 0.0))
        fail(SDDG_ERR_VALIDATION, "WalkConfig: linear scheme needs dt > 0");
    if (c.scheme == SDDG_SCHEME_EXPONENTIAL && !(c.lambda > 0.0))
        fail(SDDG_ERR_VALIDATION, "WalkConfig: exponential scheme needs lambda > 0");
    if (c.scheme != SDDG_SCHEME_LINEAR && c.scheme != SDDG_SCHEME_EXPONENTIAL)
        fail(SDDG_ERR_VALIDATION, "WalkConfig: unknown scheme");
    if (c.walks < 1) fail(SDDG_ERR_VALIDATION, "WalkConfig: walks must be >= 1");
    if (c.walks > 0xFFFFFFFFLL)
        fail(SDDG_ERR_VALIDATION, "WalkConfig: walks must fit the 32-bit stream walk id");
    if (c.max_steps < 1) fail(SDDG_ERR_VALIDATION, "WalkConfig: max_steps must be >= 1");
    // A step draws at most 7 u64s (exponential scheme: 1 + 2 + 4 edges), and
    // the per-epoch draw counter (LaneStream::n) is 32-bit: 2^29 steps keep it
    // below 2^32 draws, so the stream never wraps (the reference's counter
    // would wrap at 2^32 blocks and draw differently).  Default: 1e7.
    if (c.max_steps > (int64_t(1) << 29))
        fail(SDDG_ERR_VALIDATION, "WalkConfig: max_steps must be <= 2^29 (536870912)");
    if (c.precision != SDDG_FP64 && c.precision != SDDG_FP32)
        fail(SDDG_ERR_VALIDATION, "WalkConfig: unknown precision");
}

// A tabulated density: a table, >= 2 x 2 finite positive samples over a
// non-empty domain (the reference's user_supplied checks its rho the same
// way, monitor.cpp:105-119, on the interpolant: check_positivity).
void check_table(const sddg_density& d) {
    if (!d.table) fail(SDDG_ERR_VALIDATION, "tabulated density: table is NULL");
    if (d.tnx < 2 || d.tny < 2) fail(SDDG_ERR_VALIDATION, "tabulated density: needs at least 2 x 2 samples");
    if (!(d.tdom.xmin < d.tdom.xmax) || !(d.tdom.ymin < d.tdom.ymax))
        fail(SDDG_ERR_VALIDATION, "tabulated density: empty domain");
    if (!(d.fd_h > 0.0)) fail(SDDG_ERR_VALIDATION, "fd_h must be > 0");
    for (int64_t k = 0; k < static_cast<int64_t>(d.tnx) * d.tny; ++k)
        if (!std::isfinite(d.table[k]) || d.table[k] <= 0.0)
            fail(SDDG_ERR_EVALUATION, "tabulated density: samples must be finite and > 0");
}

int drift_variant(const sddg_density& d, int precision) {
    if (d.kind == SDDG_DENS_TABLE) {
        check_table(d);
        if (d.grad_mode == SDDG_GRAD_ANALYTIC) return 36;  // DV_TABLE_AN
        if (d.grad_mode != SDDG_GRAD_REFERENCE) fail(SDDG_ERR_VALIDATION, "unknown grad_mode");
        if (precision == SDDG_FP32)
            fail(SDDG_ERR_VALIDATION, "fp32 walks need the analytic drift (grad_mode SDDG_GRAD_ANALYTIC)");
        return 20;  // DV_TABLE_FD
    }
    const bool wkind = d.kind >= SDDG_DENS_RING_W && d.kind <= SDDG_DENS_TWOBUMP_W;
    const bool builtin = d.kind >= SDDG_DENS_CONSTANT && d.kind <= SDDG_DENS_FIVE_RING;
    if (!wkind && !builtin) fail(SDDG_ERR_VALIDATION, "unknown density kind");
    if (d.grad_mode == SDDG_GRAD_ANALYTIC) {
        if (d.kind == SDDG_DENS_FIVE_RING) return 35;  // DV_FIVE_RING_AN
        if (!wkind)
            fail(SDDG_ERR_VALIDATION,
                 "performance-mode drift exists for the BASELINE densities (kinds 16-18) and "
                 "the five-ring (kind 4)");
        return 32 + (d.kind - SDDG_DENS_RING_W);
    }
    if (d.grad_mode != SDDG_GRAD_REFERENCE) fail(SDDG_ERR_VALIDATION, "unknown grad_mode");
    if (precision == SDDG_FP32)
        fail(SDDG_ERR_VALIDATION,
             "fp32 walks need the analytic drift (grad_mode SDDG_GRAD_ANALYTIC)");
    if (wkind && !(d.fd_h > 0.0)) fail(SDDG_ERR_VALIDATION, "fd_h must be > 0");
    return d.kind;
}

void check_table(const sddg_density& d);

// The walk kernel variant of (density, walk config): the drift variant, or
// for BASELINE's literal SDE (cfg.form) its own variant (the BASELINE
// weights, performance mode, linear scheme).
int walk_variant(const sddg_density& d, const sddg_walk_config& cfg) {
    if (cfg.form == SDDG_FORM_REFERENCE) return drift_variant(d, cfg.precision);
    if (cfg.form != SDDG_FORM_LITERAL) fail(SDDG_ERR_VALIDATION, "WalkConfig: unknown SDE form");
    if (d.kind < SDDG_DENS_RING_W || d.kind > SDDG_DENS_TWOBUMP_W)
        fail(SDDG_ERR_VALIDATION, "the literal SDE form exists for the BASELINE weights (kinds 16-18)");
    if (cfg.scheme != SDDG_SCHEME_LINEAR)
        fail(SDDG_ERR_VALIDATION, "the literal SDE form runs the linear scheme");
    return 40 + (d.kind - SDDG_DENS_RING_W);  // DV_RING_LIT ..
}

HostDensity host_density(const sddg_density& d) {
    if (d.kind == SDDG_DENS_TABLE) check_table(d);
    return HostDensity::of(d);
}

// MonitorFunction::check_positivity (proj/src/monitor.cpp:105-119) over the
// density's domain: the builtins' own, the caller's for user_supplied kinds.
void check_positivity(const sddg_density& d, const sddg_domain& dom) {
    sddg_domain pd = dom;
    if (d.kind <= SDDG_DENS_MACKENZIE) pd = {0, 1, 0, 1};
    if (d.kind == SDDG_DENS_FIVE_RING) pd = {-1, 1, -1, 1};
    if (d.kind == SDDG_DENS_TABLE) pd = d.tdom;
    const HostDensity h = host_density(d);
    for (int j = 0; j < 33; ++j)
        for (int i = 0; i < 33; ++i) {
            const double x = pd.xmin + (pd.xmax - pd.xmin) * i / 32;
            const double y = pd.ymin + (pd.ymax - pd.ymin) * j / 32;
            double r;
            try {
                r = h.rho(x, y);
            } catch (const std::exception&) {
                r = NAN;
            }
            if (!std::isfinite(r) || r <= 0.0)
                fail(SDDG_ERR_EVALUATION, "monitor density not finite/positive");
        }
}

void check_domain(const sddg_domain& d) {
    if (!(d.xmin < d.xmax) || !(d.ymin < d.ymax))
        fail(SDDG_ERR_VALIDATION, "RectDomain: requires xmin < xmax and ymin < ymax");
}

void check_boundary(const sddg_boundary& b) {
    check_domain(b.dom);
    if (b.nx < 3 || b.ny < 3) fail(SDDG_ERR_VALIDATION, "GridSpec: needs nx >= 3 and ny >= 3");
    for (int k = 0; k < 4; ++k)
        if (!b.f[k] || !b.g[k]) fail(SDDG_ERR_VALIDATION, "boundary table pointer is NULL");
}

// ------------------------------------------------------------ K1 + K2

// Persistent grid of the walk kernel: (CTAs, threads per CTA)
std::pair<int, int> walk_grid(sddg_ctx* c, int dv, int prec, uint64_t total) {
    const int key = dv * 2 + prec;
    auto it = c->occ.find(key);
    std::pair<int, int> o;
    if (it == c->occ.end()) {
        ck(walk_occupancy(dv, prec, &o.first, &o.second), "occupancy");
        c->occ[key] = o;
    } else {
        o = it->second;
    }
    const uint64_t blk = static_cast<uint64_t>(o.second);
    const uint64_t full = static_cast<uint64_t>(std::max(1, o.first)) * c->sms;
    const uint64_t need = (total + blk - 1) / blk;
    return {static_cast<int>(std::max<uint64_t>(1, std::min(full, need))), o.second};
}

int64_t batch_budget_walks() {
    const char* e = std::getenv("SDDG_MAX_BATCH_WALKS");
    if (e) {
        const long long v = std::atoll(e);
        if (v > 0) return v;
    }
    return int64_t(1) << 27;  // 2.7 GB of walk records
}

void fill_args(WalkArgs& a, const sddg_density& d, const sddg_domain& dom,
               const sddg_boundary& bd, const sddg_walk_config& cfg, const double* dtab) {
    std::memset(&a, 0, sizeof(a));
    a.xmin = dom.xmin;
    a.xmax = dom.xmax;
    a.ymin = dom.ymin;
    a.ymax = dom.ymax;
    a.txmin = bd.dom.xmin;
    a.tymin = bd.dom.ymin;
    a.thx = (bd.dom.xmax - bd.dom.xmin) / (bd.nx - 1);  // GridSpec::hx (geometry.hpp:52)
    a.thy = (bd.dom.ymax - bd.dom.ymin) / (bd.ny - 1);
    a.tnx = bd.nx;
    a.tny = bd.ny;
    const int64_t nx = bd.nx, ny = bd.ny;
    const int64_t offs[4] = {0, nx, 2 * nx, 2 * nx + ny};
    for (int k = 0; k < 4; ++k) {
        a.tf[k] = dtab + offs[k];
        a.tg[k] = dtab + 2 * (nx + ny) + offs[k];
    }
    a.R = d.R;
    a.alpha = d.alpha;
    a.fd_h = d.fd_h;
    a.scheme = cfg.scheme;
    a.bridge = cfg.bridge_test ? 1 : 0;
    a.dt = cfg.dt;
    a.sqrt2dt = std::sqrt(2.0 * cfg.dt);  // step_linear (sde.cpp:27)
    a.inv_dt = 1.0 / cfg.dt;
    a.half_inv_lambda = 0.5 / cfg.lambda;
    a.lambda = cfg.lambda;
    a.nu2 = 2.0 * std::sqrt(cfg.lambda);  // step_exponential (sde.cpp:135)
    a.bridge_thr = 40.0 * cfg.dt * (1.0 + (cfg.precision == SDDG_FP32 ? 1e-5 : 1e-12));
    // inner box: both endpoints farther than s >= sqrt(bridge_thr) from every
    // edge => every d0*d1 > bridge_thr => no bridge draw possible
    // literal SDE: the bridge threshold scales with w (d0 d1 <= 40 w dt),
    // so the inner box takes w's maximum (ring 11, shock 21, two-bump < 31)
    const double wmax = cfg.form == SDDG_FORM_LITERAL
                            ? (d.kind == SDDG_DENS_RING_W ? 11.0 : (d.kind == SDDG_DENS_SHOCK_W ? 21.0 : 31.0))
                            : 1.0;
    const double sbox = std::sqrt(a.bridge_thr * wmax) * (1.0 + 1e-6);
    a.box[0] = dom.xmin + sbox;
    a.box[1] = dom.xmax - sbox;
    a.box[2] = dom.ymin + sbox;
    a.box[3] = dom.ymax - sbox;
    // integer form of the box test (performance mode): for positive doubles a
    // strictly larger high word means a strictly larger value, so comparing
    // high words is a conservative (slightly smaller) box.  Needs the box in
    // the positive quadrant; otherwise it never fires and every step takes
    // the exact path.
    const bool pos = a.box[0] > 0.0 && a.box[2] > 0.0 && a.box[0] < a.box[1] && a.box[2] < a.box[3];
    for (int k = 0; k < 4; ++k) {
        int64_t bits;
        std::memcpy(&bits, &a.box[k], 8);
        a.box_hi[k] = static_cast<int32_t>(bits >> 32);
    }
    if (!pos) a.box_hi[0] = a.box_hi[2] = INT32_MAX;
    const double dv[8] = {a.xmin, a.xmax, a.ymin, a.ymax, a.box[0], a.box[1], a.box[2], a.box[3]};
    for (int k = 0; k < 8; ++k) a.f_dom[k] = static_cast<float>(dv[k]);
    // fp32 walks: positive floats order like their bit patterns, so the box
    // test is four integer compares, and exact (same condition as for box_hi)
    for (int k = 0; k < 4; ++k) std::memcpy(&a.box_fi[k], &a.f_dom[4 + k], 4);
    if (!pos || !(a.f_dom[4] > 0.0f && a.f_dom[6] > 0.0f)) a.box_fi[0] = a.box_fi[2] = INT32_MAX;
    a.f_dt = static_cast<float>(a.dt);
    a.f_sqrt2dt = static_cast<float>(a.sqrt2dt);
    a.f_thr = static_cast<float>(a.bridge_thr);
    a.f_kd = d.kind == SDDG_DENS_RING_W    ? static_cast<float>(-8000.0 * a.dt)
             : d.kind == SDDG_DENS_SHOCK_W ? static_cast<float>(1.0 / (-160.0 * a.dt))
                                           : static_cast<float>(-3000.0 * a.dt);
    a.seed = cfg.seed;
    a.rk = make_round_keys(cfg.seed);
    a.max_steps32 = static_cast<uint32_t>(cfg.max_steps);  // <= 2^29 (validate_walk)
}

// ------------------------------------------------------------ cost model

double ExitTimeModel::at(double x, double y) const {
    double sx = (x - x0) / hx, sy = (y - y0) / hy;
    sx = std::min(std::max(sx, 0.0), static_cast<double>(g - 1));
    sy = std::min(std::max(sy, 0.0), static_cast<double>(g - 1));
    const int i = std::min(static_cast<int>(sx), g - 2), j = std::min(static_cast<int>(sy), g - 2);
    const double u = sx - i, v = sy - j;
    const double* r0 = t.data() + static_cast<size_t>(j) * g + i;
    const double* r1 = r0 + g;
    return (1 - v) * ((1 - u) * r0[0] + u * r0[1]) + v * ((1 - u) * r1[0] + u * r1[1]);
}

// div(w grad T) = -w on a 65 x 65 grid over the domain, T = 0 on the edges:
// the conservative five-point operator of solve_dirichlet (detsolver.cpp:88-111)
// with a source, red-black SOR at the grid's optimal factor until the update
// is below 1e-7 of max T (a few ms of host time, once per density/domain).
const ExitTimeModel& exit_time_model(sddg_ctx* c, const sddg_density& d, const sddg_domain& dom) {
    char key[256];
    std::snprintf(key, sizeof(key), "%d %a %a %a %a %a %a", d.kind, d.R, d.alpha, dom.xmin, dom.xmax,
                  dom.ymin, dom.ymax);
    auto it = c->cost_models.find(key);
    if (it != c->cost_models.end()) return it->second;
    ExitTimeModel m;
    const int g = 65;
    m.g = g;
    m.x0 = dom.xmin;
    m.y0 = dom.ymin;
    m.hx = (dom.xmax - dom.xmin) / (g - 1);
    m.hy = (dom.ymax - dom.ymin) / (g - 1);
    const HostDensity h = host_density(d);
    std::vector<double> w(static_cast<size_t>(g) * g);
    for (int j = 0; j < g; ++j)
        for (int i = 0; i < g; ++i) {
            double r = 1.0;
            try {
                r = h.rho(m.x0 + i * m.hx, m.y0 + j * m.hy);
            } catch (const std::exception&) {
            }
            w[static_cast<size_t>(j) * g + i] = (std::isfinite(r) && r > 0.0) ? 1.0 / r : 1.0;
        }
    const double ihx2 = 1.0 / (m.hx * m.hx), ihy2 = 1.0 / (m.hy * m.hy);
    m.t.assign(static_cast<size_t>(g) * g, 0.0);
    const double omega = 2.0 / (1.0 + std::sin(3.14159265358979323846 / (g - 1)));
    for (int sweep = 0; sweep < 4000; ++sweep) {
        double upd = 0.0, tmax = 0.0;
        for (int colour = 0; colour < 2; ++colour)
            for (int j = 1; j < g - 1; ++j)
                for (int i = 1 + ((j + colour) & 1); i < g - 1; i += 2) {
                    const size_t k = static_cast<size_t>(j) * g + i;
                    const double ce = 0.5 * (w[k] + w[k + 1]) * ihx2, cw = 0.5 * (w[k] + w[k - 1]) * ihx2;
                    const double cn = 0.5 * (w[k] + w[k + g]) * ihy2, cs = 0.5 * (w[k] + w[k - g]) * ihy2;
                    const double gs = (ce * m.t[k + 1] + cw * m.t[k - 1] + cn * m.t[k + g] + cs * m.t[k - g] +
                                       w[k]) / (ce + cw + cn + cs);
                    const double nv = m.t[k] + omega * (gs - m.t[k]);
                    upd = std::max(upd, std::fabs(nv - m.t[k]));
                    tmax = std::max(tmax, nv);
                    m.t[k] = nv;
                }
        if (upd <= 1e-7 * tmax) break;
    }
    return c->cost_models.emplace(key, std::move(m)).first->second;
}

std::vector<double> node_costs(const ExitTimeModel& m, const sddg_walk_config& cfg, const double* px,
                               const double* py, int64_t n) {
    // mean step: dt (linear) or 1/lambda (exponential, dt ~ Exp(lambda))
    const double per = cfg.scheme == SDDG_SCHEME_LINEAR ? 1.0 / cfg.dt : cfg.lambda;
    const double walks = static_cast<double>(cfg.walks);
    std::vector<double> out(n);
    for (int64_t k = 0; k < n; ++k) out[k] = walks * (1.0 + std::max(0.0, m.at(px[k], py[k])) * per);
    return out;
}

// Longest-expected-walk-first launch order (LPT): the batch tail is then made
// of short walks.
std::vector<uint32_t> cost_order(const std::vector<double>& cost, const std::vector<uint32_t>* subset) {
    std::vector<uint32_t> perm;
    if (subset) {
        perm = *subset;
    } else {
        perm.resize(cost.size());
        for (size_t k = 0; k < cost.size(); ++k) perm[k] = static_cast<uint32_t>(k);
    }
    const char* ord = std::getenv("SDDG_NODE_ORDER");  // A/B knob: "reverse" (shortest first), "index"
    if (ord && std::strcmp(ord, "index") == 0) return perm;
    const bool rev = ord && std::strcmp(ord, "reverse") == 0;
    std::stable_sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) {
        if (rev) return cost[a] < cost[b] || (cost[a] == cost[b] && a < b);
        return cost[a] > cost[b] || (cost[a] == cost[b] && a < b);
    });
    return perm;
}

// A tabulated density's padded samples in device memory (empty view for the
// formula kinds).
TableDensity upload_density(sddg_ctx* c, const sddg_density& d) {
    TableDensity t;
    if (d.kind != SDDG_DENS_TABLE) return t;
    const HostDensity h = host_density(d);
    const size_t bytes = sizeof(double) * h.padded->size();
    double* p = static_cast<double*>(c->dens_tab.ensure(bytes));
    ck(cudaMemcpy(p, h.padded->data(), bytes, cudaMemcpyHostToDevice), "h2d density table");
    t = h.td;
    t.t = p;
    return t;
}

double* upload_tables(sddg_ctx* c, const sddg_boundary& bd) {
    const size_t nx = bd.nx, ny = bd.ny;
    std::vector<double> h(4 * (nx + ny));
    const size_t lens[4] = {nx, nx, ny, ny};
    size_t o = 0;
    for (int fg = 0; fg < 2; ++fg)
        for (int k = 0; k < 4; ++k) {
            const double* src = fg == 0 ? bd.f[k] : bd.g[k];
            std::memcpy(h.data() + o, src, sizeof(double) * lens[k]);
            o += lens[k];
        }
    double* d = static_cast<double*>(c->tables.ensure(sizeof(double) * h.size()));
    ck(cudaMemcpyAsync(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c->stream),
       "upload tables");
    ck(cudaStreamSynchronize(c->stream), "sync");
    return d;
}

void raise_kernel_error(const Counters& hc) {
    if (hc.err_flag == 3)
        fail(SDDG_ERR_EVALUATION,
             "drift not finite (point_id " + std::to_string(hc.err_info) + ")");
    if (hc.err_flag == 4)
        fail(SDDG_ERR_NUMERICAL, "mc_estimate: walk failed to exit after 1024 restarts (point_id " +
                                     std::to_string(hc.err_info) + ")");
    if (hc.err_flag == 5)
        fail(SDDG_ERR_CUDA, "walk kernel: dynamic shared memory at offset " +
                                std::to_string(hc.err_info) + ", not the compiled SDDG_SMEM_ABS");
}

// The batch tail for fp64 walks (batches of at most kTailWalksPerLane walks
// per K1 lane; larger batches, whose tail is a small share, keep the plain K1
// loop: 1.5 instructions per step fewer).  Once K1's batch counter has run
// out, its lanes empty out while the longest walks run on: warps keep issuing
// every step for a few live lanes.  So at check points (every chunk32 steps)
// the walks still running move on, in stages:
//  * drain rounds: K1 resumed on the previous stage's handoffs, packed 32 per
//    warp and spread over the SMs (SDDG_DRAIN: the per-SM caps, decreasing;
//    default "256": K1 hands over once <= 256 walks per SM are in flight; a
//    list "256,64" adds a round that repacks again at 64, ...; "" none).
//    Config 1: 18.6 -> 16.6 ms (tools/tail_ab.py; a second round or an earlier
//    first one measured no better);
//  * the tail kernel (walk_tail.cuh), one warp per walk, for the last
//    SDDG_TAIL_PER_SM (16) walks per SM.
// Every stage runs the same step functions on the same draws, so results do
// not depend on where a walk finished.  SDDG_NO_TAIL=1: K1 alone.
// The handoff check points cost the step loop ~1.8% of its warp instructions, so the
// stages pay only while the tail is a large enough share: config 2 at 50 / 75 / 100 walks
// per lane: +1.0% / 0 / -1.1% against the plain kernel (SDDG_TAIL_WALKS_PER_LANE, A/B)
constexpr uint64_t kTailWalksPerLane = 72;

DrainPlan enable_tail(sddg_ctx* c, WalkArgs& a, int precision, Counters* cnt, uint64_t lanes) {
    DrainPlan dp;
    a.cont = nullptr;
    a.cont_cap = 0;
    a.src = nullptr;
    a.n_src = nullptr;
    a.src_cap = 0;
    a.chunk32 = a.max_steps32;
    if (precision != SDDG_FP64 || std::getenv("SDDG_NO_TAIL")) return dp;
    const char* wpl = std::getenv("SDDG_TAIL_WALKS_PER_LANE");  // A/B knob
    const uint64_t max_wpl = wpl ? std::strtoull(wpl, nullptr, 10) : kTailWalksPerLane;
    if (a.total > max_wpl * lanes) return dp;
    // K1's check points every chunk32 steps: the largest of 256, 128, 64
    // dividing max_steps (the restart must still fall on a chunk end)
    uint32_t chunk = 256;
    while (chunk >= 64 && a.max_steps32 % chunk != 0) chunk /= 2;
    if (chunk < 64 || chunk >= a.max_steps32) return dp;
    a.chunk32 = chunk;
    const uint32_t sms = static_cast<uint32_t>(c->sms);
    const char* per_sm = std::getenv("SDDG_TAIL_PER_SM");  // A/B knob: walks handed to K1t per SM
    const uint32_t tail_sm = per_sm ? static_cast<uint32_t>(std::max(1, std::atoi(per_sm))) : 16u;
    std::vector<uint32_t> caps;  // per SM, decreasing, above the tail's
    const char* drain = std::getenv("SDDG_DRAIN");
    std::string spec = drain ? drain : "256";
    for (size_t p = 0; p < spec.size();) {
        const size_t q = std::min(spec.find(',', p), spec.size());
        const long v = std::strtol(spec.substr(p, q - p).c_str(), nullptr, 10);
        if (v > static_cast<long>(tail_sm) && (caps.empty() || static_cast<uint32_t>(v) < caps.back()) &&
            static_cast<uint64_t>(v) * sms < lanes && caps.size() < static_cast<size_t>(kMaxDrain))
            caps.push_back(static_cast<uint32_t>(v));
        p = q + 1;
    }
    caps.push_back(tail_sm);
    dp.rounds = static_cast<int>(caps.size()) - 1;
    size_t total = 0;
    for (uint32_t v : caps) total += static_cast<size_t>(v) * sms;
    WalkCont* buf = static_cast<WalkCont*>(c->tail_cont.ensure(sizeof(WalkCont) * total));
    for (size_t r = 0; r < caps.size(); ++r) {
        dp.cap[r] = caps[r] * sms;
        dp.buf[r] = buf;
        buf += dp.cap[r];
    }
    a.cont = dp.buf[0];
    a.cont_cap = dp.cap[0];
    a.n_cont = &cnt->n_cont;
    a.live = &cnt->live;
    return dp;
}

// K1 on a batch set up by set_next_kernel, then its drain rounds and the tail
// kernel; `after_k1` (optional) is recorded between K1 and the rest.  Returns
// the kernels launched.
int launch_walk_stages(sddg_ctx* c, int dv, int precision, const WalkArgs& a, const DrainPlan& dp, int grid,
                       Counters* cnt, cudaStream_t st, cudaEvent_t after_k1) {
    ck(launch_walk(dv, precision, a, grid, st), "walk kernel launch");
    if (!a.cont) return 1;
    if (after_k1) ck(cudaEventRecord(after_k1, st), "event");
    int launches = 1;
    WalkArgs b = a;
    const unsigned int* n_prev = &cnt->n_cont;
    for (int r = 1; r <= dp.rounds; ++r) {
        b.src = dp.buf[r - 1];
        b.n_src = n_prev;
        b.src_cap = dp.cap[r - 1];
        b.cont = dp.buf[r];
        b.cont_cap = dp.cap[r];
        b.n_cont = &cnt->n_drain[r - 1];
        drain_prep_kernel<<<1, 1, 0, st>>>(cnt, b.n_src, b.src_cap);
        ck(cudaGetLastError(), "drain prep");
        // one CTA per SM holding its share of the handoffs, 32 walks per warp
        const uint32_t per_sm = (b.src_cap + c->sms - 1) / c->sms;
        const int block = static_cast<int>(std::min<uint32_t>((per_sm + 31) / 32 * 32, static_cast<uint32_t>(kDrainBlock)));
        const int g = static_cast<int>((b.src_cap + block - 1) / block);
        ck(launch_walk(dv, precision, b, g, st, block), "drain round launch");
        n_prev = b.n_cont;
        launches += 2;
    }
    b.src = nullptr;
    b.n_src = nullptr;
    b.src_cap = 0;
    b.cont = dp.buf[dp.rounds];
    b.cont_cap = dp.cap[dp.rounds];
    b.n_cont = const_cast<unsigned int*>(n_prev);
    ck(launch_walk_tail(dv, b, st), "tail kernel launch");
    return launches + 1;
}

// Walks + finalize for n device-resident nodes; estimates to d_out.
void run_estimates(sddg_ctx* c, const sddg_density& d, const sddg_domain& dom,
                   const sddg_boundary& bd, const sddg_walk_config& cfg, const double* d_px,
                   const double* d_py, const uint64_t* d_pid, int64_t n_all,
                   const std::vector<uint32_t>& perm, sddg_estimate* d_out, cudaStream_t st,
                   const GatherTargets* gt) {
    GatherTargets none;
    none.n_peers = 0;
    none.global_index = nullptr;
    const int dv = walk_variant(d, cfg);
    const int64_t n = static_cast<int64_t>(perm.size());
    c->last_ms = 0.0;
    c->last_steps = 0;
    c->last_launches = 0;
    if (n == 0) return;
    const double* dtab = upload_tables(c, bd);
    uint32_t* dperm = static_cast<uint32_t*>(c->perm.ensure(sizeof(uint32_t) * n));
    ck(cudaMemcpyAsync(dperm, perm.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st),
       "h2d perm");
    Counters* cnt = static_cast<Counters*>(c->counters.ensure(sizeof(Counters)));
    ck(cudaMemsetAsync(cnt, 0, sizeof(Counters), st), "memset counters");
    unsigned long long* nst =
        static_cast<unsigned long long*>(c->nsteps.ensure(sizeof(unsigned long long) * n_all));
    ck(cudaMemsetAsync(nst, 0, sizeof(unsigned long long) * n_all, st), "memset node steps");
    const int64_t W = cfg.walks;
    const int64_t npb = std::max<int64_t>(1, batch_budget_walks() / W);
    const int64_t cap = std::min(npb, n) * W;
    double* rf = static_cast<double*>(c->rec_f.ensure(sizeof(double) * cap));
    double* rg = static_cast<double*>(c->rec_g.ensure(sizeof(double) * cap));
    uint32_t* rm = static_cast<uint32_t*>(c->rec_meta.ensure(sizeof(uint32_t) * cap));
    WalkArgs a;
    fill_args(a, d, dom, bd, cfg, dtab);
    a.tab = upload_density(c, d);
    a.fm_tables = c->fm_tables.p;
    a.walks = W;
    a.walk_lo = 0;
    a.n_nodes = n_all;
    a.next = &cnt->next;
    a.steps = &cnt->steps;
    a.node_steps = nst;
    a.err_flag = &cnt->err_flag;
    a.err_info = &cnt->err_info;
    a.rec_f = rf;
    a.rec_g = rg;
    a.rec_meta = rm;
    int64_t launches = 0;
    const size_t nbatch = static_cast<size_t>((n + npb - 1) / npb);
    while (c->bev.size() < 3 * nbatch) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "event");
        c->bev.push_back(e);
    }
    size_t bi = 0;
    for (int64_t b = 0; b < n; b += npb, ++bi) {
        const int64_t nb = std::min(npb, n - b);
        a.px = d_px;
        a.py = d_py;
        a.pid = d_pid;
        a.perm = dperm + b;
        a.total = static_cast<uint64_t>(nb) * W;
        const auto [grid, blk] = walk_grid(c, dv, cfg.precision, a.total);
        const unsigned long long lanes = static_cast<unsigned long long>(grid) * blk;
        const DrainPlan dp = enable_tail(c, a, cfg.precision, cnt, lanes);
        set_next_kernel<<<1, 1, 0, st>>>(cnt, lanes, std::min<unsigned long long>(lanes, a.total));
        ck(cudaGetLastError(), "set_next");
        ck(cudaEventRecord(c->bev[3 * bi], st), "event");
        launches += launch_walk_stages(c, dv, cfg.precision, a, dp, grid, cnt, st, c->bev[3 * bi + 1]);
        if (!a.cont) ck(cudaEventRecord(c->bev[3 * bi + 1], st), "event");
        ck(cudaEventRecord(c->bev[3 * bi + 2], st), "event");
        ck(launch_reduce(rf, rg, rm, W, nb, dperm + b, nst, d_out, st, gt ? *gt : none), "reduce launch");
        launches += 2;
    }
    Counters hc;
    ck(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, st), "read counters");
    ck(cudaStreamSynchronize(st), "walk kernels");
    double tot_ms = 0.0, tail_ms = 0.0;
    for (size_t k = 0; k < nbatch; ++k) {
        float ms = 0.f, ms_t = 0.f;
        cudaEventElapsedTime(&ms, c->bev[3 * k], c->bev[3 * k + 2]);
        cudaEventElapsedTime(&ms_t, c->bev[3 * k + 1], c->bev[3 * k + 2]);
        tot_ms += ms;
        tail_ms += ms_t;
    }
    c->last_ms = tot_ms;
    c->last_tail_ms = a.cont ? tail_ms : 0.0;
    c->last_handoffs = a.cont ? std::min<int64_t>(hc.n_cont, a.cont_cap) : 0;
    c->last_steps = static_cast<int64_t>(hc.steps);
    c->last_launches = launches;
    raise_kernel_error(hc);
}

void check_points(const sddg_domain& dom, const double* px, const double* py, int64_t n) {
    for (int64_t k = 0; k < n; ++k)
        if (!(px[k] > dom.xmin && px[k] < dom.xmax && py[k] > dom.ymin && py[k] < dom.ymax))
            fail(SDDG_ERR_OUT_OF_DOMAIN, "mc_estimate: start point must be strictly inside");
}

void estimates_host(sddg_ctx* c, const sddg_density& d, const sddg_domain& dom,
                    const sddg_boundary& bd, const sddg_walk_config& cfg, const double* px,
                    const double* py, const uint64_t* pid, int64_t n, sddg_estimate* out,
                    const GatherTargets* gt = nullptr) {
    validate_walk(cfg);
    check_domain(dom);
    check_boundary(bd);
    walk_variant(d, cfg);
    check_positivity(d, dom);
    check_points(dom, px, py, n);
    if (n <= 0) return;
    char* buf = static_cast<char*>(c->nodes.ensure(n * (2 * sizeof(double) + sizeof(uint64_t))));
    double* dpx = reinterpret_cast<double*>(buf);
    double* dpy = dpx + n;
    uint64_t* dpid = reinterpret_cast<uint64_t*>(dpy + n);
    ck(cudaMemcpyAsync(dpx, px, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream), "h2d");
    ck(cudaMemcpyAsync(dpy, py, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream), "h2d");
    ck(cudaMemcpyAsync(dpid, pid, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, c->stream), "h2d");
    sddg_estimate* dout = static_cast<sddg_estimate*>(c->est.ensure(sizeof(sddg_estimate) * n));
    if (team_active(c) && !gt) {
        team_estimates(c, d, dom, bd, cfg, dpx, dpy, dpid, n, dout, c->stream, px, py);
    } else {
        const std::vector<uint32_t> order =
            cost_order(node_costs(exit_time_model(c, d, dom), cfg, px, py, n), nullptr);
        run_estimates(c, d, dom, bd, cfg, dpx, dpy, dpid, n, order, dout, c->stream, gt);
    }
    ck(cudaMemcpyAsync(out, dout, sizeof(sddg_estimate) * n, cudaMemcpyDeviceToHost, c->stream),
       "d2h");
    ck(cudaStreamSynchronize(c->stream), "d2h sync");
}

// ------------------------------------------------------------ K3

void solve_batch_host(sddg_ctx* c, const double* w, int gnx, int gny, double hx, double hy,
                      int64_t n, const sddg_subdomain* subs, const double* bc,
                      const sddg_solver_config& sc, double* u, sddg_solve_info* info) {
    if (!(sc.tol > 0.0)) fail(SDDG_ERR_VALIDATION, "SolverConfig: tol must be > 0");
    if (sc.max_iters < 0) fail(SDDG_ERR_VALIDATION, "SolverConfig: max_iters must be >= 0");
    if (sc.method != SDDG_SOLVER_JACOBI && sc.method != SDDG_SOLVER_RBSOR)
        fail(SDDG_ERR_VALIDATION, "SolverConfig: unknown method");
    if (n <= 0) return;
    for (int64_t k = 0; k < static_cast<int64_t>(gnx) * gny; ++k)
        if (!std::isfinite(w[k]) || w[k] <= 0.0)
            fail(SDDG_ERR_EVALUATION, "solve_dirichlet: non-positive diffusion weight");
    std::vector<SolveJob> jobs(n);
    int64_t boff = 0, uoff = 0;
    int max_n = 0, max_int = 0, max_dim = 0;
    for (int64_t s = 0; s < n; ++s) {
        const sddg_subdomain& q = subs[s];
        if (q.nx < 3 || q.ny < 3) fail(SDDG_ERR_VALIDATION, "solve_dirichlet: grid too small");
        if (q.i0 < 0 || q.j0 < 0 || q.i0 + q.nx > gnx || q.j0 + q.ny > gny)
            fail(SDDG_ERR_VALIDATION, "solve_dirichlet: subdomain outside the weight grid");
        const double* B = bc + boff;
        const double* T = B + q.nx;
        const double* L = T + q.nx;
        const double* R = L + q.ny;
        auto mismatch = [](double a, double b) {
            return std::abs(a - b) > 1e-12 * (1.0 + std::abs(a) + std::abs(b));
        };
        if (mismatch(B[0], L[0]) || mismatch(B[q.nx - 1], R[0]) || mismatch(T[0], L[q.ny - 1]) ||
            mismatch(T[q.nx - 1], R[q.ny - 1]))
            fail(SDDG_ERR_VALIDATION, "solve_dirichlet: boundary data disagrees at a corner");
        jobs[s] = SolveJob{q.i0, q.j0, q.nx, q.ny, boff, uoff};
        boff += 2 * (q.nx + q.ny);
        uoff += static_cast<int64_t>(q.nx) * q.ny;
        max_n = std::max(max_n, q.nx * q.ny);
        max_int = std::max(max_int, (q.nx - 2) * (q.ny - 2));
        max_dim = std::max(max_dim, std::max(q.nx, q.ny));
    }
    // jobs whose solution fits in shared memory go to the batched K3; larger
    // ones (e.g. the single-domain 513^2 comparison of config 4) to K3b
    const size_t smem_cap = 227 * 1024;
    const bool force_large = std::getenv("SDDG_FORCE_LARGE_SOLVER") != nullptr;
    std::vector<SolveJob> small, large;
    int max_n_s = 0, max_int_s = 0, max_dim_s = 0, max_dim_all = 0;
    int64_t max_n_l = 0;
    for (int64_t q = 0; q < n; ++q) {
        const SolveJob& j = jobs[q];
        const int nn = j.nx * j.ny;
        max_dim_all = std::max(max_dim_all, std::max(j.nx, j.ny));
        if (!force_large && sizeof(double) * static_cast<size_t>(nn) <= smem_cap) {
            small.push_back(j);
            max_n_s = std::max(max_n_s, nn);
            max_int_s = std::max(max_int_s, (j.nx - 2) * (j.ny - 2));
            max_dim_s = std::max(max_dim_s, std::max(j.nx, j.ny));
        } else {
            large.push_back(j);
            max_n_l = std::max<int64_t>(max_n_l, nn);
        }
    }
    (void)max_n;
    (void)max_int;
    (void)max_dim;
    const int ncoef = sc.method == SDDG_SOLVER_RBSOR ? 4 : 3;  // solver.cu launch_solve_batch
    const bool coef_smem = sizeof(double) * ((1 + ncoef) * static_cast<size_t>(max_n_s) + 1) <= smem_cap;
    const bool jacobi_small_ok = max_int_s <= solver_max_points();
    if (sc.method == SDDG_SOLVER_JACOBI && !jacobi_small_ok) {
        // Jacobi register budget exceeded: route those jobs to K3b as well
        std::vector<SolveJob> keep;
        for (const SolveJob& j : small) {
            if ((j.nx - 2) * (j.ny - 2) > solver_max_points()) {
                large.push_back(j);
                max_n_l = std::max<int64_t>(max_n_l, static_cast<int64_t>(j.nx) * j.ny);
            } else {
                keep.push_back(j);
            }
        }
        small.swap(keep);
        max_n_s = max_int_s = 0;
        for (const SolveJob& j : small) {
            max_n_s = std::max(max_n_s, j.nx * j.ny);
            max_int_s = std::max(max_int_s, (j.nx - 2) * (j.ny - 2));
        }
    }
    // SOR factor: sc.omega > 0 as given; 0 (default) per job from the job's
    // weights (launch_sor_omega); < 0 the constant-coefficient grid formula
    double omega = sc.omega;
    const bool omega_per_job = sc.method == SDDG_SOLVER_RBSOR && omega == 0.0;
    if (sc.method == SDDG_SOLVER_RBSOR && !(omega > 0.0)) {
        const double kPi = 3.14159265358979323846;
        omega = 2.0 / (1.0 + std::sin(kPi / (max_dim_all - 1)));
    }
    if (sc.method == SDDG_SOLVER_JACOBI) omega = 1.0;
    const size_t wbytes = sizeof(double) * static_cast<size_t>(gnx) * gny;
    double* dw = static_cast<double*>(c->s_w.ensure(wbytes));
    // device job list: small jobs (K3/K3c) then large jobs (K3b), and one SOR factor per job
    const size_t n_all = small.size() + large.size();
    SolveJob* dj = static_cast<SolveJob*>(c->s_jobs.ensure(sizeof(SolveJob) * std::max<size_t>(1, n_all)));
    double* domg = static_cast<double*>(c->s_omega.ensure(sizeof(double) * std::max<size_t>(1, n_all)));
    int* dperm = static_cast<int*>(c->s_perm.ensure(sizeof(int) * std::max<size_t>(1, small.size())));
    double* dbc = static_cast<double*>(c->s_bc.ensure(sizeof(double) * boff));
    double* du = static_cast<double*>(c->s_u.ensure(sizeof(double) * uoff));
    sddg_solve_info* dinfo = static_cast<sddg_solve_info*>(c->s_info.ensure(sizeof(sddg_solve_info) * n));
    int* derr = static_cast<int*>(c->s_err.ensure(sizeof(int)));
    // RB-SOR jobs too large for one CTA's shared memory (with their weights)
    // go to the thread-block-cluster kernel K3c when they all share one shape
    // and the batch is latency-bound (at most one job per SM: the slowest
    // job sets the time, and K3c runs each job on CL SMs from shared memory;
    // A/B config 3, 128 x 129^2: 15.5 -> 7.8 ms).  Larger batches are
    // throughput-bound, where one CTA per job wins (2048 x 129^2: 47 vs 65 ms).
    int cluster = 0;
    if (sc.method == SDDG_SOLVER_RBSOR && !small.empty() && !coef_smem &&
        static_cast<int64_t>(small.size()) <= std::max(1, c->sms)) {
        bool same = true;
        for (const SolveJob& j : small) same = same && j.nx == small[0].nx && j.ny == small[0].ny;
        if (same) cluster = solver_cluster_size(small[0].nx, small[0].ny);
    }
    double* dcoef = nullptr;
    if (!small.empty() && !coef_smem && !cluster)
        dcoef = static_cast<double*>(c->s_coef.ensure(sizeof(double) * ncoef * max_n_s * small.size()));
    double* dlarge = nullptr;
    if (!large.empty())
        dlarge = static_cast<double*>(c->s_large.ensure(sizeof(double) * (5 * max_n_l + 8)));
    cudaStream_t st = c->stream;
    ck(cudaMemcpyAsync(dw, w, wbytes, cudaMemcpyHostToDevice, st), "h2d w");
    ck(cudaMemcpyAsync(dbc, bc, sizeof(double) * boff, cudaMemcpyHostToDevice, st), "h2d bc");
    ck(cudaMemsetAsync(derr, 0, sizeof(int), st), "memset");
    // info slots: small jobs first in job order, then large jobs
    std::vector<int64_t> info_of(n);
    {
        int64_t a = 0;
        std::map<int64_t, int64_t> pos_of_uoff;
        for (int64_t q = 0; q < n; ++q) pos_of_uoff[jobs[q].u_off] = q;
        for (const SolveJob& j : small) info_of[a++] = pos_of_uoff[j.u_off];
        for (const SolveJob& j : large) info_of[a++] = pos_of_uoff[j.u_off];
    }
    std::vector<SolveJob> all_jobs(small);
    all_jobs.insert(all_jobs.end(), large.begin(), large.end());
    std::vector<double> homg(n_all, omega);
    ck(cudaEventRecord(c->ev0, st), "event");
    int launches = 0;
    if (n_all) {
        ck(cudaMemcpyAsync(dj, all_jobs.data(), sizeof(SolveJob) * n_all, cudaMemcpyHostToDevice, st),
           "h2d jobs");
        if (omega_per_job) {
            ck(launch_sor_omega(dw, gnx, hx, hy, static_cast<int64_t>(n_all), dj, domg, st), "omega launch");
            ++launches;
            // K3 blocks in descending factor order, so the slowest solves start
            // in the first waves (2048 x 129^2: 41.5 -> 39.9 ms).  Not for K3c:
            // on the config-3 batch the order measured slower (4.9-5.2 -> 5.7 ms)
            if (!small.empty() && !cluster && !std::getenv("SDDG_NO_JOB_ORDER")) {
                ck(launch_order_jobs(domg, static_cast<int64_t>(small.size()), dperm, st), "order launch");
                ++launches;
            } else {
                dperm = nullptr;
            }
        } else {
            ck(cudaMemcpyAsync(domg, homg.data(), sizeof(double) * n_all, cudaMemcpyHostToDevice, st),
               "h2d omega");
            dperm = nullptr;
        }
    }
    if (!small.empty()) {
        if (cluster)
            ck(launch_solve_cluster(dw, gnx, hx, hy, static_cast<int64_t>(small.size()), dj, dbc, sc.tol,
                                    sc.max_iters, sc.init_blend, domg, dperm, du, dinfo, derr, st, small[0].nx,
                                    small[0].ny, cluster),
               "cluster solver launch");
        else
            ck(launch_solve_batch(dw, gnx, hx, hy, static_cast<int64_t>(small.size()), dj, dbc, sc.tol,
                                  sc.max_iters, sc.init_blend, sc.method, domg, dperm, du, dinfo, derr, st,
                                  max_n_s, max_int_s, dcoef, coef_smem ? 1 : 0),
               "solver launch");
        ++launches;
    }
    for (size_t q = 0; q < large.size(); ++q) {
        ck(launch_solve_large(dw, gnx, hx, hy, large[q], dbc, sc.tol, sc.max_iters, sc.init_blend,
                              sc.method, domg + small.size() + q, du, dinfo + small.size() + q, derr, dlarge, st, c->sms),
           "large solver launch");
        ++launches;
    }
    ck(cudaEventRecord(c->ev1, st), "event");
    int herr = 0;
    std::vector<sddg_solve_info> hinfo(n);
    ck(cudaMemcpyAsync(u, du, sizeof(double) * uoff, cudaMemcpyDeviceToHost, st), "d2h u");
    ck(cudaMemcpyAsync(hinfo.data(), dinfo, sizeof(sddg_solve_info) * n, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h err");
    ck(cudaStreamSynchronize(st), "solver");
    for (int64_t a = 0; a < n; ++a) info[info_of[a]] = hinfo[a];
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    c->last_ms = ms;
    c->last_launches = launches;
    c->last_steps = 0;
    if (herr == 4) fail(SDDG_ERR_NUMERICAL, "solve_dirichlet: maximum principle violated");
}

// ------------------------------------------------------------ decomposition

struct Line {
    bool vertical;
    int fixed;
    int length;
};

struct Layout {
    int nx, ny, sx, sy, bx, by;
    sddg_domain dom;
    std::vector<Line> lines;
    double hx() const { return (dom.xmax - dom.xmin) / (nx - 1); }
    double hy() const { return (dom.ymax - dom.ymin) / (ny - 1); }
};

// build_layout (proj/src/decomposition.cpp:26-53)
Layout build_layout(const sddg_domain& dom, int nx, int ny, int sx, int sy) {
    check_domain(dom);
    if (nx < 3 || ny < 3) fail(SDDG_ERR_VALIDATION, "GridSpec: needs nx >= 3 and ny >= 3");
    if (sx < 1 || sy < 1) fail(SDDG_ERR_LAYOUT, "build_layout: subdomain counts must be >= 1");
    if ((nx - 1) % sx != 0)
        fail(SDDG_ERR_LAYOUT, "build_layout: nx-1=" + std::to_string(nx - 1) +
                                  " not divisible by " + std::to_string(sx) + " (x axis)");
    if ((ny - 1) % sy != 0)
        fail(SDDG_ERR_LAYOUT, "build_layout: ny-1=" + std::to_string(ny - 1) +
                                  " not divisible by " + std::to_string(sy) + " (y axis)");
    Layout L{nx, ny, sx, sy, (nx - 1) / sx, (ny - 1) / sy, dom, {}};
    if (L.bx < 2 || L.by < 2)
        fail(SDDG_ERR_LAYOUT, "build_layout: subdomains need at least 3 nodes per axis");
    for (int a = 1; a < sx; ++a) L.lines.push_back({true, a * L.bx, ny});
    for (int b = 1; b < sy; ++b) L.lines.push_back({false, b * L.by, nx});
    return L;
}

// Interior samples that are strict local peaks or dips of a series, skipping
// those smaller than 1e-9 of its largest magnitude (the reference's guard
// against roundoff wiggles in flat stretches, decomposition.cpp:65-79)
void flag_extrema(const std::vector<double>& series, std::vector<char>& flag) {
    double top = 0.0;
    for (size_t i = 0; i < series.size(); ++i) top = std::max(top, std::fabs(series[i]));
    const double guard = 1e-9 * top;
    for (size_t i = 1; i + 1 < series.size(); ++i) {
        const double before = series[i - 1], here = series[i], after = series[i + 1];
        if (std::fabs(here) < guard) continue;
        const bool peak = here > before && here > after;
        const bool dip = here < before && here < after;
        if (peak || dip) flag[i] = 1;
    }
}

// plan_interface_points (proj/src/decomposition.cpp:81-145)
std::vector<std::vector<int>> plan(const sddg_density& d, const Layout& L, int strategy, int k) {
    std::vector<std::vector<int>> out;
    const HostDensity h = host_density(d);
    for (const Line& line : L.lines) {
        const int n = line.length;
        std::vector<int> nodes;
        if (strategy == SDDG_PLACE_ALL) {
            for (int p = 1; p + 1 < n; ++p) nodes.push_back(p);
        } else if (strategy == SDDG_PLACE_EQUISPACED) {
            if (k < 1 || k > n - 2)
                fail(SDDG_ERR_VALIDATION, "plan_interface_points: equispaced count " +
                                              std::to_string(k) + " not in [1, " +
                                              std::to_string(n - 2) + "]");
            for (int j = 1; j <= k; ++j) {
                const int pos = static_cast<int>(std::lround(static_cast<double>(j) * (n - 1) / (k + 1)));
                nodes.push_back(std::clamp(pos, 1, n - 2));
            }
            nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
        } else if (strategy == SDDG_PLACE_OPTIMAL) {
            // the feature rule (decomposition.cpp:82-108): nodes where rho' along
            // the line (analytic) or rho'' (central difference of rho') has a
            // strict extremum, at least two nodes apart; the middle node if none
            const double spacing = line.vertical ? L.hy() : L.hx();
            std::vector<double> slope(n), curv(n, 0.0);
            for (int p = 0; p < n; ++p) {
                const int i = line.vertical ? line.fixed : p, j = line.vertical ? p : line.fixed;
                double gx, gy;
                h.grad(L.dom.xmin + i * L.hx(), L.dom.ymin + j * L.hy(), gx, gy);
                slope[p] = line.vertical ? gy : gx;
            }
            for (int p = 1; p + 1 < n; ++p) curv[p] = (slope[p + 1] - slope[p - 1]) / (2.0 * spacing);
            std::vector<char> feature(n, 0);
            flag_extrema(slope, feature);
            flag_extrema(curv, feature);
            for (int p = 1; p + 1 < n; ++p)
                if (feature[p] && (nodes.empty() || p - nodes.back() >= 2)) nodes.push_back(p);
            if (nodes.empty()) nodes.push_back(n / 2);
        } else if (strategy == SDDG_PLACE_EQUIDISTRIBUTED) {
            // BASELINE config 4: grid nodes nearest to equal shares
            // of the trapezoid integral of w = 1/rho along the line
            if (k < 1 || k > n - 2)
                fail(SDDG_ERR_VALIDATION, "plan_interface_points: equidistributed count " +
                                              std::to_string(k) + " not in [1, " +
                                              std::to_string(n - 2) + "]");
            std::vector<double> cum(n, 0.0);
            double wprev = 0.0;
            for (int p = 0; p < n; ++p) {
                const double x = line.vertical ? L.dom.xmin + line.fixed * L.hx() : L.dom.xmin + p * L.hx();
                const double y = line.vertical ? L.dom.ymin + p * L.hy() : L.dom.ymin + line.fixed * L.hy();
                const double w = 1.0 / h.rho(x, y);
                if (p > 0) cum[p] = cum[p - 1] + 0.5 * (wprev + w);
                wprev = w;
            }
            for (int j = 1; j <= k; ++j) {
                const double target = cum[n - 1] * j / (k + 1);
                int hi = static_cast<int>(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
                hi = std::min(std::max(hi, 1), n - 1);
                const int pos = (target - cum[hi - 1] < cum[hi] - target) ? hi - 1 : hi;
                const int c = std::clamp(pos, 1, n - 2);
                if (nodes.empty() || nodes.back() != c) nodes.push_back(c);
            }
        } else {
            fail(SDDG_ERR_VALIDATION, "unknown placement strategy");
        }
        out.push_back(std::move(nodes));
    }
    return out;
}

// make_boundary_data (proj/src/boundary.cpp:44-56) / identity tables.
std::vector<std::vector<double>> boundary_tables(const sddg_density& d, const sddg_domain& dom,
                                                 int nx, int ny, int mode) {
    const double hx = (dom.xmax - dom.xmin) / (nx - 1), hy = (dom.ymax - dom.ymin) / (ny - 1);
    std::vector<std::vector<double>> t(8);
    if (mode == SDDG_BC_IDENTITY) {
        std::vector<double> fx(nx), gy(ny);
        for (int i = 0; i < nx; ++i) fx[i] = ((dom.xmin + i * hx) - dom.xmin) / (dom.xmax - dom.xmin);
        for (int j = 0; j < ny; ++j) gy[j] = ((dom.ymin + j * hy) - dom.ymin) / (dom.ymax - dom.ymin);
        fx[0] = 0.0;
        fx[nx - 1] = 1.0;
        gy[0] = 0.0;
        gy[ny - 1] = 1.0;
        t = {fx, fx, std::vector<double>(ny, 0.0), std::vector<double>(ny, 1.0),
             std::vector<double>(nx, 0.0), std::vector<double>(nx, 1.0), gy, gy};
        return t;
    }
    if (mode != SDDG_BC_REFERENCE) fail(SDDG_ERR_VALIDATION, "unknown bc_mode");
    const HostDensity h = host_density(d);
    // solve_1d_boundary (proj/src/detsolver.cpp:20-48)
    // the 1-D equidistribution of rho along an edge (solve_1d_boundary,
    // detsolver.cpp:20-48): the cumulative trapezoid of rho over the edge's
    // nodes, normalised to end at exactly 1 (the spacing cancels)
    auto edge_table = [&](int edge) {
        const bool along_x = edge < 2;
        const int n = along_x ? nx : ny;
        const int fixed = edge == 1 ? ny - 1 : (edge == 3 ? nx - 1 : 0);
        std::vector<double> cum(n, 0.0);
        double prev = 0.0;
        for (int k = 0; k < n; ++k) {
            const int i = along_x ? k : fixed, j = along_x ? fixed : k;
            const double r = h.rho(dom.xmin + i * hx, dom.ymin + j * hy);
            if (!(r > 0.0)) fail(SDDG_ERR_EVALUATION, "solve_1d_boundary: non-positive density on an edge");
            if (k > 0) cum[k] = cum[k - 1] + 0.5 * (prev + r);
            prev = r;
        }
        const double total = cum[n - 1];
        for (int k = 1; k < n - 1; ++k) cum[k] /= total;
        cum[n - 1] = 1.0;
        return cum;
    };
    t[0] = edge_table(0);
    t[1] = edge_table(1);
    t[2] = std::vector<double>(ny, 0.0);
    t[3] = std::vector<double>(ny, 1.0);
    t[4] = std::vector<double>(nx, 0.0);
    t[5] = std::vector<double>(nx, 1.0);
    t[6] = edge_table(2);
    t[7] = edge_table(3);
    return t;
}

struct IfcResult {
    std::vector<std::vector<double>> xi, eta, sxi, seta;
    int64_t mc_points = 0, restarts = 0, path_steps = 0;
    int warnings = 0;
};

// Unique Monte Carlo nodes of a plan, in line order (vertical lines first):
// proj/src/decomposition.cpp:156-169.  point_id = global index j*nx + i.
struct NodeSet {
    std::map<uint64_t, size_t> index_of;
    std::vector<double> px, py;
    std::vector<uint64_t> gid;
};

uint64_t line_node_gid(const Layout& L, const Line& ln, int pos) {
    const uint64_t i = ln.vertical ? ln.fixed : pos, j = ln.vertical ? pos : ln.fixed;
    return j * static_cast<uint64_t>(L.nx) + i;
}

NodeSet interface_nodes(const Layout& L, const std::vector<std::vector<int>>& pl) {
    NodeSet ns;
    for (size_t l = 0; l < L.lines.size(); ++l)
        for (int pos : pl[l]) {
            const Line& ln = L.lines[l];
            const uint64_t g = line_node_gid(L, ln, pos);
            if (ns.index_of.emplace(g, ns.px.size()).second) {
                const int i = ln.vertical ? ln.fixed : pos, j = ln.vertical ? pos : ln.fixed;
                ns.px.push_back(L.dom.xmin + i * L.hx());
                ns.py.push_back(L.dom.ymin + j * L.hy());
                ns.gid.push_back(g);
            }
        }
    return ns;
}

// Linear fill between known nodes and crossing reconciliation
// (proj/src/decomposition.cpp:176-246) from per-node estimates in NodeSet order.
// Natural cubic spline through (xs, ys) evaluated at integer positions
// between consecutive knots (BASELINE config 4 fill).
void spline_fill(const std::vector<int>& xs, std::vector<double>& v) {
    const int m = static_cast<int>(xs.size());
    if (m < 3) return;  // two knots: the linear fill already in place is the spline
    std::vector<double> h(m - 1), a(m, 0.0), b(m, 1.0), c(m, 0.0), r(m, 0.0), M(m, 0.0);
    for (int i = 0; i + 1 < m; ++i) h[i] = xs[i + 1] - xs[i];
    for (int i = 1; i + 1 < m; ++i) {
        a[i] = h[i - 1];
        b[i] = 2.0 * (h[i - 1] + h[i]);
        c[i] = h[i];
        r[i] = 6.0 * ((v[xs[i + 1]] - v[xs[i]]) / h[i] - (v[xs[i]] - v[xs[i - 1]]) / h[i - 1]);
    }
    // Thomas algorithm with M_0 = M_{m-1} = 0
    for (int i = 1; i < m; ++i) {
        const double f = a[i] / b[i - 1];
        b[i] -= f * c[i - 1];
        r[i] -= f * r[i - 1];
    }
    M[m - 1] = 0.0;
    for (int i = m - 2; i >= 1; --i) M[i] = (r[i] - c[i] * M[i + 1]) / b[i];
    M[0] = 0.0;
    for (int i = 0; i + 1 < m; ++i) {
        const double y0 = v[xs[i]], y1 = v[xs[i + 1]], hh = h[i];
        for (int q = xs[i] + 1; q < xs[i + 1]; ++q) {
            const double t1 = q - xs[i], t0 = xs[i + 1] - q;
            v[q] = (M[i] * t0 * t0 * t0 + M[i + 1] * t1 * t1 * t1) / (6.0 * hh) +
                   (y0 / hh - M[i] * hh / 6.0) * t0 + (y1 / hh - M[i + 1] * hh / 6.0) * t1;
        }
    }
}

// v[q] for a < q < b on the straight line between v[a] and v[b], with the
// reference's weights (1 - t) v[a] + t v[b], t = (q - a) / (b - a)
// (decomposition.cpp:218-226)
void blend_between(std::vector<double>& v, int a, int b) {
    for (int q = a + 1; q < b; ++q) {
        const double t = static_cast<double>(q - a) / (b - a);
        v[q] = (1.0 - t) * v[a] + t * v[b];
    }
}

// The interface values of every line from the Monte Carlo estimates
// (decomposition.cpp:176-246): each line is anchored at its two boundary
// nodes (read from the boundary tables, so they equal the subdomain corner
// data bit for bit), takes the estimates at its Monte Carlo nodes, and is
// filled between neighbouring known nodes -- linearly as in the reference, or
// by a natural cubic spline through the known nodes (BASELINE config 4).
// Where a horizontal and a vertical line cross at a node that was not
// estimated, the vertical line's value is the one both carry.
IfcResult fill_interfaces(const Layout& L, const NodeSet& ns, const sddg_boundary& bd,
                          const sddg_estimate* est, int interp = SDDG_INTERP_LINEAR) {
    if (interp != SDDG_INTERP_LINEAR && interp != SDDG_INTERP_SPLINE)
        fail(SDDG_ERR_VALIDATION, "unknown interface interpolation");
    IfcResult out;
    out.mc_points = static_cast<int64_t>(ns.px.size());
    for (int64_t k = 0; k < out.mc_points; ++k) {
        out.restarts += est[k].restarts;
        out.warnings += est[k].warn ? 1 : 0;
    }
    const size_t n_lines = L.lines.size();
    out.xi.assign(n_lines, {});
    out.eta.assign(n_lines, {});
    out.sxi.assign(n_lines, {});
    out.seta.assign(n_lines, {});
    for (size_t l = 0; l < n_lines; ++l) {
        const Line& ln = L.lines[l];
        const int last = ln.length - 1, at = ln.fixed;
        // a vertical line runs from the bottom edge to the top one, a
        // horizontal line from the left edge to the right one
        const int e0 = ln.vertical ? 0 : 2, e1 = ln.vertical ? 1 : 3;
        std::vector<double>&xi = out.xi[l], &eta = out.eta[l], &sx = out.sxi[l], &se = out.seta[l];
        xi.assign(ln.length, 0.0);
        eta.assign(ln.length, 0.0);
        sx.assign(ln.length, 0.0);
        se.assign(ln.length, 0.0);
        xi[0] = bd.f[e0][at];
        eta[0] = bd.g[e0][at];
        xi[last] = bd.f[e1][at];
        eta[last] = bd.g[e1][at];
        std::vector<int> knots(1, 0);  // the nodes whose values are known, in order
        for (int pos = 1; pos < last; ++pos) {
            const auto hit = ns.index_of.find(line_node_gid(L, ln, pos));
            if (hit == ns.index_of.end()) continue;
            const sddg_estimate& e = est[hit->second];
            xi[pos] = e.xi;
            eta[pos] = e.eta;
            sx[pos] = e.se_xi;
            se[pos] = e.se_eta;
            knots.push_back(pos);
        }
        knots.push_back(last);
        for (size_t k = 0; k + 1 < knots.size(); ++k) {
            blend_between(xi, knots[k], knots[k + 1]);
            blend_between(eta, knots[k], knots[k + 1]);
        }
        if (interp == SDDG_INTERP_SPLINE) {
            spline_fill(knots, xi);
            spline_fill(knots, eta);
        }
    }
    for (size_t h = 0; h < n_lines; ++h) {
        if (L.lines[h].vertical) continue;
        for (size_t v = 0; v < n_lines; ++v) {
            if (!L.lines[v].vertical) continue;
            const int col = L.lines[v].fixed, row = L.lines[h].fixed;
            if (ns.index_of.count(static_cast<uint64_t>(row) * L.nx + col)) continue;  // estimated: both read it
            out.xi[h][col] = out.xi[v][row];
            out.eta[h][col] = out.eta[v][row];
        }
    }
    return out;
}

// solve_interfaces (proj/src/decomposition.cpp:147-248), walks on the GPU.
IfcResult solve_interfaces(sddg_ctx* c, const sddg_density& d, const Layout& L,
                           const std::vector<std::vector<int>>& pl, const sddg_boundary& bd,
                           const sddg_walk_config& cfg, int interp = SDDG_INTERP_LINEAR) {
    const NodeSet ns = interface_nodes(L, pl);
    std::vector<sddg_estimate> est(ns.px.size());
    int64_t steps = 0;
    if (!ns.px.empty()) {
        estimates_host(c, d, L.dom, bd, cfg, ns.px.data(), ns.py.data(), ns.gid.data(),
                       static_cast<int64_t>(ns.px.size()), est.data());
        steps = c->last_steps;
    }
    IfcResult out = fill_interfaces(L, ns, bd, est.data(), interp);
    out.path_steps = steps;
    return out;
}

// Subdomain phase of solve_sdd (proj/src/decomposition.cpp:292-355) for
// subdomains [s_lo, s_hi): global weights, per-(subdomain, field) edge data
// from the boundary tables or the interface lines, one batched K3 launch.
// u receives, per subdomain, the xi field then the eta field (nx*ny each).
void solve_subdomains(sddg_ctx* c, const sddg_density& d, const Layout& L,
                      const std::vector<std::vector<double>>& tabs,
                      const std::vector<std::vector<double>>& ixi,
                      const std::vector<std::vector<double>>& ieta, const sddg_solver_config& sc,
                      int s_lo, int s_hi, std::vector<double>& u,
                      std::vector<sddg_solve_info>& info) {
    std::map<int, size_t> vline, hline;
    for (size_t l = 0; l < L.lines.size(); ++l) {
        if (L.lines[l].vertical) vline[L.lines[l].fixed] = l;
        else hline[L.lines[l].fixed] = l;
    }
    const int nx = L.nx, ny = L.ny;
    // weight_values on the global grid (detsolver.cpp:219-224)
    const HostDensity h = host_density(d);
    std::vector<double> w(static_cast<size_t>(nx) * ny);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            w[static_cast<size_t>(j) * nx + i] =
                1.0 / h.rho(L.dom.xmin + i * L.hx(), L.dom.ymin + j * L.hy());
    std::vector<sddg_subdomain> subs;
    std::vector<double> bc;
    for (int s = s_lo; s < s_hi; ++s) {
        const int a = s % L.sx, b = s / L.sx;
        const sddg_subdomain q{a * L.bx, b * L.by, L.bx + 1, L.by + 1};
        for (int field = 0; field < 2; ++field) {
            const bool fxi = field == 0;
            const auto& lines = fxi ? ixi : ieta;
            for (int e = 0; e < 4; ++e) {
                const bool horiz = e < 2;
                const int len = horiz ? q.nx : q.ny, lo = horiz ? q.i0 : q.j0;
                const std::vector<double>* src;
                if (e == 0) src = q.j0 == 0 ? &tabs[fxi ? 0 : 4] : &lines[hline.at(q.j0)];
                else if (e == 1) {
                    const int j1 = q.j0 + q.ny - 1;
                    src = j1 == ny - 1 ? &tabs[fxi ? 1 : 5] : &lines[hline.at(j1)];
                } else if (e == 2) src = q.i0 == 0 ? &tabs[fxi ? 2 : 6] : &lines[vline.at(q.i0)];
                else {
                    const int i1 = q.i0 + q.nx - 1;
                    src = i1 == nx - 1 ? &tabs[fxi ? 3 : 7] : &lines[vline.at(i1)];
                }
                bc.insert(bc.end(), src->begin() + lo, src->begin() + lo + len);
            }
            subs.push_back(q);
        }
    }
    const int64_t nj = static_cast<int64_t>(subs.size());
    u.assign(static_cast<size_t>(nj) * (L.bx + 1) * (L.by + 1), 0.0);
    info.assign(nj, sddg_solve_info{});
    if (team_active(c))
        team_solve_batch(c, w.data(), nx, ny, L.hx(), L.hy(), nj, 2, subs.data(), bc.data(), sc, u.data(),
                         info.data());
    else
        solve_batch_host(c, w.data(), nx, ny, L.hx(), L.hy(), nj, subs.data(), bc.data(), sc, u.data(),
                         info.data());
}

// smooth_interface on the GPU (K7, smoothing.cpp:140-183)
std::vector<double> smooth_line(sddg_ctx* c, const std::vector<double>& v, int span) {
    const int n = static_cast<int>(v.size());
    if (span < 3 || span % 2 == 0 || span > n)
        fail(SDDG_ERR_VALIDATION, "smooth_interface: span must be odd and in [3, length]");
    cudaStream_t st = c->stream;
    double* d = static_cast<double*>(c->m_q.ensure(sizeof(double) * 2 * n + 64));
    int* derr = reinterpret_cast<int*>(d + 2 * n);
    ck(cudaMemcpyAsync(d, v.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "h2d");
    ck(cudaMemsetAsync(derr, 0, sizeof(int), st), "memset");
    ck(loess_run(d, d + n, n, span, derr, st), "loess launch");
    std::vector<double> out(n);
    int herr = 0;
    ck(cudaMemcpyAsync(out.data(), d + n, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "loess");
    if (herr) fail(SDDG_ERR_NUMERICAL, "smooth_interface: singular local fit");
    return out;
}

std::vector<std::vector<double>> split_lines(const Layout& L, const double* flat) {
    std::vector<std::vector<double>> out;
    size_t off = 0;
    for (const Line& ln : L.lines) {
        out.emplace_back(flat + off, flat + off + ln.length);
        off += ln.length;
    }
    return out;
}

sddg_boundary make_boundary_view(const sddg_domain& dom, int nx, int ny,
                                 const std::vector<std::vector<double>>& t) {
    sddg_boundary b;
    b.dom = dom;
    b.nx = nx;
    b.ny = ny;
    for (int k = 0; k < 4; ++k) {
        b.f[k] = t[k].data();
        b.g[k] = t[4 + k].data();
    }
    return b;
}

sddg_status finish(sddg_ctx* c, const Fail& f) {
    if (c) c->err = f.msg;
    else g_free_err = f.msg;
    return f.st;
}

// Every context entry point is an NVTX range named after the C-ABI function
// (host-side phases in nsys / ncu --nvtx; a few ns when no tool is attached).
#define API_BEGIN(ctx)                                   \
    if (!(ctx)) {                                        \
        g_free_err = "NULL context";                     \
        return SDDG_ERR_VALIDATION;                      \
    }                                                    \
    const nvtx3::scoped_range _nvtx{__func__};           \
    std::lock_guard<std::mutex> _lk((ctx)->mu);          \
    try {                                                \
        ck(cudaSetDevice((ctx)->device), "cudaSetDevice");
#define API_RETURN_OK(ctx) \
    do {                   \
        (ctx)->err.clear(); \
        return SDDG_OK;    \
    } while (0)
#define API_END(ctx)                                     \
    }                                                    \
    catch (const Fail& f) {                              \
        return finish((ctx), f);                         \
    }                                                    \
    catch (const std::exception& e) {                    \
        return finish((ctx), Fail{SDDG_ERR_INTERNAL, e.what()}); \
    }                                                    \
    (ctx)->err.clear();                                  \
    return SDDG_OK;

void set_free_error(const std::string& m) { g_free_err = m; }

}  // namespace rt
}  // namespace sddg

namespace sddg {

// Tables of fastmath.cuh, in 80-bit long double, rounded once to double.
void make_fm_tables(void* out) {
    fm::FmTables& t = *static_cast<fm::FmTables*>(out);
    const long double pi = acosl(-1.0L), ln2 = logl(2.0L);
    for (int j = 0; j < fm::kScN; ++j) {
        const long double a = 2.0L * pi * j / fm::kScN;
        t.sc[j][0] = static_cast<double>(sinl(a));
        t.sc[j][1] = static_cast<double>(cosl(a));
    }
    for (int j = 0; j < fm::kLgN; ++j) {
        // Gal's accurate table: among the 2048 doubles nearest fl(1/c_j), take
        // the rc whose log lies closest to a double (80-bit logl resolves 11
        // bits past the double; typically within 2^-8 ulp, always < 2^-5)
        const double c = 1.0 + (j + 0.5) / fm::kLgN;
        const double rc0 = static_cast<double>(1.0L / c);
        double rc = rc0, up = rc0, dn = rc0, best_rc = rc0;
        long double L = 0.0L, best_L = 0.0L, best_err = 1.0L;
        for (int t = 0; t < 2048; ++t) {  // rc0, rc0+1ulp, rc0-1ulp, rc0+2ulp, ...
            if (t > 0) rc = (t & 1) ? (up = std::nextafter(up, 2.0)) : (dn = std::nextafter(dn, 0.0));
            L = -logl(static_cast<long double>(rc));       // log(1/rc), consistent with r
            if (j >= fm::kLgSplit) L -= ln2;              // log(c/2) branch
            const double Lh = static_cast<double>(L);
            const long double ulp =
                static_cast<long double>(std::nextafter(std::fabs(Lh), 1e300) - std::fabs(Lh));
            const long double err = fabsl(L - static_cast<long double>(Lh)) / ulp;
            if (err < best_err) {
                best_err = err;
                best_rc = rc;
                best_L = L;
            }
            if (err <= 1.0L / 256.0L) break;
        }
        rc = best_rc;
        L = best_L;
        // stored pre-scaled by -2 (exact): fastmath.cuh fm2log_tab
        t.lg[j][0] = -2.0 * rc;
        t.lg[j][1] = -2.0 * static_cast<double>(L);
    }
    for (int j = 0; j < fm::kExN; ++j)
        t.e2[j] = static_cast<double>(exp2l(static_cast<long double>(j) / fm::kExN));
    using namespace fm;
    for (double& v : t.k) v = 0.0;
    t.k[K_E6] = 1.0 / 720.0;
    t.k[K_E5] = 1.0 / 120.0;
    t.k[K_E4] = 1.0 / 24.0;
    t.k[K_E3] = 1.0 / 6.0;
    t.k[K_EXS] = kExScale;
    t.k[K_EXHI] = kExHi;
    t.k[K_EXLO] = kExLo;
    t.k[K_L7] = 1.0 / 448.0;  // log1p coefficients in R = -2r (exact power-of-2 scalings)
    t.k[K_L6] = 1.0 / 192.0;
    t.k[K_L5] = 1.0 / 80.0;
    t.k[K_L3] = 1.0 / 12.0;
    t.k[K_LN2HI] = 2.0 * kLn2Hi;  // multiplies -k (fm2log_tab)
    t.k[K_LN2LO] = 2.0 * kLn2Lo;
    t.k[K_I2D] = 4503601774854144.0;
    t.k[K_TWOPI] = 6.283185307179586;
    t.k[K_S7] = -1.0 / 5040.0;
    t.k[K_S5] = 1.0 / 120.0;
    t.k[K_S3] = -1.0 / 6.0;
    t.k[K_C6] = -1.0 / 720.0;
    t.k[K_C4] = 1.0 / 24.0;
    t.k[K_OPEN] = 1.0 - 0x1.0p-53;
    t.k[K_SCB] = 4503599627370496.0 + 4503599627370496.0 / kScN;  // 2^52 + 2^52 / N
    t.k[K_TWOPI53] = 6.283185307179586 * 0x1.0p-53;
}

bool walk_variant_supported(int dv, int precision) {
    if ((dv >= 32 && dv <= 36) || (dv >= 40 && dv <= 42)) return true;  // walk_fast.cu
    return precision == SDDG_FP64 && ((dv >= 0 && dv <= 4) || (dv >= 16 && dv <= 18) || dv == 20);
}

cudaError_t launch_walk(int dv, int precision, const WalkArgs& a, int grid, cudaStream_t s, int block) {
    if (!walk_variant_supported(dv, precision)) return cudaErrorInvalidValue;
    if (dv >= 32) return launch_walk_fast(dv, precision, a, grid, s, block);
    return launch_walk_ref(dv, a, grid, s, block);
}

cudaError_t launch_walk_tail(int dv, const WalkArgs& a, cudaStream_t s) {
    if (!a.cont) return cudaSuccess;
    if (dv >= 32) return launch_walk_tail_fast(dv, a, s);
    return launch_walk_tail_ref(dv, a, s);
}

cudaError_t walk_occupancy(int dv, int precision, int* b, int* block) {
    if (!walk_variant_supported(dv, precision)) return cudaErrorInvalidValue;
    if (dv >= 32) return occupancy_walk_fast(dv, precision, b, block);
    return occupancy_walk_ref(dv, b, block);
}

}  // namespace sddg

extern "C" {

const char* sddg_version(void) { return "sddg 0.1 (sm_100a)"; }
int sddg_abi_version(void) { return SDDG_ABI_VERSION; }

sddg_status sddg_device_count(int32_t* n) {
    int k = 0;
    const cudaError_t e = cudaGetDeviceCount(&k);
    *n = e == cudaSuccess ? k : 0;
    return e == cudaSuccess ? SDDG_OK : SDDG_ERR_CUDA;
}

sddg_status sddg_create(int32_t device, sddg_ctx** out) {
    *out = nullptr;
    try {
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) fail(SDDG_ERR_CUDA, "no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp p;
        ck(cudaGetDeviceProperties(&p, device), "properties");
        if (p.major != 10 || p.minor != 0)
            fail(SDDG_ERR_CUDA, std::string("sddg is built for sm_100a (B200); device is ") + p.name);
        auto* c = new sddg_ctx();
        c->device = device;
        c->sms = p.multiProcessorCount;
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreate(&c->ev0), "event");
        ck(cudaEventCreate(&c->ev1), "event");
        {
            fm::FmTables t;
            make_fm_tables(&t);
            void* d = c->fm_tables.ensure(sizeof(t));
            ck(cudaMemcpy(d, &t, sizeof(t), cudaMemcpyHostToDevice), "fm tables");
        }
        *out = c;
    } catch (const Fail& f) {
        g_free_err = f.msg;
        return f.st;
    }
    return SDDG_OK;
}

void sddg_destroy(sddg_ctx* c) {
    if (!c) return;
    team_destroy(c);
    cudaSetDevice(c->device);
    for (DevBuf* b : {&c->rec_f, &c->rec_g, &c->rec_meta, &c->nodes, &c->est, &c->tables,
                      &c->counters, &c->dump, &c->perm, &c->nsteps, &c->t_recv, &c->t_nodes, &c->t_pts, &c->dens_tab, &c->tail_cont, &c->fm_tables, &c->gidx, &c->s_w, &c->s_jobs, &c->s_bc, &c->s_u, &c->s_info,
                      &c->s_coef, &c->s_err, &c->s_large, &c->s_omega, &c->s_perm, &c->m_in, &c->m_out, &c->m_q, &c->m_misc})
        b->release();
    for (cudaEvent_t e : c->bev) cudaEventDestroy(e);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* sddg_last_error(const sddg_ctx* c) { return c ? c->err.c_str() : g_free_err.c_str(); }

sddg_status sddg_last_stats(const sddg_ctx* c, int64_t* steps, int64_t* launches, double* ms) {
    if (!c) return SDDG_ERR_VALIDATION;
    if (steps) *steps = c->last_steps;
    if (launches) *launches = c->last_launches;
    if (ms) *ms = c->last_ms;
    return SDDG_OK;
}

sddg_status sddg_last_tail_stats(const sddg_ctx* c, int64_t* handoffs, double* tail_ms) {
    if (!c) return SDDG_ERR_VALIDATION;
    if (handoffs) *handoffs = c->last_handoffs;
    if (tail_ms) *tail_ms = c->last_tail_ms;
    return SDDG_OK;
}

sddg_status sddg_probe_fma_peak(sddg_ctx* ctx, int32_t precision, double* tflops) {
    API_BEGIN(ctx)
    if (precision != SDDG_FP64 && precision != SDDG_FP32) fail(SDDG_ERR_VALIDATION, "precision");
    ck(probe_fma_tflops(precision, ctx->sms, ctx->stream, tflops), "probe");
    API_END(ctx)
}

sddg_status sddg_probe_onchip_bandwidth(sddg_ctx* ctx, double* l2_gbps, double* smem_gbps) {
    API_BEGIN(ctx)
    ck(probe_onchip_gbps(ctx->sms, ctx->stream, l2_gbps, smem_gbps), "probe");
    API_END(ctx)
}

sddg_status sddg_selftest_fastmath(sddg_ctx* ctx, int64_t n, uint64_t max_ulp[6]) {
    API_BEGIN(ctx)
    unsigned long long m[6];
    ck(fastmath_selftest(n, ctx->fm_tables.p, m), "fastmath self-test");
    for (int k = 0; k < 6; ++k) max_ulp[k] = m[k];
    API_END(ctx)
}

sddg_status sddg_selftest_division(sddg_ctx* ctx, int64_t n, uint64_t* mismatches) {
    API_BEGIN(ctx)
    if (n < 0 || !mismatches) fail(SDDG_ERR_VALIDATION, "selftest_division: n >= 0 and an output pointer");
    unsigned long long m = 0;
    ck(division_selftest(n, &m), "division self-test");
    *mismatches = m;
    API_END(ctx)
}

sddg_status sddg_selftest_drift(sddg_ctx* ctx, int32_t kind, const sddg_domain* dom, int64_t n, double out[4]) {
    API_BEGIN(ctx)
    if (n < 1 || !out || !dom) fail(SDDG_ERR_VALIDATION, "selftest_drift: n >= 1, a domain and an output pointer");
    if (kind != SDDG_DENS_RING_W && kind != SDDG_DENS_SHOCK_W && kind != SDDG_DENS_TWOBUMP_W)
        fail(SDDG_ERR_VALIDATION, "selftest_drift: a BASELINE density (ring, shock, two-bump)");
    check_domain(*dom);
    const double box[4] = {dom->xmin, dom->xmax, dom->ymin, dom->ymax};
    ck(drift_selftest(kind, n, ctx->fm_tables.p, box, out), "drift self-test");
    API_END(ctx)
}

sddg_status sddg_mc_estimate_batch(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                   const sddg_boundary* bd, const sddg_walk_config* cfg,
                                   const double* px, const double* py, const uint64_t* pid,
                                   int64_t n, sddg_estimate* out) {
    API_BEGIN(ctx)
    estimates_host(ctx, *dens, *dom, *bd, *cfg, px, py, pid, n, out);
    API_END(ctx)
}

sddg_status sddg_mc_estimate_batch_device(sddg_ctx* ctx, const sddg_density* dens,
                                          const sddg_domain* dom, const sddg_boundary* bd,
                                          const sddg_walk_config* cfg, const double* d_px,
                                          const double* d_py, const uint64_t* d_pid, int64_t n,
                                          sddg_estimate* d_out, void* stream) {
    API_BEGIN(ctx)
    validate_walk(*cfg);
    check_domain(*dom);
    check_boundary(*bd);
    walk_variant(*dens, *cfg);
    check_positivity(*dens, *dom);
    if (n > 0) {
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
        std::vector<double> hx(n), hy(n);
        ck(cudaMemcpyAsync(hx.data(), d_px, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaMemcpyAsync(hy.data(), d_py, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        check_points(*dom, hx.data(), hy.data(), n);
        if (team_active(ctx)) {
            team_estimates(ctx, *dens, *dom, *bd, *cfg, d_px, d_py, d_pid, n, d_out, st, hx.data(),
                           hy.data());
        } else {
            const std::vector<uint32_t> order = cost_order(
                node_costs(exit_time_model(ctx, *dens, *dom), *cfg, hx.data(), hy.data(), n), nullptr);
            run_estimates(ctx, *dens, *dom, *bd, *cfg, d_px, d_py, d_pid, n, order, d_out, st);
        }
    }
    API_END(ctx)
}

sddg_status sddg_walk_dump(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                           const sddg_boundary* bd, const sddg_walk_config* cfg, double px,
                           double py, uint64_t pid, int64_t walk_lo, int64_t n, sddg_path* out) {
    API_BEGIN(ctx)
    validate_walk(*cfg);
    check_domain(*dom);
    check_boundary(*bd);
    const int dv = walk_variant(*dens, *cfg);
    check_positivity(*dens, *dom);
    check_points(*dom, &px, &py, 1);
    if (walk_lo < 0 || walk_lo + n > 0x100000000LL)
        fail(SDDG_ERR_VALIDATION, "walk range must fit the 32-bit stream walk id");
    if (n > 0) {
        cudaStream_t st = ctx->stream;
        const double* dtab = upload_tables(ctx, *bd);
        char* nb = static_cast<char*>(ctx->nodes.ensure(3 * sizeof(double)));
        double* dn = reinterpret_cast<double*>(nb);
        unsigned char hv[3 * sizeof(double)];
        std::memcpy(hv, &px, sizeof(double));
        std::memcpy(hv + sizeof(double), &py, sizeof(double));
        std::memcpy(hv + 2 * sizeof(double), &pid, sizeof(uint64_t));
        ck(cudaMemcpyAsync(dn, hv, sizeof(hv), cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaStreamSynchronize(st), "sync");
        Counters* cnt = static_cast<Counters*>(ctx->counters.ensure(sizeof(Counters)));
        ck(cudaMemsetAsync(cnt, 0, sizeof(Counters), st), "memset");
        sddg_path* dd = static_cast<sddg_path*>(ctx->dump.ensure(sizeof(sddg_path) * n));
        WalkArgs a;
        fill_args(a, *dens, *dom, *bd, *cfg, dtab);
        a.tab = upload_density(ctx, *dens);
        a.fm_tables = ctx->fm_tables.p;
        a.px = dn;
        a.py = dn + 1;
        a.pid = reinterpret_cast<const uint64_t*>(dn + 2);
        a.walks = n;
        a.walk_lo = walk_lo;
        a.n_nodes = 1;
        a.total = static_cast<uint64_t>(n);
        a.next = &cnt->next;
        a.steps = &cnt->steps;
        a.err_flag = &cnt->err_flag;
        a.err_info = &cnt->err_info;
        a.dump = dd;
        const auto [grid, blk] = walk_grid(ctx, dv, cfg->precision, a.total);
        const unsigned long long lanes = static_cast<unsigned long long>(grid) * blk;
        const DrainPlan dp = enable_tail(ctx, a, cfg->precision, cnt, lanes);
        set_next_kernel<<<1, 1, 0, st>>>(cnt, lanes, std::min<unsigned long long>(lanes, a.total));
        ck(cudaEventRecord(ctx->ev0, st), "event");
        const int nl = launch_walk_stages(ctx, dv, cfg->precision, a, dp, grid, cnt, st, nullptr);
        ck(cudaEventRecord(ctx->ev1, st), "event");
        Counters hc;
        ck(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaMemcpyAsync(out, dd, sizeof(sddg_path) * n, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "walk dump");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        ctx->last_ms = ms;
        ctx->last_steps = static_cast<int64_t>(hc.steps);
        ctx->last_launches = nl + 1;
        ctx->last_handoffs = a.cont ? std::min<int64_t>(hc.n_cont, a.cont_cap) : 0;
        ctx->last_tail_ms = 0.0;
        raise_kernel_error(hc);
    }
    API_END(ctx)
}

sddg_status sddg_solve_dirichlet_batch(sddg_ctx* ctx, const double* w, int32_t gnx, int32_t gny,
                                       double hx, double hy, int64_t n, const sddg_subdomain* subs,
                                       const double* bc, const sddg_solver_config* sc, double* u,
                                       sddg_solve_info* info) {
    API_BEGIN(ctx)
    solve_batch_host(ctx, w, gnx, gny, hx, hy, n, subs, bc, *sc, u, info);
    API_END(ctx)
}

sddg_status sddg_make_boundary_data(const sddg_density* dens, const sddg_domain* dom, int32_t nx,
                                    int32_t ny, int32_t mode, double* tables8[8]) {
    try {
        check_domain(*dom);
        if (nx < 3 || ny < 3) fail(SDDG_ERR_VALIDATION, "GridSpec: needs nx >= 3 and ny >= 3");
        const auto t = boundary_tables(*dens, *dom, nx, ny, mode);
        for (int k = 0; k < 8; ++k) std::memcpy(tables8[k], t[k].data(), sizeof(double) * t[k].size());
    } catch (const Fail& f) {
        return finish(nullptr, f);
    } catch (const std::exception& e) {
        return finish(nullptr, Fail{SDDG_ERR_EVALUATION, e.what()});
    }
    return SDDG_OK;
}

sddg_status sddg_plan_interface_points(const sddg_density* dens, const sddg_domain* dom,
                                       int32_t nx, int32_t ny, int32_t sx, int32_t sy,
                                       int32_t placement, int32_t k, int32_t* n_lines,
                                       int32_t* vert, int32_t* fixed, int32_t* counts,
                                       int32_t* nodes) {
    try {
        const Layout L = build_layout(*dom, nx, ny, sx, sy);
        const auto pl = plan(*dens, L, placement, k);
        *n_lines = static_cast<int32_t>(L.lines.size());
        int off = 0;
        for (size_t l = 0; l < L.lines.size(); ++l) {
            vert[l] = L.lines[l].vertical ? 1 : 0;
            fixed[l] = L.lines[l].fixed;
            counts[l] = static_cast<int32_t>(pl[l].size());
            for (int v : pl[l]) nodes[off++] = v;
        }
    } catch (const Fail& f) {
        return finish(nullptr, f);
    } catch (const std::exception& e) {
        return finish(nullptr, Fail{SDDG_ERR_EVALUATION, e.what()});
    }
    return SDDG_OK;
}

sddg_status sddg_solve_interfaces(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                  int32_t nx, int32_t ny, int32_t sx, int32_t sy, int32_t placement,
                                  int32_t k, const sddg_boundary* bd, const sddg_walk_config* cfg,
                                  const sddg_sdd_options* opts, double* xi, double* eta,
                                  double* sxi, double* seta, sddg_sdd_stats* stats) {
    API_BEGIN(ctx)
    const double t0 = now_s();
    const Layout L = build_layout(*dom, nx, ny, sx, sy);
    const auto pl = plan(*dens, L, placement, k);
    const IfcResult r = solve_interfaces(ctx, *dens, L, pl, *bd, *cfg,
                                         opts ? opts->interp : SDDG_INTERP_LINEAR);
    size_t off = 0;
    for (size_t l = 0; l < r.xi.size(); ++l) {
        const size_t n = r.xi[l].size();
        std::memcpy(xi + off, r.xi[l].data(), sizeof(double) * n);
        std::memcpy(eta + off, r.eta[l].data(), sizeof(double) * n);
        if (sxi) std::memcpy(sxi + off, r.sxi[l].data(), sizeof(double) * n);
        if (seta) std::memcpy(seta + off, r.seta[l].data(), sizeof(double) * n);
        off += n;
    }
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->t_stoc = r.mc_points > 0 ? now_s() - t0 : 0.0;
        stats->mc_points = r.mc_points;
        stats->restarts = r.restarts;
        stats->path_steps = r.path_steps;
        stats->warnings = r.warnings;
    }
    API_END(ctx)
}

sddg_status sddg_solve_sdd(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                           int32_t nx, int32_t ny, int32_t sx, int32_t sy, int32_t placement,
                           int32_t k, int32_t bc_mode, const sddg_walk_config* cfg,
                           const sddg_solver_config* sc, const sddg_sdd_options* opts, double* xi,
                           double* eta, sddg_sdd_stats* stats) {
    API_BEGIN(ctx)
    // solve_sdd (proj/src/decomposition.cpp:262-385)
    const Layout L = build_layout(*dom, nx, ny, sx, sy);
    const double tb0 = now_s();
    std::optional<nvtx3::scoped_range> phase{std::in_place, "solve_sdd: boundary data"};
    const auto tabs = boundary_tables(*dens, *dom, nx, ny, bc_mode);
    const double t_bd = now_s() - tb0;
    const sddg_boundary bd = make_boundary_view(*dom, nx, ny, tabs);
    const auto pl = plan(*dens, L, placement, k);
    const double t0 = now_s();
    phase.emplace("solve_sdd: interface walks (T_stoc)");
    IfcResult ifc = solve_interfaces(ctx, *dens, L, pl, bd, *cfg, opts ? opts->interp : SDDG_INTERP_LINEAR);
    const double t_stoc = ifc.mc_points > 0 ? now_s() - t0 : 0.0;
    // optional interface pre-smoothing (decomposition.cpp:274-282)
    double t_smooth = 0.0;
    if (opts && opts->smooth_interface) {
        const double ts = now_s();
        for (size_t l = 0; l < ifc.xi.size(); ++l) {
            ifc.xi[l] = smooth_line(ctx, ifc.xi[l], opts->smooth_span);
            ifc.eta[l] = smooth_line(ctx, ifc.eta[l], opts->smooth_span);
        }
        t_smooth = now_s() - ts;
    }
    const int64_t steps = ifc.path_steps;

    const double ts0 = now_s();
    phase.emplace("solve_sdd: subdomain solves + assembly (T_sub)");
    const int n_sub = sx * sy;
    std::vector<double> u;
    std::vector<sddg_solve_info> info;
    solve_subdomains(ctx, *dens, L, tabs, ifc.xi, ifc.eta, *sc, 0, n_sub, u, info);
    std::vector<sddg_subdomain> subs;
    for (int s = 0; s < n_sub; ++s)
        for (int f = 0; f < 2; ++f)
            subs.push_back(sddg_subdomain{(s % sx) * L.bx, (s / sx) * L.by, L.bx + 1, L.by + 1});
    int warns = ifc.warnings;
    size_t off = 0;
    for (int s = 0; s < 2 * n_sub; ++s) {
        const sddg_subdomain& q = subs[s];
        double* dst = (s % 2 == 0) ? xi : eta;
        for (int j = 0; j < q.ny; ++j)
            for (int i = 0; i < q.nx; ++i)
                dst[static_cast<size_t>(q.j0 + j) * nx + (q.i0 + i)] = u[off + static_cast<size_t>(j) * q.nx + i];
        off += static_cast<size_t>(q.nx) * q.ny;
        if (!info[s].converged) ++warns;
    }
    if (stats) {
        stats->t_bd = t_bd;
        stats->t_stoc = t_stoc;
        stats->t_sub = t_bd + (now_s() - ts0);
        stats->t_smooth = t_smooth;
        stats->mc_points = ifc.mc_points;
        stats->subdomain_solves = 2 * n_sub;
        stats->restarts = ifc.restarts;
        stats->path_steps = steps;
        stats->warnings = warns;
        stats->reserved = 0;
    }
    API_END(ctx)
}

sddg_status sddg_interface_nodes(const sddg_density* dens, const sddg_domain* dom, int32_t nx,
                                 int32_t ny, int32_t sx, int32_t sy, int32_t placement, int32_t k,
                                 int64_t cap, double* px, double* py, uint64_t* pid, int64_t* n) {
    try {
        const Layout L = build_layout(*dom, nx, ny, sx, sy);
        const NodeSet ns = interface_nodes(L, plan(*dens, L, placement, k));
        *n = static_cast<int64_t>(ns.px.size());
        if (*n > cap) fail(SDDG_ERR_VALIDATION, "interface_nodes: capacity too small");
        for (int64_t q = 0; q < *n; ++q) {
            px[q] = ns.px[q];
            py[q] = ns.py[q];
            pid[q] = ns.gid[q];
        }
    } catch (const Fail& f) {
        return finish(nullptr, f);
    } catch (const std::exception& e) {
        return finish(nullptr, Fail{SDDG_ERR_EVALUATION, e.what()});
    }
    return SDDG_OK;
}

sddg_status sddg_fill_interfaces(const sddg_density* dens, const sddg_domain* dom, int32_t nx,
                                 int32_t ny, int32_t sx, int32_t sy, int32_t placement, int32_t k,
                                 const sddg_boundary* bd, const sddg_estimate* est, int64_t n,
                                 const sddg_sdd_options* opts, double* xi, double* eta, double* sxi,
                                 double* seta) {
    try {
        const Layout L = build_layout(*dom, nx, ny, sx, sy);
        const NodeSet ns = interface_nodes(L, plan(*dens, L, placement, k));
        if (static_cast<int64_t>(ns.px.size()) != n)
            fail(SDDG_ERR_VALIDATION, "fill_interfaces: estimate count does not match the plan");
        check_boundary(*bd);
        const IfcResult r = fill_interfaces(L, ns, *bd, est, opts ? opts->interp : SDDG_INTERP_LINEAR);
        size_t off = 0;
        for (size_t l = 0; l < r.xi.size(); ++l) {
            const size_t m = r.xi[l].size();
            std::memcpy(xi + off, r.xi[l].data(), sizeof(double) * m);
            std::memcpy(eta + off, r.eta[l].data(), sizeof(double) * m);
            if (sxi) std::memcpy(sxi + off, r.sxi[l].data(), sizeof(double) * m);
            if (seta) std::memcpy(seta + off, r.seta[l].data(), sizeof(double) * m);
            off += m;
        }
    } catch (const Fail& f) {
        return finish(nullptr, f);
    } catch (const std::exception& e) {
        return finish(nullptr, Fail{SDDG_ERR_EVALUATION, e.what()});
    }
    return SDDG_OK;
}

sddg_status sddg_solve_subdomains(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                  int32_t nx, int32_t ny, int32_t sx, int32_t sy, int32_t bc_mode,
                                  const double* xi_lines, const double* eta_lines,
                                  const sddg_solver_config* sc, int32_t s_lo, int32_t s_hi,
                                  double* fields, sddg_solve_info* info) {
    API_BEGIN(ctx)
    const Layout L = build_layout(*dom, nx, ny, sx, sy);
    if (s_lo < 0 || s_hi > sx * sy || s_lo > s_hi)
        fail(SDDG_ERR_VALIDATION, "solve_subdomains: subdomain range out of the layout");
    const auto tabs = boundary_tables(*dens, *dom, nx, ny, bc_mode);
    const auto ixi = split_lines(L, xi_lines), ieta = split_lines(L, eta_lines);
    std::vector<double> u;
    std::vector<sddg_solve_info> inf;
    solve_subdomains(ctx, *dens, L, tabs, ixi, ieta, *sc, s_lo, s_hi, u, inf);
    std::memcpy(fields, u.data(), sizeof(double) * u.size());
    if (info) std::memcpy(info, inf.data(), sizeof(sddg_solve_info) * inf.size());
    API_END(ctx)
}

sddg_status sddg_invert_mesh(sddg_ctx* ctx, const double* xi, const double* eta, int32_t nx,
                             int32_t ny, const sddg_domain* dom, int32_t m_xi, int32_t m_eta,
                             double* x, double* y) {
    API_BEGIN(ctx)
    // invert_mesh (proj/src/invert.cpp:140-150)
    if (m_xi < 2 || m_eta < 2)
        fail(SDDG_ERR_VALIDATION, "invert_mesh: needs at least 2 target nodes per axis");
    check_domain(*dom);
    if (nx < 3 || ny < 3) fail(SDDG_ERR_VALIDATION, "GridSpec: needs nx >= 3 and ny >= 3");
    const size_t N = static_cast<size_t>(nx) * ny, M = static_cast<size_t>(m_xi) * m_eta;
    for (size_t k = 0; k < N; ++k)
        if (!std::isfinite(xi[k]) || !std::isfinite(eta[k]))
            fail(SDDG_ERR_EVALUATION, "ScalarField: non-finite value");
    cudaStream_t st = ctx->stream;
    double* din = static_cast<double*>(ctx->m_in.ensure(2 * N * sizeof(double)));
    double* dout = static_cast<double*>(ctx->m_out.ensure(2 * M * sizeof(double)));
    if (2.0 * (nx - 1.0) * (ny - 1.0) > 2147483647.0 || static_cast<double>(m_xi) * m_eta > 1073741823.0)
        fail(SDDG_ERR_VALIDATION, "invert_mesh: more than 2^31 forward triangles or 2^30 targets");
    // 16 ints of error words, then the kernels' scratch
    int* derr = static_cast<int*>(ctx->m_misc.ensure(sizeof(int) * (16 + invert_scratch_ints(m_xi, m_eta))));
    ck(cudaMemcpyAsync(din, xi, N * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    ck(cudaMemcpyAsync(din + N, eta, N * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    ck(cudaMemsetAsync(derr, 0, 4 * sizeof(int), st), "memset");
    const double ghx = (dom->xmax - dom->xmin) / (nx - 1), ghy = (dom->ymax - dom->ymin) / (ny - 1);
    ck(cudaEventRecord(ctx->ev0, st), "event");
    ck(launch_invert(din, din + N, nx, ny, dom->xmin, dom->ymin, ghx, ghy, m_xi, m_eta, dout,
                     dout + M, derr + 16, derr, derr + 1, st),
       "invert launch");
    ck(cudaEventRecord(ctx->ev1, st), "event");
    int herr[4] = {0, 0, 0, 0};
    ck(cudaMemcpyAsync(herr, derr, sizeof(herr), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(x, dout, M * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(y, dout + M, M * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "invert");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->last_ms = ms;
    ctx->last_launches = 5;
    // diagnostics of the fix-up pass: targets located again sequentially
    // (last_stats' step count) and rows it visited (the tail-handoff count)
    ctx->last_steps = herr[3];
    ctx->last_handoffs = herr[2];
    if (herr[0] == 8)
        fail(SDDG_ERR_INVERSION, "invert_mesh: a target in row " + std::to_string(herr[1]) +
                                     " is not covered by the forward tessellation");
    API_END(ctx)
}

sddg_status sddg_quality_report(sddg_ctx* ctx, const double* x, const double* y, int32_t m_xi,
                                int32_t m_eta, const double* ref_x, const double* ref_y,
                                const sddg_density* dens, sddg_quality* out) {
    API_BEGIN(ctx)
    if (m_xi < 2 || m_eta < 2) fail(SDDG_ERR_VALIDATION, "PhysicalMesh: needs at least 2 nodes per axis");
    if ((ref_x == nullptr) != (ref_y == nullptr))
        fail(SDDG_ERR_VALIDATION, "quality_report: reference mesh needs both x and y");
    const size_t M = static_cast<size_t>(m_xi) * m_eta;
    const long long cells = static_cast<long long>(m_xi - 1) * (m_eta - 1);
    cudaStream_t st = ctx->stream;
    double* dm = static_cast<double*>(ctx->m_in.ensure(4 * M * sizeof(double)));
    double* dq = static_cast<double*>(ctx->m_q.ensure(cells * sizeof(double)));
    char* misc = static_cast<char*>(ctx->m_misc.ensure(256));
    int* derr = reinterpret_cast<int*>(misc);
    double* dres = reinterpret_cast<double*>(misc + 64);
    unsigned long long* dl = reinterpret_cast<unsigned long long*>(misc + 128);
    ck(cudaMemcpyAsync(dm, x, M * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    ck(cudaMemcpyAsync(dm + M, y, M * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    if (ref_x) {
        ck(cudaMemcpyAsync(dm + 2 * M, ref_x, M * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpyAsync(dm + 3 * M, ref_y, M * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    }
    ck(cudaMemsetAsync(misc, 0, 256, st), "memset");
    ck(launch_quality(dm, dm + M, m_xi, m_eta, dq, dres, derr, st), "quality launch");
    int launches = 2;
    if (ref_x) {
        ck(launch_quality(dm + 2 * M, dm + 3 * M, m_xi, m_eta, dq, dres + 2, derr, st), "quality launch");
        launches += 2;
        if (dens) {
            drift_variant(*dens, SDDG_FP64);  // validates the kind
            ck(launch_linf(dm, dm + M, dm + 2 * M, dm + 3 * M, static_cast<long long>(M), dens->kind,
                           dens->R, dens->alpha, upload_density(ctx, *dens), dl, st),
               "linf launch");
            launches += 1;
        }
    }
    int herr = 0;
    double res[4] = {0, 0, 0, 0};
    unsigned long long lbits = 0;
    ck(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(res, dres, sizeof(res), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(&lbits, dl, sizeof(lbits), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "quality");
    ctx->last_launches = launches;
    if (herr == 9) fail(SDDG_ERR_TANGLING, "cell_quality: a cell is folded or degenerate (det J <= 0)");
    std::memset(out, 0, sizeof(*out));
    out->q_max = res[0];
    out->q_mean = res[1];
    if (ref_x) {
        out->has_reference = 1;
        out->r_max = res[2] / res[0];   // quality.cpp:64-65
        out->r_mean = res[3] / res[1];
        if (dens) {
            out->has_l_inf = 1;
            double l;
            std::memcpy(&l, &lbits, sizeof(l));
            out->l_inf = l;
        }
    }
    API_END(ctx)
}

sddg_status sddg_smooth_interface(sddg_ctx* ctx, const double* values, int32_t n, int32_t span,
                                  double* out) {
    API_BEGIN(ctx)
    const std::vector<double> r = smooth_line(ctx, std::vector<double>(values, values + n), span);
    std::memcpy(out, r.data(), sizeof(double) * n);
    API_END(ctx)
}

sddg_status sddg_perona_malik(sddg_ctx* ctx, double* xi, double* eta, int32_t nx, int32_t ny,
                              const sddg_domain* dom, const sddg_smooth_config* cfg, int32_t sx,
                              int32_t sy, int32_t* stability_warning) {
    API_BEGIN(ctx)
    // SmoothConfig::validate (smoothing.cpp:12-16)
    if (!(cfg->k > 0.0)) fail(SDDG_ERR_VALIDATION, "SmoothConfig: k must be > 0");
    if (!(cfg->dt > 0.0)) fail(SDDG_ERR_VALIDATION, "SmoothConfig: dt must be > 0");
    if (cfg->steps < 0) fail(SDDG_ERR_VALIDATION, "SmoothConfig: steps must be >= 0");
    check_domain(*dom);
    if (nx < 3 || ny < 3) fail(SDDG_ERR_VALIDATION, "GridSpec: needs nx >= 3 and ny >= 3");
    const double hx = (dom->xmax - dom->xmin) / (nx - 1), hy = (dom->ymax - dom->ymin) / (ny - 1);
    if (stability_warning) *stability_warning = cfg->dt > hx * hy / 4.0 ? 1 : 0;
    std::vector<int> blocks;
    if (cfg->scope == SDDG_SMOOTH_PER_SUBDOMAIN) {
        const Layout L = build_layout(*dom, nx, ny, sx, sy);
        for (int b = 0; b < sy; ++b)
            for (int a = 0; a < sx; ++a)
                blocks.insert(blocks.end(), {a * L.bx, b * L.by, L.bx + 1, L.by + 1});
    } else if (cfg->scope == SDDG_SMOOTH_GLOBAL) {
        blocks = {0, 0, nx, ny};
    } else {
        fail(SDDG_ERR_VALIDATION, "SmoothConfig: unknown scope");
    }
    if (cfg->steps == 0) API_RETURN_OK(ctx);
    const int nb = static_cast<int>(blocks.size() / 4);
    const size_t N = static_cast<size_t>(nx) * ny;
    cudaStream_t st = ctx->stream;
    double* du = static_cast<double*>(ctx->m_in.ensure(4 * N * sizeof(double)));
    const size_t scr = pm_scratch_doubles(blocks.data(), nb);
    double* dscr = static_cast<double*>(ctx->m_q.ensure(scr * sizeof(double)));
    unsigned long long* dupd = static_cast<unsigned long long*>(
        ctx->m_misc.ensure(sizeof(unsigned long long) * 2 * cfg->steps + 64));
    ck(cudaMemcpyAsync(du, xi, N * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    ck(cudaMemcpyAsync(du + N, eta, N * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    std::vector<double> upd(2 * cfg->steps);
    ck(pm_run(du, du + N, du + 2 * N, du + 3 * N, nx, ny, blocks.data(), nb, hx, hy, cfg->k, cfg->dt,
              cfg->steps, dscr, dupd, upd.data(), st),
       "perona-malik");
    // FTCS instability rule per field (smoothing.cpp:111-121)
    for (int f = 0; f < 2; ++f) {
        double prev = -1.0;
        for (int q = 0; q < cfg->steps; ++q) {
            const double u = upd[2 * q + f];
            if (prev >= 0.0 && u > 10.0 * prev && u > 1e-14)
                fail(SDDG_ERR_NUMERICAL, "perona_malik: FTCS unstable at dt=" + std::to_string(cfg->dt));
            prev = u;
        }
    }
    ck(cudaMemcpyAsync(xi, du, N * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(eta, du + N, N * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "d2h");
    ctx->last_launches = 2 * cfg->steps;
    API_END(ctx)
}

sddg_status sddg_laplacian_smooth(sddg_ctx* ctx, double* xi, double* eta, int32_t nx, int32_t ny,
                                  const sddg_domain* dom, int32_t sweeps) {
    if (!dom) {
        set_free_error("laplacian_smooth: domain is NULL");
        return SDDG_ERR_VALIDATION;
    }
    if (sweeps < 0) {
        if (ctx) ctx->err = "laplacian_smooth: sweeps must be >= 0";
        return SDDG_ERR_VALIDATION;
    }
    const double hx = (dom->xmax - dom->xmin) / (nx - 1), hy = (dom->ymax - dom->ymin) / (ny - 1);
    const sddg_smooth_config cfg{INFINITY, hx * hy / 4.0, sweeps, SDDG_SMOOTH_GLOBAL};
    return sddg_perona_malik(ctx, xi, eta, nx, ny, dom, &cfg, 1, 1, nullptr);
}

sddg_status sddg_stochastic_full(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                 int32_t nx, int32_t ny, const sddg_walk_config* cfg, double* xi,
                                 double* eta, sddg_sdd_stats* stats) {
    API_BEGIN(ctx)
    check_domain(*dom);
    if (nx < 3 || ny < 3) fail(SDDG_ERR_VALIDATION, "GridSpec: needs nx >= 3 and ny >= 3");
    const double t0 = now_s();
    const auto tabs = boundary_tables(*dens, *dom, nx, ny, SDDG_BC_REFERENCE);
    const sddg_boundary bd = make_boundary_view(*dom, nx, ny, tabs);
    const double hx = (dom->xmax - dom->xmin) / (nx - 1), hy = (dom->ymax - dom->ymin) / (ny - 1);
    for (int i = 0; i < nx; ++i) {
        xi[i] = tabs[0][i];
        xi[static_cast<size_t>(ny - 1) * nx + i] = tabs[1][i];
        eta[i] = tabs[4][i];
        eta[static_cast<size_t>(ny - 1) * nx + i] = tabs[5][i];
    }
    for (int j = 0; j < ny; ++j) {
        xi[static_cast<size_t>(j) * nx] = tabs[2][j];
        xi[static_cast<size_t>(j) * nx + nx - 1] = tabs[3][j];
        eta[static_cast<size_t>(j) * nx] = tabs[6][j];
        eta[static_cast<size_t>(j) * nx + nx - 1] = tabs[7][j];
    }
    const int64_t interior = static_cast<int64_t>(nx - 2) * (ny - 2);
    std::vector<double> px(interior), py(interior);
    std::vector<uint64_t> pid(interior);
    for (int64_t n = 0; n < interior; ++n) {
        const int i = 1 + static_cast<int>(n % (nx - 2)), j = 1 + static_cast<int>(n / (nx - 2));
        px[n] = dom->xmin + i * hx;
        py[n] = dom->ymin + j * hy;
        pid[n] = static_cast<uint64_t>(j) * nx + i;
    }
    std::vector<sddg_estimate> est(interior);
    estimates_host(ctx, *dens, *dom, bd, *cfg, px.data(), py.data(), pid.data(), interior, est.data());
    int64_t restarts = 0;
    for (int64_t n = 0; n < interior; ++n) {
        const size_t g = static_cast<size_t>(pid[n]);
        xi[g] = est[n].xi;
        eta[g] = est[n].eta;
        restarts += est[n].restarts;
    }
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->t_stoc = now_s() - t0;
        stats->mc_points = interior;
        stats->restarts = restarts;
        stats->path_steps = ctx->last_steps;
        stats->warnings = restarts > interior * cfg->walks / 100 ? 1 : 0;  // cli.cpp:266-268
    }
    API_END(ctx)
}

sddg_status sddg_write_mesh(const double* x, const double* y, int32_t m_xi, int32_t m_eta,
                            const double* xi, const double* eta, int32_t nx, int32_t ny,
                            const char* path) {
    try {
        if (nx != m_xi || ny != m_eta)
            fail(SDDG_ERR_VALIDATION, "write_mesh: solution grid " + std::to_string(nx) + "x" +
                                          std::to_string(ny) + " does not match mesh " +
                                          std::to_string(m_xi) + "x" + std::to_string(m_eta));
        auto f17 = [](double v) {
            char buf[40];
            std::snprintf(buf, sizeof(buf), "%.17g", v);
            return std::string(buf);
        };
        std::ostringstream os;
        os << "sddmesh v1 " << m_xi << " " << m_eta << "\n";
        for (int a = 0; a < m_xi; ++a)
            for (int b = 0; b < m_eta; ++b) {
                const size_t n = static_cast<size_t>(b) * m_xi + a;
                const size_t sidx = static_cast<size_t>(b) * nx + a;
                os << a << " " << b << " " << f17(x[n]) << " " << f17(y[n]) << " " << f17(xi[sidx])
                   << " " << f17(eta[sidx]) << "\n";
            }
        std::ofstream out(path, std::ios::binary);
        if (!out) fail(SDDG_ERR_INTERNAL, std::string("write_mesh: cannot open ") + path);
        out << os.str();
        if (!out) fail(SDDG_ERR_INTERNAL, std::string("write_mesh: write failed for ") + path);
    } catch (const Fail& f) {
        return finish(nullptr, f);
    }
    return SDDG_OK;
}

// ------------------------------------------------------------ fused gather

sddg_status sddg_gather_alloc(sddg_ctx* ctx, int64_t n_records, void** d_buf,
                              sddg_ipc_handle* handle) {
    API_BEGIN(ctx)
    if (n_records < 1) fail(SDDG_ERR_VALIDATION, "gather_alloc: n_records must be >= 1");
    void* p = nullptr;
    ck(cudaMalloc(&p, sizeof(sddg_estimate) * n_records), "cudaMalloc gather");
    ck(cudaMemset(p, 0, sizeof(sddg_estimate) * n_records), "memset gather");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        ck(e, "cudaIpcGetMemHandle");
    }
    static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(sddg_ipc_handle), "ipc handle size");
    std::memset(handle, 0, sizeof(*handle));
    std::memcpy(handle->bytes, &h, sizeof(h));
    *d_buf = p;
    API_END(ctx)
}

sddg_status sddg_gather_open(sddg_ctx* ctx, const sddg_ipc_handle* handle, void** d_peer) {
    API_BEGIN(ctx)
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle->bytes, sizeof(h));
    ck(cudaIpcOpenMemHandle(d_peer, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    API_END(ctx)
}

sddg_status sddg_gather_close(sddg_ctx* ctx, void* d_peer) {
    API_BEGIN(ctx)
    ck(cudaIpcCloseMemHandle(d_peer), "cudaIpcCloseMemHandle");
    API_END(ctx)
}

sddg_status sddg_gather_free(sddg_ctx* ctx, void* d_buf) {
    API_BEGIN(ctx)
    ck(cudaFree(d_buf), "cudaFree gather");
    API_END(ctx)
}

sddg_status sddg_gather_read(sddg_ctx* ctx, const void* d_buf, int64_t n_records,
                             sddg_estimate* out) {
    API_BEGIN(ctx)
    ck(cudaMemcpy(out, d_buf, sizeof(sddg_estimate) * n_records, cudaMemcpyDeviceToHost), "d2h gather");
    API_END(ctx)
}

sddg_status sddg_mc_estimate_gather(sddg_ctx* ctx, const sddg_density* dens, const sddg_domain* dom,
                                    const sddg_boundary* bd, const sddg_walk_config* cfg,
                                    const double* px, const double* py, const uint64_t* pid,
                                    const int64_t* global_index, int64_t n, void* const* peer_bufs,
                                    int32_t n_peers, int64_t n_total) {
    API_BEGIN(ctx)
    if (n_peers < 1 || n_peers > kMaxPeers)
        fail(SDDG_ERR_VALIDATION, "mc_estimate_gather: 1.." + std::to_string(kMaxPeers) + " peers");
    for (int64_t k = 0; k < n; ++k)
        if (global_index[k] < 0 || global_index[k] >= n_total)
            fail(SDDG_ERR_VALIDATION, "mc_estimate_gather: global index out of range");
    GatherTargets gt;
    gt.n_peers = n_peers;
    for (int p = 0; p < n_peers; ++p) gt.peers[p] = static_cast<sddg_estimate*>(peer_bufs[p]);
    int64_t* dgi = static_cast<int64_t*>(ctx->gidx.ensure(sizeof(int64_t) * std::max<int64_t>(1, n)));
    ck(cudaMemcpyAsync(dgi, global_index, sizeof(int64_t) * n, cudaMemcpyHostToDevice, ctx->stream), "h2d");
    gt.global_index = dgi;
    std::vector<sddg_estimate> local(n);
    estimates_host(ctx, *dens, *dom, *bd, *cfg, px, py, pid, n, local.data(), &gt);
    API_END(ctx)
}

}  // extern "C"
