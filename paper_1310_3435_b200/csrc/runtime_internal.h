// runtime_internal.h -- the context object behind include/sddg.h and the
// host-runtime helpers shared by runtime.cu (single device) and team.cu
// (several devices: node and subdomain sharding, NCCL all-gathers).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>  // types only: the library is loaded at run time (team.cu)

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "host_density.h"
#include "sddg_internal.h"

namespace sddg {
namespace rt {

struct Fail {
    sddg_status st;
    std::string msg;
};

[[noreturn]] inline void fail(sddg_status st, const std::string& m) { throw Fail{st, m}; }

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SDDG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

inline double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// Grow-only device buffer (allocation on the context's device).
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* ensure(size_t bytes) {
        if (bytes <= cap) return p;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        ck(cudaMalloc(&p, want), "cudaMalloc");
        cap = want;
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

constexpr int kMaxDrain = 4;  // drain rounds between K1 and the tail kernel
// The stages after K1 of a small fp64 batch (runtime.cu enable_tail): handoff
// caps (total walks) and buffers of K1 (0), the drain rounds (1..rounds) and
// the tail kernel's input (rounds)
struct DrainPlan {
    int rounds = 0;
    uint32_t cap[kMaxDrain + 1] = {};
    struct WalkCont* buf[kMaxDrain + 1] = {};
};
struct Counters {
    unsigned long long next, steps, err_info;
    int err_flag;
    unsigned int n_cont;     // walks handed over by K1
    unsigned long long live;  // walks in flight once the batch counter has run out
    unsigned int n_drain[kMaxDrain];  // walks handed over by drain round r
};

// Expected first-exit time T(x) of the walk dX = grad(w)/w dt + sqrt(2) dW
// (the reference's SDE, sde.cpp:21-29: generator (1/w) div(w grad)), i.e.
// div(w grad T) = -w in the domain, T = 0 on its edges, on a coarse grid.
// A node's expected walk cost is T / dt steps (linear scheme) or T lambda
// (exponential scheme).  Used to order nodes longest-first inside a launch
// and to balance node shards across GPUs.
struct ExitTimeModel {
    int g = 0;
    double x0 = 0, y0 = 0, hx = 1, hy = 1;
    std::vector<double> t;  // g x g, index j*g + i
    double at(double x, double y) const;
};

}  // namespace rt
}  // namespace sddg

struct Team;

struct sddg_ctx {
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::string err;
    std::mutex mu;
    sddg::rt::DevBuf rec_f, rec_g, rec_meta, nodes, est, tables, counters, dump, perm, nsteps;
    sddg::rt::DevBuf s_w, s_jobs, s_bc, s_u, s_info, s_coef, s_err, s_large, s_omega, s_perm;
    sddg::rt::DevBuf m_in, m_out, m_q, m_misc;
    int64_t last_steps = 0, last_launches = 0, last_handoffs = 0;
    double last_ms = 0.0, last_tail_ms = 0.0;
    std::map<int, std::pair<int, int>> occ;  // (dv*2+prec) -> (CTAs per SM, threads per CTA)
    std::vector<cudaEvent_t> bev;  // per-batch walk-kernel events
    sddg::rt::DevBuf fm_tables;    // fastmath.cuh FmTables (performance mode)
    sddg::rt::DevBuf gidx;         // fused-gather global indices
    // exit-time cost models by density/domain (host, cached)
    std::map<std::string, sddg::rt::ExitTimeModel> cost_models;
    // several GPUs (team.cu): null for a single-device context
    Team* team = nullptr;
    sddg::rt::DevBuf t_recv, t_nodes, t_pts;  // team exchange buffers on this device
    sddg::rt::DevBuf dens_tab;                // padded samples of a tabulated density
    sddg::rt::DevBuf tail_cont;               // walks handed from K1 to the tail kernel
};

namespace sddg {
namespace rt {

// validation (runtime.cu)
void validate_walk(const sddg_walk_config& c);
int drift_variant(const sddg_density& d, int precision);
int walk_variant(const sddg_density& d, const sddg_walk_config& cfg);
HostDensity host_density(const sddg_density& d);
void check_positivity(const sddg_density& d, const sddg_domain& dom);
void check_domain(const sddg_domain& d);
void check_boundary(const sddg_boundary& b);
void check_points(const sddg_domain& dom, const double* px, const double* py, int64_t n);

// the exit-time model of (density, domain), cached on the context
const ExitTimeModel& exit_time_model(sddg_ctx* c, const sddg_density& d, const sddg_domain& dom);
// expected path-steps of each node's cfg.walks walks
std::vector<double> node_costs(const ExitTimeModel& m, const sddg_walk_config& cfg, const double* px,
                               const double* py, int64_t n);
// nodes by descending cost, ties by index (launch order)
std::vector<uint32_t> cost_order(const std::vector<double>& cost, const std::vector<uint32_t>* subset);

// K1 + K2 for the nodes `order` (indices into the n device-resident points,
// in launch order); the record of node k lands at d_out[k].
void run_estimates(sddg_ctx* c, const sddg_density& d, const sddg_domain& dom,
                   const sddg_boundary& bd, const sddg_walk_config& cfg, const double* d_px,
                   const double* d_py, const uint64_t* d_pid, int64_t n,
                   const std::vector<uint32_t>& order, sddg_estimate* d_out, cudaStream_t st,
                   const GatherTargets* gt = nullptr);

// subdomain solves (K3/K3c/K3b) of one batch; u and info on the host
void solve_batch_host(sddg_ctx* c, const double* w, int gnx, int gny, double hx, double hy,
                      int64_t n, const sddg_subdomain* subs, const double* bc,
                      const sddg_solver_config& sc, double* u, sddg_solve_info* info);

}  // namespace rt
}  // namespace sddg

// A context spanning several GPUs (team.cu).  Global ranks 0..nranks-1; this
// process drives members[0..] as ranks rank0, rank0+1, ...  One process per
// GPU (sddg_create_dist): one member, an NCCL communicator over all ranks.
// One process for all GPUs (sddg_create_multi): one member per device, one
// communicator per member from ncclCommInitAll; a device listed twice has no
// NCCL (the exchange is a device-to-device copy).
struct Team {
    int nranks = 1;
    int rank0 = 0;
    std::vector<sddg_ctx*> members;  // members[0] is the owning context itself
    std::vector<ncclComm_t> comms;   // one per member, or empty (peer-store or copy exchange)
    // one process, every member's device can store into the owner's memory
    // (the same device, or peer access over NVLink): each member's K2 writes
    // its finished records straight into the owner's output at their node
    // index -- the reduce and the gather are one kernel, no NCCL call
    bool fused = false;
};

namespace sddg {
namespace rt {

bool team_active(const sddg_ctx* c);
// message of the last failure of a call without a context (sddg_last_error(NULL))
void set_free_error(const std::string& m);
// sharded sddg_mc_estimate_batch(_device): d_out (n records, the owner's
// device) receives every node's record on every rank
void team_estimates(sddg_ctx* c, const sddg_density& d, const sddg_domain& dom,
                    const sddg_boundary& bd, const sddg_walk_config& cfg, const double* d_px,
                    const double* d_py, const uint64_t* d_pid, int64_t n, sddg_estimate* d_out,
                    cudaStream_t st, const double* hpx, const double* hpy);
// sharded subdomain phase: jobs [0, n_jobs) split into contiguous per-rank
// ranges of whole subdomains (jobs_per_sub jobs each); u and info complete
// on every rank
void team_solve_batch(sddg_ctx* c, const double* w, int gnx, int gny, double hx, double hy,
                      int64_t n_jobs, int jobs_per_sub, const sddg_subdomain* subs, const double* bc,
                      const sddg_solver_config& sc, double* u, sddg_solve_info* info);
void team_destroy(sddg_ctx* c);

}  // namespace rt
}  // namespace sddg
