// team.cu -- several GPUs behind one sddg_ctx: the multi-GPU form of the
// reference's two parallel_for regions (proj/src/decomposition.cpp:171-174
// over interface nodes, :298-355 over subdomains).
//
//  * Nodes are sharded by expected cost: every rank computes the same
//    longest-processing-time assignment from the exit-time model
//    (runtime.cu exit_time_model: the expected first-exit time of the walk,
//    div(w grad T) = -w), so no plan is communicated.
//  * Each rank walks its nodes (K1 + K2) and packs their 128-B records into
//    its slot of an rank-major exchange buffer; ONE ncclAllGather (in place)
//    then gives every rank every record, and a scatter kernel puts them at
//    their node index.  Each node is reduced on one rank in the reference's
//    chunk order, so records are bit-identical for any rank count.
//  * The subdomain phase splits the subdomains into contiguous per-rank
//    ranges; the fields are joined by a second all-gather.
//
// One process per GPU (sddg_create_dist, ncclCommInitRank) or one process
// for all of them (sddg_create_multi, one host thread per device).  In one
// process only the owner's buffer needs the records, so when every member
// device can store into the owner's memory (peer access over NVLink, or the
// same device) the exchange is fused into K2: reduce_kernel writes each
// finished record into the owner's output at its node index through peer
// memory (GatherTargets, reduce.cu) -- no pack, no collective, no scatter.
// Without peer access sddg_create_multi falls back to ncclCommInitAll and
// the all-gather (SDDG_TEAM_NCCL=1 forces it).  A device listed twice is
// driven as independent ranks (the sharded path on a single GPU, for tests):
// fused stores by default, device copies with SDDG_TEAM_COPY=1.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstddef>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <exception>
#include <numeric>
#include <set>
#include <thread>

#include "runtime_internal.h"

using namespace sddg;
using namespace sddg::rt;

namespace {

// NCCL is loaded at run time, the first time a multi-GPU context is made,
// and never linked: a process that already holds a libnccl.so.2 (PyTorch
// loads its bundled one) must keep using that copy, because a second copy
// of the same soname loaded first would shadow the one PyTorch needs.
// Order: an already-loaded libnccl.so.2; SDDG_NCCL_PATH (the Python mirror
// points it at PyTorch's bundled library); the system libnccl.so.2.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* env = std::getenv("SDDG_NCCL_PATH");
        if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p && api.error.empty()) api.error = std::string("libnccl.so.2 lacks ") + n;
            return p;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!api.error.empty()) fail(SDDG_ERR_CUDA, api.error);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(SDDG_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

__global__ void pack_kernel(const sddg_estimate* __restrict__ in, const int* __restrict__ nodes, int count,
                            int64_t n, sddg_estimate* __restrict__ out) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < count; s += gridDim.x * blockDim.x) {
        SDDG_CHECK(nodes[s] >= 0 && nodes[s] < n);
        out[s] = in[nodes[s]];
    }
    (void)n;
}

__global__ void unpack_kernel(const sddg_estimate* __restrict__ recv, const int* __restrict__ nodes, int slots,
                              int64_t n, sddg_estimate* __restrict__ out) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < slots; s += gridDim.x * blockDim.x) {
        const int k = nodes[s];
        SDDG_CHECK(k < n);
        if (k >= 0) out[k] = recv[s];
    }
    (void)n;
}

int blocks_for(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1024))); }

// Run f(m) for every local member m, one host thread each when there are
// several (each thread sets its member's device); rethrows the first failure.
template <typename F>
void for_members(const Team& T, F&& f) {
    const int nm = static_cast<int>(T.members.size());
    if (nm == 1) {
        f(0);
        return;
    }
    std::vector<std::exception_ptr> errs(nm);
    std::vector<std::thread> th;
    for (int m = 0; m < nm; ++m)
        th.emplace_back([&, m] {
            try {
                ck(cudaSetDevice(T.members[m]->device), "cudaSetDevice");
                f(m);
            } catch (...) {
                errs[m] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    ck(cudaSetDevice(T.members[0]->device), "cudaSetDevice");
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

}  // namespace

namespace sddg {
namespace rt {

// A one-rank communicator still takes the sharded path (one LPT shard, an
// all-gather over one rank), so the NCCL exchange runs on a single GPU too.
bool team_active(const sddg_ctx* c) {
    return c && c->team && (c->team->nranks > 1 || !c->team->comms.empty());
}

// Longest-processing-time assignment: nodes by descending cost (ties by
// index) each to the least-loaded rank (ties to the lowest rank).
std::vector<int> lpt_ranks(const std::vector<double>& cost, int nranks) {
    const std::vector<uint32_t> order = cost_order(cost, nullptr);
    std::vector<double> load(nranks, 0.0);
    std::vector<int> rank_of(cost.size(), 0);
    for (uint32_t k : order) {
        int best = 0;
        for (int r = 1; r < nranks; ++r)
            if (load[r] < load[best]) best = r;
        rank_of[k] = best;
        load[best] += cost[k];
    }
    return rank_of;
}

void team_estimates(sddg_ctx* c, const sddg_density& d, const sddg_domain& dom,
                    const sddg_boundary& bd, const sddg_walk_config& cfg, const double* d_px,
                    const double* d_py, const uint64_t* d_pid, int64_t n, sddg_estimate* d_out,
                    cudaStream_t st, const double* hpx, const double* hpy) {
    Team& T = *c->team;
    const int R = T.nranks;
    const std::vector<double> cost = node_costs(exit_time_model(c, d, dom), cfg, hpx, hpy, n);
    const std::vector<int> rank_of = lpt_ranks(cost, R);
    std::vector<std::vector<uint32_t>> lists(R);
    for (int64_t k = 0; k < n; ++k) lists[rank_of[k]].push_back(static_cast<uint32_t>(k));
    size_t maxc = 1;
    for (const auto& l : lists) maxc = std::max(maxc, l.size());
    std::vector<int> all_nodes(static_cast<size_t>(R) * maxc, -1);
    for (int r = 0; r < R; ++r)
        for (size_t i = 0; i < lists[r].size(); ++i) all_nodes[r * maxc + i] = static_cast<int>(lists[r][i]);
    const size_t rec = sizeof(sddg_estimate);
    const int nm = static_cast<int>(T.members.size());
    if (T.fused) {
        // K2 fused with the gather: member m reduces its nodes and stores each
        // record at d_out[node] on the owner's device (member 0 does so
        // anyway).  run_estimates ends with a stream synchronise, so every
        // peer store has landed when for_members returns.
        std::vector<double> fms(nm, 0.0);
        std::vector<int64_t> fl(nm, 0);
        // the records land in a buffer of the library's own on the owner's
        // device (peer access covers it whatever allocator the caller's d_out
        // comes from); one small device copy then fills d_out
        sddg_estimate* gathered = static_cast<sddg_estimate*>(c->t_recv.ensure(rec * std::max<int64_t>(n, 1)));
        for_members(T, [&](int m) {
            sddg_ctx* mc = T.members[m];
            const int r = T.rank0 + m;
            cudaStream_t ms_ = m == 0 ? st : mc->stream;
            const double* px = d_px;
            const double* py = d_py;
            const uint64_t* pid = d_pid;
            sddg_estimate* out = gathered;
            GatherTargets gt;
            gt.n_peers = 0;
            gt.global_index = nullptr;
            if (m > 0) {
                char* b = static_cast<char*>(mc->t_pts.ensure(n * (2 * sizeof(double) + sizeof(uint64_t))));
                ck(cudaMemcpyPeerAsync(b, mc->device, d_px, c->device, n * sizeof(double), ms_), "peer copy");
                ck(cudaMemcpyPeerAsync(b + n * sizeof(double), mc->device, d_py, c->device, n * sizeof(double), ms_),
                   "peer copy");
                ck(cudaMemcpyPeerAsync(b + 2 * n * sizeof(double), mc->device, d_pid, c->device,
                                       n * sizeof(uint64_t), ms_),
                   "peer copy");
                px = reinterpret_cast<const double*>(b);
                py = px + n;
                pid = reinterpret_cast<const uint64_t*>(py + n);
                out = static_cast<sddg_estimate*>(mc->est.ensure(rec * n));
                gt.n_peers = 1;
                gt.peers[0] = gathered;  // the owner's records, through peer memory
            }
            const std::vector<uint32_t> order = cost_order(cost, &lists[r]);
            run_estimates(mc, d, dom, bd, cfg, px, py, pid, n, order, out, ms_, gt.n_peers ? &gt : nullptr);
            fms[m] = mc->last_ms;
            fl[m] = mc->last_launches;
        });
        ck(cudaMemcpyAsync(d_out, gathered, rec * n, cudaMemcpyDeviceToDevice, st), "records to the caller");
        std::vector<int64_t> steps(n);
        ck(cudaMemcpy2DAsync(steps.data(), sizeof(int64_t),
                             reinterpret_cast<const char*>(gathered) + offsetof(sddg_estimate, path_steps), rec,
                             sizeof(int64_t), n, cudaMemcpyDeviceToHost, st),
           "d2h path steps");
        ck(cudaStreamSynchronize(st), "team estimates");
        c->last_steps = std::accumulate(steps.begin(), steps.end(), int64_t(0));
        c->last_ms = *std::max_element(fms.begin(), fms.end());
        c->last_launches = std::accumulate(fl.begin(), fl.end(), int64_t(0));
        return;
    }
    std::vector<sddg_estimate*> recv(nm);
    std::vector<cudaStream_t> streams(nm);
    std::vector<double> ms(nm, 0.0);
    std::vector<int64_t> launches(nm, 0);
    // 1. every local rank walks its nodes and packs their records
    for_members(T, [&](int m) {
        sddg_ctx* mc = T.members[m];
        const int r = T.rank0 + m;
        cudaStream_t ms_ = m == 0 ? st : mc->stream;
        streams[m] = ms_;
        const double* px = d_px;
        const double* py = d_py;
        const uint64_t* pid = d_pid;
        sddg_estimate* out = d_out;
        if (m > 0) {  // the points live on the owner's device: copy them over
            char* b = static_cast<char*>(mc->t_pts.ensure(n * (2 * sizeof(double) + sizeof(uint64_t))));
            ck(cudaMemcpyPeerAsync(b, mc->device, d_px, c->device, n * sizeof(double), ms_), "peer copy");
            ck(cudaMemcpyPeerAsync(b + n * sizeof(double), mc->device, d_py, c->device, n * sizeof(double), ms_),
               "peer copy");
            ck(cudaMemcpyPeerAsync(b + 2 * n * sizeof(double), mc->device, d_pid, c->device, n * sizeof(uint64_t),
                                   ms_),
               "peer copy");
            px = reinterpret_cast<const double*>(b);
            py = px + n;
            pid = reinterpret_cast<const uint64_t*>(py + n);
            out = static_cast<sddg_estimate*>(mc->est.ensure(rec * n));
        }
        recv[m] = static_cast<sddg_estimate*>(mc->t_recv.ensure(rec * R * maxc));
        int* dn = static_cast<int*>(mc->t_nodes.ensure(sizeof(int) * R * maxc));
        ck(cudaMemcpyAsync(dn, all_nodes.data(), sizeof(int) * R * maxc, cudaMemcpyHostToDevice, ms_), "h2d nodes");
        const std::vector<uint32_t> order = cost_order(cost, &lists[r]);
        run_estimates(mc, d, dom, bd, cfg, px, py, pid, n, order, out, ms_);
        ms[m] = mc->last_ms;
        launches[m] = mc->last_launches;
        const int cnt = static_cast<int>(lists[r].size());
        if (cnt > 0) {
            pack_kernel<<<blocks_for(cnt), 256, 0, ms_>>>(out, dn + r * maxc, cnt, n, recv[m] + r * maxc);
            ck(cudaGetLastError(), "pack launch");
        }
    });
    // 2. the one collective: every rank's records to every rank
    if (!T.comms.empty()) {
        nck(nccl().GroupStart(), "ncclGroupStart");
        for (int m = 0; m < nm; ++m) {
            const int r = T.rank0 + m;
            nck(nccl().AllGather(recv[m] + r * maxc, recv[m], rec * maxc, ncclUint8, T.comms[m], streams[m]),
                "ncclAllGather");
        }
        nck(nccl().GroupEnd(), "ncclGroupEnd");
    } else {  // all ranks local (duplicate devices): copy into the owner's buffer
        for (int m = 0; m < nm; ++m) ck(cudaStreamSynchronize(streams[m]), "member sync");
        for (int m = 1; m < nm; ++m) {
            const int r = T.rank0 + m;
            ck(cudaMemcpyPeerAsync(recv[0] + r * maxc, c->device, recv[m] + r * maxc, T.members[m]->device,
                                   rec * lists[r].size(), st),
               "peer copy records");
        }
    }
    for (int m = 1; m < nm; ++m) ck(cudaStreamSynchronize(streams[m]), "member sync");
    // 3. records to their node slots on the owner's device
    unpack_kernel<<<blocks_for(R * maxc), 256, 0, st>>>(recv[0], static_cast<int*>(c->t_nodes.p),
                                                         static_cast<int>(R * maxc), n, d_out);
    ck(cudaGetLastError(), "unpack launch");
    std::vector<int64_t> steps(n);
    ck(cudaMemcpy2DAsync(steps.data(), sizeof(int64_t), reinterpret_cast<const char*>(d_out) +
                                                            offsetof(sddg_estimate, path_steps),
                         rec, sizeof(int64_t), n, cudaMemcpyDeviceToHost, st),
       "d2h path steps");
    ck(cudaStreamSynchronize(st), "team estimates");
    c->last_steps = std::accumulate(steps.begin(), steps.end(), int64_t(0));
    c->last_ms = *std::max_element(ms.begin(), ms.end());
    c->last_launches = std::accumulate(launches.begin(), launches.end(), int64_t(0)) + nm + 1;
}

void team_solve_batch(sddg_ctx* c, const double* w, int gnx, int gny, double hx, double hy,
                      int64_t n_jobs, int jobs_per_sub, const sddg_subdomain* subs, const double* bc,
                      const sddg_solver_config& sc, double* u, sddg_solve_info* info) {
    Team& T = *c->team;
    const int R = T.nranks;
    const int64_t n_sub = n_jobs / jobs_per_sub;
    // contiguous ranges of whole subdomains; job offsets into bc and u
    std::vector<int64_t> lo(R + 1), boff(n_jobs + 1, 0), uoff(n_jobs + 1, 0);
    for (int r = 0; r <= R; ++r) lo[r] = (n_sub * r / R) * jobs_per_sub;
    for (int64_t j = 0; j < n_jobs; ++j) {
        boff[j + 1] = boff[j] + 2 * (subs[j].nx + subs[j].ny);
        uoff[j + 1] = uoff[j] + static_cast<int64_t>(subs[j].nx) * subs[j].ny;
    }
    int64_t max_u = 1, max_j = 1;
    for (int r = 0; r < R; ++r) {
        max_u = std::max(max_u, uoff[lo[r + 1]] - uoff[lo[r]]);
        max_j = std::max(max_j, lo[r + 1] - lo[r]);
    }
    const int nm = static_cast<int>(T.members.size());
    for_members(T, [&](int m) {
        const int r = T.rank0 + m;
        const int64_t a = lo[r], b = lo[r + 1];
        solve_batch_host(T.members[m], w, gnx, gny, hx, hy, b - a, subs + a, bc + boff[a], sc, u + uoff[a],
                         info + a);
    });
    c->last_launches = 0;
    if (T.comms.empty() || nm == R) return;  // every range solved in this process
    // one process per GPU: all-gather the ranges (u then info per rank slot)
    const size_t slot = sizeof(double) * max_u + sizeof(sddg_solve_info) * max_j;
    char* dbuf = static_cast<char*>(c->t_recv.ensure(slot * R));
    const int r = T.rank0;
    ck(cudaMemcpyAsync(dbuf + r * slot, u + uoff[lo[r]], sizeof(double) * (uoff[lo[r + 1]] - uoff[lo[r]]),
                       cudaMemcpyHostToDevice, c->stream),
       "h2d fields");
    ck(cudaMemcpyAsync(dbuf + r * slot + sizeof(double) * max_u, info + lo[r],
                       sizeof(sddg_solve_info) * (lo[r + 1] - lo[r]), cudaMemcpyHostToDevice, c->stream),
       "h2d info");
    nck(nccl().AllGather(dbuf + r * slot, dbuf, slot, ncclUint8, T.comms[0], c->stream), "ncclAllGather fields");
    std::vector<char> h(slot * R);
    ck(cudaMemcpyAsync(h.data(), dbuf, slot * R, cudaMemcpyDeviceToHost, c->stream), "d2h fields");
    ck(cudaStreamSynchronize(c->stream), "fields gather");
    for (int q = 0; q < R; ++q) {
        if (q == r) continue;
        std::memcpy(u + uoff[lo[q]], h.data() + q * slot, sizeof(double) * (uoff[lo[q + 1]] - uoff[lo[q]]));
        std::memcpy(info + lo[q], h.data() + q * slot + sizeof(double) * max_u,
                    sizeof(sddg_solve_info) * (lo[q + 1] - lo[q]));
    }
    c->last_launches = 1;
}

void team_destroy(sddg_ctx* c) {
    Team* T = c->team;
    if (!T) return;
    c->team = nullptr;
    for (size_t m = 0; m < T->comms.size(); ++m) {
        cudaSetDevice(T->members[m]->device);
        nccl().CommDestroy(T->comms[m]);
    }
    for (size_t m = 1; m < T->members.size(); ++m) sddg_destroy(T->members[m]);
    delete T;
}

}  // namespace rt
}  // namespace sddg

namespace {
sddg_status team_fail(const Fail& f) {
    set_free_error(f.msg);
    return f.st;
}
}  // namespace

extern "C" {

sddg_status sddg_nccl_unique_id(sddg_nccl_id* id) {
    try {
        static_assert(sizeof(ncclUniqueId) == sizeof(sddg_nccl_id), "nccl id size");
        ncclUniqueId u;
        nck(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id->bytes, &u, sizeof(u));
    } catch (const Fail& f) {
        return team_fail(f);
    }
    return SDDG_OK;
}

sddg_status sddg_create_dist(int32_t device, int32_t rank, int32_t nranks, const sddg_nccl_id* id,
                             sddg_ctx** out) {
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks || !id) {
        set_free_error("create_dist: needs 0 <= rank < nranks and an id");
        return SDDG_ERR_VALIDATION;
    }
    sddg_ctx* c = nullptr;
    const sddg_status s = sddg_create(device, &c);
    if (s != SDDG_OK) return s;
    try {
        ncclUniqueId u;
        std::memcpy(&u, id->bytes, sizeof(u));
        ncclComm_t comm;
        ck(cudaSetDevice(device), "cudaSetDevice");
        nck(nccl().CommInitRank(&comm, nranks, u, rank), "ncclCommInitRank");
        c->team = new Team{nranks, rank, {c}, {comm}};
    } catch (const Fail& f) {
        sddg_destroy(c);
        return team_fail(f);
    }
    *out = c;
    return SDDG_OK;
}

sddg_status sddg_create_multi(int32_t n, const int32_t* devices, sddg_ctx** out) {
    *out = nullptr;
    if (n < 1 || !devices) {
        set_free_error("create_multi: needs n >= 1 devices");
        return SDDG_ERR_VALIDATION;
    }
    std::vector<sddg_ctx*> members;
    for (int m = 0; m < n; ++m) {
        sddg_ctx* c = nullptr;
        const sddg_status s = sddg_create(devices[m], &c);
        if (s != SDDG_OK) {
            for (sddg_ctx* q : members) sddg_destroy(q);
            return s;
        }
        members.push_back(c);
    }
    try {
        const std::set<int32_t> distinct(devices, devices + n);
        std::vector<ncclComm_t> comms;
        // can every member store into the owner's (devices[0]) memory?
        bool peer_ok = true;
        for (int m = 1; m < n; ++m) {
            int ok = devices[m] == devices[0] ? 1 : 0;
            if (!ok) cudaDeviceCanAccessPeer(&ok, devices[m], devices[0]);
            peer_ok = peer_ok && ok;
        }
        const char* force_nccl = std::getenv("SDDG_TEAM_NCCL");
        const char* force_copy = std::getenv("SDDG_TEAM_COPY");
        const bool all_distinct = static_cast<int32_t>(distinct.size()) == n;
        const bool fused = n > 1 && peer_ok && !(force_nccl && *force_nccl == '1' && all_distinct) &&
                           !(force_copy && *force_copy == '1' && !all_distinct);
        if (n > 1 && all_distinct && !fused) {
            comms.resize(n);
            nck(nccl().CommInitAll(comms.data(), n, devices), "ncclCommInitAll");
        }
        if (n > 1) {
            // peer access for the point copies and the copy exchange
            for (int a = 0; a < n; ++a)
                for (int b = 0; b < n; ++b) {
                    if (devices[a] == devices[b]) continue;
                    int ok = 0;
                    cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]);
                    if (!ok) continue;
                    cudaSetDevice(devices[a]);
                    const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "peer access");
                    cudaGetLastError();
                }
            ck(cudaSetDevice(devices[0]), "cudaSetDevice");
        }
        members[0]->team = new Team{n, 0, members, comms, fused};
    } catch (const Fail& f) {
        for (sddg_ctx* q : members) sddg_destroy(q);
        return team_fail(f);
    }
    *out = members[0];
    return SDDG_OK;
}

sddg_status sddg_team_info(const sddg_ctx* ctx, int32_t* rank, int32_t* nranks, int32_t* local_devices,
                           int32_t* nccl) {
    if (!ctx) return SDDG_ERR_VALIDATION;
    const Team* T = ctx->team;
    if (rank) *rank = T ? T->rank0 : 0;
    if (nranks) *nranks = T ? T->nranks : 1;
    if (local_devices) *local_devices = T ? static_cast<int32_t>(T->members.size()) : 1;
    if (nccl) *nccl = (T && !T->comms.empty()) ? 1 : 0;
    return SDDG_OK;
}

sddg_status sddg_shard_plan(const sddg_density* dens, const sddg_domain* dom, const sddg_walk_config* cfg,
                            const double* px, const double* py, int64_t n, int32_t nranks, int32_t* rank_of,
                            double* cost) {
    try {
        check_domain(*dom);
        validate_walk(*cfg);
        walk_variant(*dens, *cfg);
        if (nranks < 1) fail(SDDG_ERR_VALIDATION, "shard_plan: nranks must be >= 1");
        check_points(*dom, px, py, n);
        sddg_ctx scratch;  // host-only: the model cache of a throwaway context
        const std::vector<double> cst = node_costs(exit_time_model(&scratch, *dens, *dom), *cfg, px, py, n);
        const std::vector<int> r = lpt_ranks(cst, nranks);
        for (int64_t k = 0; k < n; ++k) {
            if (rank_of) rank_of[k] = r[k];
            if (cost) cost[k] = cst[k];
        }
    } catch (const Fail& f) {
        return team_fail(f);
    }
    return SDDG_OK;
}

}  // extern "C"
