// mesh.cu -- K4 mesh inversion and K5 quality statistics on the GPU.
//
// Reference: invert_mesh (proj/src/invert.cpp:13-196) and cell_quality /
// quality_report (proj/src/quality.cpp:8-80).  Built with -fmad=false; every
// expression keeps the reference's operation order, so the physical mesh and
// the statistics are bit-identical to the reference's (rho for l_inf uses the
// CUDA libm, ~1 ulp).
//
// K4.  The reference locates each target (xi_a, eta_b) in the forward
// tessellation by a walk that starts from the triangle of the previous target
// of the row (the hint), which makes a row sequential -- and the hint matters:
// a target within the walk tolerance of an edge, or inside several triangles
// of a folded mesh, lands in whichever triangle the walk meets first.  Here
// every target is located in parallel, and the reference's result is
// reproduced by construction rather than by assuming the hint never matters:
//   1. candidates: a containing triangle per target, found in three sweeps of
//      short walks -- a coarse lattice of targets from the uniform-mesh guess,
//      the lattice columns upwards from the lattice targets, then every row
//      in blocks of 16 targets from its column candidate (each target from
//      its predecessor's triangle: one or two triangles per target);
//   2. chain: one thread per target runs the reference's location (walk from
//      the hint, then the two exhaustive scans) with the CANDIDATE of the
//      previous target as the hint (target 0: the reference's own seed), and
//      interpolates.  If every candidate of a row equals its chain result,
//      induction over a gives: hint = candidate(a-1) = result(a-1), so each
//      chain result is the reference's -- for any mesh, folded or not;
//   3. fix-up: rows where some candidate differs from its chain result (a
//      target on an edge, a folded cell, a failed candidate walk): a warp
//      scans the row, and from each difference on one lane follows the
//      reference's sequence until it meets the candidates again; only this
//      pass raises the reference's errors.
// K5: one thread per cell computes Q = tr(J^T J) / (2 det J) and flags folded
// cells; the sum for q_mean is then taken in a fixed two-level order (see
// quality_fold), the maxima are order-free.
#include <cfloat>

#include "density.cuh"
#include "sddg_internal.h"

namespace sddg {

namespace {

// The forward tessellation (invert.cpp:13-79): cell (i, j) of the (nx-1) x
// (ny-1) cell grid is split along its (i,j)-(i+1,j+1) diagonal into triangle
// 2c (lower right: (i,j), (i+1,j), (i+1,j+1)) and 2c+1 (upper left: (i,j),
// (i+1,j+1), (i,j+1)), c = j (nx-1) + i.  Triangles are ints: the host rejects
// grids with more than 2^31 triangles.
struct Forward {
    const double* __restrict__ xi;
    const double* __restrict__ eta;
    int nx, ny;

    __device__ __forceinline__ int cells_x() const { return nx - 1; }
    __device__ __forceinline__ int triangles() const { return 2 * (nx - 1) * (ny - 1); }
    // node indices (i, j) of the three corners of triangle t
    __device__ __forceinline__ void corners(int t, int ci[3], int cj[3]) const {
        const int c = t >> 1, upper = t & 1;
        const int i = c % cells_x(), j = c / cells_x();
        ci[0] = i;
        cj[0] = j;
        ci[1] = i + 1;
        cj[1] = j + upper;
        ci[2] = i + 1 - upper;
        cj[2] = j + 1;
    }
    // the triangle across the edge opposite corner k, or -1 at the boundary
    __device__ __forceinline__ int across(int t, int k) const {
        const int c = t >> 1, upper = t & 1;
        int i = c % cells_x(), j = c / cells_x();
        int other;  // the neighbour's half
        if (!upper) {
            other = 1;
            if (k == 0) ++i;        // right cell's upper triangle
            else if (k == 2) --j;   // lower cell's upper triangle (k == 1: this cell's)
        } else {
            other = 0;
            if (k == 0) ++j;        // upper cell's lower triangle
            else if (k == 1) --i;   // left cell's lower triangle (k == 2: this cell's)
        }
        if (i < 0 || j < 0 || i >= cells_x() || j >= ny - 1) return -1;
        return 2 * (j * cells_x() + i) + other;
    }
};

// barycentric coordinates of p in triangle t (invert.cpp:81-111): weights
// a_k / det from the three sub-areas, `inside` with tolerance, and the corner
// with the smallest weight (the walk leaves through the opposite edge)
struct Weights {
    double w[3];
    double det;
    bool inside;
    int leave;  // -1: degenerate triangle
};

__device__ __forceinline__ double area2(double ax, double ay, double bx, double by) {
    return ax * by - ay * bx;
}

__device__ Weights weights_in(const Forward& F, int t, double px, double py, double tol) {
    int ci[3], cj[3];
    F.corners(t, ci, cj);
    double vx[3], vy[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const size_t n = static_cast<size_t>(cj[k]) * F.nx + ci[k];
        vx[k] = F.xi[n];
        vy[k] = F.eta[n];
    }
    Weights r;
    r.det = area2(vx[1] - vx[0], vy[1] - vy[0], vx[2] - vx[0], vy[2] - vy[0]);
    if (r.det == 0.0) {
        r.inside = false;
        r.leave = -1;
        r.w[0] = r.w[1] = r.w[2] = 0.0;
        return r;
    }
    r.w[0] = area2(vx[1] - px, vy[1] - py, vx[2] - px, vy[2] - py) / r.det;
    r.w[1] = area2(vx[2] - px, vy[2] - py, vx[0] - px, vy[0] - py) / r.det;
    r.w[2] = area2(vx[0] - px, vy[0] - py, vx[1] - px, vy[1] - py) / r.det;
    r.inside = r.w[0] >= -tol && r.w[1] >= -tol && r.w[2] >= -tol;
    r.leave = 0;
    if (r.w[1] < r.w[r.leave]) r.leave = 1;
    if (r.w[2] < r.w[r.leave]) r.leave = 2;
    return r;
}

// visibility walk (invert.cpp:113-126): -1 when it meets a degenerate
// triangle, leaves the mesh, or exceeds 2 (nx + ny) + 16 steps
__device__ int walk_to(const Forward& F, int from, double px, double py, double tol) {
    int t = from;
    for (int step = 2 * (F.nx + F.ny) + 16; step > 0; --step) {
        const Weights r = weights_in(F, t, px, py, tol);
        if (r.inside) return t;
        if (r.leave < 0) return -1;
        t = F.across(t, r.leave);
        if (t < 0) return -1;
    }
    return -1;
}

// exhaustive scan (invert.cpp:128-138): the first containing triangle of
// positive area, else the first containing one
__device__ int scan_for(const Forward& F, double px, double py, double tol) {
    int folded = -1;
    for (int t = 0; t < F.triangles(); ++t) {
        const Weights r = weights_in(F, t, px, py, tol);
        if (!r.inside) continue;
        if (r.det > 0.0) return t;
        if (folded < 0) folded = t;
    }
    return folded;
}

constexpr double kWalkTol = 1e-12, kSnapTol = 1e-9;  // invert.cpp:152-153

// the reference's location of one target given its hint (invert.cpp:168-170)
__device__ int locate_like_reference(const Forward& F, int hint, double px, double py) {
    int t = walk_to(F, hint, px, py, kWalkTol);
    if (t < 0) t = scan_for(F, px, py, kWalkTol);
    if (t < 0) t = scan_for(F, px, py, kSnapTol);
    return t;
}

struct Targets {
    int m_xi, m_eta;
    double gx0, gy0, ghx, ghy;  // GridSpec::node of the physical grid
    __device__ __forceinline__ double xi_of(int a) const { return static_cast<double>(a) / (m_xi - 1); }
    __device__ __forceinline__ double eta_of(int b) const { return static_cast<double>(b) / (m_eta - 1); }
};

// the cell a near-uniform mesh would put the target in (invert.cpp:161-166)
__device__ __forceinline__ int uniform_seed(const Forward& F, double xi_a, double eta_b) {
    int ci = static_cast<int>(xi_a * (F.nx - 2));
    ci = ci < 0 ? 0 : (ci > F.nx - 2 ? F.nx - 2 : ci);
    int cj = static_cast<int>(eta_b * (F.ny - 2));
    cj = cj < 0 ? 0 : (cj > F.ny - 2 ? F.ny - 2 : cj);
    return 2 * (cj * (F.nx - 1) + ci);
}

// physical position of a target located in triangle t (invert.cpp:176-191);
// false for a degenerate triangle
__device__ __forceinline__ bool interpolate(const Forward& F, const Targets& G, int t, double px, double py,
                                            double& X, double& Y) {
    const Weights r = weights_in(F, t, px, py, kSnapTol);
    if (r.det == 0.0) return false;
    int ci[3], cj[3];
    F.corners(t, ci, cj);
    double x = 0.0, y = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        x += r.w[k] * (G.gx0 + ci[k] * G.ghx);
        y += r.w[k] * (G.gy0 + cj[k] * G.ghy);
    }
    X = x;
    Y = y;
    return true;
}

constexpr int kLattice = 16;  // candidate lattice spacing in targets

// K4 pass 1a: candidates of the lattice targets, from the uniform-mesh seed
__global__ void invert_lattice(Forward F, Targets G, int la, int lb, int* __restrict__ lat) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= la * lb) return;
    const int a = (q % la) * kLattice, b = (q / la) * kLattice;
    const double px = G.xi_of(a), py = G.eta_of(b);
    lat[q] = walk_to(F, uniform_seed(F, px, py), px, py, kWalkTol);
}

// K4 pass 1b: candidates down the lattice columns: one thread per lattice
// column and block of kLattice rows walks from the lattice target through the
// targets above it, each from its predecessor's triangle (one or two
// triangles per target instead of a long walk from a far seed)
__global__ void invert_columns(Forward F, Targets G, int la, int lb, const int* __restrict__ lat,
                               int* __restrict__ colc) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= la * lb) return;
    const int qa = q % la, qb = q / la;
    const int a = qa * kLattice;
    const double px = G.xi_of(a);
    int t = lat[q];
    const int b_end = min((qb + 1) * kLattice, G.m_eta);
    for (int b = qb * kLattice; b < b_end; ++b) {
        const double py = G.eta_of(b);
        t = walk_to(F, t >= 0 ? t : uniform_seed(F, px, py), px, py, kWalkTol);
        colc[b * la + qa] = t;
    }
}

// K4 pass 1c: candidates along the rows: one thread per row and block of
// kLattice targets, from the column candidate at the block's first target
__global__ void invert_candidates(Forward F, Targets G, int la, const int* __restrict__ colc,
                                  int* __restrict__ cand) {
    const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (q >= static_cast<long long>(la) * G.m_eta) return;
    const int qa = static_cast<int>(q % la), b = static_cast<int>(q / la);
    const double py = G.eta_of(b);
    int t = colc[q];
    const int a_end = min((qa + 1) * kLattice, G.m_xi);
    for (int a = qa * kLattice; a < a_end; ++a) {
        const double px = G.xi_of(a);
        t = walk_to(F, t >= 0 ? t : uniform_seed(F, px, py), px, py, kWalkTol);
        cand[static_cast<long long>(b) * G.m_xi + a] = t;
    }
}

// K4 pass 2: the reference's location with the previous target's candidate as
// the hint; the row is marked when a candidate and its chain result differ
// (or the location fails, or its triangle is degenerate).  res: the triangle,
// -1 not covered, -2 located in a degenerate triangle.
__global__ void invert_chain(Forward F, Targets G, const int* __restrict__ cand, int* __restrict__ res,
                             int* __restrict__ redo, double* __restrict__ X, double* __restrict__ Y) {
    const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (q >= static_cast<long long>(G.m_xi) * G.m_eta) return;
    const int a = static_cast<int>(q % G.m_xi), b = static_cast<int>(q / G.m_xi);
    const double px = G.xi_of(a), py = G.eta_of(b);
    const int hint = a == 0 ? uniform_seed(F, px, py) : cand[q - 1];
    int t = -1;
    if (hint >= 0) {
        t = locate_like_reference(F, hint, px, py);
        if (t >= 0 && !interpolate(F, G, t, px, py, X[q], Y[q])) t = -2;
    }
    res[q] = t;
    if (t != cand[q] || t < 0) redo[b] = 1;
}

// K4 pass 3: one warp per marked row.  The warp scans the row 32 targets at a
// time; a stretch whose chain results equal their candidates stands (the
// induction of the header).  From a difference on, lane 0 follows the
// reference's sequence (invert.cpp:154-193): a target whose predecessor's
// triangle equals the hint pass 2 assumed keeps its pass-2 result, any other
// is located again from the true predecessor -- until the sequence meets the
// candidates again.  Only this pass raises the reference's errors.
// stats[0]: rows marked, stats[1]: targets located again.
__global__ void invert_fixup(Forward F, Targets G, const int* __restrict__ cand, const int* __restrict__ res,
                             const int* __restrict__ redo, double* __restrict__ X, double* __restrict__ Y,
                             int* err, int* err_row, int* stats) {
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (b >= G.m_eta || !redo[b]) return;  // warp-uniform
    const double py = G.eta_of(b);
    const long long row = static_cast<long long>(b) * G.m_xi;
    int prev = -1;            // the reference's triangle of the target before the chunk
    int as_assumed = 1;       // ... equals the hint pass 2 used for the chunk's first target
    int relocated = 0;
    for (int a0 = 0; a0 < G.m_xi; a0 += 32) {
        const int a = a0 + lane;
        const bool in = a < G.m_xi;
        const int r = in ? res[row + a] : 0, c = in ? cand[row + a] : 0;
        const unsigned differ = __ballot_sync(0xffffffffu, in && (r != c || r < 0));
        if (as_assumed && differ == 0u) continue;  // the whole chunk stands, and so does the next hint
        int failed = 0;
        if (lane == 0) {
            const int n_in = min(32, G.m_xi - a0);
            // targets before the first difference stand; start there
            int j = as_assumed ? __ffs(differ) - 1 : 0;
            for (; j < n_in && !failed; ++j) {
                const long long q = row + a0 + j;
                int t;
                if (as_assumed) {
                    t = res[q];  // pass 2 had the right hint: its result, X and Y stand
                } else {
                    const double px = G.xi_of(a0 + j);
                    t = locate_like_reference(F, prev, px, py);
                    if (t >= 0 && !interpolate(F, G, t, px, py, X[q], Y[q])) t = -2;
                    ++relocated;
                }
                if (t < 0) {
                    failed = 1;  // InversionError: not covered, or a degenerate triangle
                    break;
                }
                prev = t;
                as_assumed = t == cand[q];
            }
        }
        failed = __shfl_sync(0xffffffffu, failed, 0);
        if (failed) {
            if (lane == 0) {
                atomicCAS(err, 0, 8);
                atomicExch(err_row, b);
            }
            return;
        }
        prev = __shfl_sync(0xffffffffu, prev, 0);
        as_assumed = __shfl_sync(0xffffffffu, as_assumed, 0);
    }
    if (lane == 0) {
        atomicAdd(stats, 1);
        atomicAdd(stats + 1, relocated);
    }
}

// cell_quality (proj/src/quality.cpp:8-33)
__global__ void quality_cells(const double* __restrict__ X, const double* __restrict__ Y, int m_xi,
                              int m_eta, double* __restrict__ q, int* err) {
    const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long cells = static_cast<long long>(m_xi - 1) * (m_eta - 1);
    if (c >= cells) return;
    const int a = static_cast<int>(c % (m_xi - 1)), b = static_cast<int>(c / (m_xi - 1));
    const double dxi = 1.0 / (m_xi - 1);
    const double deta = 1.0 / (m_eta - 1);
    auto at = [&](const double* A, int i, int j) { return A[static_cast<long long>(j) * m_xi + i]; };
    const double p00x = at(X, a, b), p00y = at(Y, a, b);
    const double p10x = at(X, a + 1, b), p10y = at(Y, a + 1, b);
    const double p01x = at(X, a, b + 1), p01y = at(Y, a, b + 1);
    const double p11x = at(X, a + 1, b + 1), p11y = at(Y, a + 1, b + 1);
    const double x_xi = 0.5 * ((p10x - p00x) + (p11x - p01x)) / dxi;
    const double y_xi = 0.5 * ((p10y - p00y) + (p11y - p01y)) / dxi;
    const double x_eta = 0.5 * ((p01x - p00x) + (p11x - p10x)) / deta;
    const double y_eta = 0.5 * ((p01y - p00y) + (p11y - p10y)) / deta;
    const double det = x_xi * y_eta - x_eta * y_xi;
    const double tr = x_xi * x_xi + y_xi * y_xi + x_eta * x_eta + y_eta * y_eta;
    if (!isfinite(det) || det <= 0.0) {
        atomicCAS(err, 0, 9);  // TanglingError
        q[c] = 0.0;
        return;
    }
    q[c] = 0.5 * tr / det;
}

// quality_report folds (proj/src/quality.cpp:44-53): the sum for q_mean and
// the maximum.  The reference adds the cells in row-major order; one thread
// doing the same takes 27 ms for a 1025^2 mesh (a million dependent adds), so
// the sum is taken in a fixed two-level order instead: thread t of one CTA adds
// cells t, t + 1024, ... in order, thread 0 adds the 1024 partial sums in
// order.  The result does not depend on scheduling, and differs from the
// row-major sum by the rounding of either (a few 1e-16 of q_mean on the test
// meshes, ~1e-14 at a million cells; the bar for quality statistics is 1e-6).
constexpr int kFoldThreads = 1024;

__global__ void __launch_bounds__(kFoldThreads) quality_fold(const double* __restrict__ q, long long cells,
                                                             double* out) {
    __shared__ double psum[kFoldThreads], pmax[kFoldThreads];
    double sum = 0.0, qmax = 0.0;
    for (long long c = threadIdx.x; c < cells; c += kFoldThreads) {
        const double v = q[c];
        sum += v;
        qmax = qmax < v ? v : qmax;
    }
    psum[threadIdx.x] = sum;
    pmax[threadIdx.x] = qmax;
    __syncthreads();
    if (threadIdx.x != 0) return;
    sum = 0.0;
    qmax = 0.0;
    for (int t = 0; t < kFoldThreads; ++t) {
        sum += psum[t];
        qmax = qmax < pmax[t] ? pmax[t] : qmax;
    }
    out[0] = qmax;
    out[1] = sum / static_cast<double>(cells);
}

__device__ double rho_any(int kind, double R, double al, const TableDensity& tab, double x, double y) {
    switch (kind) {
        case SDDG_DENS_CONSTANT: return R;
        case SDDG_DENS_RUNNING: {
            const double dx = x - 0.75, dy = y - 0.5;
            return 1.0 + R * exp(-50.0 * dx * dx - 50.0 * dy * dy - 0.5);
        }
        case SDDG_DENS_HUANG_SLOAN: {
            const double E = exp(R * (x - 1.0));
            const double S = sin(kPiD * y);
            const double C = cos(kPiD * y);
            const double q = al * (R * R * E * E * S * S + (1.0 - E) * (1.0 - E) * kPiD * kPiD * C * C);
            return sqrt(1.0 + q);
        }
        case SDDG_DENS_MACKENZIE: {
            const double s = y - 0.5 - 0.25 * sin(2.0 * kPiD * x);
            return 1.0 / (1.0 + al * exp(-R * s * s));
        }
        case SDDG_DENS_FIVE_RING: {
            double ux, uy, uxx, uxy, uyy;
            five_ring_velocity(x, y, R, ux, uy, uxx, uxy, uyy);
            return sqrt(1.0 + al * (ux * ux + uy * uy));
        }
        case SDDG_DENS_RING_W: return 1.0 / w_ring(x, y);
        case SDDG_DENS_SHOCK_W: return 1.0 / w_shock(x, y);
        case SDDG_DENS_TABLE: return table_rho(tab, x, y);
        default: return 1.0 / w_twobump(x, y);
    }
}

// l_inf of rho at the node positions (proj/src/quality.cpp:68-75): max is
// order-free; per-block max then atomic max on the (non-negative) bits.
__global__ void linf_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                            const double* __restrict__ RX, const double* __restrict__ RY,
                            long long n, int kind, double R, double al, const TableDensity tab,
                            unsigned long long* out_bits) {
    const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    double v = 0.0;
    if (k < n) {
        const double rr = rho_any(kind, R, al, tab, RX[k], RY[k]);
        const double rm = rho_any(kind, R, al, tab, X[k], Y[k]);
        v = fabs(rr - rm);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, v, o);
        v = v < u ? u : v;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace

size_t invert_scratch_ints(int m_xi, int m_eta) {
    const size_t la = (m_xi + kLattice - 1) / kLattice, lb = (m_eta + kLattice - 1) / kLattice;
    return la * lb + la * m_eta + 2 * static_cast<size_t>(m_xi) * m_eta + m_eta;
}

cudaError_t launch_invert(const double* xi, const double* eta, int nx, int ny, double gx0,
                          double gy0, double ghx, double ghy, int m_xi, int m_eta, double* X,
                          double* Y, int* scratch, int* err, int* err_row, cudaStream_t s) {
    const Forward F{xi, eta, nx, ny};
    const Targets G{m_xi, m_eta, gx0, gy0, ghx, ghy};
    const int la = (m_xi + kLattice - 1) / kLattice, lb = (m_eta + kLattice - 1) / kLattice;
    const long long M = static_cast<long long>(m_xi) * m_eta;
    int* lat = scratch;
    int* colc = lat + static_cast<size_t>(la) * lb;
    int* cand = colc + static_cast<size_t>(la) * m_eta;
    int* res = cand + M;
    int* redo = res + M;
    cudaError_t e = cudaMemsetAsync(redo, 0, sizeof(int) * m_eta, s);
    if (e != cudaSuccess) return e;
    const unsigned pts = static_cast<unsigned>((M + 127) / 128);
    const unsigned segs = static_cast<unsigned>((static_cast<long long>(la) * m_eta + 63) / 64);
    invert_lattice<<<(la * lb + 31) / 32, 32, 0, s>>>(F, G, la, lb, lat);
    invert_columns<<<(la * lb + 31) / 32, 32, 0, s>>>(F, G, la, lb, lat, colc);
    invert_candidates<<<segs, 64, 0, s>>>(F, G, la, colc, cand);
    invert_chain<<<pts, 128, 0, s>>>(F, G, cand, res, redo, X, Y);
    invert_fixup<<<(m_eta + 3) / 4, 128, 0, s>>>(F, G, cand, res, redo, X, Y, err, err_row, err + 2);
    return cudaGetLastError();
}

cudaError_t launch_quality(const double* X, const double* Y, int m_xi, int m_eta, double* qbuf,
                           double* out2, int* err, cudaStream_t s) {
    const long long cells = static_cast<long long>(m_xi - 1) * (m_eta - 1);
    quality_cells<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, s>>>(X, Y, m_xi, m_eta, qbuf,
                                                                             err);
    quality_fold<<<1, kFoldThreads, 0, s>>>(qbuf, cells, out2);
    return cudaGetLastError();
}

cudaError_t launch_linf(const double* X, const double* Y, const double* RX, const double* RY,
                        long long n, int kind, double R, double al, const TableDensity& tab,
                        unsigned long long* out_bits, cudaStream_t s) {
    linf_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(X, Y, RX, RY, n, kind, R, al, tab,
                                                                       out_bits);
    return cudaGetLastError();
}

}  // namespace sddg
