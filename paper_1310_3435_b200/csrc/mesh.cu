// mesh.cu -- K4 mesh inversion and K5 quality statistics on the GPU.
//
// Reference: invert_mesh (proj/src/invert.cpp:13-196) and cell_quality /
// quality_report (proj/src/quality.cpp:8-80).  Built with -fmad=false; every
// expression keeps the reference's operation order, so the physical mesh and
// the statistics are bit-identical to the reference's (rho for l_inf uses the
// CUDA libm, ~1 ulp).
//
// K4: one thread per target row b, walking the row's targets in order with
// the previous triangle as the hint exactly like the reference's per-row
// parallel_for body (the hint chain makes a row sequential); the exhaustive
// scan fallback runs in the same thread.  K5: one thread per cell computes
// Q = tr(J^T J) / (2 det J) and flags folded cells; the sum for q_mean is
// then folded in the reference's row-major order by one thread (exactly the
// reference's rounding sequence), the maxima are order-free.
#include <cfloat>

#include "density.cuh"
#include "sddg_internal.h"

namespace sddg {

namespace {

struct Tess {
    const double* xi;
    const double* eta;
    int nx, ny;
    __device__ int cx() const { return nx - 1; }
    __device__ int cy() const { return ny - 1; }
    __device__ long long tri_count() const { return 2LL * cx() * cy(); }
    __device__ void vertices(long long t, int idx[3][2]) const {
        const long long cell = t / 2;
        const int half = static_cast<int>(t % 2);
        const int i = static_cast<int>(cell % cx());
        const int j = static_cast<int>(cell / cx());
        idx[0][0] = i;
        idx[0][1] = j;
        idx[1][0] = i + 1;
        idx[1][1] = half == 0 ? j : j + 1;
        idx[2][0] = half == 0 ? i + 1 : i;
        idx[2][1] = j + 1;
    }
    __device__ long long neighbor(long long t, int k) const {
        const long long cell = t / 2;
        const int half = static_cast<int>(t % 2);
        const int i = static_cast<int>(cell % cx());
        const int j = static_cast<int>(cell / cx());
        auto tri = [&](int ci, int cj, int h) -> long long {
            if (ci < 0 || cj < 0 || ci >= cx() || cj >= cy()) return -1;
            return 2LL * (static_cast<long long>(cj) * cx() + ci) + h;
        };
        if (half == 0) {
            if (k == 0) return tri(i + 1, j, 1);
            if (k == 1) return tri(i, j, 1);
            return tri(i, j - 1, 1);
        }
        if (k == 0) return tri(i, j + 1, 0);
        if (k == 1) return tri(i - 1, j, 0);
        return tri(i, j, 0);
    }
};

struct Bary {
    bool inside;
    double w[3];
    double det;
    int exit_vertex;
};

__device__ __forceinline__ double cross(double ax, double ay, double bx, double by) {
    return ax * by - ay * bx;
}

// barycentric (proj/src/invert.cpp:81-111)
__device__ Bary barycentric(const Tess& T, long long t, double px, double py, double tol) {
    int idx[3][2];
    T.vertices(t, idx);
    double vx[3], vy[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long n = static_cast<long long>(idx[k][1]) * T.nx + idx[k][0];
        vx[k] = T.xi[n];
        vy[k] = T.eta[n];
    }
    Bary r;
    r.det = cross(vx[1] - vx[0], vy[1] - vy[0], vx[2] - vx[0], vy[2] - vy[0]);
    if (r.det == 0.0) {
        r.inside = false;
        r.exit_vertex = -1;
        r.w[0] = r.w[1] = r.w[2] = 0.0;
        return r;
    }
    const double a0 = cross(vx[1] - px, vy[1] - py, vx[2] - px, vy[2] - py);
    const double a1 = cross(vx[2] - px, vy[2] - py, vx[0] - px, vy[0] - py);
    const double a2 = cross(vx[0] - px, vy[0] - py, vx[1] - px, vy[1] - py);
    r.w[0] = a0 / r.det;
    r.w[1] = a1 / r.det;
    r.w[2] = a2 / r.det;
    r.inside = r.w[0] >= -tol && r.w[1] >= -tol && r.w[2] >= -tol;
    r.exit_vertex = 0;
    if (r.w[1] < r.w[r.exit_vertex]) r.exit_vertex = 1;
    if (r.w[2] < r.w[r.exit_vertex]) r.exit_vertex = 2;
    return r;
}

// walk_locate (proj/src/invert.cpp:113-126)
__device__ long long walk_locate(const Tess& T, long long start, double px, double py, double tol) {
    long long t = start;
    const int limit = 2 * (T.nx + T.ny) + 16;
    for (int step = 0; step < limit; ++step) {
        const Bary r = barycentric(T, t, px, py, tol);
        if (r.inside) return t;
        if (r.exit_vertex < 0) return -1;
        const long long next = T.neighbor(t, r.exit_vertex);
        if (next < 0) return -1;
        t = next;
    }
    return -1;
}

// scan_locate (proj/src/invert.cpp:128-138)
__device__ long long scan_locate(const Tess& T, double px, double py, double tol) {
    long long flipped = -1;
    for (long long t = 0; t < T.tri_count(); ++t) {
        const Bary r = barycentric(T, t, px, py, tol);
        if (!r.inside) continue;
        if (r.det > 0.0) return t;
        if (flipped < 0) flipped = t;
    }
    return flipped;
}

// invert_mesh row body (proj/src/invert.cpp:154-193)
__global__ void invert_kernel(const double* __restrict__ xi, const double* __restrict__ eta, int nx,
                              int ny, double gx0, double gy0, double ghx, double ghy, int m_xi,
                              int m_eta, double* __restrict__ X, double* __restrict__ Y,
                              int* err, int* err_row) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= m_eta) return;
    const Tess T{xi, eta, nx, ny};
    const double kWalkTol = 1e-12, kSnapTol = 1e-9;
    const double eta_b = static_cast<double>(b) / (m_eta - 1);
    long long hint = -1;
    for (int a = 0; a < m_xi; ++a) {
        const double xi_a = static_cast<double>(a) / (m_xi - 1);
        if (hint < 0) {
            int ci = static_cast<int>(xi_a * (nx - 2));
            ci = ci < 0 ? 0 : (ci > nx - 2 ? nx - 2 : ci);
            int cj = static_cast<int>(eta_b * (ny - 2));
            cj = cj < 0 ? 0 : (cj > ny - 2 ? ny - 2 : cj);
            hint = 2LL * (static_cast<long long>(cj) * (nx - 1) + ci);
        }
        long long t = walk_locate(T, hint, xi_a, eta_b, kWalkTol);
        if (t < 0) t = scan_locate(T, xi_a, eta_b, kWalkTol);
        if (t < 0) t = scan_locate(T, xi_a, eta_b, kSnapTol);
        if (t < 0) {
            atomicCAS(err, 0, 8);  // InversionError: not covered
            atomicExch(err_row, b);
            return;
        }
        const Bary r = barycentric(T, t, xi_a, eta_b, kSnapTol);
        if (r.det == 0.0) {
            atomicCAS(err, 0, 8);  // InversionError: degenerate
            atomicExch(err_row, b);
            return;
        }
        int idx[3][2];
        T.vertices(t, idx);
        double px = 0.0, py = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double nxp = gx0 + idx[k][0] * ghx;  // GridSpec::node
            const double nyp = gy0 + idx[k][1] * ghy;
            px += r.w[k] * nxp;
            py += r.w[k] * nyp;
        }
        X[static_cast<long long>(b) * m_xi + a] = px;
        Y[static_cast<long long>(b) * m_xi + a] = py;
        hint = t;
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

// quality_report folds (proj/src/quality.cpp:44-53): row-major sequential sum,
// std::max.  One thread: the reference's exact rounding sequence.
__global__ void quality_fold(const double* __restrict__ q, long long cells, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double sum = 0.0, qmax = 0.0;
    for (long long c = 0; c < cells; ++c) {
        const double v = q[c];
        sum += v;
        qmax = qmax < v ? v : qmax;
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

cudaError_t launch_invert(const double* xi, const double* eta, int nx, int ny, double gx0,
                          double gy0, double ghx, double ghy, int m_xi, int m_eta, double* X,
                          double* Y, int* err, int* err_row, cudaStream_t s) {
    invert_kernel<<<(m_eta + 63) / 64, 64, 0, s>>>(xi, eta, nx, ny, gx0, gy0, ghx, ghy, m_xi, m_eta,
                                                   X, Y, err, err_row);
    return cudaGetLastError();
}

cudaError_t launch_quality(const double* X, const double* Y, int m_xi, int m_eta, double* qbuf,
                           double* out2, int* err, cudaStream_t s) {
    const long long cells = static_cast<long long>(m_xi - 1) * (m_eta - 1);
    quality_cells<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, s>>>(X, Y, m_xi, m_eta, qbuf,
                                                                             err);
    quality_fold<<<1, 32, 0, s>>>(qbuf, cells, out2);
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
