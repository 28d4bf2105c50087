// table_density.h -- the tabulated density (SDDG_DENS_TABLE): any
// user_supplied rho of the reference (proj/src/monitor.cpp:73-80) handed to
// the GPU as data, rho sampled at the nodes of a grid over its domain.
//
// Interpolant (fixed, part of the ABI): Catmull-Rom bicubic, i.e. cubic
// convolution with a = -1/2, on the grid padded by one node per side whose
// value is the linear extrapolation 2 f(edge) - f(edge +- 1) (first in x,
// then in y).  Cell (i, j) = clamp(floor((x - x0)/hx), 0, n - 2), local
// t = s - i (not clamped, so the interpolant continues smoothly a little
// past the domain, where the reference's central difference may look).
// Linear rho is reproduced exactly; the interpolant is C1, so the drift is
// continuous.  The operation order below is normative: the reference-mode
// walk (built with -fmad=false), the host set-up code and the quality
// kernel evaluate exactly this sequence.
#pragma once
#include <cmath>
#include <cstddef>
#include <vector>

#ifdef __CUDACC__
#define SDDG_HD __host__ __device__
#else
#define SDDG_HD
#endif

namespace sddg {

struct TableDensity {
    const double* t = nullptr;  // padded (nx+2) x (ny+2); node (i, j) at (j+1)(nx+2) + i+1
    int nx = 0, ny = 0;         // sample grid
    double x0 = 0, y0 = 0;      // grid origin
    double ihx = 1, ihy = 1;    // RN(1 / hx), hx = (xmax - xmin) / (nx - 1)
};

SDDG_HD inline void cr_weights(double t, double w[4]) {
    w[0] = 0.5 * (((2.0 - t) * t - 1.0) * t);
    w[1] = 0.5 * ((3.0 * t - 5.0) * t * t + 2.0);
    w[2] = 0.5 * (((4.0 - 3.0 * t) * t + 1.0) * t);
    w[3] = 0.5 * ((t - 1.0) * t * t);
}

SDDG_HD inline int table_cell(double s, int n) {
    int i = static_cast<int>(floor(s));
    return i < 0 ? 0 : (i > n - 2 ? n - 2 : i);
}

SDDG_HD inline double table_rho(const TableDensity& d, double x, double y) {
    const double sx = (x - d.x0) * d.ihx, sy = (y - d.y0) * d.ihy;
    const int i = table_cell(sx, d.nx), j = table_cell(sy, d.ny);
    double wx[4], wy[4];
    cr_weights(sx - i, wx);
    cr_weights(sy - j, wy);
    const int st = d.nx + 2;
    const double* p = d.t + static_cast<size_t>(j) * st + i;  // padded node (i-1, j-1)
    double v = 0.0;
    for (int b = 0; b < 4; ++b) {
        const double* r = p + b * st;
        const double row = ((wx[0] * r[0] + wx[1] * r[1]) + wx[2] * r[2]) + wx[3] * r[3];
        v = v + wy[b] * row;
    }
    return v;
}

// The padded table of nx x ny samples f (index j*nx + i).
inline std::vector<double> pad_table(const double* f, int nx, int ny) {
    const int st = nx + 2;
    std::vector<double> p(static_cast<size_t>(st) * (ny + 2), 0.0);
    for (int j = 0; j < ny; ++j) {
        double* r = p.data() + static_cast<size_t>(j + 1) * st;
        for (int i = 0; i < nx; ++i) r[i + 1] = f[static_cast<size_t>(j) * nx + i];
        r[0] = 2.0 * r[1] - r[2];
        r[nx + 1] = 2.0 * r[nx] - r[nx - 1];
    }
    for (int i = 0; i < st; ++i) {
        p[i] = 2.0 * p[st + i] - p[2 * st + i];
        p[static_cast<size_t>(ny + 1) * st + i] =
            2.0 * p[static_cast<size_t>(ny) * st + i] - p[static_cast<size_t>(ny - 1) * st + i];
    }
    return p;
}

}  // namespace sddg
