// host_density.h -- host-side density evaluation for the set-up work the
// reference does on the host before and around the hot path: boundary tables
// (solve_1d_boundary, proj/src/detsolver.cpp:20-48), nodal weights
// (weight_values, :219-224) and optimal placement gradients
// (proj/src/decomposition.cpp:81-108).  Same expressions and the same glibc
// libm as the reference (proj/src/monitor.cpp:121-223), so the tables and
// weights are bit-identical to the reference's.
#pragma once
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sddg.h"
#include "table_density.h"

namespace sddg {

struct HostDensity {
    int kind;
    double R, alpha, fd_h;
    // SDDG_DENS_TABLE: the padded samples (owned) and their interpolant view
    std::shared_ptr<const std::vector<double>> padded;
    TableDensity td;

    static HostDensity of(const sddg_density& d) {
        HostDensity h{d.kind, d.R, d.alpha, d.fd_h, nullptr, TableDensity{}};
        if (d.kind == SDDG_DENS_TABLE && d.table && d.tnx >= 2 && d.tny >= 2) {
            h.padded = std::make_shared<const std::vector<double>>(pad_table(d.table, d.tnx, d.tny));
            h.td.t = h.padded->data();
            h.td.nx = d.tnx;
            h.td.ny = d.tny;
            h.td.x0 = d.tdom.xmin;
            h.td.y0 = d.tdom.ymin;
            h.td.ihx = 1.0 / ((d.tdom.xmax - d.tdom.xmin) / (d.tnx - 1));
            h.td.ihy = 1.0 / ((d.tdom.ymax - d.tdom.ymin) / (d.tny - 1));
        }
        return h;
    }

    static double w_of(int kind, double x, double y) {
        constexpr double kPi = 3.14159265358979323846264338327950288;
        switch (kind) {
            case SDDG_DENS_RING_W: {
                const double dx = x - 0.5, dy = y - 0.5;
                const double q = dx * dx + dy * dy - 0.0625;
                return 1.0 + 10.0 * std::exp(-200.0 * q * q);
            }
            case SDDG_DENS_SHOCK_W: {
                const double s = 50.0 * (y - 0.5 - 0.15 * std::sin(2.0 * kPi * x));
                const double e = std::exp(-2.0 * std::fabs(s));
                const double d = 1.0 + e;
                return 1.0 + 20.0 * (4.0 * e / (d * d));
            }
            default: {
                const double ax = x - 0.3, ay = y - 0.3, bx = x - 0.7, by = y - 0.6;
                return 1.0 + 15.0 * std::exp(-100.0 * (ax * ax + ay * ay)) +
                       15.0 * std::exp(-100.0 * (bx * bx + by * by));
            }
        }
    }

    static void five_ring(double x, double y, double R, double& ux, double& uy, double& uxx,
                          double& uxy, double& uyy) {
        static constexpr double cx[5] = {0.0, 0.5, 0.5, -0.5, -0.5};
        static constexpr double cy[5] = {0.0, 0.5, -0.5, 0.5, -0.5};
        ux = uy = uxx = uxy = uyy = 0.0;
        for (int k = 0; k < 5; ++k) {
            const double dx = x - cx[k];
            const double dy = y - cy[k];
            const double t = std::tanh(R * (dx * dx + dy * dy - 0.125));
            const double s = 1.0 - t * t;
            const double gx = 2.0 * R * dx;
            const double gy = 2.0 * R * dy;
            ux += s * gx;
            uy += s * gy;
            uxx += s * (2.0 * R - 2.0 * t * gx * gx);
            uyy += s * (2.0 * R - 2.0 * t * gy * gy);
            uxy += -2.0 * t * s * gx * gy;
        }
    }

    // MonitorFunction::rho (proj/src/monitor.cpp:121-161)
    double rho(double x, double y) const {
        constexpr double kPi = 3.14159265358979323846264338327950288;
        double r;
        switch (kind) {
            case SDDG_DENS_CONSTANT: r = R; break;
            case SDDG_DENS_RUNNING: {
                const double dx = x - 0.75, dy = y - 0.5;
                r = 1.0 + R * std::exp(-50.0 * dx * dx - 50.0 * dy * dy - 0.5);
                break;
            }
            case SDDG_DENS_HUANG_SLOAN: {
                const double E = std::exp(R * (x - 1.0));
                const double S = std::sin(kPi * y);
                const double C = std::cos(kPi * y);
                const double q =
                    alpha * (R * R * E * E * S * S + (1.0 - E) * (1.0 - E) * kPi * kPi * C * C);
                r = std::sqrt(1.0 + q);
                break;
            }
            case SDDG_DENS_MACKENZIE: {
                const double s = y - 0.5 - 0.25 * std::sin(2.0 * kPi * x);
                r = 1.0 / (1.0 + alpha * std::exp(-R * s * s));
                break;
            }
            case SDDG_DENS_FIVE_RING: {
                double ux, uy, uxx, uxy, uyy;
                five_ring(x, y, R, ux, uy, uxx, uxy, uyy);
                r = std::sqrt(1.0 + alpha * (ux * ux + uy * uy));
                break;
            }
            case SDDG_DENS_TABLE: r = table_rho(td, x, y); break;
            default: r = 1.0 / w_of(kind, x, y); break;
        }
        if (!std::isfinite(r)) throw std::domain_error("monitor density not finite");
        return r;
    }

    // grad_rho (proj/src/monitor.cpp:163-229)
    void grad(double x, double y, double& gx, double& gy) const {
        constexpr double kPi = 3.14159265358979323846264338327950288;
        switch (kind) {
            case SDDG_DENS_CONSTANT: gx = gy = 0.0; return;
            case SDDG_DENS_RUNNING: {
                const double dx = x - 0.75, dy = y - 0.5;
                const double g = R * std::exp(-50.0 * dx * dx - 50.0 * dy * dy - 0.5);
                gx = -100.0 * dx * g;
                gy = -100.0 * dy * g;
                return;
            }
            case SDDG_DENS_HUANG_SLOAN: {
                const double E = std::exp(R * (x - 1.0));
                const double S = std::sin(kPi * y);
                const double C = std::cos(kPi * y);
                const double q =
                    alpha * (R * R * E * E * S * S + (1.0 - E) * (1.0 - E) * kPi * kPi * C * C);
                const double r = std::sqrt(1.0 + q);
                const double qx = alpha * (2.0 * R * R * R * E * E * S * S +
                                           2.0 * kPi * kPi * R * C * C * E * (E - 1.0));
                const double qy = 2.0 * kPi * S * C * alpha *
                                  (R * R * E * E - kPi * kPi * (1.0 - E) * (1.0 - E));
                gx = qx / (2.0 * r);
                gy = qy / (2.0 * r);
                return;
            }
            case SDDG_DENS_MACKENZIE: {
                const double s = y - 0.5 - 0.25 * std::sin(2.0 * kPi * x);
                const double E = std::exp(-R * s * s);
                const double D = 1.0 + alpha * E;
                const double drho_ds = 2.0 * alpha * R * s * E / (D * D);
                const double sx = -0.5 * kPi * std::cos(2.0 * kPi * x);
                gx = drho_ds * sx;
                gy = drho_ds;
                return;
            }
            case SDDG_DENS_FIVE_RING: {
                double ux, uy, uxx, uxy, uyy;
                five_ring(x, y, R, ux, uy, uxx, uxy, uyy);
                const double r = std::sqrt(1.0 + alpha * (ux * ux + uy * uy));
                gx = alpha * (ux * uxx + uy * uxy) / r;
                gy = alpha * (ux * uxy + uy * uyy) / r;
                return;
            }
            case SDDG_DENS_TABLE: {  // user_supplied central difference of the interpolant
                const double h = fd_h;
                gx = (table_rho(td, x + h, y) - table_rho(td, x - h, y)) / (2.0 * h);
                gy = (table_rho(td, x, y + h) - table_rho(td, x, y - h)) / (2.0 * h);
                return;
            }
            default: {
                const double h = fd_h;
                gx = (1.0 / w_of(kind, x + h, y) - 1.0 / w_of(kind, x - h, y)) / (2.0 * h);
                gy = (1.0 / w_of(kind, x, y + h) - 1.0 / w_of(kind, x, y - h)) / (2.0 * h);
                return;
            }
        }
    }
};

}  // namespace sddg
