/*
 * workload_w.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The BASELINE.json densities as the diffusion weight w (ring: configs 1, 2,
 * 5; shock: config 3; two-bump: config 4).  This is the workload definition
 * fed to the reference (oracle/ref_harness.cpp, as
 * MonitorFunction::user_supplied(rho = 1/w), proj/src/monitor.cpp:73-80) and
 * to the C restatement (sdd_oracle.c).  The product kernels restate the same
 * expressions in the same operation order (csrc/density.cuh).
 */
#ifndef SDD_WORKLOAD_W_H
#define SDD_WORKLOAD_W_H

#include <math.h>

#define WL_RING 16
#define WL_SHOCK 17
#define WL_TWOBUMP 18
#define WL_PI 3.14159265358979323846264338327950288

static inline double wl_w(int kind, double x, double y) {
    switch (kind) {
        case WL_RING: {
            const double dx = x - 0.5, dy = y - 0.5;
            const double q = dx * dx + dy * dy - 0.0625;
            return 1.0 + 10.0 * exp(-200.0 * q * q);
        }
        case WL_SHOCK: {
            const double s = 50.0 * (y - 0.5 - 0.15 * sin(2.0 * WL_PI * x));
            const double e = exp(-2.0 * fabs(s));
            const double d = 1.0 + e;
            return 1.0 + 20.0 * (4.0 * e / (d * d));
        }
        case WL_TWOBUMP: {
            const double ax = x - 0.3, ay = y - 0.3, bx = x - 0.7, by = y - 0.6;
            return 1.0 + 15.0 * exp(-100.0 * (ax * ax + ay * ay)) +
                   15.0 * exp(-100.0 * (bx * bx + by * by));
        }
    }
    return 1.0;
}

#endif
