// smooth.cu -- K6 Perona-Malik FTCS smoothing and K7 interface loess.
//
// Reference: perona_malik / smooth_block / smooth_field
// (proj/src/smoothing.cpp:33-138) and smooth_interface (:140-183).
//
// K6: per FTCS step two launches over every (block, field):
//   pm_cond:  c = exp(-|grad u|^2 / k^2) at every block node (centred
//             differences inside the block, one-sided on its edges; a node on
//             an interface line gets one c per adjacent block, so c is stored
//             per block);
//   pm_flux:  u_next = u + dt * div(c grad u) on block interiors, per-step
//             max |u_next - u| per field via atomicMax on the (non-negative)
//             double bits.
// Block boundaries are never written (physical boundary; in per-subdomain
// scope also the interface lines), so blocks are independent within a step
// and the ping-pong buffers equal the reference's in-place update.  The
// FTCS instability rule (update grew > 10x, smoothing.cpp:115-120) is
// evaluated on the host from the per-step maxima.  Built with -fmad=false.
//
// K7: one thread per interior line node: tricube-weighted quadratic least
// squares over the span window evaluated at the centre (smoothing.cpp:146-180).
#include "sddg_internal.h"

namespace sddg {

namespace {

struct PmBlock {
    int i0, j0, bnx, bny;
    long long c_off;  // offset of this block's c scratch (bnx*bny)
};

__global__ void pm_cond(const double* __restrict__ u0, const double* __restrict__ u1, int nx,
                        int n_per_field, const PmBlock* __restrict__ blocks, int nblocks,
                        double hx, double hy, double inv_k2, double* __restrict__ cbuf,
                        long long c_field_stride) {
    const int f = blockIdx.y;              // field: 0 xi, 1 eta
    const int b = blockIdx.z;              // smoothing block
    const PmBlock B = blocks[b];
    const double* u = f == 0 ? u0 : u1;
    double* cc = cbuf + f * c_field_stride + B.c_off;
    const int n = B.bnx * B.bny;
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n; l += gridDim.x * blockDim.x) {
        const int i = l % B.bnx, j = l / B.bnx;
        const int gi = B.i0 + i, gj = B.j0 + j;
        const long long g = static_cast<long long>(gj) * nx + gi;
        double gx, gy;
        if (i == 0) gx = (u[g + 1] - u[g]) / hx;
        else if (i == B.bnx - 1) gx = (u[g] - u[g - 1]) / hx;
        else gx = (u[g + 1] - u[g - 1]) / (2.0 * hx);
        if (j == 0) gy = (u[g + nx] - u[g]) / hy;
        else if (j == B.bny - 1) gy = (u[g] - u[g - nx]) / hy;
        else gy = (u[g + nx] - u[g - nx]) / (2.0 * hy);
        cc[l] = exp(-(gx * gx + gy * gy) * inv_k2);
    }
    (void)n_per_field;
    (void)nblocks;
}

__global__ void pm_flux(const double* __restrict__ u0, const double* __restrict__ u1,
                        double* __restrict__ v0, double* __restrict__ v1, int nx,
                        const PmBlock* __restrict__ blocks, double ihx2, double ihy2, double dt,
                        const double* __restrict__ cbuf, long long c_field_stride,
                        unsigned long long* __restrict__ upd_bits) {
    const int f = blockIdx.y;
    const int b = blockIdx.z;
    const PmBlock B = blocks[b];
    const double* u = f == 0 ? u0 : u1;
    double* v = f == 0 ? v0 : v1;
    const double* cc = cbuf + f * c_field_stride + B.c_off;
    const int mi = B.bnx - 2, mj = B.bny - 2;
    double lmax = 0.0;
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < mi * mj; l += gridDim.x * blockDim.x) {
        const int i = l % mi + 1, j = l / mi + 1;
        const int c = j * B.bnx + i;
        const long long gc = static_cast<long long>(B.j0 + j) * nx + (B.i0 + i);
        const double cE = 0.5 * (cc[c] + cc[c + 1]);
        const double cW = 0.5 * (cc[c] + cc[c - 1]);
        const double cN = 0.5 * (cc[c] + cc[c + B.bnx]);
        const double cS = 0.5 * (cc[c] + cc[c - B.bnx]);
        const double flux = (cE * (u[gc + 1] - u[gc]) - cW * (u[gc] - u[gc - 1])) * ihx2 +
                            (cN * (u[gc + nx] - u[gc]) - cS * (u[gc] - u[gc - nx])) * ihy2;
        const double nv = u[gc] + dt * flux;
        v[gc] = nv;
        const double d = fabs(nv - u[gc]);
        lmax = lmax < d ? d : lmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, lmax, o);
        lmax = lmax < t ? t : lmax;
    }
    if ((threadIdx.x & 31) == 0)
        atomicMax(&upd_bits[f], static_cast<unsigned long long>(__double_as_longlong(lmax)));
}

// smooth_interface (proj/src/smoothing.cpp:140-183), one thread per node
__global__ void loess_kernel(const double* __restrict__ in, double* __restrict__ out, int n,
                             int span, int* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (i + 1 >= n) return;
    const int half = (span - 1) / 2;
    int lo = i - half;
    lo = lo < 0 ? 0 : (lo > n - span ? n - span : lo);
    double dmax = 0.0;
    for (int j = lo; j < lo + span; ++j) {
        const double d = fabs(static_cast<double>(j - i));
        dmax = dmax < d ? d : dmax;
    }
    dmax += 1.0;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, b0 = 0, b1 = 0, b2 = 0;
    for (int j = lo; j < lo + span; ++j) {
        const double t = static_cast<double>(j - i);
        const double a = 1.0 - pow(fabs(t) / dmax, 3.0);
        const double w = a * a * a;
        const double v = in[j];
        s0 += w;
        s1 += w * t;
        s2 += w * t * t;
        s3 += w * t * t * t;
        s4 += w * t * t * t * t;
        b0 += w * v;
        b1 += w * t * v;
        b2 += w * t * t * v;
    }
    const double d = s0 * (s2 * s4 - s3 * s3) - s1 * (s1 * s4 - s2 * s3) + s2 * (s1 * s3 - s2 * s2);
    if (fabs(d) < 1e-300) {
        atomicCAS(err, 0, 4);  // NumericalError: singular local fit
        return;
    }
    const double c0 = b0 * (s2 * s4 - s3 * s3) - s1 * (b1 * s4 - b2 * s3) + s2 * (b1 * s3 - b2 * s2);
    out[i] = c0 / d;
}

}  // namespace

// Runs `steps` FTCS steps on both fields (device arrays u0=xi, u1=eta, each
// nx*ny) over the given blocks; per-step per-field max updates go to
// upd_host[steps][2].  v0, v1: ping-pong buffers (nx*ny each).
cudaError_t pm_run(double* u0, double* u1, double* v0, double* v1, int nx, int ny,
                   const int* blocks_host, int nblocks, double hx, double hy, double k, double dt,
                   int steps, double* scratch, unsigned long long* dev_upd, double* upd_host,
                   cudaStream_t s) {
    std::vector<PmBlock> hb(nblocks);
    long long off = 0;
    for (int b = 0; b < nblocks; ++b) {
        hb[b] = PmBlock{blocks_host[4 * b], blocks_host[4 * b + 1], blocks_host[4 * b + 2],
                        blocks_host[4 * b + 3], off};
        off += static_cast<long long>(hb[b].bnx) * hb[b].bny;
    }
    PmBlock* db = reinterpret_cast<PmBlock*>(scratch);
    double* cbuf = scratch + (sizeof(PmBlock) * nblocks + 7) / 8 + 8;
    cudaError_t e = cudaMemcpyAsync(db, hb.data(), sizeof(PmBlock) * nblocks, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    // v = u so the untouched boundary nodes are already in place
    cudaMemcpyAsync(v0, u0, sizeof(double) * nx * ny, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(v1, u1, sizeof(double) * nx * ny, cudaMemcpyDeviceToDevice, s);
    cudaMemsetAsync(dev_upd, 0, sizeof(unsigned long long) * 2 * (steps > 0 ? steps : 1), s);
    const double inv_k2 = 1.0 / (k * k);
    const double ihx2 = 1.0 / (hx * hx), ihy2 = 1.0 / (hy * hy);
    int maxn = 0;
    for (const auto& b : hb) maxn = std::max(maxn, b.bnx * b.bny);
    const dim3 grid(static_cast<unsigned>(std::min(1024, (maxn + 255) / 256)), 2, nblocks);
    double *a0 = u0, *a1 = u1, *b0 = v0, *b1 = v1;
    for (int st = 0; st < steps; ++st) {
        pm_cond<<<grid, 256, 0, s>>>(a0, a1, nx, nx * ny, db, nblocks, hx, hy, inv_k2, cbuf, off);
        pm_flux<<<grid, 256, 0, s>>>(a0, a1, b0, b1, nx, db, ihx2, ihy2, dt, cbuf, off,
                                     dev_upd + 2 * st);
        std::swap(a0, b0);
        std::swap(a1, b1);
    }
    if (steps % 2 == 1) {  // result sits in v: copy back into u
        cudaMemcpyAsync(u0, v0, sizeof(double) * nx * ny, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(u1, v1, sizeof(double) * nx * ny, cudaMemcpyDeviceToDevice, s);
    }
    if (steps > 0) {
        std::vector<unsigned long long> bits(2 * steps);
        cudaMemcpyAsync(bits.data(), dev_upd, sizeof(unsigned long long) * 2 * steps,
                        cudaMemcpyDeviceToHost, s);
        e = cudaStreamSynchronize(s);
        for (int q = 0; q < 2 * steps; ++q) std::memcpy(&upd_host[q], &bits[q], sizeof(double));
    }
    return e == cudaSuccess ? cudaGetLastError() : e;
}

size_t pm_scratch_doubles(const int* blocks_host, int nblocks) {
    size_t n = 0;
    for (int b = 0; b < nblocks; ++b)
        n += static_cast<size_t>(blocks_host[4 * b + 2]) * blocks_host[4 * b + 3];
    return 2 * n + (sizeof(PmBlock) * nblocks + 7) / 8 + 16;
}

cudaError_t loess_run(const double* d_in, double* d_out, int n, int span, int* d_err, cudaStream_t s) {
    cudaMemcpyAsync(d_out, d_in, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    if (n > 2) loess_kernel<<<(n - 2 + 127) / 128, 128, 0, s>>>(d_in, d_out, n, span, d_err);
    return cudaGetLastError();
}

}  // namespace sddg
