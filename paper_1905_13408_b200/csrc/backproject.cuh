// Backprojection into the kernel-regression accumulators on the device
// (reference: backproject_accumulate, backproject.cpp:12-101).
//
//   numerator(n) += P * K(n_j, n) * CTF_j * Xhat_j,  weight(n) += P * K * CTF_j^2
//
// over the nonzero-posterior (particle, candidate) entries, the image's 2D
// frequency components within the cutoff and the kernel window's in-grid taps,
// followed by the Friedel average of every orbit with its conjugated mate.
//
// Mapping: entries are grouped by pose on the host; bp_gather_kernel (one
// thread per (pose, component)) sums post * CTF * Xhat and post * CTF^2 over
// the pose's entries -- CTF, shift phase and image read per entry, no atomics
// -- and bp_spread_kernel spreads each (pose, component) once through its 8 / 27
// taps with fp64 atomics into the fp64 staging grid that commit_acc_stage then
// converts into the solver's resident W / Y. (CM_BP_DIRECT=1 selects the
// per-entry scatter, the reference's loop order, for A/B.) The arithmetic that decides
// tap positions (the rotation and the rotated point) is written with explicit
// rounding intrinsics in the reference's evaluation order, so a point on a
// floor / lround boundary (15-degree grid poses put many exactly on .5) lands
// on the same side as in the reference; transcendentals differ from glibc by an
// ulp, and the atomic sum order is not fixed, so results agree with the
// reference to ~1e-15 relative rather than bitwise.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cm_api.h"
#include "cm_common.cuh"

namespace cm {

int fail(int code, const std::string& msg);

struct BpDev {
    const double2* img;     // [n_images][n*n]
    const double* iparams;  // [n_images][6]
    const double* mats;     // [n_poses][9]
    const int2* shifts;     // [n_shifts]
    const int2* comps;      // [ncomp] (k, l)
    const long long* epart;
    const unsigned* ecand;
    const double* epost;
    double* weight;         // [L]
    double2* num;           // [L]
    long long n_entries;
    int ncomp, n, n_shifts;
    double bandwidth;
};

__device__ __forceinline__ int bp_store(int h, int n) { return h >= 0 ? h : h + n; }

// ctf_value (ctf.cpp:11-23) with electron_wavelength_A (ctf.cpp:7-10)
__device__ __forceinline__ double bp_ctf(const double* ip, double s) {
    if (ip[4] != 0.0) return 1.0;
    const double kPi = 3.14159265358979323846;
    const double v = ip[0] * 1000.0;
    const double lambda = 12.2639 / sqrt(v + 0.97845e-6 * v * v);
    const double cs_A = ip[2] * 1e7;
    const double s2 = s * s;
    const double chi = kPi * lambda * ip[1] * s2 - (kPi / 2.0) * cs_A * lambda * lambda * lambda * s2 * s2;
    const double a = ip[3];
    return -(sqrt(1.0 - a * a) * sin(chi) + a * cos(chi));
}

// The window of a rotated frequency (kernel_taps, kernel.cpp:36-78) with the
// in-grid test of backproject.cpp:58-61: f(px, py, pz, w) per tap.
template <int KIND, typename F>
__device__ __forceinline__ void bp_window(const double* R, int k, int l, double bandwidth, int n, F&& f) {
    const int lo = -n / 2, hi = n / 2 - 1;
    double nj[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)  // the reference's as-built order (see bp_scatter_kernel)
        nj[a] = __dadd_rn(__fma_rn(R[3 * a], (double)k, __dmul_rn(R[3 * a + 1], (double)l)),
                          __dmul_rn(R[3 * a + 2], 0.0));
    auto tap = [&](int px, int py, int pz, double w) {
        if (px < lo || px > hi || py < lo || py > hi || pz < lo || pz > hi) return;
        f(((size_t)bp_store(pz, n) * n + bp_store(py, n)) * n + bp_store(px, n), w);
    };
    if constexpr (KIND == 0) {
        int anc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) anc[a] = (int)llround(nj[a]);
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    const int q[3] = {anc[0] + dx, anc[1] + dy, anc[2] + dz};
                    double d2 = 0.0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const double d = __dsub_rn(nj[a], (double)q[a]);
                        d2 = __dadd_rn(d2, __dmul_rn(d, d));
                    }
                    tap(q[0], q[1], q[2], exp(-d2 / bandwidth));
                }
    } else {
        int lo3[3];
        double fr[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo3[a] = (int)floor(nj[a]);
            fr[a] = __dsub_rn(nj[a], (double)lo3[a]);
        }
        const int cz1 = fr[2] == 0.0 ? 0 : 1, cy1 = fr[1] == 0.0 ? 0 : 1, cx1 = fr[0] == 0.0 ? 0 : 1;
        for (int cz = 0; cz <= cz1; ++cz)
            for (int cy = 0; cy <= cy1; ++cy)
                for (int cx = 0; cx <= cx1; ++cx) {
                    const double wx = cx ? fr[0] : 1.0 - fr[0];
                    const double wy = cy ? fr[1] : 1.0 - fr[1];
                    const double wz = cz ? fr[2] : 1.0 - fr[2];
                    tap(lo3[0] + cx, lo3[1] + cy, lo3[2] + cz, __dmul_rn(__dmul_rn(wx, wy), wz));
                }
    }
}

// Pose-grouped form (the default). Every entry of one pose spreads its
// components through the same windows, so the per-entry sums
//   Z(pose, j) = sum_e post_e ctf_e(j) Xhat_e(j),  Wt(pose, j) = sum_e post_e ctf_e(j)^2
// are formed first (a gather, no atomics), and only (pose, component) pairs are
// spread: tap w adds w Z and w Wt. Fewer REDs by the entries-per-pose factor;
// the sums associate differently from the reference's per-entry adds (1e-16
// relative per term).
struct BpGroup {
    const int* pose_of;     // [nused] pose index of each used pose
    const int* off;         // [nused + 1] into the grouped entries
    double2* Z;             // [batch][ncomp]
    double* Wt;
    const double2* ph;      // [n] roots e^{-2 pi i t / n}: the shift phase of (k, l, s) is
                            // ph[(k sx + l sy) mod n] (slice.cpp:47-50, reduced exactly)
    const int* gpart;       // per grouped entry: particle, shift, posterior
    const int2* gsh;
    const double* gpost;
};

// the n-th roots of unity of the shift phases, from sincospi of the reduced
// argument (the integer k sx + l sy reduced mod n exactly)
__global__ void bp_roots_kernel(int n, double2* ph) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double sp, cp;
    sincospi(-2.0 * (double)t / (double)n, &sp, &cp);
    ph[t] = make_double2(cp, sp);
}

// Entries of a pose arrive in PosteriorRow order (particle-major), so the runs
// of one particle share its CTF and image sample: per run
//   Z += ctf X conj(sum_s post_s ph_s),  Wt += ctf^2 sum_s post_s
// with the phase from the table -- one CTF and one image read per
// (pose, particle, component) instead of per entry.
__global__ void __launch_bounds__(128) bp_gather_kernel(BpDev p, BpGroup g, int u0) {
    extern __shared__ double2 roots[];  // [n]
    const int n = p.n;
    for (int t = threadIdx.x; t < n; t += blockDim.x) roots[t] = g.ph[t];
    __syncthreads();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int u = u0 + blockIdx.y;
    if (j >= p.ncomp) return;
    const int k = p.comps[j].x, l = p.comps[j].y;
    // (k sx + l sy) mod n by a mask when n is a power of two
    const int kk = k < 0 ? k + n : k, ll = l < 0 ? l + n : l;
    const bool pow2 = (n & (n - 1)) == 0;
    const double r = __dsqrt_rn((double)(k * k + l * l));
    const size_t pix = (size_t)bp_store(l, n) * n + bp_store(k, n);
    double zr = 0.0, zi = 0.0, wt = 0.0;
    const int qe = g.off[u + 1];
    int q = g.off[u];
    while (q < qe) {
        const int part = g.gpart[q];
        double sr = 0.0, si = 0.0, sw = 0.0;  // sum over the particle's run of post ph, post
        for (; q < qe && g.gpart[q] == part; ++q) {
            const double post = g.gpost[q];
            const int2 sh = g.gsh[q];
            int t = kk * sh.x + ll * sh.y;  // |.| < 2 n^2 (shifts are within the box)
            t = pow2 ? (t & (n - 1)) : ((t % n) + n) % n;
            const double2 ph = roots[t];
            sr = fma(post, ph.x, sr);
            si = fma(post, ph.y, si);
            sw += post;
        }
        const double* ip = p.iparams + 6 * part;
        const double ctf = bp_ctf(ip, r / ((double)n * ip[5]));
        const double2 f = p.img[(size_t)part * n * n + pix];
        // X conj(e^{i ph}) summed: the shift moves the image by -shift (slice.cpp:47-50)
        zr += ctf * (f.x * sr + f.y * si);
        zi += ctf * (f.y * sr - f.x * si);
        wt += ctf * ctf * sw;
    }
    const size_t o = (size_t)blockIdx.y * p.ncomp + j;
    g.Z[o] = make_double2(zr, zi);
    g.Wt[o] = wt;
}

template <int KIND>
__global__ void __launch_bounds__(128) bp_spread_kernel(BpDev p, BpGroup g, int u0) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.ncomp) return;
    const size_t o = (size_t)blockIdx.y * p.ncomp + j;
    const double2 z = g.Z[o];
    const double wt = g.Wt[o];
    if (z.x == 0.0 && z.y == 0.0 && wt == 0.0) return;
    const double* R = p.mats + 9 * (size_t)g.pose_of[u0 + blockIdx.y];
    bp_window<KIND>(R, p.comps[j].x, p.comps[j].y, p.bandwidth, p.n, [&](size_t vi, double w) {
        atomicAdd(&p.num[vi].x, w * z.x);
        atomicAdd(&p.num[vi].y, w * z.y);
        atomicAdd(&p.weight[vi], w * wt);
    });
}

// Per-entry form (CM_BP_DIRECT=1; the reference's loop order, one RED triple per tap and entry)
template <int KIND>  // 0 gaussian (27 taps), 1 trilinear (<= 8 taps)
__global__ void __launch_bounds__(128) bp_scatter_kernel(BpDev p, long long nblocks_total, int cblocks) {
    const int n = p.n, lo = -n / 2, hi = n / 2 - 1;
    for (long long b = blockIdx.x; b < nblocks_total; b += gridDim.x) {
        const long long e = b / cblocks;
        const int c = (int)(b % cblocks) * blockDim.x + threadIdx.x;
        const double post = p.epost[e];
        if (!(post > 0.0) || c >= p.ncomp) continue;  // backproject.cpp:43
        const unsigned cand = p.ecand[e];
        const unsigned pose = cand / (unsigned)p.n_shifts;
        const int2 sh = p.shifts[cand % (unsigned)p.n_shifts];
        const double* R = p.mats + 9 * (size_t)pose;
        const long long part = p.epart[e];
        const double* ip = p.iparams + 6 * part;
        const int2 kl = p.comps[c];
        const int k = kl.x, l = kl.y;
        // freq_of_radius(hypot(k, l)) (simulate.hpp:32): k^2 + l^2 is exact, so
        // the correctly rounded sqrt is the correctly rounded hypot
        const double r = __dsqrt_rn((double)(k * k + l * l));
        const double s = r / ((double)n * ip[5]);
        const double ctf = bp_ctf(ip, s);
        // Xhat = X(k, l) * conj(shift_phase) (slice.cpp:47-50)
        const double2 f = p.img[(size_t)part * n * n + (size_t)bp_store(l, n) * n + bp_store(k, n)];
        const double ph = -2.0 * 3.14159265358979323846 * ((double)k * sh.x + (double)l * sh.y) / (double)n;
        double sp, cp;
        sincos(ph, &sp, &cp);
        const double xr = f.x * cp - f.y * (-sp), xi = f.x * (-sp) + f.y * cp;
        // n_j = R (k, l, 0) (pose.hpp:21-25) in the reference's evaluation order
        // as built (GCC contracts it on x86-64-v3: fma(m0, k, m1 * l) + m2 * 0,
        // read off the object code), so lround / floor ties break the same way
        double nj[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
            nj[a] = __dadd_rn(__fma_rn(R[3 * a], (double)k, __dmul_rn(R[3 * a + 1], (double)l)),
                              __dmul_rn(R[3 * a + 2], 0.0));
        auto tap = [&](int px, int py, int pz, double w) {
            if (px < lo || px > hi || py < lo || py > hi || pz < lo || pz > hi) return;
            const size_t vi = ((size_t)bp_store(pz, n) * n + bp_store(py, n)) * n + bp_store(px, n);
            const double pk = post * w;
            const double pc = pk * ctf;
            atomicAdd(&p.num[vi].x, pc * xr);
            atomicAdd(&p.num[vi].y, pc * xi);
            atomicAdd(&p.weight[vi], pc * ctf);
        };
        if constexpr (KIND == 0) {  // kernel.cpp:38-55
            int anc[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) anc[a] = (int)llround(nj[a]);
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int q[3] = {anc[0] + dx, anc[1] + dy, anc[2] + dz};
                        double d2 = 0.0;
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const double d = __dsub_rn(nj[a], (double)q[a]);
                            d2 = __dadd_rn(d2, __dmul_rn(d, d));
                        }
                        tap(q[0], q[1], q[2], exp(-d2 / p.bandwidth));
                    }
        } else {  // kernel.cpp:57-78
            int lo3[3];
            double fr[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                lo3[a] = (int)floor(nj[a]);
                fr[a] = __dsub_rn(nj[a], (double)lo3[a]);
            }
            const int cz1 = fr[2] == 0.0 ? 0 : 1, cy1 = fr[1] == 0.0 ? 0 : 1, cx1 = fr[0] == 0.0 ? 0 : 1;
            for (int cz = 0; cz <= cz1; ++cz)
                for (int cy = 0; cy <= cy1; ++cy)
                    for (int cx = 0; cx <= cx1; ++cx) {
                        const double wx = cx ? fr[0] : 1.0 - fr[0];
                        const double wy = cy ? fr[1] : 1.0 - fr[1];
                        const double wz = cz ? fr[2] : 1.0 - fr[2];
                        tap(lo3[0] + cx, lo3[1] + cy, lo3[2] + cz, __dmul_rn(__dmul_rn(wx, wy), wz));
                    }
        }
    }
}

// Friedel symmetrization (backproject.cpp:80-96): each orbit {i, mate(i)} once
__global__ void bp_friedel_kernel(int n, double* __restrict__ weight, double2* __restrict__ num) {
    const size_t L = (size_t)n * n * n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < L;
         i += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(i % n), b = (int)((i / n) % n), c = (int)(i / ((size_t)n * n));
        const int ma = a == 0 ? 0 : n - a, mb = b == 0 ? 0 : n - b, mc = c == 0 ? 0 : n - c;
        const size_t m = ((size_t)mc * n + mb) * n + ma;
        if (i > m) continue;
        const double2 zi = num[i], zm = num[m];
        const double2 zn = make_double2(0.5 * (zi.x + zm.x), 0.5 * (zi.y + (-zm.y)));
        num[i] = zn;
        num[m] = make_double2(zn.x, -zn.y);
        const double zw = 0.5 * (weight[i] + weight[m]);
        weight[i] = zw;
        weight[m] = zw;
    }
}

// rotation_matrix (pose.cpp:9-40): Rz(rot) Ry(tilt) Rz(psi), row-major. The
// products decide which grid points a rotated frequency's window covers, so
// they follow the reference's rounding exactly (std::fma is exact in libm)
inline void bp_rotation(const double* ang, double* out) {
    const double kDeg = 3.14159265358979323846 / 180.0;
    auto rz = [&](double deg, double m[3][3]) {
        const double c = std::cos(deg * kDeg), s = std::sin(deg * kDeg);
        const double r[3][3] = {{c, -s, 0.0}, {s, c, 0.0}, {0.0, 0.0, 1.0}};
        std::memcpy(m, r, sizeof r);
    };
    auto ry = [&](double deg, double m[3][3]) {
        const double c = std::cos(deg * kDeg), s = std::sin(deg * kDeg);
        const double r[3][3] = {{c, 0.0, s}, {0.0, 1.0, 0.0}, {-s, 0.0, c}};
        std::memcpy(m, r, sizeof r);
    };
    auto mul = [](const double a[3][3], const double b[3][3], double r[3][3]) {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                // the reference's mat_mul as built: an fma chain from a[i][0] * b[0][j]
                double s = a[i][0] * b[0][j];
                for (int k = 1; k < 3; ++k) s = std::fma(a[i][k], b[k][j], s);
                r[i][j] = s;
            }
    };
    double a[3][3], b[3][3], c[3][3], t[3][3], r[3][3];
    rz(ang[0], a);
    ry(ang[1], b);
    rz(ang[2], c);
    mul(b, c, t);
    mul(a, t, r);
    std::memcpy(out, r, sizeof r);
}

// Particle images resident on the device across EM iterations (cm_set_particles):
// the E-step and the backprojection of every iteration read them in place.
struct ParticleDev {
    double2* img = nullptr;  // [n_images][n*n]
    double* ip = nullptr;    // [n_images][6]
    int n_images = 0;
    ~ParticleDev() { release(); }
    void release() {
        if (img) cudaFree(img);
        if (ip) cudaFree(ip);
        img = nullptr;
        ip = nullptr;
        n_images = 0;
    }
    int set(int n, int m, const double* images, const double* params, cudaStream_t st) {
        release();
        if (m < 0 || (m > 0 && (!images || !params)))
            return fail(CM_ERR_INVALID_ARGUMENT, "set_particles: missing images");
        if (m == 0) return CM_OK;
        const size_t ni = (size_t)m * n * n;
        if (cudaMalloc(&img, sizeof(double2) * ni) != cudaSuccess ||
            cudaMalloc(&ip, sizeof(double) * 6 * (size_t)m) != cudaSuccess) {
            release();
            return fail(CM_ERR_CUDA, "set_particles: device allocation failed");
        }
        if (cudaMemcpyAsync(img, images, sizeof(double2) * ni, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaMemcpyAsync(ip, params, sizeof(double) * 6 * (size_t)m, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            release();
            return fail(CM_ERR_CUDA, "set_particles: upload failed");
        }
        n_images = m;
        return CM_OK;
    }
};

// images == NULL in a call selects the resident set, which must hold as many images
inline int particles_of(int n_images, const double* images, const double* params, const ParticleDev* res,
                        bool* host) {
    *host = images != nullptr;
    if (images) return params ? CM_OK : fail(CM_ERR_INVALID_ARGUMENT, "image_params missing");
    if (!res || res->n_images == 0) return fail(CM_ERR_STATE, "no images given and none resident (cm_set_particles)");
    if (res->n_images != n_images) return fail(CM_ERR_INVALID_ARGUMENT, "n_images differs from the resident particle set");
    return CM_OK;
}

// Device allocations of one call, released on every exit path.
struct BpBuffers {
    std::vector<void*> ptrs;
    ~BpBuffers() {
        for (void* q : ptrs) cudaFree(q);
    }
    template <typename T>
    int put(T** dst, const T* src, size_t count, cudaStream_t st) {
        *dst = nullptr;
        if (count == 0) return CM_OK;
        void* q = nullptr;
        if (cudaMalloc(&q, sizeof(T) * count) != cudaSuccess)
            return fail(CM_ERR_CUDA, "backproject: device allocation failed");
        ptrs.push_back(q);
        *dst = static_cast<T*>(q);
        if (src && cudaMemcpyAsync(q, src, sizeof(T) * count, cudaMemcpyHostToDevice, st) != cudaSuccess)
            return fail(CM_ERR_CUDA, "backproject: upload failed");
        return CM_OK;
    }
};

// Host side: validation, the component list and rotations, launch, finalize.
// `stage` = [weight L | numerator L complex] on the device (ImplBase::acc_stage).
inline int backproject_run(int n, const cm_bp_input* in, double* stage, cudaStream_t st,
                           const ParticleDev* resident = nullptr) {
    if (!in) return fail(CM_ERR_INVALID_ARGUMENT, "backproject: null input");
    if (in->kernel_kind != 0 && in->kernel_kind != 1)
        return fail(CM_ERR_INVALID_ARGUMENT, "backproject: unknown kernel kind");
    if (in->kernel_kind == 0 && !(in->bandwidth > 0.0))
        return fail(CM_ERR_INVALID_ARGUMENT, "gaussian kernel bandwidth must be positive");
    if (in->n_images < 0 || in->n_poses < 0 || in->n_shifts < 0 || in->n_entries < 0)
        return fail(CM_ERR_INVALID_ARGUMENT, "backproject: negative count");
    if (in->n_entries > 0 && (!in->entry_particle || !in->entry_candidate || !in->entry_posterior ||
                              !in->poses || !in->shifts || in->n_shifts == 0))
        return fail(CM_ERR_INVALID_ARGUMENT, "backproject: null input array");
    bool host_images = true;
    if (in->n_entries > 0) CKS(particles_of(in->n_images, in->images, in->image_params, resident, &host_images));
    const unsigned long long ncand = (unsigned long long)in->n_poses * (unsigned long long)in->n_shifts;
    for (long long e = 0; e < in->n_entries; ++e) {
        if (in->entry_particle[e] < 0 || in->entry_particle[e] >= in->n_images)
            return fail(CM_ERR_INVALID_ARGUMENT, "backproject: posterior row names an absent particle");
        if ((unsigned long long)in->entry_candidate[e] >= ncand)
            return fail(CM_ERR_INVALID_ARGUMENT, "backproject: candidate index outside the grid");
    }
    // frequency_components(n, min(cutoff, n)) (slice.cpp:7-22), storage-scan order
    const double cutoff = in->radius_cutoff < 0.0 ? double(n) : in->radius_cutoff;
    const double rc = std::min(cutoff, double(n));
    std::vector<int2> comps;
    comps.reserve((size_t)n * n);
    for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
            const int k = a < n / 2 ? a : a - n, l = b < n / 2 ? b : b - n;
            if (rc >= 0.0 && std::lround(std::hypot(double(k), double(l))) > std::lround(rc)) continue;
            comps.push_back(make_int2(k, l));
        }
    std::vector<double> mats(9 * (size_t)in->n_poses);
    for (int q = 0; q < in->n_poses; ++q) bp_rotation(in->poses + 3 * (size_t)q, mats.data() + 9 * (size_t)q);

    const size_t L = (size_t)n * n * n;
    if (cudaMemsetAsync(stage, 0, sizeof(double) * 3 * L, st) != cudaSuccess)
        return fail(CM_ERR_CUDA, "backproject: memset failed");
    BpBuffers bufs;
    BpDev p{};
    double2* img = nullptr;
    double *ipar = nullptr, *dm = nullptr, *post = nullptr;
    int2 *shf = nullptr, *cmp = nullptr;
    long long* ep = nullptr;
    unsigned* ec = nullptr;
    if (in->n_entries > 0) {
        if (host_images) {
            CKS(bufs.put(&img, reinterpret_cast<const double2*>(in->images), (size_t)in->n_images * n * n, st));
            CKS(bufs.put(&ipar, in->image_params, (size_t)in->n_images * 6, st));
        } else {
            img = resident->img;
            ipar = resident->ip;
        }
        CKS(bufs.put(&dm, mats.data(), mats.size(), st));
        CKS(bufs.put(&shf, reinterpret_cast<const int2*>(in->shifts), (size_t)in->n_shifts, st));
        CKS(bufs.put(&cmp, comps.data(), comps.size(), st));
        CKS(bufs.put(&ep, in->entry_particle, (size_t)in->n_entries, st));
        CKS(bufs.put(&ec, in->entry_candidate, (size_t)in->n_entries, st));
        CKS(bufs.put(&post, in->entry_posterior, (size_t)in->n_entries, st));
        p = BpDev{img, ipar, dm, shf, cmp, ep, ec, post, stage, reinterpret_cast<double2*>(stage + L),
                  in->n_entries, (int)comps.size(), n, in->n_shifts, in->bandwidth};
        const char* direct = getenv("CM_BP_DIRECT");
        if (!comps.empty() && !(direct && direct[0] == '1')) {
            // group the nonzero entries by pose (stable: row order within a pose)
            std::vector<int> cnt(in->n_poses + 1, 0);
            for (long long e = 0; e < in->n_entries; ++e)
                if (in->entry_posterior[e] > 0.0) ++cnt[in->entry_candidate[e] / (unsigned)in->n_shifts];
            std::vector<int> pose_of, off{0};
            std::vector<int> slot(in->n_poses, -1);
            for (int q = 0; q < in->n_poses; ++q)
                if (cnt[q] > 0) {
                    slot[q] = (int)pose_of.size();
                    pose_of.push_back(q);
                    off.push_back(off.back() + cnt[q]);
                }
            std::vector<int> fill(off.begin(), off.end() - 1);
            std::vector<int> gpart(off.back());
            std::vector<int2> gsh(off.back());
            std::vector<double> gpost(off.back());
            for (long long e = 0; e < in->n_entries; ++e)
                if (in->entry_posterior[e] > 0.0) {
                    const int at = fill[slot[in->entry_candidate[e] / (unsigned)in->n_shifts]]++;
                    gpart[at] = (int)in->entry_particle[e];
                    gsh[at] = reinterpret_cast<const int2*>(in->shifts)[in->entry_candidate[e] % (unsigned)in->n_shifts];
                    gpost[at] = in->entry_posterior[e];
                }
            const int nused = (int)pose_of.size();
            const int ncomp = (int)comps.size();
            // pose batches bounded to ~1 GB of (Z, Wt)
            const int batch = (int)std::max<size_t>(1, std::min<size_t>(std::min<size_t>((size_t)nused, (size_t)65535), (size_t(1) << 30) / (24 * (size_t)ncomp)));
            BpGroup g{};
            int *d_pose = nullptr, *d_off = nullptr;
            double2* Z = nullptr;
            double* Wt = nullptr;
            CKS(bufs.put(&d_pose, pose_of.data(), pose_of.size(), st));
            CKS(bufs.put(&d_off, off.data(), off.size(), st));
            CKS(bufs.put(&Z, (const double2*)nullptr, (size_t)batch * ncomp, st));
            CKS(bufs.put(&Wt, (const double*)nullptr, (size_t)batch * ncomp, st));
            double2* ph = nullptr;
            CKS(bufs.put(&ph, (const double2*)nullptr, (size_t)n, st));
            bp_roots_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, ph);
            int* d_gpart = nullptr;
            int2* d_gsh = nullptr;
            double* d_gpost = nullptr;
            CKS(bufs.put(&d_gpart, gpart.data(), gpart.size(), st));
            CKS(bufs.put(&d_gsh, gsh.data(), gsh.size(), st));
            CKS(bufs.put(&d_gpost, gpost.data(), gpost.size(), st));
            g = BpGroup{d_pose, d_off, Z, Wt, ph, d_gpart, d_gsh, d_gpost};
            for (int u0 = 0; u0 < nused; u0 += batch) {
                const dim3 grid((ncomp + 127) / 128, std::min(batch, nused - u0));
                bp_gather_kernel<<<grid, 128, sizeof(double2) * n, st>>>(p, g, u0);
                if (in->kernel_kind == 0)
                    bp_spread_kernel<0><<<grid, 128, 0, st>>>(p, g, u0);
                else
                    bp_spread_kernel<1><<<grid, 128, 0, st>>>(p, g, u0);
                if (cudaGetLastError() != cudaSuccess) return fail(CM_ERR_CUDA, "backproject: launch failed");
            }
        } else if (!comps.empty()) {
            const int cblocks = ((int)comps.size() + 127) / 128;
            const long long total = in->n_entries * cblocks;
            int sms = 148, dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const long long grid = std::min<long long>(total, (long long)sms * 16);
            if (in->kernel_kind == 0)
                bp_scatter_kernel<0><<<(unsigned)grid, 128, 0, st>>>(p, total, cblocks);
            else
                bp_scatter_kernel<1><<<(unsigned)grid, 128, 0, st>>>(p, total, cblocks);
            if (cudaGetLastError() != cudaSuccess) return fail(CM_ERR_CUDA, "backproject: launch failed");
        }
    }
    bp_friedel_kernel<<<(unsigned)std::min<size_t>((L + 255) / 256, 148 * 32), 256, 0, st>>>(
        n, stage, reinterpret_cast<double2*>(stage + L));
    if (cudaGetLastError() != cudaSuccess) return fail(CM_ERR_CUDA, "backproject: launch failed");
    // the staging buffers are freed at scope exit: wait for the kernels reading them
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(CM_ERR_CUDA, "backproject: kernel failed");
    return CM_OK;
}

} // namespace cm
