// Per-iteration finalize: fixed-order reduction of the block partials of the
// z pass (fit) and the x-line sweep (penalties), trace row, monotone audit and
// tolerance test. One 256-thread block; deterministic.
#pragma once

#include "cm_common.cuh"
#include "kernels.cuh"

namespace cm {

struct FinParams {
    DevState* st;
    const double* part1; int nb1;   // xline partials [nb1][NP1]
    const double* part3; int nb3;   // zpass partials [nb3][NP3]
    double* trace;                  // [max_iters][15] or null
    double alpha, beta, gamma, invL;
    int epilogue;                   // 1: close the last row after the loop
    const double* sums;             // z-slab ranks: globally reduced partials [NP1+NP3]
};

constexpr int FIN_THREADS = 1024;

// thread-strided sums of the block partials; the loads of an unrolled group are
// independent (a dependent load chain per thread made this latency bound)
__device__ __forceinline__ void sum_partials(const double* part1, int nb1, const double* part3,
                                             int nb3, double (&s)[NP1 + NP3]) {
#pragma unroll
    for (int q = 0; q < NP1 + NP3; ++q) s[q] = 0.0;
    if (part1)
#pragma unroll 2
        for (int b = threadIdx.x; b < nb1; b += blockDim.x)
#pragma unroll
            for (int q = 0; q < NP1; ++q) s[q] += __ldcg(part1 + (size_t)b * NP1 + q);
    if (part3) {
        const double2* p3 = reinterpret_cast<const double2*>(part3);
        static_assert(NP3 == 2, "z partials are (quad, cross) pairs");
#pragma unroll 4
        for (int b = threadIdx.x; b < nb3; b += blockDim.x) {
            const double2 v = __ldcg(p3 + b);
            s[NP1] += v.x;
            s[NP1 + 1] += v.y;
        }
    }
}

// z-slab ranks: this rank's partials -> out[NP1 + NP3] (then all-reduced)
static __global__ void __launch_bounds__(FIN_THREADS) fin_local_kernel(const double* part1, int nb1,
                                                                       const double* part3, int nb3,
                                                                       double* out) {
    __shared__ double red[32 * (NP1 + NP3)];
    double s[NP1 + NP3];
    sum_partials(part1, nb1, part3, nb3, s);
    block_sum<NP1 + NP3>(s, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < NP1 + NP3; ++q) out[q] = s[q];
}

static __device__ __forceinline__ double surrogate7(const double* o) { return o[0] + o[1] + o[2] + o[4]; }

static __global__ void __launch_bounds__(FIN_THREADS) finalize_kernel(FinParams p) {
    __shared__ double red[32 * (NP1 + NP3)];
    pdl_trigger();
    pdl_wait();
    DevState* st = p.st;
    if (!p.epilogue && ld_done(st)) return;
    if (p.epilogue && !(st->stop_reason == 1 && st->audit)) return;

    double s[NP1 + NP3];
#pragma unroll
    for (int q = 0; q < NP1 + NP3; ++q) s[q] = 0.0;
    if (p.sums) {  // already reduced over ranks
        if (threadIdx.x != 0) return;
        for (int q = 0; q < NP1 + NP3; ++q) s[q] = p.sums[q];
    } else {
    // fixed assignment of blocks to threads + fixed tree => deterministic
    sum_partials(p.part1, p.nb1, p.part3, p.nb3, s);
    block_sum<NP1 + NP3>(s, red);
    if (threadIdx.x != 0) return;
    }

    // work on a register copy of the state: its fields load in one round trip
    // instead of a chain of dependent global loads by one thread
    DevState S = *st;
    [&] {
        const double fit = (s[NP1 + 0] - 2.0 * s[NP1 + 1]) * p.invL;
        const int i = p.epilogue ? S.max_iters : S.iter;
        double cur[7] = {fit,
                         p.alpha * s[0],
                         p.beta * s[1],
                         p.beta * s[2],
                         p.gamma * s[5],
                         p.alpha * s[3],
                         p.beta * s[4]};
        if (S.audit && i > 0) {
            double after[7];
            for (int q = 0; q < 7; ++q) after[q] = cur[q];
            if (S.refresh_inner) { // weights of x_{i-1} at x_i
                after[1] = p.alpha * s[6];
                after[2] = p.beta * s[7];
                after[3] = p.beta * s[8];
            }
            const double sb = surrogate7(S.before);
            const double sa = surrogate7(after);
            const double slack = S.audit_slack * fmax(1.0, fabs(sb));
            if (S.check_diverge && sa > sb + slack) {
                S.diverged_iter = i - 1;
                S.stop_reason = 3;
                S.done = 1;
                S.rows = i - 1;
                return;
            }
            if (p.trace) {
                double* row = p.trace + (size_t)(i - 1) * 15;
                for (int q = 0; q < 7; ++q) row[q] = S.before[q];
                for (int q = 0; q < 7; ++q) row[7 + q] = after[q];
                row[14] = S.step;
            }
            S.rows = i;
            if (S.tol_kind == 1) {
                const double rel = fabs(sb - sa) / fmax(fabs(sb), 1e-300);
                S.last_rel = rel;
                if (!p.epilogue && rel < S.tol) {
                    // stop with x_i as the result
                    S.stop_reason = 2;
                    S.done = 1;
                    S.iter = i;
                    return;
                }
            }
        }
        if (p.epilogue) return;
        for (int q = 0; q < 7; ++q) S.before[q] = cur[q];
        S.iter = i + 1;
        if (S.fista && S.restart && s[11] > 0.0) {
            // gradient restart: the momentum sequence starts over at the next
            // iteration (theta index iter - mom_base = 0: no momentum)
            S.mom_base = S.iter;
            ++S.restarts;
        }
        if (S.tol_kind == 2) {
            // scale-free step rule: ||x_{k+1} - x_k|| relative to the largest step so
            // far (the first steps are tiny under the Lipschitz step of the TV term)
            const double dn = sqrt(s[9]);
            S.step_max = fmax(S.step_max, dn);
            const double rel = dn / fmax(S.step_max, 1e-300);
            S.last_rel = rel;
            if (i >= 1 && rel < S.tol) {
                S.stop_reason = 2;
                S.done = 1;
                return;
            }
        }
        if (S.iter >= S.max_iters) {
            S.stop_reason = 1;
            S.done = 1;
        }
    }();
    *st = S;
}

} // namespace cm
