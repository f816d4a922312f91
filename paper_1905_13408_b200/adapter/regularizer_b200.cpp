// Drop-in replacement for /root/reference/proj/src/regularizer.cpp.
//
// Implements every function declared in the reference's UNCHANGED header
// include/cryomap/regularizer.hpp (validate_reg_config :37, compute_weights
// :45-46, smoothed_tv_value :51-52, smoothed_tv_gradient :56-57, data_gradient
// :62, prox_l1 :65, penalized_objective :83-85, m_step :98-100) by calling the
// B200 solver through its C ABI (include/cm_api.h). Link this file instead of
// regularizer.cpp, plus libcm.so; nothing else in the reference changes.
//
// Status codes are rethrown as the reference's exception types
// (errors.hpp:7-30). Contexts are cached per thread and side length
// (cm_adapter.hpp), so em_refine's repeated m_step calls (refine.cpp:181, 249)
// reuse device memory, the accumulator scale_data made resident is not
// uploaded twice, and fft3_centered of the returned volume reads the resident
// result (params_b200.cpp, fourier_b200.cpp). Precision: CM_PRECISION=64
// (default here: the reference's fp64 tests pass unchanged) or 32 (product
// mode, 1e-5 objective parity). Devices: CM_DEVICES (default "0").
#include <string>
#include <vector>

#include "cm_adapter.hpp"
#include "cryomap/regularizer.hpp"

namespace cryomap {

namespace {

using cm_adapter::check;

cm_reg_config to_c(const RegConfig& c) {
    cm_reg_config r{};
    r.alpha = c.alpha;
    r.beta = c.beta;
    r.gamma = c.gamma;
    r.eps = c.eps;
    r.eps_prime = c.eps_prime;
    r.mu = c.mu;
    r.inner_iters = c.inner_iters;
    r.step_rule = c.step_rule == RegConfig::StepRule::fixed ? 1 : 0;
    r.fixed_step = c.fixed_step;
    r.refresh = c.refresh == RegConfig::Refresh::per_m_step ? 1 : 0;
    r.convex_mode = c.convex_mode ? 1 : 0;
    return r;  // extensions zero: reference ISTA semantics
}

ObjectiveValue to_obj(const double* v) {
    ObjectiveValue o;
    o.fit = v[0];
    o.l1 = v[1];
    o.tv_smooth = v[2];
    o.tv_linear = v[3];
    o.restraint = v[4];
    o.lognorm_l1 = v[5];
    o.lognorm_tv = v[6];
    return o;
}


} // namespace

void validate_reg_config(const RegConfig& config) {
    cm_reg_config c = to_c(config);
    // cm_derive_config validates too; here only the RegConfig checks
    // (regularizer.cpp:33-42 semantics, same messages)
    if (c.alpha < 0.0 || c.beta < 0.0 || c.gamma < 0.0)
        throw InvalidArgument("regularizer: alpha/beta/gamma must be >= 0");
    if (c.eps <= 0.0 || c.eps_prime <= 0.0 || c.mu <= 0.0)
        throw InvalidArgument("regularizer: eps/eps_prime/mu must be > 0");
    if (c.inner_iters < 1) throw InvalidArgument("regularizer: inner_iters must be >= 1");
    if (c.step_rule == 1 && c.fixed_step <= 0.0)
        throw InvalidArgument("regularizer: fixed step must be > 0");
}

WeightFields compute_weights(const Volume3D& x_prev, double eps, double eps_prime,
                             bool convex_mode) {
    WeightFields w;
    w.w_l1.resize(x_prev.data.size());
    w.w_tv.resize(x_prev.data.size());
    check(cm_compute_weights_n(x_prev.side_n, x_prev.data.data(), eps, eps_prime,
                               convex_mode ? 1 : 0, w.w_l1.data(), w.w_tv.data()));
    return w;
}

double smoothed_tv_value(const Volume3D& v, double mu, const std::vector<double>* w_tv) {
    double out = 0.0;
    check(cm_smoothed_tv_value_n(v.side_n, v.data.data(), mu, w_tv ? w_tv->data() : nullptr,
                                 &out));
    return out;
}

Volume3D smoothed_tv_gradient(const Volume3D& v, double mu, const std::vector<double>* w_tv) {
    Volume3D out(v.side_n, v.voxel_size);
    check(cm_smoothed_tv_gradient_n(v.side_n, v.data.data(), mu,
                                    w_tv ? w_tv->data() : nullptr, out.data.data()));
    return out;
}

Volume3D data_gradient(const Volume3D& x, const AccumulatorPair& acc) {
    if (x.side_n != acc.side_n) throw GridMismatch("data_gradient: side_n differs");
    cm_ctx* ctx = cm_adapter::component_context(acc);
    Volume3D g(x.side_n, x.voxel_size);
    check(cm_data_gradient(ctx, x.data.data(), g.data.data()));
    return g;
}

Volume3D prox_l1(const Volume3D& x_dash, const std::vector<double>& thresholds) {
    Volume3D out(x_dash.side_n, x_dash.voxel_size);
    out.data.resize(x_dash.data.size());
    check(cm_prox_l1_n((long long)x_dash.data.size(), x_dash.data.data(), thresholds.data(),
                       out.data.data()));
    return out;
}

ObjectiveValue penalized_objective(const Volume3D& x, const AccumulatorPair& acc,
                                   const RegConfig& config, const Volume3D& x_anchor,
                                   const Volume3D& x_weights_source) {
    validate_reg_config(config);
    cm_ctx* ctx = cm_adapter::component_context(acc);
    const cm_reg_config c = to_c(config);
    double o[7];
    check(cm_penalized_objective(ctx, x.data.data(), &c, x_anchor.data.data(),
                                 x_weights_source.data.data(), o));
    return to_obj(o);
}

Volume3D m_step(const AccumulatorPair& acc, const Volume3D& x_init, const Volume3D& x_anchor,
                const RegConfig& config, std::vector<MStepTraceRow>* trace) {
    validate_reg_config(config);
    if (x_init.side_n != acc.side_n || x_anchor.side_n != acc.side_n)
        throw GridMismatch("m_step: side_n differs");
    cm_adapter::Slot& s = cm_adapter::slot(acc.side_n);
    cm_ctx* ctx = s.ctx.get();
    const cm_reg_config c = to_c(config);
    std::vector<cm_trace_row> rows(trace ? (size_t)config.inner_iters : 0);
    Volume3D out(x_init.side_n, x_init.voxel_size);
    cm_solve_stats st{};
    // the accumulator scale_data(acc) made resident is not uploaded again
    // (em_refine: refine.cpp:175-181); x_init and x_anchor may be one object
    // (refine.cpp:181): pass one pointer
    cm_adapter::upload_acc(s, acc);
    const double* xa = (&x_init == &x_anchor) ? x_init.data.data() : x_anchor.data.data();
    check(cm_set_volumes(ctx, x_init.data.data(), xa));
    const int rc = cm_solve(ctx, &c, trace ? rows.data() : nullptr, trace ? config.inner_iters : 0, &st);
    if (trace)
        for (int r = 0; r < st.trace_rows; ++r)
            trace->push_back({to_obj(rows[r].before), to_obj(rows[r].after), rows[r].step});
    check(rc);
    check(cm_get_volume(ctx, out.data.data()));
    cm_adapter::note_result(s, out);  // fft3_centered(out) reads the resident result
    return out;
}

} // namespace cryomap
