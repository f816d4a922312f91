// Drop-in for scale_data (params.hpp:22; reference params.cpp:9-26) on the B200.
//
// The reference whitens the full fp64 grid, runs a host inverse FFT and takes
// the RMS; here the accumulator goes to the device once (cm_set_accumulator:
// symmetry residue, Hermitian projection, half-spectrum conversion) and s_y is
// the Parseval sum of the whitened half spectrum (cm_scale_data), no FFT at
// all. The accumulator stays resident, so em_refine's m_step(acc, ...) that
// follows (refine.cpp:175-181, 238-249) does not upload it again.
//
// Integration: compile the reference's params.cpp with -Dscale_data=scale_data_fftw
// (its other functions -- derive_config, effective_eps_prime,
// validate_refine_config, sweep_grid -- are host configuration logic and stay
// the reference's) and link this file; see INTEGRATION.md.
#include "cm_adapter.hpp"
#include "cryomap/params.hpp"

namespace cryomap {

DataScales scale_data(const AccumulatorPair& acc) {
    if (!acc.finalized)  // params.cpp:10-11
        throw NonHermitianAccumulator("scale_data: accumulator is not finalized");
    cm_adapter::Slot& s = cm_adapter::slot(acc.side_n);
    cm_adapter::upload_acc(s, acc);
    DataScales d;
    cm_adapter::check(cm_scale_data(s.ctx.get(), &d.s_y, &d.s_n));
    return d;
}

} // namespace cryomap
