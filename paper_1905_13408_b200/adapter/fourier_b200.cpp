// Drop-in for fft3_centered (fourier.hpp:24; reference fourier.cpp:109) on the B200.
//
// em_refine turns every M-step result into the spectrum the next E-step and the
// FSC read (refine.cpp:138, 182; fsc.cpp:141-144): V = fft3_centered(x). The
// reference runs a full-grid fp64 FFTW c2c of the half-shifted volume on the
// host. Here:
//   * x is the volume m_step just returned (cm_adapter.hpp identity): the
//     spectrum of the RESIDENT result is unpacked on the device
//     (cm_get_spectrum, centered) -- nothing is uploaded;
//   * any other volume: uploaded once and transformed on the device
//     (cm_fft3_centered: R2C + y + z passes, (-1)^(a+b+c) sign for the half
//     shift).
// Only the full complex grid crosses back to the host (the FourierVolume the
// API returns by value).
//
// Integration: compile the reference's fourier.cpp with
// -Dfft3_centered=fft3_centered_fftw (every other transform -- 2D particle
// images, inverse transforms of the baseline modes -- stays the reference's)
// and link this file; see INTEGRATION.md.
#include "cm_adapter.hpp"
#include "cryomap/fourier.hpp"

namespace cryomap {

FourierVolume fft3_centered(const Volume3D& v) {
    cm_adapter::Slot& s = cm_adapter::slot(v.side_n);
    FourierVolume F(v.side_n, v.voxel_size);
    double* out = reinterpret_cast<double*>(F.data.data());
    if (cm_adapter::is_result(s, v))
        cm_adapter::check(cm_get_spectrum(s.ctx.get(), 1, out));
    else
        cm_adapter::check(cm_fft3_centered(cm_adapter::transform_context(s, v.side_n), v.data.data(), out));
    return F;
}

} // namespace cryomap
