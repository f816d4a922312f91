// em_refine driver -- TEST INFRASTRUCTURE.
//
// Runs the reference's production entry em_refine (refine.hpp:54-55,
// refine.cpp:102-266) in regularized mode on a simulated particle set through
// the reference's own public API. oracle/Makefile links it twice from the same
// source:
//   _ref/em_drive_ref    the unmodified reference library (all host, FFTW shim)
//   _ref/em_drive_b200   the same objects with the drop-in adapters linked in:
//                        regularizer_b200.cpp (m_step), params_b200.cpp
//                        (scale_data), fourier_b200.cpp (fft3_centered), i.e.
//                        the M-step block of refine.cpp:174-183 / 237-250 on
//                        the B200
//
//   em_drive <n> <particles> <max_iters> <inner_iters> <angular_step> <trans_radius> <threads> [out.bin]
//
// Prints one JSON line (wall seconds of em_refine, iterations, resolution,
// ||volume||) and writes the combined volume as raw doubles when asked.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "cryomap/orientation.hpp"
#include "cryomap/phantom.hpp"
#include "cryomap/refine.hpp"
#include "cryomap/simulate.hpp"

using namespace cryomap;

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: em_drive n particles max_iters inner_iters step trans threads [out]\n");
        return 2;
    }
    const int n = std::atoi(argv[1]), np = std::atoi(argv[2]);
    const int max_iters = std::atoi(argv[3]), inner = std::atoi(argv[4]);
    const double step = std::atof(argv[5]);
    const int trans = std::atoi(argv[6]), threads = std::atoi(argv[7]);
    const double voxel = 1.5;
    try {
        const int blobs = std::max(4, (int)std::lround(0.05 * n * n * n / 270.0));
        Volume3D truth = generate_phantom(random_phantom_spec(blobs, n, 55), n, voxel);
        OrientationGrid grid = make_orientation_grid(n, step, 0);
        PoseSamplerSpec sampler;
        sampler.kind = PoseSamplerSpec::Kind::grid;
        sampler.grid = &grid;
        const KernelSpec kernel{KernelKind::gaussian, 2.0};
        CTFParams ctf;
        ctf.identity_flag = true;
        double rms = 0.0, mx = 0.0;
        for (double v : truth.data) {
            rms += v * v;
            mx = std::max(mx, std::fabs(v));
        }
        rms = std::sqrt(rms / double(truth.data.size()));
        ParticleSet parts = simulate_particles(truth, np, sampler, ctf, 0.5 * rms * n, 77, kernel, threads);

        RefineConfig config;
        config.mode = RefineMode::regularized;
        config.kernel = kernel;
        config.angular_step_deg = step;
        config.trans_radius = trans;
        config.max_iters = max_iters;
        config.seed = 3;
        config.threads = threads;
        config.init_lowpass_A = 6.0;
        config.eps = 0.1 * mx;
        config.inner_iters = inner;

        const auto t0 = std::chrono::steady_clock::now();
        RefineResult res = em_refine(parts, truth, config);
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        double norm = 0.0;
        for (double v : res.volume.data) norm += v * v;
        std::printf("{\"n\": %d, \"particles\": %d, \"iterations\": %d, \"seconds\": %.6f, "
                    "\"resolution_shell\": %.6f, \"volume_norm\": %.17g, \"converged\": %d}\n",
                    n, np, res.iterations, secs, res.resolution.crossing_shell, std::sqrt(norm),
                    res.converged ? 1 : 0);
        if (argc > 8) {
            FILE* f = std::fopen(argv[8], "wb");
            if (!f) return 3;
            std::fwrite(res.volume.data.data(), sizeof(double), res.volume.data.size(), f);
            std::fwrite(res.half_a.data.data(), sizeof(double), res.half_a.data.size(), f);
            std::fclose(f);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "em_drive: %s\n", e.what());
        return 1;
    }
    return 0;
}
