// Micro-benchmark: does a plane-chunked y-inverse -> x-C2R schedule keep the
// intermediate spectrum in L2? Times full-volume vs chunked launch orders.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1905_13408_b200/csrc \
//        profiles/micro/l2_chunk.cu -o build/l2_chunk
#include <cstdio>
#include <vector>
#include <cmath>
#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "xfft.cuh"

using namespace cm;
constexpr int N = 512, Nh = N / 2;
using G = Geo<float, N>;
using XG = XGeo<float, N>;

__global__ void fill(float2* s, size_t n) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x)
        s[q] = make_float2(__sinf(q * 1e-3f), __cosf(q * 7e-4f));
}

int main(int argc, char** argv) {
    const size_t H = (size_t)N * N * Nh, L = (size_t)N * N * N;
    float2 *S, *tw;
    float* g;
    cudaMalloc(&S, H * 8);
    cudaMalloc(&g, L * 4);
    cudaMalloc(&tw, N * 8);
    std::vector<float2> h(N);
    for (int q = 0; q < N; ++q) h[q] = make_float2(cos(-2 * M_PI * q / N), sin(-2 * M_PI * q / N));
    cudaMemcpy(tw, h.data(), N * 8, cudaMemcpyHostToDevice);
    fill<<<1184, 256>>>(S, H);
    cudaFuncSetAttribute(ypass_kernel<float, N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YSmem<float, N>::bytes);
    cudaFuncSetAttribute(xfft_kernel<float, N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XG::SMEM);
    int occ = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xfft_kernel<float, N, 0>, XG::NT, XG::SMEM);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int xgrid = sms * occ;
    const SpecLayout nat = spec_layout((long long)N * Nh, 0, N);
    auto run = [&](int B) {
        for (int p0 = 0; p0 < N; p0 += B) {
            YParams<float> yp{S + (size_t)p0 * N * Nh, tw, nullptr, nullptr, nullptr, nat, nat, B};
            ypass_kernel<float, N, false><<<dim3(Nh / G::TWY, B), G::TWY * G::TY, YSmem<float, N>::bytes>>>(yp);
            XfParams<float> xp{S + (size_t)p0 * N * Nh, g + (size_t)p0 * N * N, tw, nullptr, nullptr, 1.0, B * N};
            const int grid = std::min(xgrid, (B * N + XG::LPC - 1) / XG::LPC);
            xfft_kernel<float, N, 0><<<grid, XG::NT, XG::SMEM>>>(xp);
        }
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int Bs[] = {512, 128, 64, 32, 16, 8};
    for (int B : Bs) {
        run(B);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) run(B);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("chunk %4d planes: %.3f ms per y-inverse + C2R pass (err %s)\n", B, ms / 10,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
