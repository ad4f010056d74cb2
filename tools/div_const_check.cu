// Exhaustive check of div_by_const_rn (paper_2602_22158_b200/csrc/kernels/ieee_div.cuh)
// against __fdiv_rn: every one of the 2^32 float bit patterns a, for each divisor b given
// (the trainer's bias corrections 1 - beta^t rounded to float, plus random divisors), with
// y = const_reciprocal(b) as the trainer computes it. Results must be bitwise equal (NaN
// payloads aside). Usage: div_const_check <t_max> <n_random> [beta ...]; prints one JSON line.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "ieee_div.cuh"
#include "tailor/device.hpp"

using tailor::dev::div_by_const_rn;

__global__ void check_kernel(const float* bs, const float* ys, int nb, unsigned long long* mismatches,
                             unsigned int* first_bad) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (int k = 0; k < nb; ++k) {
        const float b = bs[k], y = ys[k];
        unsigned long long bad = 0;
        for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < (1ull << 32); i += stride) {
            const float a = __uint_as_float(static_cast<unsigned int>(i));
            const float p = div_by_const_rn(a, b, y), q = __fdiv_rn(a, b);
            const bool same = __float_as_uint(p) == __float_as_uint(q) || (p != p && q != q);
            if (!same) {
                ++bad;
                atomicCAS(&first_bad[k], 0xFFFFFFFFu, static_cast<unsigned int>(i));
            }
        }
        if (bad) atomicAdd(&mismatches[k], bad);
    }
}

int main(int argc, char** argv) {
    const int tmax = argc > 1 ? std::atoi(argv[1]) : 200;
    const int nrand = argc > 2 ? std::atoi(argv[2]) : 50;
    std::vector<double> betas;
    for (int i = 3; i < argc; ++i) betas.push_back(std::atof(argv[i]));
    if (betas.empty()) betas = {0.9, 0.999};
    std::vector<float> bs;
    for (double beta : betas)
        for (int t = 1; t <= tmax; ++t) bs.push_back(static_cast<float>(1.0 - std::pow(beta, static_cast<double>(t))));
    std::mt19937 rng(1234);
    std::uniform_real_distribution<double> ex(-20.0, 0.0);
    for (int i = 0; i < nrand; ++i) bs.push_back(static_cast<float>(std::exp2(ex(rng))));
    std::vector<float> ys(bs.size());
    for (std::size_t i = 0; i < bs.size(); ++i) ys[i] = tailor::dev::const_reciprocal(bs[i]);
    float *d_b, *d_y;
    unsigned long long* d_m;
    unsigned int* d_f;
    const int nb = static_cast<int>(bs.size());
    cudaMalloc(&d_b, nb * sizeof(float));
    cudaMalloc(&d_y, nb * sizeof(float));
    cudaMalloc(&d_m, nb * sizeof(unsigned long long));
    cudaMalloc(&d_f, nb * sizeof(unsigned int));
    cudaMemcpy(d_b, bs.data(), nb * sizeof(float), cudaMemcpyHostToDevice);
    cudaMemcpy(d_y, ys.data(), nb * sizeof(float), cudaMemcpyHostToDevice);
    cudaMemset(d_m, 0, nb * sizeof(unsigned long long));
    cudaMemset(d_f, 0xFF, nb * sizeof(unsigned int));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    check_kernel<<<sms * 8, 256>>>(d_b, d_y, nb, d_m, d_f);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        return 2;
    }
    std::vector<unsigned long long> m(nb);
    std::vector<unsigned int> f(nb);
    cudaMemcpy(m.data(), d_m, nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemcpy(f.data(), d_f, nb * sizeof(unsigned int), cudaMemcpyDeviceToHost);
    unsigned long long total = 0;
    int bad_divisors = 0;
    for (int k = 0; k < nb; ++k) {
        total += m[k];
        if (m[k]) {
            if (bad_divisors < 5)
                std::fprintf(stderr, "divisor %.9g (y %.9g): %llu mismatches, first a = 0x%08x\n", bs[k], ys[k], m[k], f[k]);
            ++bad_divisors;
        }
    }
    std::printf("{\"divisors\": %d, \"values_per_divisor\": 4294967296, \"mismatches\": %llu, \"bad_divisors\": %d}\n", nb,
                total, bad_divisors);
    return total ? 1 : 0;
}
