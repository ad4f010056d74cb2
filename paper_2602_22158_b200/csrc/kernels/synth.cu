// K5 — synthetic snapshot generator, bit-exact with the CPU restatement
// (oracle/ref_driver.cpp gen, oracle/tailor_oracle.py) of SURVEY §8(d):
//   W_0(e)  = 0.02f * u(seed, 0, e)                       (init_state, R/src/gradients.cpp:51-66)
//   W_j(e)  = W_{j-1}(e) + (sign_j(e) ? -sigma_j(m) : sigma_j(m))   FP32, round-to-nearest
//   m_k(e)  = 0.1f * u(seed ^ 0xA5, k, e)
//   v_k(e)  = |0.01f * u(seed ^ 0x5A, k, e)|
//   weights = bf16_round(W_k)                              (R/include/tailor/bf16.hpp:12-20)
// with u = unit_noise (R/src/gradients.cpp:17-23) and sign_j(e) the top bit of
// the same three-round counter hash salted with 0x51A7E5. Every FP op is an
// explicit _rn intrinsic (and the file builds with --fmad=false), mirroring
// the reference's -ffp-contract=off.
#include <algorithm>

#include "tailor/bf16.hpp"
#include "tailor/device.hpp"

namespace tailor::dev {

namespace {

constexpr std::uint64_t kSignSalt = 0x51A7E5ULL;
constexpr std::uint64_t kMSalt = 0xA5ULL;
constexpr std::uint64_t kVSalt = 0x5AULL;

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

__device__ __forceinline__ std::uint64_t hash3(std::uint64_t seed, std::uint64_t t, std::uint64_t e) {
    std::uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ULL);
    h = mix64(h ^ (t * 0xD1B54A32D192ED03ULL));
    return mix64(h ^ (e * 0x8CB92BA72F3D8DD7ULL));
}

__device__ __forceinline__ float unit_noise(std::uint64_t seed, std::uint64_t t, std::uint64_t e) {
    const double unit = __dmul_rn(__ull2double_rn(hash3(seed, t, e) >> 11), 0x1.0p-53);
    return __double2float_rn(__dadd_rn(__dmul_rn(2.0, unit), -1.0));
}

__device__ __forceinline__ float master_step(float w, const float* __restrict__ sigma, int M, std::uint32_t module,
                                             std::uint64_t seed, int j, std::uint64_t e) {
    const float s = sigma[(j - 1) * M + module];
    const bool neg = (hash3(seed ^ kSignSalt, static_cast<std::uint64_t>(j), e) >> 63) != 0;
    return __fadd_rn(w, neg ? -s : s);
}

template <typename T>
__device__ __forceinline__ int find_by_begin(const T* __restrict__ xs, std::uint32_t n, std::uint64_t v) {
    int lo = 0, hi = static_cast<int>(n) - 1, ans = 0;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        if (xs[mid].begin <= v) {
            ans = mid;
            lo = mid + 1;
        } else {
            hi = mid - 1;
        }
    }
    return ans;
}

__global__ void synth_shard_kernel(const SynthGroup* __restrict__ groups, std::uint32_t ngroups,
                                   const SynthSlice* __restrict__ slices, const float* __restrict__ sigma, int M,
                                   std::uint64_t seed, int k0, int k1, OutPtrs outs,
                                   std::uint64_t total) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t v = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; v < total; v += stride) {
        const SynthGroup& g = groups[find_by_begin(groups, ngroups, v)];
        const std::uint64_t i = v - g.begin;
        const std::uint64_t go = g.group_first + i;
        if (go >= g.true_len) {
            for (int k = k0; k <= k1; ++k) {
                std::uint8_t* o = outs.p[k - k0];
#pragma unroll
                for (int f = 0; f < 3; ++f)
                    if (g.off[f] != ~0ULL) reinterpret_cast<float*>(o + g.off[f])[i] = 0.0f;
            }
            continue;
        }
        std::uint32_t s = g.slice_begin;
        while (s + 1 < g.slice_begin + g.slice_count && static_cast<std::int64_t>(go) >= slices[s + 1].group_offset) ++s;
        const std::uint64_t e = static_cast<std::uint64_t>(slices[s].model_offset + (static_cast<std::int64_t>(go) - slices[s].group_offset));
        float w = __fmul_rn(0.02f, unit_noise(seed, 0, e));
        if (k1 == 0) { // initial state only (the trainer's init_state)
            if (g.off[2] != ~0ULL) reinterpret_cast<float*>(outs.p[0] + g.off[2])[i] = w;
            continue;
        }
        for (int j = 1; j <= k1; ++j) {
            w = master_step(w, sigma, M, g.module, seed, j, e);
            if (j < k0) continue;
            std::uint8_t* o = outs.p[j - k0];
            if (g.off[0] != ~0ULL)
                reinterpret_cast<float*>(o + g.off[0])[i] = __fmul_rn(0.1f, unit_noise(seed ^ kMSalt, static_cast<std::uint64_t>(j), e));
            if (g.off[1] != ~0ULL)
                reinterpret_cast<float*>(o + g.off[1])[i] =
                    fabsf(__fmul_rn(0.01f, unit_noise(seed ^ kVSalt, static_cast<std::uint64_t>(j), e)));
            if (g.off[2] != ~0ULL) reinterpret_cast<float*>(o + g.off[2])[i] = w;
        }
    }
}

__global__ void synth_weights_kernel(const SynthTensor* __restrict__ tensors, std::uint32_t ntensors,
                                     const float* __restrict__ sigma, int M, std::uint64_t seed, int k0, int k1,
                                     OutPtrs outs, std::uint64_t total) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t v = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; v < total; v += stride) {
        const SynthTensor& t = tensors[find_by_begin(tensors, ntensors, v)];
        const std::uint64_t i = v - t.begin;
        const std::uint64_t e = static_cast<std::uint64_t>(t.model_offset) + i;
        float w = __fmul_rn(0.02f, unit_noise(seed, 0, e));
        for (int j = 1; j <= k1; ++j) {
            w = master_step(w, sigma, M, t.module, seed, j, e);
            if (j < k0) continue;
            reinterpret_cast<std::uint16_t*>(outs.p[j - k0] + t.dst_off)[i] = bf16_round_bits(__float_as_uint(w));
        }
    }
}

unsigned grid_for(std::uint64_t total) {
    const std::uint64_t want = (total + 255) / 256;
    return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(want, static_cast<std::uint64_t>(sm_count()) * 16)));
}

} // namespace

cudaError_t launch_synth_shard(const SynthGroup* d_groups, std::uint32_t ngroups, const SynthSlice* d_slices,
                               const float* d_sigma, int M, std::uint64_t seed, int k0, int k1,
                               OutPtrs d_outs, std::uint64_t total, cudaStream_t stream) {
    if (total == 0) return cudaSuccess;
    synth_shard_kernel<<<grid_for(total), 256, 0, stream>>>(d_groups, ngroups, d_slices, d_sigma, M, seed, k0, k1, d_outs, total);
    return cudaGetLastError();
}

cudaError_t launch_synth_weights(const SynthTensor* d_tensors, std::uint32_t ntensors, const float* d_sigma, int M,
                                 std::uint64_t seed, int k0, int k1, OutPtrs d_outs, std::uint64_t total,
                                 cudaStream_t stream) {
    if (total == 0) return cudaSuccess;
    synth_weights_kernel<<<grid_for(total), 256, 0, stream>>>(d_tensors, ntensors, d_sigma, M, seed, k0, k1, d_outs, total);
    return cudaGetLastError();
}

} // namespace tailor::dev
