// K7 — device AdamW step over ZeRO rank partitions, bit-exact with the
// reference trainer step:
//   grad  g = c1*w + c2*u(seed, step, e)            synth_grad, R/src/gradients.cpp:25-49
//   m = b1*m + (1-b1)*g ; v = b2*v + (1-b2)*(g*g)    adamw_update_group, R/src/adamw.cpp:10-47
//   w = w - lr * ( (m/bias1) / (sqrt(v/bias2) + eps) + wd*w )
// Coefficients are computed on the host in FP64 and rounded to FP32 once per
// group, as the reference does; the elementwise arithmetic is FP32 with
// explicit round-to-nearest intrinsics (IEEE div/sqrt, no FMA contraction;
// the file builds with --fmad=false), so every state bit matches. The
// non-finite check runs as a separate pass before any state is touched
// (apply_step's contract, R/src/adamw.cpp:49-60). Shard padding is never
// touched. Norm partials (sum g^2, sum step^2) are FP64 per block, combined in
// block order on the host: deterministic, not bitwise equal to the
// reference's sequential sums (they only feed log.jsonl).
#include <algorithm>

#include "tailor/bf16.hpp"
#include "tailor/device.hpp"

namespace tailor::dev {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

__device__ __forceinline__ float unit_noise_from(std::uint64_t prefix, std::uint64_t e) {
    const std::uint64_t h = mix64(prefix ^ (e * 0x8CB92BA72F3D8DD7ULL));
    const double unit = __dmul_rn(__ull2double_rn(h >> 11), 0x1.0p-53);
    return __double2float_rn(__dadd_rn(__dmul_rn(2.0, unit), -1.0));
}

__device__ __forceinline__ int find_group(const TrainGroup* __restrict__ g, std::uint32_t n, std::uint64_t v) {
    int lo = 0, hi = static_cast<int>(n) - 1, ans = 0;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        if (g[mid].begin <= v) {
            ans = mid;
            lo = mid + 1;
        } else {
            hi = mid - 1;
        }
    }
    return ans;
}

// Resolves virtual element v of a rank partition to (group, chunk index, global
// element id); returns false for shard padding.
__device__ __forceinline__ bool locate(const TrainGroup* __restrict__ groups, std::uint32_t ngroups,
                                       const SynthSlice* __restrict__ slices, std::uint64_t v, const TrainGroup*& g,
                                       std::uint64_t& i, std::uint64_t& e) {
    g = &groups[find_group(groups, ngroups, v)];
    i = v - g->begin;
    const std::uint64_t go = g->group_first + i;
    if (go >= g->true_len) return false;
    std::uint32_t s = g->slice_begin;
    while (s + 1 < g->slice_begin + g->slice_count && static_cast<std::int64_t>(go) >= slices[s + 1].group_offset) ++s;
    e = static_cast<std::uint64_t>(slices[s].model_offset + (static_cast<std::int64_t>(go) - slices[s].group_offset));
    return true;
}

__device__ __forceinline__ float grad_of(float w, const TrainParams& p, std::uint64_t e) {
    return __fadd_rn(__fmul_rn(p.state_coeff, w), __fmul_rn(p.noise_coeff, unit_noise_from(p.noise_prefix, e)));
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}

__global__ void __launch_bounds__(kThreads) grad_check_kernel(const TrainGroup* __restrict__ groups, std::uint32_t ngroups,
                                                              const SynthSlice* __restrict__ slices,
                                                              const std::uint8_t* __restrict__ part, std::uint64_t total,
                                                              TrainParams p, float* __restrict__ grad,
                                                              double* __restrict__ grad_partials,
                                                              unsigned int* __restrict__ nonfinite) {
    __shared__ double red[kThreads / 32];
    double acc = 0.0;
    bool bad = false;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t v = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; v < total; v += stride) {
        const TrainGroup* g;
        std::uint64_t i, e;
        if (!locate(groups, ngroups, slices, v, g, i, e)) continue;
        const float w = reinterpret_cast<const float*>(part + g->off_w)[i];
        const float gr = grad_of(w, p, e);
        grad[v] = gr;
        bad = bad || !isfinite(gr);
        acc += static_cast<double>(gr) * static_cast<double>(gr);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) grad_partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) adamw_update_kernel(const TrainGroup* __restrict__ groups, std::uint32_t ngroups,
                                                                const AdamCoef* __restrict__ coef, std::uint8_t* __restrict__ part,
                                                                const float* __restrict__ grad, std::uint64_t total,
                                                                double* __restrict__ delta_partials) {
    __shared__ double red[kThreads / 32];
    double acc = 0.0;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t v = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; v < total; v += stride) {
        const TrainGroup* g = &groups[find_group(groups, ngroups, v)];
        const std::uint64_t i = v - g->begin;
        if (g->group_first + i >= g->true_len) continue; // shard padding stays zero
        const AdamCoef c = coef[g->coef];
        float* wp = reinterpret_cast<float*>(part + g->off_w) + i;
        float* mp = reinterpret_cast<float*>(part + g->off_m) + i;
        float* vp = reinterpret_cast<float*>(part + g->off_v) + i;
        const float w = *wp;
        const float gr = grad[v];
        const float m = __fadd_rn(__fmul_rn(c.b1, *mp), __fmul_rn(c.one_minus_b1, gr));
        const float vv = __fadd_rn(__fmul_rn(c.b2, *vp), __fmul_rn(c.one_minus_b2, __fmul_rn(gr, gr)));
        const float m_hat = __fdiv_rn(m, c.bias1);
        const float v_hat = __fdiv_rn(vv, c.bias2);
        const float update = __fadd_rn(__fdiv_rn(m_hat, __fadd_rn(__fsqrt_rn(v_hat), c.eps)), __fmul_rn(c.wd, w));
        const float step = __fmul_rn(c.lr, update);
        *mp = m;
        *vp = vv;
        *wp = __fsub_rn(w, step);
        acc += static_cast<double>(step) * static_cast<double>(step);
    }
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) delta_partials[blockIdx.x] = s;
}

// K8 — consolidated BF16 weights from sharded FP32 masters (derive_weights,
// R/src/checkpoint.cpp:287-312): element i of a tensor lives at group offset
// go = group_offset + i, i.e. in rank go / chunk at position go % chunk.
__global__ void derive_weights_kernel(const WeightTensor* __restrict__ tensors, std::uint32_t ntensors,
                                      const std::uint8_t* const* __restrict__ parts, std::uint8_t* __restrict__ out,
                                      std::uint64_t total) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t v = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; v < total; v += stride) {
        int lo = 0, hi = static_cast<int>(ntensors) - 1, k = 0;
        while (lo <= hi) {
            const int mid = (lo + hi) >> 1;
            if (tensors[mid].begin <= v) {
                k = mid;
                lo = mid + 1;
            } else {
                hi = mid - 1;
            }
        }
        const WeightTensor& t = tensors[k];
        const std::uint64_t i = v - t.begin;
        const std::uint64_t go = t.group_offset + i;
        const std::uint64_t r = go / t.chunk, pos = go % t.chunk;
        const float w = reinterpret_cast<const float*>(parts[r] + t.master_off)[pos];
        reinterpret_cast<std::uint16_t*>(out + t.dst_off)[i] = bf16_round_bits(__float_as_uint(w));
    }
}

} // namespace

cudaError_t launch_derive_weights(const WeightTensor* d_tensors, std::uint32_t ntensors,
                                  const std::uint8_t* const* d_parts, std::uint8_t* d_out, std::uint64_t total,
                                  cudaStream_t s) {
    if (total == 0) return cudaSuccess;
    derive_weights_kernel<<<adamw_grid(total), kThreads, 0, s>>>(d_tensors, ntensors, d_parts, d_out, total);
    return cudaGetLastError();
}

unsigned adamw_grid(std::uint64_t total) {
    const std::uint64_t want = (total + kThreads - 1) / kThreads;
    return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(want, static_cast<std::uint64_t>(sm_count()) * 8)));
}

std::uint64_t noise_prefix(std::uint64_t seed, std::uint64_t step) {
    const auto mix = [](std::uint64_t z) {
        z ^= z >> 30;
        z *= 0xBF58476D1CE4E5B9ULL;
        z ^= z >> 27;
        z *= 0x94D049BB133111EBULL;
        z ^= z >> 31;
        return z;
    };
    return mix(mix(seed + 0x9E3779B97F4A7C15ULL) ^ (step * 0xD1B54A32D192ED03ULL));
}

cudaError_t launch_grad_check(const TrainGroup* d_groups, std::uint32_t ngroups, const SynthSlice* d_slices,
                              const std::uint8_t* d_part, std::uint64_t total, const TrainParams& p, float* d_grad,
                              double* d_grad_partials, unsigned int* d_nonfinite, cudaStream_t s) {
    if (total == 0) return cudaSuccess;
    grad_check_kernel<<<adamw_grid(total), kThreads, 0, s>>>(d_groups, ngroups, d_slices, d_part, total, p, d_grad,
                                                            d_grad_partials, d_nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_adamw(const TrainGroup* d_groups, std::uint32_t ngroups, const AdamCoef* d_coef, std::uint8_t* d_part,
                         const float* d_grad, std::uint64_t total, double* d_delta_partials, cudaStream_t s) {
    if (total == 0) return cudaSuccess;
    adamw_update_kernel<<<adamw_grid(total), kThreads, 0, s>>>(d_groups, ngroups, d_coef, d_part, d_grad, total,
                                                              d_delta_partials);
    return cudaGetLastError();
}

} // namespace tailor::dev
