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

#include "ieee_div.cuh"
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

// float(2 * ((h >> 11) * 2^-53) - 1) of the reference (R/src/gradients.cpp:17-23).
// With x = h >> 11 (< 2^53), 2u - 1 = (x - 2^52) * 2^-52 exactly in double, so the
// float result is the round-to-nearest float of the integer x - 2^52, scaled by 2^-52
// (scaling by a power of two commutes with rounding here): one I2F instead of an
// I2F.F64 + three FP64 ops + F2F, bit-identical.
__device__ __forceinline__ float unit_noise_from(std::uint64_t prefix, std::uint64_t e) {
    const std::uint64_t h = mix64(prefix ^ (e * 0x8CB92BA72F3D8DD7ULL));
    const long long y = static_cast<long long>(h >> 11) - (1LL << 52);
    return __fmul_rn(__ll2float_rn(y), 0x1.0p-52f);
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

// Tiles (host-built, TrainTile) replace per-element group/slice searches: inside a
// tile the field index, the gradient index and the noise counter are all affine
// in j, so each thread streams float4 runs with no lookups.
template <bool kStore>
__global__ void __launch_bounds__(kThreads) grad_check_kernel(const TrainTile* __restrict__ tiles, std::uint32_t ntiles,
                                                              const TrainGroup* __restrict__ groups,
                                                              const std::uint8_t* __restrict__ part, TrainParams p,
                                                              float* __restrict__ grad, double* __restrict__ grad_partials,
                                                              unsigned int* __restrict__ nonfinite) {
    __shared__ double red[kThreads / 32];
    double acc = 0.0;
    bool bad = false;
    for (std::uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TrainTile tile = tiles[t];
        const float* w = reinterpret_cast<const float*>(part + groups[tile.group].off_w) + tile.i0;
        float* gout = grad + tile.v0;
        if (tile.vec) {
            const std::uint32_t n4 = tile.count >> 2;
#pragma unroll 2
            for (std::uint32_t q = threadIdx.x; q < n4; q += kThreads) {
                const float4 x = __ldcs(reinterpret_cast<const float4*>(w) + q);
                const std::uint64_t e = tile.e0 + 4ull * q;
                float4 gr;
                gr.x = grad_of(x.x, p, e);
                gr.y = grad_of(x.y, p, e + 1);
                gr.z = grad_of(x.z, p, e + 2);
                gr.w = grad_of(x.w, p, e + 3);
                if constexpr (kStore) reinterpret_cast<float4*>(gout)[q] = gr;
                bad = bad || !isfinite(gr.x) || !isfinite(gr.y) || !isfinite(gr.z) || !isfinite(gr.w);
                acc = fma(static_cast<double>(gr.x), static_cast<double>(gr.x), acc);
                acc = fma(static_cast<double>(gr.y), static_cast<double>(gr.y), acc);
                acc = fma(static_cast<double>(gr.z), static_cast<double>(gr.z), acc);
                acc = fma(static_cast<double>(gr.w), static_cast<double>(gr.w), acc);
            }
        } else {
            for (std::uint32_t j = threadIdx.x; j < tile.count; j += kThreads) {
                const float gr = grad_of(w[j], p, tile.e0 + j);
                if constexpr (kStore) gout[j] = gr;
                bad = bad || !isfinite(gr);
                acc = fma(static_cast<double>(gr), static_cast<double>(gr), acc);
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) grad_partials[blockIdx.x] = s;
}

// Pass 1, fast form: for the reference gradient source g = c1*w + c2*u with
// 0 < |c1| <= 1/2, |c2| <= 1 and |u| < 1, g is finite exactly when w is (|c1*w|
// <= FLT_MAX/2 cannot overflow with |c2*u| <= 1 added; c1*inf and c1*NaN are not
// finite), so the pre-update check needs only the masters' exponent bits: a
// pure 4 B/element read instead of the hash. The host picks this form only when
// the coefficients satisfy the bound; the gradient norm then comes from pass 2.
__global__ void __launch_bounds__(kThreads) finite_check_kernel(const TrainTile* __restrict__ tiles, std::uint32_t ntiles,
                                                                const TrainGroup* __restrict__ groups,
                                                                const std::uint8_t* __restrict__ part,
                                                                unsigned int* __restrict__ nonfinite) {
    bool bad = false;
    for (std::uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TrainTile tile = tiles[t];
        const std::uint32_t* w = reinterpret_cast<const std::uint32_t*>(part + groups[tile.group].off_w) + tile.i0;
        const auto inf_or_nan = [](std::uint32_t b) { return (b & 0x7F800000u) == 0x7F800000u; };
        if (tile.vec) {
            const std::uint32_t n4 = tile.count >> 2;
#pragma unroll 4
            for (std::uint32_t q = threadIdx.x; q < n4; q += kThreads) {
                const uint4 x = __ldcs(reinterpret_cast<const uint4*>(w) + q);
                bad = bad || inf_or_nan(x.x) || inf_or_nan(x.y) || inf_or_nan(x.z) || inf_or_nan(x.w);
            }
        } else {
            for (std::uint32_t j = threadIdx.x; j < tile.count; j += kThreads) bad = bad || inf_or_nan(w[j]);
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

__device__ __forceinline__ float adam_one(const AdamCoef& c, float& w, float& m, float& v, float gr) {
    m = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(c.one_minus_b1, gr));
    v = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(c.one_minus_b2, __fmul_rn(gr, gr)));
    // bias corrections: constant divisors through RN(1/bias) precomputed on the host
    // (kernels/ieee_div.cuh; bitwise __fdiv_rn, checked exhaustively)
    const float m_hat = div_by_const_rn(m, c.bias1, c.rcp1);
    const float v_hat = div_by_const_rn(v, c.bias2, c.rcp2);
    const float update = __fadd_rn(__fdiv_rn(m_hat, __fadd_rn(__fsqrt_rn(v_hat), c.eps)), __fmul_rn(c.wd, w));
    const float step = __fmul_rn(c.lr, update);
    w = __fsub_rn(w, step);
    return step;
}

// kRecompute: the gradient is recomputed from the pre-update master (the same
// _rn expression as pass 1, so the same bits) instead of being read back from a
// scratch buffer: 28 B per element for the step instead of 36.
template <bool kRecompute>
__global__ void __launch_bounds__(kThreads) adamw_update_kernel(const TrainTile* __restrict__ tiles, std::uint32_t ntiles,
                                                                const TrainGroup* __restrict__ groups,
                                                                const AdamCoef* __restrict__ coef, std::uint8_t* __restrict__ part,
                                                                const float* __restrict__ grad, TrainParams p,
                                                                double* __restrict__ delta_partials,
                                                                double* __restrict__ grad_partials,
                                                                unsigned int* __restrict__ next_nonfinite) {
    __shared__ double red[kThreads / 32];
    double acc = 0.0, gacc = 0.0;
    bool next_bad = false; // a new master is inf/NaN: the next step's gradient is not finite
    const auto inf_or_nan = [](float x) { return (__float_as_uint(x) & 0x7F800000u) == 0x7F800000u; };
    for (std::uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TrainTile tile = tiles[t];
        const TrainGroup& g = groups[tile.group];
        const AdamCoef c = coef[g.coef];
        float* wp = reinterpret_cast<float*>(part + g.off_w) + tile.i0;
        float* mp = reinterpret_cast<float*>(part + g.off_m) + tile.i0;
        float* vp = reinterpret_cast<float*>(part + g.off_v) + tile.i0;
        const float* gp = grad + tile.v0;
        if (tile.vec) {
            const std::uint32_t n4 = tile.count >> 2;
            for (std::uint32_t q = threadIdx.x; q < n4; q += kThreads) {
                float4 w = __ldcs(reinterpret_cast<const float4*>(wp) + q);
                float4 m = __ldcs(reinterpret_cast<const float4*>(mp) + q);
                float4 v = __ldcs(reinterpret_cast<const float4*>(vp) + q);
                float4 gr;
                if constexpr (kRecompute) {
                    const std::uint64_t e = tile.e0 + 4ull * q;
                    gr = make_float4(grad_of(w.x, p, e), grad_of(w.y, p, e + 1), grad_of(w.z, p, e + 2), grad_of(w.w, p, e + 3));
                } else {
                    gr = __ldcs(reinterpret_cast<const float4*>(gp) + q);
                }
                const float s0 = adam_one(c, w.x, m.x, v.x, gr.x);
                const float s1 = adam_one(c, w.y, m.y, v.y, gr.y);
                const float s2 = adam_one(c, w.z, m.z, v.z, gr.z);
                const float s3 = adam_one(c, w.w, m.w, v.w, gr.w);
                __stcs(reinterpret_cast<float4*>(mp) + q, m);
                __stcs(reinterpret_cast<float4*>(vp) + q, v);
                __stcs(reinterpret_cast<float4*>(wp) + q, w);
                if constexpr (kRecompute)
                    next_bad = next_bad || inf_or_nan(w.x) || inf_or_nan(w.y) || inf_or_nan(w.z) || inf_or_nan(w.w);
                acc = fma(static_cast<double>(s0), static_cast<double>(s0), acc);
                acc = fma(static_cast<double>(s1), static_cast<double>(s1), acc);
                acc = fma(static_cast<double>(s2), static_cast<double>(s2), acc);
                acc = fma(static_cast<double>(s3), static_cast<double>(s3), acc);
                if constexpr (kRecompute) {
                    gacc = fma(static_cast<double>(gr.x), static_cast<double>(gr.x), gacc);
                    gacc = fma(static_cast<double>(gr.y), static_cast<double>(gr.y), gacc);
                    gacc = fma(static_cast<double>(gr.z), static_cast<double>(gr.z), gacc);
                    gacc = fma(static_cast<double>(gr.w), static_cast<double>(gr.w), gacc);
                }
            }
        } else {
            for (std::uint32_t j = threadIdx.x; j < tile.count; j += kThreads) {
                float w = wp[j], m = mp[j], v = vp[j];
                const float gr = kRecompute ? grad_of(w, p, tile.e0 + j) : gp[j];
                const float st = adam_one(c, w, m, v, gr);
                mp[j] = m;
                vp[j] = v;
                wp[j] = w;
                acc = fma(static_cast<double>(st), static_cast<double>(st), acc);
                if constexpr (kRecompute) {
                    gacc = fma(static_cast<double>(gr), static_cast<double>(gr), gacc);
                    next_bad = next_bad || inf_or_nan(w);
                }
            }
        }
    }
    if constexpr (kRecompute) {
        if (next_nonfinite && __any_sync(0xffffffffu, next_bad) && (threadIdx.x & 31) == 0) atomicOr(next_nonfinite, 1u);
    }
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) delta_partials[blockIdx.x] = s;
    if constexpr (kRecompute) {
        if (grad_partials) {
            const double gs = block_sum(gacc, red);
            if (threadIdx.x == 0) grad_partials[blockIdx.x] = gs;
        }
    }
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

unsigned train_grid(std::uint32_t ntiles) {
    return std::max(1u, std::min(ntiles, static_cast<unsigned>(sm_count()) * 8u));
}

cudaError_t launch_grad_check(const TrainTile* d_tiles, std::uint32_t ntiles, const TrainGroup* d_groups,
                              const std::uint8_t* d_part, const TrainParams& p, float* d_grad, double* d_grad_partials,
                              unsigned int* d_nonfinite, cudaStream_t s) {
    if (d_grad)
        grad_check_kernel<true><<<train_grid(ntiles), kThreads, 0, s>>>(d_tiles, ntiles, d_groups, d_part, p, d_grad,
                                                                       d_grad_partials, d_nonfinite);
    else
        grad_check_kernel<false><<<train_grid(ntiles), kThreads, 0, s>>>(d_tiles, ntiles, d_groups, d_part, p, nullptr,
                                                                        d_grad_partials, d_nonfinite);
    return cudaGetLastError();
}

bool finite_check_suffices(const TrainParams& p) {
    const float c1 = p.state_coeff < 0 ? -p.state_coeff : p.state_coeff;
    const float c2 = p.noise_coeff < 0 ? -p.noise_coeff : p.noise_coeff;
    return c1 > 0.f && c1 <= 0.5f && c2 <= 1.f; // false for NaN coefficients too
}

cudaError_t launch_finite_check(const TrainTile* d_tiles, std::uint32_t ntiles, const TrainGroup* d_groups,
                                const std::uint8_t* d_part, unsigned int* d_nonfinite, cudaStream_t s) {
    finite_check_kernel<<<train_grid(ntiles), kThreads, 0, s>>>(d_tiles, ntiles, d_groups, d_part, d_nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_adamw(const TrainTile* d_tiles, std::uint32_t ntiles, const TrainGroup* d_groups, const AdamCoef* d_coef,
                         std::uint8_t* d_part, const float* d_grad, const TrainParams& p, double* d_delta_partials,
                         double* d_grad_partials, unsigned int* d_next_nonfinite, cudaStream_t s) {
    if (d_grad)
        adamw_update_kernel<false><<<train_grid(ntiles), kThreads, 0, s>>>(d_tiles, ntiles, d_groups, d_coef, d_part, d_grad, p,
                                                                          d_delta_partials, nullptr, nullptr);
    else
        adamw_update_kernel<true><<<train_grid(ntiles), kThreads, 0, s>>>(d_tiles, ntiles, d_groups, d_coef, d_part, nullptr, p,
                                                                         d_delta_partials, d_grad_partials, d_next_nonfinite);
    return cudaGetLastError();
}

} // namespace tailor::dev
