// K6 — device re-verify of a written composite, replacing the reference's
// full host re-read (execute_merge -> read_checkpoint, R/src/merge.cpp:353,
// R/src/checkpoint.cpp:515-572):
//   * weight/master duality: bf16_round(master) == stored BF16 weight, per element
//   * shard padding is zero on disk
//   * exp_avg_sq >= 0 (GroupState::validate, R/src/groups.cpp:27-32)
// One grid-stride pass over (pair | range) work; failures are counted with a
// warp-aggregated atomic (counts only, so the result is order-independent).
#include <algorithm>

#include "tailor/bf16.hpp"
#include "tailor/device.hpp"

namespace tailor::dev {

namespace {

__device__ __forceinline__ void count_fail(bool bad, unsigned long long* slot) {
    const unsigned m = __ballot_sync(__activemask(), bad);
    if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(slot, static_cast<unsigned long long>(__popc(m)));
}

__global__ void verify_pairs_kernel(const VerifyPair* __restrict__ pairs, std::uint32_t npairs, unsigned long long* err) {
    for (std::uint32_t p = blockIdx.y; p < npairs; p += gridDim.y) {
        const VerifyPair q = pairs[p];
        for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < q.count;
             i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
            const std::uint32_t bits = __float_as_uint(__ldg(q.master + i));
            count_fail(bf16_round_bits(bits) != __ldg(q.weight + i), &err[0]);
        }
    }
}

__global__ void verify_ranges_kernel(const VerifyRange* __restrict__ ranges, std::uint32_t nranges, unsigned long long* err) {
    for (std::uint32_t r = blockIdx.y; r < nranges; r += gridDim.y) {
        const VerifyRange q = ranges[r];
        for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < q.count;
             i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
            const std::uint32_t w = __ldg(q.words + i);
            if (q.kind == 0) count_fail(w != 0u, &err[1]);
            else count_fail(!(__uint_as_float(w) >= 0.0f), &err[2]);
        }
    }
}

} // namespace

cudaError_t launch_verify(const VerifyPair* d_pairs, std::uint32_t npairs, const VerifyRange* d_ranges,
                          std::uint32_t nranges, unsigned long long* d_err, cudaStream_t stream) {
    const unsigned gx = static_cast<unsigned>(sm_count()) * 4;
    if (npairs) {
        dim3 grid(std::max(1u, gx / std::min(npairs, 64u)), std::min(npairs, 64u));
        verify_pairs_kernel<<<grid, 256, 0, stream>>>(d_pairs, npairs, d_err);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (nranges) {
        dim3 grid(std::max(1u, gx / std::min(nranges, 64u)), std::min(nranges, 64u));
        verify_ranges_kernel<<<grid, 256, 0, stream>>>(d_ranges, nranges, d_err);
    }
    return cudaGetLastError();
}

} // namespace tailor::dev
