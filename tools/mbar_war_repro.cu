// Minimal reproducer for the one racecheck report left on the scorer (score_staged_kernel's
// WAR pair, profiles/r1_compute_sanitizer.txt): is it the ring protocol or racecheck's model?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2602_22158_b200/csrc/kernels \
//        tools/mbar_war_repro.cu -o tools/mbar_war_repro
//   compute-sanitizer --tool racecheck tools/mbar_war_repro {mbarrier|syncthreads}
//
// Both kernels stream 64 chunks of 4 KB through a 2-stage shared-memory ring filled by
// cp.async.bulk (completion on a `full` mbarrier, transaction bytes) and sum them.
//   mbarrier    — the scorer's protocol: one producer lane, one consumer warp; the consumer
//                 reads the stage, __syncwarp, fence.proxy.async.shared::cta, arrives on the
//                 stage's `empty` mbarrier; the producer try_waits on `empty` before it
//                 issues the next bulk copy into that stage (PTX ISA: an mbarrier
//                 arrive/complete-phase is a release/acquire pair, and the proxy fence orders
//                 the generic-proxy reads before the async-proxy write).
//   syncthreads — control: same ring, but the stage is released with __syncthreads().
// Both check the sum on the host. If racecheck reports a WAR hazard for `mbarrier` and none
// for `syncthreads`, it does not model mbarrier completion as ordering the async proxy —
// the report carries no information about the scorer.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tma.cuh"

using namespace tailor::dev::tma;

constexpr int kStages = 2;
constexpr int kChunkFloats = 1024; // 4 KB
constexpr int kChunks = 64;

__global__ void ring_mbarrier(const float* __restrict__ src, double* out) {
    __shared__ __align__(128) float ring[kStages][kChunkFloats];
    __shared__ __align__(8) std::uint64_t full[kStages], empty[kStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1); // one arrival: the consumer warp
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 1) { // producer
        if (lane == 0)
            for (int i = 0; i < kChunks; ++i) {
                const int s = i % kStages;
                if (i >= kStages) mbar_wait_parity(&empty[s], ((i / kStages) - 1) & 1u);
                mbar_arrive_expect_tx(&full[s], kChunkFloats * 4);
                bulk_load(ring[s], src + static_cast<std::size_t>(i) * kChunkFloats, kChunkFloats * 4, &full[s]);
            }
        return;
    }
    double acc = 0.0; // consumer warp
    for (int i = 0; i < kChunks; ++i) {
        const int s = i % kStages;
        mbar_wait_parity(&full[s], (i / kStages) & 1u);
        for (int e = lane; e < kChunkFloats; e += 32) acc += ring[s][e];
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive(&empty[s]);
        }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) *out = acc;
}

__global__ void ring_syncthreads(const float* __restrict__ src, double* out) {
    __shared__ __align__(128) float ring[kStages][kChunkFloats];
    __shared__ __align__(8) std::uint64_t full[kStages];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = 0; i < kStages; ++i) {
            mbar_arrive_expect_tx(&full[i], kChunkFloats * 4);
            bulk_load(ring[i], src + static_cast<std::size_t>(i) * kChunkFloats, kChunkFloats * 4, &full[i]);
        }
    double acc = 0.0;
    for (int i = 0; i < kChunks; ++i) {
        const int s = i % kStages;
        mbar_wait_parity(&full[s], (i / kStages) & 1u);
        if (threadIdx.x < 32)
            for (int e = lane; e < kChunkFloats; e += 32) acc += ring[s][e];
        fence_proxy_async_smem();
        __syncthreads(); // release the stage to the next bulk copy
        if (threadIdx.x == 0 && i + kStages < kChunks) {
            mbar_arrive_expect_tx(&full[s], kChunkFloats * 4);
            bulk_load(ring[s], src + static_cast<std::size_t>(i + kStages) * kChunkFloats, kChunkFloats * 4, &full[s]);
        }
    }
    if (threadIdx.x < 32) {
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) *out = acc;
    }
}

int main(int argc, char** argv) {
    const bool mb = argc < 2 || std::strcmp(argv[1], "syncthreads") != 0;
    std::vector<float> h(static_cast<std::size_t>(kChunks) * kChunkFloats);
    double expect = 0.0;
    for (std::size_t i = 0; i < h.size(); ++i) {
        h[i] = static_cast<float>(i % 97);
        expect += h[i];
    }
    float* d = nullptr;
    double* o = nullptr;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 8);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    if (mb) ring_mbarrier<<<1, 64>>>(d, o);
    else ring_syncthreads<<<1, 64>>>(d, o);
    double got = 0.0;
    const cudaError_t e = cudaMemcpy(&got, o, 8, cudaMemcpyDeviceToHost);
    std::printf("%s: sum %.1f expect %.1f %s (%s)\n", mb ? "mbarrier" : "syncthreads", got, expect,
                got == expect ? "OK" : "MISMATCH", cudaGetErrorString(e));
    return got == expect && e == cudaSuccess ? 0 : 1;
}
