// K9 — on-device magnitude selection + segment-table construction, so a
// score -> select -> merge step needs no host round trip (and can be captured
// in a CUDA graph). Exactly the host contract (select_by_magnitude +
// recipe_from_selection):
//   score(m) = sqrt(sum_r sd_r) / sqrt(sum_r sr_r)   (ranks summed in rank order, FP64,
//              IEEE sqrt/div — bitwise the host's value)
//   saved_1 = all; saved_k = the n highest r_k (ties -> lower canonical index)
//   source(m) = max { k : m in saved_k }
// then every output entry (owned by module m) copies from snapshot source(m) at
// the same byte offset — the plan of a selection-driven merge of full
// snapshots, which never moves layers. One CTA; M <= a few hundred modules.
#include "tailor/device.hpp"

namespace tailor::dev {

namespace {

constexpr int kSelThreads = 256;
constexpr int kMaxModules = 1024;
constexpr int kMaxPairs = kMaxSelectSnapshots - 1;

__global__ void __launch_bounds__(kSelThreads) select_plan_kernel(const double* __restrict__ parts, int nranks, int P, int M,
                                                                   int n_save, const PlanEntry* __restrict__ shard_entries,
                                                                   std::uint32_t n_shard, const PlanEntry* __restrict__ w_entries,
                                                                   std::uint32_t n_w, SnapshotBases bases,
                                                                   GatherSeg* __restrict__ shard_segs,
                                                                   GatherSeg* __restrict__ w_segs, int* __restrict__ source_of,
                                                                   double* __restrict__ scores) {
    __shared__ int src[kMaxModules];
    for (int m = threadIdx.x; m < M; m += blockDim.x) src[m] = 0;
    for (int p = 0; p < P; ++p) {
        __syncthreads();
        __shared__ double sc[kMaxModules];
        for (int m = threadIdx.x; m < M; m += blockDim.x) {
            double sd = 0.0, sr = 0.0;
            for (int r = 0; r < nranks; ++r) { // rank order
                const std::uint64_t at = ((static_cast<std::uint64_t>(r) * P + p) * M + m) * 2;
                sd = __dadd_rn(sd, parts[at]);
                sr = __dadd_rn(sr, parts[at + 1]);
            }
            const double s = sr > 0.0 ? __ddiv_rn(__dsqrt_rn(sd), __dsqrt_rn(sr)) : (sd > 0.0 ? __longlong_as_double(0x7ff0000000000000LL) : 0.0);
            sc[m] = s;
            scores[static_cast<std::uint64_t>(p) * M + m] = s;
        }
        __syncthreads();
        for (int m = threadIdx.x; m < M; m += blockDim.x) {
            int rank = 0;
            const double s = sc[m];
            for (int j = 0; j < M; ++j) rank += (sc[j] > s || (sc[j] == s && j < m)) ? 1 : 0;
            if (rank < n_save) src[m] = p + 1; // snapshot index (0-based) of S_{p+2}
        }
    }
    __syncthreads();
    for (int m = threadIdx.x; m < M; m += blockDim.x) source_of[m] = src[m];
    for (std::uint32_t i = threadIdx.x; i < n_shard; i += blockDim.x) {
        const PlanEntry e = shard_entries[i];
        shard_segs[i] = {bases.shard[src[e.module]] + e.src_off, e.dst_off, e.bytes};
    }
    for (std::uint32_t i = threadIdx.x; i < n_w; i += blockDim.x) {
        const PlanEntry e = w_entries[i];
        w_segs[i] = {bases.weights[src[e.module]] + e.src_off, e.dst_off, e.bytes};
    }
}

} // namespace

cudaError_t launch_select_plan(const double* d_parts, int nranks, int K, int M, int n_save, const PlanEntry* d_shard_entries,
                               std::uint32_t n_shard, const PlanEntry* d_w_entries, std::uint32_t n_w,
                               const SnapshotBases& bases, GatherSeg* d_shard_segs, GatherSeg* d_w_segs, int* d_source_of,
                               double* d_scores, cudaStream_t s) {
    if (M > kMaxModules || K - 1 > kMaxPairs || K < 2) return cudaErrorInvalidValue;
    select_plan_kernel<<<1, kSelThreads, 0, s>>>(d_parts, nranks, K - 1, M, n_save, d_shard_entries, n_shard, d_w_entries, n_w,
                                                 bases, d_shard_segs, d_w_segs, d_source_of, d_scores);
    return cudaGetLastError();
}

} // namespace tailor::dev
