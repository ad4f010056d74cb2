// Device tables and kernel launchers (sm_100a). Tables are built on the host
// from the layer map (tailor/model.hpp, tailor/merge.hpp), uploaded once and
// read-only during a launch; kernels never allocate. All launches are
// asynchronous on the caller's stream.
#pragma once

#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

namespace tailor::dev {

// ---- K2: segmented gather/scatter ------------------------------------------
// Destination bytes [dst_off, dst_off + bytes) <- src[0, bytes). Segments are
// sorted by dst_off and do not overlap.
struct GatherSeg {
    const std::uint8_t* src;
    std::uint64_t dst_off;
    std::uint64_t bytes;
};
static_assert(sizeof(GatherSeg) == 24, "GatherSeg is part of the C ABI");

// kGatherBulk = 3 x 64 KB ring, one CTA per SM (default); the other bulk
// shapes exist for measured comparisons (profiles/).
enum GatherVariant : int {
    kGatherAuto = 0,
    kGatherLsu = 1,
    kGatherBulk = 2,
    kGatherBulk6x32 = 3,
    kGatherBulk2Cta = 4,
    kGatherBulk4x48 = 5, // the previous default ring
    kGatherBulk8x24 = 6,
    kGatherBulkStatic = 7 // the default ring with the static tile split even when a counter is given
};

// `bulk_ok` (host-checked): every segment has 16-B aligned src/dst/bytes and
// the segments tile [0, dst_bytes) exactly — the TMA bulk path's contract.
// `d_counter` (optional, two words, zero between launches): the bulk kernel claims its
// 64 KB tiles dynamically through it and resets it before it exits; launches sharing
// one counter must be stream-ordered. Null = static tile split. Bytes never depend on it.
cudaError_t launch_gather(const GatherSeg* d_segs, std::uint32_t nseg, std::uint8_t* d_dst, std::uint64_t dst_bytes,
                          int variant, bool bulk_ok, cudaStream_t stream, unsigned int* d_counter = nullptr);
// Measurement only: read-only HBM stream over [d_src, d_src + bytes) (16-B aligned),
// XOR-folded into *d_sink.
cudaError_t launch_read_probe(const std::uint8_t* d_src, std::uint64_t bytes, unsigned int* d_sink, cudaStream_t stream);

// ---- K3/K4: update-magnitude scorer -----------------------------------------
// A tile covers `count` consecutive master elements of one field (one group's
// rank chunk) of one module; every snapshot k reads the same element range at
// field_base[k * nfields + field].
struct ScoreTile {
    std::uint32_t module;
    std::uint32_t field;
    std::uint32_t count;
    std::uint32_t pad;
    std::uint64_t elem_start;
};
static_assert(sizeof(ScoreTile) == 24, "ScoreTile is part of the C ABI");

// tile_partials[t][p][0|1] = (sum (B-A)^2, sum A^2) over tile t for pair
// p = (snapshot p, snapshot p+1), FP64. 2 <= K <= 16.
// variant: 0 auto, 1 register-staged 128-bit loads, 2 TMA-bulk smem ring (needs vec_ok).
// Register variants: 3 forces 128-bit loads, 4 forces 64-bit loads. Measured
// at K=16: 128-bit 0.938, 64-bit 0.675 (spills at the 2-CTA register cap), so
// auto always uses 128-bit loads.
enum ScoreVariant : int {
    kScoreAuto = 0,
    kScoreRegister = 1,
    kScoreStaged = 2,
    kScoreWide = 3,
    kScoreNarrow = 4,
    kScoreStagedWide = 5, // staged ring, half the rows per stage (K <= 8; the round-1 geometry for K >= 4)
    kScoreStaged2Cta = 6  // staged ring, two CTAs per SM (K <= 8)
};
constexpr int kNarrowMinK = 1 << 20;
// Staged = warp-specialised TMA ring (producer warp + 8 consumer warps, full/empty
// mbarriers). Measured on B200 (bench events, fraction of the 6543 GB/s copy peak):
// K=16 1.093 vs register 0.951; K=4 1.075 vs 1.064. At K=2 its first form lost (cfg2:
// 1.83 vs 1.28 ms: 8 KB stages need ~6 stages/us per SM from one producer lane; a deeper
// ring did not help); with 4 float4 rows per thread per stage (32 KB stages) it tied the
// register kernel (1.30 vs 1.27 ms), and with two CTAs per SM for K < 4 (half the ring
// each: more independent streams) it wins (1.23 ms; at K=4 two CTAs lose: 2.65 vs 2.47)
// -> auto picks it whenever the bases are 16-B aligned. (Its very first version, one
// CTA-wide barrier per chunk, was barrier-bound: 0.88 / 0.61.)
constexpr int kStagedMinK = 2;
// d_counter (optional, one word): the staged kernel claims tiles dynamically through it
// (zeroed on `stream` first); null = static tile split. Results do not depend on it.
cudaError_t launch_score_partials(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                                  std::uint32_t nfields, int K, bool vec_ok, double* d_tile_partials, cudaStream_t stream,
                                  int variant = kScoreAuto, unsigned int* d_counter = nullptr);
// out[p][m][0|1] = fixed-order sum over module m's tiles [tile_begin[m], tile_begin[m+1]).
cudaError_t launch_score_combine(const double* d_tile_partials, const std::uint32_t* d_module_tile_begin, int M, int K,
                                 double* d_out, cudaStream_t stream);

// ---- K5: synthetic snapshot generator (SURVEY §8d contract) -----------------
struct SynthGroup {
    std::uint64_t begin;       // first virtual element of this group in the launch
    std::uint64_t chunk;       // elements in the rank chunk
    std::uint64_t group_first; // group-local index of chunk element 0 (rank * chunk)
    std::uint64_t true_len;
    std::uint64_t off[3];      // byte offsets of exp_avg, exp_avg_sq, master; ~0 = not generated
    std::uint32_t slice_begin;
    std::uint32_t slice_count;
    std::uint32_t module; // canonical module index (sigma row)
    std::uint32_t pad;
};
struct SynthSlice {
    std::int64_t group_offset;
    std::int64_t model_offset;
    std::int64_t count;
};
struct SynthTensor {
    std::uint64_t begin;  // first virtual element
    std::uint64_t count;
    std::uint64_t dst_off; // byte offset in the output window
    std::int64_t model_offset;
    std::uint32_t module;
    std::uint32_t pad;
};

// Output buffers travel by value in the launch parameters (no upload).
constexpr int kMaxSnapshots = 16;
struct OutPtrs {
    std::uint8_t* p[kMaxSnapshots];
};

// Generates snapshots k0..k1 (1-based, k1 - k0 < 16) in one pass; outs.p[k - k0]
// receives snapshot k. sigma is [k1][M] floats (row j-1 = sigma_j).
cudaError_t launch_synth_shard(const SynthGroup* d_groups, std::uint32_t ngroups, const SynthSlice* d_slices,
                               const float* d_sigma, int M, std::uint64_t seed, int k0, int k1, OutPtrs outs,
                               std::uint64_t total, cudaStream_t stream);
cudaError_t launch_synth_weights(const SynthTensor* d_tensors, std::uint32_t ntensors, const float* d_sigma, int M,
                                 std::uint64_t seed, int k0, int k1, OutPtrs outs, std::uint64_t total,
                                 cudaStream_t stream);

// ---- K6: composite re-verify (R/src/checkpoint.cpp:515-572 invariants) ------
// Pairs: bf16_round(master[i]) == weight[i] for i < count. Zero ranges: every
// 32-bit word must be 0 (shard padding). Nonneg ranges: exp_avg_sq >= 0.
struct VerifyPair {
    const float* master;
    const std::uint16_t* weight;
    std::uint64_t count;
};
struct VerifyRange {
    const std::uint32_t* words;
    std::uint64_t count;
    std::uint32_t kind; // 0 = must be zero, 1 = must be >= 0 (float)
    std::uint32_t pad;
};
// err[0] = number of failing pair elements, err[1] = failing zero words,
// err[2] = failing non-negative elements (accumulated; caller zeroes).
cudaError_t launch_verify(const VerifyPair* d_pairs, std::uint32_t npairs, const VerifyRange* d_ranges,
                          std::uint32_t nranges, unsigned long long* d_err, cudaStream_t stream);

// ---- K7: AdamW step over rank partitions ------------------------
struct TrainGroup {
    std::uint64_t begin;       // first virtual element of this group in the partition
    std::uint64_t chunk;
    std::uint64_t group_first; // rank * chunk
    std::uint64_t true_len;
    std::uint64_t off_m, off_v, off_w; // payload byte offsets of exp_avg, exp_avg_sq, master
    std::uint32_t slice_begin;
    std::uint32_t slice_count;
    std::uint32_t coef; // index into the AdamCoef table
    std::uint32_t pad;
};
// Per-group FP32 coefficients, each rounded once from FP64 (R/src/adamw.cpp:19-27).
// y = RN(1/b) in single precision for div_by_const_rn (kernels/ieee_div.cuh); a divisor
// outside [2^-20, 2^20] (never a bias correction: those lie in [1 - beta, 1]) gets 0,
// which makes the kernel divide per element (__fdiv_rn).
inline float const_reciprocal(float b) {
    const float ab = b < 0 ? -b : b;
    if (!(ab >= 0x1p-20f && ab <= 0x1p20f)) return 0.0f;
    volatile float one = 1.0f; // an IEEE single division on the host, not a folded constant
    return one / b;
}
struct AdamCoef {
    float b1, one_minus_b1, b2, one_minus_b2, bias1, bias2, lr, eps, wd;
    float rcp1, rcp2; // RN(1/bias1), RN(1/bias2) for div_by_const_rn (kernels/ieee_div.cuh); 0 = divide
    float pad;
};
struct TrainParams {
    // unit_noise(seed, step, e) = f(mix64(noise_prefix ^ e * C3)): the first two
    // hash rounds depend only on (seed, step) and are computed once on the host.
    std::uint64_t noise_prefix;
    float state_coeff; // GradientSource c1 (R/include/tailor/gradients.hpp:20-24)
    float noise_coeff; // c2
};
std::uint64_t noise_prefix(std::uint64_t seed, std::uint64_t step);
// A run of consecutive non-padding elements of one group inside one tensor slice
// (host-built): element j of the tile is field element i0 + j, virtual element
// v0 + j (gradient scratch index) and global element id e0 + j (noise counter).
struct TrainTile {
    std::uint64_t v0, i0, e0;
    std::uint32_t count;
    std::uint16_t group; // index into the rank's TrainGroup table
    std::uint16_t vec;   // 1: i0 and count are multiples of 4 and the fields 16-B aligned
};
constexpr std::uint32_t kTrainTileElems = 16384;
// Pass 1: gradients (stored to d_grad, one float per virtual element, unless
// d_grad is null), FP64 sum g^2 per block, non-finite flag. Pass 2 (only if no
// flag): AdamW, reading d_grad or (null) recomputing the gradient from p.
cudaError_t launch_grad_check(const TrainTile* d_tiles, std::uint32_t ntiles, const TrainGroup* d_groups,
                              const std::uint8_t* d_part, const TrainParams& p, float* d_grad, double* d_grad_partials,
                              unsigned int* d_nonfinite, cudaStream_t s);
cudaError_t launch_adamw(const TrainTile* d_tiles, std::uint32_t ntiles, const TrainGroup* d_groups, const AdamCoef* d_coef,
                         std::uint8_t* d_part, const float* d_grad, const TrainParams& p, double* d_delta_partials,
                         double* d_grad_partials, unsigned int* d_next_nonfinite, cudaStream_t s);
// (recomputing form) d_next_nonfinite, if set, is OR-ed with 1 when a new master is
// inf/NaN: the exponent check of the NEXT step, done on the values as they are written.
// Pass 1 fast form (masters' exponent bits only) and when it is exact: g = c1*w +
// c2*u is finite iff w is, for 0 < |c1| <= 1/2 and |c2| <= 1. In that mode pass 2
// (recomputing) also writes the FP64 sum g^2 per block into d_grad_partials.
bool finite_check_suffices(const TrainParams& p);
cudaError_t launch_finite_check(const TrainTile* d_tiles, std::uint32_t ntiles, const TrainGroup* d_groups,
                                const std::uint8_t* d_part, unsigned int* d_nonfinite, cudaStream_t s);
// blocks of the two passes (one FP64 partial each)
unsigned train_grid(std::uint32_t ntiles);
unsigned adamw_grid(std::uint64_t total);

// ---- K8: bf16 weights derived from sharded masters ---------------------------------
struct WeightTensor {
    std::uint64_t begin;        // first virtual element
    std::uint64_t dst_off;      // byte offset in the weights payload
    std::uint64_t group_offset; // tensor's first element within its group
    std::uint64_t chunk;        // group's shard length
    std::uint64_t master_off;   // byte offset of the group's master field in every rank payload
};
cudaError_t launch_derive_weights(const WeightTensor* d_tensors, std::uint32_t ntensors,
                                  const std::uint8_t* const* d_parts, std::uint8_t* d_out, std::uint64_t total,
                                  cudaStream_t s);

// ---- K9: device-side magnitude selection + merge plan ---------------------------
struct PlanEntry {
    std::uint32_t module; // canonical owner module of the entry
    std::uint32_t pad;
    std::uint64_t src_off; // relative to the snapshot buffer base
    std::uint64_t dst_off;
    std::uint64_t bytes;
};
// K9 takes the snapshot bases by value (1 KB of launch parameters at 64 snapshots).
constexpr int kMaxSelectSnapshots = 64;
struct SnapshotBases {
    const std::uint8_t* shard[kMaxSelectSnapshots];
    const std::uint8_t* weights[kMaxSelectSnapshots];
};
cudaError_t launch_select_plan(const double* d_parts, int nranks, int K, int M, int n_save, const PlanEntry* d_shard_entries,
                               std::uint32_t n_shard, const PlanEntry* d_w_entries, std::uint32_t n_w,
                               const SnapshotBases& bases, GatherSeg* d_shard_segs, GatherSeg* d_w_segs, int* d_source_of,
                               double* d_scores, cudaStream_t s);

int sm_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device);
// `done` is the kernel's per-device bitmask. Thread-safe.
cudaError_t ensure_smem_attr(const void* fn, std::size_t smem, std::atomic<std::uint64_t>& done);

} // namespace tailor::dev
