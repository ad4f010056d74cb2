// The tailoring engine surface: recipes, plan resolution, composite assembly,
// auto-recipes — the reference's L5 API (R/include/tailor/merge.hpp:18-70,
// R/include/tailor/recipe.hpp:12-35) with identical semantics, plus the
// update-magnitude selection strategy that the reference
// lacks. execute_merge moves every payload byte through the device gather
// kernel; there is no host copy path.
#pragma once

#include "tailor/io.hpp"

#include <cstdint>
#include <filesystem>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "tailor/checkpoint.hpp"
#include "tailor/model.hpp"

namespace tailor {

struct RecipeSlice {
    std::string source;
    std::vector<int> layers;
    std::vector<int> targets;
};

struct MergeRecipe {
    std::string base_checkpoint;
    int num_ranks = 0;
    std::vector<RecipeSlice> slices;
    std::map<std::string, std::string> aux;
    std::string config_from = "latest";
};

MergeRecipe parse_recipe(const std::string& yaml_text);
MergeRecipe read_recipe_file(const std::string& path);
std::string recipe_to_yaml(const MergeRecipe& recipe);

struct MergePlan {
    ModelSpec spec;
    int num_ranks = 1;
    GroupTable table;
    struct Assignment {
        std::string source;
        ModuleId source_module;
        std::int64_t source_step = 0;
    };
    std::map<ModuleId, Assignment> assignment; // by target module
    struct GroupCopy {
        std::string source;
        int source_group = 0;
        int target_group = 0;
    };
    std::vector<GroupCopy> group_copies; // ascending target group
    std::string config_source;
    std::vector<std::string> sources;
};

using SummaryLookup = std::function<CheckpointSummary(const std::string&)>;

MergePlan resolve_plan(const MergeRecipe& recipe);
// Same resolution over summaries from any provider (device-resident sources).
MergePlan resolve_plan_with(const MergeRecipe& recipe, const SummaryLookup& lookup);

struct MergeOptions {
    int workers = 0;       // host read threads; 0 -> num_ranks
    bool uncached = false; // re-read the source shard per group copy (benchmark mode)
    int device = 0;
    bool verify = true;    // device re-verify of the written composite
    // Lanes (one output file at a time each) spread round-robin over these devices;
    // empty = {device}. Output bytes do not depend on the devices or the lane count.
    std::vector<int> devices;
    // Source reads / output writes through the page cache or O_DIRECT (tailor/io.hpp);
    // the bytes written do not depend on it.
    IoMode io = IoMode::Auto;
};
inline std::vector<int> lane_devices(const MergeOptions& o) {
    return o.devices.empty() ? std::vector<int>{o.device} : o.devices;
}

struct MergeStats {
    std::int64_t shard_files_read = 0;
    std::int64_t weight_files_read = 0;
    double wall_ms = 0.0;
    double device_ms = 0.0;        // gather kernels, CUDA events
    std::uint64_t bytes_moved = 0; // composite payload bytes
    std::uint64_t direct_read_bytes = 0;  // source bytes read with O_DIRECT
    std::uint64_t direct_write_bytes = 0; // output bytes written with O_DIRECT (whole blocks)
    std::uint64_t resident_bytes = 0;     // source bytes gathered from device copies (ResidentSources), not read
};

MergeStats execute_merge(const MergePlan& plan, const std::filesystem::path& out_dir, const MergeOptions& options = {});

// Source bytes already on the merge's device (the masters the scorer just read, in a
// combined select+merge): payload-relative byte ranges of (source, container) that the
// merge gathers from device memory instead of reading the file again. The output bytes
// are the same; only fewer bytes come off the disk / cross PCIe.
struct ResidentRange {
    std::uint64_t lo = 0, hi = 0;       // payload-relative [lo, hi) in the source container
    const std::uint8_t* dev = nullptr;  // device address of byte lo
};
struct ResidentSources {
    int device = 0;
    std::map<std::pair<std::string, int>, std::vector<ResidentRange>> ranges; // sorted by lo, disjoint
};
MergeStats execute_merge(const MergePlan& plan, const std::filesystem::path& out_dir, const MergeOptions& options,
                         const ResidentSources* resident);

// Re-slice a complete checkpoint between the coarse (2-group) and fine
// (2L+3 / 2L+2) optimizer layouts (R/src/groups.cpp:152-220)
// as a device gather; output bytes equal read_checkpoint -> coarse_to_fine /
// fine_to_coarse -> write_checkpoint.
MergeStats execute_regroup(const std::filesystem::path& src, const std::filesystem::path& out_dir, Grouping target,
                           const MergeOptions& options = {});

std::vector<std::filesystem::path> list_checkpoints(const std::filesystem::path& run_dir);
MergeRecipe recipe_from_manifests(const std::filesystem::path& run_dir, std::int64_t failure_step);

// ---- the merge plan as byte segments ------------------------------------------
// One output container (weights or one rank shard) = a list of source windows
// (a byte range of one source file's payload) and copy segments
// {window, src_off, dst_off, bytes} that tile the output payload.
struct SourceWindow {
    std::string source;    // checkpoint path / id
    int container = -1;    // -1 = weights, r >= 0 = rank r shard
    std::uint64_t lo = 0;  // payload-relative window [lo, hi)
    std::uint64_t hi = 0;
};

struct CopySegment {
    std::uint32_t window = 0;
    std::uint64_t src_off = 0; // relative to window.lo
    std::uint64_t dst_off = 0; // payload-relative in the output
    std::uint64_t bytes = 0;
};

struct PartitionPlan {
    ContainerLayout out;
    std::vector<SourceWindow> windows;
    std::vector<CopySegment> segments; // ascending dst_off, coalesced
    std::uint64_t dst_lo = 0;          // output byte range this plan produces
    std::uint64_t dst_hi = 0;
};

// Source payload layouts by source path. For files: parsed headers; for
// device-resident synthetic sources: checkpoint_layout().
struct SourceLayout {
    ContainerLayout weights;
    std::vector<ContainerLayout> shards;
};
using LayoutLookup = std::function<const SourceLayout&(const std::string&)>;

// A copy expressed against a source container: windows and coalesced
// segments are derived by finalize_partition. container -1 = weights,
// r >= 0 = rank-r shard, kZeroContainer = zero fill (no source file).
inline constexpr int kZeroContainer = -2;
struct CopyPiece {
    std::string source;
    int container;
    std::uint64_t src_off; // payload-relative in the source container
    std::uint64_t dst_off;
    std::uint64_t bytes;
};
void finalize_partition(PartitionPlan& pp, std::vector<CopyPiece> pieces);

// Weights container plan (validates tensor presence/dtype/shape exactly as
// R/src/merge.cpp:254-266) restricted to output bytes [lo, hi).
PartitionPlan plan_weights(const MergePlan& plan, const LayoutLookup& layouts, std::uint64_t lo = 0,
                           std::uint64_t hi = UINT64_MAX);
// Rank-r shard container plan (checks as copy_shard_entries, R/src/merge.cpp:207-222).
// [lo, hi): a byte sub-range of the composite shard payload (host-staged units of
// partitions that exceed one pass through HBM, e.g. cfg5).
PartitionPlan plan_shard(const MergePlan& plan, const LayoutLookup& layouts, int rank, std::uint64_t lo = 0,
                         std::uint64_t hi = UINT64_MAX);
// Byte range of a container payload owned by unit u of n: split at tensor
// boundaries, balanced by bytes (weights shares; shard sub-units).
std::pair<std::uint64_t, std::uint64_t> weights_share(const ContainerLayout& out, int unit, int units);

OptimMeta merged_optim_meta(const MergePlan& plan, const SummaryLookup& lookup);
SaveManifest merged_manifest(const MergePlan& plan, const SummaryLookup& lookup);

// ---- update-magnitude selection (no reference code) ------
// scores[p][m] = score(S_p -> S_{p+1}) of canonical module m.
struct Selection {
    std::vector<std::vector<int>> saved; // per snapshot: canonical module indices (ascending)
    std::vector<int> source_of;          // per module: snapshot index it is drawn from
    double min_boundary_gap = 0.0;       // smallest relative score gap at a top-n boundary
};
Selection select_by_magnitude(const std::vector<std::vector<double>>& scores, int num_modules, double rho);
// Latest-version rule of recipe_from_manifests (R/src/merge.cpp:375-417) over
// the selected sets; snapshots given as summaries (step, dir, num_ranks).
MergeRecipe recipe_from_selection(const std::vector<CheckpointSummary>& snapshots, const Selection& sel);
// score = sqrt(sum_delta_sq) / sqrt(sum_ref_sq) (0 when both are 0, inf when ref is 0).
double magnitude_score(double sum_delta_sq, double sum_ref_sq);

} // namespace tailor
