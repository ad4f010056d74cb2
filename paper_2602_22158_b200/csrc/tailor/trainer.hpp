// Device-resident trainer over ZeRO rank partitions: the
// reference's deterministic toy trainer (R/src/trainer.cpp:26-123) with the
// state living in HBM in checkpoint-payload layout, AdamW on the device (K7,
// bit-exact), and checkpoints written straight from the partitions. It adds the
// update-magnitude strategy at training time: at every checkpoint the current
// masters are scored against the previous checkpoint's (K3, in-situ) and only
// the top-rho modules are saved — the selective checkpointing that
// recipe_from_manifests + execute_merge later recover from.
#pragma once

#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "tailor/checkpoint.hpp"
#include "tailor/engine.hpp"

namespace tailor {

// R/src/strategy.cpp:48-91 (full / parity / filter schedules).
std::vector<ModuleId> modules_to_save(const StrategyConfig& cfg, const ModelSpec& spec, std::int64_t counter);
void validate_strategy(const StrategyConfig& cfg, const ModelSpec& spec);

struct DeviceTrainConfig {
    ModelSpec spec;
    StrategyConfig strategy;
    int total_steps = 0;
    int num_ranks = 1;
    AdamHyperparams hyper; // base; weight_decay applies to decay groups
    bool magnitude = false; // update-magnitude selective checkpointing (label "magnitude")
    double rho = 0.5;
    int device = 0;
};

class DeviceTrainer {
  public:
    // Holds rank partitions [rank_begin, rank_end) of the num_ranks layout
    // (default: all). save() needs every rank; step() works on any subset —
    // one rank partition per GPU in a ZeRO job.
    DeviceTrainer(const ModelSpec& spec, int num_ranks, const AdamHyperparams& base, int device, int rank_begin = 0,
                  int rank_end = -1);
    std::uint64_t elements() const; // true (unpadded) optimizer elements held
    ~DeviceTrainer();
    // One train_step at training step `step` (R/src/trainer.cpp:26-35): returns
    // {grad_norm, update_norm}. Throws NonFinite before touching the state.
    std::pair<double, double> step(std::int64_t step);
    std::int64_t optimizer_t() const { return t_; }
    // write_checkpoint of the given module subset (R/src/trainer.cpp:60-79).
    void save(const std::filesystem::path& dir, const TrainerMeta& meta, const std::vector<ModuleId>& modules,
              const std::string& label);
    // In-situ scorer: keep a device copy of the current masters; score the
    // current state against the kept copy -> per module (sum d^2, sum ref^2).
    void keep_masters();
    std::vector<std::pair<double, double>> score_against_kept();
    const ModelLayout& model() const { return model_; }
    // resume (R/src/trainer.cpp:125-152): replace the state with a complete fine
    // checkpoint's (rank payloads byte for byte, per-group hyperparameters from its
    // optim_meta, the optimizer step counter); the caller has verified it.
    void load(const std::filesystem::path& dir, const CheckpointSummary& s);
    // Device partition of rank r (payload layout of optim/rank_r.shard) and its
    // size, for in-situ consumers (scorers, diagnostics); synchronizes first.
    std::pair<std::uint8_t*, std::uint64_t> partition(int rank);

  private:
    struct Rank;
    ModelLayout model_;
    int N_;
    int r0_ = 0, r1_ = 0;
    std::uint64_t elements_ = 0;
    AdamHyperparams base_;
    CheckpointLayout full_;
    std::vector<std::unique_ptr<Rank>> ranks_;
    DeviceBuffer coef_, part_ptrs_, flag_;
    std::int64_t t_ = 0;
    cudaStream_t stream_ = nullptr;
    // Pass 2 recomputes the gradient (28 B/element) unless TAILOR_TRAIN_STORE_GRAD=1
    // selects the scratch-buffer variant (36 B/element; kept for comparison).
    bool store_grad_ = false;
    // The bias corrections divide by a per-step constant through its precomputed
    // reciprocal (kernels/ieee_div.cuh); TAILOR_TRAIN_FDIV=1 keeps __fdiv_rn per element.
    bool fdiv_ = false;
    std::vector<AdamHyperparams> hyper_; // per group (GroupState::hyper)
    // The fast pre-update check of step s+1 is folded into step s's update pass (it sees
    // every new master as it writes it): masters_checked_ = the current masters are known
    // finite, masters_bad_ = known not finite. Any other writer of the state (load,
    // partition() access) clears both, and the next step runs the standalone check.
    DeviceBuffer next_flag_;
    bool masters_checked_ = false, masters_bad_ = false;
};

// The reference's train() (R/src/trainer.cpp:109-123) on the device: same run
// directory layout, checkpoints byte-identical for full/parity/filter.
std::vector<std::filesystem::path> device_train(const DeviceTrainConfig& cfg, const std::filesystem::path& out_dir);

// The reference's resume() (R/src/trainer.cpp:125-152) on the device: read + verify a
// complete fine checkpoint, continue `additional_steps` steps with its strategy and
// rank count, writing checkpoints and log.jsonl into a fresh out_dir.
std::vector<std::filesystem::path> device_resume(const std::filesystem::path& checkpoint_dir, std::int64_t additional_steps,
                                                 const std::filesystem::path& out_dir, int device);

} // namespace tailor
