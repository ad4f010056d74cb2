// Host-side engine binding layer-map plans to the device kernels:
//   SnapshotSet  — layouts of snapshots S_1..S_K (synthetic, or read from checkpoint dirs)
//   SynthFamily  — a SnapshotSet plus the K5 generator of its payloads (synthetic sources)
//   ScorePlan    — K3/K4 tile tables for one rank partition of K snapshots
//   DeviceMerge  — K2 segment table for one output partition, bound to device windows
//   HostMerge    — the shard pipeline: pinned host sources -> H2D -> K2 -> D2H, chunked,
//                  on three streams (H2D / gather / D2H, event-ordered) so transfers
//                  overlap the gather
#pragma once

#include <cstdint>
#include <mutex>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "tailor/checkpoint.hpp"
#include "tailor/device.hpp"
#include "tailor/merge.hpp"

namespace tailor {

void cuda_check(cudaError_t e, const char* what);

class DeviceBuffer {
  public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) { resize(n); }
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_), cap_(o.cap_), dev_(o.dev_) {
        o.p_ = nullptr;
        o.n_ = o.cap_ = 0;
    }
    void resize(std::size_t n); // discards contents
    template <typename T = std::uint8_t>
    T* get() const { return static_cast<T*>(p_); }
    std::size_t size() const { return n_; }
    void upload(const void* src, std::size_t n, cudaStream_t s = nullptr);

  private:
    void* p_ = nullptr;
    std::size_t n_ = 0;   // bytes requested (largest so far)
    std::size_t cap_ = 0; // bytes allocated (pool size class)
    int dev_ = 0;
};

// Device bytes the file-facing paths may plan for: half of (free - 2 GB), capped by
// TAILOR_DEVICE_BUDGET (bytes; tests use it to force the streaming forms).
std::uint64_t device_budget();

// Counters of fresh (non-pooled) allocations, printed by TAILOR_TRACE=1.
struct AllocStats {
    std::mutex mu;
    std::size_t pinned_count = 0, device_count = 0, pinned_bytes = 0, device_bytes = 0;
    double pinned_ms = 0.0, device_ms = 0.0;
    void note(bool pinned, std::size_t bytes, double ms);
    void trace(const char* where);
};
AllocStats& alloc_stats();

class PinnedBuffer {
  public:
    PinnedBuffer() = default;
    explicit PinnedBuffer(std::size_t n) { resize(n); }
    ~PinnedBuffer();
    PinnedBuffer(const PinnedBuffer&) = delete;
    PinnedBuffer& operator=(const PinnedBuffer&) = delete;
    void resize(std::size_t n);
    std::uint8_t* get() const { return static_cast<std::uint8_t*>(p_); }
    std::size_t size() const { return n_; }

  private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
};

// sigma_j(m) = 1e-6 * g^{pi_j(m)}, g = 1000^{1/(M-1)} (SURVEY §8d ladder).
std::vector<float> synth_sigma(std::uint64_t seed, int M, int j);

// The layouts of K snapshots S_1..S_K of one model over N ZeRO ranks — what the
// device plans (scorer tiles, merge segments, K9 tables) are built from. Either
// synthetic (every snapshot full unless set_partial; ids "S1".."SK", step k*interval)
// or read from real checkpoint directories (read_checkpoint_summary of each: spec,
// rank count, manifest module set, step; ids = the directory paths). It owns no
// payload bytes: callers (a trainer, a loader, the generator below) own the device
// buffers and bind them to the plans.
class SnapshotSet {
  public:
    SnapshotSet(const ModelSpec& spec, int num_ranks, int snapshots, std::int64_t interval);
    // Snapshot k = dirs[k-1]; all must share geometry, rank count and the fine grouping.
    static std::unique_ptr<SnapshotSet> from_checkpoints(const std::vector<std::string>& dirs);
    virtual ~SnapshotSet() = default;
    virtual void set_partial(int k, const std::vector<ModuleId>& modules);

    const ModelLayout& model() const { return model_; }
    int num_ranks() const { return num_ranks_; }
    int snapshots() const { return K_; }
    std::int64_t step(int k) const;
    const CheckpointLayout& layout(int k) const;
    CheckpointSummary summary(int k, const std::string& dir) const;
    std::string trainer_state_json(int k) const;
    std::string manifest_json(int k) const;
    std::string optim_meta_json(int k) const;
    const std::string& id(int k) const { return ids_[static_cast<std::size_t>(k - 1)]; }
    void set_id(int k, const std::string& id) { ids_[static_cast<std::size_t>(k - 1)] = id; }
    int index_of(const std::string& id) const; // 1-based; 0 if unknown
    // Masters only, packed per field in score-field order (the scorer's packed layout).
    std::uint64_t packed_master_bytes(int rank) const;

  protected:
    ModelLayout model_;
    int num_ranks_;
    int K_;
    std::int64_t interval_;
    std::vector<std::vector<ModuleId>> modules_;
    std::vector<std::unique_ptr<CheckpointLayout>> layouts_;
    std::vector<std::string> ids_;
    std::vector<CheckpointSummary> real_; // from_checkpoints: the on-disk summaries
};

class SynthFamily : public SnapshotSet {
  public:
    SynthFamily(const ModelSpec& spec, int num_ranks, int snapshots, std::int64_t interval);
    void set_partial(int k, const std::vector<ModuleId>& modules) override;

    // Device generation. Snapshots k0..k1 must share one layout.
    void gen_shard(int rank, int k0, int k1, std::uint8_t* const* outs, cudaStream_t s);
    // Weights payload bytes [lo, hi) of snapshot layout (tensor-aligned), window base = lo.
    void gen_weights(int k0, int k1, std::uint64_t lo, std::uint64_t hi, std::uint8_t* const* outs, cudaStream_t s);
    // Masters only, packed per field in score-field order (for scorer-only sweeps).
    void gen_masters_packed(int rank, int k0, int k1, std::uint8_t* const* outs, cudaStream_t s);
    // bytes [lo, hi) of snapshot k's rank shard payload; entry-aligned (synchronous table upload)
    void gen_shard_range(int rank, int k, std::uint64_t lo, std::uint64_t hi, std::uint8_t* out, cudaStream_t s);
    // GPU-generate snapshot k and write it as a checkpoint directory.
    void write_dir(int k, const std::string& dir);

  private:
    struct ShardTables {
        DeviceBuffer groups, slices;
        std::uint32_t ngroups = 0;
        std::uint64_t total = 0;
    };
    ShardTables& shard_tables(int k, int rank, bool packed);
    void ensure_sigma(int kmax);

    std::map<std::tuple<int, int, bool>, std::unique_ptr<ShardTables>> tables_;
    DeviceBuffer sigma_;
    int sigma_rows_ = 0;
    DeviceBuffer wtab_;
};

// Score fields of one rank partition: every group's master chunk, module-major
// in canonical module order (groups in group_indices_for order).
struct ScoreField {
    int module;
    int group;
    std::int64_t chunk;
};
std::vector<ScoreField> score_fields(const ModelLayout& model, int num_ranks);

class ScorePlan {
  public:
    // field_offsets[k][f]: byte offset of field f's master chunk inside
    // snapshot k's buffer.
    ScorePlan(const ModelLayout& model, int num_ranks, std::vector<std::vector<std::uint64_t>> field_offsets,
              std::uint32_t tile_elems = 32768);
    int K() const { return K_; }
    int M() const { return M_; }
    std::uint64_t bytes_read() const { return bytes_; }
    // out: device [K-1][M][2] FP64 (sum delta^2, sum ref^2) for this rank. Any K >= 2:
    // sweeps longer than 16 snapshots run as K3 launches over windows of <= 16
    // snapshots overlapping by one (bytes_read counts the overlap snapshot twice).
    void run(const std::uint8_t* const* snap_bases, double* d_out, cudaStream_t s);
    void set_variant(int v) { variant_ = v; }

  private:
    int variant_ = dev::kScoreAuto; // TAILOR_SCORE_VARIANT (diagnostics) sets the default; set_variant overrides
    int K_, M_;
    std::vector<ScoreField> fields_;
    std::vector<std::pair<int, int>> windows_; // [first, last] snapshot of each K3 launch (<= 16, overlapping by one)
    std::vector<std::vector<std::uint64_t>> offs_;
    std::vector<dev::ScoreTile> tiles_;
    std::vector<std::uint32_t> begin_;
    DeviceBuffer d_tiles_, d_begin_, d_bases_, d_partials_;
    DeviceBuffer d_counter_; // K3's dynamic tile counter (zeroed before each launch)
    bool dynamic_ = true;    // TAILOR_SCORE_STATIC=1: static tile split (diagnostics)
    PinnedBuffer h_bases_;
    std::vector<const std::uint8_t*> bound_;
    std::uint64_t bytes_ = 0;
    bool aligned_offsets_ = true;
};

class DeviceMerge {
  public:
    explicit DeviceMerge(const PartitionPlan& plan);
    const PartitionPlan& plan() const { return plan_; }
    // window_ptrs[w] = device address of window w's first byte (window.lo).
    void bind(const std::vector<const std::uint8_t*>& window_ptrs);
    // d_dst points at output payload byte dst_lo.
    void run(std::uint8_t* d_dst, int variant, cudaStream_t s);
    bool bulk_ok() const { return bulk_ok_; }
    std::uint64_t bytes() const { return plan_.dst_hi - plan_.dst_lo; }

  private:
    PartitionPlan plan_;
    DeviceBuffer d_segs_;
    DeviceBuffer counter_; // K2's dynamic tile counter (two words, zero between launches)
    std::uint32_t nseg_ = 0;
    bool bulk_ok_ = false;
};

// A whole score -> select -> merge step on the device for one unit (rank-r
// shard + weights share u/units) of a family of FULL snapshots: K9 turns the
// (all-gathered) per-rank scorer partials into the selection and both segment
// tables, then K2 gathers. No host synchronization; graph-capturable. The
// selection is bitwise the host's (select_by_magnitude).
class DeviceSelectStep {
  public:
    DeviceSelectStep(const SnapshotSet& snaps, int rank, int unit, int units, double rho);
    std::uint64_t shard_bytes() const { return shard_bytes_; }
    std::uint64_t weights_lo() const { return wlo_; }
    std::uint64_t weights_hi() const { return whi_; }
    // shard_bases[k]: snapshot k+1's rank shard payload; wwin_bases[k]: its weights bytes [wlo, whi)
    void bind(const std::uint8_t* const* shard_bases, const std::uint8_t* const* wwin_bases);
    // phases: bitmask of kPhaseSelect (K9), kPhaseShard / kPhaseWeights (the two K2 gathers)
    static constexpr int kPhaseSelect = 1, kPhaseShard = 2, kPhaseWeights = 4, kPhaseAll = 7;
    void run(const double* d_parts, int nranks, std::uint8_t* d_out_shard, std::uint8_t* d_out_w, int variant, cudaStream_t s,
             int phases = kPhaseAll);
    std::vector<int> source_of(cudaStream_t s);
    std::vector<double> scores(cudaStream_t s);

  private:
    int K_, M_, n_save_;
    std::uint64_t shard_bytes_ = 0, wlo_ = 0, whi_ = 0;
    std::uint32_t n_shard_ = 0, n_w_ = 0;
    DeviceBuffer shard_entries_, w_entries_, shard_segs_, w_segs_, source_, scores_;
    DeviceBuffer counters_; // K2's dynamic tile counters: [0..1] shard gather, [2..3] weights gather
    dev::SnapshotBases bases_{};
    bool entries_aligned_ = false;
    bool bulk_ = false;
};

// Pipelined host->device->host assembly of one partition from host (pinned)
// source windows into a host destination: per chunk, only the bytes the
// chunk needs are copied in, gathered on the device and copied out. Source
// byte ranges listed as `resident` (window-relative) are read straight from
// device copies instead (e.g. masters already staged for scoring).
//
// All host->device copies of a GPU go through one copy engine in submission
// order (measured: a 1 MB H2D on another stream waits behind a 2 GB one,
// tools/pcie_ce_probe.cu), so the pipeline owns the order: one H2D stream
// carries the chunk inputs and, between them, slices of the caller's
// `prefetch` copies (e.g. the next unit's masters), sized so that each chunk's
// H2D time matches its D2H time; a gather stream and a D2H stream follow via
// events. The link then stays busy in both directions.
struct HostCopy {
    const std::uint8_t* src; // pinned host
    std::uint8_t* dst;       // device
    std::uint64_t bytes;
};

class HostMerge {
  public:
    // Per window: byte ranges [lo, hi) (window-relative) that are read from device
    // memory instead of crossing PCIe; byte x lives at d_windows[w] + dev_off + (x - lo)
    // (dev_off = lo: a device copy in the window's own layout).
    struct ResidentRange {
        std::uint64_t lo, hi, dev_off;
        bool operator==(const ResidentRange&) const = default;
    };
    using Resident = std::vector<std::vector<ResidentRange>>;
    explicit HostMerge(const PartitionPlan& plan, std::uint64_t chunk_bytes = 256ull << 20, Resident resident = {});
    ~HostMerge();
    // h_windows[w] = host address of window w's first byte; d_windows[w] = device
    // address (only needed for windows with resident ranges); h_dst = output byte dst_lo.
    void run(const std::vector<const std::uint8_t*>& h_windows, const std::vector<const std::uint8_t*>& d_windows,
             std::uint8_t* h_dst, int variant, bool async = false, const std::vector<HostCopy>& prefetch = {});
    void wait();
    std::uint64_t h2d_bytes() const { return h2d_; }
    std::uint64_t d2h_bytes() const { return d2h_; }

  private:
    static constexpr int kInSlots = 3, kOutSlots = 2;
    struct Piece {
        std::uint32_t w;
        std::uint64_t src, dst, n;
        bool dev;
        std::uint64_t stage = 0; // host pieces: offset in the staging slot; device pieces: offset from d_windows[w]
    };
    struct Read {
        std::uint32_t w;
        std::uint64_t a, b, at;
    };
    struct Chunk {
        std::uint64_t lo, hi; // output range (relative to dst_lo)
        std::vector<Piece> pieces;
        std::vector<Read> reads;
        std::uint64_t staging = 0, in_bytes = 0;
    };
    PartitionPlan plan_;
    Resident resident_;
    std::vector<Chunk> chunks_;
    std::uint64_t max_staging_ = 0, max_out_ = 0;
    DeviceBuffer stage_[kInSlots], segs_[kInSlots], out_[kOutSlots];
    cudaStream_t h2d_s_ = nullptr, gather_s_ = nullptr, d2h_s_ = nullptr;
    cudaEvent_t loaded_[kInSlots]{}, consumed_[kInSlots]{}, gathered_[kOutSlots]{}, drained_[kOutSlots]{};
    PinnedBuffer patched_;                 // per-chunk segment tables (pinned: the async
    std::vector<std::size_t> patched_at_;  // uploads must not sync the stream)
    std::uint64_t h2d_ = 0, d2h_ = 0;
};

// Device re-verify of a checkpoint directory (duality, zero padding,
// exp_avg_sq >= 0) plus the structural checks of read_checkpoint.
void verify_checkpoint_dir(const std::string& dir, int device);

// The pieces of the device re-verify (read_checkpoint's checks), reusable by callers
// that already hold the layouts (execute_merge verifies files as its lanes finish them):
// verify_plan = structural checks + per-rank work lists as payload offsets;
// verify_rank_resident = load one rank payload, run K6 against the device weights payload
// that `weights` returns (counters at d_err[3r..3r+2]; `weights` may block, e.g. until the
// weights are in);
// verify_counters = the errors, in rank order.
struct VerifyPlan {
    ContainerLayout weights;
    std::vector<ContainerLayout> shards;
    std::vector<std::vector<dev::VerifyPair>> pairs;   // master / weight offsets
    std::vector<std::vector<dev::VerifyRange>> ranges; // payload offsets
    std::uint64_t max_shard = 16;
};
VerifyPlan verify_plan(const std::filesystem::path& dir, const CheckpointSummary& s, ContainerLayout weights,
                       std::vector<ContainerLayout> shards);
void verify_rank_resident(const VerifyPlan& plan, int r, const std::filesystem::path& shard_file, DeviceBuffer& ds,
                          DeviceBuffer& dpairs, DeviceBuffer& dranges, PinnedBuffer* stage, int readers, std::uint64_t step,
                          unsigned long long* d_err, cudaStream_t st, const std::function<const std::uint8_t*()>& weights);
void verify_counters(const std::filesystem::path& dir, int num_ranks, const unsigned long long* d_err);
void verify_counters_host(const std::filesystem::path& dir, int num_ranks, const unsigned long long* err);
void load_payload_to(const std::filesystem::path& path, const ContainerLayout& lay, DeviceBuffer& dst, PinnedBuffer* stage,
                     int threads, std::uint64_t step);

} // namespace tailor
