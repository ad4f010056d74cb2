// Host engine: synthetic families, scorer plans, device/host merge plans and
// the device re-verify (see tailor/engine.hpp).
#include "tailor/engine.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <unistd.h>

#include "tailor/errors.hpp"
#include "tailor/io.hpp"

namespace tailor {

namespace fs = std::filesystem;

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ErrorKind::Device, std::string(what) + ": " + cudaGetErrorString(e));
}

AllocStats& alloc_stats() {
    static AllocStats* s = new AllocStats();
    return *s;
}

void AllocStats::note(bool pinned, std::size_t bytes, double ms) {
    std::lock_guard<std::mutex> lk(mu);
    (pinned ? pinned_bytes : device_bytes) += bytes;
    (pinned ? pinned_ms : device_ms) += ms;
    (pinned ? pinned_count : device_count) += 1;
}

void AllocStats::trace(const char* where) {
    if (!trace_enabled()) return;
    std::lock_guard<std::mutex> lk(mu);
    std::fprintf(stderr, "[tailor] %s: new pinned %zu blocks %.1f MB in %.1f ms (thread-sum), new device %zu blocks %.1f MB in %.1f ms\n",
                 where, pinned_count, pinned_bytes / 1048576.0, pinned_ms, device_count, device_bytes / 1048576.0, device_ms);
}

// cudaMalloc of a large block can take 10-350 ms on a busy process (measured in
// the file scorer lanes: tools/files_trace.py), so released device blocks up to
// 2 GB are kept per device in size classes (cap 8 GB per device) and reused.
// Release keeps cudaFree's implicit device synchronisation, so a block is never
// handed out while a kernel launched before the release may still use it.
namespace {
std::size_t pool_size_class(std::size_t n) {
    std::size_t base = 2u << 20;
    while (base * 2 <= n) base <<= 1;
    for (std::size_t q = 4; q <= 8; ++q)
        if (base / 4 * q >= n) return base / 4 * q;
    return base * 2;
}

struct DevicePool {
    static constexpr std::size_t kCap = 8ull << 30, kMaxBlock = 2ull << 30;
    std::mutex mu;
    std::map<int, std::multimap<std::size_t, void*>> free_; // device -> size class -> block
    std::map<int, std::size_t> pooled;

    // TAILOR_DEVICE_POOL=0 turns pooling off (plain cudaMalloc / cudaFree), for comparisons
    const bool enabled = [] {
        const char* v = std::getenv("TAILOR_DEVICE_POOL");
        return !(v && *v == '0');
    }();
    void* take(int dev, std::size_t n, std::size_t* got) {
        const std::size_t sz = enabled && n <= kMaxBlock ? pool_size_class(n) : n;
        if (sz <= kMaxBlock) {
            std::lock_guard<std::mutex> lk(mu);
            auto& f = free_[dev];
            auto it = f.find(sz);
            if (it != f.end()) {
                void* p = it->second;
                pooled[dev] -= sz;
                f.erase(it);
                *got = sz;
                return p;
            }
        }
        void* p = nullptr;
        const double t0 = clock_ms();
        cuda_check(cudaMalloc(&p, sz), "cudaMalloc");
        alloc_stats().note(false, sz, clock_ms() - t0);
        *got = sz;
        return p;
    }
    void give(int dev, void* p, std::size_t sz) {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        if (sz > kMaxBlock || !enabled) {
            cudaFree(p);
        } else {
            cudaDeviceSynchronize();
            std::lock_guard<std::mutex> lk(mu);
            free_[dev].emplace(sz, p);
            pooled[dev] += sz;
            auto& f = free_[dev];
            while (pooled[dev] > kCap && !f.empty()) {
                auto it = std::prev(f.end());
                pooled[dev] -= it->first;
                cudaFree(it->second);
                f.erase(it);
            }
        }
        if (cur != dev) cudaSetDevice(cur);
    }
};
DevicePool& device_pool() {
    static DevicePool* pool = new DevicePool(); // intentionally leaked: lives for the process
    return *pool;
}
} // namespace

std::uint64_t device_budget() {
    std::size_t free_b = 0, total_b = 0;
    cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    std::uint64_t b = free_b > (2ull << 30) ? (free_b - (2ull << 30)) / 2 : 0;
    if (const char* v = std::getenv("TAILOR_DEVICE_BUDGET"); v && *v) b = std::min<std::uint64_t>(b, std::strtoull(v, nullptr, 10));
    return b;
}

DeviceBuffer::~DeviceBuffer() {
    if (p_) device_pool().give(dev_, p_, cap_);
}

void DeviceBuffer::resize(std::size_t n) {
    if (n <= n_ && p_) return;
    if (p_ && n <= cap_) {
        n_ = n;
        return;
    }
    if (p_) device_pool().give(dev_, p_, cap_);
    p_ = nullptr;
    n_ = cap_ = 0;
    if (n == 0) return;
    cuda_check(cudaGetDevice(&dev_), "cudaGetDevice");
    p_ = device_pool().take(dev_, n, &cap_);
    n_ = n;
}

void DeviceBuffer::upload(const void* src, std::size_t n, cudaStream_t s) {
    resize(std::max<std::size_t>(n, 1));
    if (n == 0) return;
    if (s) {
        cuda_check(cudaMemcpyAsync(p_, src, n, cudaMemcpyHostToDevice, s), "upload"); // ordered before s's later work
    } else {
        // cudaMemcpy from pageable memory returns once the bytes are staged, before the DMA
        // has landed, and the legacy stream it uses is not ordered with our non-blocking
        // streams: without this sync a kernel launched right after on another stream can
        // read the buffer's previous contents (a verify table with stale pointers -> an
        // intermittent illegal address).
        cuda_check(cudaMemcpy(p_, src, n, cudaMemcpyHostToDevice), "upload");
        cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "upload");
    }
}

// Pinning pages costs ~0.4 s per GB, far more than the reads the staging
// buffers serve, so released pinned buffers are kept in a process-wide pool
// (bounded) and reused by later calls.
namespace {
struct PinnedPool {
    static constexpr std::size_t kCap = 8ull << 30;
    std::mutex mu;
    std::multimap<std::size_t, void*> free_; // size -> block
    std::size_t pooled = 0;

    // Size classes (2^k x {1, 1.25, 1.5, 1.75}, >= 2 MB), matched exactly: a request never takes a block
    // of another class, so the staging buffers of different phases (16-32 MB
    // assemble slots, 64-128 MB verify / scorer stages) each keep their own
    // blocks, and a warm process never pins again (cudaMallocHost holds a
    // driver lock that stalls every other thread's CUDA calls).
    static std::size_t size_class(std::size_t n) {
        std::size_t base = 2u << 20;
        while (base * 2 <= n) base <<= 1;
        for (std::size_t q = 4; q <= 8; ++q)
            if (base / 4 * q >= n) return base / 4 * q;
        return base * 2;
    }
    void* take(std::size_t n, std::size_t* got) {
        const std::size_t sz = size_class(n);
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = free_.find(sz);
            if (it != free_.end()) {
                void* p = it->second;
                *got = sz;
                pooled -= sz;
                free_.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        const double t0 = clock_ms();
        cuda_check(cudaMallocHost(&p, sz), "cudaMallocHost");
        alloc_stats().note(true, sz, clock_ms() - t0);
        *got = sz;
        return p;
    }
    void give(void* p, std::size_t n) {
        std::lock_guard<std::mutex> lk(mu);
        free_.emplace(n, p);
        pooled += n;
        while (pooled > kCap && !free_.empty()) { // drop the largest blocks first
            auto it = std::prev(free_.end());
            pooled -= it->first;
            cudaFreeHost(it->second);
            free_.erase(it);
        }
    }
};
PinnedPool& pinned_pool() {
    static PinnedPool* pool = new PinnedPool(); // intentionally leaked: lives for the process
    return *pool;
}
} // namespace

PinnedBuffer::~PinnedBuffer() {
    if (p_) pinned_pool().give(p_, n_);
}

void PinnedBuffer::resize(std::size_t n) {
    if (n <= n_ && p_) return;
    if (p_) pinned_pool().give(p_, n_);
    p_ = nullptr;
    n_ = 0;
    if (n == 0) return;
    p_ = pinned_pool().take(n, &n_);
}

// ---- synthetic family ---------------------------------------------------------
namespace {

std::uint64_t mix64(std::uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

std::uint64_t hash3(std::uint64_t seed, std::uint64_t t, std::uint64_t e) {
    std::uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ULL);
    h = mix64(h ^ (t * 0xD1B54A32D192ED03ULL));
    return mix64(h ^ (e * 0x8CB92BA72F3D8DD7ULL));
}

constexpr std::uint64_t kPermSalt = 0x9E2AULL;

std::uint64_t align16(std::uint64_t x) { return (x + 15) & ~15ull; }

} // namespace

std::vector<float> synth_sigma(std::uint64_t seed, int M, int j) {
    std::vector<int> perm(static_cast<std::size_t>(M));
    for (int i = 0; i < M; ++i) perm[static_cast<std::size_t>(i)] = i;
    for (int i = M - 1; i >= 1; --i) {
        const std::uint64_t r = hash3(seed ^ kPermSalt, static_cast<std::uint64_t>(j), static_cast<std::uint64_t>(i));
        std::swap(perm[static_cast<std::size_t>(i)], perm[static_cast<std::size_t>(r % static_cast<std::uint64_t>(i + 1))]);
    }
    const double g = M > 1 ? std::pow(1000.0, 1.0 / static_cast<double>(M - 1)) : 1.0;
    std::vector<float> s(static_cast<std::size_t>(M));
    for (int m = 0; m < M; ++m)
        s[static_cast<std::size_t>(m)] = static_cast<float>(1e-6 * std::pow(g, static_cast<double>(perm[static_cast<std::size_t>(m)])));
    return s;
}

SnapshotSet::SnapshotSet(const ModelSpec& spec, int num_ranks, int snapshots, std::int64_t interval)
    : model_(spec), num_ranks_(num_ranks), K_(snapshots), interval_(interval) {
    if (num_ranks < 1) fail(ErrorKind::Geometry, "num_ranks must be >= 1");
    if (snapshots < 1) fail(ErrorKind::Geometry, "need at least one snapshot");
    if (interval < 1) fail(ErrorKind::Geometry, "interval must be >= 1");
    modules_.assign(static_cast<std::size_t>(K_), model_.modules());
    layouts_.resize(static_cast<std::size_t>(K_));
    for (int k = 1; k <= K_; ++k) ids_.push_back("S" + std::to_string(k));
}

std::unique_ptr<SnapshotSet> SnapshotSet::from_checkpoints(const std::vector<std::string>& dirs) {
    if (dirs.empty()) fail(ErrorKind::Recipe, "no checkpoint directories");
    std::vector<CheckpointSummary> sums;
    for (const auto& d : dirs) sums.push_back(read_checkpoint_summary(d));
    const CheckpointSummary& s0 = sums.front();
    for (const auto& s : sums) {
        if (!s.spec.same_geometry(s0.spec)) fail(ErrorKind::Geometry, "checkpoints disagree on model geometry");
        if (s.optim.num_ranks != s0.optim.num_ranks) fail(ErrorKind::Geometry, "checkpoints disagree on the rank count");
        if (s.optim.grouping != Grouping::Fine) fail(ErrorKind::Geometry, "device plans need the fine grouping");
    }
    auto set = std::make_unique<SnapshotSet>(s0.spec, s0.optim.num_ranks, static_cast<int>(dirs.size()), 1);
    for (std::size_t i = 0; i < dirs.size(); ++i) {
        set->modules_[i] = sums[i].manifest.modules;
        set->ids_[i] = dirs[i];
    }
    set->real_ = std::move(sums);
    return set;
}

std::int64_t SnapshotSet::step(int k) const {
    return real_.empty() ? interval_ * k : real_.at(static_cast<std::size_t>(k - 1)).trainer.step;
}

void SnapshotSet::set_partial(int k, const std::vector<ModuleId>& modules) {
    if (k < 1 || k > K_) fail(ErrorKind::Geometry, "snapshot index out of range");
    if (!real_.empty()) fail(ErrorKind::Consistency, "the module set of a checkpoint on disk comes from its manifest");
    std::vector<ModuleId> sorted;
    for (const auto& m : model_.modules())
        if (std::find(modules.begin(), modules.end(), m) != modules.end()) sorted.push_back(m);
    if (sorted.empty()) fail(ErrorKind::Consistency, "manifest module list is empty");
    modules_[static_cast<std::size_t>(k - 1)] = sorted;
    layouts_[static_cast<std::size_t>(k - 1)].reset();
}

void SynthFamily::set_partial(int k, const std::vector<ModuleId>& modules) {
    SnapshotSet::set_partial(k, modules);
    for (auto it = tables_.begin(); it != tables_.end();)
        it = std::get<0>(it->first) == k ? tables_.erase(it) : std::next(it);
}

const CheckpointLayout& SnapshotSet::layout(int k) const {
    if (k < 1 || k > K_) fail(ErrorKind::Geometry, "snapshot index out of range");
    auto& slot = const_cast<std::unique_ptr<CheckpointLayout>&>(layouts_[static_cast<std::size_t>(k - 1)]);
    if (!slot) slot = std::make_unique<CheckpointLayout>(checkpoint_layout(model_, num_ranks_, modules_[static_cast<std::size_t>(k - 1)]));
    return *slot;
}

int SnapshotSet::index_of(const std::string& id) const {
    for (int k = 1; k <= K_; ++k)
        if (ids_[static_cast<std::size_t>(k - 1)] == id) return k;
    return 0;
}

CheckpointSummary SnapshotSet::summary(int k, const std::string& dir) const {
    if (!real_.empty()) {
        CheckpointSummary s = real_.at(static_cast<std::size_t>(k - 1));
        s.dir = dir;
        return s;
    }
    const CheckpointLayout& lay = layout(k);
    CheckpointSummary s;
    s.dir = dir;
    s.spec = model_.spec();
    s.trainer.step = step(k);
    s.trainer.optimizer_t = step(k);
    s.trainer.strategy.interval = static_cast<int>(interval_);
    s.trainer.checkpoint_counter = k;
    s.trainer.rng_seed = model_.spec().seed;
    s.manifest.step = step(k);
    s.manifest.strategy = lay.modules.size() == model_.modules().size() ? "full" : "manual";
    s.manifest.modules = lay.modules;
    AdamHyperparams base;
    base.weight_decay = kDefaultWeightDecay;
    std::map<int, AdamHyperparams> hyp;
    for (int g : lay.groups) hyp[g] = hyper_for_class(base, model_.table().groups[static_cast<std::size_t>(g)].decay);
    s.optim = make_optim_meta(model_.table(), hyp, ShardGeometry{num_ranks_}, step(k));
    return s;
}

SynthFamily::SynthFamily(const ModelSpec& spec, int num_ranks, int snapshots, std::int64_t interval)
    : SnapshotSet(spec, num_ranks, snapshots, interval) {}

std::string SnapshotSet::trainer_state_json(int k) const { return sidecar_text(summary(k, "").trainer); }
std::string SnapshotSet::manifest_json(int k) const { return sidecar_text(summary(k, "").manifest); }
std::string SnapshotSet::optim_meta_json(int k) const { return sidecar_text(summary(k, "").optim); }

void SynthFamily::ensure_sigma(int kmax) {
    if (kmax <= sigma_rows_) return;
    const int M = model_.module_count();
    std::vector<float> all;
    for (int j = 1; j <= kmax; ++j) {
        const auto row = synth_sigma(model_.spec().seed, M, j);
        all.insert(all.end(), row.begin(), row.end());
    }
    sigma_.upload(all.data(), all.size() * sizeof(float));
    sigma_rows_ = kmax;
}

std::vector<ScoreField> score_fields(const ModelLayout& model, int num_ranks) {
    const ShardGeometry geom{num_ranks};
    std::vector<ScoreField> out;
    for (int m = 0; m < model.module_count(); ++m)
        for (int g : group_indices_for(model.table(), model.modules()[static_cast<std::size_t>(m)]))
            out.push_back({m, g, geom.shard_length(model.table().groups[static_cast<std::size_t>(g)].element_count)});
    return out;
}

std::uint64_t SnapshotSet::packed_master_bytes(int /*rank*/) const {
    std::uint64_t off = 0;
    for (const auto& f : score_fields(model_, num_ranks_)) off = align16(off + static_cast<std::uint64_t>(f.chunk) * 4);
    return off;
}

SynthFamily::ShardTables& SynthFamily::shard_tables(int k, int rank, bool packed) {
    auto key = std::make_tuple(packed ? 0 : k, rank, packed);
    auto it = tables_.find(key);
    if (it != tables_.end()) return *it->second;
    auto t = std::make_unique<ShardTables>();
    const ShardGeometry geom{num_ranks_};
    std::vector<dev::SynthGroup> groups;
    std::vector<dev::SynthSlice> slices;
    std::uint64_t begin = 0;
    const auto add_group = [&](int g, std::uint64_t o_m, std::uint64_t o_v, std::uint64_t o_w) {
        const GroupInfo& info = model_.table().groups[static_cast<std::size_t>(g)];
        const std::int64_t chunk = geom.shard_length(info.element_count);
        dev::SynthGroup sg{};
        sg.begin = begin;
        sg.chunk = static_cast<std::uint64_t>(chunk);
        sg.group_first = static_cast<std::uint64_t>(rank) * static_cast<std::uint64_t>(chunk);
        sg.true_len = static_cast<std::uint64_t>(info.element_count);
        sg.off[0] = o_m;
        sg.off[1] = o_v;
        sg.off[2] = o_w;
        sg.slice_begin = static_cast<std::uint32_t>(slices.size());
        for (const auto& s : model_.slices(g)) slices.push_back({s.group_offset, s.model_offset, s.decl.numel()});
        sg.slice_count = static_cast<std::uint32_t>(model_.slices(g).size());
        sg.module = static_cast<std::uint32_t>(model_.owner_index(g));
        if (chunk > 0) groups.push_back(sg);
        begin += static_cast<std::uint64_t>(chunk);
    };
    if (packed) {
        std::uint64_t off = 0;
        for (const auto& f : score_fields(model_, num_ranks_)) {
            add_group(f.group, ~0ull, ~0ull, off);
            off = align16(off + static_cast<std::uint64_t>(f.chunk) * 4);
        }
    } else {
        const ContainerLayout& c = layout(k).shards[static_cast<std::size_t>(rank)];
        for (int g : layout(k).groups)
            add_group(g, c.find(shard_key(g, ".exp_avg"))->begin, c.find(shard_key(g, ".exp_avg_sq"))->begin,
                      c.find(shard_key(g, ".master"))->begin);
    }
    t->ngroups = static_cast<std::uint32_t>(groups.size());
    t->total = begin;
    t->groups.upload(groups.data(), groups.size() * sizeof(dev::SynthGroup));
    t->slices.upload(slices.data(), slices.size() * sizeof(dev::SynthSlice));
    return *tables_.emplace(key, std::move(t)).first->second;
}

namespace {
dev::OutPtrs out_ptrs(std::uint8_t* const* outs, int n) {
    if (n < 1 || n > dev::kMaxSnapshots) fail(ErrorKind::Geometry, "at most 16 snapshots per generator launch");
    dev::OutPtrs o{};
    for (int i = 0; i < n; ++i) o.p[i] = outs[i];
    return o;
}
} // namespace

void SynthFamily::gen_shard(int rank, int k0, int k1, std::uint8_t* const* outs, cudaStream_t s) {
    if (rank < 0 || rank >= num_ranks_) fail(ErrorKind::Geometry, "rank out of range");
    if (k0 < 1 || k1 > K_ || k0 > k1) fail(ErrorKind::Geometry, "snapshot range out of bounds");
    for (int k = k0 + 1; k <= k1; ++k)
        if (modules_[static_cast<std::size_t>(k - 1)] != modules_[static_cast<std::size_t>(k0 - 1)])
            fail(ErrorKind::Geometry, "snapshots generated together must share one layout");
    ensure_sigma(k1);
    ShardTables& t = shard_tables(k0, rank, false);
    for (int a = k0; a <= k1; a += dev::kMaxSnapshots) { // <= 16 snapshots per launch
        const int b = std::min(k1, a + dev::kMaxSnapshots - 1);
        cuda_check(dev::launch_synth_shard(t.groups.get<dev::SynthGroup>(), t.ngroups, t.slices.get<dev::SynthSlice>(),
                                           sigma_.get<float>(), model_.module_count(), model_.spec().seed, a, b,
                                           out_ptrs(outs + (a - k0), b - a + 1), t.total, s),
                   "synth shard");
    }
}

void SynthFamily::gen_masters_packed(int rank, int k0, int k1, std::uint8_t* const* outs, cudaStream_t s) {
    if (rank < 0 || rank >= num_ranks_) fail(ErrorKind::Geometry, "rank out of range");
    if (k0 < 1 || k1 > K_ || k0 > k1) fail(ErrorKind::Geometry, "snapshot range out of bounds");
    ensure_sigma(k1);
    ShardTables& t = shard_tables(0, rank, true);
    for (int a = k0; a <= k1; a += dev::kMaxSnapshots) {
        const int b = std::min(k1, a + dev::kMaxSnapshots - 1);
        cuda_check(dev::launch_synth_shard(t.groups.get<dev::SynthGroup>(), t.ngroups, t.slices.get<dev::SynthSlice>(),
                                           sigma_.get<float>(), model_.module_count(), model_.spec().seed, a, b,
                                           out_ptrs(outs + (a - k0), b - a + 1), t.total, s),
                   "synth masters");
    }
}

void SynthFamily::gen_shard_range(int rank, int k, std::uint64_t lo, std::uint64_t hi, std::uint8_t* out,
                                  cudaStream_t s) {
    if (rank < 0 || rank >= num_ranks_) fail(ErrorKind::Geometry, "rank out of range");
    if (k < 1 || k > K_) fail(ErrorKind::Geometry, "snapshot out of bounds");
    ensure_sigma(k);
    const ShardGeometry geom{num_ranks_};
    const ContainerLayout& c = layout(k).shards[static_cast<std::size_t>(rank)];
    std::vector<dev::SynthGroup> groups;
    std::vector<dev::SynthSlice> slices;
    std::uint64_t begin = 0;
    for (int g : layout(k).groups) {
        dev::SynthGroup sg{};
        bool any = false;
        int f = 0;
        for (const char* field : {".exp_avg", ".exp_avg_sq", ".master"}) {
            const Entry* e = c.find(shard_key(g, field));
            sg.off[f] = ~0ull;
            if (e->end > lo && e->begin < hi) {
                if (e->begin < lo || e->end > hi) fail(ErrorKind::Geometry, "shard window must be tensor-aligned");
                sg.off[f] = e->begin - lo;
                any = true;
            }
            ++f;
        }
        const GroupInfo& info = model_.table().groups[static_cast<std::size_t>(g)];
        const std::int64_t chunk = geom.shard_length(info.element_count);
        if (!any || chunk <= 0) continue;
        sg.begin = begin;
        sg.chunk = static_cast<std::uint64_t>(chunk);
        sg.group_first = static_cast<std::uint64_t>(rank) * static_cast<std::uint64_t>(chunk);
        sg.true_len = static_cast<std::uint64_t>(info.element_count);
        sg.slice_begin = static_cast<std::uint32_t>(slices.size());
        for (const auto& sl : model_.slices(g)) slices.push_back({sl.group_offset, sl.model_offset, sl.decl.numel()});
        sg.slice_count = static_cast<std::uint32_t>(model_.slices(g).size());
        sg.module = static_cast<std::uint32_t>(model_.owner_index(g));
        groups.push_back(sg);
        begin += static_cast<std::uint64_t>(chunk);
    }
    if (groups.empty()) return;
    if (s) cuda_check(cudaStreamSynchronize(s), "sync");
    DeviceBuffer dg, ds;
    dg.upload(groups.data(), groups.size() * sizeof(dev::SynthGroup));
    ds.upload(slices.data(), slices.size() * sizeof(dev::SynthSlice));
    cuda_check(dev::launch_synth_shard(dg.get<dev::SynthGroup>(), static_cast<std::uint32_t>(groups.size()),
                                       ds.get<dev::SynthSlice>(), sigma_.get<float>(), model_.module_count(),
                                       model_.spec().seed, k, k, out_ptrs(&out, 1), begin, s),
               "synth shard range");
    cuda_check(s ? cudaStreamSynchronize(s) : cudaDeviceSynchronize(), "sync"); // tables are freed on return
}

void SynthFamily::gen_weights(int k0, int k1, std::uint64_t lo, std::uint64_t hi, std::uint8_t* const* outs,
                              cudaStream_t s) {
    if (k0 < 1 || k1 > K_ || k0 > k1) fail(ErrorKind::Geometry, "snapshot range out of bounds");
    ensure_sigma(k1);
    const CheckpointLayout& lay = layout(k0);
    std::map<std::string, std::pair<std::int64_t, int>> where; // tensor -> (model offset, module)
    for (int m = 0; m < model_.module_count(); ++m) {
        std::int64_t off = model_.module_offset(m);
        for (const auto& t : tensors_of(model_.spec(), model_.modules()[static_cast<std::size_t>(m)])) {
            where[t.name] = {off, m};
            off += t.numel();
        }
    }
    std::vector<dev::SynthTensor> tabs;
    std::uint64_t begin = 0;
    for (const auto& e : lay.weights.entries) {
        if (e.end <= lo || e.begin >= hi) continue;
        if (e.begin < lo || e.end > hi) fail(ErrorKind::Geometry, "weights window must be tensor-aligned");
        const auto& w = where.at(e.name);
        const std::uint64_t n = e.bytes() / 2;
        tabs.push_back({begin, n, e.begin - lo, w.first, static_cast<std::uint32_t>(w.second), 0});
        begin += n;
    }
    if (tabs.empty()) return;
    if (s) cuda_check(cudaStreamSynchronize(s), "sync");
    wtab_.upload(tabs.data(), tabs.size() * sizeof(dev::SynthTensor));
    for (int a = k0; a <= k1; a += dev::kMaxSnapshots) {
        const int b = std::min(k1, a + dev::kMaxSnapshots - 1);
        cuda_check(dev::launch_synth_weights(wtab_.get<dev::SynthTensor>(), static_cast<std::uint32_t>(tabs.size()),
                                             sigma_.get<float>(), model_.module_count(), model_.spec().seed, a, b,
                                             out_ptrs(outs + (a - k0), b - a + 1), begin, s),
                   "synth weights");
    }
    cuda_check(cudaStreamSynchronize(s), "sync");
}

namespace {

void write_bytes_file(const fs::path& path, const std::string& prefix, const std::uint8_t* payload, std::uint64_t n) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(ErrorKind::Storage, "cannot create '" + path.string() + "'");
    out.write(prefix.data(), static_cast<std::streamsize>(prefix.size()));
    if (n) out.write(reinterpret_cast<const char*>(payload), static_cast<std::streamsize>(n));
    out.flush();
    if (!out) fail(ErrorKind::Storage, "write failed for '" + path.string() + "'");
}

} // namespace

void SynthFamily::write_dir(int k, const std::string& dir) {
    const CheckpointLayout& lay = layout(k);
    std::error_code ec;
    fs::create_directories(fs::path(dir) / "optim", ec);
    if (ec) fail(ErrorKind::Storage, "cannot create '" + dir + "': " + ec.message());
    std::uint64_t most = lay.weights.payload_bytes;
    for (const auto& c : lay.shards) most = std::max(most, c.payload_bytes);
    DeviceBuffer d(std::max<std::uint64_t>(most, 16));
    std::vector<std::uint8_t> h(most);
    std::uint8_t* outs[1] = {d.get()};
    gen_weights(k, k, 0, lay.weights.payload_bytes, outs, nullptr);
    cuda_check(cudaMemcpy(h.data(), d.get(), lay.weights.payload_bytes, cudaMemcpyDeviceToHost), "D2H");
    write_bytes_file(ckpt_file(CkptFile::Weights, dir), lay.weights.prefix(), h.data(), lay.weights.payload_bytes);
    for (int r = 0; r < num_ranks_; ++r) {
        gen_shard(r, k, k, outs, nullptr);
        const auto& c = lay.shards[static_cast<std::size_t>(r)];
        cuda_check(cudaMemcpy(h.data(), d.get(), c.payload_bytes, cudaMemcpyDeviceToHost), "D2H");
        write_bytes_file(ckpt_file(CkptFile::Shard, dir, r), c.prefix(), h.data(), c.payload_bytes);
    }
    const CheckpointSummary s = summary(k, dir);
    write_text_file(ckpt_file(CkptFile::OptimMeta, dir), sidecar_text(s.optim));
    write_text_file(ckpt_file(CkptFile::Config, dir), sidecar_text(s.spec));
    write_text_file(ckpt_file(CkptFile::TrainerState, dir), sidecar_text(s.trainer));
    write_text_file(ckpt_file(CkptFile::Manifest, dir), sidecar_text(s.manifest));
    set_id(k, dir);
}

// ---- scorer plan ----------------------------------------------------------------
ScorePlan::ScorePlan(const ModelLayout& model, int num_ranks, std::vector<std::vector<std::uint64_t>> field_offsets,
                     std::uint32_t tile_elems)
    : K_(static_cast<int>(field_offsets.size())), M_(model.module_count()), offs_(std::move(field_offsets)) {
    if (K_ < 2) fail(ErrorKind::Geometry, "scoring needs at least 2 snapshots");
    // K3 holds up to 16 snapshots per launch; longer sweeps run as windows of <= 16
    // snapshots that overlap by one (pairs never straddle a window)
    for (int s0 = 0; s0 < K_ - 1; s0 += dev::kMaxSnapshots - 1)
        windows_.push_back({s0, std::min(K_ - 1, s0 + dev::kMaxSnapshots - 1)});
    if (const char* v = std::getenv("TAILOR_SCORE_VARIANT"); v && *v) variant_ = std::atoi(v);
    if (const char* v = std::getenv("TAILOR_SCORE_STATIC"); v && *v == '1') dynamic_ = false; // diagnostics
    d_counter_.resize(16);
    tile_elems = std::max<std::uint32_t>(4, tile_elems & ~3u);
    fields_ = score_fields(model, num_ranks);
    for (const auto& o : offs_) {
        if (o.size() != fields_.size()) fail(ErrorKind::Geometry, "field offset table has the wrong size");
        for (auto x : o) aligned_offsets_ = aligned_offsets_ && (x % 16 == 0);
    }
    begin_.assign(static_cast<std::size_t>(M_) + 1, 0);
    int cur = -1;
    for (std::size_t f = 0; f < fields_.size(); ++f) {
        const ScoreField& sf = fields_[f];
        while (cur < sf.module) begin_[static_cast<std::size_t>(++cur)] = static_cast<std::uint32_t>(tiles_.size());
        for (std::int64_t s = 0; s < sf.chunk; s += tile_elems) {
            const std::uint32_t n = static_cast<std::uint32_t>(std::min<std::int64_t>(tile_elems, sf.chunk - s));
            tiles_.push_back({static_cast<std::uint32_t>(sf.module), static_cast<std::uint32_t>(f), n, 0,
                              static_cast<std::uint64_t>(s)});
        }
        for (const auto& w : windows_) bytes_ += static_cast<std::uint64_t>(sf.chunk) * 4 * static_cast<std::uint64_t>(w.second - w.first + 1);
    }
    while (cur < M_) begin_[static_cast<std::size_t>(++cur)] = static_cast<std::uint32_t>(tiles_.size());
    d_tiles_.upload(tiles_.data(), tiles_.size() * sizeof(dev::ScoreTile));
    d_begin_.upload(begin_.data(), begin_.size() * sizeof(std::uint32_t));
    d_partials_.resize(std::max<std::size_t>(1, tiles_.size()) * 2 *
                       static_cast<std::size_t>(std::min(K_, static_cast<int>(dev::kMaxSnapshots)) - 1) * sizeof(double));
    h_bases_.resize(static_cast<std::size_t>(K_) * fields_.size() * sizeof(void*) + 8);
    d_bases_.resize(static_cast<std::size_t>(K_) * fields_.size() * sizeof(void*) + 8);
}

void ScorePlan::run(const std::uint8_t* const* snap_bases, double* d_out, cudaStream_t s) {
    const std::vector<const std::uint8_t*> want(snap_bases, snap_bases + K_);
    bool vec = aligned_offsets_;
    for (auto* p : want) vec = vec && (reinterpret_cast<std::uintptr_t>(p) % 16 == 0);
    if (want != bound_) {
        const float** h = reinterpret_cast<const float**>(h_bases_.get());
        for (int k = 0; k < K_; ++k)
            for (std::size_t f = 0; f < fields_.size(); ++f)
                h[static_cast<std::size_t>(k) * fields_.size() + f] =
                    reinterpret_cast<const float*>(want[static_cast<std::size_t>(k)] + offs_[static_cast<std::size_t>(k)][f]);
        cuda_check(cudaMemcpyAsync(d_bases_.get(), h, static_cast<std::size_t>(K_) * fields_.size() * sizeof(void*),
                                   cudaMemcpyHostToDevice, s),
                   "bases upload");
        cuda_check(cudaStreamSynchronize(s), "sync");
        bound_ = want;
    }
    for (const auto& [w0, w1] : windows_) { // pairs w0..w1-1 of the sweep
        const int Kw = w1 - w0 + 1;
        cuda_check(dev::launch_score_partials(d_tiles_.get<dev::ScoreTile>(), static_cast<std::uint32_t>(tiles_.size()),
                                              d_bases_.get<const float*>() + static_cast<std::size_t>(w0) * fields_.size(),
                                              static_cast<std::uint32_t>(fields_.size()), Kw, vec, d_partials_.get<double>(), s,
                                              variant_, dynamic_ ? d_counter_.get<unsigned int>() : nullptr),
                   "score partials");
        cuda_check(dev::launch_score_combine(d_partials_.get<double>(), d_begin_.get<std::uint32_t>(), M_, Kw,
                                             d_out + static_cast<std::size_t>(w0) * M_ * 2, s),
                   "score combine");
    }
}

// ---- device merge -----------------------------------------------------------------
DeviceMerge::DeviceMerge(const PartitionPlan& plan) : plan_(plan) {
    nseg_ = static_cast<std::uint32_t>(plan_.segments.size());
}

void DeviceMerge::bind(const std::vector<const std::uint8_t*>& window_ptrs) {
    if (window_ptrs.size() != plan_.windows.size()) fail(ErrorKind::Geometry, "window pointer count mismatch");
    // The table is immutable while launches may read it: a rebind waits for all
    // outstanding device work (rare; binds happen once per plan in practice).
    if (d_segs_.size()) cuda_check(cudaDeviceSynchronize(), "bind sync");
    std::vector<dev::GatherSeg> segs;
    segs.reserve(plan_.segments.size());
    bool ok = true;
    std::uint64_t expect = plan_.dst_lo;
    for (const auto& s : plan_.segments) {
        const std::uint8_t* src = window_ptrs[s.window] + s.src_off;
        segs.push_back({src, s.dst_off - plan_.dst_lo, s.bytes});
        ok = ok && s.dst_off == expect && (s.dst_off - plan_.dst_lo) % 16 == 0 && s.bytes % 16 == 0 &&
             reinterpret_cast<std::uintptr_t>(src) % 16 == 0;
        expect = s.dst_off + s.bytes;
    }
    bulk_ok_ = ok && expect == plan_.dst_hi;
    d_segs_.upload(segs.data(), segs.size() * sizeof(dev::GatherSeg));
    if (!counter_.size()) { // plans are built without a device; the counter comes with the first bind
        const unsigned int zero[2] = {0, 0};
        counter_.upload(zero, sizeof(zero));
    }
}

void DeviceMerge::run(std::uint8_t* d_dst, int variant, cudaStream_t s) {
    const bool ok = bulk_ok_ && reinterpret_cast<std::uintptr_t>(d_dst) % 16 == 0;
    cuda_check(dev::launch_gather(d_segs_.get<dev::GatherSeg>(), nseg_, d_dst, bytes(), variant, ok, s, counter_.get<unsigned int>()),
               "gather");
}

// ---- host-staged merge (shard pipeline) ------------------------------------------
HostMerge::HostMerge(const PartitionPlan& plan, std::uint64_t chunk_bytes, Resident resident)
    : plan_(plan), resident_(std::move(resident)) {
    resident_.resize(plan_.windows.size());
    chunk_bytes = std::max<std::uint64_t>(16, chunk_bytes & ~15ull);
    const std::uint64_t total = plan_.dst_hi - plan_.dst_lo;
    std::size_t si = 0;
    for (std::uint64_t lo = 0; lo < total; lo += chunk_bytes) {
        Chunk c;
        c.lo = lo;
        c.hi = std::min(total, lo + chunk_bytes);
        std::vector<Piece> ps;
        while (si < plan_.segments.size() && plan_.segments[si].dst_off + plan_.segments[si].bytes - plan_.dst_lo <= c.lo) ++si;
        for (std::size_t j = si; j < plan_.segments.size(); ++j) {
            const auto& s = plan_.segments[j];
            const std::uint64_t d0 = s.dst_off - plan_.dst_lo, d1 = d0 + s.bytes;
            if (d0 >= c.hi) break;
            std::uint64_t a = std::max(d0, c.lo);
            const std::uint64_t b = std::min(d1, c.hi);
            // split at device-resident source ranges: those bytes never cross PCIe
            while (a < b) {
                const std::uint64_t src = s.src_off + (a - d0);
                std::uint64_t n = b - a;
                bool dev_side = false;
                std::uint64_t dev_at = 0;
                for (const auto& rr : resident_[s.window]) {
                    if (src >= rr.lo && src < rr.hi) {
                        dev_side = true;
                        dev_at = rr.dev_off + (src - rr.lo);
                        n = std::min(n, rr.hi - src);
                        break;
                    }
                    if (rr.lo > src) n = std::min(n, rr.lo - src);
                }
                ps.push_back({s.window, src, a, n, dev_side, dev_at});
                a += n;
            }
        }
        // Stage host pieces in source order per window, coalescing contiguous bytes.
        std::vector<std::size_t> order;
        for (std::size_t i = 0; i < ps.size(); ++i)
            if (!ps[i].dev) order.push_back(i);
        std::sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
            return ps[x].w != ps[y].w ? ps[x].w < ps[y].w : ps[x].src < ps[y].src;
        });
        std::uint64_t at = 0;
        for (std::size_t i : order) {
            Piece& p = ps[i];
            if (!c.reads.empty() && c.reads.back().w == p.w && c.reads.back().b == p.src) {
                p.stage = c.reads.back().at + (p.src - c.reads.back().a);
                c.reads.back().b += p.n;
                at = c.reads.back().at + (c.reads.back().b - c.reads.back().a);
                continue;
            }
            at = align16(at) + ((p.dst - c.lo) & 15); // keep src == dst (mod 16)
            c.reads.push_back({p.w, p.src, p.src + p.n, at});
            p.stage = at;
            at += p.n;
        }
        c.staging = align16(at);
        for (const auto& rd : c.reads) c.in_bytes += rd.b - rd.a;
        c.pieces = std::move(ps);
        max_staging_ = std::max(max_staging_, c.staging);
        max_out_ = std::max(max_out_, c.hi - c.lo);
        chunks_.push_back(std::move(c));
    }
}

HostMerge::~HostMerge() {
    for (cudaStream_t s : {h2d_s_, gather_s_, d2h_s_})
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    for (auto* evs : {loaded_, consumed_})
        for (int i = 0; i < kInSlots; ++i)
            if (evs[i]) cudaEventDestroy(evs[i]);
    for (auto* evs : {gathered_, drained_})
        for (int i = 0; i < kOutSlots; ++i)
            if (evs[i]) cudaEventDestroy(evs[i]);
}

void HostMerge::wait() {
    for (cudaStream_t s : {h2d_s_, gather_s_, d2h_s_})
        if (s) cuda_check(cudaStreamSynchronize(s), "sync");
}

void HostMerge::run(const std::vector<const std::uint8_t*>& h_windows, const std::vector<const std::uint8_t*>& d_windows,
                    std::uint8_t* h_dst, int variant, bool async, const std::vector<HostCopy>& prefetch) {
    if (h_windows.size() != plan_.windows.size()) fail(ErrorKind::Geometry, "window pointer count mismatch");
    wait(); // a previous asynchronous run still owns the staging buffers
    std::size_t max_segs = 1;
    for (const auto& c : chunks_) max_segs = std::max(max_segs, c.pieces.size());
    if (!h2d_s_) {
        for (cudaStream_t* s : {&h2d_s_, &gather_s_, &d2h_s_})
            cuda_check(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking), "stream");
        for (auto* evs : {loaded_, consumed_})
            for (int i = 0; i < kInSlots; ++i) cuda_check(cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming), "event");
        for (auto* evs : {gathered_, drained_})
            for (int i = 0; i < kOutSlots; ++i) cuda_check(cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming), "event");
    }
    for (int i = 0; i < kInSlots; ++i) {
        stage_[i].resize(std::max<std::uint64_t>(16, max_staging_));
        segs_[i].resize(max_segs * sizeof(dev::GatherSeg));
    }
    for (int i = 0; i < kOutSlots; ++i) out_[i].resize(std::max<std::uint64_t>(16, max_out_));
    if (patched_at_.size() != chunks_.size() + 1) {
        patched_at_.assign(1, 0);
        for (const auto& c : chunks_) patched_at_.push_back(patched_at_.back() + c.pieces.size());
        patched_.resize(std::max<std::size_t>(1, patched_at_.back()) * sizeof(dev::GatherSeg));
    }
    h2d_ = d2h_ = 0;
    // prefetch cursor: copies are sliced so each chunk's H2D (inputs + slice) matches its D2H
    std::size_t pf = 0;
    std::uint64_t pf_off = 0;
    const auto issue_prefetch = [&](std::uint64_t budget) {
        while (pf < prefetch.size() && budget > 0) {
            const HostCopy& c = prefetch[pf];
            const std::uint64_t n = std::min(budget, c.bytes - pf_off);
            if (n) cuda_check(cudaMemcpyAsync(c.dst + pf_off, c.src + pf_off, n, cudaMemcpyHostToDevice, h2d_s_), "prefetch");
            h2d_ += n;
            budget -= n;
            pf_off += n;
            if (pf_off == c.bytes) {
                ++pf;
                pf_off = 0;
            }
        }
    };
    for (std::size_t ci = 0; ci < chunks_.size(); ++ci) {
        const Chunk& c = chunks_[ci];
        const int in = static_cast<int>(ci % kInSlots), out = static_cast<int>(ci % kOutSlots);
        // H2D: the slot's previous gather must be done with its staging and table
        if (ci >= kInSlots) cuda_check(cudaStreamWaitEvent(h2d_s_, consumed_[in], 0), "wait");
        for (const auto& rd : c.reads) {
            cuda_check(cudaMemcpyAsync(stage_[in].get() + rd.at, h_windows[rd.w] + rd.a, rd.b - rd.a,
                                       cudaMemcpyHostToDevice, h2d_s_),
                       "H2D");
            h2d_ += rd.b - rd.a;
        }
        dev::GatherSeg* segs = reinterpret_cast<dev::GatherSeg*>(patched_.get()) + patched_at_[ci];
        std::size_t nseg = 0;
        bool bulk = true;
        std::uint64_t expect = c.lo;
        for (const auto& p : c.pieces) {
            const std::uint8_t* src;
            if (p.dev) {
                if (d_windows.size() <= p.w || !d_windows[p.w]) fail(ErrorKind::Geometry, "resident window without a device pointer");
                src = d_windows[p.w] + p.stage;
            } else {
                src = stage_[in].get() + p.stage;
            }
            segs[nseg++] = {src, p.dst - c.lo, p.n};
            bulk = bulk && p.dst == expect && reinterpret_cast<std::uintptr_t>(src) % 16 == 0 && p.n % 16 == 0 &&
                   (p.dst - c.lo) % 16 == 0;
            expect = p.dst + p.n;
        }
        bulk = bulk && expect == c.hi;
        cuda_check(cudaMemcpyAsync(segs_[in].get(), segs, nseg * sizeof(dev::GatherSeg), cudaMemcpyHostToDevice, h2d_s_),
                   "segs");
        cuda_check(cudaEventRecord(loaded_[in], h2d_s_), "event");
        const std::uint64_t out_bytes = c.hi - c.lo;
        issue_prefetch(out_bytes > c.in_bytes ? out_bytes - c.in_bytes : 0);
        // gather: inputs loaded, output slot drained by its previous D2H
        cuda_check(cudaStreamWaitEvent(gather_s_, loaded_[in], 0), "wait");
        if (ci >= kOutSlots) cuda_check(cudaStreamWaitEvent(gather_s_, drained_[out], 0), "wait");
        cuda_check(dev::launch_gather(segs_[in].get<dev::GatherSeg>(), static_cast<std::uint32_t>(nseg), out_[out].get(),
                                      out_bytes, variant, bulk, gather_s_),
                   "gather");
        cuda_check(cudaEventRecord(consumed_[in], gather_s_), "event");
        cuda_check(cudaEventRecord(gathered_[out], gather_s_), "event");
        // D2H
        cuda_check(cudaStreamWaitEvent(d2h_s_, gathered_[out], 0), "wait");
        cuda_check(cudaMemcpyAsync(h_dst + c.lo, out_[out].get(), out_bytes, cudaMemcpyDeviceToHost, d2h_s_), "D2H");
        cuda_check(cudaEventRecord(drained_[out], d2h_s_), "event");
        d2h_ += out_bytes;
    }
    issue_prefetch(~0ull);
    if (!async) wait();
}

// ---- device select + plan step ---------------------------------------------------------
DeviceSelectStep::DeviceSelectStep(const SnapshotSet& fam, int rank, int unit, int units, double rho)
    : K_(fam.snapshots()), M_(fam.model().module_count()) {
    if (K_ < 2 || K_ > dev::kMaxSelectSnapshots) fail(ErrorKind::Geometry, "device selection needs 2..64 snapshots");
    if (!(rho > 0.0 && rho <= 1.0)) fail(ErrorKind::Recipe, "selection ratio rho must lie in (0, 1]");
    if (rank < 0 || rank >= fam.num_ranks()) fail(ErrorKind::Geometry, "rank out of range");
    n_save_ = std::max(1, std::min(M_, static_cast<int>(std::ceil(rho * M_))));
    for (int k = 1; k <= K_; ++k)
        if (fam.layout(k).modules.size() != static_cast<std::size_t>(M_))
            fail(ErrorKind::Geometry, "device selection merges full snapshots only");
    const CheckpointLayout& lay = fam.layout(K_);
    const ModelLayout& model = fam.model();
    std::vector<dev::PlanEntry> se, we;
    const ContainerLayout& sl = lay.shards[static_cast<std::size_t>(rank)];
    for (const auto& e : sl.entries) {
        const int g = std::stoi(e.name.substr(1, e.name.find('.') - 1));
        se.push_back({static_cast<std::uint32_t>(model.owner_index(g)), 0, e.begin, e.begin, e.bytes()});
    }
    shard_bytes_ = sl.payload_bytes;
    std::tie(wlo_, whi_) = weights_share(lay.weights, unit, units);
    std::map<std::string, int> owner;
    for (int m = 0; m < M_; ++m)
        for (const auto& t : tensors_of(model.spec(), model.modules()[static_cast<std::size_t>(m)])) owner[t.name] = m;
    for (const auto& e : lay.weights.entries)
        if (e.begin >= wlo_ && e.end <= whi_)
            we.push_back({static_cast<std::uint32_t>(owner.at(e.name)), 0, e.begin - wlo_, e.begin - wlo_, e.bytes()});
    n_shard_ = static_cast<std::uint32_t>(se.size());
    n_w_ = static_cast<std::uint32_t>(we.size());
    bool aligned = true;
    for (const auto* v : {&se, &we})
        for (const auto& p : *v) aligned = aligned && p.dst_off % 16 == 0 && p.bytes % 16 == 0;
    entries_aligned_ = aligned;
    shard_entries_.upload(se.data(), se.size() * sizeof(dev::PlanEntry));
    w_entries_.upload(we.data(), we.size() * sizeof(dev::PlanEntry));
    shard_segs_.resize(std::max<std::size_t>(1, se.size()) * sizeof(dev::GatherSeg));
    w_segs_.resize(std::max<std::size_t>(1, we.size()) * sizeof(dev::GatherSeg));
    source_.resize(static_cast<std::size_t>(M_) * sizeof(int));
    scores_.resize(static_cast<std::size_t>(M_) * (K_ - 1) * sizeof(double));
    const unsigned int zero[4] = {0, 0, 0, 0};
    counters_.upload(zero, sizeof(zero));
}

void DeviceSelectStep::bind(const std::uint8_t* const* shard_bases, const std::uint8_t* const* wwin_bases) {
    // Bases travel by value in the K9 launch parameters: rebinding never races
    // with launches already queued.
    bulk_ = entries_aligned_;
    for (int k = 0; k < K_; ++k) {
        bases_.shard[k] = shard_bases[k];
        bases_.weights[k] = wwin_bases[k];
        bulk_ = bulk_ && reinterpret_cast<std::uintptr_t>(shard_bases[k]) % 16 == 0 &&
                reinterpret_cast<std::uintptr_t>(wwin_bases[k]) % 16 == 0;
    }
}

void DeviceSelectStep::run(const double* d_parts, int nranks, std::uint8_t* d_out_shard, std::uint8_t* d_out_w, int variant,
                           cudaStream_t s, int phases) {
    if (phases & kPhaseSelect)
        cuda_check(dev::launch_select_plan(d_parts, nranks, K_, M_, n_save_, shard_entries_.get<dev::PlanEntry>(), n_shard_,
                                           w_entries_.get<dev::PlanEntry>(), n_w_, bases_, shard_segs_.get<dev::GatherSeg>(),
                                           w_segs_.get<dev::GatherSeg>(), source_.get<int>(), scores_.get<double>(), s),
                   "select plan");
    const bool ok_s = bulk_ && reinterpret_cast<std::uintptr_t>(d_out_shard) % 16 == 0;
    const bool ok_w = bulk_ && reinterpret_cast<std::uintptr_t>(d_out_w) % 16 == 0;
    if (phases & kPhaseShard)
        cuda_check(dev::launch_gather(shard_segs_.get<dev::GatherSeg>(), n_shard_, d_out_shard, shard_bytes_, variant, ok_s, s,
                                      counters_.get<unsigned int>()),
                   "gather shard");
    if (phases & kPhaseWeights)
        cuda_check(dev::launch_gather(w_segs_.get<dev::GatherSeg>(), n_w_, d_out_w, whi_ - wlo_, variant, ok_w, s,
                                      counters_.get<unsigned int>() + 2),
                   "gather weights");
}

std::vector<int> DeviceSelectStep::source_of(cudaStream_t s) {
    std::vector<int> h(static_cast<std::size_t>(M_));
    cuda_check(cudaMemcpyAsync(h.data(), source_.get(), h.size() * sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    return h;
}

std::vector<double> DeviceSelectStep::scores(cudaStream_t s) {
    std::vector<double> h(static_cast<std::size_t>(M_) * (K_ - 1));
    cuda_check(cudaMemcpyAsync(h.data(), scores_.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    return h;
}

// ---- device re-verify --------------------------------------------------------------
namespace {

struct StreamHandle {
    cudaStream_t s = nullptr;
    StreamHandle() { cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream"); }
    ~StreamHandle() { cudaStreamDestroy(s); }
    StreamHandle(const StreamHandle&) = delete;
    StreamHandle& operator=(const StreamHandle&) = delete;
};

struct FileRange {
    std::uint64_t file_off, bytes;
    std::uint8_t* dst; // device
};

// Streams byte ranges of one file to device memory in `step`-byte pieces read by
// the I/O pool, alternating two pinned halves so the H2D of one piece overlaps
// the reads of the next. Returns after the copies complete.
void load_ranges(const fs::path& path, const std::vector<FileRange>& ranges, PinnedBuffer* stage /* [2] */, int threads,
                 std::uint64_t step, cudaStream_t s) {
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) fail(ErrorKind::MissingArtifact, "cannot open '" + path.string() + "'");
    // a file not in the page cache (e.g. written with O_DIRECT) is read with O_DIRECT
    std::uint64_t span_lo = ~0ull, span_hi = 0;
    for (const auto& r : ranges) {
        span_lo = std::min(span_lo, r.file_off);
        span_hi = std::max(span_hi, r.file_off + r.bytes);
    }
    const int dfd = span_hi > span_lo && want_direct_read(io_mode_from_env(IoMode::Auto), fd, span_lo, span_hi - span_lo)
                        ? open_direct_read(path.string())
                        : -1;
    stage[0].resize(step);
    stage[1].resize(step);
    cudaEvent_t done[2];
    cuda_check(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming), "event");
    bool used[2] = {false, false};
    const auto cleanup = [&] {
        cudaStreamSynchronize(s);
        cudaEventDestroy(done[0]);
        cudaEventDestroy(done[1]);
        ::close(fd);
        if (dfd >= 0) ::close(dfd);
    };
    try {
        int half = 0;
        std::size_t ri = 0;
        std::uint64_t at = 0; // progress inside ranges[ri]
        while (ri < ranges.size()) {
            // fill one half with up to `step` bytes drawn from consecutive ranges
            std::uint8_t* buf = stage[half].get();
            if (used[half]) cuda_check(cudaEventSynchronize(done[half]), "event");
            std::vector<ReadJob> jobs;
            std::vector<std::pair<std::uint64_t, const FileRange*>> pieces; // (bytes, range) with in-range offsets
            std::vector<std::uint64_t> starts;
            std::uint64_t fill = 0;
            while (ri < ranges.size() && fill < step) {
                const FileRange& r = ranges[ri];
                const std::uint64_t n = std::min(step - fill, r.bytes - at);
                if (n > 0) {
                    jobs.push_back({fd, buf + fill, n, r.file_off + at, dfd});
                    pieces.push_back({n, &r});
                    starts.push_back(at);
                }
                fill += n;
                at += n;
                if (at == r.bytes) {
                    ++ri;
                    at = 0;
                }
            }
            run_reads(jobs, threads, path.string());
            std::uint64_t off = 0;
            for (std::size_t i = 0; i < pieces.size(); ++i) {
                cuda_check(cudaMemcpyAsync(pieces[i].second->dst + starts[i], buf + off, pieces[i].first, cudaMemcpyHostToDevice, s),
                           "H2D");
                off += pieces[i].first;
            }
            cuda_check(cudaEventRecord(done[half], s), "event");
            used[half] = true;
            half ^= 1;
        }
        cuda_check(cudaStreamSynchronize(s), "sync");
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

void load_payload(const fs::path& path, const ContainerLayout& lay, DeviceBuffer& dst, PinnedBuffer* stage /* [2] */,
                  int threads = io_threads(), std::uint64_t step = 512ull << 20) {
    dst.resize(std::max<std::uint64_t>(16, lay.payload_bytes));
    StreamHandle sh;
    load_ranges(path, {{lay.payload_offset(), lay.payload_bytes, dst.get()}}, stage, threads, step, sh.s);
}

} // namespace

VerifyPlan verify_plan(const fs::path& dir, const CheckpointSummary& s, ContainerLayout weights,
                       std::vector<ContainerLayout> shards) {
    VerifyPlan out;
    out.weights = std::move(weights);
    out.shards = std::move(shards);
    const GroupTable table = s.optim.grouping == Grouping::Fine ? build_group_table(s.spec) : build_coarse_table(s.spec);
    std::map<int, std::vector<TensorSlice>> group_slices;
    for (const auto& g : s.optim.groups) group_slices[g.index] = group_tensor_slices(s.spec, table, g.index);
    const ContainerLayout& wl = out.weights;
    std::size_t expect_tensors = 0;
    for (const auto& m : s.manifest.modules)
        for (const auto& t : tensors_of(s.spec, m)) {
            ++expect_tensors;
            const Entry* e = wl.find(t.name);
            if (!e) fail(ErrorKind::CorruptContainer, ckpt_file(CkptFile::Weights, dir).string() + ": missing tensor '" + t.name + "'");
            if (e->dtype != Dtype::BF16 || e->shape != t.shape)
                fail(ErrorKind::Geometry, ckpt_file(CkptFile::Weights, dir).string() + ": tensor '" + t.name + "' has unexpected dtype/shape");
        }
    if (wl.entries.size() != expect_tensors)
        fail(ErrorKind::CorruptContainer, ckpt_file(CkptFile::Weights, dir).string() + ": contains tensors not in the manifest");

    // Structure of every rank file first (rank order), with the verify work of
    // each rank as offsets into its payload; then the payloads stream to the
    // device over parallel lanes (one rank file each) and the failure counters
    // are checked in rank order.
    const int N = s.optim.num_ranks;
    if (out.shards.size() != static_cast<std::size_t>(N)) fail(ErrorKind::Geometry, "shard layout count mismatch");
    auto& pairs = out.pairs;
    auto& ranges = out.ranges;
    pairs.assign(static_cast<std::size_t>(N), {});
    ranges.assign(static_cast<std::size_t>(N), {});
    for (int r = 0; r < N; ++r) {
        const fs::path sp = ckpt_file(CkptFile::Shard, dir, r);
        const ContainerLayout& sl = out.shards[static_cast<std::size_t>(r)];
        out.max_shard = std::max<std::uint64_t>(out.max_shard, sl.payload_bytes);
        auto mr = sl.metadata.find("rank");
        if (mr != sl.metadata.end() && mr->second != std::to_string(r))
            fail(ErrorKind::CorruptContainer, sp.string() + ": rank metadata mismatch");
        for (const auto& g : s.optim.groups) {
            const Entry* f[3];
            const char* names[3] = {".master", ".exp_avg", ".exp_avg_sq"};
            for (int i = 0; i < 3; ++i) {
                f[i] = sl.find(shard_key(g.index, names[i]));
                if (!f[i]) fail(ErrorKind::CorruptContainer, sp.string() + ": missing tensor '" + shard_key(g.index, names[i]) + "'");
                if (f[i]->dtype != Dtype::F32 || f[i]->shape != std::vector<std::int64_t>{g.shard_length})
                    fail(ErrorKind::Geometry,
                         sp.string() + ": tensor '" + shard_key(g.index, names[i]) + "' has unexpected dtype/shape");
            }
            // pointers below are payload offsets (shard) / weights offsets; rebased per lane
            const std::int64_t c = g.shard_length, first = static_cast<std::int64_t>(r) * c;
            const std::int64_t valid = std::clamp<std::int64_t>(g.true_length - first, 0, c);
            auto at = [](std::uint64_t off) { return reinterpret_cast<const std::uint32_t*>(off); };
            for (int i = 0; i < 3; ++i)
                if (valid < c)
                    ranges[static_cast<std::size_t>(r)].push_back(
                        {at(f[i]->begin + static_cast<std::uint64_t>(valid) * 4), static_cast<std::uint64_t>(c - valid), 0, 0});
            if (valid > 0) ranges[static_cast<std::size_t>(r)].push_back({at(f[2]->begin), static_cast<std::uint64_t>(valid), 1, 0});
            for (const auto& sl2 : group_slices.at(g.index)) {
                const std::int64_t a = std::max(first, sl2.group_offset);
                const std::int64_t b = std::min(first + valid, sl2.group_offset + sl2.decl.numel());
                if (a >= b) continue;
                // derive_weights (R/src/checkpoint.cpp:287-312) pairs only tensors of manifest
                // modules: a coarse checkpoint with a partial manifest has group slices
                // without a weights entry, and those are not checked
                const Entry* we = wl.find(sl2.decl.name);
                if (!we) continue;
                pairs[static_cast<std::size_t>(r)].push_back(
                    {reinterpret_cast<const float*>(f[0]->begin + static_cast<std::uint64_t>(a - first) * 4),
                     reinterpret_cast<const std::uint16_t*>(we->begin + static_cast<std::uint64_t>(a - sl2.group_offset) * 2),
                     static_cast<std::uint64_t>(b - a)});
            }
        }
    }

    return out;
}

void verify_rank_resident(const VerifyPlan& plan, int r, const fs::path& shard_file, DeviceBuffer& ds, DeviceBuffer& dpairs,
                          DeviceBuffer& dranges, PinnedBuffer* stage, int readers, std::uint64_t step, unsigned long long* d_err,
                          cudaStream_t st, const std::function<const std::uint8_t*()>& weights) {
    const auto& sl = plan.shards.at(static_cast<std::size_t>(r));
    load_payload(shard_file, sl, ds, stage, readers, step);
    const std::uint8_t* dw = weights(); // may block (e.g. until the weights file is in)
    auto pr = plan.pairs[static_cast<std::size_t>(r)];
    auto rg = plan.ranges[static_cast<std::size_t>(r)];
    for (auto& x : pr) {
        x.master = reinterpret_cast<const float*>(ds.get() + reinterpret_cast<std::uintptr_t>(x.master));
        x.weight = reinterpret_cast<const std::uint16_t*>(dw + reinterpret_cast<std::uintptr_t>(x.weight));
    }
    for (auto& x : rg) x.words = reinterpret_cast<const std::uint32_t*>(ds.get() + reinterpret_cast<std::uintptr_t>(x.words));
    dpairs.upload(pr.data(), pr.size() * sizeof(dev::VerifyPair), st); // on the verify stream: ordered before K6
    dranges.upload(rg.data(), rg.size() * sizeof(dev::VerifyRange), st);
    cuda_check(dev::launch_verify(dpairs.get<dev::VerifyPair>(), static_cast<std::uint32_t>(pr.size()),
                                  dranges.get<dev::VerifyRange>(), static_cast<std::uint32_t>(rg.size()), d_err + 3 * r, st),
               "verify");
    cuda_check(cudaStreamSynchronize(st), "verify");
}

void load_payload_to(const fs::path& path, const ContainerLayout& lay, DeviceBuffer& dst, PinnedBuffer* stage, int threads,
                     std::uint64_t step) {
    load_payload(path, lay, dst, stage, threads, step);
}

void verify_counters_host(const fs::path& dir, int num_ranks, const unsigned long long* err) {
    bool mismatch = false;
    for (int r = 0; r < num_ranks; ++r) {
        if (err[3 * r + 1]) fail(ErrorKind::CorruptContainer, dir.string() + ": nonzero padding in rank " + std::to_string(r));
        if (err[3 * r + 2]) fail(ErrorKind::Consistency, "exp_avg_sq contains a negative or non-finite element");
        mismatch = mismatch || err[3 * r] != 0;
    }
    if (mismatch) fail(ErrorKind::Consistency, dir.string() + ": a weight tensor disagrees with its FP32 master");
}

void verify_counters(const fs::path& dir, int num_ranks, const unsigned long long* d_err) {
    std::vector<unsigned long long> err(static_cast<std::size_t>(num_ranks) * 3);
    cuda_check(cudaMemcpy(err.data(), d_err, err.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H");
    verify_counters_host(dir, num_ranks, err.data());
}

void verify_checkpoint_dir(const std::string& dir_s, int device) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    const fs::path dir(dir_s);
    const CheckpointSummary s = read_checkpoint_summary(dir);
    const fs::path optim = dir / "optim";
    if (!fs::exists(optim)) fail(ErrorKind::MissingArtifact, "'" + optim.string() + "' does not exist");
    std::size_t files = 0;
    for ([[maybe_unused]] const auto& e : fs::directory_iterator(optim)) ++files;
    if (files != static_cast<std::size_t>(s.optim.num_ranks))
        fail(ErrorKind::Geometry, dir.string() + ": found " + std::to_string(files) + " shard files for " +
                                      std::to_string(s.optim.num_ranks) + " ranks");
    ContainerLayout wl_file = read_layout(ckpt_file(CkptFile::Weights, dir));
    std::vector<ContainerLayout> shard_files;
    for (int r = 0; r < s.optim.num_ranks; ++r) shard_files.push_back(read_layout(ckpt_file(CkptFile::Shard, dir, r)));
    const VerifyPlan plan = verify_plan(dir, s, std::move(wl_file), std::move(shard_files));
    const ContainerLayout& wl = plan.weights;
    const int N = s.optim.num_ranks;
    const std::uint64_t max_shard = plan.max_shard;
    const auto& pairs = plan.pairs;
    const auto& ranges = plan.ranges;
    const auto& shard_lay = plan.shards;
    DeviceBuffer dw, derr(static_cast<std::size_t>(N) * 3 * sizeof(unsigned long long));
    cuda_check(cudaMemset(derr.get(), 0, derr.size()), "memset");
    cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "memset"); // cudaMemset is async: done before the verify streams add to it
    const std::uint64_t budget = device_budget();
    // Resident form: the weights payload stays on the device and each lane holds one
    // whole rank payload. Streaming form (a 70B-shaped checkpoint: 160 GB of weights,
    // 120 GB per rank): each lane walks its rank payload in windows and loads, per
    // window, only the weight bytes its masters pair with (every byte read once).
    const bool resident = wl.payload_bytes + max_shard <= budget;
    std::atomic<int> next{0};
    std::exception_ptr lane_err;
    std::mutex mu;
    const auto run_lanes = [&](int lanes, const std::function<void()>& lane) {
        PhaseTimer pt("verify.shards");
        if (lanes == 1) {
            lane();
        } else {
            std::vector<std::thread> pool;
            for (int i = 0; i < lanes; ++i) pool.emplace_back(lane);
            for (auto& t : pool) t.join();
        }
    };
    const auto launch = [&](std::vector<dev::VerifyPair>& pr, std::vector<dev::VerifyRange>& rg, DeviceBuffer& dpairs,
                            DeviceBuffer& dranges, int r, cudaStream_t st) {
        dpairs.upload(pr.data(), pr.size() * sizeof(dev::VerifyPair), st);
        dranges.upload(rg.data(), rg.size() * sizeof(dev::VerifyRange), st);
        cuda_check(dev::launch_verify(dpairs.get<dev::VerifyPair>(), static_cast<std::uint32_t>(pr.size()),
                                      dranges.get<dev::VerifyRange>(), static_cast<std::uint32_t>(rg.size()),
                                      derr.get<unsigned long long>() + 3 * r, st),
                   "verify");
        cuda_check(cudaStreamSynchronize(st), "verify");
    };
    if (resident) {
        const int lanes = std::clamp<int>(static_cast<int>(std::min<std::uint64_t>((budget - wl.payload_bytes) / max_shard, 8)), 1,
                                          std::max(1, std::min(N, 8)));
        const int readers = std::max(1, io_threads() / lanes);
        const std::uint64_t step = lanes > 1 ? (16ull << 20) : (256ull << 20);
        // the weights payload loads on its own thread while the lanes load rank payloads;
        // a lane waits for it only before its first duality kernel
        dw.resize(std::max<std::uint64_t>(16, wl.payload_bytes));
        std::mutex wmu;
        std::condition_variable wcv;
        bool weights_ready = false;
        std::exception_ptr werr;
        std::thread wloader([&] {
            try {
                cuda_check(cudaSetDevice(device), "cudaSetDevice");
                PhaseTimer pt("verify.load_weights");
                PinnedBuffer stage[2];
                load_payload(ckpt_file(CkptFile::Weights, dir), wl, dw, stage, std::max(1, io_threads() / 2), step);
            } catch (...) {
                werr = std::current_exception();
            }
            std::lock_guard<std::mutex> lk(wmu);
            weights_ready = true;
            wcv.notify_all();
        });
        const auto wait_weights = [&] {
            std::unique_lock<std::mutex> lk(wmu);
            wcv.wait(lk, [&] { return weights_ready; });
            if (werr) std::rethrow_exception(werr);
        };
        run_lanes(lanes, [&] {
            try {
                cuda_check(cudaSetDevice(device), "cudaSetDevice");
                DeviceBuffer ds, dpairs, dranges;
                PinnedBuffer stage[2];
                StreamHandle ls;
                for (int r = next.fetch_add(1); r < N; r = next.fetch_add(1)) {
                    {
                        std::lock_guard<std::mutex> lk(mu);
                        if (lane_err) break;
                    }
                    verify_rank_resident(plan, r, ckpt_file(CkptFile::Shard, dir, r), ds, dpairs, dranges, stage, readers,
                                         step, derr.get<unsigned long long>(), ls.s, [&] {
                                             wait_weights();
                                             return static_cast<const std::uint8_t*>(dw.get());
                                         });
                }
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!lane_err) lane_err = std::current_exception();
            }
        });
        wloader.join();
        if (werr && !lane_err) std::rethrow_exception(werr);
    } else {
        // window W of shard bytes + up to W/2 of weight bytes per lane
        const int want = std::max(1, std::min(N, 8));
        std::uint64_t W = std::min<std::uint64_t>(256ull << 20, budget / (3 * static_cast<std::uint64_t>(want)) * 2);
        W = std::max<std::uint64_t>(4096, W & ~4095ull);
        const int lanes = std::clamp<int>(static_cast<int>(budget / (W + W / 2)), 1, want);
        const int readers = std::max(1, io_threads() / lanes);
        trace_count("verify.streaming window (MB)", static_cast<double>(W >> 20));
        run_lanes(lanes, [&] {
            try {
                cuda_check(cudaSetDevice(device), "cudaSetDevice");
                DeviceBuffer A(W), B(W / 2 + 16), dpairs, dranges;
                PinnedBuffer stage[2];
                StreamHandle ls;
                for (int r = next.fetch_add(1); r < N; r = next.fetch_add(1)) {
                    {
                        std::lock_guard<std::mutex> lk(mu);
                        if (lane_err) break;
                    }
                    // items by shard payload offset: pairs (master 4 B/elt, weight 2 B/elt) and word ranges
                    struct Item {
                        std::uint64_t soff, count, woff;
                        std::uint32_t kind; // 0 pair, 1 must-be-zero words, 2 must-be-nonnegative floats
                    };
                    std::vector<Item> items;
                    for (const auto& x : pairs[static_cast<std::size_t>(r)])
                        items.push_back({reinterpret_cast<std::uintptr_t>(x.master), x.count, reinterpret_cast<std::uintptr_t>(x.weight), 0});
                    for (const auto& x : ranges[static_cast<std::size_t>(r)])
                        items.push_back({reinterpret_cast<std::uintptr_t>(x.words), x.count, 0, 1 + x.kind});
                    std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.soff < b.soff; });
                    const ContainerLayout& sl = shard_lay[static_cast<std::size_t>(r)];
                    const fs::path sp = ckpt_file(CkptFile::Shard, dir, r), wp = ckpt_file(CkptFile::Weights, dir);
                    std::size_t first = 0;
                    for (std::uint64_t lo = 0; lo < sl.payload_bytes; lo += W) {
                        const std::uint64_t hi = std::min(sl.payload_bytes, lo + W);
                        std::vector<dev::VerifyPair> pr;
                        std::vector<dev::VerifyRange> rg;
                        std::vector<FileRange> wr;
                        std::uint64_t bpos = 0;
                        while (first < items.size() && items[first].soff + 4 * items[first].count <= lo) ++first;
                        for (std::size_t i = first; i < items.size() && items[i].soff < hi; ++i) {
                            const Item& it = items[i];
                            const std::uint64_t a = std::max(lo, it.soff), z = std::min(hi, it.soff + 4 * it.count);
                            if (a >= z) continue;
                            const std::uint64_t j0 = (a - it.soff) / 4, n = (z - a) / 4;
                            if (it.kind == 0) {
                                const std::uint64_t wo = it.woff + 2 * j0;
                                if (!wr.empty() && wr.back().file_off + wr.back().bytes == wl.payload_offset() + wo &&
                                    wr.back().dst + wr.back().bytes == B.get() + bpos) {
                                    wr.back().bytes += 2 * n;
                                } else {
                                    wr.push_back({wl.payload_offset() + wo, 2 * n, B.get() + bpos});
                                }
                                pr.push_back({reinterpret_cast<const float*>(A.get() + (a - lo)),
                                              reinterpret_cast<const std::uint16_t*>(B.get() + bpos), n});
                                bpos += 2 * n;
                            } else {
                                rg.push_back({reinterpret_cast<const std::uint32_t*>(A.get() + (a - lo)), n, it.kind - 1, 0});
                            }
                        }
                        load_ranges(sp, {{sl.payload_offset() + lo, hi - lo, A.get()}}, stage, readers, 16ull << 20, ls.s);
                        if (!wr.empty()) load_ranges(wp, wr, stage, readers, 16ull << 20, ls.s);
                        launch(pr, rg, dpairs, dranges, r, ls.s);
                    }
                }
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!lane_err) lane_err = std::current_exception();
            }
        });
    }
    if (lane_err) std::rethrow_exception(lane_err);
    verify_counters(dir, N, derr.get<unsigned long long>());
}

} // namespace tailor
