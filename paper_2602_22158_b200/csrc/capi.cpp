// The C ABI (include/tailor_b200.h) over the C++ engine. Every entry point
// catches: no exception crosses the boundary; the error kind becomes the
// return code and the message goes to tg_last_error().
#include "tailor_b200.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <exception>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fcntl.h>
#include <future>
#include <memory>
#include <string>
#include <unistd.h>

#include <json.hpp>

#include "tailor/comm.hpp"
#include "tailor/engine.hpp"
#include "tailor/errors.hpp"
#include "tailor/io.hpp"
#include "tailor/merge.hpp"
#include "tailor/trainer.hpp"

using nlohmann::json;
using namespace tailor;
namespace fs = std::filesystem;

// A layout handle either owns its SnapshotSet (tg_layout_create / _from_checkpoints)
// or views a family's (tg_family_layout; owned by the family, never destroyed by the caller).
struct tg_layout {
    SnapshotSet* set = nullptr;
    std::unique_ptr<SnapshotSet> owned;
};
struct tg_family {
    std::unique_ptr<SynthFamily> fam;
    tg_layout view;
};
struct tg_scorer {
    std::unique_ptr<ScorePlan> plan;
};
struct tg_trainer {
    std::unique_ptr<DeviceTrainer> tr;
};
struct tg_dstep {
    std::unique_ptr<DeviceSelectStep> step;
};
struct tg_comm {
    std::unique_ptr<Comm> comm;
};
struct tg_mplan {
    std::unique_ptr<DeviceMerge> dev;
    std::unique_ptr<HostMerge> host;
    std::uint64_t host_chunk = 0;
    HostMerge::Resident host_resident; // the resident map the host pipeline was built for
    const SnapshotSet* fam = nullptr;
    std::vector<int> window_k;
    std::vector<ContainerLayout> window_layout; // source container of each window
};

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

template <typename F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        g_kind = 0;
        return TG_OK;
    } catch (const TailorError& e) {
        g_err = e.what();
        g_kind = static_cast<int>(e.kind());
    } catch (const std::exception& e) {
        g_err = std::string("internal error: ") + e.what();
        g_kind = TG_E_INTERNAL;
    } catch (...) { // nothing may unwind across the C ABI
        g_err = "internal error: unknown exception";
        g_kind = TG_E_INTERNAL;
    }
    return g_kind;
}

int put_text(const std::string& s, char* out, size_t cap, size_t* needed) {
    if (needed) *needed = s.size() + 1;
    if (!out || cap < s.size() + 1) fail(ErrorKind::Geometry, "output buffer too small (need " + std::to_string(s.size() + 1) + ")");
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

ModelSpec to_spec(const tg_model_spec* s) {
    if (!s) fail(ErrorKind::Geometry, "null model spec");
    ModelSpec m;
    m.num_layers = s->num_layers;
    m.hidden_dim = s->hidden_dim;
    m.ffn_dim = s->ffn_dim;
    m.vocab_size = s->vocab_size;
    m.weight_tied = s->weight_tied != 0;
    m.seed = s->seed;
    m.validate();
    return m;
}

json recipe_json(const MergeRecipe& r) {
    json slices = json::array();
    for (const auto& s : r.slices) slices.push_back({{"source", s.source}, {"layers", s.layers}, {"targets", s.targets}});
    json aux = json::object();
    for (const auto& [k, v] : r.aux) aux[k] = v;
    return {{"base_checkpoint", r.base_checkpoint}, {"num_ranks", r.num_ranks}, {"slices", slices},
            {"aux", aux}, {"config_from", r.config_from}};
}

MergeRecipe recipe_from_json(const json& j) {
    MergeRecipe r;
    r.base_checkpoint = j.value("base_checkpoint", std::string());
    r.num_ranks = j.value("num_ranks", 0);
    if (j.contains("slices"))
        for (const auto& s : j.at("slices")) {
            RecipeSlice sl;
            sl.source = s.at("source").get<std::string>();
            sl.layers = s.at("layers").get<std::vector<int>>();
            sl.targets = s.contains("targets") ? s.at("targets").get<std::vector<int>>() : sl.layers;
            r.slices.push_back(sl);
        }
    if (j.contains("aux"))
        for (const auto& [k, v] : j.at("aux").items()) r.aux[k] = v.get<std::string>();
    r.config_from = j.value("config_from", std::string("latest"));
    return r;
}

json plan_json(const MergePlan& p) {
    json copies = json::array();
    for (const auto& c : p.group_copies)
        copies.push_back({{"source", c.source}, {"source_group", c.source_group}, {"target_group", c.target_group}});
    json assign = json::object();
    for (const auto& [t, a] : p.assignment)
        assign[module_name(t)] = {{"source", a.source}, {"source_module", module_name(a.source_module)},
                                  {"source_step", a.source_step}};
    return {{"num_ranks", p.num_ranks}, {"config_source", p.config_source}, {"sources", p.sources},
            {"group_copies", copies}, {"assignment", assign}};
}

CheckpointSummary family_summary(const SnapshotSet& f, const std::string& id) {
    const int k = f.index_of(id);
    if (k == 0) fail(ErrorKind::MissingArtifact, "checkpoint directory '" + id + "' does not exist");
    return f.summary(k, id);
}

// Packed layout of one snapshot's rank-r master fields: 16-B aligned, in
// score_fields order; `stride` rounds the total to 256 B (the slot size).
std::uint64_t packed_stride(const std::vector<ScoreField>& fields) {
    std::uint64_t total = 0;
    for (const auto& f : fields) total = (total + static_cast<std::uint64_t>(f.chunk) * 4 + 15) & ~15ull;
    return std::max<std::uint64_t>(256, (total + 255) & ~255ull);
}

// Streams one snapshot's rank-r master fields into `dst` (packed layout) through
// two 16 MB pinned halves: the pread of one half overlaps the H2D of the other on
// the lane's stream. `offs` receives the field offsets inside `dst`.
struct PackedLoader {
    PinnedBuffer stage;
    cudaStream_t st = nullptr;
    cudaEvent_t half_done[2]{};
    bool used[2] = {false, false};
    int half = 0, threads = 1;
    double read_ms = 0.0, load_ms = 0.0;
    std::uint64_t direct_bytes = 0;
    static constexpr std::uint64_t kHalf = 16ull << 20;
    struct LoadedEntry {
        std::uint64_t begin, end; // payload-relative master entry in the file
        std::uint64_t packed;     // its offset in the packed destination
    };
    std::vector<LoadedEntry> last_entries; // of the last load()

    ReadPool pool;

    PackedLoader(cudaStream_t s, int reader_threads) : st(s), threads(reader_threads), pool(std::max(1, reader_threads)) {
        for (auto& e : half_done) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        stage.resize(2 * kHalf);
    }
    ~PackedLoader() {
        if (st) cudaStreamSynchronize(st);
        for (auto& e : half_done) cudaEventDestroy(e);
    }
    PackedLoader(const PackedLoader&) = delete;
    PackedLoader& operator=(const PackedLoader&) = delete;

    void load(const fs::path& p, const std::vector<ScoreField>& fields, std::uint8_t* dst, std::vector<std::uint64_t>& offs) {
        const double t0 = clock_ms();
        const ContainerLayout lay = read_layout(p);
        std::uint64_t total = 0;
        std::vector<std::pair<const Entry*, std::uint64_t>> where;
        offs.clear();
        for (const auto& f : fields) {
            const Entry* e = lay.find(shard_key(f.group, ".master"));
            if (!e) fail(ErrorKind::MissingModules, p.string() + ": scoring needs every module; missing '" + shard_key(f.group, ".master") + "'");
            if (e->dtype != Dtype::F32 || e->shape != std::vector<std::int64_t>{f.chunk})
                fail(ErrorKind::Geometry, p.string() + ": master '" + e->name + "' has unexpected dtype/shape");
            where.push_back({e, total});
            offs.push_back(total);
            total = (total + e->bytes() + 15) & ~15ull;
        }
        last_entries.clear();
        for (const auto& [e, at] : where) last_entries.push_back({e->begin, e->end, at});
        const int fd = ::open(p.c_str(), O_RDONLY);
        if (fd < 0) fail(ErrorKind::MissingArtifact, "cannot open '" + p.string() + "'");
        // snapshots not in the page cache are read with O_DIRECT (tailor/io.hpp; TAILOR_IO overrides)
        const int dfd = want_direct_read(io_mode_from_env(IoMode::Auto), fd, lay.payload_offset(), lay.payload_bytes)
                            ? open_direct_read(p.string())
                            : -1;
        // half h uses buffer (half + h) & 1; its reads are queued one half ahead on the
        // reader pool (after the buffer's previous H2D), so the pieces of the next half are
        // in flight while this half's last ones finish
        const std::uint64_t nh = (total + kHalf - 1) / kHalf;
        const auto queue_half = [&](std::uint64_t h) {
            const int b = static_cast<int>((static_cast<std::uint64_t>(half) + h) & 1);
            if (used[b]) cuda_check(cudaEventSynchronize(half_done[b]), "event");
            const std::uint64_t lo = h * kHalf, hi = std::min(total, lo + kHalf);
            std::uint8_t* buf = stage.get() + static_cast<std::uint64_t>(b) * kHalf;
            std::vector<ReadJob> jobs;
            for (const auto& [e, at] : where) {
                const std::uint64_t a = std::max(lo, at), z = std::min(hi, at + e->bytes());
                if (a < z) jobs.push_back({fd, buf + (a - lo), z - a, lay.payload_offset() + e->begin + (a - at), dfd});
            }
            return pool.submit(jobs, p.string());
        };
        try {
            const bool ahead = read_lookahead();
            std::uint64_t ticket = nh ? queue_half(0) : 0;
            for (std::uint64_t h = 0; h < nh; ++h) {
                const std::uint64_t next = ahead && h + 1 < nh ? queue_half(h + 1) : 0;
                const double r0 = clock_ms();
                pool.wait(ticket);
                read_ms += clock_ms() - r0;
                const int b = static_cast<int>((static_cast<std::uint64_t>(half) + h) & 1);
                const std::uint64_t lo = h * kHalf, hi = std::min(total, lo + kHalf);
                cuda_check(cudaMemcpyAsync(dst + lo, stage.get() + static_cast<std::uint64_t>(b) * kHalf, hi - lo,
                                           cudaMemcpyHostToDevice, st),
                           "H2D");
                cuda_check(cudaEventRecord(half_done[b], st), "event");
                used[b] = true;
                ticket = ahead ? next : (h + 1 < nh ? queue_half(h + 1) : 0);
            }
            half = static_cast<int>((static_cast<std::uint64_t>(half) + nh) & 1);
        } catch (...) {
            pool.drain();
            cudaStreamSynchronize(st);
            ::close(fd);
            if (dfd >= 0) ::close(dfd);
            throw;
        }
        ::close(fd);
        if (dfd >= 0) ::close(dfd);
        if (dfd >= 0) direct_bytes += total;
        load_ms += clock_ms() - t0;
    }
};

// Device scores over snapshot directories: per rank, packed masters -> K3/K4;
// ranks combined in rank order on the host (FP64, fixed order).
// keep (optional): when every snapshot of every rank fits the budget of a single-device
// run, the packed masters stay in (*keep_mem)[rank] afterwards (one pooled buffer per rank)
// and *keep maps each (snapshot dir, rank) master entry to its device copy
// (tg_select_merge hands them to the merge).
void score_dirs(const std::vector<std::string>& dirs, const std::vector<int>& devices, std::vector<std::vector<double>>& sd,
                std::vector<std::vector<double>>& sr, std::vector<CheckpointSummary>& sums, ResidentSources* keep = nullptr,
                std::vector<DeviceBuffer>* keep_mem = nullptr) {
    if (dirs.size() < 2) fail(ErrorKind::Recipe, "scoring needs at least two snapshots");
    // the CUDA context comes up while the sidecars are parsed (a fresh process pays
    // hundreds of ms for it)
    auto cuda_ready = std::async(std::launch::async, [&devices] {
        for (int d : devices) {
            cuda_check(cudaSetDevice(d), "cudaSetDevice");
            cuda_check(cudaFree(nullptr), "cuda init");
        }
    });
    sums.clear();
    try {
        for (const auto& d : dirs) sums.push_back(read_checkpoint_summary(d));
    } catch (...) {
        cuda_ready.wait();
        throw;
    }
    cuda_ready.get();
    cuda_check(cudaSetDevice(devices.front()), "cudaSetDevice");
    const ModelSpec& spec = sums.front().spec;
    const int N = sums.front().optim.num_ranks;
    for (const auto& s : sums) {
        if (!s.spec.same_geometry(spec)) fail(ErrorKind::Geometry, "snapshots disagree on model geometry");
        if (s.optim.num_ranks != N) fail(ErrorKind::Geometry, "snapshots disagree on the rank count");
        if (s.optim.grouping != Grouping::Fine) fail(ErrorKind::Geometry, "scoring needs the fine grouping");
    }
    const ModelLayout model(spec);
    const int K = static_cast<int>(dirs.size()), M = model.module_count();
    sd.assign(static_cast<std::size_t>(K - 1), std::vector<double>(static_cast<std::size_t>(M), 0.0));
    sr = sd;
    // Ranks are independent: lanes (threads with their own buffers, spread round-robin
    // over the devices) score one rank each; the per-rank partials are summed in rank
    // order afterwards, so the result depends on neither the lane count nor the devices.
    // A lane holds all K packed snapshots of its rank when they fit the device budget;
    // otherwise it rolls through `slots` device slots (>= 2) in windows of up to
    // min(slots, 16) consecutive snapshots that overlap by one (snapshot k lives in slot
    // k % slots; every pair is scored once, inside one window), e.g. a 70B-shaped rank
    // partition (4 x 40 GB of masters) in pairs, or a 35-snapshot sweep.
    const auto fields = score_fields(model, N);
    const std::uint64_t stride = packed_stride(fields);
    std::uint64_t budget = ~0ull;
    for (int d : devices) {
        cuda_check(cudaSetDevice(d), "cudaSetDevice");
        budget = std::min(budget, device_budget());
    }
    cuda_check(cudaSetDevice(devices.front()), "cudaSetDevice");
    const bool all_resident = stride * static_cast<std::uint64_t>(K) <= budget;
    const int slots = all_resident ? K
                                   : static_cast<int>(std::clamp<std::uint64_t>(budget / stride, 2, static_cast<std::uint64_t>(dev::kMaxSnapshots)));
    const std::uint64_t all_bytes = stride * static_cast<std::uint64_t>(K) * static_cast<std::uint64_t>(N);
    const bool keep_all = keep && keep_mem && devices.size() == 1 && all_resident && all_bytes <= budget;
    if (keep_all) keep_mem->resize(static_cast<std::size_t>(N)); // per rank: K slots, kept after scoring
    const std::uint64_t per_lane = keep_all ? stride : stride * static_cast<std::uint64_t>(slots);
    if (per_lane > budget && !std::getenv("TAILOR_DEVICE_BUDGET"))
        fail(ErrorKind::Device, "scoring needs " + std::to_string(per_lane) + " B of device memory for two snapshots of one rank; " +
                                    std::to_string(budget) + " B available");
    const int nd = static_cast<int>(devices.size());
    const int per_dev = std::clamp<int>(static_cast<int>(std::min<std::uint64_t>(budget / per_lane, 8)), 1, 8);
    int lanes = std::clamp<int>(per_dev * nd, 1, N);
    if (const char* v = std::getenv("TAILOR_SCORE_LANES"); v && std::atoi(v) > 0) // diagnostics (racecheck: one lane)
        lanes = std::min(lanes, std::atoi(v));
    const int readers = std::max(1, io_threads() / lanes);
    trace_count(all_resident ? "score.lanes" : "score.lanes (rolling windows)", lanes);
    trace_count("score.slots", slots);
    const std::size_t nres = static_cast<std::size_t>(K - 1) * M * 2;
    std::vector<std::vector<double>> res(static_cast<std::size_t>(N), std::vector<double>(nres));
    std::atomic<int> next{0};
    std::exception_ptr lane_err;
    std::mutex mu;
    const auto lane = [&](int li) {
        try {
            cuda_check(cudaSetDevice(devices[static_cast<std::size_t>(li % nd)]), "cudaSetDevice");
            cudaStream_t st = nullptr;
            cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
            std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> own(st, &cudaStreamDestroy);
            DeviceBuffer dout(nres * sizeof(double)), arena(keep_all ? 0 : per_lane);
            PackedLoader loader(st, readers);
            std::map<int, std::unique_ptr<ScorePlan>> plans; // by window length (offsets are rank-independent)
            for (int r = next.fetch_add(1); r < N; r = next.fetch_add(1)) {
                {
                    std::lock_guard<std::mutex> lk(mu);
                    if (lane_err) break;
                }
                PhaseTimer pt("score.rank");
                loader.read_ms = loader.load_ms = 0.0;
                const double t0 = clock_ms();
                std::vector<std::uint64_t> offs;
                if (keep_all) (*keep_mem)[static_cast<std::size_t>(r)].resize(stride * static_cast<std::uint64_t>(K));
                const auto slot_of = [&](int k) {
                    return keep_all ? (*keep_mem)[static_cast<std::size_t>(r)].get() + static_cast<std::uint64_t>(k) * stride
                                    : arena.get() + static_cast<std::uint64_t>(k % slots) * stride;
                };
                const auto load = [&](int k) {
                    loader.load(ckpt_file(CkptFile::Shard, dirs[static_cast<std::size_t>(k)], r), fields, slot_of(k), offs);
                    if (keep_all) {
                        std::vector<ResidentRange> rr;
                        for (const auto& e : loader.last_entries) rr.push_back({e.begin, e.end, slot_of(k) + e.packed});
                        std::sort(rr.begin(), rr.end(), [](const ResidentRange& a, const ResidentRange& b) { return a.lo < b.lo; });
                        std::lock_guard<std::mutex> lk(mu);
                        keep->ranges[{fs::path(dirs[static_cast<std::size_t>(k)]).lexically_normal().string(), r}] = std::move(rr);
                    }
                };
                const auto score = [&](int k0, int k1) { // snapshots k0..k1 resident, pairs k0..k1-1
                    const int n = k1 - k0 + 1;
                    auto& plan = plans[n];
                    if (!plan) plan = std::make_unique<ScorePlan>(model, N, std::vector<std::vector<std::uint64_t>>(static_cast<std::size_t>(n), offs));
                    std::vector<const std::uint8_t*> bases;
                    for (int k = k0; k <= k1; ++k) bases.push_back(slot_of(k));
                    plan->run(bases.data(), dout.get<double>() + static_cast<std::size_t>(k0) * M * 2, st);
                    if (sync_check()) cuda_check(cudaStreamSynchronize(st), "score (TAILOR_SYNC_CHECK)");
                };
                if (all_resident) {
                    for (int k = 0; k < K; ++k) load(k);
                    score(0, K - 1); // windows of <= 16 inside ScorePlan
                } else {
                    // the slot a load overwrites was last read by a window scored earlier on
                    // this stream, so stream order keeps the reuse safe
                    const int win = std::min(slots, static_cast<int>(dev::kMaxSnapshots));
                    load(0);
                    for (int k0 = 0; k0 < K - 1;) {
                        const int k1 = std::min(K - 1, k0 + win - 1);
                        for (int k = k0 + 1; k <= k1; ++k) load(k);
                        score(k0, k1);
                        k0 = k1;
                    }
                }
                cuda_check(cudaMemcpyAsync(res[static_cast<std::size_t>(r)].data(), dout.get(), nres * sizeof(double),
                                           cudaMemcpyDeviceToHost, st),
                           "D2H");
                cuda_check(cudaStreamSynchronize(st), "sync");
                if (trace_enabled())
                    std::fprintf(stderr, "[tailor] score.rank %d: load %.1f (read %.1f) total %.1f ms\n", r, loader.load_ms,
                                 loader.read_ms, clock_ms() - t0);
            }
        } catch (...) {
            std::lock_guard<std::mutex> lk(mu);
            if (!lane_err) lane_err = std::current_exception();
        }
    };
    if (lanes == 1) {
        lane(0);
    } else {
        std::vector<std::thread> pool;
        for (int i = 0; i < lanes; ++i) pool.emplace_back(lane, i);
        for (auto& t : pool) t.join();
    }
    cuda_check(cudaSetDevice(devices.front()), "cudaSetDevice");
    if (lane_err) std::rethrow_exception(lane_err);
    if (keep_all) keep->device = devices.front();
    for (int r = 0; r < N; ++r) {
        const auto& h = res[static_cast<std::size_t>(r)];
        for (int p = 0; p < K - 1; ++p)
            for (int m = 0; m < M; ++m) {
                sd[static_cast<std::size_t>(p)][static_cast<std::size_t>(m)] += h[(static_cast<std::size_t>(p) * M + m) * 2];
                sr[static_cast<std::size_t>(p)][static_cast<std::size_t>(m)] += h[(static_cast<std::size_t>(p) * M + m) * 2 + 1];
            }
    }
}

MergeOptions merge_options(const tg_merge_options* o) {
    MergeOptions opt;
    if (!o) return opt;
    opt.workers = o->workers;
    opt.uncached = o->uncached != 0;
    opt.device = o->device;
    opt.verify = o->skip_verify == 0;
    if (o->io_mode < TG_IO_AUTO || o->io_mode > TG_IO_DIRECT_RW)
        fail(ErrorKind::Recipe, "tg_merge_options: unknown io_mode " + std::to_string(o->io_mode));
    opt.io = static_cast<IoMode>(o->io_mode);
    if (o->num_devices > 0) {
        if (!o->devices) fail(ErrorKind::Recipe, "tg_merge_options: num_devices > 0 with a null device list");
        opt.devices.assign(o->devices, o->devices + o->num_devices);
    }
    return opt;
}

void put_stats(const MergeStats& s, tg_merge_stats* st) {
    st->shard_files_read = s.shard_files_read;
    st->weight_files_read = s.weight_files_read;
    st->wall_ms = s.wall_ms;
    st->device_ms = s.device_ms;
    st->bytes_moved = s.bytes_moved;
    st->direct_read_bytes = s.direct_read_bytes;
    st->direct_write_bytes = s.direct_write_bytes;
    st->resident_bytes = s.resident_bytes;
}

// A null handle is a caller error reported through tg_last_error, never a crash.
template <typename T>
T& need(T* h, const char* fn) {
    if (!h) fail(ErrorKind::Geometry, std::string(fn) + ": null handle");
    return *h;
}

std::vector<std::string> dir_list(const char* const* dirs, int32_t n) {
    if (n < 0 || (n > 0 && !dirs)) fail(ErrorKind::Recipe, "snapshot directory list is null or has a negative length");
    std::vector<std::string> ds;
    for (int32_t i = 0; i < n; ++i) {
        if (!dirs[i]) fail(ErrorKind::Recipe, "snapshot directory " + std::to_string(i) + " is null");
        ds.emplace_back(dirs[i]);
    }
    return ds;
}

std::vector<int> device_list(const int32_t* devices, int32_t n) {
    if (n <= 0 || !devices) return {0};
    return std::vector<int>(devices, devices + n);
}

} // namespace

extern "C" {

const char* tg_last_error(void) { return g_err.c_str(); }
int tg_last_error_kind(void) { return g_kind; }
const char* tg_version(void) { return "tailor-b200 0.1 (sm_100a)"; }
int tg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int tg_parse_recipe(const char* yaml, char* out, size_t cap, size_t* needed) {
    return guard([&] { put_text(recipe_json(parse_recipe(yaml ? yaml : "")).dump(), out, cap, needed); });
}

int tg_recipe_to_yaml(const char* rj, char* out, size_t cap, size_t* needed) {
    return guard([&] { put_text(recipe_to_yaml(recipe_from_json(json::parse(rj ? rj : "{}"))), out, cap, needed); });
}

int tg_resolve_plan(const char* yaml, char* out, size_t cap, size_t* needed) {
    return guard([&] { put_text(plan_json(resolve_plan(parse_recipe(yaml ? yaml : ""))).dump(), out, cap, needed); });
}

int tg_execute_merge(const char* yaml, const char* out_dir, const tg_merge_options* o, tg_merge_stats* st) {
    return guard([&] {
        const MergePlan plan = resolve_plan(parse_recipe(yaml ? yaml : ""));
        const MergeOptions opt = merge_options(o);
        const MergeStats s = execute_merge(plan, out_dir ? out_dir : "", opt);
        if (st) put_stats(s, st);
    });
}

int tg_recipe_from_manifests(const char* run_dir, int64_t failure_step, char* out, size_t cap, size_t* needed) {
    return guard([&] { put_text(recipe_to_yaml(recipe_from_manifests(run_dir ? run_dir : "", failure_step)), out, cap, needed); });
}

int tg_regroup(const char* src_dir, const char* out_dir, int32_t to_fine, const tg_merge_options* o, tg_merge_stats* st) {
    return guard([&] {
        MergeOptions opt = merge_options(o);
        opt.uncached = false;
        const MergeStats s = execute_regroup(src_dir ? src_dir : "", out_dir ? out_dir : "",
                                             to_fine ? Grouping::Fine : Grouping::Coarse, opt);
        if (st) put_stats(s, st);
    });
}

int tg_train(const tg_model_spec* spec, const tg_train_config* c, const char* out_dir, int32_t* written) {
    return guard([&] {
        if (!c) fail(ErrorKind::Recipe, "null train config");
        DeviceTrainConfig cfg;
        cfg.spec = to_spec(spec);
        cfg.total_steps = c->total_steps;
        cfg.num_ranks = c->num_ranks;
        cfg.strategy.interval = c->interval;
        cfg.strategy.head_count = c->head_count;
        cfg.strategy.tail_count = c->tail_count;
        cfg.strategy.sparse_multiple = c->sparse_multiple;
        switch (c->strategy) {
            case 0: cfg.strategy.kind = StrategyKind::Full; break;
            case 1: cfg.strategy.kind = StrategyKind::Parity; break;
            case 2: cfg.strategy.kind = StrategyKind::Filter; break;
            case 3: // magnitude: saved on the full schedule (readable by reference tools), label "magnitude"
                cfg.strategy.kind = StrategyKind::Full;
                cfg.magnitude = true;
                break;
            default: fail(ErrorKind::Recipe, "unknown strategy code " + std::to_string(c->strategy));
        }
        cfg.hyper.lr = c->lr;
        cfg.hyper.weight_decay = c->weight_decay;
        cfg.rho = c->rho;
        cfg.device = c->device;
        const auto dirs = device_train(cfg, out_dir ? out_dir : "");
        if (written) *written = static_cast<int32_t>(dirs.size());
    });
}

tg_trainer* tg_trainer_create(const tg_model_spec* spec, int32_t num_ranks, int32_t r0, int32_t r1, double lr, double wd,
                              int32_t device) {
    tg_trainer* out = nullptr;
    guard([&] {
        AdamHyperparams h;
        h.lr = lr;
        h.weight_decay = wd;
        out = new tg_trainer{std::make_unique<DeviceTrainer>(to_spec(spec), num_ranks, h, device, r0, r1)};
    });
    return out;
}

void tg_trainer_destroy(tg_trainer* t) { delete t; }
uint64_t tg_trainer_elements(const tg_trainer* t) { return t ? t->tr->elements() : 0; }

int tg_resume(const char* checkpoint_dir, int64_t additional_steps, const char* out_dir, int32_t device, int32_t* written) {
    return guard([&] {
        const auto dirs = device_resume(checkpoint_dir ? checkpoint_dir : "", additional_steps, out_dir ? out_dir : "", device);
        if (written) *written = static_cast<int32_t>(dirs.size());
    });
}

int tg_trainer_step(tg_trainer* t, int64_t step, double* gn, double* un) {
    return guard([&] {
        const auto [g, u] = need(t, "tg_trainer_step").tr->step(step);
        if (gn) *gn = g;
        if (un) *un = u;
    });
}

int tg_trainer_partition(tg_trainer* t, int32_t rank, void** d_ptr, uint64_t* bytes) {
    return guard([&] {
        const auto [p, n] = need(t, "tg_trainer_partition").tr->partition(rank);
        if (d_ptr) *d_ptr = p;
        if (bytes) *bytes = n;
    });
}

int tg_verify_checkpoint(const char* dir, int32_t device) {
    return guard([&] { verify_checkpoint_dir(dir ? dir : "", device); });
}

int tg_score_snapshots(const char* const* dirs, int32_t n, const int32_t* devices, int32_t num_devices, double* sums,
                       double* scores, int32_t* nm) {
    return guard([&] {
        std::vector<std::string> ds = dir_list(dirs, n);
        std::vector<std::vector<double>> sd, sr;
        std::vector<CheckpointSummary> summ;
        score_dirs(ds, device_list(devices, num_devices), sd, sr, summ);
        const int M = static_cast<int>(sd.front().size());
        if (nm) *nm = M;
        for (std::size_t p = 0; p < sd.size(); ++p)
            for (int m = 0; m < M; ++m) {
                if (sums) {
                    sums[(p * M + m) * 2] = sd[p][static_cast<std::size_t>(m)];
                    sums[(p * M + m) * 2 + 1] = sr[p][static_cast<std::size_t>(m)];
                }
                if (scores) scores[p * M + m] = magnitude_score(sd[p][static_cast<std::size_t>(m)], sr[p][static_cast<std::size_t>(m)]);
            }
    });
}

int tg_select_recipe(const char* const* dirs, int32_t n, double rho, const int32_t* devices, int32_t num_devices, char* out, size_t cap,
                     size_t* needed, int32_t* source_of, double* min_gap) {
    return guard([&] {
        std::vector<std::string> ds = dir_list(dirs, n);
        std::vector<std::vector<double>> sd, sr;
        std::vector<CheckpointSummary> summ;
        score_dirs(ds, device_list(devices, num_devices), sd, sr, summ);
        std::vector<std::vector<double>> sc = sd;
        for (std::size_t p = 0; p < sd.size(); ++p)
            for (std::size_t m = 0; m < sd[p].size(); ++m) sc[p][m] = magnitude_score(sd[p][m], sr[p][m]);
        const Selection sel = select_by_magnitude(sc, static_cast<int>(sd.front().size()), rho);
        if (source_of)
            for (std::size_t m = 0; m < sel.source_of.size(); ++m) source_of[m] = sel.source_of[m];
        if (min_gap) *min_gap = sel.min_boundary_gap;
        put_text(recipe_to_yaml(recipe_from_selection(summ, sel)), out, cap, needed);
    });
}

int tg_select_merge(const char* const* dirs, int32_t n, double rho, const char* out_dir, const tg_merge_options* o,
                    tg_merge_stats* st, char* out, size_t cap, size_t* needed, int32_t* source_of, double* min_gap) {
    return guard([&] {
        const MergeOptions opt = merge_options(o);
        const fs::path dst = out_dir ? out_dir : "";
        std::error_code ec;
        if (fs::exists(dst) && !fs::is_empty(dst, ec)) // fail before any device work, as execute_merge would
            fail(ErrorKind::Storage, "refusing to write into non-empty directory '" + dst.string() + "'");
        std::vector<std::string> ds = dir_list(dirs, n);
        std::vector<std::vector<double>> sd, sr;
        std::vector<CheckpointSummary> summ;
        ResidentSources keep;
        std::vector<DeviceBuffer> keep_mem;
        score_dirs(ds, lane_devices(opt), sd, sr, summ, &keep, &keep_mem);
        std::vector<std::vector<double>> sc = sd;
        for (std::size_t p = 0; p < sd.size(); ++p)
            for (std::size_t m = 0; m < sd[p].size(); ++m) sc[p][m] = magnitude_score(sd[p][m], sr[p][m]);
        const Selection sel = select_by_magnitude(sc, static_cast<int>(sd.front().size()), rho);
        if (source_of)
            for (std::size_t m = 0; m < sel.source_of.size(); ++m) source_of[m] = sel.source_of[m];
        if (min_gap) *min_gap = sel.min_boundary_gap;
        const std::string yaml = recipe_to_yaml(recipe_from_selection(summ, sel));
        if (needed) *needed = yaml.size() + 1; // the merge runs whether or not the recipe fits yaml_out
        if (out && cap >= yaml.size() + 1) std::memcpy(out, yaml.c_str(), yaml.size() + 1);
        const MergePlan plan = resolve_plan(parse_recipe(yaml));
        const MergeStats s = execute_merge(plan, dst, opt, keep.ranges.empty() ? nullptr : &keep);
        if (st) put_stats(s, st);
    });
}

int tg_parse_config(const char* text, tg_model_spec* out) {
    return guard([&] {
        const ModelSpec s = sidecar_value<ModelSpec>(text ? text : "", "config");
        if (out) *out = tg_model_spec{s.num_layers, s.hidden_dim, s.ffn_dim, s.vocab_size, s.weight_tied ? 1 : 0, 0, s.seed};
    });
}

int tg_layer_map(const tg_model_spec* spec, int32_t num_ranks, char* out, size_t cap, size_t* needed) {
    return guard([&] {
        const ModelLayout model(to_spec(spec));
        const ShardGeometry geom{num_ranks};
        json mods = json::array();
        for (int m = 0; m < model.module_count(); ++m) {
            json ts = json::array();
            for (const auto& t : tensors_of(model.spec(), model.modules()[static_cast<std::size_t>(m)]))
                ts.push_back({{"name", t.name}, {"shape", t.shape}, {"decay", t.decay == DecayClass::Decay ? "decay" : "no_decay"}});
            mods.push_back({{"name", module_name(model.modules()[static_cast<std::size_t>(m)])},
                            {"model_offset", model.module_offset(m)},
                            {"tensors", ts},
                            {"groups", group_indices_for(model.table(), model.modules()[static_cast<std::size_t>(m)])}});
        }
        json groups = json::array();
        for (const auto& g : model.table().groups) {
            json sl = json::array();
            for (const auto& s : model.slices(g.index))
                sl.push_back({{"name", s.decl.name}, {"group_offset", s.group_offset}, {"model_offset", s.model_offset}});
            groups.push_back({{"index", g.index}, {"owner", module_name(*g.owner)},
                              {"decay", g.decay == DecayClass::Decay ? "decay" : "no_decay"},
                              {"true_length", g.element_count}, {"padded_length", geom.padded_length(g.element_count)},
                              {"shard_length", geom.shard_length(g.element_count)}, {"slices", sl}});
        }
        put_text(json{{"modules", mods}, {"groups", groups}, {"parameters", model.parameter_count()}}.dump(), out, cap, needed);
    });
}

int tg_gather(const tg_gather_seg* d_segs, uint32_t nseg, uint8_t* d_dst, uint64_t dst_bytes, int32_t variant,
              int32_t bulk_ok, void* stream) {
    return guard([&] {
        cuda_check(dev::launch_gather(reinterpret_cast<const dev::GatherSeg*>(d_segs), nseg, d_dst, dst_bytes, variant,
                                      bulk_ok != 0, static_cast<cudaStream_t>(stream)),
                   "tg_gather");
    });
}

int tg_read_probe(const void* d_src, uint64_t bytes, uint32_t* d_sink, void* stream) {
    return guard([&] {
        cuda_check(dev::launch_read_probe(static_cast<const std::uint8_t*>(d_src), bytes, d_sink, static_cast<cudaStream_t>(stream)),
                   "tg_read_probe");
    });
}

int tg_score_partials(const tg_score_tile* d_tiles, uint32_t ntiles, const float* const* d_field_base, uint32_t nfields,
                      int32_t K, int32_t vec_ok, double* d_tile_partials, void* stream) {
    return guard([&] {
        cuda_check(dev::launch_score_partials(reinterpret_cast<const dev::ScoreTile*>(d_tiles), ntiles, d_field_base, nfields,
                                              K, vec_ok != 0, d_tile_partials, static_cast<cudaStream_t>(stream)),
                   "tg_score_partials");
    });
}

int tg_score_combine(const double* d_tile_partials, const uint32_t* d_begin, int32_t M, int32_t K, double* d_out,
                     void* stream) {
    return guard([&] {
        cuda_check(dev::launch_score_combine(d_tile_partials, d_begin, M, K, d_out, static_cast<cudaStream_t>(stream)),
                   "tg_score_combine");
    });
}

tg_family* tg_family_create(const tg_model_spec* spec, int32_t num_ranks, int32_t snapshots, int64_t interval) {
    tg_family* out = nullptr;
    guard([&] {
        out = new tg_family{std::make_unique<SynthFamily>(to_spec(spec), num_ranks, snapshots, interval), {}};
        out->view.set = out->fam.get();
    });
    return out;
}

void tg_family_destroy(tg_family* f) { delete f; }

tg_layout* tg_family_layout(tg_family* f) { return f ? &f->view : nullptr; }

tg_layout* tg_layout_create(const tg_model_spec* spec, int32_t num_ranks, int32_t snapshots, int64_t interval) {
    tg_layout* out = nullptr;
    guard([&] {
        auto set = std::make_unique<SnapshotSet>(to_spec(spec), num_ranks, snapshots, interval);
        out = new tg_layout{set.get(), std::move(set)};
    });
    return out;
}

tg_layout* tg_layout_from_checkpoints(const char* const* dirs, int32_t n) {
    tg_layout* out = nullptr;
    guard([&] {
        if (!dirs || n < 1) fail(ErrorKind::Recipe, "no checkpoint directories");
        auto set = SnapshotSet::from_checkpoints(dir_list(dirs, n));
        out = new tg_layout{set.get(), std::move(set)};
    });
    return out;
}

void tg_layout_destroy(tg_layout* l) {
    if (l && l->owned) delete l; // a family's view belongs to the family
}

int tg_layout_set_partial(tg_layout* l, int32_t k, const char* csv) {
    return guard([&] {
        std::vector<ModuleId> mods;
        std::string cur;
        for (const char* c = csv; c && *c; ++c) {
            if (*c == ',') {
                if (!cur.empty()) mods.push_back(parse_module_name(cur));
                cur.clear();
            } else {
                cur.push_back(*c);
            }
        }
        if (!cur.empty()) mods.push_back(parse_module_name(cur));
        need(l, "tg_layout_set_partial").set->set_partial(k, mods);
    });
}

int tg_layout_set_id(tg_layout* l, int32_t k, const char* id) {
    return guard([&] {
        if (k < 1 || k > need(l, "tg_layout_set_id").set->snapshots()) fail(ErrorKind::Geometry, "snapshot index out of range");
        l->set->set_id(k, id ? id : "");
    });
}

int32_t tg_layout_num_modules(const tg_layout* l) { return l ? l->set->model().module_count() : 0; }
int32_t tg_layout_num_ranks(const tg_layout* l) { return l ? l->set->num_ranks() : 0; }
int32_t tg_layout_snapshots(const tg_layout* l) { return l ? l->set->snapshots() : 0; }

uint64_t tg_layout_shard_bytes(const tg_layout* l, int32_t k, int32_t rank) {
    uint64_t n = 0;
    guard([&] { n = need(l, "tg_layout_shard_bytes").set->layout(k).shards.at(static_cast<std::size_t>(rank)).payload_bytes; });
    return n;
}

uint64_t tg_layout_weights_bytes(const tg_layout* l, int32_t k) {
    uint64_t n = 0;
    guard([&] { n = need(l, "tg_layout_weights_bytes").set->layout(k).weights.payload_bytes; });
    return n;
}

uint64_t tg_layout_packed_master_bytes(const tg_layout* l, int32_t rank) {
    uint64_t n = 0;
    guard([&] { n = need(l, "tg_layout_packed_master_bytes").set->packed_master_bytes(rank); });
    return n;
}

uint64_t tg_layout_parameter_count(const tg_layout* l) { return l ? static_cast<uint64_t>(l->set->model().parameter_count()) : 0; }

int tg_family_gen_shard(tg_family* f, int32_t rank, int32_t k0, int32_t k1, uint8_t* const* outs, void* stream) {
    return guard([&] { need(f, "tg_family_gen_shard").fam->gen_shard(rank, k0, k1, outs, static_cast<cudaStream_t>(stream)); });
}

int tg_family_gen_weights(tg_family* f, int32_t k0, int32_t k1, uint64_t lo, uint64_t hi, uint8_t* const* outs,
                          void* stream) {
    return guard([&] { need(f, "tg_family_gen_weights").fam->gen_weights(k0, k1, lo, hi, outs, static_cast<cudaStream_t>(stream)); });
}

int tg_family_gen_masters(tg_family* f, int32_t rank, int32_t k0, int32_t k1, uint8_t* const* outs, void* stream) {
    return guard([&] { need(f, "tg_family_gen_masters").fam->gen_masters_packed(rank, k0, k1, outs, static_cast<cudaStream_t>(stream)); });
}

int tg_family_gen_shard_range(tg_family* f, int32_t rank, int32_t k, uint64_t lo, uint64_t hi, uint8_t* out, void* stream) {
    return guard([&] { need(f, "tg_family_gen_shard_range").fam->gen_shard_range(rank, k, lo, hi, out, static_cast<cudaStream_t>(stream)); });
}

int tg_family_write_dir(tg_family* f, int32_t k, const char* dir) {
    return guard([&] { need(f, "tg_family_write_dir").fam->write_dir(k, dir ? dir : ""); });
}

int tg_layout_select(const tg_layout* l, const double* parts, int32_t nranks, double rho, char* out, size_t cap,
                     size_t* needed, int32_t* source_of, double* scores, double* min_gap) {
    return guard([&] {
        const SnapshotSet& fam = *need(l, "tg_layout_select").set;
        const int K = fam.snapshots(), M = fam.model().module_count();
        if (nranks < 1 || !parts) fail(ErrorKind::Geometry, "tg_layout_select: no score partials");
        std::vector<std::vector<double>> sc(static_cast<std::size_t>(K - 1), std::vector<double>(static_cast<std::size_t>(M)));
        for (int p = 0; p < K - 1; ++p)
            for (int m = 0; m < M; ++m) {
                double d2 = 0.0, r2 = 0.0;
                for (int r = 0; r < nranks; ++r) { // rank order == canonical chunk order
                    const std::size_t at = ((static_cast<std::size_t>(r) * (K - 1) + p) * M + m) * 2;
                    d2 += parts[at];
                    r2 += parts[at + 1];
                }
                sc[static_cast<std::size_t>(p)][static_cast<std::size_t>(m)] = magnitude_score(d2, r2);
                if (scores) scores[static_cast<std::size_t>(p) * M + m] = sc[static_cast<std::size_t>(p)][static_cast<std::size_t>(m)];
            }
        const Selection sel = select_by_magnitude(sc, M, rho);
        std::vector<CheckpointSummary> summ;
        for (int k = 1; k <= K; ++k) summ.push_back(fam.summary(k, fam.id(k)));
        if (source_of)
            for (int m = 0; m < M; ++m) source_of[m] = sel.source_of[static_cast<std::size_t>(m)];
        if (min_gap) *min_gap = sel.min_boundary_gap;
        put_text(recipe_to_yaml(recipe_from_selection(summ, sel)), out, cap, needed);
    });
}

tg_scorer* tg_scorer_create(const tg_layout* l, int32_t rank, int32_t k0, int32_t k1, int32_t packed) {
    tg_scorer* out = nullptr;
    guard([&] {
        const SnapshotSet& fam = *need(l, "tg_scorer_create").set;
        if (rank < 0 || rank >= fam.num_ranks()) fail(ErrorKind::Geometry, "rank out of range");
        if (k0 < 1 || k1 > fam.snapshots() || k1 - k0 < 1) fail(ErrorKind::Geometry, "snapshot range out of bounds");
        const auto fields = score_fields(fam.model(), fam.num_ranks());
        std::vector<std::vector<std::uint64_t>> offs;
        for (int k = k0; k <= k1; ++k) {
            std::vector<std::uint64_t> o;
            if (packed) {
                std::uint64_t at = 0;
                for (const auto& fl : fields) {
                    o.push_back(at);
                    at = (at + static_cast<std::uint64_t>(fl.chunk) * 4 + 15) & ~15ull;
                }
            } else {
                const ContainerLayout& c = fam.layout(k).shards.at(static_cast<std::size_t>(rank));
                for (const auto& fl : fields) {
                    const Entry* e = c.find(shard_key(fl.group, ".master"));
                    if (!e) fail(ErrorKind::MissingModules, "snapshot " + std::to_string(k) + " lacks " + shard_key(fl.group, ".master"));
                    o.push_back(e->begin);
                }
            }
            offs.push_back(std::move(o));
        }
        out = new tg_scorer{std::make_unique<ScorePlan>(fam.model(), fam.num_ranks(), std::move(offs))};
    });
    return out;
}

void tg_scorer_destroy(tg_scorer* s) { delete s; }

int tg_scorer_set_variant(tg_scorer* s, int32_t variant) {
    return guard([&] {
        if (variant < 0 || variant > 6)
            fail(ErrorKind::Geometry, "scorer variant: 0 auto, 1 register, 2 staged, 3 register-128b, 4 register-64b, "
                                          "5 staged half rows, 6 staged 2 CTAs/SM");
        need(s, "tg_scorer_set_variant").plan->set_variant(variant);
    });
}
uint64_t tg_scorer_bytes(const tg_scorer* s) { return s ? s->plan->bytes_read() : 0; }

int tg_scorer_run(tg_scorer* s, const uint8_t* const* bases, double* d_out, void* stream) {
    return guard([&] { need(s, "tg_scorer_run").plan->run(bases, d_out, static_cast<cudaStream_t>(stream)); });
}

tg_mplan* tg_mplan_create(const tg_layout* l, const char* yaml, int32_t container, int32_t unit, int32_t units) {
    tg_mplan* out = nullptr;
    guard([&] {
        const SnapshotSet& fam = *need(l, "tg_mplan_create").set;
        const MergePlan plan =
            resolve_plan_with(parse_recipe(yaml ? yaml : ""), [&](const std::string& id) { return family_summary(fam, id); });
        std::map<std::string, SourceLayout> lays;
        const LayoutLookup lay_of = [&](const std::string& id) -> const SourceLayout& {
            auto it = lays.find(id);
            if (it == lays.end()) {
                const int k = fam.index_of(id);
                if (k == 0) fail(ErrorKind::MissingArtifact, "unknown snapshot '" + id + "'");
                SourceLayout sl{fam.layout(k).weights, fam.layout(k).shards};
                it = lays.emplace(id, std::move(sl)).first;
            }
            return it->second;
        };
        PartitionPlan pp;
        if (container < 0) {
            const PartitionPlan full = plan_weights(plan, lay_of);
            const auto [lo, hi] = weights_share(full.out, unit, units);
            pp = plan_weights(plan, lay_of, lo, hi);
        } else {
            if (container >= plan.num_ranks) fail(ErrorKind::Geometry, "rank out of range");
            pp = plan_shard(plan, lay_of, container);
            if (units > 1) { // sub-unit of the rank partition, split at tensor boundaries
                const auto [lo, hi] = weights_share(pp.out, unit, units);
                pp = plan_shard(plan, lay_of, container, lo, hi);
            }
        }
        auto* p = new tg_mplan{};
        p->fam = &fam;
        for (const auto& w : pp.windows) {
            p->window_k.push_back(fam.index_of(w.source));
            const SourceLayout& sl = lay_of(w.source);
            p->window_layout.push_back(w.container < 0 ? sl.weights : sl.shards.at(static_cast<std::size_t>(w.container)));
        }
        p->dev = std::make_unique<DeviceMerge>(pp);
        out = p;
    });
    return out;
}

void tg_mplan_destroy(tg_mplan* p) { delete p; }
uint64_t tg_mplan_bytes(const tg_mplan* p) { return p ? p->dev->bytes() : 0; }

int tg_mplan_range(const tg_mplan* p, uint64_t* lo, uint64_t* hi, uint64_t* payload) {
    return guard([&] {
        const PartitionPlan& pp = need(p, "tg_mplan_range").dev->plan();
        if (lo) *lo = pp.dst_lo;
        if (hi) *hi = pp.dst_hi;
        if (payload) *payload = pp.out.payload_bytes;
    });
}

int32_t tg_mplan_num_windows(const tg_mplan* p) { return p ? static_cast<int32_t>(p->dev->plan().windows.size()) : 0; }

int tg_mplan_window(const tg_mplan* p, int32_t i, int32_t* k, int32_t* container, uint64_t* lo, uint64_t* hi) {
    return guard([&] {
        const auto& w = need(p, "tg_mplan_window").dev->plan().windows.at(static_cast<std::size_t>(i));
        if (k) *k = p->window_k.at(static_cast<std::size_t>(i));
        if (container) *container = w.container;
        if (lo) *lo = w.lo;
        if (hi) *hi = w.hi;
    });
}

uint32_t tg_mplan_num_segments(const tg_mplan* p) { return p ? static_cast<uint32_t>(p->dev->plan().segments.size()) : 0; }

int tg_mplan_segment(const tg_mplan* p, uint32_t i, uint32_t* window, uint64_t* src_off, uint64_t* dst_off, uint64_t* bytes) {
    return guard([&] {
        const PartitionPlan& pp = need(p, "tg_mplan_segment").dev->plan();
        const CopySegment& s = pp.segments.at(i);
        if (window) *window = s.window;
        if (src_off) *src_off = s.src_off;
        if (dst_off) *dst_off = s.dst_off - pp.dst_lo;
        if (bytes) *bytes = s.bytes;
    });
}

int tg_mplan_prefix(const tg_mplan* p, char* out, size_t cap, size_t* needed) {
    return guard([&] {
        const std::string s = need(p, "tg_mplan_prefix").dev->plan().out.prefix();
        if (needed) *needed = s.size();
        if (!out || cap < s.size()) fail(ErrorKind::Geometry, "output buffer too small");
        std::memcpy(out, s.data(), s.size());
    });
}

int tg_mplan_bind(tg_mplan* p, const uint8_t* const* ptrs) {
    return guard([&] {
        need(p, "tg_mplan_bind");
        if (!ptrs && !p->dev->plan().windows.empty()) fail(ErrorKind::Geometry, "tg_mplan_bind: null window list");
        p->dev->bind(std::vector<const std::uint8_t*>(ptrs, ptrs + p->dev->plan().windows.size())); });
}

int32_t tg_mplan_bulk_ok(const tg_mplan* p) { return p && p->dev->bulk_ok() ? 1 : 0; }

int tg_mplan_run(tg_mplan* p, uint8_t* d_dst, int32_t variant, void* stream) {
    return guard([&] { need(p, "tg_mplan_run").dev->run(d_dst, variant, static_cast<cudaStream_t>(stream)); });
}

int tg_mplan_run_host(tg_mplan* p, const uint8_t* const* h_windows, const uint8_t* const* d_windows,
                      uint32_t resident_fields, uint8_t* h_dst, int32_t variant, uint64_t chunk, int32_t async,
                      const tg_host_copy* prefetch, uint32_t nprefetch, uint64_t* h2d, uint64_t* d2h) {
    return guard([&] {
        const PartitionPlan& pp = need(p, "tg_mplan_run_host").dev->plan();
        if (!h_windows || !h_dst) fail(ErrorKind::Geometry, "tg_mplan_run_host: null host windows or destination");
        if (!d_windows) resident_fields = 0;
        // Resident ranges: bits 0-2 read exp_avg / exp_avg_sq / master from d_windows[w], a
        // device copy of the window in shard layout; bit 3 reads the masters from
        // d_windows[w] = the window snapshot's packed masters of this rank (the scorer's
        // layout, SynthFamily::gen_masters). Windows with a null d_windows entry stay on PCIe.
        HostMerge::Resident res(pp.windows.size());
        static const char* kField[3] = {".exp_avg", ".exp_avg_sq", ".master"};
        std::map<int, std::uint64_t> packed_off; // group -> offset in the packed masters
        if (resident_fields & 8u) {
            std::uint64_t off = 0;
            for (const auto& f : score_fields(p->fam->model(), p->fam->num_ranks())) {
                packed_off[f.group] = off;
                off = (off + static_cast<std::uint64_t>(f.chunk) * 4 + 15) & ~15ull;
            }
        }
        for (std::size_t w = 0; resident_fields && w < pp.windows.size(); ++w) {
            if (pp.windows[w].container < 0 || !d_windows[w]) continue; // weights are never resident
            const std::uint64_t wlo = pp.windows[w].lo, whi = pp.windows[w].hi;
            for (const auto& e : p->window_layout[w].entries) {
                const std::uint64_t a = std::max(e.begin, wlo), b = std::min(e.end, whi);
                if (a >= b) continue;
                const std::string& n = e.name;
                const auto ends = [&](const char* suf) {
                    const std::size_t k = std::strlen(suf);
                    return n.size() >= k && n.compare(n.size() - k, k, suf) == 0;
                };
                const int f = ends(kField[1]) ? 1 : ends(kField[0]) ? 0 : ends(kField[2]) ? 2 : -1;
                if (f < 0) continue;
                if ((resident_fields & 8u) && f == 2) {
                    const int g = std::stoi(n.substr(1, n.find('.') - 1));
                    res[w].push_back({a - wlo, b - wlo, packed_off.at(g) + (a - e.begin)});
                } else if (resident_fields & (1u << f)) {
                    res[w].push_back({a - wlo, b - wlo, a - wlo});
                }
            }
            std::sort(res[w].begin(), res[w].end(),
                      [](const HostMerge::ResidentRange& x, const HostMerge::ResidentRange& y) { return x.lo < y.lo; });
        }
        if (!p->host || p->host_chunk != chunk || p->host_resident != res) {
            p->host = std::make_unique<HostMerge>(pp, chunk ? chunk : (256ull << 20), res);
            p->host_chunk = chunk;
            p->host_resident = std::move(res);
        }
        std::vector<const std::uint8_t*> dw(pp.windows.size(), nullptr);
        if (d_windows) dw.assign(d_windows, d_windows + pp.windows.size());
        std::vector<HostCopy> pf;
        for (uint32_t i = 0; prefetch && i < nprefetch; ++i) pf.push_back({prefetch[i].src, prefetch[i].dst, prefetch[i].bytes});
        p->host->run(std::vector<const std::uint8_t*>(h_windows, h_windows + pp.windows.size()), dw, h_dst, variant,
                     async != 0, pf);
        if (h2d) *h2d = p->host->h2d_bytes();
        if (d2h) *d2h = p->host->d2h_bytes();
    });
}

int tg_mplan_wait(tg_mplan* p) {
    return guard([&] {
        if (need(p, "tg_mplan_wait").host) p->host->wait();
    });
}

tg_dstep* tg_dstep_create(const tg_layout* l, int32_t rank, int32_t unit, int32_t units, double rho) {
    tg_dstep* out = nullptr;
    guard([&] { out = new tg_dstep{std::make_unique<DeviceSelectStep>(*need(l, "tg_dstep_create").set, rank, unit, units, rho)}; });
    return out;
}

void tg_dstep_destroy(tg_dstep* s) { delete s; }

int tg_dstep_range(const tg_dstep* s, uint64_t* shard_bytes, uint64_t* wlo, uint64_t* whi) {
    return guard([&] {
        need(s, "tg_dstep_range");
        if (shard_bytes) *shard_bytes = s->step->shard_bytes();
        if (wlo) *wlo = s->step->weights_lo();
        if (whi) *whi = s->step->weights_hi();
    });
}

int tg_dstep_bind(tg_dstep* s, const uint8_t* const* shard_bases, const uint8_t* const* wwin_bases) {
    return guard([&] { need(s, "tg_dstep_bind").step->bind(shard_bases, wwin_bases); });
}

int tg_dstep_run(tg_dstep* s, const double* d_parts, int32_t nranks, uint8_t* d_out_shard, uint8_t* d_out_w, int32_t variant,
                 int32_t phases, void* stream) {
    return guard([&] {
        need(s, "tg_dstep_run").step->run(d_parts, nranks, d_out_shard, d_out_w, variant, static_cast<cudaStream_t>(stream), phases);
    });
}

int tg_dstep_result(tg_dstep* s, int32_t* source_of, double* scores, void* stream) {
    return guard([&] {
        const auto src = need(s, "tg_dstep_result").step->source_of(static_cast<cudaStream_t>(stream));
        if (source_of) std::copy(src.begin(), src.end(), source_of);
        if (scores) {
            const auto sc = s->step->scores(static_cast<cudaStream_t>(stream));
            std::copy(sc.begin(), sc.end(), scores);
        }
    });
}

int tg_comm_unique_id(uint8_t id_out[128]) {
    return guard([&] {
        if (!id_out) fail(ErrorKind::Recipe, "tg_comm_unique_id: null output");
        const auto id = comm_unique_id();
        std::copy(id.begin(), id.end(), id_out);
    });
}

tg_comm* tg_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device) {
    tg_comm* out = nullptr;
    guard([&] {
        if (!id) fail(ErrorKind::Recipe, "tg_comm_create: null id");
        out = new tg_comm{std::make_unique<Comm>(id, nranks, rank, device)};
    });
    return out;
}

void tg_comm_destroy(tg_comm* c) { delete c; }

int tg_comm_allgather(tg_comm* c, const double* d_send, double* d_recv, uint64_t count, void* stream) {
    return guard([&] {
        if (!c) fail(ErrorKind::Recipe, "tg_comm_allgather: null communicator");
        c->comm->all_gather(d_send, d_recv, count, static_cast<cudaStream_t>(stream));
    });
}

} // extern "C"
