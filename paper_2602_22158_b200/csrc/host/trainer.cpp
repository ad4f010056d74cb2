// Device-resident trainer (see tailor/trainer.hpp).
#include "tailor/trainer.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <fstream>
#include <unistd.h>
#include <fcntl.h>
#include <map>
#include <set>

#include <json.hpp>

#include "tailor/errors.hpp"
#include "tailor/io.hpp"

namespace tailor {

namespace fs = std::filesystem;

void validate_strategy(const StrategyConfig& cfg, const ModelSpec& spec) {
    if (cfg.interval < 1) fail(ErrorKind::Recipe, "checkpoint interval must be >= 1");
    if (cfg.kind == StrategyKind::Filter) {
        if (cfg.head_count < 0 || cfg.tail_count < 0 || cfg.sparse_multiple < 1)
            fail(ErrorKind::Recipe, "invalid filter parameters");
        if (cfg.head_count + cfg.tail_count > spec.num_layers)
            fail(ErrorKind::Recipe, "filter head_count + tail_count exceeds the layer count");
    }
}

std::vector<ModuleId> modules_to_save(const StrategyConfig& cfg, const ModelSpec& spec, std::int64_t counter) {
    spec.validate();
    validate_strategy(cfg, spec);
    if (counter < 1) fail(ErrorKind::Geometry, "checkpoint counter starts at 1");
    const int L = spec.num_layers;
    if (cfg.kind == StrategyKind::Full) return enumerate_modules(spec);
    std::set<ModuleId> pick;
    if (cfg.kind == StrategyKind::Parity) {
        // odd counters: even layers + norm + lm_head; even counters: odd layers + embed
        const bool odd = counter % 2 == 1;
        for (int i = odd ? 0 : 1; i < L; i += 2) pick.insert(ModuleId::transformer_layer(i));
        if (odd) {
            pick.insert(ModuleId::norm());
            if (!spec.weight_tied) pick.insert(ModuleId::lm_head());
        } else {
            pick.insert(ModuleId::embed_tokens());
        }
    } else {
        for (int i = 0; i < cfg.head_count; ++i) pick.insert(ModuleId::transformer_layer(i));
        for (int i = L - cfg.tail_count; i < L; ++i) pick.insert(ModuleId::transformer_layer(i));
        pick.insert(ModuleId::norm());
        if (counter % cfg.sparse_multiple == 0) {
            const std::int64_t multiple = counter / cfg.sparse_multiple;
            const int lo = cfg.head_count, hi = L - cfg.tail_count; // middle [lo, hi)
            const int lower = (hi - lo + 1) / 2;
            if (multiple % 2 == 1) {
                for (int i = lo; i < lo + lower; ++i) pick.insert(ModuleId::transformer_layer(i));
                pick.insert(ModuleId::embed_tokens());
            } else {
                for (int i = lo + lower; i < hi; ++i) pick.insert(ModuleId::transformer_layer(i));
                if (!spec.weight_tied) pick.insert(ModuleId::lm_head());
            }
        }
    }
    std::vector<ModuleId> out;
    for (const auto& m : enumerate_modules(spec))
        if (pick.count(m)) out.push_back(m);
    return out;
}

struct DeviceTrainer::Rank {
    DeviceBuffer part, groups, slices, tiles, grad, grad_part, delta_part;
    std::uint32_t ngroups = 0, ntiles = 0;
    std::uint64_t total = 0;
    unsigned grid = 0;
    // in-situ scorer state
    DeviceBuffer kept, keep_segs, score_out;
    std::uint32_t nkeep = 0;
    std::uint64_t kept_bytes = 0;
    std::unique_ptr<ScorePlan> plan;
};

namespace {

std::uint64_t align16(std::uint64_t x) { return (x + 15) & ~15ull; }

void write_container_file(const fs::path& path, const ContainerLayout& lay, const std::vector<std::uint8_t>& payload) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(ErrorKind::Storage, "cannot create '" + path.string() + "'");
    const std::string prefix = lay.prefix();
    out.write(prefix.data(), static_cast<std::streamsize>(prefix.size()));
    out.write(reinterpret_cast<const char*>(payload.data()), static_cast<std::streamsize>(lay.payload_bytes));
    out.flush();
    if (!out) fail(ErrorKind::Storage, "write failed for '" + path.string() + "'");
}

} // namespace

DeviceTrainer::DeviceTrainer(const ModelSpec& spec, int num_ranks, const AdamHyperparams& base, int device, int rank_begin,
                             int rank_end)
    : model_(spec), N_(num_ranks), base_(base) {
    base_.validate();
    if (const char* v = std::getenv("TAILOR_TRAIN_STORE_GRAD")) store_grad_ = *v && *v != '0';
    if (const char* v = std::getenv("TAILOR_TRAIN_FDIV")) fdiv_ = *v && *v != '0';
    if (num_ranks < 1) fail(ErrorKind::Recipe, "num_ranks must be >= 1");
    r0_ = rank_begin;
    r1_ = rank_end < 0 ? num_ranks : rank_end;
    if (r0_ < 0 || r1_ > num_ranks || r0_ >= r1_) fail(ErrorKind::Geometry, "bad rank range for the trainer");
    for (const auto& g : model_.table().groups) hyper_.push_back(hyper_for_class(base_, g.decay));
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
    full_ = checkpoint_layout(model_, N_, model_.modules());
    const ShardGeometry geom{N_};
    std::vector<const std::uint8_t*> ptrs;
    for (int r = r0_; r < r1_; ++r) {
        auto rk = std::make_unique<Rank>();
        const ContainerLayout& lay = full_.shards[static_cast<std::size_t>(r)];
        rk->part.resize(std::max<std::uint64_t>(16, lay.payload_bytes));
        cuda_check(cudaMemsetAsync(rk->part.get(), 0, lay.payload_bytes, stream_), "memset");
        std::vector<dev::TrainGroup> tg;
        std::vector<dev::TrainTile> tiles;
        std::vector<dev::SynthGroup> sg;
        std::vector<dev::SynthSlice> sl;
        std::uint64_t begin = 0, vbegin = 0; // generator / gradient-scratch element spaces
        for (int g = 0; g < model_.table().group_count(); ++g) {
            const std::int64_t len = model_.table().groups[static_cast<std::size_t>(g)].element_count;
            const std::uint64_t chunk = static_cast<std::uint64_t>(geom.shard_length(len));
            const std::uint32_t sb = static_cast<std::uint32_t>(sl.size());
            for (const auto& s : model_.slices(g)) sl.push_back({s.group_offset, s.model_offset, s.decl.numel()});
            const std::uint64_t om = lay.find(shard_key(g, ".exp_avg"))->begin, ov = lay.find(shard_key(g, ".exp_avg_sq"))->begin,
                                ow = lay.find(shard_key(g, ".master"))->begin;
            if (chunk == 0) continue;
            elements_ += static_cast<std::uint64_t>(std::clamp<std::int64_t>(len - static_cast<std::int64_t>(r) * static_cast<std::int64_t>(chunk), 0,
                                                                             static_cast<std::int64_t>(chunk)));
            tg.push_back({begin, chunk, static_cast<std::uint64_t>(r) * chunk, static_cast<std::uint64_t>(len), om, ov, ow, sb,
                          static_cast<std::uint32_t>(model_.slices(g).size()), static_cast<std::uint32_t>(g), 0});
            // tiles: non-padding elements of this rank's chunk, split at tensor slices
            // and at field-index multiples of kTrainTileElems (4-aligned runs)
            const std::int64_t first = static_cast<std::int64_t>(r) * static_cast<std::int64_t>(chunk);
            const std::int64_t valid_end = std::min<std::int64_t>(len, first + static_cast<std::int64_t>(chunk));
            const bool fields16 = om % 16 == 0 && ov % 16 == 0 && ow % 16 == 0;
            for (const auto& sc : model_.slices(g)) {
                std::int64_t a = std::max<std::int64_t>(sc.group_offset, first);
                const std::int64_t b = std::min<std::int64_t>(sc.group_offset + sc.decl.numel(), valid_end);
                while (a < b) {
                    const std::uint64_t i0 = static_cast<std::uint64_t>(a - first);
                    const std::uint64_t next = (i0 / dev::kTrainTileElems + 1) * dev::kTrainTileElems;
                    const std::uint64_t n = std::min<std::uint64_t>(next - i0, static_cast<std::uint64_t>(b - a));
                    dev::TrainTile t{};
                    t.v0 = vbegin + i0;
                    t.i0 = i0;
                    t.e0 = static_cast<std::uint64_t>(sc.model_offset + (a - sc.group_offset));
                    t.count = static_cast<std::uint32_t>(n);
                    t.group = static_cast<std::uint16_t>(tg.size() - 1);
                    t.vec = fields16 && i0 % 4 == 0 && n % 4 == 0 ? 1 : 0;
                    tiles.push_back(t);
                    a += static_cast<std::int64_t>(n);
                }
            }
            vbegin = (vbegin + chunk + 3) & ~3ull;
            dev::SynthGroup s{};
            s.begin = begin;
            s.chunk = chunk;
            s.group_first = static_cast<std::uint64_t>(r) * chunk;
            s.true_len = static_cast<std::uint64_t>(len);
            s.off[0] = ~0ull; // exp_avg / exp_avg_sq start at zero (memset)
            s.off[1] = ~0ull;
            s.off[2] = ow;
            s.slice_begin = sb;
            s.slice_count = static_cast<std::uint32_t>(model_.slices(g).size());
            s.module = static_cast<std::uint32_t>(model_.owner_index(g));
            sg.push_back(s);
            begin += chunk;
        }
        rk->ngroups = static_cast<std::uint32_t>(tg.size());
        rk->total = begin;
        if (tg.size() > 0xFFFF) fail(ErrorKind::Geometry, "too many optimizer groups for the trainer tile table");
        rk->groups.upload(tg.data(), tg.size() * sizeof(dev::TrainGroup));
        rk->slices.upload(sl.data(), sl.size() * sizeof(dev::SynthSlice));
        rk->ntiles = static_cast<std::uint32_t>(tiles.size());
        rk->tiles.upload(tiles.data(), std::max<std::size_t>(1, tiles.size()) * sizeof(dev::TrainTile));
        rk->grid = dev::train_grid(rk->ntiles);
        rk->grad_part.resize(rk->grid * sizeof(double));
        if (store_grad_) rk->grad.resize(std::max<std::uint64_t>(16, vbegin * sizeof(float)));
        rk->delta_part.resize(rk->grid * sizeof(double));
        // W_0 = 0.02 * u(seed, 0, e) (init_state, R/src/gradients.cpp:51-66): the
        // generator with k1 = 0 writes exactly the initial masters.
        DeviceBuffer sgb;
        sgb.upload(sg.data(), sg.size() * sizeof(dev::SynthGroup));
        dev::OutPtrs outs{};
        outs.p[0] = rk->part.get();
        cuda_check(dev::launch_synth_shard(sgb.get<dev::SynthGroup>(), static_cast<std::uint32_t>(sg.size()),
                                           rk->slices.get<dev::SynthSlice>(), nullptr, model_.module_count(),
                                           model_.spec().seed, 0, 0, outs, begin, stream_),
                   "init masters");
        cuda_check(cudaStreamSynchronize(stream_), "sync");
        ptrs.push_back(rk->part.get());
        ranks_.push_back(std::move(rk));
    }
    part_ptrs_.upload(ptrs.data(), ptrs.size() * sizeof(void*));
    flag_.resize(sizeof(unsigned int));
    coef_.resize(static_cast<std::size_t>(model_.table().group_count()) * sizeof(dev::AdamCoef));
}

DeviceTrainer::~DeviceTrainer() {
    if (stream_) cudaStreamDestroy(stream_);
}

std::uint64_t DeviceTrainer::elements() const { return elements_; }

void DeviceTrainer::load(const fs::path& dir, const CheckpointSummary& s) {
    if (s.optim.grouping != Grouping::Fine)
        fail(ErrorKind::Geometry, "the device trainer resumes fine-grouped checkpoints; convert with `tailor regroup --to fine`");
    if (s.optim.num_ranks != N_ || !s.spec.same_geometry(model_.spec()))
        fail(ErrorKind::Geometry, "checkpoint geometry does not match the trainer");
    for (const auto& g : s.optim.groups) hyper_.at(static_cast<std::size_t>(g.index)) = g.hyper;
    masters_checked_ = masters_bad_ = false; // new state: the next step checks it
    PinnedBuffer stage;
    for (int r = r0_; r < r1_; ++r) {
        const fs::path p = ckpt_file(CkptFile::Shard, dir, r);
        const ContainerLayout lay = read_layout(p);
        const ContainerLayout& want = full_.shards[static_cast<std::size_t>(r)];
        if (lay.payload_bytes != want.payload_bytes || lay.entries.size() != want.entries.size())
            fail(ErrorKind::Geometry, p.string() + ": shard layout does not match a complete fine checkpoint");
        for (std::size_t i = 0; i < lay.entries.size(); ++i)
            if (lay.entries[i].name != want.entries[i].name || lay.entries[i].begin != want.entries[i].begin ||
                lay.entries[i].bytes() != want.entries[i].bytes())
                fail(ErrorKind::Geometry, p.string() + ": shard layout does not match a complete fine checkpoint");
        // the rank partition IS the file payload (same keys, same order)
        stage.resize(std::max<std::uint64_t>(16, lay.payload_bytes));
        const int fd = ::open(p.c_str(), O_RDONLY);
        if (fd < 0) fail(ErrorKind::MissingArtifact, "cannot open '" + p.string() + "'");
        try {
            run_reads({{fd, stage.get(), lay.payload_bytes, lay.payload_offset()}}, io_threads(), p.string());
        } catch (...) {
            ::close(fd);
            throw;
        }
        ::close(fd);
        auto& rk = ranks_[static_cast<std::size_t>(r - r0_)];
        cuda_check(cudaMemcpyAsync(rk->part.get(), stage.get(), lay.payload_bytes, cudaMemcpyHostToDevice, stream_), "H2D");
        cuda_check(cudaStreamSynchronize(stream_), "sync");
    }
    t_ = s.trainer.optimizer_t;
}

std::pair<std::uint8_t*, std::uint64_t> DeviceTrainer::partition(int rank) {
    if (rank < r0_ || rank >= r1_) fail(ErrorKind::Geometry, "rank " + std::to_string(rank) + " is not held by this trainer");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    masters_checked_ = masters_bad_ = false; // the caller may write the state
    const auto& rk = ranks_[static_cast<std::size_t>(rank - r0_)];
    return {rk->part.get(), full_.shards[static_cast<std::size_t>(rank)].payload_bytes};
}

std::pair<double, double> DeviceTrainer::step(std::int64_t s) {
    const dev::TrainParams p{dev::noise_prefix(model_.spec().seed, static_cast<std::uint64_t>(s)), 0.05f, 0.01f};
    cuda_check(cudaMemsetAsync(flag_.get(), 0, sizeof(unsigned int), stream_), "memset");
    // fast check: masters' finiteness decides the gradient's (see finite_check_kernel);
    // the gradient norm then comes from the update pass
    const bool fast = !store_grad_ && dev::finite_check_suffices(p);
    if (fast && masters_bad_) fail(ErrorKind::NonFinite, "non-finite gradient at step " + std::to_string(s));
    if (!(fast && masters_checked_)) { // otherwise the previous update pass already checked these masters
        for (auto& rk : ranks_)
            cuda_check(fast ? dev::launch_finite_check(rk->tiles.get<dev::TrainTile>(), rk->ntiles, rk->groups.get<dev::TrainGroup>(),
                                                       rk->part.get(), flag_.get<unsigned int>(), stream_)
                            : dev::launch_grad_check(rk->tiles.get<dev::TrainTile>(), rk->ntiles, rk->groups.get<dev::TrainGroup>(),
                                                     rk->part.get(), p, store_grad_ ? rk->grad.get<float>() : nullptr,
                                                     rk->grad_part.get<double>(), flag_.get<unsigned int>(), stream_),
                       "grad check");
        unsigned int bad = 0;
        cuda_check(cudaMemcpyAsync(&bad, flag_.get(), sizeof(bad), cudaMemcpyDeviceToHost, stream_), "D2H");
        cuda_check(cudaStreamSynchronize(stream_), "sync");
        if (bad) {
            masters_bad_ = fast;
            fail(ErrorKind::NonFinite, "non-finite gradient at step " + std::to_string(s));
        }
    }
    if (fast) {
        next_flag_.resize(sizeof(unsigned int));
        cuda_check(cudaMemsetAsync(next_flag_.get(), 0, sizeof(unsigned int), stream_), "memset");
    }
    t_ += 1;
    std::vector<dev::AdamCoef> coef(static_cast<std::size_t>(model_.table().group_count()));
    for (const auto& g : model_.table().groups) {
        const AdamHyperparams& h = hyper_[static_cast<std::size_t>(g.index)];
        dev::AdamCoef& c = coef[static_cast<std::size_t>(g.index)];
        c.b1 = static_cast<float>(h.beta1);
        c.one_minus_b1 = static_cast<float>(1.0 - h.beta1);
        c.b2 = static_cast<float>(h.beta2);
        c.one_minus_b2 = static_cast<float>(1.0 - h.beta2);
        c.bias1 = static_cast<float>(1.0 - std::pow(h.beta1, static_cast<double>(t_)));
        c.bias2 = static_cast<float>(1.0 - std::pow(h.beta2, static_cast<double>(t_)));
        c.lr = static_cast<float>(h.lr);
        c.eps = static_cast<float>(h.eps);
        c.wd = static_cast<float>(h.weight_decay);
        // y = 0 sends the kernel to __fdiv_rn (TAILOR_TRAIN_FDIV=1: measurement / tests)
        c.rcp1 = fdiv_ ? 0.f : dev::const_reciprocal(c.bias1);
        c.rcp2 = fdiv_ ? 0.f : dev::const_reciprocal(c.bias2);
    }
    cuda_check(cudaMemcpyAsync(coef_.get(), coef.data(), coef.size() * sizeof(dev::AdamCoef), cudaMemcpyHostToDevice, stream_),
               "coef");
    for (auto& rk : ranks_)
        cuda_check(dev::launch_adamw(rk->tiles.get<dev::TrainTile>(), rk->ntiles, rk->groups.get<dev::TrainGroup>(),
                                     coef_.get<dev::AdamCoef>(), rk->part.get(),
                                     store_grad_ ? rk->grad.get<float>() : nullptr, p, rk->delta_part.get<double>(),
                                     fast ? rk->grad_part.get<double>() : nullptr,
                                     fast ? next_flag_.get<unsigned int>() : nullptr, stream_),
                   "adamw");
    double g2 = 0.0, d2 = 0.0;
    std::vector<double> h;
    for (auto& rk : ranks_) {
        h.resize(2 * rk->grid);
        cuda_check(cudaMemcpyAsync(h.data(), rk->grad_part.get(), rk->grid * sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H");
        cuda_check(cudaMemcpyAsync(h.data() + rk->grid, rk->delta_part.get(), rk->grid * sizeof(double), cudaMemcpyDeviceToHost,
                                   stream_),
                   "D2H");
        cuda_check(cudaStreamSynchronize(stream_), "sync");
        for (unsigned b = 0; b < rk->grid; ++b) {
            g2 += h[b];
            d2 += h[rk->grid + b];
        }
    }
    if (fast) { // the stream is synchronized: the flag of the masters just written is final
        unsigned int next_bad = 0;
        cuda_check(cudaMemcpy(&next_bad, next_flag_.get(), sizeof(next_bad), cudaMemcpyDeviceToHost), "D2H");
        masters_checked_ = next_bad == 0;
        masters_bad_ = next_bad != 0;
    } else {
        masters_checked_ = masters_bad_ = false;
    }
    return {std::sqrt(g2), std::sqrt(d2)};
}

void DeviceTrainer::save(const fs::path& dir, const TrainerMeta& meta, const std::vector<ModuleId>& modules,
                         const std::string& label) {
    if (r0_ != 0 || r1_ != N_) fail(ErrorKind::Consistency, "saving a checkpoint needs every rank partition");
    const CheckpointLayout lay = checkpoint_layout(model_, N_, modules);
    const ShardGeometry geom{N_};
    std::error_code ec;
    fs::create_directories(dir / "optim", ec);
    if (ec) fail(ErrorKind::Storage, "cannot create '" + dir.string() + "': " + ec.message());
    // weights: K8 from the sharded masters
    std::map<std::string, std::pair<int, std::int64_t>> where;
    for (const auto& g : model_.table().groups)
        for (const auto& s : model_.slices(g.index)) where[s.decl.name] = {g.index, s.group_offset};
    std::vector<dev::WeightTensor> wt;
    std::uint64_t begin = 0;
    for (const auto& e : lay.weights.entries) {
        const auto [g, goff] = where.at(e.name);
        const std::uint64_t chunk = static_cast<std::uint64_t>(geom.shard_length(model_.table().groups[static_cast<std::size_t>(g)].element_count));
        wt.push_back({begin, e.begin, static_cast<std::uint64_t>(goff), chunk, full_.shards[0].find(shard_key(g, ".master"))->begin});
        begin += e.bytes() / 2;
    }
    std::uint64_t most = lay.weights.payload_bytes;
    for (const auto& c : lay.shards) most = std::max(most, c.payload_bytes);
    DeviceBuffer out(std::max<std::uint64_t>(16, most)), wtab, segs;
    std::vector<std::uint8_t> host(most);
    wtab.upload(wt.data(), wt.size() * sizeof(dev::WeightTensor));
    cuda_check(dev::launch_derive_weights(wtab.get<dev::WeightTensor>(), static_cast<std::uint32_t>(wt.size()),
                                          part_ptrs_.get<const std::uint8_t*>(), out.get(), begin, stream_),
               "derive weights");
    cuda_check(cudaMemcpyAsync(host.data(), out.get(), lay.weights.payload_bytes, cudaMemcpyDeviceToHost, stream_), "D2H");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    write_container_file(ckpt_file(CkptFile::Weights, dir), lay.weights, host);
    // shards: the kept groups' fields gathered (K2) out of the full partitions
    const bool complete = lay.groups.size() == static_cast<std::size_t>(model_.table().group_count());
    for (int r = 0; r < N_; ++r) {
        const ContainerLayout& sl = lay.shards[static_cast<std::size_t>(r)];
        const std::uint8_t* src = ranks_[static_cast<std::size_t>(r)]->part.get();
        if (complete) {
            cuda_check(cudaMemcpyAsync(host.data(), src, sl.payload_bytes, cudaMemcpyDeviceToHost, stream_), "D2H");
        } else {
            std::vector<dev::GatherSeg> gs;
            const ContainerLayout& fl = full_.shards[static_cast<std::size_t>(r)];
            for (const auto& e : sl.entries) gs.push_back({src + fl.find(e.name)->begin, e.begin, e.bytes()});
            segs.upload(gs.data(), gs.size() * sizeof(dev::GatherSeg));
            cuda_check(dev::launch_gather(segs.get<dev::GatherSeg>(), static_cast<std::uint32_t>(gs.size()), out.get(),
                                          sl.payload_bytes, dev::kGatherLsu, false, stream_),
                       "gather");
            cuda_check(cudaMemcpyAsync(host.data(), out.get(), sl.payload_bytes, cudaMemcpyDeviceToHost, stream_), "D2H");
        }
        cuda_check(cudaStreamSynchronize(stream_), "sync");
        write_container_file(ckpt_file(CkptFile::Shard, dir, r), sl, host);
    }
    std::map<int, AdamHyperparams> hyp;
    for (int g : lay.groups) hyp[g] = hyper_[static_cast<std::size_t>(g)];
    SaveManifest man;
    man.step = meta.step;
    man.strategy = label;
    man.modules = modules;
    write_text_file(ckpt_file(CkptFile::OptimMeta, dir), sidecar_text(make_optim_meta(model_.table(), hyp, geom, meta.optimizer_t)));
    write_text_file(ckpt_file(CkptFile::Config, dir), sidecar_text(model_.spec()));
    write_text_file(ckpt_file(CkptFile::TrainerState, dir), sidecar_text(meta));
    write_text_file(ckpt_file(CkptFile::Manifest, dir), sidecar_text(man));
}

void DeviceTrainer::keep_masters() {
    const auto fields = score_fields(model_, N_);
    for (int r = r0_; r < r1_; ++r) {
        Rank& rk = *ranks_[static_cast<std::size_t>(r - r0_)];
        const ContainerLayout& fl = full_.shards[static_cast<std::size_t>(r)];
        if (!rk.plan) {
            std::vector<dev::GatherSeg> gs;
            std::vector<std::vector<std::uint64_t>> offs(2);
            std::uint64_t at = 0;
            for (const auto& f : fields) {
                const Entry* e = fl.find(shard_key(f.group, ".master"));
                gs.push_back({rk.part.get() + e->begin, at, e->bytes()});
                offs[0].push_back(at);
                offs[1].push_back(e->begin);
                at = align16(at + e->bytes());
            }
            rk.kept_bytes = at;
            rk.kept.resize(std::max<std::uint64_t>(16, at));
            // zero the alignment gaps once; the gather never writes them
            cuda_check(cudaMemsetAsync(rk.kept.get(), 0, std::max<std::uint64_t>(16, at), stream_), "memset");
            rk.keep_segs.upload(gs.data(), gs.size() * sizeof(dev::GatherSeg));
            rk.nkeep = static_cast<std::uint32_t>(gs.size());
            rk.plan = std::make_unique<ScorePlan>(model_, N_, std::move(offs));
            rk.score_out.resize(static_cast<std::size_t>(model_.module_count()) * 2 * sizeof(double));
        }
        cuda_check(dev::launch_gather(rk.keep_segs.get<dev::GatherSeg>(), rk.nkeep, rk.kept.get(), rk.kept_bytes,
                                      dev::kGatherLsu, false, stream_),
                   "keep masters");
    }
    cuda_check(cudaStreamSynchronize(stream_), "sync");
}

std::vector<std::pair<double, double>> DeviceTrainer::score_against_kept() {
    const int M = model_.module_count();
    std::vector<std::pair<double, double>> sums(static_cast<std::size_t>(M), {0.0, 0.0});
    std::vector<double> h(static_cast<std::size_t>(M) * 2);
    for (auto& rk : ranks_) { // rank order == canonical chunk order
        if (!rk->plan) fail(ErrorKind::Consistency, "score_against_kept before keep_masters");
        const std::uint8_t* bases[2] = {rk->kept.get(), rk->part.get()};
        rk->plan->run(bases, rk->score_out.get<double>(), stream_);
        cuda_check(cudaMemcpyAsync(h.data(), rk->score_out.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_),
                   "D2H");
        cuda_check(cudaStreamSynchronize(stream_), "sync");
        for (int m = 0; m < M; ++m) {
            sums[static_cast<std::size_t>(m)].first += h[static_cast<std::size_t>(m) * 2];
            sums[static_cast<std::size_t>(m)].second += h[static_cast<std::size_t>(m) * 2 + 1];
        }
    }
    return sums;
}

std::vector<fs::path> device_train(const DeviceTrainConfig& cfg, const fs::path& out_dir) {
    cfg.spec.validate();
    validate_strategy(cfg.strategy, cfg.spec);
    cfg.hyper.validate();
    if (cfg.total_steps < 0) fail(ErrorKind::Recipe, "total_steps must be >= 0");
    std::error_code ec;
    if (fs::exists(out_dir) && !fs::is_empty(out_dir, ec))
        fail(ErrorKind::Storage, "refusing to write into non-empty directory '" + out_dir.string() + "'");
    fs::create_directories(out_dir, ec);
    if (ec) fail(ErrorKind::Storage, "cannot create '" + out_dir.string() + "': " + ec.message());
    DeviceTrainer tr(cfg.spec, cfg.num_ranks, cfg.hyper, cfg.device);
    std::ofstream log(out_dir / "log.jsonl", std::ios::binary);
    if (!log) fail(ErrorKind::Storage, "cannot create log in '" + out_dir.string() + "'");
    TrainerMeta meta;
    meta.lr = cfg.hyper.lr;
    meta.strategy = cfg.strategy;
    meta.rng_seed = cfg.spec.seed;
    const int M = tr.model().module_count();
    std::vector<fs::path> saved;
    for (std::int64_t s = 1; s <= cfg.total_steps; ++s) {
        const auto [gn, un] = tr.step(s);
        log << nlohmann::json{{"grad_norm", gn}, {"step", s}, {"update_norm", un}}.dump() << "\n";
        meta.step = s;
        meta.optimizer_t = tr.optimizer_t();
        if (s % cfg.strategy.interval != 0) continue;
        meta.checkpoint_counter = s / cfg.strategy.interval;
        std::vector<ModuleId> mods;
        if (!cfg.magnitude) {
            mods = modules_to_save(cfg.strategy, cfg.spec, meta.checkpoint_counter);
        } else if (meta.checkpoint_counter == 1) {
            mods = enumerate_modules(cfg.spec); // S_1 holds the complete state
        } else {
            const auto sums = tr.score_against_kept(); // r_k = score(S_{k-1} -> S_k), in situ
            std::vector<double> row(static_cast<std::size_t>(M));
            for (int m = 0; m < M; ++m) row[static_cast<std::size_t>(m)] = magnitude_score(sums[static_cast<std::size_t>(m)].first, sums[static_cast<std::size_t>(m)].second);
            const Selection sel = select_by_magnitude({row}, M, cfg.rho);
            for (int m : sel.saved[1]) mods.push_back(tr.model().modules()[static_cast<std::size_t>(m)]);
        }
        const fs::path dir = out_dir / dir_of_step(s);
        tr.save(dir, meta, mods, cfg.magnitude ? "magnitude" : strategy_kind_name(cfg.strategy.kind));
        if (cfg.magnitude) tr.keep_masters();
        saved.push_back(dir);
    }
    log.flush();
    if (!log) fail(ErrorKind::Storage, "log write failed");
    return saved;
}

std::vector<fs::path> device_resume(const fs::path& checkpoint_dir, std::int64_t additional_steps, const fs::path& out_dir,
                                    int device) {
    if (additional_steps < 0) fail(ErrorKind::Recipe, "additional_steps must be >= 0");
    // read_checkpoint: the full structural + payload verification, on the device
    verify_checkpoint_dir(checkpoint_dir.string(), device);
    const CheckpointSummary s = read_checkpoint_summary(checkpoint_dir);
    std::string missing;
    for (const auto& m : enumerate_modules(s.spec))
        if (!s.manifest.contains(m)) missing += (missing.empty() ? "" : ", ") + module_name(m);
    if (!missing.empty())
        fail(ErrorKind::MissingModules, "checkpoint '" + checkpoint_dir.string() + "' is partial (missing " + missing +
                                            "); assemble a complete checkpoint with the merge command first");
    if (s.trainer.rng_seed != s.spec.seed) fail(ErrorKind::Consistency, "trainer rng_seed disagrees with the model config seed");
    std::error_code ec;
    if (fs::exists(out_dir) && !fs::is_empty(out_dir, ec))
        fail(ErrorKind::Storage, "refusing to write into non-empty directory '" + out_dir.string() + "'");
    DeviceTrainer tr(s.spec, s.optim.num_ranks, AdamHyperparams{}, device);
    tr.load(checkpoint_dir, s);
    fs::create_directories(out_dir, ec);
    if (ec) fail(ErrorKind::Storage, "cannot create '" + out_dir.string() + "': " + ec.message());
    std::ofstream log(out_dir / "log.jsonl", std::ios::binary);
    if (!log) fail(ErrorKind::Storage, "cannot create log in '" + out_dir.string() + "'");
    TrainerMeta meta = s.trainer;
    const StrategyConfig strategy = s.trainer.strategy;
    std::vector<fs::path> saved;
    for (std::int64_t st = s.trainer.step + 1; st <= s.trainer.step + additional_steps; ++st) {
        const auto [gn, un] = tr.step(st);
        log << nlohmann::json{{"grad_norm", gn}, {"step", st}, {"update_norm", un}}.dump() << "\n";
        meta.step = st;
        meta.optimizer_t = tr.optimizer_t();
        if (st % strategy.interval != 0) continue;
        meta.checkpoint_counter = st / strategy.interval;
        const auto mods = modules_to_save(strategy, s.spec, meta.checkpoint_counter);
        const fs::path dir = out_dir / dir_of_step(st);
        tr.save(dir, meta, mods, strategy_kind_name(strategy.kind));
        saved.push_back(dir);
    }
    log.flush();
    if (!log) fail(ErrorKind::Storage, "log write failed");
    return saved;
}

} // namespace tailor
