// ref_tool — drives the REFERENCE tailor library (compiled from
// /root/reference/proj/src by oracle/Makefile) through its public C++ API.
//
// TEST INFRASTRUCTURE ONLY. This binary is the parity oracle and the
// reference arm of bench.py; nothing on the product path links or runs it.
//
// Subcommands (all print one JSON object on stdout; errors go to stderr as
// {"error": kind, "message": ...} with exit 1 = user error, 2 = internal,
// mirroring R/tools/tailor_main.cpp:351-357):
//
//   gen      synthetic snapshots S_1..S_K in reference format (write_checkpoint,
//            R/src/checkpoint.cpp:387-428) using the generator contract of
//            SURVEY.md §8(d) on reference primitives (unit_noise/mix64,
//            R/src/gradients.cpp:8-23; group_tensor_slices, R/src/groups.cpp:105-133)
//   merge    resolve_plan + execute_merge (R/src/merge.cpp:39-357) on a JSON recipe
//   plan     recipe_from_manifests (R/src/merge.cpp:359-418)
//   train    the reference toy trainer (R/src/trainer.cpp:109-123) + optional inject_failure
//   resume   resume from a complete checkpoint (R/src/trainer.cpp:125-152)
//   score    CPU restatement of the update-magnitude scorer and the
//            magnitude selection → recipe mapping (a14) over read_checkpoint output
//   select-merge   score → select → resolve_plan → execute_merge, timed (reference arm)
//   verify   verify_checkpoints (R/src/verify.cpp:46-112)
//   read     read_checkpoint (R/src/checkpoint.cpp:485-575) — full validation
//   regroup  read_checkpoint -> coarse_to_fine / fine_to_coarse -> write_checkpoint
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <iostream>
#include <map>
#include <mutex>
#include <optional>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "tailor/checkpoint.hpp"
#include "tailor/errors.hpp"
#include "tailor/gradients.hpp"
#include "tailor/groups.hpp"
#include "tailor/merge.hpp"
#include "tailor/model.hpp"
#include "tailor/trainer.hpp"
#include "tailor/verify.hpp"

using nlohmann::json;
using namespace tailor;
namespace fs = std::filesystem;

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// ---- argument parsing -------------------------------------------------------
struct Args {
    std::map<std::string, std::string> kv;
    std::set<std::string> flags;
    bool has(const std::string& k) const { return kv.count(k) || flags.count(k); }
    std::string str(const std::string& k, const std::string& d = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? d : it->second;
    }
    long long i64(const std::string& k, long long d) const {
        auto it = kv.find(k);
        return it == kv.end() ? d : std::stoll(it->second);
    }
    double f64(const std::string& k, double d) const {
        auto it = kv.find(k);
        return it == kv.end() ? d : std::stod(it->second);
    }
};

Args parse_args(int argc, char** argv, int first) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw std::runtime_error("unexpected argument " + k);
        k = k.substr(2);
        if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) a.kv[k] = argv[++i];
        else a.flags.insert(k);
    }
    return a;
}

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == sep) { out.push_back(cur); cur.clear(); }
        else cur.push_back(c);
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}

ModelSpec spec_from(const Args& a) {
    ModelSpec s;
    s.num_layers = static_cast<int>(a.i64("layers", 4));
    s.hidden_dim = static_cast<int>(a.i64("hidden", 8));
    s.ffn_dim = static_cast<int>(a.i64("ffn", 16));
    s.vocab_size = static_cast<int>(a.i64("vocab", 32));
    s.weight_tied = a.has("tied");
    s.seed = static_cast<std::uint64_t>(a.i64("seed", 42));
    s.validate();
    return s;
}

// ---- synthetic generator, restated on reference primitives -----
// hash3 is the three-round counter hash inside unit_noise (R/src/gradients.cpp:17-23).
std::uint64_t hash3(std::uint64_t seed, std::uint64_t t, std::uint64_t e) {
    std::uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ULL);
    h = mix64(h ^ (t * 0xD1B54A32D192ED03ULL));
    h = mix64(h ^ (e * 0x8CB92BA72F3D8DD7ULL));
    return h;
}
constexpr std::uint64_t kSignSalt = 0x51A7E5ULL;
constexpr std::uint64_t kMSalt = 0xA5ULL;
constexpr std::uint64_t kVSalt = 0x5AULL;
constexpr std::uint64_t kPermSalt = 0x9E2AULL;

// sigma_j(m) = 1e-6 * g^{pi_j(m)}, g = 1000^{1/(M-1)}, pi_j a seeded
// Fisher-Yates permutation of the canonical module indices.
std::vector<float> sigma_table(std::uint64_t seed, int M, int j) {
    std::vector<int> perm(static_cast<std::size_t>(M));
    for (int i = 0; i < M; ++i) perm[static_cast<std::size_t>(i)] = i;
    for (int i = M - 1; i >= 1; --i) {
        const std::uint64_t r = hash3(seed ^ kPermSalt, static_cast<std::uint64_t>(j), static_cast<std::uint64_t>(i));
        const int k = static_cast<int>(r % static_cast<std::uint64_t>(i + 1));
        std::swap(perm[static_cast<std::size_t>(i)], perm[static_cast<std::size_t>(k)]);
    }
    const double g = M > 1 ? std::pow(1000.0, 1.0 / static_cast<double>(M - 1)) : 1.0;
    std::vector<float> s(static_cast<std::size_t>(M));
    for (int m = 0; m < M; ++m)
        s[static_cast<std::size_t>(m)] = static_cast<float>(1e-6 * std::pow(g, static_cast<double>(perm[static_cast<std::size_t>(m)])));
    return s;
}

int canonical_index(const ModelSpec& spec, const ModuleId& m) {
    const auto mods = enumerate_modules(spec);
    for (std::size_t i = 0; i < mods.size(); ++i)
        if (mods[i] == m) return static_cast<int>(i);
    fail(ErrorKind::InvalidModule, "module not in spec");
}

// Writes snapshots k = 1..K at step k*interval into out/checkpoint-<step>.
// `partial[k]` (optional) restricts snapshot k's manifest to a module subset.
json cmd_gen(const Args& a) {
    const ModelSpec spec = spec_from(a);
    const int ranks = static_cast<int>(a.i64("ranks", 1));
    const int K = static_cast<int>(a.i64("snapshots", 2));
    const std::int64_t interval = a.i64("interval", 100);
    const fs::path out = a.str("out");
    std::map<int, std::vector<ModuleId>> partial;
    for (const auto& item : split(a.str("partial"), ';')) {
        auto eq = item.find('=');
        if (eq == std::string::npos) continue;
        std::vector<ModuleId> mods;
        for (const auto& n : split(item.substr(eq + 1), ',')) mods.push_back(parse_module_name(n));
        partial[std::stoi(item.substr(0, eq))] = mods;
    }

    const GroupTable table = build_group_table(spec);
    const int M = spec.module_count();
    AdamHyperparams base;
    base.weight_decay = kDefaultWeightDecay;
    OptimizerState state = zero_state(spec, table, base);
    // group -> owner module's canonical index
    std::vector<int> owner_index(static_cast<std::size_t>(table.group_count()));
    for (int g = 0; g < table.group_count(); ++g)
        owner_index[static_cast<std::size_t>(g)] = canonical_index(spec, *table.groups[static_cast<std::size_t>(g)].owner);
    // W_0 = 0.02 * u(seed, 0, e), exactly as init_state (R/src/gradients.cpp:51-66)
    for (int g = 0; g < table.group_count(); ++g) {
        auto& gs = state[static_cast<std::size_t>(g)];
        for (const auto& sl : group_tensor_slices(spec, table, g))
            for (std::int64_t i = 0; i < sl.decl.element_count(); ++i)
                gs.master[static_cast<std::size_t>(sl.group_offset + i)] =
                    0.02f * unit_noise(spec.seed, 0, sl.model_offset + i);
    }
    json dirs = json::array();
    fs::create_directories(out);
    for (int k = 1; k <= K; ++k) {
        const auto sig = sigma_table(spec.seed, M, k);
        for (int g = 0; g < table.group_count(); ++g) {
            auto& gs = state[static_cast<std::size_t>(g)];
            const float sigma = sig[static_cast<std::size_t>(owner_index[static_cast<std::size_t>(g)])];
            for (const auto& sl : group_tensor_slices(spec, table, g)) {
                for (std::int64_t i = 0; i < sl.decl.element_count(); ++i) {
                    const auto at = static_cast<std::size_t>(sl.group_offset + i);
                    const auto e = static_cast<std::uint64_t>(sl.model_offset + i);
                    const bool neg = (hash3(spec.seed ^ kSignSalt, static_cast<std::uint64_t>(k), e) >> 63) != 0;
                    gs.master[at] = gs.master[at] + (neg ? -sigma : sigma);
                    gs.exp_avg[at] = 0.1f * unit_noise(spec.seed ^ kMSalt, k, static_cast<std::int64_t>(e));
                    gs.exp_avg_sq[at] = std::fabs(0.01f * unit_noise(spec.seed ^ kVSalt, k, static_cast<std::int64_t>(e)));
                }
            }
        }
        const std::int64_t step = k * interval;
        CheckpointData data;
        data.spec = spec;
        data.trainer.step = step;
        data.trainer.optimizer_t = step;
        data.trainer.strategy.interval = static_cast<int>(interval);
        data.trainer.checkpoint_counter = k;
        data.trainer.rng_seed = spec.seed;
        data.manifest.step = step;
        data.manifest.strategy = partial.count(k) ? "manual" : "full";
        data.manifest.modules = partial.count(k) ? partial.at(k) : enumerate_modules(spec);
        data.table = table;
        data.num_ranks = ranks;
        for (int g : group_indices_for_modules(table, data.manifest.modules))
            data.groups.emplace(g, state[static_cast<std::size_t>(g)]);
        data.weights = derive_weights(spec, table, data.groups, data.manifest.modules);
        const fs::path dir = out / checkpoint_dir_name(step);
        write_checkpoint(dir, data);
        dirs.push_back(dir.string());
    }
    return {{"snapshots", dirs}};
}

// ---- recipes as JSON (yaml-cpp is absent) -----------------------------------
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

json recipe_to_json(const MergeRecipe& r) {
    json slices = json::array();
    for (const auto& s : r.slices) slices.push_back({{"source", s.source}, {"layers", s.layers}, {"targets", s.targets}});
    json aux = json::object();
    for (const auto& [k, v] : r.aux) aux[k] = v;
    return {{"base_checkpoint", r.base_checkpoint}, {"num_ranks", r.num_ranks}, {"slices", slices},
            {"aux", aux}, {"config_from", r.config_from}};
}

json plan_to_json(const MergePlan& p) {
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

json run_merge(const MergeRecipe& recipe, const Args& a) {
    const auto t0 = Clock::now();
    const MergePlan plan = resolve_plan(recipe);
    const double plan_ms = ms_since(t0);
    MergeOptions opt;
    opt.workers = static_cast<int>(a.i64("workers", 0));
    opt.uncached = a.has("uncached");
    const MergeStats st = execute_merge(plan, a.str("out"), opt);
    return {{"plan", plan_to_json(plan)},
            {"stats", {{"shard_files_read", st.shard_files_read}, {"weight_files_read", st.weight_files_read},
                       {"wall_ms", st.wall_ms}, {"plan_ms", plan_ms}}}};
}

json cmd_merge(const Args& a) {
    const auto bytes = read_file_bytes(a.str("recipe"));
    return run_merge(recipe_from_json(json::parse(bytes.begin(), bytes.end())), a);
}

json cmd_resolve(const Args& a) {
    const auto bytes = read_file_bytes(a.str("recipe"));
    return {{"plan", plan_to_json(resolve_plan(recipe_from_json(json::parse(bytes.begin(), bytes.end()))))}};
}

json cmd_plan(const Args& a) {
    return {{"recipe", recipe_to_json(recipe_from_manifests(a.str("run"), a.i64("failure-step", 0)))}};
}

// resume (R/src/trainer.cpp:125-152): continue a complete checkpoint for --steps steps.
json cmd_resume(const Args& a) {
    const TrainResult res = resume(a.str("ckpt"), static_cast<int>(a.i64("steps", 0)), a.str("out"));
    json cks = json::array();
    for (const auto& c : res.checkpoints) cks.push_back(c.string());
    return {{"checkpoints", cks}, {"step", res.meta.step}};
}

json cmd_train(const Args& a) {
    TrainRunConfig cfg;
    cfg.spec = spec_from(a);
    cfg.strategy.kind = parse_strategy_kind(a.str("strategy", "full"));
    cfg.strategy.interval = static_cast<int>(a.i64("interval", 50));
    cfg.strategy.head_count = static_cast<int>(a.i64("head", 2));
    cfg.strategy.tail_count = static_cast<int>(a.i64("tail", 2));
    cfg.strategy.sparse_multiple = static_cast<int>(a.i64("sparse-multiple", 5));
    cfg.total_steps = static_cast<int>(a.i64("steps", 100));
    cfg.num_ranks = static_cast<int>(a.i64("ranks", 1));
    cfg.grouping = a.str("grouping", "fine") == "coarse" ? Grouping::Coarse : Grouping::Fine;
    cfg.hyper.lr = a.f64("lr", kDefaultLr);
    cfg.hyper.weight_decay = a.f64("weight-decay", kDefaultWeightDecay);
    const TrainResult res = train(cfg, a.str("out"));
    if (a.has("fail-at")) inject_failure(a.str("out"), a.i64("fail-at", 0));
    json cks = json::array();
    for (const auto& c : list_checkpoints(a.str("out"))) cks.push_back(c.string());
    return {{"checkpoints", cks}};
}

// ---- scorer + selection restatement ---------------------
struct ScoreResult {
    std::vector<std::vector<double>> sd, sr, score; // [pair][module]
};

// Sequential FP64 over canonical element order: each module's groups in
// group_indices_for order (R/src/groups.cpp:84-103), true_length only.
ScoreResult score_snapshots(const std::vector<CheckpointData>& snaps) {
    const ModelSpec& spec = snaps.front().spec;
    const auto mods = enumerate_modules(spec);
    const GroupTable table = build_group_table(spec);
    ScoreResult r;
    for (std::size_t k = 1; k < snaps.size(); ++k) {
        std::vector<double> sd(mods.size()), sr(mods.size()), sc(mods.size());
        for (std::size_t m = 0; m < mods.size(); ++m) {
            double d2 = 0.0, r2 = 0.0;
            for (int g : group_indices_for(table, mods[m])) {
                const auto& A = snaps[k - 1].groups.at(g).master;
                const auto& B = snaps[k].groups.at(g).master;
                for (std::size_t i = 0; i < A.size(); ++i) {
                    const double d = static_cast<double>(B[i]) - static_cast<double>(A[i]);
                    d2 += d * d;
                    r2 += static_cast<double>(A[i]) * static_cast<double>(A[i]);
                }
            }
            sd[m] = d2;
            sr[m] = r2;
            sc[m] = r2 > 0.0 ? std::sqrt(d2) / std::sqrt(r2) : (d2 > 0.0 ? INFINITY : 0.0);
        }
        r.sd.push_back(sd);
        r.sr.push_back(sr);
        r.score.push_back(sc);
    }
    return r;
}

// saved_1 = all; saved_k = top-ceil(rho*M) by r_k, ties -> lower canonical index.
std::vector<std::vector<int>> select_modules(const ScoreResult& s, int M, double rho, double* min_gap) {
    std::vector<std::vector<int>> saved;
    std::vector<int> all(static_cast<std::size_t>(M));
    for (int i = 0; i < M; ++i) all[static_cast<std::size_t>(i)] = i;
    saved.push_back(all);
    int n = static_cast<int>(std::ceil(rho * M));
    n = std::max(1, std::min(M, n));
    *min_gap = INFINITY;
    for (const auto& sc : s.score) {
        std::vector<int> order = all;
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
            return sc[static_cast<std::size_t>(x)] > sc[static_cast<std::size_t>(y)];
        });
        if (n < M) {
            const double hi = sc[static_cast<std::size_t>(order[static_cast<std::size_t>(n - 1)])];
            const double lo = sc[static_cast<std::size_t>(order[static_cast<std::size_t>(n)])];
            *min_gap = std::min(*min_gap, (hi - lo) / hi);
        }
        std::vector<int> pick(order.begin(), order.begin() + n);
        std::sort(pick.begin(), pick.end());
        saved.push_back(pick);
    }
    return saved;
}

// The latest-version rule of recipe_from_manifests (R/src/merge.cpp:375-417)
// applied to the selected module sets instead of on-disk manifests.
MergeRecipe recipe_from_selection(const std::vector<CheckpointSummary>& snaps,
                                  const std::vector<std::vector<int>>& saved) {
    const ModelSpec& spec = snaps.front().spec;
    const auto mods = enumerate_modules(spec);
    auto newer = [](const CheckpointSummary& a, const CheckpointSummary& b) {
        return a.trainer.step != b.trainer.step ? a.trainer.step > b.trainer.step : a.dir.string() > b.dir.string();
    };
    const CheckpointSummary* latest = &snaps.front();
    for (const auto& s : snaps)
        if (newer(s, *latest)) latest = &s;
    std::map<ModuleId, const CheckpointSummary*> chosen;
    for (std::size_t m = 0; m < mods.size(); ++m) {
        const CheckpointSummary* best = nullptr;
        for (std::size_t k = 0; k < snaps.size(); ++k) {
            const auto& set = saved[k];
            if (std::find(set.begin(), set.end(), static_cast<int>(m)) == set.end()) continue;
            if (!best || newer(snaps[k], *best)) best = &snaps[k];
        }
        chosen[mods[m]] = best;
    }
    MergeRecipe recipe;
    recipe.num_ranks = latest->optim.num_ranks;
    recipe.base_checkpoint = latest->dir.string();
    recipe.config_from = latest->dir.string();
    std::map<std::string, std::vector<int>> layer_slices;
    for (const auto& [m, s] : chosen) {
        if (s == latest) continue;
        if (m.kind == ModuleKind::TransformerLayer) layer_slices[s->dir.string()].push_back(m.layer);
        else recipe.aux[module_name(m)] = s->dir.string();
    }
    for (auto& [src, layers] : layer_slices) {
        std::sort(layers.begin(), layers.end());
        recipe.slices.push_back({src, layers, layers});
    }
    return recipe;
}

json score_and_select(const Args& a, MergeRecipe* recipe_out, double* score_ms) {
    const auto t0 = Clock::now();
    // Snapshots are independent: each is read (read_checkpoint, full validation) on its
    // own thread, as the reference's ShardLoader spreads file loads over std::threads
    // (R/src/merge.cpp:157-205); the first error is rethrown after the join.
    const auto paths = split(a.str("snapshots"), ',');
    std::vector<CheckpointData> snaps(paths.size());
    std::vector<CheckpointSummary> sums(paths.size());
    {
        std::exception_ptr err;
        std::mutex mu;
        std::vector<std::thread> pool;
        for (std::size_t i = 0; i < paths.size(); ++i)
            pool.emplace_back([&, i] {
                try {
                    snaps[i] = read_checkpoint(paths[i]);
                    sums[i] = read_checkpoint_summary(paths[i]);
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!err) err = std::current_exception();
                }
            });
        for (auto& th : pool) th.join();
        if (err) std::rethrow_exception(err);
    }
    if (snaps.size() < 2) fail(ErrorKind::Recipe, "scoring needs at least two snapshots");
    const ScoreResult sr = score_snapshots(snaps);
    const int M = snaps.front().spec.module_count();
    double gap = 0.0;
    const auto saved = select_modules(sr, M, a.f64("rho", 0.5), &gap);
    const MergeRecipe recipe = recipe_from_selection(sums, saved);
    *score_ms = ms_since(t0);
    if (recipe_out) *recipe_out = recipe;
    json saved_j = json::array();
    const auto mods = enumerate_modules(snaps.front().spec);
    for (const auto& s : saved) {
        json names = json::array();
        for (int m : s) names.push_back(module_name(mods[static_cast<std::size_t>(m)]));
        saved_j.push_back(names);
    }
    return {{"sum_delta_sq", sr.sd}, {"sum_ref_sq", sr.sr}, {"scores", sr.score}, {"saved", saved_j},
            {"min_boundary_gap", std::isfinite(gap) ? json(gap) : json(nullptr)},
            {"recipe", recipe_to_json(recipe)}, {"score_ms", *score_ms}};
}

json cmd_score(const Args& a) {
    double ms = 0.0;
    return score_and_select(a, nullptr, &ms);
}

json cmd_select_merge(const Args& a) {
    MergeRecipe recipe;
    double score_ms = 0.0;
    json j = score_and_select(a, &recipe, &score_ms);
    json m = run_merge(recipe, a);
    j["merge"] = m;
    j["total_ms"] = score_ms + m["stats"]["plan_ms"].get<double>() + m["stats"]["wall_ms"].get<double>();
    return j;
}

json cmd_verify(const Args& a) {
    std::optional<std::vector<ModuleId>> mods;
    if (a.has("modules")) {
        mods.emplace();
        for (const auto& n : split(a.str("modules"), ',')) mods->push_back(parse_module_name(n));
    }
    const VerifyResult r = verify_checkpoints(a.str("a"), a.str("b"), mods);
    return {{"equal", r.equal}, {"first_divergence", r.first_divergence}};
}

// Regroup a checkpoint directory with reference primitives only:
// read_checkpoint -> coarse_to_fine / fine_to_coarse (R/src/groups.cpp:212-220)
// -> write_checkpoint (R/src/checkpoint.cpp:387-428).
json cmd_regroup(const Args& a) {
    CheckpointData d = read_checkpoint(a.str("dir"));
    const bool to_fine = a.str("to", "fine") == "fine";
    const GroupTable fine = build_group_table(d.spec);
    OptimizerState src;
    for (int g = 0; g < d.table.group_count(); ++g) src.push_back(d.groups.at(g));
    OptimizerState dst = to_fine ? coarse_to_fine(d.spec, src, fine) : fine_to_coarse(d.spec, src, fine);
    d.table = to_fine ? fine : build_coarse_table(d.spec);
    d.groups.clear();
    for (int g = 0; g < d.table.group_count(); ++g) d.groups.emplace(g, dst[static_cast<std::size_t>(g)]);
    write_checkpoint(a.str("out"), d);
    return {{"groups", d.table.group_count()}};
}

json cmd_read(const Args& a) {
    const CheckpointData d = read_checkpoint(a.str("dir"));
    return {{"ok", true}, {"groups", d.groups.size()}, {"tensors", d.weights.tensors.size()}};
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: ref_tool <gen|merge|resolve|plan|train|resume|score|select-merge|verify|read|regroup> [--k v ...]\n";
        return 1;
    }
    const std::string cmd = argv[1];
    try {
        const Args a = parse_args(argc, argv, 2);
        json out;
        if (cmd == "gen") out = cmd_gen(a);
        else if (cmd == "merge") out = cmd_merge(a);
        else if (cmd == "resolve") out = cmd_resolve(a);
        else if (cmd == "plan") out = cmd_plan(a);
        else if (cmd == "train") out = cmd_train(a);
        else if (cmd == "resume") out = cmd_resume(a);
        else if (cmd == "score") out = cmd_score(a);
        else if (cmd == "select-merge") out = cmd_select_merge(a);
        else if (cmd == "verify") out = cmd_verify(a);
        else if (cmd == "read") out = cmd_read(a);
        else if (cmd == "regroup") out = cmd_regroup(a);
        else {
            std::cerr << "unknown subcommand " << cmd << "\n";
            return 1;
        }
        std::cout << out.dump() << "\n";
        return 0;
    } catch (const TailorError& e) {
        std::cerr << json{{"error", error_kind_name(e.kind())}, {"message", e.what()}}.dump() << "\n";
        return e.is_user_error() ? 1 : 2;
    } catch (const std::exception& e) {
        std::cerr << json{{"error", "internal"}, {"message", e.what()}}.dump() << "\n";
        return 2;
    }
}
