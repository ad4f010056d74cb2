// Checkpoint sidecars, summaries and payload layouts (see tailor/checkpoint.hpp).
#include "tailor/checkpoint.hpp"

#include <algorithm>
#include <charconv>
#include <fstream>
#include <set>

#include <json.hpp>

#include "tailor/errors.hpp"

namespace tailor {

using nlohmann::json;
namespace fs = std::filesystem;

std::string strategy_kind_name(StrategyKind kind) {
    switch (kind) {
        case StrategyKind::Full: return "full";
        case StrategyKind::Parity: return "parity";
        case StrategyKind::Filter: return "filter";
    }
    fail(ErrorKind::Consistency, "unknown strategy kind");
}

StrategyKind parse_strategy_kind(const std::string& name) {
    if (name == "full") return StrategyKind::Full;
    if (name == "parity") return StrategyKind::Parity;
    if (name == "filter") return StrategyKind::Filter;
    fail(ErrorKind::Recipe, "unknown strategy '" + name + "' (expected full, parity or filter)");
}

bool SaveManifest::contains(const ModuleId& m) const {
    return std::find(modules.begin(), modules.end(), m) != modules.end();
}

const OptimGroupMeta* OptimMeta::find(int index) const {
    for (const auto& g : groups)
        if (g.index == index) return &g;
    return nullptr;
}

std::string dir_of_step(std::int64_t step) { return "checkpoint-" + std::to_string(step); }

std::optional<std::int64_t> step_of_dir(const std::string& name) {
    static const std::string kPrefix = "checkpoint-";
    if (name.compare(0, kPrefix.size(), kPrefix) != 0) return std::nullopt;
    std::int64_t step = -1;
    const char* b = name.data() + kPrefix.size();
    const char* e = name.data() + name.size();
    const auto r = std::from_chars(b, e, step);
    if (r.ec != std::errc() || r.ptr != e || step < 0) return std::nullopt;
    return step;
}

fs::path ckpt_file(CkptFile kind, const fs::path& dir, int rank) {
    switch (kind) {
    case CkptFile::Weights: return dir / "model.weights";
    case CkptFile::Shard: return dir / "optim" / ("rank_" + std::to_string(rank) + ".shard");
    case CkptFile::OptimMeta: return dir / "optim_meta.json";
    case CkptFile::Config: return dir / "config.json";
    case CkptFile::TrainerState: return dir / "trainer_state.json";
    case CkptFile::Manifest: return dir / "manifest.json";
    }
    fail(ErrorKind::Consistency, "unknown checkpoint file kind");
}

std::string read_text_file(const fs::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(ErrorKind::MissingArtifact, "cannot open '" + path.string() + "'");
    std::string s((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (in.bad()) fail(ErrorKind::Storage, "read failed for '" + path.string() + "'");
    return s;
}

void write_text_file(const fs::path& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(ErrorKind::Storage, "cannot create '" + path.string() + "'");
    out.write(text.data(), static_cast<std::streamsize>(text.size()));
    out.flush();
    if (!out) fail(ErrorKind::Storage, "write failed for '" + path.string() + "'");
}

namespace {

std::string pretty(const json& j) { return j.dump(2) + "\n"; }

json parse_json(const std::string& text, const std::string& origin) {
    try {
        return json::parse(text);
    } catch (const json::exception& e) {
        fail(ErrorKind::CorruptContainer, origin + ": invalid JSON (" + e.what() + ")");
    }
}

void exact_keys(const json& j, std::initializer_list<const char*> required, std::initializer_list<const char*> optional,
                const std::string& origin) {
    if (!j.is_object()) fail(ErrorKind::CorruptContainer, origin + ": expected a JSON object");
    std::set<std::string> req(required.begin(), required.end()), opt(optional.begin(), optional.end());
    for (const auto& [k, v] : j.items())
        if (!req.count(k) && !opt.count(k)) fail(ErrorKind::CorruptContainer, origin + ": unexpected key '" + k + "'");
    for (const auto& k : req)
        if (!j.contains(k)) fail(ErrorKind::CorruptContainer, origin + ": missing key '" + k + "'");
}

const char* decay_text(DecayClass d) { return d == DecayClass::Decay ? "decay" : "no_decay"; }

DecayClass decay_from(const std::string& s, const std::string& origin) {
    if (s == "decay") return DecayClass::Decay;
    if (s == "no_decay") return DecayClass::NoDecay;
    fail(ErrorKind::CorruptContainer, origin + ": unknown decay class '" + s + "'");
}

} // namespace

std::string sidecar_text(const ModelSpec& s) {
    json j = json::object();
    j["num_layers"] = s.num_layers;
    j["hidden_dim"] = s.hidden_dim;
    j["ffn_dim"] = s.ffn_dim;
    j["vocab_size"] = s.vocab_size;
    j["weight_tied"] = s.weight_tied;
    j["seed"] = s.seed;
    return pretty(j);
}

template <>
ModelSpec sidecar_value<ModelSpec>(const std::string& text, const std::string& origin) {
    const json j = parse_json(text, origin);
    exact_keys(j, {"num_layers", "hidden_dim", "ffn_dim", "vocab_size", "weight_tied", "seed"}, {}, origin);
    ModelSpec s;
    s.num_layers = j.at("num_layers").get<int>();
    s.hidden_dim = j.at("hidden_dim").get<int>();
    s.ffn_dim = j.at("ffn_dim").get<int>();
    s.vocab_size = j.at("vocab_size").get<int>();
    s.weight_tied = j.at("weight_tied").get<bool>();
    s.seed = j.at("seed").get<std::uint64_t>();
    s.validate();
    return s;
}

std::string sidecar_text(const TrainerMeta& m) {
    json strat = json::object();
    strat["kind"] = strategy_kind_name(m.strategy.kind);
    strat["interval"] = m.strategy.interval;
    if (m.strategy.kind == StrategyKind::Filter) {
        strat["head_count"] = m.strategy.head_count;
        strat["tail_count"] = m.strategy.tail_count;
        strat["sparse_multiple"] = m.strategy.sparse_multiple;
    }
    json j = json::object();
    j["step"] = m.step;
    j["lr"] = m.lr;
    j["optimizer_t"] = m.optimizer_t;
    j["strategy"] = std::move(strat);
    j["checkpoint_counter"] = m.checkpoint_counter;
    j["rng_seed"] = m.rng_seed;
    return pretty(j);
}

template <>
TrainerMeta sidecar_value<TrainerMeta>(const std::string& text, const std::string& origin) {
    const json j = parse_json(text, origin);
    exact_keys(j, {"step", "lr", "optimizer_t", "strategy", "checkpoint_counter", "rng_seed"}, {}, origin);
    TrainerMeta m;
    m.step = j.at("step").get<std::int64_t>();
    m.lr = j.at("lr").get<double>();
    m.optimizer_t = j.at("optimizer_t").get<std::int64_t>();
    const json& s = j.at("strategy");
    exact_keys(s, {"kind", "interval"}, {"head_count", "tail_count", "sparse_multiple"}, origin + ": strategy");
    m.strategy.kind = parse_strategy_kind(s.at("kind").get<std::string>());
    m.strategy.interval = s.at("interval").get<int>();
    if (s.contains("head_count")) m.strategy.head_count = s.at("head_count").get<int>();
    if (s.contains("tail_count")) m.strategy.tail_count = s.at("tail_count").get<int>();
    if (s.contains("sparse_multiple")) m.strategy.sparse_multiple = s.at("sparse_multiple").get<int>();
    m.checkpoint_counter = j.at("checkpoint_counter").get<std::int64_t>();
    m.rng_seed = j.at("rng_seed").get<std::uint64_t>();
    return m;
}

std::string sidecar_text(const SaveManifest& man) {
    json mods = json::array();
    for (const auto& m : man.modules) mods.push_back(module_name(m));
    json j = json::object();
    j["step"] = man.step;
    j["strategy"] = man.strategy;
    j["modules"] = std::move(mods);
    if (!man.provenance.empty()) {
        json prov = json::object();
        for (const auto& [name, p] : man.provenance) {
            json e = json::object();
            e["source"] = p.source;
            e["step"] = p.step;
            prov[name] = std::move(e);
        }
        j["provenance"] = std::move(prov);
    }
    return pretty(j);
}

template <>
SaveManifest sidecar_value<SaveManifest>(const std::string& text, const std::string& origin) {
    const json j = parse_json(text, origin);
    exact_keys(j, {"step", "strategy", "modules"}, {"provenance"}, origin);
    SaveManifest man;
    man.step = j.at("step").get<std::int64_t>();
    man.strategy = j.at("strategy").get<std::string>();
    for (const auto& n : j.at("modules")) man.modules.push_back(parse_module_name(n.get<std::string>()));
    if (man.modules.empty()) fail(ErrorKind::CorruptContainer, origin + ": empty module list");
    if (j.contains("provenance"))
        for (const auto& [name, p] : j.at("provenance").items()) {
            exact_keys(p, {"source", "step"}, {}, origin + ": provenance." + name);
            man.provenance[name] = {p.at("source").get<std::string>(), p.at("step").get<std::int64_t>()};
        }
    return man;
}

std::string sidecar_text(const OptimMeta& meta) {
    json groups = json::array();
    for (const auto& g : meta.groups) {
        json e = json::object();
        e["index"] = g.index;
        e["owner"] = g.owner;
        e["decay"] = decay_text(g.decay);
        e["true_length"] = g.true_length;
        e["padded_length"] = g.padded_length;
        e["shard_length"] = g.shard_length;
        e["lr"] = g.hyper.lr;
        e["beta1"] = g.hyper.beta1;
        e["beta2"] = g.hyper.beta2;
        e["eps"] = g.hyper.eps;
        e["weight_decay"] = g.hyper.weight_decay;
        groups.push_back(std::move(e));
    }
    json j = json::object();
    j["grouping"] = meta.grouping == Grouping::Fine ? "fine" : "coarse";
    j["num_ranks"] = meta.num_ranks;
    j["step"] = meta.step;
    j["groups"] = std::move(groups);
    return pretty(j);
}

template <>
OptimMeta sidecar_value<OptimMeta>(const std::string& text, const std::string& origin) {
    const json j = parse_json(text, origin);
    exact_keys(j, {"grouping", "num_ranks", "step", "groups"}, {}, origin);
    OptimMeta meta;
    const std::string grouping = j.at("grouping").get<std::string>();
    if (grouping == "fine") meta.grouping = Grouping::Fine;
    else if (grouping == "coarse") meta.grouping = Grouping::Coarse;
    else fail(ErrorKind::CorruptContainer, origin + ": unknown grouping '" + grouping + "'");
    meta.num_ranks = j.at("num_ranks").get<int>();
    meta.step = j.at("step").get<std::int64_t>();
    for (const auto& g : j.at("groups")) {
        exact_keys(g, {"index", "owner", "decay", "true_length", "padded_length", "shard_length", "lr", "beta1", "beta2",
                       "eps", "weight_decay"},
                   {}, origin + ": groups[]");
        OptimGroupMeta m;
        m.index = g.at("index").get<int>();
        m.owner = g.at("owner").get<std::string>();
        m.decay = decay_from(g.at("decay").get<std::string>(), origin);
        m.true_length = g.at("true_length").get<std::int64_t>();
        m.padded_length = g.at("padded_length").get<std::int64_t>();
        m.shard_length = g.at("shard_length").get<std::int64_t>();
        m.hyper.lr = g.at("lr").get<double>();
        m.hyper.beta1 = g.at("beta1").get<double>();
        m.hyper.beta2 = g.at("beta2").get<double>();
        m.hyper.eps = g.at("eps").get<double>();
        m.hyper.weight_decay = g.at("weight_decay").get<double>();
        meta.groups.push_back(std::move(m));
    }
    std::sort(meta.groups.begin(), meta.groups.end(), [](const auto& a, const auto& b) { return a.index < b.index; });
    return meta;
}

OptimMeta make_optim_meta(const GroupTable& table, const std::map<int, AdamHyperparams>& groups,
                          const ShardGeometry& geom, std::int64_t step) {
    OptimMeta meta;
    meta.grouping = table.grouping;
    meta.num_ranks = geom.num_ranks;
    meta.step = step;
    for (const auto& [idx, hyper] : groups) {
        if (idx < 0 || idx >= table.group_count()) fail(ErrorKind::Geometry, "group index out of range: " + std::to_string(idx));
        const GroupInfo& info = table.groups[static_cast<std::size_t>(idx)];
        OptimGroupMeta m;
        m.index = idx;
        m.owner = info.owner ? module_name(*info.owner) : "coarse";
        m.decay = info.decay;
        m.true_length = info.element_count;
        m.padded_length = geom.padded_length(info.element_count);
        m.shard_length = geom.shard_length(info.element_count);
        m.hyper = hyper;
        meta.groups.push_back(std::move(m));
    }
    return meta;
}

CheckpointSummary read_checkpoint_summary(const fs::path& dir) {
    if (!fs::exists(dir)) fail(ErrorKind::MissingArtifact, "checkpoint directory '" + dir.string() + "' does not exist");
    CheckpointSummary s;
    s.dir = dir;
    auto load = [&dir]<class T>(CkptFile kind, T& out) {
        const fs::path f = ckpt_file(kind, dir);
        out = sidecar_value<T>(read_text_file(f), f.string());
    };
    load(CkptFile::Config, s.spec);
    load(CkptFile::TrainerState, s.trainer);
    load(CkptFile::Manifest, s.manifest);
    load(CkptFile::OptimMeta, s.optim);
    const std::string d = dir.string();
    if (s.manifest.step != s.trainer.step) fail(ErrorKind::Consistency, d + ": manifest step disagrees with trainer state");
    if (s.optim.step != s.trainer.optimizer_t) fail(ErrorKind::Consistency, d + ": optim_meta step disagrees with trainer state");
    if (s.optim.num_ranks < 1) fail(ErrorKind::Geometry, d + ": invalid rank count");
    for (const auto& m : s.manifest.modules)
        if (!module_valid(s.spec, m))
            fail(ErrorKind::Geometry, d + ": manifest names module '" + module_name(m) + "' not in the model");
    const GroupTable table = s.optim.grouping == Grouping::Fine ? build_group_table(s.spec) : build_coarse_table(s.spec);
    const ShardGeometry geom{s.optim.num_ranks};
    const auto required = group_indices_for_modules(table, s.manifest.modules);
    if (s.optim.groups.size() != required.size())
        fail(ErrorKind::Geometry, d + ": optim_meta group set does not match the manifest");
    for (std::size_t i = 0; i < required.size(); ++i) {
        const OptimGroupMeta& g = s.optim.groups[i];
        if (g.index != required[i]) fail(ErrorKind::Geometry, d + ": optim_meta group set does not match the manifest");
        const GroupInfo& info = table.groups[static_cast<std::size_t>(g.index)];
        const std::string owner = info.owner ? module_name(*info.owner) : "coarse";
        if (g.owner != owner || g.decay != info.decay || g.true_length != info.element_count)
            fail(ErrorKind::Geometry, d + ": group " + std::to_string(g.index) + " metadata does not match the model spec");
        if (g.padded_length != geom.padded_length(g.true_length) || g.shard_length != geom.shard_length(g.true_length))
            fail(ErrorKind::Geometry, d + ": group " + std::to_string(g.index) + " sharding lengths do not match the rank count");
        g.hyper.validate();
    }
    return s;
}

std::string shard_key(int group, const char* field) { return "g" + std::to_string(group) + field; }

CheckpointLayout checkpoint_layout(const ModelLayout& model, int num_ranks, const std::vector<ModuleId>& modules) {
    CheckpointLayout c;
    c.spec = model.spec();
    c.num_ranks = num_ranks;
    c.modules = modules;
    c.groups = group_indices_for_modules(model.table(), modules);
    const ShardGeometry geom{num_ranks};
    std::vector<EntryDecl> shard_decls;
    for (int g : c.groups) {
        const std::int64_t chunk = geom.shard_length(model.table().groups[static_cast<std::size_t>(g)].element_count);
        for (const char* f : {".exp_avg", ".exp_avg_sq", ".master"}) shard_decls.push_back({shard_key(g, f), Dtype::F32, {chunk}});
    }
    for (int r = 0; r < num_ranks; ++r)
        c.shards.push_back(layout_for(shard_decls, {{"num_ranks", std::to_string(num_ranks)}, {"rank", std::to_string(r)}}));
    std::vector<EntryDecl> wdecls;
    for (const auto& m : modules)
        for (const auto& t : tensors_of(model.spec(), m)) wdecls.push_back({t.name, Dtype::BF16, t.shape});
    c.weights = layout_for(std::move(wdecls));
    return c;
}

} // namespace tailor
