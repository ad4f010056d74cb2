// Layer map implementation. Semantics follow R/src/model.cpp:22-132,
// R/src/groups.cpp:40-133 and R/src/shard.cpp:10-19; see tailor/model.hpp.
#include "tailor/model.hpp"

#include <algorithm>
#include <charconv>
#include <set>

#include "tailor/errors.hpp"

namespace tailor {

const char* error_kind_name(ErrorKind kind) {
    switch (kind) {
        case ErrorKind::InvalidModule: return "InvalidModule";
        case ErrorKind::Geometry: return "GeometryError";
        case ErrorKind::NonFinite: return "NonFiniteError";
        case ErrorKind::Recipe: return "RecipeError";
        case ErrorKind::SourceLacksModule: return "SourceLacksModule";
        case ErrorKind::MissingArtifact: return "MissingArtifact";
        case ErrorKind::CorruptContainer: return "CorruptContainer";
        case ErrorKind::UnrecoverableModule: return "UnrecoverableModule";
        case ErrorKind::MissingModules: return "MissingModules";
        case ErrorKind::Consistency: return "ConsistencyError";
        case ErrorKind::Storage: return "StorageError";
        case ErrorKind::Device: return "DeviceError";
    }
    return "UnknownError";
}

void fail(ErrorKind kind, const std::string& message) { throw TailorError(kind, message); }

void ModelSpec::validate() const {
    if (num_layers < 1) fail(ErrorKind::Geometry, "num_layers must be >= 1");
    if (hidden_dim < 1 || ffn_dim < 1 || vocab_size < 1)
        fail(ErrorKind::Geometry, "all model dimensions must be >= 1");
}

std::string module_name(const ModuleId& m) {
    switch (m.kind) {
        case ModuleKind::EmbedTokens: return "embed_tokens";
        case ModuleKind::Norm: return "norm";
        case ModuleKind::LmHead: return "lm_head";
        case ModuleKind::TransformerLayer: return "layers." + std::to_string(m.layer);
    }
    fail(ErrorKind::InvalidModule, "unknown module kind");
}

ModuleId parse_module_name(const std::string& name) {
    static const std::string kLayerPrefix = "layers.";
    if (name == "embed_tokens") return ModuleId::embed_tokens();
    if (name == "norm") return ModuleId::norm();
    if (name == "lm_head") return ModuleId::lm_head();
    if (name.size() > kLayerPrefix.size() && name.compare(0, kLayerPrefix.size(), kLayerPrefix) == 0) {
        int idx = -1;
        const char* b = name.data() + kLayerPrefix.size();
        const char* e = name.data() + name.size();
        const auto res = std::from_chars(b, e, idx);
        if (res.ec == std::errc() && res.ptr == e && idx >= 0) return ModuleId::transformer_layer(idx);
    }
    fail(ErrorKind::InvalidModule, "unrecognized module name '" + name + "'");
}

bool module_valid(const ModelSpec& spec, const ModuleId& m) {
    if (m.kind == ModuleKind::TransformerLayer) return m.layer >= 0 && m.layer < spec.num_layers;
    if (m.kind == ModuleKind::LmHead) return !spec.weight_tied;
    return true;
}

std::vector<ModuleId> enumerate_modules(const ModelSpec& spec) {
    spec.validate();
    std::vector<ModuleId> out;
    out.reserve(static_cast<std::size_t>(spec.module_count()));
    out.push_back(ModuleId::embed_tokens());
    for (int i = 0; i < spec.num_layers; ++i) out.push_back(ModuleId::transformer_layer(i));
    out.push_back(ModuleId::norm());
    if (!spec.weight_tied) out.push_back(ModuleId::lm_head());
    return out;
}

int canonical_index(const ModelSpec& spec, const ModuleId& m) {
    if (!module_valid(spec, m)) fail(ErrorKind::InvalidModule, "module '" + module_name(m) + "' is not in the model");
    switch (m.kind) {
        case ModuleKind::EmbedTokens: return 0;
        case ModuleKind::TransformerLayer: return 1 + m.layer;
        case ModuleKind::Norm: return 1 + spec.num_layers;
        case ModuleKind::LmHead: return 2 + spec.num_layers;
    }
    return -1;
}

std::vector<TensorDecl> tensors_of(const ModelSpec& spec, const ModuleId& m) {
    spec.validate();
    if (!module_valid(spec, m))
        fail(ErrorKind::InvalidModule, "module '" + module_name(m) + "' is not part of this model");
    const std::int64_t h = spec.hidden_dim, f = spec.ffn_dim, v = spec.vocab_size;
    if (m.kind == ModuleKind::EmbedTokens) return {{"embed_tokens.weight", {v, h}, DecayClass::Decay}};
    if (m.kind == ModuleKind::Norm) return {{"norm.weight", {h}, DecayClass::NoDecay}};
    if (m.kind == ModuleKind::LmHead) return {{"lm_head.weight", {v, h}, DecayClass::Decay}};
    // Transformer layer: the flattening order is the declaration order below
    // (R/src/model.cpp:96-106): two norms, attention q/k/v/o, then MLP.
    const std::string p = module_name(m) + ".";
    struct Row {
        const char* suffix;
        std::int64_t a, b; // b == 0 -> 1-D
        DecayClass d;
    };
    const Row rows[] = {
        {"input_layernorm.weight", h, 0, DecayClass::NoDecay},
        {"post_attention_layernorm.weight", h, 0, DecayClass::NoDecay},
        {"attn.q_proj.weight", h, h, DecayClass::Decay},
        {"attn.k_proj.weight", h, h, DecayClass::Decay},
        {"attn.v_proj.weight", h, h, DecayClass::Decay},
        {"attn.o_proj.weight", h, h, DecayClass::Decay},
        {"mlp.gate_proj.weight", f, h, DecayClass::Decay},
        {"mlp.up_proj.weight", f, h, DecayClass::Decay},
        {"mlp.down_proj.weight", h, f, DecayClass::Decay},
    };
    std::vector<TensorDecl> out;
    out.reserve(9);
    for (const Row& r : rows) {
        TensorDecl t;
        t.name = p + r.suffix;
        t.shape = r.b ? std::vector<std::int64_t>{r.a, r.b} : std::vector<std::int64_t>{r.a};
        t.decay = r.d;
        out.push_back(std::move(t));
    }
    return out;
}

std::int64_t total_parameter_count(const ModelSpec& spec) { return ModelLayout(spec).parameter_count(); }

void AdamHyperparams::validate() const {
    if (!(lr > 0)) fail(ErrorKind::Geometry, "lr must be > 0");
    if (!(beta1 >= 0 && beta1 < 1) || !(beta2 >= 0 && beta2 < 1))
        fail(ErrorKind::Geometry, "beta coefficients must lie in [0, 1)");
    if (!(eps > 0)) fail(ErrorKind::Geometry, "eps must be > 0");
    if (!(weight_decay >= 0)) fail(ErrorKind::Geometry, "weight_decay must be >= 0");
}

AdamHyperparams hyper_for_class(const AdamHyperparams& base, DecayClass decay) {
    AdamHyperparams h = base;
    if (decay == DecayClass::NoDecay) h.weight_decay = 0.0;
    return h;
}

namespace {
std::int64_t class_elements(const ModelSpec& spec, const ModuleId& m, DecayClass d) {
    std::int64_t n = 0;
    for (const auto& t : tensors_of(spec, m))
        if (t.decay == d) n += t.numel();
    return n;
}
} // namespace

GroupTable build_group_table(const ModelSpec& spec) {
    spec.validate();
    GroupTable t;
    t.grouping = Grouping::Fine;
    t.num_layers = spec.num_layers;
    t.weight_tied = spec.weight_tied;
    const auto add = [&](ModuleId owner, DecayClass d) {
        t.groups.push_back({t.group_count(), owner, d, class_elements(spec, owner, d)});
    };
    add(ModuleId::norm(), DecayClass::NoDecay);
    for (int i = 0; i < spec.num_layers; ++i) add(ModuleId::transformer_layer(i), DecayClass::NoDecay);
    add(ModuleId::embed_tokens(), DecayClass::Decay);
    if (!spec.weight_tied) add(ModuleId::lm_head(), DecayClass::Decay);
    for (int i = 0; i < spec.num_layers; ++i) add(ModuleId::transformer_layer(i), DecayClass::Decay);
    return t;
}

GroupTable build_coarse_table(const ModelSpec& spec) {
    spec.validate();
    GroupTable t;
    t.grouping = Grouping::Coarse;
    t.num_layers = spec.num_layers;
    t.weight_tied = spec.weight_tied;
    std::int64_t nd = 0, d = 0;
    for (const auto& m : enumerate_modules(spec)) {
        nd += class_elements(spec, m, DecayClass::NoDecay);
        d += class_elements(spec, m, DecayClass::Decay);
    }
    t.groups.push_back({0, std::nullopt, DecayClass::NoDecay, nd});
    t.groups.push_back({1, std::nullopt, DecayClass::Decay, d});
    return t;
}

std::vector<int> group_indices_for(const GroupTable& table, const ModuleId& m) {
    if (table.grouping != Grouping::Fine) fail(ErrorKind::Geometry, "per-module group lookup requires the fine layout");
    const int L = table.num_layers;
    switch (m.kind) {
        case ModuleKind::Norm: return {0};
        case ModuleKind::EmbedTokens: return {L + 1};
        case ModuleKind::LmHead:
            if (table.weight_tied) fail(ErrorKind::InvalidModule, "lm_head does not exist in a weight-tied model");
            return {L + 2};
        case ModuleKind::TransformerLayer:
            if (m.layer < 0 || m.layer >= L)
                fail(ErrorKind::InvalidModule, "layer index out of range: " + std::to_string(m.layer));
            return {1 + m.layer, (table.weight_tied ? L + 2 : L + 3) + m.layer};
    }
    fail(ErrorKind::InvalidModule, "unknown module kind");
}

std::vector<int> group_indices_for_modules(const GroupTable& table, const std::vector<ModuleId>& modules) {
    std::set<int> s;
    if (table.grouping == Grouping::Coarse) {
        for (const auto& g : table.groups) s.insert(g.index);
    } else {
        for (const auto& m : modules)
            for (int g : group_indices_for(table, m)) s.insert(g);
    }
    return {s.begin(), s.end()};
}

std::int64_t ShardGeometry::padded_length(std::int64_t true_length) const {
    if (num_ranks < 1) fail(ErrorKind::Geometry, "num_ranks must be >= 1");
    if (true_length < 0) fail(ErrorKind::Geometry, "negative group length");
    const std::int64_t n = num_ranks;
    return (true_length + n - 1) / n * n;
}

ModelLayout::ModelLayout(const ModelSpec& spec) : spec_(spec) {
    modules_ = enumerate_modules(spec);
    module_offset_.resize(modules_.size());
    std::int64_t off = 0;
    std::vector<std::vector<TensorDecl>> decls(modules_.size());
    for (std::size_t i = 0; i < modules_.size(); ++i) {
        module_offset_[i] = off;
        decls[i] = tensors_of(spec, modules_[i]);
        for (const auto& t : decls[i]) off += t.numel();
    }
    total_ = off;
    table_ = build_group_table(spec);
    owner_index_.resize(static_cast<std::size_t>(table_.group_count()));
    slices_.resize(static_cast<std::size_t>(table_.group_count()));
    for (const auto& g : table_.groups) {
        const int mi = canonical_index(spec, *g.owner);
        owner_index_[static_cast<std::size_t>(g.index)] = mi;
        std::int64_t go = 0, within = 0;
        for (const auto& t : decls[static_cast<std::size_t>(mi)]) {
            if (t.decay == g.decay) {
                slices_[static_cast<std::size_t>(g.index)].push_back({t, go, module_offset_[static_cast<std::size_t>(mi)] + within});
                go += t.numel();
            }
            within += t.numel();
        }
        if (go != g.element_count) fail(ErrorKind::Consistency, "group tensor slices do not tile the group");
    }
}

std::vector<TensorSlice> group_tensor_slices(const ModelSpec& spec, const GroupTable& table, int group) {
    if (group < 0 || group >= table.group_count())
        fail(ErrorKind::Geometry, "group index out of range: " + std::to_string(group));
    const GroupInfo& info = table.groups[static_cast<std::size_t>(group)];
    if (info.owner) return ModelLayout(spec).slices(group);
    // Coarse group: every module's tensors of this decay class, module order.
    ModelLayout lay(spec);
    std::vector<TensorSlice> out;
    std::int64_t go = 0;
    for (int mi = 0; mi < lay.module_count(); ++mi) {
        std::int64_t within = 0;
        for (const auto& t : tensors_of(spec, lay.modules()[static_cast<std::size_t>(mi)])) {
            if (t.decay == info.decay) {
                out.push_back({t, go, lay.module_offset(mi) + within});
                go += t.numel();
            }
            within += t.numel();
        }
    }
    return out;
}

} // namespace tailor
