// Layer map: parameter names -> modules -> optimizer groups -> per-rank
// flat-offset ranges. Same semantics as the reference layer
// (R/src/model.cpp:22-132, R/src/groups.cpp:40-133, R/src/shard.cpp:10-19),
// re-implemented around a precomputed ModelLayout so every lookup the device
// table builders make is O(1) instead of the reference's O(M^2) offset scans.
#pragma once

#include <compare>
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

namespace tailor {

// R/include/tailor/model.hpp:14-30 — geometry + seed; no GQA, no biases.
struct ModelSpec {
    int num_layers = 0;
    int hidden_dim = 0;
    int ffn_dim = 0;
    int vocab_size = 0;
    bool weight_tied = false;
    std::uint64_t seed = 0;

    bool operator==(const ModelSpec&) const = default;
    int module_count() const { return num_layers + (weight_tied ? 2 : 3); }
    void validate() const;
    bool same_geometry(const ModelSpec& o) const {
        return num_layers == o.num_layers && hidden_dim == o.hidden_dim && ffn_dim == o.ffn_dim &&
               vocab_size == o.vocab_size && weight_tied == o.weight_tied;
    }
};

// Enum order matters: ModuleId ordering (kind, layer) is the std::map key
// order the reference iterates in (R/include/tailor/model.hpp:35-48).
enum class ModuleKind : int { EmbedTokens = 0, TransformerLayer = 1, Norm = 2, LmHead = 3 };

struct ModuleId {
    ModuleKind kind = ModuleKind::EmbedTokens;
    int layer = -1;
    static ModuleId embed_tokens() { return {ModuleKind::EmbedTokens, -1}; }
    static ModuleId transformer_layer(int i) { return {ModuleKind::TransformerLayer, i}; }
    static ModuleId norm() { return {ModuleKind::Norm, -1}; }
    static ModuleId lm_head() { return {ModuleKind::LmHead, -1}; }
    bool operator==(const ModuleId&) const = default;
    auto operator<=>(const ModuleId&) const = default;
};

std::string module_name(const ModuleId& m);
ModuleId parse_module_name(const std::string& name);
bool module_valid(const ModelSpec& spec, const ModuleId& m);
// Canonical order [embed_tokens, layers.0..L-1, norm, lm_head?].
std::vector<ModuleId> enumerate_modules(const ModelSpec& spec);
int canonical_index(const ModelSpec& spec, const ModuleId& m);

enum class DecayClass : int { Decay = 0, NoDecay = 1 };

struct TensorDecl {
    std::string name;
    std::vector<std::int64_t> shape;
    DecayClass decay = DecayClass::Decay;
    std::int64_t numel() const {
        std::int64_t n = 1;
        for (auto d : shape) n *= d;
        return n;
    }
};

// Declared tensors of one module in canonical flattening order.
std::vector<TensorDecl> tensors_of(const ModelSpec& spec, const ModuleId& m);
std::int64_t total_parameter_count(const ModelSpec& spec);

// ---- optimizer groups (R/src/groups.cpp) ------------------------------------
struct AdamHyperparams {
    double lr = 1e-3;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;
    double weight_decay = 0.0;
    bool operator==(const AdamHyperparams&) const = default;
    void validate() const;
};
inline constexpr double kDefaultLr = 1e-3;
inline constexpr double kDefaultWeightDecay = 0.01;
AdamHyperparams hyper_for_class(const AdamHyperparams& base, DecayClass decay);

enum class Grouping { Fine, Coarse };

struct GroupInfo {
    int index = 0;
    std::optional<ModuleId> owner; // nullopt for the two coarse groups
    DecayClass decay = DecayClass::Decay;
    std::int64_t element_count = 0;
};

// Fine layout: g0 norm | g1..gL layer no-decay | gL+1 embed | gL+2 lm_head
// (untied) | then layer decay groups (R/include/tailor/groups.hpp:53-61).
struct GroupTable {
    Grouping grouping = Grouping::Fine;
    int num_layers = 0;
    bool weight_tied = false;
    std::vector<GroupInfo> groups;
    int group_count() const { return static_cast<int>(groups.size()); }
};

GroupTable build_group_table(const ModelSpec& spec);
GroupTable build_coarse_table(const ModelSpec& spec);
std::vector<int> group_indices_for(const GroupTable& table, const ModuleId& m);
std::vector<int> group_indices_for_modules(const GroupTable& table, const std::vector<ModuleId>& modules);

struct TensorSlice {
    TensorDecl decl;
    std::int64_t group_offset = 0; // first element within the flattened group
    std::int64_t model_offset = 0; // global element id of the first element
};

// ---- ZeRO-style shard geometry (R/src/shard.cpp:10-19) ----------------------
struct ShardGeometry {
    int num_ranks = 1;
    std::int64_t padded_length(std::int64_t true_length) const;
    std::int64_t shard_length(std::int64_t true_length) const { return padded_length(true_length) / num_ranks; }
};

// ---- precomputed layout ------------------------------------------------------
// Everything the table builders need, computed once per spec: canonical
// module list, per-module global element offsets, the fine group table and
// each group's tensor slices (flattening order).
class ModelLayout {
  public:
    explicit ModelLayout(const ModelSpec& spec);
    const ModelSpec& spec() const { return spec_; }
    const std::vector<ModuleId>& modules() const { return modules_; }
    const GroupTable& table() const { return table_; }
    int module_count() const { return static_cast<int>(modules_.size()); }
    std::int64_t module_offset(int canonical) const { return module_offset_[static_cast<std::size_t>(canonical)]; }
    int owner_index(int group) const { return owner_index_[static_cast<std::size_t>(group)]; }
    const std::vector<TensorSlice>& slices(int group) const { return slices_[static_cast<std::size_t>(group)]; }
    std::int64_t parameter_count() const { return total_; }

  private:
    ModelSpec spec_;
    std::vector<ModuleId> modules_;
    std::vector<std::int64_t> module_offset_;
    GroupTable table_;
    std::vector<int> owner_index_;
    std::vector<std::vector<TensorSlice>> slices_;
    std::int64_t total_ = 0;
};

std::vector<TensorSlice> group_tensor_slices(const ModelSpec& spec, const GroupTable& table, int group);

} // namespace tailor
