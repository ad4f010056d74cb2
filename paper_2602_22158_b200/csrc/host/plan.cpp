// Plan resolution and the byte-segment view of a merge.
//   resolve_plan          — R/src/merge.cpp:39-152 (same validation order and error kinds)
//   plan_weights/plan_shard — the gather/scatter of R/src/merge.cpp:244-303 expressed as
//                           {window, src_off, dst_off, bytes} copy segments for the device
//   recipe_from_manifests — R/src/merge.cpp:359-418
//   select_by_magnitude / recipe_from_selection — SURVEY §8 a14 (new)
#include <algorithm>
#include <cmath>
#include <map>
#include <set>

#include "tailor/errors.hpp"
#include "tailor/merge.hpp"

namespace tailor {

namespace fs = std::filesystem;

namespace {

std::vector<std::string> distinct_sources(const MergeRecipe& r) {
    std::vector<std::string> out;
    const auto note = [&](const std::string& p) {
        if (!p.empty() && p != "latest" && std::find(out.begin(), out.end(), p) == out.end()) out.push_back(p);
    };
    for (const auto& s : r.slices) note(s.source);
    for (const auto& [k, p] : r.aux) note(p);
    note(r.base_checkpoint);
    note(r.config_from);
    return out;
}

} // namespace

MergePlan resolve_plan(const MergeRecipe& recipe) {
    return resolve_plan_with(recipe, [](const std::string& p) { return read_checkpoint_summary(p); });
}

MergePlan resolve_plan_with(const MergeRecipe& recipe, const SummaryLookup& lookup) {
    if (recipe.num_ranks < 1) fail(ErrorKind::Recipe, "num_ranks must be >= 1");
    MergePlan plan;
    plan.sources = distinct_sources(recipe);
    if (plan.sources.empty()) fail(ErrorKind::Recipe, "recipe names no source checkpoints");
    std::map<std::string, CheckpointSummary> sum;
    for (const auto& p : plan.sources) sum.emplace(p, lookup(p));

    const ModelSpec& geo = sum.at(plan.sources.front()).spec;
    for (const auto& p : plan.sources) {
        const CheckpointSummary& s = sum.at(p);
        if (!s.spec.same_geometry(geo)) fail(ErrorKind::Geometry, "source '" + p + "' has a different model geometry");
        if (s.optim.num_ranks != recipe.num_ranks)
            fail(ErrorKind::Geometry, "source '" + p + "' was sharded over " + std::to_string(s.optim.num_ranks) +
                                          " ranks, recipe says " + std::to_string(recipe.num_ranks));
        if (s.optim.grouping != Grouping::Fine)
            fail(ErrorKind::Geometry, "source '" + p + "' uses the coarse grouping and cannot be merged");
    }
    plan.num_ranks = recipe.num_ranks;

    std::map<ModuleId, MergePlan::Assignment> assign;
    const auto put = [&](const ModuleId& tgt, const std::string& src, const ModuleId& src_mod, const std::string& where) {
        if (!module_valid(geo, tgt)) fail(ErrorKind::Recipe, where + ": module '" + module_name(tgt) + "' is not in the model");
        if (assign.count(tgt)) fail(ErrorKind::Recipe, where + ": target module '" + module_name(tgt) + "' assigned twice");
        assign[tgt] = {src, src_mod, sum.at(src).trainer.step};
    };
    for (std::size_t i = 0; i < recipe.slices.size(); ++i) {
        const RecipeSlice& s = recipe.slices[i];
        const std::string where = "slices[" + std::to_string(i) + "]";
        if (s.targets.size() != s.layers.size()) fail(ErrorKind::Recipe, where + ": targets must have the same length as layers");
        for (std::size_t k = 0; k < s.layers.size(); ++k) {
            if (s.layers[k] >= geo.num_layers)
                fail(ErrorKind::Recipe, where + ": layer " + std::to_string(s.layers[k]) + " out of range");
            put(ModuleId::transformer_layer(s.targets[k]), s.source, ModuleId::transformer_layer(s.layers[k]), where);
        }
    }
    for (const auto& [key, p] : recipe.aux) {
        const ModuleId m = parse_module_name(key);
        if (!module_valid(geo, m)) fail(ErrorKind::Recipe, "aux." + key + ": module is not in the model (weight-tied spec)");
        put(m, p, m, "aux." + key);
    }
    for (const auto& m : enumerate_modules(geo)) {
        if (assign.count(m)) continue;
        if (recipe.base_checkpoint.empty())
            fail(ErrorKind::Recipe, "module '" + module_name(m) + "' is not covered and no base_checkpoint is set");
        assign[m] = {recipe.base_checkpoint, m, sum.at(recipe.base_checkpoint).trainer.step};
    }
    for (const auto& [tgt, a] : assign)
        if (!sum.at(a.source).manifest.contains(a.source_module))
            fail(ErrorKind::SourceLacksModule,
                 "checkpoint '" + a.source + "' does not contain module '" + module_name(a.source_module) + "'");

    std::erase_if(plan.sources, [&](const std::string& p) {
        return std::none_of(assign.begin(), assign.end(), [&](const auto& kv) { return kv.second.source == p; });
    });

    if (recipe.config_from == "latest") {
        std::string best;
        std::int64_t best_step = -1;
        for (const auto& p : plan.sources) {
            const std::int64_t st = sum.at(p).trainer.step;
            if (st > best_step || (st == best_step && p > best)) {
                best = p;
                best_step = st;
            }
        }
        plan.config_source = best;
    } else {
        plan.config_source = recipe.config_from;
    }
    plan.spec = sum.at(plan.config_source).spec;
    plan.table = build_group_table(plan.spec);
    plan.assignment = std::move(assign);
    for (const auto& [tgt, a] : plan.assignment) {
        const auto tg = group_indices_for(plan.table, tgt);
        const auto sg = group_indices_for(plan.table, a.source_module);
        for (std::size_t i = 0; i < tg.size(); ++i) plan.group_copies.push_back({a.source, sg[i], tg[i]});
    }
    std::stable_sort(plan.group_copies.begin(), plan.group_copies.end(),
                     [](const auto& x, const auto& y) { return x.target_group < y.target_group; });
    if (static_cast<int>(plan.group_copies.size()) != plan.table.group_count())
        fail(ErrorKind::Consistency, "group copy list does not cover the target table");
    return plan;
}

namespace {
using Piece = CopyPiece;
void finish_plan(PartitionPlan& pp, std::vector<Piece> pieces);
} // namespace

void finalize_partition(PartitionPlan& pp, std::vector<CopyPiece> pieces) { finish_plan(pp, std::move(pieces)); }

namespace {

// Builds windows + coalesced segments from (source, container, src range,
// dst range) pieces in destination order.
void finish_plan(PartitionPlan& pp, std::vector<Piece> pieces) {
    std::map<std::pair<std::string, int>, std::pair<std::uint64_t, std::uint64_t>> span;
    for (const auto& p : pieces) {
        auto key = std::make_pair(p.source, p.container);
        auto it = span.find(key);
        if (it == span.end()) span[key] = {p.src_off, p.src_off + p.bytes};
        else {
            it->second.first = std::min(it->second.first, p.src_off);
            it->second.second = std::max(it->second.second, p.src_off + p.bytes);
        }
    }
    std::map<std::pair<std::string, int>, std::uint32_t> index;
    for (const auto& [key, range] : span) {
        index[key] = static_cast<std::uint32_t>(pp.windows.size());
        pp.windows.push_back({key.first, key.second, range.first, range.second});
    }
    std::sort(pieces.begin(), pieces.end(), [](const Piece& a, const Piece& b) { return a.dst_off < b.dst_off; });
    for (const auto& p : pieces) {
        if (p.bytes == 0) continue;
        const std::uint32_t w = index.at({p.source, p.container});
        const std::uint64_t so = p.src_off - pp.windows[w].lo;
        if (!pp.segments.empty()) {
            CopySegment& last = pp.segments.back();
            if (last.window == w && last.dst_off + last.bytes == p.dst_off && last.src_off + last.bytes == so) {
                last.bytes += p.bytes;
                continue;
            }
        }
        pp.segments.push_back({w, so, p.dst_off, p.bytes});
    }
}

} // namespace

PartitionPlan plan_weights(const MergePlan& plan, const LayoutLookup& layouts, std::uint64_t lo, std::uint64_t hi) {
    std::vector<EntryDecl> decls;
    struct From {
        std::string source;
        std::string name;
    };
    std::map<std::string, From> from;
    for (const auto& [tgt, a] : plan.assignment) {
        const auto td = tensors_of(plan.spec, tgt);
        const auto sd = tensors_of(plan.spec, a.source_module);
        const ContainerLayout& src = layouts(a.source).weights;
        for (std::size_t i = 0; i < td.size(); ++i) {
            const Entry* e = src.find(sd[i].name);
            if (!e) fail(ErrorKind::MissingArtifact, "'" + a.source + "' lacks weight tensor '" + sd[i].name + "'");
            if (e->dtype != Dtype::BF16 || e->shape != td[i].shape)
                fail(ErrorKind::Geometry, "weight tensor '" + sd[i].name + "' of '" + a.source + "' has unexpected dtype/shape");
            decls.push_back({td[i].name, Dtype::BF16, td[i].shape});
            from[td[i].name] = {a.source, sd[i].name};
        }
    }
    PartitionPlan pp;
    pp.out = layout_for(std::move(decls));
    pp.dst_lo = std::min(lo, pp.out.payload_bytes);
    pp.dst_hi = std::min(hi, pp.out.payload_bytes);
    std::vector<Piece> pieces;
    for (const auto& e : pp.out.entries) {
        const std::uint64_t a = std::max(e.begin, pp.dst_lo), b = std::min(e.end, pp.dst_hi);
        if (a >= b) continue;
        const From& f = from.at(e.name);
        const Entry* se = layouts(f.source).weights.find(f.name);
        pieces.push_back({f.source, -1, se->begin + (a - e.begin), a, b - a});
    }
    finish_plan(pp, std::move(pieces));
    return pp;
}

PartitionPlan plan_shard(const MergePlan& plan, const LayoutLookup& layouts, int rank, std::uint64_t lo, std::uint64_t hi) {
    const ShardGeometry geom{plan.num_ranks};
    std::vector<EntryDecl> decls;
    std::vector<Piece> pending; // dst offsets filled after layout
    struct Want {
        std::string dst;
        std::string source;
        std::uint64_t src_off;
        std::uint64_t bytes;
    };
    std::vector<Want> wants;
    // Field order mirrors copy_shard_entries (R/src/merge.cpp:210); the
    // output order is fixed by the sorted layout, so it is immaterial here.
    for (const auto& c : plan.group_copies) {
        const std::int64_t chunk = geom.shard_length(plan.table.groups[static_cast<std::size_t>(c.target_group)].element_count);
        const auto& src_layouts = layouts(c.source).shards;
        if (rank >= static_cast<int>(src_layouts.size()))
            fail(ErrorKind::MissingArtifact, "cannot open shard rank " + std::to_string(rank) + " of '" + c.source + "'");
        const ContainerLayout& src = src_layouts[static_cast<std::size_t>(rank)];
        for (const char* f : {".master", ".exp_avg", ".exp_avg_sq"}) {
            const std::string sk = shard_key(c.source_group, f), dk = shard_key(c.target_group, f);
            const Entry* e = src.find(sk);
            if (!e)
                fail(ErrorKind::MissingArtifact,
                     "shard rank " + std::to_string(rank) + " of '" + c.source + "' lacks '" + sk + "'");
            if (e->dtype != Dtype::F32 || e->shape != std::vector<std::int64_t>{chunk})
                fail(ErrorKind::Geometry, "shard tensor '" + sk + "' of '" + c.source + "' has unexpected dtype/shape");
            decls.push_back({dk, Dtype::F32, {chunk}});
            wants.push_back({dk, c.source, e->begin, e->bytes()});
        }
    }
    PartitionPlan pp;
    pp.out = layout_for(std::move(decls),
                        {{"num_ranks", std::to_string(plan.num_ranks)}, {"rank", std::to_string(rank)}});
    pp.dst_lo = std::min(lo, pp.out.payload_bytes);
    pp.dst_hi = std::min(hi, pp.out.payload_bytes);
    std::vector<Piece> pieces;
    for (const auto& w : wants) {
        const std::uint64_t d0 = pp.out.find(w.dst)->begin, d1 = d0 + w.bytes;
        const std::uint64_t a = std::max(d0, pp.dst_lo), b = std::min(d1, pp.dst_hi);
        if (a < b) pieces.push_back({w.source, rank, w.src_off + (a - d0), a, b - a});
    }
    finish_plan(pp, std::move(pieces));
    return pp;
}

std::pair<std::uint64_t, std::uint64_t> weights_share(const ContainerLayout& out, int unit, int units) {
    if (units < 1 || unit < 0 || unit >= units) fail(ErrorKind::Geometry, "bad weights share request");
    const auto cut = [&](int u) -> std::uint64_t {
        if (u <= 0) return 0;
        if (u >= units) return out.payload_bytes;
        const double target = static_cast<double>(out.payload_bytes) * u / units;
        // nearest tensor boundary to the balanced cut
        std::uint64_t best = 0;
        double best_d = target;
        for (const auto& e : out.entries) {
            const double d = std::fabs(static_cast<double>(e.end) - target);
            if (d < best_d) {
                best_d = d;
                best = e.end;
            }
        }
        return best;
    };
    std::uint64_t a = cut(unit), b = cut(unit + 1);
    if (b < a) b = a;
    return {a, b};
}

OptimMeta merged_optim_meta(const MergePlan& plan, const SummaryLookup& lookup) {
    const ShardGeometry geom{plan.num_ranks};
    std::map<std::string, CheckpointSummary> sums;
    const auto get = [&](const std::string& p) -> const CheckpointSummary& {
        auto it = sums.find(p);
        if (it == sums.end()) it = sums.emplace(p, lookup(p)).first;
        return it->second;
    };
    OptimMeta o;
    o.grouping = Grouping::Fine;
    o.num_ranks = plan.num_ranks;
    o.step = get(plan.config_source).optim.step;
    for (const auto& c : plan.group_copies) {
        const OptimGroupMeta* sm = get(c.source).optim.find(c.source_group);
        if (!sm) fail(ErrorKind::Consistency, "source group metadata missing for group " + std::to_string(c.source_group));
        const GroupInfo& info = plan.table.groups[static_cast<std::size_t>(c.target_group)];
        OptimGroupMeta m;
        m.index = c.target_group;
        m.owner = info.owner ? module_name(*info.owner) : "coarse";
        m.decay = info.decay;
        m.true_length = info.element_count;
        m.padded_length = geom.padded_length(info.element_count);
        m.shard_length = geom.shard_length(info.element_count);
        m.hyper = sm->hyper;
        o.groups.push_back(std::move(m));
    }
    return o;
}

SaveManifest merged_manifest(const MergePlan& plan, const SummaryLookup& lookup) {
    SaveManifest m;
    m.step = lookup(plan.config_source).trainer.step;
    m.strategy = "merged";
    m.modules = enumerate_modules(plan.spec);
    for (const auto& [tgt, a] : plan.assignment) m.provenance[module_name(tgt)] = {a.source, a.source_step};
    return m;
}

std::vector<fs::path> list_checkpoints(const fs::path& run_dir) {
    if (!fs::exists(run_dir)) fail(ErrorKind::MissingArtifact, "run directory '" + run_dir.string() + "' does not exist");
    std::vector<std::pair<std::int64_t, fs::path>> found;
    for (const auto& e : fs::directory_iterator(run_dir)) {
        if (!e.is_directory()) continue;
        if (auto st = step_of_dir(e.path().filename().string())) found.emplace_back(*st, e.path());
    }
    std::sort(found.begin(), found.end());
    std::vector<fs::path> out;
    for (auto& [st, p] : found) out.push_back(std::move(p));
    return out;
}

namespace {

bool newer(const CheckpointSummary& a, const CheckpointSummary& b) {
    return a.trainer.step != b.trainer.step ? a.trainer.step > b.trainer.step : a.dir.string() > b.dir.string();
}

// Shared tail of recipe_from_manifests / recipe_from_selection: chosen[m] is
// the snapshot each module comes from; `latest` becomes base + config.
MergeRecipe recipe_from_choice(const ModelSpec& spec, const std::vector<const CheckpointSummary*>& chosen,
                               const CheckpointSummary* latest) {
    MergeRecipe r;
    r.num_ranks = latest->optim.num_ranks;
    r.base_checkpoint = latest->dir.string();
    r.config_from = latest->dir.string();
    const auto mods = enumerate_modules(spec);
    // Iterate in ModuleId order, as the reference's std::map does.
    std::vector<int> order(mods.size());
    for (std::size_t i = 0; i < mods.size(); ++i) order[i] = static_cast<int>(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return mods[static_cast<std::size_t>(a)] < mods[static_cast<std::size_t>(b)]; });
    std::map<std::string, std::vector<int>> layer_slices;
    for (int i : order) {
        const CheckpointSummary* s = chosen[static_cast<std::size_t>(i)];
        if (s == latest) continue;
        const ModuleId& m = mods[static_cast<std::size_t>(i)];
        if (m.kind == ModuleKind::TransformerLayer) layer_slices[s->dir.string()].push_back(m.layer);
        else r.aux[module_name(m)] = s->dir.string();
    }
    for (auto& [src, layers] : layer_slices) {
        std::sort(layers.begin(), layers.end());
        r.slices.push_back({src, layers, layers});
    }
    return r;
}

} // namespace

MergeRecipe recipe_from_manifests(const fs::path& run_dir, std::int64_t failure_step) {
    std::vector<CheckpointSummary> cand;
    for (const auto& d : list_checkpoints(run_dir)) {
        CheckpointSummary s = read_checkpoint_summary(d);
        if (s.trainer.step <= failure_step) cand.push_back(std::move(s));
    }
    if (cand.empty())
        fail(ErrorKind::UnrecoverableModule,
             "no checkpoint at or before step " + std::to_string(failure_step) + " in '" + run_dir.string() + "'");
    const ModelSpec& geo = cand.front().spec;
    for (const auto& s : cand)
        if (!s.spec.same_geometry(geo))
            fail(ErrorKind::Geometry, "checkpoints in '" + run_dir.string() + "' disagree on model geometry");
    const CheckpointSummary* latest = &cand.front();
    for (const auto& s : cand)
        if (newer(s, *latest)) latest = &s;
    const auto mods = enumerate_modules(geo);
    std::vector<const CheckpointSummary*> chosen(mods.size(), nullptr);
    for (std::size_t i = 0; i < mods.size(); ++i) {
        for (const auto& s : cand)
            if (s.manifest.contains(mods[i]) && (!chosen[i] || newer(s, *chosen[i]))) chosen[i] = &s;
        if (!chosen[i])
            fail(ErrorKind::UnrecoverableModule, "module '" + module_name(mods[i]) + "' was never saved at or before step " +
                                                     std::to_string(failure_step));
    }
    return recipe_from_choice(geo, chosen, latest);
}

double magnitude_score(double sum_delta_sq, double sum_ref_sq) {
    if (sum_ref_sq > 0.0) return std::sqrt(sum_delta_sq) / std::sqrt(sum_ref_sq);
    return sum_delta_sq > 0.0 ? INFINITY : 0.0;
}

Selection select_by_magnitude(const std::vector<std::vector<double>>& scores, int M, double rho) {
    if (M < 1) fail(ErrorKind::Geometry, "no modules to select from");
    if (!(rho > 0.0 && rho <= 1.0)) fail(ErrorKind::Recipe, "selection ratio rho must lie in (0, 1]");
    Selection sel;
    std::vector<int> all(static_cast<std::size_t>(M));
    for (int i = 0; i < M; ++i) all[static_cast<std::size_t>(i)] = i;
    sel.saved.push_back(all); // S_1 holds the complete state
    const int n = std::max(1, std::min(M, static_cast<int>(std::ceil(rho * M))));
    sel.min_boundary_gap = INFINITY;
    for (const auto& sc : scores) {
        if (static_cast<int>(sc.size()) != M) fail(ErrorKind::Geometry, "score row has the wrong module count");
        std::vector<int> order = all;
        // descending score; ties -> lower canonical index (stable on ascending ids)
        std::stable_sort(order.begin(), order.end(),
                         [&](int a, int b) { return sc[static_cast<std::size_t>(a)] > sc[static_cast<std::size_t>(b)]; });
        if (n < M) {
            const double hi = sc[static_cast<std::size_t>(order[static_cast<std::size_t>(n - 1)])];
            const double lo = sc[static_cast<std::size_t>(order[static_cast<std::size_t>(n)])];
            sel.min_boundary_gap = std::min(sel.min_boundary_gap, hi > 0 ? (hi - lo) / hi : 0.0);
        }
        std::vector<int> pick(order.begin(), order.begin() + n);
        std::sort(pick.begin(), pick.end());
        sel.saved.push_back(std::move(pick));
    }
    sel.source_of.assign(static_cast<std::size_t>(M), 0);
    for (std::size_t k = 0; k < sel.saved.size(); ++k)
        for (int m : sel.saved[k]) sel.source_of[static_cast<std::size_t>(m)] = static_cast<int>(k);
    return sel;
}

MergeRecipe recipe_from_selection(const std::vector<CheckpointSummary>& snaps, const Selection& sel) {
    if (snaps.empty()) fail(ErrorKind::Recipe, "no snapshots");
    if (sel.saved.size() != snaps.size()) fail(ErrorKind::Consistency, "selection does not match the snapshot count");
    const ModelSpec& geo = snaps.front().spec;
    const CheckpointSummary* latest = &snaps.front();
    for (const auto& s : snaps)
        if (newer(s, *latest)) latest = &s;
    const auto mods = enumerate_modules(geo);
    std::vector<const CheckpointSummary*> chosen(mods.size(), nullptr);
    for (std::size_t k = 0; k < snaps.size(); ++k)
        for (int m : sel.saved[k]) {
            const CheckpointSummary*& c = chosen[static_cast<std::size_t>(m)];
            if (!c || newer(snaps[k], *c)) c = &snaps[k];
        }
    for (std::size_t i = 0; i < mods.size(); ++i)
        if (!chosen[i]) fail(ErrorKind::UnrecoverableModule, "module '" + module_name(mods[i]) + "' was never selected");
    return recipe_from_choice(geo, chosen, latest);
}

} // namespace tailor
