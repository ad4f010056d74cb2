// `tailor` CLI for the tailoring path, over the C ABI only (include/tailor_b200.h).
// Mirrors the reference's merge / plan subcommands and exit codes
// (R/tools/tailor_main.cpp:66-103, :291-299, :351-357) and adds the
// update-magnitude `select` / `score` subcommands.
//
//   tailor merge  --recipe r.yaml --out DIR [--workers W] [--uncached] [--json] [--device D | --devices 0,1,..] [--no-verify]
//                [--io auto|buffered|direct|direct-rw]
//   tailor plan   --run RUN --failure-step S --out r.yaml
//   tailor select --snapshots A,B,... [--rho 0.5] --out r.yaml [--device D | --devices 0,1,..] [--json]
//   tailor score  --snapshots A,B,... [--device D | --devices 0,1,..]
//   tailor check  --ckpt DIR [--device D]
//   tailor regroup --ckpt DIR --out DIR [--to fine|coarse] [--device D | --devices 0,1,..] [--no-verify]
//   tailor resume --ckpt DIR --steps S --out RUN [--device D]
//   tailor train  --config c.json --steps S --interval I --strategy full|parity|filter|magnitude
//                 --ranks N --out RUN [--lr --weight-decay --head --tail --sparse-multiple --rho --device]
// Exit codes: 0 success, 1 user error, 2 internal/consistency error.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "tailor_b200.h"

namespace {

struct Args {
    std::map<std::string, std::string> kv;
    std::set<std::string> flags;
};

int exit_for(int code) { return (code >= 1 && code <= 9) ? 1 : 2; }

int report(int code) {
    // as the reference CLI (R/tools/tailor_main.cpp:93-98): "error: <kind>: ..." for a
    // TailorError, "internal error: ..." for anything else (the C ABI's message already
    // carries that prefix)
    std::cerr << (code == TG_E_INTERNAL ? "" : "error: ") << tg_last_error() << "\n";
    return exit_for(code);
}

std::string read_file(const std::string& p, bool* ok) {
    std::ifstream in(p, std::ios::binary);
    *ok = static_cast<bool>(in);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

std::vector<std::string> split_csv(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string x;
    while (std::getline(ss, x, ','))
        if (!x.empty()) out.push_back(x);
    return out;
}

template <typename F>
int text_call(F&& f, std::string& out) {
    std::vector<char> buf(1 << 16);
    size_t need = 0;
    int rc = f(buf.data(), buf.size(), &need);
    if (rc != TG_OK && need > buf.size()) {
        buf.resize(need);
        rc = f(buf.data(), buf.size(), &need);
    }
    if (rc == TG_OK) out = buf.data();
    return rc;
}

// --devices 0,1,... (lanes spread over these GPUs; output bytes do not depend on them),
// else --device D, else device 0
std::vector<int32_t> devices_of(const Args& a) {
    std::vector<int32_t> out;
    if (a.kv.count("devices"))
        for (const auto& x : split_csv(a.kv.at("devices"))) out.push_back(static_cast<int32_t>(std::stoi(x)));
    if (out.empty()) out.push_back(a.kv.count("device") ? static_cast<int32_t>(std::stoi(a.kv.at("device"))) : 0);
    return out;
}

bool require(const Args& a, std::initializer_list<const char*> keys) {
    for (const char* k : keys)
        if (!a.kv.count(k)) {
            std::cerr << "missing required option --" << k << "\n";
            return false;
        }
    return true;
}

// --workers / --uncached / --devices / --no-verify / --io of merge and select-merge;
// false (after the message) on an unknown --io mode.
bool merge_options_of(const Args& a, const std::vector<int32_t>& devs, tg_merge_options& opt) {
    opt = tg_merge_options{};
    opt.workers = a.kv.count("workers") ? std::stoi(a.kv.at("workers")) : 0;
    opt.uncached = a.flags.count("uncached") ? 1 : 0;
    opt.device = devs.front();
    opt.skip_verify = a.flags.count("no-verify") ? 1 : 0;
    opt.devices = devs.data();
    opt.num_devices = static_cast<int32_t>(devs.size());
    if (a.kv.count("io")) { // --io auto|buffered|direct|direct-rw (source reads / output writes)
        const std::string m = a.kv.at("io");
        opt.io_mode = m == "buffered" ? TG_IO_BUFFERED : m == "direct" ? TG_IO_DIRECT : m == "direct-rw" ? TG_IO_DIRECT_RW
                      : m == "auto"   ? TG_IO_AUTO : -1;
        if (opt.io_mode < 0) {
            std::cerr << "error: unknown --io mode '" << m << "' (auto, buffered, direct, direct-rw)\n";
            return false;
        }
    }
    return true;
}

int cmd_merge(const Args& a) {
    if (!require(a, {"recipe", "out"})) return 1;
    bool ok = false;
    const std::string yaml = read_file(a.kv.at("recipe"), &ok);
    if (!ok) {
        std::cerr << "error: MissingArtifact: cannot open '" << a.kv.at("recipe") << "'\n";
        return 1;
    }
    const std::vector<int32_t> devs = devices_of(a);
    tg_merge_options opt{};
    if (!merge_options_of(a, devs, opt)) return 1;
    tg_merge_stats st{};
    const int rc = tg_execute_merge(yaml.c_str(), a.kv.at("out").c_str(), &opt, &st);
    if (rc != TG_OK) return report(rc);
    size_t need = 0; // plan summary for the report (sidecar reads only)
    tg_resolve_plan(yaml.c_str(), nullptr, 0, &need);
    std::string plan(need, '\0');
    if (tg_resolve_plan(yaml.c_str(), plan.data(), plan.size(), &need) != TG_OK) return report(tg_last_error_kind());
    const nlohmann::json pj = nlohmann::json::parse(plan.c_str());
    const int ranks = pj.at("num_ranks").get<int>();
    const int sources = static_cast<int>(pj.at("sources").size());
    if (a.flags.count("json")) { // the reference's keys (R/tools/tailor_main.cpp:84-91) plus the device's
        std::cout << nlohmann::json{{"out", a.kv.at("out")},
                                    {"num_ranks", ranks},
                                    {"num_sources", sources},
                                    {"shard_files_read", st.shard_files_read},
                                    {"weight_files_read", st.weight_files_read},
                                    {"wall_ms", st.wall_ms},
                                    {"bytes_moved", st.bytes_moved},
                                    {"device_ms", st.device_ms}}
                         .dump()
                  << "\n";
        return 0;
    }
    // the reference's report (R/tools/tailor_main.cpp:94-101), then the device's line
    std::cout << "merged checkpoint written to " << a.kv.at("out") << "\n";
    std::cout << "sources: " << sources << "  ranks: " << ranks << "\n";
    std::cout << "optimizer shard files read: " << st.shard_files_read << " (bound " << ranks << " x " << sources << " = "
              << ranks * sources << " cached)\n";
    std::cout << "weight files read: " << st.weight_files_read << "\n";
    std::cout << "wall time: " << st.wall_ms << " ms\n";
    std::cout << "composite bytes: " << st.bytes_moved << " (device gather " << st.device_ms << " ms)\n";
    return 0;
}

int write_out(const std::string& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    out << text;
    if (!out) {
        std::cerr << "error: StorageError: cannot write '" << path << "'\n";
        return 2;
    }
    return 0;
}

int cmd_plan(const Args& a) {
    if (!require(a, {"run", "failure-step", "out"})) return 1;
    std::string yaml;
    const long long step = std::stoll(a.kv.at("failure-step"));
    const int rc = text_call([&](char* b, size_t c, size_t* n) { return tg_recipe_from_manifests(a.kv.at("run").c_str(), step, b, c, n); }, yaml);
    if (rc != TG_OK) return report(rc);
    if (int w = write_out(a.kv.at("out"), yaml)) return w;
    std::cout << "recipe for failure at step " << step << " written to " << a.kv.at("out") << "\n" << yaml;
    return 0;
}

int cmd_select(const Args& a) {
    if (!require(a, {"snapshots", "out"})) return 1;
    const auto dirs = split_csv(a.kv.at("snapshots"));
    std::vector<const char*> ptrs;
    for (const auto& d : dirs) ptrs.push_back(d.c_str());
    const double rho = a.kv.count("rho") ? std::stod(a.kv.at("rho")) : 0.5;
    const std::vector<int32_t> devs = devices_of(a);
    std::vector<int32_t> src(4096);
    double gap = 0.0;
    std::string yaml;
    const int rc = text_call(
        [&](char* b, size_t c, size_t* n) {
            return tg_select_recipe(ptrs.data(), static_cast<int32_t>(ptrs.size()), rho, devs.data(),
                                    static_cast<int32_t>(devs.size()), b, c, n, src.data(), &gap);
        },
        yaml);
    if (rc != TG_OK) return report(rc);
    if (int w = write_out(a.kv.at("out"), yaml)) return w;
    std::cout << yaml << "# min boundary gap " << gap << "\n";
    return 0;
}

// select + merge in one call (tg_select_merge): the masters the scorer read stay on the
// device for the merge when they fit; --recipe-out keeps the recipe it chose.
int cmd_select_merge(const Args& a) {
    if (!require(a, {"snapshots", "out"})) return 1;
    const auto dirs = split_csv(a.kv.at("snapshots"));
    std::vector<const char*> ptrs;
    for (const auto& d : dirs) ptrs.push_back(d.c_str());
    const double rho = a.kv.count("rho") ? std::stod(a.kv.at("rho")) : 0.5;
    const std::vector<int32_t> devs = devices_of(a);
    tg_merge_options opt{};
    if (!merge_options_of(a, devs, opt)) return 1;
    std::vector<int32_t> src(4096);
    std::vector<char> yaml(1 << 20);
    size_t need = 0;
    double gap = 0.0;
    tg_merge_stats st{};
    const int rc = tg_select_merge(ptrs.data(), static_cast<int32_t>(ptrs.size()), rho, a.kv.at("out").c_str(), &opt, &st,
                                   yaml.data(), yaml.size(), &need, src.data(), &gap);
    if (rc != TG_OK) return report(rc);
    if (a.kv.count("recipe-out"))
        if (int w = write_out(a.kv.at("recipe-out"), std::string(yaml.data()))) return w;
    std::cout << "merged checkpoint written to " << a.kv.at("out") << "\n";
    std::cout << "composite bytes: " << st.bytes_moved << " (" << st.resident_bytes
              << " gathered from the scorer's device copies)\n";
    std::cout << "min boundary gap " << gap << "; wall time (merge): " << st.wall_ms << " ms\n";
    return 0;
}

int cmd_score(const Args& a) {
    if (!require(a, {"snapshots"})) return 1;
    const auto dirs = split_csv(a.kv.at("snapshots"));
    std::vector<const char*> ptrs;
    for (const auto& d : dirs) ptrs.push_back(d.c_str());
    const std::vector<int32_t> devs = devices_of(a);
    std::vector<double> scores(dirs.size() * 4096);
    int32_t M = 0;
    const int rc = tg_score_snapshots(ptrs.data(), static_cast<int32_t>(ptrs.size()), devs.data(), static_cast<int32_t>(devs.size()),
                                       nullptr, scores.data(), &M);
    if (rc != TG_OK) return report(rc);
    std::printf("{\"scores\":[");
    for (size_t p = 0; p + 1 < dirs.size(); ++p) {
        std::printf("%s[", p ? "," : "");
        for (int m = 0; m < M; ++m) std::printf("%s%.17g", m ? "," : "", scores[p * static_cast<size_t>(M) + static_cast<size_t>(m)]);
        std::printf("]");
    }
    std::printf("]}\n");
    return 0;
}

// R/tools/tailor_main.cpp:40-64 flags, on the device trainer; --strategy adds
// `magnitude` (in-situ update-magnitude selective checkpointing, --rho).
int cmd_train(const Args& a) {
    if (!require(a, {"config", "steps", "interval", "strategy", "ranks", "out"})) return 1;
    bool ok = false;
    const std::string text = read_file(a.kv.at("config"), &ok);
    if (!ok) {
        std::cerr << "error: MissingArtifact: cannot open '" << a.kv.at("config") << "'\n";
        return 1;
    }
    tg_model_spec spec{};
    if (int rc = tg_parse_config(text.c_str(), &spec); rc != TG_OK) return report(rc);
    static const std::map<std::string, int> kinds = {{"full", 0}, {"parity", 1}, {"filter", 2}, {"magnitude", 3}};
    const auto it = kinds.find(a.kv.at("strategy"));
    if (it == kinds.end()) {
        std::cerr << "error: RecipeError: unknown strategy '" << a.kv.at("strategy") << "'\n";
        return 1;
    }
    if (a.kv.count("grouping") && a.kv.at("grouping") != "fine") {
        std::cerr << "error: RecipeError: "
                  << (a.kv.at("grouping") == "coarse"
                          ? std::string("the device trainer writes fine grouping; convert with `tailor regroup --to coarse`")
                          : "unknown grouping '" + a.kv.at("grouping") + "' (expected fine or coarse)")
                  << "\n";
        return 1;
    }
    const auto num = [&](const char* k, double d) { return a.kv.count(k) ? std::stod(a.kv.at(k)) : d; };
    tg_train_config cfg{};
    cfg.total_steps = std::stoi(a.kv.at("steps"));
    cfg.num_ranks = std::stoi(a.kv.at("ranks"));
    cfg.interval = std::stoi(a.kv.at("interval"));
    cfg.strategy = it->second;
    cfg.head_count = static_cast<int32_t>(num("head", 2));
    cfg.tail_count = static_cast<int32_t>(num("tail", 2));
    cfg.sparse_multiple = static_cast<int32_t>(num("sparse-multiple", 5));
    cfg.device = static_cast<int32_t>(num("device", 0));
    cfg.lr = num("lr", 1e-3);
    cfg.weight_decay = num("weight-decay", 0.01);
    cfg.rho = num("rho", 0.5);
    int32_t written = 0;
    if (int rc = tg_train(&spec, &cfg, a.kv.at("out").c_str(), &written); rc != TG_OK) return report(rc);
    std::cout << "trained " << cfg.total_steps << " steps (" << a.kv.at("strategy") << ", interval " << cfg.interval
              << ", ranks " << cfg.num_ranks << "): " << written << " checkpoints in " << a.kv.at("out") << "\n";
    return 0;
}

// R/tools/tailor_main.cpp:105-110 (`resume --ckpt --steps --out`), on the device.
int cmd_resume(const Args& a) {
    if (!require(a, {"ckpt", "steps", "out"})) return 1;
    const int device = a.kv.count("device") ? std::stoi(a.kv.at("device")) : 0;
    const int steps = std::stoi(a.kv.at("steps"));
    int32_t written = 0;
    if (int rc = tg_resume(a.kv.at("ckpt").c_str(), steps, a.kv.at("out").c_str(), device, &written); rc != TG_OK)
        return report(rc);
    std::cout << "resumed from " << a.kv.at("ckpt") << " for " << steps << " steps\n";
    return 0;
}

int cmd_regroup(const Args& a) {
    if (!require(a, {"ckpt", "out"})) return 1;
    const std::string to = a.kv.count("to") ? a.kv.at("to") : "fine";
    if (to != "fine" && to != "coarse") {
        std::cerr << "error: RecipeError: --to must be fine or coarse\n";
        return 1;
    }
    tg_merge_options opt{};
    const std::vector<int32_t> devs = devices_of(a);
    opt.device = devs.front();
    opt.skip_verify = a.flags.count("no-verify") ? 1 : 0;
    opt.devices = devs.data();
    opt.num_devices = static_cast<int32_t>(devs.size());
    tg_merge_stats st{};
    const int rc = tg_regroup(a.kv.at("ckpt").c_str(), a.kv.at("out").c_str(), to == "fine" ? 1 : 0, &opt, &st);
    if (rc != TG_OK) return report(rc);
    std::cout << "regrouped (" << to << ") checkpoint written to " << a.kv.at("out") << " (" << st.bytes_moved
              << " bytes, " << st.wall_ms << " ms)\n";
    return 0;
}

int cmd_check(const Args& a) {
    if (!require(a, {"ckpt"})) return 1;
    const int device = a.kv.count("device") ? std::stoi(a.kv.at("device")) : 0;
    const int rc = tg_verify_checkpoint(a.kv.at("ckpt").c_str(), device);
    if (rc != TG_OK) return report(rc);
    std::cout << "ok\n";
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: tailor <merge|plan|select|select-merge|score|check|regroup|train|resume> [options]\n";
        return 1;
    }
    Args a;
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) {
            std::cerr << "unexpected argument " << k << "\n";
            return 1;
        }
        k = k.substr(2);
        if (const auto eq = k.find('='); eq != std::string::npos) a.kv[k.substr(0, eq)] = k.substr(eq + 1); // --key=value (CLI11)
        else if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) a.kv[k] = argv[++i];
        else a.flags.insert(k);
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "merge") return cmd_merge(a);
        if (cmd == "plan") return cmd_plan(a);
        if (cmd == "select") return cmd_select(a);
        if (cmd == "select-merge") return cmd_select_merge(a);
        if (cmd == "score") return cmd_score(a);
        if (cmd == "check") return cmd_check(a);
        if (cmd == "regroup") return cmd_regroup(a);
        if (cmd == "train") return cmd_train(a);
        if (cmd == "resume") return cmd_resume(a);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    std::cerr << "unknown subcommand " << cmd << "\n";
    return 1;
}
