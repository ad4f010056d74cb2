// INTEGRATION.md §1, compiled: the reference's `tailor merge` subcommand
// (R/tools/tailor_main.cpp:75-103) with its body replaced by the B200 drop-in
// (tg_execute_merge), built in the reference's own context — its headers
// (R/include/tailor/errors.hpp, container.hpp) and library (oracle/_ref/libtailor_ref.a
// for read_file_bytes) — exactly what a maintainer would add to the reference.
// Same flags, same --json object, same error -> exit-code mapping
// (R/tools/tailor_main.cpp:351-357). TEST INFRASTRUCTURE: built by
// tests/integration/Makefile into tests/integration/_build/.
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>

#include <json.hpp>

#include "tailor/container.hpp" // reference: read_file_bytes
#include "tailor/errors.hpp"    // reference: TailorError, ErrorKind
#include "tailor_b200.h"

using nlohmann::json;
using namespace tailor;

namespace {

// TG_E_* 1..11 follow the reference's ErrorKind declaration order; 12 (device) and 100
// (internal) are internal errors (exit 2), i.e. Storage-class.
[[noreturn]] void throw_last(int rc) {
    std::string msg = tg_last_error();
    if (const auto c = msg.find(": "); c != std::string::npos) msg = msg.substr(c + 2); // TailorError re-prefixes the kind
    const ErrorKind kind = (rc >= 1 && rc <= 11) ? static_cast<ErrorKind>(rc - 1) : ErrorKind::Storage;
    throw TailorError(kind, msg);
}

int cmd_merge(const std::string& recipe_path, const std::string& out, int workers, bool uncached, bool as_json) {
    const auto bytes = read_file_bytes(recipe_path); // the reference's helper, unchanged
    const std::string yaml(bytes.begin(), bytes.end());
    // num_ranks / sources for the report, as the reference prints them from its MergePlan
    std::string plan_text(1 << 16, '\0');
    size_t need = 0;
    int rc = tg_resolve_plan(yaml.c_str(), plan_text.data(), plan_text.size(), &need);
    if (rc != TG_OK && need > plan_text.size()) {
        plan_text.assign(need, '\0');
        rc = tg_resolve_plan(yaml.c_str(), plan_text.data(), plan_text.size(), &need);
    }
    if (rc != TG_OK) throw_last(rc);
    const json plan = json::parse(plan_text.c_str());
    tg_merge_options opt{};
    opt.workers = workers;
    opt.uncached = uncached ? 1 : 0; // zero-initialised: device 0, re-verify on
    tg_merge_stats st{};
    if ((rc = tg_execute_merge(yaml.c_str(), out.c_str(), &opt, &st)) != TG_OK) throw_last(rc);
    const int num_ranks = plan["num_ranks"].get<int>();
    const std::size_t num_sources = plan["sources"].size();
    if (as_json) {
        std::cout << json{{"out", out},
                          {"num_ranks", num_ranks},
                          {"num_sources", num_sources},
                          {"shard_files_read", st.shard_files_read},
                          {"weight_files_read", st.weight_files_read},
                          {"wall_ms", st.wall_ms}}
                         .dump()
                  << "\n";
        return 0;
    }
    std::cout << "merged checkpoint written to " << out << "\n";
    std::cout << "sources: " << num_sources << "  ranks: " << num_ranks << "\n";
    std::cout << "optimizer shard files read: " << st.shard_files_read << " (bound " << num_ranks << " x " << num_sources
              << " = " << num_ranks * static_cast<int>(num_sources) << " cached)\n";
    std::cout << "weight files read: " << st.weight_files_read << "\n";
    std::cout << "wall time: " << st.wall_ms << " ms\n";
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    // `merge --recipe R --out O [--workers W] [--uncached] [--json]` (R/tools/tailor_main.cpp:291-299)
    std::string recipe, out;
    int workers = 0;
    bool uncached = false, as_json = false;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "merge") continue;
        if (a == "--recipe" && i + 1 < argc) recipe = argv[++i];
        else if (a == "--out" && i + 1 < argc) out = argv[++i];
        else if (a == "--workers" && i + 1 < argc) workers = std::atoi(argv[++i]);
        else if (a == "--uncached") uncached = true;
        else if (a == "--json") as_json = true;
        else {
            std::cerr << "unknown argument " << a << "\n";
            return 1;
        }
    }
    try {
        return cmd_merge(recipe, out, workers, uncached, as_json);
    } catch (const TailorError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return e.is_user_error() ? 1 : 2;
    } catch (const std::exception& e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return 2;
    }
}
