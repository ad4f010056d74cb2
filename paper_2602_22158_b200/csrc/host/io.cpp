// Parallel pread (see tailor/io.hpp).
#include "tailor/io.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <unistd.h>

#include "tailor/errors.hpp"

namespace tailor {

namespace {
double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
bool trace_on() {
    static const bool on = [] {
        const char* v = std::getenv("TAILOR_TRACE");
        return v && *v && *v != '0';
    }();
    return on;
}
} // namespace

PhaseTimer::PhaseTimer(const char* name) : name_(name), on_(trace_on()) {
    if (on_) t0_ = now_ms();
}

PhaseTimer::~PhaseTimer() {
    if (on_) std::fprintf(stderr, "[tailor] %s %.2f ms\n", name_, now_ms() - t0_);
}

ScopedAccum::ScopedAccum(double& sink) : sink_(sink), t0_(now_ms()) {}
ScopedAccum::~ScopedAccum() { sink_ += now_ms() - t0_; }

bool trace_enabled() { return trace_on(); }
double clock_ms() { return now_ms(); }

void trace_count(const char* name, double count) {
    if (trace_on()) std::fprintf(stderr, "[tailor] %s %g\n", name, count);
}

void trace_value(const char* name, double ms) {
    if (trace_on()) std::fprintf(stderr, "[tailor] %s %.2f ms\n", name, ms);
}

int io_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return static_cast<int>(std::clamp<unsigned>(hw ? hw : 4u, 1u, 16u));
}

void run_reads(const std::vector<ReadJob>& jobs, int threads, const std::string& what) {
    constexpr std::uint64_t kPiece = 16ull << 20;
    std::vector<ReadJob> pieces;
    for (const auto& j : jobs)
        for (std::uint64_t at = 0; at < j.bytes; at += kPiece)
            pieces.push_back({j.fd, j.dst + at, std::min(kPiece, j.bytes - at), j.offset + at});
    const auto read_one = [&](const ReadJob& p) {
        std::uint64_t got = 0;
        while (got < p.bytes) {
            const ssize_t r = ::pread(p.fd, p.dst + got, p.bytes - got, static_cast<off_t>(p.offset + got));
            if (r <= 0) fail(ErrorKind::Storage, "read failed for '" + what + "'");
            got += static_cast<std::uint64_t>(r);
        }
    };
    const int n = std::max(1, std::min<int>(threads, static_cast<int>(pieces.size())));
    if (n == 1) {
        for (const auto& p : pieces) read_one(p);
        return;
    }
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex mu;
    std::vector<std::thread> pool;
    pool.reserve(static_cast<std::size_t>(n));
    for (int t = 0; t < n; ++t)
        pool.emplace_back([&] {
            for (std::size_t i = next.fetch_add(1); i < pieces.size(); i = next.fetch_add(1)) {
                try {
                    read_one(pieces[i]);
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!err) err = std::current_exception();
                }
            }
        });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

} // namespace tailor
