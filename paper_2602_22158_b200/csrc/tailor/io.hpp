// Parallel positional file I/O for the file-facing drop-ins (execute_merge,
// score_snapshots, verify). The reference reads each file through an
// istreambuf byte loop (R/src/container.cpp:193-199, ~0.25 GB/s per thread);
// here large reads are split into 16 MB pieces pulled by a small thread pool
// with pread, straight into pinned staging buffers.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace tailor {

struct ReadJob {
    int fd;
    std::uint8_t* dst;
    std::uint64_t bytes;
    std::uint64_t offset;
};

// Executes all jobs (any order); the first failure is rethrown as StorageError.
void run_reads(const std::vector<ReadJob>& jobs, int threads, const std::string& what);
// Default worker count for host I/O: hardware threads, capped at 16.
int io_threads();

// Phase timer for the file-facing paths: prints "[tailor] <name> <ms>" to
// stderr at scope exit when TAILOR_TRACE=1 (no cost otherwise).
class PhaseTimer {
  public:
    explicit PhaseTimer(const char* name);
    ~PhaseTimer();
    PhaseTimer(const PhaseTimer&) = delete;
    PhaseTimer& operator=(const PhaseTimer&) = delete;

  private:
    const char* name_;
    double t0_ = 0.0;
    bool on_;
};

// Adds the scope's wall time (ms) to `sink`.
class ScopedAccum {
  public:
    explicit ScopedAccum(double& sink);
    ~ScopedAccum();
    ScopedAccum(const ScopedAccum&) = delete;
    ScopedAccum& operator=(const ScopedAccum&) = delete;

  private:
    double& sink_;
    double t0_;
};
// Prints "[tailor] <name> <ms> ms" / "[tailor] <name> <count>" when TAILOR_TRACE=1.
void trace_value(const char* name, double ms);
void trace_count(const char* name, double count);
bool trace_enabled();
// Monotonic clock in ms (for phase breakdowns).
double clock_ms();

} // namespace tailor
