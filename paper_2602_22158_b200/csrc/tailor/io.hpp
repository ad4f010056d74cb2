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

} // namespace tailor
