// Parallel positional file I/O for the file-facing drop-ins (execute_merge,
// score_snapshots, verify). The reference reads each file through an
// istreambuf byte loop (R/src/container.cpp:193-199, ~0.25 GB/s per thread);
// here large reads are split into 16 MB pieces pulled by a small thread pool
// with pread, straight into pinned staging buffers.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace tailor {

struct ReadJob {
    int fd;
    std::uint8_t* dst;
    std::uint64_t bytes;
    std::uint64_t offset;
    int dfd = -1; // O_DIRECT descriptor of the same file (-1: buffered pread on fd)
};

// Executes all jobs (any order); the first failure is rethrown as StorageError.
// Jobs with a direct descriptor read with O_DIRECT: whole 4 KB blocks straight into
// `dst` where dst and the file offset are congruent mod 4 KB (the staging layouts
// of the merge lanes arrange that), the partial head/tail blocks and any
// incongruent job through an aligned bounce buffer.
void run_reads(const std::vector<ReadJob>& jobs, int threads, const std::string& what);

// Persistent reader threads over one FIFO of pieces (cut as run_reads cuts them). Each
// submit() is a batch with its own completion, so a lane can queue the reads of its next
// chunk while the current chunk's last pieces are still in flight: the device queue never
// drains at chunk boundaries. Buffers and descriptors of a batch must outlive its wait()
// (or drain()); the destructor finishes the queued pieces before joining.
// TAILOR_READ_LOOKAHEAD=0 (measurement): queue a chunk's reads only when the previous
// chunk's have completed, as a per-call read pool would.
bool read_lookahead();
// TAILOR_SYNC_CHECK=1 (diagnostics): synchronise each device step's stream right after its
// launch, so an asynchronous fault is reported by the step that caused it.
bool sync_check();
class ReadPool {
  public:
    explicit ReadPool(int threads);
    ~ReadPool();
    ReadPool(const ReadPool&) = delete;
    ReadPool& operator=(const ReadPool&) = delete;
    void grow(int threads); // never shrinks
    std::uint64_t submit(const std::vector<ReadJob>& jobs, const std::string& what);
    void wait(std::uint64_t ticket); // rethrows the batch's first failure (StorageError)
    void drain();                    // waits for every batch, dropping their errors

  private:
    struct Piece {
        std::uint64_t ticket = 0;
        ReadJob job{};
        std::shared_ptr<const std::string> what;
    };
    struct Batch {
        std::size_t remaining = 0;
        std::exception_ptr err;
        std::shared_ptr<const std::string> what;
    };
    void worker();
    std::mutex mu_;
    std::condition_variable work_, done_;
    std::deque<Piece> queue_;
    std::map<std::uint64_t, Batch> batches_;
    std::vector<std::thread> threads_;
    std::uint64_t next_ = 0;
    bool stop_ = false;
};

// ---- direct I/O ------------------------------------------------
// The reference reads every byte through the page cache with an istreambuf loop
// (R/src/container.cpp:193-207). Sources that are not in the page cache (a
// recovery reading checkpoints written long ago or elsewhere) are read here with
// O_DIRECT: deep parallel queues straight into pinned staging, no page-cache
// insertion, no readahead limits. Warm sources keep buffered reads (a memcpy from
// the page cache beats the device).
enum class IoMode : int {
    Auto = 0,        // O_DIRECT reads for source files mostly absent from the page cache
    Buffered = 1,    // everything through the page cache (the reference's behaviour)
    DirectRead = 2,  // O_DIRECT reads of every source file
    DirectRW = 3,    // + O_DIRECT writes of the output files (and direct re-verify reads)
};
constexpr std::uint64_t kDirectAlign = 4096;
// TAILOR_IO=auto|buffered|direct|direct-rw overrides `requested` when set.
IoMode io_mode_from_env(IoMode requested);
const char* io_mode_name(IoMode m);
// Fraction of the file's pages [off, off+len) resident in the page cache (mincore).
double page_cache_fraction(int fd, std::uint64_t off, std::uint64_t len);
// Whether a source read of [off, off+len) of `fd` should use O_DIRECT under `mode`.
bool want_direct_read(IoMode mode, int fd, std::uint64_t off, std::uint64_t len);
// open(path, O_RDONLY | O_DIRECT), -1 if the filesystem refuses O_DIRECT.
int open_direct_read(const std::string& path);

// Aligned host memory for O_DIRECT bounce buffers (page-aligned, freed with free()).
struct AlignedBuffer {
    std::uint8_t* p = nullptr;
    std::uint64_t n = 0;
    AlignedBuffer() = default;
    explicit AlignedBuffer(std::uint64_t bytes);
    ~AlignedBuffer();
    AlignedBuffer(const AlignedBuffer&) = delete;
    AlignedBuffer& operator=(const AlignedBuffer&) = delete;
};
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
