// Parallel pread, buffered or O_DIRECT (see tailor/io.hpp).
#include "tailor/io.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <fcntl.h>
#include <memory>
#include <sys/mman.h>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>
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

AlignedBuffer::AlignedBuffer(std::uint64_t bytes) : n(bytes) {
    void* q = nullptr;
    if (posix_memalign(&q, kDirectAlign, std::max<std::uint64_t>(bytes, kDirectAlign)) != 0)
        fail(ErrorKind::Storage, "out of host memory");
    p = static_cast<std::uint8_t*>(q);
}
AlignedBuffer::~AlignedBuffer() { std::free(p); }

IoMode io_mode_from_env(IoMode requested) {
    const char* v = std::getenv("TAILOR_IO");
    if (!v || !*v) return requested;
    const std::string s(v);
    if (s == "auto") return IoMode::Auto;
    if (s == "buffered") return IoMode::Buffered;
    if (s == "direct") return IoMode::DirectRead;
    if (s == "direct-rw") return IoMode::DirectRW;
    return requested;
}

const char* io_mode_name(IoMode m) {
    switch (m) {
        case IoMode::Auto: return "auto";
        case IoMode::Buffered: return "buffered";
        case IoMode::DirectRead: return "direct";
        case IoMode::DirectRW: return "direct-rw";
    }
    return "?";
}

double page_cache_fraction(int fd, std::uint64_t off, std::uint64_t len) {
    if (len == 0) return 1.0;
    // sampled: up to 256 pages spread over the range (mincore of a whole 15 GB
    // window would walk ~4 M page-cache entries)
    const std::uint64_t pg = static_cast<std::uint64_t>(::sysconf(_SC_PAGESIZE));
    const std::uint64_t a = off / pg * pg, b = off + len;
    const std::uint64_t pages = (b - a + pg - 1) / pg;
    const std::uint64_t probes = std::min<std::uint64_t>(pages, 256);
    void* m = ::mmap(nullptr, b - a, PROT_READ, MAP_SHARED, fd, static_cast<off_t>(a)); // lazy: no page touched
    if (m == MAP_FAILED) return 1.0; // unknown: keep the page cache
    std::size_t in = 0, seen = 0;
    for (std::uint64_t i = 0; i < probes; ++i) {
        unsigned char v = 0;
        if (::mincore(static_cast<std::uint8_t*>(m) + (pages * i / probes) * pg, pg, &v) == 0) {
            in += v & 1u;
            ++seen;
        }
    }
    ::munmap(m, b - a);
    return seen ? static_cast<double>(in) / static_cast<double>(seen) : 1.0;
}

bool want_direct_read(IoMode mode, int fd, std::uint64_t off, std::uint64_t len) {
    switch (mode) {
        case IoMode::Buffered: return false;
        case IoMode::DirectRead:
        case IoMode::DirectRW: return true;
        case IoMode::Auto: return page_cache_fraction(fd, off, len) < 0.5;
    }
    return false;
}

int open_direct_read(const std::string& path) { return ::open(path.c_str(), O_RDONLY | O_DIRECT); }

namespace {

// Bounce buffers of the direct path, reused across calls (a 16 MB piece plus the
// two partial blocks around it).
constexpr std::uint64_t kPiece = 16ull << 20;
constexpr std::uint64_t kBounce = kPiece + 2 * kDirectAlign;

struct BouncePool {
    std::mutex mu;
    std::vector<std::unique_ptr<AlignedBuffer>> free;
    std::unique_ptr<AlignedBuffer> take() {
        std::lock_guard<std::mutex> lk(mu);
        if (free.empty()) return std::make_unique<AlignedBuffer>(kBounce);
        auto b = std::move(free.back());
        free.pop_back();
        return b;
    }
    void give(std::unique_ptr<AlignedBuffer> b) {
        std::lock_guard<std::mutex> lk(mu);
        free.push_back(std::move(b));
    }
};
BouncePool& bounce_pool() {
    static BouncePool* p = new BouncePool(); // process lifetime
    return *p;
}

// pread of n bytes, stopping early only at EOF; returns the bytes read
std::uint64_t pread_full(int fd, std::uint8_t* dst, std::uint64_t n, std::uint64_t off, const std::string& what) {
    std::uint64_t got = 0;
    while (got < n) {
        const ssize_t r = ::pread(fd, dst + got, n - got, static_cast<off_t>(off + got));
        if (r < 0) fail(ErrorKind::Storage, "read failed for '" + what + "'");
        if (r == 0) break;
        got += static_cast<std::uint64_t>(r);
    }
    return got;
}

void read_buffered(const ReadJob& p, const std::string& what) {
    if (pread_full(p.fd, p.dst, p.bytes, p.offset, what) != p.bytes) fail(ErrorKind::Storage, "read failed for '" + what + "'");
}

// O_DIRECT read of [offset, offset+bytes) into dst (either may be unaligned).
void read_direct(const ReadJob& p, const std::string& what) {
    constexpr std::uint64_t A = kDirectAlign;
    const std::uint64_t lo = p.offset, hi = p.offset + p.bytes;
    const std::uint64_t a0 = lo / A * A, a1 = (hi + A - 1) / A * A;
    std::unique_ptr<AlignedBuffer> bounce;
    const auto via_bounce = [&](std::uint64_t blo, std::uint64_t bhi) { // aligned blocks -> copy the overlap
        if (!bounce) bounce = bounce_pool().take();
        const std::uint64_t got = pread_full(p.dfd, bounce->p, bhi - blo, blo, what);
        const std::uint64_t x = std::max(lo, blo), y = std::min(hi, bhi);
        if (got < y - blo) fail(ErrorKind::Storage, "read failed for '" + what + "' (short direct read)");
        std::memcpy(p.dst + (x - lo), bounce->p + (x - blo), y - x);
    };
    const bool congruent = (reinterpret_cast<std::uintptr_t>(p.dst) - lo) % A == 0;
    const std::uint64_t m0 = (lo + A - 1) / A * A, m1 = hi / A * A; // whole blocks inside [lo, hi)
    if (congruent && m0 < m1) {
        if (lo < m0) via_bounce(a0, m0);
        if (pread_full(p.dfd, p.dst + (m0 - lo), m1 - m0, m0, what) != m1 - m0)
            fail(ErrorKind::Storage, "read failed for '" + what + "' (short direct read)");
        if (m1 < hi) via_bounce(m1, a1);
    } else {
        for (std::uint64_t b = a0; b < a1; b += kPiece) via_bounce(b, std::min(a1, b + kPiece));
    }
    if (bounce) bounce_pool().give(std::move(bounce));
}

} // namespace

namespace {
// O_DIRECT reads go to the device, not the page cache: queue depth is what they need
// (tools/disk_probe reaches the device's bandwidth with 32 readers), so direct jobs are
// cut into 4 MB pieces served by at least 4 threads
constexpr std::uint64_t kDirectPiece = 4ull << 20;

bool cut_pieces(const std::vector<ReadJob>& jobs, std::vector<ReadJob>& pieces) {
    bool direct = false;
    for (const auto& j : jobs) {
        const std::uint64_t piece = j.dfd >= 0 ? kDirectPiece : kPiece;
        direct = direct || j.dfd >= 0;
        for (std::uint64_t at = 0; at < j.bytes; at += piece)
            pieces.push_back({j.fd, j.dst + at, std::min(piece, j.bytes - at), j.offset + at, j.dfd});
    }
    return direct;
}

void read_one(const ReadJob& p, const std::string& what) {
    if (p.dfd >= 0) read_direct(p, what);
    else read_buffered(p, what);
}
} // namespace

bool sync_check() {
    static const bool on = [] {
        const char* v = std::getenv("TAILOR_SYNC_CHECK");
        return v && *v == '1';
    }();
    return on;
}

bool read_lookahead() {
    static const bool on = [] {
        const char* v = std::getenv("TAILOR_READ_LOOKAHEAD");
        return !(v && *v == '0');
    }();
    return on;
}

// ---- ReadPool ---------------------------------------------------------------------
ReadPool::ReadPool(int threads) { grow(threads); }

ReadPool::~ReadPool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    work_.notify_all();
    for (auto& t : threads_) t.join();
}

void ReadPool::grow(int threads) {
    std::lock_guard<std::mutex> lk(mu_);
    while (static_cast<int>(threads_.size()) < threads) threads_.emplace_back([this] { worker(); });
}

void ReadPool::worker() {
    for (;;) {
        Piece pc;
        {
            std::unique_lock<std::mutex> lk(mu_);
            work_.wait(lk, [&] { return stop_ || !queue_.empty(); });
            if (queue_.empty()) return; // stop_ with nothing left
            pc = std::move(queue_.front());
            queue_.pop_front();
        }
        std::exception_ptr err;
        try {
            read_one(pc.job, *pc.what);
        } catch (...) {
            err = std::current_exception();
        }
        std::lock_guard<std::mutex> lk(mu_);
        Batch& b = batches_[pc.ticket];
        if (err && !b.err) b.err = err;
        if (--b.remaining == 0) done_.notify_all();
    }
}

std::uint64_t ReadPool::submit(const std::vector<ReadJob>& jobs, const std::string& what) {
    std::vector<ReadJob> pieces;
    if (cut_pieces(jobs, pieces)) grow(4);
    std::lock_guard<std::mutex> lk(mu_);
    const std::uint64_t ticket = next_++;
    Batch& b = batches_[ticket];
    b.remaining = pieces.size();
    b.what = std::make_shared<const std::string>(what);
    for (auto& p : pieces) queue_.push_back({ticket, p, b.what});
    work_.notify_all();
    return ticket;
}

void ReadPool::wait(std::uint64_t ticket) {
    std::unique_lock<std::mutex> lk(mu_);
    auto it = batches_.find(ticket);
    if (it == batches_.end()) return;
    done_.wait(lk, [&] { return it->second.remaining == 0; });
    const std::exception_ptr err = it->second.err;
    batches_.erase(it);
    lk.unlock();
    if (err) std::rethrow_exception(err);
}

void ReadPool::drain() {
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] {
        for (const auto& [t, b] : batches_)
            if (b.remaining) return false;
        return true;
    });
    batches_.clear();
}

void run_reads(const std::vector<ReadJob>& jobs, int threads, const std::string& what) {
    std::vector<ReadJob> pieces;
    if (cut_pieces(jobs, pieces)) threads = std::max(threads, 4);
    const auto read_one = [&](const ReadJob& p) { tailor::read_one(p, what); };
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
