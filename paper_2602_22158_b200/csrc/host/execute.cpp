// execute_merge — the drop-in for R/src/merge.cpp:226-357 on files.
//
// Same contract: refuse a non-empty out_dir, validate everything before the
// first write, output bytes identical to the reference (headers and sidecars
// render through the same JSON library; payload bytes are copied exactly), a
// full re-verify before returning, MergeStats counting files read. Different
// mechanism: only the byte ranges the composite needs are read from each
// source (the reference loads every shard file whole), staged through pinned
// memory, assembled by the device gather kernel, and streamed back out — the
// output files in parallel lanes (one file per lane, 3-slot pipeline each); the
// re-verify is the device kernel K6.
#include <algorithm>
#include <atomic>
#include <exception>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <fcntl.h>
#include <filesystem>
#include <functional>
#include <future>
#include <map>
#include <mutex>
#include <thread>
#include <unistd.h>

#include "tailor/engine.hpp"
#include "tailor/errors.hpp"
#include "tailor/io.hpp"

namespace tailor {

namespace fs = std::filesystem;

namespace {

struct Fd {
    int fd = -1;
    explicit Fd(const fs::path& p, int flags, mode_t mode = 0644) : fd(::open(p.c_str(), flags, mode)) {}
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

void pwrite_all(int fd, const std::uint8_t* src, std::uint64_t n, std::uint64_t off, const std::string& what) {
    std::uint64_t put = 0;
    while (put < n) {
        const ssize_t r = ::pwrite(fd, src + put, n - put, static_cast<off_t>(off + put));
        if (r <= 0) fail(ErrorKind::Storage, "write failed for '" + what + "'");
        put += static_cast<std::uint64_t>(r);
    }
}

std::uint64_t align16(std::uint64_t x) { return (x + 15) & ~15ull; }
std::uint64_t floor_blk(std::uint64_t x) { return x / kDirectAlign * kDirectAlign; }
std::uint64_t ceil_blk(std::uint64_t x) { return (x + kDirectAlign - 1) / kDirectAlign * kDirectAlign; }

// One lane of the file pipeline: assembles whole output container files, one
// chunk at a time through kSlots slots: the lane thread preads chunk i while the
// GPU runs chunk i-1 (H2D -> K2 -> D2H on the slot's stream) and the lane's
// writer thread pwrites chunk i-2. Lanes run on their own threads, each writing
// a different file: buffered writes to ONE file serialise on its inode lock
// (tools/write_probe.cpp: 8 threads on one file ~4.7 GB/s, on 8 files 20-30 GB/s
// on the B200 host), so the parallelism is across files.
// Direct I/O (IoMode): a source window read with O_DIRECT is staged at a pinned
// offset congruent to its file offset mod 4 KB, so whole blocks land in place;
// with O_DIRECT writes the chunk grid follows the output file's 4 KB blocks
// (chunk 0 carries the tail of the header) and the file is truncated to size.
class FileAssembler {
  public:
    static constexpr int kSlots = 3;

    FileAssembler(int read_threads, bool uncached, std::uint64_t chunk, IoMode io = IoMode::Buffered)
        : uncached_(uncached), chunk_(chunk), io_(io), pool_(std::max(1, read_threads)) {
        for (auto& s : stream_) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
        for (int i = 0; i < kSlots; ++i) {
            cuda_check(cudaEventCreate(&ev0_[i]), "event");
            cuda_check(cudaEventCreate(&ev1_[i]), "event");
        }
    }
    ~FileAssembler() {
        for (auto& s : stream_) cudaStreamDestroy(s);
        for (int i = 0; i < kSlots; ++i) {
            cudaEventDestroy(ev0_[i]);
            cudaEventDestroy(ev1_[i]);
        }
    }

    double device_ms = 0.0, read_ms = 0.0, wait_ms = 0.0, write_ms = 0.0;
    std::uint64_t bytes = 0, direct_read_bytes = 0, direct_write_bytes = 0;
    void set_read_threads(int n) { pool_.grow(std::max(1, n)); }

    // resident[w] (may be empty): window-relative byte ranges of window w already on the
    // device (ResidentSources); those bytes are gathered from there, not read.
    void assemble(const PartitionPlan& pp, const std::vector<fs::path>& window_files, const fs::path& out_path,
                  const std::vector<std::vector<ResidentRange>>& resident = {}) {
        Fd out(out_path, O_WRONLY | O_CREAT | O_TRUNC);
        if (out.fd < 0) fail(ErrorKind::Storage, "cannot create '" + out_path.string() + "'");
        const std::string prefix = pp.out.prefix();
        const std::uint64_t base = pp.out.payload_offset();
        // Payload offsets of each window inside its source file; which windows read direct.
        std::vector<std::uint64_t> file_off(pp.windows.size());
        std::vector<std::unique_ptr<Fd>> fds(pp.windows.size()), dfds(pp.windows.size());
        std::vector<char> direct(pp.windows.size(), 0);
        for (std::size_t w = 0; w < pp.windows.size(); ++w) {
            if (pp.windows[w].container == kZeroContainer) continue; // zero fill: no source file
            file_off[w] = source_payload_offset(window_files[w]) + pp.windows[w].lo;
            if (!uncached_) {
                fds[w] = std::make_unique<Fd>(window_files[w], O_RDONLY);
                if (fds[w]->fd < 0) fail(ErrorKind::MissingArtifact, "cannot open '" + window_files[w].string() + "'");
                if (io_ != IoMode::Buffered &&
                    want_direct_read(io_, fds[w]->fd, file_off[w], pp.windows[w].hi - pp.windows[w].lo)) {
                    dfds[w] = std::make_unique<Fd>(window_files[w], O_RDONLY | O_DIRECT);
                    direct[w] = dfds[w]->fd >= 0; // the filesystem may refuse O_DIRECT: buffered then
                }
            }
        }
        // O_DIRECT output: a second descriptor on the same file; every write is whole blocks
        std::unique_ptr<Fd> dout;
        bool dwrite = io_ == IoMode::DirectRW && pp.dst_hi > pp.dst_lo;
        if (dwrite) {
            dout = std::make_unique<Fd>(out_path, O_WRONLY | O_DIRECT);
            dwrite = dout->fd >= 0;
        }
        const std::uint64_t head = dwrite ? base % kDirectAlign : 0; // header bytes that ride in chunk 0
        HostMergeChunks plan(pp, chunk_, dwrite ? chunk_ - head : chunk_, file_off, direct, resident);
        for (int i = 0; i < kSlots; ++i) {
            // one pinned buffer per slot carries the chunk both ways: the D2H of the
            // gathered chunk lands in it after its H2D has completed (same stream)
            pin_io_[i].resize(std::max<std::uint64_t>(16, std::max(plan.max_staging, ceil_blk(plan.max_out + head))));
            dwrite = dwrite && reinterpret_cast<std::uintptr_t>(pin_io_[i].get()) % kDirectAlign == 0;
            d_in_[i].resize(std::max<std::uint64_t>(16, plan.max_staging));
            d_out_[i].resize(std::max<std::uint64_t>(16, plan.max_out));
            d_segs_[i].resize(std::max<std::size_t>(1, plan.max_segs) * sizeof(dev::GatherSeg));
            pin_segs_[i].resize(std::max<std::size_t>(1, plan.max_segs) * sizeof(dev::GatherSeg));
        }
        if (dwrite) { // the header's whole blocks now; its tail goes out with chunk 0
            const std::uint64_t whole = floor_blk(base);
            if (whole) {
                AlignedBuffer hb(whole);
                std::memcpy(hb.p, prefix.data(), whole);
                pwrite_all(dout->fd, hb.p, whole, 0, out_path.string());
            }
        } else {
            pwrite_all(out.fd, reinterpret_cast<const std::uint8_t*>(prefix.data()), prefix.size(), 0, out_path.string());
        }

        // Writer: takes chunks in order, waits for the slot's stream, pwrites,
        // frees the slot. `written` counts chunks fully on disk (page cache).
        std::mutex mu;
        std::condition_variable cv;
        std::size_t issued = 0, written = 0;
        std::exception_ptr werr;
        std::thread writer([&] {
            try {
                for (std::size_t ci = 0; ci < plan.chunks.size(); ++ci) {
                    {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [&] { return issued > ci || werr; });
                        if (werr) return;
                    }
                    const int slot = static_cast<int>(ci % kSlots);
                    {
                        ScopedAccum acc(wait_ms);
                        cuda_check(cudaStreamSynchronize(stream_[slot]), "sync");
                    }
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, ev0_[slot], ev1_[slot]);
                    device_ms += ms;
                    const auto& c = plan.chunks[ci];
                    {
                        ScopedAccum acc(write_ms);
                        if (dwrite) {
                            const std::uint64_t h = ci == 0 ? head : 0;
                            if (h) std::memcpy(pin_io_[slot].get(), prefix.data() + (base - head), h);
                            const std::uint64_t n = ceil_blk(h + c.hi - c.lo);
                            pwrite_all(dout->fd, pin_io_[slot].get(), n, base + c.lo - h, out_path.string());
                            direct_write_bytes += n;
                        } else {
                            pwrite_all(out.fd, pin_io_[slot].get(), c.hi - c.lo, base + c.lo, out_path.string());
                        }
                    }
                    std::lock_guard<std::mutex> lk(mu);
                    written = ci + 1;
                    cv.notify_all();
                }
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                werr = std::current_exception();
                cv.notify_all();
            }
        });
        // Reads run one chunk ahead on the lane's reader pool: chunk ci+1's pieces are
        // queued (its slot free once chunk ci+1-kSlots is written) before chunk ci's
        // reads are waited for, so the device queue does not drain between chunks.
        std::exception_ptr rerr;
        std::uint64_t ticket[kSlots] = {};
        const auto slot_free = [&](std::size_t ci) { // the slot's previous chunk is written
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return written + kSlots > ci || werr; });
            return !werr;
        };
        // A chunk's reads are queued as soon as its slot is free: before the previous chunk's
        // reads are waited for when the slot is already free then (no blocking for it), else
        // at the top of its own iteration (as without lookahead).
        const auto slot_is_free = [&](std::size_t ci) {
            std::lock_guard<std::mutex> lk(mu);
            return written + kSlots > ci;
        };
        const bool lookahead = read_lookahead();
        try {
            const std::size_t nchunks = plan.chunks.size();
            std::size_t queued = 0; // chunks [0, queued) have their reads queued
            for (std::size_t ci = 0; ci < nchunks; ++ci) {
                const int slot = static_cast<int>(ci % kSlots);
                if (queued == ci) {
                    if (!slot_free(ci)) break;
                    ticket[slot] = queue_reads(plan.chunks[ci], pp, window_files, file_off, fds, dfds, slot, out_path);
                    queued = ci + 1;
                }
                if (lookahead && ci + 1 < nchunks && queued == ci + 1 && slot_is_free(ci + 1)) {
                    const int ns = static_cast<int>((ci + 1) % kSlots);
                    ticket[ns] = queue_reads(plan.chunks[ci + 1], pp, window_files, file_off, fds, dfds, ns, out_path);
                    queued = ci + 2;
                }
                {
                    ScopedAccum acc(read_ms);
                    pool_.wait(ticket[slot]);
                }
                launch_chunk(plan.chunks[ci], slot, ci == 0 ? head : 0);
                std::lock_guard<std::mutex> lk(mu);
                issued = ci + 1;
                cv.notify_all();
            }
        } catch (...) {
            rerr = std::current_exception();
        }
        pool_.drain(); // no read may still target a slot or descriptor of this file
        for (auto& o : opened_) o.clear();
        {
            std::lock_guard<std::mutex> lk(mu);
            if (rerr && !werr) werr = rerr; // stops the writer
            cv.notify_all();
        }
        writer.join();
        for (auto& st : stream_) cudaStreamSynchronize(st);
        if (rerr) std::rethrow_exception(rerr);
        if (werr) std::rethrow_exception(werr);
        if (plan.chunks.empty() && pp.out.payload_bytes != 0) fail(ErrorKind::Consistency, "empty merge plan");
        if (dwrite && ::ftruncate(out.fd, static_cast<off_t>(base + pp.out.payload_bytes)) != 0) // drop the last block's tail
            fail(ErrorKind::Storage, "cannot truncate '" + out_path.string() + "'");
    }

  private:
    struct ChunkPlan;

    // Queues one chunk's source reads into the slot's pinned staging on the lane's
    // reader pool (uncached mode re-opens the source file per read, as the reference
    // reloads a shard per group copy; those descriptors live in the slot until its next
    // use, after the reads were waited for).
    std::uint64_t queue_reads(const ChunkPlan& c, const PartitionPlan& pp, const std::vector<fs::path>& window_files,
                              const std::vector<std::uint64_t>& file_off, const std::vector<std::unique_ptr<Fd>>& fds,
                              const std::vector<std::unique_ptr<Fd>>& dfds, int slot, const fs::path& out_path) {
        auto& opened = opened_[slot];
        opened.clear();
        std::vector<ReadJob> jobs;
        for (const auto& rd : c.reads) {
            int fd;
            if (pp.windows[rd.w].container == kZeroContainer) {
                std::memset(pin_io_[slot].get() + rd.at, 0, rd.b - rd.a);
                continue;
            }
            if (uncached_) {
                opened.push_back(std::make_unique<Fd>(window_files[rd.w], O_RDONLY));
                if (opened.back()->fd < 0) fail(ErrorKind::MissingArtifact, "cannot open '" + window_files[rd.w].string() + "'");
                fd = opened.back()->fd;
            } else {
                fd = fds[rd.w]->fd;
            }
            const int dfd = !uncached_ && dfds[rd.w] && dfds[rd.w]->fd >= 0 ? dfds[rd.w]->fd : -1;
            if (dfd >= 0) direct_read_bytes += rd.b - rd.a;
            jobs.push_back({fd, pin_io_[slot].get() + rd.at, rd.b - rd.a, file_off[rd.w] + rd.a, dfd});
        }
        return pool_.submit(jobs, out_path.string());
    }

    // The slot's reads are complete: H2D -> K2 -> D2H on the slot's stream.
    void launch_chunk(const ChunkPlan& c, int slot, std::uint64_t d2h_shift) {
        cudaStream_t s = stream_[slot];
        cuda_check(cudaMemcpyAsync(d_in_[slot].get(), pin_io_[slot].get(), c.staging, cudaMemcpyHostToDevice, s), "H2D");
        auto* segs = reinterpret_cast<dev::GatherSeg*>(pin_segs_[slot].get());
        for (std::size_t i = 0; i < c.segs.size(); ++i) {
            segs[i] = c.segs[i];
            if (!c.abs[i]) segs[i].src = d_in_[slot].get() + reinterpret_cast<std::uintptr_t>(c.segs[i].src);
        }
        cuda_check(cudaMemcpyAsync(d_segs_[slot].get(), segs, c.segs.size() * sizeof(dev::GatherSeg), cudaMemcpyHostToDevice, s),
                   "segs");
        cuda_check(cudaEventRecord(ev0_[slot], s), "event");
        cuda_check(dev::launch_gather(d_segs_[slot].get<dev::GatherSeg>(), static_cast<std::uint32_t>(c.segs.size()),
                                      d_out_[slot].get(), c.hi - c.lo, dev::kGatherAuto, c.bulk_ok, s),
                   "gather");
        cuda_check(cudaEventRecord(ev1_[slot], s), "event");
        if (sync_check()) cuda_check(cudaStreamSynchronize(s), "gather (TAILOR_SYNC_CHECK)");
        cuda_check(cudaMemcpyAsync(pin_io_[slot].get() + d2h_shift, d_out_[slot].get(), c.hi - c.lo, cudaMemcpyDeviceToHost, s),
                   "D2H");
        bytes += c.hi - c.lo;
    }

    struct Read {
        std::uint32_t w;
        std::uint64_t a, b, at;
    };
    struct ChunkPlan {
        std::uint64_t lo, hi, staging = 0;
        std::vector<Read> reads;
        std::vector<dev::GatherSeg> segs; // src = staging offset, or a device address where abs[i]
        std::vector<std::uint8_t> abs;    // 1: the segment reads resident device bytes
        bool bulk_ok = true;
    };
    struct HostMergeChunks {
        std::vector<ChunkPlan> chunks;
        std::uint64_t max_staging = 0, max_out = 0;
        std::size_t max_segs = 0;
        // first: the size of chunk 0 (chunk, or less so that later chunks start on
        // 4 KB blocks of the output file); direct[w]: window w is read with O_DIRECT,
        // so its reads are staged congruent to file_off[w] + src mod 4 KB
        HostMergeChunks(const PartitionPlan& pp, std::uint64_t chunk, std::uint64_t first,
                        const std::vector<std::uint64_t>& file_off, const std::vector<char>& direct,
                        const std::vector<std::vector<ResidentRange>>& resident) {
            const std::uint64_t total = pp.dst_hi - pp.dst_lo;
            first = std::max<std::uint64_t>(1, first);
            std::size_t si = 0;
            for (std::uint64_t lo = 0; lo < total; lo = lo == 0 ? first : lo + chunk) {
                ChunkPlan c;
                c.lo = lo;
                c.hi = std::min(total, lo == 0 ? first : lo + chunk);
                struct P {
                    std::uint32_t w;
                    std::uint64_t src, dst, n;
                    const std::uint8_t* dev = nullptr; // resident: gathered from here, not read
                };
                std::vector<P> ps;
                const auto push = [&](std::uint32_t w, std::uint64_t src, std::uint64_t dst, std::uint64_t n) {
                    // split at the window's resident ranges (sorted, disjoint)
                    if (w < resident.size())
                        for (const auto& r : resident[w]) {
                            if (r.hi <= src) continue;
                            if (r.lo >= src + n) break;
                            if (r.lo > src) { // a non-resident gap first
                                const std::uint64_t g = r.lo - src;
                                ps.push_back({w, src, dst, g});
                                src += g, dst += g, n -= g;
                            }
                            const std::uint64_t k = std::min(n, r.hi - src);
                            ps.push_back({w, src, dst, k, r.dev + (src - r.lo)});
                            src += k, dst += k, n -= k;
                            if (!n) return;
                        }
                    ps.push_back({w, src, dst, n});
                };
                while (si < pp.segments.size() && pp.segments[si].dst_off + pp.segments[si].bytes - pp.dst_lo <= c.lo) ++si;
                for (std::size_t j = si; j < pp.segments.size(); ++j) {
                    const auto& s = pp.segments[j];
                    const std::uint64_t d0 = s.dst_off - pp.dst_lo, d1 = d0 + s.bytes;
                    if (d0 >= c.hi) break;
                    const std::uint64_t a = std::max(d0, c.lo), b = std::min(d1, c.hi);
                    if (a < b) push(s.window, s.src_off + (a - d0), a, b - a);
                }
                std::vector<std::size_t> order;
                for (std::size_t i = 0; i < ps.size(); ++i)
                    if (!ps[i].dev) order.push_back(i); // only non-resident pieces are read
                std::sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
                    return ps[x].w != ps[y].w ? ps[x].w < ps[y].w : ps[x].src < ps[y].src;
                });
                std::vector<std::uint64_t> at_of(ps.size(), 0);
                std::uint64_t at = 0;
                for (std::size_t i : order) {
                    const P& p = ps[i];
                    const bool dw = direct[p.w] != 0;
                    // contiguous (buffered) or within one block of the previous read
                    // (direct: the gap is read along; its block is read anyway)
                    if (!c.reads.empty() && c.reads.back().w == p.w && p.src >= c.reads.back().b &&
                        p.src - c.reads.back().b <= (dw ? kDirectAlign : 0)) {
                        at_of[i] = c.reads.back().at + (p.src - c.reads.back().a);
                        c.reads.back().b = p.src + p.n;
                        at = c.reads.back().at + (c.reads.back().b - c.reads.back().a);
                        continue;
                    }
                    if (dw) { // whole blocks straight into place: congruent to the file offset mod 4 KB
                        at = ceil_blk(at) + (file_off[p.w] + p.src) % kDirectAlign;
                        c.reads.push_back({p.w, p.src, p.src + p.n, at});
                        at_of[i] = at;
                        at += p.n;
                        continue;
                    }
                    // keep src/dst congruent mod 16 so the vector path applies
                    at = align16(at) + ((p.dst - c.lo) & 15);
                    c.reads.push_back({p.w, p.src, p.src + p.n, at});
                    at_of[i] = at;
                    at += p.n;
                }
                c.staging = ceil_blk(at);
                std::uint64_t expect = c.lo;
                for (std::size_t i = 0; i < ps.size(); ++i) {
                    const bool res = ps[i].dev != nullptr;
                    const std::uintptr_t src = res ? reinterpret_cast<std::uintptr_t>(ps[i].dev) : at_of[i];
                    c.segs.push_back({reinterpret_cast<const std::uint8_t*>(src), ps[i].dst - c.lo, ps[i].n});
                    c.abs.push_back(res ? 1 : 0);
                    c.bulk_ok = c.bulk_ok && ps[i].dst == expect && src % 16 == 0 && ps[i].n % 16 == 0 &&
                                (ps[i].dst - c.lo) % 16 == 0;
                    expect = ps[i].dst + ps[i].n;
                }
                c.bulk_ok = c.bulk_ok && expect == c.hi;
                max_staging = std::max(max_staging, c.staging);
                max_out = std::max(max_out, c.hi - c.lo);
                max_segs = std::max(max_segs, c.segs.size());
                chunks.push_back(std::move(c));
            }
        }
    };

    std::uint64_t source_payload_offset(const fs::path& p) {
        auto it = payload_off_.find(p.string());
        if (it != payload_off_.end()) return it->second;
        const std::uint64_t off = read_layout(p).payload_offset();
        payload_off_[p.string()] = off;
        return off;
    }

    bool uncached_;
    std::uint64_t chunk_;
    IoMode io_;
    cudaStream_t stream_[kSlots]{};
    cudaEvent_t ev0_[kSlots]{}, ev1_[kSlots]{};
    PinnedBuffer pin_io_[kSlots], pin_segs_[kSlots]; // pinned: async copies never sync the stream
    DeviceBuffer d_in_[kSlots], d_out_[kSlots], d_segs_[kSlots];
    std::vector<std::unique_ptr<Fd>> opened_[kSlots]; // uncached mode: per-read descriptors of the slot's chunk
    std::map<std::string, std::uint64_t> payload_off_;
    ReadPool pool_; // last: destroyed (joined) before the buffers its reads target
};

// Failure injection for tests (TAILOR_FAULT = comma-separated point names), in the
// spirit of the reference's inject_failure (R/src/trainer.cpp:170-193): lets a test
// make one output lane fail and check that the others are released.
bool fault_injected(const char* point) {
    const char* v = std::getenv("TAILOR_FAULT");
    if (!v || !*v) return false;
    const std::string s = std::string(",") + v + ",";
    return s.find(std::string(",") + point + ",") != std::string::npos;
}

struct OutputJob {
    const PartitionPlan* plan;
    std::vector<fs::path> window_files;
    fs::path out;
    int tag = 0; // passed to on_done: -1 = weights, r >= 0 = rank-r shard file
    std::vector<std::vector<ResidentRange>> resident; // per window, window-relative (may be empty)
};

struct AssembleTotals {
    double device_ms = 0.0, read_ms = 0.0, wait_ms = 0.0, write_ms = 0.0;
    std::uint64_t bytes = 0, direct_read_bytes = 0, direct_write_bytes = 0;
};

// Runs the output files over up to 16 lanes (weights first, then largest first,
// pulled from a shared queue). Output bytes do not depend on the lane count or timing: each
// file is produced by exactly one lane, in chunk order.
// on_done(tag), if set, runs on the lane's thread right after a file is complete (the
// pipelined re-verify of execute_merge hooks in here).
// on_error, if set, runs once on the thread of the first lane that fails (before the pool
// joins), so that lanes blocked on a hook's condition can be released.
// Lane li runs on devices[li % devices.size()] (the reference's loader pool,
// R/src/merge.cpp:156-205, spread over GPUs; which lane writes a file never changes its bytes).
AssembleTotals assemble_outputs(std::vector<OutputJob> jobs, int workers, bool uncached, const std::vector<int>& devices,
                                IoMode io, const std::function<void(int)>& on_done = {},
                                const std::function<void()>& on_error = {}) {
    // the weights file first (a lane verifying a rank file waits for it: with fewer lanes
    // than files, taking it last could block every lane), then largest first
    std::stable_sort(jobs.begin(), jobs.end(), [](const OutputJob& a, const OutputJob& b) {
        if ((a.tag < 0) != (b.tag < 0)) return a.tag < 0;
        return a.plan->dst_hi - a.plan->dst_lo > b.plan->dst_hi - b.plan->dst_lo;
    });
    const int lanes = std::clamp<int>(std::min<int>(static_cast<int>(jobs.size()), std::max<int>(workers, static_cast<int>(devices.size()))),
                                      1, 16 * static_cast<int>(devices.size()));
    const int readers = std::max(1, workers / lanes);
    // Chunks a little under a pool size class (16 / 32 / 128 MB), so a slot's
    // staging (chunk + <= 31 B of alignment per read) stays in that class and the
    // verify stages (16 MB halves) reuse the same pinned blocks.
    const std::uint64_t chunk = lanes >= 4 ? (15ull << 20) : lanes > 1 ? (31ull << 20) : (127ull << 20);
    std::vector<AssembleTotals> part(static_cast<std::size_t>(lanes));
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex mu;
    const auto lane = [&](int li) {
        try {
            cuda_check(cudaSetDevice(devices[static_cast<std::size_t>(li) % devices.size()]), "cudaSetDevice");
            FileAssembler fa(readers, uncached, chunk, io);
            for (std::size_t j = next.fetch_add(1); j < jobs.size(); j = next.fetch_add(1)) {
                {
                    std::lock_guard<std::mutex> lk(mu);
                    if (err) break;
                }
                // the weights file is the longest job and the one everything waits for: more readers
                fa.set_read_threads(jobs[j].tag < 0 ? std::max(readers, 4) : readers);
                if (jobs[j].tag < 0 && fault_injected("assemble-weights"))
                    fail(ErrorKind::Storage, "injected fault (TAILOR_FAULT=assemble-weights): " + jobs[j].out.string());
                fa.assemble(*jobs[j].plan, jobs[j].window_files, jobs[j].out, jobs[j].resident);
                if (on_done) on_done(jobs[j].tag);
            }
            part[static_cast<std::size_t>(li)] = {fa.device_ms, fa.read_ms,  fa.wait_ms,           fa.write_ms,
                                                  fa.bytes,     fa.direct_read_bytes, fa.direct_write_bytes};
        } catch (...) {
            bool first = false;
            {
                std::lock_guard<std::mutex> lk(mu);
                if (!err) {
                    err = std::current_exception();
                    first = true;
                }
            }
            if (first && on_error) on_error();
        }
    };
    if (lanes == 1) {
        lane(0);
    } else {
        std::vector<std::thread> pool;
        for (int li = 0; li < lanes; ++li) pool.emplace_back(lane, li);
        for (auto& t : pool) t.join();
    }
    if (err) std::rethrow_exception(err);
    AssembleTotals tot;
    for (const auto& x : part) {
        tot.device_ms += x.device_ms;
        tot.read_ms += x.read_ms;
        tot.wait_ms += x.wait_ms;
        tot.write_ms += x.write_ms;
        tot.bytes += x.bytes;
        tot.direct_read_bytes += x.direct_read_bytes;
        tot.direct_write_bytes += x.direct_write_bytes;
    }
    trace_count("assemble.lanes", lanes);
    trace_count("assemble.devices", static_cast<long long>(devices.size()));
    trace_value("assemble.read (sum over lanes)", tot.read_ms);
    trace_value("assemble.wait (sum over lanes)", tot.wait_ms);
    trace_value("assemble.write (sum over lanes)", tot.write_ms);
    trace_count("assemble.direct_read_bytes", static_cast<double>(tot.direct_read_bytes));
    trace_count("assemble.direct_write_bytes", static_cast<double>(tot.direct_write_bytes));
    return tot;
}

// Pipelined re-verify (resident form, when weights + one rank payload per lane fit the
// budget of every device): the lane that finished the weights file loads it to its
// device; a lane that finished a rank file re-reads it and runs K6 on its own device
// (after the weights are in; a device's first such lane loads its own copy of the
// weights payload). The on-disk headers are compared with the planned layouts
// afterwards. Otherwise the whole directory is verified after assembly
// (verify_checkpoint_dir). The sidecars must be written before the assembly starts.
class LaneVerifier {
  public:
    LaneVerifier(const fs::path& out_dir, const PartitionPlan* wplan, const std::vector<PartitionPlan>& splans, int workers,
                 bool verify, const std::vector<int>& devices)
        : out_(out_dir), wplan_(wplan), splans_(splans), verify_(verify), devices_(devices), N_(static_cast<int>(splans.size())) {
        std::uint64_t max_shard = 16;
        for (const auto& sp : splans) max_shard = std::max<std::uint64_t>(max_shard, sp.out.payload_bytes);
        const int nd = static_cast<int>(devices_.size());
        lanes_ = std::clamp<int>(std::min<int>(N_ + 1, std::max(workers, nd)), 1, 16 * nd);
        const std::uint64_t lanes_per_dev = static_cast<std::uint64_t>((lanes_ + nd - 1) / nd);
        pipelined_ = verify;
        for (int d : devices_) {
            if (!pipelined_) break;
            cuda_check(cudaSetDevice(d), "cudaSetDevice");
            pipelined_ = wplan->out.payload_bytes + lanes_per_dev * max_shard <= device_budget();
        }
        cuda_check(cudaSetDevice(devices_.front()), "cudaSetDevice");
        if (!pipelined_) return;
        const CheckpointSummary vs = read_checkpoint_summary(out_dir);
        std::vector<ContainerLayout> sl;
        for (const auto& sp : splans) sl.push_back(sp.out);
        vplan_ = verify_plan(out_dir, vs, wplan->out, std::move(sl));
        for (int d : devices_) {
            if (dev_.count(d)) continue;
            cuda_check(cudaSetDevice(d), "cudaSetDevice");
            auto st = std::make_unique<DevState>();
            st->derr.resize(static_cast<std::size_t>(N_) * 3 * sizeof(unsigned long long));
            cuda_check(cudaMemset(st->derr.get(), 0, st->derr.size()), "memset");
            cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "memset"); // cudaMemset is async: done before the verify streams add to it
            dev_.emplace(d, std::move(st));
        }
        cuda_check(cudaSetDevice(devices_.front()), "cudaSetDevice");
    }

    // on_done hook for assemble_outputs (empty when not pipelined); runs on the lane's
    // thread, with the lane's device current
    std::function<void(int)> hook() {
        if (!pipelined_) return {};
        const int readers = std::max(1, io_threads() / lanes_);
        return [this, readers](int tag) {
            int d = 0;
            cuda_check(cudaGetDevice(&d), "cudaGetDevice");
            DevState& ds_ = *dev_.at(d);
            PinnedBuffer stage[2];
            if (tag < 0) {
                try {
                    std::lock_guard<std::mutex> dl(ds_.mu);
                    load_payload_to(ckpt_file(CkptFile::Weights, out_), wplan_->out, ds_.dw, stage, std::max(readers, 8), 16ull << 20);
                    ds_.loaded = true;
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu_);
                    if (!werr_) werr_ = std::current_exception();
                }
                std::lock_guard<std::mutex> lk(mu_);
                weights_in_ = true;
                cv_.notify_all();
                if (werr_) std::rethrow_exception(werr_);
                return;
            }
            DeviceBuffer ds, dpairs, dranges;
            cudaStream_t st = nullptr;
            cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
            std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> own(st, &cudaStreamDestroy);
            // the last argument blocks until the weights file is complete and loaded on this
            // device, and returns its device address
            verify_rank_resident(vplan_, tag, ckpt_file(CkptFile::Shard, out_, tag), ds, dpairs, dranges, stage, readers,
                                 16ull << 20, ds_.derr.get<unsigned long long>(), st, [this, &ds_, readers] {
                                     {
                                         std::unique_lock<std::mutex> lk(mu_);
                                         cv_.wait(lk, [this] { return weights_in_; });
                                         if (werr_) std::rethrow_exception(werr_);
                                     }
                                     std::lock_guard<std::mutex> dl(ds_.mu);
                                     if (!ds_.loaded) { // first lane of a device other than the weights lane's
                                         PinnedBuffer st2[2];
                                         load_payload_to(ckpt_file(CkptFile::Weights, out_), wplan_->out, ds_.dw, st2,
                                                         std::max(readers, 8), 16ull << 20);
                                         ds_.loaded = true;
                                     }
                                     return static_cast<const std::uint8_t*>(ds_.dw.get());
                                 });
        };
    }

    // on_error hook for assemble_outputs: a lane failed (e.g. while assembling the weights
    // file, before it could release the others), so lanes waiting for the weights must not
    // wait forever; they fail with this error (the first lane's error is the one reported).
    std::function<void()> abort_hook() {
        if (!pipelined_) return {};
        return [this] {
            std::lock_guard<std::mutex> lk(mu_);
            if (!werr_)
                werr_ = std::make_exception_ptr(TailorError(ErrorKind::Storage, "merge aborted: another output lane failed"));
            weights_in_ = true;
            cv_.notify_all();
        };
    }

    // after assembly: headers on disk == the planned layouts (what read_checkpoint's
    // deserialize checks) and the counters, or the whole post-assembly verify
    void finish() {
        cuda_check(cudaSetDevice(devices_.front()), "cudaSetDevice");
        if (!pipelined_) {
            if (verify_) verify_checkpoint_dir(out_.string(), devices_.front());
            return;
        }
        const auto same = [](const ContainerLayout& a, const ContainerLayout& b) {
            if (a.payload_offset() != b.payload_offset() || a.payload_bytes != b.payload_bytes ||
                a.entries.size() != b.entries.size() || a.metadata != b.metadata)
                return false;
            for (std::size_t i = 0; i < a.entries.size(); ++i)
                if (a.entries[i].name != b.entries[i].name || a.entries[i].begin != b.entries[i].begin ||
                    a.entries[i].end != b.entries[i].end || a.entries[i].dtype != b.entries[i].dtype ||
                    a.entries[i].shape != b.entries[i].shape)
                    return false;
            return true;
        };
        std::size_t files = 0;
        for ([[maybe_unused]] const auto& e : fs::directory_iterator(out_ / "optim")) ++files;
        if (files != static_cast<std::size_t>(N_)) fail(ErrorKind::Consistency, out_.string() + ": unexpected shard file count");
        if (!same(read_layout(ckpt_file(CkptFile::Weights, out_)), wplan_->out))
            fail(ErrorKind::CorruptContainer, out_.string() + ": weights header differs from the plan");
        for (int r = 0; r < N_; ++r)
            if (!same(read_layout(ckpt_file(CkptFile::Shard, out_, r)), splans_[static_cast<std::size_t>(r)].out))
                fail(ErrorKind::CorruptContainer, out_.string() + ": shard " + std::to_string(r) + " header differs from the plan");
        // each rank was verified on exactly one device; the others' counters for it stay 0
        std::vector<unsigned long long> err(static_cast<std::size_t>(N_) * 3, 0), part(err.size());
        for (auto& [d, st] : dev_) {
            cuda_check(cudaSetDevice(d), "cudaSetDevice");
            cuda_check(cudaMemcpy(part.data(), st->derr.get(), part.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H");
            for (std::size_t i = 0; i < err.size(); ++i) err[i] += part[i];
        }
        cuda_check(cudaSetDevice(devices_.front()), "cudaSetDevice");
        verify_counters_host(out_, N_, err.data());
    }

  private:
    struct DevState {
        std::mutex mu;
        bool loaded = false;
        DeviceBuffer dw, derr;
    };
    fs::path out_;
    const PartitionPlan* wplan_;
    const std::vector<PartitionPlan>& splans_;
    bool verify_, pipelined_ = false;
    std::vector<int> devices_;
    int N_, lanes_ = 1;
    VerifyPlan vplan_;
    std::map<int, std::unique_ptr<DevState>> dev_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool weights_in_ = false;
    std::exception_ptr werr_;
};

} // namespace

MergeStats execute_merge(const MergePlan& plan, const fs::path& out_dir, const MergeOptions& options) {
    return execute_merge(plan, out_dir, options, nullptr);
}

MergeStats execute_merge(const MergePlan& plan, const fs::path& out_dir, const MergeOptions& options,
                         const ResidentSources* resident) {
    const auto t0 = std::chrono::steady_clock::now();
    MergeStats stats;
    const std::vector<int> devices = lane_devices(options);
    std::error_code ec;
    if (fs::exists(out_dir) && !fs::is_empty(out_dir, ec))
        fail(ErrorKind::Storage, "refusing to write into non-empty directory '" + out_dir.string() + "'");
    // CUDA context creation (hundreds of ms in a fresh process) overlaps the header
    // parsing and planning below; joined before the first device allocation.
    auto cuda_ready = std::async(std::launch::async, [&devices] {
        PhaseTimer pt("merge.cuda_init (overlapped)");
        for (int d : devices) {
            cuda_check(cudaSetDevice(d), "cudaSetDevice");
            cuda_check(cudaFree(nullptr), "cuda init");
        }
    });
    struct JoinOnExit { // a validation error below must not leave the init running past the call
        std::future<void>& f;
        ~JoinOnExit() {
            if (f.valid()) f.wait();
        }
    } join_on_exit{cuda_ready};

    auto phase = std::make_unique<PhaseTimer>("merge.headers+plan");
    std::map<std::string, CheckpointSummary> sums;
    for (const auto& p : plan.sources) sums.emplace(p, read_checkpoint_summary(p));
    if (!sums.count(plan.config_source)) sums.emplace(plan.config_source, read_checkpoint_summary(plan.config_source));
    const SummaryLookup sum_of = [&](const std::string& p) { return sums.at(p); };

    // Parse every source header the composite reads (validating container
    // structure as deserialize does) — weights once per source, shards per
    // (source, rank).
    std::map<std::string, SourceLayout> layouts;
    for (const auto& [tgt, a] : plan.assignment) {
        if (layouts.count(a.source)) continue;
        SourceLayout sl;
        sl.weights = read_layout(ckpt_file(CkptFile::Weights, a.source));
        stats.weight_files_read += 1;
        layouts.emplace(a.source, std::move(sl));
    }
    for (const auto& src : plan.sources) {
        auto& sl = layouts[src];
        for (int r = 0; r < plan.num_ranks; ++r) sl.shards.push_back(read_layout(ckpt_file(CkptFile::Shard, src, r)));
    }
    stats.shard_files_read = options.uncached
                                 ? static_cast<std::int64_t>(plan.num_ranks) * static_cast<std::int64_t>(plan.group_copies.size())
                                 : static_cast<std::int64_t>(plan.sources.size()) * plan.num_ranks;
    const LayoutLookup lay_of = [&](const std::string& p) -> const SourceLayout& { return layouts.at(p); };

    const PartitionPlan wplan = plan_weights(plan, lay_of);
    std::vector<PartitionPlan> splans;
    for (int r = 0; r < plan.num_ranks; ++r) splans.push_back(plan_shard(plan, lay_of, r));
    const OptimMeta optim = merged_optim_meta(plan, sum_of);
    const SaveManifest manifest = merged_manifest(plan, sum_of);

    // All inputs validated; write.
    cuda_ready.get(); // rethrows a device error
    cuda_check(cudaSetDevice(devices.front()), "cudaSetDevice");
    fs::create_directories(out_dir / "optim", ec);
    if (ec) fail(ErrorKind::Storage, "cannot create '" + out_dir.string() + "': " + ec.message());
    const int workers = options.workers > 0 ? options.workers : std::max(plan.num_ranks, io_threads());
    phase = std::make_unique<PhaseTimer>("merge.assemble");
    // Sidecars first: the re-verify reads them back, and it starts while the payload
    // files are still being assembled.
    write_text_file(ckpt_file(CkptFile::OptimMeta, out_dir), sidecar_text(optim));
    write_text_file(ckpt_file(CkptFile::Config, out_dir), read_text_file(ckpt_file(CkptFile::Config, plan.config_source)));
    write_text_file(ckpt_file(CkptFile::TrainerState, out_dir), read_text_file(ckpt_file(CkptFile::TrainerState, plan.config_source)));
    write_text_file(ckpt_file(CkptFile::Manifest, out_dir), sidecar_text(manifest));

    std::vector<OutputJob> jobs;
    {
        OutputJob j{&wplan, {}, ckpt_file(CkptFile::Weights, out_dir), -1, {}};
        for (const auto& w : wplan.windows) j.window_files.push_back(ckpt_file(CkptFile::Weights, w.source));
        jobs.push_back(std::move(j));
    }
    // resident source bytes are usable when every lane runs on their device
    const bool use_resident = resident && !resident->ranges.empty() && devices.size() == 1 && devices.front() == resident->device;
    std::uint64_t resident_bytes = 0;
    for (int r = 0; r < plan.num_ranks; ++r) {
        const PartitionPlan& sp = splans[static_cast<std::size_t>(r)];
        OutputJob j{&sp, {}, ckpt_file(CkptFile::Shard, out_dir, r), r, {}};
        for (const auto& w : sp.windows) j.window_files.push_back(ckpt_file(CkptFile::Shard, w.source, w.container));
        if (use_resident) {
            j.resident.resize(sp.windows.size());
            for (std::size_t wi = 0; wi < sp.windows.size(); ++wi) {
                const SourceWindow& w = sp.windows[wi];
                const auto it = resident->ranges.find({fs::path(w.source).lexically_normal().string(), w.container});
                if (it == resident->ranges.end()) continue;
                for (const ResidentRange& rr : it->second) { // payload-relative -> window-relative
                    const std::uint64_t lo = std::max(rr.lo, w.lo), hi = std::min(rr.hi, w.hi);
                    if (lo < hi) j.resident[wi].push_back({lo - w.lo, hi - w.lo, rr.dev + (lo - rr.lo)});
                }
            }
            for (const auto& seg : sp.segments) // bytes the plan will take from the device
                for (const auto& rr : j.resident[seg.window]) {
                    const std::uint64_t lo = std::max(rr.lo, seg.src_off), hi = std::min(rr.hi, seg.src_off + seg.bytes);
                    if (lo < hi) resident_bytes += hi - lo;
                }
        }
        jobs.push_back(std::move(j));
    }
    trace_count("merge.resident_source_bytes", static_cast<double>(resident_bytes));

    LaneVerifier lv(out_dir, &wplan, splans, workers, options.verify, devices);
    const IoMode io = io_mode_from_env(options.io);
    trace_count(("merge.io_mode " + std::string(io_mode_name(io))).c_str(), static_cast<double>(io));
    const AssembleTotals fa =
        assemble_outputs(std::move(jobs), workers, options.uncached, devices, io, lv.hook(), lv.abort_hook());
    alloc_stats().trace("merge.assemble allocations");
    phase = std::make_unique<PhaseTimer>("merge.verify");
    lv.finish();
    phase.reset();
    alloc_stats().trace("merge.verify allocations (cumulative)");

    stats.device_ms = fa.device_ms;
    stats.bytes_moved = fa.bytes;
    stats.resident_bytes = resident_bytes;
    stats.direct_read_bytes = fa.direct_read_bytes;
    stats.direct_write_bytes = fa.direct_write_bytes;
    stats.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return stats;
}

// ---- regroup: coarse <-> fine re-slicing on files -------------------
// Same result as read_checkpoint -> coarse_to_fine / fine_to_coarse
// (R/src/groups.cpp:152-220, a gather by model offset) -> write_checkpoint, but
// expressed as byte segments: every target rank chunk is a run of pieces of
// source rank chunks (split at tensor and rank-chunk boundaries) plus zero
// padding, assembled by K2 without materialising the unsharded state.
MergeStats execute_regroup(const fs::path& src, const fs::path& out_dir, Grouping target, const MergeOptions& options) {
    const auto t0 = std::chrono::steady_clock::now();
    MergeStats stats;
    std::error_code ec;
    if (fs::exists(out_dir) && !fs::is_empty(out_dir, ec))
        fail(ErrorKind::Storage, "refusing to write into non-empty directory '" + out_dir.string() + "'");
    const std::vector<int> devices = lane_devices(options);
    cuda_check(cudaSetDevice(devices.front()), "cudaSetDevice");
    const CheckpointSummary s = read_checkpoint_summary(src);
    const ModelSpec& spec = s.spec;
    const int N = s.optim.num_ranks;
    for (const auto& m : enumerate_modules(spec))
        if (!s.manifest.contains(m))
            fail(ErrorKind::MissingModules, "regrouping needs a complete checkpoint; '" + src.string() + "' lacks '" +
                                                module_name(m) + "'");
    const GroupTable src_table = s.optim.grouping == Grouping::Fine ? build_group_table(spec) : build_coarse_table(spec);
    const GroupTable dst_table = target == Grouping::Fine ? build_group_table(spec) : build_coarse_table(spec);
    const ShardGeometry geom{N};
    const std::string key = src.string();

    // source side: tensor -> (group, group offset); shard layouts per rank
    std::map<std::string, std::pair<int, std::int64_t>> where;
    for (int g = 0; g < src_table.group_count(); ++g)
        for (const auto& sl : group_tensor_slices(spec, src_table, g)) where[sl.decl.name] = {g, sl.group_offset};
    std::vector<ContainerLayout> shards;
    for (int r = 0; r < N; ++r) {
        shards.push_back(read_layout(ckpt_file(CkptFile::Shard, src, r)));
        for (const auto& gm : s.optim.groups)
            for (const char* f : {".master", ".exp_avg", ".exp_avg_sq"}) {
                const Entry* e = shards.back().find(shard_key(gm.index, f));
                if (!e) fail(ErrorKind::CorruptContainer, ckpt_file(CkptFile::Shard, src, r).string() + ": missing tensor '" + shard_key(gm.index, f) + "'");
                if (e->dtype != Dtype::F32 || e->shape != std::vector<std::int64_t>{gm.shard_length})
                    fail(ErrorKind::Geometry, ckpt_file(CkptFile::Shard, src, r).string() + ": tensor '" + e->name + "' has unexpected dtype/shape");
            }
    }
    stats.shard_files_read = N;

    // target optim_meta: hyper inherited from the source group of the first slice,
    // weight decay by decay class; conflicts are a GeometryError (as reslice).
    std::map<int, AdamHyperparams> hyp;
    std::vector<std::vector<TensorSlice>> dst_slices(static_cast<std::size_t>(dst_table.group_count()));
    for (int g = 0; g < dst_table.group_count(); ++g) {
        dst_slices[static_cast<std::size_t>(g)] = group_tensor_slices(spec, dst_table, g);
        const DecayClass d = dst_table.groups[static_cast<std::size_t>(g)].decay;
        bool set = false;
        for (const auto& sl : dst_slices[static_cast<std::size_t>(g)]) {
            const AdamHyperparams h = hyper_for_class(s.optim.find(where.at(sl.decl.name).first)->hyper, d);
            if (!set) {
                hyp[g] = h;
                set = true;
            } else if (!(hyp[g] == h)) {
                fail(ErrorKind::Geometry, "conflicting hyperparams while re-slicing group " + std::to_string(g));
            }
        }
    }
    const OptimMeta optim = make_optim_meta(dst_table, hyp, geom, s.optim.step);

    std::vector<PartitionPlan> plans;
    for (int r = 0; r < N; ++r) {
        std::vector<EntryDecl> decls;
        for (int g = 0; g < dst_table.group_count(); ++g)
            for (const char* f : {".exp_avg", ".exp_avg_sq", ".master"})
                decls.push_back({shard_key(g, f), Dtype::F32, {geom.shard_length(dst_table.groups[static_cast<std::size_t>(g)].element_count)}});
        PartitionPlan pp;
        pp.out = layout_for(std::move(decls), {{"num_ranks", std::to_string(N)}, {"rank", std::to_string(r)}});
        pp.dst_lo = 0;
        pp.dst_hi = pp.out.payload_bytes;
        std::vector<CopyPiece> pieces;
        for (int g = 0; g < dst_table.group_count(); ++g) {
            const std::int64_t len = dst_table.groups[static_cast<std::size_t>(g)].element_count;
            const std::int64_t c = geom.shard_length(len), first = static_cast<std::int64_t>(r) * c;
            for (const char* f : {".exp_avg", ".exp_avg_sq", ".master"}) {
                const std::uint64_t dbase = pp.out.find(shard_key(g, f))->begin;
                for (const auto& sl : dst_slices[static_cast<std::size_t>(g)]) {
                    std::int64_t a = std::max(first, sl.group_offset);
                    const std::int64_t b = std::min(first + c, sl.group_offset + sl.decl.numel());
                    const auto [sg, soff] = where.at(sl.decl.name);
                    const std::int64_t sc = geom.shard_length(src_table.groups[static_cast<std::size_t>(sg)].element_count);
                    while (a < b) { // split at source rank-chunk boundaries
                        const std::int64_t x = soff + (a - sl.group_offset); // source group element
                        const std::int64_t rr = x / sc, pos = x % sc;
                        const std::int64_t n = std::min(b - a, sc - pos);
                        const Entry* se = shards[static_cast<std::size_t>(rr)].find(shard_key(sg, f));
                        pieces.push_back({key, static_cast<int>(rr), se->begin + static_cast<std::uint64_t>(pos) * 4,
                                          dbase + static_cast<std::uint64_t>(a - first) * 4, static_cast<std::uint64_t>(n) * 4});
                        a += n;
                    }
                }
                const std::int64_t valid = std::clamp<std::int64_t>(len - first, 0, c);
                if (valid < c) // zero padding
                    pieces.push_back({"", kZeroContainer, 0, dbase + static_cast<std::uint64_t>(valid) * 4,
                                      static_cast<std::uint64_t>(c - valid) * 4});
            }
        }
        finalize_partition(pp, std::move(pieces));
        plans.push_back(std::move(pp));
    }
    // weights: the tensor set and order do not depend on the grouping
    PartitionPlan wp;
    wp.out = read_layout(ckpt_file(CkptFile::Weights, src));
    stats.weight_files_read = 1;
    wp.dst_lo = 0;
    wp.dst_hi = wp.out.payload_bytes;
    finalize_partition(wp, {{key, -1, 0, 0, wp.out.payload_bytes}});

    // The reference regroups what read_checkpoint returned (R/src/checkpoint.cpp:485-575):
    // a source with nonzero shard padding, a negative exp_avg_sq or a weight that
    // disagrees with its master fails before anything is written. Same here: the
    // device re-verify of the source directory runs before out_dir is created.
    verify_checkpoint_dir(src.string(), devices.front());

    fs::create_directories(out_dir / "optim", ec);
    if (ec) fail(ErrorKind::Storage, "cannot create '" + out_dir.string() + "': " + ec.message());
    const int workers = options.workers > 0 ? options.workers : std::max(N, io_threads());
    const auto files_of = [&](const PartitionPlan& pp) {
        std::vector<fs::path> files;
        for (const auto& w : pp.windows)
            files.push_back(w.container == kZeroContainer ? fs::path() : w.container < 0 ? ckpt_file(CkptFile::Weights, src) : ckpt_file(CkptFile::Shard, src, w.container));
        return files;
    };
    std::vector<OutputJob> jobs;
    jobs.push_back({&wp, files_of(wp), ckpt_file(CkptFile::Weights, out_dir), -1, {}});
    for (int r = 0; r < N; ++r)
        jobs.push_back({&plans[static_cast<std::size_t>(r)], files_of(plans[static_cast<std::size_t>(r)]), ckpt_file(CkptFile::Shard, out_dir, r), r,
                        {}});
    // sidecars first: the pipelined re-verify reads them back while the files assemble
    write_text_file(ckpt_file(CkptFile::OptimMeta, out_dir), sidecar_text(optim));
    write_text_file(ckpt_file(CkptFile::Config, out_dir), sidecar_text(spec));
    write_text_file(ckpt_file(CkptFile::TrainerState, out_dir), sidecar_text(s.trainer));
    write_text_file(ckpt_file(CkptFile::Manifest, out_dir), sidecar_text(s.manifest));
    LaneVerifier lv(out_dir, &wp, plans, workers, options.verify, devices);
    const AssembleTotals fa =
        assemble_outputs(std::move(jobs), workers, false, devices, io_mode_from_env(options.io), lv.hook(), lv.abort_hook());
    lv.finish();
    stats.device_ms = fa.device_ms;
    stats.bytes_moved = fa.bytes;
    stats.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return stats;
}

} // namespace tailor
