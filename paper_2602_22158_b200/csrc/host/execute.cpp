// execute_merge — the drop-in for R/src/merge.cpp:226-357 on files.
//
// Same contract: refuse a non-empty out_dir, validate everything before the
// first write, output bytes identical to the reference (headers and sidecars
// render through the same JSON library; payload bytes are copied exactly), a
// full re-verify before returning, MergeStats counting files read. Different
// mechanism: only the byte ranges the composite needs are read from each
// source (the reference loads every shard file whole), staged through pinned
// memory, assembled by the device gather kernel, and streamed back out in
// chunks on two CUDA streams; the re-verify is the device kernel K6.
#include <algorithm>
#include <chrono>
#include <fcntl.h>
#include <filesystem>
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

// Assembles one output container file from source files through the device.
class FileAssembler {
  public:
    FileAssembler(int workers, bool uncached) : workers_(std::max(1, workers)), uncached_(uncached) {
        for (auto& s : stream_) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
        for (int i = 0; i < 2; ++i) {
            cuda_check(cudaEventCreate(&ev0_[i]), "event");
            cuda_check(cudaEventCreate(&ev1_[i]), "event");
        }
    }
    ~FileAssembler() {
        for (auto& s : stream_) cudaStreamDestroy(s);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(ev0_[i]);
            cudaEventDestroy(ev1_[i]);
        }
    }

    double device_ms = 0.0;
    std::uint64_t bytes = 0;

    void assemble(const PartitionPlan& pp, const std::vector<fs::path>& window_files, const fs::path& out_path) {
        const std::uint64_t chunk = 256ull << 20;
        Fd out(out_path, O_WRONLY | O_CREAT | O_TRUNC);
        if (out.fd < 0) fail(ErrorKind::Storage, "cannot create '" + out_path.string() + "'");
        const std::string prefix = pp.out.prefix();
        pwrite_all(out.fd, reinterpret_cast<const std::uint8_t*>(prefix.data()), prefix.size(), 0, out_path.string());
        const std::uint64_t base = pp.out.payload_offset();
        // Payload offsets of each window inside its source file.
        std::vector<std::uint64_t> file_off(pp.windows.size());
        std::vector<std::unique_ptr<Fd>> fds(pp.windows.size());
        for (std::size_t w = 0; w < pp.windows.size(); ++w) {
            file_off[w] = source_payload_offset(window_files[w]) + pp.windows[w].lo;
            if (!uncached_) {
                fds[w] = std::make_unique<Fd>(window_files[w], O_RDONLY);
                if (fds[w]->fd < 0) fail(ErrorKind::MissingArtifact, "cannot open '" + window_files[w].string() + "'");
            }
        }
        HostMergeChunks plan(pp, chunk);
        for (int i = 0; i < 2; ++i) {
            pin_in_[i].resize(std::max<std::uint64_t>(16, plan.max_staging));
            pin_out_[i].resize(std::max<std::uint64_t>(16, plan.max_out));
            d_in_[i].resize(std::max<std::uint64_t>(16, plan.max_staging));
            d_out_[i].resize(std::max<std::uint64_t>(16, plan.max_out));
            d_segs_[i].resize(std::max<std::size_t>(1, plan.max_segs) * sizeof(dev::GatherSeg));
        }
        int pending[2] = {-1, -1};
        std::vector<std::vector<dev::GatherSeg>> patched(plan.chunks.size());
        const auto flush = [&](int slot) {
            if (pending[slot] < 0) return;
            cuda_check(cudaStreamSynchronize(stream_[slot]), "sync");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev0_[slot], ev1_[slot]);
            device_ms += ms;
            const auto& c = plan.chunks[static_cast<std::size_t>(pending[slot])];
            pwrite_all(out.fd, pin_out_[slot].get(), c.hi - c.lo, base + c.lo, out_path.string());
            pending[slot] = -1;
        };
        for (std::size_t ci = 0; ci < plan.chunks.size(); ++ci) {
            const int slot = static_cast<int>(ci & 1);
            flush(slot);
            const auto& c = plan.chunks[ci];
            // This chunk's source ranges -> pinned staging, via the parallel pread pool
            // (uncached mode re-opens the source file per read, as the reference
            // reloads a shard per group copy).
            std::vector<std::unique_ptr<Fd>> opened;
            std::vector<ReadJob> jobs;
            for (const auto& rd : c.reads) {
                int fd;
                if (uncached_) {
                    opened.push_back(std::make_unique<Fd>(window_files[rd.w], O_RDONLY));
                    if (opened.back()->fd < 0) fail(ErrorKind::MissingArtifact, "cannot open '" + window_files[rd.w].string() + "'");
                    fd = opened.back()->fd;
                } else {
                    fd = fds[rd.w]->fd;
                }
                jobs.push_back({fd, pin_in_[slot].get() + rd.at, rd.b - rd.a, file_off[rd.w] + rd.a});
            }
            run_reads(jobs, workers_, out_path.string());
            cudaStream_t s = stream_[slot];
            cuda_check(cudaMemcpyAsync(d_in_[slot].get(), pin_in_[slot].get(), c.staging, cudaMemcpyHostToDevice, s), "H2D");
            patched[ci] = c.segs;
            for (auto& g : patched[ci]) g.src = d_in_[slot].get() + reinterpret_cast<std::uintptr_t>(g.src);
            cuda_check(cudaMemcpyAsync(d_segs_[slot].get(), patched[ci].data(), patched[ci].size() * sizeof(dev::GatherSeg),
                                       cudaMemcpyHostToDevice, s),
                       "segs");
            cuda_check(cudaEventRecord(ev0_[slot], s), "event");
            cuda_check(dev::launch_gather(d_segs_[slot].get<dev::GatherSeg>(), static_cast<std::uint32_t>(patched[ci].size()),
                                          d_out_[slot].get(), c.hi - c.lo, dev::kGatherAuto, c.bulk_ok, s),
                       "gather");
            cuda_check(cudaEventRecord(ev1_[slot], s), "event");
            cuda_check(cudaMemcpyAsync(pin_out_[slot].get(), d_out_[slot].get(), c.hi - c.lo, cudaMemcpyDeviceToHost, s), "D2H");
            pending[slot] = static_cast<int>(ci);
            bytes += c.hi - c.lo;
        }
        flush(0);
        flush(1);
        if (plan.chunks.empty() && pp.out.payload_bytes != 0) fail(ErrorKind::Consistency, "empty merge plan");
    }

  private:
    struct Read {
        std::uint32_t w;
        std::uint64_t a, b, at;
    };
    struct ChunkPlan {
        std::uint64_t lo, hi, staging = 0;
        std::vector<Read> reads;
        std::vector<dev::GatherSeg> segs; // src = staging offset
        bool bulk_ok = true;
    };
    struct HostMergeChunks {
        std::vector<ChunkPlan> chunks;
        std::uint64_t max_staging = 0, max_out = 0;
        std::size_t max_segs = 0;
        HostMergeChunks(const PartitionPlan& pp, std::uint64_t chunk) {
            const std::uint64_t total = pp.dst_hi - pp.dst_lo;
            std::size_t si = 0;
            for (std::uint64_t lo = 0; lo < total; lo += chunk) {
                ChunkPlan c;
                c.lo = lo;
                c.hi = std::min(total, lo + chunk);
                struct P {
                    std::uint32_t w;
                    std::uint64_t src, dst, n;
                };
                std::vector<P> ps;
                while (si < pp.segments.size() && pp.segments[si].dst_off + pp.segments[si].bytes - pp.dst_lo <= c.lo) ++si;
                for (std::size_t j = si; j < pp.segments.size(); ++j) {
                    const auto& s = pp.segments[j];
                    const std::uint64_t d0 = s.dst_off - pp.dst_lo, d1 = d0 + s.bytes;
                    if (d0 >= c.hi) break;
                    const std::uint64_t a = std::max(d0, c.lo), b = std::min(d1, c.hi);
                    if (a < b) ps.push_back({s.window, s.src_off + (a - d0), a, b - a});
                }
                std::vector<std::size_t> order(ps.size());
                for (std::size_t i = 0; i < ps.size(); ++i) order[i] = i;
                std::sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
                    return ps[x].w != ps[y].w ? ps[x].w < ps[y].w : ps[x].src < ps[y].src;
                });
                std::vector<std::uint64_t> at_of(ps.size());
                std::uint64_t at = 0;
                for (std::size_t i : order) {
                    const P& p = ps[i];
                    if (!c.reads.empty() && c.reads.back().w == p.w && c.reads.back().b == p.src) {
                        at_of[i] = c.reads.back().at + (p.src - c.reads.back().a);
                        c.reads.back().b += p.n;
                        at = c.reads.back().at + (c.reads.back().b - c.reads.back().a);
                        continue;
                    }
                    // keep src/dst congruent mod 16 so the vector path applies
                    at = align16(at) + ((p.dst - c.lo) & 15);
                    c.reads.push_back({p.w, p.src, p.src + p.n, at});
                    at_of[i] = at;
                    at += p.n;
                }
                c.staging = align16(at);
                std::uint64_t expect = c.lo;
                for (std::size_t i = 0; i < ps.size(); ++i) {
                    c.segs.push_back({reinterpret_cast<const std::uint8_t*>(at_of[i]), ps[i].dst - c.lo, ps[i].n});
                    c.bulk_ok = c.bulk_ok && ps[i].dst == expect && at_of[i] % 16 == 0 && ps[i].n % 16 == 0 &&
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

    int workers_;
    bool uncached_;
    cudaStream_t stream_[2]{};
    cudaEvent_t ev0_[2]{}, ev1_[2]{};
    PinnedBuffer pin_in_[2], pin_out_[2];
    DeviceBuffer d_in_[2], d_out_[2], d_segs_[2];
    std::map<std::string, std::uint64_t> payload_off_;
};

} // namespace

MergeStats execute_merge(const MergePlan& plan, const fs::path& out_dir, const MergeOptions& options) {
    const auto t0 = std::chrono::steady_clock::now();
    MergeStats stats;
    std::error_code ec;
    if (fs::exists(out_dir) && !fs::is_empty(out_dir, ec))
        fail(ErrorKind::Storage, "refusing to write into non-empty directory '" + out_dir.string() + "'");
    cuda_check(cudaSetDevice(options.device), "cudaSetDevice");

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
        sl.weights = read_layout(weights_path(a.source));
        stats.weight_files_read += 1;
        layouts.emplace(a.source, std::move(sl));
    }
    for (const auto& src : plan.sources) {
        auto& sl = layouts[src];
        for (int r = 0; r < plan.num_ranks; ++r) sl.shards.push_back(read_layout(shard_path(src, r)));
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
    fs::create_directories(out_dir / "optim", ec);
    if (ec) fail(ErrorKind::Storage, "cannot create '" + out_dir.string() + "': " + ec.message());
    const int workers = options.workers > 0 ? options.workers : std::max(plan.num_ranks, io_threads());
    phase = std::make_unique<PhaseTimer>("merge.assemble");
    FileAssembler fa(workers, options.uncached);
    {
        std::vector<fs::path> files;
        for (const auto& w : wplan.windows) files.push_back(weights_path(w.source));
        fa.assemble(wplan, files, weights_path(out_dir));
    }
    for (int r = 0; r < plan.num_ranks; ++r) {
        std::vector<fs::path> files;
        for (const auto& w : splans[static_cast<std::size_t>(r)].windows) files.push_back(shard_path(w.source, w.container));
        fa.assemble(splans[static_cast<std::size_t>(r)], files, shard_path(out_dir, r));
    }
    write_text_file(optim_meta_path(out_dir), render_optim_meta_json(optim));
    write_text_file(config_path(out_dir), read_text_file(config_path(plan.config_source)));
    write_text_file(trainer_state_path(out_dir), read_text_file(trainer_state_path(plan.config_source)));
    write_text_file(manifest_path(out_dir), render_manifest_json(manifest));

    phase = std::make_unique<PhaseTimer>("merge.verify");
    if (options.verify) verify_checkpoint_dir(out_dir.string(), options.device);
    phase.reset();

    stats.device_ms = fa.device_ms;
    stats.bytes_moved = fa.bytes;
    stats.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return stats;
}

} // namespace tailor
