// Host-only test of tailor::ReadPool (tailor/io.hpp), the per-lane reader pool of the file
// drop-ins: batches of pread jobs queued ahead of their waits (the one-chunk lookahead),
// pieces larger than the cut size, O_DIRECT jobs staged congruent and incongruent to the
// file offset (when the filesystem takes O_DIRECT), a failing batch that does not poison
// the next ones, drain(), and destruction with work still queued. Needs no GPU.
// Test infrastructure: links libtailor_b200.so for its internal C++ symbols.
#include <fcntl.h>
#include <unistd.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tailor/errors.hpp"
#include "tailor/io.hpp"

using tailor::ReadJob;
using tailor::ReadPool;

namespace {
std::uint64_t rng = 0x9E3779B97F4A7C15ull;
std::uint64_t next_u64() {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return rng;
}
int failures = 0;
void check(bool ok, const char* what) {
    if (!ok) {
        std::fprintf(stderr, "FAIL: %s\n", what);
        ++failures;
    }
}
} // namespace

int main(int argc, char** argv) {
    const std::string path = argc > 1 ? argv[1] : "/tmp/readpool_test.bin";
    const std::uint64_t size = 48ull << 20;
    std::vector<std::uint8_t> data(size);
    for (auto& b : data) b = static_cast<std::uint8_t>(next_u64() >> 56);
    {
        FILE* f = std::fopen(path.c_str(), "wb");
        if (!f || std::fwrite(data.data(), 1, size, f) != size) return 2;
        std::fclose(f);
    }
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) return 2;
    const int dfd = tailor::open_direct_read(path);

    // 1. lookahead: batch i+1 queued before batch i is waited for; random ranges, some
    //    larger than the 16 MB buffered / 4 MB direct piece size
    {
        ReadPool pool(3);
        constexpr int kBatches = 24;
        std::vector<std::vector<std::uint8_t>> bufs(kBatches);
        std::vector<std::vector<std::pair<std::uint64_t, std::uint64_t>>> ranges(kBatches); // (offset, bytes)
        std::vector<std::uint64_t> tickets(kBatches);
        const auto queue = [&](int i) {
            std::vector<ReadJob> jobs;
            std::uint64_t total = 0;
            const int n = 1 + static_cast<int>(next_u64() % 5);
            for (int j = 0; j < n; ++j) {
                const std::uint64_t len = 1 + next_u64() % (i % 6 == 0 ? (40ull << 20) : (3ull << 20));
                const std::uint64_t off = next_u64() % (size - len);
                ranges[i].push_back({off, len});
                total += len;
            }
            bufs[i].assign(total + 4096, 0xEE);
            std::uint64_t at = 0;
            for (const auto& [off, len] : ranges[i]) {
                // direct jobs (every third batch) mostly incongruent to the file offset: bounce path
                jobs.push_back({fd, bufs[i].data() + at, len, off, (i % 3 == 1 && dfd >= 0) ? dfd : -1});
                at += len;
            }
            tickets[i] = pool.submit(jobs, path);
        };
        queue(0);
        for (int i = 0; i < kBatches; ++i) {
            if (i + 1 < kBatches) queue(i + 1);
            pool.wait(tickets[i]);
            std::uint64_t at = 0;
            bool ok = true;
            for (const auto& [off, len] : ranges[i]) {
                ok = ok && std::memcmp(bufs[i].data() + at, data.data() + off, len) == 0;
                at += len;
            }
            ok = ok && bufs[i][at] == 0xEE; // nothing written past the batch
            check(ok, "lookahead batch bytes");
        }
    }
    // 2. O_DIRECT staged congruent to the file offset (whole blocks straight into place)
    if (dfd >= 0) {
        void* raw = nullptr;
        if (posix_memalign(&raw, 4096, 24ull << 20) != 0) return 2;
        std::unique_ptr<void, decltype(&std::free)> hold(raw, &std::free);
        auto* dst = static_cast<std::uint8_t*>(raw);
        ReadPool pool(4);
        const std::uint64_t off = 3 * 4096 + 123, len = (20ull << 20) + 77; // partial head and tail blocks
        pool.wait(pool.submit({{fd, dst + (off % 4096), len, off, dfd}}, path));
        check(std::memcmp(dst + (off % 4096), data.data() + off, len) == 0, "direct congruent bytes");
    } else {
        std::printf("O_DIRECT not supported here: direct cases covered by the bounce path only\n");
    }
    // 3. a failing batch reports Storage; the pool keeps serving later batches
    {
        ReadPool pool(2);
        std::vector<std::uint8_t> a(1 << 20), b(1 << 20);
        const auto bad = pool.submit({{-1, a.data(), a.size(), 0, -1}}, "bad-fd");
        const auto good = pool.submit({{fd, b.data(), b.size(), 4096, -1}}, path);
        bool threw = false;
        try {
            pool.wait(bad);
        } catch (const tailor::TailorError& e) {
            threw = e.kind() == tailor::ErrorKind::Storage;
        }
        check(threw, "failing batch raises Storage");
        pool.wait(good);
        check(std::memcmp(b.data(), data.data() + 4096, b.size()) == 0, "batch after a failure");
        std::vector<std::uint8_t> c(5 << 20), d(7 << 20);
        pool.submit({{fd, c.data(), c.size(), 0, -1}}, path);
        pool.submit({{fd, d.data(), d.size(), 1 << 20, -1}}, path);
        pool.drain(); // waits for both without their tickets
        check(std::memcmp(c.data(), data.data(), c.size()) == 0 && std::memcmp(d.data(), data.data() + (1 << 20), d.size()) == 0,
              "drain completes every batch");
    }
    // 4. destruction with pieces still queued finishes them before the buffers go away
    {
        std::vector<std::uint8_t> e(32 << 20);
        {
            ReadPool pool(1);
            pool.submit({{fd, e.data(), e.size(), 0, -1}}, path);
        }
        check(std::memcmp(e.data(), data.data(), e.size()) == 0, "destructor finishes queued pieces");
    }
    ::close(fd);
    if (dfd >= 0) ::close(dfd);
    std::remove(path.c_str());
    if (failures) return 1;
    std::printf("readpool ok\n");
    return 0;
}
