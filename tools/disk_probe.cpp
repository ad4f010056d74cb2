// Disk / page-cache bandwidth probe for the files drop-in's roofline (bench.py
// --workload files reports its cold and warm lines against these numbers).
//
//   disk_probe <dir> [gib_per_file=2] [files=8] [threads_per_file=4]
//
// Writes `files` files of `gib_per_file` GiB in <dir> and prints one JSON line:
//   write_cached_gbs    pwrite into the page cache (no fsync)
//   write_buffered_gbs  the same + fsync (includes the writeback to the device)
//   write_direct_gbs    O_DIRECT pwrite (null if the filesystem refuses O_DIRECT)
//   read_direct_gbs     O_DIRECT pread (the device's read bandwidth)
//   read_cold_gbs       buffered pread after POSIX_FADV_DONTNEED (cold page cache)
//   read_warm_gbs       buffered pread of the same files again (page cache)
// Every file is read/written by `threads_per_file` threads in 16 MB pieces.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <string>
#include <sys/statvfs.h>
#include <thread>
#include <unistd.h>
#include <vector>

namespace {

constexpr std::size_t kPiece = 16u << 20;

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

struct Buf {
    void* p = nullptr;
    explicit Buf(std::size_t n) {
        if (posix_memalign(&p, 4096, n)) std::abort();
        std::memset(p, 0x5a, n);
    }
    ~Buf() { std::free(p); }
};

// Runs `fn(fd, piece_offset, buffer)` over every 16 MB piece of every file with
// threads_per_file threads per file; returns GB/s (1e9) or -1 on an I/O error.
template <class Fn>
double run(const std::vector<int>& fds, std::size_t bytes, int tpf, Fn fn) {
    std::atomic<bool> bad{false};
    const double t0 = now();
    std::vector<std::thread> pool;
    for (int fd : fds)
        for (int t = 0; t < tpf; ++t)
            pool.emplace_back([&, fd, t] {
                Buf b(kPiece);
                for (std::size_t off = static_cast<std::size_t>(t) * kPiece; off < bytes; off += kPiece * tpf)
                    if (!fn(fd, off, static_cast<char*>(b.p))) bad = true;
            });
    for (auto& th : pool) th.join();
    const double dt = now() - t0;
    return bad ? -1.0 : static_cast<double>(bytes) * fds.size() / dt / 1e9;
}

std::string num(double v) {
    if (v < 0) return "null";
    char s[32];
    std::snprintf(s, sizeof s, "%.3f", v);
    return s;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: disk_probe <dir> [gib_per_file] [files] [threads_per_file]\n");
        return 2;
    }
    const std::string dir = argv[1];
    const double gib = argc > 2 ? std::atof(argv[2]) : 2.0;
    const int nfiles = argc > 3 ? std::atoi(argv[3]) : 8;
    const int tpf = argc > 4 ? std::atoi(argv[4]) : 4;
    const std::size_t bytes = static_cast<std::size_t>(gib * (1ull << 30)) / kPiece * kPiece;
    std::vector<std::string> paths;
    for (int i = 0; i < nfiles; ++i) paths.push_back(dir + "/disk_probe_" + std::to_string(i) + ".bin");
    const auto open_all = [&](int flags) {
        std::vector<int> fds;
        for (const auto& p : paths) {
            const int fd = ::open(p.c_str(), flags, 0644);
            if (fd < 0) {
                for (int f : fds) ::close(f);
                return std::vector<int>{};
            }
            fds.push_back(fd);
        }
        return fds;
    };
    const auto close_all = [](std::vector<int>& fds) {
        for (int f : fds) ::close(f);
        fds.clear();
    };
    const auto pw = [&](int fd, std::size_t off, char* b) { return ::pwrite(fd, b, kPiece, static_cast<off_t>(off)) == static_cast<ssize_t>(kPiece); };
    const auto pr = [&](int fd, std::size_t off, char* b) { return ::pread(fd, b, kPiece, static_cast<off_t>(off)) == static_cast<ssize_t>(kPiece); };

    // buffered write + fsync
    auto fds = open_all(O_WRONLY | O_CREAT | O_TRUNC);
    if (fds.empty()) {
        std::fprintf(stderr, "cannot create files in %s\n", dir.c_str());
        return 1;
    }
    double t0 = now();
    const double wc = run(fds, bytes, tpf, pw); // into the page cache
    for (int f : fds) ::fsync(f);
    double wb = wc > 0 ? static_cast<double>(bytes) * fds.size() / (now() - t0) / 1e9 : -1.0; // incl. writeback
    close_all(fds);

    // O_DIRECT write (overwrites in place)
    double wd = -1.0;
    fds = open_all(O_WRONLY | O_DIRECT);
    const bool direct_ok = !fds.empty();
    if (direct_ok) {
        t0 = now();
        wd = run(fds, bytes, tpf, pw);
        for (int f : fds) ::fsync(f);
        if (wd > 0) wd = static_cast<double>(bytes) * fds.size() / (now() - t0) / 1e9;
        close_all(fds);
    }

    // O_DIRECT read
    double rd = -1.0;
    if (direct_ok) {
        fds = open_all(O_RDONLY | O_DIRECT);
        if (!fds.empty()) rd = run(fds, bytes, tpf, pr);
        close_all(fds);
    }

    // buffered cold read: drop the files' pages first
    fds = open_all(O_RDONLY);
    for (int f : fds) {
        ::fdatasync(f);
        ::posix_fadvise(f, 0, 0, POSIX_FADV_DONTNEED);
    }
    const double rc = run(fds, bytes, tpf, pr);
    const double rw = run(fds, bytes, tpf, pr);
    close_all(fds);

    struct statvfs sv {};
    statvfs(dir.c_str(), &sv);
    std::printf("{\"dir\": \"%s\", \"files\": %d, \"gib_per_file\": %.2f, \"threads_per_file\": %d, \"free_gb\": %.1f, "
                "\"write_cached_gbs\": %s, \"write_buffered_gbs\": %s, \"write_direct_gbs\": %s, \"read_direct_gbs\": %s, \"read_cold_gbs\": %s, "
                "\"read_warm_gbs\": %s, \"o_direct\": %s}\n",
                dir.c_str(), nfiles, static_cast<double>(bytes) / (1ull << 30), tpf,
                static_cast<double>(sv.f_bavail) * sv.f_frsize / 1e9, num(wc).c_str(), num(wb).c_str(), num(wd).c_str(), num(rd).c_str(),
                num(rc).c_str(), num(rw).c_str(), direct_ok ? "true" : "false");
    for (const auto& p : paths) ::unlink(p.c_str());
    return 0;
}
