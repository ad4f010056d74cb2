// Host write-path probe for the file drop-ins: how fast can a merge output reach
// the page cache? Compares one thread vs T threads on disjoint ranges of ONE
// file (buffered pwrite takes the inode lock) vs T threads on T files, and
// memcpy into a shared mmap of a ftruncate'd file.
//   g++ -O2 -std=c++17 -pthread tools/write_probe.cpp -o /tmp/write_probe
//   /tmp/write_probe <dir> [GB] [threads]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <string>
#include <sys/mman.h>
#include <thread>
#include <unistd.h>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void pw(int fd, const char* src, size_t n, off_t off) {
    size_t put = 0;
    while (put < n) {
        ssize_t r = pwrite(fd, src + put, n - put, off + put);
        if (r <= 0) { perror("pwrite"); exit(1); }
        put += r;
    }
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    const double gb = argc > 2 ? atof(argv[2]) : 2.0;
    const int T = argc > 3 ? atoi(argv[3]) : 8;
    const size_t total = static_cast<size_t>(gb * 1e9) & ~((size_t)(1 << 20) - 1);
    std::vector<char> src(total);
    for (size_t i = 0; i < total; i += 4096) src[i] = static_cast<char>(i >> 12);
    const size_t piece = 16 << 20;

    auto run = [&](const char* name, auto fn) {
        for (int rep = 0; rep < 2; ++rep) {
            double t0 = now();
            fn();
            double dt = now() - t0;
            printf("%-34s rep%d %7.1f ms  %6.2f GB/s\n", name, rep, dt * 1e3, total / dt / 1e9);
            fflush(stdout);
        }
    };
    const std::string f1 = dir + "/wp_one.bin";
    run("1 thread, 1 file (pwrite)", [&] {
        unlink(f1.c_str());
        int fd = open(f1.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        for (size_t at = 0; at < total; at += piece) pw(fd, src.data() + at, std::min(piece, total - at), at);
        close(fd);
    });
    run("T threads, 1 file (pwrite)", [&] {
        unlink(f1.c_str());
        int fd = open(f1.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                for (size_t at = t * piece; at < total; at += T * piece) pw(fd, src.data() + at, std::min(piece, total - at), at);
            });
        for (auto& x : th) x.join();
        close(fd);
    });
    run("T threads, 1 file (ftruncate first)", [&] {
        unlink(f1.c_str());
        int fd = open(f1.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (ftruncate(fd, total)) perror("ftruncate");
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                for (size_t at = t * piece; at < total; at += T * piece) pw(fd, src.data() + at, std::min(piece, total - at), at);
            });
        for (auto& x : th) x.join();
        close(fd);
    });
    run("T threads, T files (pwrite)", [&] {
        std::vector<std::thread> th;
        const size_t per = total / T;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                const std::string f = dir + "/wp_" + std::to_string(t) + ".bin";
                unlink(f.c_str());
                int fd = open(f.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
                for (size_t at = 0; at < per; at += piece) pw(fd, src.data() + t * per + at, std::min(piece, per - at), at);
                close(fd);
            });
        for (auto& x : th) x.join();
    });
    run("T threads, 1 file (mmap memcpy)", [&] {
        unlink(f1.c_str());
        int fd = open(f1.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
        if (ftruncate(fd, total)) perror("ftruncate");
        char* m = static_cast<char*>(mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
        if (m == MAP_FAILED) { perror("mmap"); exit(1); }
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                for (size_t at = t * piece; at < total; at += T * piece) memcpy(m + at, src.data() + at, std::min(piece, total - at));
            });
        for (auto& x : th) x.join();
        munmap(m, total);
        close(fd);
    });
    run("T threads, 1 file (read back pread)", [&] {
        int fd = open(f1.c_str(), O_RDONLY);
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                for (size_t at = t * piece; at < total; at += T * piece) {
                    size_t n = std::min(piece, total - at), got = 0;
                    while (got < n) got += pread(fd, src.data() + at + got, n - got, at + got);
                }
            });
        for (auto& x : th) x.join();
        close(fd);
    });
    unlink(f1.c_str());
    for (int t = 0; t < T; ++t) unlink((dir + "/wp_" + std::to_string(t) + ".bin").c_str());
    return 0;
}
