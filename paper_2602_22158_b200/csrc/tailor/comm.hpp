// NCCL communicator for the score-partials all-gather (host/comm.cpp).
#pragma once

#include <array>
#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>

namespace tailor {

constexpr std::size_t kCommIdBytes = 128; // ncclUniqueId

// A fresh NCCL unique id (rank 0 creates it; the caller ships it to the other ranks).
std::array<std::uint8_t, kCommIdBytes> comm_unique_id();

class Comm {
  public:
    Comm(const std::uint8_t* id, int nranks, int rank, int device); // collective over the ranks
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    // d_recv[r * count + i] = rank r's d_send[i]; asynchronous on s.
    void all_gather(const double* d_send, double* d_recv, std::uint64_t count, cudaStream_t s);
    int nranks() const { return nranks_; }
    int rank() const { return rank_; }

  private:
    void* comm_ = nullptr;
    int nranks_, rank_, device_;
};

} // namespace tailor
