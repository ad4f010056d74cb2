// The one collective of the path: an all-gather of the scorer's FP64
// per-rank partials across the GPUs that share a job, so every GPU combines them in
// rank order and selects identically (no broadcast of the selection, no payload byte on
// NVLink). NCCL is loaded at run time (dlopen "libnccl.so.2"): a process that already
// holds torch's NCCL reuses that library, and the single-GPU library has no link-time
// dependency on it.
#include "tailor/comm.hpp"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include <nccl.h>

#include "tailor/engine.hpp"
#include "tailor/errors.hpp"

namespace tailor {

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string load_error;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
            return a;
        }
        const auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p && a.load_error.empty()) a.load_error = std::string("libnccl.so.2 lacks ") + name;
            return p;
        };
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(sym("ncclAllGather"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
        return a;
    }();
    if (!api.load_error.empty()) fail(ErrorKind::Device, api.load_error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const NcclApi& a = nccl();
    fail(ErrorKind::Device, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
}

} // namespace

std::array<std::uint8_t, kCommIdBytes> comm_unique_id() {
    static_assert(sizeof(ncclUniqueId) == kCommIdBytes, "NCCL unique id size");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::array<std::uint8_t, kCommIdBytes> out{};
    std::memcpy(out.data(), &id, kCommIdBytes);
    return out;
}

Comm::Comm(const std::uint8_t* id, int nranks, int rank, int device) : nranks_(nranks), rank_(rank), device_(device) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(ErrorKind::Geometry, "communicator rank out of range");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId uid;
    std::memcpy(&uid, id, kCommIdBytes);
    ncclComm_t c = nullptr;
    nccl_check(nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    comm_ = c;
}

Comm::~Comm() {
    if (comm_) nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
}

void Comm::all_gather(const double* d_send, double* d_recv, std::uint64_t count, cudaStream_t s) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    nccl_check(nccl().all_gather(d_send, d_recv, static_cast<size_t>(count), ncclFloat64, static_cast<ncclComm_t>(comm_), s),
               "ncclAllGather");
}

} // namespace tailor
