// Fabric over NCCL (NVLink 5 / NVSwitch): the B200 replacement of the
// reference's value-level collectives (proj/src/collectives.cpp:36-91).
// One rank per process / GPU; rank order = worker id.
#include "acco.h"
#include "capi_util.h"
#include "comm.h"
#include "host_util.h"
#include "lm_kernels.h"

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace acco {

#define ACCO_NCCL(expr)                                                                             \
    do {                                                                                            \
        ncclResult_t _r = (expr);                                                                   \
        if (_r != ncclSuccess)                                                                      \
            throw Error(kCudaError, std::string(#expr) + ": " + ncclGetErrorString(_r));            \
    } while (0)

Comm::Comm(int nranks, int rank, const ncclUniqueId& id, int device) : nranks_(nranks), rank_(rank), device_(device) {
    ACCO_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "comm: bad rank/size");
    ACCO_CUDA(cudaSetDevice(device));
    ACCO_NCCL(ncclCommInitRank(&comm_, nranks, id, rank));
}

Comm::~Comm() {
    if (comm_ && !aborted_) ncclCommDestroy(comm_);
}

double Comm::timeout_s() {
    const char* e = std::getenv("ACCO_NCCL_TIMEOUT_S");  // read per wait: tests shorten it
    const double v = e ? std::atof(e) : 600.0;
    return v > 0 ? v : 600.0;
}

void Comm::abort_and_throw(const std::string& why) {
    if (!aborted_) {
        ncclCommAbort(comm_);  // NCCL's kernels observe the abort flag and exit
        aborted_ = true;
    }
    throw Error(kCudaError, "nccl rank " + std::to_string(rank_) + "/" + std::to_string(nranks_) + ": " + why);
}

void Comm::wait(cudaEvent_t ev) {
    ACCO_REQUIRE(!aborted_, "comm: communicator was aborted after an earlier failure");
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = timeout_s();
    int spins = 0;
    while (true) {
        const cudaError_t q = cudaEventQuery(ev);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) ACCO_CUDA(q);
        ncclResult_t async = ncclSuccess;
        ACCO_NCCL(ncclCommGetAsyncError(comm_, &async));
        if (async != ncclSuccess && async != ncclInProgress)
            abort_and_throw(std::string("asynchronous NCCL error: ") + ncclGetErrorString(async));
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > limit)
            abort_and_throw("no progress for " + std::to_string(static_cast<int>(limit)) +
                            " s (a rank died or stopped issuing collectives); communicator aborted");
        // poll tightly at first (the common case is a short wait), then back off
        if (++spins > 1000) std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
}

void Comm::all_reduce_f32(const float* send, float* recv, size_t n, cudaStream_t s) {
    ACCO_NCCL(ncclAllReduce(send, recv, n, ncclFloat32, ncclSum, comm_, s));
}
void Comm::all_reduce_i64(const int64_t* send, int64_t* recv, size_t n, cudaStream_t s) {
    ACCO_NCCL(ncclAllReduce(send, recv, n, ncclInt64, ncclSum, comm_, s));
}
void Comm::reduce_scatter_f32(const float* send, float* recv, size_t n, cudaStream_t s) {
    ACCO_NCCL(ncclReduceScatter(send, recv, n, ncclFloat32, ncclSum, comm_, s));
}
void Comm::all_gather(const void* send, void* recv, size_t n, int dtype, cudaStream_t s) {
    ACCO_NCCL(ncclAllGather(send, recv, n, dtype == ACCO_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32, comm_, s));
}
void Comm::all_gather_u64(const uint64_t* send, uint64_t* recv, size_t n, cudaStream_t s) {
    ACCO_NCCL(ncclAllGather(send, recv, n, ncclUint64, comm_, s));
}

}  // namespace acco

using namespace acco;

struct acco_comm {
    Comm* impl;
};

extern "C" {

int acco_comm_unique_id(unsigned char id_out[128]) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        ACCO_NCCL(ncclGetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int acco_comm_init_rank(int nranks, int rank, const unsigned char id[128], int device, acco_comm** out) {
    return guarded([&] {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        *out = new acco_comm{new Comm(nranks, rank, uid, device)};
    });
}

int acco_comm_destroy(acco_comm* c) {
    return guarded([&] {
        if (c) {
            delete c->impl;
            delete c;
        }
    });
}

int acco_comm_size(const acco_comm* c) { return c ? c->impl->size() : 0; }
int acco_comm_rank(const acco_comm* c) { return c ? c->impl->rank() : -1; }

int acco_all_reduce_f32(acco_comm* c, const float* send, float* recv, uint64_t count, void* stream) {
    return guarded([&] { c->impl->all_reduce_f32(send, recv, count, static_cast<cudaStream_t>(stream)); });
}
int acco_all_reduce_i64(acco_comm* c, const int64_t* send, int64_t* recv, uint64_t count, void* stream) {
    return guarded([&] { c->impl->all_reduce_i64(send, recv, count, static_cast<cudaStream_t>(stream)); });
}
int acco_reduce_scatter_f32(acco_comm* c, const float* send, float* recv, uint64_t count, void* stream) {
    return guarded([&] { c->impl->reduce_scatter_f32(send, recv, count, static_cast<cudaStream_t>(stream)); });
}
int acco_pack_padded(const float* flat, float* padded, uint64_t dim, int n, void* stream) {
    return guarded([&] {
        ShardLayout l = shard_partition(dim, n);
        std::vector<uint64_t> lo, sz;
        for (int w = 0; w < n; ++w) {
            lo.push_back(l.lo(w));
            sz.push_back(l.size(w));
        }
        pack_padded(flat, padded, lo.data(), sz.data(), n, l.chunk(), static_cast<cudaStream_t>(stream));
    });
}

int acco_unpack_padded(const void* padded, void* flat, uint64_t dim, int n, int dtype, void* stream) {
    return guarded([&] {
        ACCO_REQUIRE(dtype == ACCO_DTYPE_F32 || dtype == ACCO_DTYPE_BF16, "unpack_padded: bad dtype");
        ShardLayout l = shard_partition(dim, n);
        std::vector<uint64_t> lo, sz;
        for (int w = 0; w < n; ++w) {
            lo.push_back(l.lo(w));
            sz.push_back(l.size(w));
        }
        unpack_padded(padded, flat, dtype == ACCO_DTYPE_F32 ? 4 : 2, lo.data(), sz.data(), n, l.chunk(),
                      static_cast<cudaStream_t>(stream));
    });
}

int acco_all_gather(acco_comm* c, const void* send, void* recv, uint64_t count, int dtype, void* stream) {
    return guarded([&] {
        ACCO_REQUIRE(dtype == ACCO_DTYPE_F32 || dtype == ACCO_DTYPE_BF16, "all_gather: bad dtype");
        c->impl->all_gather(send, recv, count, dtype, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"

namespace acco {
Comm* comm_impl(acco_comm* c) { return c ? c->impl : nullptr; }
}  // namespace acco
