// NCCL communicator (see comm.cu).
#pragma once

#include <nccl.h>

#include "acco.h"
#include "common.cuh"

namespace acco {

class Comm {
public:
    Comm(int nranks, int rank, const ncclUniqueId& id, int device);
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    int size() const { return nranks_; }
    int rank() const { return rank_; }
    void all_reduce_f32(const float* send, float* recv, size_t n, cudaStream_t s);
    void all_reduce_i64(const int64_t* send, int64_t* recv, size_t n, cudaStream_t s);
    void reduce_scatter_f32(const float* send, float* recv, size_t n, cudaStream_t s);
    void all_gather(const void* send, void* recv, size_t n, int dtype, cudaStream_t s);
    void all_gather_u64(const uint64_t* send, uint64_t* recv, size_t n, cudaStream_t s);
    // Failure detection (the reference's deadlock detection, protocols.cpp:476-482):
    // block until `ev` completes while polling ncclCommGetAsyncError; an NCCL
    // error, or no progress for timeout_s() seconds (a dead or stuck rank),
    // aborts the communicator and throws instead of hanging forever.
    void wait(cudaEvent_t ev);
    static double timeout_s();  // ACCO_NCCL_TIMEOUT_S, default 600
    bool aborted() const { return aborted_; }

private:
    ncclComm_t comm_ = nullptr;
    int nranks_, rank_, device_;
    bool aborted_ = false;
    void abort_and_throw(const std::string& why);
};

Comm* comm_impl(acco_comm* c);

}  // namespace acco
