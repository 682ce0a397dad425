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

private:
    ncclComm_t comm_ = nullptr;
    int nranks_, rank_, device_;
};

Comm* comm_impl(acco_comm* c);

}  // namespace acco
