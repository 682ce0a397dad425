// Peer fabric: the comm phase as ONE fused kernel over NVLink peer memory
// (CUDA IPC between the one-process-per-GPU ranks of a box), replacing NCCL's
// counts all-reduce + reduce-scatter + all-gather around the optimizer.
//
// Per comm phase (sequence number seq), on the comm stream of every rank:
//   1. signal: write this rank's sample count and post flag = seq into every
//      peer's flag block (system-scope release after a system fence);
//   2. wait:   one thread spins until every rank's post flag >= seq, then sums
//      the counts in rank order (Fabric::all_reduce_counts, collectives.cpp:48-53);
//   3. fold:   the optimizer kernel (optim.cu opt_fold) reads the shard
//      [lo, hi) of EVERY rank's accumulator directly over NVLink, sums them in
//      ascending rank order — exactly the reference Fabric's reduce-scatter
//      fold (collectives.cpp:55-75), which NCCL does not guarantee — applies
//      AdamW and stores the new bf16 parameters into EVERY rank's replica
//      (Fabric::all_gather, collectives.cpp:77-91) — one kernel, no staging;
//   4. done:   write done flag = seq into every peer's flag block.
// A rank's compute stream waits for every rank's done flag of phase p-2
// before stage p (it reuses that accumulator and reads those parameters).
// With world size 1 the "peers" are this process's own buffers.
#pragma once

#include <vector>

#include "common.cuh"

namespace acco {

constexpr int kMaxPeers = 16;

struct PeerFlags {  // device memory, one block per rank, written by the peers
    unsigned long long post[kMaxPeers];
    unsigned long long done[kMaxPeers];
    long long counts[2][kMaxPeers];  // [phase parity][rank]
    unsigned long long csum_seq[kMaxPeers];  // replica checksums (debug check_replicas)
    unsigned long long csum[kMaxPeers][2];
};

struct PeerFlagPtrs {
    PeerFlags* p[kMaxPeers];
};

class PeerFabric {
public:
    PeerFabric(int world, int rank, int device);
    ~PeerFabric();
    PeerFabric(const PeerFabric&) = delete;
    PeerFabric& operator=(const PeerFabric&) = delete;
    int size() const { return world_; }
    int rank() const { return rank_; }

    // Exchange: every rank exports the IPC handles of its registered buffers
    // (+ its flag block); the caller all-gathers the blobs (torch.distributed)
    // and connects. Buffers must be cudaMalloc allocation bases.
    void register_buffers(const std::vector<void*>& bufs);
    size_t blob_bytes() const;
    void export_blob(void* out) const;
    void connect(const void* blobs);  // [world][blob_bytes()]
    bool connected() const { return connected_; }
    void* peer_buffer(int r, int i) const { return peers_[static_cast<size_t>(r)][static_cast<size_t>(i)]; }

    // Stream-ordered protocol steps (see the header comment).
    void signal_post(unsigned long long seq, int parity, long long count, cudaStream_t s);
    void wait_posts(unsigned long long seq, int parity, int64_t* total_out, cudaStream_t s);
    void signal_done(unsigned long long seq, cudaStream_t s);
    void wait_done(unsigned long long seq, cudaStream_t s);
    // Debug replica check: publish this rank's 2 replica hashes for phase seq
    // into every rank's block, wait for every rank's, compare (flag |= bit).
    void check_hashes(unsigned long long seq, const uint64_t* local_hash2, int* flag, int bit, cudaStream_t s);

private:
    int world_, rank_, device_;
    PeerFlags* flags_ = nullptr;         // local block (peers write into it)
    std::vector<void*> local_;            // registered local buffers
    std::vector<std::vector<void*>> peers_;  // [rank][buffer]; own rank = local pointers
    std::vector<void*> opened_;           // IPC mappings to close
    PeerFlagPtrs flag_ptrs_{};            // every rank's flag block (mapped)
    bool connected_ = false;
};

}  // namespace acco
