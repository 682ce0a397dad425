// Peer fabric over CUDA IPC / NVLink (see peer.h).
#include "peer.h"

#include <cstring>

namespace acco {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// one thread: publish (count,) flag = seq into every rank's block
__global__ void peer_signal_kernel(PeerFlagPtrs fp, int world, int rank, unsigned long long seq, int parity,
                                   long long count, int post) {
    __threadfence_system();  // this rank's accumulator / replica writes before the flag
    for (int r = 0; r < world; ++r) {
        PeerFlags* f = fp.p[r];
        if (post) {
            f->counts[parity][rank] = count;
            __threadfence_system();
            st_release_sys(&f->post[rank], seq);
        } else {
            st_release_sys(&f->done[rank], seq);
        }
    }
}

// one thread: wait until every rank's flag >= seq; posts also fold the counts
__global__ void peer_wait_kernel(PeerFlags* local, int world, unsigned long long seq, int parity, int post,
                                 int64_t* total_out) {
    const unsigned long long* flags = post ? local->post : local->done;
    for (int r = 0; r < world; ++r) {
        uint64_t t0 = 0;
        while (ld_acquire_sys(&flags[r]) < seq) {
            __nanosleep(200);
            uint64_t now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (!t0) t0 = now;
            else if (now - t0 > 60000000000ull) __trap();  // 60 s: a rank died; fail instead of hanging
        }
    }
    if (post && total_out) {
        long long tot = 0;
        for (int r = 0; r < world; ++r) tot += *(volatile long long*)&local->counts[parity][r];
        *total_out = tot;
    }
    __threadfence_system();
}

__global__ void peer_hash_kernel(PeerFlagPtrs fp, PeerFlags* local, int world, int rank, unsigned long long seq,
                                 const unsigned long long* h2, int* flag, int bit) {
    const unsigned long long a = h2[0], b = h2[1];
    for (int r = 0; r < world; ++r) {
        PeerFlags* f = fp.p[r];
        f->csum[rank][0] = a;
        f->csum[rank][1] = b;
        __threadfence_system();
        st_release_sys(&f->csum_seq[rank], seq);
    }
    bool bad = false;
    for (int r = 0; r < world; ++r) {
        uint64_t t0 = 0;
        while (ld_acquire_sys(&local->csum_seq[r]) < seq) {
            __nanosleep(200);
            uint64_t now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (!t0) t0 = now;
            else if (now - t0 > 60000000000ull) __trap();
        }
        bad |= *(volatile unsigned long long*)&local->csum[r][0] != a ||
               *(volatile unsigned long long*)&local->csum[r][1] != b;
    }
    if (bad) atomicOr(flag, bit);
}

}  // namespace

PeerFabric::PeerFabric(int world, int rank, int device) : world_(world), rank_(rank), device_(device) {
    ACCO_REQUIRE(world >= 1 && world <= kMaxPeers, "peer fabric: 1..16 ranks");
    ACCO_REQUIRE(rank >= 0 && rank < world, "peer fabric: bad rank");
    ACCO_CUDA(cudaSetDevice(device));
    ACCO_CUDA(cudaMalloc(&flags_, sizeof(PeerFlags)));
    ACCO_CUDA(cudaMemset(flags_, 0, sizeof(PeerFlags)));
}

PeerFabric::~PeerFabric() {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    cudaFree(flags_);
}

void PeerFabric::register_buffers(const std::vector<void*>& bufs) {
    ACCO_REQUIRE(!connected_, "peer fabric: already connected");
    local_ = bufs;
}

// blob: [int device][pad to 64 B][IPC handle of the flag block][handles of the buffers]
constexpr size_t kBlobHeader = 64;

size_t PeerFabric::blob_bytes() const { return kBlobHeader + (local_.size() + 1) * sizeof(cudaIpcMemHandle_t); }

void PeerFabric::export_blob(void* out) const {
    std::memset(out, 0, kBlobHeader);
    std::memcpy(out, &device_, sizeof(int));
    auto* h = reinterpret_cast<cudaIpcMemHandle_t*>(static_cast<char*>(out) + kBlobHeader);
    if (world_ == 1) return;  // no peers: nothing to map
    ACCO_CUDA(cudaIpcGetMemHandle(&h[0], flags_));
    for (size_t i = 0; i < local_.size(); ++i) ACCO_CUDA(cudaIpcGetMemHandle(&h[i + 1], local_[i]));
}

void PeerFabric::connect(const void* blobs) {
    ACCO_REQUIRE(!connected_, "peer fabric: already connected");
    const size_t nb = local_.size();
    peers_.assign(static_cast<size_t>(world_), std::vector<void*>(nb, nullptr));
    for (int r = 0; r < world_; ++r) {
        if (r == rank_) {
            peers_[static_cast<size_t>(r)] = local_;
            flag_ptrs_.p[r] = flags_;
            continue;
        }
        const char* blob = static_cast<const char*>(blobs) + static_cast<size_t>(r) * blob_bytes();
        int dev = 0;
        std::memcpy(&dev, blob, sizeof(int));
        int can = 0;
        if (dev == device_)
            can = 1;  // ranks sharing a device (single-GPU multi-process tests): IPC without P2P
        else
            ACCO_CUDA(cudaDeviceCanAccessPeer(&can, device_, dev));
        ACCO_REQUIRE(can, "peer fabric: no peer access between the GPUs (NVLink/P2P required)");
        const auto* h = reinterpret_cast<const cudaIpcMemHandle_t*>(blob + kBlobHeader);
        void* p = nullptr;
        ACCO_CUDA(cudaIpcOpenMemHandle(&p, h[0], cudaIpcMemLazyEnablePeerAccess));
        opened_.push_back(p);
        flag_ptrs_.p[r] = static_cast<PeerFlags*>(p);
        for (size_t i = 0; i < nb; ++i) {
            ACCO_CUDA(cudaIpcOpenMemHandle(&p, h[i + 1], cudaIpcMemLazyEnablePeerAccess));
            opened_.push_back(p);
            peers_[static_cast<size_t>(r)][i] = p;
        }
    }
    connected_ = true;
}

void PeerFabric::signal_post(unsigned long long seq, int parity, long long count, cudaStream_t s) {
    peer_signal_kernel<<<1, 1, 0, s>>>(flag_ptrs_, world_, rank_, seq, parity, count, 1);
    ACCO_CHECK_LAUNCH();
}

void PeerFabric::wait_posts(unsigned long long seq, int parity, int64_t* total_out, cudaStream_t s) {
    peer_wait_kernel<<<1, 1, 0, s>>>(flags_, world_, seq, parity, 1, total_out);
    ACCO_CHECK_LAUNCH();
}

void PeerFabric::signal_done(unsigned long long seq, cudaStream_t s) {
    peer_signal_kernel<<<1, 1, 0, s>>>(flag_ptrs_, world_, rank_, seq, 0, 0, 0);
    ACCO_CHECK_LAUNCH();
}

void PeerFabric::wait_done(unsigned long long seq, cudaStream_t s) {
    peer_wait_kernel<<<1, 1, 0, s>>>(flags_, world_, seq, 0, 0, nullptr);
    ACCO_CHECK_LAUNCH();
}

void PeerFabric::check_hashes(unsigned long long seq, const uint64_t* local_hash2, int* flag, int bit, cudaStream_t s) {
    peer_hash_kernel<<<1, 1, 0, s>>>(flag_ptrs_, flags_, world_, rank_, seq,
                                     reinterpret_cast<const unsigned long long*>(local_hash2), flag, bit);
    ACCO_CHECK_LAUNCH();
}

}  // namespace acco
