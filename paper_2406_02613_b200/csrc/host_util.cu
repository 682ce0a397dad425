// C-ABI for the integer pieces of the path: shard_partition, rng::derive and
// the micro-batch index draw. See host_util.h.
#include "acco.h"
#include "capi_util.h"
#include "common.cuh"
#include "host_util.h"

namespace acco {

ShardLayout shard_partition(uint64_t dim, int n) {
    // proj/include/accosim/shard.hpp:24-38
    if (n < 1) throw Error(kInvalidArg, "shard_partition: need at least one worker");
    ShardLayout l;
    l.dim = dim;
    const uint64_t base = dim / static_cast<uint64_t>(n);
    const uint64_t extra = dim % static_cast<uint64_t>(n);
    uint64_t lo = 0;
    for (int w = 0; w < n; ++w) {
        uint64_t len = base + (static_cast<uint64_t>(w) < extra ? 1 : 0);
        l.ranges.emplace_back(lo, lo + len);
        lo += len;
    }
    return l;
}

}  // namespace acco

using namespace acco;

extern "C" {

int acco_shard_partition(uint64_t dim, int n, uint64_t* lo_out, uint64_t* hi_out) {
    return guarded([&] {
        ShardLayout l = shard_partition(dim, n);
        for (int w = 0; w < n; ++w) {
            if (lo_out) lo_out[w] = l.lo(w);
            if (hi_out) hi_out[w] = l.hi(w);
        }
    });
}

uint64_t acco_rng_derive(uint64_t master, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    return rng_derive(master, a, b, c, d);
}

int acco_sample_indices(uint64_t stream_seed, int batch, int n_samples, int32_t* out) {
    return guarded([&] {
        ACCO_REQUIRE(batch >= 1, "stochastic_grad: empty batch");
        ACCO_REQUIRE(n_samples >= 1, "sample_indices: n_samples >= 1");
        Stream s(stream_seed);
        for (int b = 0; b < batch; ++b) out[b] = static_cast<int32_t>(s.below(static_cast<uint64_t>(n_samples)));
    });
}

}  // extern "C"
