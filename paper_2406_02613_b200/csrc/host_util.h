// Host-side restatements shared by the engine and the model plugin:
// counter-based rng (proj/include/accosim/rng.hpp:13-56), shard layout
// (proj/include/accosim/shard.hpp:24-38). Integer work: bit-exact by design.
#pragma once

#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

namespace acco {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ inline uint64_t splitmix_finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

inline uint64_t splitmix64(uint64_t& state) { return splitmix_finalize(state += kGolden); }

inline uint64_t rng_mix(uint64_t a, uint64_t b) {
    uint64_t s = a;
    uint64_t h = splitmix64(s);
    s = h ^ (b + kGolden + (h << 6) + (h >> 2));
    return splitmix64(s);
}

inline uint64_t rng_derive(uint64_t master, uint64_t a, uint64_t b = 0, uint64_t c = 0,
                           uint64_t d = 0) {
    return rng_mix(rng_mix(rng_mix(rng_mix(master, a), b), c), d);
}

// The i-th (0-based) draw of Stream(seed).next_u64(): the stream is a counter,
// so any draw can be computed independently (used on device for batch indices).
__host__ __device__ inline uint64_t stream_draw(uint64_t seed, uint64_t i) {
    return splitmix_finalize(seed + (i + 1) * kGolden);
}

struct Stream {
    uint64_t state;
    explicit Stream(uint64_t s) : state(s) {}
    uint64_t next_u64() { return splitmix64(state); }
    double uniform01() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
    uint64_t below(uint64_t n) { return next_u64() % n; }
};

struct ShardLayout {
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    uint64_t dim = 0;
    int n() const { return static_cast<int>(ranges.size()); }
    uint64_t lo(int w) const { return ranges[static_cast<size_t>(w)].first; }
    uint64_t hi(int w) const { return ranges[static_cast<size_t>(w)].second; }
    uint64_t size(int w) const { return hi(w) - lo(w); }
    uint64_t chunk() const { return n() ? (dim + n() - 1) / n() : 0; }  // owner-padded chunk
};

ShardLayout shard_partition(uint64_t dim, int n);

}  // namespace acco
