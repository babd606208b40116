// kpm_rng.cuh -- counter-based Rademacher start vectors, generated on the fly.
//
// The paper draws the random vector inside its GPU kernel ("including the random
// number generation for r") from iid real xi with <<xi>> = 0 and
// <<xi xi'>> = delta delta (Eq 14).  Reading X1:
// xi_{r,i} = 1 - 2 * (mix64(key ^ ctr) >> 63), key = mix64(seed + 0x9E3779B97F4A7C15),
// ctr = r * D + i over global indices; mix64 = the splitmix64 finaliser.  A vector
// element is a pure function of (seed, r, i), so the first-step kernel regenerates
// neighbours instead of reading a stored a_0, and the vector set is independent of
// how vectors or rows are split across GPUs.
#pragma once
#include <cstdint>

namespace kpm {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t vector_key(uint64_t seed) {
    return mix64(seed + 0x9E3779B97F4A7C15ull);
}

// +1.0 or -1.0
__device__ __forceinline__ double rademacher(uint64_t key, uint64_t ctr) {
    return 1.0 - 2.0 * (double)(mix64(key ^ ctr) >> 63);
}

}  // namespace kpm
