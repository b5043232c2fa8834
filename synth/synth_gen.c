/*
 * synth_gen.c -- the seeded input generator of synth/__init__.py in plain C
 * (test / bench infrastructure; holds none of the method's arithmetic).
 *
 *   byte(seed, i) = splitmix64(seed * 0x9E3779B97F4A7C15 + i) >> 56
 *
 * splitmix64(x) = z ^ (z >> 31) with z = x + 0x9E3779B97F4A7C15 passed
 * through z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 and
 * z = (z ^ (z >> 27)) * 0x94D049BB133111EB (the SplitMix64 finaliser).
 * Identical bytes to synth.random_bytes (numpy), checked by
 * tests/test_oracle.py; about 30x faster, which the every-frame
 * verification of multi-GB streams needs.
 */
#include <stdint.h>

void synth_random_bytes(uint64_t seed, uint64_t start, uint64_t count, uint8_t* out) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ull;
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t z = base + start + i + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        out[i] = (uint8_t)((z ^ (z >> 31)) >> 56);
    }
}
