/* ORACLE (test infrastructure only) -- splitmix64 keys.
 *
 * Restates reference pkg/src/boardbatch/rng.py:22-29 (mix64), :43-45
 * (child_state), :97-101 (randint = state % bound), :107-117 (permutation;
 * for n=2 the Lehmer code is state % 2 and the permutation is (c, 1-c)).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this code.
 */
#ifndef ORC_RNG_H
#define ORC_RNG_H
#include <stdint.h>

#define ORC_GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t orc_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

static inline uint64_t orc_child(uint64_t state, uint64_t index) {
    return orc_mix64(state + (index + 1) * ORC_GOLDEN);
}

/* Slot key: explicit per-slot keys (scalar API) or child(key, slot0+i). */
static inline uint64_t orc_slot_key(const uint64_t* slot_keys, uint64_t key_state, int64_t slot0, int64_t i) {
    return slot_keys ? slot_keys[i] : orc_child(key_state, (uint64_t)(slot0 + i));
}

#endif
