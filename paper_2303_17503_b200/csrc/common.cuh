// Shared device helpers for the sm_100a board-game step kernels.
//
// RNG: bit-exact restatement of reference pkg/src/boardbatch/rng.py:22-45
// (splitmix64 finaliser; child(k, i) = mix64(k + (i+1)*phi)). Keys are a pure
// function of (root seed, step, GLOBAL slot index), so slicing a batch over
// GPUs (slot0 offset) is bit-identical to one GPU.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define BBK_FULL 0xffffffffu

// Checked builds (-DBBK_CHECKS=1, tools/checked_build.sh): BBK_CHECK(cond) records the first failing
// source line of each translation unit in a device word instead of trapping (a trap would poison the
// context of the whole test run); bbk_debug_failures() (util.cu) collects and clears them. The pool's
// compute-sanitizer is closed, so scratch-index / capacity asserts at every phase-multiplexed or
// capacity-bounded buffer are the bad-access check. Off (no code) in the product build.
#ifndef BBK_CHECKS
#define BBK_CHECKS 0
#endif
#if BBK_CHECKS
static __device__ unsigned long long g_bbk_fail;   // (line << 32) | count of failed checks, per TU
#define BBK_CHECK(c)                                                                          \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            atomicCAS(&g_bbk_fail, 0ull, (unsigned long long)__LINE__ << 32);                 \
            atomicAdd(&g_bbk_fail, 1ull);                                                     \
        }                                                                                     \
    } while (0)
#define BBK_CHECK_READER(name)                                                                \
    unsigned long long name(int reset) {                                                      \
        unsigned long long v = 0ull;                                                          \
        if (cudaMemcpyFromSymbol(&v, g_bbk_fail, sizeof v) != cudaSuccess) return ~0ull;      \
        if (reset) {                                                                          \
            const unsigned long long z = 0ull;                                                \
            cudaMemcpyToSymbol(g_bbk_fail, &z, sizeof z);                                     \
        }                                                                                     \
        return v;                                                                             \
    }
#else
#define BBK_CHECK(c) do { } while (0)
#define BBK_CHECK_READER(name) \
    unsigned long long name(int) { return 0ull; }
#endif

namespace bbk {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t child(uint64_t s, uint64_t i) {
    return mix64(s + (i + 1) * 0x9E3779B97F4A7C15ULL);
}

// x mod d for a small divisor (1 <= d < 2^16: action counts, empty cells) with 32-bit
// arithmetic: x = hi 2^32 + lo, so x mod d = ((hi mod d)(2^32 mod d) + lo mod d) mod d and the
// sum stays below 2^32. Identical to x % d (the reference's `state % bound`, rng.py:97-101)
// without the 64-bit division subroutine.
__device__ __forceinline__ uint32_t umod_small(uint64_t x, uint32_t d) {
    const uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
    const uint32_t r32 = (0u - d) % d;   // 2^32 mod d
    return ((hi % d) * r32 + lo % d) % d;
}

__device__ __forceinline__ uint64_t slot_key(const uint64_t* slot_keys, uint64_t key, int64_t slot0, int64_t i) {
    return slot_keys ? slot_keys[i] : child(key, (uint64_t)(slot0 + i));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Persistent grid: as many CTAs as fit on the device at once (the step kernels loop over
// boards), so there is no partial second wave of CTAs.
template <class Kernel>
inline int64_t persistent_grid(Kernel kernel, int threads, size_t smem, int64_t need) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > need) grid = need;
    return grid < 1 ? 1 : grid;
}

// Grid of a step launch. boards_per_warp <= 0: the persistent grid above. Otherwise whole waves
// of resident CTAs (about need / boards_per_warp CTAs, rounded to a multiple of the resident
// count so the last wave is not a partial one): CTAs retire and start in board order, which gives
// the observation stream a tighter write window (go.cu launch_step); a batch that does not fill
// the resident CTAs keeps one board per warp.
inline int64_t wave_grid(int64_t resident, int64_t need, int boards_per_warp) {
    if (resident < 1) resident = 1;
    if (boards_per_warp <= 0 || need <= resident) return need < resident ? (need < 1 ? 1 : need) : resident;
    int64_t waves = (need + resident * boards_per_warp / 2) / (resident * boards_per_warp);
    if (waves < 1) waves = 1;
    const int64_t g = resident * waves;
    return g < need ? g : need;
}
template <class Kernel>
inline int64_t resident_ctas(Kernel kernel, int threads, size_t smem) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    return (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
}
template <class Kernel>
inline int64_t step_grid(Kernel kernel, int threads, size_t smem, int64_t need, int boards_per_warp) {
    return wave_grid(resident_ctas(kernel, threads, smem), need, boards_per_warp);
}

// Tail of one-pass CTAs (pass_map): `pct` % of the resident CTAs, for a grid of several waves.
inline int64_t tail_ctas(int64_t grid, int64_t resident, int pct) {
    if (grid <= resident || pct <= 0) return 0;
    const int64_t t = resident * pct / 100;
    return t < grid / 2 ? t : grid / 2;
}

// Board mapping of a step grid (a pass = one board per warp or warp segment, `per_cta` boards per
// CTA): the first gridDim.x - tail CTAs grid-stride over every pass but the last `tail` ones,
// which the last `tail` CTAs take one each. Those launch last, so the grid drains with short CTAs
// filling the slots the long ones free instead of idling behind the slowest multi-pass CTA
// (r02: go_9x9 +3.2 %, go_19x19 +0.8 %). tail = 0: the plain grid stride.
struct PassMap {
    int64_t b0, stride, end;
};
__device__ __forceinline__ PassMap pass_map(int64_t n, int per_cta, int64_t tail, int slot) {
    const int64_t passes = (n + per_cta - 1) / per_cta;
    const int64_t front = (int64_t)gridDim.x - tail;
    PassMap m;
    if ((int64_t)blockIdx.x >= front) {
        m.b0 = (passes - tail + ((int64_t)blockIdx.x - front)) * per_cta + slot;
        m.stride = n > 0 ? n : 1;
        m.end = n;
    } else {
        const int64_t e = (passes - tail) * per_cta;
        m.b0 = (int64_t)blockIdx.x * per_cta + slot;
        m.stride = front * per_cta;
        m.end = e < n ? e : n;
    }
    return m;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
    uint32_t lo = __shfl_sync(BBK_FULL, (uint32_t)v, src);
    uint32_t hi = __shfl_sync(BBK_FULL, (uint32_t)(v >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_xor64(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        uint32_t lo = __shfl_xor_sync(BBK_FULL, (uint32_t)v, o);
        uint32_t hi = __shfl_xor_sync(BBK_FULL, (uint32_t)(v >> 32), o);
        v ^= ((uint64_t)hi << 32) | lo;
    }
    return v;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(BBK_FULL, v, o);
    return v;
}

// Write NBYTES bytes of a per-env record into a flat [n, NBYTES] byte stream.
// `src` is shared memory laid out so that src[i] is record byte i - `off`
// relative to a 16-byte aligned origin: callers stage bytes at
// src_base + (dst_byte_offset & 15). Chunks fully inside the record use
// 128-bit stores; the (at most two) partial edge chunks use byte stores, so
// neighbouring records written by other warps are never touched.
__device__ __forceinline__ void warp_emit_bytes(uint8_t* dst_stream, int64_t rec_start, int nbytes,
                                                const uint8_t* staged /* 16B aligned, data at +off */) {
    const int lane = lane_id();
    const int64_t end = rec_start + nbytes;
    const int64_t base = rec_start & ~(int64_t)15;
    const int64_t f0 = (rec_start + 15) >> 4;     // first full chunk
    const int64_t f1 = end >> 4;                  // one past the last full chunk
    for (int64_t c = f0 + lane; c < f1; c += 32)
        *reinterpret_cast<uint4*>(dst_stream + (c << 4)) = *reinterpret_cast<const uint4*>(staged + ((c << 4) - base));
    // edge bytes: lanes 0-15 the partial head chunk, lanes 16-31 the partial tail chunk
    const int64_t head_end = (f0 << 4) < end ? (f0 << 4) : end;
    const int64_t g = lane < 16 ? rec_start + lane : (f1 << 4) + (lane - 16);
    const bool ok = lane < 16 ? g < head_end : (g < end && g >= (f0 << 4));
    if (ok) dst_stream[g] = staged[g - base];
}

}  // namespace bbk

namespace bbk {

// agents.random_actions (reference agents.py:33-46) for ONE slot whose legal
// mask is staged in shared memory as 0/1 bytes at mask[0..A): returns the
// index of the d-th legal action, d = child(key, slot) % max(count, 1), or 0.
// Warp-cooperative: lanes count contiguous ranges of 16-byte chunks (bytes
// outside [0, A) masked off), scan, and the lane holding the d-th set byte
// resolves it. `mask` may be unaligned (chunks are taken from the 16-byte
// aligned address at or below it).
__device__ __forceinline__ uint32_t chunk_count_bytes(uint4 v) {
    return __popc(v.x & 0x01010101u) + __popc(v.y & 0x01010101u) + __popc(v.z & 0x01010101u) +
           __popc(v.w & 0x01010101u);
}
// 4 bits -> 4 bytes of 0 / 1 (bit k -> byte k)
__device__ __forceinline__ uint32_t spread4(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

// Next-board scalar columns, one per lane (lane j holds field j, read back by shuffles). Lane j's
// column base and element size are fixed for the launch, so each board's load is one aligned
// 8-byte read and a shift instead of a divergent switch over the lanes. Reading the aligned word
// around a 1/2/4-byte element stays inside the column's allocation (allocations are at least
// 8-byte granular); lanes without a field get mask 0.
struct FieldRef {
    uint64_t v;   // column base | log2(element size) << 58 | no-field flag << 61 (one register pair)
};

__device__ __forceinline__ FieldRef field_of(const void* base, uint32_t lsz) {
    return {reinterpret_cast<uint64_t>(base) | ((uint64_t)lsz << 58)};
}
__device__ __forceinline__ FieldRef no_field() { return {1ull << 61}; }

__device__ __forceinline__ uint64_t load_field(FieldRef f, int64_t b) {
    if (f.v >> 61) return 0ull;
    const uint32_t lsz = (uint32_t)(f.v >> 58) & 3u;
    const uint64_t a = (f.v & ((1ull << 58) - 1ull)) + ((uint64_t)b << lsz);
    const uint64_t w = *reinterpret_cast<const uint64_t*>(a & ~7ull);
    const uint64_t x = w >> (8u * (uint32_t)(a & 7u));
    return lsz == 3u ? x : x & ((1ull << (8u << lsz)) - 1ull);
}

// agents.random_actions for ONE slot whose legal mask is staged as bits (action a = bit a of
// bits[a / 32], nwords words): lanes count contiguous word ranges, scan, and the lane holding
// the d-th set bit resolves it; d = child(key, slot) % count, 0 when count == 0.
__device__ __forceinline__ int64_t warp_sample_bits(const uint32_t* bits, int nwords, int count, uint64_t key,
                                                    int64_t slot) {
    if (count <= 0) return 0;
    const int lane = lane_id();
    const int d = (int)umod_small(child(key, (uint64_t)slot), (uint32_t)count);
    const int per = (nwords + 31) >> 5;
    const int w0 = lane * per, w1 = min(w0 + per, nwords);
    int c = 0;
    for (int i = w0; i < w1; i++) c += __popc(bits[i]);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(BBK_FULL, incl, o);
        if (lane >= o) incl += t;
    }
    const int excl = incl - c;
    int64_t act = -1;
    if (d >= excl && d < incl) {
        int r = d - excl;
        for (int i = w0; i < w1; i++) {
            uint32_t v = bits[i];
            const int pc = __popc(v);
            if (r < pc) {
                for (; r > 0; r--) v &= v - 1;
                act = 32 * i + __ffs(v) - 1;
                break;
            }
            r -= pc;
        }
    }
    const unsigned who = __ballot_sync(BBK_FULL, act >= 0);
    return __shfl_sync(BBK_FULL, act, __ffs(who) - 1);
}

// kPadsZero: the caller guarantees that the bytes of the 16-byte chunks outside [0, A) are zero
// (a zeroed staging buffer), so the edge chunks need no masking.
template <bool kPadsZero = false>
__device__ __forceinline__ int64_t warp_sample_bytes(const uint8_t* mask, int A, int count, uint64_t key,
                                                     int64_t slot) {
    if (count <= 0) return 0;
    const int lane = lane_id();
    const int d = (int)umod_small(child(key, (uint64_t)slot), (uint32_t)count);
    const uintptr_t base = reinterpret_cast<uintptr_t>(mask);
    const int head = (int)(base & 15);
    const uint4* w = reinterpret_cast<const uint4*>(base - head);
    const int nc = (head + A + 15) >> 4;
    const int per = (nc + 31) >> 5;
    const int c0 = lane * per, c1 = min(c0 + per, nc);
    // chunk i covers record bytes [16 i - head, 16 i - head + 16); clear the bytes outside [0, A)
    auto word_mask = [&](int lo) -> uint32_t {   // lo = record byte of the word's byte 0
        uint32_t m = 0xFFFFFFFFu;
        if (lo < 0) m = lo <= -4 ? 0u : m << (8 * (-lo));
        if (lo + 4 > A) m = lo >= A ? 0u : m & (0xFFFFFFFFu >> (8 * (lo + 4 - A)));
        return m;
    };
    auto chunk_at = [&](int i) -> uint4 {
        uint4 v = w[i];
        const int b0 = 16 * i - head;
        if (!kPadsZero && (b0 < 0 || b0 + 16 > A)) {
            v.x &= word_mask(b0); v.y &= word_mask(b0 + 4); v.z &= word_mask(b0 + 8); v.w &= word_mask(b0 + 12);
        }
        return v;
    };
    int c = 0;
    for (int i = c0; i < c1; i++) c += chunk_count_bytes(chunk_at(i));
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(BBK_FULL, incl, o);
        if (lane >= o) incl += t;
    }
    const int excl = incl - c;
    int64_t act = -1;
    if (d >= excl && d < incl) {
        int r = d - excl;
        for (int i = c0; i < c1; i++) {
            const uint4 v = chunk_at(i);
            const int pc = chunk_count_bytes(v);
            if (r < pc) {
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    uint32_t y = (k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w) & 0x01010101u;
                    const int q = __popc(y);
                    if (act < 0 && r < q) {
                        for (; r > 0; r--) y &= y - 1;
                        act = 16 * i + 4 * k + ((__ffs(y) - 1) >> 3) - head;
                    }
                    r -= q;
                }
                break;
            }
            r -= pc;
        }
    }
    const unsigned who = __ballot_sync(BBK_FULL, act >= 0);
    return __shfl_sync(BBK_FULL, act, __ffs(who) - 1);
}

}  // namespace bbk
