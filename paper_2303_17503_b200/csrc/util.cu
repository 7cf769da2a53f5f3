// Generic per-slot kernels shared by every game.
//   bbk_random_actions  -- agents.random_actions (reference agents.py:33-46)
//   bbk_check_actions   -- IllegalAction detection (core.py:234-239, tictactoe.py:111-121)
//   bbk_count_finished  -- episode counter of bench_run (bench.py:129)
//   bbk_latch_finished  -- first-episode returns / lengths of a batched rollout (agents.py:113-116)
#include <climits>
#include "common.cuh"
#include "../../include/bbk.h"

namespace util {
using namespace bbk;

// Byte j of a mask row packed as 0/1 per byte; returns the word's flags
// restricted to bytes in [lo, hi) of the row (row byte = 4*w + k - head).
__device__ __forceinline__ uint32_t row_word(const uint8_t* mask, int64_t rs, int A, int w) {
    // covered row bytes: [4w - head, 4w - head + 4)
    const int64_t g0 = ((rs & ~(int64_t)3)) + 4 * (int64_t)w;   // global byte of this word
    if (g0 >= rs && g0 + 4 <= rs + A) return *reinterpret_cast<const uint32_t*>(mask + g0) & 0x01010101u;
    uint32_t v = 0u;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        int64_t g = g0 + k;
        if (g >= rs && g < rs + A) v |= (uint32_t)(mask[g] & 1u) << (8 * k);
    }
    return v;
}

__global__ void random_actions_kernel(const uint8_t* mask, int64_t n, int A, uint64_t key, int64_t slot0,
                                      int64_t* out) {
    const int lane = lane_id();
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < n; b += nwarps) {
        const int64_t rs = b * (int64_t)A;
        const int head = (int)(rs & 3);
        const int nwords = (head + A + 3) >> 2;
        int cnt = 0;
        for (int w = lane; w < nwords; w += 32) cnt += __popc(row_word(mask, rs, A, w));
        const int total = warp_sum(cnt);
        const uint64_t d64 = umod_small(child(key, (uint64_t)(slot0 + b)), (uint32_t)(total > 0 ? total : 1));
        const int d = (int)d64;
        int64_t action = 0;
        if (total > 0) {
            int base = 0;
            for (int w0 = 0; w0 < nwords; w0 += 32) {
                const int w = w0 + lane;
                const uint32_t v = w < nwords ? row_word(mask, rs, A, w) : 0u;
                const int c = __popc(v);
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int t = __shfl_up_sync(BBK_FULL, incl, o);
                    if (lane >= o) incl += t;
                }
                const int tot = __shfl_sync(BBK_FULL, incl, 31);
                if (base + tot > d) {
                    const int excl = base + incl - c;
                    const bool mine = d >= excl && d < base + incl;
                    int pos = 0;
                    if (mine) {
                        uint32_t x = v;
                        for (int r = d - excl; r > 0; r--) x &= x - 1;
                        pos = 4 * w + ((__ffs(x) - 1) >> 3) - head;
                    }
                    const unsigned who = __ballot_sync(BBK_FULL, mine);
                    action = __shfl_sync(BBK_FULL, pos, __ffs(who) - 1);
                    break;
                }
                base += tot;
            }
        }
        if (lane == 0) out[b] = action;
    }
}

// One CTA: the lowest live offending slot (or INT32_MAX) by a grid-stride scan and a block min,
// written with a plain store -- the caller needs no initialisation launch (a single kernel per check).
__global__ void __launch_bounds__(1024) check_actions_kernel(const uint8_t* mask, const uint8_t* term,
                                                             const uint8_t* trunc, const int64_t* actions, int64_t n,
                                                             int A, int32_t* first_bad) {
    __shared__ int32_t wmin[32];
    int32_t best = INT32_MAX;
    for (int64_t b = threadIdx.x; b < n && b < best; b += blockDim.x) {
        if (term[b] || trunc[b]) continue;
        const int64_t a = actions[b];
        if (a < 0 || a >= A || !mask[b * (int64_t)A + a]) best = (int32_t)b;   // b increases per thread
    }
    best = __reduce_min_sync(BBK_FULL, best);
    if (lane_id() == 0) wmin[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        int32_t v = threadIdx.x < (blockDim.x >> 5) ? wmin[threadIdx.x] : INT32_MAX;
        v = __reduce_min_sync(BBK_FULL, v);
        if (threadIdx.x == 0) *first_bad = v;
    }
}

__global__ void count_finished_kernel(const uint8_t* term, const uint8_t* trunc, int64_t n,
                                      unsigned long long* count) {
    int c = 0;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x)
        c += (term[b] | trunc[b]) ? 1 : 0;
    c = warp_sum(c);
    __shared__ int part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        int v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0;
        v = warp_sum(v);
        if (threadIdx.x == 0 && v) atomicAdd(count, (unsigned long long)v);
    }
}

// Record each slot's first finished episode: returns by player and its length; count newly
// finished slots (the host polls the count to stop the rollout).
__global__ void latch_finished_kernel(const uint8_t* term, const uint8_t* trunc, const float* rewards,
                                      const int32_t* step_count, int P, int64_t n, uint8_t* done, float* ret,
                                      int32_t* len, unsigned long long* count) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool fresh = false;
    if (b < n && !done[b] && (term[b] | trunc[b])) {
        fresh = true;
        done[b] = 1;
        for (int q = 0; q < P; q++) ret[P * b + q] = rewards[P * b + q];
        len[b] = step_count[b];
    }
    const unsigned m = __ballot_sync(BBK_FULL, fresh);
    if (lane_id() == 0 && m) atomicAdd(count, (unsigned long long)__popc(m));
}

}  // namespace util

// per-translation-unit failed-check readers (common.cuh BBK_CHECK_READER)
unsigned long long bbk_tu_fail_go(int), bbk_tu_fail_chess(int), bbk_tu_fail_shogi(int), bbk_tu_fail_backgammon(int),
    bbk_tu_fail_small(int), bbk_tu_fail_mcts(int), bbk_tu_fail_fingerprint(int);
BBK_CHECK_READER(bbk_tu_fail_util)

extern "C" {

int bbk_random_actions(const uint8_t* mask, int64_t n, int32_t num_actions, uint64_t key_state,
                       int64_t slot0, int64_t* actions, void* stream) {
    if (n <= 0) return 0;
    int64_t blocks = (n + 7) / 8;
    if (blocks > 148 * 32) blocks = 148 * 32;
    util::random_actions_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(mask, n, num_actions, key_state,
                                                                                  slot0, actions);
    return (int)cudaGetLastError();
}

int bbk_check_actions(const uint8_t* mask, const uint8_t* terminated, const uint8_t* truncated,
                      const int64_t* actions, int64_t n, int32_t num_actions, int32_t* first_bad, void* stream) {
    if (n <= 0) return 0;
    util::check_actions_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
        mask, terminated, truncated, actions, n, num_actions, first_bad);
    return (int)cudaGetLastError();
}

int bbk_count_finished(const uint8_t* terminated, const uint8_t* truncated, int64_t n,
                       unsigned long long* count, void* stream) {
    if (n <= 0) return 0;
    int64_t blocks = (n + 1023) / 1024;
    if (blocks > 148 * 4) blocks = 148 * 4;
    util::count_finished_kernel<<<(unsigned)blocks, 1024, 0, (cudaStream_t)stream>>>(terminated, truncated, n, count);
    return (int)cudaGetLastError();
}

int bbk_latch_finished(const uint8_t* term, const uint8_t* trunc, const float* rewards, const int32_t* step_count,
                       int players, int64_t n, uint8_t* done, float* returns, int32_t* lengths,
                       unsigned long long* count, void* stream) {
    if (n <= 0) return 0;
    util::latch_finished_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        term, trunc, rewards, step_count, players, n, done, returns, lengths, count);
    return (int)cudaGetLastError();
}

int bbk_fetch_async(int count, void* const* dst, const void* const* src, const int64_t* bytes,
                    void* main_stream, void* copy_stream, void* after, void* done) {
    if (count < 0 || count > 8) return (int)cudaErrorInvalidValue;
    cudaStream_t ms = (cudaStream_t)main_stream, cs = (cudaStream_t)copy_stream;
    cudaError_t e = cudaEventRecord((cudaEvent_t)after, ms);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, (cudaEvent_t)after, 0);
    for (int i = 0; i < count && e == cudaSuccess; i++)
        if (bytes[i] > 0) e = cudaMemcpyAsync(dst[i], src[i], (size_t)bytes[i], cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && done) e = cudaEventRecord((cudaEvent_t)done, cs);
    return (int)e;
}

int bbk_abi_version(void) { return BBK_ABI_VERSION; }

const char* bbk_build_info(void) {
    return BBK_CHECKS ? "libbbk: sm_100a (compute_100a), checked build (BBK_CHECKS)" : "libbbk: sm_100a (compute_100a)";
}

int bbk_debug_checks(void) { return BBK_CHECKS; }

int bbk_debug_failures(int reset, unsigned long long* out, int n) {
    unsigned long long (*const tus[])(int) = {bbk_tu_fail_go, bbk_tu_fail_chess, bbk_tu_fail_shogi,
                                              bbk_tu_fail_backgammon, bbk_tu_fail_small, bbk_tu_fail_mcts,
                                              bbk_tu_fail_fingerprint, bbk_tu_fail_util};
    int bad = 0;
    for (int i = 0; i < 8; i++) {
        const unsigned long long v = tus[i](reset);
        if (i < n && out) out[i] = v;
        bad += v != 0ull;
    }
    return bad;
}

}  // extern "C"
