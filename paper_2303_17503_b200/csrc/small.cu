// Batched init / step / observe for the reference's small engines
// (small.cuh), one thread per slot: the env-core contract of
// core._make_state / batch_step (core.py:192-220, 353-386) around each
// engine -- auto-reset of finished slots from child(key, slot) (permutation
// from child(k, 0), core from child(k, 1)), step count, truncation at
// max_steps, rewards by player (zero when truncated), mask zeroed when
// finished, current_player = perm.index(role_to_move), the observation of the
// side to move, and the same fused next-step random actions / episode counter
// as the big games.
#include "small.cuh"
#include "../../include/bbk.h"

namespace small {

struct Params {
    bbk_cols in, out;
    const uint8_t* in_blob;
    uint8_t* out_blob;
    const int64_t* actions;
    const uint64_t* slot_keys;
    int64_t n, slot0;
    uint64_t key;
    int32_t max_steps;
    int force_reset;
};

__device__ __forceinline__ void load(St& s, const uint8_t* p) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4* d = reinterpret_cast<uint4*>(s.b);
#pragma unroll
    for (int i = 0; i < kStateBytes / 16; i++) d[i] = q[i];
}
__device__ __forceinline__ void store(uint8_t* p, const St& s) {
    uint4* q = reinterpret_cast<uint4*>(p);
    const uint4* d = reinterpret_cast<const uint4*>(s.b);
#pragma unroll
    for (int i = 0; i < kStateBytes / 16; i++) q[i] = d[i];
}

// d-th set bit of a mask (agents.random_actions, agents.py:33-46)
__device__ __forceinline__ int64_t select_bit(Mask128 m, int d) {
    const int cl = __popcll(m.lo);
    uint64_t w = d < cl ? m.lo : m.hi;
    int r = d < cl ? d : d - cl;
    for (; r > 0; r--) w &= w - 1;
    return (d < cl ? 0 : 64) + __ffsll((long long)w) - 1;
}

// one slot's env-core step (everything but the observation, which the warp emits)
template <class G>
__device__ __forceinline__ void step_slot(const Params& p, int64_t b, uint8_t* sblob, uint8_t& srole, uint8_t& sterm) {
    constexpr int P = G::P;
    const bool reset = p.force_reset || p.in.terminated[b] || p.in.truncated[b];
    const uint64_t k = slot_key(p.slot_keys, p.key, p.slot0, b);
    St s;
    int perm0 = 0, step;
    bool terminal;
    float rr0 = 0.0f, rr1 = 0.0f;
    if (reset) {   // core.init (core.py:223-229)
        if (P == 2) perm0 = (int)(child(k, 0) % 2ull);
        terminal = G::init(s, child(k, 1));
        step = 0;
    } else {
        load(s, p.in_blob + b * kStateBytes);
        perm0 = P == 2 ? (int)p.in.player_to_role[2 * b] : 0;
        step = p.in.step_count[b] + 1;
        const Out o = G::apply(s, (int)p.actions[b], k);
        terminal = o.terminal;
        rr0 = o.r0; rr1 = o.r1;
    }
    const bool truncated = !terminal && step >= p.max_steps;
    float r[2] = {0.0f, 0.0f};
    if (!truncated && (rr0 != 0.0f || rr1 != 0.0f)) {   // role_rewards[perm[p]] (core.py:197-204)
        if (P == 2) { r[0] = perm0 == 0 ? rr0 : rr1; r[1] = perm0 == 0 ? rr1 : rr0; }
        else r[0] = rr0;
    }
    const Mask128 m = (terminal || truncated) ? Mask128{0, 0} : G::mask(s);
    uint8_t* mk = p.out.legal_action_mask + b * (int64_t)G::A;
    for (int a = 0; a < G::A; a++) mk[a] = m.has(a) ? 1 : 0;
    const int role = G::role(s);
    *reinterpret_cast<St*>(sblob) = s;
    srole = (uint8_t)role;
    sterm = terminal ? 1 : 0;
    for (int q = 0; q < P; q++) p.out.rewards[P * b + q] = r[q];
    p.out.terminated[b] = terminal;
    p.out.truncated[b] = truncated;
    p.out.step_count[b] = step;
    p.out.current_player[b] = P == 2 ? (perm0 == role ? 0 : 1) : 0;
    p.out.player_to_role[P * b] = (int8_t)perm0;
    if (P == 2) p.out.player_to_role[P * b + 1] = (int8_t)(1 - perm0);
    store(p.out_blob + b * kStateBytes, s);
    if (p.out.next_actions) {
        const int cnt = m.count();
        int64_t act = 0;
        if (cnt > 0) act = select_bit(m, (int)umod_small(child(p.out.next_key, (uint64_t)(p.slot0 + b)), (uint32_t)cnt));
        p.out.next_actions[b] = act;
    }
    if (p.out.episodes && (terminal || truncated)) atomicAdd(p.out.episodes, 1ull);
}

constexpr int kWarps = 4;

template <class G>
__global__ void __launch_bounds__(kWarps * 32) step_kernel(Params p) {
    // each warp's 32 slots' Cores are staged in shared memory so the warp can write their
    // observation records (one contiguous region) with coalesced float4 stores
    __shared__ __align__(16) uint8_t sblob[kWarps][32][kStateBytes];
    __shared__ uint8_t srole[kWarps][32], sterm[kWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t base = ((int64_t)blockIdx.x * kWarps + warp) * 32;
    if (base >= p.n) return;   // whole warp past the batch
    const int64_t b = base + lane;
    const int cnt = p.n - base < 32 ? (int)(p.n - base) : 32;
    if (b < p.n) step_slot<G>(p, b, sblob[warp][lane], srole[warp][lane], sterm[warp][lane]);
    __syncwarp();
    if (p.out.observation) {
        constexpr int OBS = G::OBS;
        float* reg = p.out.observation + base * (int64_t)OBS;   // 16-byte aligned (base % 32 == 0)
        const int nf = cnt * OBS;
        for (int j = lane; 4 * j < nf; j += 32) {
            float v[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int g = 4 * j + t, slot = g / OBS, f = g - OBS * slot;
                v[t] = g < nf ? G::obs_at(*reinterpret_cast<const St*>(sblob[warp][slot]), srole[warp][slot],
                                          sterm[warp][slot] != 0, f) : 0.0f;
            }
            if (4 * j + 3 < nf) reinterpret_cast<float4*>(reg)[j] = make_float4(v[0], v[1], v[2], v[3]);
            else
                for (int t = 0; t < 4 && 4 * j + t < nf; t++) reg[4 * j + t] = v[t];
        }
    }
}

template <class G>
__global__ void observe_kernel(const uint8_t* blob, const uint8_t* terminated, const uint8_t* role, float* obs, int64_t n) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    St s;
    load(s, blob + b * kStateBytes);
    G::observe(s, role[b], terminated[b] != 0, obs + b * (int64_t)G::OBS);
}

template <class G>
int launch_step(const Params& p, cudaStream_t st) {
    if (p.n <= 0) return 0;
    step_kernel<G><<<(unsigned)((p.n + kWarps * 32 - 1) / (kWarps * 32)), kWarps * 32, 0, st>>>(p);
    return (int)cudaGetLastError();
}

template <class F>
int dispatch(int game, F&& f) {
    switch (game) {
        case 0: return f(TicTacToe{});
        case 1: return f(ConnectFour{});
        case 2: return f(Othello{});
        case 3: return f(Hex{});
        case 4: return f(Play2048{});
        case 5: return f(Kuhn{});
        case 6: return f(Leduc{});
        default: return (int)cudaErrorInvalidValue;
    }
}

}  // namespace small

extern "C" {

int bbk_small_state_bytes(void) { return small::kStateBytes; }

int bbk_small_init(int game, const bbk_cols* out, uint8_t* out_blob, int64_t n, int64_t slot0, uint64_t key_state,
                   const uint64_t* slot_keys, int32_t max_steps, void* stream) {
    small::Params p{};
    p.in = *out;
    p.out = *out;
    p.out_blob = out_blob;
    p.slot_keys = slot_keys;
    p.n = n; p.slot0 = slot0; p.key = key_state; p.max_steps = max_steps; p.force_reset = 1;
    return small::dispatch(game, [&](auto g) { return small::launch_step<decltype(g)>(p, (cudaStream_t)stream); });
}

int bbk_small_step(int game, const bbk_cols* in, const uint8_t* in_blob, const bbk_cols* out, uint8_t* out_blob,
                   const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                   int32_t max_steps, void* stream) {
    small::Params p{};
    p.in = *in;
    p.out = *out;
    p.in_blob = in_blob;
    p.out_blob = out_blob;
    p.actions = actions;
    p.slot_keys = slot_keys;
    p.n = n; p.slot0 = slot0; p.key = key_state; p.max_steps = max_steps; p.force_reset = 0;
    return small::dispatch(game, [&](auto g) { return small::launch_step<decltype(g)>(p, (cudaStream_t)stream); });
}

int bbk_small_observe(int game, const uint8_t* blob, const uint8_t* terminated, const uint8_t* role, float* obs,
                      int64_t n, void* stream) {
    if (n <= 0) return 0;
    return small::dispatch(game, [&](auto g) {
        small::observe_kernel<decltype(g)><<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
            blob, terminated, role, obs, n);
        return (int)cudaGetLastError();
    });
}

}  // extern "C"

// checked builds: this translation unit's failed-check word (common.cuh BBK_CHECK)
BBK_CHECK_READER(bbk_tu_fail_small)
