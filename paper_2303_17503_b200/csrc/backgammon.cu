// Backgammon batched step for sm_100a.
//
// Replaces reference pkg/src/boardbatch/games/backgammon.py: _legal_mask
// :62-95, _roll :125-130 (dice from child(k,0)%6+1, child(k,1)%6+1),
// _init_core :133-134, _final :137-147, _apply :150-193, _observe :196-206,
// and the env-core wrapping (core.py:192-243, 353-386).
//
// The state is 36 bytes per env, so one THREAD owns one board; the warp
// stages its 32 boards' mask (156 B each) and observation (34 floats each)
// rows in shared memory and writes them as contiguous 16-byte chunks.
#include "common.cuh"
#include "../../include/bbk.h"

namespace bg {
using namespace bbk;

constexpr int A = 156;
constexpr int OBS = 34;
constexpr int kWarps = 4;

struct WarpSmem {
    alignas(16) uint8_t mb[32 * A + 32];
    alignas(16) float ob[32 * OBS + 8];
};

struct Params {
    bbk_cols in, out;
    bbk_bg_state in_s, out_s;
    const int64_t* actions;
    const uint64_t* slot_keys;
    int64_t n, slot0;
    uint64_t key;
    int32_t max_steps;
    int force_reset;
};

struct Board {
    int8_t pts[24];
    uint8_t bar[2], off[2];
    uint8_t role, d1, d2, nrem;
    uint8_t rem[4];
    bool terminal;
    float rr0, rr1;
};

__device__ __constant__ int8_t kStart[24] = {2, 0, 0, 0, 0, -5, 0, -3, 0, 0, 0, 5, -5, 0, 0, 0, 3, 0, 5, 0, 0, 0, 0, -2};

// Board points are read and written with run-time indices through these unrolled
// compare-and-select loops, so `pts` stays in registers (a dynamically indexed local array
// would live in local memory: every access a long-scoreboard round trip).
__device__ __forceinline__ int get_pt(const Board& s, int a) {
    int v = 0;
#pragma unroll
    for (int j = 0; j < 24; j++) v = j == a ? (int)s.pts[j] : v;
    return v;
}
__device__ __forceinline__ void add_pt(Board& s, int a, int d) {
#pragma unroll
    for (int j = 0; j < 24; j++) s.pts[j] = (int8_t)(j == a ? s.pts[j] + d : s.pts[j]);
}
__device__ __forceinline__ void set_pt(Board& s, int a, int v) {
#pragma unroll
    for (int j = 0; j < 24; j++) s.pts[j] = (int8_t)(j == a ? v : s.pts[j]);
}
// bar / off of a run-time role, by select (a role-indexed array would live in local memory)
__device__ __forceinline__ int bar_of(const Board& s, int r) { return r ? s.bar[1] : s.bar[0]; }
__device__ __forceinline__ int off_of(const Board& s, int r) { return r ? s.off[1] : s.off[0]; }
__device__ __forceinline__ void add_bar(Board& s, int r, int d) { if (r) s.bar[1] += d; else s.bar[0] += d; }
__device__ __forceinline__ void add_off(Board& s, int r, int d) { if (r) s.off[1] += d; else s.off[0] += d; }

// OR action bit `bit` into the 5 mask words (held in registers)
__device__ __forceinline__ void set_bit5(uint32_t m[5], int bit) {
    const int w = bit >> 5;
    const uint32_t v = 1u << (bit & 31);
#pragma unroll
    for (int j = 0; j < 5; j++) m[j] |= j == w ? v : 0u;
}

// _legal_mask (backgammon.py:62-95) as 5 words of action bits, bit-parallel over pips:
// OWN / BLOCK (>= 2 opponent checkers) as 24-bit pip masks (bit p-1 = pip p, mover frame), then
// per die the movable pips are OWN & ~(BLOCK << die) above the die, plus bear-offs.
__device__ __forceinline__ void legal_mask(const Board& s, uint32_t m[5]) {
#pragma unroll
    for (int j = 0; j < 5; j++) m[j] = 0u;
    const int role = s.role, sign = role == 0 ? 1 : -1;
    uint32_t dset = 0u;
#pragma unroll
    for (int j = 0; j < 4; j++) dset |= j < s.nrem ? 1u << s.rem[j] : 0u;
    uint32_t own = 0u, blk = 0u;   // absolute point order first
#pragma unroll
    for (int j = 0; j < 24; j++) {
        const int v = s.pts[j] * sign;
        own |= (uint32_t)(v > 0) << j;
        blk |= (uint32_t)(v <= -2) << j;
    }
    if (role == 0) { own = __brev(own) >> 8; blk = __brev(blk) >> 8; }   // pip p <-> point 24 - p
    bool any = false;
    if (bar_of(s, role) > 0) {   // enter on pip 25 - die
        for (int die = 1; die <= 6; die++) {
            if (!((dset >> die) & 1u)) continue;
            if (!((blk >> (24 - die)) & 1u)) { set_bit5(m, 6 + die - 1); any = true; }
        }
        if (!any) m[0] |= 1u;
        return;
    }
    const int rear = own ? 32 - __clz(own) : 0;   // rearmost own pip
    const bool can_bear_off = rear <= 6;
    for (int die = 1; die <= 6; die++) {
        if (!((dset >> die) & 1u)) continue;
        uint32_t mv = own & ~(blk << die) & ~((1u << die) - 1u);   // pip - die >= 1, target not blocked
        if (can_bear_off) {                                        // pip - die < 1: die == pip or pip == rear
            mv |= own & (1u << (die - 1));
            if (rear >= 1 && rear <= die) mv |= 1u << (rear - 1);
        }
        for (; mv; mv &= mv - 1) {
            const int pip = __ffs(mv);
            set_bit5(m, (pip + 1) * 6 + die - 1);
            any = true;
        }
    }
    if (!any) m[0] |= 1u;
}

__device__ __forceinline__ void roll(Board& s, int role, uint64_t key) {
    int d1 = (int)(child(key, 0) % 6ull) + 1;
    int d2 = (int)(child(key, 1) % 6ull) + 1;
    s.role = (uint8_t)role; s.d1 = (uint8_t)d1; s.d2 = (uint8_t)d2;
    if (d1 == d2) { s.nrem = 4; s.rem[0] = s.rem[1] = s.rem[2] = s.rem[3] = (uint8_t)d1; }
    else { s.nrem = 2; s.rem[0] = (uint8_t)d1; s.rem[1] = (uint8_t)d2; s.rem[2] = s.rem[3] = 0; }
    s.terminal = false; s.rr0 = s.rr1 = 0.0f;
}

__device__ __forceinline__ int sgn_at(const Board& s, int role, int a) { const int v = get_pt(s, a); return role == 0 ? v : -v; }
__device__ __forceinline__ int abs_point(int role, int pip) { return role == 0 ? 24 - pip : pip - 1; }

__device__ __forceinline__ void final_(Board& s, int winner) {
    int loser = 1 - winner;
    float value = 1.0f;
    if (off_of(s, loser) == 0) {
        value = 2.0f;
        bool in_home = false;
        int lo = winner == 0 ? 18 : 0;
        for (int a = lo; a < lo + 6; a++) in_home |= sgn_at(s, loser, a) > 0;
        if (bar_of(s, loser) > 0 || in_home) value = 3.0f;
    }
    s.rr0 = winner == 0 ? value : -value;
    s.rr1 = winner == 0 ? -value : value;
    s.role = (uint8_t)loser; s.d1 = s.d2 = 0; s.nrem = 0;
    s.rem[0] = s.rem[1] = s.rem[2] = s.rem[3] = 0;
    s.terminal = true;
}

// _apply (backgammon.py:150-193)
__device__ __forceinline__ void apply(Board& s, int action, uint64_t key) {
    const int role = s.role;
    const int src = action / 6, die = action - 6 * src + 1;
    if (src == 0) { roll(s, 1 - role, key); return; }
    const int delta = role == 0 ? 1 : -1;
    int target;
    if (src == 1) { add_bar(s, role, -1); target = 25 - die; }
    else { int pip = src - 1; add_pt(s, abs_point(role, pip), -delta); target = pip - die; }
    if (src != 1 && target < 1) {
        add_off(s, role, 1);
    } else {
        int a = abs_point(role, target);
        if (sgn_at(s, role, a) == -1) { set_pt(s, a, delta); add_bar(s, 1 - role, 1); }
        else add_pt(s, a, delta);
    }
    if (off_of(s, role) == 15) { final_(s, role); return; }
    // consume the first remaining die equal to `die` (unrolled: rem stays in registers)
    int idx = 4;
#pragma unroll
    for (int j = 0; j < 4; j++) idx = (idx == 4 && j < s.nrem && s.rem[j] == die) ? j : idx;
#pragma unroll
    for (int j = 0; j < 3; j++) s.rem[j] = (j >= idx && j + 1 < s.nrem) ? s.rem[j + 1] : s.rem[j];
    if (s.nrem > 0) {
        s.nrem -= 1;
#pragma unroll
        for (int j = 0; j < 4; j++) s.rem[j] = j == s.nrem ? (uint8_t)0 : s.rem[j];
    }
    if (s.nrem == 0) { roll(s, 1 - role, key); return; }
    s.rr0 = s.rr1 = 0.0f;
}

__device__ __forceinline__ void observe(const Board& s, int role, float* o /* 34, shared */) {
#pragma unroll
    for (int pip = 1; pip <= 24; pip++)   // role 0: point 24 - pip, role 1: point pip - 1 (negated)
        o[pip - 1] = role == 0 ? (float)s.pts[24 - pip] : (float)(-s.pts[pip - 1]);
    o[24] = bar_of(s, role); o[25] = bar_of(s, 1 - role);
    o[26] = off_of(s, role); o[27] = off_of(s, 1 - role);
#pragma unroll
    for (int d = 0; d < 6; d++) {   // remaining-dice histogram
        int c = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) c += (j < s.nrem && s.rem[j] == d + 1) ? 1 : 0;
        o[28 + d] = (float)c;
    }
}

__device__ __forceinline__ void load_board(Board& s, const bbk_bg_state& st, int64_t b) {
    const int8_t* p = st.points + b * 24;
#pragma unroll
    for (int j = 0; j < 24; j++) s.pts[j] = p[j];
    const uint8_t* m = st.misc + b * 12;
    s.bar[0] = m[0]; s.bar[1] = m[1]; s.off[0] = m[2]; s.off[1] = m[3];
    s.role = m[4]; s.d1 = m[5]; s.d2 = m[6];
    s.rem[0] = m[7]; s.rem[1] = m[8]; s.rem[2] = m[9]; s.rem[3] = m[10]; s.nrem = m[11];
}

__device__ __forceinline__ void store_board(const Board& s, const bbk_bg_state& st, int64_t b) {
    int8_t* p = st.points + b * 24;
#pragma unroll
    for (int j = 0; j < 24; j++) p[j] = s.pts[j];
    uint8_t* m = st.misc + b * 12;
    m[0] = s.bar[0]; m[1] = s.bar[1]; m[2] = s.off[0]; m[3] = s.off[1];
    m[4] = s.role; m[5] = s.d1; m[6] = s.d2;
    m[7] = s.rem[0]; m[8] = s.rem[1]; m[9] = s.rem[2]; m[10] = s.rem[3]; m[11] = s.nrem;
}

__global__ void __launch_bounds__(kWarps * 32) step_kernel(Params p) {
    __shared__ WarpSmem sm[kWarps];
    WarpSmem& S = sm[threadIdx.x >> 5];
    const int lane = lane_id();
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    unsigned long long eps = 0;
    for (int64_t base = ((int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5)) * 32; base < p.n; base += nwarps * 32) {
        const int64_t b = base + lane;
        const bool live = b < p.n;
        Board s;
        int8_t p2r0 = 0, p2r1 = 0;
        int step = 0;
        bool truncated = false;
        uint32_t m[5] = {0u, 0u, 0u, 0u, 0u};
        if (live) {
            const uint64_t k = slot_key(p.slot_keys, p.key, p.slot0, b);
            const bool reset = p.force_reset || p.in.terminated[b] || p.in.truncated[b];
            if (reset) {
                int c = (int)(child(k, 0) % 2ull);
                p2r0 = (int8_t)c; p2r1 = (int8_t)(1 - c);
#pragma unroll
                for (int j = 0; j < 24; j++) s.pts[j] = kStart[j];
                s.bar[0] = s.bar[1] = s.off[0] = s.off[1] = 0;
                roll(s, 0, child(k, 1));
                step = 0;
            } else {
                load_board(s, p.in_s, b);
                s.terminal = false; s.rr0 = s.rr1 = 0.0f;
                p2r0 = p.in.player_to_role[2 * b]; p2r1 = p.in.player_to_role[2 * b + 1];
                step = p.in.step_count[b] + 1;
                int a = (int)p.actions[b];
                if (a < 0 || a >= A) a = 0;
                apply(s, a, k);
            }
            truncated = !s.terminal && step >= p.max_steps;
            if (!s.terminal && !truncated) legal_mask(s, m);
            eps += (s.terminal || truncated) ? 1 : 0;
            if (p.out.next_actions) {   // fused agents.random_actions on the new mask
                const int count = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]) + __popc(m[4]);
                int64_t act = 0;
                if (count > 0) {
                    int d = (int)(child(p.out.next_key, (uint64_t)(p.slot0 + b)) % (uint64_t)count);   // (umod_small measured slower here)
#pragma unroll
                    for (int j = 0; j < 5; j++) {
                        const int pc = __popc(m[j]);
                        if (d < pc) {
                            uint32_t v = m[j];
                            for (; d > 0; d--) v &= v - 1;
                            act = 32 * j + __ffs(v) - 1;
                            break;
                        }
                        d -= pc;
                    }
                }
                p.out.next_actions[b] = act;
            }
            store_board(s, p.out_s, b);
            float r0 = 0.0f, r1 = 0.0f;
            if (!truncated && (s.rr0 != 0.0f || s.rr1 != 0.0f)) {
                r0 = p2r0 == 0 ? s.rr0 : s.rr1;
                r1 = p2r1 == 0 ? s.rr0 : s.rr1;
            }
            p.out.rewards[2 * b] = r0; p.out.rewards[2 * b + 1] = r1;
            p.out.terminated[b] = s.terminal; p.out.truncated[b] = truncated;
            p.out.step_count[b] = step;
            p.out.current_player[b] = p2r0 == s.role ? 0 : 1;
            p.out.player_to_role[2 * b] = p2r0; p.out.player_to_role[2 * b + 1] = p2r1;
            // stage mask bytes (record phase = (base*A) & 15, constant per warp)
            // base is a multiple of 32, so the record phase is 0 and rows are 4-byte aligned (A = 4 * 39)
            uint32_t* mrow = reinterpret_cast<uint32_t*>(S.mb + lane * A);
#pragma unroll
            for (int w = 0; w < A / 4; w++) mrow[w] = spread4((m[(4 * w) >> 5] >> ((4 * w) & 31)) & 15u);
            if (p.out.observation) observe(s, s.role, S.ob + ((base * OBS) & 3) + lane * OBS);
        }
        __syncwarp();
        const int64_t cnt = p.n - base < 32 ? p.n - base : 32;
        warp_emit_bytes(p.out.legal_action_mask, base * A, (int)(cnt * A), S.mb);
        if (p.out.observation)
            warp_emit_bytes(reinterpret_cast<uint8_t*>(p.out.observation), base * OBS * 4, (int)(cnt * OBS * 4),
                            reinterpret_cast<const uint8_t*>(S.ob));
        __syncwarp();
    }
    if (p.out.episodes) {
        const int e = warp_sum((int)eps);
        if (lane == 0 && e) atomicAdd(p.out.episodes, (unsigned long long)e);
    }
}

__global__ void observe_kernel(bbk_bg_state st, const uint8_t* role, float* obs, int64_t n) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    Board s;
    load_board(s, st, b);
    float o[OBS];
    observe(s, role[b], o);
    for (int j = 0; j < OBS; j++) obs[b * OBS + j] = o[j];
}

static int launch(const Params& p, cudaStream_t stream) {
    int64_t warps = (p.n + 31) / 32;
    int64_t grid = (warps + kWarps - 1) / kWarps;
    if (grid > 148 * 16) grid = 148 * 16;
    step_kernel<<<(unsigned)(grid < 1 ? 1 : grid), kWarps * 32, 0, stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace bg

extern "C" {

int bbk_bg_init(const bbk_cols* out, const bbk_bg_state* out_s, int64_t n, int64_t slot0,
                uint64_t key_state, const uint64_t* slot_keys, int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    bg::Params p{};
    p.out = *out; p.out_s = *out_s; p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state;
    p.max_steps = max_steps; p.force_reset = 1;
    return bg::launch(p, (cudaStream_t)stream);
}

int bbk_bg_step(const bbk_cols* in, const bbk_bg_state* in_s, const bbk_cols* out, const bbk_bg_state* out_s,
                const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state,
                const uint64_t* slot_keys, int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    bg::Params p{};
    p.in = *in; p.in_s = *in_s; p.out = *out; p.out_s = *out_s; p.actions = actions;
    p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state; p.max_steps = max_steps;
    p.force_reset = 0;
    return bg::launch(p, (cudaStream_t)stream);
}

int bbk_bg_observe(const bbk_bg_state* s, const uint8_t* role, float* obs, int64_t n, void* stream) {
    if (n <= 0) return 0;
    bg::observe_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*s, role, obs, n);
    return (int)cudaGetLastError();
}

}  // extern "C"

// checked builds: this translation unit's failed-check word (common.cuh BBK_CHECK)
BBK_CHECK_READER(bbk_tu_fail_backgammon)
