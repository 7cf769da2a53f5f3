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

// _legal_mask (backgammon.py:62-95) as 5 words of action bits.
__device__ void legal_mask(const Board& s, uint32_t m[5]) {
#pragma unroll
    for (int j = 0; j < 5; j++) m[j] = 0u;
    const int role = s.role, sign = role == 0 ? 1 : -1;
    uint32_t dset = 0u;
    for (int j = 0; j < s.nrem; j++) dset |= 1u << s.rem[j];
    bool any = false;
    if (s.bar[role] > 0) {
        for (int die = 1; die <= 6; die++) {
            if (!((dset >> die) & 1u)) continue;
            int dest = role == 0 ? die - 1 : 24 - die;
            if (s.pts[dest] * sign >= -1) { int bit = 6 + die - 1; m[bit >> 5] |= 1u << (bit & 31); any = true; }
        }
        if (!any) m[0] |= 1u;
        return;
    }
    int rear = 0;
    for (int a = 0; a < 24; a++)
        if (s.pts[a] * sign > 0) { int pip = role == 0 ? 24 - a : a + 1; rear = pip > rear ? pip : rear; }
    const bool can_bear_off = rear <= 6;
    for (int die = 1; die <= 6; die++) {
        if (!((dset >> die) & 1u)) continue;
        for (int pip = 1; pip <= 24; pip++) {
            int src = role == 0 ? 24 - pip : pip - 1;
            if (s.pts[src] * sign < 1) continue;
            int target = pip - die;
            bool ok;
            if (target >= 1) {
                int dest = role == 0 ? 24 - target : target - 1;
                ok = s.pts[dest] * sign >= -1;
            } else {
                ok = can_bear_off && (die == pip || pip == rear);
            }
            if (ok) { int bit = (pip + 1) * 6 + die - 1; m[bit >> 5] |= 1u << (bit & 31); any = true; }
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

__device__ __forceinline__ int sgn_at(const Board& s, int role, int a) { return role == 0 ? s.pts[a] : -s.pts[a]; }
__device__ __forceinline__ int abs_point(int role, int pip) { return role == 0 ? 24 - pip : pip - 1; }

__device__ void final_(Board& s, int winner) {
    int loser = 1 - winner;
    float value = 1.0f;
    if (s.off[loser] == 0) {
        value = 2.0f;
        bool in_home = false;
        int lo = winner == 0 ? 18 : 0;
        for (int a = lo; a < lo + 6; a++) in_home |= sgn_at(s, loser, a) > 0;
        if (s.bar[loser] > 0 || in_home) value = 3.0f;
    }
    s.rr0 = winner == 0 ? value : -value;
    s.rr1 = winner == 0 ? -value : value;
    s.role = (uint8_t)loser; s.d1 = s.d2 = 0; s.nrem = 0;
    s.rem[0] = s.rem[1] = s.rem[2] = s.rem[3] = 0;
    s.terminal = true;
}

// _apply (backgammon.py:150-193)
__device__ void apply(Board& s, int action, uint64_t key) {
    const int role = s.role;
    const int src = action / 6, die = action - 6 * src + 1;
    if (src == 0) { roll(s, 1 - role, key); return; }
    const int delta = role == 0 ? 1 : -1;
    int target;
    if (src == 1) { s.bar[role] -= 1; target = 25 - die; }
    else { int pip = src - 1; s.pts[abs_point(role, pip)] -= (int8_t)delta; target = pip - die; }
    if (src != 1 && target < 1) {
        s.off[role] += 1;
    } else {
        int a = abs_point(role, target);
        if (sgn_at(s, role, a) == -1) { s.pts[a] = (int8_t)delta; s.bar[1 - role] += 1; }
        else s.pts[a] += (int8_t)delta;
    }
    if (s.off[role] == 15) { final_(s, role); return; }
    int j = 0;
    while (j < s.nrem && s.rem[j] != die) j++;
    for (; j + 1 < s.nrem; j++) s.rem[j] = s.rem[j + 1];
    if (s.nrem > 0) { s.nrem -= 1; s.rem[s.nrem & 3] = 0; }
    if (s.nrem == 0) { roll(s, 1 - role, key); return; }
    s.rr0 = s.rr1 = 0.0f;
}

__device__ void observe(const Board& s, int role, float* o /* 34, shared */) {
    for (int pip = 1; pip <= 24; pip++) o[pip - 1] = (float)sgn_at(s, role, abs_point(role, pip));
    o[24] = s.bar[role]; o[25] = s.bar[1 - role];
    o[26] = s.off[role]; o[27] = s.off[1 - role];
    float cnt[6] = {0, 0, 0, 0, 0, 0};
    for (int j = 0; j < s.nrem; j++) cnt[s.rem[j] - 1] += 1.0f;
    for (int d = 0; d < 6; d++) o[28 + d] = cnt[d];
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
                    int d = (int)(child(p.out.next_key, (uint64_t)(p.slot0 + b)) % (uint64_t)count);
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
            uint8_t* mrow = S.mb + ((base * A) & 15) + lane * A;
            for (int j = 0; j < A; j++) mrow[j] = (uint8_t)((m[j >> 5] >> (j & 31)) & 1u);
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
