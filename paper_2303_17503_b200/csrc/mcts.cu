// Batched UCT search (reference agents.py:49-131, mcts_agent) on the device.
//
// One search per root state, all searches advancing in lockstep one simulation at a time:
//   select   one thread per search walks its tree (UCB over the children of fully expanded
//            nodes, agents.py:89-101), then pops a random untried action (agents.py:103-109)
//            and allocates the child node;
//   expand   the host copies the parent rows of the node pool into a staging batch, runs the
//            game's own step kernel once and scatters the children back into the pool
//            (bbk_copy_rows);
//   rollout  uniform random play to the end of the episode (agents.py:111-116) with the game's
//            step kernel, one warp per search drawing the actions;
//   backup   one thread per search credits every edge of its path from the mover's
//            perspective (agents.py:117-122).
// Each search owns a Mersenne Twister stream seeded like Python's random.Random(key.state)
// (agents.py:85) and consumes it in the reference's order -- the expansion draw, then one draw
// per rollout move -- through randrange(n) = getrandbits(bit_length(n)) with rejection
// (CPython Lib/random.py _randbelow_with_getrandbits, Modules/_randommodule.c). UCB scores are
// evaluated in double precision with the reference's operation order and no FMA contraction
// (explicit _rn intrinsics); log(visits) comes from a host table computed with the host's libm
// (Python math.log), so the chosen actions are bit-for-bit the reference's.
#include "common.cuh"
#include "../../include/bbk.h"

namespace mcts {
using namespace bbk;

constexpr int kN = 624, kM = 397;

// ---- MT19937 (Matsumoto & Nishimura 2002; CPython _randommodule.c init_genrand /
// init_by_array / genrand_uint32), state block: mt[0..623] words, mt[624] = index.
__host__ __device__ inline void mt_seed_u64(uint32_t* mt, uint64_t seed) {
    // random.Random(int): abs(seed) split into little-endian 32-bit words, at least one
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const int klen = (seed >> 32) ? 2 : 1;
    mt[0] = 19650218u;
    for (int i = 1; i < kN; i++) mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
    int i = 1, j = 0;
    for (int k = kN > klen ? kN : klen; k; k--) {
        mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
        i++; j++;
        if (i >= kN) { mt[0] = mt[kN - 1]; i = 1; }
        if (j >= klen) j = 0;
    }
    for (int k = kN - 1; k; k--) {
        mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
        i++;
        if (i >= kN) { mt[0] = mt[kN - 1]; i = 1; }
    }
    mt[0] = 0x80000000u;
    mt[kN] = kN;
}

__host__ __device__ inline uint32_t mt_next(uint32_t* mt) {
    uint32_t idx = mt[kN];
    if (idx >= (uint32_t)kN) {   // regenerate the block
        int kk = 0;
        uint32_t y;
        for (; kk < kN - kM; kk++) {
            y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
            mt[kk] = mt[kk + kM] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        for (; kk < kN - 1; kk++) {
            y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
            mt[kk] = mt[kk + (kM - kN)] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        y = (mt[kN - 1] & 0x80000000u) | (mt[0] & 0x7fffffffu);
        mt[kN - 1] = mt[kM - 1] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        idx = 0;
    }
    uint32_t y = mt[idx];
    mt[kN] = idx + 1;
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    return y ^ (y >> 18);
}

// random.randrange(n) for 1 <= n < 2^31: k = n.bit_length(); r = getrandbits(k) until r < n
__host__ __device__ inline uint32_t mt_below(uint32_t* mt, uint32_t n) {
    int k = 0;
    for (uint32_t t = n; t; t >>= 1) k++;
    uint32_t r;
    do { r = mt_next(mt) >> (32 - k); } while (r >= n);
    return r;
}

// ---- tree accessors
struct Tree {
    bbk_mcts_tree t;
    __device__ __forceinline__ int64_t at(int64_t s, int node) const { return s * t.max_nodes + node; }
    __device__ __forceinline__ uint32_t* mt(int64_t s) const { return t.mt + s * (int64_t)(kN + 1); }
    __device__ __forceinline__ uint32_t* untried(int64_t s, int node) const {
        return t.untried + at(s, node) * t.mask_words;
    }
};

__device__ __forceinline__ void new_node(const Tree& T, int64_t s, int node, int parent, int action) {
    const int64_t q = T.at(s, node);
    T.t.visits[q] = 0;
    T.t.value_sum[q] = 0.0;
    T.t.parent[q] = parent;
    T.t.first_child[q] = -1;
    T.t.last_child[q] = -1;
    T.t.next_sibling[q] = -1;
    T.t.action[q] = action;
    if (parent >= 0) {   // append: children stay in creation order (agents.py:108)
        const int64_t pq = T.at(s, parent);
        const int last = T.t.last_child[pq];
        if (last < 0) T.t.first_child[pq] = node;
        else T.t.next_sibling[T.at(s, last)] = node;
        T.t.last_child[pq] = node;
    }
}

__global__ void seed_kernel(bbk_mcts_tree t, const uint64_t* keys) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= t.n_search) return;
    Tree T{t};
    mt_seed_u64(T.mt(s), keys[s]);
    new_node(T, s, 0, -1, -1);
    t.next_node[s] = 1;
    t.leaf[s] = 0;
}

// Untried actions of node[s] (flatnonzero of its mask, agents.py:55-57; empty when finished
// because finished masks are all-zero, core.py:205-208) and the role to move there.
__global__ void untried_kernel(bbk_mcts_tree t, const uint8_t* mask, const int32_t* cur, const int8_t* p2r,
                               const int32_t* node) {
    const int lane = lane_id();
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (s >= t.n_search) return;
    const int nd = node ? node[s] : 0;
    if (nd < 0) return;
    Tree T{t};
    const int A = t.num_actions;
    const uint8_t* row = mask + s * (int64_t)A;
    uint32_t* u = T.untried(s, nd);
    int cnt = 0;
    for (int w = lane; w < t.mask_words; w += 32) {
        uint32_t bits = 0u;
        const int a0 = 32 * w;
        for (int k = 0; k < 32 && a0 + k < A; k++) bits |= (uint32_t)(row[a0 + k] & 1u) << k;
        u[w] = bits;
        cnt += __popc(bits);
    }
    cnt = warp_sum(cnt);
    if (lane == 0) {
        const int64_t q = T.at(s, nd);
        t.untried_count[q] = cnt;
        t.role[q] = (uint8_t)p2r[2 * s + cur[s]];
    }
}

// i-th set bit of a node's untried set, removed from it (list.pop(i) on the sorted list)
__device__ __forceinline__ int pop_untried(uint32_t* u, int words, uint32_t i) {
    for (int w = 0; w < words; w++) {
        uint32_t bits = u[w];
        const uint32_t c = __popc(bits);
        if (i < c) {
            for (uint32_t r = 0; r < i; r++) bits &= bits - 1u;
            const int b = __ffs(bits) - 1;
            u[w] &= ~(1u << b);
            return 32 * w + b;
        }
        i -= c;
    }
    return -1;
}

// Selection + expansion of one simulation (agents.py:89-109). Outputs per search: the pool row
// of the state to expand from (src_row), the pool row of the new child (dst_row, -1 when the
// selected node is finished and nothing is expanded), the action, and the new node's id
// (new_node, -1 likewise). The pool row of node k of search s is s * max_nodes + k.
__global__ void select_kernel(bbk_mcts_tree t, double c, const double* logtab, int32_t* src_row, int32_t* dst_row,
                              int64_t* act, int32_t* new_id) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= t.n_search) return;
    Tree T{t};
    int node = 0;
    for (;;) {
        const int64_t q = T.at(s, node);
        if (t.untried_count[q] != 0 || t.first_child[q] < 0) break;
        // ucb: value_sum / visits + c * sqrt(log(visits_parent) / visits), first maximum wins
        const double log_n = logtab[t.visits[q]];
        int best = -1;
        double best_score = -INFINITY;
        for (int ch = t.first_child[q]; ch >= 0; ch = t.next_sibling[T.at(s, ch)]) {
            const int64_t cq = T.at(s, ch);
            const double nv = (double)t.visits[cq];
            const double score = __dadd_rn(__ddiv_rn(t.value_sum[cq], nv),
                                           __dmul_rn(c, __dsqrt_rn(__ddiv_rn(log_n, nv))));
            if (score > best_score) { best_score = score; best = ch; }
        }
        node = best;
    }
    const int64_t q = T.at(s, node);
    src_row[s] = (int32_t)q;
    const int cnt = t.untried_count[q];
    if (cnt > 0) {
        const uint32_t i = mt_below(T.mt(s), (uint32_t)cnt);
        const int a = pop_untried(T.untried(s, node), t.mask_words, i);
        t.untried_count[q] = cnt - 1;
        const int nd = t.next_node[s];
        t.next_node[s] = nd + 1;
        new_node(T, s, nd, node, a);
        dst_row[s] = (int32_t)T.at(s, nd);
        new_id[s] = nd;
        act[s] = a;
        t.leaf[s] = nd;
    } else {
        dst_row[s] = -1;
        new_id[s] = -1;
        act[s] = 0;
        t.leaf[s] = node;
    }
}

// Rollout moves (agents.py:113-116): legal[randrange(len(legal))] for every unfinished search.
// Searches whose rollout is over keep stepping (the batched step auto-resets them) on their
// lowest legal action; nothing of theirs is read again and their Twister is left untouched.
__global__ void rollout_actions_kernel(bbk_mcts_tree t, const uint8_t* mask, const uint8_t* done, int64_t* act) {
    const int lane = lane_id();
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (s >= t.n_search) return;
    const int A = t.num_actions;
    const uint8_t* row = mask + s * (int64_t)A;
    // lane l holds the flags of actions [32 w + ... ) for words w = l, l + 32, ...
    int cnt = 0;
    for (int a = lane; a < A; a += 32) cnt += row[a] & 1;
    cnt = warp_sum(cnt);
    uint32_t d = 0;
    if (lane == 0 && cnt > 0 && !done[s]) d = mt_below(Tree{t}.mt(s), (uint32_t)cnt);
    d = __shfl_sync(BBK_FULL, d, 0);
    // the d-th set flag in action order: scan 32 actions per round
    int base = 0;
    int64_t out = 0;
    for (int a0 = 0; a0 < A; a0 += 32) {
        const int a = a0 + lane;
        const bool f = a < A && (row[a] & 1);
        const uint32_t m = __ballot_sync(BBK_FULL, f);
        const int c = __popc(m);
        if ((uint32_t)(base + c) > d) {
            uint32_t bits = m;
            for (uint32_t r = d - base; r > 0; r--) bits &= bits - 1u;
            out = a0 + __ffs(bits) - 1;
            break;
        }
        base += c;
    }
    if (lane == 0) act[s] = cnt > 0 ? out : 0;
}

// Record the role rewards of every search whose rollout just ended (agents.py:117,
// _role_rewards agents.py:126-131): ret[s, p2r[s, p]] = rewards[s, p]. Only searches with
// sel[s] == want are considered when sel is given.
__global__ void latch_kernel(const uint8_t* term, const uint8_t* trunc, const float* rewards, const int8_t* p2r,
                             const int32_t* sel, int want, int64_t n, uint8_t* done, float* ret,
                             unsigned long long* count) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool fresh = false;
    if (s < n && !done[s] && (term[s] | trunc[s]) && (!sel || ((sel[s] >= 0) == (want != 0)))) {
        fresh = true;
        done[s] = 1;
        ret[2 * s + p2r[2 * s]] = rewards[2 * s];
        ret[2 * s + p2r[2 * s + 1]] = rewards[2 * s + 1];
    }
    const unsigned m = __ballot_sync(BBK_FULL, fresh);
    if (lane_id() == 0 && m) atomicAdd(count, (unsigned long long)__popc(m));
}

// Backup (agents.py:117-122): every node of the path below the root gains a visit and
// scale * role_reward[mover] + offset, mover = the role to move at its parent.
__global__ void backup_kernel(bbk_mcts_tree t, const float* ret, double scale, double offset) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= t.n_search) return;
    Tree T{t};
    int node = t.leaf[s];
    while (node > 0) {
        const int64_t q = T.at(s, node);
        const int parent = t.parent[q];
        const double r = (double)ret[2 * s + t.role[T.at(s, parent)]];
        t.visits[q] += 1;
        t.value_sum[q] = __dadd_rn(t.value_sum[q], __dadd_rn(__dmul_rn(scale, r), offset));
        node = parent;
    }
    t.visits[T.at(s, 0)] += 1;
}

// Most visited root child, ties to the lowest action (agents.py:124-129).
__global__ void best_kernel(bbk_mcts_tree t, int64_t* out) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= t.n_search) return;
    Tree T{t};
    int best_action = -1, best_visits = -1;
    for (int ch = t.first_child[T.at(s, 0)]; ch >= 0; ch = t.next_sibling[T.at(s, ch)]) {
        const int64_t cq = T.at(s, ch);
        const int v = t.visits[cq], a = t.action[cq];
        if (v > best_visits || (v == best_visits && a < best_action)) { best_visits = v; best_action = a; }
    }
    out[s] = best_action;
}

// ---- row gather / scatter between batches (node pool <-> staging)
__global__ void copy_rows_kernel(bbk_row_copy_set set, const int32_t* src_idx, const int32_t* dst_idx, int64_t n) {
    const bbk_row_copy d = set.t[blockIdx.y];
    const int64_t units = d.row_bytes / d.unit;
    const int64_t total = n * units;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = g / units, u = g - i * units;
        const int64_t si = src_idx ? src_idx[i] : i, di = dst_idx ? dst_idx[i] : i;
        if (si < 0 || di < 0) continue;
        const char* sp = static_cast<const char*>(d.src) + si * d.row_bytes + u * d.unit;
        char* dp = static_cast<char*>(d.dst) + di * d.row_bytes + u * d.unit;
        switch (d.unit) {
            case 16: *reinterpret_cast<uint4*>(dp) = *reinterpret_cast<const uint4*>(sp); break;
            case 8: *reinterpret_cast<uint2*>(dp) = *reinterpret_cast<const uint2*>(sp); break;
            case 4: *reinterpret_cast<uint32_t*>(dp) = *reinterpret_cast<const uint32_t*>(sp); break;
            default: *dp = *sp; break;
        }
    }
}

inline unsigned blocks(int64_t threads, int per) { return (unsigned)((threads + per - 1) / per); }

}  // namespace mcts

extern "C" {

int bbk_mcts_seed(const bbk_mcts_tree* t, const uint64_t* key_states, void* stream) {
    if (t->n_search <= 0) return 0;
    mcts::seed_kernel<<<mcts::blocks(t->n_search, 128), 128, 0, (cudaStream_t)stream>>>(*t, key_states);
    return (int)cudaGetLastError();
}

int bbk_mcts_untried(const bbk_mcts_tree* t, const uint8_t* mask, const int32_t* current_player,
                     const int8_t* player_to_role, const int32_t* node, void* stream) {
    if (t->n_search <= 0) return 0;
    mcts::untried_kernel<<<mcts::blocks(32 * t->n_search, 128), 128, 0, (cudaStream_t)stream>>>(
        *t, mask, current_player, player_to_role, node);
    return (int)cudaGetLastError();
}

int bbk_mcts_select(const bbk_mcts_tree* t, double c, const double* log_table, int32_t* src_row, int32_t* dst_row,
                    int64_t* actions, int32_t* new_node, void* stream) {
    if (t->n_search <= 0) return 0;
    mcts::select_kernel<<<mcts::blocks(t->n_search, 64), 64, 0, (cudaStream_t)stream>>>(
        *t, c, log_table, src_row, dst_row, actions, new_node);
    return (int)cudaGetLastError();
}

int bbk_mcts_rollout_actions(const bbk_mcts_tree* t, const uint8_t* mask, const uint8_t* done, int64_t* actions,
                             void* stream) {
    if (t->n_search <= 0) return 0;
    mcts::rollout_actions_kernel<<<mcts::blocks(32 * t->n_search, 128), 128, 0, (cudaStream_t)stream>>>(
        *t, mask, done, actions);
    return (int)cudaGetLastError();
}

int bbk_mcts_latch(const uint8_t* terminated, const uint8_t* truncated, const float* rewards,
                   const int8_t* player_to_role, const int32_t* sel, int want, int64_t n, uint8_t* done,
                   float* role_returns, unsigned long long* count, void* stream) {
    if (n <= 0) return 0;
    mcts::latch_kernel<<<mcts::blocks(n, 128), 128, 0, (cudaStream_t)stream>>>(
        terminated, truncated, rewards, player_to_role, sel, want, n, done, role_returns, count);
    return (int)cudaGetLastError();
}

int bbk_mcts_backup(const bbk_mcts_tree* t, const float* role_returns, double scale, double offset, void* stream) {
    if (t->n_search <= 0) return 0;
    mcts::backup_kernel<<<mcts::blocks(t->n_search, 128), 128, 0, (cudaStream_t)stream>>>(*t, role_returns, scale,
                                                                                          offset);
    return (int)cudaGetLastError();
}

int bbk_mcts_best(const bbk_mcts_tree* t, int64_t* actions, void* stream) {
    if (t->n_search <= 0) return 0;
    mcts::best_kernel<<<mcts::blocks(t->n_search, 128), 128, 0, (cudaStream_t)stream>>>(*t, actions);
    return (int)cudaGetLastError();
}

int bbk_copy_rows(const bbk_row_copy_set* set, const int32_t* src_idx, const int32_t* dst_idx, int64_t n,
                  void* stream) {
    if (n <= 0 || set->count <= 0) return 0;
    if (set->count > BBK_ROW_COPY_MAX) return (int)cudaErrorInvalidValue;
    for (int k = 0; k < set->count; k++) {
        const bbk_row_copy& d = set->t[k];
        if (d.unit != 1 && d.unit != 4 && d.unit != 8 && d.unit != 16) return (int)cudaErrorInvalidValue;
        if (d.row_bytes % d.unit) return (int)cudaErrorInvalidValue;
    }
    int64_t most = 0;
    for (int k = 0; k < set->count; k++) {
        const int64_t u = n * (set->t[k].row_bytes / set->t[k].unit);
        most = u > most ? u : most;
    }
    int64_t gx = (most + 255) / 256;
    if (gx > 4096) gx = 4096;
    dim3 grid((unsigned)(gx < 1 ? 1 : gx), (unsigned)set->count);
    mcts::copy_rows_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(*set, src_idx, dst_idx, n);
    return (int)cudaGetLastError();
}

int bbk_mt19937_host(uint64_t seed, const uint32_t* below, int64_t n, uint32_t* out) {
    // host twin of the device Twister: out[i] = randrange(below[i]) (0 -> raw 32-bit word)
    static thread_local uint32_t mt[mcts::kN + 1];
    mcts::mt_seed_u64(mt, seed);
    for (int64_t i = 0; i < n; i++) out[i] = below[i] ? mcts::mt_below(mt, below[i]) : mcts::mt_next(mt);
    return 0;
}

}  // extern "C"

// checked builds: this translation unit's failed-check word (common.cuh BBK_CHECK)
BBK_CHECK_READER(bbk_tu_fail_mcts)
