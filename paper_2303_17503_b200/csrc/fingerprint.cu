// Device-side state fingerprints: the reference's
// core.state_fingerprint (pkg/src/boardbatch/core.py:417-434) for every slot
// of a device batch, without a host round trip per slot.
//
// Per slot the digest is blake2b (16-byte digest, RFC 7693) over
//   game_id | <i i B B>(current_player, step_count, terminated, truncated)
//   | player_to_role (2 x int8) | rewards (2 x float32, by player)
//   | packbits(legal_action_mask) (numpy default, most significant bit first)
//   | Core.encode()
// where encode is the game's byte encoding (go.py:103-111, backgammon.py:113-119,
// and the chess / shogi encodings of DESIGN.md §3.3-3.4). One thread per slot
// assembles the message into a scratch row, then one thread per slot hashes it.
// batch_fingerprint (core.py:437-441) is blake2b over the per-slot digests in
// slot order, done by the host over n x 16 bytes.
#include "common.cuh"
#include "small.cuh"
#include "../../include/bbk.h"

namespace fp {
using namespace bbk;

// ---------------------------------------------------------------- blake2b
__device__ __constant__ uint8_t D_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
[[maybe_unused]] static const uint8_t H_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__host__ __device__ __forceinline__ uint64_t iv(int i) {
    switch (i) {
        case 0: return 0x6a09e667f3bcc908ULL;
        case 1: return 0xbb67ae8584caa73bULL;
        case 2: return 0x3c6ef372fe94f82bULL;
        case 3: return 0xa54ff53a5f1d36f1ULL;
        case 4: return 0x510e527fade682d1ULL;
        case 5: return 0x9b05688c2b3e6c1fULL;
        case 6: return 0x1f83d9abfb41bd6bULL;
        default: return 0x5be0cd19137e2179ULL;
    }
}
__host__ __device__ __forceinline__ uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

#define BB_G(a, b, c, d, x, y)               \
    do {                                     \
        v[a] = v[a] + v[b] + (x);            \
        v[d] = rotr(v[d] ^ v[a], 32);        \
        v[c] = v[c] + v[d];                  \
        v[b] = rotr(v[b] ^ v[c], 24);        \
        v[a] = v[a] + v[b] + (y);            \
        v[d] = rotr(v[d] ^ v[a], 16);        \
        v[c] = v[c] + v[d];                  \
        v[b] = rotr(v[b] ^ v[c], 63);        \
    } while (0)

// Compress one 128-byte block (RFC 7693 §3.2); t = bytes hashed so far incl. this block.
__host__ __device__ void compress(uint64_t h[8], const uint8_t* blk, uint64_t t, bool last) {
    uint64_t m[16], v[16];
    for (int i = 0; i < 16; i++) {
        uint64_t w = 0;
        for (int k = 7; k >= 0; k--) w = (w << 8) | blk[8 * i + k];
        m[i] = w;
    }
    for (int i = 0; i < 8; i++) { v[i] = h[i]; v[i + 8] = iv(i); }
    v[12] ^= t;
    if (last) v[14] = ~v[14];
    for (int r = 0; r < 12; r++) {
#ifdef __CUDA_ARCH__
        const uint8_t* s = D_SIGMA[r];
#else
        const uint8_t* s = H_SIGMA[r];
#endif
        BB_G(0, 4, 8, 12, m[s[0]], m[s[1]]);
        BB_G(1, 5, 9, 13, m[s[2]], m[s[3]]);
        BB_G(2, 6, 10, 14, m[s[4]], m[s[5]]);
        BB_G(3, 7, 11, 15, m[s[6]], m[s[7]]);
        BB_G(0, 5, 10, 15, m[s[8]], m[s[9]]);
        BB_G(1, 6, 11, 12, m[s[10]], m[s[11]]);
        BB_G(2, 7, 8, 13, m[s[12]], m[s[13]]);
        BB_G(3, 4, 9, 14, m[s[14]], m[s[15]]);
    }
    for (int i = 0; i < 8; i++) h[i] ^= v[i] ^ v[i + 8];
}

// blake2b with a 16-byte digest, no key.
__host__ __device__ void blake2b16(const uint8_t* msg, int64_t len, uint8_t out[16]) {
    uint64_t h[8];
    for (int i = 0; i < 8; i++) h[i] = iv(i);
    h[0] ^= 0x01010000ULL ^ 16ULL;
    int64_t off = 0;
    while (len - off > 128) {
        compress(h, msg + off, (uint64_t)(off + 128), false);
        off += 128;
    }
    uint8_t last[128];
    const int rem = (int)(len - off);
    for (int i = 0; i < 128; i++) last[i] = i < rem ? msg[off + i] : (uint8_t)0;
    compress(h, last, (uint64_t)len, true);
    for (int i = 0; i < 16; i++) out[i] = (uint8_t)(h[i >> 3] >> (8 * (i & 7)));
}

// ---------------------------------------------------------------- message prefix
struct Writer {
    uint8_t* p;
    int n;
    __device__ __forceinline__ void u8(uint32_t v) { p[n++] = (uint8_t)v; }
    __device__ __forceinline__ void u32(uint32_t v) { for (int k = 0; k < 4; k++) u8(v >> (8 * k)); }
    __device__ __forceinline__ void u64(uint64_t v) { for (int k = 0; k < 8; k++) u8((uint32_t)(v >> (8 * k))); }
    __device__ __forceinline__ void str(const char* s) { while (*s) u8((uint8_t)*s++); }
};

// game id, scalar fields, rewards and the MSB-first packed legal mask (core.py:421-426)
__device__ void write_prefix(Writer& w, const char* gid, const bbk_cols& c, int64_t b, int A, int P = 2) {
    w.str(gid);
    w.u32((uint32_t)c.current_player[b]);
    w.u32((uint32_t)c.step_count[b]);
    w.u8(c.terminated[b] ? 1u : 0u);
    w.u8(c.truncated[b] ? 1u : 0u);
    for (int q = 0; q < P; q++) w.u8((uint8_t)c.player_to_role[P * b + q]);
    for (int q = 0; q < P; q++) w.u32(__float_as_uint(c.rewards[P * b + q]));
    const uint8_t* m = c.legal_action_mask + b * (int64_t)A;
    for (int j = 0; j < (A + 7) / 8; j++) {
        uint32_t byte = 0;
        for (int k = 0; k < 8; k++) {
            const int a = 8 * j + k;
            byte |= (a < A && m[a]) ? (0x80u >> k) : 0u;
        }
        w.u8(byte);
    }
}

// ---------------------------------------------------------------- per-game messages
__global__ void go_msg_kernel(int N, bbk_cols c, bbk_go_state s, int64_t n, uint8_t* msgs, int64_t stride,
                              int32_t* lens) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const int C = N * N, PS = (C + 7) & ~7;
    char gid[12] = {'g', 'o', '_', 0};
    int q = 3;
    if (N >= 10) gid[q++] = (char)('0' + N / 10);
    gid[q++] = (char)('0' + N % 10);
    gid[q++] = 'x';
    if (N >= 10) gid[q++] = (char)('0' + N / 10);
    gid[q++] = (char)('0' + N % 10);
    gid[q] = 0;
    Writer w{msgs + b * stride, 0};
    write_prefix(w, gid, c, b, C + 1);
    // Core.encode (go.py:103-111): board, role, pass count, hash, hist_xor, hist_len (u16),
    // then boards_hist newest first (min(step + 1, 8) boards)
    const uint16_t* pat = s.pat + b * (int64_t)PS;
    for (int i = 0; i < C; i++) w.u8((pat[i] & 1u) + 2u * ((pat[i] >> 1) & 1u));
    w.u8(s.role_to_move[b]);
    w.u8(s.pass_count[b]);
    w.u64(s.hash[b]);
    w.u64(s.hist_xor[b]);
    const uint32_t hl = (uint32_t)s.hist_len[b];
    w.u8(hl & 0xFF);
    w.u8((hl >> 8) & 0xFF);
    const int step = c.step_count[b];
    const int nbh = step + 1 < 8 ? step + 1 : 8;
    for (int t = 0; t < nbh; t++)
        for (int i = 0; i < C; i++) w.u8(((pat[i] >> (2 * t)) & 1u) + 2u * ((pat[i] >> (2 * t + 1)) & 1u));
    lens[b] = w.n;
}

__global__ void bg_msg_kernel(bbk_cols c, bbk_bg_state s, int64_t n, uint8_t* msgs, int64_t stride, int32_t* lens) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    Writer w{msgs + b * stride, 0};
    write_prefix(w, "backgammon", c, b, 156);
    // Core.encode (backgammon.py:113-119): points + 16, bar, off, role, dice, remaining (zero padded)
    for (int i = 0; i < 24; i++) w.u8((uint8_t)(s.points[b * 24 + i] + 16));
    const uint8_t* m = s.misc + b * 12;
    for (int i = 0; i < 7; i++) w.u8(m[i]);
    const int nrem = m[11];
    for (int i = 0; i < 4; i++) w.u8(i < nrem ? m[7 + i] : 0u);
    lens[b] = w.n;
}

__global__ void chess_msg_kernel(bbk_cols c, bbk_chess_state s, int64_t n, uint8_t* msgs, int64_t stride,
                                 int32_t* lens) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    Writer w{msgs + b * stride, 0};
    write_prefix(w, "chess", c, b, 4672);
    // board[64] + stm, castling, ep, half-move clock, repetition
    for (int i = 0; i < 64; i++) w.u8(s.board[b * 64 + i]);
    for (int i = 0; i < 5; i++) w.u8(s.misc[b * 8 + i]);
    lens[b] = w.n;
}

__global__ void shogi_msg_kernel(bbk_cols c, bbk_shogi_state s, int64_t n, uint8_t* msgs, int64_t stride,
                                 int32_t* lens) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    Writer w{msgs + b * stride, 0};
    write_prefix(w, "shogi", c, b, 2187);
    // board[81] + hands[14] + side to move + repetition count
    for (int i = 0; i < 81; i++) w.u8(s.board[b * 96 + i]);
    for (int i = 0; i < 16; i++) w.u8(s.misc[b * 16 + i]);
    lens[b] = w.n;
}

template <class G>
__global__ void small_msg_kernel(int game, bbk_cols c, const uint8_t* blob, int64_t n,
                                 uint8_t* msgs, int64_t stride, int32_t* lens) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const char* ids[7] = {"tic_tac_toe", "connect_four", "othello", "hex", "2048", "kuhn_poker", "leduc_holdem"};
    Writer w{msgs + b * stride, 0};
    write_prefix(w, ids[game], c, b, G::A, G::P);
    small::St s;
    for (int i = 0; i < small::kStateBytes; i++) s.b[i] = blob[b * small::kStateBytes + i];
    G::encode(s, w);   // the engine's Core.encode
    lens[b] = w.n;
}

__global__ void hash_kernel(const uint8_t* msgs, int64_t stride, const int32_t* lens, int64_t n, uint8_t* out) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    uint8_t d[16];
    blake2b16(msgs + b * stride, lens[b], d);
    for (int i = 0; i < 16; i++) out[b * 16 + i] = d[i];
}

template <typename K>
int run(K launch_msg, const uint8_t* msgs, int64_t stride, int32_t* lens, int64_t n, uint8_t* out, cudaStream_t st) {
    if (n <= 0) return 0;
    const unsigned grid = (unsigned)((n + 127) / 128);
    launch_msg(grid, st);
    hash_kernel<<<grid, 128, 0, st>>>(msgs, stride, lens, n, out);
    return (int)cudaGetLastError();
}

}  // namespace fp

extern "C" {

int bbk_fingerprint_stride(int game_code, int size) {
    // upper bound of the message length (prefix + encode), rounded to 16 bytes
    int A, enc;
    switch (game_code) {
        case 0: { const int C = size * size; A = C + 1; enc = C + 2 + 8 + 8 + 2 + 8 * C; break; }
        case 1: A = 156; enc = 24 + 7 + 4; break;
        case 2: A = 4672; enc = 64 + 5; break;
        case 3: A = 2187; enc = 81 + 16; break;
        default: A = 128; enc = 64; break;   // small engines (game_code 10 + bbk_small game)
    }
    return ((16 + 10 + 2 + 8 + (A + 7) / 8 + enc) + 15) & ~15;
}

int bbk_go_fingerprint(int size, const bbk_cols* c, const bbk_go_state* s, int64_t n, uint8_t* scratch,
                       int64_t stride, int32_t* lens, uint8_t* out, void* stream) {
    const bbk_cols cc = *c;
    const bbk_go_state ss = *s;
    return fp::run([&](unsigned g, cudaStream_t st) { fp::go_msg_kernel<<<g, 128, 0, st>>>(size, cc, ss, n, scratch, stride, lens); },
                   scratch, stride, lens, n, out, (cudaStream_t)stream);
}

int bbk_bg_fingerprint(const bbk_cols* c, const bbk_bg_state* s, int64_t n, uint8_t* scratch, int64_t stride,
                       int32_t* lens, uint8_t* out, void* stream) {
    const bbk_cols cc = *c;
    const bbk_bg_state ss = *s;
    return fp::run([&](unsigned g, cudaStream_t st) { fp::bg_msg_kernel<<<g, 128, 0, st>>>(cc, ss, n, scratch, stride, lens); },
                   scratch, stride, lens, n, out, (cudaStream_t)stream);
}

int bbk_chess_fingerprint(const bbk_cols* c, const bbk_chess_state* s, int64_t n, uint8_t* scratch, int64_t stride,
                          int32_t* lens, uint8_t* out, void* stream) {
    const bbk_cols cc = *c;
    const bbk_chess_state ss = *s;
    return fp::run([&](unsigned g, cudaStream_t st) { fp::chess_msg_kernel<<<g, 128, 0, st>>>(cc, ss, n, scratch, stride, lens); },
                   scratch, stride, lens, n, out, (cudaStream_t)stream);
}

int bbk_shogi_fingerprint(const bbk_cols* c, const bbk_shogi_state* s, int64_t n, uint8_t* scratch, int64_t stride,
                          int32_t* lens, uint8_t* out, void* stream) {
    const bbk_cols cc = *c;
    const bbk_shogi_state ss = *s;
    return fp::run([&](unsigned g, cudaStream_t st) { fp::shogi_msg_kernel<<<g, 128, 0, st>>>(cc, ss, n, scratch, stride, lens); },
                   scratch, stride, lens, n, out, (cudaStream_t)stream);
}

int bbk_small_fingerprint(int game, const bbk_cols* c, const uint8_t* blob, int64_t n, uint8_t* scratch,
                          int64_t stride, int32_t* lens, uint8_t* out, void* stream) {
    const bbk_cols cc = *c;
    auto go = [&](auto g) {
        using G = decltype(g);
        return fp::run([&](unsigned gr, cudaStream_t st) {
            fp::small_msg_kernel<G><<<gr, 128, 0, st>>>(game, cc, blob, n, scratch, stride, lens);
        }, scratch, stride, lens, n, out, (cudaStream_t)stream);
    };
    switch (game) {
        case 0: return go(small::TicTacToe{});
        case 1: return go(small::ConnectFour{});
        case 2: return go(small::Othello{});
        case 3: return go(small::Hex{});
        case 4: return go(small::Play2048{});
        case 5: return go(small::Kuhn{});
        case 6: return go(small::Leduc{});
        default: return (int)cudaErrorInvalidValue;
    }
}

// Host build of the same blake2b (CPU tests pin it against hashlib).
int bbk_blake2b16_host(const uint8_t* msg, int64_t len, uint8_t* out) {
    fp::blake2b16(msg, len, out);
    return 0;
}

}  // extern "C"

// checked builds: this translation unit's failed-check word (common.cuh BBK_CHECK)
BBK_CHECK_READER(bbk_tu_fail_fingerprint)
