// Write-pattern microbenchmark: how fast can HBM absorb the observation stream when each warp
// writes whole per-board records (the step kernels' pattern) vs a flat grid-stride fill?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wp tools/write_pattern.cu && /tmp/wp
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

// one warp per record (records of `rec` floats, flat stream, 16-B chunks of the aligned interior)
__global__ void per_record(float* out, int64_t n, int rec, int pad_iters) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); b < n; b += nw) {
        const int64_t F0 = b * rec;
        const int head = (int)((4 - (F0 & 3)) & 3);
        const int nchunk = (rec - head) >> 2;
        float4* o4 = reinterpret_cast<float4*>(out + F0 + head);
        const float v = (float)(b & 1);
        for (int j = lane; j < nchunk; j += 32) o4[j] = make_float4(v, v, v, v);
        // simulated per-board logic (dependent ALU chain), so warps desynchronise as in a step
        uint32_t x = (uint32_t)b;
        for (int i = 0; i < pad_iters; i++) x = x * 1664525u + 1013904223u;
        if (x == 0xFFFFFFFFu) out[0] = 1.0f;
    }
}

// the same records, but the warps of a CTA write one record together (chunk j by lane j of warp w)
__global__ void per_cta_record(float* out, int64_t n, int rec) {
    const int t = threadIdx.x;
    for (int64_t b = blockIdx.x; b < n; b += gridDim.x) {
        const int64_t F0 = b * rec;
        const int head = (int)((4 - (F0 & 3)) & 3);
        const int nchunk = (rec - head) >> 2;
        float4* o4 = reinterpret_cast<float4*>(out + F0 + head);
        const float v = (float)(b & 1);
        for (int j = t; j < nchunk; j += blockDim.x) o4[j] = make_float4(v, v, v, v);
    }
}

__global__ void flat(float4* out, int64_t n4) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}

// 32-byte stores (st.global.v8.f32, sm_100)
__device__ __forceinline__ void st256(float* p, float v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(v) : "memory");
}
__global__ void flat256(float* out, int64_t n8) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x)
        st256(out + 8 * i, 1.0f);
}
__global__ void flat_unroll4(float4* out, int64_t n4) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 3 * stride < n4; i += 4 * stride) {
#pragma unroll
        for (int u = 0; u < 4; u++) out[i + u * stride] = make_float4(1.f, 1.f, 1.f, 1.f);
    }
}
__device__ __forceinline__ void st256cs(float* p, float v) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st256na(float* p, float v) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st256ef(float* p, float v) {
    asm volatile("st.global.L2::evict_first.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(v) : "memory");
}
template <int MODE>
__global__ void per_record256m(float* out, int64_t n, int rec) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); b < n; b += nw) {
        const int64_t F0 = b * rec;
        const int head = (int)((8 - (F0 & 7)) & 7);
        const int nchunk = (rec - head) >> 3;
        float* o = out + F0 + head;
        const float v = (float)(b & 1);
        for (int j = lane; j < nchunk; j += 32) {
            if (MODE == 0) st256cs(o + 8 * j, v);
            else if (MODE == 1) st256na(o + 8 * j, v);
            else st256ef(o + 8 * j, v);
        }
    }
}
template <int MODE>
__global__ void flat256m(float* out, int64_t n8) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
        if (MODE == 0) st256cs(out + 8 * i, 1.0f);
        else if (MODE == 1) st256na(out + 8 * i, 1.0f);
        else st256ef(out + 8 * i, 1.0f);
    }
}
// per-record with 32-byte stores over the 32-B aligned interior
__global__ void per_record256(float* out, int64_t n, int rec) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); b < n; b += nw) {
        const int64_t F0 = b * rec;
        const int head = (int)((8 - (F0 & 7)) & 7);
        const int nchunk = (rec - head) >> 3;
        float* o = out + F0 + head;
        const float v = (float)(b & 1);
        for (int j = lane; j < nchunk; j += 32) st256(o + 8 * j, v);
    }
}

__device__ __forceinline__ void write_rec256(float* out, int64_t b, int rec, int lane) {
    const int64_t F0 = b * rec;
    const int head = (int)((8 - (F0 & 7)) & 7);
    const int nchunk = (rec - head) >> 3;
    float* o = out + F0 + head;
    const float v = (float)(b & 1);
    for (int j = lane; j < nchunk; j += 32) st256(o + 8 * j, v);
}
// (a) persistent, boards taken from a global counter in order (dynamic scheduling)
__global__ void rec_dynamic(float* out, int64_t n, int rec, unsigned long long* ctr) {
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(ctr, 1ull);
        b = __shfl_sync(0xffffffffu, b, 0);
        if ((int64_t)b >= n) break;
        write_rec256(out, (int64_t)b, rec, lane);
    }
}
// (b) persistent, each warp a contiguous range of boards
__global__ void rec_ranges(float* out, int64_t n, int rec) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t per = (n + nw - 1) / nw;
    for (int64_t b = w * per; b < n && b < (w + 1) * per; b++) write_rec256(out, b, rec, lane);
}
// (c) non-persistent, K consecutive boards per warp
template <int K>
__global__ void rec_nonpersist_k(float* out, int64_t n, int rec) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    for (int k = 0; k < K; k++) {
        const int64_t b = w * K + k;
        if (b < n) write_rec256(out, b, rec, lane);
    }
}
// (d) non-persistent, K boards per warp strided by the number of warps in the grid (interleaved)
template <int K>
__global__ void rec_nonpersist_strided(float* out, int64_t n, int rec) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    for (int k = 0; k < K; k++) {
        const int64_t b = w + k * nw;
        if (b < n) write_rec256(out, b, rec, lane);
    }
}

// (e) bulk (TMA-engine) stores: each warp fills a CHUNK-byte shared-memory buffer (double
// buffered) and one lane hands it to cp.async.bulk.global.shared::cta; K boards per warp strided
// by the grid's warp count. The record's unaligned head/tail floats go out as plain stores.
template <int CHUNK, int K>
__global__ void rec_bulk(float* out, int64_t n, int rec) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float* buf0 = reinterpret_cast<float*>(sm + wid * 2 * CHUNK);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + wid;
    int par = 0;
    for (int k = 0; k < K; k++) {
        const int64_t b = w + k * nw;
        if (b >= n) break;
        const int64_t F0 = b * rec;
        const int head = (int)((4 - (F0 & 3)) & 3);
        const float v = (float)(b & 1);
        const int body = ((rec - head) >> 2) << 2;
        const int tail = rec - head - body;
        if (lane < head) out[F0 + lane] = v;
        if (lane < tail) out[F0 + head + body + lane] = v;
        float* g = out + F0 + head;
        for (int off = 0; off < body; off += CHUNK / 4) {
            const int cnt = min(CHUNK / 4, body - off);
            float* buf = buf0 + par * (CHUNK / 4);
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            for (int j = lane * 4; j < cnt; j += 128) *reinterpret_cast<float4*>(buf + j) = make_float4(v, v, v, v);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             :: "l"(g + off), "r"((unsigned)__cvta_generic_to_shared(buf)), "r"(cnt * 4) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            par ^= 1;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int64_t n = 131072;
    const int rec = 19 * 19 * 17;
    float* out;
    const size_t bytes = (size_t)n * rec * 4;
    cudaMalloc(&out, bytes + 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; i++) launch();
        cudaEventRecord(a);
        const int K = 20;
        for (int i = 0; i < K; i++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= K;
        printf("%-40s %.3f ms  %.0f GB/s\n", name, ms, bytes / (ms * 1e6));
    };
    if (getenv("WP_BULK")) {
        timeit("per record 256, 1/warp (n/4 CTAs)", [&] { per_record256<<<(unsigned)(n / 4), 128>>>(out, n, rec); });
        timeit("per record 256, 3 strided/warp", [&] { rec_nonpersist_strided<3><<<(unsigned)((n + 11) / 12), 128>>>(out, n, rec); });
        cudaFuncSetAttribute(rec_bulk<4096, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        cudaFuncSetAttribute(rec_bulk<4096, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        cudaFuncSetAttribute(rec_bulk<8192, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        timeit("bulk 2K chunks, 1/warp", [&] { rec_bulk<2048, 1><<<(unsigned)(n / 4), 128, 4 * 2 * 2048>>>(out, n, rec); });
        timeit("bulk 2K chunks, 3 strided/warp", [&] { rec_bulk<2048, 3><<<(unsigned)((n + 11) / 12), 128, 4 * 2 * 2048>>>(out, n, rec); });
        timeit("bulk 4K chunks, 1/warp", [&] { rec_bulk<4096, 1><<<(unsigned)(n / 4), 128, 4 * 2 * 4096>>>(out, n, rec); });
        timeit("bulk 4K chunks, 3 strided/warp", [&] { rec_bulk<4096, 3><<<(unsigned)((n + 11) / 12), 128, 4 * 2 * 4096>>>(out, n, rec); });
        timeit("bulk 8K chunks, 3 strided/warp", [&] { rec_bulk<8192, 3><<<(unsigned)((n + 11) / 12), 128, 4 * 2 * 8192>>>(out, n, rec); });
        timeit("bulk 1K chunks, 3 strided/warp", [&] { rec_bulk<1024, 3><<<(unsigned)((n + 11) / 12), 128, 4 * 2 * 1024>>>(out, n, rec); });
        timeit("flat 256 (again)", [&] { flat256<<<148 * 8, 256>>>(out, (int64_t)(bytes / 32)); });
        cudaError_t e = cudaDeviceSynchronize();
        printf("%s\n", cudaGetErrorString(e));
        return 0;
    }
    timeit("flat grid-stride (148x8 x 256)", [&] { flat<<<148 * 8, 256>>>((float4*)out, (int64_t)(bytes / 16)); });
    timeit("flat 256-bit stores", [&] { flat256<<<148 * 8, 256>>>(out, (int64_t)(bytes / 32)); });
    timeit("flat unroll 4", [&] { flat_unroll4<<<148 * 8, 256>>>((float4*)out, (int64_t)(bytes / 16)); });
    for (int ctas : {4, 6, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "warp per record 256-bit, %d x 4 / SM", ctas);
        timeit(nm, [&] { per_record256<<<148 * ctas, 128>>>(out, n, rec); });
    }
    unsigned long long* ctr;
    cudaMalloc(&ctr, 8);
    timeit("per record 256, persistent dynamic counter 6x4", [&] { cudaMemsetAsync(ctr, 0, 8); rec_dynamic<<<148 * 6, 128>>>(out, n, rec, ctr); });
    timeit("per record 256, persistent contiguous ranges 6x4", [&] { rec_ranges<<<148 * 6, 128>>>(out, n, rec); });
    timeit("per record 256, non-persistent 4 consecutive/warp", [&] { rec_nonpersist_k<4><<<(unsigned)(n / 16), 128>>>(out, n, rec); });
    timeit("per record 256, non-persistent 16 consecutive/warp", [&] { rec_nonpersist_k<16><<<(unsigned)(n / 64), 128>>>(out, n, rec); });
    timeit("per record 256, non-persistent 4 strided/warp", [&] { rec_nonpersist_strided<4><<<(unsigned)(n / 16), 128>>>(out, n, rec); });
    timeit("per record 256, NON-persistent (n/4 CTAs)", [&] { per_record256<<<(unsigned)(n / 4), 128>>>(out, n, rec); });
    timeit("per record 128, NON-persistent (n/4 CTAs)", [&] { per_record<<<(unsigned)(n / 4), 128>>>(out, n, rec, 0); });
    timeit("flat 256, NON-persistent (1 chunk/thread)", [&] { flat256<<<(unsigned)(bytes / 32 / 256), 256>>>(out, (int64_t)(bytes / 32)); });
    timeit("flat 128, NON-persistent (1 chunk/thread)", [&] { flat<<<(unsigned)(bytes / 16 / 256), 256>>>((float4*)out, (int64_t)(bytes / 16)); });
    timeit("flat 256 .cs", [&] { flat256m<0><<<148 * 8, 256>>>(out, (int64_t)(bytes / 32)); });
    timeit("flat 256 L1::no_allocate", [&] { flat256m<1><<<148 * 8, 256>>>(out, (int64_t)(bytes / 32)); });
    timeit("flat 256 L2::evict_first", [&] { flat256m<2><<<148 * 8, 256>>>(out, (int64_t)(bytes / 32)); });
    timeit("per record 256 .cs, 6x4", [&] { per_record256m<0><<<148 * 6, 128>>>(out, n, rec); });
    timeit("per record 256 no_allocate, 6x4", [&] { per_record256m<1><<<148 * 6, 128>>>(out, n, rec); });
    timeit("per record 256 evict_first, 6x4", [&] { per_record256m<2><<<148 * 6, 128>>>(out, n, rec); });
    timeit("flat 256 (again)", [&] { flat256<<<148 * 8, 256>>>(out, (int64_t)(bytes / 32)); });
    for (int t : {128, 512, 1024}) {
        char nm[64];
        snprintf(nm, sizeof nm, "flat 256, %d threads x 148x(2048/%d)", t, t);
        timeit(nm, [&] { flat256<<<148 * (2048 / t), t>>>(out, (int64_t)(bytes / 32)); });
    }
    for (int ctas : {4, 6, 8, 16}) {
        char nm[64];
        snprintf(nm, sizeof nm, "warp per record, %d x 4 warps / SM", ctas);
        timeit(nm, [&] { per_record<<<148 * ctas, 128>>>(out, n, rec, 0); });
    }
    for (int pad : {200, 1000}) {
        char nm[64];
        snprintf(nm, sizeof nm, "warp per record + %d ALU, 6x4 / SM", pad);
        timeit(nm, [&] { per_record<<<148 * 6, 128>>>(out, n, rec, pad); });
    }
    for (int ctas : {4, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "CTA (4 warps) per record, %d / SM", ctas);
        timeit(nm, [&] { per_cta_record<<<148 * ctas, 128>>>(out, n, rec); });
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
