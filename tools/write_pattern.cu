// Write-pattern microbenchmark: how fast can HBM absorb the observation stream when each warp
// writes whole per-board records (the step kernels' pattern) vs a flat grid-stride fill?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wp tools/write_pattern.cu && /tmp/wp
#include <cstdio>
#include <cstdint>
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
    timeit("flat grid-stride (148x8 x 256)", [&] { flat<<<148 * 8, 256>>>((float4*)out, (int64_t)(bytes / 16)); });
    timeit("flat 256-bit stores", [&] { flat256<<<148 * 8, 256>>>(out, (int64_t)(bytes / 32)); });
    timeit("flat unroll 4", [&] { flat_unroll4<<<148 * 8, 256>>>((float4*)out, (int64_t)(bytes / 16)); });
    for (int ctas : {4, 6, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "warp per record 256-bit, %d x 4 / SM", ctas);
        timeit(nm, [&] { per_record256<<<148 * ctas, 128>>>(out, n, rec); });
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
