// microbench.cu -- roofline denominators the walker needs that
// MEASURED_PEAKS.json does not carry (SURVEY §8(d) "Microbenchmarks the build
// must add"): random 32-B gathers (L2- and HBM-resident), L2 streaming reads,
// fp64 FMA rate, f64 RED throughput.  Separate library (libtetmicro.so);
// not part of the operator path.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// Each thread issues `iters` independent 32-B gathers (one 256-bit load at a
// pseudo-random record index) and folds them into a checksum.  The record
// count is a power of two: the index is a 32-bit xorshift state masked to
// the buffer (7 integer ops per load, no 64-bit modulo), so the loop is
// bound by the memory system, not by index arithmetic.
__global__ void gather32_kernel(const int4* __restrict__ buf, uint32_t mask, int iters,
                                unsigned* __restrict__ sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t s = hash32(tid) | 1u;
    unsigned acc = 0;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        s ^= s << 13; s ^= s >> 17; s ^= s << 5;
        const uint32_t r = s & mask;
        int a0, a1, a2, a3, a4, a5, a6, a7;
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3), "=r"(a4), "=r"(a5), "=r"(a6),
                       "=r"(a7)
                     : "l"(buf + 2 * (size_t)r));
        acc += a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// The same with 16-B records (the walker's vertex gather).
__global__ void gather16_kernel(const int4* __restrict__ buf, uint32_t mask, int iters,
                                unsigned* __restrict__ sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t s = hash32(tid) | 1u;
    unsigned acc = 0;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        s ^= s << 13; s ^= s >> 17; s ^= s << 5;
        const int4 v = __ldg(buf + (s & mask));
        acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// Coalesced reads; in pass r block b reads the slice of block (b + 37 r) so no
// SM re-reads its own slice from L1 (the buffer is L2-resident, not L1).
__global__ void stream_kernel(const int4* __restrict__ buf, uint64_t n16, int reps,
                              unsigned* __restrict__ sink) {
    unsigned acc = 0;
    const uint64_t per = (n16 + gridDim.x - 1) / gridDim.x;
    for (int r = 0; r < reps; ++r) {
        const uint64_t blk = (blockIdx.x + 37ull * r) % gridDim.x;
        const uint64_t lo = blk * per, hi = lo + per < n16 ? lo + per : n16;
        for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            int4 v;
            asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + i));
            acc += v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void dfma_kernel(double* __restrict__ out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double m = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 0.123) out[0] = s;
}

__global__ void red_kernel(double* __restrict__ acc, uint64_t n, int iters) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) atomicAdd(acc + hash32(tid * 31u + i * 0x85ebca6bu) % n, 1.0);
}

// REDs with the walker's pattern: per iteration a warp picks one random base
// and lane l adds to base + (l >> 2) (8 addresses per warp instruction, 4
// lanes on each -- coherent rays crossing the same tets).
template <typename T>
__global__ void red_coherent_kernel(T* __restrict__ acc, uint64_t n, int iters) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t warp = tid >> 5, lane = tid & 31;
    for (int i = 0; i < iters; ++i) {
        const uint64_t base = hash32(warp * 31u + i * 0x85ebca6bu) % (n - 8);
        atomicAdd(acc + base + (lane >> 2), (T)1);
    }
}

__global__ void red32_kernel(float* __restrict__ acc, uint64_t n, int iters) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) atomicAdd(acc + hash32(tid * 31u + i * 0x85ebca6bu) % n, 1.0f);
}

}  // namespace

extern "C" {

// Returns the kernel time in ms (CUDA events), or a negative value on error.
// kind: 0 gather32 (power-of-two buffer of 32-B records), 1 stream, 2 dfma,
// 3 red.f64, 4 red.f32, 5 red.f64 coherent (8 addresses x 4 lanes per warp),
// 6 red.f32 coherent, 7 gather16 (power-of-two buffer of 16-B records)
double tetmicro_run(int kind, uint64_t buffer_bytes, int iters, int blocks, int threads) {
    void* buf = nullptr;
    unsigned* sink = nullptr;
    if (cudaMalloc(&buf, buffer_bytes ? buffer_bytes : 256) != cudaSuccess) return -1;
    cudaMalloc((void**)&sink, 16);
    cudaMemset(buf, 1, buffer_bytes ? buffer_bytes : 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {   // rep 0 = warm-up
        cudaEventRecord(a);
        if (kind == 0)   // buffer_bytes must be a power of two
            gather32_kernel<<<blocks, threads>>>((const int4*)buf, (uint32_t)(buffer_bytes / 32 - 1),
                                                 iters, sink);
        else if (kind == 7)
            gather16_kernel<<<blocks, threads>>>((const int4*)buf, (uint32_t)(buffer_bytes / 16 - 1),
                                                 iters, sink);
        else if (kind == 1)
            stream_kernel<<<blocks, threads>>>((const int4*)buf, buffer_bytes / 16, iters, sink);
        else if (kind == 2)
            dfma_kernel<<<blocks, threads>>>((double*)buf, iters);
        else if (kind == 3)
            red_kernel<<<blocks, threads>>>((double*)buf, buffer_bytes / 8, iters);
        else if (kind == 4)
            red32_kernel<<<blocks, threads>>>((float*)buf, buffer_bytes / 4, iters);
        else if (kind == 5)
            red_coherent_kernel<double><<<blocks, threads>>>((double*)buf, buffer_bytes / 8, iters);
        else if (kind == 6)
            red_coherent_kernel<float><<<blocks, threads>>>((float*)buf, buffer_bytes / 4, iters);
        cudaEventRecord(b);
    }
    cudaEventSynchronize(b);
    float ms = -1;
    if (cudaGetLastError() == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    cudaFree(sink);
    return ms;
}

}  // extern "C"
