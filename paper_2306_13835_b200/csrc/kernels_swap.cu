// sm_100a swap-path kernels: zero-copy shard copy and the order-independent checksum.
//
// Zero-copy (north star: "a hand-written sm_100a zero-copy kernel that reads mapped host
// memory with 128-bit coalesced loads and writes the device layout"): each thread keeps
// kUnroll independent 16-B loads in flight (PCIe needs ~64 GB/s x ~2 us ~ 128 KB
// outstanding per GPU), reads with ld.global.nc.L1::no_allocate (streamed once; no L1
// pollution) and writes with st.global.L1::no_allocate. The same kernel serves D2H when dst
// is a mapped host pointer (posted PCIe writes). Grid is small by design (zc_ctas) so a
// concurrent forward of another model keeps the remaining SMs (loads overlap
// unrelated batches).
//
// Checksum (C4): H = sum_j splitmix64(word_j ^ j*0x9E3779B97F4A7C15) mod 2^64,
// HBM-bound: 128-bit loads, per-thread u64 sum, warp shuffle + one atomicAdd per warp.
#include "internal.h"

namespace mpsw {

namespace {

__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_na_v4(uint4* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

constexpr int kZcThreads = 512;
constexpr int kUnroll = 8;

__global__ void __launch_bounds__(kZcThreads) zero_copy_kernel(uint4* __restrict__ dst,
                                                               const uint4* __restrict__ src,
                                                               uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * kZcThreads;
    uint64_t i = (uint64_t)blockIdx.x * kZcThreads + threadIdx.x;
    // main loop: kUnroll loads in flight, then kUnroll stores
    for (; i + (kUnroll - 1) * stride < n16; i += kUnroll * stride) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ld_nc_v4(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) st_na_v4(dst + i + u * stride, v[u]);
    }
    for (; i < n16; i += stride) st_na_v4(dst + i, ld_nc_v4(src + i));
}

__device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

constexpr int kCkThreads = 256;

__global__ void __launch_bounds__(kCkThreads) checksum_kernel(const uint4* __restrict__ buf, uint64_t n16,
                                                              unsigned long long* __restrict__ out) {
    const uint64_t K = 0x9E3779B97F4A7C15ull;
    const uint64_t stride = (uint64_t)gridDim.x * kCkThreads;
    uint64_t h = 0;
    uint64_t i = (uint64_t)blockIdx.x * kCkThreads + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ld_nc_v4(buf + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t j = 2 * (i + u * stride);
            const uint64_t w0 = ((uint64_t)v[u].y << 32) | v[u].x;
            const uint64_t w1 = ((uint64_t)v[u].w << 32) | v[u].z;
            h += sm64(w0 ^ (j * K)) + sm64(w1 ^ ((j + 1) * K));
        }
    }
    for (; i < n16; i += stride) {
        const uint4 v = ld_nc_v4(buf + i);
        const uint64_t j = 2 * i;
        h += sm64((((uint64_t)v.y << 32) | v.x) ^ (j * K)) + sm64((((uint64_t)v.w << 32) | v.z) ^ ((j + 1) * K));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)h);
}

__global__ void checksum_tail_kernel(const uint64_t* __restrict__ buf, uint64_t w0, uint64_t nw,
                                     unsigned long long* __restrict__ out) {
    // words [w0, nw) when the buffer is not a multiple of 16 B (at most one word)
    const uint64_t K = 0x9E3779B97F4A7C15ull;
    uint64_t h = 0;
    for (uint64_t j = w0 + threadIdx.x; j < nw; j += blockDim.x) h += sm64(buf[j] ^ (j * K));
    atomicAdd(out, (unsigned long long)h);
}

}  // namespace

void launch_zero_copy(void* dst, const void* src, uint64_t bytes, int ctas, cudaStream_t s) {
    if (bytes == 0) return;
    if ((bytes & 15) || ((uintptr_t)dst & 15) || ((uintptr_t)src & 15))
        throw Error(MPSW_EINVAL, "zero-copy needs 16-B aligned pointers and sizes");
    const uint64_t n16 = bytes / 16;
    uint64_t need = (n16 + (uint64_t)kZcThreads * kUnroll - 1) / ((uint64_t)kZcThreads * kUnroll);
    int grid = (int)std::min<uint64_t>(need, (uint64_t)std::max(1, ctas));
    zero_copy_kernel<<<grid, kZcThreads, 0, s>>>((uint4*)dst, (const uint4*)src, n16);
    MPSW_CU(cudaGetLastError());
}

// Residency stamps (mpsw_config.debug_checks): a load writes its entry id, an offload the evicted
// marker, behind its copies on the copy stream; the forward checks the stamp first.
__global__ void stamp_kernel(unsigned long long* slot, unsigned long long value) { *slot = value; }

__global__ void check_stamp_kernel(const unsigned long long* slot, unsigned long long expect, unsigned int* err) {
    const unsigned long long v = *(volatile const unsigned long long*)slot;
    if (v != expect) *(volatile unsigned int*)err = 1u;   // mapped pinned host word: a plain store
}

void launch_stamp(unsigned long long* slot, unsigned long long value, cudaStream_t s) {
    stamp_kernel<<<1, 1, 0, s>>>(slot, value);
}

void launch_check_stamp(const unsigned long long* slot, unsigned long long expect, unsigned int* err, cudaStream_t s) {
    check_stamp_kernel<<<1, 1, 0, s>>>(slot, expect, err);
}

void launch_checksum(const void* buf, uint64_t bytes, unsigned long long* d_out, cudaStream_t s) {
    if (bytes & 7) throw Error(MPSW_EINVAL, "checksum needs a multiple of 8 bytes");
    const uint64_t n16 = bytes / 16;
    if (n16) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        uint64_t need = (n16 + kCkThreads - 1) / kCkThreads;
        int grid = (int)std::min<uint64_t>(need, (uint64_t)sms * 8);
        checksum_kernel<<<grid, kCkThreads, 0, s>>>((const uint4*)buf, n16, d_out);
        MPSW_CU(cudaGetLastError());
    }
    if (bytes / 8 > 2 * n16) {
        checksum_tail_kernel<<<1, 32, 0, s>>>((const uint64_t*)buf, 2 * n16, bytes / 8, d_out);
        MPSW_CU(cudaGetLastError());
    }
}

}  // namespace mpsw
