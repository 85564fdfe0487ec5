// Pinned shard store ("the parameters are kept pinned in CPU memory") and the POSIX
// shared-memory segments of the multi-process control plane.
#include "runtime.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <fstream>

namespace mpsw {

int gpu_numa_node(int dev) {
    if (const char* f = getenv("MPSW_NUMA_NODE")) return atoi(f);   // forced (tests, remote-node runs)
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) return -1;
    for (char* c = bus; *c; ++c) *c = (char)tolower(*c);
    std::ifstream f(std::string("/sys/bus/pci/devices/") + bus + "/numa_node");
    int node = -1;
    if (f) f >> node;
    return node;
}

// MemAvailable of /proc/meminfo in bytes (0 if unknown): the register_model preflight.
uint64_t host_mem_available() {
    std::ifstream f("/proc/meminfo");
    std::string key;
    uint64_t kb = 0;
    while (f >> key >> kb) {
        if (key == "MemAvailable:") return kb * 1024;
        f.ignore(256, '\n');
    }
    return 0;
}

// NUMA-affine page-locked arena: anonymous mmap, transparent huge pages, bound to the
// GPU's NUMA node when the platform reports one, then registered (portable + mapped so the
// zero-copy kernel can read it through UVA).
PinnedBuf pin_alloc(uint64_t bytes, int numa_node) {
    PinnedBuf b;
    b.bytes = bytes;
    b.map_bytes = (std::max<uint64_t>(bytes, 1) + (2ull << 20) - 1) / (2ull << 20) * (2ull << 20);
    void* p = mmap(nullptr, b.map_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) throw Error(MPSW_ENOMEM, "mmap of pinned arena failed");
    madvise(p, b.map_bytes, MADV_HUGEPAGE);
    if (numa_node >= 0 && numa_node < 64) {
        unsigned long mask = 1ul << numa_node;
        if (syscall(SYS_mbind, p, b.map_bytes, 2 /*MPOL_BIND*/, &mask, 64, 0) == 0) b.numa = numa_node;
    }
    cudaError_t e = cudaHostRegister(p, b.map_bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e != cudaSuccess) {
        cudaGetLastError();
        munmap(p, b.map_bytes);
        throw Error(MPSW_ENOMEM, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
    }
    b.p = (uint8_t*)p;
    if (b.numa >= 0) {
        // registration faulted every page in under the binding policy: check where 16 sampled
        // pages live (move_pages with no target nodes only reports)
        void* pages[16];
        int status[16];
        const uint64_t step = std::max<uint64_t>(4096, b.map_bytes / 16 / 4096 * 4096);
        int n = 0;
        for (uint64_t off = 0; off < b.map_bytes && n < 16; off += step) pages[n++] = (uint8_t*)p + off;
        b.numa_ok = syscall(SYS_move_pages, 0, n, pages, nullptr, status, 0) == 0 &&
                    std::all_of(status, status + n, [&](int s) { return s == b.numa; });
    }
    return b;
}

void pin_free(PinnedBuf& b) {
    if (!b.p) return;
    cudaHostUnregister(b.p);
    munmap(b.p, b.map_bytes);
    b.p = nullptr;
}

// Write a freshly filled arena back from the CPU caches to DRAM (clflushopt per 64-B line, in
// parallel). Measured on the B200 box: a copy-engine read of host memory that is still dirty in
// the CPU's L3 runs at 1/3 – 1/5 of the link rate (a 4 MiB swap-in: 0.38 ms instead of 0.082 ms,
// profiles/r02_ce_dirty_cache.ndjson), so every arena the library writes (synthetic fill,
// caller shards copied in) is flushed once; a DMA read of clean lines runs at full speed.
// MPSW_NO_FLUSH=1 skips it (A/B measurement).
static bool has_clflushopt() {
    unsigned a, b, c, d;
    __asm__ __volatile__("cpuid" : "=a"(a), "=b"(b), "=c"(c), "=d"(d) : "a"(7), "c"(0));
    return (b >> 23) & 1u;          // CPUID.(EAX=7,ECX=0):EBX[23] = CLFLUSHOPT
}

void flush_to_memory(uint8_t* p, uint64_t n) {
    static const bool off = getenv("MPSW_NO_FLUSH") != nullptr;
    static const bool opt = has_clflushopt();
    if (off || !n) return;
    const uint64_t lines = (n + 63) / 64;
    const int T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    auto work = [=](uint64_t l0, uint64_t l1) {
        if (opt)
            for (uint64_t l = l0; l < l1; ++l) asm volatile("clflushopt (%0)" ::"r"(p + l * 64) : "memory");
        else
            for (uint64_t l = l0; l < l1; ++l) asm volatile("clflush (%0)" ::"r"(p + l * 64) : "memory");
        asm volatile("sfence" ::: "memory");
    };
    if (n < (16ull << 20)) {
        work(0, lines);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(work, lines * t / T, lines * (t + 1) / T);
    for (auto& x : th) x.join();
}

void parallel_memcpy(uint8_t* dst, const uint8_t* src, uint64_t n) {
    const int T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (n < (64ull << 20)) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([=] {
            const uint64_t b = n * t / T, e = n * (t + 1) / T;
            std::memcpy(dst + b, src + b, e - b);
        });
    for (auto& x : th) x.join();
}

void* shm_map(const std::string& name, size_t bytes, bool create) {
    int fd = create ? shm_open(name.c_str(), O_CREAT | O_RDWR | O_TRUNC, 0600) : shm_open(name.c_str(), O_RDWR, 0600);
    if (fd < 0) return nullptr;
    if (create && ftruncate(fd, (off_t)bytes) != 0) {
        close(fd);
        throw Error(MPSW_ENOMEM, "ftruncate of shm segment failed");
    }
    if (!create) {
        struct stat st;
        if (fstat(fd, &st) != 0 || (size_t)st.st_size < bytes) {
            close(fd);
            return nullptr;
        }
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(MPSW_ENOMEM, "mmap of shm segment failed");
    return p;
}

}  // namespace mpsw
