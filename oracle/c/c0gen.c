/* oracle/c/c0gen.c — TEST INFRASTRUCTURE (oracle side), not product code.
 *
 * Plain C, OpenMP-parallel transcription of the C0 synthetic-weight spec (DESIGN.md §3,
 * SURVEY §8(c) C0), used only so the oracle can generate full-size (OPT-13B/30B) weights in
 * seconds instead of minutes:
 *     x = splitmix64(seed ^ (tensor_id << 40) ^ flat_index);  u = x >> 40;
 *     w = (u - 2^23) * 2^-28;  value = (gamma ? 1 + w : w) rounded RNE to fp32,
 *     optionally then RNE to bf16 (returned widened to fp32).
 * Pinned against the numpy oracle (oracle/weights.py) element for element in
 * tests/test_oracle_cgen.py. Shares no code with the CUDA path.
 */
#include <stdint.h>
#include <string.h>

static uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static float round_bf16(float f) {
    uint32_t b;
    memcpy(&b, &f, 4);
    b = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
    memcpy(&f, &b, 4);
    return f;
}

/* values of flat indices [start, start + count) of one tensor, written to out[0..count) */
void c0_values(uint64_t seed, uint64_t tensor_id, uint64_t start, uint64_t count, int gamma, int bf16,
               float* out) {
    const uint64_t key = seed ^ (tensor_id << 40);
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)count; ++i) {
        const uint64_t x = splitmix64(key ^ (start + (uint64_t)i));
        const double w = (double)((int64_t)(x >> 40) - (1 << 23)) * (1.0 / 268435456.0);
        float v = (float)(gamma ? 1.0 + w : w);
        if (bf16) v = round_bf16(v);
        out[i] = v;
    }
}
