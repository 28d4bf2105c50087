// philox.cuh -- device Philox4x32-10 with the reference counter layout.
//
// Reference: Philox4x32::block and RandomStream (proj/include/sdd/rng.hpp:12-83).
// Key (k0, k1) = (seed lo, seed hi); counter = {block, walk, point_id lo32,
// (point_id >> 32 & 0xFFFF) | epoch << 16}.  u64 number n of a stream is
// (hi << 32 | lo) with lo, hi = words 2(n&1), 2(n&1)+1 of block n >> 1: the
// reference hands out 4-word blocks two words at a time (rng.hpp:41-55), so a
// u64 never straddles two blocks.  A lane's stream state is therefore just the
// u64 index n plus the upper half of the last block it generated.
#pragma once
#include <cstdint>

namespace sddg {

struct PhiloxWords {
    uint32_t w0, w1, w2, w3;
};

__device__ __forceinline__ PhiloxWords philox4x32_10(uint32_t k0, uint32_t k1, uint32_t c0,
                                                     uint32_t c1, uint32_t c2, uint32_t c3) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return {c0, c1, c2, c3};
}

__device__ __forceinline__ uint64_t join64(uint32_t lo, uint32_t hi) {
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Philox round keys of a seed: k0 + r*W0, k1 + r*W1 for r = 0..9.  Passed
// as a kernel parameter so every LOP3 of the rounds reads its key straight
// from the constant bank (no per-block key schedule in the step loop).
struct RoundKeys {
    uint32_t k[20];
};

__host__ __device__ inline RoundKeys make_round_keys(uint64_t seed) {
    RoundKeys r;
    uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
    for (int i = 0; i < 10; ++i) {
        r.k[2 * i] = k0;
        r.k[2 * i + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return r;
}

__device__ __forceinline__ PhiloxWords philox4x32_10(const RoundKeys& rk, uint32_t c0,
                                                     uint32_t c1, uint32_t c2, uint32_t c3) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
        c0 = hi1 ^ c1 ^ rk.k[2 * r];
        c1 = lo1;
        c2 = hi0 ^ c3 ^ rk.k[2 * r + 1];
        c3 = lo0;
    }
    return {c0, c1, c2, c3};
}

// Per-lane stream (one walk, one epoch); the seed lives in RoundKeys.
//
// Within one stream only the block counter c0 changes, so part of the first
// two rounds is the same for every block and is computed once per walk:
// round 1's product of the third word, M1 * c2, gives the round-1 outputs
// c0' = hi(M1 c2) ^ walk ^ k0 and c1' = lo(M1 c2); round 2's product of that
// c0', M0 * c0', is then fixed as well.  Per block the first two rounds cost
// one 32x32->64 multiply each instead of two (the same words as
// philox4x32_10; tests/test_gpu_walk.py compares every stream with the
// reference's).
struct LaneStream {
    uint32_t c3;         // point id hi16 | epoch << 16 (round-1 input)
    uint32_t r1c1;       // round-1 output word 1: lo(M1 * c2)
    uint32_t r2lo, r2hi; // round 2: lo/hi of M0 * c0'
    uint32_t n;          // u64s consumed this epoch
    uint32_t cw2, cw3;   // words 2,3 of the last generated block

    __device__ __forceinline__ void init(const RoundKeys& rk, uint64_t pid, uint32_t walk, uint32_t epoch) {
        const uint32_t c2 = static_cast<uint32_t>(pid);
        c3 = static_cast<uint32_t>((pid >> 32) & 0xFFFFu) | (epoch << 16);
        r1c1 = 0xCD9E8D57u * c2;
        const uint32_t c0p = __umulhi(0xCD9E8D57u, c2) ^ walk ^ rk.k[0];
        r2lo = 0xD2511F53u * c0p;
        r2hi = __umulhi(0xD2511F53u, c0p);
        n = 0;
        cw2 = cw3 = 0;
    }

    // Philox4x32-10 of block c0 of this stream (philox4x32_10 with rounds 1
    // and 2 partly precomputed)
    __device__ __forceinline__ PhiloxWords block(const RoundKeys& rk, uint32_t c0) const {
        // round 1: (c0, walk, c2, c3) -> (c0', r1c1, hi(M0 c0) ^ c3 ^ k1, lo(M0 c0))
        const uint32_t a2 = __umulhi(0xD2511F53u, c0) ^ c3 ^ rk.k[1];
        const uint32_t a3 = 0xD2511F53u * c0;
        // round 2: M0 * c0' precomputed
        uint32_t x0 = __umulhi(0xCD9E8D57u, a2) ^ r1c1 ^ rk.k[2];
        uint32_t x1 = 0xCD9E8D57u * a2;
        uint32_t x2 = r2hi ^ a3 ^ rk.k[3];
        uint32_t x3 = r2lo;
#pragma unroll
        for (int r = 2; r < 10; ++r) {
            const uint32_t lo0 = 0xD2511F53u * x0;
            const uint32_t hi0 = __umulhi(0xD2511F53u, x0);
            const uint32_t lo1 = 0xCD9E8D57u * x2;
            const uint32_t hi1 = __umulhi(0xCD9E8D57u, x2);
            x0 = hi1 ^ x1 ^ rk.k[2 * r];
            x1 = lo1;
            x2 = hi0 ^ x3 ^ rk.k[2 * r + 1];
            x3 = lo0;
        }
        return {x0, x1, x2, x3};
    }

    // Two consecutive u64s (n, n+1): exactly one new block, index (n+1)>>1,
    // for either parity of n -- the per-step Philox call is warp-uniform.
    __device__ __forceinline__ void next_pair(const RoundKeys& rk, uint64_t& a, uint64_t& b) {
        const PhiloxWords w = block(rk, (n + 1) >> 1);
        const bool odd = n & 1u;
        a = odd ? join64(cw2, cw3) : join64(w.w0, w.w1);
        b = odd ? join64(w.w0, w.w1) : join64(w.w2, w.w3);
        cw2 = w.w2;
        cw3 = w.w3;
        n += 2;
    }

    // One u64 (bridge / exponential draws): a new block only when n is even.
    __device__ __forceinline__ uint64_t next_one(const RoundKeys& rk) {
        uint64_t v;
        if (n & 1u) {
            v = join64(cw2, cw3);
        } else {
            const PhiloxWords w = block(rk, n >> 1);
            v = join64(w.w0, w.w1);
            cw2 = w.w2;
            cw3 = w.w3;
        }
        n += 1;
        return v;
    }
};

// rng.hpp:58 u01 = (u >> 11) 2^-53 in [0,1); rng.hpp:61-63 u01_open.
__device__ __forceinline__ double u01_d(uint64_t u) {
    return __dmul_rn(static_cast<double>(u >> 11), 0x1.0p-53);
}
__device__ __forceinline__ double u01_open_d(uint64_t u) {
    return __dmul_rn(__dadd_rn(static_cast<double>(u >> 12), 0.5), 0x1.0p-52);
}
// fp32 views of the same draws: the top 24 bits.
__device__ __forceinline__ float u01_f(uint64_t u) {
    return static_cast<float>(static_cast<uint32_t>(u >> 40)) * 0x1.0p-24f;
}
__device__ __forceinline__ float u01_open_f(uint64_t u) {
    return __fmaf_rn(static_cast<float>(static_cast<uint32_t>(u >> 40)), 0x1.0p-24f, 0x1.0p-25f);
}

}  // namespace sddg
