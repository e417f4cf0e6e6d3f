// records.cuh -- key-value records merged by their key: the reference's own
// key-value call shape, a struct plus a key-only less (tagged<K> /
// tagged_key_less, /root/reference/proj/include/comerge/oracle.hpp:22-37;
// merge_parallel<T> with `less`, parallel.hpp:304-317).
//
// A record is S bytes: the key (int32 / uint32 / uint64) at offset 0 and
// S - sizeof(key) bytes of payload that travel with it untouched (padding
// included, so a record is copied byte for byte).  S = 8 ({32-bit key,
// uint32 val}), 12 ({32-bit key, 8 bytes}: the reference's tagged<int32_t>)
// or 16 ({uint64 key, uint32 val, 4 bytes padding}: the reference's struct
// layout, and its tagged<uint64_t>).  A is the alignment every record position has in
// global and shared memory for a launch (the arrays' common alignment), used
// for vector shared-memory accesses: the pipeline keeps windows at their
// address offset modulo 16, so a record's shared position has the alignment of
// its global one.
#pragma once

#include <cstdint>
#include <type_traits>

namespace comerge_b200 {

template <typename KT, int S, int A>
struct rec {
    static_assert(S % 4 == 0 && S > int(sizeof(KT)) && (A == 4 || A == 8 || A == 16), "record");
    KT key;
    uint32_t rest[(S - sizeof(KT)) / 4];
    __host__ __device__ __forceinline__ bool operator<(const rec& o) const { return key < o.key; }
};

template <typename T>
struct is_rec : std::false_type {};
template <typename KT, int S, int A>
struct is_rec<rec<KT, S, A>> : std::true_type {};

// Shared-memory element access at a shared-window address (u32).
template <typename K>
struct smem_io;

template <>
struct smem_io<int32_t> {
    static __device__ __forceinline__ int32_t ld(uint32_t addr) {
        int32_t v;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
        return v;
    }
    static __device__ __forceinline__ void st(uint32_t addr, int32_t v) {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
    }
};
template <>
struct smem_io<uint32_t> {
    static __device__ __forceinline__ uint32_t ld(uint32_t addr) {
        uint32_t v;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
        return v;
    }
    static __device__ __forceinline__ void st(uint32_t addr, uint32_t v) {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
    }
};
template <>
struct smem_io<uint64_t> {
    static __device__ __forceinline__ uint64_t ld(uint32_t addr) {
        unsigned long long v;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
        return uint64_t(v);
    }
    static __device__ __forceinline__ void st(uint32_t addr, uint64_t v) {
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"((unsigned long long)v) : "memory");
    }
};

// 8-byte records {32-bit key, uint32}: one 64-bit access (A = 8) or two 32-bit
template <typename KT, int A>
struct smem_io<rec<KT, 8, A>> {
    using R = rec<KT, 8, A>;
    static __device__ __forceinline__ R ld(uint32_t addr) {
        uint32_t k, v;
        if constexpr (A >= 8) {
            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(k), "=r"(v) : "r"(addr));
        } else {
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(k) : "r"(addr));
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr + 4));
        }
        R r;
        r.key = static_cast<KT>(k);
        r.rest[0] = v;
        return r;
    }
    static __device__ __forceinline__ void st(uint32_t addr, const R& r) {
        const uint32_t k = static_cast<uint32_t>(r.key);
        if constexpr (A >= 8) {
            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(k), "r"(r.rest[0])
                         : "memory");
        } else {
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(k) : "memory");
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr + 4), "r"(r.rest[0]) : "memory");
        }
    }
};

// 16-byte records {uint64 key, uint32, uint32 pad}: one 128-bit access (A =
// 16) or two 64-bit
template <int A>
struct smem_io<rec<uint64_t, 16, A>> {
    using R = rec<uint64_t, 16, A>;
    static __device__ __forceinline__ R ld(uint32_t addr) {
        unsigned long long k, v;
        if constexpr (A >= 16) {
            asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(k), "=l"(v) : "r"(addr));
        } else {
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(k) : "r"(addr));
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr + 8));
        }
        R r;
        r.key = uint64_t(k);
        r.rest[0] = uint32_t(v);
        r.rest[1] = uint32_t(v >> 32);
        return r;
    }
    static __device__ __forceinline__ void st(uint32_t addr, const R& r) {
        const unsigned long long v = (unsigned long long)r.rest[0] |
                                     ((unsigned long long)r.rest[1] << 32);
        if constexpr (A >= 16) {
            asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(addr),
                         "l"((unsigned long long)r.key), "l"(v)
                         : "memory");
        } else {
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"((unsigned long long)r.key)
                         : "memory");
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr + 8), "l"(v) : "memory");
        }
    }
};

// 12-byte records {32-bit key, 8 payload bytes} -- the reference's own
// tagged<int32_t> / tagged<uint32_t> (key, origin byte + 3 padding bytes,
// uint32 index; oracle.hpp:22-27): three 32-bit accesses (a 12-byte record
// position is 4-byte aligned in general)
template <typename KT, int A>
struct smem_io<rec<KT, 12, A>> {
    using R = rec<KT, 12, A>;
    static __device__ __forceinline__ R ld(uint32_t addr) {
        uint32_t k, v0, v1;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(k) : "r"(addr));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v0) : "r"(addr + 4));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v1) : "r"(addr + 8));
        R r;
        r.key = static_cast<KT>(k);
        r.rest[0] = v0;
        r.rest[1] = v1;
        return r;
    }
    static __device__ __forceinline__ void st(uint32_t addr, const R& r) {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(static_cast<uint32_t>(r.key))
                     : "memory");
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr + 4), "r"(r.rest[0]) : "memory");
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr + 8), "r"(r.rest[1]) : "memory");
    }
};

// The key a co-rank search compares (a record's key; a plain key itself).
template <typename T>
struct key_of {
    using type = T;
};
template <typename KT, int S, int A>
struct key_of<rec<KT, S, A>> {
    using type = KT;
};

}  // namespace comerge_b200
